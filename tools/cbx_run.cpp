// cbx_run -- C++ host driver over the drop-in API (include/cbinfer_b200.hpp),
// the B200 counterpart of the reference CLI's `cbench run`
// (/root/reference/proj/tools/cbench.cpp:95-173): runs a frame sequence
// through one Network and prints one CSV row per frame.
//
//   cbx_run --net spec.json --weights DIR [--seq DIR | --synth C,H,W,N,SIZE,VEL,SEED]
//           [--engine cbinfer|baseline] [--precision tf32|exact] [--thresholds a,b,c]
//           [--mode run|analyze-prop|sweep|calibrate] [--factors f1,f2,...] [--budget PCT] [--grid N]
//
// --mode analyze-prop is the counterpart of `cbench analyze-prop`
// (cbench.cpp:242-302): per steady frame and CBCONV layer k >= 2, the actual
// updated count next to the worst case propagated from layer k-1.
// --mode sweep / calibrate are `cbench sweep` / `cbench calibrate`
// (cbench.cpp:174-240) over cbinfer_b200_calibration.hpp.
//
// --seq reads frame_%04d.f32le + manifest.json (synth.cpp:130-186 layout).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "cbinfer_b200.hpp"
#include "cbinfer_b200_calibration.hpp"

namespace cb = cbinfer_b200;

static std::vector<float> parse_floats(const std::string& s) {
    std::vector<float> v;
    std::stringstream ss(s);
    std::string tok;
    while (std::getline(ss, tok, ',')) v.push_back(std::stof(tok));
    return v;
}

int main(int argc, char** argv) {
    std::string net_path, wdir, seq, synth, engine = "cbinfer", precision = "tf32", taus, mode = "run";
    std::string factors = "0,0.25,0.5,0.75,1,1.25,1.5,1.75,2";
    double budget = 1.0;
    int gridSize = 16;
    for (int i = 1; i + 1 < argc; i += 2) {
        const std::string k = argv[i], v = argv[i + 1];
        if (k == "--net") net_path = v;
        else if (k == "--weights") wdir = v;
        else if (k == "--seq") seq = v;
        else if (k == "--synth") synth = v;
        else if (k == "--engine") engine = v;
        else if (k == "--precision") precision = v;
        else if (k == "--thresholds") taus = v;
        else if (k == "--mode") mode = v;
        else if (k == "--factors") factors = v;
        else if (k == "--budget") budget = std::stod(v);
        else if (k == "--grid") gridSize = std::stoi(v);
        else {
            std::cerr << "unknown option " << k << "\n";
            return 1;
        }
    }
    if (net_path.empty() || wdir.empty() || (seq.empty() && synth.empty())) {
        std::cerr << "usage: cbx_run --net spec.json --weights DIR (--seq DIR | --synth C,H,W,N,SIZE,VEL,SEED)\n";
        return 1;
    }
    try {
        cb::NetworkSpec spec = cb::load_network_spec(net_path);
        cb::Network net(spec, wdir, 0, precision == "exact" ? cb::Precision::Exact : cb::Precision::TF32);
        if (!taus.empty()) net.set_thresholds(parse_floats(taus));
        const cb::Engine eng = engine == "baseline" ? cb::Engine::Baseline : cb::Engine::CBInfer;
        std::vector<cb::FrameTensor> frames;
        if (!seq.empty()) {
            auto man = nlohmann::json::parse(std::ifstream(seq + "/manifest.json"));
            const int C = man.at("channels"), H = man.at("height"), W = man.at("width"), N = man.at("frames");
            for (int f = 0; f < N; ++f) {
                char name[64];
                std::snprintf(name, sizeof(name), "/frame_%04d.f32le", f);
                cb::FrameTensor t(C, H, W);
                std::ifstream in(seq + name, std::ios::binary);
                if (!in) throw cb::io_error(std::string("missing frame ") + seq + name);
                in.read(reinterpret_cast<char*>(t.data.data()), std::streamsize(t.data.size() * 4));
                frames.push_back(std::move(t));
            }
        } else {
            const auto v = parse_floats(synth);
            if (v.size() != 7) throw cb::spec_error("--synth needs C,H,W,N,SIZE,VEL,SEED");
            cbx_sprite sp{int(v[4]), int(v[5]), 0.9f};
            cbx_synth_cfg cfg{int(v[0]), int(v[1]), int(v[2]), int(v[3]), 1, &sp, 0.0f, uint32_t(v[6])};
            for (int f = 0; f < cfg.frames; ++f) {
                cb::FrameTensor t(cfg.channels, cfg.height, cfg.width);
                cb::check(cbx_synth_frame(&cfg, f, t.data.data()));
                frames.push_back(std::move(t));
            }
        }
        if (mode == "analyze-prop") {
            std::vector<size_t> cbl;
            for (size_t k = 0; k < spec.layers.size(); ++k)
                if (spec.layers[k].kind == cb::LayerKind::CBCONV) cbl.push_back(k);
            if (cbl.size() < 2) throw cb::spec_error("analyze-prop needs at least two CBCONV layers");
            const auto dims = cb::chain_dims(spec);
            std::cout << "frameIndex,layer,detectedCount,worstCaseCount,detectedFraction,worstCaseFraction\n";
            for (size_t f = 0; f < frames.size(); ++f) {
                cb::ForwardResult r = cb::forward_frame(net, frames[f], cb::Engine::CBInfer);
                if (f == 0) continue;  // full evaluation, no propagation to compare
                const auto worst = net.worst_case_counts();
                for (size_t k = 1; k < cbl.size(); ++k) {
                    const double grid = double(dims[cbl[k]].out.height) * dims[cbl[k]].out.width;
                    const long long det = (long long)r.stats[cbl[k]].changedOutputPixels;
                    char buf[160];
                    std::snprintf(buf, sizeof(buf), "%d,%zu,%lld,%lld,%.9g,%.9g", int(f), k + 1, det,
                                  (long long)worst[k - 1], 100.0 * det / grid, 100.0 * double(worst[k - 1]) / grid);
                    std::cout << buf << "\n";
                }
            }
            return 0;
        }
        if (mode == "sweep" || mode == "calibrate") {
            std::vector<cb::Sequence> seqs(1);
            seqs[0].name = seq.empty() ? std::string("synth") : seq;
            seqs[0].frames = std::move(frames);
            char buf[192];
            if (mode == "sweep") {
                std::vector<double> fs;
                for (float f : parse_floats(factors)) fs.push_back(f);
                const auto pts = cb::sweep_threshold_factor(net, seqs, net.thresholds(), fs);
                std::cout << "sequence,factor,errorIncrease,numChangeTotal,throughput,macsTotal\n";
                for (const auto& p : pts) {
                    std::snprintf(buf, sizeof(buf), "%s,%.9g,%.9g,%lld,%.9g,%llu", seqs[0].name.c_str(),
                                  p.thresholdFactor, p.errorIncrease, (long long)p.changedPixelsTotal,
                                  p.framesPerSecond, (unsigned long long)p.macsTotal);
                    std::cout << buf << "\n";
                }
            } else {
                const auto grids = cb::default_threshold_grids(net, seqs, gridSize);
                const auto res = cb::calibrate_thresholds(net, seqs, grids, budget);
                std::cout << "layer,threshold,errorIncrease\n";
                for (const auto& p : res.sweep) {
                    std::snprintf(buf, sizeof(buf), "%d,%.9g,%.9g", p.layer, double(p.threshold), p.errorIncrease);
                    std::cout << buf << "\n";
                }
                std::string line;
                for (size_t k = 0; k < res.thresholds.size(); ++k) {
                    std::snprintf(buf, sizeof(buf), "%.9g", double(res.thresholds[k]));
                    line += (k ? "," : "") + std::string(buf);
                }
                std::cout << "thresholds: " << line << "\n";
            }
            return 0;
        }
        if (mode != "run") throw cb::spec_error("unknown --mode " + mode);
        std::cout << "frame,wallNanos,macsTotal";
        for (size_t k = 0; k < spec.layers.size(); ++k)
            if (spec.layers[k].kind == cb::LayerKind::CBCONV) std::cout << ",changedIn" << k + 1 << ",changedOut" << k + 1;
        std::cout << ",labelChecksum\n";
        for (size_t f = 0; f < frames.size(); ++f) {
            const auto t0 = std::chrono::steady_clock::now();
            cb::ForwardResult r = cb::forward_frame(net, frames[f], eng);
            const auto t1 = std::chrono::steady_clock::now();
            uint64_t sum = 0;
            for (size_t i = 0; i < r.labels.labels.size(); ++i) sum += uint64_t(r.labels.labels[i]) * (i % 9973 + 1);
            std::cout << f << "," << std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count() << ","
                      << r.macsTotal;
            for (size_t k = 0; k < spec.layers.size(); ++k)
                if (spec.layers[k].kind == cb::LayerKind::CBCONV)
                    std::cout << "," << r.stats[k].changedInputPixels << "," << r.stats[k].changedOutputPixels;
            std::cout << "," << sum << "\n";
        }
        return 0;
    } catch (const cb::error& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    }
}
