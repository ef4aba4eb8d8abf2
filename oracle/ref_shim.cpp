// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the UNMODIFIED reference library
// (/root/reference/proj/core, compiled from its own sources by
// oracle/Makefile into oracle/_ref/libcbinfer_ref.so). Used to pin the C
// restatement (cbinfer_oracle.c) and to time the reference CPU path in
// bench.py --impl reference. Nothing in the product links this.
#include <cstdint>
#include <cstring>
#include <exception>
#include <filesystem>
#include <string>
#include <thread>
#include <vector>

#include "cbinfer/baseline.hpp"
#include "cbinfer/cbconv.hpp"
#include "cbinfer/error.hpp"
#include "cbinfer/calibration.hpp"
#include "cbinfer/network.hpp"
#include "cbinfer/synth.hpp"

using namespace cbinfer;

namespace {

thread_local std::string g_err;

int code_of(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const shape_error*>(&e)) return -1;
    if (dynamic_cast<const geometry_error*>(&e)) return -2;
    if (dynamic_cast<const bounds_error*>(&e)) return -3;
    if (dynamic_cast<const io_error*>(&e)) return -4;
    if (dynamic_cast<const spec_error*>(&e)) return -5;
    return -9;
}

FrameTensor to_tensor(const float* d, int c, int h, int w) {
    FrameTensor t(c, h, w);
    std::memcpy(t.data.data(), d, t.data.size() * sizeof(float));
    return t;
}

ConvGeometry geom_of(const int* g) {
    ConvGeometry x;
    x.kernelH = g[0];
    x.kernelW = g[1];
    x.strideH = g[2];
    x.strideW = g[3];
    x.padH = g[4];
    x.padW = g[5];
    x.inChannels = g[6];
    x.outChannels = g[7];
    return x;
}

struct RefNet {
    Network net;
    ForwardTrace trace;
};

}  // namespace

#define GUARD(...)                           \
    try {                                    \
        __VA_ARGS__                          \
    } catch (const std::exception& e) {      \
        return code_of(e);                   \
    }

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int64_t ref_detect_changes(const float* cur, const float* prev, int C, int H, int W, float tau,
                           uint8_t* m) {
    GUARD({
        ChangeMap cm = detect_changes(to_tensor(cur, C, H, W), to_tensor(prev, C, H, W), tau);
        std::memcpy(m, cm.bits.data(), cm.bits.size());
        return cm.count();
    })
}

int ref_dilate_changes(const uint8_t* m, int H, int W, const int* g, uint8_t* out) {
    GUARD({
        ChangeMap cm(H, W);
        std::memcpy(cm.bits.data(), m, cm.bits.size());
        ChangeMap d = dilate_changes(cm, geom_of(g));
        std::memcpy(out, d.bits.data(), d.bits.size());
        return 0;
    })
}

int64_t ref_extract_indexes(const uint8_t* m, int H, int W, int32_t* idx) {
    GUARD({
        ChangeMap cm(H, W);
        std::memcpy(cm.bits.data(), m, cm.bits.size());
        ChangeIndexList l = extract_indexes(cm);
        std::memcpy(idx, l.indices.data(), l.indices.size() * sizeof(int32_t));
        return l.count();
    })
}

int ref_conv_full(const float* in, int C, int H, int W, const float* K, const float* bias,
                  const int* g, float* out) {
    GUARD({
        ConvGeometry geom = geom_of(g);
        FilterMatrix f(geom.outChannels, geom.inChannels * geom.kernelH * geom.kernelW);
        std::memcpy(f.data.data(), K, f.data.size() * sizeof(float));
        std::memcpy(f.bias.data(), bias, f.bias.size() * sizeof(float));
        FrameTensor o = conv_full(to_tensor(in, C, H, W), f, geom);
        std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
        return 0;
    })
}

int ref_maxpool(const float* in, int C, int H, int W, int window, int stride, float* out) {
    GUARD({
        FrameTensor o = maxpool(to_tensor(in, C, H, W), window, stride);
        std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
        return 0;
    })
}

int ref_synth_frame(int C, int H, int W, int nSprites, const int* sizes, const int* vels,
                    const float* intens, float noise, uint32_t seed, int f, float* out) {
    GUARD({
        SynthConfig cfg;
        cfg.channels = C;
        cfg.height = H;
        cfg.width = W;
        cfg.frames = f + 1;
        for (int s = 0; s < nSprites; ++s) cfg.sprites.push_back({sizes[s], vels[s], intens[s]});
        cfg.noiseAmplitude = noise;
        cfg.seed = seed;
        FrameTensor t = synth_frame(cfg, f);
        std::memcpy(out, t.data.data(), t.data.size() * sizeof(float));
        return 0;
    })
}

int ref_random_filters(const int* g, uint32_t seed, float* K, float* bias) {
    GUARD({
        FilterMatrix f = random_filters(geom_of(g), seed);
        std::memcpy(K, f.data.data(), f.data.size() * sizeof(float));
        std::memcpy(bias, f.bias.data(), f.bias.size() * sizeof(float));
        return 0;
    })
}

// Network level: the reference's own JSON parsing, weight loading and
// forward_frame. weightsDir must hold files written by ref_generate_weights
// (or any reference-format weights).
int ref_generate_weights(const char* specJson, const char* dir, uint32_t seed) {
    GUARD({
        generate_weights(network_spec_from_json(specJson), dir, seed);
        return 0;
    })
}

int ref_net_load(const char* specJson, const char* dir, void** out) {
    GUARD({
        auto* r = new RefNet;
        r->net = load_network(network_spec_from_json(specJson), dir);
        *out = r;
        return 0;
    })
}

void ref_net_free(void* h) { delete static_cast<RefNet*>(h); }

int ref_net_reset(void* h) {
    reset_state(static_cast<RefNet*>(h)->net);
    return 0;
}

int ref_net_set_thresholds(void* h, const float* taus, int n) {
    GUARD({
        static_cast<RefNet*>(h)->net.set_thresholds(std::vector<float>(taus, taus + n));
        return 0;
    })
}

// stats: per layer {changedIn, changedOut, macs} as int64 triples.
int ref_forward_frame(void* h, const float* frame, int engine, uint16_t* labels, int64_t* stats,
                      uint64_t* macsTotal, int keepTrace) {
    GUARD({
        auto* r = static_cast<RefNet*>(h);
        const auto& s = r->net.spec;
        FrameTensor f = to_tensor(frame, s.inputChannels, s.inputHeight, s.inputWidth);
        ForwardResult res = forward_frame(r->net, f, engine ? Engine::CBInfer : Engine::Baseline,
                                          keepTrace ? &r->trace : nullptr);
        if (labels)
            std::memcpy(labels, res.labels.labels.data(), res.labels.labels.size() * 2);
        if (stats)
            for (std::size_t k = 0; k < res.stats.size(); ++k) {
                stats[3 * k + 0] = res.stats[k].changedInputPixels;
                stats[3 * k + 1] = res.stats[k].changedOutputPixels;
                stats[3 * k + 2] = static_cast<int64_t>(res.stats[k].gemmMacs);
            }
        if (macsTotal) *macsTotal = res.macsTotal;
        return 0;
    })
}

// Warm-up for timing runs: leaves the network in exactly the state one
// forward_frame(frame) would (every CBCONV evaluated in full, prevInput /
// prevOutput stored), but computes each full-frame convolution with the
// reference's own gen_x_reduced + gemm over disjoint output-pixel chunks on
// `nthreads` threads. Each output column is an independent gemm column, so
// the result is bitwise identical to the serial first frame
// (cbconv.cpp:170-192, 225-226).
int ref_net_warm(void* h, const float* frame, int nthreads) {
    GUARD({
        auto* r = static_cast<RefNet*>(h);
        Network& net = r->net;
        const auto& s = net.spec;
        FrameTensor cur = to_tensor(frame, s.inputChannels, s.inputHeight, s.inputWidth);
        if (nthreads < 1) nthreads = 1;
        for (Layer& layer : net.layers) {
            const LayerKind kind = layer.spec.kind;
            if (kind == LayerKind::CBCONV || kind == LayerKind::CONV) {
                const ConvGeometry& g = layer.state.geom;
                const int O = layer.outDims.channels, oh = layer.outDims.height, ow = layer.outDims.width;
                const bool fuse = kind == LayerKind::CBCONV && layer.spec.fuseRelu;
                FrameTensor out(O, oh, ow);
                const int pixels = oh * ow;
                const int chunk = (pixels + nthreads - 1) / nthreads;
                std::vector<std::thread> pool;
                for (int t = 0; t < nthreads; ++t) {
                    const int a = t * chunk, b = std::min(pixels, a + chunk);
                    if (a >= b) break;
                    pool.emplace_back([&, a, b] {
                        ChangeIndexList idx;
                        idx.indices.resize(b - a);
                        for (int p = a; p < b; ++p) idx.indices[p - a] = p;
                        PatchMatrix X = gen_x_reduced(cur, idx, g);
                        ResultMatrix Y = gemm(layer.state.filters, X);
                        for (int o = 0; o < O; ++o)
                            for (int n = 0; n < b - a; ++n) {
                                const float v = Y.data[static_cast<std::size_t>(o) * Y.cols + n];
                                out.plane(o)[a + n] = fuse ? std::max(0.0f, v) : v;
                            }
                    });
                }
                for (auto& th : pool) th.join();
                if (kind == LayerKind::CBCONV) {
                    layer.state.prevInput = cur;
                    layer.state.prevOutput = out;
                }
                cur = std::move(out);
            } else if (kind == LayerKind::RELU) {
                cur = relu(cur);
            } else if (kind == LayerKind::MAXPOOL) {
                cur = maxpool(cur, layer.spec.window, layer.spec.stride);
            }
        }
        return 0;
    })
}

// Copies the whole Network (spec, filters, change-based state) of src into dst.
int ref_net_copy_state(void* dst, const void* src) {
    GUARD({
        static_cast<RefNet*>(dst)->net = static_cast<const RefNet*>(src)->net;
        return 0;
    })
}

int ref_net_final_activation(void* h, const float** data, int* dims) {
    auto* r = static_cast<RefNet*>(h);
    const FrameTensor& t = r->trace.finalActivation;
    *data = t.data.data();
    dims[0] = t.channels;
    dims[1] = t.height;
    dims[2] = t.width;
    return 0;
}

int ref_net_trace(void* h, int cb, const uint8_t** detected, int* dims, const int32_t** updated,
                  int64_t* n) {
    auto* r = static_cast<RefNet*>(h);
    if (cb < 0 || cb >= static_cast<int>(r->trace.cb.size())) return -5;
    const CBConvTrace& t = r->trace.cb[cb];
    *detected = t.detected.bits.empty() ? nullptr : t.detected.bits.data();
    dims[0] = t.detected.height;
    dims[1] = t.detected.width;
    *updated = t.updated.indices.data();
    *n = t.updated.count();
    return 0;
}

// calibration.cpp over one sequence of nframes frames (no ground truth):
// default_threshold_grids(gridSize) + calibrate_thresholds(budget).
// thresholds[ncb]; sweep arrays of ncb*gridSize entries (layer, tau, err).
int ref_calibrate(void* h, const float* frames, int nframes, int gridSize, double budget, float* thresholds,
                  int* sweepLayer, float* sweepTau, double* sweepErr) {
    GUARD({
        auto* r = static_cast<RefNet*>(h);
        const auto& s = r->net.spec;
        std::vector<Sequence> seqs(1);
        seqs[0].name = "seq";
        const size_t per = (size_t)s.inputChannels * s.inputHeight * s.inputWidth;
        for (int f = 0; f < nframes; ++f)
            seqs[0].frames.push_back(to_tensor(frames + per * f, s.inputChannels, s.inputHeight, s.inputWidth));
        const auto grids = default_threshold_grids(r->net, seqs, gridSize);
        const auto res = calibrate_thresholds(r->net, seqs, grids, budget);
        for (size_t k = 0; k < res.thresholds.size(); ++k) thresholds[k] = res.thresholds[k];
        for (size_t i = 0; i < res.sweep.size(); ++i) {
            sweepLayer[i] = res.sweep[i].layer;
            sweepTau[i] = res.sweep[i].threshold;
            sweepErr[i] = res.sweep[i].errorIncrease;
        }
        return 0;
    })
}

// sweep_threshold_factor over one sequence; per factor: errorIncrease,
// changedPixelsTotal, macsTotal (framesPerSecond is wall-clock, not compared).
int ref_sweep(void* h, const float* frames, int nframes, const double* factors, int nf, double* err,
              int64_t* changed, uint64_t* macs) {
    GUARD({
        auto* r = static_cast<RefNet*>(h);
        const auto& s = r->net.spec;
        std::vector<Sequence> seqs(1);
        seqs[0].name = "seq";
        const size_t per = (size_t)s.inputChannels * s.inputHeight * s.inputWidth;
        for (int f = 0; f < nframes; ++f)
            seqs[0].frames.push_back(to_tensor(frames + per * f, s.inputChannels, s.inputHeight, s.inputWidth));
        const auto pts = sweep_threshold_factor(r->net, seqs, r->net.thresholds(),
                                                std::vector<double>(factors, factors + nf));
        for (int i = 0; i < nf; ++i) {
            err[i] = pts[i].errorIncrease;
            changed[i] = pts[i].changedPixelsTotal;
            macs[i] = pts[i].macsTotal;
        }
        return 0;
    })
}

}  // extern "C"
