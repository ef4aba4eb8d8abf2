// cbinfer_b200.hpp -- header-only C++ drop-in for the reference's per-frame
// network API (namespace cbinfer, /root/reference/proj/core/include/cbinfer),
// implemented over the C-ABI in cbx.h (link with -lcbx).
//
// Same names, value types and exception classes as the reference:
//   NetworkSpec / LayerSpec / ConvGeometry      network.hpp:17-35, geometry.hpp:12-49
//   network_spec_from_json / load_network_spec  network.hpp:39-40 (nlohmann/json, like the reference)
//   chain_dims                                  network.hpp:45
//   load_network / forward_frame / reset_state  network.hpp:88-97
//   Network::thresholds / set_thresholds        network.hpp:66-67
//   FrameTensor / LabelMap / LayerStats / ForwardResult / ForwardTrace
//   error, shape_error, geometry_error, bounds_error, io_error, spec_error  error.hpp:9-42
// A Network here lives on a B200: forward_frame uploads the frame, runs the
// change-based pipeline as one CUDA graph and returns labels + stats. There is
// no CPU fallback; a CUDA failure throws cuda_error (derived from error).
#pragma once

#include <cstdint>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "cbx.h"
#include "json.hpp"  // nlohmann/json (the reference's own JSON dependency)

namespace cbinfer_b200 {

class error : public std::runtime_error {
public:
    explicit error(const std::string& m) : std::runtime_error(m) {}
};
class shape_error : public error { public: using error::error; };
class geometry_error : public error { public: using error::error; };
class bounds_error : public error { public: using error::error; };
class io_error : public error { public: using error::error; };
class spec_error : public error { public: using error::error; };
class cuda_error : public error { public: using error::error; };

inline void check(int rc, const cbx_ctx* ctx = nullptr) {
    if (rc == CBX_OK) return;
    const std::string m = cbx_last_error(ctx);
    switch (rc) {
        case CBX_E_SHAPE: throw shape_error(m);
        case CBX_E_GEOMETRY: throw geometry_error(m);
        case CBX_E_BOUNDS: throw bounds_error(m);
        case CBX_E_IO: throw io_error(m);
        case CBX_E_SPEC: throw spec_error(m);
        case CBX_E_CUDA: throw cuda_error(m);
        default: throw error(m);
    }
}

struct ConvGeometry {
    int kernelH = 1, kernelW = 1, strideH = 1, strideW = 1, padH = 0, padW = 0, inChannels = 1, outChannels = 1;
    int outHeight(int h) const { return (h + 2 * padH - kernelH) / strideH + 1; }
    int outWidth(int w) const { return (w + 2 * padW - kernelW) / strideW + 1; }
};

enum class LayerKind { CBCONV = CBX_CBCONV, CONV = CBX_CONV, RELU = CBX_RELU, MAXPOOL = CBX_MAXPOOL, CLASSIFY = CBX_CLASSIFY };
enum class Engine { Baseline = CBX_ENGINE_BASELINE, CBInfer = CBX_ENGINE_CBINFER };
enum class Precision { Exact = CBX_PREC_EXACT, TF32 = CBX_PREC_TF32, F16 = CBX_PREC_F16 };

inline LayerKind layer_kind_from_string(const std::string& s) {
    if (s == "CBCONV") return LayerKind::CBCONV;
    if (s == "CONV") return LayerKind::CONV;
    if (s == "RELU") return LayerKind::RELU;
    if (s == "MAXPOOL") return LayerKind::MAXPOOL;
    if (s == "CLASSIFY") return LayerKind::CLASSIFY;
    throw spec_error("unknown layer kind \"" + s + "\"");
}

struct LayerSpec {
    LayerKind kind = LayerKind::CONV;
    ConvGeometry geom;
    int window = 0, stride = 0;
    float threshold = 0.0f;
    bool fuseRelu = false;
    std::string weightsFile;
    bool is_conv() const { return kind == LayerKind::CBCONV || kind == LayerKind::CONV; }
};

struct NetworkSpec {
    int inputChannels = 0, inputHeight = 0, inputWidth = 0, numClasses = 0;
    std::vector<LayerSpec> layers;
};

// network.cpp:43-85 semantics: same keys, defaults and error classes.
inline NetworkSpec network_spec_from_json(const std::string& text) {
    nlohmann::json doc;
    try {
        doc = nlohmann::json::parse(text);
    } catch (const nlohmann::json::exception& e) {
        throw spec_error(std::string("network spec: invalid JSON: ") + e.what());
    }
    try {
        NetworkSpec spec;
        spec.inputChannels = doc.at("inputChannels").get<int>();
        spec.inputHeight = doc.at("inputHeight").get<int>();
        spec.inputWidth = doc.at("inputWidth").get<int>();
        spec.numClasses = doc.at("numClasses").get<int>();
        for (const auto& jl : doc.at("layers")) {
            LayerSpec l;
            l.kind = layer_kind_from_string(jl.at("kind").get<std::string>());
            if (l.is_conv()) {
                l.geom.kernelH = jl.at("kernelH").get<int>();
                l.geom.kernelW = jl.at("kernelW").get<int>();
                l.geom.strideH = jl.value("strideH", 1);
                l.geom.strideW = jl.value("strideW", 1);
                l.geom.padH = jl.value("padH", 0);
                l.geom.padW = jl.value("padW", 0);
                l.geom.outChannels = jl.at("outChannels").get<int>();
                l.weightsFile = jl.at("weightsFile").get<std::string>();
            }
            if (l.kind == LayerKind::CBCONV) {
                l.threshold = jl.value("threshold", 0.0f);
                l.fuseRelu = jl.value("fuseRelu", false);
                if (l.threshold < 0.0f) throw spec_error("network spec: negative threshold");
            }
            if (l.kind == LayerKind::MAXPOOL) {
                l.window = jl.at("window").get<int>();
                l.stride = jl.at("stride").get<int>();
            }
            spec.layers.push_back(l);
        }
        return spec;
    } catch (const nlohmann::json::exception& e) {
        throw spec_error(std::string("network spec: ") + e.what());
    }
}

inline NetworkSpec load_network_spec(const std::filesystem::path& file) {
    std::ifstream in(file);
    if (!in) throw io_error("cannot open network spec " + file.string());
    std::stringstream ss;
    ss << in.rdbuf();
    return network_spec_from_json(ss.str());
}

struct TensorDims {
    int channels = 0, height = 0, width = 0;
};
struct LayerShape {
    TensorDims in, out;
};

namespace detail {
inline std::vector<cbx_layer_desc> descs(const NetworkSpec& spec) {
    std::vector<cbx_layer_desc> d(spec.layers.size());
    for (size_t k = 0; k < spec.layers.size(); ++k) {
        const auto& l = spec.layers[k];
        d[k].kind = static_cast<int>(l.kind);
        d[k].geom = cbx_geom{l.geom.kernelH, l.geom.kernelW, l.geom.strideH, l.geom.strideW,
                             l.geom.padH, l.geom.padW, l.geom.inChannels, l.geom.outChannels};
        d[k].window = l.window;
        d[k].stride = l.stride;
        d[k].threshold = l.threshold;
        d[k].fuseRelu = l.fuseRelu ? 1 : 0;
    }
    return d;
}
inline cbx_net_desc net(const NetworkSpec& spec, const std::vector<cbx_layer_desc>& d) {
    return cbx_net_desc{spec.inputChannels, spec.inputHeight, spec.inputWidth, spec.numClasses,
                        static_cast<int>(d.size()), d.data()};
}
}  // namespace detail

// network.cpp:128-188: validates the chain, fills inChannels.
inline std::vector<LayerShape> chain_dims(NetworkSpec& spec) {
    auto d = detail::descs(spec);
    auto n = detail::net(spec, d);
    std::vector<cbx_layer_desc> out(d.size() ? d.size() : 1);
    std::vector<int> dims(6 * (d.size() ? d.size() : 1));
    check(cbx_chain_dims(&n, out.data(), dims.data()));
    std::vector<LayerShape> shapes(d.size());
    for (size_t k = 0; k < d.size(); ++k) {
        spec.layers[k].geom.inChannels = out[k].geom.inChannels;
        shapes[k] = {{dims[6 * k], dims[6 * k + 1], dims[6 * k + 2]}, {dims[6 * k + 3], dims[6 * k + 4], dims[6 * k + 5]}};
    }
    return shapes;
}

// Planar CHW fp32 frame / activation (tensor.hpp:28-63).
struct FrameTensor {
    int channels = 0, height = 0, width = 0;
    std::vector<float> data;
    FrameTensor() = default;
    FrameTensor(int c, int h, int w) : channels(c), height(h), width(w), data(size_t(c) * h * w, 0.0f) {}
};

struct LabelMap {
    int height = 0, width = 0;
    std::vector<std::uint16_t> labels;
};

struct LayerStats {
    std::int64_t changedInputPixels = 0, changedOutputPixels = 0;
    std::uint64_t gemmMacs = 0;
};

struct ForwardResult {
    LabelMap labels;
    std::vector<LayerStats> stats;
    std::uint64_t macsTotal = 0;
};

// read_weights_f32le (io.cpp:121-139): exact byte length, finite values.
inline void read_weights_f32le(const std::filesystem::path& file, const ConvGeometry& g, std::vector<float>& K,
                               std::vector<float>& bias) {
    const size_t kv = size_t(g.outChannels) * g.inChannels * g.kernelH * g.kernelW;
    std::ifstream in(file, std::ios::binary | std::ios::ate);
    if (!in) throw io_error("cannot open " + file.string());
    const auto size = static_cast<size_t>(in.tellg());
    if (size != (kv + g.outChannels) * 4)
        throw io_error(file.string() + ": expected " + std::to_string((kv + g.outChannels) * 4) + " bytes, got " +
                       std::to_string(size));
    in.seekg(0);
    K.resize(kv);
    bias.resize(g.outChannels);
    in.read(reinterpret_cast<char*>(K.data()), std::streamsize(kv * 4));
    in.read(reinterpret_cast<char*>(bias.data()), std::streamsize(g.outChannels * 4));
}

// One reference Network (one camera stream) on one B200.
class Network {
public:
    Network(const NetworkSpec& spec, const std::filesystem::path& weightsDir, int device = 0,
            Precision precision = Precision::TF32)
        : spec_(spec) {
        shapes_ = chain_dims(spec_);
        auto d = detail::descs(spec_);
        auto n = detail::net(spec_, d);
        check(cbx_create(&n, device, 1, static_cast<int>(precision), &ctx_));
        for (size_t k = 0; k < spec_.layers.size(); ++k) {
            const auto& l = spec_.layers[k];
            if (!l.is_conv()) continue;
            std::vector<float> K, b;
            try {
                read_weights_f32le(weightsDir / l.weightsFile, l.geom, K, b);
            } catch (const io_error& e) {
                throw io_error("layer " + std::to_string(k + 1) + ": " + e.what());
            }
            check(cbx_load_layer(ctx_, int(k), K.data(), b.data()), ctx_);
        }
        const auto& last = shapes_.back();
        const bool cls = spec_.layers.back().kind == LayerKind::CLASSIFY;
        lh_ = cls ? last.in.height : last.out.height;
        lw_ = cls ? last.in.width : last.out.width;
    }
    Network(const Network&) = delete;
    Network& operator=(const Network&) = delete;
    ~Network() { cbx_destroy(ctx_); }

    std::vector<float> thresholds() const {
        std::vector<float> t;
        for (const auto& l : spec_.layers)
            if (l.kind == LayerKind::CBCONV) t.push_back(0.0f);
        check(cbx_get_thresholds(ctx_, t.data(), int(t.size())), ctx_);
        return t;
    }
    void set_thresholds(const std::vector<float>& taus) {
        check(cbx_set_thresholds(ctx_, taus.data(), int(taus.size())), ctx_);
    }
    ForwardResult forward(const FrameTensor& frame, Engine engine) {
        if (frame.channels != spec_.inputChannels || frame.height != spec_.inputHeight ||
            frame.width != spec_.inputWidth)
            throw shape_error("forward_frame: frame does not match network input dimensions");
        ForwardResult r;
        r.labels.height = lh_;
        r.labels.width = lw_;
        r.labels.labels.resize(size_t(lh_) * lw_);
        std::vector<cbx_layer_stats> st(spec_.layers.size());
        std::uint64_t macs = 0;
        check(cbx_forward(ctx_, static_cast<int>(engine), frame.data.data(), r.labels.labels.data(), st.data(), &macs),
              ctx_);
        r.stats.resize(st.size());
        for (size_t k = 0; k < st.size(); ++k)
            r.stats[k] = {st[k].changedInputPixels, st[k].changedOutputPixels, st[k].gemmMacs};
        r.macsTotal = macs;
        return r;
    }
    // Pipelined serving (cbx_submit / cbx_wait): enqueue the next frame and
    // return at once; the upload of the next submission overlaps this one's
    // kernels. `frame` and `labels` must stay alive until wait(ticket).
    std::int64_t submit(const FrameTensor& frame, LabelMap& labels) {
        if (frame.channels != spec_.inputChannels || frame.height != spec_.inputHeight ||
            frame.width != spec_.inputWidth)
            throw shape_error("forward_frame: frame does not match network input dimensions");
        labels.height = lh_;
        labels.width = lw_;
        labels.labels.resize(size_t(lh_) * lw_);
        std::int64_t t = -1;
        check(cbx_submit(ctx_, static_cast<int>(Engine::CBInfer), frame.data.data(), labels.labels.data(), &t), ctx_);
        return t;
    }
    void wait(std::int64_t ticket, std::vector<LayerStats>* stats = nullptr, std::uint64_t* macsTotal = nullptr) {
        std::vector<cbx_layer_stats> st(spec_.layers.size());
        std::uint64_t macs = 0;
        check(cbx_wait(ctx_, ticket, st.data(), &macs), ctx_);
        if (stats) {
            stats->resize(st.size());
            for (size_t k = 0; k < st.size(); ++k)
                (*stats)[k] = {st[k].changedInputPixels, st[k].changedOutputPixels, st[k].gemmMacs};
        }
        if (macsTotal) *macsTotal = macs;
    }
    // Output activation of `layer` (0-based) after the last change-based frame,
    // planar CHW like the reference's tensors (ForwardTrace, network.hpp:80-83).
    std::vector<float> activation(int layer) {
        const auto& sh = shapes_.at(size_t(layer)).out;
        std::vector<float> out(size_t(sh.channels) * sh.height * sh.width);
        check(cbx_get_activation(ctx_, static_cast<int>(Engine::CBInfer), layer, 0, out.data()), ctx_);
        return out;
    }
    // cbench analyze-prop (cbench.cpp:242-302) for the last change-based frame:
    // worst-case updated count of every CBCONV after the first.
    std::vector<std::int64_t> worst_case_counts() {
        int ncb = 0;
        for (const auto& l : spec_.layers) ncb += l.kind == LayerKind::CBCONV;
        std::vector<std::int64_t> w(ncb > 1 ? ncb - 1 : 0);
        check(cbx_worst_case_counts(ctx_, w.data()), ctx_);
        return w;
    }
    void reset() { check(cbx_reset(ctx_), ctx_); }
    const NetworkSpec& spec() const { return spec_; }
    cbx_ctx* handle() { return ctx_; }

private:
    NetworkSpec spec_;
    std::vector<LayerShape> shapes_;
    cbx_ctx* ctx_ = nullptr;
    int lh_ = 0, lw_ = 0;
};

inline ForwardResult forward_frame(Network& net, const FrameTensor& frame, Engine engine = Engine::CBInfer) {
    return net.forward(frame, engine);
}
inline void reset_state(Network& net) { net.reset(); }

}  // namespace cbinfer_b200
