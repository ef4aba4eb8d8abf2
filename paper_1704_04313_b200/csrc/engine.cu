// engine.cu -- device runtime of one change-based network (see engine.hpp).
//
// Frame recipe (reference: forward_frame network.cpp:252-315, cbconv_forward
// cbconv.cpp:157-228). Tensor t is the input of layer t (t = 0: the camera
// frame, planar, addressed through a per-stream pointer table).
//
//   steady frame, for each layer k
//     CBCONV  : U_k = dilate(chg_k)              (K3)   cbconv.cpp:73-82
//               idx_k = compact(U_k)             (K2)   cbconv.cpp:99-113
//               T_{k+1}[idx_k] = conv(T_k)       (K4)   cbconv.cpp:115-155
//               + chg_{k+1} by compare-before-write when layer k+1 is CBCONV
//     MAXPOOL : recompute windows touched by upd_k, compare-before-write
//     RELU    : recompute pixels in upd_k, compare-before-write
//     CONV    : recompute dilate(upd_k) (== upd_k for 1x1), reusing idx lists
//     CLASSIFY: argmax over upd_k
//   chg_0 = detect(frame_t, frame_{t-1}) (K1) cbconv.cpp:57-71
//
// chg_t ("changed by more than the consumer's tau") equals the reference's
// detect_changes(input, prevInput) because the tensor is updated in place:
// pixels outside the producer's updated set are bitwise unchanged and the
// writer compares the new value with the one it overwrites.
//
// First frame after reset and the Baseline engine run the same kernels in
// "full" mode: no masks, every output pixel evaluated.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>

#include "engine.hpp"
#include "kernels.hpp"
#include "conv_tc.hpp"

namespace cbx {

// Programmatic dependent launch is opt-in (CBX_PDL=1): with two lanes the
// early-launched successors sit on SM slots the other lane's kernels would
// use, and the step measured slower (27.8k vs 30.6k frames/s, 16 x 1080p).
bool pdl_enabled() {
    static const bool on = std::getenv("CBX_PDL") && std::atoi(std::getenv("CBX_PDL")) == 1;
    return on;
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        (void)cudaGetLastError();  // a non-sticky error must not leak into the caller's next CUDA call
        throw Error(CBX_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    }
}

namespace {

int fdiv(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

bool is_conv(int kind) { return kind == CBX_CBCONV || kind == CBX_CONV; }

bool identity_geom(const cbx_geom& g) {
    return g.kernelH == 1 && g.kernelW == 1 && g.strideH == 1 && g.strideW == 1 && g.padH == 0 &&
           g.padW == 0;
}

std::string where(int k, int kind) {
    static const char* names[] = {"CBCONV", "CONV", "RELU", "MAXPOOL", "CLASSIFY"};
    return "layer " + std::to_string(k + 1) + " (" + (kind >= 0 && kind < 5 ? names[kind] : "?") + ")";
}

template <class T>
T* dmalloc(size_t n) {
    void* p = nullptr;
    CBX_CUDA(cudaMalloc(&p, n * sizeof(T) + 16));
    // cudaMemset runs on the legacy default stream, which the engine's
    // non-blocking streams do not order against: wait for it, or a later
    // copy into the buffer (a lazily allocated staging slot) can be zeroed
    CBX_CUDA(cudaMemset(p, 0, n * sizeof(T) + 16));
    CBX_CUDA(cudaStreamSynchronize(nullptr));
    return static_cast<T*>(p);
}

}  // namespace

// chain_dims, network.cpp:128-188
std::vector<int> chain_dims(const cbx_net_desc& net, std::vector<cbx_layer_desc>& L) {
    if (net.numLayers < 1 || !net.layers) throw Error(CBX_E_SPEC, "network spec has no layers");
    if (net.inputChannels < 1 || net.inputHeight < 1 || net.inputWidth < 1)
        throw Error(CBX_E_SPEC, "network spec has invalid input dimensions");
    if (net.numClasses < 1) throw Error(CBX_E_SPEC, "network spec has invalid class count");
    L.assign(net.layers, net.layers + net.numLayers);
    std::vector<int> dims(6 * L.size());
    int c = net.inputChannels, h = net.inputHeight, w = net.inputWidth;
    for (size_t k = 0; k < L.size(); ++k) {
        cbx_layer_desc& l = L[k];
        int oc = c, oh = h, ow = w;
        dims[6 * k + 0] = c;
        dims[6 * k + 1] = h;
        dims[6 * k + 2] = w;
        switch (l.kind) {
            case CBX_CBCONV:
            case CBX_CONV: {
                cbx_geom& g = l.geom;
                g.inChannels = c;
                if (g.kernelH < 1 || g.kernelW < 1 || g.strideH < 1 || g.strideW < 1 || g.padH < 0 || g.padW < 0)
                    throw Error(CBX_E_GEOMETRY, where((int)k, l.kind) + ": invalid convolution geometry");
                if (h + 2 * g.padH < g.kernelH || w + 2 * g.padW < g.kernelW)
                    throw Error(CBX_E_GEOMETRY, where((int)k, l.kind) + ": convolution output would be empty");
                if (g.outChannels < 1) throw Error(CBX_E_SPEC, where((int)k, l.kind) + ": invalid outChannels");
                if (l.kind == CBX_CBCONV && l.threshold < 0.0f)
                    throw Error(CBX_E_SPEC, "network spec: negative threshold");
                oc = g.outChannels;
                oh = (h + 2 * g.padH - g.kernelH) / g.strideH + 1;
                ow = (w + 2 * g.padW - g.kernelW) / g.strideW + 1;
                break;
            }
            case CBX_RELU:
                break;
            case CBX_MAXPOOL:
                if (l.window < 1 || l.stride < 1 || l.window > h || l.window > w)
                    throw Error(CBX_E_GEOMETRY, where((int)k, l.kind) + ": invalid pooling window");
                oh = (h - l.window) / l.stride + 1;
                ow = (w - l.window) / l.stride + 1;
                break;
            case CBX_CLASSIFY:
                if (k + 1 != L.size()) throw Error(CBX_E_SPEC, where((int)k, l.kind) + ": CLASSIFY must be the last layer");
                if (c != net.numClasses)
                    throw Error(CBX_E_SPEC, where((int)k, l.kind) + ": classification input has " + std::to_string(c) +
                                                " channels, expected " + std::to_string(net.numClasses) + " classes");
                oc = 1;
                break;
            default:
                throw Error(CBX_E_SPEC, "unknown layer kind");
        }
        dims[6 * k + 3] = oc;
        dims[6 * k + 4] = oh;
        dims[6 * k + 5] = ow;
        c = oc;
        h = oh;
        w = ow;
    }
    const bool hasClassify = L.back().kind == CBX_CLASSIFY;
    const int finalC = hasClassify ? dims[6 * (L.size() - 1)] : dims[6 * (L.size() - 1) + 3];
    if (finalC != net.numClasses)
        throw Error(CBX_E_SPEC, "network produces " + std::to_string(finalC) + " channels, expected " +
                                    std::to_string(net.numClasses) + " classes");
    return dims;
}

struct Engine::Plan {
    bool baseline = false;
    std::vector<TensorView> T;      // nl+1; T[0] = frame (planar) unless ingested
    std::vector<TensorView> T16;    // nl+1; fp16 shadows (4-byte channel units) of kind::f16 conv inputs
    std::vector<TensorView> T16b;   // packed shadows: the same shifted by 8 bytes (d[v + 2] = T16.d[v])
    bool ingest = false;            // first layer is not a conv: frame copied to HWC T[0]
    std::vector<BitMask> chg;       // nl+1
    std::vector<bool> chg_by_conv;  // chg written with 1s only -> cleared per frame
    std::vector<BitMask> upd;       // nl+1 (aliases)
    std::vector<int> upd_owner;     // producing layer of upd[t] (-1 detect, -2 none)
    std::vector<BitMask> U;         // nl (owned)
    std::vector<int32_t*> idx;
    std::vector<int*> cnt;
    std::vector<int> idx_src;       // conv layer whose list is reused (-1: own)
    std::vector<void*> allocs;
    uint16_t* labels = nullptr;
    unsigned long long* stats = nullptr;  // [nl][S][2]
    // graphs: [steady, full] x [fp32 frames, 8-bit native frames]
    cudaGraphExec_t gexec[4] = {nullptr, nullptr, nullptr, nullptr};
    int launches[4] = {0, 0, 0, 0};
    // CBX_OPT_STEP_TIMES: event-record nodes at the kernel boundaries of each graph
    std::vector<Engine::ProfMark> tm[4];
    void drop_marks(int m) {
        for (auto& x : tm[m]) cudaEventDestroy(x.ev);
        tm[m].clear();
    }
    bool dirty = true;
    int fused_from = -1;            // conv layer whose epilogue runs the per-pixel tail (-1: none)
    uint32_t* work = nullptr;       // touched-pixel list shared by the MAXPOOL/RELU layers
    TensorView rgbx_tv{};           // 8-bit path: RGBX copy of this plan's last frame (layer-1 input)
    Rgbx8View rgbx{};
    int* ovf = nullptr;             // fp16 shadow overflow flag (sticky until a full frame)
    // Frame scratch zeroed by ONE memset at the start of a steady frame:
    // stats counters, each compaction's look-back status words, each
    // MAXPOOL/RELU's work-list counter (no per-kernel memset nodes).
    uint8_t* scratch = nullptr;
    size_t scratch_bytes = 0;
    std::vector<void*> ws_k;        // per conv layer
    std::vector<int*> wcount_k;     // per MAXPOOL/RELU layer

    ~Plan() {
        for (auto& g : gexec)
            if (g) cudaGraphExecDestroy(g);
        for (int m = 0; m < 4; ++m) drop_marks(m);
        for (void* p : allocs) cudaFree(p);
    }
    template <class T>
    T* alloc(size_t n) {
        T* p = dmalloc<T>(n);
        allocs.push_back(p);
        return p;
    }
    BitMask mask(int S, int H, int W) {
        const int wpr = (W + 31) / 32;
        BitMask m{nullptr, H, W, wpr, round_up((int64_t)H * wpr, 2048)};
        m.d = alloc<uint32_t>((size_t)(m.stride * S));
        return m;
    }
};

Engine::Engine(const cbx_net_desc& net, int device, int S, int precision)
    : device_(device), S_(S), precision_(precision) {
    if (S < 1) throw Error(CBX_E_ARG, "num_streams must be >= 1");
    if (precision != CBX_PREC_EXACT && precision != CBX_PREC_TF32 && precision != CBX_PREC_F16)
        throw Error(CBX_E_ARG, "bad precision (CBX_PREC_EXACT, CBX_PREC_TF32 or CBX_PREC_F16)");
    dims_ = chain_dims(net, layers_);
    net_ = net;
    net_.layers = layers_.data();
    CBX_CUDA(cudaSetDevice(device));
    int ndev = 0;
    CBX_CUDA(cudaGetDeviceCount(&ndev));
    CBX_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    const int nl = (int)layers_.size();
    dK_.assign(nl, nullptr);
    dBias_.assign(nl, nullptr);
    hK_.assign(nl, {});
    hB_.assign(nl, {});
    tc_.resize(nl);
    mpr_.resize(nl);
    for (int k = 0; k < nl; ++k) {
        if (layers_[k].kind == CBX_CBCONV) cb_layers_.push_back(k);
        if (is_conv(layers_[k].kind)) {
            const cbx_geom& g = layers_[k].geom;
            const size_t kd = (size_t)g.inChannels * g.kernelH * g.kernelW;
            dK_[k] = dmalloc<float>(kd * g.outChannels);
            dBias_[k] = dmalloc<float>(g.outChannels);
            // tcgen05 for channels-last inputs in TF32 mode (every conv but a
            // first layer reading the planar frame).
            // (N >= 32 output channels: narrower 1x1 heads stay exact on CUDA cores,
            //  usually fused into the epilogue of the preceding tcgen05 layer)
            if (precision_ != CBX_PREC_EXACT && k > 0 && g.outChannels >= 32 && tc_supported(g)) {
                const int te = tail_end(k);
                const int c1 = te > 0 ? layers_[k + 1].geom.outChannels : 0;
                const int tail_floats = te > 0 ? (c1 <= 8 ? 8 : 16) * g.outChannels : 0;
                // CBX_PREC_F16: fp16 operands (kind::f16: 10 explicit mantissa
                // bits like tf32, twice the rate, half the bytes) for a wide
                // layer fed by a MAXPOOL, which also writes an fp16
                // (round-to-nearest) shadow of its output.
                const bool f16 = precision_ == CBX_PREC_F16 && g.outChannels > 128 &&
                                 layers_[k - 1].kind == CBX_MAXPOOL;
                if (f16) f16_layers_.push_back(k);
                tc_[k] = make_tc_layer(g, tail_floats, -1, f16, false, group_width_for(g), pack_f16(k));
                // narrow layer on a 4-channel input (paper layer 2): groups of
                // R adjacent output pixels per tensor-core row, fp16 operands
                // converted while gathering. Opt-in (CBX_MPR_F16=1): on the
                // paper's layer 2 the fp32 output scatter (52 channels per
                // pixel) bounds it, and it measured slower than conv_tc's tf32
                // path (R = 1/2/4: 52/63/87 vs 44 us per 8 x 1080p lane-frame)
                const char* me = std::getenv("CBX_MPR_F16");
                if (precision_ == CBX_PREC_F16 && !f16 && te < 0 && g.inChannels <= 4 && me && std::atoi(me) == 1) {
                    int R = 4;
                    if (const char* re = std::getenv("CBX_MPR_R")) R = std::atoi(re);  // (tuning)
                    while (R > 1 && !mpr_supported(g, 1, R)) R /= 2;
                    if (mpr_supported(g, 1, R)) mpr_[k] = make_mpr_layer(g, 1, R, 0);
                }
            }
        }
    }
    any_f16_ = !f16_layers_.empty();
    for (const auto& m : mpr_) any_f16_ = any_f16_ || (m && mpr_mode(*m) == 1);
    const bool hasClassify = layers_.back().kind == CBX_CLASSIFY;
    const int fl = nl - 1;
    lh_ = hasClassify ? dims_[6 * fl + 1] : dims_[6 * fl + 4];
    lw_ = hasClassify ? dims_[6 * fl + 2] : dims_[6 * fl + 5];
    const float** tbl = dmalloc<const float*>(2 * (size_t)S);
    d_cur_ = tbl;
    d_prev_ = tbl + S;
    // 8-bit camera path: layer 1 as kind::i8 over an RGBX copy of the frame
    // (tensor-core precisions; exact mode decodes to fp32 and stays bitwise)
    if (precision_ != CBX_PREC_EXACT && is_conv(layers_[0].kind) && rgb8_native_ok(net.inputChannels, net.inputHeight, net.inputWidth) &&
        tc_i8_supported(layers_[0].geom)) {
        const cbx_geom& g = layers_[0].geom;
        tc8_ = make_tc_layer(g, 0, -1, false, true);
        const char* me = std::getenv("CBX_MPR");
        if (mpr_supported(g, 0, 4) && !(me && std::atoi(me) == 0))
            mpr8_ = make_mpr_layer(g, 0, 4, (int)round_up(g.padW, 4));
        const uint8_t** t8 = dmalloc<const uint8_t*>(2 * (size_t)S);
        d_cur8_ = t8;
        d_prev8_ = t8 + S;
    }
    const size_t frame = (size_t)net.inputChannels * net.inputHeight * net.inputWidth * S;
    for (auto& s : slots_) s = dmalloc<float>(frame);
    CBX_CUDA(cudaMallocHost(&h_stats_, sizeof(unsigned long long) * 2 * stats_words()));
    last_cb_frames_.assign(S, nullptr);
    for (int e = 0; e < 2; ++e) {
        last_stats_[e].assign((size_t)S * nl, cbx_layer_stats{0, 0, 0});
        last_macs_[e].assign(S, 0);
    }
    cb_.reset(new Plan);
    build_plan(*cb_, false);
}

Engine::~Engine() {
    cudaSetDevice(device_);
    if (stream_) cudaStreamSynchronize(stream_);
    cb_.reset();
    base_.reset();
    tc_.clear();
    for (float* p : dK_) cudaFree(p);
    for (float* p : dBias_) cudaFree(p);
    cudaFree(d_cur_);
    for (auto& s : slots_) cudaFree(s);
    tc8_.reset();
    mpr8_.reset();
    mpr_.clear();
    if (d_cur8_) cudaFree(d_cur8_);
    if (prev_dec_) cudaFree(prev_dec_);
    for (auto& s : slots8_)
        if (s) cudaFree(s);
    cudaFreeHost(h_stats_);
    if (copy_st_) cudaStreamSynchronize(copy_st_);
    for (int q = 0; q < kRing; ++q) {
        if (ring_u8_[q]) cudaFree(ring_u8_[q]);
        if (ring_[q]) cudaFree(ring_[q]);
        if (copied_[q]) cudaEventDestroy(copied_[q]);
        if (done_[q]) cudaEventDestroy(done_[q]);
    }
    if (h_ring_stats_) cudaFreeHost(h_ring_stats_);
    if (copy_st_) cudaStreamDestroy(copy_st_);
    if (stream_) cudaStreamDestroy(stream_);
}

int Engine::list_group(int k, bool u8) const {
    if (k == 0 && u8 && mpr8_) return mpr_group_width(*mpr8_);
    if (mpr_[k]) return mpr_group_width(*mpr_[k]);
    if (tc_[k]) return tc_group_width(*tc_[k]);
    return 1;
}

// Pixel groups for a narrow tcgen05 layer on a 4-channel input (the paper's
// layer 2): R adjacent output pixels per tensor-core row share their window
// (R = 4: K = 7 x 10 taps instead of 4 x 7 x 7, N = 4 x 64) -- 2.8x fewer
// gathered bytes and 1.7x fewer MMA cycles per pixel. Opt-in (CBX_TC_GROUP =
// 2 or 4): on the paper's layer 2 the kernel time did not follow (8-stream
// lane-frame: 49 / 47 / 53 us for R = 4 / 2 / 1) and the two-lane step was
// best with R = 1 (31.7k vs 31.0k frames/s). make_tc_layer falls back to 1
// where unsupported.
// fp16 operands from the unpadded shadow (packed kernel rows) when the
// input's padded row pitch is even (CBX_TC_PACK=0 keeps the padded layout;
// tuning): the paper's layer 3 gathers 46 instead of 49 chunks per kernel
// row, 41 instead of 43 K-blocks.
bool Engine::pack_f16(int k) const {
    const char* e = std::getenv("CBX_TC_PACK");
    if (e && std::atoi(e) == 0) return false;
    const int W = dims_[6 * k + 2];
    return ((W + 2 * layers_[k].geom.padW) & 1) == 0;
}

// Pixel groups of R = 2 for narrow tcgen05 layers on a 4-channel input (the
// paper's layer 2): one tensor-core row carries two adjacent output pixels
// (N = 2 x 64 costs what N = 64 does: profiles/r2_mma_cost_by_n.log), 56 K
// taps for two pixels instead of 49 for one. CBX_TC_GROUP overrides (1 = one
// pixel per row).
int Engine::group_width_for(const cbx_geom& g) const {
    int R = 2;
    if (const char* e = std::getenv("CBX_TC_GROUP")) R = std::max(1, std::min(4, std::atoi(e)));
    while (R > 1 && !tc_group_supported(g, R)) R /= 2;
    return R;
}

int Engine::layer_operands(int layer) const {
    if (layer < 0 || layer >= (int)layers_.size() || !is_conv(layers_[layer].kind)) return -1;
    if (layer == 0 && u8_native()) return 3;
    if (mpr_[layer]) return 2;
    if (!tc_[layer]) return 0;
    return tc_is_f16(*tc_[layer]) ? 2 : 1;
}

Engine::Plan& Engine::plan(int engine) {
    if (engine == CBX_ENGINE_CBINFER) return *cb_;
    if (!base_) {
        base_.reset(new Plan);
        build_plan(*base_, true);
    }
    return *base_;
}

void Engine::build_plan(Plan& p, bool baseline) {
    const int nl = (int)layers_.size(), S = S_;
    p.baseline = baseline;
    p.T.assign(nl + 1, TensorView{});
    p.chg.assign(nl + 1, BitMask{nullptr, 0, 0, 0, 0});
    p.chg_by_conv.assign(nl + 1, false);
    p.upd.assign(nl + 1, BitMask{nullptr, 0, 0, 0, 0});
    p.upd_owner.assign(nl + 1, -2);
    p.U.assign(nl, BitMask{nullptr, 0, 0, 0, 0});
    p.idx.assign(nl, nullptr);
    p.cnt.assign(nl, nullptr);
    p.idx_src.assign(nl, -1);
    const bool hasClassify = layers_.back().kind == CBX_CLASSIFY;

    auto consumer_kind = [&](int t) -> int {  // kind of the layer reading tensor t; 4 = final argmax
        if (t < nl) return layers_[t].kind;
        return CBX_CLASSIFY;
    };
    auto tensor_dims = [&](int t, int& c, int& h, int& w) {
        if (t == 0) {
            c = net_.inputChannels;
            h = net_.inputHeight;
            w = net_.inputWidth;
        } else {
            c = dims_[6 * (t - 1) + 3];
            h = dims_[6 * (t - 1) + 4];
            w = dims_[6 * (t - 1) + 5];
        }
    };
    auto alloc_tensor = [&](int t) {
        int c, h, w;
        tensor_dims(t, c, h, w);
        TensorView v{};
        v.C = c;
        v.H = h;
        v.W = w;
        v.Cp = (int)round_up(c, 4);
        if (t < nl && is_conv(layers_[t].kind)) {
            v.hh = layers_[t].geom.padH;
            v.hw = layers_[t].geom.padW;
        }
        v.Hp = h + 2 * v.hh;
        v.Wp = w + 2 * v.hw;
        v.ss = round_up((int64_t)v.Hp * v.Wp * v.Cp, 64);
        // (slack: a multi-pixel-row gather window of the last row may run a
        // few pixels past the last stream's right halo; zero weights there)
        v.d = p.alloc<float>((size_t)(v.ss * S) + 64 * (size_t)v.Cp);
        p.T[t] = v;
    };

    // tensors
    p.ingest = !is_conv(layers_[0].kind);
    if (p.ingest) alloc_tensor(0);
    for (int k = 0; k < nl; ++k) {
        if (layers_[k].kind == CBX_CLASSIFY) {
            p.T[k + 1] = p.T[k];
            continue;
        }
        alloc_tensor(k + 1);
    }
    p.T16.assign(nl + 1, TensorView{});
    p.T16b.assign(nl + 1, TensorView{});
    for (int k : f16_layers_) {
        // the layer's fp16 shadow: channels padded to 8, or packed (Cp = C/2
        // units) plus a copy shifted by 8 bytes (T16b, element v + 2 = T16's v)
        TensorView v = p.T[k];
        v.Cp = tc_input_cp(*tc_[k]);
        v.ss = round_up((int64_t)v.Hp * v.Wp * v.Cp, 64);
        v.d = p.alloc<float>((size_t)(v.ss * S) + 64);
        p.T16[k] = v;
        if (v.Cp * 2 == v.C) {
            TensorView b = v;
            b.d = p.alloc<float>((size_t)(v.ss * S) + 64);
            p.T16b[k] = b;
        }
    }
    if (p.T[0].d == nullptr) {
        int c, h, w;
        tensor_dims(0, c, h, w);
        p.T[0] = TensorView{nullptr, c, h, w, c, h, w, 0, 0, (int64_t)c * h * w};
    }
    if (tc8_) {
        // RGBX copy of the 8-bit frame for the kind::i8 layer 1 (zero halo,
        // never written; + slack for the last row's gather window). One per
        // plan: a change-based frame rewrites only the pixel groups whose
        // bytes differ from the previous frame, so the buffer must hold the
        // change-based engine's previous frame (the dense engine has its own).
        const cbx_geom& g = layers_[0].geom;
        TensorView v{};
        v.C = net_.inputChannels;
        v.H = net_.inputHeight;
        v.W = net_.inputWidth;
        v.Cp = 1;
        v.hh = g.padH;
        v.hw = (int)round_up(g.padW, 4);
        v.Hp = v.H + 2 * v.hh;
        v.Wp = v.W + 2 * v.hw;
        v.ss = round_up((int64_t)v.Hp * v.Wp, 64);
        v.d = p.alloc<float>((size_t)(v.ss * S) + 2 * (size_t)v.Wp + 64);
        p.rgbx_tv = v;
        p.rgbx = Rgbx8View{reinterpret_cast<uint32_t*>(v.d), v.ss, v.Wp, v.hh, v.hw};
    }
    p.labels = p.alloc<uint16_t>((size_t)S * lh_ * lw_);
    p.stats = p.alloc<unsigned long long>(stats_words());
    if (any_f16_) p.ovf = p.alloc<int>(1);
    if (baseline) return;  // full mode only: no masks, no lists

    // change masks (inputs of CBCONV layers) and updated masks
    const int nt = hasClassify ? nl : nl + 1;
    std::vector<size_t> ws_bytes(nl, 0);
    for (int t = 0; t < nt; ++t) {
        int c, h, w;
        tensor_dims(t, c, h, w);
        const int ck = consumer_kind(t);
        if (ck == CBX_CBCONV) {
            p.chg[t] = p.mask(S, h, w);
            p.chg_by_conv[t] = t > 0 && is_conv(layers_[t - 1].kind);
        } else {
            if (t == 0) {
                p.upd[0] = p.mask(S, h, w);
                p.upd_owner[0] = -1;
            } else {
                const int pk = layers_[t - 1].kind;
                if (is_conv(pk) || pk == CBX_MAXPOOL) {
                    p.upd_owner[t] = t - 1;
                } else if (pk == CBX_RELU) {
                    p.upd_owner[t] = -3;  // alias of the RELU input, resolved below
                }
            }
        }
    }
    for (int k = 0; k < nl; ++k) {
        const auto& l = layers_[k];
        const int Ho = dims_[6 * k + 4], Wo = dims_[6 * k + 5];
        if (l.kind == CBX_CBCONV) {
            p.U[k] = p.mask(S, Ho, Wo);
        } else if (l.kind == CBX_CONV) {
            if (!identity_geom(l.geom)) p.U[k] = p.mask(S, Ho, Wo);
        } else if (l.kind == CBX_MAXPOOL) {
            if (p.upd_owner[k + 1] == k) p.U[k] = p.mask(S, Ho, Wo);
        }
    }
    // resolve upd aliases in layer order (upd[t] of a RELU output = upd of its input)
    for (int t = 1; t <= nl; ++t) {
        if (p.upd_owner[t] == -3) {
            p.upd_owner[t] = p.upd_owner[t - 1];
            p.upd[t] = p.upd[t - 1];
        } else if (p.upd_owner[t] >= 0) {
            const int k = p.upd_owner[t];
            if (layers_[k].kind == CBX_CONV && identity_geom(layers_[k].geom)) {
                p.upd[t] = p.upd[k];  // U of an identity conv is its input's upd
                p.upd_owner[t] = p.upd_owner[k];
            } else {
                p.upd[t] = p.U[k];
            }
        }
    }
    // index lists
    for (int k = 0; k < nl; ++k) {
        const auto& l = layers_[k];
        if (!is_conv(l.kind)) continue;
        const int Ho = dims_[6 * k + 4], Wo = dims_[6 * k + 5];
        if (l.kind == CBX_CONV && identity_geom(l.geom) && p.upd_owner[k] >= 0 &&
            is_conv(layers_[p.upd_owner[k]].kind) && list_group(p.upd_owner[k], true) == 1 &&
            list_group(p.upd_owner[k], false) == 1) {  // (a pixel-group list cannot be reused as a pixel list)
            const int j = p.upd_owner[k];
            p.idx_src[k] = p.idx_src[j] >= 0 ? p.idx_src[j] : j;
            continue;
        }
        p.idx[k] = p.alloc<int32_t>((size_t)S * Ho * Wo);
        const int wpr = (Wo + 31) / 32;
        ws_bytes[k] = round_up(dilate_compact_workspace(BitMask{nullptr, Ho, Wo, wpr, round_up((int64_t)Ho * wpr, 2048)}, S), 256);
        // strided geometries dilate separately, then compact the dilated mask
        if (!identity_geom(l.geom) && (l.geom.strideH != 1 || l.geom.strideW != 1 || l.geom.kernelW - 1 - l.geom.padW > 31 ||
                                       l.geom.padW > 31) && !p.U[k].d)
            p.U[k] = p.mask(S, Ho, Wo);
    }
    int64_t wk = 0;
    for (int k = 0; k < nl; ++k)
        if (layers_[k].kind == CBX_MAXPOOL || layers_[k].kind == CBX_RELU)
            wk = std::max<int64_t>(wk, (int64_t)S * dims_[6 * k + 4] * dims_[6 * k + 5]);
    if (wk) {
        if (wk >= (int64_t)1 << 32) throw Error(CBX_E_ARG, "pooling work list exceeds 2^32 pixels");
        p.work = p.alloc<uint32_t>((size_t)wk);
    }
    // frame scratch: [stats][look-back status per conv][work counter per pool/relu]
    size_t off = round_up(sizeof(unsigned long long) * stats_words(), 256);
    std::vector<size_t> ws_off(nl, 0), wc_off(nl, 0);
    for (int k = 0; k < nl; ++k) {
        if (ws_bytes[k]) {
            ws_off[k] = off;
            off += ws_bytes[k];
        }
        if (layers_[k].kind == CBX_MAXPOOL || layers_[k].kind == CBX_RELU) {
            wc_off[k] = off;
            off += 256;
        }
    }
    p.scratch_bytes = off;
    p.scratch = p.alloc<uint8_t>(off);
    p.stats = reinterpret_cast<unsigned long long*>(p.scratch);
    p.ws_k.assign(nl, nullptr);
    p.wcount_k.assign(nl, nullptr);
    for (int k = 0; k < nl; ++k) {
        if (ws_bytes[k]) {
            p.ws_k[k] = p.scratch + ws_off[k];
            // the compaction's list counter lives in the frame scratch: zeroed
            // by the frame's one memset, incremented by the compaction blocks
            p.cnt[k] = reinterpret_cast<int*>(p.ws_k[k]);
        }
        if (wc_off[k]) p.wcount_k[k] = reinterpret_cast<int*>(p.scratch + wc_off[k]);
    }
}

void Engine::record(Plan& p, bool full) {
    const int nl = (int)layers_.size(), S = S_;
    cudaStream_t st = stream_;
    auto stats_of = [&](int layer, int field) { return p.stats + (size_t)layer * S * 2 + field; };
    if (full && p.ovf) CBX_CUDA(cudaMemsetAsync(p.ovf, 0, sizeof(int), st));  // full evaluation clears it
    if (!full) {
        CBX_CUDA(cudaMemsetAsync(p.scratch, 0, p.scratch_bytes, st));
        for (int t = 0; t <= nl; ++t)
            if (p.chg_by_conv[t] && p.chg[t].d)
                CBX_CUDA(cudaMemsetAsync(p.chg[t].d, 0, sizeof(uint32_t) * (size_t)(p.chg[t].stride * S), st));
    }
    mark("memset", -1);  // (profile pass: the scratch memsets get their own interval)
    // K1: detection on the raw frames
    if (rec_u8_) {
        // 8-bit frames: detection on the bytes + RGBX copy for the i8 layer 1
        const auto& in = p.T[0];
        if (!full && p.chg[0].d) {
            launch_detect_rgb8(d_cur8_, d_prev8_, S, in.H, in.W, layers_[0].threshold, 0, p.chg[0], stats_of(0, 0), 2,
                               p.rgbx, st);
            mark("detect", 0);
        } else if (!full && p.upd[0].d && p.upd_owner[0] == -1) {
            launch_detect_rgb8(d_cur8_, d_prev8_, S, in.H, in.W, 0.0f, 1, p.upd[0], nullptr, 2, p.rgbx, st);
            mark("detect_bitwise", 0);
        } else {
            launch_detect_rgb8(d_cur8_, d_cur8_, S, in.H, in.W, 0.0f, 2, BitMask{nullptr, 0, 0, 0, 0}, nullptr, 2, p.rgbx, st);
            mark("expand", 0);
        }
    } else if (!full) {
        const auto& in = p.T[0];
        if (p.chg[0].d) {
            launch_detect_bits(d_cur_, d_prev_, S, in.C, in.H, in.W, layers_[0].threshold, 0, p.chg[0],
                               stats_of(0, 0), 2, st);
            mark("detect", 0);
        }
        if (p.upd[0].d && p.upd_owner[0] == -1) {
            launch_detect_bits(d_cur_, d_prev_, S, in.C, in.H, in.W, 0.0f, 1, p.upd[0], nullptr, 2, st);
            mark("detect_bitwise", 0);
        }
    }
    if (p.ingest) {
        launch_ingest(d_cur_, p.T[0], S, st);
        mark("ingest", 0);
    }
    p.fused_from = -1;
    for (int k = 0; k < nl; ++k) {
        const auto& l = layers_[k];
        const bool has_next = k + 1 < nl;
        BitMask chg_next = (!full && has_next) ? p.chg[k + 1] : BitMask{nullptr, 0, 0, 0, 0};
        const float tau_next = has_next ? layers_[k + 1].threshold : 0.0f;
        unsigned long long* cnt_next = has_next ? stats_of(k + 1, 0) : nullptr;
        switch (l.kind) {
            case CBX_CBCONV:
            case CBX_CONV: {
                const cbx_geom& g = l.geom;
                const int32_t* idx = nullptr;
                const int* count = nullptr;
                if (!full) {
                    if (p.idx_src[k] < 0) {
                        // U_k = dilate(input change mask) (CBCONV) or dilate(input updated mask) (CONV)
                        const BitMask& src = l.kind == CBX_CBCONV ? p.chg[k] : p.upd[k];
                        unsigned long long* cnt = l.kind == CBX_CBCONV ? stats_of(k, 1) : nullptr;
                        const bool fused = g.strideH == 1 && g.strideW == 1 && g.padW <= 31 &&
                                           g.kernelW - 1 - g.padW <= 31 && 2 * g.padW <= g.kernelW - 1;
                        const int R = list_group(k, rec_u8_);
                        if (identity_geom(g)) {
                            const bool own = p.U[k].d != nullptr;  // CBCONV 1x1: U_k is its own mask
                            launch_dilate_compact(src, own ? p.U[k] : src, own, S, 1, 1, 0, 0, p.idx[k], p.cnt[k], p.ws_k[k],
                                                  cnt, 2, st, true, R);
                            mark("compact", k);
                        } else if (fused) {
                            launch_dilate_compact(src, p.U[k], true, S, g.kernelH, g.kernelW, g.padH, g.padW, p.idx[k],
                                                  p.cnt[k], p.ws_k[k], cnt, 2, st, true, R);
                            mark("dilate_compact", k);
                        } else {
                            launch_dilate_bits(src, p.U[k], S, g.kernelH, g.kernelW, g.strideH, g.strideW, g.padH, g.padW, st);
                            mark("dilate", k);
                            launch_dilate_compact(p.U[k], p.U[k], false, S, 1, 1, 0, 0, p.idx[k], p.cnt[k], p.ws_k[k], cnt, 2,
                                                  st, true);
                            mark("compact", k);
                        }
                    }
                    const int src = p.idx_src[k] >= 0 ? p.idx_src[k] : k;
                    idx = p.idx[src];
                    count = p.cnt[src];
                }
                const bool planar_in = (k == 0 && !p.ingest);
                const bool relu = l.kind == CBX_CBCONV && l.fuseRelu;
                const int64_t full_count = (int64_t)S * dims_[6 * k + 4] * dims_[6 * k + 5];
                if (k == 0 && rec_u8_) {
                    if (mpr8_)
                        launch_conv_mpr(*mpr8_, p.rgbx_tv, p.T[1], dBias_[0], reinterpret_cast<const uint32_t*>(idx), count,
                                        S, relu, chg_next, tau_next, cnt_next, 2, nullptr, st);
                    else
                        launch_conv_tc(*tc8_, p.rgbx_tv, p.T[1], dBias_[0], idx, count, full_count, relu, chg_next, tau_next,
                                       cnt_next, 2, S, st);
                    mark("conv_tc", 0);
                    break;
                }
                if (mpr_[k] && !planar_in) {
                    launch_conv_mpr(*mpr_[k], p.T[k], p.T[k + 1], dBias_[k], reinterpret_cast<const uint32_t*>(idx), count,
                                    S, relu, chg_next, tau_next, cnt_next, 2, p.ovf, st);
                    mark("conv_tc", k);
                    break;
                }
                const int tail_last = (tc_[k] && !planar_in) ? tail_end(k) : -1;
                if (tail_last > 0) {
                    // per-pixel layers k+1..tail_last fused into this conv's epilogue
                    TcTail t{};
                    int prevC = l.geom.outChannels;
                    for (int j = k + 1; j <= tail_last && layers_[j].kind != CBX_CLASSIFY; ++j) {
                        if (layers_[j].kind == CBX_CONV) {
                            t.kind[t.n] = 0;
                            t.cout[t.n] = layers_[j].geom.outChannels;
                            t.W[t.n] = dK_[j];
                            t.b[t.n] = dBias_[j];
                            prevC = t.cout[t.n];
                        } else {
                            t.kind[t.n] = 1;
                            t.cout[t.n] = prevC;
                        }
                        ++t.n;
                    }
                    const TensorView& fo = p.T[final_tensor()];
                    t.final_out = fo.d;
                    t.fo_ss = fo.ss;
                    t.fo_Wp = fo.Wp;
                    t.fo_Cp = fo.Cp;
                    t.fo_hh = fo.hh;
                    t.fo_hw = fo.hw;
                    t.labels = p.labels;
                    t.l_ss = (int64_t)lh_ * lw_;
                    launch_conv_tc(*tc_[k], p.T16[k].d ? p.T16[k] : p.T[k], p.T[k + 1], dBias_[k], idx, count, full_count, relu,
                                   chg_next, tau_next, cnt_next, 2, S, st, &t, p.T16b[k].d);
                    mark("conv_tc_tail", k);
                    p.fused_from = k;
                    break;
                } else if (tc_[k] && !planar_in) {
                    launch_conv_tc(*tc_[k], p.T16[k].d ? p.T16[k] : p.T[k], p.T[k + 1], dBias_[k], idx, count, full_count, relu,
                                   chg_next, tau_next, cnt_next, 2, S, st, nullptr, p.T16b[k].d);
                    mark("conv_tc", k);
                } else {
                    ConvArgs a{};
                    a.in = p.T[k];
                    a.in_ptrs = planar_in ? d_cur_ : nullptr;
                    a.out = p.T[k + 1];
                    a.K = dK_[k];
                    a.bias = dBias_[k];
                    a.kh = g.kernelH;
                    a.kw = g.kernelW;
                    a.sh = g.strideH;
                    a.sw = g.strideW;
                    a.ph = g.padH;
                    a.pw = g.padW;
                    a.idx = idx;
                    a.count = count;
                    a.full_count = full_count;
                    a.relu = relu;
                    a.chg = chg_next;
                    a.tau = tau_next;
                    a.chg_cnt = cnt_next;
                    a.cnt_stride = 2;
                    a.S = S;
                    a.hK = hK_[k].data();
                    a.hB = hB_[k].data();
                    launch_conv_exact(a, st); mark("conv_exact", k);
                }
                break;
            }
            case CBX_RELU:
            case CBX_MAXPOOL: {
                const BitMask none{nullptr, 0, 0, 0, 0};
                PointBitsArgs a{};
                a.in = p.T[k];
                a.out = p.T[k + 1];
                a.relu = l.kind == CBX_RELU;
                a.window = a.relu ? 1 : l.window;
                a.stride = a.relu ? 1 : l.stride;
                a.upd_in = full ? none : p.upd[k];
                a.U_out = (full || a.relu) ? none : p.U[k];
                a.chg = chg_next;
                a.tau = tau_next;
                a.chg_cnt = cnt_next;
                a.cnt_stride = 2;
                a.S = S;
                a.work = p.work;
                a.work_count = p.wcount_k.empty() ? nullptr : p.wcount_k[k];  // (sparse frames only)
                a.count_zeroed = 1;
                a.out16 = p.T16[k + 1];
                a.out16b = p.T16b[k + 1];
                a.f16_overflow = p.T16[k + 1].d ? p.ovf : nullptr;
                launch_point_bits(a, st);
                mark(a.relu ? "relu" : "pool", k);
                break;
            }
            case CBX_CLASSIFY:
                launch_classify_bits(p.T[k], full ? BitMask{nullptr, 0, 0, 0, 0} : p.upd[k], p.labels, S, st);
                mark("classify", k);
                break;
        }
        if (p.fused_from == k) break;  // the rest of the network ran in that epilogue
    }
    if (p.fused_from < 0 && layers_.back().kind != CBX_CLASSIFY) {
        launch_classify_bits(p.T[nl], full ? BitMask{nullptr, 0, 0, 0, 0} : p.upd[nl], p.labels, S, st);
        mark("classify", nl);
    }
    // this frame's view of the (sticky) fp16 overflow flag, read back with its counters
    if (p.ovf)
        CBX_CUDA(cudaMemcpyAsync(p.stats + stats_words() - 1, p.ovf, sizeof(int), cudaMemcpyDeviceToDevice, st));
    CBX_CUDA(cudaGetLastError());
}

void Engine::launch(Plan& p, bool full) {
    const int m = (full ? 1 : 0) + (rec_u8_ ? 2 : 0);
    if (p.dirty) {
        for (auto& g : p.gexec)
            if (g) {
                cudaGraphExecDestroy(g);
                g = nullptr;
            }
        p.dirty = false;
    }
    if (!p.gexec[m]) {
        cudaGraph_t graph = nullptr;
        p.drop_marks(m);
        if (step_times_) {  // events exist before the capture records them
            for (int i = 0; i < 64; ++i) {
                cudaEvent_t e;
                CBX_CUDA(cudaEventCreate(&e));
                p.tm[m].push_back(ProfMark{"", -1, e});
            }
        }
        CBX_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
        try {
            if (step_times_) {
                tmarks_ = &p.tm[m];
                tmarks_used_ = 0;
                mark("start", -1);
            }
            record(p, full);
            tmarks_ = nullptr;
        } catch (...) {
            tmarks_ = nullptr;
            cudaStreamEndCapture(stream_, &graph);
            if (graph) cudaGraphDestroy(graph);
            throw;
        }
        if (step_times_) {
            for (size_t i = tmarks_used_; i < p.tm[m].size(); ++i) cudaEventDestroy(p.tm[m][i].ev);
            p.tm[m].resize(tmarks_used_);
        }
        CBX_CUDA(cudaStreamEndCapture(stream_, &graph));
        size_t n = 0;
        CBX_CUDA(cudaGraphGetNodes(graph, nullptr, &n));
        std::vector<cudaGraphNode_t> nodes(n);
        if (n) CBX_CUDA(cudaGraphGetNodes(graph, nodes.data(), &n));
        int kernels = 0;
        for (auto nd : nodes) {
            cudaGraphNodeType t;
            CBX_CUDA(cudaGraphNodeGetType(nd, &t));
            kernels += t == cudaGraphNodeTypeKernel;
        }
        p.launches[m] = kernels;
        CBX_CUDA(cudaGraphInstantiate(&p.gexec[m], graph, 0));
        cudaGraphDestroy(graph);
    }
    CBX_CUDA(cudaGraphLaunch(p.gexec[m], stream_));
    last_launches_ = p.launches[m];
    last_tm_ = step_times_ ? &p.tm[m] : nullptr;
}

void Engine::stage_frame_pointers(int engine, const float* const* cur, const float* const* prev) {
    (void)engine;
    for (int s = 0; s < S_; ++s)
        if (!cur[s] || reinterpret_cast<uintptr_t>(cur[s]) % 16)
            throw Error(CBX_E_ARG, "frame pointers must be non-null and 16-byte aligned");
    std::vector<const float*> tbl(2 * (size_t)S_);
    for (int s = 0; s < S_; ++s) {
        tbl[s] = cur[s];
        tbl[S_ + s] = prev ? prev[s] : cur[s];
    }
    // pageable source: staged by the driver before return, safe to reuse
    CBX_CUDA(cudaMemcpyAsync(d_cur_, tbl.data(), sizeof(const float*) * 2 * S_, cudaMemcpyHostToDevice, stream_));
}

void Engine::forward_host(int engine, const float* frames, uint16_t* labels, cbx_layer_stats* stats,
                          uint64_t* macs) {
    enqueue_host(engine, frames);
    if (labels) read_labels(engine, labels);
    read_stats(engine, stats, macs);
}

// 8-bit host frames (S x H x W x C interleaved, the PPM raster): H2D of the
// bytes into a staging buffer, decoded on the device into the frame slot
// (px / 255, read_ppm io.cpp:60-104), then the frame as enqueue_host.
void Engine::enqueue_host_u8(int engine, const uint8_t* frames) {
    if (!frames) throw Error(CBX_E_ARG, "frames is null");
    if (engine != CBX_ENGINE_CBINFER && engine != CBX_ENGINE_BASELINE) throw Error(CBX_E_ARG, "bad engine");
    CBX_CUDA(cudaSetDevice(device_));
    const size_t per = (size_t)net_.inputChannels * net_.inputHeight * net_.inputWidth;
    // byte staging (CB ping-pong: the previous frame stays the detection
    // reference; the dense comparator has its own slot)
    const int q = engine == CBX_ENGINE_CBINFER ? parity8_ : 2;
    if (!slots8_[q]) slots8_[q] = dmalloc<uint8_t>(per * S_);
    CBX_CUDA(cudaMemcpyAsync(slots8_[q], frames, per * S_, cudaMemcpyHostToDevice, stream_));
    std::vector<const uint8_t*> cur(S_);
    for (int s = 0; s < S_; ++s) cur[s] = slots8_[q] + per * s;
    forward_device_u8(engine, cur.data());
    if (engine == CBX_ENGINE_CBINFER) parity8_ ^= 1;
}

void Engine::forward_host_u8(int engine, const uint8_t* frames, uint16_t* labels, cbx_layer_stats* stats,
                             uint64_t* macs) {
    enqueue_host_u8(engine, frames);
    if (labels) read_labels(engine, labels);
    read_stats(engine, stats, macs);
}

// Host frames -> staging slot (CB ping-pong / baseline) -> forward, all
// asynchronous on the context stream.
void Engine::enqueue_host(int engine, const float* frames) {
    if (!frames) throw Error(CBX_E_ARG, "frames is null");
    if (engine != CBX_ENGINE_CBINFER && engine != CBX_ENGINE_BASELINE) throw Error(CBX_E_ARG, "bad engine");
    CBX_CUDA(cudaSetDevice(device_));
    const size_t per = (size_t)net_.inputChannels * net_.inputHeight * net_.inputWidth;
    float* slot = engine == CBX_ENGINE_CBINFER ? slots_[parity_] : slots_[2];
    CBX_CUDA(cudaMemcpyAsync(slot, frames, per * S_ * sizeof(float), cudaMemcpyHostToDevice, stream_));
    std::vector<const float*> cur(S_);
    for (int s = 0; s < S_; ++s) cur[s] = slot + per * s;
    forward_device(engine, cur.data());
    if (engine == CBX_ENGINE_CBINFER) parity_ ^= 1;
}

void Engine::forward_device(int engine, const float* const* frames_dev) {
    // counters stay on the device until cbx_read_stats asks for them (the
    // frame scratch holds the last frame's counters until the next frame)
    enqueue(engine, frames_dev, nullptr, nullptr);
    stats_pending_[engine] = true;
}

void Engine::forward_device_u8(int engine, const uint8_t* const* frames_dev) {
    enqueue(engine, nullptr, frames_dev, nullptr);
    stats_pending_[engine] = true;
}

bool Engine::u8_native() const {
    return u8_opt_ && tc8_ && rgb8_native_ok(net_.inputChannels, net_.inputHeight, net_.inputWidth);
}

// Frame path selection. 8-bit frames run natively (detection on the bytes,
// kind::i8 layer 1) when the engine supports it and the change-based history
// is 8-bit too (or there is none); otherwise they are decoded (px / 255.0f,
// read_ppm) into an fp32 slot that then serves as the history. An fp32 frame
// after 8-bit history gets the previous frames decoded as its detection
// reference. Either way the change masks are those of the reference on
// read_ppm's tensors.
bool Engine::prepare_frame(int engine, const float* const* f32, const uint8_t* const* u8) {
    if (engine != CBX_ENGINE_CBINFER && engine != CBX_ENGINE_BASELINE) throw Error(CBX_E_ARG, "bad engine");
    if (!f32 && !u8) throw Error(CBX_E_ARG, "frames is null");
    CBX_CUDA(cudaSetDevice(device_));
    const bool cb = engine == CBX_ENGINE_CBINFER;
    const bool full = !cb || !has_history_;
    const size_t per = (size_t)net_.inputChannels * net_.inputHeight * net_.inputWidth;
    cur_u8_.clear();
    cur_f32_.clear();
    if (u8) {
        for (int s = 0; s < S_; ++s)
            if (!u8[s] || reinterpret_cast<uintptr_t>(u8[s]) % 16)
                throw Error(CBX_E_ARG, "frame pointers must be non-null and 16-byte aligned");
        rec_u8_ = u8_native() && (full || hist_u8_);
        if (rec_u8_) {
            cur_u8_.assign(u8, u8 + S_);
            std::vector<const uint8_t*> tbl(2 * (size_t)S_);
            for (int s = 0; s < S_; ++s) {
                tbl[s] = u8[s];
                tbl[S_ + s] = full ? u8[s] : last_cb_frames8_[s];
            }
            CBX_CUDA(cudaMemcpyAsync(d_cur8_, tbl.data(), sizeof(const uint8_t*) * 2 * S_, cudaMemcpyHostToDevice, stream_));
            return full;
        }
        // decode into the fp32 staging slot of this frame
        float* slot = cb ? slots_[parity_] : slots_[2];
        if (cb) parity_ ^= 1;
        for (int s = 0; s < S_; ++s) {
            launch_decode_u8(u8[s], 1, net_.inputChannels, net_.inputHeight, net_.inputWidth, slot + per * s, stream_);
            cur_f32_.push_back(slot + per * s);
        }
    } else {
        rec_u8_ = false;
        cur_f32_.assign(f32, f32 + S_);
    }
    const float* const* prev = nullptr;
    std::vector<const float*> dec;
    if (cb && !full) {
        if (hist_u8_) {
            if (!prev_dec_) prev_dec_ = dmalloc<float>(per * S_);
            for (int s = 0; s < S_; ++s) {
                launch_decode_u8(last_cb_frames8_[s], 1, net_.inputChannels, net_.inputHeight, net_.inputWidth,
                                 prev_dec_ + per * s, stream_);
                dec.push_back(prev_dec_ + per * s);
            }
            prev = dec.data();
        } else {
            prev = last_cb_frames_.data();
        }
    }
    stage_frame_pointers(engine, cur_f32_.data(), prev);
    return full;
}

void Engine::frame_done(int engine) {
    if (engine != CBX_ENGINE_CBINFER) return;
    has_history_ = true;
    hist_u8_ = rec_u8_;
    if (rec_u8_)
        last_cb_frames8_ = cur_u8_;
    else
        last_cb_frames_ = cur_f32_;
}

// Enqueues one frame on the context stream (pointer table, graph, counter
// readback into stats_dst); returns whether it is a full evaluation.
bool Engine::enqueue(int engine, const float* const* frames_dev, const uint8_t* const* frames_u8,
                     unsigned long long* stats_dst) {
    const bool full = prepare_frame(engine, frames_dev, frames_u8);
    Plan& p = plan(engine);
    launch(p, full);
    if (stats_dst)
        CBX_CUDA(cudaMemcpyAsync(stats_dst, p.stats, sizeof(unsigned long long) * stats_words(), cudaMemcpyDeviceToHost,
                                 stream_));
    last_full_[engine] = full;
    frame_done(engine);
    return full;
}

// Pipelined host-frame path (cbx_submit / cbx_wait). Frame j is copied into
// ring slot j % 3 on a copy stream and evaluated on the context stream once
// the copy has landed, so the H2D copy of frame j+1 overlaps the kernels of
// frame j. Slot j % 3 was last read by frame j-2 (as its detection
// reference), hence the copy of frame j waits for frame j-2 only.
int64_t Engine::submit(int engine, const float* frames, uint16_t* labels) {
    return submit_any(engine, frames, nullptr, labels);
}

int64_t Engine::submit_u8(int engine, const uint8_t* frames, uint16_t* labels) {
    return submit_any(engine, nullptr, frames, labels);
}

// f32: planar fp32 host frames copied into the ring slot; u8: 8-bit
// interleaved host frames copied into a byte ring and decoded into the slot
// on the context stream (4x fewer PCIe bytes).
int64_t Engine::submit_any(int engine, const float* frames, const uint8_t* frames_u8, uint16_t* labels) {
    if (engine != CBX_ENGINE_CBINFER)
        throw Error(CBX_E_ARG, "cbx_submit runs the change-based engine (use cbx_forward for the dense comparator)");
    if ((!frames && !frames_u8) || !labels) throw Error(CBX_E_ARG, "null frames or labels");
    CBX_CUDA(cudaSetDevice(device_));
    const int nl = (int)layers_.size();
    const size_t per = (size_t)net_.inputChannels * net_.inputHeight * net_.inputWidth;
    if (!copy_st_) {
        CBX_CUDA(cudaStreamCreateWithFlags(&copy_st_, cudaStreamNonBlocking));
        for (int q = 0; q < kRing; ++q) {
            CBX_CUDA(cudaEventCreateWithFlags(&copied_[q], cudaEventDisableTiming));
            CBX_CUDA(cudaEventCreateWithFlags(&done_[q], cudaEventDisableTiming));
        }
        CBX_CUDA(cudaMallocHost(&h_ring_stats_, sizeof(unsigned long long) * kRing * stats_words()));
    }
    const int64_t j = submitted_;
    const int q = (int)(j % kRing);
    if (j >= 2) CBX_CUDA(cudaStreamWaitEvent(copy_st_, done_[(j - 2) % kRing], 0));
    if (frames_u8) {
        if (!ring_u8_[q]) ring_u8_[q] = dmalloc<uint8_t>(per * S_);
        CBX_CUDA(cudaMemcpyAsync(ring_u8_[q], frames_u8, per * S_, cudaMemcpyHostToDevice, copy_st_));
    } else {
        if (!ring_[q]) ring_[q] = dmalloc<float>(per * S_);
        CBX_CUDA(cudaMemcpyAsync(ring_[q], frames, per * S_ * sizeof(float), cudaMemcpyHostToDevice, copy_st_));
    }
    CBX_CUDA(cudaEventRecord(copied_[q], copy_st_));
    CBX_CUDA(cudaStreamWaitEvent(stream_, copied_[q], 0));
    // ring slot q was last read by frame j-2 (as its detection reference)
    if (frames_u8) {
        std::vector<const uint8_t*> cur(S_);
        for (int s = 0; s < S_; ++s) cur[s] = ring_u8_[q] + per * s;
        ring_full_[q] = enqueue(engine, nullptr, cur.data(), h_ring_stats_ + (size_t)q * stats_words());
    } else {
        std::vector<const float*> cur(S_);
        for (int s = 0; s < S_; ++s) cur[s] = ring_[q] + per * s;
        ring_full_[q] = enqueue(engine, cur.data(), nullptr, h_ring_stats_ + (size_t)q * stats_words());
    }
    CBX_CUDA(cudaMemcpyAsync(labels, plan(engine).labels, sizeof(uint16_t) * S_ * lh_ * lw_, cudaMemcpyDeviceToHost,
                             stream_));
    CBX_CUDA(cudaEventRecord(done_[q], stream_));
    ring_ticket_[q] = j;
    submitted_ = j + 1;
    return j;
}

void Engine::wait(int64_t ticket, cbx_layer_stats* stats, uint64_t* macs) {
    const int q = (int)(((ticket % kRing) + kRing) % kRing);
    if (ticket < 0 || ticket >= submitted_ || ring_ticket_[q] != ticket)
        throw Error(CBX_E_ARG, "cbx_wait: unknown or expired ticket (at most the last 3 submissions can be waited on)");
    CBX_CUDA(cudaSetDevice(device_));
    CBX_CUDA(cudaEventSynchronize(done_[q]));
    const int nl = (int)layers_.size();
    const unsigned long long* hs = h_ring_stats_ + (size_t)q * stats_words();
    check_f16_overflow(hs, CBX_ENGINE_CBINFER);
    std::vector<cbx_layer_stats> st((size_t)S_ * nl);
    std::vector<uint64_t> mc(S_);
    stats_from(hs, ring_full_[q], CBX_ENGINE_CBINFER, st.data(), mc.data());
    if (stats) std::memcpy(stats, st.data(), sizeof(cbx_layer_stats) * st.size());
    if (macs) std::memcpy(macs, mc.data(), sizeof(uint64_t) * S_);
}

void Engine::sync() { CBX_CUDA(cudaStreamSynchronize(stream_)); }

void Engine::finish_stats(Plan& p, bool full, int engine) {
    (void)p;
    const int nl = (int)layers_.size();
    stats_from(h_stats_ + (size_t)engine * stats_words(), full, engine, last_stats_[engine].data(), last_macs_[engine].data());
    last_ovf_[engine] = h_stats_[(size_t)engine * stats_words() + stats_words() - 1] != 0;
}

// Per-stream LayerStats from the device counters (cbconv.cpp:170-192,
// 212-220; non-CB convs report full-frame work, network.cpp:241-248,290-294).
void Engine::stats_from(const unsigned long long* hs, bool full, int engine, cbx_layer_stats* out, uint64_t* macs) const {
    const int nl = (int)layers_.size();
    for (int s = 0; s < S_; ++s) {
        uint64_t total = 0;
        for (int k = 0; k < nl; ++k) {
            const auto& l = layers_[k];
            cbx_layer_stats st{0, 0, 0};
            const int64_t inHW = (int64_t)dims_[6 * k + 1] * dims_[6 * k + 2];
            const int64_t outHW = (int64_t)dims_[6 * k + 4] * dims_[6 * k + 5];
            if (is_conv(l.kind)) {
                const uint64_t rc = (uint64_t)l.geom.outChannels * l.geom.inChannels * l.geom.kernelH * l.geom.kernelW;
                if (l.kind == CBX_CBCONV && engine == CBX_ENGINE_CBINFER) {
                    if (full) {
                        st.changedInputPixels = inHW;
                        st.changedOutputPixels = outHW;
                    } else {
                        st.changedInputPixels = (int64_t)hs[((size_t)k * S_ + s) * 2 + 0];
                        st.changedOutputPixels = (int64_t)hs[((size_t)k * S_ + s) * 2 + 1];
                    }
                    st.gemmMacs = rc * (uint64_t)st.changedOutputPixels;
                } else {
                    st.changedOutputPixels = outHW;
                    st.gemmMacs = rc * (uint64_t)outHW;
                }
            }
            out[(size_t)s * nl + k] = st;
            total += st.gemmMacs;
        }
        macs[s] = total;
    }
}

// fp16 operand range: the MAXPOOL that writes a kind::f16 layer's fp16 shadow
// raises the plan's overflow flag when a value exceeds 65504. The flag is
// sticky until the next full evaluation (a change-based frame only rewrites
// changed pixels, so outputs computed from an inf operand persist), and every
// frame copies it into its stats block: each frame whose outputs may carry
// the overflow reports it, and the next frame is evaluated in full.
void Engine::check_f16_overflow(const unsigned long long* hs, int engine) {
    if (!any_f16_ || !hs[stats_words() - 1]) return;
    if (engine == CBX_ENGINE_CBINFER) has_history_ = false;
    throw Error(CBX_E_ARG,
                "fp16 operand overflow: an input of a kind::f16 layer exceeded 65504 in magnitude "
                "(create the context with CBX_PREC_TF32 to keep tf32 operands); the next frame is a full evaluation");
}

void Engine::read_stats(int engine, cbx_layer_stats* stats, uint64_t* macs) {
    if (engine != CBX_ENGINE_CBINFER && engine != CBX_ENGINE_BASELINE) throw Error(CBX_E_ARG, "bad engine");
    if (stats_pending_[engine]) {
        const int nl = (int)layers_.size();
        CBX_CUDA(cudaMemcpyAsync(h_stats_ + (size_t)engine * stats_words(), plan(engine).stats,
                                 sizeof(unsigned long long) * stats_words(), cudaMemcpyDeviceToHost, stream_));
        sync();
        finish_stats(plan(engine), last_full_[engine], engine);
        stats_pending_[engine] = false;
    } else {
        sync();
    }
    if (last_ovf_[engine]) check_f16_overflow(h_stats_ + (size_t)engine * stats_words(), engine);
    const int nl = (int)layers_.size();
    if (stats) std::memcpy(stats, last_stats_[engine].data(), sizeof(cbx_layer_stats) * S_ * nl);
    if (macs) std::memcpy(macs, last_macs_[engine].data(), sizeof(uint64_t) * S_);
}

void Engine::read_labels(int engine, uint16_t* labels) {
    Plan& p = plan(engine);
    CBX_CUDA(cudaMemcpyAsync(labels, p.labels, sizeof(uint16_t) * S_ * lh_ * lw_, cudaMemcpyDeviceToHost, stream_));
    sync();
}

const uint16_t* Engine::labels_device(int engine) { return plan(engine).labels; }

void Engine::load_layer(int layer, const float* K, const float* bias) {
    if (layer < 0 || layer >= (int)layers_.size() || !is_conv(layers_[layer].kind))
        throw Error(CBX_E_SPEC, "layer " + std::to_string(layer + 1) + " has no filters");
    if (!K || !bias) throw Error(CBX_E_ARG, "null weights");
    const cbx_geom& g = layers_[layer].geom;
    const size_t kd = (size_t)g.inChannels * g.kernelH * g.kernelW;
    for (size_t i = 0; i < kd * g.outChannels; ++i)
        if (!std::isfinite(K[i])) throw Error(CBX_E_IO, where(layer, layers_[layer].kind) + ": non-finite weight");
    for (int i = 0; i < g.outChannels; ++i)
        if (!std::isfinite(bias[i])) throw Error(CBX_E_IO, where(layer, layers_[layer].kind) + ": non-finite bias");
    CBX_CUDA(cudaSetDevice(device_));
    CBX_CUDA(cudaMemcpy(dK_[layer], K, kd * g.outChannels * sizeof(float), cudaMemcpyHostToDevice));
    CBX_CUDA(cudaMemcpy(dBias_[layer], bias, g.outChannels * sizeof(float), cudaMemcpyHostToDevice));
    hK_[layer].assign(K, K + kd * g.outChannels);
    hB_[layer].assign(bias, bias + g.outChannels);
    // recorded graphs may carry filters as kernel parameters: re-record
    if (cb_) cb_->dirty = true;
    if (base_) base_->dirty = true;
    if (tc_[layer]) tc_load_weights(*tc_[layer], K, stream_);
    if (layer == 0 && tc8_) tc_load_weights(*tc8_, K, stream_);
    if (layer == 0 && mpr8_) mpr_load_weights(*mpr8_, K, stream_);
    if (mpr_[layer]) mpr_load_weights(*mpr_[layer], K, stream_);
    CBX_CUDA(cudaStreamSynchronize(stream_));
}

void Engine::set_thresholds(const float* taus, int n) {
    if (n != (int)cb_layers_.size())
        throw Error(CBX_E_SPEC, "expected " + std::to_string(cb_layers_.size()) + " thresholds, got " + std::to_string(n));
    for (int k = 0; k < n; ++k)
        if (!(taus[k] >= 0.0f)) throw Error(CBX_E_SPEC, "negative threshold");
    for (int k = 0; k < n; ++k) layers_[cb_layers_[k]].threshold = taus[k];
    cb_->dirty = true;
}

void Engine::get_thresholds(float* taus, int n) const {
    for (int k = 0; k < n && k < (int)cb_layers_.size(); ++k) taus[k] = layers_[cb_layers_[k]].threshold;
}

void Engine::reset() { has_history_ = false; }

void Engine::get_activation(int engine, int layer, int s, float* out) {
    if (layer < 0 || layer >= (int)layers_.size() || s < 0 || s >= S_) throw Error(CBX_E_BOUNDS, "layer/stream out of range");
    if (layers_[layer].kind == CBX_CLASSIFY) throw Error(CBX_E_SPEC, "CLASSIFY produces labels, not an activation");
    Plan& p = plan(engine);
    if (p.fused_from >= 0 && layer + 1 > p.fused_from && layer + 1 < final_tensor())
        throw Error(CBX_E_SPEC, "layer " + std::to_string(layer + 1) +
                                    " output is not materialized (fused tail); set CBX_OPT_FUSE_TAIL = 0");
    const TensorView& t = p.T[layer + 1];
    const size_t n = (size_t)t.C * t.H * t.W;
    float* tmp = nullptr;
    CBX_CUDA(cudaMallocAsync(&tmp, n * sizeof(float), stream_));
    launch_hwc_to_chw(t, s, tmp, stream_);
    CBX_CUDA(cudaMemcpyAsync(out, tmp, n * sizeof(float), cudaMemcpyDeviceToHost, stream_));
    CBX_CUDA(cudaFreeAsync(tmp, stream_));
    sync();
}

// Input tensor of `layer` (planar CHW) after the last frame: prevInput of a
// CBCONV (cbconv.hpp:71). Layer 0 reads the frame the engine last consumed.
void Engine::get_input(int engine, int layer, int s, float* out) {
    if (layer < 0 || layer >= (int)layers_.size() || s < 0 || s >= S_) throw Error(CBX_E_BOUNDS, "layer/stream out of range");
    if (layer > 0) return get_activation(engine, layer - 1, s, out);
    if (engine != CBX_ENGINE_CBINFER) throw Error(CBX_E_ARG, "the dense engine keeps no frame history");
    if (!has_history_) throw Error(CBX_E_SPEC, "no frame has been evaluated since the last reset");
    const size_t n = (size_t)net_.inputChannels * net_.inputHeight * net_.inputWidth;
    if (hist_u8_) {  // 8-bit history: the frame the reference would hold, px / 255.0f
        float* tmp = nullptr;
        CBX_CUDA(cudaMallocAsync(&tmp, n * sizeof(float), stream_));
        launch_decode_u8(last_cb_frames8_[s], 1, net_.inputChannels, net_.inputHeight, net_.inputWidth, tmp, stream_);
        CBX_CUDA(cudaMemcpyAsync(out, tmp, n * sizeof(float), cudaMemcpyDeviceToHost, stream_));
        CBX_CUDA(cudaFreeAsync(tmp, stream_));
    } else {
        CBX_CUDA(cudaMemcpyAsync(out, last_cb_frames_[s], n * sizeof(float), cudaMemcpyDeviceToHost, stream_));
    }
    sync();
}

void Engine::get_trace(int cb, int s, uint8_t* detected, int32_t* updated, int64_t* n, int* first) {
    if (cb < 0 || cb >= (int)cb_layers_.size() || s < 0 || s >= S_) throw Error(CBX_E_BOUNDS, "trace index out of range");
    const int k = cb_layers_[cb];
    Plan& p = *cb_;
    const int H = dims_[6 * k + 1], W = dims_[6 * k + 2];
    const int64_t N = (int64_t)dims_[6 * k + 4] * dims_[6 * k + 5];
    sync();
    const bool full = last_full_[CBX_ENGINE_CBINFER];
    if (first) *first = full;
    if (detected) {
        if (full) {
            std::memset(detected, 0, (size_t)H * W);
        } else {
            uint8_t* tmp = nullptr;
            CBX_CUDA(cudaMallocAsync(&tmp, (size_t)H * W, stream_));
            launch_unpack_bits(p.chg[k], s, tmp, stream_);
            CBX_CUDA(cudaMemcpyAsync(detected, tmp, (size_t)H * W, cudaMemcpyDeviceToHost, stream_));
            CBX_CUDA(cudaFreeAsync(tmp, stream_));
            sync();
        }
    }
    if (full) {
        if (updated)
            for (int64_t i = 0; i < N; ++i) updated[i] = (int32_t)i;
        if (n) *n = N;
        return;
    }
    int total = 0;
    CBX_CUDA(cudaMemcpy(&total, p.cnt[k], sizeof(int), cudaMemcpyDeviceToHost));
    std::vector<int32_t> all(total);
    if (total) CBX_CUDA(cudaMemcpy(all.data(), p.idx[k], sizeof(int32_t) * total, cudaMemcpyDeviceToHost));
    // (the compaction writes each tile's ascending run where its atomic
    // landed: sort for the reference's extract_indexes order)
    std::sort(all.begin(), all.end(), [](int32_t a, int32_t b) { return (uint32_t)a < (uint32_t)b; });
    const int R = list_group(k, hist_u8_);
    const int Wo = dims_[6 * k + 5], Gw = (Wo + R - 1) / R;
    const int64_t Ng = (int64_t)dims_[6 * k + 4] * Gw;
    int64_t m = 0;
    for (int32_t g : all) {
        if (R == 1) {
            if (g >= s * N && g < (s + 1) * N) {
                if (updated) updated[m] = (int32_t)(g - s * N);
                ++m;
            }
            continue;
        }
        // group entry (gid << 4 | mask): its set pixels, ascending
        const int64_t gid = (uint32_t)g >> 4;
        if (gid < s * Ng || gid >= (s + 1) * Ng) continue;
        const int64_t rem = gid - s * Ng;
        const int64_t y = rem / Gw, x0 = (rem % Gw) * R;
        for (int j = 0; j < R; ++j)
            if ((g >> j) & 1) {
                if (updated) updated[m] = (int32_t)(y * Wo + x0 + j);
                ++m;
            }
    }
    if (n) *n = m;
}

}  // namespace cbx

namespace cbx {

void Engine::mark(const char* name, int layer) {
    if (tmarks_) {  // graph capture with CBX_OPT_STEP_TIMES: an event-record node
        if (tmarks_used_ >= tmarks_->size()) throw Error(CBX_E_ARG, "too many step-time marks");
        ProfMark& pm = (*tmarks_)[tmarks_used_++];
        pm.name = name;
        pm.layer = layer;
        // an event-record node (a plain cudaEventRecord under capture only
        // becomes a graph edge and is never timestamped)
        CBX_CUDA(cudaEventRecordWithFlags(pm.ev, stream_, cudaEventRecordExternal));
        return;
    }
    if (!prof_) return;
    cudaEvent_t e;
    CBX_CUDA(cudaEventCreate(&e));
    CBX_CUDA(cudaEventRecord(e, stream_));
    prof_->push_back(ProfMark{name, layer, e});
}

// One forward without the graph, each kernel bracketed by CUDA events on the
// context stream (the stream every kernel is launched on). Advances the state
// exactly like forward_device.
void Engine::profile(int engine, const float* const* frames_dev, const uint8_t* const* frames_u8,
                     std::vector<cbx_kernel_time>& out) {
    const bool full = prepare_frame(engine, frames_dev, frames_u8);
    Plan& p = plan(engine);
    std::vector<ProfMark> marks;
    prof_ = &marks;
    try {
        mark("start", -1);
        record(p, full);
    } catch (...) {
        prof_ = nullptr;
        throw;
    }
    prof_ = nullptr;
    const int nl = (int)layers_.size();
    CBX_CUDA(cudaMemcpyAsync(h_stats_ + (size_t)engine * stats_words(), p.stats, sizeof(unsigned long long) * stats_words(),
                             cudaMemcpyDeviceToHost, stream_));
    sync();
    out.clear();
    for (size_t i = 1; i < marks.size(); ++i) {
        float ms = 0;
        CBX_CUDA(cudaEventElapsedTime(&ms, marks[i - 1].ev, marks[i].ev));
        cbx_kernel_time t{};
        std::snprintf(t.name, sizeof(t.name), "%s", marks[i].name.c_str());
        t.layer = marks[i].layer;
        t.ms = ms;
        out.push_back(t);
    }
    for (auto& m : marks) cudaEventDestroy(m.ev);
    last_full_[engine] = full;
    finish_stats(p, full, engine);  // h_stats_ was filled above
    stats_pending_[engine] = false;
    frame_done(engine);
}

}  // namespace cbx

namespace cbx {

// Index of the tensor classified into labels (input of CLASSIFY, or the last
// layer's output when the network has no CLASSIFY).
int Engine::final_tensor() const {
    const int nl = (int)layers_.size();
    return layers_.back().kind == CBX_CLASSIFY ? nl - 1 : nl;
}

// Last layer of a per-pixel tail that can run in the epilogue of tcgen05 conv
// k: 1x1 CONVs (<= kTailMaxC outputs) and RELUs up to the end of the network
// (optionally closed by CLASSIFY), first op a CONV. -1 when not fusable.
int Engine::tail_end(int k) const {
    const int nl = (int)layers_.size();
    if (!fuse_tail_ || k + 1 >= nl) return -1;
    const auto& first = layers_[k + 1];
    if (first.kind != CBX_CONV || !identity_geom(first.geom) || first.geom.outChannels > kTailMaxC) return -1;
    int ops = 0;
    for (int j = k + 1; j < nl; ++j) {
        const auto& l = layers_[j];
        if (l.kind == CBX_CLASSIFY) return j == nl - 1 ? j : -1;
        if (l.kind == CBX_RELU) {
            ++ops;
        } else if (l.kind == CBX_CONV && identity_geom(l.geom) && l.geom.outChannels <= kTailMaxC) {
            ++ops;
        } else {
            return -1;
        }
        if (ops > kTailMaxOps) return -1;
    }
    return nl - 1;
}

// cbench analyze-prop (tools/cbench.cpp:242-302) on the device: for every
// CBCONV k >= 1, the previous CBCONV's updated set (its U mask of the last
// frame) pushed through the layers in between (MAXPOOL: pooling support,
// CONV: its receptive field, RELU: unchanged) and dilated by layer k's
// geometry -- worst_case_propagation / dilate_changes (cbconv.cpp:73-97) --
// counted per stream. worst[s * (ncb - 1) + (k - 1)].
void Engine::worst_case_counts(int64_t* worst) {
    const int ncb = (int)cb_layers_.size();
    if (ncb < 2) throw Error(CBX_E_SPEC, "analyze-prop needs at least two CBCONV layers");
    if (!has_history_ || last_full_[CBX_ENGINE_CBINFER])
        throw Error(CBX_E_ARG, "analyze-prop: the last change-based frame was a full evaluation (no propagation)");
    if (!worst) throw Error(CBX_E_ARG, "null output");
    CBX_CUDA(cudaSetDevice(device_));
    Plan& p = *cb_;
    std::vector<void*> tmp;
    auto mask = [&](int H, int W) {
        const int wpr = (W + 31) / 32;
        BitMask m{nullptr, H, W, wpr, round_up((int64_t)H * wpr, 2048)};
        m.d = dmalloc<uint32_t>((size_t)(m.stride * S_));
        tmp.push_back(m.d);
        return m;
    };
    unsigned long long* cnt = dmalloc<unsigned long long>((size_t)S_ * (ncb - 1));
    tmp.push_back(cnt);
    try {
        CBX_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * S_ * (ncb - 1), stream_));
        for (int k = 1; k < ncb; ++k) {
            const int prev = cb_layers_[k - 1], next = cb_layers_[k];
            BitMask wave = p.U[prev];
            for (int li = prev + 1; li < next; ++li) {
                const auto& l = layers_[li];
                const int Ho = dims_[6 * li + 4], Wo = dims_[6 * li + 5];
                if (l.kind == CBX_MAXPOOL) {
                    BitMask o = mask(Ho, Wo);
                    launch_dilate_bits(wave, o, S_, l.window, l.window, l.stride, l.stride, 0, 0, stream_);
                    wave = o;
                } else if (l.kind == CBX_CONV) {
                    const cbx_geom& g = l.geom;
                    BitMask o = mask(Ho, Wo);
                    launch_dilate_bits(wave, o, S_, g.kernelH, g.kernelW, g.strideH, g.strideW, g.padH, g.padW, stream_);
                    wave = o;
                }
            }
            const cbx_geom& g = layers_[next].geom;
            BitMask w = mask(dims_[6 * next + 4], dims_[6 * next + 5]);
            launch_dilate_bits(wave, w, S_, g.kernelH, g.kernelW, g.strideH, g.strideW, g.padH, g.padW, stream_);
            for (int s = 0; s < S_; ++s) {
                BitMask one = w;
                one.d = w.d + (int64_t)s * w.stride;
                launch_popcount_bits(one, 1, cnt + (size_t)s * (ncb - 1) + (k - 1), stream_);
            }
        }
        std::vector<unsigned long long> h((size_t)S_ * (ncb - 1));
        CBX_CUDA(cudaMemcpyAsync(h.data(), cnt, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost, stream_));
        CBX_CUDA(cudaStreamSynchronize(stream_));
        for (size_t i = 0; i < h.size(); ++i) worst[i] = (int64_t)h[i];
    } catch (...) {
        for (void* q : tmp) cudaFree(q);
        throw;
    }
    for (void* q : tmp) cudaFree(q);
}

// StepTimes (cbconv.hpp:44-52) of the last frame launched as a graph, per
// layer: [nl][5] = detect, extract, generate, multiply, update (ns). Mapping
// of the fused B200 kernels onto the reference's five steps: detect = the
// frame detection kernel (first CBCONV; a later CBCONV's detection is fused
// into its producer's compare-before-write), extract = dilation + index
// compaction (one kernel), multiply = the gathered convolution, which also
// generates the patches (producer warps) and updates the output (epilogue
// scatter), so generate and update are 0. Every stream of the engine shares
// the same kernels, hence the same times.
void Engine::read_step_times(int64_t* out) {
    const int nl = (int)layers_.size();
    std::memset(out, 0, sizeof(int64_t) * 5 * nl);
    if (!last_tm_ || last_tm_->size() < 2) return;
    sync();
    const auto& v = *last_tm_;
    for (size_t i = 1; i < v.size(); ++i) {
        float ms = 0;
        CBX_CUDA(cudaEventElapsedTime(&ms, v[i - 1].ev, v[i].ev));
        const int64_t ns = (int64_t)((double)ms * 1e6);
        const std::string& n = v[i].name;
        const int k = v[i].layer;
        if (k < 0 || k >= nl) continue;
        int slot = -1;
        if (n == "detect") slot = 0;
        else if (n == "dilate_compact" || n == "compact" || n == "dilate") slot = 1;
        else if (n.rfind("conv", 0) == 0) slot = 3;
        if (slot >= 0) out[5 * k + slot] += ns;
    }
}

void Engine::set_option(int option, int value) {
    if (option == CBX_OPT_STEP_TIMES) {
        step_times_ = value != 0;
        cb_->dirty = true;
        if (base_) base_->dirty = true;
        last_tm_ = nullptr;
        return;
    }
    if (option == CBX_OPT_TC_PAIR) {
        if (value < -1 || value > 1) throw Error(CBX_E_ARG, "CBX_OPT_TC_PAIR takes -1, 0 or 1");
        bool relayout = false;
        // rebuild every tcgen05 layer with the requested CTA grouping; the
        // filters come back from the device copy in the reference layout
        for (int k = 0; k < (int)layers_.size(); ++k) {
            if (!tc_[k]) continue;
            const cbx_geom& g = layers_[k].geom;
            const int te = tail_end(k);
            const int c1 = te > 0 ? layers_[k + 1].geom.outChannels : 0;
            const int tail_floats = te > 0 ? (c1 <= 8 ? 8 : 16) * g.outChannels : 0;
            std::vector<float> K((size_t)g.outChannels * g.inChannels * g.kernelH * g.kernelW);
            CBX_CUDA(cudaMemcpy(K.data(), dK_[k], K.size() * sizeof(float), cudaMemcpyDeviceToHost));
            const int cp_before = tc_input_cp(*tc_[k]);
            tc_[k] = make_tc_layer(g, tail_floats, value, tc_is_f16(*tc_[k]), false,
                                   tail_floats ? 1 : group_width_for(g), pack_f16(k));
            tc_load_weights(*tc_[k], K.data(), stream_);
            if (tc_input_cp(*tc_[k]) != cp_before) relayout = true;
        }
        if (relayout) {
            // the fp16 shadow layout changed (packing depends on the layer shape):
            // new plans, and the next frame is a full evaluation
            CBX_CUDA(cudaStreamSynchronize(stream_));
            cb_.reset(new Plan);
            build_plan(*cb_, false);
            base_.reset();
            has_history_ = false;
        }
    } else if (option == CBX_OPT_FUSE_TAIL) {
        fuse_tail_ = value != 0;
    } else if (option == CBX_OPT_U8_NATIVE) {
        // switching paths keeps results within the tolerance, not bitwise:
        // the next frame is a full evaluation
        if (u8_opt_ != (value != 0)) has_history_ = false;
        u8_opt_ = value != 0;
        return;
    } else {
        throw Error(CBX_E_ARG, "unknown option");
    }
    cb_->dirty = true;
    if (base_) base_->dirty = true;
}

}  // namespace cbx
