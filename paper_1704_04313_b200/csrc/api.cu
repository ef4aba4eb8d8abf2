// api.cu -- the extern "C" boundary declared in include/cbx.h.
//
// Every entry point converts C++ exceptions into cbx_status codes (the
// reference's exception hierarchy, core/include/cbinfer/error.hpp:9-42) and
// records the message for cbx_last_error.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/cbx.h"
#include "context.hpp"
#include "engine.hpp"
#include "kernels.hpp"

struct cbx_ctx {
    cbx::Context* eng = nullptr;
    std::string err;
};

namespace {

thread_local std::string g_err;

template <class F>
int guarded(cbx_ctx* ctx, F&& f) {
    try {
        f();
        return CBX_OK;
    } catch (const cbx::Error& e) {
        (ctx ? ctx->err : g_err) = e.what();
        return e.code;
    } catch (const std::bad_alloc& e) {
        (ctx ? ctx->err : g_err) = "out of host memory";
        return CBX_E_CUDA;
    } catch (const std::exception& e) {
        (ctx ? ctx->err : g_err) = e.what();
        return CBX_E_CUDA;
    }
}

cbx::Context& E(cbx_ctx* c) {
    if (!c || !c->eng) throw cbx::Error(CBX_E_ARG, "null context");
    return *c->eng;
}

// std::mt19937, the engine the reference seeds in synth.cpp / testutil.hpp.
struct Mt19937 {
    uint32_t st[624];
    int pos;
    explicit Mt19937(uint32_t seed) {
        st[0] = seed;
        for (int i = 1; i < 624; ++i) st[i] = 1812433253u * (st[i - 1] ^ (st[i - 1] >> 30)) + (uint32_t)i;
        pos = 624;
    }
    uint32_t operator()() {
        if (pos >= 624) {
            for (int i = 0; i < 624; ++i) {
                const uint32_t y = (st[i] & 0x80000000u) | (st[(i + 1) % 624] & 0x7fffffffu);
                st[i] = st[(i + 397) % 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
            }
            pos = 0;
        }
        uint32_t y = st[pos++];
        y ^= y >> 11;
        y ^= (y << 7) & 0x9d2c5680u;
        y ^= (y << 15) & 0xefc60000u;
        y ^= y >> 18;
        return y;
    }
    float unit() { return (float)((*this)() >> 8) * (1.0f / 16777216.0f); }  // synth.cpp:18-20
};

// sprite placement, synth.cpp:33-58
void sprite_rect(const cbx_synth_cfg& cfg, int s, int f, int r[4]) {
    const cbx_sprite& sp = cfg.sprites[s];
    if (sp.size > cfg.height || sp.size > cfg.width) throw cbx::Error(CBX_E_SPEC, "sprite larger than frame");
    static const int dirs[8][2] = {{-1, -1}, {-1, 0}, {-1, 1}, {0, -1}, {0, 1}, {1, -1}, {1, 0}, {1, 1}};
    Mt19937 rng(cfg.seed ^ (0x9e3779b9u * (uint32_t)(s + 1)));
    const int sy = (int)(rng() % (uint32_t)(cfg.height - sp.size + 1));
    const int sx = (int)(rng() % (uint32_t)(cfg.width - sp.size + 1));
    const int* d = dirs[rng() % 8];
    const int travel = sp.velocity * f;
    int y = sy + d[0] * travel, x = sx + d[1] * travel;
    y = std::min(std::max(y, 0), cfg.height - sp.size);
    x = std::min(std::max(x, 0), cfg.width - sp.size);
    r[0] = y;
    r[1] = x;
    r[2] = y + sp.size;
    r[3] = x + sp.size;
}

}  // namespace

extern "C" {

CBX_API const char* cbx_last_error(const cbx_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }
CBX_API const char* cbx_version(void) { return "cbx 0.1 (sm_100a)"; }

CBX_API int cbx_chain_dims(const cbx_net_desc* net, cbx_layer_desc* layers_out, int* dims) {
    return guarded(nullptr, [&] {
        if (!net) throw cbx::Error(CBX_E_ARG, "null net");
        std::vector<cbx_layer_desc> L;
        auto d = cbx::chain_dims(*net, L);
        if (layers_out) std::memcpy(layers_out, L.data(), sizeof(cbx_layer_desc) * L.size());
        if (dims) std::memcpy(dims, d.data(), sizeof(int) * d.size());
    });
}

CBX_API int cbx_create_ex(const cbx_net_desc* net, int device, int num_streams, int precision, int lanes,
                          cbx_ctx** out) {
    return guarded(nullptr, [&] {
        if (!net || !out) throw cbx::Error(CBX_E_ARG, "null argument");
        *out = nullptr;
        if (lanes <= 0) lanes = num_streams >= 2 ? 2 : 1;
        auto* c = new cbx_ctx;
        try {
            c->eng = new cbx::Context(*net, device, num_streams, precision, lanes);
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

CBX_API int cbx_create(const cbx_net_desc* net, int device, int num_streams, int precision, cbx_ctx** out) {
    return cbx_create_ex(net, device, num_streams, precision, 0, out);
}

CBX_API int cbx_num_lanes(const cbx_ctx* ctx) { return ctx && ctx->eng ? ctx->eng->lanes() : -1; }
CBX_API int cbx_layer_operands(const cbx_ctx* ctx, int layer) {
    return ctx && ctx->eng ? ctx->eng->lane(0).layer_operands(layer) : -1;
}

CBX_API void cbx_destroy(cbx_ctx* ctx) {
    if (!ctx) return;
    delete ctx->eng;
    delete ctx;
}

CBX_API int cbx_load_layer(cbx_ctx* ctx, int layer, const float* K, const float* bias) {
    return guarded(ctx, [&] { E(ctx).load_layer(layer, K, bias); });
}

CBX_API int cbx_set_thresholds(cbx_ctx* ctx, const float* taus, int n) {
    return guarded(ctx, [&] { E(ctx).set_thresholds(taus, n); });
}

CBX_API int cbx_get_thresholds(const cbx_ctx* ctx, float* taus, int n) {
    return guarded(const_cast<cbx_ctx*>(ctx), [&] { E(const_cast<cbx_ctx*>(ctx)).get_thresholds(taus, n); });
}

CBX_API int cbx_set_option(cbx_ctx* ctx, int option, int value) {
    return guarded(ctx, [&] { E(ctx).set_option(option, value); });
}

CBX_API int cbx_reset(cbx_ctx* ctx) {
    return guarded(ctx, [&] { E(ctx).reset(); });
}

CBX_API int cbx_forward(cbx_ctx* ctx, int engine, const float* frames, uint16_t* labels,
                        cbx_layer_stats* stats, uint64_t* macs) {
    return guarded(ctx, [&] { E(ctx).forward_host(engine, frames, labels, stats, macs); });
}

CBX_API int cbx_forward_device(cbx_ctx* ctx, int engine, const float* const* frames_dev) {
    return guarded(ctx, [&] { E(ctx).forward_device(engine, frames_dev); });
}

CBX_API int cbx_forward_device_u8(cbx_ctx* ctx, int engine, const uint8_t* const* frames_dev) {
    return guarded(ctx, [&] { E(ctx).forward_device_u8(engine, frames_dev); });
}

CBX_API int cbx_submit(cbx_ctx* ctx, int engine, const float* frames, uint16_t* labels, int64_t* ticket) {
    return guarded(ctx, [&] {
        if (!ticket) throw cbx::Error(CBX_E_ARG, "null ticket");
        *ticket = E(ctx).submit(engine, frames, labels);
    });
}

CBX_API int cbx_forward_u8(cbx_ctx* ctx, int engine, const uint8_t* frames, uint16_t* labels, cbx_layer_stats* stats,
                           uint64_t* macs) {
    return guarded(ctx, [&] { E(ctx).forward_host_u8(engine, frames, labels, stats, macs); });
}

CBX_API int cbx_submit_u8(cbx_ctx* ctx, int engine, const uint8_t* frames, uint16_t* labels, int64_t* ticket) {
    return guarded(ctx, [&] {
        const int64_t t = E(ctx).submit_u8(engine, frames, labels);
        if (ticket) *ticket = t;
    });
}

CBX_API int cbx_wait(cbx_ctx* ctx, int64_t ticket, cbx_layer_stats* stats, uint64_t* macs) {
    return guarded(ctx, [&] { E(ctx).wait(ticket, stats, macs); });
}

CBX_API int cbx_worst_case_counts(cbx_ctx* ctx, int64_t* worst) {
    return guarded(ctx, [&] { E(ctx).worst_case_counts(worst); });
}

CBX_API int cbx_sync(cbx_ctx* ctx) {
    return guarded(ctx, [&] { E(ctx).sync(); });
}

CBX_API int cbx_read_labels(cbx_ctx* ctx, int engine, uint16_t* labels) {
    return guarded(ctx, [&] {
        if (!labels) throw cbx::Error(CBX_E_ARG, "null labels");
        E(ctx).read_labels(engine, labels);
    });
}

CBX_API int cbx_read_stats(cbx_ctx* ctx, int engine, cbx_layer_stats* stats, uint64_t* macs) {
    return guarded(ctx, [&] { E(ctx).read_stats(engine, stats, macs); });
}

CBX_API int cbx_labels_device(cbx_ctx* ctx, int engine, const uint16_t** labels_dev) {
    return guarded(ctx, [&] { *labels_dev = E(ctx).labels_device(engine); });
}

CBX_API void* cbx_stream(cbx_ctx* ctx) { return ctx && ctx->eng ? (void*)ctx->eng->stream() : nullptr; }

CBX_API int cbx_last_launch_count(const cbx_ctx* ctx) {
    return ctx && ctx->eng ? ctx->eng->last_launch_count() : -1;
}

CBX_API int cbx_get_activation(cbx_ctx* ctx, int engine, int layer, int s, float* out) {
    return guarded(ctx, [&] {
        if (!out) throw cbx::Error(CBX_E_ARG, "null out");
        E(ctx).get_activation(engine, layer, s, out);
    });
}

CBX_API int cbx_get_trace(cbx_ctx* ctx, int cb, int s, uint8_t* detected, int32_t* updated, int64_t* n,
                          int* first) {
    return guarded(ctx, [&] { E(ctx).get_trace(cb, s, detected, updated, n, first); });
}

CBX_API int cbx_profile_forward(cbx_ctx* ctx, int engine, const float* const* frames_dev, cbx_kernel_time* out,
                                int cap, int* n) {
    return guarded(ctx, [&] {
        if (!frames_dev) throw cbx::Error(CBX_E_ARG, "frames is null");
        std::vector<cbx_kernel_time> v;
        E(ctx).profile(engine, frames_dev, nullptr, v);
        const int m = std::min<int>((int)v.size(), cap);
        if (out && m > 0) std::memcpy(out, v.data(), sizeof(cbx_kernel_time) * m);
        if (n) *n = (int)v.size();
    });
}

CBX_API int cbx_profile_forward_u8(cbx_ctx* ctx, int engine, const uint8_t* const* frames_dev, cbx_kernel_time* out,
                                   int cap, int* n) {
    return guarded(ctx, [&] {
        if (!frames_dev) throw cbx::Error(CBX_E_ARG, "frames is null");
        std::vector<cbx_kernel_time> v;
        E(ctx).profile(engine, nullptr, frames_dev, v);
        const int m = std::min<int>((int)v.size(), cap);
        if (out && m > 0) std::memcpy(out, v.data(), sizeof(cbx_kernel_time) * m);
        if (n) *n = (int)v.size();
    });
}

CBX_API int cbx_get_input(cbx_ctx* ctx, int engine, int layer, int s, float* out) {
    return guarded(ctx, [&] {
        if (!out) throw cbx::Error(CBX_E_ARG, "null output");
        E(ctx).get_input(engine, layer, s, out);
    });
}

CBX_API int cbx_has_history(const cbx_ctx* ctx) {
    return ctx && ctx->eng ? (ctx->eng->has_history() ? 1 : 0) : -1;
}

CBX_API int cbx_read_step_times(cbx_ctx* ctx, int64_t* nanos) {
    return guarded(ctx, [&] { E(ctx).read_step_times(nanos); });
}

// ---- op level ---------------------------------------------------------
CBX_API int cbx_op_detect(const float* cur, const float* prev, int C, int H, int W, float tau, uint8_t* mask,
                          unsigned long long* count_dev, void* stream) {
    return guarded(nullptr, [&] {
        if (!cur || !prev || !mask) throw cbx::Error(CBX_E_ARG, "null pointer");
        if (C < 1 || H < 1 || W < 1) throw cbx::Error(CBX_E_SHAPE, "detect_changes: empty frame");
        cudaStream_t st = (cudaStream_t)stream;
        const float** tbl = nullptr;
        CBX_CUDA(cudaMallocAsync((void**)&tbl, 2 * sizeof(float*), st));
        const float* h[2] = {cur, prev};
        CBX_CUDA(cudaMemcpyAsync(tbl, h, sizeof(h), cudaMemcpyHostToDevice, st));
        cbx::MaskView m{mask, H, W, (int64_t)H * W};
        // the op-level mask is dense (stride H*W); use the scalar path when W*H % 4 != 0
        cbx::launch_detect_planar(tbl, tbl + 1, 1, C, H, W, tau, 0, m, count_dev, 2, st);
        CBX_CUDA(cudaFreeAsync(tbl, st));
        CBX_CUDA(cudaGetLastError());
    });
}

CBX_API int cbx_op_dilate(const uint8_t* mask, int H, int W, const cbx_geom* g, uint8_t* out, void* stream) {
    return guarded(nullptr, [&] {
        if (!mask || !out || !g) throw cbx::Error(CBX_E_ARG, "null pointer");
        if (g->kernelH < 1 || g->kernelW < 1 || g->strideH < 1 || g->strideW < 1 || g->padH < 0 || g->padW < 0)
            throw cbx::Error(CBX_E_GEOMETRY, "invalid convolution geometry");
        if (H + 2 * g->padH < g->kernelH || W + 2 * g->padW < g->kernelW)
            throw cbx::Error(CBX_E_GEOMETRY, "convolution output would be empty");
        const int Ho = (H + 2 * g->padH - g->kernelH) / g->strideH + 1;
        const int Wo = (W + 2 * g->padW - g->kernelW) / g->strideW + 1;
        cbx::launch_dilate(cbx::MaskView{const_cast<uint8_t*>(mask), H, W, (int64_t)H * W},
                           cbx::MaskView{out, Ho, Wo, (int64_t)Ho * Wo}, 1, g->kernelH, g->kernelW, g->strideH,
                           g->strideW, g->padH, g->padW, (cudaStream_t)stream);
        CBX_CUDA(cudaGetLastError());
    });
}

CBX_API size_t cbx_op_extract_workspace(int64_t n) { return cbx::compact_workspace_bytes(1, n); }

CBX_API int cbx_op_extract(const uint8_t* mask, int64_t n, int32_t* idx, int* count_dev, void* workspace,
                           void* stream) {
    return guarded(nullptr, [&] {
        if (!mask || !idx || !count_dev || !workspace) throw cbx::Error(CBX_E_ARG, "null pointer");
        if (reinterpret_cast<uintptr_t>(mask) % 16) throw cbx::Error(CBX_E_ARG, "mask must be 16-byte aligned");
        if (n <= 0) {
            CBX_CUDA(cudaMemsetAsync(count_dev, 0, sizeof(int), (cudaStream_t)stream));
            return;
        }
        cbx::launch_compact(cbx::MaskView{const_cast<uint8_t*>(mask), 1, (int)n, cbx::round_up(n, 16)}, 1, idx,
                            count_dev, workspace, nullptr, 2, (cudaStream_t)stream);
        CBX_CUDA(cudaGetLastError());
    });
}

CBX_API int cbx_op_maxpool(const float* in, int C, int H, int W, int window, int stride, float* out, void* stream) {
    return guarded(nullptr, [&] {
        if (window < 1 || stride < 1) throw cbx::Error(CBX_E_GEOMETRY, "maxpool: window and stride must be positive");
        if (window > H || window > W) throw cbx::Error(CBX_E_GEOMETRY, "maxpool: window exceeds input");
        cudaStream_t st = (cudaStream_t)stream;
        const int Ho = (H - window) / stride + 1, Wo = (W - window) / stride + 1;
        const int Cp = (int)cbx::round_up(C, 4);
        cbx::TensorView ti{nullptr, C, H, W, Cp, H, W, 0, 0, (int64_t)H * W * Cp};
        cbx::TensorView to{nullptr, C, Ho, Wo, Cp, Ho, Wo, 0, 0, (int64_t)Ho * Wo * Cp};
        CBX_CUDA(cudaMallocAsync((void**)&ti.d, ti.ss * 4, st));
        CBX_CUDA(cudaMallocAsync((void**)&to.d, to.ss * 4, st));
        CBX_CUDA(cudaMemsetAsync(ti.d, 0, ti.ss * 4, st));
        cbx::launch_chw_to_hwc(in, ti, 0, st);
        cbx::PoolArgs a{};
        a.in = ti;
        a.out = to;
        a.window = window;
        a.stride = stride;
        a.S = 1;
        cbx::launch_pool(a, st);
        cbx::launch_hwc_to_chw(to, 0, out, st);
        CBX_CUDA(cudaFreeAsync(ti.d, st));
        CBX_CUDA(cudaFreeAsync(to.d, st));
        CBX_CUDA(cudaGetLastError());
    });
}

CBX_API int cbx_op_argmax(const float* t, int C, int H, int W, uint16_t* labels, void* stream) {
    return guarded(nullptr, [&] {
        cudaStream_t st = (cudaStream_t)stream;
        const int Cp = (int)cbx::round_up(C, 4);
        cbx::TensorView ti{nullptr, C, H, W, Cp, H, W, 0, 0, (int64_t)H * W * Cp};
        CBX_CUDA(cudaMallocAsync((void**)&ti.d, ti.ss * 4, st));
        CBX_CUDA(cudaMemsetAsync(ti.d, 0, ti.ss * 4, st));
        cbx::launch_chw_to_hwc(t, ti, 0, st);
        cbx::PointArgs a{};
        a.in = ti;
        a.labels = labels;
        a.S = 1;
        cbx::launch_classify(a, st);
        CBX_CUDA(cudaFreeAsync(ti.d, st));
        CBX_CUDA(cudaGetLastError());
    });
}

CBX_API int cbx_op_gen_x(const float* in, int C, int H, int W, const cbx_geom* g, const int32_t* idx,
                         int64_t n, float* X, void* stream) {
    return guarded(nullptr, [&] {
        if (!in || !g || (n > 0 && !X)) throw cbx::Error(CBX_E_ARG, "null pointer");
        if (C != g->inChannels) throw cbx::Error(CBX_E_SHAPE, "gen_x_reduced: channel count mismatch");
        if (g->kernelH < 1 || g->kernelW < 1 || g->strideH < 1 || g->strideW < 1 || g->padH < 0 || g->padW < 0 ||
            H + 2 * g->padH < g->kernelH || W + 2 * g->padW < g->kernelW)
            throw cbx::Error(CBX_E_GEOMETRY, "invalid convolution geometry or empty output");
        cbx::launch_gen_x(in, C, H, W, g->kernelH, g->kernelW, g->strideH, g->strideW, g->padH, g->padW, idx, n, X,
                          (cudaStream_t)stream);
        CBX_CUDA(cudaGetLastError());
    });
}

CBX_API int cbx_op_gemm(const float* K, const float* bias, int rows, int cols, const float* X, int64_t n, float* Y,
                        void* stream) {
    return guarded(nullptr, [&] {
        if (rows < 0 || cols < 0 || n < 0) throw cbx::Error(CBX_E_SHAPE, "gemm: negative dimension");
        if (rows && n && (!K || !bias || !Y || (cols && !X))) throw cbx::Error(CBX_E_ARG, "null pointer");
        cbx::launch_gemm_exact(K, bias, rows, cols, X, n, Y, (cudaStream_t)stream);
        CBX_CUDA(cudaGetLastError());
    });
}

CBX_API int cbx_op_scatter(float* out, int C, int H, int W, const float* Y, const int32_t* idx, int64_t n, int relu,
                           void* stream) {
    return guarded(nullptr, [&] {
        if (n > 0 && (!out || !Y || !idx)) throw cbx::Error(CBX_E_ARG, "null pointer");
        cbx::launch_scatter(out, C, (int64_t)H * W, Y, idx, n, relu, (cudaStream_t)stream);
        CBX_CUDA(cudaGetLastError());
    });
}

CBX_API int cbx_op_decode_u8(const uint8_t* in, int S, int C, int H, int W, float* out, void* stream) {
    return guarded(nullptr, [&] {
        if (!in || !out) throw cbx::Error(CBX_E_ARG, "null pointer");
        if (S < 1 || C < 1 || H < 1 || W < 1) throw cbx::Error(CBX_E_SHAPE, "decode_u8: empty frame");
        cbx::launch_decode_u8(in, S, C, H, W, out, (cudaStream_t)stream);
        CBX_CUDA(cudaGetLastError());
    });
}

CBX_API int cbx_op_relu(const float* in, int C, int H, int W, float* out, void* stream) {
    return guarded(nullptr, [&] {
        if (!in || !out) throw cbx::Error(CBX_E_ARG, "null pointer");
        if (C < 1 || H < 1 || W < 1) throw cbx::Error(CBX_E_SHAPE, "relu: empty tensor");
        cudaStream_t st = (cudaStream_t)stream;
        const int Cp = (int)cbx::round_up(C, 4);
        cbx::TensorView ti{nullptr, C, H, W, Cp, H, W, 0, 0, (int64_t)H * W * Cp};
        cbx::TensorView to = ti;
        CBX_CUDA(cudaMallocAsync((void**)&ti.d, ti.ss * 4, st));
        CBX_CUDA(cudaMallocAsync((void**)&to.d, to.ss * 4, st));
        CBX_CUDA(cudaMemsetAsync(ti.d, 0, ti.ss * 4, st));
        cbx::launch_chw_to_hwc(in, ti, 0, st);
        cbx::PointArgs a{};
        a.in = ti;
        a.out = to;
        a.S = 1;
        cbx::launch_relu(a, st);
        cbx::launch_hwc_to_chw(to, 0, out, st);
        CBX_CUDA(cudaFreeAsync(ti.d, st));
        CBX_CUDA(cudaFreeAsync(to.d, st));
        CBX_CUDA(cudaGetLastError());
    });
}

CBX_API int cbx_op_cbconv_update(const float* in, int C, int H, int W, const float* K, const float* bias,
                                 const cbx_geom* g, const int32_t* idx, int n, int fuseRelu, float* out,
                                 void* stream) {
    return guarded(nullptr, [&] {
        if (!g || !in || !K || !bias || !out) throw cbx::Error(CBX_E_ARG, "null pointer");
        if (C != g->inChannels) throw cbx::Error(CBX_E_SHAPE, "gen_x_reduced: channel count mismatch");
        if (H + 2 * g->padH < g->kernelH || W + 2 * g->padW < g->kernelW)
            throw cbx::Error(CBX_E_GEOMETRY, "convolution output would be empty");
        cudaStream_t st = (cudaStream_t)stream;
        const int Ho = (H + 2 * g->padH - g->kernelH) / g->strideH + 1;
        const int Wo = (W + 2 * g->padW - g->kernelW) / g->strideW + 1;
        const int O = g->outChannels;
        const int Cp = (int)cbx::round_up(O, 4);
        const float** tbl = nullptr;
        cbx::TensorView to{nullptr, O, Ho, Wo, Cp, Ho, Wo, 0, 0, (int64_t)Ho * Wo * Cp};
        int* cnt = nullptr;
        CBX_CUDA(cudaMallocAsync((void**)&tbl, sizeof(float*), st));
        CBX_CUDA(cudaMemcpyAsync(tbl, &in, sizeof(float*), cudaMemcpyHostToDevice, st));
        CBX_CUDA(cudaMallocAsync((void**)&to.d, to.ss * 4, st));
        CBX_CUDA(cudaMallocAsync((void**)&cnt, sizeof(int), st));
        CBX_CUDA(cudaMemcpyAsync(cnt, &n, sizeof(int), cudaMemcpyHostToDevice, st));
        CBX_CUDA(cudaMemsetAsync(to.d, 0, to.ss * 4, st));
        cbx::launch_chw_to_hwc(out, to, 0, st);
        cbx::ConvArgs a{};
        a.in = cbx::TensorView{nullptr, C, H, W, C, H, W, 0, 0, (int64_t)C * H * W};
        a.in_ptrs = tbl;
        a.out = to;
        a.K = K;
        a.bias = bias;
        a.kh = g->kernelH;
        a.kw = g->kernelW;
        a.sh = g->strideH;
        a.sw = g->strideW;
        a.ph = g->padH;
        a.pw = g->padW;
        a.idx = idx;
        a.count = cnt;
        a.full_count = (int64_t)Ho * Wo;
        a.relu = fuseRelu;
        a.S = 1;
        cbx::launch_conv_exact(a, st);
        cbx::launch_hwc_to_chw(to, 0, out, st);
        CBX_CUDA(cudaFreeAsync(to.d, st));
        CBX_CUDA(cudaFreeAsync(cnt, st));
        CBX_CUDA(cudaFreeAsync(tbl, st));
        CBX_CUDA(cudaGetLastError());
    });
}

// ---- fixtures -----------------------------------------------------------
// random_filters, synth.cpp:188-196
CBX_API int cbx_random_filters(const cbx_geom* g, uint32_t seed, float* K, float* bias) {
    return guarded(nullptr, [&] {
        if (!g || !K || !bias) throw cbx::Error(CBX_E_ARG, "null pointer");
        Mt19937 rng(seed);
        const int fanIn = g->inChannels * g->kernelH * g->kernelW;
        const float scale = 1.0f / std::sqrt((float)fanIn);
        const size_t n = (size_t)g->outChannels * fanIn;
        for (size_t i = 0; i < n; ++i) K[i] = scale * (2.0f * rng.unit() - 1.0f);
        for (int o = 0; o < g->outChannels; ++o) bias[o] = 0.1f * (2.0f * rng.unit() - 1.0f);
    });
}

// synth_frame, synth.cpp:60-91
CBX_API int cbx_synth_frame(const cbx_synth_cfg* cfg, int f, float* out) {
    return guarded(nullptr, [&] {
        if (!cfg || !out) throw cbx::Error(CBX_E_ARG, "null pointer");
        const int C = cfg->channels, H = cfg->height, W = cfg->width;
        for (int c = 0; c < C; ++c)
            for (int j = 0; j < H; ++j)
                for (int i = 0; i < W; ++i) {
                    const unsigned v = (unsigned)(i * 31 + j * 17 + c * 47) % 101u;
                    out[((size_t)c * H + j) * W + i] = 0.2f + 0.25f * ((float)v / 100.0f);
                }
        for (int s = 0; s < cfg->numSprites; ++s) {
            int r[4];
            sprite_rect(*cfg, s, f, r);
            const float v = cfg->sprites[s].intensity;
            for (int c = 0; c < C; ++c)
                for (int j = r[0]; j < r[2]; ++j)
                    for (int i = r[1]; i < r[3]; ++i) out[((size_t)c * H + j) * W + i] = v;
        }
        if (cfg->noiseAmplitude > 0.0f) {
            Mt19937 rng(cfg->seed * 2654435761u + (uint32_t)f + 1u);
            const size_t n = (size_t)C * H * W;
            for (size_t k = 0; k < n; ++k) out[k] += cfg->noiseAmplitude * (2.0f * rng.unit() - 1.0f);
        }
    });
}

CBX_API int cbx_synth_frame_device(const cbx_synth_cfg* cfg, int f, float* out_dev, void* stream) {
    return guarded(nullptr, [&] {
        if (!cfg || !out_dev) throw cbx::Error(CBX_E_ARG, "null pointer");
        if (cfg->noiseAmplitude > 0.0f) throw cbx::Error(CBX_E_ARG, "device synth supports noise-free clips only");
        cudaStream_t st = (cudaStream_t)stream;
        std::vector<cbx::SpriteRect> rects(cfg->numSprites);
        for (int s = 0; s < cfg->numSprites; ++s) {
            int r[4];
            sprite_rect(*cfg, s, f, r);
            rects[s] = cbx::SpriteRect{r[0], r[1], r[2], r[3], cfg->sprites[s].intensity};
        }
        cbx::SpriteRect* d = nullptr;
        const size_t bytes = sizeof(cbx::SpriteRect) * std::max(1, cfg->numSprites);
        CBX_CUDA(cudaMallocAsync((void**)&d, bytes, st));
        if (cfg->numSprites)
            CBX_CUDA(cudaMemcpyAsync(d, rects.data(), sizeof(cbx::SpriteRect) * cfg->numSprites,
                                     cudaMemcpyHostToDevice, st));
        cbx::launch_synth_frame(out_dev, cfg->channels, cfg->height, cfg->width, d, cfg->numSprites, st);
        CBX_CUDA(cudaFreeAsync(d, st));
        CBX_CUDA(cudaStreamSynchronize(st));
    });
}

}  // extern "C"
