// kernels.hpp -- host launchers of the cbx CUDA kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace cbx {

// ---- k_change.cu ----
void launch_detect_planar(const float* const* cur, const float* const* prev, int S, int C, int H,
                          int W, float tau, int mode, MaskView m, unsigned long long* cnt,
                          int cstride, cudaStream_t st);
void launch_dilate(MaskView in, MaskView out, int S, int kh, int kw, int sh, int sw, int ph, int pw,
                   cudaStream_t st);
size_t compact_workspace_bytes(int S, int64_t N);
void launch_compact(MaskView m, int S, int32_t* idx, int* total, void* workspace,
                    unsigned long long* cnt, int cstride, cudaStream_t st);

// ---- k_layers.cu ----
// Gathered convolution over an output-pixel list (or all pixels when idx is
// null), result written in place into the output tensor.
struct ConvArgs {
    // input: HWC tensor, or the planar frame table when in_ptrs != nullptr
    TensorView in;
    const float* const* in_ptrs;
    TensorView out;
    const float* K;     // [O][Kdim], columns (c,kj,ki) -- reference layout
    const float* bias;  // [O]
    int kh, kw, sh, sw, ph, pw;
    const int32_t* idx;  // global output indices s*Ho*Wo + p, ascending; null => all
    const int* count;    // device count for idx
    int64_t full_count;  // S*Ho*Wo
    int relu;
    // change test of the consumer CBCONV (compare new vs stored value)
    MaskView chg;        // chg.d == nullptr => no test
    float tau;
    unsigned long long* chg_cnt;
    int cnt_stride;
    int S;
};
void launch_conv_exact(const ConvArgs& a, cudaStream_t st);

struct PoolArgs {
    TensorView in, out;
    int window, stride;
    const uint8_t* upd_in;  // updated mask of the input grid; null => all pixels
    int64_t upd_in_stride;
    uint8_t* upd_out;       // touched mask of the output grid (optional)
    int64_t upd_out_stride;
    MaskView chg;           // consumer CBCONV change mask (optional)
    float tau;
    unsigned long long* chg_cnt;
    int cnt_stride;
    int S;
};
void launch_pool(const PoolArgs& a, cudaStream_t st);

struct PointArgs {  // RELU / CLASSIFY over updated pixels
    TensorView in, out;
    const uint8_t* upd;  // null => all
    int64_t upd_stride;
    MaskView chg;
    float tau;
    unsigned long long* chg_cnt;
    int cnt_stride;
    uint16_t* labels;    // CLASSIFY output [S][H][W]
    int S;
};
void launch_relu(const PointArgs& a, cudaStream_t st);
void launch_classify(const PointArgs& a, cudaStream_t st);

// Channels-last <-> planar helpers (trace readback, op-level API).
void launch_hwc_to_chw(TensorView t, int s, float* out, cudaStream_t st);
void launch_chw_to_hwc(const float* in, TensorView t, int s, cudaStream_t st);
// planar frames (device pointer table) -> channels-last tensor, all streams
void launch_ingest(const float* const* frames, TensorView t, int S, cudaStream_t st);

// ---- k_synth.cu ----
struct SpriteRect {
    int y0, x0, y1, x1;
    float v;
};
void launch_synth_frame(float* out, int C, int H, int W, const SpriteRect* rects_dev, int n,
                        cudaStream_t st);

// ---- k_conv_tc.cu (tcgen05) ----
struct TcConvArgs;  // defined in conv_tc.hpp

}  // namespace cbx
