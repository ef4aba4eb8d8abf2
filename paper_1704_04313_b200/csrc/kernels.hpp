// kernels.hpp -- host launchers of the cbx CUDA kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"

namespace cbx {

// ---- k_change.cu: byte-mask kernels behind the op-level C-ABI (cbx_op_*) ----
void launch_detect_planar(const float* const* cur, const float* const* prev, int S, int C, int H,
                          int W, float tau, int mode, MaskView m, unsigned long long* cnt,
                          int cstride, cudaStream_t st);
void launch_dilate(MaskView in, MaskView out, int S, int kh, int kw, int sh, int sw, int ph, int pw,
                   cudaStream_t st);
size_t compact_workspace_bytes(int S, int64_t N);
void launch_compact(MaskView m, int S, int32_t* idx, int* total, void* workspace,
                    unsigned long long* cnt, int cstride, cudaStream_t st);

// ---- k_bits.cu: the engine's packed-bit mask pipeline ----
void launch_detect_bits(const float* const* cur, const float* const* prev, int S, int C, int H, int W, float tau,
                        int mode, BitMask m, unsigned long long* cnt, int cstride, cudaStream_t st);
// 8-bit interleaved RGB frames (W % 16 == 0): detection (mode 0 threshold,
// 1 bitwise) fused with the RGBX expansion of the current frame; mode 2 =
// expansion only (full evaluations).
bool rgb8_native_ok(int C, int H, int W);
void launch_detect_rgb8(const uint8_t* const* cur, const uint8_t* const* prev, int S, int H, int W, float tau, int mode,
                        BitMask m, unsigned long long* cnt, int cstride, Rgbx8View x, cudaStream_t st);
size_t dilate_compact_workspace(const BitMask& out, int S);
// ws_zeroed: the caller zeroed `workspace` (the look-back status words) in
// the same stream, e.g. with the frame's single scratch memset.
void launch_dilate_compact(BitMask in, BitMask out, bool write_out, int S, int kh, int kw, int ph, int pw,
                           int32_t* idx, int* total, void* workspace, unsigned long long* cnt, int cstride,
                           cudaStream_t st, bool ws_zeroed = false, int R = 1);
void launch_dilate_bits(BitMask in, BitMask out, int S, int kh, int kw, int sh, int sw, int ph, int pw,
                        cudaStream_t st);

struct PointBitsArgs {  // MAXPOOL (window/stride) or RELU (relu=1, window=stride=1)
    TensorView in, out;
    int window, stride, relu;
    BitMask upd_in;   // updated pixels of the input grid; d == nullptr => all
    BitMask U_out;    // touched output pixels (optional)
    BitMask chg;      // consumer CBCONV change mask (optional)
    float tau;
    unsigned long long* chg_cnt;
    int cnt_stride;
    int S;
    uint32_t* work;   // touched-pixel list s*Ho*Wo + y*Wo + x (capacity S*Ho*Wo), sparse mode only
    int* work_count;
    int count_zeroed;  // work_count already zeroed in-stream (frame scratch memset)
    // optional fp16 shadow of `out` (round to nearest even) for a kind::f16
    // consumer; channels counted in 4-byte units (Cp = fp16 channels / 2)
    TensorView out16;
    TensorView out16b;  // packed shadows: the same written again 8 bytes further (conv_tc packed gather)
    int* f16_overflow;  // set to 1 when a value written to out16 exceeds the fp16 range
};
void launch_point_bits(const PointBitsArgs& a, cudaStream_t st);
void launch_classify_bits(TensorView in, BitMask upd, uint16_t* labels, int S, cudaStream_t st);
void launch_unpack_bits(BitMask m, int s, uint8_t* out, cudaStream_t st);
// out[s] += number of set bits of stream s (out zeroed by the caller)
void launch_popcount_bits(BitMask m, int S, unsigned long long* out, cudaStream_t st);

// ---- k_layers.cu ----
// Gathered convolution over an output-pixel list (or all pixels when idx is
// null), exact fp32 reference order, result written in place.
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
    BitMask chg;         // chg.d == nullptr => no test
    float tau;
    unsigned long long* chg_cnt;
    int cnt_stride;
    int S;
    // host copies of K / bias (optional): lets a geometry-specialised kernel
    // carry the filters as kernel parameters (constant-bank FMUL operands)
    const float* hK;
    const float* hB;
};
void launch_conv_exact(const ConvArgs& a, cudaStream_t st);

// byte-mask pool / classify used by the op-level API
struct PoolArgs {
    TensorView in, out;
    int window, stride;
    const uint8_t* upd_in;
    int64_t upd_in_stride;
    uint8_t* upd_out;
    int64_t upd_out_stride;
    MaskView chg;
    float tau;
    unsigned long long* chg_cnt;
    int cnt_stride;
    int S;
};
void launch_pool(const PoolArgs& a, cudaStream_t st);

struct PointArgs {
    TensorView in, out;
    const uint8_t* upd;
    int64_t upd_stride;
    MaskView chg;
    float tau;
    unsigned long long* chg_cnt;
    int cnt_stride;
    uint16_t* labels;
    int S;
};
void launch_relu(const PointArgs& a, cudaStream_t st);
void launch_classify(const PointArgs& a, cudaStream_t st);

// Channels-last <-> planar helpers (trace readback, op-level API).
void launch_hwc_to_chw(TensorView t, int s, float* out, cudaStream_t st);
void launch_chw_to_hwc(const float* in, TensorView t, int s, cudaStream_t st);
// planar frames (device pointer table) -> channels-last tensor, all streams
void launch_ingest(const float* const* frames, TensorView t, int S, cudaStream_t st);

// 8-bit interleaved camera frames -> planar fp32 px / 255 (read_ppm, io.cpp:60-104)
void launch_decode_u8(const uint8_t* in, int S, int C, int H, int W, float* out, cudaStream_t st);

// ---- matrix-form reference ops (op-level API only; k_ops.cu) ----
void launch_gen_x(const float* in, int C, int H, int W, int kh, int kw, int sh, int sw, int ph, int pw,
                  const int32_t* idx, int64_t n, float* X, cudaStream_t st);
void launch_gemm_exact(const float* K, const float* bias, int rows, int cols, const float* X, int64_t n, float* Y,
                       cudaStream_t st);
void launch_scatter(float* out, int C, int64_t HW, const float* Y, const int32_t* idx, int64_t n, int relu,
                    cudaStream_t st);

// ---- synthetic frames ----
struct SpriteRect {
    int y0, x0, y1, x1;
    float v;
};
void launch_synth_frame(float* out, int C, int H, int W, const SpriteRect* rects_dev, int n,
                        cudaStream_t st);

}  // namespace cbx
