// conv_tc.hpp -- tcgen05 (5th-gen tensor core) gathered convolution.
#pragma once

#include <cuda_runtime.h>

#include <memory>

#include "../../include/cbx.h"
#include "common.cuh"

namespace cbx {

struct TcLayer;
struct TcLayerDeleter {
    void operator()(TcLayer* p) const;
};

// A chain of per-pixel layers fused into the epilogue of the preceding
// tcgen05 conv: ops[0] is a 1x1 CONV over the conv's outputs, then RELU (1)
// / 1x1 CONV (0) ops on at most kTailMaxC channels; the result (the input of
// CLASSIFY) is stored to final_out and argmax-classified into labels.
constexpr int kTailMaxC = 16;
constexpr int kTailMaxOps = 8;
struct TcTail {
    int n;
    int kind[kTailMaxOps];  // 0 = CONV 1x1, 1 = RELU
    int cout[kTailMaxOps];
    const float* W[kTailMaxOps];  // [cout][cin] reference layout
    const float* b[kTailMaxOps];
    float* final_out;
    int64_t fo_ss;
    int fo_Wp, fo_Cp, fo_hh, fo_hw;
    uint16_t* labels;
    int64_t l_ss;
    int keep_out;  // also store the conv's own output tensor
};

bool tc_supported(const cbx_geom& g);
// tail_floats: shared memory (floats) to reserve for a fused tail's first 1x1 conv.
// pair_mode: -1 = auto (single-CTA tiles), 0 = never, 1 = CTA pairs (cta_group::2).
// f16: fp16 operands (kind::f16) read from an fp16 shadow of the input whose
// TensorView counts channels in 4-byte units (tc_input_cp).
// i8: layer 1 of the 8-bit camera path -- kind::i8 over the RGBX bytes of the
// frame (TensorView with Cp = 1: one 4-byte unit per pixel), filters as three
// signed base-256 digits of a 22-bit fixed-point weight (relative weight
// error <= 2^-23 of the channel's largest weight, exact integer accumulation).
// grpR > 1: pixel groups -- each tensor-core row is grpR horizontally
// adjacent output pixels (stride-1 layers with a <= 4-channel fp32 input,
// tf32, no fused tail); the update lists hold group entries (gid << 4 | mask)
// from dilate_compact with R = grpR. Falls back to 1 when unsupported.
// pack: fp16 operands from an UNPADDED shadow (Cp = C/2 4-byte units, C even)
// plus the same shadow shifted by 8 bytes (in_shifted of launch_conv_tc):
// each kernel row's kw x C halves are gathered as contiguous 16-byte chunks.
std::unique_ptr<TcLayer, TcLayerDeleter> make_tc_layer(const cbx_geom& g, int tail_floats = 0, int pair_mode = -1,
                                                       bool f16 = false, bool i8 = false, int grpR = 1, bool pack = false);
int tc_input_cp(const TcLayer& t);
int tc_group_width(const TcLayer& t);
bool tc_group_supported(const cbx_geom& g, int R);
bool tc_is_f16(const TcLayer& t);
bool tc_is_i8(const TcLayer& t);
bool tc_i8_supported(const cbx_geom& g);
// K in the reference layout [O][Cin*kh*kw], columns (c,kj,ki); host memory.
void tc_load_weights(TcLayer& t, const float* K, cudaStream_t st);
void launch_conv_tc(const TcLayer& t, TensorView in, TensorView out, const float* bias,
                    const int32_t* idx, const int* count, int64_t full_count, bool relu,
                    BitMask chg, float tau, unsigned long long* cnt, int cstride, int S,
                    cudaStream_t st, const TcTail* tail = nullptr, const float* in_shifted = nullptr);

}  // namespace cbx
