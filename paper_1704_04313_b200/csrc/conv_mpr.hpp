// conv_mpr.hpp -- multi-pixel-row tcgen05 convolution for narrow layers (see conv_mpr.cu).
#pragma once

#include <cuda_runtime.h>

#include <memory>

#include "../../include/cbx.h"
#include "common.cuh"

namespace cbx {

struct MprLayer;
struct MprLayerDeleter {
    void operator()(MprLayer* p) const;
};

// mode 0: kind::i8 over the RGBX bytes of an 8-bit frame (R = 4 only);
// mode 1: kind::f16 over a 4-channel fp32 channels-last input.
bool mpr_supported(const cbx_geom& g, int mode, int R);
// in_hw: the input tensor's left halo (pixels); mode 0 aligns its windows to it
std::unique_ptr<MprLayer, MprLayerDeleter> make_mpr_layer(const cbx_geom& g, int mode, int R, int in_hw);
int mpr_group_width(const MprLayer& t);
int mpr_mode(const MprLayer& t);
// K in the reference layout [O][Cin*kh*kw], columns (c,kj,ki); host memory.
void mpr_load_weights(MprLayer& t, const float* K, cudaStream_t st);
// list: group entries (gid << 4 | mask) from dilate_compact with R = the
// layer's group width, or nullptr for a full evaluation of the S streams.
void launch_conv_mpr(const MprLayer& t, TensorView in, TensorView out, const float* bias, const uint32_t* list,
                     const int* count, int S, bool relu, BitMask chg, float tau, unsigned long long* cnt, int cstride,
                     int* ovf, cudaStream_t st);

}  // namespace cbx
