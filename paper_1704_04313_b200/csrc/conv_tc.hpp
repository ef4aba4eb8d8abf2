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

bool tc_supported(const cbx_geom& g);
std::unique_ptr<TcLayer, TcLayerDeleter> make_tc_layer(const cbx_geom& g);
// K in the reference layout [O][Cin*kh*kw], columns (c,kj,ki); host memory.
void tc_load_weights(TcLayer& t, const float* K, cudaStream_t st);
void launch_conv_tc(const TcLayer& t, TensorView in, TensorView out, const float* bias,
                    const int32_t* idx, const int* count, int64_t full_count, bool relu,
                    BitMask chg, float tau, unsigned long long* cnt, int cstride, int S,
                    cudaStream_t st);

}  // namespace cbx
