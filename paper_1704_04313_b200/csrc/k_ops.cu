// k_ops.cu -- the reference's matrix-form ops on the GPU, for the op-level
// API only (cbx_op_gen_x / cbx_op_gemm / cbx_op_scatter; the C++ drop-in's
// im2col_full, gen_x_reduced, fill_patch_column, gemm, update_output). The
// network path never materializes X or Y: there the gather, the contraction
// and the scatter are one kernel (conv_tc.cu, k_layers.cu).
//
//   gen_x   <- fill_patch_column / gen_x_reduced  baseline.cpp:9-31, cbconv.cpp:115-133
//   gemm    <- gemm                               baseline.cpp:47-63
//   scatter <- update_output (without the copy)   cbconv.cpp:135-155
#include "common.cuh"
#include "kernels.hpp"

namespace cbx {

namespace {

// X column-major [n][K]: column j = receptive field of output pixel idx[j]
// (all pixels when idx is null) in (c, kj, ki) order, zeros outside the frame.
__global__ void gen_x_kernel(const float* __restrict__ in, int C, int H, int W, int kh, int kw, int sh, int sw,
                             int ph, int pw, int Wo, const int32_t* __restrict__ idx, int64_t n,
                             float* __restrict__ X) {
    const int K = C * kh * kw;
    const int64_t total = n * K;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t col = t / K;
        const int r = (int)(t - col * K);
        const int p = idx ? idx[col] : (int)col;
        const int yo = p / Wo, xo = p - (p / Wo) * Wo;
        const int c = r / (kh * kw), rem = r - c * kh * kw;
        const int kj = rem / kw, ki = rem - kj * kw;
        const int y = yo * sh + kj - ph, x = xo * sw + ki - pw;
        X[t] = (y >= 0 && y < H && x >= 0 && x < W) ? in[((int64_t)c * H + y) * W + x] : 0.0f;
    }
}

// Y row-major [rows][n] = bias + K X, accumulated in ascending r with one
// rounding per multiply and per add (no FMA): bitwise the reference gemm.
__global__ void gemm_exact_kernel(const float* __restrict__ Kf, const float* __restrict__ bias, int rows, int cols,
                                  const float* __restrict__ X, int64_t n, float* __restrict__ Y) {
    const int64_t total = (int64_t)rows * n;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int o = (int)(t / n);
        const int64_t j = t - (int64_t)o * n;
        const float* krow = Kf + (int64_t)o * cols;
        const float* xcol = X + j * cols;
        float acc = bias[o];
        for (int r = 0; r < cols; ++r) acc = __fadd_rn(acc, __fmul_rn(krow[r], xcol[r]));
        Y[t] = acc;
    }
}

// out[c][idx[j]] = Y[c][j] (through max(0, .) when relu), planar, in place.
__global__ void scatter_kernel(float* __restrict__ out, int C, int64_t HW, const float* __restrict__ Y,
                               const int32_t* __restrict__ idx, int64_t n, int relu) {
    const int64_t total = (int64_t)C * n;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(t / n);
        const int64_t j = t - (int64_t)c * n;
        const float v = Y[t];
        out[(int64_t)c * HW + idx[j]] = relu ? ref_relu(v) : v;
    }
}

// 8-bit interleaved frames (PPM raster: pixel-major, C bytes per pixel) ->
// planar fp32 in [0, 1], exactly read_ppm's px / 255.0f (io.cpp:60-104):
// one IEEE-rounded division per value. One thread per pixel; the C loads of
// a warp cover 32*C contiguous bytes, each plane's stores are coalesced.
__global__ void decode_u8_kernel(const uint8_t* __restrict__ in, int C, int64_t HW, float* __restrict__ out) {
    const int s = blockIdx.y;
    const uint8_t* src = in + (int64_t)s * HW * C;
    float* dst = out + (int64_t)s * HW * C;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < HW; p += (int64_t)gridDim.x * blockDim.x)
        for (int c = 0; c < C; ++c) dst[(int64_t)c * HW + p] = __fdiv_rn((float)src[p * C + c], 255.0f);
}

int grid_for(int64_t total) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, (int64_t)kNumSMs * 32));
}

}  // namespace

void launch_decode_u8(const uint8_t* in, int S, int C, int H, int W, float* out, cudaStream_t st) {
    const int64_t HW = (int64_t)H * W;
    const int gx = (int)std::max<int64_t>(1, std::min<int64_t>((HW + 255) / 256, (int64_t)kNumSMs * 8));
    if (HW > 0 && S > 0) decode_u8_kernel<<<dim3(gx, S), 256, 0, st>>>(in, C, HW, out);
}

void launch_gen_x(const float* in, int C, int H, int W, int kh, int kw, int sh, int sw, int ph, int pw,
                  const int32_t* idx, int64_t n, float* X, cudaStream_t st) {
    const int Wo = (W + 2 * pw - kw) / sw + 1;
    const int64_t total = n * C * kh * kw;
    if (total > 0) gen_x_kernel<<<grid_for(total), 256, 0, st>>>(in, C, H, W, kh, kw, sh, sw, ph, pw, Wo, idx, n, X);
}

void launch_gemm_exact(const float* K, const float* bias, int rows, int cols, const float* X, int64_t n, float* Y,
                       cudaStream_t st) {
    const int64_t total = (int64_t)rows * n;
    if (total > 0) gemm_exact_kernel<<<grid_for(total), 256, 0, st>>>(K, bias, rows, cols, X, n, Y);
}

void launch_scatter(float* out, int C, int64_t HW, const float* Y, const int32_t* idx, int64_t n, int relu,
                    cudaStream_t st) {
    const int64_t total = (int64_t)C * n;
    if (total > 0) scatter_kernel<<<grid_for(total), 256, 0, st>>>(out, C, HW, Y, idx, n, relu);
}

}  // namespace cbx
