// k_change.cu -- change detection, change propagation (dilation) and
// change-index extraction (stream compaction) on B200.
//
//   detect   <- detect_changes   /root/reference/proj/core/src/cbconv.cpp:57-71
//   dilate   <- dilate_changes   cbconv.cpp:73-82 (+ scatter_support :28-41)
//   compact  <- extract_indexes  cbconv.cpp:99-113
//
// All three are HBM/L2-bound byte and fp32 streams; none uses tensor cores.
#include "common.cuh"
#include "kernels.hpp"

namespace cbx {

// ---------------------------------------------------------------------------
// K1: detection on planar frames. m(j,i) = OR_c (d > tau || -d > tau), with
// d = cur - prev in fp32. One thread per 4 consecutive pixels, 128-bit loads
// of every channel plane of both frames (the frame read is the O(frame) cost
// of the whole change-based pipeline: 8*C*H*W bytes per stream).
// mode 0: threshold test; mode 1: bitwise inequality (exact-incremental
// consumers that are not CBCONV).
template <int MODE>
__global__ void __launch_bounds__(256) detect_planar_kernel(const float* const* cur,
                                                            const float* const* prev, int C,
                                                            int64_t HW, float tau, uint8_t* mask,
                                                            int64_t mstride,
                                                            unsigned long long* cnt, int cstride) {
    const int s = blockIdx.y;
    const float* a = cur[s];
    const float* b = prev[s];
    uint8_t* m = mask + (int64_t)s * mstride;
    const bool vec = (HW % 4 == 0) && ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) % 16 == 0);
    const int64_t nq = (HW + 3) / 4;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < nq; base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = base + threadIdx.x;
        const bool act = q < nq;
        unsigned flags = 0;
        if (act) {
            if (vec) {
                for (int c = 0; c < C; ++c) {
                    const float4 x = __ldcs(reinterpret_cast<const float4*>(a + c * HW) + q);
                    const float4 y = __ldcs(reinterpret_cast<const float4*>(b + c * HW) + q);
                    if (MODE == 0) {
                        flags |= ref_changed(x.x, y.x, tau) ? 1u : 0u;
                        flags |= ref_changed(x.y, y.y, tau) ? 2u : 0u;
                        flags |= ref_changed(x.z, y.z, tau) ? 4u : 0u;
                        flags |= ref_changed(x.w, y.w, tau) ? 8u : 0u;
                    } else {
                        flags |= (__float_as_uint(x.x) != __float_as_uint(y.x)) ? 1u : 0u;
                        flags |= (__float_as_uint(x.y) != __float_as_uint(y.y)) ? 2u : 0u;
                        flags |= (__float_as_uint(x.z) != __float_as_uint(y.z)) ? 4u : 0u;
                        flags |= (__float_as_uint(x.w) != __float_as_uint(y.w)) ? 8u : 0u;
                    }
                }
                uint32_t packed = (flags & 1u) | ((flags & 2u) << 7) | ((flags & 4u) << 14) | ((flags & 8u) << 21);
                reinterpret_cast<uint32_t*>(m)[q] = packed;
            } else {
                for (int k = 0; k < 4; ++k) {
                    const int64_t p = q * 4 + k;
                    if (p >= HW) break;
                    bool f = false;
                    for (int c = 0; c < C; ++c) {
                        const float x = a[c * HW + p], y = b[c * HW + p];
                        f |= MODE == 0 ? ref_changed(x, y, tau) : (__float_as_uint(x) != __float_as_uint(y));
                    }
                    m[p] = f;
                    flags |= f ? (1u << k) : 0u;
                }
            }
        }
        // per-stream count of changed input pixels (LayerStats::changedInputPixels)
        const int n = __popc(flags);
        const int warp_sum = __reduce_add_sync(0xffffffffu, n);
        if ((threadIdx.x & 31) == 0 && warp_sum && cnt) atomicAdd(cnt + (int64_t)s * cstride, (unsigned long long)warp_sum);
    }
}

void launch_detect_planar(const float* const* cur, const float* const* prev, int S, int C, int H,
                          int W, float tau, int mode, MaskView m, unsigned long long* cnt,
                          int cstride, cudaStream_t st) {
    const int64_t HW = (int64_t)H * W;
    const int64_t nq = (HW + 3) / 4;
    int gx = (int)((nq + 255) / 256);
    const int cap = (kNumSMs * 8 + S - 1) / S;
    if (gx > cap) gx = cap < 1 ? 1 : cap;
    dim3 grid(gx, S);
    if (mode == 0)
        detect_planar_kernel<0><<<grid, 256, 0, st>>>(cur, prev, C, HW, tau, m.d, m.stride, cnt, cstride);
    else
        detect_planar_kernel<1><<<grid, 256, 0, st>>>(cur, prev, C, HW, tau, m.d, m.stride, cnt, cstride);
}

// ---------------------------------------------------------------------------
// K3: dilation of an input-grid mask by a conv geometry (any k, stride, pad):
// out(y,x) = OR over the zero-padded receptive field of (y,x). Separable OR on
// a shared-memory tile: vertical OR over kh rows, then horizontal OR over kw
// columns. Equivalent to the reference's scatter formulation (a set input
// pixel marks every output whose receptive field holds it).
constexpr int kDilTH = 8, kDilTW = 128;

__global__ void __launch_bounds__(256) dilate_kernel(const uint8_t* __restrict__ in, int64_t istride,
                                                     int H, int W, uint8_t* __restrict__ out,
                                                     int64_t ostride, int Ho, int Wo, int kh, int kw,
                                                     int sh, int sw, int ph, int pw) {
    extern __shared__ uint8_t smem[];
    const int s = blockIdx.z;
    const int oy0 = blockIdx.y * kDilTH, ox0 = blockIdx.x * kDilTW;
    const int iy0 = oy0 * sh - ph, ix0 = ox0 * sw - pw;
    const int IH = (kDilTH - 1) * sh + kh, IW = (kDilTW - 1) * sw + kw;
    uint8_t* tin = smem;              // [IH][IW]
    uint8_t* tv = smem + IH * IW;     // [kDilTH][IW]
    const uint8_t* src = in + (int64_t)s * istride;
    for (int t = threadIdx.x; t < IH * IW; t += blockDim.x) {
        const int r = t / IW, c = t - r * IW;
        const int y = iy0 + r, x = ix0 + c;
        tin[t] = (y >= 0 && y < H && x >= 0 && x < W) ? (src[(int64_t)y * W + x] != 0) : 0;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < kDilTH * IW; t += blockDim.x) {
        const int r = t / IW, c = t - r * IW;
        uint8_t v = 0;
        for (int kj = 0; kj < kh; ++kj) v |= tin[(r * sh + kj) * IW + c];
        tv[t] = v;
    }
    __syncthreads();
    uint8_t* dst = out + (int64_t)s * ostride;
    for (int t = threadIdx.x; t < kDilTH * kDilTW; t += blockDim.x) {
        const int r = t / kDilTW, c = t - r * kDilTW;
        const int y = oy0 + r, x = ox0 + c;
        if (y >= Ho || x >= Wo) continue;
        uint8_t v = 0;
        for (int ki = 0; ki < kw; ++ki) v |= tv[r * IW + c * sw + ki];
        dst[(int64_t)y * Wo + x] = v;
    }
}

void launch_dilate(MaskView in, MaskView out, int S, int kh, int kw, int sh, int sw, int ph, int pw,
                   cudaStream_t st) {
    const int IH = (kDilTH - 1) * sh + kh, IW = (kDilTW - 1) * sw + kw;
    const size_t smem = (size_t)IH * IW + (size_t)kDilTH * IW;
    dim3 grid((out.W + kDilTW - 1) / kDilTW, (out.H + kDilTH - 1) / kDilTH, S);
    dilate_kernel<<<grid, 256, smem, st>>>(in.d, in.stride, in.H, in.W, out.d, out.stride, out.H,
                                           out.W, kh, kw, sh, sw, ph, pw);
}

// ---------------------------------------------------------------------------
// K2: stream compaction of a byte mask into the ascending list of set linear
// indices, single pass with decoupled look-back. Tiles of 4096 mask bytes
// (256 threads x 16 bytes, 128-bit loads) never straddle a stream; the list
// is global over [S][N] (index = s*N + p), so it is ascending per stream, and
// per-stream counts are accumulated for LayerStats::changedOutputPixels.
constexpr int kCmpThreads = 256, kCmpPerThread = 16, kCmpTile = kCmpThreads * kCmpPerThread;
constexpr unsigned long long kFlagAgg = 1ull << 62, kFlagPre = 2ull << 62, kValMask = (1ull << 62) - 1;

__global__ void __launch_bounds__(kCmpThreads) compact_kernel(const uint8_t* __restrict__ mask,
                                                              int64_t mstride, int64_t N, int S,
                                                              int tiles_per_stream,
                                                              int32_t* __restrict__ idx, int* total,
                                                              unsigned long long* status,
                                                              unsigned* tile_counter,
                                                              unsigned long long* cnt, int cstride) {
    __shared__ unsigned s_tile;
    __shared__ int s_warp[kCmpThreads / 32];
    __shared__ long long s_base;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const unsigned tile = s_tile;
    const int s = tile / tiles_per_stream;
    const int64_t t_in = tile - (int64_t)s * tiles_per_stream;
    const int64_t p0 = t_in * kCmpTile + (int64_t)threadIdx.x * kCmpPerThread;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (p0 < N) {
        if (p0 + kCmpPerThread <= N) {
            v = __ldcs(reinterpret_cast<const uint4*>(mask + (int64_t)s * mstride + p0));
        } else {
            uint8_t b[16] = {0};
            for (int k = 0; p0 + k < N; ++k) b[k] = mask[(int64_t)s * mstride + p0 + k];
            v = *reinterpret_cast<uint4*>(b);
        }
    }
    // one bit per set byte
    unsigned bits = 0;
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 16; ++k) bits |= ((w[k >> 2] >> ((k & 3) * 8)) & 0xffu) ? (1u << k) : 0u;
    const int my = __popc(bits);
    // block exclusive scan
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = my;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int x = lane < kCmpThreads / 32 ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += t;
        }
        if (lane < kCmpThreads / 32) s_warp[lane] = x;  // inclusive warp prefix
    }
    __syncthreads();
    const int warp_excl = warp ? s_warp[warp - 1] : 0;
    const int agg = s_warp[kCmpThreads / 32 - 1];
    // decoupled look-back (warp 0)
    if (warp == 0) {
        long long base = 0;
        if (tile == 0) {
            if (lane == 0) atomicExch(status, kFlagPre | (unsigned long long)agg);
        } else {
            if (lane == 0) atomicExch(status + tile, kFlagAgg | (unsigned long long)agg);
            long long pos = (long long)tile - 1;
            while (true) {
                const long long j = pos - lane;
                unsigned long long st = 0;
                if (j >= 0) {
                    do {
                        st = atomicAdd(status + j, 0ull);
                    } while ((st >> 62) == 0);
                } else {
                    st = kFlagPre;  // before the first tile: prefix 0
                }
                const unsigned pre = __ballot_sync(0xffffffffu, (st >> 62) == 2);
                const int stop = pre ? __ffs(pre) - 1 : 32;  // first lane (closest tile) with a prefix
                long long val = (lane <= stop) ? (long long)(st & kValMask) : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
                base += val;
                if (pre) break;
                pos -= 32;
            }
            if (lane == 0) atomicExch(status + tile, kFlagPre | (unsigned long long)(base + agg));
        }
        if (lane == 0) {
            s_base = base;
            if (agg) {
                atomicAdd(total, agg);
                if (cnt) atomicAdd(cnt + (int64_t)s * cstride, (unsigned long long)agg);
            }
        }
    }
    __syncthreads();
    int64_t out = s_base + warp_excl + (incl - my);
    const int64_t gbase = (int64_t)s * N + p0;
    while (bits) {
        const int k = __ffs(bits) - 1;
        bits &= bits - 1;
        idx[out++] = (int32_t)(gbase + k);
    }
}

size_t compact_workspace_bytes(int S, int64_t N) {
    const int64_t tiles = (int64_t)S * ((N + kCmpTile - 1) / kCmpTile);
    return (size_t)round_up(tiles * 8 + 16, 256);
}

// workspace: [status: tiles*8][tile_counter: 4][pad]
void launch_compact(MaskView m, int S, int32_t* idx, int* total, void* workspace,
                    unsigned long long* cnt, int cstride, cudaStream_t st) {
    const int64_t N = (int64_t)m.H * m.W;
    const int tps = (int)((N + kCmpTile - 1) / kCmpTile);
    const int64_t tiles = (int64_t)S * tps;
    unsigned long long* status = reinterpret_cast<unsigned long long*>(workspace);
    unsigned* counter = reinterpret_cast<unsigned*>(status + tiles);
    cudaMemsetAsync(workspace, 0, tiles * 8 + 16, st);
    cudaMemsetAsync(total, 0, sizeof(int), st);
    compact_kernel<<<(unsigned)tiles, kCmpThreads, 0, st>>>(m.d, m.stride, N, S, tps, idx, total,
                                                             status, counter, cnt, cstride);
}

}  // namespace cbx
