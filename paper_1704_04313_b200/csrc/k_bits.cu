// k_bits.cu -- the engine's change-mask pipeline on packed bit masks.
//
// Every mask the engine keeps (change masks "chg", updated-pixel masks "U")
// is one bit per pixel, rows padded to 32-bit words (see BitMask in
// common.cuh), so the O(frame) mask traffic is 1/8 of the reference's
// uint8 ChangeMap (cbconv.hpp:17-29) and dilation is a handful of funnel
// shifts per 32 pixels.
//
//   detect_bits        <- detect_changes  cbconv.cpp:57-71      (K1)
//   dilate_compact     <- dilate_changes + extract_indexes
//                         cbconv.cpp:73-82, 99-113              (K3+K2, one pass)
//   dilate_bits        <- dilate_changes for strided geometries (K3)
//   point_bits         <- maxpool / relu over updated pixels     (K5)
//                         baseline.cpp:113-145, fused with the next
//                         layer's change detection
//   classify_bits      <- argmax_classify  baseline.cpp:147-163
#include <cuda_fp16.h>

#include <cstdlib>
#include <stdexcept>

#include "common.cuh"
#include "kernels.hpp"

namespace cbx {

// ---------------------------------------------------------------------------
// K1: detection on the planar frames, 4 pixels per thread (128-bit loads of
// every channel plane of both frames), packed with warp shuffles into words.
template <int MODE, bool VEC>
__global__ void __launch_bounds__(256) detect_bits_kernel(const float* const* cur, const float* const* prev, int C,
                                                          int H, int W, float tau, BitMask m,
                                                          unsigned long long* cnt, int cstride) {
    pdl_entry();
    const int s = blockIdx.y;
    const float* a = cur[s];
    const float* b = prev[s];
    const int64_t HW = (int64_t)H * W;
    constexpr bool vec = VEC;
    const int qpr = m.wpr * 8;  // pixel quads per (padded) row
    const int64_t nq = (int64_t)H * qpr;
    const int lane = threadIdx.x & 31;
    uint32_t* dst = m.d + (int64_t)s * m.stride;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < nq; base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = base + threadIdx.x;
        const bool act = q < nq;
        uint32_t flags = 0;
        if (act) {
            const int y = (int)(q / qpr);
            const int x0 = (int)(q - (int64_t)y * qpr) * 4;
            if (x0 < W) {
                const int64_t p0 = (int64_t)y * W + x0;
                if constexpr (vec) {
                    // all channel planes of both frames in flight before the compares
                    for (int c0 = 0; c0 < C; c0 += 4) {
                        float4 u[4], v[4];
#pragma unroll
                        for (int c = 0; c < 4; ++c)
                            if (c0 + c < C) {
                                u[c] = __ldcs(reinterpret_cast<const float4*>(a + (c0 + c) * HW + p0));
                                v[c] = __ldcs(reinterpret_cast<const float4*>(b + (c0 + c) * HW + p0));
                            }
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            if (c0 + c >= C) break;
                            if (MODE == 0) {
                                flags |= (ref_changed(u[c].x, v[c].x, tau) ? 1u : 0u) | (ref_changed(u[c].y, v[c].y, tau) ? 2u : 0u) |
                                         (ref_changed(u[c].z, v[c].z, tau) ? 4u : 0u) | (ref_changed(u[c].w, v[c].w, tau) ? 8u : 0u);
                            } else {
                                flags |= (__float_as_uint(u[c].x) != __float_as_uint(v[c].x) ? 1u : 0u) |
                                         (__float_as_uint(u[c].y) != __float_as_uint(v[c].y) ? 2u : 0u) |
                                         (__float_as_uint(u[c].z) != __float_as_uint(v[c].z) ? 4u : 0u) |
                                         (__float_as_uint(u[c].w) != __float_as_uint(v[c].w) ? 8u : 0u);
                            }
                        }
                    }
                } else {
                    for (int e = 0; e < 4 && x0 + e < W; ++e)
                        for (int c = 0; c < C; ++c) {
                            const float u = a[c * HW + p0 + e], v = b[c * HW + p0 + e];
                            const bool f = MODE == 0 ? ref_changed(u, v, tau) : (__float_as_uint(u) != __float_as_uint(v));
                            flags |= f ? (1u << e) : 0u;
                        }
                }
            }
        }
        uint32_t word = flags << (4 * (lane & 7));
        word |= __shfl_xor_sync(0xffffffffu, word, 1);
        word |= __shfl_xor_sync(0xffffffffu, word, 2);
        word |= __shfl_xor_sync(0xffffffffu, word, 4);
        if (act && (lane & 7) == 0) dst[q >> 3] = word;
        if (cnt) {
            const int n = __reduce_add_sync(0xffffffffu, __popc(flags));
            if (lane == 0 && n) atomicAdd(cnt + (int64_t)s * cstride, (unsigned long long)n);
        }
    }
}

// K1 for 3-channel frames (the paper's RGB input), QPT pixel quads per thread:
// all 6*QPT 128-bit loads (both frames, every plane) are issued before any
// compare, so each thread keeps QPT*96 bytes in flight.
template <int QPT>
__global__ void __launch_bounds__(256) detect_c3_kernel(const float* const* cur, const float* const* prev, int H, int W,
                                                        float tau, BitMask m, unsigned long long* cnt, int cstride) {
    pdl_entry();
    const int s = blockIdx.y;
    const float* a = cur[s];
    const float* b = prev[s];
    const int HW = H * W;
    const int qpr = m.wpr * 8;
    const int nq = H * qpr;
    const int lane = threadIdx.x & 31;
    uint32_t* dst = m.d + (int64_t)s * m.stride;
    for (int base = blockIdx.x * blockDim.x * QPT; base < nq; base += gridDim.x * blockDim.x * QPT) {
        float4 u[QPT][3], v[QPT][3];
        bool ok[QPT];
#pragma unroll
        for (int k = 0; k < QPT; ++k) {
            const int q = base + k * blockDim.x + threadIdx.x;
            const int y = q / qpr;
            const int x0 = (q - y * qpr) * 4;
            ok[k] = q < nq && x0 < W;
            if (ok[k]) {
                const int p0 = y * W + x0;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    u[k][c] = __ldcs(reinterpret_cast<const float4*>(a + c * HW + p0));
                    v[k][c] = __ldcs(reinterpret_cast<const float4*>(b + c * HW + p0));
                }
            }
        }
        int n = 0;
#pragma unroll
        for (int k = 0; k < QPT; ++k) {
            const int q = base + k * blockDim.x + threadIdx.x;
            uint32_t flags = 0;
            if (ok[k]) {
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    flags |= (ref_changed(u[k][c].x, v[k][c].x, tau) ? 1u : 0u) | (ref_changed(u[k][c].y, v[k][c].y, tau) ? 2u : 0u) |
                             (ref_changed(u[k][c].z, v[k][c].z, tau) ? 4u : 0u) | (ref_changed(u[k][c].w, v[k][c].w, tau) ? 8u : 0u);
            }
            uint32_t word = flags << (4 * (lane & 7));
            word |= __shfl_xor_sync(0xffffffffu, word, 1);
            word |= __shfl_xor_sync(0xffffffffu, word, 2);
            word |= __shfl_xor_sync(0xffffffffu, word, 4);
            if (q < nq && (lane & 7) == 0) dst[q >> 3] = word;
            n += __popc(flags);
        }
        if (cnt) {
            n = __reduce_add_sync(0xffffffffu, n);
            if (lane == 0 && n) atomicAdd(cnt + (int64_t)s * cstride, (unsigned long long)n);
        }
    }
}

// K1 on 8-bit camera frames (the PPM raster read_ppm decodes, io.cpp:60-104):
// H x W x 3 interleaved bytes per stream, W a multiple of 16. A thread owns 16
// pixels (48 bytes = three 128-bit loads per frame). Pixel values are the
// reference's px / 255.0f (correctly rounded like the host division), so the
// change test is detect_changes on read_ppm's tensors bit for bit: per
// channel byte pair, |a - b| >= dhi is changed for every pair and < dlo for
// none (bounds precomputed on the host for tau by brute force,
// rgb8_tau_bounds); only differences in [dlo, dhi) -- none unless tau sits
// within an ulp of some k / 255 -- take the exact decode + compare. The same
// pass writes the current frame as 4-byte RGBX pixels (channel 3 = 0) into
// the zero-halo tensor the layer-1 tcgen05 conv gathers from; a steady frame
// rewrites only the 16-pixel groups whose bytes changed (the buffer holds the
// previous frame's expansion).
//   MODE 0: threshold test (CBCONV); MODE 1: any byte differs (updated
//   pixels of a non-CB first layer); MODE 2: full frame, expansion only.
// SWAR "some byte of x is >= t" (1 <= t <= 256; t = 256: never), branch
// free with per-launch constants (ByteGe::make on the host): bytes below 128
// carry into bit 7 when (b & 0x7f) + 0x80 - t overflows 7 bits (t <= 128:
// OR with x's own bit 7); for t > 128 a byte needs bit 7 set AND its low 7
// bits >= t - 128 (AND with x).
struct ByteGe {
    uint32_t add, and_sel, mask;  // and_sel: ~0 selects the AND form
    static ByteGe make(int t) {
        ByteGe b{0u, 0u, 0x80808080u};
        if (t > 255) {
            b.mask = 0u;
        } else if (t <= 128) {
            b.add = (uint32_t)(0x80 - t) * 0x01010101u;
        } else {
            b.add = (uint32_t)(0x80 - (t - 128)) * 0x01010101u;
            b.and_sel = 0xffffffffu;
        }
        return b;
    }
    __device__ __forceinline__ uint32_t test(uint32_t x) const {
        const uint32_t r = (x & 0x7f7f7f7fu) + add;
        return ((r & x) | ((r | x) & ~and_sel)) & mask;
    }
};

template <int MODE>
__global__ void __launch_bounds__(256) detect_rgb8_kernel(const uint8_t* const* cur, const uint8_t* const* prev, int H,
                                                          int W, float tau, ByteGe ge_lo, ByteGe ge_hi, BitMask m,
                                                          unsigned long long* cnt, int cstride, Rgbx8View x) {
    pdl_entry();
    // px / 255.0f of every byte value: the reference's read_ppm decode
    // (correctly rounded division, like the host's)
    __shared__ float lut[256];
    if (MODE == 0) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) lut[i] = __fdiv_rn((float)i, 255.0f);
        __syncthreads();
    }
    const int s = blockIdx.y;
    const uint4* a = reinterpret_cast<const uint4*>(cur[s]);
    const uint4* b = MODE == 2 ? nullptr : reinterpret_cast<const uint4*>(prev[s]);
    const int wpr = (W + 31) >> 5;
    const int gpr = 2 * wpr;  // 16-pixel groups per row, padded to whole mask words
    const int ng = H * gpr;
    const int lane = threadIdx.x & 31;
    uint32_t* dst = MODE == 2 ? nullptr : m.d + (int64_t)s * m.stride;
    uint32_t* xs = x.d + (int64_t)s * x.ss;
    for (int base = blockIdx.x * blockDim.x; base < ng; base += gridDim.x * blockDim.x) {
        const int g = base + threadIdx.x;
        const int y = g / gpr, gx = g - y * gpr;
        const bool act = g < ng && 16 * gx < W;
        uint32_t flags = 0, amb = 0;
        uint32_t o[16], op[16];
        if (act) {
            const int64_t q = ((int64_t)y * W + 16 * gx) / 16 * 3;  // uint4 index of the 48-byte group
            uint32_t cw[12], pw[12];
            {
                const uint4 c0 = __ldg(a + q), c1 = __ldg(a + q + 1), c2 = __ldg(a + q + 2);
                cw[0] = c0.x; cw[1] = c0.y; cw[2] = c0.z; cw[3] = c0.w;
                cw[4] = c1.x; cw[5] = c1.y; cw[6] = c1.z; cw[7] = c1.w;
                cw[8] = c2.x; cw[9] = c2.y; cw[10] = c2.z; cw[11] = c2.w;
            }
            uint32_t anyd = 1u;  // full frames: every group is expanded
            if constexpr (MODE != 2) {
                const uint4 p0 = __ldcs(b + q), p1 = __ldcs(b + q + 1), p2 = __ldcs(b + q + 2);
                pw[0] = p0.x; pw[1] = p0.y; pw[2] = p0.z; pw[3] = p0.w;
                pw[4] = p1.x; pw[5] = p1.y; pw[6] = p1.z; pw[7] = p1.w;
                pw[8] = p2.x; pw[9] = p2.y; pw[10] = p2.z; pw[11] = p2.w;
                anyd = 0u;
#pragma unroll
                for (int i = 0; i < 12; ++i) anyd |= cw[i] ^ pw[i];
            }
            // A group whose 48 bytes equal the previous frame's has no change
            // and its RGBX pixels (the buffer holds the previous frame's
            // expansion) are already right: only changed groups are expanded,
            // tested and rewritten (a static camera changes a few %).
            if (anyd) {
                // RGBX expansion: pixel p = bytes 3p..3p+2 of the group
#pragma unroll
                for (int p = 0; p < 16; ++p) {
                    const int bi = 3 * p, wi = bi >> 2, r = bi & 3;
                    const uint32_t sel = (uint32_t)(r | ((r + 1) << 4) | ((r + 2) << 8));
                    o[p] = __byte_perm(cw[wi], wi + 1 < 12 ? cw[wi + 1] : 0u, sel) & 0x00ffffffu;
                    if constexpr (MODE != 2) {
                        op[p] = __byte_perm(pw[wi], wi + 1 < 12 ? pw[wi + 1] : 0u, sel) & 0x00ffffffu;
                        // |a - b| per channel byte: >= dhi is changed for every
                        // byte pair, < dlo for none; in between decide exactly below
                        const uint32_t ad = __vabsdiffu4(o[p], op[p]);
                        if (ge_hi.test(ad)) flags |= 1u << p;
                        else if (ge_lo.test(ad)) amb |= 1u << p;
                    }
                }
                uint4* xo = reinterpret_cast<uint4*>(xs + (int64_t)(y + x.hh) * x.Wp + x.hw + 16 * gx);
                xo[0] = make_uint4(o[0], o[1], o[2], o[3]);
                xo[1] = make_uint4(o[4], o[5], o[6], o[7]);
                xo[2] = make_uint4(o[8], o[9], o[10], o[11]);
                xo[3] = make_uint4(o[12], o[13], o[14], o[15]);
            }
        }
        if constexpr (MODE != 2) {
            // the exact test (decode + reference compare) for pixels whose
            // channel differences straddle tau's byte-difference boundary --
            // none for a tau that is not within an ulp of some k / 255
            if (__any_sync(0xffffffffu, amb != 0u)) {
#pragma unroll
                for (int p = 0; p < 16; ++p) {
                    if ((amb >> p) & 1u) {
                        bool c = false;
#pragma unroll
                        for (int e = 0; e < 3; ++e) {
                            const uint32_t u = (o[p] >> (8 * e)) & 0xffu, v = (op[p] >> (8 * e)) & 0xffu;
                            c |= MODE == 1 ? u != v : ref_changed(lut[u], lut[v], tau);
                        }
                        if (c) flags |= 1u << p;
                    }
                }
            }
            uint32_t word = flags << (16 * (gx & 1));
            word |= __shfl_xor_sync(0xffffffffu, word, 1);
            if (g < ng && (gx & 1) == 0) dst[(int64_t)y * m.wpr + (gx >> 1)] = word;
            if (cnt) {
                const int n = __reduce_add_sync(0xffffffffu, __popc(flags));
                if (lane == 0 && n) atomicAdd(cnt + (int64_t)s * cstride, (unsigned long long)n);
            }
        }
    }
}

// Byte-difference bounds of the reference change test on read_ppm values for
// threshold tau: a channel pair (u, v) of bytes is changed
// (ref_changed(u / 255.0f, v / 255.0f, tau)) for every pair with
// |u - v| >= dhi and for no pair with |u - v| < dlo (brute force over all
// 65536 pairs with the same IEEE division and subtraction as the device).
// dhi = 256 when some difference class is never entirely changed above dlo.
static void rgb8_tau_bounds(float tau, int mode, int& dlo, int& dhi) {
    if (mode == 1) {  // bitwise: any differing byte
        dlo = dhi = 1;
        return;
    }
    // (one tau per layer-1 threshold setting: remember the last one)
    thread_local float last_tau = -1.0f;
    thread_local int last_lo = 0, last_hi = 0;
    if (tau == last_tau) {
        dlo = last_lo;
        dhi = last_hi;
        return;
    }
    bool any[256] = {}, all[256];
    for (int k = 0; k < 256; ++k) all[k] = true;
    for (int u = 0; u < 256; ++u)
        for (int v = 0; v < 256; ++v) {
            const float fu = (float)u / 255.0f, fv = (float)v / 255.0f;
            const float d = fu - fv;
            const bool c = d > tau || -d > tau;
            const int k = u > v ? u - v : v - u;
            any[k] = any[k] || c;
            all[k] = all[k] && c;
        }
    dlo = 256;
    for (int k = 0; k < 256; ++k)
        if (any[k]) {
            dlo = k;
            break;
        }
    dhi = 256;
    for (int k = 255; k >= 0 && all[k]; --k) dhi = k;
    if (dhi < dlo) dhi = dlo;
    last_tau = tau;
    last_lo = dlo;
    last_hi = dhi;
}

bool rgb8_native_ok(int C, int H, int W) { return C == 3 && W % 16 == 0 && W > 0 && H > 0 && (int64_t)H * W < (1 << 30); }

void launch_detect_rgb8(const uint8_t* const* cur, const uint8_t* const* prev, int S, int H, int W, float tau, int mode,
                        BitMask m, unsigned long long* cnt, int cstride, Rgbx8View x, cudaStream_t st) {
    const int ng = H * 2 * ((W + 31) / 32);
    int gx = (ng + 255) / 256;
    const int cap = (kNumSMs * 8 + S - 1) / S;
    if (gx > cap) gx = cap < 1 ? 1 : cap;
    const dim3 grid(gx, S);
    int dlo = 256, dhi = 256;
    if (mode != 2) rgb8_tau_bounds(tau, mode, dlo, dhi);
    if (mode == 0)
        launch_k(detect_rgb8_kernel<0>, grid, dim3(256), 0, st, cur, prev, H, W, tau, ByteGe::make(dlo), ByteGe::make(dhi), m, cnt, cstride, x);
    else if (mode == 1)
        launch_k(detect_rgb8_kernel<1>, grid, dim3(256), 0, st, cur, prev, H, W, tau, ByteGe::make(dlo), ByteGe::make(dhi), m, cnt, cstride, x);
    else
        launch_k(detect_rgb8_kernel<2>, grid, dim3(256), 0, st, cur, prev, H, W, tau, ByteGe::make(dlo), ByteGe::make(dhi), m, cnt, cstride, x);
}

void launch_detect_bits(const float* const* cur, const float* const* prev, int S, int C, int H, int W, float tau,
                        int mode, BitMask m, unsigned long long* cnt, int cstride, cudaStream_t st) {
    const int64_t nq = (int64_t)H * m.wpr * 8;
    int gx = (int)((nq + 255) / 256);
    const int cap = (kNumSMs * 8 + S - 1) / S;
    if (gx > cap) gx = cap < 1 ? 1 : cap;
    dim3 grid(gx, S);
    // frame pointers are 16-byte aligned (engine slots; checked for user frames in forward_device)
    const bool vec = W % 4 == 0;
    if (mode == 0 && vec && C == 3 && (int64_t)H * W < ((int64_t)1 << 31)) {
        constexpr int QPT = 2;
        int g3 = (int)((nq + 256 * QPT - 1) / (256 * QPT));
        const int cap3 = (kNumSMs * 8 + S - 1) / S;
        if (g3 > cap3) g3 = cap3 < 1 ? 1 : cap3;
        launch_k(detect_c3_kernel<QPT>, dim3(g3, S), dim3(256), 0, st, cur, prev, H, W, tau, m, cnt, cstride);
        return;
    }
    if (mode == 0 && vec)
        launch_k(detect_bits_kernel<0, true>, grid, dim3(256), 0, st, cur, prev, C, H, W, tau, m, cnt, cstride);
    else if (mode == 0)
        launch_k(detect_bits_kernel<0, false>, grid, dim3(256), 0, st, cur, prev, C, H, W, tau, m, cnt, cstride);
    else if (vec)
        launch_k(detect_bits_kernel<1, true>, grid, dim3(256), 0, st, cur, prev, C, H, W, tau, m, cnt, cstride);
    else
        launch_k(detect_bits_kernel<1, false>, grid, dim3(256), 0, st, cur, prev, C, H, W, tau, m, cnt, cstride);
}

// ---------------------------------------------------------------------------
// K3+K2 fused, stride-1 geometries: each thread owns one output word (32
// output pixels of a row): vertical OR over kh input rows of the horizontally
// dilated row slices (funnel shifts over the neighbouring words), optional
// write of the dilated word (the layer's updated-pixel mask), then
// single-pass stream compaction with decoupled look-back. Tiles of 256 words
// never straddle a stream (stride is a multiple of 256 words).
constexpr int kDcThreads = 256;
constexpr unsigned long long kFlagAgg = 1ull << 62, kFlagPre = 2ull << 62, kValMask = (1ull << 62) - 1;

__device__ __forceinline__ uint32_t hslice(uint32_t prev, uint32_t cur, uint32_t next, int t) {
    // bits of the input row at output positions x + t, x in this word
    if (t == 0) return cur;
    if (t > 0) return __funnelshift_r(cur, next, t);
    return __funnelshift_l(prev, cur, -t);
}

// Returns the block-exclusive prefix of `my` and the block total (all threads).
__device__ __forceinline__ int block_scan(int my, int* s_warp, int& total) {
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
        int x = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += t;
        }
        if (lane < (int)(blockDim.x >> 5)) s_warp[lane] = x;
    }
    __syncthreads();
    total = s_warp[(blockDim.x >> 5) - 1];
    return (warp ? s_warp[warp - 1] : 0) + incl - my;
}

// OR over a horizontal window: output bit x of the word = OR of input bits
// x + t, t in [-pw, kw - 1 - pw], with the neighbouring words supplying the
// bits that cross the word boundary (64-bit doubling: ~log2(kw) shift/or).
__device__ __forceinline__ uint32_t hdilate(uint32_t prev, uint32_t cur, uint32_t next, int kw, int pw) {
    const int tmax = kw - 1 - pw;  // rightward reach (may be negative)
    uint32_t out = 0;
    if (tmax >= 0) {
        uint64_t r = ((uint64_t)next << 32) | cur;  // bit j = input position j
        int covered = 1;
        const int wdt = tmax + 1;
        uint64_t acc = r;
        while (covered * 2 <= wdt) {
            acc |= acc >> covered;
            covered *= 2;
        }
        if (covered < wdt) acc |= acc >> (wdt - covered);
        out |= (uint32_t)acc;  // positions x .. x + tmax
        if (pw > 0) {
            // positions x - pw .. x - 1: bits of (prev, cur) shifted
            uint64_t l = ((uint64_t)cur << 32) | prev;  // bit j = input position j - 32
            uint64_t accl = l;
            int cv = 1;
            while (cv * 2 <= pw) {
                accl |= accl >> cv;
                cv *= 2;
            }
            if (cv < pw) accl |= accl >> (pw - cv);
            out |= (uint32_t)(accl >> (32 - pw));  // bit x <- OR of positions x-pw .. x-1
        }
    } else {
        // window entirely left of x: positions x - pw .. x - pw + kw - 1
        uint64_t l = ((uint64_t)cur << 32) | prev;
        uint64_t accl = l;
        int cv = 1;
        while (cv * 2 <= kw) {
            accl |= accl >> cv;
            cv *= 2;
        }
        if (cv < kw) accl |= accl >> (kw - cv);
        out = (uint32_t)(accl >> (32 - pw));
    }
    return out;
}

// Output words [t0, t0 + tile) of one stream need input rows
// [y(t0) - ph, y(t0 + tile - 1) - ph + kh) -- one contiguous range of input
// words. It is staged into shared memory with coalesced 16-byte loads,
// horizontally dilated once per input word, and every output word is then
// the OR of kh shared-memory words.
//
// R = 1: the list holds pixel indices s*Ho*Wo + y*Wo + x (extract_indexes
// order). R = 2 / 4: it holds GROUP entries (gid << 4 | mask) of R
// horizontally adjacent pixels, gid = s*Ho*Gw + y*Gw + x / R, mask = the
// group's set pixels (the multi-pixel-row conv's tiles, conv_mpr.cu); the
// per-stream counter still counts pixels. The list is written warp-
// cooperatively: each non-empty word is expanded by the 32 lanes at once, so
// every store instruction writes consecutive entries (coalesced).
template <int WPT, int R>
__global__ void __launch_bounds__(kDcThreads) dilate_compact_kernel(BitMask in, BitMask out, bool write_out,
                                                                    int kh, int kw, int ph, int pw, bool identity,
                                                                    int32_t* __restrict__ idx, int* total,
                                                                    unsigned long long* cnt, int cstride) {
    pdl_entry();
    extern __shared__ uint4 s_rows4[];
    uint32_t* s_rows = reinterpret_cast<uint32_t*>(s_rows4);
    __shared__ int s_warp[kDcThreads / 32];
    __shared__ long long s_base;
    const unsigned tile = blockIdx.x;
    constexpr int kTile = kDcThreads * WPT;
    const int tps = (int)(out.stride / kTile);
    const int s = tile / tps;
    const int64_t t0 = (int64_t)(tile - (unsigned)s * tps) * kTile;
    const int64_t w0 = t0 + (int64_t)threadIdx.x * WPT;
    const int ya = (int)(t0 / out.wpr);
    const int yb = (int)((t0 + kTile - 1) / out.wpr);
    const int ra = identity ? ya : max(0, ya - ph);
    const int rb = identity ? min(in.H - 1, yb) : min(in.H - 1, yb - ph + kh - 1);
    const uint32_t* src = in.d + (int64_t)s * in.stride;
    const int64_t sw0 = (int64_t)ra * in.wpr;
    const int nwords = rb >= ra ? (rb - ra + 1) * in.wpr : 0;
    const int64_t a4 = sw0 & ~int64_t(3);
    const int shift = (int)(sw0 - a4);
    const int n4 = (int)((sw0 + nwords - a4 + 3) >> 2);
    {
        const uint4* g4 = reinterpret_cast<const uint4*>(src + a4);
        for (int i = threadIdx.x; i < n4; i += kDcThreads) s_rows4[i] = __ldg(g4 + i);
    }
    __syncthreads();
    const uint32_t* rows = s_rows + shift;
    uint32_t* hrows = s_rows + 4 * n4 + 4;  // horizontally dilated copy
    if (!identity) {
        for (int i = threadIdx.x; i < nwords; i += kDcThreads) {
            const int w = i % in.wpr;
            const uint32_t prev = w > 0 ? rows[i - 1] : 0u;
            const uint32_t next = w + 1 < in.wpr ? rows[i + 1] : 0u;
            const uint32_t cur = rows[i];
            hrows[i] = (prev | cur | next) ? hdilate(prev, cur, next, kw, pw) : 0u;  // (most words are empty)
        }
        __syncthreads();
    }
    uint32_t words[WPT];
    int my = 0, mypx = 0;
    // per-group "non-empty" bit at the group's lowest bit position
    auto group_bits = [](uint32_t w) -> uint32_t {
        if (R == 1) return w;
        if (R == 2) return (w | (w >> 1)) & 0x55555555u;
        uint32_t t = w | (w >> 1);
        return (t | (t >> 2)) & 0x11111111u;
    };
    const int y0 = (int)(w0 / out.wpr), wr0 = (int)(w0 - (int64_t)y0 * out.wpr);
    int wy[WPT], ww[WPT];  // row / word of each of the thread's words (kept for the list writes)
#pragma unroll
    for (int i = 0; i < WPT; ++i) {
        int y = y0, w = wr0 + i;
        if (w >= out.wpr) {  // (a thread's WPT words may wrap into the next rows)
            y += w / out.wpr;
            w -= (w / out.wpr) * out.wpr;
        }
        wy[i] = y;
        ww[i] = w;
        uint32_t word = 0;
        if (y < out.H && w < in.wpr) {
            if (identity) {
                word = rows[(y - ra) * in.wpr + w];
            } else {
                const int k0 = max(0, ph - y), k1 = min(kh, in.H + ph - y);
                for (int kj = k0; kj < k1; ++kj) word |= hrows[(y - ph + kj - ra) * in.wpr + w];
            }
        }
        if (y < out.H) {
            const int rem = out.W - 32 * w;
            if (rem < 32) word &= rem > 0 ? ((1u << rem) - 1u) : 0u;
        } else {
            word = 0;
        }
        words[i] = word;
        mypx += __popc(word);
        my += __popc(group_bits(word));
    }
    if (write_out) {
        uint32_t* o = out.d + (int64_t)s * out.stride + w0;
#pragma unroll
        for (int i = 0; i < WPT; ++i) o[i] = words[i];
    }
    if (cnt) {  // changed pixels per stream (a tile never straddles two streams)
        const int wpx = __reduce_add_sync(0xffffffffu, mypx);
        if ((threadIdx.x & 31) == 0 && wpx) atomicAdd(cnt + (int64_t)s * cstride, (unsigned long long)wpx);
    }
    // The block's entries go to a range claimed with ONE atomic on the list
    // counter (zeroed by the frame's scratch memset): no tile waits for
    // another (a decoupled look-back chains the tiles through ~tiles/32 L2
    // round trips). Entries are ascending within a tile and the tiles land in
    // completion order -- the convolutions do not depend on the order (every
    // output pixel is computed from its own receptive field), traces are
    // sorted when read back (extract_indexes order, cbconv.cpp:99-113).
    int agg;
    const int excl = block_scan(my, s_warp, agg);
    if (threadIdx.x == 0) s_base = agg ? atomicAdd(total, agg) : 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    int64_t o = s_base + excl;  // this thread's first entry
    const int Gw = (out.W + R - 1) / R;
    const int64_t sbase = R == 1 ? (int64_t)s * out.H * out.W : (int64_t)s * out.H * Gw;
#pragma unroll
    for (int i = 0; i < WPT; ++i) {
        const uint32_t word = words[i];
        const uint32_t gb = group_bits(word);
        unsigned todo = __ballot_sync(0xffffffffu, gb != 0u);
        while (todo) {  // expand lane src's word with all 32 lanes
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            const uint32_t wsrc = __shfl_sync(0xffffffffu, word, src);
            const uint32_t gsrc = __shfl_sync(0xffffffffu, gb, src);
            const int64_t osrc = __shfl_sync(0xffffffffu, o, src);
            const int ys = __shfl_sync(0xffffffffu, wy[i], src), ws = __shfl_sync(0xffffffffu, ww[i], src);
            const int bit = lane * R;
            if (bit < 32 && ((gsrc >> bit) & 1u)) {
                const int64_t pos = osrc + __popc(gsrc & ((1u << bit) - 1u));
                if (R == 1) {
                    idx[pos] = (int32_t)(sbase + (int64_t)ys * out.W + 32 * ws + lane);
                } else {
                    const int64_t gid = sbase + (int64_t)ys * Gw + (32 * ws) / R + lane;
                    idx[pos] = (int32_t)((gid << 4) | ((wsrc >> bit) & ((1u << R) - 1u)));
                }
            }
        }
        o += __popc(gb);
    }
}

static size_t dc_smem_bytes(const BitMask& in, const BitMask& out, int kh, int wpt) {
    const int rows = (kDcThreads * wpt) / out.wpr + 2 + kh;
    return (2 * ((size_t)rows * in.wpr + 8) + 16) * sizeof(uint32_t);
}

size_t dilate_compact_workspace(const BitMask& out, int S) {
    (void)out;
    (void)S;
    return 256;  // the list counter (the kernel's `total`)
}

template <int WPT, int R>
static void launch_dc_r(BitMask in, BitMask out, bool write_out, int S, int kh, int kw, int ph, int pw, bool identity,
                        int32_t* idx, int* total, unsigned long long* cnt, int cstride, cudaStream_t st) {
    const int64_t tiles = (int64_t)S * (out.stride / (kDcThreads * WPT));
    const size_t smem = dc_smem_bytes(in, out, identity ? 1 : kh, WPT);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(dilate_compact_kernel<WPT, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_k(dilate_compact_kernel<WPT, R>, dim3((unsigned)tiles), dim3(kDcThreads), smem, st, in, out, write_out, kh, kw,
             ph, pw, identity, idx, total, cnt, cstride);
}

template <int WPT>
static void launch_dc(BitMask in, BitMask out, bool write_out, int S, int kh, int kw, int ph, int pw, bool identity,
                      int32_t* idx, int* total, unsigned long long* cnt, int cstride, cudaStream_t st, int R) {
    if (R == 4)
        launch_dc_r<WPT, 4>(in, out, write_out, S, kh, kw, ph, pw, identity, idx, total, cnt, cstride, st);
    else if (R == 2)
        launch_dc_r<WPT, 2>(in, out, write_out, S, kh, kw, ph, pw, identity, idx, total, cnt, cstride, st);
    else
        launch_dc_r<WPT, 1>(in, out, write_out, S, kh, kw, ph, pw, identity, idx, total, cnt, cstride, st);
}

void launch_dilate_compact(BitMask in, BitMask out, bool write_out, int S, int kh, int kw, int ph, int pw,
                           int32_t* idx, int* total, void* workspace, unsigned long long* cnt, int cstride,
                           cudaStream_t st, bool ws_zeroed, int R) {
    (void)workspace;  // (the counter `total` must be zero: ws_zeroed means the caller zeroed it in-stream)
    const bool identity = kh == 1 && kw == 1 && ph == 0 && pw == 0;
    const int64_t words = (int64_t)S * out.stride;
    // enough tiles to cover the SMs twice, at most 8 words per thread
    int wpt = 8;
    while (wpt > 1 && words / (kDcThreads * wpt) < 2 * kNumSMs) wpt /= 2;
    const int64_t tiles = words / (kDcThreads * wpt);
    if (!ws_zeroed) cudaMemsetAsync(total, 0, sizeof(int), st);
    (void)tiles;
    switch (wpt) {
        case 8: launch_dc<8>(in, out, write_out, S, kh, kw, ph, pw, identity, idx, total, cnt, cstride, st, R); break;
        case 4: launch_dc<4>(in, out, write_out, S, kh, kw, ph, pw, identity, idx, total, cnt, cstride, st, R); break;
        case 2: launch_dc<2>(in, out, write_out, S, kh, kw, ph, pw, identity, idx, total, cnt, cstride, st, R); break;
        default: launch_dc<1>(in, out, write_out, S, kh, kw, ph, pw, identity, idx, total, cnt, cstride, st, R); break;
    }
}

// ---------------------------------------------------------------------------
// Generic dilation (any stride): one thread per output word; every output
// pixel ORs its zero-padded receptive field via bit tests.
__global__ void dilate_bits_kernel(BitMask in, BitMask out, int kh, int kw, int sh, int sw, int ph, int pw) {
    pdl_entry();
    const int s = blockIdx.y;
    const int64_t nw = (int64_t)out.H * out.wpr;
    for (int64_t wi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; wi < nw; wi += (int64_t)gridDim.x * blockDim.x) {
        const int y = (int)(wi / out.wpr), w = (int)(wi % out.wpr);
        uint32_t word = 0;
        for (int b = 0; b < 32; ++b) {
            const int x = 32 * w + b;
            if (x >= out.W) break;
            bool any = false;
            for (int kj = 0; kj < kh && !any; ++kj) {
                const int yy = y * sh - ph + kj;
                if (yy < 0 || yy >= in.H) continue;
                for (int ki = 0; ki < kw; ++ki) {
                    const int xx = x * sw - pw + ki;
                    if (xx >= 0 && xx < in.W && bit_test(in, s, yy, xx)) {
                        any = true;
                        break;
                    }
                }
            }
            word |= any ? (1u << b) : 0u;
        }
        out.d[(int64_t)s * out.stride + wi] = word;
    }
}

void launch_dilate_bits(BitMask in, BitMask out, int S, int kh, int kw, int sh, int sw, int ph, int pw,
                        cudaStream_t st) {
    const int64_t nw = (int64_t)out.H * out.wpr;
    int gx = (int)std::min<int64_t>((nw + 127) / 128, 4096);
    launch_k(dilate_bits_kernel, dim3(gx < 1 ? 1 : gx, S), dim3(128), 0, st, in, out, kh, kw, sh, sw, ph, pw);
}

// ---------------------------------------------------------------------------
// K5: max-pool (window/stride) or ReLU (window 1) recomputed for the output
// pixels whose input window holds an updated pixel, compare-before-write
// feeding the next CBCONV's change mask.
//
// Phase 1 (sparse frames, point_scan_kernel): one thread per output word (32
// pixels of a row) forms the touched word from the input grid's updated mask
// with word operations (2x2/2 pooling: OR of two rows, then pairs of bits
// folded together; ReLU: the word itself; other windows: per-bit window
// tests), writes U_out, resets the consumer's change word, and appends the
// touched PIXELS to a flat work list (one atomic per warp).
// Phase 2 (point_work_kernel): a flat grid-stride loop over (pixel, 4-channel)
// items of the list; max-pool (first element seeds the max, then every
// window element, baseline.cpp:134-138) or ReLU (baseline.cpp:115), compare
// with the stored value, store; the change bits of a warp are merged per
// mask word (match + OR-reduce) into one atomicOr, which also yields the
// newly set bits for the per-stream changed-pixel counter.
constexpr int kPtThreads = 256;

// bit j of the result = bit 2j | bit 2j+1 of v (64 -> 32 bits)
__device__ __forceinline__ uint32_t fold_pairs(uint64_t v) {
    v = (v | (v >> 1)) & 0x5555555555555555ull;
    v = (v | (v >> 1)) & 0x3333333333333333ull;
    v = (v | (v >> 2)) & 0x0f0f0f0f0f0f0f0full;
    v = (v | (v >> 4)) & 0x00ff00ff00ff00ffull;
    v = (v | (v >> 8)) & 0x0000ffff0000ffffull;
    v = (v | (v >> 16)) & 0x00000000ffffffffull;
    return (uint32_t)v;
}

__device__ __forceinline__ uint32_t touched_word(const PointBitsArgs& a, int s, int y, int w) {
    const BitMask& u = a.upd_in;
    const uint32_t* row0 = u.d + (int64_t)s * u.stride;
    uint32_t tw = 0;
    if (a.window == 1 && a.stride == 1) {
        tw = row0[(int64_t)y * u.wpr + w];
    } else if (a.window == 2 && a.stride == 2) {
        const uint32_t* r0 = row0 + (int64_t)(2 * y) * u.wpr;
        const uint32_t* r1 = r0 + u.wpr;
        const int w0 = 2 * w, w1 = 2 * w + 1;
        const uint32_t lo = r0[w0] | r1[w0];
        const uint32_t hi = w1 < u.wpr ? (r0[w1] | r1[w1]) : 0u;
        tw = fold_pairs(((uint64_t)hi << 32) | lo);
    } else {
        for (int j = 0; j < 32; ++j) {
            const int x = 32 * w + j;
            bool t = false;
            for (int kj = 0; kj < a.window && !t; ++kj)
                for (int ki = 0; ki < a.window; ++ki) {
                    const int xi = x * a.stride + ki;
                    if (xi < u.W && bit_test(u, s, y * a.stride + kj, xi)) {
                        t = true;
                        break;
                    }
                }
            tw |= t ? (1u << j) : 0u;
        }
    }
    const int rem = a.out.W - 32 * w;  // pixels past the last full window do not exist
    if (rem < 32) tw &= rem > 0 ? ((1u << rem) - 1u) : 0u;
    return tw;
}

// (index arithmetic: every count here is below 2^31 -- launch_point_bits
// checks -- so divisions are multiply-shifts, FastDiv)
__global__ void __launch_bounds__(kPtThreads) point_scan_kernel(PointBitsArgs a, FastDiv fd_plane, FastDiv fd_wpr) {
    pdl_entry();
    const int Ho = a.out.H, Wo = a.out.W;
    const int wpr = (Wo + 31) / 32;
    const int nseg = a.S * Ho * wpr;
    const int lane = threadIdx.x & 31;
    for (int base = blockIdx.x * kPtThreads; base < nseg; base += gridDim.x * kPtThreads) {
        const int seg = base + threadIdx.x;
        uint32_t tw = 0;
        int s = 0, y = 0, w = 0;
        if (seg < nseg) {
            s = (int)fd_plane.div((uint32_t)seg);
            const int r = seg - s * Ho * wpr;
            y = (int)fd_wpr.div((uint32_t)r);
            w = r - y * wpr;
            tw = touched_word(a, s, y, w);
            const int64_t wo = (int64_t)y * wpr + w;
            if (a.U_out.d) a.U_out.d[(int64_t)s * a.U_out.stride + wo] = tw;
            if (a.chg.d) a.chg.d[(int64_t)s * a.chg.stride + wo] = 0u;
        }
        // warp-aggregated append of the touched pixels
        const int n = __popc(tw);
        int incl = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int wtotal = __shfl_sync(0xffffffffu, incl, 31);
        if (!wtotal) continue;
        int wbase = 0;
        if (lane == 31) wbase = atomicAdd(a.work_count, wtotal);
        wbase = __shfl_sync(0xffffffffu, wbase, 31);
        int pos = wbase + incl - n;
        const uint32_t gbase = (uint32_t)((int64_t)s * Ho * Wo + (int64_t)y * Wo + 32 * w);
        while (tw) {
            const int j = __ffs(tw) - 1;
            tw &= tw - 1;
            a.work[pos++] = gbase + (uint32_t)j;
        }
    }
}

template <bool FULL>
__global__ void __launch_bounds__(kPtThreads) point_work_kernel(PointBitsArgs a, FastDiv fd_c4, FastDiv fd_howo,
                                                                FastDiv fd_wo) {
    pdl_entry();
    const int Ho = a.out.H, Wo = a.out.W;
    const int wpr = (Wo + 31) / 32;
    const int c4n = a.in.Cp / 4;
    const int HoWo = Ho * Wo;
    const int npix = FULL ? a.S * HoWo : *a.work_count;
    const int items = npix * c4n;
    const int rowq = a.in.Wp * c4n;
    const int lane = threadIdx.x & 31;
    for (int base = blockIdx.x * kPtThreads; base < items; base += gridDim.x * kPtThreads) {
        const int it = base + threadIdx.x;
        const bool act = it < items;
        bool ch = false;
        uint32_t* waddr = nullptr;
        int s = 0, x = 0;
        if (act) {
            const int pi = (int)fd_c4.div((uint32_t)it);
            const int c4 = it - pi * c4n;
            const uint32_t g = FULL ? (uint32_t)pi : __ldg(a.work + pi);
            s = (int)fd_howo.div(g);
            const int p = (int)(g - (uint32_t)s * (uint32_t)HoWo);
            const int y = (int)fd_wo.div((uint32_t)p);
            x = p - y * Wo;
            const float4* src = reinterpret_cast<const float4*>(
                a.in.d + (int64_t)s * a.in.ss + ((int64_t)(y * a.stride + a.in.hh) * a.in.Wp + x * a.stride + a.in.hw) * a.in.Cp) + c4;
            float4* dst = reinterpret_cast<float4*>(
                a.out.d + (int64_t)s * a.out.ss + ((int64_t)(y + a.out.hh) * a.out.Wp + x + a.out.hw) * a.out.Cp) + c4;
            // the stored value is loaded with the window, so all loads are in flight together
            const float4 o = (!FULL && a.chg.d) ? *dst : make_float4(0.f, 0.f, 0.f, 0.f);
            float4 m = *src;
            if (a.relu) {
                m = make_float4(ref_relu(m.x), ref_relu(m.y), ref_relu(m.z), ref_relu(m.w));
            } else if (a.window == 2) {
                // 2x2 window (the paper's pools): same max sequence as below
                const float4 v01 = src[c4n], v10 = src[rowq], v11 = src[rowq + c4n];
                const float4 w[4] = {m, v01, v10, v11};
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    m = make_float4(ref_max(m.x, w[k].x), ref_max(m.y, w[k].y), ref_max(m.z, w[k].z),
                                    ref_max(m.w, w[k].w));
            } else {
                for (int kj = 0; kj < a.window; ++kj)
                    for (int ki = 0; ki < a.window; ++ki) {
                        const float4 v = src[kj * rowq + ki * c4n];
                        m = make_float4(ref_max(m.x, v.x), ref_max(m.y, v.y), ref_max(m.z, v.z), ref_max(m.w, v.w));
                    }
            }
            if (!FULL && a.chg.d) {
                ch = ref_changed(m.x, o.x, a.tau) | ref_changed(m.y, o.y, a.tau) | ref_changed(m.z, o.z, a.tau) |
                     ref_changed(m.w, o.w, a.tau);
                waddr = a.chg.d + (int64_t)s * a.chg.stride + (int64_t)y * wpr + (x >> 5);
            }
            *dst = m;
            if (a.out16.d) {
                // fp16 operands are only valid below 65504 in magnitude: flag it (the
                // host raises an error when the frame's stats are read)
                if (a.f16_overflow && fmaxf(fmaxf(fabsf(m.x), fabsf(m.y)), fmaxf(fabsf(m.z), fabsf(m.w))) > 65504.0f)
                    atomicOr(a.f16_overflow, 1);
                const __half2 h01 = __floats2half2_rn(m.x, m.y), h23 = __floats2half2_rn(m.z, m.w);
                uint2 hv;
                hv.x = *reinterpret_cast<const uint32_t*>(&h01);
                hv.y = *reinterpret_cast<const uint32_t*>(&h23);
                const int64_t u16 = (int64_t)s * a.out16.ss + ((int64_t)(y + a.out16.hh) * a.out16.Wp + x + a.out16.hw) * a.out16.Cp;
                reinterpret_cast<uint2*>(a.out16.d + u16)[c4] = hv;
                if (a.out16b.d) reinterpret_cast<uint2*>(a.out16b.d + u16 + 2)[c4] = hv;
            }
        }
        if (!FULL && a.chg.d) {
            // one atomicOr per distinct mask word in the warp
            const unsigned peers = __match_any_sync(0xffffffffu, reinterpret_cast<unsigned long long>(waddr));
            const uint32_t bits = __reduce_or_sync(peers, ch ? (1u << (x & 31)) : 0u);
            if (act && bits && lane == __ffs(peers) - 1) {
                const uint32_t old = atomicOr(waddr, bits);
                const uint32_t fresh = bits & ~old;
                if (fresh && a.chg_cnt) atomicAdd(a.chg_cnt + (int64_t)s * a.cnt_stride, (unsigned long long)__popc(fresh));
            }
        }
    }
}

// Single-pass sparse MAXPOOL / RELU: one warp per output row. The lanes form
// the row's touched words (as point_scan), write U_out and the consumer's
// cleared change words, then the warp walks the touched pixels of the row in
// batches of 32 (pixel, 4-channel) items -- window max, compare-before-write,
// store (+ fp16 shadow) -- and collects the row's change bits in registers:
// the warp owns the row's change words, so they are written once, without
// atomics, and counted with one atomic per row. No global work list, no
// second launch, no dependent global round trip between the two phases.
// Rows are processed grid-stride (rows without touched pixels cost the mask
// loads only).
constexpr int kPfWarps = 8;
__global__ void __launch_bounds__(32 * kPfWarps) point_fused_kernel(PointBitsArgs a, FastDiv fd_ho, FastDiv fd_c4) {
    pdl_entry();
    __shared__ uint32_t s_tw[kPfWarps][64];   // touched words of the row (Wo <= 2048)
    __shared__ uint32_t s_ch[kPfWarps][64];   // change bits of the row
    __shared__ int s_pre[kPfWarps][65];       // exclusive prefix of the touched words' popcounts
    const int Ho = a.out.H, Wo = a.out.W;
    const int wpr = (Wo + 31) / 32;
    const int c4n = a.in.Cp / 4;
    const int rowq = a.in.Wp * c4n;
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int nrows = a.S * Ho;
    for (int row = blockIdx.x * kPfWarps + wl; row < nrows; row += gridDim.x * kPfWarps) {
        const int s = (int)fd_ho.div((uint32_t)row);
        const int y = row - s * Ho;
        int ntouched = 0;
        for (int w = lane; w < wpr; w += 32) {
            const uint32_t tw = touched_word(a, s, y, w);
            const int64_t wo = (int64_t)y * wpr + w;
            if (a.U_out.d) a.U_out.d[(int64_t)s * a.U_out.stride + wo] = tw;
            s_tw[wl][w] = tw;
            s_ch[wl][w] = 0u;
            ntouched += __popc(tw);
        }
        ntouched = __reduce_add_sync(0xffffffffu, ntouched);
        __syncwarp();
        if (ntouched) {
            // word prefix counts (<= 64 words: two per lane, one warp scan)
            const int p0 = lane < wpr ? __popc(s_tw[wl][lane]) : 0;
            const int p1 = lane + 32 < wpr ? __popc(s_tw[wl][lane + 32]) : 0;
            int v = p0 + p1, incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            // exclusive prefix of word pairs (lane, lane+32) is not contiguous:
            // scan words 0..31 and 32..63 separately
            int i0 = p0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, i0, o);
                if (lane >= o) i0 += t;
            }
            const int tot0 = __shfl_sync(0xffffffffu, i0, 31);
            int i1 = p1;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, i1, o);
                if (lane >= o) i1 += t;
            }
            s_pre[wl][lane] = i0 - p0;
            s_pre[wl][lane + 32] = tot0 + i1 - p1;
            if (lane == 0) s_pre[wl][64] = ntouched;
            (void)incl;
            __syncwarp();
        }
        if (ntouched) {
            // items (pixel j of the row's touched list, channel quad c4),
            // 32 at a time; pixel j is found by a warp-wide prefix over words
            const int items = ntouched * c4n;
            for (int i0 = 0; i0 < items; i0 += 32) {
                const int it = i0 + lane;
                bool ch = false;
                int x = 0;
                if (it < items) {
                    const int j = (int)fd_c4.div((uint32_t)it);
                    const int c4 = it - j * c4n;
                    // the j-th set bit of the row: binary search of the word
                    // prefix counts, then the n-th set bit of the word
                    int lo = 0, hi = wpr - 1;
                    while (lo < hi) {
                        const int mid = (lo + hi + 1) >> 1;
                        if (s_pre[wl][mid] <= j) lo = mid; else hi = mid - 1;
                    }
                    const int w = lo;
                    x = 32 * w + (int)__fns(s_tw[wl][w], 0, j - s_pre[wl][w] + 1);
                    const float4* src = reinterpret_cast<const float4*>(
                        a.in.d + (int64_t)s * a.in.ss +
                        ((int64_t)(y * a.stride + a.in.hh) * a.in.Wp + x * a.stride + a.in.hw) * a.in.Cp) + c4;
                    float4* dst = reinterpret_cast<float4*>(
                        a.out.d + (int64_t)s * a.out.ss + ((int64_t)(y + a.out.hh) * a.out.Wp + x + a.out.hw) * a.out.Cp) + c4;
                    const float4 o = a.chg.d ? *dst : make_float4(0.f, 0.f, 0.f, 0.f);
                    float4 m = *src;
                    if (a.relu) {
                        m = make_float4(ref_relu(m.x), ref_relu(m.y), ref_relu(m.z), ref_relu(m.w));
                    } else if (a.window == 2) {
                        const float4 v01 = src[c4n], v10 = src[rowq], v11 = src[rowq + c4n];
                        const float4 wv[4] = {m, v01, v10, v11};
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            m = make_float4(ref_max(m.x, wv[k].x), ref_max(m.y, wv[k].y), ref_max(m.z, wv[k].z),
                                            ref_max(m.w, wv[k].w));
                    } else {
                        for (int kj = 0; kj < a.window; ++kj)
                            for (int ki = 0; ki < a.window; ++ki) {
                                const float4 v = src[kj * rowq + ki * c4n];
                                m = make_float4(ref_max(m.x, v.x), ref_max(m.y, v.y), ref_max(m.z, v.z),
                                                ref_max(m.w, v.w));
                            }
                    }
                    if (a.chg.d)
                        ch = ref_changed(m.x, o.x, a.tau) | ref_changed(m.y, o.y, a.tau) |
                             ref_changed(m.z, o.z, a.tau) | ref_changed(m.w, o.w, a.tau);
                    *dst = m;
                    if (a.out16.d) {
                        if (a.f16_overflow && fmaxf(fmaxf(fabsf(m.x), fabsf(m.y)), fmaxf(fabsf(m.z), fabsf(m.w))) > 65504.0f)
                            atomicOr(a.f16_overflow, 1);
                        const __half2 h01 = __floats2half2_rn(m.x, m.y), h23 = __floats2half2_rn(m.z, m.w);
                        uint2 hv;
                        hv.x = *reinterpret_cast<const uint32_t*>(&h01);
                        hv.y = *reinterpret_cast<const uint32_t*>(&h23);
                        const int64_t u16 = (int64_t)s * a.out16.ss +
                                            ((int64_t)(y + a.out16.hh) * a.out16.Wp + x + a.out16.hw) * a.out16.Cp;
                        reinterpret_cast<uint2*>(a.out16.d + u16)[c4] = hv;
                        if (a.out16b.d) reinterpret_cast<uint2*>(a.out16b.d + u16 + 2)[c4] = hv;
                    }
                }
                if (a.chg.d && ch) atomicOr(&s_ch[wl][x >> 5], 1u << (x & 31));  // (shared memory)
            }
            __syncwarp();
        }
        if (a.chg.d) {
            int nch = 0;
            for (int w = lane; w < wpr; w += 32) {
                const uint32_t c = s_ch[wl][w];
                a.chg.d[(int64_t)s * a.chg.stride + (int64_t)y * wpr + w] = c;
                nch += __popc(c);
            }
            nch = __reduce_add_sync(0xffffffffu, nch);
            if (lane == 0 && nch && a.chg_cnt) atomicAdd(a.chg_cnt + (int64_t)s * a.cnt_stride, (unsigned long long)nch);
        }
        __syncwarp();
    }
}

void launch_point_bits(const PointBitsArgs& a, cudaStream_t st) {
    const int wpr = (a.out.W + 31) / 32;
    const int64_t nseg = (int64_t)a.S * a.out.H * wpr;
    const int c4n = a.in.Cp / 4;
    if ((int64_t)a.S * a.out.H * a.out.W * c4n >= ((int64_t)1 << 31) || nseg * 32 >= ((int64_t)1 << 31))
        throw std::runtime_error("pooling: more than 2^31 items per frame");
    const FastDiv fd_c4 = FastDiv::make((uint32_t)c4n), fd_howo = FastDiv::make((uint32_t)(a.out.H * a.out.W)),
                  fd_wo = FastDiv::make((uint32_t)a.out.W), fd_plane = FastDiv::make((uint32_t)(a.out.H * wpr)),
                  fd_wpr = FastDiv::make((uint32_t)wpr);
    if (!a.upd_in.d) {  // full frame: every pixel, no change test (the next layer evaluates in full)
        const int64_t items = (int64_t)a.S * a.out.H * a.out.W * c4n;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((items + kPtThreads - 1) / kPtThreads, (int64_t)kNumSMs * 16));
        launch_k(point_work_kernel<true>, dim3(grid), dim3(kPtThreads), 0, st, a, fd_c4, fd_howo, fd_wo);
        return;
    }
    static const bool two_pass = std::getenv("CBX_POOL_TWO_PASS") != nullptr;  // (tuning: the scan + work pair)
    // (one warp walks a row's items serially, a dependent load round trip
    // per 32 items: it wins for 4-channel rows -- pool 1: 28 -> 19 us per
    // 8 x 1080p lane-frame -- and loses for wide ones -- pool 2's 52
    // channels: 36 -> 92 us --, which keep the scan + flat work-list pair)
    if (!two_pass && wpr <= 64 && c4n == 1) {
        const int nrows = a.S * a.out.H;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((nrows + kPfWarps - 1) / kPfWarps, (int64_t)kNumSMs * 16));
        launch_k(point_fused_kernel, dim3(grid), dim3(32 * kPfWarps), 0, st, a, FastDiv::make((uint32_t)a.out.H), fd_c4);
        return;
    }
    if (!a.count_zeroed) cudaMemsetAsync(a.work_count, 0, sizeof(int), st);
    const int g1 = (int)std::max<int64_t>(1, std::min<int64_t>((nseg + kPtThreads - 1) / kPtThreads, (int64_t)kNumSMs * 8));
    launch_k(point_scan_kernel, dim3(g1), dim3(kPtThreads), 0, st, a, fd_plane, fd_wpr);
    launch_k(point_work_kernel<false>, dim3(kNumSMs * 8), dim3(kPtThreads), 0, st, a, fd_c4, fd_howo, fd_wo);
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) classify_bits_kernel(TensorView in, BitMask upd, uint16_t* labels, int S) {
    pdl_entry();
    const int H = in.H, W = in.W;
    const int64_t HW = (int64_t)H * W, total = HW * S;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int s = (int)(i / HW);
        const int p = (int)(i - (int64_t)s * HW);
        const int y = p / W, x = p - (p / W) * W;
        if (upd.d && !bit_test(upd, s, y, x)) continue;
        const float* src = in.d + (int64_t)s * in.ss + ((int64_t)(y + in.hh) * in.Wp + x + in.hw) * in.Cp;
        int best = 0;
        float bv = src[0];
        for (int c = 1; c < in.C; ++c) {
            const float v = src[c];
            if (v > bv) {
                bv = v;
                best = c;
            }
        }
        labels[i] = (uint16_t)best;
    }
}

void launch_classify_bits(TensorView in, BitMask upd, uint16_t* labels, int S, cudaStream_t st) {
    const int64_t total = (int64_t)in.H * in.W * S;
    int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)kNumSMs * 16);
    launch_k(classify_bits_kernel, dim3(grid < 1 ? 1 : grid), dim3(256), 0, st, in, upd, labels, S);
}

// Per-stream number of set bits of a mask (analyze-prop worst-case counts).
__global__ void popcount_bits_kernel(BitMask m, unsigned long long* out) {
    const int s = blockIdx.y;
    const int64_t nw = (int64_t)m.H * m.wpr;
    unsigned long long c = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += (int64_t)gridDim.x * blockDim.x)
        c += __popc(m.d[(int64_t)s * m.stride + i]);
    c = __reduce_add_sync(0xffffffffu, (unsigned)c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out + s, c);
}

void launch_popcount_bits(BitMask m, int S, unsigned long long* out, cudaStream_t st) {
    const int64_t nw = (int64_t)m.H * m.wpr;
    const int gx = (int)std::max<int64_t>(1, std::min<int64_t>((nw + 255) / 256, 256));
    popcount_bits_kernel<<<dim3(gx, S), 256, 0, st>>>(m, out);
}

// Unpacks one stream of a bit mask into bytes (trace readback).
__global__ void unpack_bits_kernel(BitMask m, int s, uint8_t* out) {
    const int64_t n = (int64_t)m.H * m.W;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int y = (int)(i / m.W), x = (int)(i % m.W);
        out[i] = bit_test(m, s, y, x) ? 1 : 0;
    }
}

void launch_unpack_bits(BitMask m, int s, uint8_t* out, cudaStream_t st) {
    const int64_t n = (int64_t)m.H * m.W;
    int grid = (int)std::min<int64_t>((n + 255) / 256, 4096);
    unpack_bits_kernel<<<grid < 1 ? 1 : grid, 256, 0, st>>>(m, s, out);
}

}  // namespace cbx
