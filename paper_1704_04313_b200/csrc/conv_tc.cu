// conv_tc.cu -- gathered ("sparse") convolution on the 5th-generation tensor
// cores (tcgen05, kind::tf32, fp32 accumulation in TMEM).
//
// Replaces gen_x_reduced + gemm + update_output
// (/root/reference/proj/core/src/cbconv.cpp:115-155, baseline.cpp:47-63) for
// every convolution whose input is a channels-last device tensor:
//
//   Y[n, o] = bias[o] + sum_K X[n, K] * W[o, K],  n over the change-index list
//
// * M = 128 output pixels per tile (one tile = 128 consecutive entries of the
//   ascending index list, or of all pixels in full mode). A is the im2col of
//   those pixels, GATHERED straight into shared memory: 4 producer warps, one
//   thread per tile row, 16-byte cp.async per (tap, 4-channel) chunk of the
//   zero-halo HWC input, written in the canonical K-major SWIZZLE_128B layout
//   the UMMA descriptor expects (chunk j of row r at slot j ^ (r & 7)). K is
//   ordered (kj, ki, c) and blocked by 32 tf32 values (128 B per row per
//   K-block); chunks past the real K are zero-filled.
// * B = the filter bank, pre-arranged on the host into exactly the smem image
//   of every K-block (N_pad rows x 128 B, swizzled, tf32-rounded), loaded with
//   one cp.async.bulk per stage that completes on the stage's mbarrier.
// * The MMA warp runs its loop converged; one elect.sync lane issues
//   tcgen05.mma (M=128, N<=256 per instruction; two instructions when
//   N_pad > 256, e.g. 304 = 128 + 176) into a TMEM accumulator;
//   tcgen05.commit releases smem stages and hands finished accumulators to
//   the epilogue. Persistent CTAs walk tiles; with N_pad <= 256 the
//   accumulator is double-buffered so the epilogue of tile t overlaps the
//   MMAs of tile t+1, wider layers split it (shared head columns + a tail
//   region per tile parity, see make_tc_layer).
// * Epilogue (4 warps, thread = TMEM lane = tile row): tcgen05.ld 32 columns at
//   a time, + bias, fused ReLU, compare with the value being overwritten
//   (next CBCONV's change detection, cbconv.cpp:66-67), in-place scatter into
//   the persistent output tensor (update_output without the full copy).
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_fp16.h>

#include "conv_tc.hpp"
#include "engine.hpp"
#include "tc_ptx.cuh"

namespace cbx {

namespace {

using namespace tc;

constexpr int kKBlock = 32;        // tf32 elements per K-block (128 B per row)
constexpr int kChunksPerKB = 8;    // 16-byte chunks per K-block row
constexpr int kABytes = tc::kTileM * 128;
constexpr int kEpiThreads = 128, kProdThreads = 128;
constexpr int kThreads = kEpiThreads + kProdThreads + 32;
constexpr int kMaxSmem = 232448;   // 227 KB opt-in

// Output pixel of list entry g: stream s, linear pixel p = y*Wo + x.
struct TcArgs;
template <class A>
__device__ __forceinline__ void pixel_of(const A& a, int64_t g, int64_t HoWo, int& s, int& p, int& y, int& x) {
    if (a.fast) {
        const uint32_t gg = (uint32_t)g;
        const uint32_t ss = a.fd_howo.div(gg);
        const uint32_t pp = gg - ss * (uint32_t)HoWo;
        const uint32_t yy = a.fd_wo.div(pp);
        s = (int)ss;
        p = (int)pp;
        y = (int)yy;
        x = (int)(pp - yy * (uint32_t)a.Wo);
    } else {
        s = (int)(g / HoWo);
        p = (int)(g - (int64_t)s * HoWo);
        y = p / a.Wo;
        x = p - y * a.Wo;
    }
}

// List entry n of a launch: the list's value, or in full mode the pixel index
// n / the group entry (n << 4 | mask of the group's pixels inside the row).
template <class A>
__device__ __forceinline__ int64_t entry_at(const A& a, int64_t n) {
    if (a.idx) return (int64_t)__ldg(a.idx + n);
    if (a.grp_R <= 1) return n;
    const uint32_t gid = (uint32_t)n;
    const uint32_t rem = gid - a.fd_gplane.div(gid) * (uint32_t)(a.Ho * a.Gw);
    const int x0 = (int)(rem - a.fd_gw.div(rem) * (uint32_t)a.Gw) * a.grp_R;
    return (n << 4) | ((1 << min(a.grp_R, a.Wo - x0)) - 1);
}

// Group entry -> stream, output row, first output column.
template <class A>
__device__ __forceinline__ void group_of_tc(const A& a, int64_t e, int& s, int& y, int& x0) {
    const uint32_t gid = (uint32_t)(e >> 4);
    const uint32_t ss = a.fd_gplane.div(gid);
    const uint32_t rem = gid - ss * (uint32_t)(a.Ho * a.Gw);
    const uint32_t yy = a.fd_gw.div(rem);
    s = (int)ss;
    y = (int)yy;
    x0 = (int)(rem - yy * (uint32_t)a.Gw) * a.grp_R;
}

// Remaining per-pixel ops of a fused tail (after the first 1x1 CONV, whose
// outputs arrive in `cur`): RELU (ref_relu), 1x1 CONV (bias-first, ascending
// channel order, one rounding per multiply and add -- the reference gemm
// order), then the final activation is stored and argmax-classified with the
// reference tie rule (strict >, lowest channel wins).
template <int TC>
__device__ __forceinline__ void run_tail(const TcTail& t, float (&cur)[TC], int s, int y, int x, int p) {
    int C = t.cout[0];
    for (int k = 1; k < t.n; ++k) {
        if (t.kind[k] == 1) {
#pragma unroll
            for (int q = 0; q < TC; ++q) cur[q] = ref_relu(cur[q]);
        } else {
            const int O = t.cout[k];
            float nxt[TC];
#pragma unroll
            for (int q = 0; q < TC; ++q) {
                float acc = (q < O) ? __ldg(t.b[k] + q) : 0.0f;
#pragma unroll
                for (int c = 0; c < TC; ++c)
                    if (q < O && c < C) acc = __fadd_rn(acc, __fmul_rn(__ldg(t.W[k] + q * C + c), cur[c]));
                nxt[q] = acc;
            }
#pragma unroll
            for (int q = 0; q < TC; ++q) cur[q] = nxt[q];
            C = O;
        }
    }
    float* fo = t.final_out + (int64_t)s * t.fo_ss + ((int64_t)(y + t.fo_hh) * t.fo_Wp + (x + t.fo_hw)) * t.fo_Cp;
    int best = 0;
    float bv = cur[0];
#pragma unroll
    for (int q = 0; q < TC; ++q) {
        if (q < C) {
            fo[q] = cur[q];
            if (q > 0 && cur[q] > bv) {
                bv = cur[q];
                best = q;
            }
        }
    }
    t.labels[(int64_t)s * t.l_ss + p] = (uint16_t)best;
}

struct TcArgs {
    const float* in;
    int64_t in_ss;
    int in_Wp, in_Cp, in_hh, in_hw;
    float* out;
    int64_t out_ss;
    int out_Wp, out_Cp, out_hh, out_hw;
    int O, Ho, Wo;
    int kh, kw, sh, sw, ph, pw;
    const int32_t* idx;
    const int* count;
    int64_t full_count;
    const float* Bw;     // [ranks][NKB][Brows][32] swizzled smem images
    const float* bias;   // [O]
    int NKB, Npad, N0, N1;
    int Brows;           // filter rows held per CTA (Npad, or Npad/2 for a CTA pair)
    int stages, acc_stages, acc_cols, tmem_cols;
    // split accumulator (N_pad > 256, single CTA): the first instruction's N0
    // channels always land in the shared columns [ovl_s, ovl_s + N0), the
    // second's alternate between ovl_b[0] and ovl_b[1] by tile parity, so the
    // next tile's MMAs wait only for the shared columns to be drained
    int ovl, ovl_s, ovl_b0, ovl_b1;
    int tap4x7;  // row-lane gather specialised for Cp = 4, 7x7 (NKB = 7)
    int xrow;    // row-lane gather of 4-channel inputs as 8 rows x 4 chunks per warp instruction
    // kind::i8 (8-bit camera path, layer 1): A = RGBX bytes of the frame, one
    // 4-byte chunk per tap (32 taps per K-block); B = the filters as three
    // signed base-256 digits per weight, digit q of channel j in accumulator
    // column q * i8_opad + j; y_j = bias_j + qsc[j] * (A2 * 65536 + A1 * 256 + A0)
    int i8_opad;
    const float* qsc;
    // pixel index -> (stream, y, x) by multiply-shift when S*Ho*Wo < 2^31
    int fast;
    FastDiv fd_howo, fd_wo;
    // pixel groups (grp_R > 1, stride-1 layers with a 4-channel input): an A
    // row is R horizontally adjacent output pixels, K its union window
    // (kh x (kw + R - 1) taps), N = R x grp_N (sub-pixel j's channels at
    // columns j * grp_N); list entries (gid << 4 | mask), gid over Ho x Gw
    int grp_R, grp_N, Gw;
    FastDiv fd_gplane, fd_gw;
    // packed fp16 input (pack_cpr > 0): channels not padded, each kernel row's
    // kw x C halves gathered as pack_cpr contiguous 16-byte chunks (the last
    // may run into the next pixel: zero weights there); `in2` is the same
    // shadow shifted by 8 bytes, used for windows that start 8-byte aligned
    int pack_cpr;
    const float* in2;
    int kinst_last;  // MMA instructions of the last K-block (its 32-byte K steps that hold data)
    int f16;     // operands are fp16 (kind::f16): the input is an fp16 shadow tensor
                 // addressed in 4-byte units (in_Cp = fp16 channels / 2)
    int relu;
    BitMask chg;
    float tau;
    unsigned long long* chg_cnt;
    int cnt_stride;
    int write_out;  // store this layer's output tensor (off when a fused tail consumes it)
    float one, nzero;  // 1.0f / -0.0f as runtime values (paired-fp32 rounding, common.cuh)
    int tail_w_floats;  // shared memory reserved for the first tail conv's filters
    TcTail tail;
};

// Epilogue of one 32-column TMEM chunk for one pixel: + bias, fused ReLU,
// the first tail 1x1 conv accumulated in ascending channel order, and (when
// the layer output is kept) compare-before-write against the stored value.
// FULL: all 32 channels exist, so every loop is branch-free and the shared
// memory loads of bias / tail filters can be hoisted ahead of their use.
// t1p: the first tail conv's TC accumulators as TC/2 packed fp32 pairs.
template <int TC>
using TailAcc = unsigned long long[TC > 1 ? TC / 2 : 1];

template <int TC, bool FULL>
__device__ __forceinline__ void epi_chunk(const TcArgs& a, float (&v)[32], int c0, int nv, const float* sBias,
                                          const float* sTailW, TailAcc<TC>& t1p, float* dst, bool& changed) {
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
        if (!FULL && j >= nv) break;
        const float4 b4 = *reinterpret_cast<const float4*>(sBias + c0 + j);
        const float bb[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float t = (FULL || j + e < nv) ? __fadd_rn(v[j + e], bb[e]) : 0.0f;
            v[j + e] = a.relu ? ref_relu(t) : t;
        }
    }
    if constexpr (TC > 0) {
        // the TC filters of one channel are TC/4 broadcast LDS.128 = TC/2
        // packed pairs; two output channels per paired-fp32 step, each with
        // the reference's two roundings (common.cuh)
        const unsigned long long one2 = f2_pack(a.one, a.one), nz2 = f2_pack(a.nzero, a.nzero);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            if (!FULL && j >= nv) break;
            const ulonglong2* w = reinterpret_cast<const ulonglong2*>(sTailW + (c0 + j) * TC);
            const unsigned long long vv = f2_pack(v[j], v[j]);
#pragma unroll
            for (int q4 = 0; q4 < TC / 4; ++q4) {
                const ulonglong2 wq = w[q4];
                t1p[2 * q4 + 0] = f2_fma(f2_fma(wq.x, vv, nz2), one2, t1p[2 * q4 + 0]);
                t1p[2 * q4 + 1] = f2_fma(f2_fma(wq.y, vv, nz2), one2, t1p[2 * q4 + 1]);
            }
        }
    }
    if (!a.write_out) return;
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
        if (!FULL && j >= nv) break;
        const int o = c0 + j;
        if (FULL || j + 3 < nv) {
            float4* q = reinterpret_cast<float4*>(dst + o);
            if (a.chg.d) {
                const float4 old = *q;
                changed |= ref_changed(v[j], old.x, a.tau) | ref_changed(v[j + 1], old.y, a.tau) |
                           ref_changed(v[j + 2], old.z, a.tau) | ref_changed(v[j + 3], old.w, a.tau);
            }
            *q = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if (j + e < nv) {
                    if (a.chg.d) changed |= ref_changed(v[j + e], dst[o + e], a.tau);
                    dst[o + e] = v[j + e];
                }
            }
        }
    }
}

// ROWLANE: producer thread = tile row (each lane gathers its own pixel; best
// when a pixel's taps are 16 B, i.e. 4 channels, so a warp's 32 rows of one
// tap are 32 neighbouring pixels). Otherwise 8 lanes cooperate on a row's 128
// contiguous K-block bytes and a warp instruction covers 4 rows.
//
// PAIR: the CTA pair of a 2-CTA cluster (the two SMs of one TPC) runs one
// M=256 tcgen05.mma.cta_group::2: each CTA gathers its own 128 pixel rows (A)
// and holds HALF of the filter bank (B: N/2 rows per instruction), so every
// SM streams 16 KB of A + Npad*64 B of B per K-block instead of
// 16 KB + Npad*128 B -- the filter bytes, which dominate wide layers
// (Npad = 304: 39 KB vs 16 KB of A), are halved in L2 traffic and in shared
// memory. The leader (cluster rank 0) issues the MMAs; the peer's stage-full
// state reaches it through a relay thread (cp.async completions can only
// arrive on a CTA-local mbarrier), and the leader's commits are multicast to
// both CTAs' empty / accumulator-full barriers. Each CTA's TMEM holds the
// accumulator rows of its own 128 pixels, so the epilogue is unchanged.
template <bool ROWLANE, int TC, bool PAIR, bool I8 = false>
__global__ void __launch_bounds__(kThreads, PAIR ? 1 : 2) conv_tc_kernel(TcArgs a) {
    pdl_trigger();  // (the prologue below touches only this launch's constants)
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // align by offsetting the shared array itself (not via an integer round
    // trip), so the compiler keeps emitting LDS/STS for the smem tables below
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int NS = a.stages;
    const uint32_t b_bytes = (uint32_t)a.Brows * 128u;
    uint8_t* sA = smem;                                  // NS x 16 KB
    uint8_t* sB = sA + (size_t)NS * kABytes;             // NS x b_bytes
    // NKB*8 chunk offsets (floats); I8: NKB*32 tap offsets (4-byte units)
    const int tab_n = I8 ? 0 : a.NKB * kChunksPerKB;
    int* sTab = reinterpret_cast<int*>(sB + (size_t)NS * b_bytes);
    float* sBias = reinterpret_cast<float*>(sTab + tab_n);
    float* sTailW = sBias + ((a.O + 3) & ~3);  // first tail conv's filters, transposed [O][TC] (16B aligned)
    float* sQs = sTailW + a.tail_w_floats;
    uint64_t* bars = reinterpret_cast<uint64_t*>(
        (reinterpret_cast<uintptr_t>(sQs + (I8 ? a.O : 0)) + 7) & ~uintptr_t(7));
    uint64_t* full = bars;
    uint64_t* empty = full + NS;
    uint64_t* pfull = empty + NS;  // PAIR, leader only: the peer's stage is full
    uint64_t* tfull = pfull + NS;
    uint64_t* tempty = tfull + 2;
    uint64_t* tshared = tempty + 2;  // ovl: the shared columns of the last tile are drained
    uint32_t* sTmem = reinterpret_cast<uint32_t*>(tshared + 1);

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int C4 = a.in_Cp >> 2;
    const int nchunks = a.kh * a.kw * C4;
    const uint32_t crank = PAIR ? cluster_rank() : 0u;
    const int64_t tile_first = PAIR ? (int64_t)cluster_id_x() : (int64_t)blockIdx.x;
    const int64_t tile_step = PAIR ? (int64_t)nclusters_x() : (int64_t)gridDim.x;
    constexpr int kRowsPerTile = PAIR ? 2 * tc::kTileM : tc::kTileM;
    const int64_t row_off = (int64_t)crank * tc::kTileM;  // this CTA's rows within a tile
    const float* Bw = a.Bw + (size_t)crank * a.NKB * a.Brows * kKBlock;

    // ---- setup
    for (int j = tid; j < tab_n; j += kThreads) {
        int off = -1;
        if (I8) {
            // (unused: the register-staged gather computes its offsets)
        } else if (a.pack_cpr > 0) {
            if (j < a.kh * a.pack_cpr) {
                const int kj = j / a.pack_cpr, i = j - kj * a.pack_cpr;
                off = kj * a.in_Wp * a.in_Cp + 4 * i;  // 4-byte units from the window origin
            }
        } else if (a.grp_R > 1) {
            const int span = a.kw + a.grp_R - 1;  // window columns per kernel row
            if (j < a.kh * span * C4) {
                const int tap = j / C4, c4 = j - tap * C4;
                const int kj = tap / span, w = tap - kj * span;
                off = (kj * a.in_Wp + w) * a.in_Cp + c4 * 4;
            }
        } else if (j < nchunks) {
            const int tap = j / C4, c4 = j - tap * C4;
            const int kj = tap / a.kw, ki = tap - kj * a.kw;
            off = (kj * a.in_Wp + ki) * a.in_Cp + c4 * 4;
        }
        sTab[j] = off;
    }
    for (int o = tid; o < a.O; o += kThreads) sBias[o] = a.bias[o];
    if (I8)
        for (int o = tid; o < a.O; o += kThreads) sQs[o] = a.qsc[o];
    if (TC > 0) {
        const int c1 = a.tail.cout[0];
        for (int i = tid; i < a.O * TC; i += kThreads) {
            const int o = i / TC, q = i - o * TC;
            sTailW[i] = q < c1 ? a.tail.W[0][q * a.O + o] : 0.0f;
        }
    }
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], kProdThreads + 1);
            mbar_init(&empty[s], 1);
            mbar_init(&pfull[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], PAIR ? 2 * (kEpiThreads / 32) : kEpiThreads);
        }
        mbar_init(tshared, PAIR ? 2 * (kEpiThreads / 32) : kEpiThreads);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 8) {
        if constexpr (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(sTmem)),
                         "r"(a.tmem_cols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(sTmem)),
                         "r"(a.tmem_cols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    tc_fence_before();
    if constexpr (PAIR) cluster_sync_all(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *sTmem;

    pdl_wait();  // the index list / count and the input tensor come from the previous kernels
    const int64_t total = a.idx ? (int64_t)*a.count : a.full_count;
    const int64_t ntiles = (total + kRowsPerTile - 1) / kRowsPerTile;
    const int64_t HoWo = (int64_t)a.Ho * a.Wo;

    if (warp >= 4 && warp < 8) {
        // ================= producers =================
        if constexpr (I8) {
            // RGBX bytes, register-staged: thread = tile row. Kernel row kr's
            // kw taps are kw neighbouring 4-byte pixels (consecutive lanes
            // read consecutive pixels: coalesced LDG.32), padded with zero
            // words to kwp = 8 taps (two 16-byte granules, the padding tap has
            // zero weights), written with STS.128 into the SW128 K-major row
            // (granule g of row r at g ^ (r & 7): conflict-free), then made
            // visible to the tensor core (fence.proxy.async) before the
            // stage's barrier arrive. 4 kernel rows per 128-byte K-block.
            const int r = tid - kEpiThreads;
            const uint32_t swz = (uint32_t)(r & 7);
            Ring rg;
            auto row_index = [&](int64_t t) -> int64_t {
                const int64_t n = t * kRowsPerTile + r;
                return (t < ntiles && n < total) ? (a.idx ? (int64_t)__ldg(a.idx + n) : n) : -1;
            };
            int64_t gnext = row_index(tile_first);
            for (int64_t tile = tile_first; tile < ntiles; tile += tile_step) {
                const int64_t g = gnext;
                gnext = row_index(tile + tile_step);
                const bool valid = g >= 0;
                const uint32_t* base = reinterpret_cast<const uint32_t*>(a.in);
                if (valid) {
                    int s, p, y, x;
                    pixel_of(a, g, HoWo, s, p, y, x);
                    base += (int64_t)s * a.in_ss + ((int64_t)(y * a.sh - a.ph + a.in_hh) * a.in_Wp + (x * a.sw - a.pw + a.in_hw));
                }
                for (int kb = 0; kb < a.NKB; ++kb, rg.next(NS)) {
                    const uint32_t st = rg.st, ph = rg.ph;
                    uint32_t v[4][8];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int kr = 4 * kb + q;
#pragma unroll
                        for (int ki = 0; ki < 8; ++ki)
                            v[q][ki] = (valid && kr < a.kh && ki < a.kw) ? __ldg(base + (int64_t)kr * a.in_Wp + ki) : 0u;
                    }
                    mbar_wait(&empty[st], ph ^ 1u);
                    if (r == 0) {
                        mbar_arrive_expect_tx(&full[st], b_bytes);
                        bulk_g2s(sB + (size_t)st * b_bytes, Bw + (size_t)kb * a.Brows * kKBlock, b_bytes, &full[st]);
                    }
                    uint4* row = reinterpret_cast<uint4*>(sA + (size_t)st * kABytes + r * 128);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        row[(2 * q) ^ swz] = make_uint4(v[q][0], v[q][1], v[q][2], v[q][3]);
                        row[(2 * q + 1) ^ swz] = make_uint4(v[q][4], v[q][5], v[q][6], v[q][7]);
                    }
                    fence_proxy_async();
                    mbar_arrive(&full[st]);
                }
            }
        } else if constexpr (ROWLANE) {
          if (a.xrow) {
            // 4-channel input (one 16-byte chunk per tap), shared-memory
            // conflict-free: a warp instruction copies 8 tile rows x 4
            // consecutive chunks -- the 8 rows' swizzled positions
            // (j ^ (r & 7)) are distinct, so its 32 x 16 bytes land in 4
            // wavefronts (thread-per-row LDGSTS hit 8 bank groups 4 ways:
            // 16 wavefronts, and the L2 conv was bound by it). Lane l: rows
            // 32w + 8i + (l & 7), i < 4; chunks 4h + (l >> 3), h < 2.
            const int pw = warp - 4, e = lane >> 3, rl = lane & 7;
            Ring rg;
            auto load_rows = [&](int64_t t, int64_t (&gr)[4]) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int64_t n = t * kRowsPerTile + row_off + 32 * pw + 8 * i + rl;
                    gr[i] = (t < ntiles && n < total) ? (a.idx ? (int64_t)__ldg(a.idx + n) : n) : -1;
                }
            };
            int64_t gnext4[4];
            load_rows(tile_first, gnext4);
            for (int64_t tile = tile_first; tile < ntiles; tile += tile_step) {
                const float* base[4];
                uint32_t vmask = 0;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    base[i] = a.in;
                    if (gnext4[i] >= 0) {
                        int s, p, y, x;
                        pixel_of(a, gnext4[i], HoWo, s, p, y, x);
                        vmask |= 1u << i;
                        base[i] = a.in + (int64_t)s * a.in_ss +
                                  ((int64_t)(y * a.sh - a.ph + a.in_hh) * a.in_Wp + (x * a.sw - a.pw + a.in_hw)) * a.in_Cp;
                    }
                }
                load_rows(tile + tile_step, gnext4);
                for (int kb = 0; kb < a.NKB; ++kb, rg.next(NS)) {
                    const uint32_t st = rg.st, ph = rg.ph;
                    mbar_wait(&empty[st], ph ^ 1u);
                    if (pw == 0 && lane == 0) {
                        mbar_arrive_expect_tx(&full[st], b_bytes);
                        bulk_g2s(sB + (size_t)st * b_bytes, Bw + (size_t)kb * a.Brows * kKBlock, b_bytes, &full[st]);
                    }
                    const uint32_t stage = smem_u32(sA + (size_t)st * kABytes);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int j = 4 * h + e;
                        const int off = sTab[kb * kChunksPerKB + j];
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const int r = 32 * pw + 8 * i + rl;
                            if ((vmask >> i) & 1u)
                                cp_async16(stage + r * 128 + ((j ^ rl) << 4), off >= 0 ? base[i] + off : a.in,
                                           off >= 0 ? 16u : 0u);
                        }
                    }
                    cp_async_arrive_noinc(&full[st]);
                }
            }
          } else {
            const int r = tid - kEpiThreads;
            const uint32_t swz = (uint32_t)(r & 7);
            Ring rg;
            // the next tile's index is loaded while this tile's K-blocks are
            // gathered, so a tile never starts with a dependent index load
            auto row_index = [&](int64_t t) -> int64_t {
                const int64_t n = t * kRowsPerTile + row_off + r;
                return (t < ntiles && n < total) ? entry_at(a, n) : -1;
            };
            int64_t gnext = row_index(tile_first);
            for (int64_t tile = tile_first; tile < ntiles; tile += tile_step) {
                const int64_t g = gnext;
                gnext = row_index(tile + tile_step);
                const bool valid = g >= 0;
                const float* base = a.in;
                if (valid) {
                    int s, p, y, x;
                    if (a.grp_R > 1) {  // the group's window: stride 1, columns from x0 - pw
                        group_of_tc(a, g, s, y, x);
                    } else {
                        pixel_of(a, g, HoWo, s, p, y, x);
                    }
                    base = a.in + (int64_t)s * a.in_ss +
                           ((int64_t)(y * a.sh - a.ph + a.in_hh) * a.in_Wp + (x * a.sw - a.pw + a.in_hw)) * a.in_Cp;
                }
                if (a.tap4x7) {
                    // 4-channel input, 7x7 window (the paper's layer 2): a tap is
                    // one 16-byte chunk, K-block kb holds taps 8kb..8kb+7, so
                    // every copy is a row pointer + a compile-time offset (no
                    // offset table, no per-copy address registers to recycle)
                    const float* rowp[7];
#pragma unroll
                    for (int kj = 0; kj < 7; ++kj) rowp[kj] = base + (int64_t)kj * a.in_Wp * 4;
#pragma unroll
                    for (int kb = 0; kb < 7; ++kb, rg.next(NS)) {
                        const uint32_t st = rg.st, ph = rg.ph;
                        mbar_wait(&empty[st], ph ^ 1u);
                        if (r == 0) {
                            mbar_arrive_expect_tx(&full[st], b_bytes);
                            bulk_g2s(sB + (size_t)st * b_bytes, Bw + (size_t)kb * a.Brows * kKBlock, b_bytes, &full[st]);
                        }
                        const uint32_t row = smem_u32(sA + (size_t)st * kABytes + r * 128);
                        if (valid) {
#pragma unroll
                            for (int j = 0; j < kChunksPerKB; ++j) {
                                const int t = kb * kChunksPerKB + j;
                                if (t < 49)
                                    cp_async16(row + ((j ^ swz) << 4), rowp[t / 7] + (t % 7) * 4, 16u);
                                else
                                    cp_async16(row + ((j ^ swz) << 4), a.in, 0u);
                            }
                        }
                        cp_async_arrive_noinc(&full[st]);
                    }
                    continue;
                }
                for (int kb = 0; kb < a.NKB; ++kb, rg.next(NS)) {
                    const uint32_t st = rg.st, ph = rg.ph;
                    mbar_wait(&empty[st], ph ^ 1u);
                    if (r == 0) {
                        mbar_arrive_expect_tx(&full[st], b_bytes);
                        bulk_g2s(sB + (size_t)st * b_bytes, Bw + (size_t)kb * a.Brows * kKBlock, b_bytes, &full[st]);
                    }
                    const uint32_t row = smem_u32(sA + (size_t)st * kABytes + r * 128);
                    if (valid) {
                        // the K-block's 8 chunk offsets in two 16-byte loads, so
                        // their latencies overlap instead of one LDS per copy
                        const int4* tab4 = reinterpret_cast<const int4*>(sTab + kb * kChunksPerKB);
                        const int4 o0 = tab4[0], o1 = tab4[1];
                        const int offs[kChunksPerKB] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
#pragma unroll
                        for (int j = 0; j < kChunksPerKB; ++j) {
                            const int off = offs[j];
                            cp_async16(row + ((j ^ swz) << 4), off >= 0 ? base + off : a.in, off >= 0 ? 16u : 0u);
                        }
                    }
                    cp_async_arrive_noinc(&full[st]);
                }
            }
          }
        } else {
        // Thread pt copies chunk j = pt % 8 of rows rsub + 16*i (i < 8), so the
        // 8 lanes of a row fetch its 128 contiguous-ish bytes together and a
        // warp instruction touches 4 rows instead of 32 scattered pixels.
        const int pt = tid - kEpiThreads;
        const int j = pt & 7, rsub = pt >> 3;
        const uint32_t swz_off = (uint32_t)((j ^ (rsub & 7)) << 4);
        constexpr int kRowsPerThread = tc::kTileM / 16;
        Ring rg;
        // indices of the next tile's rows are loaded during this tile's K-loop
        int32_t gnext[kRowsPerThread];
        auto load_rows = [&](int64_t t) {
#pragma unroll
            for (int i = 0; i < kRowsPerThread; ++i) {
                const int64_t n = t * kRowsPerTile + row_off + rsub + 16 * i;
                gnext[i] = (t < ntiles && n < total) ? (a.idx ? __ldg(a.idx + n) : (int32_t)n) : -1;
            }
        };
        load_rows(tile_first);
        for (int64_t tile = tile_first; tile < ntiles; tile += tile_step) {
            const float* base[kRowsPerThread];
            uint32_t vmask = 0;
            int32_t gcur[kRowsPerThread];
#pragma unroll
            for (int i = 0; i < kRowsPerThread; ++i) gcur[i] = gnext[i];
            load_rows(tile + tile_step);
#pragma unroll
            for (int i = 0; i < kRowsPerThread; ++i) {
                base[i] = a.in;
                if (gcur[i] >= 0) {
                    vmask |= 1u << i;
                    const int64_t g = gcur[i];
                    int s, p, y, x;
                    pixel_of(a, g, HoWo, s, p, y, x);
                    const int64_t u = (int64_t)s * a.in_ss +
                                      ((int64_t)(y * a.sh - a.ph + a.in_hh) * a.in_Wp + (x * a.sw - a.pw + a.in_hw)) * a.in_Cp;
                    // packed: a window origin on an odd 8-byte boundary reads
                    // the 8-byte-shifted copy, where it is 16-byte aligned
                    base[i] = (a.pack_cpr > 0 && (u & 2)) ? a.in2 + u + 2 : a.in + u;
                }
            }
            for (int kb = 0; kb < a.NKB; ++kb, rg.next(NS)) {
                const uint32_t st = rg.st, ph = rg.ph;
                mbar_wait(&empty[st], ph ^ 1u);
                if (pt == 0) {
                    mbar_arrive_expect_tx(&full[st], b_bytes);
                    bulk_g2s(sB + (size_t)st * b_bytes, Bw + (size_t)kb * a.Brows * kKBlock, b_bytes, &full[st]);
                }
                const int off = sTab[kb * kChunksPerKB + j];
                const uint32_t stage = smem_u32(sA + (size_t)st * kABytes) + swz_off;
                if (off >= 0) {
#pragma unroll
                    for (int i = 0; i < kRowsPerThread; ++i)
                        if ((vmask >> i) & 1u) cp_async16(stage + (rsub + 16 * i) * 128, base[i] + off, 16u);
                } else {
                    // chunk past the real K (last K-block only): zero-fill
#pragma unroll
                    for (int i = 0; i < kRowsPerThread; ++i)
                        if ((vmask >> i) & 1u) cp_async16(stage + (rsub + 16 * i) * 128, a.in, 0u);
                }
                cp_async_arrive_noinc(&full[st]);
            }
        }
        }
    } else if (warp == 8) {
        if (PAIR && crank != 0) {
            // ================= peer: relay "stage full" to the leader =================
            if (lane == 0) {
                Ring rg;
                for (int64_t tile = tile_first; tile < ntiles; tile += tile_step)
                    for (int kb = 0; kb < a.NKB; ++kb, rg.next(NS)) {
                        const uint32_t st = rg.st, ph = rg.ph;
                        mbar_wait(&full[st], ph);
                        fence_proxy_async();
                        mbar_arrive_cluster(mapa(&pfull[st], 0));
                    }
            }
        } else {
            // ================= MMA issuer (whole warp, one elected lane issues) =================
            const int M = PAIR ? 2 * tc::kTileM : tc::kTileM;
            const uint32_t id0 = I8 ? idesc_i8(a.N0, M) : a.f16 ? idesc_f16(a.N0, M) : idesc_tf32(a.N0, M);
            const uint32_t id1 = a.f16 ? idesc_f16(a.N1 > 0 ? a.N1 : 16, M) : idesc_tf32(a.N1 > 0 ? a.N1 : 16, M);
            const bool two = a.N1 > 0;
            const bool f16 = a.f16 != 0;
            // B rows of the second instruction start after this CTA's share of the first
            const uint32_t b1_off = (uint32_t)(PAIR ? a.N0 / 2 : a.N0) * 128u;
            const uint64_t a_desc0 = smem_desc(smem_u32(sA)), b_desc0 = smem_desc(smem_u32(sB));
            // descriptor start-address field is in 16-byte units
            const uint64_t a_st = kABytes >> 4, b_st = b_bytes >> 4, b1_d = b1_off >> 4;
#ifdef CBX_EXP_SOLO
#define MMA_ELECT true
#define MMA_SYNCWARP (void)0
            if (lane == 0) {
#else
#define MMA_ELECT elect_one()
#define MMA_SYNCWARP __syncwarp()
#endif
            Ring rg;
            uint32_t acc_it = 0;
            for (int64_t tile = tile_first; tile < ntiles; tile += tile_step, ++acc_it) {
                const uint32_t as = acc_it % a.acc_stages, aph = (acc_it / a.acc_stages) & 1u;
                if constexpr (PAIR) mbar_wait_cluster(&tempty[as], aph ^ 1u); else mbar_wait(&tempty[as], aph ^ 1u);
                if (a.ovl && acc_it > 0) {
                    if constexpr (PAIR) mbar_wait_cluster(tshared, (acc_it - 1) & 1u); else mbar_wait(tshared, (acc_it - 1) & 1u);
                }
                tc_fence_after();
                const uint32_t d = tmem_base + (a.ovl ? (uint32_t)a.ovl_s : as * a.acc_cols);
                const uint32_t d1 = a.ovl ? tmem_base + (uint32_t)(as ? a.ovl_b1 : a.ovl_b0) : d + a.N0;
                for (int kb = 0; kb < a.NKB; ++kb, rg.next(NS)) {
                    const uint32_t st = rg.st, ph = rg.ph;
                    mbar_wait(&full[st], ph);
                    if constexpr (PAIR) mbar_wait_cluster(&pfull[st], ph);
                    // no proxy fence here: the cp.async -> mbarrier -> tcgen05.mma
                    // hand-off is the one CUTLASS's SM100 cp.async UMMA mainloop
                    // uses (producer_commit with cpasync_barrier_arrive, then
                    // consumer_wait, then the MMAs); the fence cost 1-2 % of L3
                    tc_fence_after();
                    const uint64_t ad = a_desc0 + st * a_st, bd = b_desc0 + st * b_st;
                    const int nk = kb + 1 == a.NKB ? a.kinst_last : kKBlock / 8;
                    if (MMA_ELECT) {
#pragma unroll
                        for (int k = 0; k < kKBlock / 8; ++k) {
                            if (k >= nk) break;
                            const uint32_t accum = (kb | k) ? 1u : 0u;
                            if constexpr (I8) {
                                mma_i8(d, ad + 2 * k, bd + 2 * k, id0, accum);
                            } else if constexpr (PAIR) {
                                if (f16) {
                                    mma_f16_pair(d, ad + 2 * k, bd + 2 * k, id0, accum);
                                    if (two) mma_f16_pair(d1, ad + 2 * k, bd + b1_d + 2 * k, id1, accum);
                                } else {
                                    mma_tf32_pair(d, ad + 2 * k, bd + 2 * k, id0, accum);
                                    if (two) mma_tf32_pair(d1, ad + 2 * k, bd + b1_d + 2 * k, id1, accum);
                                }
                            } else if (f16) {
                                mma_f16(d, ad + 2 * k, bd + 2 * k, id0, accum);
                                if (two) mma_f16(d1, ad + 2 * k, bd + b1_d + 2 * k, id1, accum);
                            } else {
                                mma_tf32(d, ad + 2 * k, bd + 2 * k, id0, accum);
                                if (two) mma_tf32(d1, ad + 2 * k, bd + b1_d + 2 * k, id1, accum);
                            }
                        }
                        if constexpr (PAIR) mma_commit_pair(&empty[st]); else mma_commit(&empty[st]);
                    }
                    MMA_SYNCWARP;
                }
                if (MMA_ELECT) {
                    if constexpr (PAIR) mma_commit_pair(&tfull[as]); else mma_commit(&tfull[as]);
                }
                MMA_SYNCWARP;
            }
#ifdef CBX_EXP_SOLO
            }
#endif
#undef MMA_ELECT
#undef MMA_SYNCWARP
        }
        __syncwarp();
    } else {
        // ================= epilogue: thread = TMEM lane = tile row =================
        const int r = tid;
        uint32_t acc_it = 0;
        // the index of this row in the NEXT tile is loaded while this tile is
        // processed: a tile's epilogue never starts with a dependent global
        // load (short K-loops, e.g. the 2-K-block layer 1, are otherwise
        // bound by that latency)
        auto row_index = [&](int64_t t) -> int64_t {
            const int64_t n = t * kRowsPerTile + row_off + r;
            return (t < ntiles && n < total) ? entry_at(a, n) : -1;
        };
        int64_t gnext = row_index(tile_first);
        for (int64_t tile = tile_first; tile < ntiles; tile += tile_step, ++acc_it) {
            const uint32_t as = acc_it % a.acc_stages, aph = (acc_it / a.acc_stages) & 1u;
            const int64_t gi = gnext;
            gnext = row_index(tile + tile_step);
            const bool valid = gi >= 0;
            // output address resolved before waiting for the accumulator
            const int64_t g = valid ? gi : 0;
            int s = 0, p = 0, y = 0, x = 0;
            float* dst = nullptr;
            if (valid && a.grp_R <= 1) {
                pixel_of(a, g, HoWo, s, p, y, x);
                dst = a.out + (int64_t)s * a.out_ss + ((int64_t)(y + a.out_hh) * a.out_Wp + (x + a.out_hw)) * a.out_Cp;
                // the values this pixel overwrites (compare-before-write) are
                // pulled into L2 while the MMAs run
                if (a.chg.d && a.write_out)
                    for (int b = 0; b < a.O * 4; b += 128)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(dst) + b));
            }
            mbar_wait(&tfull[as], aph);
            tc_fence_after();
            bool changed = false;
            const uint32_t trow = tmem_base + ((uint32_t)(warp * 32) << 16);
            if constexpr (I8) {
                // digits -> fp32: the s32 digit sums are exact, recombined in
                // fp64 (exact below 2^53) and rounded once with the bias
                const uint32_t tb = trow + as * a.acc_cols;
                const int Op = a.i8_opad;
                for (int j0 = 0; j0 < a.O; j0 += 4) {
                    int32_t q0[4], q1[4], q2[4];
                    tmem_ld4(tb + j0, q0);
                    tmem_ld4(tb + Op + j0, q1);
                    tmem_ld4(tb + 2 * Op + j0, q2);
                    tmem_wait_ld();
                    if (j0 + 4 >= a.O) {
                        tc_fence_before();
                        mbar_arrive(&tempty[as]);
                    }
                    if (!valid) continue;
                    float v[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        // |digit sums| < 2^23: exact in fp32; the scaled
                        // recombination rounds at most three times (~2^-23 rel.)
                        const int j = min(j0 + e, a.O - 1);
                        const float tot = fmaf((float)q2[e], 65536.0f, fmaf((float)q1[e], 256.0f, (float)q0[e]));
                        const float t = fmaf(tot, sQs[j], sBias[j]);
                        v[e] = a.relu ? ref_relu(t) : t;
                    }
                    if (j0 + 4 <= a.O) {  // channel stride is a multiple of 4: aligned 16-byte store
                        float4* q4 = reinterpret_cast<float4*>(dst + j0);
                        if (a.chg.d) {
                            const float4 old = *q4;
                            changed |= ref_changed(v[0], old.x, a.tau) | ref_changed(v[1], old.y, a.tau) |
                                       ref_changed(v[2], old.z, a.tau) | ref_changed(v[3], old.w, a.tau);
                        }
                        *q4 = make_float4(v[0], v[1], v[2], v[3]);
                    } else {
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            if (j0 + e < a.O) {
                                if (a.chg.d) changed |= ref_changed(v[e], dst[j0 + e], a.tau);
                                dst[j0 + e] = v[e];
                            }
                        }
                    }
                }
                if (a.chg.d) {
                    if (valid && changed) bit_set(a.chg, s, y, x);
                    if (a.chg_cnt) warp_count_add(a.chg_cnt, a.cnt_stride, s, changed, valid);
                }
                continue;
            }
            if (a.grp_R > 1) {
                // pixel group: sub-pixel j's channels at columns j * grp_N;
                // each live sub-pixel (mask bit) gets the per-pixel epilogue
                int gs = 0, gy = 0, gx0 = 0;
                const uint32_t gm = valid ? (uint32_t)(gi & 15) : 0u;
                if (valid) group_of_tc(a, gi, gs, gy, gx0);
                const uint32_t tb = trow + as * a.acc_cols;
                TailAcc<TC> t1g;
                uint32_t chb = 0;
                for (int j = 0; j < a.grp_R; ++j) {
                    const bool live = (gm >> j) & 1u;
                    float* dj = a.out + (int64_t)gs * a.out_ss +
                                ((int64_t)(gy + a.out_hh) * a.out_Wp + (gx0 + j + a.out_hw)) * a.out_Cp;
                    bool chj = false;
                    for (int c0 = 0; c0 < a.O; c0 += 32) {
                        float v[32];
                        tmem_ld32(tb + (uint32_t)(j * a.grp_N + c0), v);
                        if (!live) continue;
                        if (c0 + 32 <= a.O)
                            epi_chunk<TC, true>(a, v, c0, 32, sBias, sTailW, t1g, dj, chj);
                        else
                            epi_chunk<TC, false>(a, v, c0, a.O - c0, sBias, sTailW, t1g, dj, chj);
                    }
                    if (live && chj) chb |= 1u << j;
                }
                tc_fence_before();
                mbar_arrive(&tempty[as]);
                if (a.chg.d) {
                    for (int j = 0; j < a.grp_R; ++j)
                        if ((chb >> j) & 1u) bit_set(a.chg, gs, gy, gx0 + j);
                    if (a.chg_cnt) {
                        const unsigned act = __ballot_sync(0xffffffffu, valid);
                        const int n = __popc(chb);
                        if (valid) {
                            const unsigned same = __match_any_sync(act, gs);
                            if (same == act) {
                                const int sum = __reduce_add_sync(act, n);
                                if (lane == __ffs(act) - 1 && sum)
                                    atomicAdd(a.chg_cnt + (int64_t)gs * a.cnt_stride, (unsigned long long)sum);
                            } else if (n) {
                                atomicAdd(a.chg_cnt + (int64_t)gs * a.cnt_stride, (unsigned long long)n);
                            }
                        }
                    }
                }
                continue;
            }
            // TMEM column of channel c0: one accumulator per stage, or (ovl)
            // the shared columns for c0 < N0 and this parity's own after
            const uint32_t col_lo = a.ovl ? (uint32_t)a.ovl_s : as * a.acc_cols;
            const uint32_t col_hi = a.ovl ? (uint32_t)(as ? a.ovl_b1 : a.ovl_b0) - (uint32_t)a.N0 : col_lo;
            // fused per-pixel tail: first op is a 1x1 CONV over this layer's
            // outputs, accumulated chunk by chunk in ascending channel order
            constexpr int TCA = TC > 0 ? TC : 1;
            TailAcc<TC> t1p;
#pragma unroll
            for (int q = 0; q < (TC > 1 ? TC / 2 : 1); ++q)
                t1p[q] = f2_pack((TC > 0 && 2 * q < a.tail.cout[0]) ? __ldg(a.tail.b[0] + 2 * q) : 0.0f,
                                 (TC > 0 && 2 * q + 1 < a.tail.cout[0]) ? __ldg(a.tail.b[0] + 2 * q + 1) : 0.0f);
            for (int c0 = 0; c0 < a.O; c0 += 32) {
                float v[32];
                tmem_ld32(trow + (c0 < a.N0 ? col_lo : col_hi) + c0, v);
                if (a.ovl && c0 + 32 == a.N0) {
                    // shared columns drained: the next tile's MMAs may start
                    tc_fence_before();
                    if constexpr (PAIR) {
                        __syncwarp();
                        if (lane == 0) mbar_arrive_cluster(mapa(tshared, 0));
                    } else {
                        mbar_arrive(tshared);
                    }
                }
                if (!valid) continue;
                if (c0 + 32 <= a.O)
                    epi_chunk<TC, true>(a, v, c0, 32, sBias, sTailW, t1p, dst, changed);
                else
                    epi_chunk<TC, false>(a, v, c0, a.O - c0, sBias, sTailW, t1p, dst, changed);
            }
            float t1[TCA];
#pragma unroll
            for (int q = 0; q < TCA; ++q) t1[q] = 0.0f;
            if constexpr (TC > 1) {
#pragma unroll
                for (int q = 0; q < TC / 2; ++q) f2_unpack(t1p[q], t1[2 * q], t1[2 * q + 1]);
            }
            tc_fence_before();
            if constexpr (PAIR) {
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(mapa(&tempty[as], 0));
            } else {
                mbar_arrive(&tempty[as]);
            }
            if constexpr (TC > 0) {
                if (valid) run_tail<TC>(a.tail, t1, s, y, x, p);
            }
            if (a.chg.d) {
                if (valid && changed) bit_set(a.chg, s, y, x);
                if (a.chg_cnt) warp_count_add(a.chg_cnt, a.cnt_stride, s, changed, valid);
            }
        }
    }
    tc_fence_before();
    // PAIR: no CTA may leave (or free its TMEM) while the other still signals
    // its barriers or the leader's MMAs still target its TMEM
    if constexpr (PAIR) cluster_sync_all(); else __syncthreads();
    if (warp == 8) {
        tc_fence_after();
        if constexpr (PAIR)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(a.tmem_cols));
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(a.tmem_cols));
    }
}

float round_tf32(float x) {
    // round-to-nearest (ties away) to 10 explicit mantissa bits, as cvt.rna.tf32.f32
    uint32_t u;
    std::memcpy(&u, &x, 4);
    if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & 0xffffe000u;
    float r;
    std::memcpy(&r, &u, 4);
    return r;
}

}  // namespace

struct TcLayer {
    cbx_geom g;
    int Cp = 0, NKB = 0, Npad = 0, N0 = 0, N1 = 0;
    int stages = 0, acc_stages = 1, acc_cols = 0, tmem_cols = 32;
    int tail_w_floats = 0;
    int ctas_per_sm = 1;
    bool pair = false;   // CTA pair (cta_group::2, M = 256)
    bool ovl = false;    // split accumulator (see make_tc_layer)
    bool f16 = false;    // fp16 operands (kind::f16): Cp counts 4-byte units of the fp16 shadow input
    bool i8 = false;     // kind::i8 over RGBX camera bytes (Cp = 1 unit per pixel), digit filters
    int Opad = 0;        // i8: output channels padded to 4 (digit column stride)
    int grpR = 1, grpN = 0;  // pixel groups: R adjacent output pixels per row, column stride per sub-pixel
    int pack_cpr = 0;        // packed fp16 input: 16-byte chunks per kernel row (0: channels padded to 8)
    int kinst_last = 4;
    float* qsc = nullptr;   // i8: per-channel scale / 255
    int ovl_s = 0, ovl_b0 = 0, ovl_b1 = 0;
    int max_ctas = 0;    // persistent grid cap (0: one per SM x ctas_per_sm)
    int Brows = 0;       // filter rows per CTA
    int max_clusters = 0;
    size_t smem = 0;
    float* Bw = nullptr;
};

void TcLayerDeleter::operator()(TcLayer* p) const {
    if (p && p->Bw) cudaFree(p->Bw);
    if (p && p->qsc) cudaFree(p->qsc);
    delete p;
}

bool tc_is_f16(const TcLayer& t) { return t.f16; }
bool tc_is_i8(const TcLayer& t) { return t.i8; }

bool tc_i8_supported(const cbx_geom& g) {
    return g.inChannels >= 1 && g.inChannels <= 4 && g.outChannels >= 1 && 3 * round_up(g.outChannels, 4) <= 256 &&
           g.kernelW <= 8 && g.kernelH <= 64;
}

bool tc_supported(const cbx_geom& g) {
    const int Npad = (int)round_up(g.outChannels, 16);
    return g.outChannels >= 1 && Npad <= 512 && g.kernelH * g.kernelW * round_up(g.inChannels, 4) <= 65536;
}

namespace {
template <bool R, int T, bool P, bool I = false>
void set_smem_attr() {
    CBX_CUDA(cudaFuncSetAttribute(conv_tc_kernel<R, T, P, I>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
}
template <int T, bool P>
void set_smem_attrs() {
    set_smem_attr<true, T, P>();
    set_smem_attr<false, T, P>();
}
}  // namespace

int tc_group_width(const TcLayer& t) { return t.grpR; }
int tc_input_cp(const TcLayer& t) { return t.Cp; }

bool tc_group_supported(const cbx_geom& g, int R) {
    return R > 1 && R <= 4 && g.strideH == 1 && g.strideW == 1 && g.inChannels <= 4 &&
           R * round_up(g.outChannels, 32) <= 256 && g.kernelH * (g.kernelW + R - 1) <= 8 * 64;
}

std::unique_ptr<TcLayer, TcLayerDeleter> make_tc_layer(const cbx_geom& g, int tail_floats, int pair_mode, bool f16,
                                                       bool i8, int grpR, bool pack) {
    std::unique_ptr<TcLayer, TcLayerDeleter> t(new TcLayer);
    t->g = g;
    if (i8) {
        // layer 1 of the 8-bit camera path: one 4-byte RGBX chunk per tap,
        // 32 taps per 128-byte K-block; N = three digit columns per channel
        if (!tc_i8_supported(g)) throw Error(CBX_E_ARG, "kind::i8 conv: unsupported geometry");
        t->i8 = true;
        t->Cp = 1;
        t->NKB = (g.kernelH + 3) / 4;  // 4 kernel rows (8 tap slots each) per K-block
        t->Opad = (int)round_up(g.outChannels, 4);
        t->Npad = (int)round_up(3 * t->Opad, 16);
        t->N0 = t->Npad;
        t->N1 = 0;
        t->acc_cols = (int)round_up(t->Npad, 32);
        t->acc_stages = 2;
        int cols = 32;
        while (cols < 2 * t->acc_cols) cols *= 2;
        t->tmem_cols = cols;
        t->Brows = t->Npad;
        t->ctas_per_sm = 2;
        const size_t b_bytes = (size_t)t->Brows * 128;
        const size_t fixed = 1024 + round_up(g.outChannels, 4) * 4 + 16 +
                             (size_t)g.outChannels * 8 + 8 * (3 * 16 + 5) + 16;
        const size_t budget = (size_t)kMaxSmem / 2 - 1024;
        int ns = 6;
        if (const char* e = std::getenv("CBX_TC_STAGES")) ns = std::max(2, std::min(16, std::atoi(e)));
        while (ns > 2 && fixed + (size_t)ns * (kABytes + b_bytes) > budget) --ns;
        t->stages = ns;
        if (const char* e = std::getenv("CBX_TC_MAXCTAS")) t->max_ctas = std::max(1, std::atoi(e));
        t->smem = fixed + (size_t)ns * (kABytes + b_bytes);
        set_smem_attr<true, 0, false, true>();
        CBX_CUDA(cudaMalloc(&t->Bw, (size_t)t->NKB * b_bytes));
        CBX_CUDA(cudaMemset(t->Bw, 0, (size_t)t->NKB * b_bytes));
        CBX_CUDA(cudaMalloc(&t->qsc, sizeof(float) * g.outChannels));
        CBX_CUDA(cudaMemset(t->qsc, 0, sizeof(float) * g.outChannels));
        CBX_CUDA(cudaStreamSynchronize(nullptr));  // (legacy-stream memsets before the non-blocking uploads)
        return t;
    }
    // fp16 operands: 8 channels per 16-byte chunk; Cp stays in 4-byte units so
    // the gather's address arithmetic is the same for both operand types
    t->f16 = f16;
    t->Cp = f16 ? (int)round_up(g.inChannels, 8) / 2 : (int)round_up(g.inChannels, 4);
    if (grpR > 1 && (f16 || pair_mode > 0 || tail_floats > 0 || !tc_group_supported(g, grpR))) grpR = 1;
    t->grpR = grpR;
    // pixel groups: K = kh x (kw + R - 1) window taps; sub-pixel j's outputs in
    // columns [j * grpN, j * grpN + O), grpN = O rounded up to 32 (the
    // epilogue's tcgen05.ld granularity)
    int nchunks = g.kernelH * (g.kernelW + grpR - 1) * (t->Cp / 4);
    if (f16 && pack && g.inChannels % 4 == 0 && grpR == 1) {
        // packed fp16 operands: a kernel row's kw x C halves are contiguous in
        // the unpadded shadow (Cp = C/2 units) -> ceil(kw C 2 / 16) chunks per
        // kernel row instead of kw ceil(C / 8) (paper layer 3: 46 vs 49).
        // C % 4 == 0 keeps every window origin 8-byte aligned (even Cp), so it
        // is 16-byte aligned in the shadow or in its 8-byte-shifted copy
        t->Cp = g.inChannels / 2;
        t->pack_cpr = (g.kernelW * g.inChannels * 2 + 15) / 16;
        nchunks = g.kernelH * t->pack_cpr;
    }
    t->NKB = (nchunks + kChunksPerKB - 1) / kChunksPerKB;
    t->kinst_last = (nchunks - kChunksPerKB * (t->NKB - 1) + 1) / 2;  // 2 chunks (32 B of K) per instruction
    t->grpN = grpR > 1 ? (int)round_up(g.outChannels, 32) : 0;
    t->Npad = grpR > 1 ? grpR * t->grpN : (int)round_up(g.outChannels, 16);
    // N > 256 needs two MMAs per K-step; split evenly (304 = 160 + 144, not
    // 256 + 48): a narrow instruction re-reads the whole A slice for few
    // columns and is shared-memory-bound, a balanced pair is not.
    // CBX_TC_NSPLIT=0 keeps the 256 + rest split (tuning).
    const char* ns_env = std::getenv("CBX_TC_NSPLIT");
    const bool even = !(ns_env && std::atoi(ns_env) == 0);
    t->N0 = t->Npad > 256 ? (even ? (int)round_up(t->Npad / 2, 16) : 256) : t->Npad;
    t->N1 = t->Npad - t->N0;
    t->acc_cols = (int)round_up(t->Npad, 32);  // tcgen05.ld reads 32-column groups
    t->acc_stages = (2 * t->acc_cols <= 512) ? 2 : 1;
    int cols = 32;
    while (cols < t->acc_stages * t->acc_cols) cols *= 2;
    t->tmem_cols = cols;
    // A wide layer's accumulator (N_pad > 256) cannot be double-buffered in
    // 512 TMEM columns, so the MMAs of tile t+1 would wait for the whole
    // epilogue of tile t. Split accumulator instead: the first instruction
    // (N0 = 128 channels, drained first by the epilogue) always writes the
    // shared columns [s, s + 128); the second (N1 = N_pad - 128) alternates
    // between [0, N1) and [s + 128, s + 128 + N1) by tile parity. Tile t+1
    // then waits only for tile t's first four 32-channel chunks.
    // CBX_TC_OVL=0 keeps the single accumulator (tuning).
    const char* ovl_env = std::getenv("CBX_TC_OVL");
    if (t->Npad > 256 && !(ovl_env && std::atoi(ovl_env) == 0)) {
        const int n0 = 128, n1 = t->Npad - n0;
        const int s0 = (int)round_up(n1, 32);
        if (n1 <= 256 && s0 + t->Npad <= 512) {
            t->ovl = true;
            t->N0 = n0;
            t->N1 = n1;
            t->acc_stages = 2;
            t->ovl_s = s0;
            t->ovl_b0 = 0;
            t->ovl_b1 = s0 + n0;
            t->tmem_cols = 512;
        }
    }
    // CTA pairs (M = 256, each SM streams half the filter bank) are opt-in:
    // measured on B200 they lose to single-CTA tiles for the paper's L3
    // (1.54 vs 1.42 ms dense 4x1080p): the shallower per-SM shared memory
    // leaves the gather's tap reuse less L1 (hit rate 45% vs 85%), and the
    // pair handshake adds a relay per K-block. Narrow layers run two
    // independent CTAs per SM so that one CTA's gather latency overlaps the
    // other's MMAs/epilogue.
    t->pair = pair_mode > 0;
    t->Brows = t->pair ? t->Npad / 2 : t->Npad;
    // one CTA per SM: with two lanes the second CTA's shared memory is worth
    // more to the other lane's kernels (16 x 1080p: 31.7k -> 32.3k frames/s)
    t->ctas_per_sm = 1;
    if (const char* e = std::getenv("CBX_TC_CTAS_PER_SM"))  // tuning
        if (!t->pair && t->Npad <= 128) t->ctas_per_sm = std::max(1, std::min(2, std::atoi(e)));
    const size_t b_bytes = (size_t)t->Brows * 128;
    t->tail_w_floats = (int)round_up(tail_floats, 4);
    const size_t fixed = 1024 + (size_t)t->NKB * kChunksPerKB * 4 + round_up(g.outChannels, 4) * 4 +
                         (size_t)t->tail_w_floats * 4 + 16 + 8 * (3 * 16 + 5) + 16 + 8;
    const size_t budget = t->ctas_per_sm == 2 ? (size_t)kMaxSmem / 2 - 1024 : (size_t)kMaxSmem;
    // stage count: deep enough to cover the gather latency, shallow enough to
    // leave L1 for the gather's tap reuse (neighbouring output pixels share
    // input pixels across taps; the L1 hit rate collapses when shared memory
    // takes the whole carve-out). CBX_TC_STAGES overrides (tuning).
    // Three stages: the layers do not get faster with more (measured: the
    // paper's layer 3 155.6 us with 3 or 4 stages, layer 2 44-46 us with
    // 2..8), and the smaller shared-memory footprint lets the other lane's
    // kernels co-reside with the persistent CTAs (16 x 1080p: 30.3k -> 30.9k
    // frames/s; with the 3-stage layer-1 conv, 31.4k). CBX_TC_STAGES /
    // CBX_TC_STAGES_WIDE (N > 256) override (tuning).
    // grouped layers: two stages keep the footprint of the wider N (the
    // other lane's kernels run beside it) at the one-pixel layer's size
    int ns = t->pair ? 4 : t->grpR > 1 ? 2 : 3;
    if (const char* e = std::getenv("CBX_TC_STAGES")) ns = std::max(2, std::min(16, std::atoi(e)));
    if (t->Npad > 256)
        if (const char* e = std::getenv("CBX_TC_STAGES_WIDE")) ns = std::max(2, std::min(16, std::atoi(e)));
    while (ns > 2 && fixed + (size_t)ns * (kABytes + b_bytes) > budget) --ns;
    if (fixed + (size_t)ns * (kABytes + b_bytes) > budget)
        throw Error(CBX_E_ARG, "tcgen05 conv: layer too wide for shared memory");
    t->stages = ns;
    // CBX_TC_MAXCTAS caps the persistent grid (tuning: SMs left free for the
    // other lane's kernels; tests: many tiles per CTA on small frames)
    if (const char* e = std::getenv("CBX_TC_MAXCTAS")) t->max_ctas = std::max(1, std::atoi(e));
    if (t->Npad > 256)  // (tuning: SMs left to the other lane's kernels while the wide layer runs)
        if (const char* e = std::getenv("CBX_TC_MAXCTAS_WIDE")) t->max_ctas = std::max(1, std::atoi(e));
    t->smem = fixed + (size_t)ns * (kABytes + b_bytes);
    set_smem_attrs<0, false>();
    set_smem_attrs<8, false>();
    set_smem_attrs<16, false>();
    set_smem_attrs<0, true>();
    set_smem_attrs<8, true>();
    set_smem_attrs<16, true>();
    if (t->pair) {
        // co-resident 2-CTA clusters at this shared-memory size
        cudaLaunchConfig_t cfg{};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(2 * kNumSMs);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = t->smem;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int n = 0;
        CBX_CUDA(cudaOccupancyMaxActiveClusters(&n, conv_tc_kernel<false, 8, true>, &cfg));
        t->max_clusters = std::max(1, std::min(n, kNumSMs / 2));
    }
    CBX_CUDA(cudaMalloc(&t->Bw, (size_t)t->NKB * b_bytes * (t->pair ? 2 : 1)));
    CBX_CUDA(cudaMemset(t->Bw, 0, (size_t)t->NKB * b_bytes * (t->pair ? 2 : 1)));
    CBX_CUDA(cudaStreamSynchronize(nullptr));  // (legacy-stream memset before the non-blocking uploads)
    return t;
}

// Host-side re-layout of the reference filter matrix K[o][(c*kh + kj)*kw + ki]
// into per-K-block swizzled smem images: element (n, kb*32 + j*4 + e) at
// float offset kb*Brows*32 + row*32 + ((j ^ (row & 7)) * 4) + e, where chunk
// J = kb*8 + j covers tap J / C4 = (kj, ki) and channels 4*(J % C4) + e.
// Single CTA: row = n. CTA pair: the two CTAs hold the two N-halves of every
// MMA instruction (channels [0, N0/2) and [N0, N0 + N1/2) on rank 0, the rest
// on rank 1), each in its own image.
void tc_load_weights(TcLayer& t, const float* K, cudaStream_t st) {
    const cbx_geom& g = t.g;
    const int C4 = t.Cp / 4, khw = g.kernelH * g.kernelW;
    const int Kref = g.inChannels * khw;
    const int ranks = t.pair ? 2 : 1;
    // filter row of output channel n: single CTA -> row n of the one image; CTA
    // pair -> each rank holds its half of every instruction's N columns
    auto place = [&](int n, int& rank, int& row) {
        rank = 0;
        row = n;
        if (!t.pair) return;
        if (n < t.N0) {
            rank = n / (t.N0 / 2);
            row = n % (t.N0 / 2);
        } else {
            const int m = n - t.N0;
            rank = m / (t.N1 / 2);
            row = t.N0 / 2 + m % (t.N1 / 2);
        }
    };
    if (t.i8) {
        // Each weight as a 22-bit integer multiple of its channel's scale
        // s_j = max|w_j| / 2^22, split into three balanced base-256 digits
        // (d0 + 256 d1 + 65536 d2, each in [-128, 127]); digit q of channel j
        // is filter row q * Opad + j. Tap (kj, ki) has slot t = kj * 8 + ki
        // (kernel rows padded to 8 taps, the A gather's order); byte
        // (row, t * 4 + c) of K-block t / 32 sits at
        // row * 128 + ((k / 16) ^ (row & 7)) * 16 + k % 16, k = (t % 32) * 4 + c.
        std::vector<int8_t> img((size_t)t.NKB * t.Brows * 128, 0);
        std::vector<float> qs(g.outChannels, 0.0f);
        for (int j = 0; j < g.outChannels; ++j) {
            double mx = 0.0;
            for (int i = 0; i < Kref; ++i) mx = std::max(mx, (double)std::fabs(K[(size_t)j * Kref + i]));
            const double sc = mx > 0.0 ? mx / 4194304.0 : 1.0;
            qs[j] = (float)(sc / 255.0);
            for (int c = 0; c < g.inChannels; ++c)
                for (int tap = 0; tap < khw; ++tap) {
                    long long wi = std::llround((double)K[(size_t)j * Kref + (size_t)c * khw + tap] / sc);
                    const int slot = (tap / g.kernelW) * 8 + tap % g.kernelW;
                    const int kb = slot / 32, k = (slot % 32) * 4 + c, jj = k / 16;
                    for (int q = 0; q < 3; ++q) {
                        long long r = ((wi % 256) + 256) % 256;
                        if (r >= 128) r -= 256;
                        wi = (wi - r) / 256;
                        const int row = q * t.Opad + j;
                        img[(size_t)kb * t.Brows * 128 + (size_t)row * 128 + ((jj ^ (row & 7)) * 16) + (k % 16)] =
                            (int8_t)r;
                    }
                    if (wi != 0) throw Error(CBX_E_ARG, "kind::i8 filter digits overflow");
                }
        }
        CBX_CUDA(cudaMemcpyAsync(t.Bw, img.data(), img.size(), cudaMemcpyHostToDevice, st));
        CBX_CUDA(cudaMemcpyAsync(t.qsc, qs.data(), sizeof(float) * qs.size(), cudaMemcpyHostToDevice, st));
        CBX_CUDA(cudaStreamSynchronize(st));
        return;
    }
    if (t.f16 && t.pack_cpr > 0) {
        for (size_t i = 0; i < (size_t)g.outChannels * Kref; ++i)
            if (std::fabs(K[i]) > 65504.0f)
                throw Error(CBX_E_ARG, "a filter weight of a kind::f16 layer exceeds the fp16 range (|w| > 65504); "
                                       "create the context with CBX_PREC_TF32");
        // packed fp16 image: chunk J = kj * pack_cpr + i holds halves
        // h = 8 i + e of kernel row kj's window (tap ki = h / C, channel
        // c = h % C; h >= kw C: next pixel, zero weight)
        const int C = g.inChannels;
        std::vector<__half> img((size_t)ranks * t.NKB * t.Brows * 64, __float2half_rn(0.0f));
        for (int n = 0; n < g.outChannels; ++n) {
            int rank, row;
            place(n, rank, row);
            __half* base = img.data() + (size_t)rank * t.NKB * t.Brows * 64;
            for (int kj = 0; kj < g.kernelH; ++kj)
                for (int h = 0; h < g.kernelW * C; ++h) {
                    const int ki = h / C, c = h % C;
                    const int J = kj * t.pack_cpr + h / 8, e = h % 8;
                    const int kb = J / kChunksPerKB, jj = J % kChunksPerKB;
                    base[(size_t)kb * t.Brows * 64 + (size_t)row * 64 + ((jj ^ (row & 7)) * 8) + e] =
                        __float2half_rn(K[(size_t)n * Kref + ((size_t)c * g.kernelH + kj) * g.kernelW + ki]);
                }
        }
        CBX_CUDA(cudaMemcpyAsync(t.Bw, img.data(), img.size() * sizeof(__half), cudaMemcpyHostToDevice, st));
        CBX_CUDA(cudaStreamSynchronize(st));
        return;
    }
    if (t.f16) {
        // fp16 image (round to nearest even): chunk J = tap * C4 + c4 holds
        // channels 8*c4 .. 8*c4+7 of that tap; half (row, kb*64 + j*8 + e) at
        // kb*Brows*64 + row*64 + (j ^ (row & 7))*8 + e of its rank's image
        // fp16 range: a weight beyond 65504 would become inf (the activations
        // are range-checked per frame by the shadow writer, engine.cu)
        for (size_t i = 0; i < (size_t)g.outChannels * Kref; ++i)
            if (std::fabs(K[i]) > 65504.0f)
                throw Error(CBX_E_ARG, "a filter weight of a kind::f16 layer exceeds the fp16 range (|w| > 65504); "
                                       "create the context with CBX_PREC_TF32");
        std::vector<__half> img((size_t)ranks * t.NKB * t.Brows * 64, __float2half_rn(0.0f));
        for (int n = 0; n < g.outChannels; ++n) {
            int rank, row;
            place(n, rank, row);
            __half* base = img.data() + (size_t)rank * t.NKB * t.Brows * 64;
            for (int J = 0; J < t.NKB * kChunksPerKB; ++J) {
                const int tap = J / C4, c4 = J - tap * C4;
                if (tap >= khw) continue;
                const int kb = J / kChunksPerKB, j = J - kb * kChunksPerKB;
                for (int e = 0; e < 8; ++e) {
                    const int c = c4 * 8 + e;
                    if (c >= g.inChannels) continue;
                    base[(size_t)kb * t.Brows * 64 + (size_t)row * 64 + ((j ^ (row & 7)) * 8) + e] =
                        __float2half_rn(K[(size_t)n * Kref + (size_t)c * khw + tap]);
                }
            }
        }
        CBX_CUDA(cudaMemcpyAsync(t.Bw, img.data(), img.size() * sizeof(__half), cudaMemcpyHostToDevice, st));
        CBX_CUDA(cudaStreamSynchronize(st));
        return;
    }
    if (t.grpR > 1) {
        // pixel groups (tf32, 4-channel input, C4 = 1): chunk J = kj * span + w
        // holds the 4 channels of window column w; B row j * grpN + o carries
        // filter o shifted by j: K[o][c][kj][w - j] for 0 <= w - j < kw
        const int span = g.kernelW + t.grpR - 1;
        std::vector<float> img((size_t)t.NKB * t.Brows * kKBlock, 0.0f);
        for (int j = 0; j < t.grpR; ++j)
            for (int o = 0; o < g.outChannels; ++o) {
                const int row = j * t.grpN + o;
                for (int kj = 0; kj < g.kernelH; ++kj)
                    for (int w = 0; w < span; ++w) {
                        const int ki = w - j;
                        if (ki < 0 || ki >= g.kernelW) continue;
                        const int J = kj * span + w, kb = J / kChunksPerKB, jj = J % kChunksPerKB;
                        for (int c = 0; c < g.inChannels; ++c)
                            img[(size_t)kb * t.Brows * kKBlock + (size_t)row * kKBlock + ((jj ^ (row & 7)) * 4) + c] =
                                round_tf32(K[(size_t)o * Kref + ((size_t)c * g.kernelH + kj) * g.kernelW + ki]);
                    }
            }
        CBX_CUDA(cudaMemcpyAsync(t.Bw, img.data(), img.size() * sizeof(float), cudaMemcpyHostToDevice, st));
        CBX_CUDA(cudaStreamSynchronize(st));
        return;
    }
    std::vector<float> img((size_t)ranks * t.NKB * t.Brows * kKBlock, 0.0f);
    for (int n = 0; n < g.outChannels; ++n) {
        int rank, row;
        place(n, rank, row);
        float* base = img.data() + (size_t)rank * t.NKB * t.Brows * kKBlock;
        for (int J = 0; J < t.NKB * kChunksPerKB; ++J) {
            const int tap = J / C4, c4 = J - tap * C4;
            if (tap >= khw) continue;
            const int kb = J / kChunksPerKB, j = J - kb * kChunksPerKB;
            for (int e = 0; e < 4; ++e) {
                const int c = c4 * 4 + e;
                if (c >= g.inChannels) continue;
                const float w = K[(size_t)n * Kref + (size_t)c * khw + tap];
                base[(size_t)kb * t.Brows * kKBlock + (size_t)row * kKBlock + ((j ^ (row & 7)) * 4) + e] = round_tf32(w);
            }
        }
    }
    CBX_CUDA(cudaMemcpyAsync(t.Bw, img.data(), img.size() * sizeof(float), cudaMemcpyHostToDevice, st));
    CBX_CUDA(cudaStreamSynchronize(st));
}

void launch_conv_tc(const TcLayer& t, TensorView in, TensorView out, const float* bias, const int32_t* idx,
                    const int* count, int64_t full_count, bool relu, BitMask chg, float tau,
                    unsigned long long* cnt, int cstride, int S, cudaStream_t st, const TcTail* tail,
                    const float* in_shifted) {
    if (in.Cp != t.Cp) throw Error(CBX_E_SHAPE, "tcgen05 conv: input channel stride mismatch");
    TcArgs a{};
    a.in = in.d;
    a.in_ss = in.ss;
    a.in_Wp = in.Wp;
    a.in_Cp = in.Cp;
    a.in_hh = in.hh;
    a.in_hw = in.hw;
    a.out = out.d;
    a.out_ss = out.ss;
    a.out_Wp = out.Wp;
    a.out_Cp = out.Cp;
    a.out_hh = out.hh;
    a.out_hw = out.hw;
    a.O = out.C;
    a.Ho = out.H;
    a.Wo = out.W;
    a.kh = t.g.kernelH;
    a.kw = t.g.kernelW;
    a.sh = t.g.strideH;
    a.sw = t.g.strideW;
    a.ph = t.g.padH;
    a.pw = t.g.padW;
    a.idx = idx;
    a.count = count;
    a.full_count = full_count;
    a.Bw = t.Bw;
    a.bias = bias;
    a.NKB = t.NKB;
    a.Npad = t.Npad;
    a.N0 = t.N0;
    a.N1 = t.N1;
    a.Brows = t.Brows;
    a.stages = t.stages;
    a.acc_stages = t.acc_stages;
    a.acc_cols = t.acc_cols;
    a.tmem_cols = t.tmem_cols;
    a.ovl = t.ovl;
    a.f16 = t.f16;
    a.i8_opad = t.Opad;
    a.qsc = t.qsc;
    {
        const int64_t HoWo = (int64_t)out.H * out.W;
        a.fast = full_count < ((int64_t)1 << 31);
        a.fd_howo = FastDiv::make((uint32_t)std::min<int64_t>(HoWo, 0x7fffffff));
        a.fd_wo = FastDiv::make((uint32_t)out.W);
    }
    a.grp_R = t.grpR;
    a.grp_N = t.grpN;
    a.pack_cpr = t.pack_cpr;
    a.in2 = in_shifted;
    a.kinst_last = t.kinst_last;
    if (t.pack_cpr > 0 && (!in_shifted || (in.Wp & 1) || (in.ss & 3)))
        throw Error(CBX_E_ARG, "tcgen05 conv: packed fp16 input needs the shifted copy, an even row pitch and 16-byte streams");
    if (t.grpR > 1) {
        // full mode walks every group; entries carry gid << 4 (below 2^31)
        a.Gw = (out.W + t.grpR - 1) / t.grpR;
        a.fd_gplane = FastDiv::make((uint32_t)(out.H * a.Gw));
        a.fd_gw = FastDiv::make((uint32_t)a.Gw);
        a.full_count = full_count = (int64_t)S * out.H * a.Gw;
        if (full_count >= ((int64_t)1 << 27)) throw Error(CBX_E_ARG, "tcgen05 conv: too many pixel groups");
        if (in.Cp != 4) throw Error(CBX_E_SHAPE, "tcgen05 conv: pixel groups need a 4-channel input");
    }
    static const bool no_tap4x7 = std::getenv("CBX_TC_NO_TAP4X7") != nullptr;  // (tuning)
    a.tap4x7 = !no_tap4x7 && in.Cp == 4 && t.g.kernelH == 7 && t.g.kernelW == 7 && t.NKB == 7 && t.grpR == 1;
    // (8-row x 4-chunk gather: conflict-free but measured slower than the
    // row-lane tap4x7 gather on the paper's layer 2, 50 vs 46 us per lane-frame;
    // CBX_TC_XROW=1 selects it, tuning)
    static const bool xrow = std::getenv("CBX_TC_XROW") != nullptr;
    a.xrow = xrow && in.Cp == 4 && !t.f16 && !t.pair && t.grpR == 1;
    a.ovl_s = t.ovl_s;
    a.ovl_b0 = t.ovl_b0;
    a.ovl_b1 = t.ovl_b1;
    a.tail_w_floats = t.tail_w_floats;
    if (tail && tail->n && (tail->cout[0] <= 8 ? 8 : 16) * out.C > t.tail_w_floats)
        throw Error(CBX_E_ARG, "tcgen05 conv: fused tail filters exceed the reserved shared memory");
    a.relu = relu;
    a.chg = chg;
    a.tau = tau;
    a.chg_cnt = chg.d ? cnt : nullptr;
    a.cnt_stride = cstride;
    a.write_out = !(tail && tail->n && !tail->keep_out);
    a.one = 1.0f;
    a.nzero = -0.0f;
    if (tail) a.tail = *tail;
    const int tc = (tail && tail->n) ? (tail->cout[0] <= 8 ? 8 : 16) : 0;
    static const int rowlane_env = std::getenv("CBX_TC_ROWLANE") ? std::atoi(std::getenv("CBX_TC_ROWLANE")) : -1;
    const bool rowlane = t.grpR > 1 || (rowlane_env >= 0 ? rowlane_env != 0 : in.Cp <= 4);  // (env: tuning)
    if (t.pair) {
        const int64_t max_tiles = (full_count + 2 * tc::kTileM - 1) / (2 * tc::kTileM);
        int64_t ccap = t.max_clusters;
        if (t.max_ctas > 0) ccap = std::min<int64_t>(ccap, std::max(1, t.max_ctas / 2));
        const int clusters = (int)std::max<int64_t>(1, std::min<int64_t>(max_tiles, ccap));
        cudaLaunchConfig_t cfg{};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(2 * clusters);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = t.smem;
        cfg.stream = st;
        cfg.attrs = at;
        cfg.numAttrs = 1;
#define CBX_TC_LAUNCH(R, T) CBX_CUDA(cudaLaunchKernelEx(&cfg, conv_tc_kernel<R, T, true>, a))
        if (tc == 0) {
            if (rowlane) CBX_TC_LAUNCH(true, 0); else CBX_TC_LAUNCH(false, 0);
        } else if (tc == 8) {
            if (rowlane) CBX_TC_LAUNCH(true, 8); else CBX_TC_LAUNCH(false, 8);
        } else {
            if (rowlane) CBX_TC_LAUNCH(true, 16); else CBX_TC_LAUNCH(false, 16);
        }
#undef CBX_TC_LAUNCH
        return;
    }
    const int64_t max_tiles = (full_count + tc::kTileM - 1) / tc::kTileM;
    const int64_t cap = t.max_ctas > 0 ? t.max_ctas : (int64_t)kNumSMs * t.ctas_per_sm;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(max_tiles, cap));
    if (t.i8) {
        launch_k(conv_tc_kernel<true, 0, false, true>, dim3(grid), dim3(kThreads), t.smem, st, a);
        return;
    }
#define CBX_TC_LAUNCH(R, T) launch_k(conv_tc_kernel<R, T, false>, dim3(grid), dim3(kThreads), t.smem, st, a)
    if (tc == 0) {
        if (rowlane) CBX_TC_LAUNCH(true, 0); else CBX_TC_LAUNCH(false, 0);
    } else if (tc == 8) {
        if (rowlane) CBX_TC_LAUNCH(true, 8); else CBX_TC_LAUNCH(false, 8);
    } else {
        if (rowlane) CBX_TC_LAUNCH(true, 16); else CBX_TC_LAUNCH(false, 16);
    }
#undef CBX_TC_LAUNCH
}

}  // namespace cbx
