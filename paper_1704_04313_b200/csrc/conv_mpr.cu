// conv_mpr.cu -- "multi-pixel row" gathered convolution on tcgen05 for the
// narrow layers of the change-based network (paper: layer 1, 3 -> 4 channels
// and layer 2, 4 -> 52 channels, both 7x7).
//
// Replaces gen_x_reduced + gemm + update_output (cbconv.cpp:115-155,
// baseline.cpp:47-63) like conv_tc.cu, with two changes that matter for a
// layer with few output channels:
//
// * A tcgen05.mma instruction costs ~84 clk per 32 K-bytes at M = 128 for any
//   N <= 64 (~136 clk at N = 256; scripts/mma_shape_probe.cu,
//   profiles/r2_mma_shape.log), so a 4- or 52-channel layer with one output
//   pixel per A row uses the tensor core at 2-25 %. Here an A row is a GROUP
//   of R horizontally adjacent output pixels: its K is the union receptive
//   field (kh rows x (kw + R - 1) columns, shared by the R pixels) and its N
//   holds the R pixels' output channels (B row j*Opad + o carries the filter
//   of channel o shifted to column offset j; zero elsewhere). Per output
//   pixel the MMA work drops by R * (kw) / (kw + R - 1) while N grows into
//   the free range.
// * The gather is register-staged (LDG.128 -> convert -> STS.128 into the
//   SW128 K-major row, fence.proxy.async, mbarrier arrive): the per-K-block
//   LDGSTS of conv_tc moves ~23 B/clk/SM, plain vector loads and stores
//   several times that, and the conversion (fp32 -> fp16 operands) happens
//   on the way, with no fp16 shadow tensor in HBM.
//
// Modes: MODE 0 = kind::i8 over the RGBX bytes of an 8-bit camera frame
// (filters as three base-256 digits, exact integer accumulation, see
// conv_tc.hpp); MODE 1 = kind::f16 over an fp32 channels-last input with 4
// channels per pixel (rounded to nearest fp16 while gathering; values beyond
// the fp16 range raise the frame's overflow flag).
//
// The tile list holds GROUP entries (gid << 4 | mask): gid = s*Ho*Gw + y*Gw + gx
// (Gw = ceil(Wo / R)), mask = the group's updated pixels (dilate_compact with
// R > 1). Pixels outside the mask are computed and discarded (the stored
// tensor keeps its previous value there, like the reference's update_output).
#include <algorithm>
#include <cmath>
#include <type_traits>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_fp16.h>

#include "conv_mpr.hpp"
#include "engine.hpp"
#include "tc_ptx.cuh"

namespace cbx {

namespace {

using namespace tc;

constexpr int kABytes = kTileM * 128;
constexpr int kEpi = 128, kProd = 256;  // 8 producer warps: thread = (tile row, half of its granules)
constexpr int kThreads = kEpi + kProd + 32;
constexpr int kMmaWarp = (kEpi + kProd) / 32;
constexpr int kMaxSmem = 232448;
constexpr int kMaxGran = 64;  // granule table entries (8 K-blocks)

struct MprArgs {
    const void* in;
    int64_t in_ss;  // input units per stream (MODE 0: 4-byte RGBX pixels, MODE 1: floats)
    int in_Wp, in_Cp, in_hh, in_hw;
    float* out;
    int64_t out_ss;
    int out_Wp, out_Cp, out_hh, out_hw;
    int O, Ho, Wo, Gw;
    int kh, kw, ph, pw;
    const uint32_t* list;
    const int* count;
    int64_t full_groups;
    const uint8_t* Bw;  // [NKB][Npad][128 B]
    const float* bias;
    const float* qsc;   // MODE 0: per-channel scale / 255
    int NKB, Npad, Opad, kinst_last;
    int stages, acc_cols, tmem_cols;
    int relu;
    BitMask chg;
    float tau;
    unsigned long long* chg_cnt;
    int cnt_stride;
    int* ovf;
    int fast;
    FastDiv fd_plane, fd_gw;  // Ho * Gw, Gw
    int win0;                 // input column of window slot 0 relative to the group's x0 (units: pixels)
    int gpr;                  // granules per kernel row
};

// Ring position without a division per K-block.
struct RingPos {
    uint32_t st = 0, ph = 0;
    __device__ __forceinline__ void next(int n) {
        if (++st == (uint32_t)n) {
            st = 0;
            ph ^= 1u;
        }
    }
};

__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

template <int R>
__device__ __forceinline__ void group_of(const MprArgs& a, uint32_t gid, int& s, int& y, int& x0) {
    if (a.fast) {
        const uint32_t ss = a.fd_plane.div(gid);
        const uint32_t rem = gid - ss * (uint32_t)(a.Ho * a.Gw);
        const uint32_t yy = a.fd_gw.div(rem);
        s = (int)ss;
        y = (int)yy;
        x0 = (int)(rem - yy * (uint32_t)a.Gw) * R;
    } else {
        const int64_t plane = (int64_t)a.Ho * a.Gw;
        s = (int)(gid / plane);
        const int rem = (int)(gid - (int64_t)s * plane);
        y = rem / a.Gw;
        x0 = (rem - y * a.Gw) * R;
    }
}

template <int MODE, int R>
__global__ void __launch_bounds__(kThreads, MODE == 0 ? 2 : 1) conv_mpr_kernel(MprArgs a) {
    pdl_trigger();  // (the prologue below touches only this launch's constants)
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int NS = a.stages;
    const uint32_t b_kb = (uint32_t)a.Npad * 128u;  // bytes of one K-block of B
    uint8_t* sA = smem;
    uint8_t* sB = sA + (size_t)NS * kABytes;  // resident filter image
    int2* sGran = reinterpret_cast<int2*>(sB + (size_t)a.NKB * b_kb);  // granule -> (source offset, pixels)
    float* sBias = reinterpret_cast<float*>(sGran + kMaxGran);
    float* sQs = sBias + ((a.O + 3) & ~3);
    uint64_t* bars = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(sQs + ((a.O + 3) & ~3)) + 7) & ~uintptr_t(7));
    uint64_t* full = bars;
    uint64_t* empty = full + NS;
    uint64_t* tfull = empty + NS;
    uint64_t* tempty = tfull + 2;
    uint64_t* bready = tempty + 2;
    uint32_t* sTmem = reinterpret_cast<uint32_t*>(bready + 1);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // granule table: granule G of the A row (16 bytes) holds kernel row
    // G / gpr, window slots covering 16 bytes from slot (G % gpr) * spg
    // (MODE 0: 4 RGBX pixels, MODE 1: 2 pixels of 4 fp32 channels -> fp16);
    // .x = source offset in input units from the group's window origin, .y =
    // number of real pixels in the granule (0: zero granule)
    if (tid < kMaxGran) {
        int2 e = make_int2(0, 0);
        const int G = tid;
        if (G < a.kh * a.gpr) {
            const int kj = G / a.gpr, part = G - kj * a.gpr;
            if (MODE == 0) {
                e = make_int2(kj * a.in_Wp + 4 * part, 4);
            } else {
                const int c0 = 2 * part, span = a.kw + R - 1;
                e = make_int2((kj * a.in_Wp + c0) * a.in_Cp, c0 < span ? min(2, span - c0) : 0);
            }
        }
        sGran[G] = e;
    }
    for (int o = tid; o < a.O; o += kThreads) {
        sBias[o] = a.bias[o];
        if (MODE == 0) sQs[o] = a.qsc[o];
    }
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], kProd);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], kEpi);
        }
        mbar_init(bready, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(sTmem)),
                     "r"(a.tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *sTmem;
    if (tid == 0) {  // the whole filter image, once per CTA
        mbar_arrive_expect_tx(bready, (uint32_t)a.NKB * b_kb);
        for (int kb = 0; kb < a.NKB; ++kb) bulk_g2s(sB + (size_t)kb * b_kb, a.Bw + (size_t)kb * b_kb, b_kb, bready);
    }

    pdl_wait();  // the group list / count and the input tensor come from the previous kernels
    const int64_t total = a.list ? (int64_t)*a.count : a.full_groups;
    const int64_t ntiles = (total + kTileM - 1) / kTileM;
    const int64_t tile_first = blockIdx.x, tile_step = gridDim.x;
    auto entry = [&](int64_t t, int r) -> int64_t {  // group entry of row r of tile t, -1 past the end
        const int64_t n = t * kTileM + r;
        if (t >= ntiles || n >= total) return -1;
        if (a.list) {  // R = 1 lists hold plain pixel indices (extract_indexes order)
            const uint32_t v = __ldg(a.list + n);
            return R == 1 ? (((int64_t)v << 4) | 1) : (int64_t)v;
        }
        // full mode: every group, mask = its pixels inside the row
        const uint32_t gid = (uint32_t)n;
        int s, y, x0;
        group_of<R>(a, gid, s, y, x0);
        const int m = (1 << min(R, a.Wo - x0)) - 1;
        return ((int64_t)gid << 4) | m;
    };

    if (warp >= 4 && warp < kMmaWarp) {
        // ================= producers =================
        // thread = (tile row r, half hf): granules 4hf .. 4hf+3 of every
        // K-block of row r. Software-pipelined two deep: the loads of the
        // next K-block (or of the next tile's first) are in flight while
        // this one is converted and stored, so a producer keeps up to two
        // K-blocks of gathers outstanding (register staging has no cp.async
        // to run ahead with).
        const int pt = tid - kEpi;
        const int r = pt & (kTileM - 1), hf = pt >> 7;
        const uint32_t swz = (uint32_t)(r & 7);
        using Raw = typename std::conditional<MODE == 0, uint4[4], float4[4][2]>::type;
        auto issue = [&](int64_t base, bool valid, int kb, Raw& raw) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int2 t = sGran[kb * 8 + 4 * hf + q];
                if constexpr (MODE == 0) {
                    const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const uint32_t*>(a.in) + base);
                    raw[q] = (valid && t.y) ? __ldg(src + (t.x >> 2)) : make_uint4(0u, 0u, 0u, 0u);
                } else {
                    const float* src = reinterpret_cast<const float*>(a.in) + base;
                    raw[q][0] = (valid && t.y > 0) ? __ldg(reinterpret_cast<const float4*>(src + t.x))
                                                   : make_float4(0.f, 0.f, 0.f, 0.f);
                    raw[q][1] = (valid && t.y > 1) ? __ldg(reinterpret_cast<const float4*>(src + t.x + a.in_Cp))
                                                   : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
        };
        auto row_base = [&](int64_t e, int64_t& base) -> bool {
            if (e < 0) return false;
            int s, y, x0;
            group_of<R>(a, (uint32_t)(e >> 4), s, y, x0);
            base = (int64_t)s * a.in_ss + ((int64_t)(y - a.ph + a.in_hh) * a.in_Wp + (x0 + a.win0 + a.in_hw)) * a.in_Cp;
            return true;
        };
        RingPos rg;
        int64_t tile = tile_first;
        int64_t base = 0, nbase = 0;
        bool valid = tile < ntiles && row_base(entry(tile, r), base);
        int64_t enext = entry(tile + tile_step, r);
        Raw cur, nxt;
        if (tile < ntiles) issue(base, valid, 0, cur);
        while (tile < ntiles) {
            for (int kb = 0; kb < a.NKB; ++kb, rg.next(NS)) {
                // prefetch: the next K-block, or the next tile's first
                const bool last = kb + 1 == a.NKB;
                if (!last) {
                    issue(base, valid, kb + 1, nxt);
                } else if (tile + tile_step < ntiles) {
                    const bool nv = row_base(enext, nbase);
                    issue(nbase, nv, 0, nxt);
                }
                uint4 g[4];
                if constexpr (MODE == 0) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) g[q] = cur[q];
                } else {
                    bool big = false;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                            big |= fabsf(cur[q][h].x) > 65504.0f || fabsf(cur[q][h].y) > 65504.0f ||
                                   fabsf(cur[q][h].z) > 65504.0f || fabsf(cur[q][h].w) > 65504.0f;
                        g[q] = make_uint4(pack_f16x2(cur[q][0].x, cur[q][0].y), pack_f16x2(cur[q][0].z, cur[q][0].w),
                                          pack_f16x2(cur[q][1].x, cur[q][1].y), pack_f16x2(cur[q][1].z, cur[q][1].w));
                    }
                    if (big && a.ovf) atomicOr(a.ovf, 1);
                }
                const uint32_t st = rg.st, ph = rg.ph;
                mbar_wait(&empty[st], ph ^ 1u);
                uint4* row = reinterpret_cast<uint4*>(sA + (size_t)st * kABytes + r * 128);
#pragma unroll
                for (int q = 0; q < 4; ++q) row[(4 * hf + q) ^ swz] = g[q];
                fence_proxy_async();
                mbar_arrive(&full[st]);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if constexpr (MODE == 0) {
                        cur[q] = nxt[q];
                    } else {
                        cur[q][0] = nxt[q][0];
                        cur[q][1] = nxt[q][1];
                    }
                }
            }
            tile += tile_step;
            base = nbase;
            valid = tile < ntiles && enext >= 0;
            enext = entry(tile + tile_step, r);
        }
    } else if (warp == kMmaWarp) {
        // ================= MMA issuer =================
        const uint32_t id = MODE == 0 ? idesc_i8(a.Npad) : idesc_f16(a.Npad);
        const uint64_t a_desc0 = smem_desc(smem_u32(sA)), b_desc0 = smem_desc(smem_u32(sB));
        const uint64_t a_st = kABytes >> 4, b_st = b_kb >> 4;
        mbar_wait(bready, 0);
        RingPos rg;
        uint32_t acc_it = 0;
        for (int64_t tile = tile_first; tile < ntiles; tile += tile_step, ++acc_it) {
            const uint32_t as = acc_it & 1u, aph = (acc_it >> 1) & 1u;
            mbar_wait(&tempty[as], aph ^ 1u);
            tc_fence_after();
            const uint32_t d = tmem_base + as * a.acc_cols;
            for (int kb = 0; kb < a.NKB; ++kb, rg.next(NS)) {
                const uint32_t st = rg.st, ph = rg.ph;
                mbar_wait(&full[st], ph);
                tc_fence_after();
                const uint64_t ad = a_desc0 + st * a_st, bd = b_desc0 + kb * b_st;
                const int nk = kb + 1 == a.NKB ? a.kinst_last : 4;
                if (elect_one()) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        if (k < nk) {
                            const uint32_t acc = (kb | k) ? 1u : 0u;
                            if (MODE == 0)
                                mma_i8(d, ad + 2 * k, bd + 2 * k, id, acc);
                            else
                                mma_f16(d, ad + 2 * k, bd + 2 * k, id, acc);
                        }
                    }
                    mma_commit(&empty[st]);
                }
                __syncwarp();
            }
            if (elect_one()) mma_commit(&tfull[as]);
            __syncwarp();
        }
    } else {
        // ================= epilogue: thread = TMEM lane = tile row =================
        const int r = tid;
        const uint32_t trow = tmem_base + ((uint32_t)(warp * 32) << 16);
        const int64_t plane = (int64_t)a.Ho * a.Wo;
        uint32_t acc_it = 0;
        int64_t enext = entry(tile_first, r);
        for (int64_t tile = tile_first; tile < ntiles; tile += tile_step, ++acc_it) {
            const uint32_t as = acc_it & 1u, aph = (acc_it >> 1) & 1u;
            const int64_t e = enext;
            enext = entry(tile + tile_step, r);
            const bool valid = e >= 0;
            const uint32_t mask = valid ? (uint32_t)(e & 15) : 0u;
            int s = 0, y = 0, x0 = 0;
            if (valid) group_of<R>(a, (uint32_t)(e >> 4), s, y, x0);
            float* drow = a.out + (int64_t)s * a.out_ss + ((int64_t)(y + a.out_hh) * a.out_Wp + (x0 + a.out_hw)) * a.out_Cp;
            mbar_wait(&tfull[as], aph);
            tc_fence_after();
            const uint32_t tb = trow + as * a.acc_cols;
            uint32_t chg_bits = 0;
            // TMEM -> registers in batches (several tcgen05.ld, one wait):
            // MODE 0 the three digit columns of 4 channels of every sub-pixel,
            // MODE 1 up to 64 channels of one sub-pixel
            auto store4 = [&](float* dst, int o0, const float (&v)[4], bool& changed) {
                if (o0 + 4 <= a.O) {
                    float4* q4 = reinterpret_cast<float4*>(dst + o0);
                    if (a.chg.d) {
                        const float4 old = *q4;
                        changed |= ref_changed(v[0], old.x, a.tau) | ref_changed(v[1], old.y, a.tau) |
                                   ref_changed(v[2], old.z, a.tau) | ref_changed(v[3], old.w, a.tau);
                    }
                    *q4 = make_float4(v[0], v[1], v[2], v[3]);
                } else {
                    for (int k = 0; k < 4 && o0 + k < a.O; ++k) {
                        if (a.chg.d) changed |= ref_changed(v[k], dst[o0 + k], a.tau);
                        dst[o0 + k] = v[k];
                    }
                }
            };
            if constexpr (MODE == 0) {
                for (int o0 = 0; o0 < a.O; o0 += 4) {
                    int32_t q[R][3][4];
#pragma unroll
                    for (int j = 0; j < R; ++j)
#pragma unroll
                        for (int d = 0; d < 3; ++d) tmem_ld4(tb + (uint32_t)((j * 3 + d) * a.Opad + o0), q[j][d]);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < R; ++j) {
                        float v[4];
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const int o = min(o0 + k, a.O - 1);
                            const float tot = fmaf((float)q[j][2][k], 65536.0f, fmaf((float)q[j][1][k], 256.0f, (float)q[j][0][k]));
                            const float t = fmaf(tot, sQs[o], sBias[o]);
                            v[k] = a.relu ? ref_relu(t) : t;
                        }
                        if ((mask >> j) & 1u) {
                            bool changed = false;
                            store4(drow + j * a.out_Cp, o0, v, changed);
                            if (changed) chg_bits |= 1u << j;
                        }
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    const bool live = (mask >> j) & 1u;
                    float* dst = drow + j * a.out_Cp;
                    bool changed = false;
                    for (int c0 = 0; c0 < a.O; c0 += 64) {
                        const int ng = min(16, (a.O - c0 + 3) / 4);
                        int32_t q[16][4];
#pragma unroll
                        for (int g = 0; g < 16; ++g)
                            if (g < ng) tmem_ld4(tb + (uint32_t)(j * a.Opad + c0 + 4 * g), q[g]);
                        tmem_wait_ld();
                        if (!live) continue;
#pragma unroll
                        for (int g = 0; g < 16; ++g) {
                            if (g < ng) {
                                float v[4];
#pragma unroll
                                for (int k = 0; k < 4; ++k) {
                                    const int o = min(c0 + 4 * g + k, a.O - 1);
                                    const float t = __fadd_rn(__int_as_float(q[g][k]), sBias[o]);
                                    v[k] = a.relu ? ref_relu(t) : t;
                                }
                                store4(dst, c0 + 4 * g, v, changed);
                            }
                        }
                    }
                    if (live && changed) chg_bits |= 1u << j;
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty[as]);
            if (a.chg.d) {
                for (int j = 0; j < R; ++j)
                    if ((chg_bits >> j) & 1u) bit_set(a.chg, s, y, x0 + j);
                if (a.chg_cnt) {
                    // per-stream count of newly changed pixels: one atomic per
                    // warp when its groups share a stream (the common case)
                    const unsigned act = __ballot_sync(0xffffffffu, valid);
                    const int n = __popc(chg_bits);
                    if (valid) {
                        const unsigned same = __match_any_sync(act, s);
                        if (same == act) {
                            const int sum = __reduce_add_sync(act, n);
                            if ((int)(threadIdx.x & 31) == __ffs(act) - 1 && sum)
                                atomicAdd(a.chg_cnt + (int64_t)s * a.cnt_stride, (unsigned long long)sum);
                        } else if (n) {
                            atomicAdd(a.chg_cnt + (int64_t)s * a.cnt_stride, (unsigned long long)n);
                        }
                    }
                }
            }
            (void)plane;
            (void)lane;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(a.tmem_cols));
    }
}

template <int MODE, int R>
void set_attr() {
    CBX_CUDA(cudaFuncSetAttribute(conv_mpr_kernel<MODE, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
}

}  // namespace

struct MprLayer {
    cbx_geom g;
    int mode = 0, R = 4;
    int NKB = 0, Npad = 0, Opad = 0, kinst_last = 4, gpr = 0, win0 = 0;
    int stages = 0, acc_cols = 0, tmem_cols = 0;
    int ctas_per_sm = 1;
    int max_ctas = 0;  // persistent grid cap (CBX_TC_MAXCTAS: tests walk several tiles per CTA)
    size_t smem = 0;
    uint8_t* Bw = nullptr;
    float* qsc = nullptr;
};

void MprLayerDeleter::operator()(MprLayer* p) const {
    if (!p) return;
    if (p->Bw) cudaFree(p->Bw);
    if (p->qsc) cudaFree(p->qsc);
    delete p;
}

int mpr_group_width(const MprLayer& t) { return t.R; }
int mpr_mode(const MprLayer& t) { return t.mode; }

bool mpr_supported(const cbx_geom& g, int mode, int R) {
    if (g.strideH != 1 || g.strideW != 1 || g.kernelW > 16 || g.kernelH > 32 || (R != 1 && R != 2 && R != 4)) return false;
    if (mode == 0) return R == 4 && g.inChannels <= 4 && 3 * R * round_up(g.outChannels, 4) <= 256;
    return g.inChannels <= 4 && R * round_up(g.outChannels, 4) <= 256;
}

std::unique_ptr<MprLayer, MprLayerDeleter> make_mpr_layer(const cbx_geom& g, int mode, int R, int in_hw) {
    if (!mpr_supported(g, mode, R)) throw Error(CBX_E_ARG, "multi-pixel-row conv: unsupported geometry");
    std::unique_ptr<MprLayer, MprLayerDeleter> t(new MprLayer);
    t->g = g;
    t->mode = mode;
    t->R = R;
    t->Opad = (int)round_up(g.outChannels, 4);
    const int span = g.kernelW + R - 1;  // window columns that carry real taps
    if (mode == 0) {
        // RGBX windows start on a 16-byte boundary: x0 is a multiple of R = 4
        // (R divides 4 here), so the window origin x0 - pw - a with
        // a = (in_hw - pw) mod 4 is aligned in the halo'd row
        const int a = ((in_hw - g.padW) % 4 + 4) % 4;
        t->win0 = -g.padW - a;
        t->gpr = (a + span + 3) / 4;
        t->Npad = (int)round_up(3 * R * t->Opad, 16);
    } else {
        t->win0 = -g.padW;
        t->gpr = (span + 1) / 2;
        t->Npad = (int)round_up(R * t->Opad, 16);
    }
    const int gran = g.kernelH * t->gpr;
    if (gran > kMaxGran) throw Error(CBX_E_ARG, "multi-pixel-row conv: receptive field too large");
    t->NKB = (gran + 7) / 8;
    t->kinst_last = ((gran - 8 * (t->NKB - 1)) + 1) / 2;
    t->acc_cols = (int)round_up(t->Npad, 32);
    int cols = 32;
    while (cols < 2 * t->acc_cols) cols *= 2;
    t->tmem_cols = cols;
    const size_t b_bytes = (size_t)t->NKB * t->Npad * 128;
    const size_t fixed = 1024 + b_bytes + kMaxGran * 8 + 2 * round_up(g.outChannels, 4) * 4 + 16 + 8 * (2 * 16 + 5) + 16;
    // CTAs per SM: two when the filters and a few stages fit twice (more
    // independent producers in flight), else one; CBX_MPR_CTAS overrides (tuning)
    t->ctas_per_sm = mode == 0 && fixed + 4 * (size_t)kABytes <= (size_t)kMaxSmem / 2 - 1024 ? 2 : 1;
    if (const char* e = std::getenv("CBX_MPR_CTAS")) t->ctas_per_sm = std::max(1, std::min(2, std::atoi(e)));
    const size_t budget = t->ctas_per_sm == 2 ? (size_t)kMaxSmem / 2 - 1024 : (size_t)kMaxSmem;
    // three A stages (plus the two K-blocks in flight in the producers'
    // registers): a small footprint so the other lane's kernels fit beside it
    int ns = 3;
    if (const char* e = std::getenv("CBX_MPR_STAGES")) ns = std::max(2, std::min(12, std::atoi(e)));  // (tuning)
    while (ns > 2 && fixed + (size_t)ns * kABytes > budget) --ns;
    if (fixed + (size_t)ns * kABytes > budget) throw Error(CBX_E_ARG, "multi-pixel-row conv: filters too large");
    t->stages = ns;
    t->smem = fixed + (size_t)ns * kABytes;
    if (const char* e = std::getenv("CBX_TC_MAXCTAS")) t->max_ctas = std::max(1, std::atoi(e));
    if (mode == 0) {
        if (R == 4) set_attr<0, 4>(); else if (R == 2) set_attr<0, 2>(); else set_attr<0, 1>();
    } else {
        if (R == 4) set_attr<1, 4>(); else if (R == 2) set_attr<1, 2>(); else set_attr<1, 1>();
    }
    CBX_CUDA(cudaMalloc(&t->Bw, b_bytes));
    CBX_CUDA(cudaMemset(t->Bw, 0, b_bytes));  // (legacy stream: synchronized below)
    if (mode == 0) {
        CBX_CUDA(cudaMalloc(&t->qsc, sizeof(float) * g.outChannels));
        CBX_CUDA(cudaMemset(t->qsc, 0, sizeof(float) * g.outChannels));
    }
    // the zeroing ran on the legacy default stream; the weight uploads run
    // on the engine's non-blocking stream, which is not ordered after it
    CBX_CUDA(cudaStreamSynchronize(nullptr));
    return t;
}

// Filter image. K of an A row: kernel row kj, window slot w (input column
// x0 + win0 + w), channel c. MODE 0: byte k = (kj * gpr * 4 + w) * 4 + c;
// MODE 1: fp16 element k = (kj * gpr * 2 + w) * 4 + c. B row n: MODE 0
// n = (j * 3 + q) * Opad + o (digit q of channel o of sub-pixel j); MODE 1
// n = j * Opad + o. Weight of (kj, w, c) for sub-pixel j is
// K[o][c][kj][ki] with ki = w + win0 + pw - j when 0 <= ki < kw, else 0.
void mpr_load_weights(MprLayer& t, const float* K, cudaStream_t st) {
    const cbx_geom& g = t.g;
    const int khw = g.kernelH * g.kernelW, Kref = g.inChannels * khw;
    const int R = t.R, O = g.outChannels;
    std::vector<uint8_t> img((size_t)t.NKB * t.Npad * 128, 0);
    auto put = [&](int row, int kbyte, const void* v, int n) {  // kbyte: byte offset of the element in the A row
        const int kb = kbyte / 128, inb = kbyte % 128, gran = inb / 16;
        uint8_t* dst = img.data() + (size_t)kb * t.Npad * 128 + (size_t)row * 128 + ((gran ^ (row & 7)) * 16) + inb % 16;
        std::memcpy(dst, v, n);
    };
    const int lead = t.win0 + g.padW;  // window slot w maps to tap ki = w + lead - j
    const int slots = t.mode == 0 ? 4 * t.gpr : 2 * t.gpr;
    if (t.mode == 0) {
        std::vector<float> qs(O, 0.0f);
        for (int o = 0; o < O; ++o) {
            double mx = 0.0;
            for (int i = 0; i < Kref; ++i) mx = std::max(mx, (double)std::fabs(K[(size_t)o * Kref + i]));
            const double sc = mx > 0.0 ? mx / 4194304.0 : 1.0;
            qs[o] = (float)(sc / 255.0);
            for (int c = 0; c < g.inChannels; ++c)
                for (int kj = 0; kj < g.kernelH; ++kj)
                    for (int ki = 0; ki < g.kernelW; ++ki) {
                        long long wi = std::llround((double)K[(size_t)o * Kref + ((size_t)c * g.kernelH + kj) * g.kernelW + ki] / sc);
                        int8_t d[3];
                        for (int q = 0; q < 3; ++q) {
                            long long r = ((wi % 256) + 256) % 256;
                            if (r >= 128) r -= 256;
                            wi = (wi - r) / 256;
                            d[q] = (int8_t)r;
                        }
                        if (wi != 0) throw Error(CBX_E_ARG, "kind::i8 filter digits overflow");
                        for (int j = 0; j < R; ++j) {
                            const int w = ki - lead + j;
                            if (w < 0 || w >= slots) continue;
                            const int kbyte = (kj * slots + w) * 4 + c;
                            for (int q = 0; q < 3; ++q) put((j * 3 + q) * t.Opad + o, kbyte, &d[q], 1);
                        }
                    }
        }
        CBX_CUDA(cudaMemcpyAsync(t.qsc, qs.data(), sizeof(float) * O, cudaMemcpyHostToDevice, st));
    } else {
        for (size_t i = 0; i < (size_t)O * Kref; ++i)
            if (std::fabs(K[i]) > 65504.0f)
                throw Error(CBX_E_ARG, "a filter weight of a kind::f16 layer exceeds the fp16 range (|w| > 65504); "
                                       "create the context with CBX_PREC_TF32");
        for (int o = 0; o < O; ++o)
            for (int c = 0; c < g.inChannels; ++c)
                for (int kj = 0; kj < g.kernelH; ++kj)
                    for (int ki = 0; ki < g.kernelW; ++ki) {
                        const __half h = __float2half_rn(K[(size_t)o * Kref + ((size_t)c * g.kernelH + kj) * g.kernelW + ki]);
                        for (int j = 0; j < R; ++j) {
                            const int w = ki - lead + j;
                            if (w < 0 || w >= slots) continue;
                            put(j * t.Opad + o, ((kj * slots + w) * 4 + c) * 2, &h, 2);
                        }
                    }
    }
    CBX_CUDA(cudaMemcpyAsync(t.Bw, img.data(), img.size(), cudaMemcpyHostToDevice, st));
    CBX_CUDA(cudaStreamSynchronize(st));
}

void launch_conv_mpr(const MprLayer& t, TensorView in, TensorView out, const float* bias, const uint32_t* list,
                     const int* count, int S, bool relu, BitMask chg, float tau, unsigned long long* cnt, int cstride,
                     int* ovf, cudaStream_t st) {
    MprArgs a{};
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
    a.Gw = (out.W + t.R - 1) / t.R;
    a.kh = t.g.kernelH;
    a.kw = t.g.kernelW;
    a.ph = t.g.padH;
    a.pw = t.g.padW;
    a.list = list;
    a.count = count;
    a.full_groups = (int64_t)S * a.Ho * a.Gw;
    a.Bw = t.Bw;
    a.bias = bias;
    a.qsc = t.qsc;
    a.NKB = t.NKB;
    a.Npad = t.Npad;
    a.Opad = t.Opad;
    a.kinst_last = t.kinst_last;
    a.stages = t.stages;
    a.acc_cols = t.acc_cols;
    a.tmem_cols = t.tmem_cols;
    a.relu = relu;
    a.chg = chg;
    a.tau = tau;
    a.chg_cnt = chg.d ? cnt : nullptr;
    a.cnt_stride = cstride;
    a.ovf = ovf;
    a.fast = a.full_groups < ((int64_t)1 << 27);  // gid << 4 stays below 2^31
    a.fd_plane = FastDiv::make((uint32_t)std::max(1, a.Ho * a.Gw));
    a.fd_gw = FastDiv::make((uint32_t)a.Gw);
    a.win0 = t.win0;
    a.gpr = t.gpr;
    if (t.mode == 0 && in.Cp != 1) throw Error(CBX_E_SHAPE, "kind::i8 conv: the input must be the RGBX frame");
    if (t.mode == 1 && in.Cp != 4) throw Error(CBX_E_SHAPE, "multi-pixel-row f16 conv: the input must have 4 channels");
    const int64_t max_tiles = (a.full_groups + kTileM - 1) / kTileM;
    const int64_t cap = t.max_ctas > 0 ? t.max_ctas : (int64_t)kNumSMs * t.ctas_per_sm;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(max_tiles, cap));
#define CBX_MPR(M_, R_) launch_k(conv_mpr_kernel<M_, R_>, dim3(grid), dim3(kThreads), t.smem, st, a)
    if (t.mode == 0) {
        if (t.R == 4) CBX_MPR(0, 4); else if (t.R == 2) CBX_MPR(0, 2); else CBX_MPR(0, 1);
    } else {
        if (t.R == 4) CBX_MPR(1, 4); else if (t.R == 2) CBX_MPR(1, 2); else CBX_MPR(1, 1);
    }
#undef CBX_MPR
}

}  // namespace cbx
