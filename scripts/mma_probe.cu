// mma_probe.cu -- tcgen05 kind::tf32 issue-rate probe (tuning aid, not product).
//
// One persistent CTA per SM (or one 2-CTA cluster per TPC); an elected thread
// issues ITERS K-blocks of MMAs (4 K=8 steps per 128-byte K-block) from shared
// memory stages, committing each K-block to an mbarrier; optional producer
// warps refill A/B stages from global memory with cp.async.bulk (TMA engine)
// through a full/empty pipeline. Reports TFLOP/s and flop/clk/SM, so the
// shapes of conv_tc (M=128 N=160+144, 256+48, pair M=256) can be compared
// against the MMA-only ceiling and the ceiling with shared-memory fills.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_probe scripts/mma_probe.cu
//   ./mma_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n\t.reg .pred P;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}" ::"r"(su32(b)), "r"(ph));
}
__device__ __forceinline__ void mbar_wait_cl(uint64_t* b, uint32_t ph) {
    asm volatile("{\n\t.reg .pred P;\n\tW_%=:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(b)) : "memory");
}
__device__ __forceinline__ uint64_t desc(uint32_t addr) {
    return (uint64_t)((addr & 0x3FFFFu) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc(int N, int M) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma1(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit1(uint64_t* b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void commit2(uint64_t* b) {
    asm volatile("{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\ttcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ uint32_t crank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t r) { uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(su32(p)), "r"(r)); return o; }
__device__ __forceinline__ void csync() { asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory"); }

struct P {
    int pair;          // 0: cta_group::1 M=128; 1: cta_group::2 M=256
    int N0, N1;        // instruction widths (N1 = 0: one instruction per K step)
    int iters;         // K-blocks
    int stages;
    int fillA, fillB;  // refill A (16 KB) / B (rows*128 B) per K-block with TMA
    int sync_each;     // wait for each K-block's commit before the next (MMA round-trip latency)
    const uint8_t* gA; const uint8_t* gB;  // sources of the fills (L2-resident)
    long long* cyc;
};

template <bool PAIR>
__global__ void __launch_bounds__(128, 1) probe(P p) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);
    const uint32_t rank = PAIR ? crank() : 0;
    const int Brows = PAIR ? (p.N0 + p.N1) / 2 : (p.N0 + p.N1);
    const uint32_t aB = 16384, bB = Brows * 128;
    uint8_t* sA = sm;
    uint8_t* sB = sA + p.stages * aB;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + p.stages * bB);
    uint64_t* empty = full + p.stages;
    uint64_t* pfull = empty + p.stages;
    uint64_t* done = pfull + p.stages;
    uint32_t* tm = reinterpret_cast<uint32_t*>(done + 1);
    const int tid = threadIdx.x, warp = tid >> 5;
    for (uint32_t i = tid * 16; i < p.stages * (aB + bB); i += 128 * 16) *reinterpret_cast<uint4*>(sm + i) = make_uint4(0, 0, 0, 0);
    if (tid == 0) {
        for (int s = 0; s < p.stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); mbar_init(&pfull[s], 1); }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 0) {
        if (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tm)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tm)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (PAIR) csync(); else __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = *tm;
    const bool fills = p.fillA || p.fillB;
    const uint32_t fill_bytes = (p.fillA ? aB : 0) + (p.fillB ? bB : 0);
    long long t0 = clock64();
    if (warp == 1 && (tid & 31) == 0 && fills) {
        // producer: one bulk copy per operand per K-block, from an L2-resident source
        for (int it = 0; it < p.iters; ++it) {
            const int st = it % p.stages; const uint32_t ph = (it / p.stages) & 1;
            if (PAIR) mbar_wait_cl(&empty[st], ph ^ 1); else mbar_wait(&empty[st], ph ^ 1);
            const size_t src = (size_t)(it % 64);
            if (PAIR) {
                // each CTA's bytes complete on its own full barrier; the peer's
                // relay thread forwards "full" to the leader (pfull)
                mbar_expect(&full[st], fill_bytes);
                if (p.fillA) bulk(sA + st * aB, p.gA + src * aB, aB, &full[st]);
                if (p.fillB) bulk(sB + st * bB, p.gB + src * bB, bB, &full[st]);
            } else {
                mbar_expect(&full[st], fill_bytes);
                if (p.fillA) bulk(sA + st * aB, p.gA + src * aB, aB, &full[st]);
                if (p.fillB) bulk(sB + st * bB, p.gB + src * bB, bB, &full[st]);
            }
        }
    } else if (PAIR && warp == 2 && (tid & 31) == 0 && rank != 0 && fills) {
        for (int it = 0; it < p.iters; ++it) {
            const int st = it % p.stages; const uint32_t ph = (it / p.stages) & 1;
            mbar_wait(&full[st], ph);
            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa(&pfull[st], 0)) : "memory");
        }
    } else if (warp == 2 && (tid & 31) == 0 && rank == 0) {
        const int M = PAIR ? 256 : 128;
        const uint32_t i0 = idesc(p.N0, M), i1 = idesc(p.N1 ? p.N1 : 16, M);
        const uint32_t b1 = (uint32_t)(PAIR ? p.N0 / 2 : p.N0) * 128u;
        for (int it = 0; it < p.iters; ++it) {
            const int st = it % p.stages; const uint32_t ph = (it / p.stages) & 1;
            if (fills) { mbar_wait(&full[st], ph); if (PAIR) mbar_wait_cl(&pfull[st], ph); }
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t aa = su32(sA + st * aB), bb = su32(sB + st * bB);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (PAIR) {
                    mma2(tbase, desc(aa + k * 32), desc(bb + k * 32), i0, (it | k) ? 1u : 0u);
                    if (p.N1) mma2(tbase + p.N0, desc(aa + k * 32), desc(bb + b1 + k * 32), i1, (it | k) ? 1u : 0u);
                } else {
                    mma1(tbase, desc(aa + k * 32), desc(bb + k * 32), i0, (it | k) ? 1u : 0u);
                    if (p.N1) mma1(tbase + p.N0, desc(aa + k * 32), desc(bb + b1 + k * 32), i1, (it | k) ? 1u : 0u);
                }
            }
            if (PAIR) commit2(&empty[st]); else commit1(&empty[st]);
            if (p.sync_each) mbar_wait(&empty[st], ph);
        }
        if (PAIR) commit2(done); else commit1(done);
    }
    if (tid == 64) mbar_wait(done, 0);
    if (PAIR) csync(); else __syncthreads();
    long long t1 = clock64();
    if (tid == 64) p.cyc[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) {
        if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tbase));
        else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
    }
}

int main() {
    int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    uint8_t *gA, *gB; long long* cyc;
    CK(cudaMalloc(&gA, 64 << 14)); CK(cudaMalloc(&gB, 64 * 320 * 128));
    CK(cudaMemset(gA, 0, 64 << 14)); CK(cudaMemset(gB, 0, 64 * 320 * 128));
    CK(cudaMalloc(&cyc, 1024 * sizeof(long long)));
    CK(cudaFuncSetAttribute(probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
    CK(cudaFuncSetAttribute(probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
    struct Case { const char* name; int pair, N0, N1, fillA, fillB, stages, sync_each = 0; };
    const Case cases[] = {
        {"M128 N256", 0, 256, 0, 0, 0, 3},
        {"M128 N128", 0, 128, 0, 0, 0, 3},
        {"M128 N160+144", 0, 160, 144, 0, 0, 3},
        {"M128 N256+48", 0, 256, 48, 0, 0, 3},
        {"M256pair N160+144", 1, 160, 144, 0, 0, 3},
        {"M256pair N256+48", 1, 256, 48, 0, 0, 3},
        {"M256pair N256", 1, 256, 0, 0, 0, 3},
        {"M128 N160+144 fillB", 0, 160, 144, 0, 1, 3},
        {"M128 N160+144 fillA+B", 0, 160, 144, 1, 1, 3},
        {"M128 N160+144 fillA+B s4", 0, 160, 144, 1, 1, 4},
        {"M256pair N160+144 fillA+B s4", 1, 160, 144, 1, 1, 4},
        {"M256pair N160+144 fillA+B s6", 1, 160, 144, 1, 1, 6},
        {"M128 N64 commit+wait per K-block", 0, 64, 0, 0, 0, 3, 1},
        {"M128 N160+144 commit+wait per K-blk", 0, 160, 144, 0, 0, 3, 1},
    };
    cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    for (const Case& c : cases) {
        P p{}; p.pair = c.pair; p.N0 = c.N0; p.N1 = c.N1; p.iters = 4000; p.stages = c.stages;
        p.fillA = c.fillA; p.fillB = c.fillB; p.gA = gA; p.gB = gB; p.cyc = cyc; p.sync_each = c.sync_each;
        const int Brows = c.pair ? (c.N0 + c.N1) / 2 : c.N0 + c.N1;
        const size_t smem = 1024 + (size_t)c.stages * (16384 + Brows * 128) + 512;
        cudaLaunchConfig_t cfg{}; cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = c.pair ? 2 : 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(c.pair ? (sms / 2) * 2 : sms); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem; cfg.attrs = at; cfg.numAttrs = 1;
        float best = 1e30f;
        for (int r = 0; r < 3; ++r) {
            CK(cudaEventRecord(e0));
            if (c.pair) CK(cudaLaunchKernelEx(&cfg, probe<true>, p)); else CK(cudaLaunchKernelEx(&cfg, probe<false>, p));
            CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
            float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
        }
        long long hc[1024]; CK(cudaMemcpy(hc, cyc, cfg.gridDim.x * sizeof(long long), cudaMemcpyDeviceToHost));
        double mc = 0; for (unsigned i = 0; i < cfg.gridDim.x; ++i) mc += hc[i]; mc /= cfg.gridDim.x;
        const int M = c.pair ? 256 : 128;
        const double flop_per_cta = 2.0 * M * (c.N0 + c.N1) * 32.0 * p.iters / (c.pair ? 2 : 1);
        const double tf = flop_per_cta * cfg.gridDim.x / (best * 1e-3) / 1e12;
        printf("%-36s %8.3f ms  %7.1f TFLOP/s  %7.0f flop/clk/SM  (%.2f GHz eff)  %.0f clk/K-block\n", c.name, best, tf,
               flop_per_cta / mc, mc / (best * 1e-3) / 1e9, mc / p.iters);
    }
    return 0;
}
