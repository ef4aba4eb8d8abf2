// ldgsts_probe.cu -- shared-memory fill rate per SM of the gather patterns the
// tcgen05 conv uses (tuning aid, not product): 16-byte cp.async (LDGSTS) by 4
// producer warps into 16 KB stages, completion tracked per stage with
// cp.async.mbarrier.arrive.noinc (as conv_tc.cu), against one TMA bulk copy
// per stage. Sources are L2-resident.
//   pattern 0: 8 lanes per row, a row = 128 contiguous bytes (layer 3 style)
//   pattern 1: lane per row, 16 bytes per lane, rows 16 bytes apart (layer 2
//              style, x-consecutive pixels)
//   pattern 2: one cp.async.bulk of 16 KB per stage
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ldgsts_probe scripts/probes/ldgsts_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n\t.reg .pred P;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}" ::"r"(
                     su32(b)),
                 "r"(ph));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}

template <int PAT>
__global__ void __launch_bounds__(160, 1) probe(const uint8_t* src, int iters, long long* cyc, int span) {
    extern __shared__ __align__(1024) uint8_t sm[];
    constexpr int NS = 4, SB = 16384;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + NS * SB);
    uint64_t* empty = full + NS;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], PAT == 2 ? 1 : 128);
            mbar_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long t0 = clock64();
    // span 4: each CTA cycles through its own 64 KB (L1-hot); larger spans walk
    // a shared L2-resident buffer (L1 misses)
    const uint8_t* base = span == 4 ? src + (size_t)blockIdx.x * 65536 : src;
    if (warp < 4) {
        for (int it = 0; it < iters; ++it) {
            const int st = it % NS;
            const uint32_t ph = (it / NS) & 1;
            mbar_wait(&empty[st], ph ^ 1);
            const uint8_t* s = base + (size_t)((it + (span == 4 ? 0 : blockIdx.x * 37)) % span) * SB;
            const uint32_t d = su32(sm + st * SB);
            if (PAT == 0) {  // thread = chunk j of rows rsub + 16 i
                const int j = tid & 7, rsub = tid >> 3;
                for (int i = 0; i < 8; ++i) {
                    const int r = rsub + 16 * i;
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(d + r * 128 + ((j ^ (r & 7)) << 4)),
                                 "l"(s + r * 128 + j * 16)
                                 : "memory");
                }
            } else if (PAT == 1) {  // thread = row r, 8 chunks 16 B apart in source rows 16 B apart
                const int r = tid;
                for (int j = 0; j < 8; ++j)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(d + r * 128 + ((j ^ (r & 7)) << 4)),
                                 "l"(s + (j * 128 + r) * 16 % SB)
                                 : "memory");
            } else {
                if (tid == 0) {
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[st])), "r"(SB)
                                 : "memory");
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
                        "l"(s), "r"(SB), "r"(su32(&full[st]))
                        : "memory");
                }
            }
            if (PAT != 2) asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[st])) : "memory");
        }
    } else if (tid == 128) {  // consumer: releases each stage once full
        for (int it = 0; it < iters; ++it) {
            const int st = it % NS;
            mbar_wait(&full[st], (it / NS) & 1);
            mbar_arrive(&empty[st]);
        }
        cyc[blockIdx.x] = clock64() - t0;
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint8_t* src;
    long long* cyc;
    const int big = 3072;  // 48 MB of 16 KB blocks: L2-resident, not L1
    cudaMalloc(&src, (size_t)big * 16384);
    cudaMemset(src, 1, (size_t)big * 16384);
    cudaMalloc(&cyc, sms * sizeof(long long));
    const int smem = 4 * 16384 + 1024;
    cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const char* names[3] = {"8 lanes/row, 128 B rows (L3)", "lane/row, 16 B chunks (L2)", "TMA bulk 16 KB"};
    for (int span : {4, big})
    for (int p = 0; p < 3; ++p) {
        const int iters = 20000;
        for (int rep = 0; rep < 2; ++rep) {
            if (p == 0) probe<0><<<sms, 160, smem>>>(src, iters, cyc, span);
            if (p == 1) probe<1><<<sms, 160, smem>>>(src, iters, cyc, span);
            if (p == 2) probe<2><<<sms, 160, smem>>>(src, iters, cyc, span);
            cudaDeviceSynchronize();
        }
        long long h[1024];
        cudaMemcpy(h, cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
        double m = 0;
        for (int i = 0; i < sms; ++i) m += h[i];
        m /= sms;
        printf("%-32s %s %6.1f B/clk/SM\n", names[p], span == 4 ? "L1-hot " : "L2     ", 16384.0 * iters / m);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
