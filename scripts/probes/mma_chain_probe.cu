// mma_chain_probe.cu -- is the per-instruction tcgen05.mma cost at small N a
// dependency latency (every MMA accumulates into the same D) or a throughput
// limit? One CTA per SM, one thread issues K-blocks of 4 instructions from a
// resident stage; consecutive instructions rotate over CH independent
// accumulators (TMEM columns c*N). Tuning aid, not product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_chain_probe scripts/probes/mma_chain_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr) {
    return (uint64_t)((addr & 0x3FFFFu) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc_f16(int N, int M) {
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__host__ __device__ constexpr uint32_t idesc_tf32(int N, int M) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}

__global__ void probe(int tf32, int N, int N2, int CH, int iters, unsigned long long* clk) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* s = sm + ((1024u - (su32(sm) & 1023u)) & 1023u);
    uint8_t* sA = s;             // 128 rows x 128 B
    uint8_t* sB = s + 16384;     // 256 rows x 128 B
    __shared__ uint64_t bar;
    __shared__ uint32_t tm;
    for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tm)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t d = tm;
    if (threadIdx.x == 0) {
        const uint64_t ad = desc(su32(sA)), bd = desc(su32(sB));
        const uint32_t id = tf32 ? idesc_tf32(N, 128) : idesc_f16(N, 128);
        const uint32_t id2 = N2 ? (tf32 ? idesc_tf32(N2, 128) : idesc_f16(N2, 128)) : 0;
        unsigned long long t0 = clock64();
        uint32_t ph = 0;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (N2) {  // L3-like: two instructions per k-step into two regions
                    if (tf32) { mma_tf32(d, ad + 2 * k, bd + 2 * k, id, 1u); mma_tf32(d + 256, ad + 2 * k, bd + 2 * k, id2, 1u); }
                    else { mma_f16(d, ad + 2 * k, bd + 2 * k, id, 1u); mma_f16(d + 256, ad + 2 * k, bd + 2 * k, id2, 1u); }
                } else {
                    const uint32_t dd = d + (uint32_t)(((it * 4 + k) % CH) * N);
                    if (tf32) mma_tf32(dd, ad + 2 * k, bd + 2 * k, id, 1u); else mma_f16(dd, ad + 2 * k, bd + 2 * k, id, 1u);
                }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
            if ((it & 7) == 7 || it == iters - 1) {
                asm volatile("{\n\t.reg .pred P;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}" ::"r"(su32(&bar)), "r"(ph));
            }
            ph ^= 1u;
        }
        unsigned long long t1 = clock64();
        clk[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(d));
}


template <int TF32, int CH, int ACC0>
__global__ void probe2(int N, int iters, unsigned long long* clk) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* s = sm + ((1024u - (su32(sm) & 1023u)) & 1023u);
    uint8_t* sA = s;
    uint8_t* sB = s + 16384;
    __shared__ uint64_t bar;
    __shared__ uint32_t tm;
    for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tm)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t d = tm;
    if (threadIdx.x == 0) {
        const uint64_t ad = desc(su32(sA)), bd = desc(su32(sB));
        const uint32_t id = TF32 ? idesc_tf32(N, 128) : idesc_f16(N, 128);
        unsigned long long t0 = clock64();
        uint32_t ph = 0;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t dd = d + (uint32_t)((k % CH) * N);
                const uint32_t acc = ACC0 ? ((it | k) ? 1u : 0u) : 1u;
                if (TF32) mma_tf32(dd, ad + 2 * k, bd + 2 * k, id, acc); else mma_f16(dd, ad + 2 * k, bd + 2 * k, id, acc);
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
            if ((it & 7) == 7 || it == iters - 1) {
                asm volatile("{\n\t.reg .pred P;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}" ::"r"(su32(&bar)), "r"(ph));
            }
            ph ^= 1u;
        }
        unsigned long long t1 = clock64();
        clk[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(d));
}

template <int TF32, int CH, int ACC0>
int run2(int N, unsigned long long* clk) {
    const int iters = 4096, smem = 16384 + 32768 + 1024;
    CK(cudaFuncSetAttribute(probe2<TF32, CH, ACC0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    for (int rep = 0; rep < 2; ++rep) {
        probe2<TF32, CH, ACC0><<<148, 128, smem>>>(N, iters, clk);
        CK(cudaDeviceSynchronize());
    }
    unsigned long long h[148];
    CK(cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost));
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("probe2 %-5s N%-4d chains %d acc0 %d : %7.1f clk/instr\n", TF32 ? "tf32" : "f16", N, CH, ACC0, mx / (iters * 4.0));
    return 0;
}

// stages: NS distinct (A 16 KB, B 32 KB) buffers rotated per K-block (fresh operands every K-block)
template <int TF32, int NS, int RND>
__global__ void probe3(int N, int iters, unsigned long long* clk) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* s = sm + ((1024u - (su32(sm) & 1023u)) & 1023u);
    __shared__ uint64_t bar;
    __shared__ uint32_t tm;
    for (int i = threadIdx.x; i < NS * (16384 + 32768) / 4; i += blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u + 12345u * RND;
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        // RND: random fp32/fp16 values of moderate magnitude (exponent forced into [-4, 3])
        reinterpret_cast<uint32_t*>(s)[i] = RND ? ((h & 0x807fffffu) | ((123u + (h >> 28)) << 23)) : 0u;
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tm)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t d = tm;
    if (threadIdx.x == 0) {
        const uint32_t id = TF32 ? idesc_tf32(N, 128) : idesc_f16(N, 128);
        unsigned long long t0 = clock64();
        uint32_t ph = 0;
        for (int it = 0; it < iters; ++it) {
            const int st = it % NS;
            const uint64_t ad = desc(su32(s + st * 49152)), bd = desc(su32(s + st * 49152 + 16384));
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (TF32) mma_tf32(d, ad + 2 * k, bd + 2 * k, id, 1u); else mma_f16(d, ad + 2 * k, bd + 2 * k, id, 1u);
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
            if ((it & 7) == 7 || it == iters - 1) {
                asm volatile("{\n\t.reg .pred P;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}" ::"r"(su32(&bar)), "r"(ph));
            }
            ph ^= 1u;
        }
        unsigned long long t1 = clock64();
        clk[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(d));
}

template <int TF32, int NS, int RND>
int run3(int N, unsigned long long* clk) {
    const int iters = 4096, smem = NS * 49152 + 1024;
    CK(cudaFuncSetAttribute(probe3<TF32, NS, RND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    for (int rep = 0; rep < 2; ++rep) {
        probe3<TF32, NS, RND><<<148, 128, smem>>>(N, iters, clk);
        CK(cudaDeviceSynchronize());
    }
    unsigned long long h[148];
    CK(cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost));
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("probe3 %-5s N%-4d stages %d random %d : %7.1f clk/instr\n", TF32 ? "tf32" : "f16", N, NS, RND, mx / (iters * 4.0));
    return 0;
}

int main(int argc, char**) {
    unsigned long long* clk;
    CK(cudaMalloc(&clk, 148 * sizeof(unsigned long long)));
    const int iters = 4096;
    const int smem = 16384 + 32768 + 1024;
    CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    struct C { int tf32, N, N2, CH; };
    const C cs[] = {{1, 64, 0, 1}, {1, 64, 0, 2}, {1, 64, 0, 4}, {1, 64, 0, 8}, {0, 64, 0, 1}, {0, 64, 0, 4},
                    {0, 128, 0, 1}, {0, 128, 0, 2}, {0, 128, 0, 4}, {0, 256, 0, 1}, {0, 256, 0, 2},
                    {0, 160, 144, 1}, {0, 128, 176, 1}, {0, 256, 48, 1}, {0, 192, 112, 1}};
    if (argc > 1) {  // f16 cost per N (rotating stages), then exit
        for (int N = 16; N <= 256; N += 16) run3<0, 3, 1>(N, clk);
        for (int N = 16; N <= 256; N += 16) run2<0, 1, 1>(N, clk);
        return 0;
    }
    run3<1, 3, 0>(64, clk); run3<1, 3, 1>(64, clk); run3<0, 3, 0>(256, clk); run3<0, 3, 1>(256, clk); run3<0, 3, 1>(160, clk); run3<0, 3, 1>(128, clk);
    run2<1, 1, 1>(64, clk); run2<1, 1, 0>(64, clk); run2<1, 2, 1>(64, clk); run2<1, 4, 1>(64, clk);
    run2<0, 1, 1>(128, clk); run2<0, 2, 1>(128, clk); run2<0, 1, 1>(256, clk); run2<0, 2, 1>(256, clk);
    for (const C& c : cs) {
        for (int rep = 0; rep < 2; ++rep) {
            probe<<<148, 128, smem>>>(c.tf32, c.N, c.N2, c.CH, iters, clk);
            CK(cudaDeviceSynchronize());
        }
        unsigned long long h[148];
        CK(cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost));
        double mx = 0;
        for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("%-5s M128 N%-4d N2 %-4d chains %d : %7.1f clk per k-step (32 K-bytes)\n", c.tf32 ? "tf32" : "f16", c.N, c.N2, c.CH,
               mx / (iters * 4.0));
    }
    return 0;
}
