// mma_shape_probe.cu -- tcgen05.mma issue cost per instruction by kind and
// shape (tuning aid, not product). One CTA per SM, one elected thread issues
// ITERS 128-byte K-blocks (4 instructions of 32 K-bytes each) from one
// resident shared-memory stage, committing every K-block; reports clk per
// instruction. Answers: does the cost depend on N (<= 256) and on M (64/128)?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_shape_probe scripts/mma_shape_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr) {
    return (uint64_t)((addr & 0x3FFFFu) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
// kind: 0 f16, 1 tf32, 2 i8
__host__ __device__ constexpr uint32_t idesc(int kind, int N, int M) {
    return kind == 2 ? ((2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24))
         : kind == 1 ? ((1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24))
                     : ((1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24));
}
template <int KIND>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    if (KIND == 2)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
    else if (KIND == 1)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
    else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}

template <int KIND>
__global__ void probe(int M, int N, int iters, unsigned long long* clk) {
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
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tm)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t d = tm;
    if (threadIdx.x == 0) {
        const uint64_t ad = desc(su32(sA)), bd = desc(su32(sB));
        const uint32_t id = idesc(KIND, N, M);
        unsigned long long t0 = clock64();
        uint32_t ph = 0;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 4; ++k) mma<KIND>(d, ad + 2 * k, bd + 2 * k, id, (it | k) ? 1u : 0u);
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
            if ((it & 7) == 7 || it == iters - 1) {  // keep <= 8 K-blocks in flight
                asm volatile("{\n\t.reg .pred P;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}" ::"r"(su32(&bar)), "r"(ph));
            }
            ph ^= 1u;
        }
        unsigned long long t1 = clock64();
        clk[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(d));
}

int main() {
    unsigned long long* clk;
    CK(cudaMalloc(&clk, 148 * sizeof(unsigned long long)));
    const int iters = 4096;
    const int smem = 16384 + 32768 + 1024;
    CK(cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const char* kinds[] = {"f16", "tf32", "i8"};
    for (int kind = 0; kind < 3; ++kind)
        for (int M : {64, 128})
            for (int N : {16, 32, 64, 128, 256}) {
                for (int rep = 0; rep < 2; ++rep) {
                    if (kind == 0) probe<0><<<148, 128, smem>>>(M, N, iters, clk);
                    if (kind == 1) probe<1><<<148, 128, smem>>>(M, N, iters, clk);
                    if (kind == 2) probe<2><<<148, 128, smem>>>(M, N, iters, clk);
                    CK(cudaDeviceSynchronize());
                }
                unsigned long long h[148];
                CK(cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost));
                double mx = 0;
                for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
                printf("%-5s M%-4d N%-4d  %7.1f clk/instr (32 K-bytes)\n", kinds[kind], M, N, mx / (iters * 4.0));
            }
    return 0;
}
