// common.cuh -- shared device/host definitions of the cbx engine.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

namespace cbx {

constexpr int kNumSMs = 148;  // B200

// Activation tensor on the device. All intermediate activations are
// channels-last (HWC) with the channel stride padded to a multiple of 4
// floats (one 16-byte chunk) and a zero halo of `hh`/`hw` pixels so that the
// consumer's zero padding is free. Layout per stream: [Hp][Wp][Cp]; streams
// are `ss` floats apart. The network input (the camera frame) is the only
// planar (CHW) tensor; it is addressed through a per-stream pointer table.
struct TensorView {
    float* d;
    int C, H, W;     // logical
    int Cp, Hp, Wp;  // padded
    int hh, hw;      // halo
    int64_t ss;      // floats per stream
};

// The layer-1 input of the 8-bit camera path: RGBX pixels (4 bytes, channel
// 3 zero) in rows of Wp pixels with a zero halo of hh rows / hw pixels (hw a
// multiple of 4 so every row's interior starts 16-byte aligned); streams ss
// pixels apart. The tcgen05 conv reads it as a TensorView with Cp = 1
// (one 4-byte unit per pixel).
struct Rgbx8View {
    uint32_t* d;
    int64_t ss;
    int Wp, hh, hw;
};

// Byte mask on a pixel grid: [S][stride], pixel p = y*W + x.
struct MaskView {
    uint8_t* d;
    int H, W;
    int64_t stride;
};

// Packed bit mask on a pixel grid (the engine's change / updated-pixel masks):
// [S][stride] 32-bit words, row y occupies words [y*wpr, (y+1)*wpr), pixel x
// is bit (x & 31) of word x >> 5; bits past W are always zero. stride is a
// multiple of 2048 words so compaction tiles never straddle two streams.
struct BitMask {
    uint32_t* d;
    int H, W, wpr;
    int64_t stride;
};

__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

// Programmatic dependent launch (the frame's kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, see launch_k): every
// kernel lets its successor start launching at once (pdl_trigger) and waits
// for its predecessor's grid to complete -- memory included -- before it
// touches anything the predecessor produced (pdl_wait). The successor's
// CTAs are then scheduled onto the SMs the predecessor's last wave frees,
// and can run their prologue there, instead of starting after the drain.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_entry() {
    pdl_trigger();
    pdl_wait();
}

// Launch with the programmatic-stream-serialization attribute when
// CBX_PDL=1 (opt-in, see pdl_enabled in engine.cu); plain stream order else.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Division by a runtime-constant divisor as a multiply-high and a shift, for
// numerators below 2^31 (the per-pixel index arithmetic of the hot kernels:
// a 64-bit division is a ~100-instruction subroutine call per pixel):
// m = ceil(2^(31 + l) / d), l = ceil(log2 d), q = umulhi(n, m) >> (l - 1).
struct FastDiv {
    uint32_t d = 1, m = 0, sh = 0;
    static FastDiv make(uint32_t d) {
        FastDiv f;
        f.d = d;
        if (d > 1) {
            int l = 0;
            while ((1ull << l) < d) ++l;
            f.m = (uint32_t)(((1ull << (31 + l)) + d - 1) / d);
            f.sh = (uint32_t)(l - 1);
        }
        return f;
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const { return d == 1 ? n : (__umulhi(n, m) >> sh); }
};

__device__ __forceinline__ bool bit_test(const BitMask& m, int s, int y, int x) {
    return (m.d[(int64_t)s * m.stride + (int64_t)y * m.wpr + (x >> 5)] >> (x & 31)) & 1u;
}
__device__ __forceinline__ void bit_set(const BitMask& m, int s, int y, int x) {
    atomicOr(m.d + (int64_t)s * m.stride + (int64_t)y * m.wpr + (x >> 5), 1u << (x & 31));
}

// Reference ReLU: std::max(0.0f, v) == (0.0f < v) ? v : 0.0f (baseline.cpp:115).
__device__ __forceinline__ float ref_relu(float v) { return (0.0f < v) ? v : 0.0f; }
// Reference max: std::max(m, v) == (m < v) ? v : m (baseline.cpp:138).
__device__ __forceinline__ float ref_max(float m, float v) { return (m < v) ? v : m; }
// Reference change test (cbconv.cpp:66-67): strict on both signs.
__device__ __forceinline__ bool ref_changed(float now, float before, float tau) {
    const float d = __fsub_rn(now, before);
    return d > tau || -d > tau;
}

// Two fp32 lanes per instruction (FFMA2), each IEEE round-to-nearest. The
// reference's separately rounded multiply and add are f2_fma(w, x, -0) and
// f2_fma(p, 1, acc) with 1 and -0 passed as RUNTIME values: with literal
// constants ptxas contracts the pair into one fused multiply-add.
__device__ __forceinline__ unsigned long long f2_pack(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void f2_unpack(unsigned long long v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ unsigned long long f2_fma(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// Adds `flag` into counters[s*stride] with one atomic per (warp, stream).
__device__ __forceinline__ void warp_count_add(unsigned long long* counters, int stride, int s,
                                               bool flag, bool active) {
    const unsigned act = __ballot_sync(0xffffffffu, active);
    if (!active) return;
    const unsigned same = __match_any_sync(act, s);
    const unsigned hits = __ballot_sync(act, flag) & same;
    const int leader = __ffs(same) - 1;
    if ((int)(threadIdx.x & 31) == leader && hits)
        atomicAdd(counters + (int64_t)s * stride, (unsigned long long)__popc(hits));
}

}  // namespace cbx
