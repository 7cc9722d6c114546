// Shared device helpers for the sm_100a integral-image regularizer.
//
// Coordinate convention (reference model.py:1-8): grids are 2^k x 2^k, row-major,
// values[j * s + i] with i = x (column), j = y (row); fields are (s, s, 2), x then y.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "../../include/inim.h"

#define INIM_DEV __device__ __forceinline__

namespace inim {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;

// ------------------------------------------------------------------ warp primitives
// three-input maximum (one FMNMX3 on sm_100a); NaN handling as fmaxf
INIM_DEV float fmax3f(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

INIM_DEV float warp_inclusive_scan(float v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        float n = __shfl_up_sync(kFull, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

INIM_DEV double warp_inclusive_scan_d(double v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        double n = __shfl_up_sync(kFull, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

INIM_DEV float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

INIM_DEV float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
    return v;
}

// Half-sample symmetric reflection with period 2n (scipy.ndimage mode="reflect";
// reference density.py:49-50, restated in tests/oracles.py:95-102).  n is a power of
// two (every grid side is 2^k), so the residue mod 2n is a mask, negative idx included.
INIM_DEV int reflect_index(int idx, int n) {
    idx &= 2 * n - 1;
    return idx >= n ? 2 * n - 1 - idx : idx;
}

// Non-negative float max through integer atomics (bit patterns of non-negative IEEE
// floats order like unsigned ints).
INIM_DEV void atomic_max_nonneg(float* addr, float v) {
    atomicMax(reinterpret_cast<unsigned int*>(addr), __float_as_uint(fmaxf(v, 0.0f)));
}

// ------------------------------------------------------------------ mbarrier + TMA (PTX)
INIM_DEV uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

INIM_DEV void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

INIM_DEV void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

INIM_DEV void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

INIM_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

INIM_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 2-D TMA tile load global -> shared, completion signalled on an mbarrier.
INIM_DEV void tma_load_2d(void* smem_dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

// 16-byte asynchronous global -> shared copy through L2 (cp.async.cg) and its wait.
INIM_DEV void cp_async16(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}

INIM_DEV void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;" ::: "memory");
}

INIM_DEV void prefetch_tensormap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// Streaming (evict-first) 32-bit global store: the eight tables are written once and
// never re-read by the producing kernel.
INIM_DEV void st_stream(float* p, float v) {
    asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

INIM_DEV void st_stream2(float2* p, float2 v) {
    asm volatile("st.global.cs.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}


#define INIM_CUDA_TRY(expr)                                       \
    do {                                                          \
        cudaError_t _e = (expr);                                  \
        if (_e != cudaSuccess) return static_cast<int>(_e);       \
    } while (0)

// ---------------------------------------------------- programmatic dependent launch
// Kernels of the iteration chain are launched with programmatic stream serialisation:
// a kernel's CTAs may be scheduled while its predecessor drains, and every kernel first
// waits (griddepcontrol.wait: the predecessor grid has completed and its writes are
// visible) and then lets its own successor start launching.  The wait is the kernel's
// first statement, before any early exit, so completion stays transitive along the
// chain.  Without the launch attribute both instructions are no-ops.
INIM_DEV void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef INIM_PDL_EARLY_TRIGGER
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

bool pdl_enabled();  // abi.cu: INIM_PDL=0 disables

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace inim
