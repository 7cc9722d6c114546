// HBM ceilings for the integral pass's access mixes (run on the GPU box):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/bw_probe tools/bw_probe.cu && gpurun_out/bw_probe
// read-only (the reduce), write-only, 1 read : 8 writes into eight planes (the tables
// write pass), and copy; grid = SMs x blocks-per-SM, grid-stride 16-byte accesses.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void read_sum(const float4* __restrict__ a, size_t n4, float* out) {
    float acc = 0.f;
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n4; q += (size_t)gridDim.x * blockDim.x) {
        const float4 v = __ldcs(a + q);
        acc += v.x + v.y + v.z + v.w;
    }
    if (acc == 1234.5f) out[0] = acc;
}

__global__ void write_only(float4* __restrict__ a, size_t n4) {
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n4; q += (size_t)gridDim.x * blockDim.x)
        __stcs(a + q, make_float4(1.f, 2.f, 3.f, (float)q));
}

__global__ void read1_write8(const float4* __restrict__ a, float4* __restrict__ t, size_t n4) {
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n4; q += (size_t)gridDim.x * blockDim.x) {
        const float4 v = __ldcs(a + q);
#pragma unroll
        for (int p = 0; p < 8; ++p)
            __stcs(t + (size_t)p * n4 + q, make_float4(v.x + p, v.y, v.z, v.w));
    }
}

__global__ void copy_k(const float4* __restrict__ a, float4* __restrict__ b, size_t n4) {
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n4; q += (size_t)gridDim.x * blockDim.x)
        __stcs(b + q, __ldcs(a + q));
}


// TMA bulk stores (cp.async.bulk.global.shared::cta): each CTA streams CH-byte chunks
// of a shared-memory buffer to grid-strided destinations, up to 4 bulk groups in flight.
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
                 "r"((unsigned)__cvta_generic_to_shared(ssrc)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

constexpr unsigned CH = 8192;
__global__ void write_bulk(char* __restrict__ t, size_t bytes) {
    __shared__ __align__(128) float buf[CH / 4];
    for (int q = threadIdx.x; q < CH / 4; q += blockDim.x) buf[q] = (float)q;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        for (size_t off = (size_t)blockIdx.x * CH; off < bytes; off += (size_t)gridDim.x * CH) {
            bulk_store(t + off, buf, CH);
            bulk_commit();
        }
        bulk_wait_all();
    }
}

// read one plane with 16-byte loads, stage 8 output planes in shared memory, bulk-store
// each plane's chunk (the tables write pass's traffic mix through TMA stores)
__global__ void read1_write8_bulk(const float4* __restrict__ a, char* __restrict__ t, size_t n4) {
    constexpr int C4 = 512;  // float4 per chunk per plane (8 KB)
    extern __shared__ __align__(128) float4 dsm[];  // [2][8][C4]: 128 KB double buffer
    auto buf = reinterpret_cast<float4 (*)[8][C4]>(dsm);
    int slot = 0;
    for (size_t c0 = (size_t)blockIdx.x * C4; c0 < n4; c0 += (size_t)gridDim.x * C4, slot ^= 1) {
        if (threadIdx.x == 0) bulk_wait_read<1>();
        __syncthreads();
        for (int q = threadIdx.x; q < C4; q += blockDim.x) {
            const float4 v = __ldcs(a + c0 + q);
#pragma unroll
            for (int p = 0; p < 8; ++p) buf[slot][p][q] = make_float4(v.x + p, v.y, v.z, v.w);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
#pragma unroll
            for (int p = 0; p < 8; ++p) bulk_store(t + ((size_t)p * n4 + c0) * 16, buf[slot][p], C4 * 16);
            bulk_commit();
        }
    }
    if (threadIdx.x == 0) bulk_wait_all();
}

template <typename F>
static float best_ms(F f, int reps = 10) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        f();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t px = (size_t)16384 * 16384;  // one 16384^2 fp32 plane = 1 GiB
    const size_t n4 = px / 4;
    float4 *a, *t;
    float* out;
    cudaMalloc(&a, px * 4);
    cudaMalloc(&t, px * 4 * 8);
    cudaMalloc(&out, 4);
    cudaMemset(a, 0, px * 4);
    cudaMemset(t, 0, px * 32);
    for (int bps : {4, 8, 16}) {
        const dim3 g(sms * bps), b(256);
        const float r = best_ms([&] { read_sum<<<g, b>>>(a, n4, out); });
        const float w = best_ms([&] { write_only<<<g, b>>>(t, n4 * 8); });
        const float m = best_ms([&] { read1_write8<<<g, b>>>(a, t, n4); });
        const float c = best_ms([&] { copy_k<<<g, b>>>(a, t, n4); });
        printf("blocks/SM %2d: read %.0f GB/s  write %.0f GB/s  read1:write8 %.0f GB/s  copy %.0f GB/s\n", bps,
               px * 4 / r / 1e6, px * 32 / w / 1e6, px * 36 / m / 1e6, px * 8 / c / 1e6);
    }

    for (int bps : {1, 2, 4, 8}) {
        const dim3 g(sms * bps), b(256);
        const float w = best_ms([&] { write_bulk<<<g, b>>>((char*)t, px * 32); });
        cudaFuncSetAttribute(read1_write8_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
        const float m = best_ms([&] { read1_write8_bulk<<<dim3(sms), dim3(128 * bps), 131072>>>(a, (char*)t, n4); });
        printf("bulk, blocks/SM %d: write %.0f GB/s  read1:write8 (1 CTA/SM, 128*bps thr) %.0f GB/s\n", bps, px * 32 / w / 1e6,
               px * 36 / m / 1e6);
    }
    const float ms = best_ms([&] { cudaMemsetAsync(t, 0, px * 32); });
    printf("cudaMemset 8 GiB: %.0f GB/s\n", px * 32 / ms / 1e6);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
