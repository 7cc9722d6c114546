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
    const float ms = best_ms([&] { cudaMemsetAsync(t, 0, px * 32); });
    printf("cudaMemset 8 GiB: %.0f GB/s\n", px * 32 / ms / 1e6);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
