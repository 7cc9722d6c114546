// L2 reduction throughput probe on sm_100a: requests per second of scalar u32 REDs,
// 64-bit REDs and 16-byte f32x4 REDs to pseudo-random addresses of a count grid
// (1024^2 and 4096^2 words), in order to size the splat's atomic cost.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/red_probe_bin tools/red_probe.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t hash(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16;
    return x;
}

template <int MODE>
__global__ void red_kernel(void* buf, uint32_t mask, int per_thread) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int i = 0; i < per_thread; ++i) {
        const uint32_t h = hash(t * 131u + i * 7919u) & mask;  // word index
        if (MODE == 0) atomicAdd(reinterpret_cast<uint32_t*>(buf) + h, 1u);
        else if (MODE == 1) {
            unsigned long long* q = reinterpret_cast<unsigned long long*>(buf) + (h >> 1);
            asm volatile("red.global.add.u64 [%0], %1;" ::"l"(q), "l"(1ull) : "memory");
        } else {
            float* q = reinterpret_cast<float*>(buf) + (h & ~3u);
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(q), "f"(1.f), "f"(0.f), "f"(1.f), "f"(0.f)
                         : "memory");
        }
    }
}

int main() {
    void* buf;
    cudaMalloc(&buf, sizeof(uint32_t) << 24);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int blocks = 148 * 8, threads = 256, per = 64;
    const double reqs = (double)blocks * threads * per;
    const char* names[] = {"u32 RED", "u64 RED", "f32x4 RED"};
    for (int k : {20, 24}) {
        const uint32_t mask = (1u << k) - 1;
        for (int mode = 0; mode < 3; ++mode) {
            for (int rep = 0; rep < 3; ++rep) {
                cudaMemset(buf, 0, sizeof(uint32_t) << k);
                cudaEventRecord(a);
                if (mode == 0) red_kernel<0><<<blocks, threads>>>(buf, mask, per);
                if (mode == 1) red_kernel<1><<<blocks, threads>>>(buf, mask, per);
                if (mode == 2) red_kernel<2><<<blocks, threads>>>(buf, mask, per);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (rep == 2) printf("grid 2^%d words  %-10s %8.1f G requests/s\n", k, names[mode], reqs / ms / 1e6);
            }
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
