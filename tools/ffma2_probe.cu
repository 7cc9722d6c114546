// FP32 FMA issue-rate probe on sm_100a: FFMA with an immediate multiplier, FFMA with a
// register multiplier, and the packed FFMA2 (fma.rn.f32x2) with a register pair and
// with a constant-bank pair.  Reports FMAs per cycle per SM (clock64 inside the kernel).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffma2_probe tools/ffma2_probe.cu && /tmp/ffma2_probe
#include <cstdio>
#include <cstdint>

__constant__ unsigned long long ctap[64];

__device__ __forceinline__ unsigned long long f2(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}

template <int MODE>
__global__ void probe(float* out, long long* cycles, int iters, float w) {
    float acc[16];
    unsigned long long acc2[8];
#pragma unroll
    for (int q = 0; q < 16; ++q) acc[q] = threadIdx.x * 1e-3f + q;
#pragma unroll
    for (int q = 0; q < 8; ++q) acc2[q] = f2(acc[2 * q], acc[2 * q + 1]);
    const unsigned long long w2 = f2(w, w);
    const unsigned long long x2 = f2(1.0001f, 0.9999f);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (MODE == 0) {  // FFMA, immediate multiplier
#pragma unroll
                for (int q = 0; q < 16; ++q) acc[q] = fmaf(acc[q], 0.999f, 1e-7f);
            } else if (MODE == 1) {  // FFMA, register multiplier
#pragma unroll
                for (int q = 0; q < 16; ++q) acc[q] = fmaf(acc[q], w, 1e-7f);
            } else if (MODE == 2) {  // FFMA2, register pairs
#pragma unroll
                for (int q = 0; q < 8; ++q) asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc2[q]) : "l"(w2), "l"(x2));
            } else {  // FFMA2, constant-bank pair
#pragma unroll
                for (int q = 0; q < 8; ++q) asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc2[q]) : "l"(ctap[q & 3]), "l"(x2));
            }
        }
    }
    long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < 16; ++q) s += acc[q];
#pragma unroll
    for (int q = 0; q < 8; ++q) s += __uint_as_float((unsigned)acc2[q]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

int main() {
    const int blocks = 148, threads = 512, iters = 4096;
    float* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(float) * blocks * threads);
    cudaMalloc(&cyc, sizeof(long long) * blocks);
    unsigned long long h[64];
    for (int i = 0; i < 64; ++i) {
        float a = 0.999f;
        unsigned ua = *reinterpret_cast<unsigned*>(&a);
        h[i] = ((unsigned long long)ua << 32) | ua;
    }
    cudaMemcpyToSymbol(ctap, h, sizeof(h));
    const char* names[] = {"FFMA imm", "FFMA reg", "FFMA2 reg pair", "FFMA2 const pair"};
    for (int mode = 0; mode < 4; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            if (mode == 0) probe<0><<<blocks, threads>>>(out, cyc, iters, 0.999f);
            if (mode == 1) probe<1><<<blocks, threads>>>(out, cyc, iters, 0.999f);
            if (mode == 2) probe<2><<<blocks, threads>>>(out, cyc, iters, 0.999f);
            if (mode == 3) probe<3><<<blocks, threads>>>(out, cyc, iters, 0.999f);
        }
        cudaDeviceSynchronize();
        long long c;
        cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
        const double fmas = (double)threads * iters * 8 * 16;  // per SM (one block per SM)
        printf("%-18s %8.1f FMA/cycle/SM  (%lld cycles)\n", names[mode], fmas / c, c);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
