// Density smoothing kernels: gaussian_smooth + background (reference density.py:30-78).
//
// Two passes, horizontal then vertical, exactly the reference order (density.py:49-50),
// each a 6*ks+1-tap FIR with half-sample-symmetric reflection at the borders
// (scipy.ndimage mode="reflect", period 2s).  The tile bodies live in inim_smooth.cuh
// (shared with the persistent iteration kernel); these are the standalone launches.
#include <type_traits>

#include "inim_smooth.cuh"

namespace inim {

template <int R, typename T>
__global__ void __launch_bounds__(256, std::is_same<T, float>::value ? 1 : 4) smooth_h_kernel(const T* __restrict__ in, float* __restrict__ out, int s,
                                                       const HGeo h, const Taps taps, const int* state,
                                                       uint32_t* __restrict__ zero_next, uint32_t* ctr, int nctr) {
    pdl_enter();
    if (state && state[0]) return;
    if (ctr && blockIdx.x == 0 && blockIdx.y == 0)
        for (int q = threadIdx.x; q < nctr; q += blockDim.x) ctr[q] = 0u;  // band counters of the reduce
    extern __shared__ __align__(16) float hsm[];
    smooth_h_tile<R, T>(in, out, s, h, taps, zero_next, blockIdx.x, blockIdx.y, hsm);
}

template <int R>
__global__ void __launch_bounds__(512) smooth_v_kernel(const float* __restrict__ tmp, float* __restrict__ d,
                                                       const Geo g, const VGeo v, const Ws ws, const Taps taps,
                                                       float background, int emit, const int* state) {
    pdl_enter();
    if (state && state[0]) return;
    extern __shared__ __align__(16) float vsm[];
    smooth_v_tile<R>(tmp, d, g, v, ws, taps, background, emit, blockIdx.x, blockIdx.y, vsm);
}

// ---------------------------------------------------------------------------- launch
void make_taps(int kernel_size, Taps* taps) {
    // smoothing_kernel (density.py:30-37) in float64, rounded to float32.
    const int R = 3 * kernel_size;
    const double sigma = kernel_size / 2.0;
    double w[2 * kMaxR + 1];
    double tot = 0.0;
    for (int t = -R; t <= R; ++t) {
        const double u = t / sigma;
        w[t + R] = exp(-0.5 * (u * u));
        tot += w[t + R];
    }
    for (int t = 0; t <= 2 * R; ++t) taps->w[t] = (float)(w[t] / tot);
}

template <int R, typename T>
static int launch_h(const T* in, float* out, int s, const Taps& taps, const int* state, uint32_t* zero_next,
                    uint32_t* ctr, int nctr, cudaStream_t st) {
    const HGeo h = make_hgeo(s);
    const size_t smem = h_smem_bytes(h, R);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(smooth_h_kernel<R, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    dim3 grid(s / h.TWH, s / h.RH);
    INIM_CUDA_TRY(launch_pdl(smooth_h_kernel<R, T>, grid, dim3(h.NWH * 32), smem, st, in, out, s, h, taps, state,
                             zero_next, ctr, nctr));
    prof_mark(st, "smooth_h");
    return (int)cudaGetLastError();
}

template <int R>
static int launch_v(const float* tmp, float* d, const Geo& g, const Ws& ws, const Taps& taps, float bg, int emit,
                    const int* state, cudaStream_t st) {

    const VGeo v = make_vgeo(g);
    const size_t smem = v_smem_bytes(g, v, R);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(smooth_v_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr = true;
    }
    dim3 grid(g.NX, g.s / v.VR);
    INIM_CUDA_TRY(launch_pdl(smooth_v_kernel<R>, grid, dim3(v.VB * v.GT), smem, st, tmp, d, g, v, ws, taps, bg, emit,
                             state));
    prof_mark(st, emit ? "smooth_v_reduce" : "smooth_v");
    return (int)cudaGetLastError();
}

template <int KS>
static int launch_pair(const void* in, bool counts, const Geo& g, const Ws& ws, const Taps& taps, float bg,
                       float* d, int emit, const int* state, uint32_t* zero_next, cudaStream_t st) {
    constexpr int R = 3 * KS;
    uint32_t* ctr = nullptr;  // the standalone reduce has no band counters (lines_kernel)
    int rc = counts ? launch_h<R, uint32_t>(static_cast<const uint32_t*>(in), ws.tmp, g.s, taps, state, zero_next,
                                            ctr, g.B, st)
                    : launch_h<R, float>(static_cast<const float*>(in), ws.tmp, g.s, taps, state, zero_next, ctr,
                                         g.B, st);
    if (rc) return rc;
    return launch_v<R>(ws.tmp, d, g, ws, taps, bg, emit, state, st);
}

int launch_smooth_state(const void* in, bool in_is_counts, const Geo& g, const Ws& ws, int kernel_size,
                        float background, float* d, bool emit_aggregates, const int* state, cudaStream_t st,
                        uint32_t* zero_next) {
    if (kernel_size < 1 || 3 * kernel_size > kMaxR) return INIM_EKERNEL;  // 1 <= ks <= 16
    Taps taps;
    make_taps(kernel_size, &taps);
    const int emit = emit_aggregates ? 1 : 0;
    switch (kernel_size) {
#define INIM_KS(K) \
    case K: return launch_pair<K>(in, in_is_counts, g, ws, taps, background, d, emit, state, zero_next, st);
        INIM_KS(1) INIM_KS(2) INIM_KS(3) INIM_KS(4) INIM_KS(5) INIM_KS(6) INIM_KS(7) INIM_KS(8)
        INIM_KS(9) INIM_KS(10) INIM_KS(11) INIM_KS(12) INIM_KS(13) INIM_KS(14) INIM_KS(15) INIM_KS(16)
#undef INIM_KS
        default: break;
    }
    return INIM_EKERNEL;
}

}  // namespace inim
