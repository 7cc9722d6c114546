// Density smoothing: gaussian_smooth + background (reference density.py:30-78).
//
// Two passes, horizontal then vertical, exactly the reference order (density.py:49-50),
// each a 6*ks+1-tap FIR with half-sample-symmetric reflection at the borders
// (scipy.ndimage mode="reflect", period 2s).  Kernel sizes 1..16 run the compiled FIRs
// (tile bodies in inim_smooth.cuh, launches in inim_smooth_launch.cuh, instantiated in
// smooth_ks*.cu); larger kernels the runtime-tap kernels below.
#include <type_traits>

#include "inim_smooth.cuh"

namespace inim {

// ------------------------------------------------------- generic taps (kernel_size > 16)
// The compiled FIRs carry the taps of kernel_size 1..16 as FFMA immediates.  Any
// larger kernel (the reference accepts every kernel_size >= 1, density.py:40-51) runs
// these runtime-tap kernels: the taps are evaluated on the device in float64 (the same
// exp / sum as smoothing_kernel, the sum passed in from the host) and stored float32.
// Reflection has period 2s, so when the kernel is longer than 2s its taps are folded
// onto one period: tap t (offset t - R) adds into slot (t - R) mod 2s, and the pass
// becomes a 2s-tap circular FIR with offsets 0..2s-1.
//   nt taps, offset o0: out[p] = sum_{q < nt} taps[q] * line[reflect(p + o0 + q)]
struct GenericTaps {
    int R, nt, o0;
    double sigma, inv_tot;
};

__global__ void generic_taps_kernel(float* __restrict__ taps, int s, const GenericTaps gt, int64_t zslab) {
    pdl_enter();
    taps = zoff(taps, zslab_off(zslab));
    const int64_t period = 2 * (int64_t)s;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < gt.nt; q += gridDim.x * blockDim.x) {
        double acc = 0.0;
        if (gt.o0 != 0) {  // unfolded: tap q is offset q - R
            const double u = (double)(q - gt.R) / gt.sigma;
            acc = exp(-0.5 * (u * u));
        } else {  // folded: every offset o = q (mod 2s) in [-R, R]
            int64_t o = (int64_t)q - ((int64_t)q + gt.R) / period * period;  // smallest o >= -R, o = q mod 2s
            if (o < -gt.R) o += period;
            for (; o <= gt.R; o += period) {
                const double u = (double)o / gt.sigma;
                acc += exp(-0.5 * (u * u));
            }
        }
        taps[q] = (float)(acc * gt.inv_tot);
    }
}

template <typename T>
__global__ void __launch_bounds__(256) generic_h_kernel(const T* __restrict__ in, float* __restrict__ out, int s,
                                                        const float* __restrict__ taps, const GenericTaps gt,
                                                        const int* state, uint32_t* __restrict__ zero_next,
                                                        int64_t zslab) {
    pdl_enter();
    state = zstate(state, zslab);
    if (state && state[0]) return;
    {
        const int64_t zo = zslab_off(zslab);
        in = zoff(in, zo);
        out = zoff(out, zo);
        taps = zoff(taps, zo);
        zero_next = zoff_opt(zero_next, zo);
    }
    const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
    if (i >= s) return;
    const T* row = in + (int64_t)j * s;
    float acc = 0.f;
    for (int q = 0; q < gt.nt; ++q) acc = fmaf(__ldg(taps + q), (float)__ldg(row + reflect_index(i + gt.o0 + q, s)), acc);
    out[(int64_t)j * s + i] = acc;
    if (zero_next) zero_next[(int64_t)j * s + i] = 0u;
}

__global__ void __launch_bounds__(256) generic_v_kernel(const float* __restrict__ tmp, float* __restrict__ d, int s,
                                                        const float* __restrict__ taps, const GenericTaps gt,
                                                        float background, const int* state, int64_t zslab) {
    pdl_enter();
    state = zstate(state, zslab);
    if (state && state[0]) return;
    {
        const int64_t zo = zslab_off(zslab);
        tmp = zoff(tmp, zo);
        d = zoff(d, zo);
        taps = zoff(taps, zo);
    }
    const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
    if (i >= s) return;
    float acc = 0.f;
    for (int q = 0; q < gt.nt; ++q)
        acc = fmaf(__ldg(taps + q), __ldg(tmp + (int64_t)reflect_index(j + gt.o0 + q, s) * s + i), acc);
    d[(int64_t)j * s + i] = acc + background;
}

static int launch_generic(const void* in, bool counts, const Geo& g, const Ws& ws, int kernel_size, float bg,
                          float* d, bool emit, const int* state, uint32_t* zero_next, cudaStream_t st,
                          const Bat& bt) {
    GenericTaps gt;
    const int64_t R64 = 3 * (int64_t)kernel_size;
    if (R64 > (int64_t)1 << 29) return INIM_EKERNEL;  // 6*ks+1 taps beyond int range
    gt.R = (int)R64;
    gt.sigma = kernel_size / 2.0;
    {  // the normalisation of smoothing_kernel (density.py:30-37), float64 on the host
        double tot = 0.0;
        for (int t = -gt.R; t <= gt.R; ++t) {
            const double u = t / gt.sigma;
            tot += exp(-0.5 * (u * u));
        }
        gt.inv_tot = 1.0 / tot;
    }
    const bool fold = 2 * (int64_t)gt.R + 1 > 2 * (int64_t)g.s;
    gt.nt = fold ? 2 * g.s : 2 * gt.R + 1;
    gt.o0 = fold ? 0 : -gt.R;
    const unsigned z = (unsigned)bt.B;
    INIM_CUDA_TRY(launch_pdl(generic_taps_kernel, dim3((gt.nt + 255) / 256, 1, z), dim3(256), 0, st, ws.taps, g.s, gt,
                             bt.slab));
    const dim3 grid((g.s + 255) / 256, g.s, z), block(256);
    if (counts)
        INIM_CUDA_TRY(launch_pdl(generic_h_kernel<uint32_t>, grid, block, 0, st, static_cast<const uint32_t*>(in),
                                 ws.tmp, g.s, (const float*)ws.taps, gt, state, zero_next, bt.slab));
    else
        INIM_CUDA_TRY(launch_pdl(generic_h_kernel<float>, grid, block, 0, st, static_cast<const float*>(in), ws.tmp,
                                 g.s, (const float*)ws.taps, gt, state, zero_next, bt.slab));
    prof_mark(st, "smooth_h");
    INIM_CUDA_TRY(launch_pdl(generic_v_kernel, grid, block, 0, st, (const float*)ws.tmp, d, g.s,
                             (const float*)ws.taps, gt, bg, state, bt.slab));
    prof_mark(st, "smooth_v");
    if (emit) return launch_reduce_from_global(d, g, ws, nullptr, st, bt);  // the integral pass's tile aggregates
    return (int)cudaGetLastError();
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

template <int KS>
int launch_pair(const void* in, int kind, const Geo& g, const Ws& ws, const Taps& taps, float bg, float* d,
                int emit, const int* state, uint32_t* zero_next, cudaStream_t st, const Bat& bt);

// in_kind: 0 = a float grid (gaussian_smooth), 1 = uint32 counts, 2 = float32 counts
// (integers; the move's 16-byte float reductions).  Counts smoothing also clears
// zero_next for the next iteration.
int launch_smooth_state(const void* in, int in_kind, const Geo& g, const Ws& ws, int kernel_size,
                        float background, float* d, bool emit_aggregates, const int* state, cudaStream_t st,
                        uint32_t* zero_next, const Bat& bt) {
    if (kernel_size < 1) return INIM_EKERNEL;
    if (3 * kernel_size > kMaxR)
        return launch_generic(in, in_kind == 1, g, ws, kernel_size, background, d, emit_aggregates, state, zero_next,
                              st, bt);
    Taps taps;
    make_taps(kernel_size, &taps);
    static const bool fuse = [] {
        const char* e = getenv("INIM_V_EMIT");
        return !(e && e[0] == '0');
    }();
    const int emit = emit_aggregates && fuse ? 1 : 0;
    int rc = INIM_EKERNEL;
    switch (kernel_size) {
#define INIM_KS(K) \
    case K: rc = launch_pair<K>(in, in_kind, g, ws, taps, background, d, emit, state, zero_next, st, bt); break;
        INIM_KS(1) INIM_KS(2) INIM_KS(3) INIM_KS(4) INIM_KS(5) INIM_KS(6) INIM_KS(7) INIM_KS(8)
        INIM_KS(9) INIM_KS(10) INIM_KS(11) INIM_KS(12) INIM_KS(13) INIM_KS(14) INIM_KS(15) INIM_KS(16)
#undef INIM_KS
        default: break;
    }
    if (rc || !emit_aggregates || emit) return rc;
    return launch_reduce_from_global(d, g, ws, nullptr, st, bt);
}

}  // namespace inim
