// Density smoothing: gaussian_smooth + background (reference density.py:30-78).
//
// Two passes, horizontal then vertical, exactly the reference order (density.py:49-50),
// each a 6*ks+1-tap FIR with half-sample-symmetric reflection at the borders
// (scipy.ndimage mode="reflect", period 2s).  Both passes use the same "one lane per
// line, slide along the line" register-blocked FIR: the lane reads a line from shared
// memory with stride-1 lane addressing (conflict-free) and keeps P partial outputs in
// registers, so each input is read from shared memory once per P outputs; the taps
// are kernel parameters (constant bank operands of FFMA).
//
// The vertical pass runs on exactly the integral pipeline's TH x TW tiles and, when
// asked, hands its tile of d (still in shared memory) to tile_reduce, so the fused
// iteration reads d once for the integral pass.
#include "inim_tiles.cuh"

namespace inim {

constexpr int kMaxR = 48;  // kernel_size <= 16 uses the unrolled paths

struct Taps {
    float w[2 * kMaxR + 1];
};

// out[p] = sum_{t=0}^{2R} w[t] * line[base + p + t],  p in [0, n)
// `line(q)` returns input q of the extended line.  R is a compile-time radius (R > 0)
// or 0 for the runtime-radius path (rr).
template <int R, int P, typename Load, typename Store>
__device__ __forceinline__ void fir_line(const Taps& taps, int rr, int n, Load line, Store store) {
    if constexpr (R > 0) {
        constexpr int NT = 2 * R + 1;
        int p0 = 0;
        for (; p0 + P <= n; p0 += P) {
            float acc[P];
#pragma unroll
            for (int pp = 0; pp < P; ++pp) acc[pp] = 0.f;
#pragma unroll
            for (int q = 0; q < P + NT - 1; ++q) {
                const float v = line(p0 + q);
#pragma unroll
                for (int pp = 0; pp < P; ++pp) {
                    const int t = q - pp;
                    if (t >= 0 && t < NT) acc[pp] = fmaf(taps.w[t], v, acc[pp]);
                }
            }
#pragma unroll
            for (int pp = 0; pp < P; ++pp) store(p0 + pp, acc[pp]);
        }
        for (; p0 < n; ++p0) {
            float acc = 0.f;
#pragma unroll
            for (int t = 0; t < NT; ++t) acc = fmaf(taps.w[t], line(p0 + t), acc);
            store(p0, acc);
        }
    } else {
        const int NT = 2 * rr + 1;
        for (int p0 = 0; p0 < n; ++p0) {
            float acc = 0.f;
            for (int t = 0; t < NT; ++t) acc = fmaf(taps.w[t], line(p0 + t), acc);
            store(p0, acc);
        }
    }
}

// ------------------------------------------------------------------------ horizontal
// Tile: RH rows x TWH columns; lane = row, warp = a CW-wide column chunk.
struct HGeo {
    int RH, TWH, NWH, CW;
};

inline HGeo make_hgeo(int s) {
    HGeo h;
    h.RH = s < 32 ? s : 32;
    h.TWH = s < 256 ? s : 256;
    h.NWH = h.TWH >= 32 ? h.TWH / 32 : 1;
    h.CW = h.TWH / h.NWH;
    return h;
}

inline size_t h_smem_bytes(const HGeo& h, int R) {
    return ((size_t)(h.TWH + 2 * R) * (h.RH + 1) + (size_t)h.RH * (h.TWH + 1)) * sizeof(float);
}

template <int R, typename T>
__global__ void __launch_bounds__(256) smooth_h_kernel(const T* __restrict__ in, float* __restrict__ out, int s,
                                                       const HGeo h, const Taps taps, int rr, const int* state) {
    if (state && state[0]) return;
    extern __shared__ __align__(16) float hsm[];
    const int RR = R > 0 ? R : rr;
    const int RH = h.RH, TWH = h.TWH, ld = RH + 1;
    float* sh = hsm;                                  // [(TWH + 2R)][RH + 1]  transposed input
    float* so = hsm + (size_t)(TWH + 2 * RR) * ld;    // [RH][TWH + 1]          output staging
    const int j0 = blockIdx.y * RH, i0 = blockIdx.x * TWH;
    const int W = TWH + 2 * RR;
    for (int q = threadIdx.x; q < RH * W; q += blockDim.x) {
        const int r = q / W, c = q % W;
        const int col = reflect_index(i0 - RR + c, s);
        sh[c * ld + r] = (float)in[(int64_t)(j0 + r) * s + col];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane < RH) {
        const int c0 = w * h.CW;
        fir_line<R, 8>(
            taps, RR, h.CW, [&](int q) { return sh[(c0 + q) * ld + lane]; },
            [&](int p, float v) { so[lane * (TWH + 1) + c0 + p] = v; });
    }
    __syncthreads();
    for (int q = threadIdx.x; q < RH * TWH; q += blockDim.x) {
        const int r = q / TWH, c = q % TWH;
        out[(int64_t)(j0 + r) * s + i0 + c] = so[r * (TWH + 1) + c];
    }
}

// -------------------------------------------------------------------------- vertical
inline size_t v_smem_bytes(const Geo& g, int R) {
    return ((size_t)(g.TH + 2 * R) * g.TW + (size_t)g.TH * g.TW + 5 * (size_t)g.NW * g.TH) * sizeof(float);
}

template <int R>
__global__ void __launch_bounds__(256) smooth_v_kernel(const float* __restrict__ tmp, float* __restrict__ d,
                                                       const Geo g, const Ws ws, const Taps taps, int rr,
                                                       float background, int emit, const int* state) {
    if (state && state[0]) return;
    extern __shared__ __align__(16) float vsm[];
    const int RR = R > 0 ? R : rr;
    const int TH = g.TH, TW = g.TW, s = g.s;
    float* sh = vsm;                                  // [(TH + 2R)][TW]
    float* sd = vsm + (size_t)(TH + 2 * RR) * TW;     // [TH][TW]  the tile of d
    float* rec = sd + (size_t)TH * TW;                // tile_reduce scratch
    const int x = blockIdx.x, b = blockIdx.y;
    const int a = b * TH, i0 = x * TW;
    const int H = TH + 2 * RR;
    for (int q = threadIdx.x; q < H * TW; q += blockDim.x) {
        const int r = q / TW, c = q % TW;
        const int row = reflect_index(a - RR + r, s);
        sh[q] = tmp[(int64_t)row * s + i0 + c];
    }
    __syncthreads();
    const int u = threadIdx.x;
    if (u < TW) {
        fir_line<R, 8>(
            taps, RR, TH, [&](int q) { return sh[q * TW + u]; },
            [&](int p, float v) {
                const float dv = v + background;
                sd[p * TW + u] = dv;
                d[(int64_t)(a + p) * s + i0 + u] = dv;
            });
    }
    __syncthreads();
    if (emit) tile_reduce(sd, rec, g, ws, b, x);
}

// ---------------------------------------------------------------------------- launch
static void make_taps(int kernel_size, Taps* taps) {
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
static int launch_h(const T* in, float* out, int s, const Taps& taps, int rr, const int* state, cudaStream_t st) {
    const HGeo h = make_hgeo(s);
    const size_t smem = h_smem_bytes(h, R > 0 ? R : rr);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(smooth_h_kernel<R, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    dim3 grid(s / h.TWH, s / h.RH);
    smooth_h_kernel<R, T><<<grid, h.NWH * 32, smem, st>>>(in, out, s, h, taps, rr, state);
    prof_mark(st, "smooth_h");
    return (int)cudaGetLastError();
}

template <int R>
static int launch_v(const float* tmp, float* d, const Geo& g, const Ws& ws, const Taps& taps, int rr, float bg,
                    int emit, const int* state, cudaStream_t st) {
    const size_t smem = v_smem_bytes(g, R > 0 ? R : rr);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(smooth_v_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        attr = true;
    }
    dim3 grid(g.NX, g.B);
    smooth_v_kernel<R><<<grid, g.NW * 32, smem, st>>>(tmp, d, g, ws, taps, rr, bg, emit, state);
    prof_mark(st, emit ? "smooth_v_reduce" : "smooth_v");
    return (int)cudaGetLastError();
}

template <int KS>
static int launch_pair(const void* in, bool counts, const Geo& g, const Ws& ws, const Taps& taps, float bg,
                       float* d, int emit, const int* state, cudaStream_t st) {
    constexpr int R = 3 * KS;
    int rc = counts ? launch_h<R, uint32_t>(static_cast<const uint32_t*>(in), ws.tmp, g.s, taps, R, state, st)
                    : launch_h<R, float>(static_cast<const float*>(in), ws.tmp, g.s, taps, R, state, st);
    if (rc) return rc;
    return launch_v<R>(ws.tmp, d, g, ws, taps, R, bg, emit, state, st);
}

int launch_smooth_state(const void* in, bool in_is_counts, const Geo& g, const Ws& ws, int kernel_size,
                        float background, float* d, bool emit_aggregates, const int* state, cudaStream_t st) {
    if (kernel_size < 1) return INIM_EKERNEL;
    if (3 * kernel_size > kMaxR) return INIM_EKERNEL;  // taps array bound (ks <= 16)
    Taps taps;
    make_taps(kernel_size, &taps);
    const int emit = emit_aggregates ? 1 : 0;
    switch (kernel_size) {
#define INIM_KS(K) \
    case K: return launch_pair<K>(in, in_is_counts, g, ws, taps, background, d, emit, state, st);
        INIM_KS(1) INIM_KS(2) INIM_KS(3) INIM_KS(4) INIM_KS(5) INIM_KS(6) INIM_KS(7) INIM_KS(8)
        INIM_KS(9) INIM_KS(10) INIM_KS(11) INIM_KS(12) INIM_KS(13) INIM_KS(14) INIM_KS(15) INIM_KS(16)
#undef INIM_KS
        default: break;
    }
    const int rr = 3 * kernel_size;
    int rc = in_is_counts ? launch_h<0, uint32_t>(static_cast<const uint32_t*>(in), ws.tmp, g.s, taps, rr, state, st)
                          : launch_h<0, float>(static_cast<const float*>(in), ws.tmp, g.s, taps, rr, state, st);
    if (rc) return rc;
    return launch_v<0>(ws.tmp, d, g, ws, taps, rr, background, emit, state, st);
}

int launch_smooth(const void* in, bool in_is_counts, const Geo& g, const Ws& ws, int kernel_size, float background,
                  float* d, bool emit_aggregates, const int* state, cudaStream_t st) {
    return launch_smooth_state(in, in_is_counts, g, ws, kernel_size, background, d, emit_aggregates, state, st);
}

}  // namespace inim
