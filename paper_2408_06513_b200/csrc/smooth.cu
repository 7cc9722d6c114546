// Density smoothing: gaussian_smooth + background (reference density.py:30-78).
//
// Two passes, horizontal then vertical, exactly the reference order (density.py:49-50),
// each a 6*ks+1-tap FIR with half-sample-symmetric reflection at the borders
// (scipy.ndimage mode="reflect", period 2s).  Both passes use the same "one lane per
// line, slide along the line" register-blocked FIR: the lane reads its line from
// shared memory with stride-1 lane addressing (conflict-free) and keeps P partial
// outputs in registers, so each input is read from shared memory once per P outputs;
// the taps are kernel parameters (constant-bank operands of FFMA).
//
// The vertical pass covers VB consecutive bands of the integral pipeline's TH x TW
// tiles per CTA (one thread group per band) and, when asked, hands each band's tile
// of d -- still in shared memory -- to tile_reduce, so the fused iteration never
// re-reads d for the integral pass's reduce phase.
#include "inim_tiles.cuh"

namespace inim {

constexpr int kMaxR = 48;  // kernel_size <= 16

struct Taps {
    float w[2 * kMaxR + 1];
};

// out[p] = sum_{t=0}^{2R} w[t] * line(p + t),  p in [0, n).  R is a compile-time radius.
template <int R, int P, typename Load, typename Store>
__device__ __forceinline__ void fir_line(const Taps& taps, int n, Load line, Store store) {
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
}

// ------------------------------------------------------------------------ horizontal
// Tile: RH rows x TWH columns; lane = row, warp = a CW-wide column chunk.
struct HGeo {
    int RH, TWH, NWH, CW;
};

inline HGeo make_hgeo(int s) {
    HGeo h;
    h.RH = s < 32 ? s : 32;
    h.TWH = s < 128 ? s : 128;
    int nw = h.TWH / 16;
    h.NWH = nw < 1 ? 1 : (nw > 8 ? 8 : nw);
    h.CW = h.TWH / h.NWH;
    return h;
}

inline size_t h_smem_bytes(const HGeo& h, int R) {
    return ((size_t)(h.TWH + 2 * R) * (h.RH + 1) + (size_t)h.RH * (h.TWH + 1)) * sizeof(float);
}

// zero_next (optional): the other counts buffer of the iteration's ping-pong pair; each
// CTA clears its own RH x TWH block of it, so the next splat needs no memset.
template <int R, typename T>
__global__ void __launch_bounds__(256) smooth_h_kernel(const T* __restrict__ in, float* __restrict__ out, int s,
                                                       const HGeo h, const Taps taps, const int* state,
                                                       uint32_t* __restrict__ zero_next) {
    if (state && state[0]) return;
    extern __shared__ __align__(16) float hsm[];
    const int RH = h.RH, TWH = h.TWH, ld = RH + 1;
    float* sh = hsm;                                 // [(TWH + 2R)][RH + 1]  transposed input
    float* so = hsm + (size_t)(TWH + 2 * R) * ld;    // [RH][TWH + 1]          output staging
    const int j0 = blockIdx.y * RH, i0 = blockIdx.x * TWH;
    const int W = TWH + 2 * R;
    const bool interior = i0 - R >= 0 && i0 + TWH + R <= s;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // warps over rows, lanes over columns: coalesced reads, no index division
    for (int r = w; r < RH; r += nw) {
        const T* row = in + (int64_t)(j0 + r) * s;
        constexpr int U = 4;
        for (int c0 = lane; c0 < W; c0 += 32 * U) {
            float v[U];
#pragma unroll
            for (int e = 0; e < U; ++e) {
                const int c = c0 + 32 * e;
                if (c < W) v[e] = (float)__ldg(row + (interior ? i0 - R + c : reflect_index(i0 - R + c, s)));
            }
#pragma unroll
            for (int e = 0; e < U; ++e) {
                const int c = c0 + 32 * e;
                if (c < W) sh[c * ld + r] = v[e];
            }
        }
        if (zero_next)
            for (int c = lane; c < TWH; c += 32) zero_next[(int64_t)(j0 + r) * s + i0 + c] = 0u;
    }
    __syncthreads();
    if (lane < RH) {
        const int c0 = w * h.CW;
        fir_line<R, 8>(
            taps, h.CW, [&](int q) { return sh[(c0 + q) * ld + lane]; },
            [&](int p, float v) { so[lane * (TWH + 1) + c0 + p] = v; });
    }
    __syncthreads();
    for (int r = w; r < RH; r += nw)
        for (int c = lane; c < TWH; c += 32) out[(int64_t)(j0 + r) * s + i0 + c] = so[r * (TWH + 1) + c];
}

// -------------------------------------------------------------------------- vertical
struct VGeo {
    int VR, VB, GT;  // rows per CTA, bands per CTA, threads per band group
};

inline VGeo make_vgeo(const Geo& g) {
    VGeo v;
    v.VR = g.s < 64 ? g.s : 64;
    v.VB = v.VR / g.TH;
    v.GT = g.TW < 32 ? 32 : g.TW;  // one thread per column per band
    return v;
}

inline size_t v_smem_bytes(const Geo& g, const VGeo& v, int R) {
    return ((size_t)(v.VR + 2 * R) * g.TW + (size_t)v.VR * g.TW) * sizeof(float);
}

template <int R>
__global__ void __launch_bounds__(512) smooth_v_kernel(const float* __restrict__ tmp, float* __restrict__ d,
                                                       const Geo g, const VGeo v, const Ws ws, const Taps taps,
                                                       float background, int emit, const int* state) {
    if (state && state[0]) return;
    extern __shared__ __align__(16) float vsm[];
    const int TH = g.TH, TW = g.TW, s = g.s, VR = v.VR;
    float* sh = vsm;                                 // [(VR + 2R)][TW]
    float* sd = vsm + (size_t)(VR + 2 * R) * TW;     // [VR][TW]  d for VB bands
    const int x = blockIdx.x;
    const int a0 = blockIdx.y * VR, i0 = x * TW;
    const int H = VR + 2 * R;
    const bool interior = a0 - R >= 0 && a0 + VR + R <= s;
    if ((TW & 3) == 0) {
        // (TW/4) float4 per row; threads tile (rows x float4 columns) without division
        const int TW4 = TW >> 2;
        const int cpr = TW4 < (int)blockDim.x ? TW4 : (int)blockDim.x;  // threads per row
        const int rpp = blockDim.x / cpr;                                // rows per pass
        const int c4 = threadIdx.x % cpr, r0 = threadIdx.x / cpr;        // once per thread
        constexpr int U = 4;
        for (int rb = r0; rb < H; rb += U * rpp) {
            float4 v4[U];
#pragma unroll
            for (int e = 0; e < U; ++e) {
                const int r = rb + e * rpp;
                if (r < H && c4 < TW4) {
                    const int row = interior ? a0 - R + r : reflect_index(a0 - R + r, s);
                    v4[e] = __ldg(reinterpret_cast<const float4*>(tmp + (int64_t)row * s + i0) + c4);
                }
            }
#pragma unroll
            for (int e = 0; e < U; ++e) {
                const int r = rb + e * rpp;
                if (r < H && c4 < TW4) reinterpret_cast<float4*>(sh)[r * TW4 + c4] = v4[e];
            }
        }
    } else {
        for (int q = threadIdx.x; q < H * TW; q += blockDim.x) {
            const int r = q / TW, c = q - r * TW;
            sh[q] = tmp[(int64_t)reflect_index(a0 - R + r, s) * s + i0 + c];
        }
    }
    __syncthreads();
    const int grp = threadIdx.x / v.GT, tid = threadIdx.x - grp * v.GT;
    const int u = tid;
    if (u < TW) {
        const int rb = grp * TH;  // first row of this group's band within the CTA
        fir_line<R, 8>(
            taps, TH, [&](int q) { return sh[(rb + q) * TW + u]; },
            [&](int p, float val) {
                const float dv = val + background;
                sd[(rb + p) * TW + u] = dv;
                d[(int64_t)(a0 + rb + p) * s + i0 + u] = dv;
            });
    }
    __syncthreads();
    if (emit) {
        // one warp per band tile of d, straight from shared memory
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
        for (int gb = warp; gb < v.VB; gb += nwarps) {
            const float* src = sd + (size_t)gb * TH * TW;
            const int b = a0 / TH + gb;
            if (g.CPL == 4) warp_tile_reduce<4>(src, TW, g, ws, b, x, lane);
            else if (g.CPL == 2) warp_tile_reduce<2>(src, TW, g, ws, b, x, lane);
            else warp_tile_reduce<1>(src, TW, g, ws, b, x, lane);
        }
    }
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
static int launch_h(const T* in, float* out, int s, const Taps& taps, const int* state, uint32_t* zero_next,
                    cudaStream_t st) {
    const HGeo h = make_hgeo(s);
    const size_t smem = h_smem_bytes(h, R);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(smooth_h_kernel<R, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    dim3 grid(s / h.TWH, s / h.RH);
    smooth_h_kernel<R, T><<<grid, h.NWH * 32, smem, st>>>(in, out, s, h, taps, state, zero_next);
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
    smooth_v_kernel<R><<<grid, v.VB * v.GT, smem, st>>>(tmp, d, g, v, ws, taps, bg, emit, state);
    prof_mark(st, emit ? "smooth_v_reduce" : "smooth_v");
    return (int)cudaGetLastError();
}

template <int KS>
static int launch_pair(const void* in, bool counts, const Geo& g, const Ws& ws, const Taps& taps, float bg,
                       float* d, int emit, const int* state, uint32_t* zero_next, cudaStream_t st) {
    constexpr int R = 3 * KS;
    int rc = counts ? launch_h<R, uint32_t>(static_cast<const uint32_t*>(in), ws.tmp, g.s, taps, state, zero_next, st)
                    : launch_h<R, float>(static_cast<const float*>(in), ws.tmp, g.s, taps, state, zero_next, st);
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
