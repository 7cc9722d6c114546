// Smoothing tile functions (gaussian_smooth + background, reference density.py:30-78),
// used by the smoothing kernels (smooth.cu).  Each function processes one tile with the whole CTA and contains
// CTA-wide barriers, so every thread of the CTA must call it.
#pragma once

#include <type_traits>

#include "inim_taps.cuh"

#ifndef INIM_FFMA2_V
#define INIM_FFMA2_V 1  // vertical pass on packed fma.rn.f32x2 (0: scalar FFMA immediates)
#endif
#ifndef INIM_V_CPASYNC
#define INIM_V_CPASYNC 1  // vertical staging by cp.async (0: register-staged loads, four rows in flight)
#endif
#ifndef INIM_FFMA2_H
#define INIM_FFMA2_H 1  // horizontal pass on packed fma.rn.f32x2 (0: scalar FFMA immediates)
#endif
#include "inim_tiles.cuh"

namespace inim {

constexpr int kMaxR = 48;  // kernel_size <= 16

struct Taps {
    float w[2 * kMaxR + 1];
};

// out[p] = sum_{t=0}^{2R} w[t] * line(p + t),  p in [0, n), w = TapsOf<R / 3> (the taps are
// compile-time immediates of FFMA; `taps` is unused).  Register-blocked: P partial
// outputs per thread, every input read once per P outputs; taps are constant-bank
// operands of FFMA.
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
                if (t >= 0 && t < NT) acc[pp] = fmaf(TapsOf<R / 3>::w(t), v, acc[pp]);
            }
        }
#pragma unroll
        for (int pp = 0; pp < P; ++pp) store(p0 + pp, acc[pp]);
    }
    for (; p0 < n; ++p0) {
        float acc = 0.f;
#pragma unroll
        for (int t = 0; t < NT; ++t) acc = fmaf(TapsOf<R / 3>::w(t), line(p0 + t), acc);
        store(p0, acc);
    }
}

// The same FIR with the input line read as float4 (inputs 4*q4 .. 4*q4 + 3) and the
// outputs stored four at a time: n is a multiple of P, P a multiple of 4, and line4 may
// read up to 3 floats past the last input (they are never used).
template <int R, int P, typename Load4, typename Store4>
__device__ __forceinline__ void fir_line4(int n, Load4 line4, Store4 store4) {
    constexpr int NT = 2 * R + 1;
    constexpr int NQ = P + NT - 1;
    constexpr int NQ4 = (NQ + 3) / 4;
    for (int p0 = 0; p0 < n; p0 += P) {
        float acc[P];
#pragma unroll
        for (int pp = 0; pp < P; ++pp) acc[pp] = 0.f;
#pragma unroll
        for (int q4 = 0; q4 < NQ4; ++q4) {
            const float4 v4 = line4((p0 >> 2) + q4);
            const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int q = 4 * q4 + e;
#pragma unroll
                for (int pp = 0; pp < P; ++pp) {
                    const int t = q - pp;
                    if (q < NQ && t >= 0 && t < NT) acc[pp] = fmaf(TapsOf<R / 3>::w(t), vv[e], acc[pp]);
                }
            }
        }
#pragma unroll
        for (int pp = 0; pp < P; pp += 4) store4(p0 + pp, make_float4(acc[pp], acc[pp + 1], acc[pp + 2], acc[pp + 3]));
    }
}

// fir_line4 on packed fma.rn.f32x2: outputs (2m, 2m + 1) form one accumulator pair, and
// input x[i] enters it as a broadcast operand (ptxas encodes the {x, x} pair as `R.F32`,
// no moves) times the shifted tap pair (w[i - 2m], w[i - 2m - 1]) from constant memory
// (uniform registers; zero outside the kernel).  Each output still accumulates
// fma.rn(w[t], x[p + t], acc) for t ascending; the extra zero-tap terms at the two ends
// add +0 to an accumulator that is +0 or positive, so with finite inputs (counts) the
// result is bit-identical to fir_line4, with (NT + 1) x P/2 FFMA2 instead of NT x P FFMA.
template <int R, int P, typename Load4, typename Store4>
__device__ __forceinline__ void fir_line4_x2(int n, Load4 line4, Store4 store4) {
    static_assert(P % 4 == 0, "P: whole float4 groups of outputs");
    constexpr int NT = 2 * R + 1;
    constexpr int NQ = P + NT - 1;
    constexpr int NQ4 = (NQ + 3) / 4;
    constexpr int M = P / 2;
    for (int p0 = 0; p0 < n; p0 += P) {
        uint64_t acc[M];
#pragma unroll
        for (int m = 0; m < M; ++m) acc[m] = 0ull;
#pragma unroll
        for (int q4 = 0; q4 < NQ4; ++q4) {
            const float4 v4 = line4((p0 >> 2) + q4);
            const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int i = 4 * q4 + e;
                uint64_t xx;
                asm("mov.b64 %0, {%1, %1};" : "=l"(xx) : "f"(vv[e]));
#pragma unroll
                for (int m = 0; m < M; ++m) {
                    const int t = i - 2 * m;
                    if (i < NQ && t >= 0 && t <= NT) {
                        const uint64_t w2 = TapsOf<R / 3>::spair(t);
                        asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[m]) : "l"(w2), "l"(xx));
                    }
                }
            }
        }
#pragma unroll
        for (int m = 0; m < M; m += 2) {
            float4 o;
            asm("mov.b64 {%0, %1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(acc[m]));
            asm("mov.b64 {%0, %1}, %2;" : "=f"(o.z), "=f"(o.w) : "l"(acc[m + 1]));
            store4(p0 + 2 * m, o);
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
    h.TWH = s < 128 ? s : 128;
    int nw = h.TWH / 16;
    h.NWH = nw < 1 ? 1 : (nw > 8 ? 8 : nw);
    h.CW = h.TWH / h.NWH;
    return h;
}

// Row pitch of the staged input tile: at least TWH + 2R + 3 floats (the float4 reads
// of fir_line4 run up to 3 past the line), a multiple of 4 with pitch/4 odd, so that
// the 16-byte row stores and the 16-byte per-row FIR reads (lane = row) are both free
// of bank conflicts.
__host__ __device__ inline int h_pitch(int TWH, int R) {
    int p = (TWH + 2 * R + 3 + 3) & ~3;
    if (((p >> 2) & 1) == 0) p += 4;
    return p;
}

// Row pitch of the output staging tile: a multiple of 4 with pitch/4 odd (16-byte FIR
// stores, lane = row, and 16-byte row reads are conflict-free); TWH + 1 when the tile
// is narrower than a 16-byte group.
__host__ __device__ inline int h_opitch(int TWH) {
    if (TWH & 3) return TWH + 1;
    int p = TWH + 4;
    if (((p >> 2) & 1) == 0) p += 4;
    return p;
}

__host__ __device__ inline size_t h_smem_bytes(const HGeo& h, int R) {
    return ((size_t)h.RH * h_pitch(h.TWH, R) + (size_t)h.RH * h_opitch(h.TWH)) * sizeof(float);
}

// Horizontal pass of tile (bx, by).  zero_next (optional): the other count buffer of
// the iteration's ping-pong pair; the tile clears its own RH x TWH block of it.  CNT:
// the input is the iteration's counts (uint32, or float32 integers when the move
// splats with 16-byte float reductions); otherwise a float grid (gaussian_smooth).
// FULL: the geometry every grid of side >= 128 gets (32 x 128 tiles, 8 warps) as
// compile-time constants, so the staging, clearing and store loops fold to straight
// code (the runtime-geometry form spent ~40% of the kernel's instructions on them).
template <int R, typename T, bool CNT = !std::is_same<T, float>::value, bool FULL = false>
__device__ __forceinline__ void smooth_h_tile(const T* __restrict__ in, float* __restrict__ out, int s, const HGeo& h,
                                              const Taps& taps, uint32_t* __restrict__ zero_next, int bx, int by,
                                              float* hsm) {
    const int RH = FULL ? 32 : h.RH, TWH = FULL ? 128 : h.TWH, NWH = FULL ? 8 : h.NWH, CW = FULL ? 16 : h.CW;
    const int ld = h_pitch(TWH, R), op = h_opitch(TWH);
    float* sh = hsm;                      // [RH][ld]  input rows (row-major)
    float* so = hsm + (size_t)RH * ld;    // [RH][op]  output staging
    const int j0 = by * RH, i0 = bx * TWH;
    const int W = TWH + 2 * R;
    const bool interior = i0 - R >= 0 && i0 + TWH + R <= s;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = FULL ? 8 : (int)(blockDim.x >> 5);
    // warps over rows, lanes over columns (coalesced, no index division); every load of
    // a pass is issued before any of its shared-memory stores (up to RPW x NPR loads in
    // flight per thread)
    constexpr int RPW = CNT ? 2 : 4;  // rows per warp per pass
    constexpr int NPR = (128 + 2 * R + 31) / 32;  // columns per lane per row (TWH <= 128)
    constexpr int NP4 = (128 + 2 * R + 127) / 128;  // 16-byte groups per lane per row (interior tiles)
    const bool vec = interior && (TWH & 3) == 0 && ((i0 - R) & 3) == 0 && (s & 3) == 0;
    for (int r0 = w; r0 < RH; r0 += RPW * nw) {
        if (vec) {  // 16-byte loads of 4 consecutive columns -> 16-byte row stores
            uint4 v4[RPW][NP4];
#pragma unroll
            for (int q = 0; q < RPW; ++q) {
                const int r = r0 + q * nw;
                const uint4* row4 = reinterpret_cast<const uint4*>(
                    reinterpret_cast<const uint32_t*>(in) + (int64_t)(j0 + (r < RH ? r : 0)) * s + i0 - R);
#pragma unroll
                for (int e = 0; e < NP4; ++e) {
                    const int c4 = lane + 32 * e;
                    if (r < RH && 4 * c4 < W) v4[q][e] = __ldg(row4 + c4);
                }
            }
#pragma unroll
            for (int q = 0; q < RPW; ++q) {
                const int r = r0 + q * nw;
#pragma unroll
                for (int e = 0; e < NP4; ++e) {
                    const int c = 4 * (lane + 32 * e);
                    if (r < RH && c < W) {
                        const uint4 u = v4[q][e];
                        float4 f;
                        if (std::is_same<T, float>::value) {
                            f = make_float4(__uint_as_float(u.x), __uint_as_float(u.y), __uint_as_float(u.z),
                                            __uint_as_float(u.w));
                        } else {
                            f = make_float4((float)u.x, (float)u.y, (float)u.z, (float)u.w);
                        }
                        *reinterpret_cast<float4*>(sh + r * ld + c) = f;
                    }
                }
            }
        } else {
            T v[RPW][NPR];
#pragma unroll
            for (int q = 0; q < RPW; ++q) {
                const int r = r0 + q * nw;
                const T* row = in + (int64_t)(j0 + (r < RH ? r : 0)) * s;
#pragma unroll
                for (int e = 0; e < NPR; ++e) {
                    const int c = lane + 32 * e;
                    if (r < RH && c < W) v[q][e] = __ldg(row + (interior ? i0 - R + c : reflect_index(i0 - R + c, s)));
                }
            }
#pragma unroll
            for (int q = 0; q < RPW; ++q) {
                const int r = r0 + q * nw;
#pragma unroll
                for (int e = 0; e < NPR; ++e) {
                    const int c = lane + 32 * e;
                    if (r < RH && c < W) sh[r * ld + c] = (float)v[q][e];
                }
            }
        }
        if (zero_next) {  // clear this tile's block of the next count buffer (16-byte stores)
#pragma unroll
            for (int q = 0; q < RPW; ++q) {
                const int r = r0 + q * nw;
                if (r >= RH) break;
                if ((TWH & 3) == 0) {  // TWH <= 128: at most one 16-byte group per lane
                    uint4* z4 = reinterpret_cast<uint4*>(zero_next + (int64_t)(j0 + r) * s + i0);
                    if (lane < (TWH >> 2)) z4[lane] = make_uint4(0u, 0u, 0u, 0u);
                } else {
                    for (int c = lane; c < TWH; c += 32) zero_next[(int64_t)(j0 + r) * s + i0 + c] = 0u;
                }
            }
        }
    }
    __syncthreads();
    if (lane < RH && w < NWH) {
        const int c0 = w * CW;
        const float* row = sh + lane * ld + c0;
        float* orow = so + lane * op + c0;
        if ((CW & 15) == 0) {  // 16-byte reads of the row and 16-byte stores of the outputs
            auto ld4 = [&](int q4) { return *reinterpret_cast<const float4*>(row + 4 * q4); };
            auto st4 = [&](int p, float4 v) { *reinterpret_cast<float4*>(orow + p) = v; };
            if (INIM_FFMA2_H && CNT) fir_line4_x2<R, 16>(CW, ld4, st4);  // counts: finite
            else fir_line4<R, 16>(CW, ld4, st4);
        } else {
            fir_line<R, 16>(taps, CW, [&](int q) { return row[q]; }, [&](int p, float v) { orow[p] = v; });
        }
    }
    __syncthreads();
    if ((TWH & 3) == 0) {  // 16-byte row reads of the staging tile, 16-byte stores
        const int TW4 = TWH >> 2, l4 = FULL ? 5 : 31 - __clz(TW4);  // TWH is a power of two
        float* obase = out + (int64_t)j0 * s + i0;
        const int nthr = FULL ? 256 : (int)blockDim.x;
#pragma unroll 4
        for (int q = threadIdx.x; q < RH * TW4; q += nthr) {
            const int r = q >> l4, c = 4 * (q & (TW4 - 1));
            *reinterpret_cast<float4*>(obase + (int64_t)r * s + c) = *reinterpret_cast<const float4*>(so + r * op + c);
        }
    } else {
        for (int r = w; r < RH; r += nw)
            for (int c = lane; c < TWH; c += 32) out[(int64_t)(j0 + r) * s + i0 + c] = so[r * op + c];
    }
    __syncthreads();  // the tile's shared memory may be reused by the caller's next tile
}

// -------------------------------------------------------------------------- vertical
// Vertical FIR of one band's TH = 4P rows over TW columns by TW threads: thread t owns
// the column quad (t % (TW/4)) and the row group (t / (TW/4)) of P output rows, reads
// its P + 2R input rows as 16-byte loads (a warp reads whole 512-byte row segments),
// keeps its 4P outputs in registers across a CTA barrier, then writes them in place over
// the staged input (output row p of the CTA -> row p of `sh`): the tile needs no second
// shared-memory buffer.  Every thread of the CTA calls it (`live` = owns a quad).
template <int R, int P>
__device__ __forceinline__ void fir_cols4_inplace(float* __restrict__ sh, int TW, int rb, int t, bool live,
                                                  float background, int ld = 0) {
    constexpr int NT = 2 * R + 1;
    if (ld == 0) ld = TW;  // row pitch of sh (floats)
    const int nq = TW >> 2;
    const int quad = t % nq, rg = t / nq;
    const int r0 = rb + rg * P;
    float4 acc[P];
#pragma unroll
    for (int pp = 0; pp < P; ++pp) acc[pp] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (live) {
#if INIM_FFMA2_V
        // packed FP32: the column pairs (x, y) and (z, w) of the quad share each tap, so
        // one fma.rn.f32x2 (FFMA2) does two of the FMAs; the tap pairs come from constant
        // memory and stay in uniform registers.  Each lane's arithmetic is the same
        // fma.rn as the scalar form, in the same order: bit-identical results, half the
        // FMA instructions (issue slots for the loads and address math).
        uint64_t a2[P][2];
#pragma unroll
        for (int pp = 0; pp < P; ++pp) a2[pp][0] = a2[pp][1] = 0ull;
#pragma unroll
        for (int q = 0; q < P + NT - 1; ++q) {
            const float4 v4 = *reinterpret_cast<const float4*>(sh + (r0 + q) * ld + 4 * quad);
            uint64_t lo, hi;
            asm("mov.b64 %0, {%1, %2};" : "=l"(lo) : "f"(v4.x), "f"(v4.y));
            asm("mov.b64 %0, {%1, %2};" : "=l"(hi) : "f"(v4.z), "f"(v4.w));
#pragma unroll
            for (int pp = 0; pp < P; ++pp) {
                const int tp = q - pp;
                if (tp >= 0 && tp < NT) {
                    const uint64_t w2 = TapsOf<R / 3>::pair(tp);
                    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a2[pp][0]) : "l"(w2), "l"(lo));
                    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a2[pp][1]) : "l"(w2), "l"(hi));
                }
            }
        }
#pragma unroll
        for (int pp = 0; pp < P; ++pp) {
            asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[pp].x), "=f"(acc[pp].y) : "l"(a2[pp][0]));
            asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[pp].z), "=f"(acc[pp].w) : "l"(a2[pp][1]));
        }
#else
#pragma unroll
        for (int q = 0; q < P + NT - 1; ++q) {
            const float4 v4 = *reinterpret_cast<const float4*>(sh + (r0 + q) * ld + 4 * quad);
#pragma unroll
            for (int pp = 0; pp < P; ++pp) {
                const int tp = q - pp;
                if (tp >= 0 && tp < NT) {
                    const float w = TapsOf<R / 3>::w(tp);
                    acc[pp].x = fmaf(w, v4.x, acc[pp].x);
                    acc[pp].y = fmaf(w, v4.y, acc[pp].y);
                    acc[pp].z = fmaf(w, v4.z, acc[pp].z);
                    acc[pp].w = fmaf(w, v4.w, acc[pp].w);
                }
            }
        }
#endif
    }
    __syncthreads();  // every input row has been read
    if (live) {
#pragma unroll
        for (int pp = 0; pp < P; ++pp)
            *reinterpret_cast<float4*>(sh + (r0 + pp) * ld + 4 * quad) = make_float4(
                acc[pp].x + background, acc[pp].y + background, acc[pp].z + background, acc[pp].w + background);
    }
}

__host__ __device__ inline bool v_inplace(int TH, int TW, int GT) { return (TW & 3) == 0 && GT == TW && (TH == 32 || TH == 16); }

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

__host__ __device__ inline size_t v_smem_bytes(const Geo& g, const VGeo& v, int R) {
    if (v_inplace(g.TH, g.TW, v.GT)) return (size_t)(v.VR + 2 * R) * g.TW * sizeof(float);
    return ((size_t)(v.VR + 2 * R) * g.TW + (size_t)v.VR * g.TW) * sizeof(float);
}

// Vertical pass + background of tile (bx, by) = VB bands x TW columns; with `emit`,
// each band's tile of d goes straight from shared memory into the tile reduce.
// VG: the two geometries the runs use as compile-time constants (1: 32 x 128 bands of
// batches and grids above 2048^2, 2: the 16 x 64 bands up to 2048^2, both 64-row CTAs of
// 256 threads), so the staging, FIR and reduce dispatch and the store loop fold; 0: the
// runtime geometry of small grids.
template <int R, int VG = 0>
__device__ __forceinline__ void smooth_v_tile(const float* __restrict__ tmp, float* __restrict__ d, const Geo& g,
                                              const VGeo& v, const Ws& ws, const Taps& taps, float background,
                                              int emit, int bx, int by, float* vsm, uint32_t* zero_next = nullptr) {
    const int TH = VG == 1 ? 32 : (VG == 2 ? 16 : g.TH);
    const int TW = VG == 1 ? 128 : (VG == 2 ? 64 : g.TW);
    const int VR = VG ? 64 : v.VR, VB = VG == 1 ? 2 : (VG == 2 ? 4 : v.VB), GT = VG ? TW : v.GT;
    const int CPL = VG == 1 ? 4 : (VG == 2 ? 2 : g.CPL);
    const int NT = VG ? 256 : (int)blockDim.x;
    const int s = g.s;
    const bool inplace = VG ? true : v_inplace(TH, TW, GT);
    float* sh = vsm;                                                 // [(VR + 2R)][TW]
    float* sd = inplace ? vsm : vsm + (size_t)(VR + 2 * R) * TW;     // [VR][TW]  d for VB bands
    const int x = bx;
    const int a0 = by * VR, i0 = x * TW;
    const int H = VR + 2 * R;
    const bool interior = a0 - R >= 0 && a0 + VR + R <= s;
    if ((TW & 3) == 0 && INIM_V_CPASYNC) {
        // (TW/4) float4 per row: every 16-byte piece of the staging tile is requested at
        // once as an asynchronous global -> shared copy (cp.async.cg, no register
        // staging), so the tile costs one memory round trip
        const int TW4 = TW >> 2;
        const int cpr = TW4 < NT ? TW4 : NT;  // threads per row
        const int rpp = NT / cpr;              // rows per pass
        const int c4 = threadIdx.x % cpr;
        if (c4 < TW4) {
            for (int r = threadIdx.x / cpr; r < H; r += rpp) {
                const int row = interior ? a0 - R + r : reflect_index(a0 - R + r, s);
                cp_async16(reinterpret_cast<float4*>(sh) + r * TW4 + c4,
                           reinterpret_cast<const float4*>(tmp + (int64_t)row * s + i0) + c4);
            }
        }
        cp_async_wait_all();
    } else if ((TW & 3) == 0) {
        // (TW/4) float4 per row; threads tile (rows x float4 columns) without division
        const int TW4 = TW >> 2;
        const int cpr = TW4 < (int)blockDim.x ? TW4 : (int)blockDim.x;  // threads per row
        const int rpp = blockDim.x / cpr;                                // rows per pass
        const int c4 = threadIdx.x % cpr, r0 = threadIdx.x / cpr;
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
    const int grp = threadIdx.x / GT, tid = threadIdx.x - grp * GT;
    if (inplace) {  // (the branch is uniform over the CTA: it contains a barrier)
        const bool live = grp < VB;
        if (TH == 32) fir_cols4_inplace<R, 8>(sh, TW, grp * TH, tid, live, background);
        else fir_cols4_inplace<R, 4>(sh, TW, grp * TH, tid, live, background);
    } else if (grp < VB && tid < TW) {
        const int rb = grp * TH;  // first row of this group's band within the CTA
        fir_line<R, 8>(
            taps, TH, [&](int q) { return sh[(rb + q) * TW + tid]; },
            [&](int p, float val) { sd[(rb + p) * TW + tid] = val + background; });
    }
    __syncthreads();
    if (emit) {
        // one warp per band tile of d, straight from shared memory
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = NT >> 5;
        for (int gb = warp; gb < VB; gb += nwarps) {
            const float* src = sd + (size_t)gb * TH * TW;
            const int b = a0 / TH + gb;
            if (CPL == 4) warp_tile_reduce<4>(src, TW, g, ws, b, x, lane);
            else if (CPL == 2) warp_tile_reduce<2>(src, TW, g, ws, b, x, lane);
            else warp_tile_reduce<1>(src, TW, g, ws, b, x, lane);
        }
    }
    // the VR x TW tile of d out; zero_next (optional): the same block of the other count
    // buffer cleared for the next iteration's splat (the horizontal pass read it one
    // iteration ago; clearing it here keeps those stores off the horizontal pass, whose
    // traffic is a third clears otherwise, and on warps that would idle at the barrier)
    if ((TW & 3) == 0) {
        const int TW4 = TW >> 2, l4 = VG == 1 ? 5 : (VG == 2 ? 4 : 31 - __clz(TW4));  // TW is a power of two
        for (int q = threadIdx.x; q < VR * TW4; q += NT) {
            const int r = q >> l4, c4 = q & (TW4 - 1);
            reinterpret_cast<float4*>(d + (int64_t)(a0 + r) * s + i0)[c4] = reinterpret_cast<const float4*>(sd)[q];
            if (zero_next)
                reinterpret_cast<uint4*>(zero_next + (int64_t)(a0 + r) * s + i0)[c4] = make_uint4(0u, 0u, 0u, 0u);
        }
    } else {
        for (int q = threadIdx.x; q < VR * TW; q += blockDim.x) {
            const int r = q / TW, c = q - r * TW;
            d[(int64_t)(a0 + r) * s + i0 + c] = sd[q];
            if (zero_next) zero_next[(int64_t)(a0 + r) * s + i0 + c] = 0u;
        }
    }
    __syncthreads();
}

}  // namespace inim
