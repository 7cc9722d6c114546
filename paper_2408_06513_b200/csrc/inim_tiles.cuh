// Warp-per-tile integral kernels (phase 1 reduce, phase 3 write), shared by the
// standalone integral kernels (integral.cu) and the vertical smoothing pass (smooth.cu).
//
// One warp owns one TH x TW tile (TW = 32 * CPL, TH <= 32); lane l owns the CPL
// consecutive columns 4l..4l+3 (CPL = 4) and sweeps the TH rows.  Nothing crosses a
// warp: the row scan is one warp scan per row, the diagonal chains move one column per
// row through registers and one shuffle, and everything a tile needs from outside
// (carries from the band above, the neighbouring tiles' edge chains, the marginals) is
// loaded once into lane-distributed registers and delivered by shuffles as the sweep
// advances.
#pragma once

#include "inim_internal.cuh"

namespace inim {

template <int CPL>
INIM_DEV void load_row(const float* __restrict__ p, float (&v)[CPL]) {
    if constexpr (CPL == 4) {
        const float4 q = *reinterpret_cast<const float4*>(p);
        v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else if constexpr (CPL == 2) {
        const float2 q = *reinterpret_cast<const float2*>(p);
        v[0] = q.x; v[1] = q.y;
    } else {
        v[0] = *p;
    }
}

template <int CPL>
INIM_DEV void load_row_g(const float* __restrict__ p, float (&v)[CPL]) {
    if constexpr (CPL == 4) {
        const float4 q = __ldg(reinterpret_cast<const float4*>(p));
        v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else if constexpr (CPL == 2) {
        const float2 q = __ldg(reinterpret_cast<const float2*>(p));
        v[0] = q.x; v[1] = q.y;
    } else {
        v[0] = __ldg(p);
    }
}

template <int CPL>
INIM_DEV void store_row(float* p, const float (&v)[CPL]) {
    if constexpr (CPL == 4) {
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    } else if constexpr (CPL == 2) {
        *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
    } else {
        *p = v[0];
    }
}

template <int CPL>
INIM_DEV void store_row_cs(float* p, const float (&v)[CPL]) {
    if constexpr (CPL == 4) {
        __stcs(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
    } else if constexpr (CPL == 2) {
        __stcs(reinterpret_cast<float2*>(p), make_float2(v[0], v[1]));
    } else {
        __stcs(p, v[0]);
    }
}

// ------------------------------------------------------------------ phase 1: reduce
// src: tile origin (shared or global), row stride ld.  Writes the per-tile aggregates:
//   inpre[b][c] (in-tile row prefix of the column sums), tiletot[b][x], ulbot[b][c],
//   urbot[b][c] (in-tile chains of the column prefix V at the
//   band's last row), ule/ure[b][x][r] (chains at the tile's last / first column, complete
//   in-band values since TW >= TH), rowsum[j][x].
// Exclusive prefix of a line of n values (one warp, float64, loads through L2 so other
// warps' writes of this launch are seen); returns the line total.
template <typename T>
__device__ __forceinline__ double warp_line_prefix(const T* src, double* __restrict__ dst, int n, int lane) {
    double carry = 0.0;
    for (int base = 0; base < n; base += 32) {
        const int x = base + lane;
        const double v = x < n ? (double)__ldcg(src + x) : 0.0;
        const double inc = warp_inclusive_scan_d(v, lane);
        if (x < n) dst[x] = carry + inc - v;
        carry += __shfl_sync(kFull, inc, 31);
    }
    return carry;
}

// Per-tile aggregates of the reduce, fed one row at a time (lane l holds columns
// CPL*l .. CPL*l + CPL - 1 of the row).  finish() writes inpre / tiletot / ulbot / urbot
// / rowsum; the band lines are a launch of their own (lines_kernel).
template <int CPL>
struct TileReducer {
    const Geo& g;
    const Ws& ws;
    int b, x, lane, last;
    bool act;
    float* ule_t;  // edge chains, stored row by row by the edge lanes
    float* ure_t;
    float V[CPL], UL[CPL], UR[CPL];
    float rs_mine;
    __device__ __forceinline__ TileReducer(const Geo& g_, const Ws& ws_, int b_, int x_, int lane_)
        : g(g_), ws(ws_), b(b_), x(x_), lane(lane_), last(g_.WL - 1), act(lane_ <= g_.WL - 1), rs_mine(0.f) {
        const int64_t tile = (int64_t)b * g.NX + x;
        ule_t = ws.ule + tile * g.TH;
        ure_t = ws.ure + tile * g.TH;
#pragma unroll
        for (int e = 0; e < CPL; ++e) V[e] = UL[e] = UR[e] = 0.f;
    }
    // ROWSUM: reduce the row's sum over the warp here (else the caller supplies the row
    // sums through set_rowsum)
    template <bool ROWSUM = true>
    __device__ __forceinline__ void row(int r, const float (&dv)[CPL]) {
        float rsum = 0.f;
#pragma unroll
        for (int e = 0; e < CPL; ++e) {
            V[e] += dv[e];
            rsum += dv[e];
        }
        float fromL = __shfl_up_sync(kFull, UL[CPL - 1], 1);
        float fromR = __shfl_down_sync(kFull, UR[0], 1);
        if (lane == 0) fromL = 0.f;     // clipped at the tile's left edge
        if (lane >= last) fromR = 0.f;  // clipped at the tile's right edge
#pragma unroll
        for (int e = CPL - 1; e > 0; --e) UL[e] = V[e] + UL[e - 1];
        UL[0] = V[0] + fromL;
#pragma unroll
        for (int e = 0; e < CPL - 1; ++e) UR[e] = V[e] + UR[e + 1];
        UR[CPL - 1] = V[CPL - 1] + fromR;
        if (ROWSUM) {
            rsum = warp_sum(rsum);
            if (lane == r) rs_mine = rsum;
        }
        if (lane == last) ule_t[r] = UL[CPL - 1];
        if (lane == 0) ure_t[r] = UR[0];
    }
    __device__ __forceinline__ void set_rowsum(int r, float v) {
        if (lane == r) rs_mine = v;
    }
    __device__ __forceinline__ void finish() {
        const int TH = g.TH, TW = g.TW, s = g.s, NX = g.NX;
        const int a = b * TH, i0 = x * TW, u0 = lane * CPL;
        // in-tile inclusive row prefix of the column sums (float64 scan over the lanes)
        // and the tile total
        double lsum = 0.0;
#pragma unroll
        for (int e = 0; e < CPL; ++e) lsum += (double)V[e];
        const double linc = warp_inclusive_scan_d(lsum, lane);
        if (act) {
            float* ip = ws.inpre + (int64_t)b * s + i0 + u0;
            float* ub = ws.ulbot + (int64_t)b * s + i0 + u0;
            float* rb = ws.urbot + (int64_t)b * s + i0 + u0;
            double run = linc - lsum;
#pragma unroll
            for (int e = 0; e < CPL; ++e) {
                run += (double)V[e];
                ip[e] = (float)run;
                ub[e] = UL[e];
                rb[e] = UR[e];
            }
        }
        if (lane == 31) ws.tiletot[(int64_t)b * NX + x] = linc;
        if (lane < TH) ws.rowsum[(int64_t)(a + lane) * NX + x] = rs_mine;
    }
};

// The reduce of one tile from `src` (tile origin, row stride ld): a staged tile
// (shared memory), or with GSRC global memory read through a ring of PF rows in flight
// per lane, refilled as rows retire (PF = 8 measured slower than 2: registers).
template <int CPL, bool GSRC = false>
__device__ __forceinline__ void warp_tile_reduce(const float* src, int ld, const Geo g, const Ws ws, int b, int x,
                                                 int lane) {
    const int TH = g.TH;
    const int u0 = lane * CPL;
    const bool act = lane <= g.WL - 1;
    TileReducer<CPL> red(g, ws, b, x, lane);
    constexpr int PF = GSRC ? (CPL <= 2 ? 16 : 2) : 1;
    float ring[PF][CPL];
    if (GSRC) {
#pragma unroll
        for (int q = 0; q < PF; ++q) {
#pragma unroll
            for (int e = 0; e < CPL; ++e) ring[q][e] = 0.f;
            if (act && q < TH) load_row_g<CPL>(src + (size_t)q * ld + u0, ring[q]);
        }
    }
    for (int r0 = 0; r0 < TH; r0 += PF) {  // PF rows per trip: the ring slot is a compile-time index
#pragma unroll
        for (int q = 0; q < PF; ++q) {
            const int r = r0 + q;
            if (r >= TH) break;
            float dv[CPL];
            if (GSRC) {
#pragma unroll
                for (int e = 0; e < CPL; ++e) dv[e] = ring[q][e];
                if (act && r + PF < TH) load_row_g<CPL>(src + (size_t)(r + PF) * ld + u0, ring[q]);
            } else if (act) {
                load_row<CPL>(src + (size_t)r * ld + u0, dv);
            } else {
#pragma unroll
                for (int e = 0; e < CPL; ++e) dv[e] = 0.f;
            }
            red.row(r, dv);
        }
    }
    red.finish();
}

// --------------------------------------------------------- flat response / anchors
// Region pixel counts of a constant texture (exact integers) -> raw map, float64, in
// the operation order of _per_pixel_targets (mapping.py:146-178).
__device__ __forceinline__ double2 flat_response_at(int i, int j, int k) {
    const int64_t S = (int64_t)1 << k, s2 = S * S;
    const int64_t I = i, J = j;
    auto f = [&](int64_t L) { return L * (J + 1) - L * (L + 1) / 2; };
    const int64_t up1 = (J + 1) + f(min(J, I)) + f(min(J, S - 1 - I));
    const int64_t sg = I + J;
    const int64_t A1 = sg <= S - 1 ? (sg + 1) * (sg + 2) / 2 : s2 - (2 * S - 2 - sg) * (2 * S - 1 - sg) / 2;
    const int64_t dl = I - J;
    const int64_t D1 = dl >= 0 ? (S - dl) * (S - dl + 1) / 2 : s2 - (S + dl - 1) * (S + dl) / 2;
    const double tl = (double)((I + 1) * (J + 1)), bl = (double)((I + 1) * (S - 1 - J));
    const double tr = (double)((S - 1 - I) * (J + 1)), br = (double)((S - 1 - I) * (S - 1 - J));
    const double up = (double)up1, left = (double)(A1 - up1), right = (double)(D1 - up1);
    const double down = (double)s2 - up - left - right;
    const double scale = ldexp(1.0, -k);
    const double x = i * scale, y = j * scale;
    const bool below = y < x, near = x + y < 1.0;
    const double drx = below ? 1.0 : 1.0 - y + x, dry = below ? 1.0 + y - x : 1.0;
    const double ulx = below ? x - y : 0.0, uly = below ? 0.0 : y - x;
    const double urx = near ? x + y : 1.0, ury = near ? 0.0 : x + y - 1.0;
    const double dlx = near ? 0.0 : x + y - 1.0, dly = near ? x + y : 1.0;
    const double inv = 0.5 / (double)s2;
    double2 t;
    t.x = (tl * drx + bl * urx + br * ulx + tr * dlx + (up + down) * x + left) * inv;
    t.y = (tl * dry + bl * ury + br * uly + tr * dly + (left + right) * y + up) * inv;
    return t;
}

// ------------------------------------------------------------------- phase 3: write
struct WriteOut {
    float* tables8;       // MODE 0
    float* targets;       // MODE 1/2: (s, s, 2), or null
    const float* defect;  // MODE 2: (s, s, 2)
    float* max_exc;       // MODE 1/2
    float* pairs;         // MODE 1/2: (s, s, 4) = (t(i, j), t(i + 1, j)), or null
};

// Sliding window over a per-band vector indexed by (column +/- row): lane l holds the
// CPL entries of its columns for the current row; entering entries come from the
// neighbouring lane or, at the tile edge, from `ext` (lane q holds the entry entering
// at row q + 1).
template <int CPL, typename T>
INIM_DEV void slide_left(T (&w)[CPL], T ext, int r, int lane) {  // index decreases by one per row
    T in = __shfl_up_sync(kFull, w[CPL - 1], 1);
    const T e = __shfl_sync(kFull, ext, r);
    if (lane == 0) in = e;
#pragma unroll
    for (int q = CPL - 1; q > 0; --q) w[q] = w[q - 1];
    w[0] = in;
}

template <int CPL, typename T>
INIM_DEV void slide_right(T (&w)[CPL], T ext, int r, int lane, int last) {  // index increases by one per row
    T in = __shfl_down_sync(kFull, w[0], 1);
    const T e = __shfl_sync(kFull, ext, r);
    if (lane == last) in = e;
#pragma unroll
    for (int q = 0; q < CPL - 1; ++q) w[q] = w[q + 1];
    w[CPL - 1] = in;
}

// Region pixel counts of a constant s x s texture (exact).
// wedge_up count: (j + 1) + g(min(j, i)) + g(min(j, s - 1 - i)),  g(L) = L (2j + 1 - L) / 2
// (each L (2j + 1 - L) is even).  ri = s - 1 - i, tj1 = 2j + 1.  Each product is at
// most j (j + 1) < s^2, so their sum fits uint32 up to s = 2^15 (INIM_MAX_K).
INIM_DEV uint32_t flat_up_count(int i, int ri, int j, int tj1) {
    const uint32_t l1 = (uint32_t)min(j, i), l2 = (uint32_t)min(j, ri), t = (uint32_t)tj1;
    return (uint32_t)(j + 1) + ((l1 * (t - l1) + l2 * (t - l2)) >> 1);
}
INIM_DEV int64_t flat_apre_count(int sg, int s) {  // #{i' + j' <= sg}
    const int64_t S = s;
    return sg <= s - 1 ? (int64_t)(sg + 1) * (sg + 2) / 2 : S * S - (2 * S - 2 - sg) * (2 * S - 1 - sg) / 2;
}
INIM_DEV int64_t flat_dsuf_count(int dl, int s) {  // #{i' - j' >= dl}
    const int64_t S = s;
    return dl >= 0 ? (S - dl) * (S - dl + 1) / 2 : S * S - (S + dl - 1) * (S + dl) / 2;
}


// MODE 0: stream the eight tables (float32 assembly from float64-rounded constants).
// MODE 1 / 2: deformation field (build_field, mapping.py:194-204), with the raw map in the
// collapsed form  2C tx = tl(1-2y) + up(2x-1) + Gx,  2C ty = tl(1-2x) + up(1-2y) + Gy
// (the anchor coefficients of tl and up are constant across the mapping.py:42/47
// branches; Gx, Gy carry the column / row / diagonal marginals Cp, Rp, Ap, Ds).  Every
// quantity is normalised by its total (C for the data, s^2 for the flat texture) so the
// arithmetic is O(1) float32.  Without an explicit defect array the flat response is
// folded in term by term: the same linear form is evaluated on (data/C - flat/s^2)
// differences, which are small where the density is near uniform, so the cancellation
// of raw - defect happens before rounding instead of after (MODE 1); MODE 2 subtracts an
// explicit defect array (build_field with a caller-supplied flat response).
// GSRC: `src` is the tile origin in global memory (row stride ld) and rows are fetched
// two ahead into registers; otherwise `src` is a staged (shared-memory) tile.
// GEO: the run geometry as compile-time constants (TW = 32 CPL with every lane holding
// columns, TH = 32 for CPL = 4, 16 for CPL = 2), so the row sweep and the per-row lane
// tests fold; the caller checks the geometry.
template <int CPL, int MODE, bool GSRC = false, bool GEO = false>
__device__ __forceinline__ void warp_tile_write(const float* src, int ld, const Geo g, const Ws ws, int b, int x,
                                                int lane, const WriteOut out) {
    const int TH = GEO ? (CPL == 4 ? 32 : 16) : g.TH, TW = GEO ? 32 * CPL : g.TW, s = g.s, NX = g.NX, B = g.B;
    const int last = GEO ? 31 : g.WL - 1;
    const int u0 = lane * CPL;
    const bool act = lane <= last;
    const int a = b * TH, i0 = x * TW;
    const int64_t tile = (int64_t)b * NX + x;
    const double* __restrict__ bandpre = ws.bandpre;
    const double C = bandpre[B];
    const double invC = 1.0 / C;
    constexpr bool diff = MODE == 1;  // fold the flat response in
    const double inv_s = ldexp(1.0, -g.k), inv_s2 = inv_s * inv_s;
    const float* __restrict__ tlc = ws.tlcar + (int64_t)b * s;
    const float* __restrict__ cpre = ws.tlcar + (int64_t)B * s;
    const float* __restrict__ x1 = ws.x1 + (int64_t)b * s;
    const float* __restrict__ x2 = ws.x2 + (int64_t)b * (s + TH);
    // diagonal marginals read off the chain carries (inim_scan.cuh "marg")
    auto apre = [&](int sg) -> double {  // Apre[sigma]
        if (sg < s) {
            const int bb = sg / TH, r = sg - bb * TH;
            return (double)ws.ure[(int64_t)bb * NX * TH + r] + (double)ws.x2[(int64_t)bb * (s + TH) + r + 1];
        }
        return (double)ws.x2[(int64_t)B * (s + TH) + sg - (s - 1)];
    };
    auto dsuf = [&](int dl) -> double {  // Dsuf[delta]
        if (dl >= 0) {
            const int j = s - 1 - dl, bb = j / TH, r = j - bb * TH, c2 = s - 2 - r;
            return (double)ws.ule[((int64_t)bb * NX + NX - 1) * TH + r] + bandpre[bb] +
                   (c2 >= 0 ? (double)ws.x1[(int64_t)bb * s + c2] : 0.0);
        }
        return (double)ws.x1[(int64_t)B * s + s - 1 + dl] + C;
    };
    // normalised marginal entries (MODE 1): value / C, minus the flat value when folding.
    // The field's marginal coefficients are kept HALVED (exact: a power-of-two scale) so
    // the 1/2 of the raw map folds into them instead of costing a multiply per pixel.
    auto nap = [&](int sg) {
        const double v = apre(sg) * invC;
        return (float)(0.5 * (diff ? v - (double)flat_apre_count(sg, s) * inv_s2 : v));
    };
    auto nds = [&](int dl) {
        const double v = dsuf(dl) * invC;
        return (float)(0.5 * (diff ? v - (double)flat_dsuf_count(dl, s) * inv_s2 : v));
    };
    // per-column constants and initial windows (row 0)
    float A[CPL], Bc[CPL], w1[CPL], w2[CPL], wa[CPL], wd[CPL];
#pragma unroll
    for (int e = 0; e < CPL; ++e) {
        const int i = i0 + u0 + e;
        const bool ok = act && i < s;
        const double tv = ok ? (double)tlc[i] : 0.0, cv = ok ? (double)cpre[i] : 0.0;
        A[e] = (float)tv;
        w1[e] = (float)(ok && i - 1 >= 0 ? x1[i - 1] : 0.0);  // X1[i - r - 1]
        w2[e] = (float)(ok ? x2[i + 1] : 0.0);                // X2[i + r + 1]
        if (MODE == 0) {
            Bc[e] = (float)(cv - tv);
            wa[e] = (float)(ok ? apre(a + i) : 0.0);  // Apre[i + j]
            wd[e] = (float)(ok ? dsuf(i - a) : 0.0);  // Dsuf[i - j]
        } else {
            Bc[e] = (float)(0.5 * (diff ? cv * invC - (i + 1) * inv_s : cv * invC));  // Cp / 2
            wa[e] = ok ? nap(a + i) : 0.f;
            wd[e] = ok ? nds(i - a) : 0.f;
        }
    }
    // lane-distributed: row constants (lane q = row q) and window / chain edge entries
    float P = 0, Q = 0, S = 0;
    float e1 = 0, e2 = 0, ea = 0, ed = 0;
    float ulel = 0.f, urer = 0.f;
    {
        const double hc = lane < TH ? ws.hc[(int64_t)(a + lane) * NX + x] : 0.0;
        const double vh = warp_inclusive_scan_d(hc, lane);
        if (lane < TH) {
            const double Rp = bandpre[b] + ws.rpre[a + lane];
            P = (float)vh;
            if (MODE == 0) {
                Q = (float)(Rp - vh);
                S = (float)(C - Rp + vh);
            } else {
                Q = (float)(0.5 * (diff ? Rp * invC - (a + lane + 1) * inv_s : Rp * invC));  // Rp / 2
            }
            if (lane < TH - 1) {  // entry q feeds row q + 1
                const int c1 = i0 - 2 - lane;
                e1 = (float)(c1 >= 0 ? x1[c1] : 0.0);
                e2 = (float)x2[i0 + TW + 1 + lane];
                ea = MODE == 0 ? (float)apre(a + i0 + TW + lane) : nap(a + i0 + TW + lane);
                ed = MODE == 0 ? (float)dsuf(i0 - a - 1 - lane) : nds(i0 - a - 1 - lane);
            }
            ulel = x > 0 ? ws.ule[(tile - 1) * TH + lane] : 0.f;
            urer = x < NX - 1 ? ws.ure[(tile + 1) * TH + lane] : 0.f;
        }
    }
    const float Ct = (float)C;
    const float invCf = (float)invC;
    const float scale = (float)inv_s, invs2f = (float)inv_s2;
    constexpr float one = diff ? 0.f : 1.f;
    float V[CPL], UL[CPL], UR[CPL];
#pragma unroll
    for (int e = 0; e < CPL; ++e) V[e] = UL[e] = UR[e] = 0.f;
    float exc = 0.f;
    // the field's excursion max(0, -min, max - 1) (mapping.py:198-203) tracked as two
    // running maxima, max(-gx, -gy) and max(gx, gy); max(g) - 1 == max(g - 1) exactly
    float excHi = -1.f;
    // per-column geometry of the field (hoisted out of the row sweep)
    float colx[CPL], colip1[CPL];
    uint32_t upcnt[CPL];  // flat wedge_up count of (i, a + r), advanced row by row
#pragma unroll
    for (int e = 0; e < CPL; ++e) {
        const int i = i0 + u0 + e;
        colx[e] = (float)i * scale;
        colip1[e] = (float)(i + 1) * scale;
        upcnt[e] = diff ? flat_up_count(i, s - 1 - i, a, 2 * a + 1) : 0u;
    }
    // MODE 1 with an explicit defect: the row's values are fetched one row ahead so their
    // latency hides behind the previous row's work.
    const float2* defrow = (MODE == 2 && act)
                               ? reinterpret_cast<const float2*>(out.defect) + (int64_t)a * s + i0 + u0
                               : nullptr;
    float2 dnext[CPL];
    if (defrow) {
#pragma unroll
        for (int e = 0; e < CPL; ++e) dnext[e] = __ldg(defrow + e);
    }
    // GSRC: a ring of PF rows in flight per lane, refilled as rows retire; the tables
    // pass with two columns per lane (16-row tiles) requests the whole tile up front.  The
    // field pass keeps a two-row ring there too: its fully unrolled 16-row sweep was 4k
    // instructions of code per warp, fetched anew in every iteration of a graph replay
    // (C2 44.4 -> 43.4 us per iteration with the ring)
    constexpr int PF = GSRC ? (CPL <= 2 && MODE == 0 ? 16 : 2) : 1;
    float ring[PF][CPL];
    if (GSRC) {
#pragma unroll
        for (int q = 0; q < PF; ++q) {
#pragma unroll
            for (int e = 0; e < CPL; ++e) ring[q][e] = 0.f;
            if (act && q < TH) load_row_g<CPL>(src + (size_t)q * ld + u0, ring[q]);
        }
    }
    // one row of the sweep; GSRC: `cb` holds row r and is refilled with row r + PF
    auto step = [&](const int r, float (&cb)[CPL]) {
        float2 dcur[CPL];
        if (defrow) {
#pragma unroll
            for (int e = 0; e < CPL; ++e) dcur[e] = dnext[e];
            if (r + 1 < TH) {
#pragma unroll
                for (int e = 0; e < CPL; ++e) dnext[e] = __ldg(defrow + (int64_t)(r + 1) * s + e);
            }
        }
        float dv[CPL];
        if (GSRC) {
#pragma unroll
            for (int e = 0; e < CPL; ++e) dv[e] = cb[e];
            if (act && r + PF < TH) load_row_g<CPL>(src + (size_t)(r + PF) * ld + u0, cb);
        } else if (act) {
            load_row<CPL>(src + (size_t)r * ld + u0, dv);
        } else {
#pragma unroll
            for (int e = 0; e < CPL; ++e) dv[e] = 0.f;
        }
#pragma unroll
        for (int e = 0; e < CPL; ++e) V[e] += dv[e];
        // band chains with the neighbouring tiles' edge chains injected at the tile edges
        float fromL = __shfl_up_sync(kFull, UL[CPL - 1], 1);
        float fromR = __shfl_down_sync(kFull, UR[0], 1);
        const float injL = __shfl_sync(kFull, ulel, r > 0 ? r - 1 : 0);
        const float injR = __shfl_sync(kFull, urer, r > 0 ? r - 1 : 0);
        if (lane == 0) fromL = r > 0 ? injL : 0.f;
        if (lane >= last) fromR = r > 0 ? injR : 0.f;
#pragma unroll
        for (int e = CPL - 1; e > 0; --e) UL[e] = V[e] + UL[e - 1];
        UL[0] = V[0] + fromL;
#pragma unroll
        for (int e = 0; e < CPL - 1; ++e) UR[e] = V[e] + UR[e + 1];
        UR[CPL - 1] = V[CPL - 1] + fromR;
        // in-tile row prefix of V
        float loc[CPL];
        loc[0] = V[0];
#pragma unroll
        for (int e = 1; e < CPL; ++e) loc[e] = loc[e - 1] + V[e];
        const float inc = warp_inclusive_scan(loc[CPL - 1], lane);
        const float off = inc - loc[CPL - 1];
        const float Pr = __shfl_sync(kFull, P, r);
        const float Qr = __shfl_sync(kFull, Q, r);
        if (MODE == 0) {
            const float Sr = __shfl_sync(kFull, S, r);
            float o[8][CPL];
#pragma unroll
            for (int e = 0; e < CPL; ++e) {
                const float L = off + loc[e];
                const float Tt = UL[e] + UR[e] - V[e];
                const float up = Tt + (w1[e] + w2[e]);
                o[0][e] = (A[e] + Pr) + L;            // rect_tl
                o[1][e] = Bc[e] - (Pr + L);           // rect_bl
                o[2][e] = (Sr - Bc[e]) + L;           // rect_br
                o[3][e] = Qr - (A[e] + L);            // rect_tr
                o[4][e] = up;                         // wedge_up
                o[5][e] = wa[e] - up;                 // wedge_left
                o[6][e] = ((Ct - wa[e]) - wd[e]) + up;  // wedge_down
                o[7][e] = wd[e] - up;                 // wedge_right
            }
            if (act) {
                const int64_t q = (int64_t)(a + r) * s + i0 + u0;
#pragma unroll
                for (int t = 0; t < 8; ++t) store_row_cs<CPL>(out.tables8 + (int64_t)t * g.m + q, o[t]);
            }
        } else {
            const int j = a + r;
            const float yy = j * scale, fj = (j + 1) * scale;
            // halved coefficients (see nap): a1 = (1 - 2y) / 2, b1 = (2x - 1) / 2, Qr = Rp / 2,
            // cp = Cp / 2, ap / ds = Apre / 2, Dsuf / 2; the x and y terms then read
            //   gx = tl a1 + up b1 + cp u + (omq - cp) ulx + Q hp + (1 + one/2 - ap - ds) x + ap
            //   gy = -tl b1 + up a1 + cp hp + (omq - cp) uly + Q u + (ap + ds) y + y
            // with ulx - uly = x - y and u + hp = x + y (anchors, mapping.py:42-47).
            const float a1 = 0.5f - yy, omq = 0.5f * one - Qr;
            constexpr float kx = 1.f + 0.5f * one;
            const uint32_t jp1 = (uint32_t)(j + 1);
            float res[2 * CPL];
#pragma unroll
            for (int e = 0; e < CPL; ++e) {
                const float xx = colx[e], b1 = xx - 0.5f;
                const float tl = (A[e] + Pr) + (off + loc[e]);
                const float up = (UL[e] + UR[e] - V[e]) + (w1[e] + w2[e]);
                float tln, upn;
                if (diff) {
                    tln = fmaf(tl, invCf, -colip1[e] * fj);
                    upn = fmaf(up, invCf, -(float)upcnt[e] * invs2f);
                    // count(i, j + 1) - count(i, j) = 1 + min(j + 1, i) + min(j + 1, s - 1 - i)
                    const uint32_t i = (uint32_t)(i0 + u0 + e);
                    upcnt[e] += 1u + min(jp1, i) + min(jp1, (uint32_t)(s - 1) - i);
                } else {
                    tln = tl * invCf;
                    upn = up * invCf;
                }
                const float cp = Bc[e], ap = wa[e], sad = ap + wd[e];
                // anchors without branches: x + y and x - y are exact, and so are
                // uly = ulx - (x - y) and hp = (x + y) - u
                const float dxy = xx - yy, sxy = xx + yy;
                const float ulx = fmaxf(dxy, 0.f), uly = ulx - dxy;
                const float u = fminf(sxy, 1.f), hp = sxy - u;  // urx = dly, ury = dlx
                const float m = omq - cp;
                float gx = fmaf(tln, a1, fmaf(upn, b1, fmaf(cp, u, fmaf(m, ulx, fmaf(Qr, hp, fmaf(kx - sad, xx, ap))))));
                float gy = fmaf(tln, -b1, fmaf(upn, a1, fmaf(cp, hp, fmaf(m, uly, fmaf(Qr, u, fmaf(sad, yy, yy))))));
                if (MODE == 2) {
                    gx -= dcur[e].x;
                    gy -= dcur[e].y;
                }
                if (act) {
                    exc = fmax3f(exc, -gx, -gy);
                    excHi = fmax3f(excHi, gx, gy);
                }
                res[2 * e] = __saturatef(gx);
                res[2 * e + 1] = __saturatef(gy);
            }
            if (out.pairs) {
                // paired layout for the move: slot i holds (t(i), t(i + 1)), so the
                // bilinear footprint is two 16-byte loads.  The half that belongs to
                // the next tile's first column is written by that tile's warp.
                const float nx = __shfl_down_sync(kFull, res[0], 1), ny = __shfl_down_sync(kFull, res[1], 1);
                if (act) {
                    float4* pd = reinterpret_cast<float4*>(out.pairs) + ((int64_t)j * s + i0 + u0);
#pragma unroll
                    for (int e = 0; e < CPL - 1; ++e)
                        pd[e] = make_float4(res[2 * e], res[2 * e + 1], res[2 * e + 2], res[2 * e + 3]);
                    if (lane < last) pd[CPL - 1] = make_float4(res[2 * CPL - 2], res[2 * CPL - 1], nx, ny);
                    else reinterpret_cast<float2*>(pd + CPL - 1)[0] = make_float2(res[2 * CPL - 2], res[2 * CPL - 1]);
                    if (lane == 0 && i0 > 0) reinterpret_cast<float2*>(pd - 1)[1] = make_float2(res[0], res[1]);
                }
            }
            if (act && out.targets) {  // default cache policy: the move gathers from it next
                float* dst = out.targets + 2 * ((int64_t)j * s + i0 + u0);
                if constexpr (CPL == 4) {
                    reinterpret_cast<float4*>(dst)[0] = make_float4(res[0], res[1], res[2], res[3]);
                    reinterpret_cast<float4*>(dst)[1] = make_float4(res[4], res[5], res[6], res[7]);
                } else if constexpr (CPL == 2) {
                    reinterpret_cast<float4*>(dst)[0] = make_float4(res[0], res[1], res[2], res[3]);
                } else {
                    reinterpret_cast<float2*>(dst)[0] = make_float2(res[0], res[1]);
                }
            }
        }
        // advance the diagonal windows to row r + 1
        slide_left<CPL>(w1, e1, r, lane);
        slide_left<CPL>(wd, ed, r, lane);
        slide_right<CPL>(w2, e2, r, lane, last);
        slide_right<CPL>(wa, ea, r, lane, last);
    };
    for (int r0 = 0; r0 < TH; r0 += PF) {  // PF rows per trip: the ring slot is a compile-time index
#pragma unroll
        for (int q = 0; q < PF; ++q)
            if (r0 + q < TH) step(r0 + q, ring[q]);
    }
    if (MODE != 0) {
        exc = fmaxf(exc, excHi - 1.f);
        exc = warp_max(exc);
        if (lane == 0 && exc > 0.f) atomic_max_nonneg(out.max_exc, exc);
    }
}

}  // namespace inim
