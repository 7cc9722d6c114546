// Warp-per-tile integral kernels (phase 1 reduce, phase 3 write), shared by the
// standalone integral kernels (integral.cu) and the fused smoothing kernel (smooth.cu).
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
//   colsum[b][c], ulbot[b][c], urbot[b][c] (in-tile chains of the column prefix V at the
//   band's last row), ule/ure[b][x][r] (chains at the tile's last / first column, complete
//   in-band values since TW >= TH), rowsum[j][x].
template <int CPL>
__device__ __forceinline__ void warp_tile_reduce(const float* src, int ld, const Geo g, const Ws ws, int b, int x,
                                                 int lane) {
    const int TH = g.TH, TW = g.TW, s = g.s, NX = g.NX;
    const int last = g.WL - 1;
    const int u0 = lane * CPL;
    const bool act = lane <= last;
    float V[CPL], UL[CPL], UR[CPL];
#pragma unroll
    for (int e = 0; e < CPL; ++e) V[e] = UL[e] = UR[e] = 0.f;
    float ule_mine = 0.f, ure_mine = 0.f, rs_mine = 0.f;
    for (int r = 0; r < TH; ++r) {
        float dv[CPL];
        if (act) load_row<CPL>(src + (size_t)r * ld + u0, dv);
        else {
#pragma unroll
            for (int e = 0; e < CPL; ++e) dv[e] = 0.f;
        }
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
        rsum = warp_sum(rsum);
        const float ulr = __shfl_sync(kFull, UL[CPL - 1], last);
        const float url = __shfl_sync(kFull, UR[0], 0);
        if (lane == r) {
            ule_mine = ulr;
            ure_mine = url;
            rs_mine = rsum;
        }
    }
    const int a = b * TH, i0 = x * TW;
    const int64_t tile = (int64_t)b * NX + x;
    if (act) {
        float* cs = ws.colsum + (int64_t)b * s + i0 + u0;
        float* ub = ws.ulbot + (int64_t)b * s + i0 + u0;
        float* rb = ws.urbot + (int64_t)b * s + i0 + u0;
#pragma unroll
        for (int e = 0; e < CPL; ++e) {
            cs[e] = V[e];
            ub[e] = UL[e];
            rb[e] = UR[e];
        }
    }
    if (lane < TH) {
        ws.ule[tile * TH + lane] = ule_mine;
        ws.ure[tile * TH + lane] = ure_mine;
        ws.rowsum[(int64_t)(a + lane) * NX + x] = rs_mine;
    }
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
    float* targets;       // MODE 1: (s, s, 2)
    const float* defect;  // MODE 1: (s, s, 2) or null (closed form)
    float* max_exc;       // MODE 1
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

// MODE 0: stream the eight tables (float32 assembly from float64-rounded constants).
// MODE 1: deformation field (build_field, mapping.py:194-204) in float64, with the raw
// map in the collapsed form  2C tx = tl(1-2y) + up(2x-1) + Gx,  2C ty = tl(1-2x) +
// up(1-2y) + Gy  (the anchor coefficients of tl and up are constant across the
// mapping.py:42/47 branches; Gx, Gy carry the marginal terms).
template <int CPL, int MODE>
__device__ __forceinline__ void warp_tile_write(const float* src, int ld, const Geo g, const Ws ws, int b, int x,
                                                int lane, const WriteOut out) {
    using T = typename std::conditional<MODE == 0, float, double>::type;
    const int TH = g.TH, TW = g.TW, s = g.s, NX = g.NX, B = g.B;
    const int last = g.WL - 1;
    const int u0 = lane * CPL;
    const bool act = lane <= last;
    const int a = b * TH, i0 = x * TW;
    const int64_t tile = (int64_t)b * NX + x;
    const double C = *ws.total;
    const double* __restrict__ tlc = ws.tlcar + (int64_t)b * s;
    const double* __restrict__ cpre = ws.tlcar + (int64_t)B * s;
    const double* __restrict__ x1 = ws.x1 + (int64_t)b * s;
    const double* __restrict__ x2 = ws.x2 + (int64_t)b * (s + TH);
    const double* __restrict__ apre = ws.apre;
    const double* __restrict__ dsuf = ws.dsuf + (s - 1);  // index by delta = i - j
    // per-column constants and initial windows (row 0)
    T A[CPL], Bc[CPL], w1[CPL], w2[CPL], wa[CPL], wd[CPL];
#pragma unroll
    for (int e = 0; e < CPL; ++e) {
        const int i = i0 + u0 + e;
        const bool ok = act && i < s;
        const double tv = ok ? tlc[i] : 0.0, cv = ok ? cpre[i] : 0.0;
        A[e] = (T)tv;
        Bc[e] = (T)(cv - tv);  // MODE 1 uses Bc = Cp
        if (MODE == 1) Bc[e] = (T)cv;
        w1[e] = (T)(ok && i - 1 >= 0 ? x1[i - 1] : 0.0);  // X1[i - r - 1]
        w2[e] = (T)(ok ? x2[i + 1] : 0.0);                // X2[i + r + 1]
        wa[e] = (T)(ok ? apre[a + i] : 0.0);              // Apre[i + j]
        wd[e] = (T)(ok ? dsuf[i - a] : 0.0);              // Dsuf[i - j]
    }
    // lane-distributed: row constants (lane q = row q) and window / chain edge entries
    T P = 0, Q = 0, S = 0;
    double Rp = 0.0;
    T e1 = 0, e2 = 0, ea = 0, ed = 0;
    float ulel = 0.f, urer = 0.f;
    {
        const double hc = lane < TH ? ws.hc[(int64_t)(a + lane) * NX + x] : 0.0;
        const double vh = warp_inclusive_scan_d(hc, lane);
        if (lane < TH) {
            Rp = ws.rpre[a + lane];
            P = (T)vh;
            Q = (T)(Rp - vh);
            S = (T)(C - Rp + vh);
            if (lane < TH - 1) {  // entry q feeds row q + 1
                const int c1 = i0 - 2 - lane;
                e1 = (T)(c1 >= 0 ? x1[c1] : 0.0);
                e2 = (T)x2[i0 + TW + 1 + lane];
                ea = (T)apre[a + i0 + TW + lane];
                ed = (T)dsuf[i0 - a - 1 - lane];
            }
            ulel = x > 0 ? ws.ule[(tile - 1) * TH + lane] : 0.f;
            urer = x < NX - 1 ? ws.ure[(tile + 1) * TH + lane] : 0.f;
        }
    }
    const T Ct = (T)C;
    const double inv = 0.5 / C;
    const double scale = ldexp(1.0, -g.k);
    float V[CPL], UL[CPL], UR[CPL];
#pragma unroll
    for (int e = 0; e < CPL; ++e) V[e] = UL[e] = UR[e] = 0.f;
    float exc = 0.f;
    // MODE 1 with a precomputed flat response: the row's defect values are fetched one
    // row ahead so their latency hides behind the previous row's work.
    const float2* defrow = (MODE == 1 && out.defect && act)
                               ? reinterpret_cast<const float2*>(out.defect) + (int64_t)a * s + i0 + u0
                               : nullptr;
    float2 dnext[CPL];
    if (defrow) {
#pragma unroll
        for (int e = 0; e < CPL; ++e) dnext[e] = __ldg(defrow + e);
    }
    for (int r = 0; r < TH; ++r) {
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
        if (act) load_row<CPL>(src + (size_t)r * ld + u0, dv);
        else {
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
        const T Pr = __shfl_sync(kFull, P, r);
        if (MODE == 0) {
            const T Qr = __shfl_sync(kFull, Q, r), Sr = __shfl_sync(kFull, S, r);
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
            const double Rr = __shfl_sync(kFull, Rp, r);
            const int j = a + r;
            const double yy = j * scale;
            float res[2 * CPL];
#pragma unroll
            for (int e = 0; e < CPL; ++e) {
                const int i = i0 + u0 + e;
                const double xx = i * scale;
                const double L = (double)(off + loc[e]);
                const double tl = (A[e] + Pr) + L;
                const double up = (double)(UL[e] + UR[e] - V[e]) + (w1[e] + w2[e]);
                const double Cp = Bc[e], Ap = wa[e], Ds = wd[e];
                const bool below = yy < xx, near = xx + yy < 1.0;
                const double ulx = below ? xx - yy : 0.0, uly = below ? 0.0 : yy - xx;
                const double urx = near ? xx + yy : 1.0, ury = near ? 0.0 : xx + yy - 1.0;
                const double dlx = near ? 0.0 : xx + yy - 1.0, dly = near ? xx + yy : 1.0;
                const double Gx = Cp * (urx - ulx) + (C - Rr) * ulx + Rr * dlx + (C - Ap - Ds) * xx + Ap;
                const double Gy = Cp * (ury - uly) + (C - Rr) * uly + Rr * dly + (Ap + Ds) * yy;
                const double tx = (tl * (1.0 - 2.0 * yy) + up * (2.0 * xx - 1.0) + Gx) * inv;
                const double ty = (tl * (1.0 - 2.0 * xx) + up * (1.0 - 2.0 * yy) + Gy) * inv;
                double2 def;
                if (defrow) {
                    def.x = dcur[e].x;
                    def.y = dcur[e].y;
                } else if (out.defect) {
                    const float2 dfv = reinterpret_cast<const float2*>(out.defect)[(int64_t)j * s + i];
                    def.x = dfv.x;
                    def.y = dfv.y;
                } else {
                    def = flat_response_at(i, j, g.k);
                }
                const float gx = (float)(tx - def.x + xx), gy = (float)(ty - def.y + yy);
                if (act) exc = fmaxf(exc, fmaxf(fmaxf(-gx, -gy), fmaxf(gx - 1.f, gy - 1.f)));
                res[2 * e] = fminf(fmaxf(gx, 0.f), 1.f);
                res[2 * e + 1] = fminf(fmaxf(gy, 0.f), 1.f);
            }
            if (act) {
                float* dst = out.targets + 2 * ((int64_t)j * s + i0 + u0);
                if constexpr (CPL == 4) {
                    __stcs(reinterpret_cast<float4*>(dst), make_float4(res[0], res[1], res[2], res[3]));
                    __stcs(reinterpret_cast<float4*>(dst) + 1, make_float4(res[4], res[5], res[6], res[7]));
                } else if constexpr (CPL == 2) {
                    __stcs(reinterpret_cast<float4*>(dst), make_float4(res[0], res[1], res[2], res[3]));
                } else {
                    __stcs(reinterpret_cast<float2*>(dst), make_float2(res[0], res[1]));
                }
            }
        }
        // advance the diagonal windows to row r + 1
        slide_left<CPL>(w1, e1, r, lane);
        slide_left<CPL>(wd, ed, r, lane);
        slide_right<CPL>(w2, e2, r, lane, last);
        slide_right<CPL>(wa, ea, r, lane, last);
    }
    if (MODE == 1) {
        exc = warp_max(exc);
        if (lane == 0 && exc > 0.f) atomic_max_nonneg(out.max_exc, exc);
    }
}

}  // namespace inim
