// Carry scan (phase 2 of the integral pass) as per-item device functions, shared by
// the standalone scan launches (scan.cu) and the persistent iteration kernel (mega.cu).
// Every function is called by a whole CTA (blockDim a multiple of 32, <= 1024) for one
// work item and may contain CTA-wide barriers.
//
//   lines   item = band b: for each row j of the band the exclusive prefix over tiles
//           of the row sums (HC[j][x]) and the in-band prefix of the row totals; for the
//           band the exclusive prefix over tiles of the tile totals (tilepre) and the
//           band total.
//   chains  item = 32 consecutive chains of one kind x NY band chunks.  With the
//           band-local row prefix of the column sums  batl_b[c] = tilepre_b[c/TW] +
//           inpre_b[c]  every carry is a plain scan over the bands of band-local terms:
//             TL: TLcar_{b+1}[c] = TLcar_b[c] + batl_b[c]
//             X1: X1_{b+1}[c]    = X1_b[c-TH] + ULbot2_b[c] - batl_b[c]
//             X2: X2_{b+1}[c]    = X2_b[c+TH] + URbot2_b[c] + batl_b[c-1],
//                 X2_b[c >= s]   = TLcar_b[s-1]  (injected where a chain enters the grid)
//           where X1 = ULcar - TLcar and X2 = URcar + TLcar[c-1] are the write pass's
//           diagonal carries and ULbot2 / URbot2 complete the band-bottom chains with
//           the neighbouring tiles' edge chains.  Substituting TLcar_{b+1} = TLcar_b +
//           batl_b into the ULcar / URcar recurrences gives the X1 / X2 forms, so the
//           three scans are independent of each other.
//   marg    Rpre (TLcar_b[s-1] + in-band prefix), C, and the diagonal marginals:
//             Dsuf[d>=0] = ULE + TLcar_b[s-1] + X1_b[s-2-r]   (row j = s-1-d = bTH + r)
//             Dsuf[d<0]  = X1_B[s-1+d] + C
//             Apre[q<s]  = URE + X2_b[r+1]                     (row q = bTH + r)
//             Apre[q>=s] = X2_B[q-s+1]
// tests/tile_model.py restates the algebra in numpy against the oracle.  Every sum has
// a fixed order (deterministic).
#pragma once

#include "inim_internal.cuh"

namespace inim {

constexpr int kMaxBands = 1024;  // s / TH: 16384 / 16 (k = 14) and 32768 / 32 (k = 15)

// Block-wide exclusive scan of one double per thread.  *total receives the block total.
__device__ __forceinline__ double block_excl_scan(double v, double* sh /* 33 */, double* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const double inc = warp_inclusive_scan_d(v, lane);
    if (lane == 31) sh[w] = inc;
    __syncthreads();
    if (w == 0) {
        const double t = lane < nw ? sh[lane] : 0.0;
        const double ti = warp_inclusive_scan_d(t, lane);
        sh[lane] = ti - t;
        if (lane == 31) sh[32] = ti;
    }
    __syncthreads();
    const double r = sh[w] + inc - v;
    *total = sh[32];
    __syncthreads();
    return r;
}

// Exclusive prefix of the band totals into shared memory bp[0..B] (whole CTA).
__device__ __forceinline__ void band_prefix(const Geo& g, const Ws& ws, double* bp, double* sh /* 33 */) {
    const int B = g.B;
    double carry = 0.0;
    for (int base = 0; base < B; base += blockDim.x) {
        const int q = base + threadIdx.x;
        const double v = q < B ? ws.btot[q] : 0.0;
        double tot;
        const double ex = block_excl_scan(v, sh, &tot);
        if (q < B) bp[q] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) bp[B] = carry;
    __syncthreads();
}

__host__ __device__ inline int chain_groups_tl(const Geo& g) { return (g.s + 31) / 32; }
__host__ __device__ inline int chain_groups_x(const Geo& g) { return (g.s + g.B * g.TH + 31) / 32; }
__host__ __device__ inline int chains_items(const Geo& g) { return chain_groups_tl(g) + 2 * chain_groups_x(g); }
__host__ __device__ inline int chain_kind(const Geo& g, int item) {
    const int ntl = chain_groups_tl(g);
    return item < ntl ? 0 : (item < ntl + chain_groups_x(g) ? 1 : 2);
}
// band chunks per chain (warps per CTA): short serial chunks on small grids
__host__ __device__ inline int chain_warps(const Geo& g, int per = 4) {
    const int ny = g.B / per;
    return ny < 1 ? 1 : (ny > 16 ? 16 : ny);
}

// One chain: columns TL c = kk; X1 c_b = kk - (B - b) TH (moves right); X2 c_b = kk - b TH
// (moves left).  Its step terms are non-zero exactly for bands b in [lo, hi) (the
// column c_{b+1} is inside the grid) and its values are stored for b in [lo, hi].
template <int KIND>
struct Chain {
    const Geo& g;
    const Ws& ws;
    const double* bp;
    int kk, lo, hi;
    __device__ __forceinline__ Chain(const Geo& g_, const Ws& ws_, const double* bp_, int kk_)
        : g(g_), ws(ws_), bp(bp_), kk(kk_) {
        const int s = g.s, B = g.B, TH = g.TH;
        if (KIND == 0) {
            lo = 0;
            hi = B;
        } else if (KIND == 1) {  // col(b) in [0, s) for b in [e0, e1]
            const int kap = kk - B * TH;
            const int e0 = kap >= 0 ? 0 : (-kap + TH - 1) / TH;
            const int e1 = s - 1 - kap < 0 ? -1 : min(B, (s - 1 - kap) / TH);
            lo = max(0, e0 - 1);
            hi = e1;
        } else {  // col(b) in [0, s) for b in [f0, f1]; entry step / border store at f0 - 1
            const int f0 = kk <= s - 1 ? 0 : (kk - s + TH) / TH;
            const int f1 = min(B, kk / TH);
            lo = max(0, f0 - 1);
            hi = f1;
        }
    }
    __device__ __forceinline__ int col(int b) const {
        return KIND == 0 ? kk : (KIND == 1 ? kk - (g.B - b) * g.TH : kk - b * g.TH);
    }
    // step b -> b + 1, b in [lo, hi): the column col(b + 1) is inside the grid.  BP = false
    // leaves out the X2 border injection (added later by border_term once bp is ready).
    template <bool BP = true>
    __device__ __forceinline__ double term(int b) const {
        // The in-tile aggregates (inpre, ulbot, urbot, ule, ure: sums over at most one
        // TH x TW tile) are combined in float32 and converted once; only the tile prefix
        // tilepre (a band-wide sum) is added in float64.  Indices stay below B * s <= 2^24.
        const int s = g.s, TH = g.TH, TW = g.TW, NX = g.NX, tl = g.twlog;
        const double* __restrict__ tilepre = ws.tilepre;
        const float* __restrict__ inpre = ws.inpre;
        if (KIND == 0) {
            const int q = b * s + kk;
            return tilepre[b * NX + (kk >> tl)] + (double)__ldg(inpre + q);
        }
        const int c = col(b + 1);
        const int x = c >> tl, u = c & (TW - 1);
        const int q = b * s + c;
        if (KIND == 1) {
            float f = __ldg(ws.ulbot + q) - __ldg(inpre + q);
            const int rr = TH - 2 - u;  // row where the chain leaves the tile on the left
            if (rr >= 0 && x > 0) f += __ldg(ws.ule + ((b * NX + x - 1) * TH + rr));
            return (double)f - tilepre[b * NX + x];
        }
        float f = __ldg(ws.urbot + q);
        double t = 0.0;
        if (c > 0) {
            f += __ldg(inpre + q - 1);
            t = tilepre[b * NX + ((c - 1) >> tl)];
        }
        const int rq = TH - 1 - (TW - u);
        if (rq >= 0 && x < NX - 1) f += __ldg(ws.ure + ((b * NX + x + 1) * TH + rq));
        double v = (double)f + t;
        if (BP && c + TH >= s) v += bp[b];  // the chain enters the grid: X2_b beyond the border
        return v;
    }
    __device__ __forceinline__ double border_term(int b) const {  // KIND 2: the BP part of term(b)
        return col(b + 1) + g.TH >= g.s ? bp[b] : 0.0;
    }
    __device__ __forceinline__ void emit(int b, double run) const {
        const int s = g.s, TH = g.TH;
        const int c = col(b);
        if (KIND == 0) {
            ws.tlcar[(int64_t)b * s + c] = (float)run;
        } else if (KIND == 1) {
            if (c >= 0) ws.x1[(int64_t)b * s + c] = (float)run;
        } else {
            ws.x2[(int64_t)b * (s + TH) + c] = (float)(c < s ? run : bp[b]);  // c < s + TH always
        }
    }
};

// 32 chains (lanes) x NY chunks of each chain's band range (warps); two passes: chunk
// sums, then the scan with stores.
template <int KIND>
__device__ __forceinline__ void chains_body(const Geo& g, const Ws& ws, int kk, double (*part)[33], const double* bp) {
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, NY = blockDim.x >> 5;
    const bool live = kk < (KIND == 0 ? g.s : g.s + g.B * g.TH);
    const Chain<KIND> T(g, ws, bp, kk);
    const int len = live && T.hi >= T.lo ? T.hi - T.lo + 1 : 0;  // bands lo..hi
    const int CH = (len + NY - 1) / NY;
    const int b0 = T.lo + min(len, ty * CH), b1 = T.lo + min(len, ty * CH + CH);  // [b0, b1)
    const int tb1 = min(b1, T.hi);  // step terms for b < hi
#ifndef INIM_CHAIN_U
#define INIM_CHAIN_U 2  // measured: 2 beats 4 (+0.9% on the 16384^2 integral sweep) and 8
#endif
    constexpr int U = INIM_CHAIN_U;  // terms in flight per thread
    double loc = 0.0;
    {
        int b = b0;
        for (; b + U <= tb1; b += U) {
            double t[U];
#pragma unroll
            for (int q = 0; q < U; ++q) t[q] = T.term(b + q);
#pragma unroll
            for (int q = 0; q < U; ++q) loc += t[q];
        }
        for (; b < tb1; ++b) loc += T.term(b);
    }
    part[ty][tx] = loc;
    __syncthreads();
    double run = 0.0;
    for (int q = 0; q < ty; ++q) run += part[q][tx];
    __syncthreads();  // `part` is reused by the caller's next item
    int b = b0;
    for (; b + U <= tb1; b += U) {
        double t[U];
#pragma unroll
        for (int q = 0; q < U; ++q) t[q] = T.term(b + q);
#pragma unroll
        for (int q = 0; q < U; ++q) {
            T.emit(b + q, run);
            run += t[q];
        }
    }
    for (; b < b1; ++b) {
        T.emit(b, run);
        if (b < T.hi) run += T.term(b);
    }
}

// Single-read variant (the standalone chains kernel): the band range of each chain's
// step terms is split into NY chunks of at most MAXCH terms; each thread loads its
// chunk's terms once into registers (all loads in flight together, issued before the
// X2 items' band prefix so its latency overlaps them), then scans them.  X2 items
// compute the band prefix into bp here; `publish` stores it and the total.
template <int KIND, int MAXCH>
__device__ __forceinline__ void chains_body_reg(const Geo& g, const Ws& ws, int kk, double (*part)[33], double* bp,
                                                double* sh, bool publish) {
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, NY = blockDim.x >> 5;
    const bool live = kk < (KIND == 0 ? g.s : g.s + g.B * g.TH);
    const Chain<KIND> T(g, ws, bp, kk);
    const int nt = live && T.hi > T.lo ? T.hi - T.lo : 0;  // step terms b in [lo, hi)
    const int CH = (g.B + NY - 1) / NY;                    // <= MAXCH (host dispatch)
    const int b0 = T.lo + min(nt, ty * CH), b1 = T.lo + min(nt, ty * CH + CH);
    double t[MAXCH];
#pragma unroll
    for (int q = 0; q < MAXCH; ++q) t[q] = b0 + q < b1 ? T.template term<false>(b0 + q) : 0.0;
    if (KIND == 2) {
        band_prefix(g, ws, bp, sh);
        if (publish) {
            for (int q = threadIdx.x; q <= g.B; q += blockDim.x) ws.bandpre[q] = bp[q];
            if (threadIdx.x == 0) *ws.total = bp[g.B];
        }
#pragma unroll
        for (int q = 0; q < MAXCH; ++q)
            if (b0 + q < b1) t[q] += T.border_term(b0 + q);
    }
    double loc = 0.0;
#pragma unroll
    for (int q = 0; q < MAXCH; ++q) loc += t[q];
    part[ty][tx] = loc;
    __syncthreads();
    double run = 0.0;
    for (int q = 0; q < ty; ++q) run += part[q][tx];
#pragma unroll
    for (int q = 0; q < MAXCH; ++q) {
        if (b0 + q < b1) {
            T.emit(b0 + q, run);
            run += t[q];
        }
    }
    // the value after the last step (band hi) belongs to the chunk holding the last term
    if (live && T.hi >= T.lo && ((nt > 0 && b0 < b1 && b1 == T.hi) || (nt == 0 && ty == 0))) T.emit(T.hi, run);
}

template <int MAXCH>
__device__ __forceinline__ void chains_item_reg(const Geo& g, const Ws& ws, int item, double (*part)[33], double* bp,
                                                double* sh) {
    const int tx = threadIdx.x & 31;
    const int ntl = chain_groups_tl(g), nxg = chain_groups_x(g);
    if (item < ntl) chains_body_reg<0, MAXCH>(g, ws, item * 32 + tx, part, bp, sh, false);
    else if (item < ntl + nxg) chains_body_reg<1, MAXCH>(g, ws, (item - ntl) * 32 + tx, part, bp, sh, false);
    else chains_body_reg<2, MAXCH>(g, ws, (item - ntl - nxg) * 32 + tx, part, bp, sh, item == ntl + nxg);
}

// bp: the band prefix (band_prefix) for X2 items, else unused.
__device__ __forceinline__ void chains_item(const Geo& g, const Ws& ws, int item, double (*part)[33],
                                            const double* bp) {
    const int tx = threadIdx.x & 31;
    const int ntl = chain_groups_tl(g), nxg = chain_groups_x(g);
    if (item < ntl) chains_body<0>(g, ws, item * 32 + tx, part, bp);
    else if (item < ntl + nxg) chains_body<1>(g, ws, (item - ntl) * 32 + tx, part, bp);
    else chains_body<2>(g, ws, (item - ntl - nxg) * 32 + tx, part, bp);
}

}  // namespace inim
