// Carry scan (phase 2 of the integral pass) as per-item device functions, shared by
// the standalone scan launches (scan.cu) and the persistent iteration kernel (mega.cu).
// Every function is called by a whole CTA (blockDim a multiple of 32, <= 1024) for one
// work item and contains CTA-wide barriers.
//
//   band_rows  item = band b: inclusive row prefix of the column sums (BATL) and
//              completion of the band-bottom chains with the neighbouring tiles' edges
//   colscan    item < ceil(s/32): TLcar_b[c] = sum_{b'<b} BATL[b'][c] for 32 columns
//              (32 columns x NY band chunks, chunk sums scanned in shared memory);
//              item >= ceil(s/32): NY rows each (one warp per row): HC and row totals
//   diagscan   the diagonal recurrences as prefix sums along sheared columns:
//                ULcar_{b+1}[c] = G_b[c] + ULcar_b[c-TH],  G_b[c] = ULbot_b[c] + TLcar_b[c] - TLcar_b[c-TH]
//                URcar_{b+1}[c] = H_b[c] + URcar_b[c+TH],  H_b[c] = URbot_b[c] + TLcar_b[min(c+TH-1,s-1)] - TLcar_b[c-1]
//              stored as X1 = ULcar - TLcar, X2 = URcar + TLcar[c-1] (+ border), and the
//              virtual band b = B gives the chains along the last row (ULrow, URrow)
//   marg       Rpre per band (TLcar_b[s-1] + in-band prefix of the row totals),
//              C = TLcar_B[s-1], and the diagonal marginals read off the chains:
//                Dsuf[d>=0] = UL[s-1-d][s-1],  Dsuf[d<0] = UL[s-1][s-1+d] + C - Cpre[s-1+d]
//                Apre[q<s]  = UR[q][0],        Apre[q>=s] = UR[s-1][q-s+1] + Cpre[q-s]
// Every sum has a fixed order (deterministic).
#pragma once

#include "inim_internal.cuh"

namespace inim {

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

// Inclusive prefix of a row of n elements into dst, 4 elements per thread per tile.
template <typename T>
__device__ __forceinline__ void row_prefix(const T* __restrict__ src, double* __restrict__ dst, int n, double* sh) {
    constexpr int per = 4;
    double carry = 0.0;
    for (int base = 0; base < n; base += per * blockDim.x) {
        const int i0 = base + per * threadIdx.x;
        double v[per];
        double loc = 0.0;
#pragma unroll
        for (int e = 0; e < per; ++e) {
            v[e] = i0 + e < n ? (double)src[i0 + e] : 0.0;
            loc += v[e];
        }
        double tot;
        const double off = block_excl_scan(loc, sh, &tot);
        double run = carry + off;
#pragma unroll
        for (int e = 0; e < per; ++e) {
            run += v[e];
            if (i0 + e < n) dst[i0 + e] = run;
        }
        carry += tot;
    }
}

__device__ __forceinline__ void band_rows_item(const Geo& g, const Ws& ws, int b, double* sh) {
    const int s = g.s, TH = g.TH, TW = g.TW, NX = g.NX;
    row_prefix<float>(ws.colsum + (int64_t)b * s, ws.batl + (int64_t)b * s, s, sh);
    const float* __restrict__ ulbot = ws.ulbot + (int64_t)b * s;
    const float* __restrict__ urbot = ws.urbot + (int64_t)b * s;
    const float* __restrict__ ule = ws.ule + (int64_t)b * NX * TH;
    const float* __restrict__ ure = ws.ure + (int64_t)b * NX * TH;
    for (int c = threadIdx.x; c < s; c += blockDim.x) {
        const int x = c / TW, u = c - x * TW;
        double ul = ulbot[c];
        const int rr = TH - 2 - u;  // row where the chain leaves the tile on the left
        if (x > 0 && rr >= 0) ul += ule[(x - 1) * TH + rr];
        double ur = urbot[c];
        const int rq = TH - 1 - (TW - u);
        if (x < NX - 1 && rq >= 0) ur += ure[(x + 1) * TH + rq];
        ws.ulb2[(int64_t)b * s + c] = ul;
        ws.urb2[(int64_t)b * s + c] = ur;
    }
}

// Exclusive prefix over the NY chunk rows of part[ty][tx], per column tx.
__device__ __forceinline__ double chunk_exclusive(double (*part)[33], int tx, int ty) {
    double off = 0.0;
    for (int q = 0; q < ty; ++q) off += part[q][tx];
    return off;
}

__host__ __device__ inline int colscan_items(const Geo& g, int ny) { return (g.s + 31) / 32 + (g.s + ny - 1) / ny; }

__device__ __forceinline__ void colscan_item(const Geo& g, const Ws& ws, int item, double (*part)[33]) {
    const int s = g.s, B = g.B, NX = g.NX;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, NY = blockDim.x >> 5;
    const int ncb = (s + 31) / 32;
    if (item < ncb) {
        const int c = item * 32 + tx;
        const int CH = (B + NY - 1) / NY;
        const int b0 = ty * CH, b1 = min(B, b0 + CH);
        const double* __restrict__ batl = ws.batl;
        double loc = 0.0;
        if (c < s)
            for (int b = b0; b < b1; ++b) loc += batl[(int64_t)b * s + c];
        part[ty][tx] = loc;
        __syncthreads();
        double run = chunk_exclusive(part, tx, ty);
        if (c < s) {
            double* __restrict__ tl = ws.tlcar;
            for (int b = b0; b < b1; ++b) {
                tl[(int64_t)b * s + c] = run;
                run += batl[(int64_t)b * s + c];
            }
            if (b1 == B && b0 < b1) tl[(int64_t)B * s + c] = run;
        }
        __syncthreads();
        return;
    }
    // rows: HC[j][x] = exclusive prefix over x of rowsum[j][x]; row total -> rpre[j]
    const int j = (item - ncb) * NY + ty;
    if (j < s) {
        const float* __restrict__ rs = ws.rowsum + (int64_t)j * NX;
        double* __restrict__ hc = ws.hc + (int64_t)j * NX;
        double carry = 0.0;
        for (int base = 0; base < NX; base += 32) {
            const int x = base + tx;
            const double v = x < NX ? (double)rs[x] : 0.0;
            const double inc = warp_inclusive_scan_d(v, tx);
            if (x < NX) hc[x] = carry + inc - v;
            carry += __shfl_sync(kFull, inc, 31);
        }
        if (tx == 0) ws.rpre[j] = carry;
    }
}

// items: [0, 2*nchunk) chain groups (UL then UR), then ceil(B*TH/blockDim) border items.
__host__ __device__ inline int diagscan_items(const Geo& g, int nthreads) {
    const int nk = g.s + g.B * g.TH;
    return 2 * ((nk + 31) / 32) + (g.B * g.TH + nthreads - 1) / nthreads;
}

__device__ __forceinline__ void diagscan_item(const Geo& g, const Ws& ws, int item, double (*part)[33]) {
    const int s = g.s, B = g.B, TH = g.TH;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, NY = blockDim.x >> 5;
    const double* __restrict__ TLc = ws.tlcar;
    auto TL = [&](int b, int c) -> double { return c >= 0 ? TLc[(int64_t)b * s + c] : 0.0; };
    const int nk = s + B * TH;
    const int ngroups = (nk + 31) / 32;
    if (item >= 2 * ngroups) {  // X2 beyond the right border: TLcar_b[s-1]
        const int q = (item - 2 * ngroups) * blockDim.x + threadIdx.x;
        if (q < B * TH) {
            const int b = q / TH, e = q % TH;
            ws.x2[(int64_t)b * (s + TH) + s + e] = TL(b, s - 1);
        }
        return;
    }
    const bool up_left = item < ngroups;
    const int kk = (up_left ? item : item - ngroups) * 32 + tx;  // chain index
    const int CH = (B + NY - 1) / NY;
    const int b0 = ty * CH, b1 = min(B, b0 + CH);
    // UL: kappa = kk - B*TH in [-B*TH, s); step term G_b[kappa + (b+1) TH]
    // UR: kappa = kk in [0, s + B*TH);       step term H_b[kappa - (b+1) TH]
    const int kappa = up_left ? kk - B * TH : kk;
    auto term = [&](int b) -> double {
        if (kk >= nk) return 0.0;
        if (up_left) {
            const int c = kappa + (b + 1) * TH;
            if (c < 0 || c >= s) return 0.0;
            return ws.ulb2[(int64_t)b * s + c] + TL(b, c) - TL(b, c - TH);
        }
        const int c = kappa - (b + 1) * TH;
        if (c < 0 || c >= s) return 0.0;
        return ws.urb2[(int64_t)b * s + c] + TL(b, min(c + TH - 1, s - 1)) - TL(b, c - 1);
    };
    double loc = 0.0;
    for (int b = b0; b < b1; ++b) loc += term(b);
    part[ty][tx] = loc;
    __syncthreads();
    double run = chunk_exclusive(part, tx, ty);  // chain value at band b0
    __syncthreads();
    if (kk >= nk) return;
    const int bend = (b1 == B) ? B + 1 : b1;  // the last chunk also emits the virtual band B
    for (int b = b0; b < bend; ++b) {
        const int c = up_left ? kappa + b * TH : kappa - b * TH;
        if (c >= 0 && c < s) {
            if (b < B) {
                if (up_left) ws.x1[(int64_t)b * s + c] = run - TL(b, c);
                else ws.x2[(int64_t)b * (s + TH) + c] = run + TL(b, c - 1);
            } else {
                if (up_left) ws.ulrow[c] = run;
                else ws.urrow[c] = run;
            }
        }
        if (b < B) run += term(b);
    }
}

// items: ceil(B / NY) band groups (one warp per band: Rpre), then the 2s-1 marginal
// entries in chunks of blockDim.
__host__ __device__ inline int marg_items(const Geo& g, int nthreads) {
    const int ny = nthreads / 32;
    return (g.B + ny - 1) / ny + (2 * g.s - 1 + nthreads - 1) / nthreads;
}

__device__ __forceinline__ void marg_item(const Geo& g, const Ws& ws, int item) {
    const int s = g.s, TH = g.TH, NX = g.NX, B = g.B;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, NY = blockDim.x >> 5;
    const int nbg = (B + NY - 1) / NY;
    const double* __restrict__ cpre = ws.tlcar + (int64_t)B * s;
    const double C = cpre[s - 1];
    if (item < nbg) {
        const int b = item * NY + w;
        if (b < B) {
            const int a = b * TH;
            const double tot = lane < TH ? ws.rpre[a + lane] : 0.0;  // row totals (colscan)
            const double inc = warp_inclusive_scan_d(tot, lane);
            __syncwarp();
            if (lane < TH) ws.rpre[a + lane] = ws.tlcar[(int64_t)b * s + s - 1] + inc;
        }
        if (item == 0 && threadIdx.x == 0) *ws.total = C;
        return;
    }
    const int q = (item - nbg) * blockDim.x + threadIdx.x;
    if (q >= 2 * s - 1) return;
    const int delta = q - (s - 1);
    double dv;
    if (delta >= 0) {
        const int j = s - 1 - delta, b = j / TH, r = j - b * TH, c2 = s - 2 - r;
        dv = (double)ws.ule[((int64_t)b * NX + NX - 1) * TH + r] + ws.tlcar[(int64_t)b * s + s - 1] +
             (c2 >= 0 ? ws.x1[(int64_t)b * s + c2] : 0.0);
    } else {
        const int c = s - 1 + delta;
        dv = ws.ulrow[c] + C - cpre[c];
    }
    ws.dsuf[q] = dv;
    double av;
    if (q < s) {
        const int b = q / TH, r = q - b * TH;
        av = (double)ws.ure[(int64_t)b * NX * TH + r] + ws.x2[(int64_t)b * (s + TH) + r + 1];
    } else {
        const int i = q - (s - 1);
        av = ws.urrow[i] + cpre[i - 1];
    }
    ws.apre[q] = av;
}

}  // namespace inim
