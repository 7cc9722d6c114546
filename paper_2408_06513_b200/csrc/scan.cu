// Carry scan (phase 2 of the integral pass): float64 recurrences over the per-tile
// aggregates, 1/TH of the texture's size.  Four launches, none of which waits on
// another CTA:
//   band_rows  per band: inclusive row prefix of the column sums (BATL) and completion
//              of the band-bottom chains with the neighbouring tiles' edge chains
//   colscan    per column: TLcar_b[c] = sum_{b'<b} BATL[b'][c] (rect_tl above each band);
//              per row: the row carries HC and the row totals
//   diagscan   per diagonal chain through the bands (slope TH columns per band):
//                ULcar_{b+1}[c] = G_b[c] + ULcar_b[c-TH],
//                  G_b[c] = ULbot_b[c] + TLcar_b[c] - TLcar_b[c-TH]
//                URcar_{b+1}[c] = H_b[c] + URcar_b[c+TH],
//                  H_b[c] = URbot_b[c] + TLcar_b[min(c+TH-1,s-1)] - TLcar_b[c-1]
//              i.e. prefix sums of G / H along sheared columns; stored as
//              X1 = ULcar - TLcar, X2 = URcar + TLcar[c-1]; the virtual band b = B gives
//              the chains along the last row (ULrow, URrow)
//   marg       prefix of the row totals (C), then the diagonal-suffix and
//              anti-diagonal-prefix marginals read directly off the chains:
//                Dsuf[d>=0] = UL[s-1-d][s-1],  Dsuf[d<0] = UL[s-1][s-1+d] + C - Cpre[s-1+d]
//                Apre[q<s]  = UR[q][0],        Apre[q>=s] = UR[s-1][q-s+1] + Cpre[q-s]
// The band-axis scans are 2-D block scans: 32 columns (or chains) x 32 band chunks per
// CTA, chunk sums scanned with one warp shuffle scan, so the dependent chain is
// B/32 + 5 steps instead of B.  Every sum has a fixed order (deterministic).
#include "inim_internal.cuh"

namespace inim {

// Block-wide exclusive scan of one double per thread (blockDim.x multiple of 32,
// <= 1024).  Returns the exclusive prefix; *total receives the block total.
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

// Inclusive prefix of a float/double row of n elements into dst, 4 elements per
// thread per tile.
template <typename T>
__device__ void row_prefix(const T* __restrict__ src, double* __restrict__ dst, int n, double* sh) {
    const int per = 4;
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

__global__ void __launch_bounds__(1024) band_rows_kernel(const Geo g, const Ws ws, const int* state) {
    if (state && state[0]) return;
    __shared__ double sh[33];
    const int b = blockIdx.x, s = g.s, TH = g.TH, TW = g.TW, NX = g.NX;
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

// Exclusive scan over ty (the band-chunk index) of part[ty][tx] for each tx, in place.
__device__ __forceinline__ void chunk_scan_32x32(double (*part)[33]) {
    __syncthreads();
    const int tx = threadIdx.x, ty = threadIdx.y;
    // warp ty scans column tx' = ty over lanes = chunks
    const double v = part[tx][ty];
    const double inc = warp_inclusive_scan_d(v, tx);
    __syncthreads();
    part[tx][ty] = inc - v;
    __syncthreads();
}

// blockDim (32, 32).  Blocks [0, ceil(s/32)): TLcar for 32 columns.  Blocks beyond:
// 32 rows each (one warp per row): HC and row totals.
__global__ void __launch_bounds__(1024) colscan_kernel(const Geo g, const Ws ws, const int* state) {
    if (state && state[0]) return;
    __shared__ double part[32][33];
    const int s = g.s, B = g.B, NX = g.NX;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int ncb = (s + 31) / 32;
    if ((int)blockIdx.x < ncb) {
        const int c = blockIdx.x * 32 + tx;
        const int CH = (B + 31) / 32;
        const int b0 = ty * CH, b1 = min(B, b0 + CH);
        const double* __restrict__ batl = ws.batl;
        double loc = 0.0;
        if (c < s)
            for (int b = b0; b < b1; ++b) loc += batl[(int64_t)b * s + c];
        part[ty][tx] = loc;
        chunk_scan_32x32(part);
        if (c < s) {
            double run = part[ty][tx];
            double* __restrict__ tl = ws.tlcar;
            for (int b = b0; b < b1; ++b) {
                tl[(int64_t)b * s + c] = run;
                run += batl[(int64_t)b * s + c];
            }
            if (b1 == B && b0 < b1) tl[(int64_t)B * s + c] = run;
            if (B == 0 && ty == 0) tl[c] = 0.0;
        }
        return;
    }
    // rows: HC[j][x] = exclusive prefix over x of rowsum[j][x]; row total -> rpre[j]
    const int j = (blockIdx.x - ncb) * 32 + ty;
    if (j >= s) return;
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

// blockDim (32, 32); blockIdx.y = 0: up-left chains, 1: up-right chains, 2: X2 border.
// Chain kappa: UL positions (b, kappa + b*TH), UR positions (b, kappa - b*TH).
__global__ void __launch_bounds__(1024) diagscan_kernel(const Geo g, const Ws ws, const int* state) {
    if (state && state[0]) return;
    __shared__ double part[32][33];
    const int s = g.s, B = g.B, TH = g.TH;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const double* __restrict__ TLc = ws.tlcar;
    auto TL = [&](int b, int c) -> double { return c >= 0 ? TLc[(int64_t)b * s + c] : 0.0; };
    if (blockIdx.y == 2) {  // X2 beyond the right border: TLcar_b[s-1]
        const int q = (blockIdx.x * 32 + ty) * 32 + tx;
        if (q < B * TH) {
            const int b = q / TH, e = q % TH;
            ws.x2[(int64_t)b * (s + TH) + s + e] = TL(b, s - 1);
        }
        return;
    }
    const bool up_left = blockIdx.y == 0;
    const int nk = s + B * TH;
    const int kk = blockIdx.x * 32 + tx;  // chain index
    const int CH = (B + 31) / 32;
    const int b0 = ty * CH, b1 = min(B, b0 + CH);
    // UL: kappa = kk - B*TH in [-B*TH, s); step term g_b = G_b[kappa + (b+1) TH]
    // UR: kappa = kk in [0, s + B*TH);       step term h_b = H_b[kappa - (b+1) TH]
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
    chunk_scan_32x32(part);
    if (kk >= nk) return;
    double run = part[ty][tx];  // chain value at band b0
    // emit positions b in [b0, b1) and, for the last chunk, b = B
    const int bend = (b1 == B) ? B + 1 : b1;
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

__global__ void __launch_bounds__(1024) marg_kernel(const Geo g, const Ws ws, const int* state) {
    if (state && state[0]) return;
    __shared__ double sh[33];
    const int s = g.s, TH = g.TH, NX = g.NX, B = g.B;
    row_prefix<double>(ws.rpre, ws.rpre, s, sh);
    __syncthreads();
    const double C = ws.rpre[s - 1];
    if (threadIdx.x == 0) *ws.total = C;
    const double* __restrict__ cpre = ws.tlcar + (int64_t)B * s;
    for (int q = threadIdx.x; q < 2 * s - 1; q += blockDim.x) {
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
}

int launch_carry_scan_state(const Geo& g, const Ws& ws, const int* state, cudaStream_t st) {
    band_rows_kernel<<<g.B, 1024, 0, st>>>(g, ws, state);
    prof_mark(st, "band_rows");
    const int ncb = (g.s + 31) / 32;
    colscan_kernel<<<2 * ncb, dim3(32, 32), 0, st>>>(g, ws, state);
    prof_mark(st, "colscan");
    const int nk = g.s + g.B * g.TH;
    diagscan_kernel<<<dim3((nk + 31) / 32, 3), dim3(32, 32), 0, st>>>(g, ws, state);
    prof_mark(st, "diagscan");
    marg_kernel<<<1, 1024, 0, st>>>(g, ws, state);
    prof_mark(st, "marg");
    return (int)cudaGetLastError();
}

}  // namespace inim
