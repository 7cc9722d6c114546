// Carry scan launch (phase 2 of the integral pass; the item bodies and their derivation
// are in inim_scan.cuh).  The per-band lines run at the end of the reduce (the warp that
// completes a band) and the marginals are read off the chains by the write pass, so
// phase 2 is one launch over 1/TH of the texture.
#include "inim_scan.cuh"
#include "inim_tiles.cuh"

namespace inim {

// The diagonal marginals the write pass needs (DESIGN.md 4.1 "marg"), one entry per
// chain and read off the chains right after the scan (the CTA's own x1 / x2 stores are
// visible after a barrier): X2 chain kk gives Apre[kk - 1], X1 chain kk gives
// Dsuf[kk - (s - 1)].  Stored raw (the tables, MODE 0), normalised by C with the flat
// texture's value folded in (the field, MODE 1) and normalised only (the field with an
// explicit defect, MODE 2), rows of 2s floats:
//   marg[2 q][sigma] = Apre, marg[2 q + 1][delta + s - 1] = Dsuf,  q = MODE.
template <int KIND>
__device__ __forceinline__ void chain_marginal(const Geo& g, const Ws& ws, int kk, const double* bp) {
    const int s = g.s, TH = g.TH, NX = g.NX, B = g.B;
    const double C = bp[B], invC = 1.0 / C;
    const double inv_s = ldexp(1.0, -g.k), inv_s2 = inv_s * inv_s;
    if (KIND == 2) {  // Apre[sigma]: URE + X2_b[r + 1] (sigma = b TH + r < s), X2_B[sigma - s + 1] (above)
        const int sg = kk - 1;
        if (sg < 0 || sg > 2 * s - 2) return;
        double v;
        if (sg < s) {
            const int bb = sg >> g.thlog, r = sg - bb * TH;
            v = (double)ws.ure[(int64_t)bb * NX * TH + r] + (double)ws.x2[(int64_t)bb * (s + TH) + r + 1];
        } else {
            v = (double)ws.x2[(int64_t)B * (s + TH) + sg - (s - 1)];
        }
        ws.marg[sg] = (float)v;
        ws.marg[4 * s + sg] = (float)(v * invC - (double)flat_apre_count(sg, s) * inv_s2);
        ws.marg[8 * s + sg] = (float)(v * invC);
    } else {  // Dsuf[delta]: ULE + TLcar_b[s - 1] + X1_b[s - 2 - r] (delta >= 0), X1_B[s - 1 + delta] + C
        const int dl = kk - (s - 1);
        if (dl < -(s - 1) || dl > s - 1) return;
        double v;
        if (dl >= 0) {
            const int j = s - 1 - dl, bb = j >> g.thlog, r = j - bb * TH, c2 = s - 2 - r;
            v = (double)ws.ule[((int64_t)bb * NX + NX - 1) * TH + r] + bp[bb] +
                (c2 >= 0 ? (double)ws.x1[(int64_t)bb * s + c2] : 0.0);
        } else {
            v = (double)ws.x1[(int64_t)B * s + s - 1 + dl] + C;
        }
        ws.marg[2 * s + kk] = (float)v;
        ws.marg[6 * s + kk] = (float)(v * invC - (double)flat_dsuf_count(dl, s) * inv_s2);
        ws.marg[10 * s + kk] = (float)(v * invC);
    }
}

// After the chain scan of an X1 / X2 item: the item's marginal entries (needs the band
// prefix bp in shared memory; X2 items built it for their border terms).
__device__ __forceinline__ void chains_marginals(const Geo& g, const Ws& ws, int item, double* bp, double* sh) {
    const int kind = chain_kind(g, item);
    if (kind == 0) return;
    if (kind == 1) band_prefix(g, ws, bp, sh);  // (ends with a barrier)
    else __syncthreads();
    if (threadIdx.x < 32) {
        const int ntl = chain_groups_tl(g), nxg = chain_groups_x(g);
        if (kind == 1) chain_marginal<1>(g, ws, (item - ntl) * 32 + threadIdx.x, bp);
        else chain_marginal<2>(g, ws, (item - ntl - nxg) * 32 + threadIdx.x, bp);
    }
}

// Launch bounds: 40 registers (3 CTAs/SM) measured best for the two-pass chains of
// the large grids (72 registers / 1 CTA per SM cost 4% of the 16384^2
// integral pass; 4 CTAs/SM spill); the marginal tail step alone would lift it to 55.  BATCH: the
// plot offsets of a SPLOM batch (grid.z) are a separate instantiation, so the
// single-plot kernels keep their register budget.
template <bool BATCH>
__global__ void __launch_bounds__(512, BATCH ? 1 : 3) chains_kernel(const Geo g, const Ws ws0, const int* state, int64_t zslab) {
    pdl_enter();
    if (state && state[0]) return;
    const Ws ws = BATCH ? ws_shift(ws0, zslab_off(zslab)) : ws0;
    __shared__ double part[16][33];
    __shared__ double bp[kMaxBands + 1];
    __shared__ double sh[33];
    const int item = blockIdx.x;
    if (chain_kind(g, item) == 2) {
        band_prefix(g, ws, bp, sh);
        if (item == chain_groups_tl(g) + chain_groups_x(g)) {  // first X2 item publishes it
            for (int q = threadIdx.x; q <= g.B; q += blockDim.x) ws.bandpre[q] = bp[q];
            if (threadIdx.x == 0) *ws.total = bp[g.B];
        }
    }
    chains_item(g, ws, item, part, bp);
    chains_marginals(g, ws, item, bp, sh);
}

// Single-read chains: each thread holds its chunk of step terms in registers.
template <int MAXCH, bool BATCH>
__global__ void __launch_bounds__(512) chains_reg_kernel(const Geo g, const Ws ws0, const int* state, int64_t zslab) {
    pdl_enter();
    if (state && state[0]) return;
    const Ws ws = BATCH ? ws_shift(ws0, zslab_off(zslab)) : ws0;
    __shared__ double part[16][33];
    __shared__ double bp[kMaxBands + 1];
    __shared__ double sh[33];
    chains_item_reg<MAXCH>(g, ws, blockIdx.x, part, bp, sh);
    chains_marginals(g, ws, blockIdx.x, bp, sh);
}

// Band lines (one CTA per band, one warp per row): HC[j][x] = exclusive prefix over the
// tiles of row j's tile row sums, rpre = the band's in-band prefix of the row totals,
// tilepre / btot = the exclusive prefix and the total of the band's tile totals.  A
// launch of its own so that no reduce warp has to fence and count its band's arrivals.
__global__ void __launch_bounds__(1024) lines_kernel(const Geo g, const Ws ws0, const int* state, int64_t zslab) {
    pdl_enter();
    if (state && state[0]) return;
    const Ws ws = ws_shift(ws0, zslab_off(zslab));
    __shared__ double rowtot[32];
    const int b = blockIdx.x, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int TH = g.TH, NX = g.NX, a = b * TH;
    {
        const double t = warp_line_prefix(ws.rowsum + (int64_t)(a + w) * NX, ws.hc + (int64_t)(a + w) * NX, NX, lane);
        if (lane == 0) rowtot[w] = t;
    }
    __syncthreads();
    // VH: HC scanned down the band's rows per tile (inclusive), what the write pass adds
    // to every row of a tile (in place; the CTA's own writes above are visible after the
    // barrier)
    for (int x = threadIdx.x; x < NX; x += blockDim.x) {
        double* col = ws.hc + (int64_t)a * NX + x;
        double run = 0.0;
        for (int r = 0; r < TH; ++r) {
            run += __ldcg(col + (int64_t)r * NX);
            col[(int64_t)r * NX] = run;
        }
    }
    if (w == 0) {
        const double v = lane < TH ? rowtot[lane] : 0.0;
        const double inc = warp_inclusive_scan_d(v, lane);
        if (lane < TH) ws.rpre[a + lane] = inc;
    }
    if (w == (TH > 1 ? 1 : 0)) {
        const double bt = warp_line_prefix(ws.tiletot + (int64_t)b * NX, ws.tilepre + (int64_t)b * NX, NX, lane);
        if (lane == 0) ws.btot[b] = bt;
    }
}

int launch_carry_scan_state(const Geo& g, const Ws& ws, const int* state, cudaStream_t st, const Bat& bt) {
    INIM_CUDA_TRY(launch_pdl(lines_kernel, dim3(g.B, 1, bt.B), dim3(32 * g.TH), 0, st, g, ws, state, bt.slab));
    prof_mark(st, "lines");
    const int ny = chain_warps(g), ch = (g.B + ny - 1) / ny;
    const dim3 grid(chains_items(g), 1, bt.B), block(32 * ny);
    // register-held chunks pay off only while they are short (measured: 1024^2 +7% on
    // the integral sweep; 4096^2 +-0; 8192^2 and up -10%, occupancy); longer chunks run
    // the two-pass kernel
    const bool batch = bt.B > 1;
    if (ch <= 4) {
        INIM_CUDA_TRY(launch_pdl(batch ? chains_reg_kernel<4, true> : chains_reg_kernel<4, false>, grid, block, 0, st,
                                 g, ws, state, bt.slab));
    } else {
        INIM_CUDA_TRY(launch_pdl(batch ? chains_kernel<true> : chains_kernel<false>, grid, block, 0, st, g, ws, state,
                                 bt.slab));
    }
    prof_mark(st, "chains");
    return (int)cudaGetLastError();
}

}  // namespace inim
