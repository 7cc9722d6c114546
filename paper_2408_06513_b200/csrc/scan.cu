// Carry scan launch (phase 2 of the integral pass; the item bodies and their derivation
// are in inim_scan.cuh).  The per-band lines run at the end of the reduce (the warp that
// completes a band) and the marginals are read off the chains by the write pass, so
// phase 2 is one launch over 1/TH of the texture.
#include "inim_scan.cuh"
#include "inim_tiles.cuh"

namespace inim {

// Launch bounds: the plain 512-thread bound settles at 40 registers (3 CTAs/SM),
// measured best (an explicit minimum of 1 CTA/SM lets ptxas spend 72
// registers and costs 4% of the 16384^2 integral pass; 4 CTAs/SM spill).  BATCH: the
// plot offsets of a SPLOM batch (grid.z) are a separate instantiation, so the
// single-plot kernels keep their register budget.
template <bool BATCH, int GEO = 0>
__global__ void __launch_bounds__(512) chains_kernel(const Geo g0, const Ws ws0, const int* state, int64_t zslab) {
    pdl_enter();
    if (BATCH) state = zstate(state, zslab);
    if (state && state[0]) return;
    const Geo g = fixed_geo<GEO>(g0);
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
}

// Single-read chains: each thread holds its chunk of step terms in registers.
template <int MAXCH, bool BATCH, int GEO = 0>
__global__ void __launch_bounds__(512) chains_reg_kernel(const Geo g0, const Ws ws0, const int* state, int64_t zslab) {
    pdl_enter();
    if (BATCH) state = zstate(state, zslab);
    if (state && state[0]) return;
    const Geo g = fixed_geo<GEO>(g0);
    const Ws ws = BATCH ? ws_shift(ws0, zslab_off(zslab)) : ws0;
    __shared__ double part[16][33];
    __shared__ double bp[kMaxBands + 1];
    __shared__ double sh[33];
    chains_item_reg<MAXCH>(g, ws, blockIdx.x, part, bp, sh);
}

// Band lines (one CTA per band, one warp per row): HC[j][x] = exclusive prefix over the
// tiles of row j's tile row sums, rpre = the band's in-band prefix of the row totals,
// tilepre / btot = the exclusive prefix and the total of the band's tile totals.  A
// launch of its own so that no reduce warp has to fence and count its band's arrivals.
template <int GEO>
__global__ void __launch_bounds__(1024) lines_kernel(const Geo g0, const Ws ws0, const int* state, int64_t zslab) {
    pdl_enter();
    const Geo g = fixed_geo<GEO>(g0);
    state = zstate(state, zslab);
    if (state && state[0]) return;
    const Ws ws = ws_shift(ws0, zslab_off(zslab));
    __shared__ double rowtot[32];
    const int b = blockIdx.x, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int TH = g.TH, NX = g.NX, a = b * TH;
    if (NX < 32) {
        // 32 / NX rows per warp, one NX-lane segment each (the same adds, in the same
        // order, as warp_line_prefix's full-warp scan, whose upper lanes hold zeros)
        const int row = w * (32 / NX) + lane / NX, x = lane % NX;
        if (row < TH) {
            const double v = (double)__ldcg(ws.rowsum + (int64_t)(a + row) * NX + x);
            double inc = v;
            for (int d = 1; d < NX; d <<= 1) {
                const double t = __shfl_up_sync(kFull, inc, d, NX);
                if (x >= d) inc += t;
            }
            ws.hc[(int64_t)(a + row) * NX + x] = inc - v;
            if (x == NX - 1) rowtot[row] = inc;
        }
    } else {
        const double t = warp_line_prefix(ws.rowsum + (int64_t)(a + w) * NX, ws.hc + (int64_t)(a + w) * NX, NX, lane);
        if (lane == 0) rowtot[w] = t;
    }
    __syncthreads();
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
    // one warp per row, or 32 / NX rows per warp on narrow grids (at least two warps: the
    // band-total scan runs on warp 1)
    int lt = g.NX < 32 ? (g.TH * g.NX + 31) / 32 * 32 : 32 * g.TH;
    if (lt < 64) lt = 64;
    const int gk = geo_kind(g);
    auto lk = gk == 1 ? lines_kernel<1> : (gk == 2 ? lines_kernel<2> : lines_kernel<0>);
    INIM_CUDA_TRY(launch_pdl(lk, dim3(g.B, 1, bt.B), dim3(lt), 0, st, g, ws, state, bt.slab));
    prof_mark(st, "lines");
    const bool batch = bt.B > 1;
    static const int batch_per = [] {  // INIM_CHAIN_PER: step terms per thread in a batch (4 or 8)
        const char* e = getenv("INIM_CHAIN_PER");
        const int v = e ? atoi(e) : 8;
        return v == 16 ? 16 : (v == 4 ? 4 : 8);
    }();
    // one plot: 4 (C2 43.6 vs 45.0 us, C3 307.9 vs 309.3 us with 8); a batch: 8
    const int per = batch ? batch_per : 4;
    const int ny = chain_warps(g, per), ch = (g.B + ny - 1) / ny;
    const dim3 grid(chains_items(g), 1, bt.B), block(32 * ny);
    if (batch && ch > 4 && ch <= 16) {
        auto kern = ch <= 8 ? (gk == 1 ? chains_reg_kernel<8, true, 1> : chains_reg_kernel<8, true>)
                            : chains_reg_kernel<16, true>;
        INIM_CUDA_TRY(launch_pdl(kern, grid, block, 0, st, g, ws, state, bt.slab));
        prof_mark(st, "chains");
        return (int)cudaGetLastError();
    }
    // register-held chunks pay off only while they are short (measured: 1024^2 +7% on
    // the integral sweep; 4096^2 +-0; 8192^2 and up -10%, occupancy); longer chunks run
    // the two-pass kernel
    if (ch <= 4) {
        auto kern = batch ? chains_reg_kernel<4, true>
                          : (gk == 2 ? chains_reg_kernel<4, false, 2> : chains_reg_kernel<4, false>);
        INIM_CUDA_TRY(launch_pdl(kern, grid, block, 0, st, g, ws, state, bt.slab));
    } else {
        // (no compile-time geometry here: it costs this kernel 16 registers and a CTA per SM)
        auto kern = batch ? chains_kernel<true> : chains_kernel<false>;
        INIM_CUDA_TRY(launch_pdl(kern, grid, block, 0, st, g, ws, state, bt.slab));
    }
    prof_mark(st, "chains");
    return (int)cudaGetLastError();
}

}  // namespace inim
