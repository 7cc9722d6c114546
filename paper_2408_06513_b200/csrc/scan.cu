// Carry scan launch (phase 2 of the integral pass; the item bodies and their derivation
// are in inim_scan.cuh).  The per-band lines run at the end of the reduce (the warp that
// completes a band) and the marginals are read off the chains by the write pass, so
// phase 2 is one launch over 1/TH of the texture.
#include "inim_scan.cuh"
#include "inim_tiles.cuh"

namespace inim {

// INIM_CHAIN_MINB: experiment switch (measured: forcing 4 CTAs/SM = 32 registers spills
// and is no faster than 3 CTAs/SM).  Left undefined on purpose: an explicit minimum of 1
// lets ptxas spend 72 registers (1 CTA/SM, -4% on the integral sweep), while the plain
// bound settles at 40 (3 CTAs/SM).
#ifdef INIM_CHAIN_MINB
#define INIM_CHAIN_BOUNDS __launch_bounds__(512, INIM_CHAIN_MINB)
#else
#define INIM_CHAIN_BOUNDS __launch_bounds__(512)
#endif
__global__ void INIM_CHAIN_BOUNDS chains_kernel(const Geo g, const Ws ws, const int* state) {
    pdl_enter();
    if (state && state[0]) return;
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
template <int MAXCH>
__global__ void __launch_bounds__(512) chains_reg_kernel(const Geo g, const Ws ws, const int* state) {
    pdl_enter();
    if (state && state[0]) return;
    __shared__ double part[16][33];
    __shared__ double bp[kMaxBands + 1];
    __shared__ double sh[33];
    chains_item_reg<MAXCH>(g, ws, blockIdx.x, part, bp, sh);
}

// Band lines (one CTA per band, one warp per row): HC[j][x] = exclusive prefix over the
// tiles of row j's tile row sums, rpre = the band's in-band prefix of the row totals,
// tilepre / btot = the exclusive prefix and the total of the band's tile totals.  A
// launch of its own so that no reduce warp has to fence and count its band's arrivals.
__global__ void __launch_bounds__(1024) lines_kernel(const Geo g, const Ws ws, const int* state) {
    pdl_enter();
    if (state && state[0]) return;
    __shared__ double rowtot[32];
    const int b = blockIdx.x, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int TH = g.TH, NX = g.NX, a = b * TH;
    {
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

int launch_carry_scan_state(const Geo& g, const Ws& ws, const int* state, cudaStream_t st) {
    INIM_CUDA_TRY(launch_pdl(lines_kernel, dim3(g.B), dim3(32 * g.TH), 0, st, g, ws, state));
    prof_mark(st, "lines");
    const int ny = chain_warps(g), ch = (g.B + ny - 1) / ny;
    const dim3 grid(chains_items(g)), block(32 * ny);
    // register-held chunks pay off only while they are short (measured: 1024^2 +7% on
    // the integral sweep; 4096^2 +-0; 8192^2 and up -10%, occupancy); longer chunks run
    // the two-pass kernel
    if (ch <= 4) {
        INIM_CUDA_TRY(launch_pdl(chains_reg_kernel<4>, grid, block, 0, st, g, ws, state));
    } else {
        INIM_CUDA_TRY(launch_pdl(chains_kernel, grid, block, 0, st, g, ws, state));
    }
    prof_mark(st, "chains");
    return (int)cudaGetLastError();
}

}  // namespace inim
