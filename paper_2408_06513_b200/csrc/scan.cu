// Carry scan launch (phase 2 of the integral pass; the item bodies and their derivation
// are in inim_scan.cuh).  The per-band lines run at the end of the reduce (the warp that
// completes a band) and the marginals are read off the chains by the write pass, so
// phase 2 is one launch over 1/TH of the texture.
#include "inim_scan.cuh"

namespace inim {

__global__ void __launch_bounds__(512) chains_kernel(const Geo g, const Ws ws, const int* state) {
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

int launch_carry_scan_state(const Geo& g, const Ws& ws, const int* state, cudaStream_t st) {
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
