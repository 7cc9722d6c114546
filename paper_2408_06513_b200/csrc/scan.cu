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

int launch_carry_scan_state(const Geo& g, const Ws& ws, const int* state, cudaStream_t st) {
    INIM_CUDA_TRY(launch_pdl(chains_kernel, dim3(chains_items(g)), dim3(32 * chain_warps(g)), 0, st, g, ws, state));
    prof_mark(st, "chains");
    return (int)cudaGetLastError();
}

}  // namespace inim
