// Carry scan launches (phase 2 of the integral pass; the item bodies and their
// derivation are in inim_scan.cuh): lines -> chains -> marg, three launches over
// 1/TH of the texture, none of which waits on another CTA.
#include "inim_scan.cuh"

namespace inim {

constexpr int kLineThreads = 256;
constexpr int kMargThreads = 256;

__global__ void __launch_bounds__(kLineThreads) lines_kernel(const Geo g, const Ws ws, const int* state) {
    if (state && state[0]) return;
    __shared__ double sh[33];
    lines_item(g, ws, blockIdx.x, sh);
}

__global__ void __launch_bounds__(512) chains_kernel(const Geo g, const Ws ws, const int* state) {
    if (state && state[0]) return;
    __shared__ double part[16][33];
    __shared__ double bp[kMaxBands + 1];
    __shared__ double sh[33];
    const int item = blockIdx.x;
    if (chain_kind(g, item) == 2) {
        band_prefix(g, ws, bp, sh);
        if (item == chain_groups_tl(g) + chain_groups_x(g))  // first X2 item publishes it for marg
            for (int q = threadIdx.x; q <= g.B; q += blockDim.x) ws.bandpre[q] = bp[q];
    }
    chains_item(g, ws, item, part, bp);
}

__global__ void __launch_bounds__(kMargThreads) marg_kernel(const Geo g, const Ws ws, const int* state) {
    if (state && state[0]) return;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < marg_entries(g)) marg_entry(g, ws, q);
}

int launch_carry_scan_state(const Geo& g, const Ws& ws, const int* state, cudaStream_t st) {
    lines_kernel<<<g.B, kLineThreads, 0, st>>>(g, ws, state);
    prof_mark(st, "lines");
    chains_kernel<<<chains_items(g), 32 * chain_warps(g), 0, st>>>(g, ws, state);
    prof_mark(st, "chains");
    marg_kernel<<<(marg_entries(g) + kMargThreads - 1) / kMargThreads, kMargThreads, 0, st>>>(g, ws, state);
    prof_mark(st, "marg");
    return (int)cudaGetLastError();
}

}  // namespace inim
