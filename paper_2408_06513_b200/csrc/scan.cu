// Carry scan launches (phase 2 of the integral pass; the item bodies and their
// derivation are in inim_scan.cuh).  Four launches over 1/TH of the texture, none of
// which waits on another CTA.
#include "inim_scan.cuh"

namespace inim {

constexpr int kScanThreads = 256;

__global__ void __launch_bounds__(kScanThreads) band_rows_kernel(const Geo g, const Ws ws, const int* state) {
    if (state && state[0]) return;
    __shared__ double sh[33];
    band_rows_item(g, ws, blockIdx.x, sh);
}

__global__ void __launch_bounds__(kScanThreads) colscan_kernel(const Geo g, const Ws ws, const int* state) {
    if (state && state[0]) return;
    __shared__ double part[kScanThreads / 32][33];
    colscan_item(g, ws, blockIdx.x, part);
}

__global__ void __launch_bounds__(kScanThreads) diagscan_kernel(const Geo g, const Ws ws, const int* state) {
    if (state && state[0]) return;
    __shared__ double part[kScanThreads / 32][33];
    diagscan_item(g, ws, blockIdx.x, part);
}

__global__ void __launch_bounds__(kScanThreads) marg_kernel(const Geo g, const Ws ws, const int* state) {
    if (state && state[0]) return;
    marg_item(g, ws, blockIdx.x);
}

int launch_carry_scan_state(const Geo& g, const Ws& ws, const int* state, cudaStream_t st) {
    band_rows_kernel<<<g.B, kScanThreads, 0, st>>>(g, ws, state);
    prof_mark(st, "band_rows");
    colscan_kernel<<<colscan_items(g, kScanThreads / 32), kScanThreads, 0, st>>>(g, ws, state);
    prof_mark(st, "colscan");
    diagscan_kernel<<<diagscan_items(g, kScanThreads), kScanThreads, 0, st>>>(g, ws, state);
    prof_mark(st, "diagscan");
    marg_kernel<<<marg_items(g, kScanThreads), kScanThreads, 0, st>>>(g, ws, state);
    prof_mark(st, "marg");
    return (int)cudaGetLastError();
}

}  // namespace inim
