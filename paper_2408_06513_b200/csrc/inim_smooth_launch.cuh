// Smoothing launches per kernel size (the taps are compile-time FFMA immediates, so
// every kernel_size 1..16 is its own set of kernels).  The definitions are
// instantiated in smooth_ks*.cu (four translation units compiled in parallel) and
// dispatched by launch_smooth_state (smooth.cu).
#pragma once

#include <type_traits>

#include "inim_smooth.cuh"

namespace inim {

template <int R, typename T>
__global__ void __launch_bounds__(256, std::is_same<T, float>::value ? 1 : 4) smooth_h_kernel(const T* __restrict__ in, float* __restrict__ out, int s,
                                                       const HGeo h, const Taps taps, const int* state,
                                                       uint32_t* __restrict__ zero_next, int64_t zslab) {
    pdl_enter();
    if (state && state[0]) return;
    if (zslab) {  // plot blockIdx.z of a batch (the input is the plot's counts)
        const int64_t zo = zslab_off(zslab);
        in = zoff(in, zo);
        out = zoff(out, zo);
        zero_next = zoff_opt(zero_next, zo);
    }
    extern __shared__ __align__(16) float hsm[];
    smooth_h_tile<R, T>(in, out, s, h, taps, zero_next, blockIdx.x, blockIdx.y, hsm);
}

template <int R>
__global__ void __launch_bounds__(512) smooth_v_kernel(const float* __restrict__ tmp, float* __restrict__ d,
                                                       const Geo g, const VGeo v, const Ws ws, const Taps taps,
                                                       float background, int emit, const int* state, int64_t zslab) {
    pdl_enter();
    if (state && state[0]) return;
    extern __shared__ __align__(16) float vsm[];
    const int64_t zo = zslab_off(zslab);
    smooth_v_tile<R>(zoff(tmp, zo), zoff(d, zo), g, v, ws_shift(ws, zo), taps, background, emit, blockIdx.x,
                     blockIdx.y, vsm);
}

// The iteration's smoothing of the counts in one launch: horizontal + vertical pass +
// tile reduce, vertical halos exchanged through distributed shared memory within
// clusters of vertically adjacent tiles (inim_smooth.cuh smooth_cluster_tile).
template <int R, int CPL>
__global__ void __launch_bounds__(kCThreads) smooth_cluster_kernel(const uint32_t* __restrict__ in,
                                                                   float* __restrict__ d,
                                                                   uint32_t* __restrict__ zero_next, const Geo g,
                                                                   const Ws ws, float background, int emit,
                                                                   const int* state, int64_t zslab) {
    pdl_enter();
    if (state && state[0]) return;  // uniform over the grid: no CTA waits at a cluster barrier alone
    extern __shared__ __align__(16) float csm[];
    const int64_t zo = zslab_off(zslab);  // plot blockIdx.z of a batch
    const cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
    smooth_cluster_tile<R, CPL>(zoff(in, zo), zoff(d, zo), zoff_opt(zero_next, zo), g, ws_shift(ws, zo), background,
                                emit, blockIdx.x, blockIdx.y, (int)cl.block_rank(), (int)cl.num_blocks(), csm);
}

constexpr int kMaxClusterRows = 8;  // portable cluster size

template <int R, int CPL>
inline int launch_cluster(const uint32_t* counts, float* d, uint32_t* zero_next, const Geo& g, const Ws& ws, float bg,
                          int emit, const int* state, cudaStream_t st, const Bat& bt) {
    const size_t smem = cl_smem_bytes(g.TW, R);
    INIM_CUDA_TRY(ensure_smem_limit((const void*)smooth_cluster_kernel<R, CPL>, (int)smem));
    const int ty = g.s / kCRows;
    const int cy = ty < kMaxClusterRows ? ty : kMaxClusterRows;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(g.NX, ty, bt.B);
    cfg.blockDim = dim3(kCThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = cy;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    INIM_CUDA_TRY(cudaLaunchKernelEx(&cfg, smooth_cluster_kernel<R, CPL>, counts, d, zero_next, g, ws, bg, emit, state,
                                     bt.slab));
    prof_mark(st, emit ? "smooth_cluster_reduce" : "smooth_cluster");
    return (int)cudaGetLastError();
}

bool cluster_smooth_enabled();  // smooth.cu (INIM_CLUSTER_SMOOTH=0 selects the two-kernel path)

template <int R, typename T>
inline int launch_h(const T* in, float* out, int s, const Taps& taps, const int* state, uint32_t* zero_next,
                    cudaStream_t st, const Bat& bt) {
    const HGeo h = make_hgeo(s);
    const size_t smem = h_smem_bytes(h, R);
    INIM_CUDA_TRY(ensure_smem_limit((const void*)smooth_h_kernel<R, T>, 200 * 1024));
    dim3 grid(s / h.TWH, s / h.RH, bt.B);
    INIM_CUDA_TRY(launch_pdl(smooth_h_kernel<R, T>, grid, dim3(h.NWH * 32), smem, st, in, out, s, h, taps, state,
                             zero_next, bt.slab));
    prof_mark(st, "smooth_h");
    return (int)cudaGetLastError();
}

template <int R>
inline int launch_v(const float* tmp, float* d, const Geo& g, const Ws& ws, const Taps& taps, float bg, int emit,
                    const int* state, cudaStream_t st, const Bat& bt) {

    const VGeo v = make_vgeo(g);
    const size_t smem = v_smem_bytes(g, v, R);
    INIM_CUDA_TRY(ensure_smem_limit((const void*)smooth_v_kernel<R>, 227 * 1024));
    dim3 grid(g.NX, g.s / v.VR, bt.B);
    INIM_CUDA_TRY(launch_pdl(smooth_v_kernel<R>, grid, dim3(v.VB * v.GT), smem, st, tmp, d, g, v, ws, taps, bg, emit,
                             state, bt.slab));
    prof_mark(st, emit ? "smooth_v_reduce" : "smooth_v");
    return (int)cudaGetLastError();
}

template <int KS>
int launch_pair(const void* in, bool counts, const Geo& g, const Ws& ws, const Taps& taps, float bg,
                       float* d, int emit, const int* state, uint32_t* zero_next, cudaStream_t st, const Bat& bt) {
    constexpr int R = 3 * KS;
    // the counts of the iteration on grids of 64^2 and up: one cluster launch
    if (counts && g.s >= kCRows && cluster_smooth_enabled()) {
        const uint32_t* c = static_cast<const uint32_t*>(in);
        if (g.CPL == 4) return launch_cluster<R, 4>(c, d, zero_next, g, ws, bg, emit, state, st, bt);
        if (g.CPL == 2) return launch_cluster<R, 2>(c, d, zero_next, g, ws, bg, emit, state, st, bt);
    }
    int rc = counts ? launch_h<R, uint32_t>(static_cast<const uint32_t*>(in), ws.tmp, g.s, taps, state, zero_next, st,
                                            bt)
                    : launch_h<R, float>(static_cast<const float*>(in), ws.tmp, g.s, taps, state, zero_next, st, bt);
    if (rc) return rc;
    return launch_v<R>(ws.tmp, d, g, ws, taps, bg, emit, state, st, bt);
}

}  // namespace inim
