// Smoothing launches per kernel size (the taps are compile-time FFMA immediates, so
// every kernel_size 1..16 is its own set of kernels).  The definitions are
// instantiated in smooth_ks*.cu (four translation units compiled in parallel) and
// dispatched by launch_smooth_state (smooth.cu).
#pragma once

#include <type_traits>

#include "inim_smooth.cuh"

namespace inim {

template <int R, typename T, bool CNT, bool FULL>
__global__ void __launch_bounds__(256, CNT ? 4 : 1) smooth_h_kernel(const T* __restrict__ in, float* __restrict__ out, int s,
                                                       const HGeo h, const Taps taps, const int* state,
                                                       uint32_t* __restrict__ zero_next, int64_t zslab) {
    pdl_enter();
    state = zstate(state, zslab);
    if (state && state[0]) return;
    if (zslab) {  // plot blockIdx.z of a batch (the input is the plot's counts)
        const int64_t zo = zslab_off(zslab);
        in = zoff(in, zo);
        out = zoff(out, zo);
        zero_next = zoff_opt(zero_next, zo);
    }
    extern __shared__ __align__(16) float hsm[];
    smooth_h_tile<R, T, CNT, FULL>(in, out, s, h, taps, zero_next, blockIdx.x, blockIdx.y, hsm);
}

template <int R, int VG>
__global__ void __launch_bounds__(512) smooth_v_kernel(const float* __restrict__ tmp, float* __restrict__ d,
                                                       const Geo g, const VGeo v, const Ws ws, const Taps taps,
                                                       float background, int emit, const int* state, int64_t zslab,
                                                       uint32_t* zero_next, int zrev) {
    pdl_enter();
    const int64_t zo = (zrev ? (int64_t)(gridDim.z - 1 - blockIdx.z) : (int64_t)blockIdx.z) * zslab;
    state = zoff_opt(state, zo);
    if (state && state[0]) return;
    extern __shared__ __align__(16) float vsm[];
    smooth_v_tile<R, VG>(zoff(tmp, zo), zoff(d, zo), g, v, ws_shift(ws, zo), taps, background, emit, blockIdx.x,
                     blockIdx.y, vsm, zoff_opt(zero_next, zo));
}

template <int R, typename T, bool CNT>
inline int launch_h(const T* in, float* out, int s, const Taps& taps, const int* state, uint32_t* zero_next,
                    cudaStream_t st, const Bat& bt) {
    const HGeo h = make_hgeo(s);
    const size_t smem = h_smem_bytes(h, R);
    // grids of side >= 128 all get the 32 x 128 x 8-warp geometry: compile it in
    const bool full = h.RH == 32 && h.TWH == 128 && h.NWH == 8;
    auto kern = full ? smooth_h_kernel<R, T, CNT, true> : smooth_h_kernel<R, T, CNT, false>;
    INIM_CUDA_TRY(ensure_smem_limit((const void*)kern, 200 * 1024));
    dim3 grid(s / h.TWH, s / h.RH, bt.B);
    INIM_CUDA_TRY(launch_pdl(kern, grid, dim3(h.NWH * 32), smem, st, in, out, s, h, taps, state, zero_next, bt.slab));
    prof_mark(st, "smooth_h");
    return (int)cudaGetLastError();
}

template <int R>
inline int launch_v(const float* tmp, float* d, const Geo& g, const Ws& ws, const Taps& taps, float bg, int emit,
                    const int* state, cudaStream_t st, const Bat& bt, uint32_t* zero_next = nullptr) {

    const VGeo v = make_vgeo(g);
    const size_t smem = v_smem_bytes(g, v, R);
    // the two geometries of the runs as compile-time constants (smooth_v_tile VG)
    const bool vg1 = g.TH == 32 && g.TW == 128 && g.CPL == 4 && v.VR == 64 && v.VB == 2 && v.GT == 128;
    const bool vg2 = g.TH == 16 && g.TW == 64 && g.CPL == 2 && v.VR == 64 && v.VB == 4 && v.GT == 64;
    auto kern = vg1 ? smooth_v_kernel<R, 1> : (vg2 ? smooth_v_kernel<R, 2> : smooth_v_kernel<R, 0>);
    INIM_CUDA_TRY(ensure_smem_limit((const void*)kern, 227 * 1024));
    dim3 grid(g.NX, g.s / v.VR, bt.B);
    INIM_CUDA_TRY(launch_pdl(kern, grid, dim3(v.VB * v.GT), smem, st, tmp, d, g, v, ws, taps, bg, emit,
                             state, bt.slab, zero_next, bt.B > 1 && zrev_enabled() ? 1 : 0));
    prof_mark(st, emit ? "smooth_v_reduce" : "smooth_v");
    return (int)cudaGetLastError();
}

// kind: kSmoothGrid (a float grid), kSmoothCountsU32, kSmoothCountsF32 (smooth.cu)
template <int KS>
int launch_pair(const void* in, int kind, const Geo& g, const Ws& ws, const Taps& taps, float bg,
                       float* d, int emit, const int* state, uint32_t* zero_next, cudaStream_t st, const Bat& bt) {
    constexpr int R = 3 * KS;
    // the clear of the next count buffer rides on the vertical pass (INIM_CLEAR_IN_V=0:
    // on the horizontal pass, as before)
    static const bool clear_in_v = [] {
        const char* e = getenv("INIM_CLEAR_IN_V");
        return !(e && e[0] == '0');
    }();
    uint32_t* zh = clear_in_v ? nullptr : zero_next;
    uint32_t* zv = clear_in_v ? zero_next : nullptr;
    int rc = kind == 1   ? launch_h<R, uint32_t, true>(static_cast<const uint32_t*>(in), ws.tmp, g.s, taps, state,
                                                      zh, st, bt)
             : kind == 2 ? launch_h<R, float, true>(static_cast<const float*>(in), ws.tmp, g.s, taps, state, zh, st,
                                                   bt)
                         : launch_h<R, float, false>(static_cast<const float*>(in), ws.tmp, g.s, taps, state, zh,
                                                    st, bt);
    if (rc) return rc;
    return launch_v<R>(ws.tmp, d, g, ws, taps, bg, emit, state, st, bt, zv);
}

}  // namespace inim
