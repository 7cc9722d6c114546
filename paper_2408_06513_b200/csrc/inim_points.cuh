// Point-stream device helpers shared by points.cu and mega.cu: pixel_of
// (reference model.py:189-198) and the bilinear field evaluation of _bilinear_kernel
// (mapping.py:207-232).
#pragma once

#include "inim_internal.cuh"

namespace inim {

template <typename T>
__device__ __forceinline__ int pixel_of(T v, int s) {
    // i = min(floor(v * s), s - 1); v * s is exact for s = 2^k, so float32 and
    // float64 coordinates bin identically when the values are identical.
    const T f = floor(v * (T)s);
    int i = (int)f;
    i = i > s - 1 ? s - 1 : i;
    return i < 0 ? 0 : i;
}

// i0 = clamp(floor(x*s), 0, s-2), fx = x*s - i0 (in [1, 2] on the last strip: one-sided
// extrapolation keeps an identity field the identity), then the four-tap blend.
template <typename T>
__device__ __forceinline__ void bilinear(const float2* __restrict__ tg, int s, T x, T y, T& ox, T& oy) {
    const T sx = x * (T)s, sy = y * (T)s;
    int i0 = (int)floor(sx), j0 = (int)floor(sy);
    i0 = i0 < 0 ? 0 : (i0 > s - 2 ? s - 2 : i0);
    j0 = j0 < 0 ? 0 : (j0 > s - 2 ? s - 2 : j0);
    const T fx = sx - (T)i0, fy = sy - (T)j0;
    const T w00 = ((T)1 - fx) * ((T)1 - fy);
    const T w10 = fx * ((T)1 - fy);
    const T w01 = ((T)1 - fx) * fy;
    const T w11 = fx * fy;
    const int64_t base = (int64_t)j0 * s + i0;
    const float2 t00 = __ldg(tg + base), t10 = __ldg(tg + base + 1);
    const float2 t01 = __ldg(tg + base + s), t11 = __ldg(tg + base + s + 1);
    ox = w00 * (T)t00.x + w10 * (T)t10.x + w01 * (T)t01.x + w11 * (T)t11.x;
    oy = w00 * (T)t00.y + w10 * (T)t10.y + w01 * (T)t01.y + w11 * (T)t11.y;
}

// The same blend from the paired field layout (slot i of row j = (t(i, j), t(i + 1, j)),
// see WriteOut::pairs): two 16-byte loads instead of four 8-byte ones, identical values
// and arithmetic.
__device__ __forceinline__ void bilinear_pairs(const float4* __restrict__ tp, int s, float x, float y, float& ox,
                                               float& oy) {
    const float sx = x * (float)s, sy = y * (float)s;
    int i0 = (int)floorf(sx), j0 = (int)floorf(sy);
    i0 = i0 < 0 ? 0 : (i0 > s - 2 ? s - 2 : i0);
    j0 = j0 < 0 ? 0 : (j0 > s - 2 ? s - 2 : j0);
    const float fx = sx - (float)i0, fy = sy - (float)j0;
    const float w00 = (1.f - fx) * (1.f - fy);
    const float w10 = fx * (1.f - fy);
    const float w01 = (1.f - fx) * fy;
    const float w11 = fx * fy;
    const int64_t base = (int64_t)j0 * s + i0;
    const float4 r0 = __ldg(tp + base), r1 = __ldg(tp + base + s);
    ox = w00 * r0.x + w10 * r0.z + w01 * r1.x + w11 * r1.z;
    oy = w00 * r0.y + w10 * r0.w + w01 * r1.y + w11 * r1.w;
}

template <typename T>
__device__ __forceinline__ T clip01(T v) {
    return v < (T)0 ? (T)0 : (v > (T)1 ? (T)1 : v);
}

}  // namespace inim
