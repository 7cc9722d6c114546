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

// The float32 bilinear sample split into its gathers and its blend, so a caller can put
// the gathers of several points in flight before the first blend (same values and
// arithmetic as bilinear / bilinear_pairs).
struct Tap4 {
    float4 r0, r1;  // (t00, t10) and (t01, t11) as (x, y, x, y)
    float fx, fy;
};

template <bool PAIRS>
__device__ __forceinline__ Tap4 bilinear_fetch(const float* tg, int s, float x, float y) {
    const float sx = x * (float)s, sy = y * (float)s;
    int i0 = (int)floorf(sx), j0 = (int)floorf(sy);
    i0 = i0 < 0 ? 0 : (i0 > s - 2 ? s - 2 : i0);
    j0 = j0 < 0 ? 0 : (j0 > s - 2 ? s - 2 : j0);
    Tap4 t;
    t.fx = sx - (float)i0;
    t.fy = sy - (float)j0;
    const int64_t base = (int64_t)j0 * s + i0;
    if (PAIRS) {
        const float4* tp = reinterpret_cast<const float4*>(tg);
        t.r0 = __ldg(tp + base);
        t.r1 = __ldg(tp + base + s);
    } else {
        const float2* tp = reinterpret_cast<const float2*>(tg);
        const float2 a = __ldg(tp + base), b = __ldg(tp + base + 1);
        const float2 c = __ldg(tp + base + s), d = __ldg(tp + base + s + 1);
        t.r0 = make_float4(a.x, a.y, b.x, b.y);
        t.r1 = make_float4(c.x, c.y, d.x, d.y);
    }
    return t;
}

__device__ __forceinline__ void bilinear_blend(const Tap4& t, float& ox, float& oy) {
    const float w00 = (1.f - t.fx) * (1.f - t.fy);
    const float w10 = t.fx * (1.f - t.fy);
    const float w01 = (1.f - t.fx) * t.fy;
    const float w11 = t.fx * t.fy;
    ox = w00 * t.r0.x + w10 * t.r0.z + w01 * t.r1.x + w11 * t.r1.z;
    oy = w00 * t.r0.y + w10 * t.r0.w + w01 * t.r1.y + w11 * t.r1.w;
}

template <typename T>
__device__ __forceinline__ T clip01(T v) {
    return v < (T)0 ? (T)0 : (v > (T)1 ? (T)1 : v);
}

}  // namespace inim
