// Device kernels behind the reference's secondary (non-iteration) API functions:
//   anchors / raw_map / corrected_map at arbitrary query points (mapping.py:40-143),
//   tilted_wedges arithmetic (integral.py:212-228),
//   sample_field on float64 targets (mapping.py:207-246),
//   flat_response in float64 (mapping.py:104-129).
// None of these is on the per-iteration path; they exist so the drop-in exposes the
// reference's whole hot-path module surface on the device.
#include "inim_internal.cuh"

namespace inim {

struct AnchorsD {
    double drx, dry, ulx, uly, urx, ury, dlx, dly;
};

__device__ __forceinline__ AnchorsD anchors_d(double x, double y) {
    AnchorsD A;
    const bool below = y < x;  // mapping.py:42
    A.drx = below ? 1.0 : 1.0 - y + x;
    A.dry = below ? 1.0 + y - x : 1.0;
    A.ulx = below ? x - y : 0.0;
    A.uly = below ? 0.0 : y - x;
    const bool near = x + y < 1.0;  // mapping.py:47
    A.urx = near ? x + y : 1.0;
    A.ury = near ? 0.0 : x + y - 1.0;
    A.dlx = near ? 0.0 : x + y - 1.0;
    A.dly = near ? x + y : 1.0;
    return A;
}

__device__ __forceinline__ int pix_d(double v, int s) {
    int i = (int)floor(v * (double)s);
    i = i > s - 1 ? s - 1 : i;
    return i < 0 ? 0 : i;
}

// mode 0: anchors -> out[8] = dr, ur, ul, dl (x, y each)
// mode 1: raw_map -> out[2]
// mode 2: corrected_map -> out[2] = clip((x, y) + raw - defect[j, i])
__global__ void map_points_kernel(const float* __restrict__ t8, int k, const double* total,
                                  const double* __restrict__ defect, const double* __restrict__ xs,
                                  const double* __restrict__ ys, int64_t n, int mode, double* __restrict__ out) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const double x = xs[p], y = ys[p];
    const AnchorsD A = anchors_d(x, y);
    if (mode == 0) {
        double* o = out + 8 * p;
        o[0] = A.drx; o[1] = A.dry; o[2] = A.urx; o[3] = A.ury;
        o[4] = A.ulx; o[5] = A.uly; o[6] = A.dlx; o[7] = A.dly;
        return;
    }
    const int s = 1 << k;
    const int64_t m = (int64_t)s * s;
    const int i = pix_d(x, s), j = pix_d(y, s);
    const int64_t q = (int64_t)j * s + i;
    const double tl = t8[q], bl = t8[m + q], br = t8[2 * m + q], tr = t8[3 * m + q];
    const double up = t8[4 * m + q], left = t8[5 * m + q], down = t8[6 * m + q], right = t8[7 * m + q];
    const double inv = 0.5 / *total;
    // _weighted_components (mapping.py:64-77)
    double tx = (tl * A.drx + bl * A.urx + br * A.ulx + tr * A.dlx + (up + down) * x + left) * inv;
    double ty = (tl * A.dry + bl * A.ury + br * A.uly + tr * A.dly + (left + right) * y + up) * inv;
    if (mode == 2) {
        tx = x + tx - defect[2 * q];
        ty = y + ty - defect[2 * q + 1];
        tx = tx < 0.0 ? 0.0 : (tx > 1.0 ? 1.0 : tx);
        ty = ty < 0.0 ? 0.0 : (ty > 1.0 ? 1.0 : ty);
    }
    out[2 * p] = tx;
    out[2 * p + 1] = ty;
}

// left_half / right_half (integral.py:220-222): prefix / suffix of the column sums
// (upper's last row), float64, one block.
__global__ void __launch_bounds__(1024) half_planes_kernel(const float* __restrict__ upper, int s,
                                                           double* __restrict__ lh, double* __restrict__ rh) {
    __shared__ double sh[1024 + 1];
    const float* cs = upper + (int64_t)(s - 1) * s;
    const int nt = blockDim.x, t = threadIdx.x;
    const int chunk = (s + nt - 1) / nt;
    const int lo = t * chunk, hi = min(s, lo + chunk);
    double acc = 0.0;
    for (int c = lo; c < hi; ++c) acc += (double)cs[c];
    sh[t] = acc;
    __syncthreads();
    if (t == 0) {
        double run = 0.0;
        for (int v = 0; v < nt; ++v) {
            const double a = sh[v];
            sh[v] = run;
            run += a;
        }
        sh[nt] = run;
    }
    __syncthreads();
    double run = sh[t];
    const double tot = sh[nt];
    for (int c = lo; c < hi; ++c) {
        const double before = run;
        run += (double)cs[c];
        lh[c] = run;               // columns <= c
        rh[c] = tot - before;      // columns >= c
    }
}

// tilted_wedges (integral.py:224-227): out4 = up, left, down, right.
__global__ void tilted_wedges_kernel(const float* __restrict__ ul, const float* __restrict__ ur,
                                     const float* __restrict__ dl, const float* __restrict__ dr,
                                     const float* __restrict__ upper, const float* __restrict__ lower,
                                     const double* __restrict__ lh, const double* __restrict__ rh, int k,
                                     float* __restrict__ out4) {
    const int s = 1 << k;
    const int64_t m = (int64_t)s * s;
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= m) return;
    const int i = (int)(q & (s - 1));
    const double a = ul[q], b = ur[q], c = dl[q], e = dr[q];
    out4[q] = (float)(a + b - (double)upper[q]);
    out4[m + q] = (float)(lh[i] - a - c);
    out4[2 * m + q] = (float)(c + e - (double)lower[q]);
    out4[3 * m + q] = (float)(rh[i] - b - e);
}

// sample_field on float64 targets and float64 points (mapping.py:207-246) [+ clip].
__global__ void sample_t64_kernel(const double* __restrict__ tg, int k, const double* __restrict__ in,
                                  double* __restrict__ out, int64_t n, int clip) {
    const int s = 1 << k;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const double sx = in[2 * p] * s, sy = in[2 * p + 1] * s;
        int i0 = (int)floor(sx), j0 = (int)floor(sy);
        i0 = i0 < 0 ? 0 : (i0 > s - 2 ? s - 2 : i0);
        j0 = j0 < 0 ? 0 : (j0 > s - 2 ? s - 2 : j0);
        const double fx = sx - i0, fy = sy - j0;
        const double w00 = (1.0 - fx) * (1.0 - fy), w10 = fx * (1.0 - fy), w01 = (1.0 - fx) * fy, w11 = fx * fy;
        const int64_t b = (int64_t)j0 * s + i0;
        for (int c = 0; c < 2; ++c) {
            double v = w00 * tg[2 * b + c] + w10 * tg[2 * (b + 1) + c] + w01 * tg[2 * (b + s) + c] +
                       w11 * tg[2 * (b + s + 1) + c];
            if (clip) v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
            out[2 * p + c] = v;
        }
    }
}

// The closed-form flat response is evaluated here in float64 and stored as float64.
__global__ void flat_response_f64_kernel(int k, double* __restrict__ defect) {
    const int s = 1 << k;
    const int64_t m = (int64_t)s * s;
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= m) return;
    const int i = (int)(q & (s - 1)), j = (int)(q >> k);
    // Region pixel counts of a constant texture (see integral.cu flat_response_at).
    const int64_t S = s, s2 = S * S, I = i, J = j;
    auto f = [&](int64_t L) { return L * (J + 1) - L * (L + 1) / 2; };
    const int64_t up1 = (J + 1) + f(min(J, I)) + f(min(J, S - 1 - I));
    const int64_t sg = I + J;
    const int64_t A1 = sg <= S - 1 ? (sg + 1) * (sg + 2) / 2 : s2 - (2 * S - 2 - sg) * (2 * S - 1 - sg) / 2;
    const int64_t dl = I - J;
    const int64_t D1 = dl >= 0 ? (S - dl) * (S - dl + 1) / 2 : s2 - (S + dl - 1) * (S + dl) / 2;
    const double tl = (double)((I + 1) * (J + 1)), bl = (double)((I + 1) * (S - 1 - J));
    const double tr = (double)((S - 1 - I) * (J + 1)), br = (double)((S - 1 - I) * (S - 1 - J));
    const double up = (double)up1, left = (double)(A1 - up1), right = (double)(D1 - up1);
    const double down = (double)s2 - up - left - right;
    const double scale = ldexp(1.0, -k);
    const double x = i * scale, y = j * scale;
    const AnchorsD A = anchors_d(x, y);
    const double inv = 0.5 / (double)s2;
    // Same operation order as _per_pixel_targets (mapping.py:175-178); __dmul_rn /
    // __dadd_rn keep a*b+c as two roundings like the reference's numba code.
    double tx = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(tl, A.drx), __dmul_rn(bl, A.urx)),
                                                          __dmul_rn(br, A.ulx)),
                                                 __dmul_rn(tr, A.dlx)),
                                        __dmul_rn(__dadd_rn(up, down), x)),
                               left);
    double ty = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(tl, A.dry), __dmul_rn(bl, A.ury)),
                                                          __dmul_rn(br, A.uly)),
                                                 __dmul_rn(tr, A.dly)),
                                        __dmul_rn(__dadd_rn(left, right), y)),
                               up);
    defect[2 * q] = __dmul_rn(tx, inv);
    defect[2 * q + 1] = __dmul_rn(ty, inv);
}

// transition_positions (regularize.py:83-93) rounded to float32 for the service's
// binary payload (service.py:170-172): (1 - frac) * lo + frac * hi in float64, each
// operation rounded as numpy does (no FMA), then one rounding to float32.
template <typename TL, typename TH>
__global__ void blend_frames_kernel(const TL* __restrict__ lo, const TH* __restrict__ hi, int64_t count, double frac,
                                    int same, float* __restrict__ out) {
    const double wl = 1.0 - frac;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < count; q += (int64_t)gridDim.x * blockDim.x) {
        const double a = (double)lo[q];
        out[q] = __double2float_rn(same ? a : __dadd_rn(__dmul_rn(wl, a), __dmul_rn(frac, (double)hi[q])));
    }
}

}  // namespace inim

using namespace inim;

extern "C" {

int inim_map_points(const float* tables8, int k, const double* total, const double* defect, const double* xs,
                    const double* ys, int64_t n, int mode, double* out, cudaStream_t stream) {
    if (k < 0 || k > INIM_MAX_K || n < 0 || mode < 0 || mode > 2 || (n > 0 && (!xs || !ys || !out))) return INIM_EINVAL;
    if (mode >= 1 && (!tables8 || !total)) return INIM_EINVAL;
    if (mode == 2 && !defect) return INIM_EINVAL;
    if (n == 0) return 0;
    map_points_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(tables8, k, total, defect, xs, ys, n, mode, out);
    return (int)cudaGetLastError();
}

int inim_tilted_wedges(const float* ul, const float* ur, const float* dl, const float* dr, const float* upper,
                       const float* lower, int k, double* scratch2s, float* out4, cudaStream_t stream) {
    if (k < 0 || k > INIM_MAX_K || !ul || !ur || !dl || !dr || !upper || !lower || !scratch2s || !out4)
        return INIM_EINVAL;
    const int s = 1 << k;
    half_planes_kernel<<<1, 1024, 0, stream>>>(upper, s, scratch2s, scratch2s + s);
    const int64_t m = (int64_t)s * s;
    tilted_wedges_kernel<<<(unsigned)((m + 255) / 256), 256, 0, stream>>>(ul, ur, dl, dr, upper, lower, scratch2s,
                                                                          scratch2s + s, k, out4);
    return (int)cudaGetLastError();
}

int inim_sample_t64(const double* targets, int k, const double* pts_in, double* pts_out, int64_t n, int clip,
                    cudaStream_t stream) {
    if (k < 1 || k > INIM_MAX_K || !targets || n < 0 || (n > 0 && (!pts_in || !pts_out))) return INIM_EINVAL;
    if (n == 0) return 0;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    sample_t64_kernel<<<(unsigned)blocks, 256, 0, stream>>>(targets, k, pts_in, pts_out, n, clip);
    return (int)cudaGetLastError();
}

int inim_flat_response_f64(int k, double* defect, cudaStream_t stream) {
    if (k < 0 || k > INIM_MAX_K || !defect) return INIM_EINVAL;
    const int64_t m = (int64_t)1 << (2 * k);
    flat_response_f64_kernel<<<(unsigned)((m + 255) / 256), 256, 0, stream>>>(k, defect);
    return (int)cudaGetLastError();
}

int inim_blend_frames(const void* lo, int lo_f64, const void* hi, int hi_f64, int64_t count, double frac, int same,
                      float* out, cudaStream_t stream) {
    if (count < 0 || (count > 0 && (!lo || !hi || !out))) return INIM_EINVAL;
    if (count == 0) return 0;
    const unsigned g = (unsigned)((count + 255) / 256 < 4096 ? (count + 255) / 256 : 4096);
    if (lo_f64 && hi_f64)
        blend_frames_kernel<<<g, 256, 0, stream>>>((const double*)lo, (const double*)hi, count, frac, same, out);
    else if (lo_f64)
        blend_frames_kernel<<<g, 256, 0, stream>>>((const double*)lo, (const float*)hi, count, frac, same, out);
    else if (hi_f64)
        blend_frames_kernel<<<g, 256, 0, stream>>>((const float*)lo, (const double*)hi, count, frac, same, out);
    else
        blend_frames_kernel<<<g, 256, 0, stream>>>((const float*)lo, (const float*)hi, count, frac, same, out);
    return (int)cudaGetLastError();
}

}  // extern "C"
