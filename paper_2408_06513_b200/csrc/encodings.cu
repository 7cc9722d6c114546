// deform_background (reference encodings.py:124-162) on the device: the iteration-0
// density carried into the deformed domain.
//
// Every source pixel q (pushed through the composed fields by the caller: `targets`)
// splats its density value with bilinear weights onto the 2x2 pixels of its cell; the
// per-pixel sums are weight-normalised; uncovered pixels copy their nearest covered
// pixel (Euclidean, scipy distance_transform_edt(return_indices=True)).
//
// Determinism and exactness: instead of float atomics, the splat is inverted into a
// gather.  Sources are bucketed by cell (counting sort, each bucket then ordered by
// source index), and every output pixel walks the four cells that reach it in the
// reference's np.add.at order -- pass (0,0), (1,0), (0,1), (1,1), sources ascending --
// accumulating  acc += w*v,  weight += w  in float64 without FMA contraction.  For the
// same targets and values the sums are therefore bit-identical to the reference's.
//
// The nearest-covered fill is an exact separable Euclidean distance transform with
// argmin tracking: per column the nearest covered row, then per row the lower envelope
// of the parabolas (i - q)^2 + g_q^2 (Felzenszwalb-Huttenlocher).  Among equidistant
// covered pixels any one is "nearest"; the tests check distances, not tie-breaks.
#include "inim_internal.cuh"

namespace inim {

int launch_exclusive_scan_u32(const uint32_t* counts, int64_t m, uint32_t* bsum, uint32_t* out, cudaStream_t st);
size_t sort_bsum_words(int k);

// Cell of a mapped source pixel and its bilinear fractions (encodings.py:141-145):
// scaled = t * size; cell = clip(floor(scaled), 0, size - 2); frac = clip(scaled - cell, 0, 1).
INIM_DEV void bg_cell(float tx, float ty, int s, int& ci, int& cj, double& fx, double& fy) {
    const double sx = (double)tx * s, sy = (double)ty * s;
    const double cx = fmin(fmax(floor(sx), 0.0), (double)(s - 2));
    const double cy = fmin(fmax(floor(sy), 0.0), (double)(s - 2));
    ci = (int)cx;
    cj = (int)cy;
    fx = fmin(fmax(sx - cx, 0.0), 1.0);
    fy = fmin(fmax(sy - cy, 0.0), 1.0);
}

// Also the value range of the (positive) density: min / max through the bit patterns.
__global__ void bg_cells_kernel(const float2* __restrict__ tg, const float* __restrict__ values, int k, int64_t m,
                                uint32_t* __restrict__ cellof, uint32_t* __restrict__ counts, float* range2) {
    const int s = 1 << k;
    float lo = __int_as_float(0x7f800000), hi = 0.f;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
        const float v = values[q];
        lo = fminf(lo, v);
        hi = fmaxf(hi, v);
        const float2 t = tg[q];
        int ci, cj;
        double fx, fy;
        bg_cell(t.x, t.y, s, ci, cj, fx, fy);
        const uint32_t c = (uint32_t)cj * s + ci;
        cellof[q] = c;
        atomicAdd(counts + c, 1u);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(kFull, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(kFull, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(reinterpret_cast<unsigned*>(range2), __float_as_uint(lo));
        atomicMax(reinterpret_cast<unsigned*>(range2) + 1, __float_as_uint(hi));
    }
}

__global__ void bg_range_init_kernel(float* range2) {
    range2[0] = __int_as_float(0x7f800000);
    range2[1] = 0.f;
}

__global__ void bg_place_kernel(const uint32_t* __restrict__ cellof, int64_t m, uint32_t* __restrict__ cursor,
                                uint32_t* __restrict__ list) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x)
        list[atomicAdd(cursor + cellof[q], 1u)] = (uint32_t)q;
}

// Order every bucket by source index (insertion sort for short buckets, heapsort for
// long ones: any bucket size stays O(c log c)).
INIM_DEV void sift_down(uint32_t* a, int64_t root, int64_t n) {
    while (true) {
        int64_t c = 2 * root + 1;
        if (c >= n) return;
        if (c + 1 < n && a[c + 1] > a[c]) ++c;
        if (a[root] >= a[c]) return;
        const uint32_t t = a[root];
        a[root] = a[c];
        a[c] = t;
        root = c;
    }
}

__global__ void bg_bucket_sort_kernel(const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ counts,
                                      int64_t m, uint32_t* __restrict__ list) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < m; c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t n = counts[c];
        if (n < 2) continue;
        uint32_t* a = list + offsets[c];
        if (n <= 32) {
            for (int64_t x = 1; x < n; ++x) {
                const uint32_t v = a[x];
                int64_t y = x - 1;
                while (y >= 0 && a[y] > v) {
                    a[y + 1] = a[y];
                    --y;
                }
                a[y + 1] = v;
            }
        } else {
            for (int64_t r = n / 2 - 1; r >= 0; --r) sift_down(a, r, n);
            for (int64_t e = n - 1; e > 0; --e) {
                const uint32_t t = a[0];
                a[0] = a[e];
                a[e] = t;
                sift_down(a, 0, e);
            }
        }
    }
}

// One output pixel: the four cells reaching it, in np.add.at order (encodings.py:150-153).
__global__ void bg_gather_kernel(const float2* __restrict__ tg, const float* __restrict__ values, int k,
                                 const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ counts,
                                 const uint32_t* __restrict__ list, double* __restrict__ out,
                                 uint8_t* __restrict__ covered) {
    const int s = 1 << k;
    const int64_t m = (int64_t)s * s;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(p >> k), i = (int)(p & (s - 1));
        double acc = 0.0, wsum = 0.0;
#pragma unroll
        for (int pass = 0; pass < 4; ++pass) {
            const int di = pass & 1, dj = pass >> 1;  // (0,0), (1,0), (0,1), (1,1)
            const int ci = i - di, cj = j - dj;
            if (ci < 0 || cj < 0 || ci > s - 2 || cj > s - 2) continue;
            const int64_t c = (int64_t)cj * s + ci;
            const uint32_t o = offsets[c], n = counts[c];
            for (uint32_t e = 0; e < n; ++e) {
                const uint32_t q = list[o + e];
                const float2 t = tg[q];
                int qi, qj;
                double fx, fy;
                bg_cell(t.x, t.y, s, qi, qj, fx, fy);
                const double gx = di ? fx : __dsub_rn(1.0, fx);
                const double gy = dj ? fy : __dsub_rn(1.0, fy);
                const double w = __dmul_rn(gx, gy);
                acc = __dadd_rn(acc, __dmul_rn(w, (double)values[q]));
                wsum = __dadd_rn(wsum, w);
            }
        }
        const bool cov = wsum > 0.0;
        covered[p] = cov;
        out[p] = cov ? __ddiv_rn(acc, wsum) : 0.0;
    }
}

__host__ __device__ inline size_t edt_env_bytes(int s) {
    return (((size_t)(s + 1) * sizeof(double) + (size_t)2 * s * sizeof(int)) + 255) & ~(size_t)255;
}
constexpr int kEdtSmemMaxK = 13;  // 16 * 8192 bytes = 128 KiB of shared memory
constexpr int kEdtGlobalCtas = 296;

// Column pass of the distance transform: nearest covered row per pixel (-1: none).
__global__ void edt_cols_kernel(const uint8_t* __restrict__ covered, int k, int* __restrict__ nrow) {
    const int s = 1 << k;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= s) return;
    int last = -1;
    for (int j = 0; j < s; ++j) {
        if (covered[(int64_t)j * s + i]) last = j;
        nrow[(int64_t)j * s + i] = last;
    }
    last = -1;
    for (int j = s - 1; j >= 0; --j) {
        const int64_t p = (int64_t)j * s + i;
        if (covered[p]) last = j;
        const int up = nrow[p];
        if (last >= 0 && (up < 0 || last - j < j - up)) nrow[p] = last;
    }
}

// Row pass: one warp per row; lane 0 builds the lower envelope of the column
// parabolas in shared memory (or, above 8192^2 where 16 s bytes exceed it, in a
// per-CTA slice of global scratch `genv`), then the warp fills the row's uncovered
// pixels from their nearest covered pixel.
__global__ void edt_rows_fill_kernel(const uint8_t* __restrict__ covered, const int* __restrict__ nrow, int k,
                                     double* __restrict__ out, unsigned char* genv) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int s = 1 << k;
    unsigned char* env = genv ? genv + (size_t)blockIdx.x * edt_env_bytes(s) : sm;
    double* z = reinterpret_cast<double*>(env);       // s + 1 boundaries
    int* v = reinterpret_cast<int*>(z + (s + 1));      // s apex columns
    int* best = v + s;                                 // s: nearest column per pixel
    const int lane = threadIdx.x;
    for (int j = blockIdx.x; j < s; j += gridDim.x) {
        const int64_t row = (int64_t)j * s;
        bool any = false;
        for (int i = lane; i < s; i += 32) any |= !covered[row + i];
        if (!__any_sync(kFull, any)) continue;
        if (lane == 0) {
            auto f = [&](int q) -> double {
                const int r = nrow[row + q];
                return r < 0 ? -1.0 : (double)(r - j) * (double)(r - j);
            };
            int kk = -1;
            for (int q = 0; q < s; ++q) {
                const double fq = f(q);
                if (fq < 0.0) continue;
                const double hq = fq + (double)q * q;
                double sint = -1e300;
                while (kk >= 0) {
                    const int p = v[kk];
                    const double hp = f(p) + (double)p * p;
                    sint = (hq - hp) / (2.0 * (q - p));
                    if (sint <= z[kk]) --kk;
                    else break;
                }
                ++kk;
                v[kk] = q;
                z[kk] = kk == 0 ? -1e300 : sint;
                z[kk + 1] = 1e300;
            }
            int e = 0;
            for (int i = 0; i < s; ++i) {
                while (z[e + 1] < (double)i) ++e;
                best[i] = v[e];
            }
        }
        __syncwarp();
        for (int i = lane; i < s; i += 32) {
            if (covered[row + i]) continue;
            const int c = best[i];
            out[row + i] = out[(int64_t)nrow[row + c] * s + c];
        }
        __syncwarp();
    }
}

struct BgScratch {
    uint32_t *counts, *offsets, *cursor, *cellof, *list, *bsum;
    uint8_t* covered;
    int* nrow;
    unsigned char* env;  // k > kEdtSmemMaxK: per-CTA envelopes of the row pass
    size_t bytes;
};

static BgScratch bg_layout(int k, void* base) {
    const int64_t m = (int64_t)1 << (2 * k);
    BgScratch b{};
    size_t o = 0;
    auto take = [&](size_t bytes) {
        size_t r = o;
        o = align256(o + bytes);
        return reinterpret_cast<char*>(base) + r;
    };
    b.counts = reinterpret_cast<uint32_t*>(take(4 * m));
    b.offsets = reinterpret_cast<uint32_t*>(take(4 * m));
    b.cursor = reinterpret_cast<uint32_t*>(take(4 * m));
    b.cellof = reinterpret_cast<uint32_t*>(take(4 * m));
    b.list = reinterpret_cast<uint32_t*>(take(4 * m));
    b.bsum = reinterpret_cast<uint32_t*>(take(4 * sort_bsum_words(k)));
    b.covered = reinterpret_cast<uint8_t*>(take(m));
    b.nrow = reinterpret_cast<int*>(take(4 * m));
    b.env = k > kEdtSmemMaxK ? reinterpret_cast<unsigned char*>(take(kEdtGlobalCtas * edt_env_bytes(1 << k))) : nullptr;
    b.bytes = o;
    return b;
}

static unsigned grid_cap(int64_t work, int per_block) {
    int64_t b = (work + per_block - 1) / per_block;
    if (b > 148 * 16) b = 148 * 16;
    return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace inim

using namespace inim;

extern "C" {

size_t inim_deform_background_scratch_bytes(int k) {
    if (k < 1 || k > INIM_MAX_K) return 0;
    return bg_layout(k, nullptr).bytes;
}

int inim_deform_background(const float* targets, const float* values, int k, double* out, float* range2,
                           void* scratch, cudaStream_t stream) {
    if (k < 1 || k > INIM_MAX_K || !targets || !values || !out || !range2 || !scratch) return INIM_EINVAL;
    const int s = 1 << k;
    const int64_t m = (int64_t)s * s;
    BgScratch b = bg_layout(k, scratch);
    const float2* tg = reinterpret_cast<const float2*>(targets);
    INIM_CUDA_TRY(cudaMemsetAsync(b.counts, 0, 4 * m, stream));
    bg_range_init_kernel<<<1, 1, 0, stream>>>(range2);
    bg_cells_kernel<<<grid_cap(m, 256), 256, 0, stream>>>(tg, values, k, m, b.cellof, b.counts, range2);
    int rc = launch_exclusive_scan_u32(b.counts, m, b.bsum, b.offsets, stream);
    if (rc) return rc;
    INIM_CUDA_TRY(cudaMemcpyAsync(b.cursor, b.offsets, 4 * m, cudaMemcpyDeviceToDevice, stream));
    bg_place_kernel<<<grid_cap(m, 256), 256, 0, stream>>>(b.cellof, m, b.cursor, b.list);
    bg_bucket_sort_kernel<<<grid_cap(m, 128), 128, 0, stream>>>(b.offsets, b.counts, m, b.list);
    bg_gather_kernel<<<grid_cap(m, 256), 256, 0, stream>>>(tg, values, k, b.offsets, b.counts, b.list, out,
                                                           b.covered);
    edt_cols_kernel<<<(s + 127) / 128, 128, 0, stream>>>(b.covered, k, b.nrow);
    if (b.env) {
        edt_rows_fill_kernel<<<kEdtGlobalCtas, 32, 0, stream>>>(b.covered, b.nrow, k, out, b.env);
    } else {
        const size_t smem = (size_t)(s + 1) * sizeof(double) + (size_t)2 * s * sizeof(int);
        if (smem > 48 * 1024) INIM_CUDA_TRY(ensure_smem_limit((const void*)edt_rows_fill_kernel, (int)smem));
        edt_rows_fill_kernel<<<(unsigned)(s < 148 * 8 ? s : 148 * 8), 32, smem, stream>>>(b.covered, b.nrow, k, out,
                                                                                        nullptr);
    }
    return (int)cudaGetLastError();
}

}  // extern "C"
