// Layout-quality metrics on the device (reference metrics.py): the occupancy statistics
// of a frame read off its splat counts, and the neighbourhood metrics of a (sub)sample.
//
// Every kernel here produces INTEGERS (occupied pixels, sum of squared bin counts,
// trustworthiness penalty sum, preserved pair count) accumulated with 64-bit integer
// atomics, so the results are order-independent and, for identical coordinates,
// identical to the reference's own integer intermediates.  The host turns them into
// the reference's floats with the reference's formulas (metrics.py:59,71,112-113,144).
#include <type_traits>

#include "inim_internal.cuh"

namespace inim {

typedef unsigned long long u64;

template <typename T>
INIM_DEV T block_sum(T v, T* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    T r = 0;
    if (threadIdx.x == 0)
        for (int q = 0; q < (int)(blockDim.x >> 5); ++q) r += red[q];
    return r;  // valid in thread 0
}

// ---------------------------------------------------------------- occupancy statistics
// binned_stddev (metrics.py:46-59): 4x4-pixel bins on the 2^k grid; the bin counts are
// sums of the per-pixel counts.  overplotting (metrics.py:62-71): occupied pixels =
// nonzero counts.  out[0] += occupied pixels, out[1] += sum over bins of count^2,
// out[2] += sum of counts (= n).  One thread per bin; each of its four rows is one
// 16-byte load, consecutive threads read consecutive bins of a row (coalesced).
// T: uint32 counts, or float32 counts (exact integers) from the moves' 16-byte reductions
template <typename T>
__global__ void __launch_bounds__(256) frame_stats_kernel(const T* __restrict__ counts, int k, u64* out,
                                                          int64_t zslab, int64_t zout) {
    pdl_enter();
    counts = zoff(counts, zslab_off(zslab));  // plot blockIdx.z of a batch
    out += blockIdx.z * zout;
    __shared__ u64 red[8];
    const int s = 1 << k;
    u64 occ = 0, sq = 0, tot = 0;
    if (k >= 2) {
        const int bps = s >> 2;  // bins per side
        const int64_t nb = (int64_t)bps * bps;
        for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
            const int bi = (int)(b % bps), bj = (int)(b / bps);
            const uint4* row = reinterpret_cast<const uint4*>(counts + (size_t)(4 * bj) * s) + bi;
            uint32_t bin = 0;
            int nz = 0;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                uint4 v = __ldg(row + (size_t)r * (s >> 2));
                if (std::is_same<T, float>::value)
                    v = make_uint4((uint32_t)__uint_as_float(v.x), (uint32_t)__uint_as_float(v.y),
                                   (uint32_t)__uint_as_float(v.z), (uint32_t)__uint_as_float(v.w));
                bin += v.x + v.y + v.z + v.w;
                nz += (v.x != 0) + (v.y != 0) + (v.z != 0) + (v.w != 0);
            }
            occ += nz;
            tot += bin;
            sq += (u64)bin * bin;
        }
    } else if (blockIdx.x == 0 && threadIdx.x < s * s) {  // 1x1 and 2x2 grids: no bins
        const uint32_t c = (uint32_t)counts[threadIdx.x];
        occ = c != 0;
        tot = c;
    }
    const u64 a = block_sum(occ, red);
    const u64 b2 = block_sum(sq, red);
    const u64 c3 = block_sum(tot, red);
    if (threadIdx.x == 0) {
        if (a) atomicAdd(out, a);
        if (b2) atomicAdd(out + 1, b2);
        if (c3) atomicAdd(out + 2, c3);
    }
}

// ------------------------------------------------------------------- subsample gather
// out[q] = pts[perm(rows(q))] widened to float64 (exact); rows = the fixed-seed pick of
// metrics.py:139-141 (NULL = identity), perm = input row -> slot of a pixel-sorted
// point buffer (NULL = identity).
template <typename T>
__global__ void gather_points_kernel(const T* __restrict__ pts, const int64_t* __restrict__ rows,
                                     const uint32_t* __restrict__ perm, int64_t m, double* __restrict__ out) {
    pdl_enter();
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = rows ? rows[q] : q;
        if (perm) r = perm[r];
        out[2 * q] = (double)pts[2 * r];
        out[2 * q + 1] = (double)pts[2 * r + 1];
    }
}

// Squared distance exactly as numpy forms it (metrics.py:82-83): the differences, then
// dx*dx + dy*dy, each step rounded (no FMA contraction).
INIM_DEV double dist2(double xi, double yi, const double* p, int64_t j) {
    const double dx = __dsub_rn(xi, p[2 * j]);
    const double dy = __dsub_rn(yi, p[2 * j + 1]);
    return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
}

// (d, j) < (e, l) in the order of a stable argsort of the distance row (metrics.py:85).
INIM_DEV bool key_less(double d, int64_t j, double e, int64_t l) { return d < e || (d == e && j < l); }

// ------------------------------------------------------------------ trustworthiness
// metrics.py:74-113.  For sample i: the n_neighbors nearest OTHER samples in the
// deformed layout (ties -> lower index), and for each of them its rank in i's ordering
// of the original layout (self = rank 0, so rank = 1 + #{l != i closer}).  The
// penalty sum  sum max(0, rank - n_neighbors)  is exact in 64-bit integers.
// One CTA per sample; the selection is n_neighbors rounds of a block arg-min over keys
// strictly after the previous round's key.
__global__ void __launch_bounds__(256) trust_kernel(const double* __restrict__ orig, const double* __restrict__ moved,
                                                    int64_t n, int nn, u64* out) {
    pdl_enter();
    extern __shared__ int64_t sel[];  // [nn] selected indices, then [nn] double dist (orig)
    double* dsel = reinterpret_cast<double*>(sel + nn);
    __shared__ double wd[8];
    __shared__ int64_t wj[8];
    __shared__ unsigned int cnt_sh[1];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const double mxi = moved[2 * i], myi = moved[2 * i + 1];
        const double oxi = orig[2 * i], oyi = orig[2 * i + 1];
        double last_d = -1.0;
        int64_t last_j = -1;
        for (int r = 0; r < nn; ++r) {
            double bd = __longlong_as_double(0x7ff0000000000000LL);  // +inf
            int64_t bj = INT64_MAX;
            for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
                if (j == i) continue;
                const double d = dist2(mxi, myi, moved, j);
                if (key_less(last_d, last_j, d, j) && key_less(d, j, bd, bj)) {
                    bd = d;
                    bj = j;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double od = __shfl_xor_sync(kFull, bd, o);
                const int64_t oj = __shfl_xor_sync(kFull, bj, o);
                if (key_less(od, oj, bd, bj)) {
                    bd = od;
                    bj = oj;
                }
            }
            __syncthreads();
            if (lane == 0) {
                wd[w] = bd;
                wj[w] = bj;
            }
            __syncthreads();
            bd = wd[0];
            bj = wj[0];
            for (int q = 1; q < nw; ++q)
                if (key_less(wd[q], wj[q], bd, bj)) {
                    bd = wd[q];
                    bj = wj[q];
                }
            if (threadIdx.x == 0) {
                sel[r] = bj;
                dsel[r] = dist2(oxi, oyi, orig, bj);
            }
            last_d = bd;
            last_j = bj;
        }
        __syncthreads();
        // original-layout rank of every selected neighbour
        u64 pen = 0;
        for (int r = 0; r < nn; ++r) {
            const int64_t jr = sel[r];
            const double dr = dsel[r];
            unsigned int c = 0;
            for (int64_t l = threadIdx.x; l < n; l += blockDim.x) {
                if (l == i) continue;
                c += key_less(dist2(oxi, oyi, orig, l), l, dr, jr);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
            if (threadIdx.x == 0) cnt_sh[0] = 0;
            __syncthreads();
            if (lane == 0) atomicAdd(cnt_sh, c);
            __syncthreads();
            const int64_t rank = 1 + (int64_t)cnt_sh[0];
            if (rank > nn) pen += (u64)(rank - nn);
            __syncthreads();
        }
        if (threadIdx.x == 0 && pen) atomicAdd(out, pen);
        __syncthreads();
    }
}

// --------------------------------------------------------------- orthogonal ordering
// metrics.py:116-144: pairs i < j whose x-order sign and y-order sign agree between the
// two layouts.  sign(a - b) of finite doubles is the comparison of a and b.
INIM_DEV int sgn_cmp(double a, double b) { return (a > b) - (a < b); }

__global__ void __launch_bounds__(256) order_pairs_kernel(const double* __restrict__ orig,
                                                          const double* __restrict__ moved, int64_t n, u64* out) {
    pdl_enter();
    __shared__ u64 red[8];
    u64 kept = 0;
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const double oxi = orig[2 * i], oyi = orig[2 * i + 1], mxi = moved[2 * i], myi = moved[2 * i + 1];
        for (int64_t j = i + 1 + threadIdx.x; j < n; j += blockDim.x) {
            const bool sx = sgn_cmp(oxi, orig[2 * j]) == sgn_cmp(mxi, moved[2 * j]);
            const bool sy = sgn_cmp(oyi, orig[2 * j + 1]) == sgn_cmp(myi, moved[2 * j + 1]);
            kept += (sx && sy);
        }
    }
    const u64 t = block_sum(kept, red);
    if (threadIdx.x == 0 && t) atomicAdd(out, t);
}

static int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

static unsigned blocks_for(int64_t work, int per_block, int per_sm) {
    int64_t b = (work + per_block - 1) / per_block;
    const int64_t cap = (int64_t)num_sms() * per_sm;
    if (b > cap) b = cap;
    return (unsigned)(b < 1 ? 1 : b);
}

// zout: u64 between consecutive plots' outputs of a batch
int launch_frame_stats(const uint32_t* counts, int k, u64* out3, cudaStream_t st, const Bat& bt, int64_t zout,
                       bool f32_counts) {
    const int64_t bins = k >= 2 ? ((int64_t)1 << (2 * k - 4)) : 1;
    const dim3 grid(blocks_for(bins, 256, bt.B > 1 ? 1 : 8), 1, bt.B);
    if (f32_counts)
        INIM_CUDA_TRY(launch_pdl(frame_stats_kernel<float>, grid, dim3(256), 0, st,
                                 reinterpret_cast<const float*>(counts), k, out3, bt.slab, zout));
    else
        INIM_CUDA_TRY(launch_pdl(frame_stats_kernel<uint32_t>, grid, dim3(256), 0, st, counts, k, out3, bt.slab, zout));
    prof_mark(st, "frame_stats");
    return (int)cudaGetLastError();
}

int launch_gather_points(const void* pts, int is_f64, const int64_t* rows, const uint32_t* perm, int64_t m,
                         double* out, cudaStream_t st) {
    const dim3 g(blocks_for(m, 256, 4));
    if (is_f64)
        INIM_CUDA_TRY(launch_pdl(gather_points_kernel<double>, g, dim3(256), 0, st, static_cast<const double*>(pts),
                                 rows, perm, m, out));
    else
        INIM_CUDA_TRY(launch_pdl(gather_points_kernel<float>, g, dim3(256), 0, st, static_cast<const float*>(pts),
                                 rows, perm, m, out));
    prof_mark(st, "gather_points");
    return (int)cudaGetLastError();
}

int launch_trust(const double* orig, const double* moved, int64_t n, int nn, u64* out, cudaStream_t st) {
    const size_t smem = (size_t)nn * (sizeof(int64_t) + sizeof(double));
    if (smem > 48 * 1024) {
        INIM_CUDA_TRY(cudaFuncSetAttribute(trust_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    const int64_t ctas = n < (int64_t)num_sms() * 64 ? n : (int64_t)num_sms() * 64;
    INIM_CUDA_TRY(launch_pdl(trust_kernel, dim3((unsigned)(ctas > 0 ? ctas : 1)), dim3(256), smem, st, orig, moved, n,
                             nn, out));
    prof_mark(st, "trust");
    return (int)cudaGetLastError();
}

int launch_order_pairs(const double* orig, const double* moved, int64_t n, u64* out, cudaStream_t st) {
    const int64_t ctas = n < (int64_t)num_sms() * 64 ? n : (int64_t)num_sms() * 64;
    INIM_CUDA_TRY(launch_pdl(order_pairs_kernel, dim3((unsigned)(ctas > 0 ? ctas : 1)), dim3(256), 0, st, orig, moved,
                             n, out));
    prof_mark(st, "order_pairs");
    return (int)cudaGetLastError();
}

}  // namespace inim
