// Point-stream kernels: the density splat (reference density.py:14-27 with pixel_of,
// model.py:189-198) and the bilinear move (mapping.py:207-246 + the clip of
// regularize.py:36).  Both stream the (n, 2) interleaved positions with 16-byte
// vector accesses (two points per float4) and touch the grid through L2.
#include <mutex>
#include <unordered_map>

#include "inim_points.cuh"

namespace inim {

// Warp-aggregated integer atomics: lanes hitting the same pixel in one step are
// merged (__match_any_sync) and the leader issues one red.add for the group.
__device__ __forceinline__ void splat_one(uint32_t* counts, int pix) {
    const unsigned mask = __match_any_sync(kFull, pix);
    const int lane = threadIdx.x & 31;
    if (pix >= 0 && lane == __ffs(mask) - 1) atomicAdd(counts + pix, (uint32_t)__popc(mask));
}

// The iteration's splat.  Points are in no particular spatial order, so lanes rarely
// share a pixel: plain red.global.add (no return) per point, two points per 16-byte
// load.  zero0/zero1: per-iteration device scalars (max excursion, max displacement)
// cleared here so the iteration needs no separate reset launch.
__global__ void __launch_bounds__(256) splat_f32_kernel(const float4* __restrict__ pts2, const float* __restrict__ pts,
                                                        int64_t n, int k, uint32_t* __restrict__ counts,
                                                        const int* state, float* zero0, float* zero1) {
    pdl_enter();
    if (state && state[0]) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (zero0) *zero0 = 0.f;
        if (zero1) *zero1 = 0.f;
    }
    const int s = 1 << k;
    const int64_t npair = n >> 1;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    constexpr int U = 4;  // four 16-byte loads in flight per thread before its atomics
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npair; p += U * stride) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (p + u * stride < npair) v[u] = __ldcs(pts2 + p + u * stride);  // streamed: read once per splat
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (p + u * stride < npair) {
                atomicAdd(counts + pixel_of(v[u].y, s) * s + pixel_of(v[u].x, s), 1u);
                atomicAdd(counts + pixel_of(v[u].w, s) * s + pixel_of(v[u].z, s), 1u);
            }
        }
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const float x = pts[2 * (n - 1)], y = pts[2 * (n - 1) + 1];
        atomicAdd(counts + pixel_of(y, s) * s + pixel_of(x, s), 1u);
    }
}

__global__ void __launch_bounds__(256) splat_f64_kernel(const double* __restrict__ pts, int64_t n, int k,
                                                        uint32_t* __restrict__ counts) {
    const int s = 1 << k;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t iters = (n + stride - 1) / stride;
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t it = 0; it < iters; ++it, p += stride) {
        int pix = -1;
        if (p < n) {
            const double2 v = reinterpret_cast<const double2*>(pts)[p];
            pix = pixel_of(v.y, s) * s + pixel_of(v.x, s);
        }
        splat_one(counts, pix);
    }
}

// PAIRS: `tg` is the paired (s, s, 4) field layout (bilinear_pairs), else (s, s, 2).
template <bool PAIRS>
__device__ __forceinline__ void move_point(const float* tg, int s, float x, float y, float& ox, float& oy) {
    if (PAIRS) bilinear_pairs(reinterpret_cast<const float4*>(tg), s, x, y, ox, oy);
    else bilinear<float>(reinterpret_cast<const float2*>(tg), s, x, y, ox, oy);
}

template <bool PAIRS>
__global__ void __launch_bounds__(256) sample_f32_kernel(const float* __restrict__ tg, int k,
                                                         const float4* __restrict__ in2, const float* __restrict__ in,
                                                         float4* __restrict__ out2, float* __restrict__ out, int64_t n,
                                                         int clip, float* max_disp, const int* state,
                                                         uint32_t* __restrict__ splat_next, float* zn0, float* zn1) {
    pdl_enter();
    const bool stopped = state && state[0];
    const int s = 1 << k;
    // fused splat of the next iteration (its count buffer was cleared by this
    // iteration's smoothing) and the reset of the next iteration's device scalars
    if (splat_next && !stopped && blockIdx.x == 0 && threadIdx.x == 0) {
        if (zn0) *zn0 = 0.f;
        if (zn1) *zn1 = 0.f;
    }
    const int64_t npair = n >> 1;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    float md = 0.f;
    // U pairs of points (U 16-byte loads) per thread per step, all gathers in flight
    constexpr int U = 2;
    for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p0 < npair; p0 += U * stride) {
        float4 v[U], o[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t q = p0 + u * stride;
            v[u] = q < npair ? __ldcs(in2 + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (stopped) {
                o[u] = v[u];  // keep the ping-pong buffers consistent after a displacement stop
                continue;
            }
            move_point<PAIRS>(tg, s, v[u].x, v[u].y, o[u].x, o[u].y);
            move_point<PAIRS>(tg, s, v[u].z, v[u].w, o[u].z, o[u].w);
            if (clip) {
                o[u].x = clip01(o[u].x); o[u].y = clip01(o[u].y); o[u].z = clip01(o[u].z); o[u].w = clip01(o[u].w);
            }
            if (p0 + u * stride < npair)
                md = fmaxf(md, fmaxf(fmaxf(fabsf(o[u].x - v[u].x), fabsf(o[u].y - v[u].y)),
                                     fmaxf(fabsf(o[u].z - v[u].z), fabsf(o[u].w - v[u].w))));
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (p0 + u * stride < npair) __stcs(out2 + p0 + u * stride, o[u]);
        if (splat_next && !stopped) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (p0 + u * stride < npair) {
                    atomicAdd(splat_next + pixel_of(o[u].y, s) * s + pixel_of(o[u].x, s), 1u);
                    atomicAdd(splat_next + pixel_of(o[u].w, s) * s + pixel_of(o[u].z, s), 1u);
                }
            }
        }
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const float x = in[2 * (n - 1)], y = in[2 * (n - 1) + 1];
        float ox = x, oy = y;
        if (!stopped) {
            move_point<PAIRS>(tg, s, x, y, ox, oy);
            if (clip) { ox = clip01(ox); oy = clip01(oy); }
            md = fmaxf(md, fmaxf(fabsf(ox - x), fabsf(oy - y)));
        }
        out[2 * (n - 1)] = ox;
        out[2 * (n - 1) + 1] = oy;
        if (splat_next && !stopped) atomicAdd(splat_next + pixel_of(oy, s) * s + pixel_of(ox, s), 1u);
    }
    if (max_disp && !stopped) {
        md = warp_max(md);
        if ((threadIdx.x & 31) == 0 && md > 0.f) atomic_max_nonneg(max_disp, md);
    }
}

__global__ void __launch_bounds__(256) sample_f64_kernel(const float2* __restrict__ tg, int k,
                                                         const double* __restrict__ in, double* __restrict__ out,
                                                         int64_t n, int clip) {
    const int s = 1 << k;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) {
        const double2 v = reinterpret_cast<const double2*>(in)[p];
        double ox, oy;
        bilinear<double>(tg, s, v.x, v.y, ox, oy);
        if (clip) { ox = clip01(ox); oy = clip01(oy); }
        reinterpret_cast<double2*>(out)[p] = make_double2(ox, oy);
    }
}

// ---------------------------------------------------------------- spatial point order
// A counting sort of the points by cell (a 2^cs x 2^cs grid of cells, at most 64 per
// side), done once per run: consecutive points (one warp) then fall in the same cell, so
// the bilinear gathers hit L1 and the splat's atomics share addresses.  Both passes
// privatise the histogram in shared memory (one CTA per contiguous chunk of points), so
// hot cells of clustered data cost one global atomic per CTA, not one per point.  No
// result depends on the order (integer counts, independent per-point moves); frames are
// scattered back through `perm`.
__host__ __device__ inline int cells_log2(int k) { return k < 6 ? k : 6; }

__device__ __forceinline__ int cell_of(float x, float y, int k) {
    const int s = 1 << k;
    const int cs = cells_log2(k);
    const int sh = k - cs;
    return (pixel_of(y, s) >> sh) * (1 << cs) + (pixel_of(x, s) >> sh);
}

// pass 1: per-CTA shared-memory histogram of its chunk, flushed with one atomic per bin
__global__ void __launch_bounds__(256) cell_hist_kernel(const float2* __restrict__ pts, int64_t n, int k,
                                                        int* __restrict__ hist, int ncells, int64_t chunk) {
    extern __shared__ int cnt[];
    for (int i = threadIdx.x; i < ncells; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    const int64_t p0 = (int64_t)blockIdx.x * chunk, p1 = min(n, p0 + chunk);
    for (int64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
        const float2 v = pts[p];
        atomicAdd(cnt + cell_of(v.x, v.y, k), 1);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < ncells; i += blockDim.x)
        if (cnt[i]) atomicAdd(hist + i, cnt[i]);
}

// pass 2: the CTA reserves one contiguous block per bin (one atomic each), then places
// its points with shared-memory cursors
__global__ void __launch_bounds__(256) cell_place_kernel(const float2* __restrict__ pts, int64_t n, int k,
                                                         int* __restrict__ cursor, int ncells, int64_t chunk,
                                                         float2* __restrict__ sorted, int* __restrict__ perm) {
    extern __shared__ int sm[];
    int* cnt = sm;
    int* base = sm + ncells;
    for (int i = threadIdx.x; i < ncells; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    const int64_t p0 = (int64_t)blockIdx.x * chunk, p1 = min(n, p0 + chunk);
    for (int64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
        const float2 v = pts[p];
        atomicAdd(cnt + cell_of(v.x, v.y, k), 1);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < ncells; i += blockDim.x) {
        base[i] = cnt[i] ? atomicAdd(cursor + i, cnt[i]) : 0;
        cnt[i] = 0;
    }
    __syncthreads();
    for (int64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
        const float2 v = pts[p];
        const int c = cell_of(v.x, v.y, k);
        const int slot = base[c] + atomicAdd(cnt + c, 1);
        sorted[slot] = v;
        perm[slot] = (int)p;
    }
}

// Exclusive scan of the cell histogram, one block (cells <= 65536 for k <= 12,
// 1M for k = 14: loops over tiles).
__global__ void __launch_bounds__(1024) cell_scan_kernel(int* __restrict__ hist, int ncells) {
    __shared__ int sh[33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int carry = 0;
    for (int base = 0; base < ncells; base += blockDim.x) {
        const int i = base + threadIdx.x;
        const int v = i < ncells ? hist[i] : 0;
        int inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(kFull, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) sh[w] = inc;
        __syncthreads();
        if (w == 0) {
            const int t = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0;
            int ti = t;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(kFull, ti, o);
                if (lane >= o) ti += u;
            }
            sh[lane] = ti - t;
            if (lane == 31) sh[32] = ti;
        }
        __syncthreads();
        if (i < ncells) hist[i] = carry + sh[w] + inc - v;
        carry += sh[32];
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) unpermute_kernel(const float2* __restrict__ sorted, const int* __restrict__ perm,
                                                        int64_t n, float2* __restrict__ out) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
        out[perm[q]] = sorted[q];
}

__global__ void cast_f64_f32_kernel(const double* __restrict__ in, float* __restrict__ out, int64_t count) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < count; q += (int64_t)gridDim.x * blockDim.x)
        out[q] = (float)in[q];
}

__global__ void cast_f32_f64_kernel(const float* __restrict__ in, double* __restrict__ out, int64_t count) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < count; q += (int64_t)gridDim.x * blockDim.x)
        out[q] = (double)in[q];
}

// --------------------------------------------------------------------------- launchers
static int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// Grid of at most one full wave: blocks x threads covers `work` items (capped at what is
// co-resident on all SMs given the kernel's registers / shared memory).
static unsigned resident_grid(const void* kernel, int64_t work, int threads, size_t smem = 0) {
    static std::mutex mu;
    static std::unordered_map<const void*, int> occ;
    int per_sm = 0;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = occ.find(kernel);
        if (it == occ.end()) {
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) != cudaSuccess ||
                per_sm < 1)
                per_sm = 1;
            occ[kernel] = per_sm;
        } else {
            per_sm = it->second;
        }
    }
    int64_t blocks = (work + threads - 1) / threads;
    const int64_t cap = (int64_t)sm_count() * per_sm;
    if (blocks > cap) blocks = cap;
    return (unsigned)(blocks < 1 ? 1 : blocks);
}

static unsigned grid_for(int64_t work, int per_block) {
    int64_t blocks = (work + per_block - 1) / per_block;
    const int64_t cap = (int64_t)sm_count() * 8;  // 8 resident 256-thread CTAs per SM
    if (blocks > cap) blocks = cap;
    return (unsigned)(blocks < 1 ? 1 : blocks);
}

int launch_splat_f32(const float* pts, int64_t n, int k, uint32_t* counts, const int* state, cudaStream_t st,
                     float* zero0, float* zero1) {
    const int64_t npair = n >> 1;
    INIM_CUDA_TRY(launch_pdl(splat_f32_kernel, dim3(grid_for(npair > 0 ? npair : 1, 256)), dim3(256), 0, st,
                             reinterpret_cast<const float4*>(pts), pts, n, k, counts, state, zero0, zero1));
    prof_mark(st, "splat");
    return (int)cudaGetLastError();
}

int cell_count(int k) { return 1 << (2 * cells_log2(k)); }

// hist: cell_count(k) ints (zeroed here, then the cursors); perm: n ints; sorted: n
// float2.  `rank` is unused (kept for the workspace layout).
int launch_sort_points(const float* pts, int64_t n, int k, int* hist, int* rank, float* sorted, int* perm,
                       cudaStream_t st) {
    (void)rank;
    const int nc = cell_count(k);
    INIM_CUDA_TRY(cudaMemsetAsync(hist, 0, sizeof(int) * nc, st));
    const int ctas = sm_count() * 2;
    const int64_t chunk = (n + ctas - 1) / ctas;
    const float2* p2 = reinterpret_cast<const float2*>(pts);
    cell_hist_kernel<<<ctas, 256, sizeof(int) * nc, st>>>(p2, n, k, hist, nc, chunk);
    cell_scan_kernel<<<1, 1024, 0, st>>>(hist, nc);
    cell_place_kernel<<<ctas, 256, 2 * sizeof(int) * nc, st>>>(p2, n, k, hist, nc, chunk,
                                                               reinterpret_cast<float2*>(sorted), perm);
    prof_mark(st, "sort_points");
    return (int)cudaGetLastError();
}

int launch_unpermute(const float* sorted, const int* perm, int64_t n, float* out, cudaStream_t st) {
    unpermute_kernel<<<grid_for(n > 0 ? n : 1, 256), 256, 0, st>>>(reinterpret_cast<const float2*>(sorted), perm, n,
                                                                    reinterpret_cast<float2*>(out));
    prof_mark(st, "unpermute");
    return (int)cudaGetLastError();
}

int launch_splat_f64(const double* pts, int64_t n, int k, uint32_t* counts, cudaStream_t st) {
    splat_f64_kernel<<<grid_for(n > 0 ? n : 1, 256), 256, 0, st>>>(pts, n, k, counts);
    return (int)cudaGetLastError();
}

int launch_sample_f32(const float* tg, int k, const float* in, float* out, int64_t n, int clip, float* max_disp,
                      const int* state, cudaStream_t st, bool pairs, uint32_t* splat_next, float* zn0, float* zn1) {
    const int64_t npair = n >> 1;
    auto kern = pairs ? sample_f32_kernel<true> : sample_f32_kernel<false>;
    INIM_CUDA_TRY(launch_pdl(kern, dim3(resident_grid((const void*)kern, npair > 0 ? npair : 1, 256)), dim3(256), 0,
                             st, tg, k, reinterpret_cast<const float4*>(in), in, reinterpret_cast<float4*>(out), out, n,
                             clip, max_disp, state, splat_next, zn0, zn1));
    prof_mark(st, "sample");
    return (int)cudaGetLastError();
}

int launch_sample_f64(const float* tg, int k, const double* in, double* out, int64_t n, int clip, cudaStream_t st) {
    sample_f64_kernel<<<grid_for(n > 0 ? n : 1, 256), 256, 0, st>>>(reinterpret_cast<const float2*>(tg), k, in, out,
                                                                     n, clip);
    return (int)cudaGetLastError();
}

int launch_cast_f64_f32(const double* in, float* out, int64_t count, cudaStream_t st) {
    cast_f64_f32_kernel<<<grid_for(count > 0 ? count : 1, 256), 256, 0, st>>>(in, out, count);
    return (int)cudaGetLastError();
}

int launch_cast_f32_f64(const float* in, double* out, int64_t count, cudaStream_t st) {
    cast_f32_f64_kernel<<<grid_for(count > 0 ? count : 1, 256), 256, 0, st>>>(in, out, count);
    return (int)cudaGetLastError();
}

}  // namespace inim
