// Point-stream kernels: the density splat (reference density.py:14-27 with pixel_of,
// model.py:189-198) and the bilinear move (mapping.py:207-246 + the clip of
// regularize.py:36).  Both stream the (n, 2) interleaved positions with 16-byte
// vector accesses (two points per float4) and touch the grid through L2.
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "inim_points.cuh"

#ifndef INIM_BATCH_MOVE_U
#define INIM_BATCH_MOVE_U 4
#endif


namespace inim {

// 16-byte float reduction (REDG.E.ADD.F32x4): four adjacent counts in one L2 request.
__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

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
__global__ void __launch_bounds__(256) splat_f32_kernel(const float* __restrict__ pts, int64_t n, int k,
                                                        uint32_t* __restrict__ counts, const int* state, float* zero0,
                                                        float* zero1, int64_t zpts, int64_t zslab) {
    pdl_enter();
    state = zstate(state, zslab);
    if (state && state[0]) return;
    {  // plot blockIdx.z of a batch
        const int64_t zo = zslab_off(zslab);
        pts += blockIdx.z * zpts;
        counts = zoff(counts, zo);
        zero0 = zoff_opt(zero0, zo);
        zero1 = zoff_opt(zero1, zo);
    }
    const float4* __restrict__ pts2 = reinterpret_cast<const float4*>(pts);
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

// Move of U point pairs per thread (pair u at index q[u], valid when ok[u]) and the
// fused splat of the next iteration: shared by the grid-stride move and the pipelined
// batch move.  Returns the thread's largest displacement.
template <bool PAIRS, int U, bool GATHER_FIRST = false>
__device__ __forceinline__ float move_pairs(const float* tg, int s, const float4 (&v)[U], const int64_t (&q)[U],
                                            const bool (&ok)[U], float4* __restrict__ out2, int clip, bool stopped,
                                            uint32_t* __restrict__ splat_next, int agg) {
    float4 o[U];
    float md = 0.f;
    if (GATHER_FIRST && !stopped) {
        // every gather of the thread's 2U points in flight before the first blend
        Tap4 t[U][2];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            t[u][0] = bilinear_fetch<PAIRS>(tg, s, v[u].x, v[u].y);
            t[u][1] = bilinear_fetch<PAIRS>(tg, s, v[u].z, v[u].w);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            bilinear_blend(t[u][0], o[u].x, o[u].y);
            bilinear_blend(t[u][1], o[u].z, o[u].w);
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if (stopped) {
            o[u] = v[u];  // keep the ping-pong buffers consistent after a displacement stop
            continue;
        }
        if (!GATHER_FIRST) {
            move_point<PAIRS>(tg, s, v[u].x, v[u].y, o[u].x, o[u].y);
            move_point<PAIRS>(tg, s, v[u].z, v[u].w, o[u].z, o[u].w);
        }
        if (clip) {
            o[u].x = clip01(o[u].x); o[u].y = clip01(o[u].y); o[u].z = clip01(o[u].z); o[u].w = clip01(o[u].w);
        }
        if (ok[u])
            md = fmaxf(md, fmaxf(fmaxf(fabsf(o[u].x - v[u].x), fabsf(o[u].y - v[u].y)),
                                 fmaxf(fabsf(o[u].z - v[u].z), fabsf(o[u].w - v[u].w))));
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
        if (ok[u]) __stcs(out2 + q[u], o[u]);
    if (splat_next && !stopped) {
        if (agg == 2) {
            // float counts (exact integers below 2^24): lanes whose points fall in the
            // same aligned group of four pixels merge into ONE 16-byte reduction
            // (red.global.add.v4.f32), so the L2 sees a request per group, not per
            // point (the splat's bound is the L2 reduction request rate)
            const unsigned am = __activemask();
            const int lane = threadIdx.x & 31;
            float* fc = reinterpret_cast<float*>(splat_next);
#pragma unroll
            for (int u = 0; u < U; ++u) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int pix = ok[u] ? pixel_of(h ? o[u].w : o[u].y, s) * s + pixel_of(h ? o[u].z : o[u].x, s)
                                          : -1;
                    const int g4 = pix >> 2;  // -1 for padding lanes
                    const unsigned grp = __match_any_sync(am, g4);
                    const int sub = pix & 3;
                    const unsigned b1 = __ballot_sync(am, ok[u] && sub == 1);
                    const unsigned b2 = __ballot_sync(am, ok[u] && sub == 2);
                    const unsigned b3 = __ballot_sync(am, ok[u] && sub == 3);
                    if (ok[u] && lane == __ffs(grp) - 1) {
                        const int c1 = __popc(grp & b1), c2 = __popc(grp & b2), c3 = __popc(grp & b3);
                        red_add_v4(fc + 4 * (int64_t)g4, (float)(__popc(grp) - c1 - c2 - c3), (float)c1,
                                   (float)c2, (float)c3);
                    }
                }
            }
        } else if (agg) {  // points in pixel order: lanes sharing a pixel merge into one red.add
            const unsigned am = __activemask();
            const int lane = threadIdx.x & 31;
#pragma unroll
            for (int u = 0; u < U; ++u) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int pix = ok[u] ? pixel_of(h ? o[u].w : o[u].y, s) * s + pixel_of(h ? o[u].z : o[u].x, s)
                                          : -1;
                    const unsigned grp = __match_any_sync(am, pix);
                    if (ok[u] && lane == __ffs(grp) - 1) atomicAdd(splat_next + pix, (uint32_t)__popc(grp));
                }
            }
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (ok[u]) {
                    atomicAdd(splat_next + pixel_of(o[u].y, s) * s + pixel_of(o[u].x, s), 1u);
                    atomicAdd(splat_next + pixel_of(o[u].w, s) * s + pixel_of(o[u].z, s), 1u);
                }
            }
        }
    }
    return md;
}

// The last point of an odd n (one thread).
template <bool PAIRS>
__device__ __forceinline__ float move_odd_tail(const float* tg, int s, const float* in, float* out, int64_t n, int clip,
                                               bool stopped, uint32_t* splat_next, int agg) {
    const float x = in[2 * (n - 1)], y = in[2 * (n - 1) + 1];
    float ox = x, oy = y, md = 0.f;
    if (!stopped) {
        move_point<PAIRS>(tg, s, x, y, ox, oy);
        if (clip) { ox = clip01(ox); oy = clip01(oy); }
        md = fmaxf(fabsf(ox - x), fabsf(oy - y));
    }
    out[2 * (n - 1)] = ox;
    out[2 * (n - 1) + 1] = oy;
    if (splat_next && !stopped) {
        const int pix = pixel_of(oy, s) * s + pixel_of(ox, s);
        if (agg == 2) atomicAdd(reinterpret_cast<float*>(splat_next) + pix, 1.f);
        else atomicAdd(splat_next + pix, 1u);
    }
    return md;
}

// BATCH: plot offsets of a SPLOM batch (grid.z), a separate instantiation so the
// single-plot move keeps its register budget.
template <bool PAIRS, int U, bool BATCH>
__global__ void __launch_bounds__(256) sample_f32_kernel(const float* __restrict__ tg, int k,
                                                         const float4* __restrict__ in2, const float* __restrict__ in,
                                                         float4* __restrict__ out2, float* __restrict__ out, int64_t n,
                                                         int clip, float* max_disp, const int* state,
                                                         uint32_t* __restrict__ splat_next, float* zn0, float* zn1,
                                                         int agg, int64_t zin, int64_t zout, int64_t zslab) {
    pdl_enter();
    if (BATCH) {  // plot blockIdx.z of a batch
        const int64_t zo = zslab_off(zslab);
        tg = zoff(tg, zo);
        in += blockIdx.z * zin;
        out += blockIdx.z * zout;
        in2 = reinterpret_cast<const float4*>(in);
        out2 = reinterpret_cast<float4*>(out);
        max_disp = zoff_opt(max_disp, zo);
        splat_next = zoff_opt(splat_next, zo);
        zn0 = zoff_opt(zn0, zo);
        zn1 = zoff_opt(zn1, zo);
        state = zstate(state, zslab);
    }
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
    for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p0 < npair; p0 += U * stride) {
        float4 v[U];
        int64_t q[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            q[u] = p0 + u * stride;
            ok[u] = q[u] < npair;
            v[u] = ok[u] ? __ldcs(in2 + q[u]) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        md = fmaxf(md, move_pairs<PAIRS, U>(tg, s, v, q, ok, out2, clip, stopped, splat_next, agg));
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0)
        md = fmaxf(md, move_odd_tail<PAIRS>(tg, s, in, out, n, clip, stopped, splat_next, agg));
    if (max_disp && !stopped) {
        md = warp_max(md);
        if ((threadIdx.x & 31) == 0 && md > 0.f) atomic_max_nonneg(max_disp, md);
    }
}

// Batch move with the point pairs staged by bulk copies: each CTA walks chunks of
// kMoveChunk pairs of its plot (grid.x CTAs per plot, grid-stride; two pairs per thread
// per chunk and eight chunks per CTA measured best), and one thread
// issues the cp.async.bulk of chunk i + 1 into the other half of a two-slot shared
// buffer before the CTA works on chunk i, so the positions' HBM latency overlaps the
// previous chunk's gathers (the grid-stride move exposes it once per thread).  Same
// per-point arithmetic and splat as sample_f32_kernel: bit-identical results.
#ifndef INIM_GATHER_FIRST
#define INIM_GATHER_FIRST 1  // pipelined move: all gathers of a thread issued before the blends
#endif
#ifndef INIM_BULK_U
#define INIM_BULK_U 2
#endif
constexpr int kMoveU = INIM_BULK_U;
constexpr int kMoveChunk = 256 * kMoveU;  // pairs per chunk (8 KB)

// Six CTAs per SM (40 registers): 48 warps of gathers in flight per SM (C4 -0.9% against
// five at 48 registers; seven spill).
template <bool PAIRS>
__global__ void __launch_bounds__(256, 6) move_bulk_kernel(const float* __restrict__ tg, int k,
                                                        const float* __restrict__ in, float* __restrict__ out,
                                                        int64_t n, int clip, float* max_disp, const int* state,
                                                        uint32_t* __restrict__ splat_next, float* zn0, float* zn1,
                                                        int agg, int64_t zin, int64_t zout, int64_t zslab,
                                                        int zrev) {
    __shared__ __align__(128) float4 buf[2][kMoveChunk];
    __shared__ __align__(8) uint64_t bar[2];
    // zrev: plots in reverse launch order, so the move starts on the plots whose fields
    // the write pass produced last (still in L2)
    const int64_t zi = zrev ? (int64_t)(gridDim.z - 1 - blockIdx.z) : (int64_t)blockIdx.z;
    const int64_t zo = zi * zslab;
    tg = zoff(tg, zo);
    in += zi * zin;
    out += zi * zout;
    max_disp = zoff_opt(max_disp, zo);
    splat_next = zoff_opt(splat_next, zo);
    zn0 = zoff_opt(zn0, zo);
    zn1 = zoff_opt(zn1, zo);
    const int tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_barrier_init();
    }
    __syncthreads();
    pdl_enter();
    state = zoff_opt(state, zo);
    const bool stopped = state && state[0];
    const int s = 1 << k;
    if (splat_next && !stopped && blockIdx.x == 0 && tid == 0) {
        if (zn0) *zn0 = 0.f;
        if (zn1) *zn1 = 0.f;
    }
    const int64_t npair = n >> 1;
    const int64_t nchunk = (npair + kMoveChunk - 1) / kMoveChunk;
    const float4* in2 = reinterpret_cast<const float4*>(in);
    float4* out2 = reinterpret_cast<float4*>(out);
    auto issue = [&](int64_t c, int slot) {  // one thread: chunk c -> buf[slot]
        const int64_t p = c * kMoveChunk;
        const int64_t cnt = npair - p < kMoveChunk ? npair - p : kMoveChunk;
        const uint32_t bytes = (uint32_t)(cnt * 16);
        fence_proxy_async();  // the slot's previous contents were read by the generic proxy
        mbar_arrive_expect_tx(&bar[slot], bytes);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(&buf[slot][0])),
                     "l"(reinterpret_cast<uint64_t>(in2 + p)), "r"(bytes), "r"(smem_u32(&bar[slot]))
                     : "memory");
    };
    float md = 0.f;
    int64_t c = blockIdx.x;
    if (tid == 0 && c < nchunk) issue(c, 0);
    for (int i = 0; c < nchunk; ++i, c += gridDim.x) {
        const int slot = i & 1;
        if (tid == 0 && c + gridDim.x < nchunk) issue(c + gridDim.x, slot ^ 1);
        mbar_wait(&bar[slot], (uint32_t)((i >> 1) & 1));
        const int64_t p = c * kMoveChunk;
        float4 v[kMoveU];
        int64_t q[kMoveU];
        bool ok[kMoveU];
#pragma unroll
        for (int u = 0; u < kMoveU; ++u) {
            const int e = u * 256 + tid;
            q[u] = p + e;
            ok[u] = q[u] < npair;
            v[u] = ok[u] ? buf[slot][e] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        md = fmaxf(md, move_pairs<PAIRS, kMoveU, INIM_GATHER_FIRST>(tg, s, v, q, ok, out2, clip, stopped, splat_next,
                                                                     agg));
        __syncthreads();  // buf[slot] is refilled two chunks later
    }
    if ((n & 1) && blockIdx.x == 0 && tid == 0)
        md = fmaxf(md, move_odd_tail<PAIRS>(tg, s, in, out, n, clip, stopped, splat_next, agg));
    if (max_disp && !stopped) {
        md = warp_max(md);
        if ((tid & 31) == 0 && md > 0.f) atomic_max_nonneg(max_disp, md);
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
// A counting sort of the points by pixel (row-major), once per run, from the counts the
// run's first splat produced anyway:
//   scan    offsets = exclusive prefix of the counts (three launches: block sums, one
//           CTA over the block sums, block scans)
//   place   slot = atomicAdd(offsets[pixel], 1) (warp-aggregated with __match_any_sync
//           when lanes share a pixel); the point goes to sorted[slot], its row to
//           perm[slot]
// Consecutive points then share field rows (coalesced bilinear gathers) and count
// words (aggregated atomics).  No result depends on the order (integer counts,
// independent per-point moves); the final positions (and recorded frames) are
// scattered back through perm.
constexpr int kScanItems = 16;                     // counts per thread
constexpr int kScanBlock = 256 * kScanItems;       // counts per block

__global__ void __launch_bounds__(256) scan_block_sums_kernel(const uint32_t* __restrict__ counts, int64_t m,
                                                              uint32_t* __restrict__ bsum, int64_t zslab) {
    pdl_enter();
    counts = zoff(counts, zslab_off(zslab));
    bsum = zoff(bsum, zslab_off(zslab));
    const int64_t base = (int64_t)blockIdx.x * kScanBlock + (int64_t)threadIdx.x * kScanItems;
    uint32_t v = 0;
#pragma unroll
    for (int q = 0; q < kScanItems; q += 4) {
        if (base + q < m) {
            const uint4 c = __ldg(reinterpret_cast<const uint4*>(counts + base + q));
            v += c.x + c.y + c.z + c.w;
        }
    }
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    __shared__ uint32_t ws[8];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int q = 0; q < 8; ++q) t += ws[q];
        bsum[blockIdx.x] = t;
    }
}

// one CTA: exclusive scan of the block sums in place
__global__ void __launch_bounds__(1024) scan_top_kernel(uint32_t* __restrict__ bsum, int nb, int64_t zslab) {
    pdl_enter();
    bsum = zoff(bsum, zslab_off(zslab));
    __shared__ uint32_t ws[33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t carry = 0;
    for (int base = 0; base < nb; base += blockDim.x) {
        const int q = base + threadIdx.x;
        const uint32_t v = q < nb ? bsum[q] : 0u;
        uint32_t inc = v;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t n = __shfl_up_sync(kFull, inc, o);
            if (lane >= o) inc += n;
        }
        if (lane == 31) ws[w] = inc;
        __syncthreads();
        if (w == 0) {
            const uint32_t t = lane < (int)(blockDim.x >> 5) ? ws[lane] : 0u;
            uint32_t ti = t;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t n = __shfl_up_sync(kFull, ti, o);
                if (lane >= o) ti += n;
            }
            ws[lane] = ti - t;
            if (lane == 31) ws[32] = ti;
        }
        __syncthreads();
        if (q < nb) bsum[q] = carry + ws[w] + inc - v;
        carry += ws[32];
        __syncthreads();
    }
}

// self_prefix: bsum holds the raw block sums and each block adds up its predecessors'
// itself (up to kScanSelfMax blocks: a strided block reduction, exact integers), so the
// one-CTA scan_top launch is skipped; otherwise bsum is already scanned by scan_top.
constexpr int kScanSelfMax = 8192;

__global__ void __launch_bounds__(256) scan_blocks_kernel(const uint32_t* __restrict__ counts, int64_t m,
                                                          const uint32_t* __restrict__ bsum,
                                                          uint32_t* __restrict__ offsets, int64_t zslab,
                                                          int self_prefix) {
    pdl_enter();
    counts = zoff(counts, zslab_off(zslab));
    bsum = zoff(bsum, zslab_off(zslab));
    offsets = zoff(offsets, zslab_off(zslab));
    __shared__ uint32_t pre[8];
    if (self_prefix) {
        uint32_t a = 0;
        for (int q = threadIdx.x; q < (int)blockIdx.x; q += blockDim.x) a += __ldcg(bsum + q);
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(kFull, a, o);
        if ((threadIdx.x & 31) == 0) pre[threadIdx.x >> 5] = a;
    }
    const int64_t base = (int64_t)blockIdx.x * kScanBlock + (int64_t)threadIdx.x * kScanItems;
    uint32_t c[kScanItems];
    uint32_t v = 0;
#pragma unroll
    for (int q = 0; q < kScanItems; q += 4) {
        uint4 u = make_uint4(0u, 0u, 0u, 0u);
        if (base + q < m) u = __ldg(reinterpret_cast<const uint4*>(counts + base + q));
        c[q] = u.x; c[q + 1] = u.y; c[q + 2] = u.z; c[q + 3] = u.w;
        v += u.x + u.y + u.z + u.w;
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t inc = v;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t n = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += n;
    }
    __shared__ uint32_t ws[8];
    if (lane == 31) ws[w] = inc;
    __syncthreads();
    uint32_t blk = 0;
    if (self_prefix) {
#pragma unroll
        for (int q = 0; q < 8; ++q) blk += pre[q];
    } else {
        blk = bsum[blockIdx.x];
    }
    uint32_t run = blk + inc - v;
    for (int q = 0; q < w; ++q) run += ws[q];
#pragma unroll
    for (int q = 0; q < kScanItems; q += 4) {
        uint4 o;
        o.x = run; run += c[q];
        o.y = run; run += c[q + 1];
        o.z = run; run += c[q + 2];
        o.w = run; run += c[q + 3];
        if (base + q < m) *reinterpret_cast<uint4*>(offsets + base + q) = o;
    }
}

__global__ void __launch_bounds__(256) place_points_kernel(const float2* __restrict__ pts, int64_t n, int k,
                                                           uint32_t* __restrict__ cursor, float2* __restrict__ sorted,
                                                           uint32_t* __restrict__ rank, int64_t zpts, int64_t zslab) {
    pdl_enter();
    {
        const int64_t zo = zslab_off(zslab);
        pts += blockIdx.z * (zpts >> 1);
        cursor = zoff(cursor, zo);
        sorted = zoff(sorted, zo);
        rank = zoff(rank, zo);
    }
    const int s = 1 << k;
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t iters = (n + stride - 1) / stride;  // uniform trip count: whole warps in __match_any_sync
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t it = 0; it < iters; ++it, p += stride) {
        const bool live = p < n;
        float2 v = make_float2(0.f, 0.f);
        int pix = -1;
        if (live) {
            v = __ldg(pts + p);
            pix = pixel_of(v.y, s) * s + pixel_of(v.x, s);
        }
        const unsigned grp = __match_any_sync(kFull, pix);
        const int leader = __ffs(grp) - 1;
        uint32_t base = 0;
        if (live && lane == leader) base = atomicAdd(cursor + pix, (uint32_t)__popc(grp));
        base = __shfl_sync(kFull, base, leader);
        if (live) {
            const uint32_t slot = base + __popc(grp & ((1u << lane) - 1u));
            sorted[slot] = v;
            rank[p] = slot;  // coalesced: the way back is a gather
        }
    }
}

// out[p] = sorted[rank[p]]: coalesced rank reads and output writes, gathered reads.
__global__ void __launch_bounds__(256) unpermute_kernel(const float2* __restrict__ sorted,
                                                        const uint32_t* __restrict__ rank, int64_t n,
                                                        float2* __restrict__ out, int64_t zout, int64_t zslab) {
    pdl_enter();
    sorted = zoff(sorted, zslab_off(zslab));
    rank = zoff(rank, zslab_off(zslab));
    out += blockIdx.z * (zout >> 1);
    constexpr int U = 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += U * stride) {
        uint32_t r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) r[u] = p + u * stride < n ? __ldg(rank + p + u * stride) : 0u;
        float2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = p + u * stride < n ? __ldg(sorted + r[u]) : make_float2(0.f, 0.f);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (p + u * stride < n) __stcs(out + p + u * stride, v[u]);
    }
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

// Batches: one launch covers every plot (grid.z = plot); the per-plot grid is not
// capped at one resident wave, B of them fill the GPU.
static dim3 batch_grid(unsigned per_plot_resident, int64_t work, int per_block, const Bat& bt) {
    if (bt.B <= 1) return dim3(per_plot_resident);
    int64_t blocks = (work + per_block - 1) / per_block;
    return dim3((unsigned)(blocks < 1 ? 1 : blocks), 1, (unsigned)bt.B);
}

int launch_splat_f32(const float* pts, int64_t n, int k, uint32_t* counts, const int* state, cudaStream_t st,
                     float* zero0, float* zero1, const Bat& bt) {
    const int64_t npair = n >> 1;
    const dim3 grid = batch_grid(grid_for(npair > 0 ? npair : 1, 256), npair, 256 * 4, bt);
    INIM_CUDA_TRY(launch_pdl(splat_f32_kernel, grid, dim3(256), 0, st, pts, n, k, counts, state, zero0, zero1, bt.pts,
                             bt.slab));
    prof_mark(st, "splat");
    return (int)cudaGetLastError();
}

// Sort the points by pixel: `counts` are the points' per-pixel counts (the run's first
// splat), `cursor` an m-word scratch (destroyed), bsum ceil(m / kScanBlock) words.
int launch_sort_points(const float* pts, int64_t n, int k, const uint32_t* counts, uint32_t* cursor,
                       uint32_t* bsum, float* sorted, uint32_t* rank, cudaStream_t st, const Bat& bt) {
    const int64_t m = (int64_t)1 << (2 * k);
    const unsigned nb = (unsigned)((m + kScanBlock - 1) / kScanBlock);
    const unsigned z = (unsigned)bt.B;
    INIM_CUDA_TRY(launch_pdl(scan_block_sums_kernel, dim3(nb, 1, z), dim3(256), 0, st, counts, m, bsum, bt.slab));
    const int self_prefix = nb <= (unsigned)kScanSelfMax ? 1 : 0;
    if (!self_prefix)
        INIM_CUDA_TRY(launch_pdl(scan_top_kernel, dim3(1, 1, z), dim3(1024), 0, st, bsum, (int)nb, bt.slab));
    INIM_CUDA_TRY(launch_pdl(scan_blocks_kernel, dim3(nb, 1, z), dim3(256), 0, st, counts, m, (const uint32_t*)bsum,
                             cursor, bt.slab, self_prefix));
    INIM_CUDA_TRY(launch_pdl(place_points_kernel, batch_grid(grid_for(n > 0 ? n : 1, 256), n, 256, bt), dim3(256), 0,
                             st, reinterpret_cast<const float2*>(pts), n, k, cursor, reinterpret_cast<float2*>(sorted),
                             rank, bt.pts, bt.slab));
    prof_mark(st, "sort_points");
    return (int)cudaGetLastError();
}

// Exclusive prefix of m (a multiple of 4) u32 counts into `out`; bsum: sort_bsum_words.
int launch_exclusive_scan_u32(const uint32_t* counts, int64_t m, uint32_t* bsum, uint32_t* out, cudaStream_t st) {
    const unsigned nb = (unsigned)((m + kScanBlock - 1) / kScanBlock);
    INIM_CUDA_TRY(launch_pdl(scan_block_sums_kernel, dim3(nb), dim3(256), 0, st, counts, m, bsum, (int64_t)0));
    const int self_prefix = nb <= (unsigned)kScanSelfMax ? 1 : 0;
    if (!self_prefix)
        INIM_CUDA_TRY(launch_pdl(scan_top_kernel, dim3(1), dim3(1024), 0, st, bsum, (int)nb, (int64_t)0));
    INIM_CUDA_TRY(launch_pdl(scan_blocks_kernel, dim3(nb), dim3(256), 0, st, counts, m, (const uint32_t*)bsum, out,
                             (int64_t)0, self_prefix));
    return (int)cudaGetLastError();
}

size_t sort_bsum_words(int k) { return (size_t)((((int64_t)1 << (2 * k)) + kScanBlock - 1) / kScanBlock); }

int launch_unpermute(const float* sorted, const uint32_t* rank, int64_t n, float* out, cudaStream_t st,
                     const Bat& bt) {
    INIM_CUDA_TRY(launch_pdl(unpermute_kernel, batch_grid(grid_for(n > 0 ? n : 1, 256), n, 256 * 4, bt), dim3(256), 0,
                             st, reinterpret_cast<const float2*>(sorted), rank, n, reinterpret_cast<float2*>(out),
                             bt.pts, bt.slab));
    prof_mark(st, "unpermute");
    return (int)cudaGetLastError();
}

int launch_splat_f64(const double* pts, int64_t n, int k, uint32_t* counts, cudaStream_t st) {
    splat_f64_kernel<<<grid_for(n > 0 ? n : 1, 256), 256, 0, st>>>(pts, n, k, counts);
    return (int)cudaGetLastError();
}

// zin / zout: floats between consecutive plots' input / output points (a batch reads
// the caller's (B, n, 2) array or the workspace ping-pong buffers).
int launch_sample_f32(const float* tg, int k, const float* in, float* out, int64_t n, int clip, float* max_disp,
                      const int* state, cudaStream_t st, bool pairs, uint32_t* splat_next, float* zn0, float* zn1,
                      bool sorted, const Bat& bt, int64_t zin, int64_t zout, bool f32_counts) {
    const int64_t npair = n >> 1;
    // point pairs (16-byte loads) per thread per step, measured per regime (DESIGN.md
    // 4.5): two for one plot on the L2-resident paired field (C2: one 50.6, four 49.2
    // vs 46.2 us per iteration), one on the plain field above 2048^2 (C3: 336.6 vs
    // 346.6 us), four in a batch (C4: 50.4 vs 55.0 ms)
    // a batch (HBM-latency bound, work for many waves): UB point pairs per thread
    constexpr int UB = INIM_BATCH_MOVE_U;
    static const int bulk_cpc = [] {  // chunks per CTA of the pipelined batch move (0: grid-stride move)
        const char* e = getenv("INIM_MOVE_BULK");
        return e ? atoi(e) : 8;
    }();
    static const int64_t bulk_single = [] {  // single plots: pipelined move from this many pairs on
        const char* e = getenv("INIM_MOVE_BULK_SINGLE");
        return e ? (int64_t)atoll(e) : (int64_t)-1;
    }();
    if (bulk_cpc > 0 && (n >> 1) > 0 && (bt.B > 1 || (bulk_single >= 0 && (n >> 1) >= bulk_single))) {
        auto kb = pairs ? move_bulk_kernel<true> : move_bulk_kernel<false>;
        // many CTAs of a few chunks each: the prefetch overlaps all but the first chunk's
        // load, and the grid is many waves deep (no tail)
        const int64_t nchunk = ((n >> 1) + kMoveChunk - 1) / kMoveChunk;
        const int64_t per_plot = (nchunk + bulk_cpc - 1) / bulk_cpc;
        INIM_CUDA_TRY(launch_pdl(kb, dim3((unsigned)per_plot, 1, (unsigned)bt.B), dim3(256), 0, st, tg, k, in, out, n,
                                 clip, max_disp, state, splat_next, zn0, zn1, sorted ? (f32_counts ? 2 : 1) : 0, zin,
                                 zout, bt.slab, zrev_enabled() ? 1 : 0));
        prof_mark(st, "sample");
        return (int)cudaGetLastError();
    }
    auto kern = bt.B > 1 ? (pairs ? sample_f32_kernel<true, UB, true> : sample_f32_kernel<false, UB, true>)
                         : (pairs ? sample_f32_kernel<true, 2, false> : sample_f32_kernel<false, 1, false>);
    const dim3 grid = batch_grid(resident_grid((const void*)kern, npair > 0 ? npair : 1, 256), npair,
                                 256 * (bt.B > 1 ? UB : (pairs ? 2 : 1)), bt);
    INIM_CUDA_TRY(launch_pdl(kern, grid, dim3(256), 0, st, tg, k, reinterpret_cast<const float4*>(in), in,
                             reinterpret_cast<float4*>(out), out, n, clip, max_disp, state, splat_next, zn0, zn1,
                             sorted ? (f32_counts ? 2 : 1) : 0, zin, zout, bt.slab));
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
