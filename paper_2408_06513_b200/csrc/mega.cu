// Persistent, cooperative iteration kernel: the whole regularization run
// (regularize.run, reference regularize.py:40-80) in ONE launch.  Every CTA stays
// resident; the phases of each iteration are separated by grid-wide barriers instead
// of kernel boundaries:
//
//   splat -> | smooth_h (+ clear next counts) -> | smooth_v + tile reduce -> |
//   band_rows -> | colscan -> | diagscan -> | marg -> | field (warp tiles, TMA) -> |
//   move + clip (+ frame, displacement) -> | [stop test] -> next iteration
//
// The phase bodies are the same device functions the standalone kernels use
// (inim_smooth.cuh, inim_scan.cuh, inim_tiles.cuh, inim_points.cuh), so the two paths
// are bit-identical.  Used for grids 64^2..2048^2 (where the per-iteration work is tens
// of microseconds and launch gaps dominated); larger grids use the graph of standalone
// kernels.
#include <cooperative_groups.h>

#include "inim_points.cuh"
#include "inim_scan.cuh"
#include "inim_smooth.cuh"

namespace cg = cooperative_groups;

namespace inim {

constexpr int kMegaThreads = 256;
constexpr int kMegaWarps = kMegaThreads / 32;
constexpr int kMaxPhaseStamps = 16;

struct MegaArgs {
    Geo g;
    HGeo h;
    VGeo v;
    Ws ws;
    Taps taps;
    float* ptsA;           // caller's positions: input, and output at the end
    float* ptsB;           // ping-pong partner
    int64_t n;
    uint32_t* counts;      // 2 * m (ping-pong)
    float* d;              // density
    float* targets;        // field scratch (when fields == null)
    float* fields;         // optional: iters * m * 2
    const float* defect;   // flat response (float32, precomputed) or null (closed form)
    float* frames;         // optional: (iters + 1) * n * 2 (frame 0 written by the host side)
    float* disp;           // optional: [iters]
    float* excs;           // optional: [iters]
    float* scratch;        // >= 4 floats
    int* state;            // {stopped, iterations_done} for the displacement criterion
    unsigned long long* stamps;  // optional: globaltimer at each phase boundary (first iteration)
    float bg, eps;
    int iters;
    unsigned bar_off;  // byte offset of the per-warp mbarriers (past every phase's footprint)
};

INIM_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

INIM_DEV unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

template <int R, int CPL>
__global__ void __launch_bounds__(kMegaThreads, 2)
    mega_kernel(const __grid_constant__ CUtensorMap map, const __grid_constant__ MegaArgs A) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(128) unsigned char smem[];
    const Geo& g = A.g;
    const int s = g.s;
    const int64_t m = g.m;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles = g.B * g.NX;
    const size_t slot_bytes = (size_t)g.TH * g.TW * sizeof(float);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + A.bar_off);
    float* slot = reinterpret_cast<float*>(smem + warp * slot_bytes);
    if (lane == 0) {
        mbar_init(&bars[warp], 1);
        fence_barrier_init();
    }
    __syncwarp();
    uint32_t parity = 0;
    int nst = 0;
    auto stamp = [&](int t) {
        if (A.stamps && t == 0 && blockIdx.x == 0 && threadIdx.x == 0 && nst < kMaxPhaseStamps)
            A.stamps[nst] = globaltimer();
        ++nst;
    };
    const int64_t npair = A.n >> 1;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
    const int nH = (s / A.h.TWH) * (s / A.h.RH), nHx = s / A.h.TWH;
    const int nV = g.NX * (s / A.v.VR);
    const int nchain = chains_items(g);
    double(*part)[33] = reinterpret_cast<double(*)[33]>(smem);
    double* bp = reinterpret_cast<double*>(smem) + kMegaWarps * 33;
    double* shs = bp + g.B + 1;
    int done = 0;
    for (int t = 0; t < A.iters; ++t) {
        nst = 0;
        const float* src = (t & 1) ? A.ptsB : A.ptsA;
        float* dst = (t & 1) ? A.ptsA : A.ptsB;
        uint32_t* cur = A.counts + (size_t)(t & 1) * m;
        uint32_t* next = A.counts + (size_t)((t + 1) & 1) * m;
        float* tg = A.fields ? A.fields + (size_t)t * 2 * m : A.targets;
        float* dsp = A.disp ? A.disp + t : A.scratch;
        float* exc = A.excs ? A.excs + t : A.scratch + 1;
        stamp(t);
        // ---- splat (density.py:14-27): one red.add per point, two points per 16-byte load
        if (gtid == 0) {
            *dsp = 0.f;
            *exc = 0.f;
        }
        {
            const float4* p2 = reinterpret_cast<const float4*>(src);
            for (int64_t p = gtid; p < npair; p += gstride) {
                const float4 v = __ldcs(p2 + p);
                atomicAdd(cur + pixel_of(v.y, s) * s + pixel_of(v.x, s), 1u);
                atomicAdd(cur + pixel_of(v.w, s) * s + pixel_of(v.z, s), 1u);
            }
            if ((A.n & 1) && gtid == 0) {
                const float x = src[2 * (A.n - 1)], y = src[2 * (A.n - 1) + 1];
                atomicAdd(cur + pixel_of(y, s) * s + pixel_of(x, s), 1u);
            }
        }
        grid.sync();
        stamp(t);
        // ---- smoothing, horizontal (and clear the other count buffer)
        for (int item = blockIdx.x; item < nH; item += gridDim.x)
            smooth_h_tile<R, uint32_t>(cur, A.ws.tmp, s, A.h, A.taps, next, item % nHx, item / nHx,
                                       reinterpret_cast<float*>(smem));
        grid.sync();
        stamp(t);
        // ---- smoothing, vertical + background + tile reduce
        for (int item = blockIdx.x; item < nV; item += gridDim.x)
            smooth_v_tile<R>(A.ws.tmp, A.d, g, A.v, A.ws, A.taps, A.bg, 2, item % g.NX, item / g.NX,
                             reinterpret_cast<float*>(smem));
        fence_proxy_async_global();  // d (generic-proxy stores) is read by TMA in the field phase
        grid.sync();
        stamp(t);
        // ---- carry scan (the band lines ran at the end of the reduce)
        band_prefix(g, A.ws, bp, shs);  // every CTA: X2 chains need it
        if (blockIdx.x == 0) {
            for (int q = threadIdx.x; q <= g.B; q += blockDim.x) A.ws.bandpre[q] = bp[q];
            if (threadIdx.x == 0) *A.ws.total = bp[g.B];
        }
        for (int item = blockIdx.x; item < nchain; item += gridDim.x) chains_item(g, A.ws, item, part, bp);
        grid.sync();
        stamp(t);
        // ---- field: one warp per tile, tile staged by TMA into the warp's slot
        {
            fence_proxy_async_global();
            const WriteOut out{nullptr, tg, A.defect, exc, nullptr};
            for (int tile = blockIdx.x * kMegaWarps + warp; tile < tiles; tile += gridDim.x * kMegaWarps) {
                const int b = tile / g.NX, x = tile - b * g.NX;
                if (lane == 0) {
                    fence_proxy_async();  // the slot was last written through the generic proxy
                    mbar_arrive_expect_tx(&bars[warp], (uint32_t)slot_bytes);
                    tma_load_2d(slot, &map, x * g.TW, b * g.TH, &bars[warp]);
                }
                __syncwarp();
                mbar_wait(&bars[warp], parity);
                parity ^= 1u;
                warp_tile_write<CPL, 1, false>(slot, g.TW, g, A.ws, b, x, lane, out);
                __syncwarp();
            }
        }
        grid.sync();
        stamp(t);
        // ---- move + clip (mapping.py:207-246, regularize.py:36), frame, displacement
        {
            const float2* tg2 = reinterpret_cast<const float2*>(tg);
            const float4* in2 = reinterpret_cast<const float4*>(src);
            float4* out2 = reinterpret_cast<float4*>(dst);
            // frames are only 8-byte aligned when n is odd: float2 stores
            float2* fr2 = A.frames ? reinterpret_cast<float2*>(A.frames + (size_t)(t + 1) * 2 * A.n) : nullptr;
            float md = 0.f;
            for (int64_t p = gtid; p < npair; p += gstride) {
                const float4 v = __ldcs(in2 + p);
                float4 o;
                bilinear<float>(tg2, s, v.x, v.y, o.x, o.y);
                bilinear<float>(tg2, s, v.z, v.w, o.z, o.w);
                o.x = clip01(o.x); o.y = clip01(o.y); o.z = clip01(o.z); o.w = clip01(o.w);
                md = fmaxf(md, fmaxf(fmaxf(fabsf(o.x - v.x), fabsf(o.y - v.y)), fmaxf(fabsf(o.z - v.z), fabsf(o.w - v.w))));
                __stcs(out2 + p, o);
                if (fr2) {
                    __stcs(fr2 + 2 * p, make_float2(o.x, o.y));
                    __stcs(fr2 + 2 * p + 1, make_float2(o.z, o.w));
                }
            }
            if ((A.n & 1) && gtid == 0) {
                const float x = src[2 * (A.n - 1)], y = src[2 * (A.n - 1) + 1];
                float ox, oy;
                bilinear<float>(tg2, s, x, y, ox, oy);
                ox = clip01(ox);
                oy = clip01(oy);
                md = fmaxf(md, fmaxf(fabsf(ox - x), fabsf(oy - y)));
                dst[2 * (A.n - 1)] = ox;
                dst[2 * (A.n - 1) + 1] = oy;
                if (A.frames) {
                    A.frames[(size_t)(t + 1) * 2 * A.n + 2 * (A.n - 1)] = ox;
                    A.frames[(size_t)(t + 1) * 2 * A.n + 2 * (A.n - 1) + 1] = oy;
                }
            }
            md = warp_max(md);
            if (lane == 0 && md > 0.f) atomic_max_nonneg(dsp, md);
        }
        grid.sync();
        stamp(t);
        done = t + 1;
        if (A.eps > 0.f) {  // stop="displacement" (regularize.py:76-79), uniform across the grid
            const bool stop = *((volatile float*)dsp) < A.eps;
            if (gtid == 0) {
                A.state[1] = done;
                if (stop) A.state[0] = 1;
            }
            if (stop) break;
        }
    }
    // final positions live in ptsA when `done` is even, else in ptsB
    if (done & 1) {
        const float4* fin = reinterpret_cast<const float4*>(A.ptsB);
        float4* o = reinterpret_cast<float4*>(A.ptsA);
        for (int64_t p = gtid; p < npair; p += gstride) o[p] = fin[p];
        if ((A.n & 1) && gtid == 0) {
            A.ptsA[2 * (A.n - 1)] = A.ptsB[2 * (A.n - 1)];
            A.ptsA[2 * (A.n - 1) + 1] = A.ptsB[2 * (A.n - 1) + 1];
        }
    }
}

void make_taps(int kernel_size, Taps* taps);  // smooth.cu

// Largest shared-memory footprint over the phases (the per-warp mbarriers go after it).
static size_t mega_body_bytes(const Geo& g, const HGeo& h, const VGeo& v, int R) {
    size_t b = h_smem_bytes(h, R);
    b = b > v_smem_bytes(g, v, R) ? b : v_smem_bytes(g, v, R);
    const size_t w = kMegaWarps * (size_t)g.TH * g.TW * sizeof(float);
    b = b > w ? b : w;
    const size_t sc = sizeof(double) * (33 * kMegaWarps + g.B + 1 + 33);
    b = b > sc ? b : sc;
    return (b + 127) & ~size_t(127);
}

template <int R, int CPL>
static int launch_mega_t(MegaArgs& A, const CUtensorMap& map, cudaStream_t st) {
    auto fn = mega_kernel<R, CPL>;
    A.bar_off = (unsigned)mega_body_bytes(A.g, A.h, A.v, R);
    const size_t smem = A.bar_off + kMegaWarps * sizeof(uint64_t);
    static int grid = 0;
    static size_t grid_smem = 0;
    if (!grid || grid_smem != smem) {
        INIM_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0, dev = 0, sms = 0;
        INIM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kMegaThreads, smem));
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (per_sm < 1) return INIM_EINVAL;
        grid = per_sm * sms;
        grid_smem = smem;
    }
    void* args[] = {(void*)&map, (void*)&A};
    INIM_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)fn, dim3(grid), dim3(kMegaThreads), args, smem, st));
    prof_mark(st, "iteration_kernel");
    return (int)cudaGetLastError();
}

bool mega_supported(const Geo& g, int kernel_size) { return kernel_size == 8 && g.s >= 64 && g.s <= 2048; }

// Enqueue one persistent launch for `iters` iterations.  pts (in/out), pong, counts
// (2*m, zeroed by the caller), d, targets, defect, frames/fields/disp/excs/state as
// in inim_run.
int launch_mega(const Geo& g, const Ws& ws, int kernel_size, float bg, float eps, int iters, float* pts, float* pong,
                int64_t n, uint32_t* counts, float* d, float* targets, const float* defect, float* frames,
                float* fields, float* disp, float* excs, float* scratch, int* state, unsigned long long* stamps,
                cudaStream_t st) {
    MegaArgs A;
    memset(&A, 0, sizeof(A));
    A.g = g;
    A.h = make_hgeo(g.s);
    A.v = make_vgeo(g);
    A.ws = ws;
    make_taps(kernel_size, &A.taps);
    A.ptsA = pts; A.ptsB = pong; A.n = n; A.counts = counts; A.d = d; A.targets = targets;
    A.fields = fields; A.defect = defect; A.frames = frames; A.disp = disp; A.excs = excs;
    A.scratch = scratch; A.state = state; A.stamps = stamps; A.bg = bg; A.eps = eps; A.iters = iters;
    CUtensorMap map;
    int rc = make_tensor_map_2d(&map, d, g.s, g.TW, g.TH);
    if (rc) return rc;
    if (g.CPL == 2) return launch_mega_t<24, 2>(A, map, st);
    if (g.CPL == 4) return launch_mega_t<24, 4>(A, map, st);
    return INIM_EINVAL;
}

}  // namespace inim
