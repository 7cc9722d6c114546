// Integral-image pass: the eight region tables of a density texture
// (reference integral.py:180-247, tables per model.py:59-85) and the deformation
// field built from them (mapping.py:146-204).
//
// Pipeline:
//   reduce : one warp per TH x 128 tile, the tile staged into shared memory by TMA
//            (cp.async.bulk.tensor.2d, one mbarrier per warp); emits per-tile aggregates
//   scan   : float64 carry scan over the aggregates (scan.cu)
//   write  : one warp per tile re-sweeps its TMA-staged tile and produces
//              rect_tl = TLcar + VH + in-tile row prefix of the column prefix
//              wedge_up = (in-band up-left + up-right chains - column prefix) + X1 + X2
//            and the six other tables from the marginals
//              tr = Rpre - tl, bl = Cpre - tl, br = C - Rpre - Cpre + tl,
//              left = Apre - up, right = Dsuf - up, down = C - Apre - Dsuf + up,
//            then streams the eight tables out (MODE 0) or evaluates the field (MODE 1).
// No warp ever waits on another; every sum has a fixed order (deterministic).
#include "inim_tiles.cuh"

namespace inim {

constexpr int kWarpsPerCta = 4;

// Reduce with a TMA ring: each warp streams its tile through two shared-memory slots
// of kChunk rows (cp.async.bulk.tensor.2d, one mbarrier per slot): the next chunk is
// in flight while the current one is reduced, and 8 KB of shared memory per warp keeps
// ~28 warps resident per SM.  Warps are independent (no CTA barrier).
constexpr int kChunk = 8;

__host__ __device__ inline size_t ring_smem_bytes(const Geo& g) {
    return (size_t)kWarpsPerCta * (2 * kChunk * g.TW * sizeof(float) + 2 * sizeof(uint64_t));
}

template <int CPL>
__global__ void __launch_bounds__(kWarpsPerCta * 32) reduce_ring_kernel(const __grid_constant__ CUtensorMap map,
                                                                        const Geo g, const Ws ws) {
    pdl_enter();  // (standalone API only: one plot)
    extern __shared__ __align__(128) unsigned char smem[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles = g.B * g.NX;
    const int stride = gridDim.x * kWarpsPerCta;  // persistent warps: tiles t0, t0 + stride, ...
    const int t0 = blockIdx.x * kWarpsPerCta + w;
    if (t0 >= tiles) return;  // the whole warp
    const int TW = g.TW, nch = g.TH / kChunk;
    const int mine = (tiles - t0 + stride - 1) / stride;
    const int K = mine * nch;  // this warp's chunk sequence over its tiles
    const uint32_t chunk_bytes = (uint32_t)(kChunk * TW * sizeof(float));
    float* buf = reinterpret_cast<float*>(smem) + (size_t)w * 2 * kChunk * TW;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (size_t)kWarpsPerCta * 2 * chunk_bytes) + 2 * w;
    auto issue = [&](int kq) {  // lane 0: chunk kq of the sequence into slot kq & 1
        const int tile = t0 + (kq / nch) * stride, c = kq % nch;
        const int b = tile / g.NX, x = tile - b * g.NX;
        mbar_arrive_expect_tx(&bar[kq & 1], chunk_bytes);
        tma_load_2d(buf + (size_t)(kq & 1) * kChunk * TW, &map, x * TW, b * g.TH + c * kChunk, &bar[kq & 1]);
    };
    if (lane == 0) {
        prefetch_tensormap(&map);
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_barrier_init();
        issue(0);
        if (K > 1) issue(1);
    }
    __syncwarp();
    const bool act = lane <= g.WL - 1;
    uint32_t ph0 = 0, ph1 = 0;
    // row sums of a chunk: lane group q (32 / kChunk lanes) sums row q of the slot
    constexpr int LPR = 32 / kChunk;
    const int rq = lane / LPR, rl = lane - rq * LPR;
    int kq = 0;
    for (int tile = t0; tile < tiles; tile += stride) {
        const int b = tile / g.NX, x = tile - b * g.NX;
        TileReducer<CPL> red(g, ws, b, x, lane);
        for (int c = 0; c < nch; ++c, ++kq) {
            const int slot = kq & 1;
            if (slot == 0) {
                mbar_wait(&bar[0], ph0);
                ph0 ^= 1u;
            } else {
                mbar_wait(&bar[1], ph1);
                ph1 ^= 1u;
            }
            const float* sl = buf + (size_t)slot * kChunk * TW;
            {  // the chunk's kChunk row sums, one shuffle pair per chunk instead of a warp sum per row
                float acc = 0.f;
                for (int u = rl * 4; u < TW; u += LPR * 4) {
                    const float4 v4 = *reinterpret_cast<const float4*>(sl + rq * TW + u);
                    acc += (v4.x + v4.y) + (v4.z + v4.w);
                }
#pragma unroll
                for (int o = LPR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
#pragma unroll
                for (int q = 0; q < kChunk; ++q) red.set_rowsum(c * kChunk + q, __shfl_sync(kFull, acc, q * LPR));
            }
#pragma unroll
            for (int q = 0; q < kChunk; ++q) {
                float dv[CPL];
                if (act) load_row<CPL>(sl + q * TW + lane * CPL, dv);
                else {
#pragma unroll
                    for (int e = 0; e < CPL; ++e) dv[e] = 0.f;
                }
                red.template row<false>(c * kChunk + q, dv);
            }
            __syncwarp();  // every lane is done with the slot before it is refilled
            if (lane == 0 && kq + 2 < K) {
                fence_proxy_async();
                issue(kq + 2);
            }
        }
        red.finish();  // band lines: lines_kernel
    }
}

// The reduce reads its tile straight from global memory (rows prefetched two ahead in
// registers), so residency is bounded by registers only.
template <int CPL>
__global__ void __launch_bounds__(kWarpsPerCta * 32) reduce_kernel(const float* __restrict__ d, const Geo g,
                                                                   const Ws ws0, int64_t zslab) {
    pdl_enter();
    const int64_t zo = zslab_off(zslab);
    d = zoff(d, zo);
    const Ws ws = ws_shift(ws0, zo);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tile = blockIdx.x * kWarpsPerCta + w;
    if (tile >= g.B * g.NX) return;
    const int b = tile / g.NX, x = tile - b * g.NX;
    warp_tile_reduce<CPL, true>(d + (int64_t)b * g.TH * g.s + (int64_t)x * g.TW, g.s, g, ws, b, x, lane);
}

// The write pass re-reads its tile straight from global memory (rows prefetched two
// ahead in registers): no shared memory, so residency is bounded by registers only.
template <int CPL, int MODE, bool GEO = false>
__global__ void __launch_bounds__(kWarpsPerCta * 32, CPL == 4 ? (GEO ? 4 : 5) : 1) write_kernel(const float* __restrict__ d, const Geo g,
                                                                  const Ws ws0, const WriteOut out0, const int* state,
                                                                  int64_t zslab) {
    pdl_enter();
    state = zstate(state, zslab);
    if (state && state[0]) return;  // displacement stop already reached
    const int64_t zo = zslab_off(zslab);  // plot blockIdx.z of a batch
    d = zoff(d, zo);
    const Ws ws = ws_shift(ws0, zo);
    WriteOut out = out0;
    if (zo) {
        out.targets = zoff_opt(out.targets, zo);
        out.max_exc = zoff_opt(out.max_exc, zo);
        out.pairs = zoff_opt(out.pairs, zo);
    }
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tile = blockIdx.x * kWarpsPerCta + w;
    if (tile >= g.B * g.NX) return;
    const int b = tile / g.NX, x = tile - b * g.NX;
    const float* src = d + (int64_t)b * g.TH * g.s + (int64_t)x * g.TW;
    warp_tile_write<CPL, MODE, true, GEO>(src, g.s, g, ws, b, x, lane, out);
}

// ---- standalone helpers --------------------------------------------------------------

// build_field from eight precomputed tables (mapping.py:194-204).
__global__ void field_from_tables_kernel(const float* __restrict__ t8, int k, const double* total,
                                         const float* __restrict__ defect, float* __restrict__ targets,
                                         float* max_exc) {
    const int s = 1 << k;
    const int64_t m = (int64_t)s * s;
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    float exc = 0.f;
    if (q < m) {
        const int j = (int)(q >> k), i = (int)(q & (s - 1));
        const double scale = ldexp(1.0, -k);
        const double x = i * scale, y = j * scale;
        const bool below = y < x, near = x + y < 1.0;
        const double drx = below ? 1.0 : 1.0 - y + x, dry = below ? 1.0 + y - x : 1.0;
        const double ulx = below ? x - y : 0.0, uly = below ? 0.0 : y - x;
        const double urx = near ? x + y : 1.0, ury = near ? 0.0 : x + y - 1.0;
        const double dlx = near ? 0.0 : x + y - 1.0, dly = near ? x + y : 1.0;
        const double tl = t8[q], bl = t8[m + q], br = t8[2 * m + q], tr = t8[3 * m + q];
        const double up = t8[4 * m + q], left = t8[5 * m + q], down = t8[6 * m + q], right = t8[7 * m + q];
        const double inv = 0.5 / *total;
        const double tx = (tl * drx + bl * urx + br * ulx + tr * dlx + (up + down) * x + left) * inv;
        const double ty = (tl * dry + bl * ury + br * uly + tr * dly + (left + right) * y + up) * inv;
        double2 def;
        if (defect) {
            def.x = defect[2 * q];
            def.y = defect[2 * q + 1];
        } else {
            def = flat_response_at(i, j, k);
        }
        const float gx = (float)(tx - def.x + x), gy = (float)(ty - def.y + y);
        exc = fmaxf(fmaxf(-gx, -gy), fmaxf(gx - 1.f, gy - 1.f));
        targets[2 * q] = fminf(fmaxf(gx, 0.f), 1.f);
        targets[2 * q + 1] = fminf(fmaxf(gy, 0.f), 1.f);
    }
    exc = warp_max(exc);
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(max_exc, exc);
}

__global__ void flat_response_kernel(int k, float* __restrict__ defect) {
    const int s = 1 << k;
    const int64_t m = (int64_t)s * s;
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= m) return;
    const double2 f = flat_response_at((int)(q & (s - 1)), (int)(q >> k), k);
    defect[2 * q] = (float)f.x;
    defect[2 * q + 1] = (float)f.y;
}

// Generic line scan along direction (dj, di) with a float64 accumulator: inclusive
// (out = sum of the line up to and including the cell) or exclusive.  Serves the
// staged API functions column_integrals / classical_rects / triangle_integrals
// (integral.py:180-209), whose per-stage outputs the reference also exports.
__global__ void line_scan_kernel(const float* __restrict__ in, float* __restrict__ out, int s, int dj, int di,
                                 int exclusive) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    int j, i;
    const int nrow = dj != 0 ? s : 0;  // starts on the entry row
    if (q < nrow) {
        j = dj > 0 ? 0 : s - 1;
        i = q;
    } else {
        const int q2 = q - nrow;
        if (di == 0) return;
        const int ncol = dj != 0 ? s - 1 : s;  // entry column minus the corner already covered
        if (q2 >= ncol) return;
        i = di > 0 ? 0 : s - 1;
        j = dj == 0 ? q2 : (dj > 0 ? q2 + 1 : q2);
    }
    double acc = 0.0;
    while (j >= 0 && j < s && i >= 0 && i < s) {
        const int64_t idx = (int64_t)j * s + i;
        const double v = in[idx];
        if (exclusive) {
            out[idx] = (float)acc;
            acc += v;
        } else {
            acc += v;
            out[idx] = (float)acc;
        }
        j += dj;
        i += di;
    }
}

// =====================================================================================
// Host launchers
// =====================================================================================

static unsigned tile_ctas(const Geo& g) { return (unsigned)((g.B * g.NX + kWarpsPerCta - 1) / kWarpsPerCta); }

template <int CPL>
static int launch_reduce_cpl(const float* d, const Geo& g, const Ws& ws, const CUtensorMap* ring_map,
                             cudaStream_t st, const Bat& bt) {
    if (ring_map && g.TH % kChunk == 0 && g.TW >= 32 && bt.B == 1) {
        const size_t smem = ring_smem_bytes(g);
        INIM_CUDA_TRY(ensure_smem_limit((const void*)reduce_ring_kernel<CPL>, (int)smem));
        // one tile per warp: persistent warps (grid capped at residency, several tiles
        // per warp through the same ring) measured 2x slower at 16384^2
        const unsigned ctas = tile_ctas(g);
        INIM_CUDA_TRY(launch_pdl(reduce_ring_kernel<CPL>, dim3(ctas), dim3(kWarpsPerCta * 32), smem, st, *ring_map, g,
                                 ws));
    } else {
        INIM_CUDA_TRY(launch_pdl(reduce_kernel<CPL>, dim3(tile_ctas(g), 1, bt.B), dim3(kWarpsPerCta * 32), 0, st, d, g,
                                 ws, bt.slab));
    }
    prof_mark(st, "reduce");
    return (int)cudaGetLastError();
}

int launch_reduce_from_global(const float* d, const Geo& g, const Ws& ws, const CUtensorMap* map, cudaStream_t st,
                              const Bat& bt) {
    switch (g.CPL) {
        case 4: return launch_reduce_cpl<4>(d, g, ws, map, st, bt);
        case 2: return launch_reduce_cpl<2>(d, g, ws, map, st, bt);
        default: return launch_reduce_cpl<1>(d, g, ws, map, st, bt);
    }
}

template <int CPL, int MODE>
static int launch_write_cpl(const float* d, const Geo& g, const Ws& ws, const WriteOut& out, const int* state,
                            cudaStream_t st, const Bat& bt) {
    // the 16 x 64 tiles of grids up to 2048^2 as compile-time constants (C2 41.4 -> 40.45
    // us per iteration; the 32 x 128 instance spills at its 96-register cap and is slower)
    // (tables pass: below 2048^2 only -- its constant-geometry instance holds the whole
    // tile in 250 registers: 512^2 +8%, 1024^2 +11%, 2048^2 -9% on the integral sweep)
    auto kern = write_kernel<CPL, MODE>;
    if constexpr (CPL == 2) {
        if (g.WL == 32 && g.TW == 64 && g.TH == 16 && (MODE != 0 || g.s < 2048)) kern = write_kernel<CPL, MODE, true>;
    }
    // the 32 x 128 field pass likewise, at 4 CTAs per SM (127 registers, no spills; at the
    // 5-CTA cap of the generic instance it spilled): C4 37.78 -> 37.19 ms, C3 -1.9%
    // (the tables pass too: integral 4096^2 3,733 -> 4,095 GB/s, 8192^2 +1%, 16384^2 +-0)
    if constexpr (CPL == 4 && MODE != 2) {
        if (g.WL == 32 && g.TW == 128 && g.TH == 32) kern = write_kernel<CPL, MODE, true>;
    }
    INIM_CUDA_TRY(launch_pdl(kern, dim3(tile_ctas(g), 1, bt.B), dim3(kWarpsPerCta * 32), 0, st, d, g, ws, out, state,
                             bt.slab));
    prof_mark(st, MODE == 0 ? "write_tables" : "write_field");
    return (int)cudaGetLastError();
}

template <int MODE>
static int launch_write_mode(const float* d, const Geo& g, const Ws& ws, const CUtensorMap* map, const WriteOut& out,
                             const int* state, cudaStream_t st, const Bat& bt = Bat{}) {
    switch (g.CPL) {
        case 4: return launch_write_cpl<4, MODE>(d, g, ws, out, state, st, bt);
        case 2: return launch_write_cpl<2, MODE>(d, g, ws, out, state, st, bt);
        default: return launch_write_cpl<1, MODE>(d, g, ws, out, state, st, bt);
    }
}

int launch_write_tables(const float* d, const Geo& g, const Ws& ws, const CUtensorMap* map, float* tables8,
                        cudaStream_t st) {
    WriteOut o{tables8, nullptr, nullptr, nullptr, nullptr};
    return launch_write_mode<0>(d, g, ws, map, o, nullptr, st);
}

int launch_write_field(const float* d, const Geo& g, const Ws& ws, const CUtensorMap* map, const float* defect,
                       float* targets, float* max_exc, const int* state, cudaStream_t st, float* pairs, const Bat& bt) {
    WriteOut o{nullptr, targets, defect, max_exc, pairs};
    return defect ? launch_write_mode<2>(d, g, ws, map, o, state, st, bt)
                  : launch_write_mode<1>(d, g, ws, map, o, state, st, bt);
}

int launch_field_from_tables(const float* t8, int k, const double* total, const float* defect, float* targets,
                             float* max_exc, cudaStream_t st) {
    const int64_t m = (int64_t)1 << (2 * k);
    field_from_tables_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(t8, k, total, defect, targets, max_exc);
    return (int)cudaGetLastError();
}

int launch_flat_response(int k, float* defect, cudaStream_t st) {
    const int64_t m = (int64_t)1 << (2 * k);
    flat_response_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(k, defect);
    prof_mark(st, "flat_response");
    return (int)cudaGetLastError();
}

int launch_line_scan(const float* in, float* out, int s, int dj, int di, int exclusive, cudaStream_t st) {
    const int n = 2 * s;
    line_scan_kernel<<<(n + 127) / 128, 128, 0, st>>>(in, out, s, dj, di, exclusive);
    return (int)cudaGetLastError();
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int make_tensor_map_2d(CUtensorMap* map, const float* base, int s, int box_w, int box_h) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !p)
            return INIM_EDRIVER;
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    cuuint64_t dims[2] = {(cuuint64_t)s, (cuuint64_t)s};
    cuuint64_t strides[1] = {(cuuint64_t)s * sizeof(float)};
    cuuint32_t box[2] = {(cuuint32_t)box_w, (cuuint32_t)box_h};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : INIM_EDRIVER;
}

}  // namespace inim
