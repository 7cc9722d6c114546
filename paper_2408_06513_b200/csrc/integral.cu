// Integral-image pass: the eight region tables of a density texture
// (reference integral.py:180-247, tables per model.py:59-85) and the deformation
// field built from them (mapping.py:146-204).
//
// Pipeline:
//   reduce  : one CTA per TH x TW tile; d staged into shared memory by TMA; each lane
//             owns a column and sweeps the rows.  Emits per-tile aggregates: column
//             sums, row sums, the in-tile up-left / up-right chains of the column
//             prefix at the band's last row and at the tile's edge columns, and the
//             tile's diagonal / anti-diagonal partial sums.
//   scan    : float64 carry scan over the aggregates (1/TH of the data): rect_tl at
//             every band boundary (TLcar), the two diagonal carries X1/X2, the row
//             carries HC and the four marginals (row/column/diagonal/anti-diagonal).
//   write   : one CTA per tile re-sweeps its tile and produces
//               rect_tl = TLcar + VH + in-tile 2D prefix
//               wedge_up = T (in-band triangle, warp-shuffle chains) + X1 + X2
//             and derives the six other tables from the marginals
//               tr = Rpre - tl, bl = Cpre - tl, br = C - Rpre - Cpre + tl,
//               left = Apre - up, right = Dsuf - up, down = C - Apre - Dsuf + up,
//             then either streams the eight tables out or evaluates the field.
// No CTA ever waits on another CTA; everything is deterministic (fixed-order sums,
// no float atomics).
#include "inim_tiles.cuh"

namespace inim {

// =====================================================================================
// Flat response in closed form (mapping.py:104-129 evaluated analytically): the eight
// tables of a constant texture are pixel counts of the regions, integers computed
// exactly in int64, then combined exactly as _per_pixel_targets does.
// =====================================================================================
struct Anchors {
    double drx, dry, ulx, uly, urx, ury, dlx, dly;
};

// _anchor_components / _per_pixel_targets branch structure (mapping.py:40-52, 155-166).
__device__ __forceinline__ Anchors anchors_at(double x, double y) {
    Anchors A;
    if (y < x) {
        A.drx = 1.0; A.dry = 1.0 + y - x; A.ulx = x - y; A.uly = 0.0;
    } else {
        A.drx = 1.0 - y + x; A.dry = 1.0; A.ulx = 0.0; A.uly = y - x;
    }
    if (x + y < 1.0) {
        A.urx = x + y; A.ury = 0.0; A.dlx = 0.0; A.dly = x + y;
    } else {
        A.urx = 1.0; A.ury = x + y - 1.0; A.dlx = x + y - 1.0; A.dly = 1.0;
    }
    return A;
}

__device__ __forceinline__ double2 raw_map(const Anchors& A, double x, double y, double tl, double bl, double br,
                                           double tr, double up, double left, double down, double right,
                                           double inv) {
    double2 t;
    t.x = (tl * A.drx + bl * A.urx + br * A.ulx + tr * A.dlx + (up + down) * x + left) * inv;
    t.y = (tl * A.dry + bl * A.ury + br * A.uly + tr * A.dly + (left + right) * y + up) * inv;
    return t;
}

__device__ __forceinline__ double2 flat_response_at(int i, int j, int k) {
    const int64_t S = (int64_t)1 << k, s2 = S * S;
    const int64_t I = i, J = j;
    const double tl = (double)((I + 1) * (J + 1));
    const double bl = (double)((I + 1) * (S - 1 - J));
    const double tr = (double)((S - 1 - I) * (J + 1));
    const double br = (double)((S - 1 - I) * (S - 1 - J));
    auto f = [&](int64_t L) { return L * (J + 1) - L * (L + 1) / 2; };
    const int64_t up1 = (J + 1) + f(min(J, I)) + f(min(J, S - 1 - I));
    const int64_t sg = I + J;
    const int64_t A1 = sg <= S - 1 ? (sg + 1) * (sg + 2) / 2 : s2 - (2 * S - 2 - sg) * (2 * S - 1 - sg) / 2;
    const int64_t dl = I - J;
    const int64_t D1 = dl >= 0 ? (S - dl) * (S - dl + 1) / 2 : s2 - (S + dl - 1) * (S + dl) / 2;
    const int64_t left1 = A1 - up1, right1 = D1 - up1;
    const int64_t down1 = s2 - up1 - left1 - right1;
    const double scale = ldexp(1.0, -k);
    const double x = i * scale, y = j * scale;
    const Anchors A = anchors_at(x, y);
    return raw_map(A, x, y, tl, bl, br, tr, (double)up1, (double)left1, (double)down1, (double)right1,
                   0.5 / (double)s2);
}

// =====================================================================================
// Tile write (phase 3).  MODE 0: stream the eight tables.  MODE 1: evaluate the
// deformation field (build_field, mapping.py:194-204) in registers.
// =====================================================================================
struct WriteOut {
    float* tables8;      // MODE 0
    float* targets;      // MODE 1: (s, s, 2)
    const float* defect; // MODE 1: (s, s, 2) or null (closed form)
    float* max_exc;      // MODE 1
};

// Shared-memory carve-up of the write kernel.
struct WriteSmem {
    float* sd;      // TH*TW
    float* ULR;     // NW*TH
    float* URL;     // NW*TH
    float* WT;      // NW*TH
    float* OFF;     // NW*TH
    float* ule;     // TH
    float* ure;     // TH
    double* tl;     // TW
    double* x1;     // TW+TH
    double* x2;     // TW+TH
    double* cpre;   // TW
    double* apre;   // TW+TH
    double* dsuf;   // TW+TH
    double* rpre;   // TH
    double* vh;     // TH
    float* red;     // 32
    uint64_t* bar;  // 1
};

__host__ __device__ inline size_t write_smem_bytes(const Geo& g) {
    size_t f = (size_t)g.TH * g.TW + 4 * (size_t)g.NW * g.TH + 2 * (size_t)g.TH + 32;
    size_t fb = ((f * 4 + 15) / 16) * 16;
    size_t d = 2 * (size_t)g.TW + 4 * ((size_t)g.TW + g.TH) + 2 * (size_t)g.TH;
    return fb + d * 8 + 16;
}

__device__ inline WriteSmem carve_write(unsigned char* base, const Geo& g) {
    WriteSmem S;
    float* f = reinterpret_cast<float*>(base);
    S.sd = f; f += g.TH * g.TW;
    S.ULR = f; f += g.NW * g.TH;
    S.URL = f; f += g.NW * g.TH;
    S.WT = f; f += g.NW * g.TH;
    S.OFF = f; f += g.NW * g.TH;
    S.ule = f; f += g.TH;
    S.ure = f; f += g.TH;
    S.red = f; f += 32;
    size_t fb = (((size_t)(reinterpret_cast<unsigned char*>(f) - base)) + 15) / 16 * 16;
    double* d = reinterpret_cast<double*>(base + fb);
    S.tl = d; d += g.TW;
    S.x1 = d; d += g.TW + g.TH;
    S.x2 = d; d += g.TW + g.TH;
    S.cpre = d; d += g.TW;
    S.apre = d; d += g.TW + g.TH;
    S.dsuf = d; d += g.TW + g.TH;
    S.rpre = d; d += g.TH;
    S.vh = d; d += g.TH;
    S.bar = reinterpret_cast<uint64_t*>(d);
    return S;
}

__host__ __device__ inline size_t reduce_smem_bytes(const Geo& g) {
    return ((size_t)g.TH * g.TW + 3 * (size_t)g.NW * g.TH) * 4 + 16 + 16;
}

// Stage the tile of d into shared memory: TMA when the tile is TMA-shaped, otherwise
// a cooperative copy (tiny textures).
__device__ inline void load_tile(float* sd, uint64_t* bar, const CUtensorMap* map, const float* d, const Geo& g,
                                 int b, int x, bool use_tma) {
    const int TH = g.TH, TW = g.TW;
    if (use_tma) {
        if (threadIdx.x == 0) {
            mbar_init(bar, 1);
            fence_barrier_init();
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            mbar_arrive_expect_tx(bar, (uint32_t)(TH * TW * sizeof(float)));
            tma_load_2d(sd, map, x * TW, b * TH, bar);
        }
        mbar_wait(bar, 0);
    } else {
        for (int q = threadIdx.x; q < TH * TW; q += blockDim.x) {
            const int r = q / TW, u = q % TW;
            sd[q] = d[(int64_t)(b * TH + r) * g.s + x * TW + u];
        }
        __syncthreads();
    }
}

template <int MODE>
__device__ void tile_write(const WriteSmem& S, const Geo g, const Ws ws, int b, int x, const WriteOut out) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int TH = g.TH, TW = g.TW, NW = g.NW, WL = g.WL, s = g.s, NX = g.NX;
    const int u = w * 32 + lane;
    const bool act = u < TW;
    const int edge = WL - 1;
    const int a = b * TH, i0 = x * TW;
    const double C = *ws.total;

    // ---- stage the band vectors and marginal windows this tile needs
    for (int q = tid; q < TW + TH - 1; q += blockDim.x) {
        const int c1 = i0 - TH + q;
        S.x1[q] = c1 >= 0 ? ws.x1[(int64_t)b * s + c1] : 0.0;
        S.x2[q] = ws.x2[(int64_t)b * (s + TH) + i0 + 1 + q];
        S.apre[q] = ws.apre[a + i0 + q];
        S.dsuf[q] = ws.dsuf[i0 - a - (TH - 1) + q + (s - 1)];
    }
    for (int q = tid; q < TW; q += blockDim.x) {
        S.tl[q] = ws.tlcar[(int64_t)b * s + i0 + q];
        S.cpre[q] = ws.tlcar[(int64_t)g.B * s + i0 + q];
    }
    if (tid < 32) {
        // VH[r] = sum_{r' <= r} HC[a + r'][x]  (row carries of the tile's rows)
        const double hcv = tid < TH ? ws.hc[(int64_t)(a + tid) * NX + x] : 0.0;
        const double vh = warp_inclusive_scan_d(hcv, lane);
        if (tid < TH) {
            S.vh[tid] = vh;
            S.rpre[tid] = ws.rpre[a + tid];
            S.ule[tid] = x > 0 ? ws.ule[((int64_t)b * NX + x - 1) * TH + tid] : 0.f;
            S.ure[tid] = x < NX - 1 ? ws.ure[((int64_t)b * NX + x + 1) * TH + tid] : 0.f;
        }
    }

    // ---- pass A: per-warp row totals of the column prefix and warp-edge chain values
    {
        float V = 0.f, ULw = 0.f, URw = 0.f;
        for (int r = 0; r < TH; ++r) {
            const float dv = act ? S.sd[r * TW + u] : 0.f;
            V += dv;
            const float upUL = __shfl_up_sync(kFull, ULw, 1);
            const float dnUR = __shfl_down_sync(kFull, URw, 1);
            ULw = V + (lane > 0 ? upUL : 0.f);
            URw = V + (lane < 31 ? dnUR : 0.f);
            const float wt = warp_sum(V);
            if (lane == edge) S.ULR[w * TH + r] = ULw;
            if (lane == 0) {
                S.URL[w * TH + r] = URw;
                S.WT[w * TH + r] = wt;
            }
        }
    }
    __syncthreads();
    for (int q = tid; q < NW * TH; q += blockDim.x) {
        const int ww = q / TH, r = q % TH;
        float o = 0.f;
        for (int v = 0; v < ww; ++v) o += S.WT[v * TH + r];
        S.OFF[q] = o;
    }
    __syncthreads();

    // ---- pass B: final values row by row
    const float* Esrc = w > 0 ? S.ULR + (w - 1) * TH : S.ule;
    const float* Fsrc = w < NW - 1 ? S.URL + (w + 1) * TH : S.ure;
    const double scale = ldexp(1.0, -g.k);
    const double inv = 0.5 / C;
    float exc = 0.f;
    float V = 0.f, ULw = 0.f, URw = 0.f;
    for (int r = 0; r < TH; ++r) {
        const float dv = act ? S.sd[r * TW + u] : 0.f;
        V += dv;
        const float upUL = __shfl_up_sync(kFull, ULw, 1);
        const float dnUR = __shfl_down_sync(kFull, URw, 1);
        ULw = V + (lane > 0 ? upUL : 0.f);
        URw = V + (lane < 31 ? dnUR : 0.f);
        const float inc = warp_inclusive_scan(V, lane);
        if (!act) continue;
        const float local = inc + S.OFF[w * TH + r];
        const int re = r - lane - 1;
        const int rq = r - (WL - lane);
        const float eUL = re >= 0 ? Esrc[re] : 0.f;
        const float eUR = rq >= 0 ? Fsrc[rq] : 0.f;
        const float T = (ULw + eUL) + (URw + eUR) - V;

        const double tl = S.tl[u] + S.vh[r] + (double)local;
        const double up = (double)T + S.x1[u - r - 1 + TH] + S.x2[u + r];
        const double Rp = S.rpre[r], Cp = S.cpre[u], Ap = S.apre[u + r], Ds = S.dsuf[u - r + TH - 1];
        const double tr = Rp - tl;
        const double bl = Cp - tl;
        const double br = C - Rp - Cp + tl;
        const double left = Ap - up;
        const double right = Ds - up;
        const double down = C - Ap - Ds + up;
        const int j = a + r, i = i0 + u;
        const int64_t q = (int64_t)j * s + i;
        if (MODE == 0) {
            float* T8 = out.tables8;
            const int64_t m = g.m;
            st_stream(T8 + q, (float)tl);
            st_stream(T8 + m + q, (float)bl);
            st_stream(T8 + 2 * m + q, (float)br);
            st_stream(T8 + 3 * m + q, (float)tr);
            st_stream(T8 + 4 * m + q, (float)up);
            st_stream(T8 + 5 * m + q, (float)left);
            st_stream(T8 + 6 * m + q, (float)down);
            st_stream(T8 + 7 * m + q, (float)right);
        } else {
            const double xx = i * scale, yy = j * scale;
            const Anchors A = anchors_at(xx, yy);
            const double2 raw = raw_map(A, xx, yy, tl, bl, br, tr, up, left, down, right, inv);
            double2 def;
            if (out.defect) {
                const float2 dfv = reinterpret_cast<const float2*>(out.defect)[q];
                def.x = dfv.x;
                def.y = dfv.y;
            } else {
                def = flat_response_at(i, j, g.k);
            }
            const float gx = (float)(raw.x - def.x + xx);
            const float gy = (float)(raw.y - def.y + yy);
            exc = fmaxf(exc, fmaxf(fmaxf(-gx, -gy), fmaxf(gx - 1.f, gy - 1.f)));
            st_stream2(reinterpret_cast<float2*>(out.targets) + q,
                       make_float2(fminf(fmaxf(gx, 0.f), 1.f), fminf(fmaxf(gy, 0.f), 1.f)));
        }
    }
    if (MODE == 1) {
        exc = warp_max(exc);
        if (lane == 0) S.red[w] = exc;
        __syncthreads();
        if (tid == 0) {
            float e = 0.f;
            for (int v = 0; v < NW; ++v) e = fmaxf(e, S.red[v]);
            atomic_max_nonneg(out.max_exc, e);
        }
    }
}

// =====================================================================================
// Kernels
// =====================================================================================
__global__ void __launch_bounds__(256) reduce_kernel(const __grid_constant__ CUtensorMap map, const float* d,
                                                     const Geo g, const Ws ws, int use_tma) {
    extern __shared__ __align__(128) unsigned char smem[];
    float* sd = reinterpret_cast<float*>(smem);
    float* rec = sd + g.TH * g.TW;
    uint64_t* bar = reinterpret_cast<uint64_t*>(
        (reinterpret_cast<uintptr_t>(rec + 3 * g.NW * g.TH) + 15) & ~uintptr_t(15));
    const int x = blockIdx.x, b = blockIdx.y;
    if (use_tma && threadIdx.x == 0) prefetch_tensormap(&map);
    load_tile(sd, bar, &map, d, g, b, x, use_tma);
    tile_reduce(sd, rec, g, ws, b, x, threadIdx.x);
}

template <int MODE>
__global__ void __launch_bounds__(256) write_kernel(const __grid_constant__ CUtensorMap map, const float* d,
                                                    const Geo g, const Ws ws, const WriteOut out, int use_tma,
                                                    const int* state) {
    if (state && state[0]) return;  // displacement stop already reached
    extern __shared__ __align__(128) unsigned char smem[];
    WriteSmem S = carve_write(smem, g);
    const int x = blockIdx.x, b = blockIdx.y;
    if (use_tma && threadIdx.x == 0) prefetch_tensormap(&map);
    load_tile(S.sd, S.bar, &map, d, g, b, x, use_tma);
    tile_write<MODE>(S, g, ws, b, x, out);
}

// ---- standalone helpers ----------------------------------------------------------------

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
        const double xx = i * scale, yy = j * scale;
        const Anchors A = anchors_at(xx, yy);
        const double2 raw = raw_map(A, xx, yy, t8[q], t8[m + q], t8[2 * m + q], t8[3 * m + q], t8[4 * m + q],
                                    t8[5 * m + q], t8[6 * m + q], t8[7 * m + q], 0.5 / *total);
        double2 def;
        if (defect) {
            def.x = defect[2 * q];
            def.y = defect[2 * q + 1];
        } else {
            def = flat_response_at(i, j, k);
        }
        const float gx = (float)(raw.x - def.x + xx), gy = (float)(raw.y - def.y + yy);
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
    // start cells: predecessor (j - dj, i - di) out of range
    int j, i;
    int nrow = dj != 0 ? s : 0;  // starts on the entry row
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
static bool tma_ok(const Geo& g) { return g.TW >= 32; }

int launch_reduce_from_global(const float* d, const Geo& g, const Ws& ws, const CUtensorMap* map,
                              cudaStream_t st) {
    const size_t smem = reduce_smem_bytes(g);
    const int use_tma = (map != nullptr && tma_ok(g)) ? 1 : 0;
    CUtensorMap dummy;
    memset(&dummy, 0, sizeof(dummy));
    dim3 grid(g.NX, g.B);
    reduce_kernel<<<grid, g.NW * 32, smem, st>>>(use_tma ? *map : dummy, d, g, ws, use_tma);
    prof_mark(st, "reduce");
    return (int)cudaGetLastError();
}


template <int MODE>
static int launch_write_mode(const float* d, const Geo& g, const Ws& ws, const CUtensorMap* map,
                             const WriteOut& out, const int* state, cudaStream_t st) {
    const size_t smem = write_smem_bytes(g);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(write_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        attr_set = true;
    }
    const int use_tma = (map != nullptr && tma_ok(g)) ? 1 : 0;
    CUtensorMap dummy;
    memset(&dummy, 0, sizeof(dummy));
    dim3 grid(g.NX, g.B);
    write_kernel<MODE><<<grid, g.NW * 32, smem, st>>>(use_tma ? *map : dummy, d, g, ws, out, use_tma, state);
    prof_mark(st, MODE == 0 ? "write_tables" : "write_field");
    return (int)cudaGetLastError();
}

int launch_write_tables(const float* d, const Geo& g, const Ws& ws, const CUtensorMap* map, float* tables8,
                        cudaStream_t st) {
    WriteOut o{tables8, nullptr, nullptr, nullptr};
    return launch_write_mode<0>(d, g, ws, map, o, nullptr, st);
}

int launch_write_field(const float* d, const Geo& g, const Ws& ws, const CUtensorMap* map, const float* defect,
                       float* targets, float* max_exc, const int* state, cudaStream_t st) {
    WriteOut o{nullptr, targets, defect, max_exc};
    return launch_write_mode<1>(d, g, ws, map, o, state, st);
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
