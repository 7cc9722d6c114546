// C ABI (include/inim.h): argument checks, launch sequencing, the device-resident
// iteration (regularize.iterate_once / run, reference regularize.py:25-80) and its
// CUDA-graph replay.
#include <string.h>

#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

#include <omp.h>

#include "inim_internal.cuh"

namespace inim {
int launch_splat_f32(const float* pts, int64_t n, int k, uint32_t* counts, const int* state, cudaStream_t st,
                     float* zero0 = nullptr, float* zero1 = nullptr, const Bat& bt = Bat{});
int launch_splat_f64(const double* pts, int64_t n, int k, uint32_t* counts, cudaStream_t st);
int launch_sample_f32(const float* tg, int k, const float* in, float* out, int64_t n, int clip, float* max_disp,
                      const int* state, cudaStream_t st, bool pairs = false, uint32_t* splat_next = nullptr,
                      float* zn0 = nullptr, float* zn1 = nullptr, bool sorted = false, const Bat& bt = Bat{},
                      int64_t zin = 0, int64_t zout = 0, bool f32_counts = false);
int launch_sample_f64(const float* tg, int k, const double* in, double* out, int64_t n, int clip, cudaStream_t st);
int launch_cast_f64_f32(const double* in, float* out, int64_t count, cudaStream_t st);
int launch_cast_f32_f64(const float* in, double* out, int64_t count, cudaStream_t st);
int launch_smooth_state(const void* in, int in_kind, const Geo& g, const Ws& ws, int kernel_size,
                        float background, float* d, bool emit_aggregates, const int* state, cudaStream_t st,
                        uint32_t* zero_next = nullptr, const Bat& bt = Bat{});
int launch_field_from_tables(const float* t8, int k, const double* total, const float* defect, float* targets,
                             float* max_exc, cudaStream_t st);
int launch_flat_response(int k, float* defect, cudaStream_t st);
int launch_line_scan(const float* in, float* out, int s, int dj, int di, int exclusive, cudaStream_t st);
size_t sort_bsum_words(int k);
int launch_sort_points(const float* pts, int64_t n, int k, const uint32_t* counts, uint32_t* cursor,
                       uint32_t* bsum, float* sorted, uint32_t* rank, cudaStream_t st, const Bat& bt = Bat{});
int launch_unpermute(const float* sorted, const uint32_t* rank, int64_t n, float* out, cudaStream_t st,
                     const Bat& bt = Bat{});
int launch_frame_stats(const uint32_t* counts, int k, unsigned long long* out3, cudaStream_t st,
                       const Bat& bt = Bat{}, int64_t zout = 0, bool f32_counts = false);
int launch_gather_points(const void* pts, int is_f64, const int64_t* rows, const uint32_t* perm, int64_t m,
                         double* out, cudaStream_t st);
int launch_trust(const double* orig, const double* moved, int64_t n, int nn, unsigned long long* out,
                 cudaStream_t st);
int launch_order_pairs(const double* orig, const double* moved, int64_t n, unsigned long long* out, cudaStream_t st);

// Field layout the move gathers from: the paired layout (slot i = (t(i), t(i+1)), two
// 16-byte gathers per point) while the field stays L2-resident, the plain (s, s, 2)
// layout (half the bytes written and gathered, four 8-byte gathers) above 2048^2
// (measured: 1024^2 paired -5% per iteration; 4096^2 plain -11%), and for plot batches,
// whose fields stream through HBM.  INIM_PAIRS=0/1 forces either.
static bool use_pairs(const Geo& g, bool batched) {
    static int env = -1;
    if (env < 0) {
        const char* e = getenv("INIM_PAIRS");
        env = e ? (e[0] == '0' ? 0 : 1) : 2;
    }
    return env == 2 ? g.s <= 2048 && !batched : env == 1;
}

// Float32 counts with 16-byte reductions in the sorted moves (INIM_F32_COUNTS=0: uint32
// counts and one reduction per distinct pixel; A/B and the bit-identity test).
static bool f32_counts_enabled() {
    static int env = -1;
    if (env < 0) {
        const char* e = getenv("INIM_F32_COUNTS");
        env = (e && e[0] == '0') ? 0 : 1;
    }
    return env == 1;
}

// Pixel-order sort of the points inside inim_run (INIM_SORT=0 disables).
constexpr int64_t kSortMinPoints = 1 << 16;
constexpr int kSortMinIters = 3;
static bool sort_points_enabled() {
    static int env = -1;
    if (env < 0) {
        const char* e = getenv("INIM_SORT");
        env = (e && e[0] == '0') ? 0 : 1;
    }
    return env == 1;
}

bool pdl_enabled() {
    static int env = -1;
    if (env < 0) {
        const char* e = getenv("INIM_PDL");
        env = (e && e[0] == '0') ? 0 : 1;
    }
    return env == 1;
}

// Per-iteration bookkeeping for the displacement criterion (regularize.py:76-79).
__global__ void iter_end_kernel(const float* disp, float eps, int* state, int64_t zslab) {
    pdl_enter();
    state = zoff(state, zslab_off(zslab));  // plot blockIdx.z of a batch
    disp = zoff(disp, zslab_off(zslab));
    if (state[0]) return;
    state[1] += 1;
    if (*disp < eps) state[0] = 1;
}

// Workspace = integral layout + grid buffers (two count buffers: the splat of
// iteration t+1 fills the one the smoothing of iteration t cleared; the flat response
// for grids up to 2048^2, read from L2 instead of re-derived per pixel) + point
// ping-pong.
struct FullLayout {
    WsLayout L;
    size_t counts, d, targets, defect, scratch, state, sortA, sortB, perm, rank, hist, bytes;
};

// The field kernel folds the closed-form flat response into its normalised arithmetic,
// so the run loop keeps no defect array.
static bool precomputed_defect(const Geo&) { return false; }

static FullLayout full_layout(const Geo& g, int64_t n) {
    FullLayout F;
    F.L = make_layout(g);
    size_t o = F.L.bytes;
    auto take = [&](size_t bytes) {
        size_t r = o;
        o = align256(o + bytes);
        return r;
    };
    F.counts = take(sizeof(uint32_t) * 2 * g.m);
    F.d = take(sizeof(float) * g.m);
    F.targets = take(sizeof(float) * 4 * g.m);  // paired field layout (also holds a plain field)
    F.defect = take(precomputed_defect(g) ? sizeof(float) * 2 * g.m : 0);
    F.scratch = take(sizeof(float) * 64);
    F.state = take(sizeof(int) * 4);  // a batched run's per-plot {stopped, iterations done}
    const size_t nn = (size_t)(n > 0 ? n : 1);
    F.sortA = take(sizeof(float) * 2 * nn);  // points in cell order (ping)
    F.sortB = take(sizeof(float) * 2 * nn);  // (pong)
    F.perm = take(sizeof(uint32_t) * nn);    // input row -> sorted slot
    F.rank = take(0);
    F.hist = take(sizeof(uint32_t) * sort_bsum_words(g.k));  // block sums of the sort's scan
    F.bytes = o;
    return F;
}

static bool k_ok(int k) { return k >= 0 && k <= INIM_MAX_K; }

// Chaining of consecutive iterations inside a run: the move of iteration t splats its
// output into iteration t+1's count buffer and clears t+1's device scalars.
struct Chain {
    bool splatted;       // this iteration's counts were filled by the previous move
    bool splat_next;     // fuse the next iteration's splat into this move
    float *next_exc, *next_disp;
    bool sorted;         // the points are in pixel order (aggregated splat atomics)
    bool f32_in = false;   // this iteration's counts are float32 (the previous move's 16-byte reductions)
    bool f32_next = false; // the move splats float32 counts
};

// One iteration.  `counts` must be zero on entry (or already filled, chain.splatted);
// `counts_next` (optional) is cleared by the smoothing pass for the next iteration.
// With `pairs` the field is (also) written in the paired layout and the move reads
// that; `targets` may then be null.  `bt`: a batch of plots (grid.z), with zin / zout
// the plot strides (floats) of pts_in / pts_out.
static int enqueue_iteration(const float* pts_in, float* pts_out, int64_t n, const Geo& g, int kernel_size,
                             float background, const float* defect, uint32_t* counts, uint32_t* counts_next, float* d,
                             float* targets, float* max_exc, float* disp, float stop_eps, int* state, const Ws& ws,
                             const CUtensorMap* map, cudaStream_t st, float* pairs = nullptr,
                             const Chain& chain = Chain{false, false, nullptr, nullptr, false},
                             const Bat& bt = Bat{}, int64_t zin = 0, int64_t zout = 0) {
    const int* flag = stop_eps > 0.f ? state : nullptr;
    int rc = 0;
    if (!chain.splatted) {
        rc = launch_splat_f32(pts_in, n, g.k, counts, flag, st, max_exc, disp, Bat{bt.B, bt.slab, zin});
        if (rc) return rc;
    }
    rc = launch_smooth_state(counts, chain.f32_in ? 2 : 1, g, ws, kernel_size, background, d, true, flag, st,
                             counts_next, bt);
    if (rc) return rc;
    rc = launch_carry_scan_state(g, ws, flag, st, bt);
    if (rc) return rc;
    rc = launch_write_field(d, g, ws, map, defect, targets, max_exc, flag, st, pairs, bt);
    if (rc) return rc;
    uint32_t* sn = chain.splat_next ? counts_next : nullptr;
    rc = pairs ? launch_sample_f32(pairs, g.k, pts_in, pts_out, n, 1, disp, flag, st, true, sn, chain.next_exc,
                                   chain.next_disp, chain.sorted, bt, zin, zout, chain.f32_next)
               : launch_sample_f32(targets, g.k, pts_in, pts_out, n, 1, disp, flag, st, false, sn, chain.next_exc,
                                   chain.next_disp, chain.sorted, bt, zin, zout, chain.f32_next);
    if (rc) return rc;
    if (flag) {
        INIM_CUDA_TRY(launch_pdl(iter_end_kernel, dim3(1, 1, bt.B), dim3(1), 0, st, (const float*)disp, stop_eps,
                                 state, bt.slab));
        prof_mark(st, "iter_end");
    }
    return (int)cudaGetLastError();
}

Prof* g_prof = nullptr;

static float auto_background(int64_t n, int k, float background) {
    if (background > 0.f) return background;
    double bg = (double)n / (double)((int64_t)1 << (2 * k));
    return bg == 0.0 ? 1.0f : (float)bg;
}

// ---- graph cache for inim_run ---------------------------------------------------------
struct RunKey {
    const void* pts;
    int64_t n;
    int k, ks;
    float bg;
    int iters;
    float eps;
    const void *frames, *fields, *disp, *exc, *state, *ws;
    cudaStream_t st;
    // per-frame metrics (regularize.py:55-59,71-75); all null = none
    const void *fstats, *orig_sub, *pick, *moved_sub, *nbstats;
    int64_t n_sub;
    int n_neighbors;
    int B;  // plots of an inim_run_batched call (>= 1); 0 for inim_run
    bool operator==(const RunKey& o) const { return memcmp(this, &o, sizeof(RunKey)) == 0; }
};

struct RunEntry {
    RunKey key;
    cudaGraphExec_t exec;
};

static std::mutex g_mu;
static std::vector<RunEntry> g_cache;

// The run (regularize.run's numeric loop) for one plot, or for a batch of key.B plots
// with the plot index in every launch's grid.z (then frames / fields / disp /
// excursions / state / neighbourhood metrics are not recorded: fixed iterations only).
static int enqueue_run(const RunKey& key, float* pts, float* frames, float* fields, float* disp, float* excursions,
                       int* state, void* ws, cudaStream_t st) {
    const int B = key.B > 1 ? key.B : 1;
    const bool batched = key.B > 0;              // inim_run_batched (any B, one plot included)
    const Geo g = make_geo(key.k, batched);      // batches: the wide tile geometry
    const FullLayout F = full_layout(g, key.n);
    const Ws w = make_ws(ws, F.L);
    // plot strides: workspace slabs (bytes) and the caller's (B, n, 2) points (floats)
    const Bat bt{B, B > 1 ? (int64_t)F.bytes : 0, B > 1 ? 2 * key.n : 0};
    const int64_t zs = bt.slab / (int64_t)sizeof(float);  // slab stride in floats (workspace point buffers)
    char* base = static_cast<char*>(ws);
    uint32_t* counts = reinterpret_cast<uint32_t*>(base + F.counts);
    float* d = reinterpret_cast<float*>(base + F.d);
    float* tg_scratch = reinterpret_cast<float*>(base + F.targets);
    float* defect = precomputed_defect(g) ? reinterpret_cast<float*>(base + F.defect) : nullptr;
    float* scratch = reinterpret_cast<float*>(base + F.scratch);
    float* sortA = reinterpret_cast<float*>(base + F.sortA);
    float* sortB = reinterpret_cast<float*>(base + F.sortB);
    int* perm = reinterpret_cast<int*>(base + F.perm);
    int* hist = reinterpret_cast<int*>(base + F.hist);
    // a batch's displacement stop runs on per-plot state words in the slabs (every
    // kernel offsets them by its plot); the caller's states[B][4] receive them at the end
    int* const caller_states = batched ? state : nullptr;
    if (batched) state = key.eps > 0.f ? reinterpret_cast<int*>(base + F.state) : nullptr;
    if (batched && state)
        INIM_CUDA_TRY(cudaMemset2DAsync(state, B > 1 ? (size_t)bt.slab : 4 * sizeof(int), 0, 4 * sizeof(int), (size_t)B,
                                        st));
    CUtensorMap map;
    const CUtensorMap* mp = nullptr;
    if (g.TW >= 32) {
        int rc = make_tensor_map_2d(&map, d, g.s, g.TW, g.TH);
        if (rc) return rc;
        mp = &map;
    }
    // once per run: the first count buffer cleared (iteration 0's smoothing clears the
    // other one for iteration 1); a batch clears every plot's with one 2-D memset
    if (B > 1)
        INIM_CUDA_TRY(cudaMemset2DAsync(counts, (size_t)bt.slab, 0, sizeof(uint32_t) * g.m, (size_t)B, st));
    else
        INIM_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(uint32_t) * g.m, st));
    prof_mark(st, "memset_counts");
    if (defect) {
        int rc = launch_flat_response(g.k, defect, st);
        if (rc) return rc;
    }
    const size_t pbytes = sizeof(float) * 2 * (size_t)key.n;
    if (frames && key.n > 0) INIM_CUDA_TRY(cudaMemcpyAsync(frames, pts, pbytes, cudaMemcpyDeviceToDevice, st));
    // Per-frame metrics: occupancy statistics of frame t+1 come off the counts the move
    // of iteration t splats (so the last move splats too); neighbourhood metrics of the
    // fixed subsample against frame 0.  A batch keeps plot z's statistics at
    // fstats[z][t][3].
    unsigned long long* fstats = (unsigned long long*)key.fstats;
    unsigned long long* nbstats = (unsigned long long*)key.nbstats;
    const bool nb = fstats && key.orig_sub && nbstats && key.moved_sub && key.n_sub > 0 && B == 1;
    if (fstats) INIM_CUDA_TRY(cudaMemsetAsync(fstats, 0, sizeof(unsigned long long) * 3 * key.iters * B, st));
    if (nb) INIM_CUDA_TRY(cudaMemsetAsync(nbstats, 0, sizeof(unsigned long long) * 2 * key.iters, st));
    // Spatial order: for runs long enough to amortise it, the points are sorted by pixel
    // once (from the counts of iteration 0's splat, which the run needs anyway), the
    // moves then gather coalesced field rows and merge their splat atomics, and the
    // final positions (and recorded frames) are scattered back through perm.
    const bool sorted = sort_points_enabled() && key.n >= kSortMinPoints && key.iters >= kSortMinIters;
    // sorted runs splat the moves' points with 16-byte float reductions (a request per
    // group of four pixels): float32 counts stay exact integers below 2^24 points.
    // Measured: C4 -2%, C2 -0.4%; one 4096^2 plot +1.4% (kept on uint32)
    const bool f32 = sorted && key.n < ((int64_t)1 << 24) && (batched || g.s <= 2048) && f32_counts_enabled();
    auto disp_at = [&](int t) { return disp ? disp + t : scratch + 2 * (t & 1); };
    auto exc_at = [&](int t) { return excursions ? excursions + t : scratch + 2 * (t & 1) + 1; };
    if (sorted) {
        const int* flag = key.eps > 0.f ? state : nullptr;
        int rc = launch_splat_f32(pts, key.n, g.k, counts, flag, st, exc_at(0), disp_at(0), bt);
        if (rc) return rc;
        // the other count buffer is the sort's cursor; iteration 0's smoothing clears it
        rc = launch_sort_points(pts, key.n, g.k, counts, counts + g.m, reinterpret_cast<uint32_t*>(hist), sortA,
                                reinterpret_cast<uint32_t*>(perm), st, bt);
        if (rc) return rc;
    }
    // Point buffers: unsorted, the first move reads the caller's array and the last one
    // writes it back (no staging copies); in between the moves ping-pong through
    // sortA / sortB.  Each buffer's plot stride: the caller's array bt.pts, the
    // workspace buffers one slab.
    float* bufs[2] = {sortB, sortA};
    auto pos_in = [&](int t) -> float* {
        if (t == 0) return sorted ? sortA : pts;
        return bufs[t & 1];
    };
    auto pos_out = [&](int t) -> float* {
        if (t == key.iters - 1 && !sorted) return pts;
        return bufs[(t + 1) & 1];
    };
    auto zstride = [&](const float* p) -> int64_t { return p == pts ? bt.pts : zs; };
    // per-iteration device scalars: recorded arrays, else two alternating scratch slots
    // (the move of iteration t clears iteration t+1's slot while t's is still live)
    for (int t = 0; t < key.iters; ++t) {
        float* src = pos_in(t);
        float* dst = pos_out(t);
        float* tg = fields ? fields + (size_t)t * 2 * g.m : nullptr;  // plain field only when recorded
        uint32_t* cur = counts + (size_t)(t & 1) * g.m;
        uint32_t* next = counts + (size_t)((t + 1) & 1) * g.m;
        const bool more = t + 1 < key.iters && key.n > 0;
        const bool splat_next = more || (fstats && key.n > 0);
        const Chain chain{t > 0 || sorted, splat_next, more ? exc_at(t + 1) : nullptr,
                          more ? disp_at(t + 1) : nullptr, sorted, f32 && t > 0, f32};
        // the move reads the paired field layout (two 16-byte gathers per point) while the
        // field stays L2-resident: one plot up to 2048^2 (INIM_PAIRS overrides); a batch's
        // fields stream through HBM, where the plain (s, s, 2) layout's half bytes win
        const bool pairs = use_pairs(g, batched);
        float* plain = tg ? tg : (pairs ? nullptr : tg_scratch);
        int rc = enqueue_iteration(src, dst, key.n, g, key.ks, key.bg, defect, cur, next, d, plain, exc_at(t),
                                   disp_at(t), key.eps, state, w, mp, st, pairs ? tg_scratch : nullptr, chain, bt,
                                   zstride(src), zstride(dst));
        if (rc) return rc;
        if (frames && key.n > 0) {
            float* fr = frames + (size_t)(t + 1) * 2 * key.n;
            rc = sorted ? launch_unpermute(dst, reinterpret_cast<const uint32_t*>(perm), key.n, fr, st)
                        : (int)cudaMemcpyAsync(fr, dst, pbytes, cudaMemcpyDeviceToDevice, st);
            if (rc) return rc;
        }
        if (fstats && key.n > 0) {
            rc = launch_frame_stats(next, g.k, fstats + 3 * t, st, bt, 3 * (int64_t)key.iters, f32);
            if (rc) return rc;
        }
        if (nb && key.n > 0) {
            double* msub = (double*)key.moved_sub;
            rc = launch_gather_points(dst, 0, (const int64_t*)key.pick, sorted ? (const uint32_t*)perm : nullptr,
                                      key.n_sub, msub, st);
            if (!rc) rc = launch_trust((const double*)key.orig_sub, msub, key.n_sub, key.n_neighbors, nbstats + 2 * t, st);
            if (!rc) rc = launch_order_pairs((const double*)key.orig_sub, msub, key.n_sub, nbstats + 2 * t + 1, st);
            if (rc) return rc;
        }
    }
    if (sorted && key.iters > 0) {
        int rc = launch_unpermute(pos_out(key.iters - 1), reinterpret_cast<const uint32_t*>(perm), key.n, pts, st, bt);
        if (rc) return rc;
    }
    if (caller_states && state)
        INIM_CUDA_TRY(cudaMemcpy2DAsync(caller_states, 4 * sizeof(int), state, B > 1 ? (size_t)bt.slab : 4 * sizeof(int),
                                        4 * sizeof(int), (size_t)B, cudaMemcpyDeviceToDevice, st));
    return 0;
}

}  // namespace inim

using namespace inim;

// ------------------------------------------------------------ host <-> device staging
// Pipelined host transfers for host (pageable) float64 buffers: the host narrows /
// widens chunks in parallel (OpenMP) through two page-locked float32 slots while the
// DMA engine moves the other slot, so the copy runs at page-locked PCIe speed on half
// the bytes instead of a single-threaded pageable float64 copy.  float64 <-> float32 on
// the host is the same IEEE round-to-nearest conversion as the device cast kernels.
namespace {
constexpr int64_t kStageChunk = int64_t(1) << 18;  // floats per slot (1 MiB)

struct Staging {
    std::mutex mu;
    float* slot[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    int dev = -1;
};
Staging g_stage;

int staging_ready(Staging& S) {
    int dev = 0;
    INIM_CUDA_TRY(cudaGetDevice(&dev));
    if (S.slot[0] && S.dev == dev) return 0;
    for (int q = 0; q < 2; ++q) {
        if (S.slot[q]) {
            cudaFreeHost(S.slot[q]);
            cudaEventDestroy(S.done[q]);
        }
        INIM_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&S.slot[q]), kStageChunk * sizeof(float),
                                    cudaHostAllocDefault));
        INIM_CUDA_TRY(cudaEventCreateWithFlags(&S.done[q], cudaEventDisableTiming));
        INIM_CUDA_TRY(cudaEventRecord(S.done[q], 0));
    }
    S.dev = dev;
    return 0;
}

int stage_threads(int64_t count) {
    const int t = omp_get_max_threads();
    const int cap = count >= (int64_t(1) << 16) ? 16 : 1;
    return t < cap ? t : cap;
}
}  // namespace

extern "C" {

const char* inim_version(void) { return "libinim sm_100a 0.1"; }

size_t inim_workspace_bytes(int k, int64_t n, int B) {
    if (!k_ok(k) || n < 0) return 0;
    // a slab holds either geometry: inim_run (16 x 64 tiles up to 2048^2) and
    // inim_run_batched (32 x 128 tiles from 128^2 up, any B) share the size
    const size_t slab = std::max(full_layout(make_geo(k, false), n).bytes, full_layout(make_geo(k, true), n).bytes);
    return slab * (size_t)(B > 1 ? B : 1);
}

int inim_splat(const void* pts, int pts_is_f64, int64_t n, int k, uint32_t* counts, cudaStream_t stream) {
    if (!k_ok(k) || n < 0 || !counts || (n > 0 && !pts)) return INIM_EINVAL;
    if (n == 0) return 0;
    return pts_is_f64 ? launch_splat_f64(static_cast<const double*>(pts), n, k, counts, stream)
                      : launch_splat_f32(static_cast<const float*>(pts), n, k, counts, nullptr, stream);
}

int inim_smooth_counts(const uint32_t* counts, int k, int kernel_size, float background, float* d, void* ws,
                       cudaStream_t stream) {
    if (!k_ok(k) || !counts || !d || !ws) return INIM_EINVAL;
    const Geo g = make_geo(k);
    return launch_smooth_state(counts, true, g, make_ws(ws, make_layout(g)), kernel_size, background, d, true, nullptr,
                               stream);
}

int inim_smooth_grid(const float* grid, int k, int kernel_size, float* out, void* ws, cudaStream_t stream) {
    if (!k_ok(k) || !grid || !out || !ws) return INIM_EINVAL;
    const Geo g = make_geo(k);
    return launch_smooth_state(grid, false, g, make_ws(ws, make_layout(g)), kernel_size, 0.f, out, false, nullptr,
                               stream);
}

int inim_integral_set(const float* d, int k, float* tables8, double* total, void* ws, cudaStream_t stream) {
    if (!k_ok(k) || !d || !tables8 || !ws) return INIM_EINVAL;
    const Geo g = make_geo(k);
    const Ws w = make_ws(ws, make_layout(g));
    CUtensorMap map;
    const CUtensorMap* mp = nullptr;
    if (g.TW >= 32) {
        int rc = make_tensor_map_2d(&map, d, g.s, g.TW, 8);  // the reduce's TMA ring (8-row chunks)
        if (rc) return rc;
        mp = &map;
    }
    int rc = launch_reduce_from_global(d, g, w, mp, stream);
    if (rc) return rc;
    rc = launch_carry_scan_state(g, w, nullptr, stream);
    if (rc) return rc;
    rc = launch_write_tables(d, g, w, mp, tables8, stream);
    if (rc) return rc;
    if (total) INIM_CUDA_TRY(cudaMemcpyAsync(total, w.total, sizeof(double), cudaMemcpyDeviceToDevice, stream));
    return 0;
}

int inim_column_integrals(const float* d, int k, float* upper, float* lower, cudaStream_t stream) {
    if (!k_ok(k) || !d || !upper || !lower) return INIM_EINVAL;
    const int s = 1 << k;
    int rc = launch_line_scan(d, upper, s, 1, 0, 0, stream);   // rows <= j (integral.py:185)
    if (rc) return rc;
    return launch_line_scan(d, lower, s, -1, 0, 1, stream);    // rows > j (integral.py:186)
}

int inim_line_scan(const float* in, float* out, int k, int dj, int di, int exclusive, cudaStream_t stream) {
    if (!k_ok(k) || !in || !out || dj < -1 || dj > 1 || di < -1 || di > 1 || (dj == 0 && di == 0)) return INIM_EINVAL;
    return launch_line_scan(in, out, 1 << k, dj, di, exclusive, stream);
}

int inim_field_from_density(const float* d, int k, const float* defect, float* targets, float* max_excursion,
                            double* total, void* ws, cudaStream_t stream) {
    if (!k_ok(k) || !d || !targets || !max_excursion || !ws) return INIM_EINVAL;
    const Geo g = make_geo(k);
    const Ws w = make_ws(ws, make_layout(g));
    CUtensorMap map;
    const CUtensorMap* mp = nullptr;
    if (g.TW >= 32) {
        int rc = make_tensor_map_2d(&map, d, g.s, g.TW, 8);  // the reduce's TMA ring (8-row chunks)
        if (rc) return rc;
        mp = &map;
    }
    int rc = launch_reduce_from_global(d, g, w, mp, stream);
    if (rc) return rc;
    rc = launch_carry_scan_state(g, w, nullptr, stream);
    if (rc) return rc;
    rc = launch_write_field(d, g, w, mp, defect, targets, max_excursion, nullptr, stream);
    if (rc) return rc;
    if (total) INIM_CUDA_TRY(cudaMemcpyAsync(total, w.total, sizeof(double), cudaMemcpyDeviceToDevice, stream));
    return 0;
}

int inim_field_from_tables(const float* tables8, int k, const double* total, const float* defect, float* targets,
                           float* max_excursion, cudaStream_t stream) {
    if (!k_ok(k) || !tables8 || !total || !targets || !max_excursion) return INIM_EINVAL;
    return launch_field_from_tables(tables8, k, total, defect, targets, max_excursion, stream);
}

int inim_flat_response(int k, float* defect, cudaStream_t stream) {
    if (!k_ok(k) || !defect) return INIM_EINVAL;
    return launch_flat_response(k, defect, stream);
}

int inim_sample(const float* targets, int k, const float* pts_in, float* pts_out, int64_t n, int clip,
                float* max_disp, cudaStream_t stream) {
    if (k < 1 || k > INIM_MAX_K || !targets || n < 0 || (n > 0 && (!pts_in || !pts_out))) return INIM_EINVAL;
    if (n == 0) return 0;
    return launch_sample_f32(targets, k, pts_in, pts_out, n, clip, max_disp, nullptr, stream);
}

int inim_sample_f64(const float* targets, int k, const double* pts_in, double* pts_out, int64_t n, int clip,
                    cudaStream_t stream) {
    if (k < 1 || k > INIM_MAX_K || !targets || n < 0 || (n > 0 && (!pts_in || !pts_out))) return INIM_EINVAL;
    if (n == 0) return 0;
    return launch_sample_f64(targets, k, pts_in, pts_out, n, clip, stream);
}

int inim_cast_f64_to_f32(const double* in, float* out, int64_t count, cudaStream_t stream) {
    if (count < 0 || (count > 0 && (!in || !out))) return INIM_EINVAL;
    if (count == 0) return 0;
    return launch_cast_f64_f32(in, out, count, stream);
}

int inim_h2d_narrow(const double* host, float* dev, int64_t count, cudaStream_t stream) {
    if (count < 0 || (count > 0 && (!host || !dev))) return INIM_EINVAL;
    if (count == 0) return 0;
    std::lock_guard<std::mutex> lock(g_stage.mu);
    int rc = staging_ready(g_stage);
    if (rc) return rc;
    const int nt = stage_threads(count);
    for (int64_t off = 0, c = 0; off < count; off += kStageChunk, ++c) {
        const int q = (int)(c & 1);
        const int64_t len = count - off < kStageChunk ? count - off : kStageChunk;
        INIM_CUDA_TRY(cudaEventSynchronize(g_stage.done[q]));  // the slot's previous DMA has finished
        float* dst = g_stage.slot[q];
        const double* src = host + off;
#pragma omp parallel for num_threads(nt) schedule(static)
        for (int64_t i = 0; i < len; ++i) dst[i] = (float)src[i];
        INIM_CUDA_TRY(cudaMemcpyAsync(dev + off, dst, len * sizeof(float), cudaMemcpyHostToDevice, stream));
        INIM_CUDA_TRY(cudaEventRecord(g_stage.done[q], stream));
    }
    return 0;
}

int inim_d2h_widen(const float* dev, double* host, int64_t count, cudaStream_t stream) {
    if (count < 0 || (count > 0 && (!host || !dev))) return INIM_EINVAL;
    if (count == 0) return 0;
    std::lock_guard<std::mutex> lock(g_stage.mu);
    int rc = staging_ready(g_stage);
    if (rc) return rc;
    const int nt = stage_threads(count);
    const int64_t nchunk = (count + kStageChunk - 1) / kStageChunk;
    auto issue = [&](int64_t c) -> int {  // DMA chunk c into its slot
        const int q = (int)(c & 1);
        const int64_t off = c * kStageChunk;
        const int64_t len = count - off < kStageChunk ? count - off : kStageChunk;
        INIM_CUDA_TRY(cudaMemcpyAsync(g_stage.slot[q], dev + off, len * sizeof(float), cudaMemcpyDeviceToHost,
                                      stream));
        INIM_CUDA_TRY(cudaEventRecord(g_stage.done[q], stream));
        return 0;
    };
    if ((rc = issue(0))) return rc;
    for (int64_t c = 0; c < nchunk; ++c) {
        const int q = (int)(c & 1);
        INIM_CUDA_TRY(cudaEventSynchronize(g_stage.done[q]));
        if (c + 1 < nchunk && (rc = issue(c + 1))) return rc;  // the other slot was widened last step
        const int64_t off = c * kStageChunk;
        const int64_t len = count - off < kStageChunk ? count - off : kStageChunk;
        const float* src = g_stage.slot[q];
        double* dst = host + off;
#pragma omp parallel for num_threads(nt) schedule(static)
        for (int64_t i = 0; i < len; ++i) dst[i] = (double)src[i];
    }
    return 0;
}

int inim_cast_f32_to_f64(const float* in, double* out, int64_t count, cudaStream_t stream) {
    if (count < 0 || (count > 0 && (!in || !out))) return INIM_EINVAL;
    if (count == 0) return 0;
    return launch_cast_f32_f64(in, out, count, stream);
}

int inim_iterate(const float* pts_in, float* pts_out, int64_t n, int k, int kernel_size, float background,
                 const float* defect, uint32_t* counts, float* d, float* targets, float* max_excursion,
                 float* disp_out, float stop_eps, int* state, void* ws, cudaStream_t stream) {
    if (k < 1 || k > INIM_MAX_K || n < 0 || !counts || !d || !targets || !max_excursion || !ws) return INIM_EINVAL;
    if (n > 0 && (!pts_in || !pts_out)) return INIM_EINVAL;
    if (kernel_size < 1) return INIM_EKERNEL;
    if (stop_eps > 0.f && !state) return INIM_EINVAL;
    const Geo g = make_geo(k);
    const FullLayout F = full_layout(g, n);
    const Ws w = make_ws(ws, F.L);
    float* scratch = reinterpret_cast<float*>(static_cast<char*>(ws) + F.scratch);
    CUtensorMap map;
    const CUtensorMap* mp = nullptr;
    if (g.TW >= 32) {
        int rc = make_tensor_map_2d(&map, d, g.s, g.TW, g.TH);
        if (rc) return rc;
        mp = &map;
    }
    INIM_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(uint32_t) * g.m, stream));
    return enqueue_iteration(pts_in, pts_out, n, g, kernel_size, auto_background(n, k, background), defect, counts,
                             nullptr, d, targets, max_excursion, disp_out ? disp_out : scratch, stop_eps, state, w, mp,
                             stream);
}

// Replay the cached executable graph of `key`, capturing it on first use.
static int run_graph(const RunKey& key, float* pts, float* frames, float* fields, float* disp, float* excursions,
                     int* state, void* ws, cudaStream_t stream) {
    {
        std::lock_guard<std::mutex> lock(g_mu);
        for (auto& e : g_cache)
            if (e.key == key) return (int)cudaGraphLaunch(e.exec, stream);
    }
    // First call with these arguments: capture once (on a private stream of the current
    // device: the legacy default stream cannot be captured), keep the executable graph,
    // launch it on the caller's stream.
    int dev = 0;
    INIM_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= kMaxDevices) return INIM_EINVAL;
    static cudaStream_t caps[kMaxDevices] = {};
    cudaStream_t& cap = caps[dev];
    if (!cap) INIM_CUDA_TRY(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    cudaGraph_t graph;
    INIM_CUDA_TRY(cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed));
    int rc = enqueue_run(key, pts, frames, fields, disp, excursions, state, ws, cap);
    cudaError_t ec = cudaStreamEndCapture(cap, &graph);
    if (rc) {
        if (ec == cudaSuccess) cudaGraphDestroy(graph);
        return rc;
    }
    INIM_CUDA_TRY(ec);
    cudaGraphExec_t exec;
    ec = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    INIM_CUDA_TRY(ec);
    {
        std::lock_guard<std::mutex> lock(g_mu);
        if (g_cache.size() >= 16) {
            cudaGraphExecDestroy(g_cache.front().exec);
            g_cache.erase(g_cache.begin());
        }
        g_cache.push_back({key, exec});
    }
    return (int)cudaGraphLaunch(exec, stream);
}

int inim_run(float* pts, int64_t n, int k, int kernel_size, float background, int iterations, float stop_eps,
             float* frames, float* fields, float* disp, float* excursions, int* state, void* ws, cudaStream_t stream) {
    if (k < 1 || k > INIM_MAX_K || n < 0 || iterations < 0 || !ws || (n > 0 && !pts)) return INIM_EINVAL;
    if (kernel_size < 1) return INIM_EKERNEL;
    if (stop_eps > 0.f && !state) return INIM_EINVAL;
    if (iterations == 0) return 0;
    RunKey key;
    memset(&key, 0, sizeof(key));
    key.pts = pts; key.n = n; key.k = k; key.ks = kernel_size; key.bg = auto_background(n, k, background);
    key.iters = iterations; key.eps = stop_eps; key.frames = frames; key.fields = fields; key.disp = disp;
    key.exc = excursions; key.state = state; key.ws = ws; key.st = stream;
    return run_graph(key, pts, frames, fields, disp, excursions, state, ws, stream);
}

int inim_run_metrics(float* pts, int64_t n, int k, int kernel_size, float background, int iterations, float stop_eps,
                     float* frames, float* fields, float* disp, float* excursions, int* state, void* ws,
                     cudaStream_t stream, unsigned long long* frame_stats, const double* orig_sub, const int64_t* pick,
                     int64_t n_sub, int n_neighbors, double* moved_sub, unsigned long long* nb_stats) {
    if (k < 1 || k > INIM_MAX_K || n < 0 || iterations < 0 || !ws || (n > 0 && !pts) || !frame_stats) return INIM_EINVAL;
    if (kernel_size < 1) return INIM_EKERNEL;
    if (stop_eps > 0.f && !state) return INIM_EINVAL;
    if (orig_sub && (!moved_sub || !nb_stats || n_sub < 2 || n_sub > n || n_neighbors < 1 || n_neighbors >= n_sub))
        return INIM_EINVAL;
    if (iterations == 0) return 0;
    RunKey key;
    memset(&key, 0, sizeof(key));
    key.pts = pts; key.n = n; key.k = k; key.ks = kernel_size; key.bg = auto_background(n, k, background);
    key.iters = iterations; key.eps = stop_eps; key.frames = frames; key.fields = fields; key.disp = disp;
    key.exc = excursions; key.state = state; key.ws = ws; key.st = stream;
    key.fstats = frame_stats;
    if (orig_sub) {
        key.orig_sub = orig_sub; key.pick = pick; key.n_sub = n_sub; key.n_neighbors = n_neighbors;
        key.moved_sub = moved_sub; key.nbstats = nb_stats;
    }
    return run_graph(key, pts, frames, fields, disp, excursions, state, ws, stream);
}

int inim_run_batched(float* pts, int64_t n, int B, int k, int kernel_size, float background, int iterations,
                     float stop_eps, int* states, unsigned long long* frame_stats, void* ws, cudaStream_t stream) {
    if (k < 1 || k > INIM_MAX_K || n < 0 || B < 1 || iterations < 0 || !ws || (n > 0 && !pts)) return INIM_EINVAL;
    if (kernel_size < 1) return INIM_EKERNEL;
    if (stop_eps > 0.f && !states) return INIM_EINVAL;
    if (iterations == 0) return 0;
    if (B > 1 && (n & 1)) return INIM_EINVAL;  // every plot's points 16-byte aligned (two points per access)
    RunKey key;
    memset(&key, 0, sizeof(key));
    key.pts = pts; key.n = n; key.k = k; key.ks = kernel_size; key.bg = auto_background(n, k, background);
    key.iters = iterations; key.ws = ws; key.st = stream; key.B = B;
    key.eps = stop_eps; key.state = stop_eps > 0.f ? states : nullptr;
    key.fstats = frame_stats;
    return run_graph(key, pts, nullptr, nullptr, nullptr, nullptr, key.eps > 0.f ? states : nullptr, ws, stream);
}

int inim_frame_stats(const uint32_t* counts, int k, unsigned long long* out3, cudaStream_t stream) {
    if (!k_ok(k) || !counts || !out3) return INIM_EINVAL;
    return launch_frame_stats(counts, k, out3, stream);
}

int inim_gather_points(const void* pts, int pts_is_f64, const int64_t* rows, const uint32_t* perm, int64_t m,
                       double* out, cudaStream_t stream) {
    if (m < 0 || (m > 0 && (!pts || !out))) return INIM_EINVAL;
    if (m == 0) return 0;
    return launch_gather_points(pts, pts_is_f64, rows, perm, m, out, stream);
}

int inim_trust_penalty(const double* orig, const double* moved, int64_t n, int n_neighbors, unsigned long long* out,
                       cudaStream_t stream) {
    if (n < 0 || !out || n_neighbors < 1 || (n > 0 && (!orig || !moved)) || n_neighbors >= n) return INIM_EINVAL;
    if ((size_t)n_neighbors * 16 > 200 * 1024) return INIM_EINVAL;
    return launch_trust(orig, moved, n, n_neighbors, out, stream);
}

int inim_order_pairs(const double* orig, const double* moved, int64_t n, unsigned long long* out,
                     cudaStream_t stream) {
    if (n < 0 || !out || (n > 0 && (!orig || !moved))) return INIM_EINVAL;
    if (n < 2) return 0;
    return launch_order_pairs(orig, moved, n, out, stream);
}

int inim_run_uncached(float* pts, int64_t n, int k, int kernel_size, float background, int iterations,
                      float stop_eps, float* frames, float* fields, float* disp, float* excursions, int* state,
                      void* ws, cudaStream_t stream) {
    // Same work as inim_run launched eagerly (no graph): used for per-kernel timing.
    if (k < 1 || k > INIM_MAX_K || n < 0 || iterations < 0 || !ws || (n > 0 && !pts)) return INIM_EINVAL;
    if (kernel_size < 1) return INIM_EKERNEL;
    RunKey key;
    memset(&key, 0, sizeof(key));
    key.pts = pts; key.n = n; key.k = k; key.ks = kernel_size; key.bg = auto_background(n, k, background);
    key.iters = iterations; key.eps = stop_eps;
    return enqueue_run(key, pts, frames, fields, disp, excursions, state, ws, stream);
}

int inim_profile_run(float* pts, int64_t n, int k, int kernel_size, float background, int iterations, void* ws,
                     cudaStream_t stream, float* ms_out, int cap, char* names_out, int names_len) {
    if (k < 1 || k > INIM_MAX_K || n < 0 || iterations < 1 || !ws || !ms_out || cap < 1 || (n > 0 && !pts))
        return INIM_EINVAL;
    std::vector<cudaEvent_t> ev(cap + 1);
    std::vector<const char*> names(cap + 1, "");
    for (auto& e : ev) INIM_CUDA_TRY(cudaEventCreate(&e));
    Prof p{ev.data(), names.data(), 0, cap + 1};
    INIM_CUDA_TRY(cudaEventRecord(ev[0], stream));
    p.names[0] = "start";
    p.n = 1;
    RunKey key;
    memset(&key, 0, sizeof(key));
    key.pts = pts; key.n = n; key.k = k; key.ks = kernel_size; key.bg = auto_background(n, k, background);
    key.iters = iterations;
    g_prof = &p;
    int rc = enqueue_run(key, pts, nullptr, nullptr, nullptr, nullptr, nullptr, ws, stream);
    g_prof = nullptr;
    if (rc) return rc;
    INIM_CUDA_TRY(cudaStreamSynchronize(stream));
    int count = p.n - 1;
    std::string joined;
    for (int q = 0; q < count; ++q) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev[q], ev[q + 1]);
        ms_out[q] = ms;
        joined += names[q + 1];
        joined += "\n";
    }
    if (names_out && names_len > 0) {
        strncpy(names_out, joined.c_str(), names_len - 1);
        names_out[names_len - 1] = 0;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    return count;
}

void inim_clear_graph_cache(void) {
    std::lock_guard<std::mutex> lock(g_mu);
    for (auto& e : g_cache) cudaGraphExecDestroy(e.exec);
    g_cache.clear();
}

int inim_run_host(const double* pts_host, double* out_host, int64_t n, int k, int kernel_size, double background,
                  int iterations) {
    if (k < 1 || k > INIM_MAX_K || n < 0 || iterations < 0 || (n > 0 && (!pts_host || !out_host))) return INIM_EINVAL;
    if (kernel_size < 1) return INIM_EKERNEL;
    // Grow-only device buffers owned by this entry point (the documented exception to
    // "the library never allocates").
    static std::mutex mu;
    static void* ws = nullptr;
    static size_t ws_bytes = 0;
    static double* pd = nullptr;
    static float* pf = nullptr;
    static int64_t cap = 0;
    static cudaStream_t st = nullptr;
    std::lock_guard<std::mutex> lock(mu);
    if (!st) INIM_CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    const size_t need = inim_workspace_bytes(k, n, 1);
    if (need > ws_bytes) {
        if (ws) cudaFree(ws);
        INIM_CUDA_TRY(cudaMalloc(&ws, need));
        ws_bytes = need;
        inim_clear_graph_cache();
    }
    if (n > cap) {
        if (pd) cudaFree(pd);
        if (pf) cudaFree(pf);
        INIM_CUDA_TRY(cudaMalloc(&pd, sizeof(double) * 2 * n));
        INIM_CUDA_TRY(cudaMalloc(&pf, sizeof(float) * 2 * n));
        cap = n;
        inim_clear_graph_cache();
    }
    if (n > 0) {  // narrowed on the host while the DMA runs (page-locked float32 slots)
        int rc = inim_h2d_narrow(pts_host, pf, 2 * n, st);
        if (rc) return rc;
    }
    int rc = inim_run(pf, n, k, kernel_size, (float)background, iterations, 0.f, nullptr, nullptr, nullptr, nullptr,
                      nullptr, ws, st);
    if (rc) return rc;
    if (n > 0) {
        rc = inim_d2h_widen(pf, out_host, 2 * n, st);
        if (rc) return rc;
    }
    INIM_CUDA_TRY(cudaStreamSynchronize(st));
    return 0;
}

int inim_kernels_per_iteration(int k) {
    // smooth_h, smooth_v(+reduce), lines, chains, write_field, move (+ iter_end when the
    // displacement criterion is on).  The move of iteration t splats iteration t+1, so a
    // run adds one splat kernel (plus the point sort and unpermute) and a memset node.
    (void)k;
    return 6;
}

}  // extern "C"
