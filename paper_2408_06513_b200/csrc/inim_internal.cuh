// Tile geometry and workspace layout of the integral-image pipeline.
//
// The texture (s x s, s = 2^k) is cut into bands of TH rows; each band into tiles of
// TW = 32 * CPL columns.  One warp owns one tile; lane l owns columns CPL*l .. CPL*l +
// CPL - 1 and sweeps the TH rows.  TH <= 32 (lane-distributed row constants) and
// TW >= TH (a chain ending in a tile's last column stays inside that tile).  See DESIGN.md "Integral pass" for the derivation of every carry.
#pragma once

#include <stdlib.h>

#include <mutex>
#include <set>
#include <type_traits>
#include <utility>

#include "inim_common.cuh"

namespace inim {

constexpr int kMaxDevices = 64;

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: raise a kernel's
// limit once for every device it is launched on.
inline cudaError_t ensure_smem_limit(const void* kernel, int bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    if (done.count({kernel, dev})) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.insert({kernel, dev});
    return e;
}

struct Geo {
    int k, s, TH, TW, B, NX, NW, WL, CPL;  // WL = lanes holding columns; CPL = columns per lane
    int twlog;                             // log2(TW)
    int64_t m;
};

// Bands of 16 rows up to 2048^2 (more CTAs for latency-bound small grids), 32 rows
// above (fewer carry vectors per pixel for bandwidth-bound large grids).  `wide`: the
// large-grid geometry from 128^2 up, for plot batches (thousands of tiles in flight
// anyway: the per-tile prologue is amortised over 4x the pixels).
inline Geo make_geo(int k, bool wide = false) {
    Geo g;
    g.k = k;
    g.s = 1 << k;
    g.m = (int64_t)g.s * g.s;
    const bool large = g.s > 2048 || (wide && g.s >= 128);
    g.TH = g.s < 16 ? g.s : (large ? 32 : 16);
    // one warp per tile: 64 columns (2 per lane) up to 2048^2 for more warps on small
    // grids, 128 columns (4 per lane, 16-byte accesses) above
    g.TW = large ? 128 : (g.s < 64 ? g.s : 64);
    g.CPL = g.TW >= 128 ? 4 : (g.TW >= 64 ? 2 : 1);
    g.B = g.s / g.TH;
    g.NX = g.s / g.TW;
    g.NW = 1;
    g.WL = g.TW >= 32 ? 32 : g.TW;
    g.twlog = 0;
    while ((1 << g.twlog) < g.TW) ++g.twlog;
    return g;
}

// Byte offsets into the caller-provided workspace (all 256-byte aligned).
struct WsLayout {
    size_t tmp;      // float [s*s]            horizontal smoothing pass
    size_t inpre;    // float [B][s]           in-tile inclusive row prefix of the band's column sums
    size_t tiletot;  // double [B][NX]         tile totals
    size_t rowsum;   // float [s][NX]          per-tile row sums
    size_t ulbot;    // float [B][s]           in-tile up-left chain of V at the band's last row
    size_t urbot;    // float [B][s]           in-tile up-right chain of V at the band's last row
    size_t ule;      // float [B][NX][TH]      up-left chain at each tile's last column
    size_t ure;      // float [B][NX][TH]      up-right chain at each tile's first column
    size_t tilepre;  // double [B][NX]         exclusive prefix over tiles of the tile totals
    size_t btot;     // double [B]             band totals
    size_t bandpre;  // double [B+1]           exclusive prefix of the band totals (TLcar_b[s-1])
    size_t tlcar;    // float [B+1][s]         rect_tl at the row above each band (row s-1 for b=B)
    size_t x1;       // float [B+1][s]         ULcar - TLcar (row B: along the last row)
    size_t x2;       // float [B+1][s+TH]      URcar + TLcar[c-1], extended with TLcar[s-1]
    size_t hc;       // double [s][NX]         row prefix of d up to each tile's first column
    size_t rpre;     // double [s]             in-band inclusive prefix of the row totals
    size_t taps;     // float [2s]             runtime taps of the generic smoothing (kernel_size > 16)
    size_t total;    // double [1]
    size_t misc;     // float [16]             scratch scalars
    size_t bytes;
};

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

inline WsLayout make_layout(const Geo& g) {
    WsLayout L;
    size_t o = 0;
    auto take = [&](size_t bytes) {
        size_t r = o;
        o = align256(o + bytes);
        return r;
    };
    const size_t s = g.s, B = g.B, NX = g.NX, TH = g.TH;
    L.tmp = take(sizeof(float) * s * s);
    L.inpre = take(sizeof(float) * B * s);
    L.tiletot = take(sizeof(double) * B * NX);
    L.rowsum = take(sizeof(float) * s * NX);
    L.ulbot = take(sizeof(float) * B * s);
    L.urbot = take(sizeof(float) * B * s);
    L.ule = take(sizeof(float) * B * NX * TH);
    L.ure = take(sizeof(float) * B * NX * TH);
    L.tilepre = take(sizeof(double) * B * NX);
    L.btot = take(sizeof(double) * B);
    L.bandpre = take(sizeof(double) * (B + 1));
    L.tlcar = take(sizeof(float) * (B + 1) * s);
    L.x1 = take(sizeof(float) * (B + 1) * s);
    L.x2 = take(sizeof(float) * (B + 1) * (s + TH));
    L.hc = take(sizeof(double) * s * NX);
    L.rpre = take(sizeof(double) * s);
    L.taps = take(sizeof(float) * 2 * s);
    L.total = take(sizeof(double));
    L.misc = take(sizeof(float) * 16);
    L.bytes = o;
    return L;
}

// Typed view of the workspace, passed by value to kernels.
struct Ws {
    float* tmp;
    float* inpre;
    double* tiletot;
    float* rowsum;
    float* ulbot;
    float* urbot;
    float* ule;
    float* ure;
    double* tilepre;
    double* btot;
    double* bandpre;
    float* tlcar;  // carries: float64 scans, stored float32 (the write pass computes in float32)
    float* x1;
    float* x2;
    double* hc;
    double* rpre;
    float* taps;
    double* total;
    float* misc;
};

inline Ws make_ws(void* base, const WsLayout& L) {
    char* b = static_cast<char*>(base);
    Ws w;
    w.tmp = reinterpret_cast<float*>(b + L.tmp);
    w.inpre = reinterpret_cast<float*>(b + L.inpre);
    w.tiletot = reinterpret_cast<double*>(b + L.tiletot);
    w.rowsum = reinterpret_cast<float*>(b + L.rowsum);
    w.ulbot = reinterpret_cast<float*>(b + L.ulbot);
    w.urbot = reinterpret_cast<float*>(b + L.urbot);
    w.ule = reinterpret_cast<float*>(b + L.ule);
    w.ure = reinterpret_cast<float*>(b + L.ure);
    w.tilepre = reinterpret_cast<double*>(b + L.tilepre);
    w.btot = reinterpret_cast<double*>(b + L.btot);
    w.bandpre = reinterpret_cast<double*>(b + L.bandpre);
    w.tlcar = reinterpret_cast<float*>(b + L.tlcar);
    w.x1 = reinterpret_cast<float*>(b + L.x1);
    w.x2 = reinterpret_cast<float*>(b + L.x2);
    w.hc = reinterpret_cast<double*>(b + L.hc);
    w.rpre = reinterpret_cast<double*>(b + L.rpre);
    w.taps = reinterpret_cast<float*>(b + L.taps);
    w.total = reinterpret_cast<double*>(b + L.total);
    w.misc = reinterpret_cast<float*>(b + L.misc);
    return w;
}

// ---------------------------------------------------------------- plot batches
// A batch of B independent plots (a SPLOM) runs every stage as ONE launch with the plot
// index in blockIdx.z.  Each plot owns a slab of the workspace (inim_workspace_bytes(k,
// n, 1) bytes, 256-aligned); plot z's workspace pointers are plot 0's plus z * slab
// bytes, and its points are the caller's (B, n, 2) array at z * 2n floats.  B = 1 with
// slab = 0 is the single-plot path (every offset is zero).
struct Bat {
    int B = 1;
    int64_t slab = 0;  // bytes between consecutive plots' workspace slabs
    int64_t pts = 0;   // floats between consecutive plots' caller point arrays
};

template <typename T>
__host__ __device__ __forceinline__ T* zoff(T* p, int64_t bytes) {
    return reinterpret_cast<T*>(reinterpret_cast<char*>(const_cast<typename std::remove_const<T>::type*>(p)) + bytes);
}
template <typename T>
__host__ __device__ __forceinline__ T* zoff_opt(T* p, int64_t bytes) {  // null stays null
    return p ? zoff(p, bytes) : p;
}

__host__ __device__ __forceinline__ Ws ws_shift(Ws w, int64_t b) {
    if (b == 0) return w;
    w.tmp = zoff(w.tmp, b);
    w.inpre = zoff(w.inpre, b);
    w.tiletot = zoff(w.tiletot, b);
    w.rowsum = zoff(w.rowsum, b);
    w.ulbot = zoff(w.ulbot, b);
    w.urbot = zoff(w.urbot, b);
    w.ule = zoff(w.ule, b);
    w.ure = zoff(w.ure, b);
    w.tilepre = zoff(w.tilepre, b);
    w.btot = zoff(w.btot, b);
    w.bandpre = zoff(w.bandpre, b);
    w.tlcar = zoff(w.tlcar, b);
    w.x1 = zoff(w.x1, b);
    w.x2 = zoff(w.x2, b);
    w.hc = zoff(w.hc, b);
    w.rpre = zoff(w.rpre, b);
    w.taps = zoff(w.taps, b);
    w.total = zoff(w.total, b);
    w.misc = zoff(w.misc, b);
    return w;
}

// byte offset of this CTA's plot
INIM_DEV int64_t zslab_off(int64_t slab) { return (int64_t)blockIdx.z * slab; }

// The run tile geometries as compile-time constants of a local Geo (GEO 1: 32 x 128
// tiles, 2: 16 x 64 tiles, 0: as passed), so the index arithmetic of the scans folds.
template <int GEO>
__device__ __forceinline__ Geo fixed_geo(const Geo& g) {
    Geo f = g;
    if (GEO == 1) { f.TH = 32; f.TW = 128; f.twlog = 7; f.CPL = 4; f.WL = 32; }
    if (GEO == 2) { f.TH = 16; f.TW = 64; f.twlog = 6; f.CPL = 2; f.WL = 32; }
    return f;
}

inline int geo_kind(const Geo& g) {
    if (g.WL != 32) return 0;
    if (g.TH == 32 && g.TW == 128) return 1;
    if (g.TH == 16 && g.TW == 64) return 2;
    return 0;
}

// INIM_ZREV=0: every batched kernel walks the plots in launch order.  Otherwise the
// vertical pass and the move walk them backwards, so each consumer starts on the plots
// its producer wrote last (still in L2): h up, v down, write up, move down.
inline bool zrev_enabled() {
    static const bool on = [] {
        const char* e = getenv("INIM_ZREV");
        return !(e && e[0] == '0');
    }();
    return on;
}

// the run's device state word pair {stopped, iterations done} of this CTA's plot: one
// per plot, inside its workspace slab, in a batch
INIM_DEV const int* zstate(const int* state, int64_t slab) { return state ? zoff(state, zslab_off(slab)) : state; }

// ---------------------------------------------------------------- launch profiler
// When g_prof is set (inim_profile_run only), every launcher records a CUDA event
// after its launch; consecutive events bracket exactly one launch.
struct Prof {
    cudaEvent_t* ev;
    const char** names;
    int n, cap;
};
extern Prof* g_prof;

inline void prof_mark(cudaStream_t st, const char* name) {
    if (g_prof && g_prof->n < g_prof->cap) {
        g_prof->names[g_prof->n] = name;
        cudaEventRecord(g_prof->ev[g_prof->n++], st);
    }
}

// ---------------------------------------------------------------- host-side launchers
int launch_reduce_from_global(const float* d, const Geo& g, const Ws& ws, const CUtensorMap* map,
                              cudaStream_t st, const Bat& bt = Bat{});
int launch_carry_scan_state(const Geo& g, const Ws& ws, const int* state, cudaStream_t st, const Bat& bt = Bat{});
int launch_write_tables(const float* d, const Geo& g, const Ws& ws, const CUtensorMap* map, float* tables8,
                        cudaStream_t st);
// targets: standard (s, s, 2) field or null; pairs: paired (s, s, 4) layout for the
// move kernel or null.
int launch_write_field(const float* d, const Geo& g, const Ws& ws, const CUtensorMap* map, const float* defect,
                       float* targets, float* max_exc, const int* state, cudaStream_t st, float* pairs = nullptr,
                       const Bat& bt = Bat{});
int make_tensor_map_2d(CUtensorMap* map, const float* base, int s, int box_w, int box_h);

}  // namespace inim
