/*
 * inim.h -- C ABI of libinim.so, the sm_100a integral-image scatterplot regularizer
 * (arXiv 2408.06513).  Drop-in compute layer under the reference package's Python API
 * (uncrowd: density.py / integral.py / mapping.py / regularize.py).
 *
 * The reference has no FFI of its own: its hot path is Python calling numpy/scipy/numba
 * (SURVEY.md section 8(b)).  Each entry point below names the reference function it
 * replaces; the Python mirror (paper_2408_06513_b200/*.py) and a ctypes binding that a
 * maintainer would add to uncrowd call these symbols.
 *
 * Conventions
 *  - All buffers are DEVICE pointers allocated by the caller (PyTorch in the mirror).
 *    The library never allocates device memory, never synchronises the device, and is
 *    stream-ordered: every call enqueues work on `stream` and returns.  The one
 *    exception is inim_run_host(), the host-buffer convenience used for end-to-end
 *    measurement, which copies in, runs, copies out and synchronises.
 *  - Grids are 2^k x 2^k row-major (values[j*s + i], i = x column, j = y row; reference
 *    model.py:1-8).  Fields are (s, s, 2) float32, x then y.  Points are (n, 2)
 *    interleaved [x, y] float32 (or float64 where stated).
 *  - The eight tables are one float32 buffer of 8*s*s in the reference order
 *    rect_tl, rect_bl, rect_br, rect_tr, wedge_up, wedge_left, wedge_down, wedge_right
 *    (model.py:81-85).
 *  - Return value: 0 = success; > 0 = a cudaError_t; < 0 = an INIM_E* argument error.
 *    The Python mirror validates arguments first and raises the reference's exceptions.
 */
#ifndef INIM_H_
#define INIM_H_

#include <stddef.h>
#include <stdint.h>

#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

#define INIM_OK 0
#define INIM_EINVAL (-1)      /* bad argument (k out of range, n < 0, null pointer) */
#define INIM_ENOTPOW2 (-2)    /* texture not square power-of-two (integral.py:183-184) */
#define INIM_EKERNEL (-3)     /* kernel_size < 1 (density.py:46-47) */
#define INIM_EDRIVER (-4)     /* could not resolve cuTensorMapEncodeTiled */

#define INIM_MAX_K 15 /* 32768^2 = 2^30 pixels (int32 pixel indices); eight fp32 tables = 32 GiB */

/* Library identification: returns a static string, e.g. "libinim sm_100a 0.1". */
const char* inim_version(void);

/* Bytes of device workspace needed by the calls below for a 2^k grid and n points
 * (integral aggregates and carries, the smoothing scratch, and for inim_run the
 * counts / density / field buffers plus a point ping-pong buffer of n*2 floats), for
 * B plots (inim_run_batched: B slabs of the single-plot size; B <= 1 means one).
 * `ws` arguments must be at least this large and 256-byte aligned.  0 if k is out of
 * range. */
size_t inim_workspace_bytes(int k, int64_t n, int B);

/* accumulate (density.py:14-27) + pixel_of (model.py:189-198): counts[j*s+i] += number
 * of points in pixel (i, j).  Integer atomics: bit-exact for identical coordinates.
 * pts_is_f64 != 0 bins float64 coordinates (the reference's dtype); else float32.
 * Counts are NOT cleared first. */
int inim_splat(const void* pts, int pts_is_f64, int64_t n, int k, uint32_t* counts, cudaStream_t stream);

/* gaussian_smooth + background (density.py:40-51, 54-78) on integer counts:
 * d = convolve1d(convolve1d(counts, w, axis=1), w, axis=0) + background, reflect mode,
 * w = smoothing_kernel(kernel_size).  Also emits, into ws, the per-tile aggregates the
 * integral pass needs (so the fused iteration reads d only once). */
int inim_smooth_counts(const uint32_t* counts, int k, int kernel_size, float background, float* d, void* ws,
                       cudaStream_t stream);

/* gaussian_smooth (density.py:40-51) of an arbitrary float32 grid (no background). */
int inim_smooth_grid(const float* grid, int k, int kernel_size, float* out, void* ws, cudaStream_t stream);

/* build_integral_set (integral.py:231-247): the eight tables of d, plus the total mass
 * (float64, device).  Reduce pass (tile aggregates + marginals) -> carry scan -> one
 * write pass. */
int inim_integral_set(const float* d, int k, float* tables8, double* total, void* ws, cudaStream_t stream);

/* The staged intermediates the reference also exports (integral.py:180-228), each
 * float32 s*s on device: column_integrals -> upper, lower. */
int inim_column_integrals(const float* d, int k, float* upper, float* lower, cudaStream_t stream);

/* Generic float64-accumulated line scan of an s*s float32 grid along direction
 * (dj, di) in {-1,0,1}^2: out = running sum along the line, inclusive or exclusive.
 * Serves classical_rects / triangle_integrals (integral.py:189-209): e.g. rect_tl =
 * row prefix of upper (0,+1), rect_tr = exclusive scan of upper along (0,-1),
 * up_left = inclusive scan of upper along (+1,+1). */
int inim_line_scan(const float* in, float* out, int k, int dj, int di, int exclusive, cudaStream_t stream);

/* build_field (mapping.py:194-204) from a density texture d, fused with the integral
 * pass (tables never leave registers): targets (s,s,2) float32, clipped to [0,1];
 * *max_excursion (device float, must be zeroed by the caller) receives the pre-clip
 * overshoot.  defect = flat response (s,s,2) float32, or NULL for the closed form. */
int inim_field_from_density(const float* d, int k, const float* defect, float* targets, float* max_excursion,
                            double* total, void* ws, cudaStream_t stream);

/* build_field (mapping.py:194-204) from eight precomputed float32 tables and a total. */
int inim_field_from_tables(const float* tables8, int k, const double* total, const float* defect, float* targets,
                           float* max_excursion, cudaStream_t stream);

/* flat_response.get(k) (mapping.py:104-129): raw map of a constant texture, evaluated
 * from the closed-form region pixel counts (integers, exact) in float64, stored fp32. */
int inim_flat_response(int k, float* defect, cudaStream_t stream);

/* sample_field (mapping.py:207-246) [+ clip to [0,1] as regularize.py:36 when clip]:
 * bilinear blend of the four pixel targets around each point; one-sided last cell.
 * If max_disp != NULL it receives max |out - in| (device float, zeroed by caller). */
int inim_sample(const float* targets, int k, const float* pts_in, float* pts_out, int64_t n, int clip,
                float* max_disp, cudaStream_t stream);

/* Same on float64 points (the interpolate()/sample_field() API with fp64 inputs). */
int inim_sample_f64(const float* targets, int k, const double* pts_in, double* pts_out, int64_t n, int clip,
                    cudaStream_t stream);

/* sample_field (mapping.py:207-246) of float64 targets at float64 points (a field the
 * caller built in float64, e.g. DeformationField(targets=ndarray)). */
int inim_sample_t64(const double* targets, int k, const double* pts_in, double* pts_out, int64_t n, int clip,
                    cudaStream_t stream);

/* anchors / raw_map / corrected_map (mapping.py:40-143) at n float64 query points:
 * mode 0 -> out[8n] anchors (down_right, up_right, up_left, down_left; x,y each);
 * mode 1 -> out[2n] raw map from float32 tables8 at the containing pixel;
 * mode 2 -> out[2n] corrected map clip((x,y) + raw - defect[j,i]) with a float64 defect. */
int inim_map_points(const float* tables8, int k, const double* total, const double* defect, const double* xs,
                    const double* ys, int64_t n, int mode, double* out, cudaStream_t stream);

/* tilted_wedges (integral.py:212-228): out4 = (up, left, down, right) from the four
 * triangle tables and the column integrals; scratch2s: 2*s doubles of device scratch. */
int inim_tilted_wedges(const float* ul, const float* ur, const float* dl, const float* dr, const float* upper,
                       const float* lower, int k, double* scratch2s, float* out4, cudaStream_t stream);

/* flat_response.get(k) in float64 (same closed form, float64 output). */
int inim_flat_response_f64(int k, double* defect, cudaStream_t stream);

/* Element-wise helpers used by the mirror (fp64 <-> fp32 casts, in-place). */
int inim_cast_f64_to_f32(const double* in, float* out, int64_t count, cudaStream_t stream);
int inim_cast_f32_to_f64(const float* in, double* out, int64_t count, cudaStream_t stream);

/* Host float64 <-> device float32 transfers for pageable host buffers (the mirror's
 * to_device / to_host of the reference's float64 position arrays): the host narrows or
 * widens 1 MiB chunks with its cores while the DMA engine moves the previous one through
 * two page-locked slots.  h2d returns once the last chunk is queued on `stream` (the host
 * buffer may be reused immediately); d2h returns with `host` complete.  Same IEEE
 * round-to-nearest conversion as inim_cast_*. */
int inim_h2d_narrow(const double* host, float* dev, int64_t count, cudaStream_t stream);
int inim_d2h_widen(const float* dev, double* host, int64_t count, cudaStream_t stream);

/* One iteration of regularize.iterate_once (regularize.py:25-37), device resident:
 * counts <- 0; splat(pts_in); smooth (+background); integral+field; sample+clip into
 * pts_out.  counts: s*s uint32; d: s*s float; targets: s*s*2 float.  background <= 0
 * means auto (n / 4^k, 1.0 if n == 0).  defect may be NULL (closed form).
 * stop_eps > 0 enables the displacement criterion: `state` (device int[4], zeroed
 * before the first iteration) holds {stopped, iterations_done, 0, 0}; once an
 * iteration's max |delta| < stop_eps, later calls are no-ops on the device.
 * disp_out (device float, may be NULL) receives this iteration's max |delta|. */
int inim_iterate(const float* pts_in, float* pts_out, int64_t n, int k, int kernel_size, float background,
                 const float* defect, uint32_t* counts, float* d, float* targets, float* max_excursion,
                 float* disp_out, float stop_eps, int* state, void* ws, cudaStream_t stream);

/* Device-resident run (regularize.run, regularize.py:40-80, numeric path only):
 * `iterations` iterations of inim_iterate captured once into a CUDA graph and
 * replayed.  frames: optional device buffer of (iterations+1) * n * 2 floats receiving
 * every frame (frame 0 = pts); fields: optional (iterations) * s*s*2 floats.
 * pts is updated in place to the final positions.  disp: optional device float
 * [iterations] of per-iteration max displacement.  excursions: optional device float
 * [iterations].  stop_eps as in inim_iterate. */
int inim_run(float* pts, int64_t n, int k, int kernel_size, float background, int iterations, float stop_eps,
             float* frames, float* fields, float* disp, float* excursions, int* state, void* ws,
             cudaStream_t stream);

/* inim_run without graph capture (every kernel launched eagerly on `stream`); used to
 * time individual kernels with events. */
int inim_run_uncached(float* pts, int64_t n, int k, int kernel_size, float background, int iterations,
                      float stop_eps, float* frames, float* fields, float* disp, float* excursions, int* state,
                      void* ws, cudaStream_t stream);

/* Profiling: `iterations` iterations launched eagerly with a CUDA event recorded after
 * every launch; synchronises.  ms_out[q] = duration of launch q, names_out = the
 * launch names joined by '\n'.  Returns the number of launches (>= 0) or an error. */
int inim_profile_run(float* pts, int64_t n, int k, int kernel_size, float background, int iterations, void* ws,
                     cudaStream_t stream, float* ms_out, int cap, char* names_out, int names_len);

/* Drop every cached executable graph of inim_run (call before freeing buffers that a
 * cached graph references). */
void inim_clear_graph_cache(void);

/* inim_run with per-frame layout metrics (regularize.py:55-59,71-75 -> metrics.py:147-168).
 * frame_stats: device u64[iterations][3] (cleared by the call) receives, for frame t+1
 *   (the positions after iteration t): {occupied pixels, sum over 4x4-pixel bins of
 *   count^2, sum of counts}, from which binned_stddev (metrics.py:46-59) and
 *   overplotting (metrics.py:62-71) follow exactly.
 * orig_sub (optional, "full" mode): device (n_sub, 2) float64 = frame 0 at the rows
 *   `pick` (device int64[n_sub], NULL = the first n_sub rows, i.e. all of them);
 *   moved_sub: device scratch (n_sub, 2) float64; nb_stats: device u64[iterations][2]
 *   (cleared by the call) = {trustworthiness penalty sum, preserved pair count} of frame
 *   t+1 against frame 0 (metrics.py:74-144), 1 <= n_neighbors < n_sub. */
int inim_run_metrics(float* pts, int64_t n, int k, int kernel_size, float background, int iterations, float stop_eps,
                     float* frames, float* fields, float* disp, float* excursions, int* state, void* ws,
                     cudaStream_t stream, unsigned long long* frame_stats, const double* orig_sub, const int64_t* pick,
                     int64_t n_sub, int n_neighbors, double* moved_sub, unsigned long long* nb_stats);

/* A batch of B independent plots of n points each (a scatterplot matrix; the reference
 * runs regularize.run per plot in a process pool, tests/test_acceptance.py:107-128):
 * `iterations` fixed iterations of every plot, every stage ONE launch over all plots
 * (plot index in grid.z), captured once into a CUDA graph and replayed.
 * pts: device (B, n, 2) float32, updated in place to each plot's final positions (n
 * even when B > 1); ws: inim_workspace_bytes(k, n, B) bytes.  stop_eps > 0 runs the
 * displacement criterion per plot (regularize.py:76-79): a plot stops after the
 * iteration whose max |delta| < stop_eps, the others go on; states (device int[B][4],
 * required then) receives each plot's {stopped, iterations done, 0, 0}.  frame_stats: NULL, or
 * device u64[B][iterations][3] (cleared by the call) receiving the per-frame occupancy
 * statistics of every plot (as inim_run_metrics; collect_metrics="basic").  Batches
 * (any B, one plot included) use the wide tile geometry (32 x 128 tiles from 128^2 up;
 * inim_run uses 16 x 64 up to 2048^2), so each plot matches inim_run on that plot alone
 * within float32 rounding (the tile sums associate differently), and a plot's result
 * does not depend on B or on its position in the batch (bit-identical). */
int inim_run_batched(float* pts, int64_t n, int B, int k, int kernel_size, float background, int iterations,
                     float stop_eps, int* states, unsigned long long* frame_stats, void* ws, cudaStream_t stream);

/* Occupancy statistics of a count grid (binned_stddev metrics.py:46-59, overplotting
 * metrics.py:62-71): out3 (device u64[3], NOT cleared) += {occupied pixels, sum over the
 * 4x4-pixel bins of count^2 (k >= 2; 0 otherwise), sum of counts}. */
int inim_frame_stats(const uint32_t* counts, int k, unsigned long long* out3, cudaStream_t stream);

/* out[q] = float64(pts[perm[rows[q]]]) for q < m (rows / perm NULL = identity):
 * gathers the fixed-seed subsample of metrics.py:139-141, 164-166. */
int inim_gather_points(const void* pts, int pts_is_f64, const int64_t* rows, const uint32_t* perm, int64_t m,
                       double* out, cudaStream_t stream);

/* trustworthiness (metrics.py:74-113) numerator: *out (device u64, NOT cleared) += sum
 * over samples i and their n_neighbors nearest others j in `moved` (ties -> lower
 * index) of max(0, rank_orig(i, j) - n_neighbors).  1 <= n_neighbors < n. */
int inim_trust_penalty(const double* orig, const double* moved, int64_t n, int n_neighbors, unsigned long long* out,
                       cudaStream_t stream);

/* orthogonal_ordering (metrics.py:116-144) numerator: *out (device u64, NOT cleared) +=
 * number of pairs i < j whose x-order and y-order signs agree between the layouts. */
int inim_order_pairs(const double* orig, const double* moved, int64_t n, unsigned long long* out,
                     cudaStream_t stream);

/* transition_positions (regularize.py:83-93) as the service's float32 payload
 * (service.py:170-172): out[q] = f32((1 - frac) * lo[q] + frac * hi[q]) computed in
 * float64 (out = f32(lo) when `same`, i.e. an integer level).  lo / hi are float64
 * (flag 1) or float32 device arrays of `count` values. */
int inim_blend_frames(const void* lo, int lo_f64, const void* hi, int hi_f64, int64_t count, double frac, int same,
                      float* out, cudaStream_t stream);

/* Scratch bytes of inim_deform_background for a 2^k grid (0 if k outside 1..13). */
size_t inim_deform_background_scratch_bytes(int k);

/* deform_background (encodings.py:124-162): targets = the 4^k source pixel coordinates
 * (x = i/s, y = j/s, row-major) pushed through the composed fields (float32 (m, 2)),
 * values = the iteration-0 density (float32 (s, s)).  out (float64 (s, s)) = the
 * weight-normalised bilinear splat of the values at the targets, summed per pixel in
 * the reference's np.add.at order (bit-identical sums for identical inputs); pixels
 * without weight copy their nearest covered pixel (exact Euclidean distance transform).
 * range2 (device float[2]) receives min and max of the (positive) values. */
int inim_deform_background(const float* targets, const float* values, int k, double* out, float* range2,
                           void* scratch, cudaStream_t stream);

/* Host-buffer end-to-end call (the FFI a C/ctypes caller of the reference would bind):
 * pts_host (n,2) float64 in, final positions float64 out (may alias), `iterations`
 * fixed iterations.  Allocates and frees its own device memory; synchronises. */
int inim_run_host(const double* pts_host, double* out_host, int64_t n, int k, int kernel_size, double background,
                  int iterations);

/* Kernels per iteration of inim_run in steady state (launch accounting); a run adds
 * one splat kernel (the move of iteration t splats iteration t+1). */
int inim_kernels_per_iteration(int k);

#ifdef __cplusplus
}
#endif

#endif /* INIM_H_ */
