/*
 * inim_oracle.c -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).
 *
 * This file is the parity oracle for the B200 framework.  It restates, in plain C and
 * float64, the algorithm of the reference package `uncrowd`
 * (/root/reference/pkg/src/uncrowd/, the *.py modules), function by function, in the same arithmetic
 * order as the reference so that integer work is bit-exact and float work matches to
 * rounding.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load it, and only as the checker or the CPU baseline; the
 * product path (paper_2408_06513_b200) never links or calls it.
 *
 * Pinned against: the tests/golden npz fixtures, produced by tests/golden/make_golden.py, which
 * imports the unmodified reference package and records its outputs (see
 * tests/test_oracle_golden.py).
 *
 * Threading: loops whose iterations are independent run under OpenMP.  Parallelising
 * them does not change any result: each output element is computed by exactly the same
 * sequence of float operations as the sequential reference.  The doubling scans are
 * restated out-of-place per step, which is bit-identical to the reference's in-place
 * descending sweep (the sweep order exists only to keep the sources at pre-step values,
 * integral.py:45).
 *
 * Layout conventions follow model.py:1-8: grids are (2^k x 2^k) row-major, values[j*s+i],
 * i = x (column), j = y (row); fields are (s, s, 2) with x then y.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_ENOMEM 2
#define ORC_ESINGULAR 3

int orc_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}

/* ------------------------------------------------------------------ model.py */

/* pixel_of (model.py:189-198): i = min(floor(x * size), size - 1) as int64. */
static inline int64_t pixel_index(double x, int64_t size) {
    double f = floor(x * (double)size);
    int64_t i = (int64_t)f;
    if (i > size - 1) i = size - 1;
    return i;
}

int orc_pixel_of(const double* x, const double* y, int64_t n, int k, int64_t* i_out, int64_t* j_out) {
    int64_t size = (int64_t)1 << k;
    for (int64_t p = 0; p < n; ++p) {
        i_out[p] = pixel_index(x[p], size);
        j_out[p] = pixel_index(y[p], size);
    }
    return ORC_OK;
}

/* ---------------------------------------------------------------- density.py */

/* accumulate (density.py:14-27): per-pixel integer counts via bincount of j*s+i.
 * pos is (n, 2) row-major [x, y].  Counting is integer-exact, so per-thread partial
 * histograms reduce to the same grid.  Returns ORC_EINVAL on a negative index
 * (np.bincount raises ValueError there). */
int orc_accumulate(const double* pos, int64_t n, int k, double* grid) {
    int64_t size = (int64_t)1 << k;
    int64_t m = size * size;
    memset(grid, 0, sizeof(double) * (size_t)m);
    if (n == 0) return ORC_OK;
    int64_t* counts = (int64_t*)calloc((size_t)m, sizeof(int64_t));
    if (!counts) return ORC_ENOMEM;
    int bad = 0;
    for (int64_t p = 0; p < n; ++p) {
        int64_t i = pixel_index(pos[2 * p], size);
        int64_t j = pixel_index(pos[2 * p + 1], size);
        if (i < 0 || j < 0 || pos[2 * p] != pos[2 * p] || pos[2 * p + 1] != pos[2 * p + 1]) { bad = 1; break; }
        counts[j * size + i] += 1;
    }
    if (!bad) {
        for (int64_t q = 0; q < m; ++q) grid[q] = (double)counts[q];
    }
    free(counts);
    return bad ? ORC_EINVAL : ORC_OK;
}

/* smoothing_kernel (density.py:30-37): 6*ks+1 taps, sigma = ks/2, normalised by the
 * numpy pairwise sum of the taps. */
static double pairwise_sum(const double* a, int64_t n);

int orc_smoothing_kernel(int ks, double* w) {
    if (ks < 1) return ORC_EINVAL;
    int radius = 3 * ks;
    double sigma = ks / 2.0;
    int nt = 2 * radius + 1;
    for (int t = 0; t < nt; ++t) {
        double u = (double)(t - radius) / sigma;
        w[t] = exp(-0.5 * (u * u));
    }
    double s = pairwise_sum(w, nt);
    for (int t = 0; t < nt; ++t) w[t] = w[t] / s;
    return ORC_OK;
}

/* Half-sample symmetric reflection with period 2n (scipy.ndimage mode="reflect",
 * restated as tests/oracles.py:95-102): ... 1 0 | 0 1 ... n-1 | n-1 n-2 ... */
static inline int64_t reflect_index(int64_t idx, int64_t n) {
    int64_t p = 2 * n;
    idx %= p;
    if (idx < 0) idx += p;
    if (idx >= n) idx = p - 1 - idx;
    return idx;
}

/* convolve1d(grid, w, axis, mode="reflect") for a symmetric odd kernel
 * (density.py:49-50).  The accumulation order restates the symmetric branch of the
 * scipy.ndimage 1-D correlation loop: out = x[0]*w[0], then for the outermost tap
 * inwards out += (x[-t] + x[+t]) * w[t]. */
static void convolve_reflect_axis(const double* in, int64_t s, const double* w, int nt, int axis, double* out) {
    int r = nt / 2;
    const double* wc = w + r;
#pragma omp parallel
    {
        double* line = (double*)malloc(sizeof(double) * (size_t)(s + 2 * r));
#pragma omp for schedule(static)
        for (int64_t L = 0; L < s; ++L) {
            /* gather the extended line */
            for (int64_t q = -r; q < s + r; ++q) {
                int64_t src = reflect_index(q, s);
                line[q + r] = axis == 1 ? in[L * s + src] : in[src * s + L];
            }
            const double* c = line + r;
            for (int64_t q = 0; q < s; ++q) {
                const double* x = c + q;
                double acc = x[0] * wc[0];
                for (int t = -r; t < 0; ++t) acc += (x[t] + x[-t]) * wc[t];
                if (axis == 1) out[L * s + q] = acc; else out[q * s + L] = acc;
            }
        }
        free(line);
    }
}

/* gaussian_smooth (density.py:40-51): horizontal pass (axis=1) then vertical (axis=0). */
int orc_gaussian_smooth(const double* grid, int64_t s, int ks, double* out) {
    if (ks < 1) return ORC_EINVAL;
    int nt = 6 * ks + 1;
    double* w = (double*)malloc(sizeof(double) * nt);
    double* tmp = (double*)malloc(sizeof(double) * (size_t)(s * s));
    if (!w || !tmp) { free(w); free(tmp); return ORC_ENOMEM; }
    orc_smoothing_kernel(ks, w);
    convolve_reflect_axis(grid, s, w, nt, 1, tmp);
    convolve_reflect_axis(tmp, s, w, nt, 0, out);
    free(w);
    free(tmp);
    return ORC_OK;
}

/* build_density (density.py:54-78).  background <= 0 on entry means "auto"
 * (n / 4^k, or 1.0 for an empty dataset); the caller raises ZeroBackground for an
 * explicit non-positive value before calling. */
int orc_build_density(const double* pos, int64_t n, int k, int ks, double background,
                      double* values, double* background_out) {
    int64_t s = (int64_t)1 << k;
    if (background <= 0.0) {
        background = (double)n / (double)((int64_t)1 << (2 * k));
        if (background == 0.0) background = 1.0;
    }
    double* counts = (double*)malloc(sizeof(double) * (size_t)(s * s));
    if (!counts) return ORC_ENOMEM;
    int rc = orc_accumulate(pos, n, k, counts);
    if (rc == ORC_OK) rc = orc_gaussian_smooth(counts, s, ks, values);
    free(counts);
    if (rc != ORC_OK) return rc;
    for (int64_t q = 0; q < s * s; ++q) values[q] += background;
    *background_out = background;
    return ORC_OK;
}

/* --------------------------------------------------------------- integral.py */

/* numpy's pairwise summation (the algorithm behind ndarray.sum for contiguous
 * float64): used for `total = float(values.sum())` (integral.py:246). */
static double pairwise_sum(const double* a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; ++i) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
    }
}

double orc_sum(const double* a, int64_t n) { return pairwise_sum(a, n); }

/* One doubling stage, restated out-of-place per step.  (dj, di) is the source offset
 * of a step of length 1 (the source is (j - step*dj, i - step*di)).  This covers
 * _scan_rows_down (dj=1,di=0; integral.py:43-52), _scan_rows_up (dj=-1; 55-63),
 * _scan_cols_right (di=1; 66-74), _scan_cols_left (di=-1; 77-85) and the four
 * _scan_diagonal variants (88-110).  Each element is updated from pre-step values
 * exactly as in the reference's in-place sweep. */
static int doubling_scan(double* a, int64_t s, int dj, int di) {
    double* b = (double*)malloc(sizeof(double) * (size_t)(s * s));
    if (!b) return ORC_ENOMEM;
    for (int64_t step = 1; step < s; step *= 2) {
        memcpy(b, a, sizeof(double) * (size_t)(s * s));
#pragma omp parallel for schedule(static)
        for (int64_t j = 0; j < s; ++j) {
            int64_t sj = j - step * dj;
            if (sj < 0 || sj >= s) continue;
            for (int64_t i = 0; i < s; ++i) {
                int64_t si = i - step * di;
                if (si < 0 || si >= s) continue;
                a[j * s + i] = b[j * s + i] + b[sj * s + si];
            }
        }
    }
    free(b);
    return ORC_OK;
}

/* _scan_1d (integral.py:113-120) */
static void scan_1d(double* a, int64_t n) {
    for (int64_t step = 1; step < n; step *= 2)
        for (int64_t i = n - 1; i >= step; --i) a[i] += a[i - step];
}

static int is_pow2_square(int64_t s) { return s >= 1 && (s & (s - 1)) == 0; }

/* column_integrals (integral.py:180-186): upper = inclusive column prefix (rows <= j),
 * lower = strict column suffix (rows > j), both by k doubling steps. */
int orc_column_integrals(const double* d, int64_t s, double* upper, double* lower) {
    if (!is_pow2_square(s)) return ORC_EINVAL;
    memcpy(upper, d, sizeof(double) * (size_t)(s * s));
    int rc = doubling_scan(upper, s, 1, 0);
    if (rc) return rc;
    /* _suffix_scan_exclusive axis 0 (integral.py:159-169): out[:-1] = values[1:] */
    memset(lower, 0, sizeof(double) * (size_t)(s * s));
    if (s > 1) memcpy(lower, d + s, sizeof(double) * (size_t)((s - 1) * s));
    return doubling_scan(lower, s, -1, 0);
}

/* classical_rects (integral.py:189-200): returns (tl, bl, br, tr). */
int orc_classical_rects(const double* upper, const double* lower, int64_t s,
                        double* tl, double* bl, double* br, double* tr) {
    int rc;
    memcpy(tl, upper, sizeof(double) * (size_t)(s * s));
    if ((rc = doubling_scan(tl, s, 0, 1))) return rc;
    memcpy(bl, lower, sizeof(double) * (size_t)(s * s));
    if ((rc = doubling_scan(bl, s, 0, 1))) return rc;
    /* _suffix_scan_exclusive axis 1: out[:, :-1] = values[:, 1:] */
    memset(tr, 0, sizeof(double) * (size_t)(s * s));
    memset(br, 0, sizeof(double) * (size_t)(s * s));
    for (int64_t j = 0; j < s; ++j)
        for (int64_t i = 0; i + 1 < s; ++i) {
            tr[j * s + i] = upper[j * s + i + 1];
            br[j * s + i] = lower[j * s + i + 1];
        }
    if ((rc = doubling_scan(tr, s, 0, -1))) return rc;
    return doubling_scan(br, s, 0, -1);
}

/* triangle_integrals (integral.py:203-209): chains of upper toward up-left /
 * up-right, of lower toward down-left / down-right. */
int orc_triangle_integrals(const double* upper, const double* lower, int64_t s,
                           double* up_left, double* up_right, double* down_left, double* down_right) {
    int rc;
    memcpy(up_left, upper, sizeof(double) * (size_t)(s * s));
    if ((rc = doubling_scan(up_left, s, 1, 1))) return rc;       /* a[j,i] += a[j-st, i-st] */
    memcpy(up_right, upper, sizeof(double) * (size_t)(s * s));
    if ((rc = doubling_scan(up_right, s, 1, -1))) return rc;     /* a[j,i] += a[j-st, i+st] */
    memcpy(down_left, lower, sizeof(double) * (size_t)(s * s));
    if ((rc = doubling_scan(down_left, s, -1, 1))) return rc;    /* a[j,i] += a[j+st, i-st] */
    memcpy(down_right, lower, sizeof(double) * (size_t)(s * s));
    return doubling_scan(down_right, s, -1, -1);                 /* a[j,i] += a[j+st, i+st] */
}

/* tilted_wedges (integral.py:212-228): returns (up, left, down, right). */
int orc_tilted_wedges(const double* up_left, const double* up_right, const double* down_left,
                      const double* down_right, const double* upper, const double* lower, int64_t s,
                      double* w_up, double* w_left, double* w_down, double* w_right) {
    double* left_half = (double*)malloc(sizeof(double) * (size_t)s);
    double* right_half = (double*)malloc(sizeof(double) * (size_t)s);
    if (!left_half || !right_half) { free(left_half); free(right_half); return ORC_ENOMEM; }
    for (int64_t i = 0; i < s; ++i) left_half[i] = upper[(s - 1) * s + i];
    scan_1d(left_half, s);
    /* _prefix_scan(colsum[::-1])[::-1] */
    for (int64_t i = 0; i < s; ++i) right_half[i] = upper[(s - 1) * s + (s - 1 - i)];
    scan_1d(right_half, s);
    for (int64_t lo = 0, hi = s - 1; lo < hi; ++lo, --hi) {
        double t = right_half[lo]; right_half[lo] = right_half[hi]; right_half[hi] = t;
    }
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < s; ++j)
        for (int64_t i = 0; i < s; ++i) {
            int64_t q = j * s + i;
            w_up[q] = up_left[q] + up_right[q] - upper[q];
            w_down[q] = down_left[q] + down_right[q] - lower[q];
            w_left[q] = left_half[i] - up_left[q] - down_left[q];
            w_right[q] = right_half[i] - up_right[q] - down_right[q];
        }
    free(left_half);
    free(right_half);
    return ORC_OK;
}

/* build_integral_set (integral.py:231-247).  tables8 is 8*s*s in the order
 * tl, bl, br, tr, up, left, down, right (model.py:81-85). */
int orc_build_integral_set(const double* d, int64_t s, double* tables8, double* total) {
    if (!is_pow2_square(s)) return ORC_EINVAL;
    int64_t m = s * s;
    double* upper = (double*)malloc(sizeof(double) * (size_t)m);
    double* lower = (double*)malloc(sizeof(double) * (size_t)m);
    double* tri = (double*)malloc(sizeof(double) * (size_t)(4 * m));
    int rc = ORC_ENOMEM;
    if (upper && lower && tri) {
        rc = orc_column_integrals(d, s, upper, lower);
        if (!rc) rc = orc_classical_rects(upper, lower, s, tables8, tables8 + m, tables8 + 2 * m, tables8 + 3 * m);
        if (!rc) rc = orc_triangle_integrals(upper, lower, s, tri, tri + m, tri + 2 * m, tri + 3 * m);
        if (!rc) rc = orc_tilted_wedges(tri, tri + m, tri + 2 * m, tri + 3 * m, upper, lower, s,
                                        tables8 + 4 * m, tables8 + 5 * m, tables8 + 6 * m, tables8 + 7 * m);
        if (!rc) *total = pairwise_sum(d, m);
    }
    free(upper);
    free(lower);
    free(tri);
    return rc;
}

/* ---------------------------------------------------------------- mapping.py */

/* _per_pixel_targets (mapping.py:146-178) / _raw_targets_per_pixel (181-191). */
int orc_raw_targets_per_pixel(const double* tables8, double total, int k, double* out) {
    if (!(total > 0.0)) return ORC_ESINGULAR;
    int64_t size = (int64_t)1 << k;
    int64_t m = size * size;
    double scale = ldexp(1.0, -k);
    double inv = 0.5 / total;
    const double *rtl = tables8, *rbl = tables8 + m, *rbr = tables8 + 2 * m, *rtr = tables8 + 3 * m;
    const double *wup = tables8 + 4 * m, *wleft = tables8 + 5 * m, *wdown = tables8 + 6 * m, *wright = tables8 + 7 * m;
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < size; ++j) {
        double y = j * scale;
        for (int64_t i = 0; i < size; ++i) {
            double x = i * scale;
            double dr_x, dr_y, ul_x, ul_y, ur_x, ur_y, dl_x, dl_y;
            if (y < x) { dr_x = 1.0; dr_y = 1.0 + y - x; ul_x = x - y; ul_y = 0.0; }
            else { dr_x = 1.0 - y + x; dr_y = 1.0; ul_x = 0.0; ul_y = y - x; }
            if (x + y < 1.0) { ur_x = x + y; ur_y = 0.0; dl_x = 0.0; dl_y = x + y; }
            else { ur_x = 1.0; ur_y = x + y - 1.0; dl_x = x + y - 1.0; dl_y = 1.0; }
            int64_t q = j * size + i;
            double tl = rtl[q], bl = rbl[q], br = rbr[q], tr = rtr[q];
            double up = wup[q], left = wleft[q], down = wdown[q], right = wright[q];
            out[2 * q] = (tl * dr_x + bl * ur_x + br * ul_x + tr * dl_x + (up + down) * x + left) * inv;
            out[2 * q + 1] = (tl * dr_y + bl * ur_y + br * ul_y + tr * dl_y + (left + right) * y + up) * inv;
        }
    }
    return ORC_OK;
}

/* flat_response.get(k) (mapping.py:120-126): raw targets of build_integral_set(ones). */
int orc_flat_response(int k, double* out) {
    int64_t s = (int64_t)1 << k, m = s * s;
    double* ones = (double*)malloc(sizeof(double) * (size_t)m);
    double* t8 = (double*)malloc(sizeof(double) * (size_t)(8 * m));
    int rc = ORC_ENOMEM;
    if (ones && t8) {
        for (int64_t q = 0; q < m; ++q) ones[q] = 1.0;
        double total;
        rc = orc_build_integral_set(ones, s, t8, &total);
        if (!rc) rc = orc_raw_targets_per_pixel(t8, total, k, out);
    }
    free(ones);
    free(t8);
    return rc;
}

/* build_field (mapping.py:194-204): targets = raw - defect + (X, Y); excursion before
 * the clip; clip to [0, 1].  unit_coordinates (model.py:183-186): arange * 2^-k. */
int orc_build_field(const double* tables8, double total, int k, const double* defect,
                    double* targets, double* max_excursion) {
    int rc = orc_raw_targets_per_pixel(tables8, total, k, targets);
    if (rc) return rc;
    int64_t size = (int64_t)1 << k, m = size * size;
    double scale = ldexp(1.0, -k);
    double mn = INFINITY, mx = -INFINITY;
    for (int64_t j = 0; j < size; ++j)
        for (int64_t i = 0; i < size; ++i) {
            int64_t q = j * size + i;
            double tx = targets[2 * q] - defect[2 * q];
            double ty = targets[2 * q + 1] - defect[2 * q + 1];
            tx += (double)i * scale;
            ty += (double)j * scale;
            targets[2 * q] = tx;
            targets[2 * q + 1] = ty;
            if (tx < mn) mn = tx;
            if (ty < mn) mn = ty;
            if (tx > mx) mx = tx;
            if (ty > mx) mx = ty;
        }
    double exc = 0.0;
    if (-mn > exc) exc = -mn;
    if (mx - 1.0 > exc) exc = mx - 1.0;
    *max_excursion = exc;
    for (int64_t q = 0; q < 2 * m; ++q) {
        double v = targets[q];
        targets[q] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    }
    return ORC_OK;
}

/* _bilinear_kernel (mapping.py:207-232), sample_field (235-246). */
int orc_sample_field(const double* targets, int k, const double* pts, int64_t n, double* out) {
    int64_t size = (int64_t)1 << k;
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < n; ++r) {
        double sx = pts[2 * r] * (double)size;
        double sy = pts[2 * r + 1] * (double)size;
        int64_t i0 = (int64_t)floor(sx), j0 = (int64_t)floor(sy);
        if (i0 < 0) i0 = 0; else if (i0 > size - 2) i0 = size - 2;
        if (j0 < 0) j0 = 0; else if (j0 > size - 2) j0 = size - 2;
        double fx = sx - (double)i0, fy = sy - (double)j0;
        double w00 = (1.0 - fx) * (1.0 - fy);
        double w10 = fx * (1.0 - fy);
        double w01 = (1.0 - fx) * fy;
        double w11 = fx * fy;
        for (int c = 0; c < 2; ++c) {
            out[2 * r + c] = (w00 * targets[2 * (j0 * size + i0) + c] + w10 * targets[2 * (j0 * size + i0 + 1) + c]
                              + w01 * targets[2 * ((j0 + 1) * size + i0) + c]
                              + w11 * targets[2 * ((j0 + 1) * size + i0 + 1) + c]);
        }
    }
    return ORC_OK;
}

/* -------------------------------------------------------------- regularize.py */

/* iterate_once (regularize.py:25-37): density -> tables -> field -> clip(sample).
 * defect may be NULL (then flat_response(k) is built here).  Outputs new_pos (n,2);
 * field_out (s,s,2) and density_out (s,s) are optional. */
int orc_iterate_once(const double* pos, int64_t n, int k, int ks, double background,
                     const double* defect, double* new_pos, double* field_out,
                     double* density_out, double* max_excursion) {
    int64_t s = (int64_t)1 << k, m = s * s;
    double* values = density_out ? density_out : (double*)malloc(sizeof(double) * (size_t)m);
    double* t8 = (double*)malloc(sizeof(double) * (size_t)(8 * m));
    double* field = field_out ? field_out : (double*)malloc(sizeof(double) * (size_t)(2 * m));
    double* own_defect = NULL;
    int rc = ORC_ENOMEM;
    if (!values || !t8 || !field) goto done;
    if (!defect) {
        own_defect = (double*)malloc(sizeof(double) * (size_t)(2 * m));
        if (!own_defect) goto done;
        if ((rc = orc_flat_response(k, own_defect))) goto done;
        defect = own_defect;
    }
    double bg, total, exc;
    if ((rc = orc_build_density(pos, n, k, ks, background, values, &bg))) goto done;
    if ((rc = orc_build_integral_set(values, s, t8, &total))) goto done;
    if ((rc = orc_build_field(t8, total, k, defect, field, &exc))) goto done;
    if (max_excursion) *max_excursion = exc;
    if ((rc = orc_sample_field(field, k, pos, n, new_pos))) goto done;
    for (int64_t q = 0; q < 2 * n; ++q) {
        double v = new_pos[q];
        new_pos[q] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    }
done:
    if (!density_out) free(values);
    if (!field_out) free(field);
    free(t8);
    free(own_defect);
    return rc;
}

/* ================================================================ layout metrics
 * metrics.py restated over integers (the quantities the reference reduces to floats
 * at its last step).  The neighbour ranks are counted directly instead of through the
 * reference's full argsort: rank_i(j) = 1 + #{l != i : (d(i,l), l) < (d(i,j), j)},
 * which is the position of j in a stable argsort of row i with self first
 * (metrics.py:77-90).
 */

/* binned_stddev / overplotting moments (metrics.py:46-71) of a float64 layout:
 * out[0] = occupied pixels, out[1] = sum over 4x4 bins of count^2 (k >= 2, else 0),
 * out[2] = n. */
int orc_frame_stats(const double* pos, int64_t n, int k, int64_t* out) {
    if (k < 0 || k > 14 || n < 0 || !out) return 1;
    const int64_t s = (int64_t)1 << k;
    int64_t* cnt = (int64_t*)calloc((size_t)(s * s), sizeof(int64_t));
    if (!cnt) return 2;
    for (int64_t q = 0; q < n; ++q) cnt[pixel_index(pos[2 * q + 1], s) * s + pixel_index(pos[2 * q], s)] += 1;
    int64_t occ = 0, sq = 0;
    for (int64_t p = 0; p < s * s; ++p) occ += cnt[p] != 0;
    if (k >= 2) {
        const int64_t b = s / 4;
        for (int64_t bj = 0; bj < b; ++bj)
            for (int64_t bi = 0; bi < b; ++bi) {
                int64_t c = 0;
                for (int r = 0; r < 4; ++r)
                    for (int q = 0; q < 4; ++q) c += cnt[(4 * bj + r) * s + 4 * bi + q];
                sq += c * c;
            }
    }
    free(cnt);
    out[0] = occ;
    out[1] = sq;
    out[2] = n;
    return 0;
}

static inline double orc_dist2(const double* p, int64_t i, int64_t j) {
    const double dx = p[2 * i] - p[2 * j];
    const double dy = p[2 * i + 1] - p[2 * j + 1];
    return dx * dx + dy * dy; /* -ffp-contract=off: (dx*dx) + (dy*dy), two roundings */
}

static inline int key_before(double d, int64_t j, double e, int64_t l) { return d < e || (d == e && j < l); }

/* trustworthiness numerator (metrics.py:95-108): sum over i of
 * max(0, rank_orig_i(j) - nn) for the nn nearest j != i of the deformed layout. */
int orc_trust_penalty(const double* orig, const double* moved, int64_t n, int nn, int64_t* out) {
    if (n < 0 || nn < 1 || nn >= n || !out) return 1;
    int64_t total = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : total)
    for (int64_t i = 0; i < n; ++i) {
        int64_t sel[64];
        int64_t* selp = nn <= 64 ? sel : (int64_t*)malloc(sizeof(int64_t) * (size_t)nn);
        double last_d = -1.0;
        int64_t last_j = -1;
        for (int r = 0; r < nn; ++r) { /* r-th nearest by (distance, index) */
            double bd = INFINITY;
            int64_t bj = INT64_MAX;
            for (int64_t j = 0; j < n; ++j) {
                if (j == i) continue;
                const double d = orc_dist2(moved, i, j);
                if (key_before(last_d, last_j, d, j) && key_before(d, j, bd, bj)) {
                    bd = d;
                    bj = j;
                }
            }
            selp[r] = bj;
            last_d = bd;
            last_j = bj;
        }
        for (int r = 0; r < nn; ++r) {
            const int64_t j = selp[r];
            const double dj = orc_dist2(orig, i, j);
            int64_t rank = 1;
            for (int64_t l = 0; l < n; ++l)
                if (l != i && key_before(orc_dist2(orig, i, l), l, dj, j)) ++rank;
            if (rank > nn) total += rank - nn;
        }
        if (selp != sel) free(selp);
    }
    *out = total;
    return 0;
}

/* orthogonal_ordering numerator (metrics.py:136-143): pairs i < j whose x-order and
 * y-order signs agree between the two layouts. */
static inline int sgn3(double a, double b) { return (a > b) - (a < b); }

int orc_order_pairs(const double* orig, const double* moved, int64_t n, int64_t* out) {
    if (n < 0 || !out) return 1;
    int64_t kept = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : kept)
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = i + 1; j < n; ++j)
            kept += sgn3(orig[2 * i], orig[2 * j]) == sgn3(moved[2 * i], moved[2 * j]) &&
                    sgn3(orig[2 * i + 1], orig[2 * j + 1]) == sgn3(moved[2 * i + 1], moved[2 * j + 1]);
    *out = kept;
    return 0;
}

/* ============================================================ deform_background
 * encodings.py:141-156: cell / fractions of every mapped source pixel, then the four
 * np.add.at passes in order, each sequential over the sources (unbuffered in-place
 * accumulation), then acc / weight on covered pixels.  covered[p] = weight > 0.  The
 * nearest-covered fill (scipy distance_transform_edt) is done by the Python wrapper
 * with the reference's own scipy call.
 */
int orc_background_splat(const double* targets, const double* values, int k, double* out, unsigned char* covered) {
    if (k < 1 || k > 14) return 1;
    const int64_t s = (int64_t)1 << k, m = s * s;
    double* acc = (double*)calloc((size_t)m, sizeof(double));
    double* wgt = (double*)calloc((size_t)m, sizeof(double));
    int64_t* cell = (int64_t*)malloc(sizeof(int64_t) * 2 * (size_t)m);
    double* frac = (double*)malloc(sizeof(double) * 2 * (size_t)m);
    if (!acc || !wgt || !cell || !frac) {
        free(acc); free(wgt); free(cell); free(frac);
        return 2;
    }
    for (int64_t q = 0; q < m; ++q)
        for (int a = 0; a < 2; ++a) {
            const double sc = targets[2 * q + a] * (double)s;
            double c = floor(sc);
            if (c < 0.0) c = 0.0;
            if (c > (double)(s - 2)) c = (double)(s - 2);
            double f = sc - c;
            if (f < 0.0) f = 0.0;
            if (f > 1.0) f = 1.0;
            cell[2 * q + a] = (int64_t)c;
            frac[2 * q + a] = f;
        }
    for (int pass = 0; pass < 4; ++pass) {
        const int di = pass & 1, dj = pass >> 1;
        for (int64_t q = 0; q < m; ++q) {
            const double fx = frac[2 * q], fy = frac[2 * q + 1];
            const double w = (di ? fx : 1.0 - fx) * (dj ? fy : 1.0 - fy);
            const int64_t p = (cell[2 * q + 1] + dj) * s + cell[2 * q] + di;
            acc[p] += w * values[q];
            wgt[p] += w;
        }
    }
    for (int64_t p = 0; p < m; ++p) {
        covered[p] = wgt[p] > 0.0;
        out[p] = covered[p] ? acc[p] / wgt[p] : 0.0;
    }
    free(acc); free(wgt); free(cell); free(frac);
    return 0;
}
