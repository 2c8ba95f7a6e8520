/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker + CPU baseline).
 *
 * A float64, matrix-free CPU restatement of the reference's hot path
 * (arxiv/paper_2602_09527, package `proxtomo`, pure Python/numpy/scipy):
 *
 *   - Joseph ray-driven forward projector     pkg/src/proxtomo/projector.py:26-61,114-126
 *   - its exact algebraic adjoint (as a gather) pkg/src/proxtomo/projector.py:64-97,129-140
 *   - FGP (Beck-Teboulle) dual TV prox          pkg/src/proxtomo/regularizers.py:62-76,90-133
 *   - a 3D slice-stacked extension of FGP (no reference code, "parity unpinned"
 *     for the 3D stencil, pinned instead by a dense dual-PG QP oracle in tests/)
 *
 * The reference stores A as an explicit scipy CSR matrix and applies it with
 * csr_matvec; this file evaluates the same COO entries on the fly, with every
 * floating-point expression written in the reference's operation order so the
 * weights are bitwise identical (built with -ffp-contract=off, no FMA).
 * Summation order: forward sums along the ray in step order (the CSR sums in
 * ascending flat-pixel order; identical for row-stepping rays, a permutation for
 * column-stepping ones -> differences at the 1e-16 relative level); the adjoint
 * gather sums in ascending A-row order, which is exactly the CSR of A^T order.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library.  The product path never does.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int branch_rows; /* 1: |cos| >= |sin| -> one sample per image row (projector.py:32-40) */
    double cos_t, sin_t, step_len;
} angle_par;

static angle_par angle_params(double theta, double h)
{
    angle_par a;
    a.cos_t = cos(theta);
    a.sin_t = sin(theta);
    if (fabs(a.cos_t) >= fabs(a.sin_t)) {
        a.branch_rows = 1;
        a.step_len = h / fabs(a.cos_t);
    } else {
        a.branch_rows = 0;
        a.step_len = h / fabs(a.sin_t);
    }
    return a;
}

/* pos exactly as projector.py:28,36-37,43-44,49 */
static inline double joseph_pos(const angle_par* a, int b, int step, int n_bins, int height,
                                int width, double ds, double h)
{
    double s = ((double)b - (n_bins - 1) / 2.0) * ds;
    double cross;
    int n_lanes;
    if (a->branch_rows) {
        double axis = ((double)step - (height - 1) / 2.0) * h;
        cross = (s - axis * a->sin_t) / a->cos_t;
        n_lanes = width;
    } else {
        double axis = ((double)step - (width - 1) / 2.0) * h;
        cross = (s - axis * a->cos_t) / a->sin_t;
        n_lanes = height;
    }
    return cross / h + (n_lanes - 1) / 2.0;
}

int oracle_nthreads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* y[k, b] = sum over the ray (angle thetas[k], bin b) of Joseph taps * x.
 * x: (n_slices, height, width) row-major; y: (n_slices, n_sel, n_bins).
 * n_slices > 1 is the slice-stacked 3D geometry (rotation about z): every
 * z-slice is an independent 2D problem with the same operator. */
void oracle_forward(int height, int width, int n_bins, double ds, double h, int n_sel,
                    const double* thetas, int n_slices, const double* x, double* y)
{
    long total = (long)n_slices * n_sel * n_bins;
#pragma omp parallel for schedule(static)
    for (long idx = 0; idx < total; ++idx) {
        int b = (int)(idx % n_bins);
        long t = idx / n_bins;
        int k = (int)(t % n_sel);
        int z = (int)(t / n_sel);
        const double* img = x + (long)z * height * width;
        angle_par a = angle_params(thetas[k], h);
        int n_steps = a.branch_rows ? height : width;
        int n_lanes = a.branch_rows ? width : height;
        double acc = 0.0;
        for (int st = 0; st < n_steps; ++st) {
            double pos = joseph_pos(&a, b, st, n_bins, height, width, ds, h);
            double fl = floor(pos);
            long lane0 = (long)fl;
            double frac = pos - fl;
            double w0 = (1.0 - frac) * a.step_len;
            double w1 = frac * a.step_len;
            /* projector.py:55-60: keep iff lane in range and w > 0 */
            if (lane0 >= 0 && lane0 < n_lanes && w0 > 0.0) {
                long flat = a.branch_rows ? (long)st * width + lane0 : lane0 * width + st;
                acc += w0 * img[flat];
            }
            long lane1 = lane0 + 1;
            if (lane1 >= 0 && lane1 < n_lanes && w1 > 0.0) {
                long flat = a.branch_rows ? (long)st * width + lane1 : lane1 * width + st;
                acc += w1 * img[flat];
            }
        }
        y[idx] = acc;
    }
}

/* x[r, c] = sum over rays (subset order, then ascending bin) of the tap that
 * lands on pixel (r, c) times y: the CSR-of-A^T row of pixel (r, c)
 * (projector.py:83,96,140) evaluated as a per-pixel gather. */
void oracle_adjoint(int height, int width, int n_bins, double ds, double h, int n_sel,
                    const double* thetas, int n_slices, const double* y, double* x)
{
    angle_par* ap = (angle_par*)malloc(sizeof(angle_par) * (n_sel > 0 ? n_sel : 1));
    for (int k = 0; k < n_sel; ++k) ap[k] = angle_params(thetas[k], h);
    long total = (long)n_slices * height * width;
#pragma omp parallel for schedule(static)
    for (long idx = 0; idx < total; ++idx) {
        int c = (int)(idx % width);
        long t = idx / width;
        int r = (int)(t % height);
        int z = (int)(t / height);
        const double* sino = y + (long)z * n_sel * n_bins;
        double acc = 0.0;
        for (int k = 0; k < n_sel; ++k) {
            const angle_par* a = &ap[k];
            int step = a->branch_rows ? r : c;
            int lane = a->branch_rows ? c : r;
            /* bin where pos == lane, from the linear pos(b) relation */
            double trig = a->branch_rows ? a->cos_t : a->sin_t;
            double sigma = ds / (h * trig); /* d pos / d b */
            double p0 = joseph_pos(a, 0, step, n_bins, height, width, ds, h);
            double bf = ((double)lane - p0) / sigma;
            int half = (int)ceil(1.0 / fabs(sigma)) + 1;
            long b_lo = (long)floor(bf) - half;
            long b_hi = (long)floor(bf) + half;
            if (b_lo < 0) b_lo = 0;
            if (b_hi > n_bins - 1) b_hi = n_bins - 1;
            for (long b = b_lo; b <= b_hi; ++b) {
                double pos = joseph_pos(a, (int)b, step, n_bins, height, width, ds, h);
                double fl = floor(pos);
                long lane0 = (long)fl;
                double frac = pos - fl;
                double v = sino[(long)k * n_bins + b];
                if (lane0 == lane) {
                    double w0 = (1.0 - frac) * a->step_len;
                    if (w0 > 0.0) acc += w0 * v;
                } else if (lane0 + 1 == lane) {
                    double w1 = frac * a->step_len;
                    if (w1 > 0.0) acc += w1 * v;
                }
            }
        }
        x[idx] = acc;
    }
    free(ap);
}

/* ---------------------------------------------------------------------- */
/* FGP TV prox, 2D: regularizers.py:90-133, expression by expression.      */
/* p, q: in = warm duals (zeros for a cold start), out = final duals.      */
/* ---------------------------------------------------------------------- */
void oracle_fgp2d(int height, int width, const double* image, double lam, int iters,
                  int nonneg, double* p, double* q, double* out)
{
    long n = (long)height * width;
    double* r = (double*)malloc(sizeof(double) * n);
    double* s = (double*)malloc(sizeof(double) * n);
    double* pp = (double*)malloc(sizeof(double) * n);
    double* qp = (double*)malloc(sizeof(double) * n);
    double* u = (double*)malloc(sizeof(double) * n);
    memcpy(r, p, sizeof(double) * n);
    memcpy(s, q, sizeof(double) * n);
    memcpy(pp, p, sizeof(double) * n);
    memcpy(qp, q, sizeof(double) * n);
    double t = 1.0;
    double step = 1.0 / (8.0 * lam);
    for (int it = 0; it < iters; ++it) {
#pragma omp parallel for schedule(static)
        for (long idx = 0; idx < n; ++idx) {
            int i = (int)(idx / width), j = (int)(idx % width);
            /* _diff_adjoint (regularizers.py:70-76) in numpy's statement order */
            double o = 0.0;
            if (i < height - 1) o -= r[idx];
            if (i > 0) o += r[idx - width];
            if (j < width - 1) o -= s[idx];
            if (j > 0) o += s[idx - 1];
            double uu = image[idx] - lam * o;
            if (nonneg) uu = (uu < 0.0) ? 0.0 : uu; /* np.maximum(u, 0) */
            u[idx] = uu;
        }
        double t_next = (1.0 + sqrt(1.0 + 4.0 * t * t)) / 2.0;
        double beta = (t - 1.0) / t_next;
#pragma omp parallel for schedule(static)
        for (long idx = 0; idx < n; ++idx) {
            int i = (int)(idx / width), j = (int)(idx % width);
            double gv = (i < height - 1) ? u[idx + width] - u[idx] : 0.0;
            double gh = (j < width - 1) ? u[idx + 1] - u[idx] : 0.0;
            double ph = r[idx] + step * gv;
            double qh = s[idx] + step * gh;
            double nrm = sqrt(ph * ph + qh * qh);
            double scale = (nrm > 1.0 || nrm != nrm) ? nrm : 1.0; /* np.maximum(1, .) */
            double pn = ph / scale, qn = qh / scale;
            double rn = pn + beta * (pn - pp[idx]);
            double sn = qn + beta * (qn - qp[idx]);
            pp[idx] = pn;
            qp[idx] = qn;
            r[idx] = rn;
            s[idx] = sn;
        }
        t = t_next;
    }
    /* p, q = final duals (= p_prev after the swap, regularizers.py:129) */
#pragma omp parallel for schedule(static)
    for (long idx = 0; idx < n; ++idx) {
        int i = (int)(idx / width), j = (int)(idx % width);
        double o = 0.0;
        if (i < height - 1) o -= pp[idx];
        if (i > 0) o += pp[idx - width];
        if (j < width - 1) o -= qp[idx];
        if (j > 0) o += qp[idx - 1];
        double v = image[idx] - lam * o;
        if (nonneg) v = (v < 0.0) ? 0.0 : v;
        out[idx] = v;
    }
    if (iters > 0) {
        memcpy(p, pp, sizeof(double) * n);
        memcpy(q, qp, sizeof(double) * n);
    }
    free(r); free(s); free(pp); free(qp); free(u);
}

/* 3D isotropic FGP on a (depth, height, width) volume: the 2D algorithm with
 * a third forward difference along z and dual step 1/(12*lam) (the 3D bound
 * ||D||^2 <= 12).  No reference code exists. */
void oracle_fgp3d(int depth, int height, int width, const double* image, double lam,
                  int iters, int nonneg, double* p, double* q, double* w, double* out)
{
    long plane = (long)height * width;
    long n = (long)depth * plane;
    double* r = (double*)malloc(sizeof(double) * n);
    double* s = (double*)malloc(sizeof(double) * n);
    double* o3 = (double*)malloc(sizeof(double) * n);
    double* pp = (double*)malloc(sizeof(double) * n);
    double* qp = (double*)malloc(sizeof(double) * n);
    double* wp = (double*)malloc(sizeof(double) * n);
    double* u = (double*)malloc(sizeof(double) * n);
    memcpy(r, p, sizeof(double) * n);
    memcpy(s, q, sizeof(double) * n);
    memcpy(o3, w, sizeof(double) * n);
    memcpy(pp, p, sizeof(double) * n);
    memcpy(qp, q, sizeof(double) * n);
    memcpy(wp, w, sizeof(double) * n);
    double t = 1.0;
    double step = 1.0 / (12.0 * lam);
    for (int it = 0; it < iters; ++it) {
#pragma omp parallel for schedule(static)
        for (long idx = 0; idx < n; ++idx) {
            int k = (int)(idx / plane);
            long rem = idx % plane;
            int i = (int)(rem / width), j = (int)(rem % width);
            double o = 0.0;
            if (i < height - 1) o -= r[idx];
            if (i > 0) o += r[idx - width];
            if (j < width - 1) o -= s[idx];
            if (j > 0) o += s[idx - 1];
            if (k < depth - 1) o -= o3[idx];
            if (k > 0) o += o3[idx - plane];
            double uu = image[idx] - lam * o;
            if (nonneg) uu = (uu < 0.0) ? 0.0 : uu;
            u[idx] = uu;
        }
        double t_next = (1.0 + sqrt(1.0 + 4.0 * t * t)) / 2.0;
        double beta = (t - 1.0) / t_next;
#pragma omp parallel for schedule(static)
        for (long idx = 0; idx < n; ++idx) {
            int k = (int)(idx / plane);
            long rem = idx % plane;
            int i = (int)(rem / width), j = (int)(rem % width);
            double gv = (i < height - 1) ? u[idx + width] - u[idx] : 0.0;
            double gh = (j < width - 1) ? u[idx + 1] - u[idx] : 0.0;
            double gz = (k < depth - 1) ? u[idx + plane] - u[idx] : 0.0;
            double ph = r[idx] + step * gv;
            double qh = s[idx] + step * gh;
            double wh = o3[idx] + step * gz;
            double nrm = sqrt(ph * ph + qh * qh + wh * wh);
            double scale = (nrm > 1.0 || nrm != nrm) ? nrm : 1.0;
            double pn = ph / scale, qn = qh / scale, wn = wh / scale;
            r[idx] = pn + beta * (pn - pp[idx]);
            s[idx] = qn + beta * (qn - qp[idx]);
            o3[idx] = wn + beta * (wn - wp[idx]);
            pp[idx] = pn;
            qp[idx] = qn;
            wp[idx] = wn;
        }
        t = t_next;
    }
#pragma omp parallel for schedule(static)
    for (long idx = 0; idx < n; ++idx) {
        int k = (int)(idx / plane);
        long rem = idx % plane;
        int i = (int)(rem / width), j = (int)(rem % width);
        double o = 0.0;
        if (i < height - 1) o -= pp[idx];
        if (i > 0) o += pp[idx - width];
        if (j < width - 1) o -= qp[idx];
        if (j > 0) o += qp[idx - 1];
        if (k < depth - 1) o -= wp[idx];
        if (k > 0) o += wp[idx - plane];
        double v = image[idx] - lam * o;
        if (nonneg) v = (v < 0.0) ? 0.0 : v;
        out[idx] = v;
    }
    if (iters > 0) {
        memcpy(p, pp, sizeof(double) * n);
        memcpy(q, qp, sizeof(double) * n);
        memcpy(w, wp, sizeof(double) * n);
    }
    free(r); free(s); free(o3); free(pp); free(qp); free(wp); free(u);
}

/* ---------------------------------------------------------------------- */
/* "fast" variants for the timed CPU baseline: the same operator with the  */
/* per-angle constants hoisted (pos = a0 + b*sigma + step*m, no divisions  */
/* per sample; the adjoint gathers the two bins around the crossing with   */
/* the hat weight).  Algebraically identical to the exact variants above;  */
/* tests pin them to <= 1e-12 relative against the reference.              */
/* ---------------------------------------------------------------------- */
typedef struct {
    int branch_rows;
    double sigma, m, a0, step_len;
} fast_par;

static fast_par fast_params(double theta, int height, int width, int n_bins, double ds, double h)
{
    fast_par f;
    double c = cos(theta), s = sin(theta);
    double cB = (n_bins - 1) / 2.0, cH = (height - 1) / 2.0, cW = (width - 1) / 2.0;
    if (fabs(c) >= fabs(s)) {
        f.branch_rows = 1;
        f.sigma = ds / (h * c);
        f.m = -(s / c);
        f.a0 = -cB * f.sigma + cH * (s / c) + cW;
        f.step_len = h / fabs(c);
    } else {
        f.branch_rows = 0;
        f.sigma = ds / (h * s);
        f.m = -(c / s);
        f.a0 = -cB * f.sigma + cW * (c / s) + cH;
        f.step_len = h / fabs(s);
    }
    return f;
}

void oracle_forward_fast(int height, int width, int n_bins, double ds, double h, int n_sel,
                         const double* thetas, int n_slices, const double* x, double* y)
{
    fast_par* fp = (fast_par*)malloc(sizeof(fast_par) * (n_sel > 0 ? n_sel : 1));
    for (int k = 0; k < n_sel; ++k) fp[k] = fast_params(thetas[k], height, width, n_bins, ds, h);
    long total = (long)n_slices * n_sel * n_bins;
#pragma omp parallel for schedule(static)
    for (long idx = 0; idx < total; ++idx) {
        int b = (int)(idx % n_bins);
        long t = idx / n_bins;
        int k = (int)(t % n_sel);
        int z = (int)(t / n_sel);
        const fast_par* f = &fp[k];
        const double* img = x + (long)z * height * width;
        int n_steps = f->branch_rows ? height : width;
        int n_lanes = f->branch_rows ? width : height;
        long lstride = f->branch_rows ? 1 : width, sstride = f->branch_rows ? width : 1;
        double p0 = f->a0 + b * f->sigma;
        double acc = 0.0;
        for (int st = 0; st < n_steps; ++st) {
            double pos = p0 + st * f->m;
            double fl = floor(pos);
            long l0 = (long)fl;
            double fr = pos - fl;
            if (l0 >= 0 && l0 < n_lanes) acc += (1.0 - fr) * img[st * sstride + l0 * lstride];
            if (l0 + 1 >= 0 && l0 + 1 < n_lanes) acc += fr * img[st * sstride + (l0 + 1) * lstride];
        }
        y[idx] = acc * f->step_len;
    }
    free(fp);
}

void oracle_adjoint_fast(int height, int width, int n_bins, double ds, double h, int n_sel,
                         const double* thetas, int n_slices, const double* y, double* x)
{
    fast_par* fp = (fast_par*)malloc(sizeof(fast_par) * (n_sel > 0 ? n_sel : 1));
    for (int k = 0; k < n_sel; ++k) fp[k] = fast_params(thetas[k], height, width, n_bins, ds, h);
    long total = (long)n_slices * height * width;
#pragma omp parallel for schedule(static)
    for (long idx = 0; idx < total; ++idx) {
        int c = (int)(idx % width);
        long t = idx / width;
        int r = (int)(t % height);
        int z = (int)(t / height);
        const double* sino = y + (long)z * n_sel * n_bins;
        double acc = 0.0;
        for (int k = 0; k < n_sel; ++k) {
            const fast_par* f = &fp[k];
            int step = f->branch_rows ? r : c;
            int lane = f->branch_rows ? c : r;
            double bf = (lane - f->a0 - step * f->m) / f->sigma; /* pos(bf) == lane */
            double as = fabs(f->sigma);
            int half = (int)ceil(1.0 / as);
            long b0 = (long)floor(bf);
            double part = 0.0;
            for (long b = b0 - half + 1; b <= b0 + half; ++b) {
                if (b < 0 || b >= n_bins) continue;
                double w = 1.0 - as * fabs((double)b - bf);
                if (w > 0.0) part += w * sino[(long)k * n_bins + b];
            }
            acc += part * f->step_len;
        }
        x[idx] = acc;
    }
    free(fp);
}
