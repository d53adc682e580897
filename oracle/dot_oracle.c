/*
 * dot_oracle.c -- CPU parity ORACLE for the DOT render / backward path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is a plain-C restatement of the
 * reference's Numba kernels (/root/reference/pkg/src/octrf/_kernels.py) and is
 * used exclusively as the checker by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py.  The product path
 * (paper_2307_15333_b200/) never links or calls it.
 *
 * Parity pin: tests/test_oracle_golden.py checks every entry point against
 * golden vectors produced by the reference itself (tests/golden/make_golden.py).
 *
 * Numerics follow the reference exactly: float64 geometry and accumulation,
 * float32 payloads widened on read, NO fused multiply-add (build with
 * -ffp-contract=off; Numba compiles these kernels with fastmath=False), IEEE
 * division, glibc exp().  Parallel loops are per-ray and write disjoint
 * slices, the per-leaf reduction is serial in ray-major order -- exactly the
 * reference's determinism model (_kernels.py:1-8).
 *
 * Tree layout is the reference's pool layout (octree.py:94-102):
 *   child  int64[cap][8], leaf uint8[cap], center f64[cap][3], depth i32[cap],
 *   half_tab f64[max_depth+1]; sigma f32[cap]; sh f32[cap][3B] channel-major.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define NUDGE_REL 2e-12 /* _kernels.py:16 */
#define SH_C0 0.28209479177387814
#define SH_C1 0.4886025119029199

/* _kernels.py:22-27 */
static inline double sigmoid(double x) {
    if (x >= 0.0) return 1.0 / (1.0 + exp(-x));
    double e = exp(x);
    return e / (1.0 + e);
}

/* _kernels.py:30-53 (svox / 3DGS sign convention) */
static void eval_basis(int degree, double x, double y, double z, double* out) {
    out[0] = SH_C0;
    if (degree >= 1) {
        out[1] = -SH_C1 * y;
        out[2] = SH_C1 * z;
        out[3] = -SH_C1 * x;
    }
    if (degree >= 2) {
        double xx = x * x, yy = y * y, zz = z * z;
        out[4] = 1.0925484305920792 * x * y;
        out[5] = -1.0925484305920792 * y * z;
        out[6] = 0.31539156525252005 * (2.0 * zz - xx - yy);
        out[7] = -1.0925484305920792 * x * z;
        out[8] = 0.5462742152960396 * (xx - yy);
        if (degree >= 3) {
            out[9] = -0.5900435899266435 * y * (3.0 * xx - yy);
            out[10] = 2.890611442640554 * x * y * z;
            out[11] = -0.4570457994644658 * y * (4.0 * zz - xx - yy);
            out[12] = 0.3731763325901154 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
            out[13] = -0.4570457994644658 * x * (4.0 * zz - xx - yy);
            out[14] = 1.445305721320277 * z * (xx - yy);
            out[15] = -0.5900435899266435 * x * (xx - 3.0 * yy);
        }
    }
}

static int degree_for_basis(int b) { return b == 1 ? 0 : b == 4 ? 1 : b == 9 ? 2 : 3; }

/* _kernels.py:56-68: root-to-leaf point location, ties to the upper octant. */
static inline int64_t descend(const int64_t* child, const uint8_t* leaf,
                              const double* center, double px, double py, double pz) {
    int64_t node = 0;
    while (leaf[node] == 0) {
        int o = 0;
        if (px >= center[node * 3 + 0]) o |= 1;
        if (py >= center[node * 3 + 1]) o |= 2;
        if (pz >= center[node * 3 + 2]) o |= 4;
        node = child[node * 8 + o];
    }
    return node;
}

/* _kernels.py:71-158: exact per-leaf segmentation of one ray. */
static int64_t trace_ray(const int64_t* child, const uint8_t* leaf, const double* center,
                         const int32_t* depth, const double* half_tab,
                         double ox, double oy, double oz, double dx, double dy, double dz,
                         double t_near, double t_far,
                         int64_t* seg_leaf, double* seg_t, double* seg_delta, int store) {
    double root_half = half_tab[0];
    double t0 = t_near, t1 = t_far;
    for (int axis = 0; axis < 3; ++axis) {
        double o = axis == 0 ? ox : axis == 1 ? oy : oz;
        double d = axis == 0 ? dx : axis == 1 ? dy : dz;
        double c = center[axis];
        double lo = c - root_half, hi = c + root_half;
        if (d != 0.0) {
            double ta = (lo - o) / d, tb = (hi - o) / d;
            if (ta > tb) { double tmp = ta; ta = tb; tb = tmp; }
            if (ta > t0) t0 = ta;
            if (tb < t1) t1 = tb;
        } else if (o < lo || o >= hi) {
            return 0;
        }
    }
    if (t1 <= t0) return 0;
    double nudge0 = root_half * NUDGE_REL, nudge = nudge0, t = t0;
    int64_t n = 0;
    for (;;) {
        double probe = t + nudge;
        if (probe >= t1) break;
        double px = ox + probe * dx, py = oy + probe * dy, pz = oz + probe * dz;
        int64_t node = descend(child, leaf, center, px, py, pz);
        double h = half_tab[depth[node]];
        double tex = t1, cand;
        const double* c = center + node * 3;
        if (dx > 0.0) { cand = (c[0] + h - ox) / dx; if (cand < tex) tex = cand; }
        else if (dx < 0.0) { cand = (c[0] - h - ox) / dx; if (cand < tex) tex = cand; }
        if (dy > 0.0) { cand = (c[1] + h - oy) / dy; if (cand < tex) tex = cand; }
        else if (dy < 0.0) { cand = (c[1] - h - oy) / dy; if (cand < tex) tex = cand; }
        if (dz > 0.0) { cand = (c[2] + h - oz) / dz; if (cand < tex) tex = cand; }
        else if (dz < 0.0) { cand = (c[2] - h - oz) / dz; if (cand < tex) tex = cand; }
        if (tex <= probe) { nudge *= 4.0; continue; }
        if (store) { seg_leaf[n] = node; seg_t[n] = t; seg_delta[n] = tex - t; }
        ++n;
        t = tex;
        nudge = nudge0;
    }
    return n;
}

/* _kernels.py:161-170 */
void oracle_count_segments(const int64_t* child, const uint8_t* leaf, const double* center,
                           const int32_t* depth, const double* half_tab,
                           const double* origins, const double* dirs, int64_t n_rays,
                           double t_near, double t_far, int64_t* counts) {
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t r = 0; r < n_rays; ++r) {
        const double* o = origins + 3 * r;
        const double* d = dirs + 3 * r;
        counts[r] = trace_ray(child, leaf, center, depth, half_tab, o[0], o[1], o[2],
                              d[0], d[1], d[2], t_near, t_far, 0, 0, 0, 0);
    }
}

/* _kernels.py:173-182 */
void oracle_fill_segments(const int64_t* child, const uint8_t* leaf, const double* center,
                          const int32_t* depth, const double* half_tab,
                          const double* origins, const double* dirs, int64_t n_rays,
                          double t_near, double t_far, const int64_t* offsets,
                          int64_t* seg_leaf, double* seg_t, double* seg_delta) {
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t r = 0; r < n_rays; ++r) {
        const double* o = origins + 3 * r;
        const double* d = dirs + 3 * r;
        int64_t b = offsets[r];
        trace_ray(child, leaf, center, depth, half_tab, o[0], o[1], o[2], d[0], d[1], d[2],
                  t_near, t_far, seg_leaf + b, seg_t + b, seg_delta + b, 1);
    }
}

/* _kernels.py:185-224 */
void oracle_composite(const float* sigma, const float* sh, int64_t sh_stride, int basis_count,
                      const double* dirs, int64_t n_rays, const int64_t* offsets,
                      const int64_t* seg_leaf, const double* seg_delta, const double* bg,
                      double eps_t, double* rgb_out, double* tfin_out, double* wsum_out) {
    int degree = degree_for_basis(basis_count);
    int B = basis_count;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t r = 0; r < n_rays; ++r) {
        double basis[16];
        eval_basis(degree, dirs[3 * r], dirs[3 * r + 1], dirs[3 * r + 2], basis);
        double trans = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0, wsum = 0.0;
        for (int64_t s = offsets[r]; s < offsets[r + 1]; ++s) {
            int64_t node = seg_leaf[s];
            double sg = (double)sigma[node];
            double a = exp(-sg * seg_delta[s]);
            double q = 1.0 - a;
            if (q > 0.0) {
                const float* row = sh + node * sh_stride;
                double e0 = 0.0, e1 = 0.0, e2 = 0.0;
                for (int b = 0; b < B; ++b) {
                    double bb = basis[b];
                    e0 += (double)row[b] * bb;
                    e1 += (double)row[B + b] * bb;
                    e2 += (double)row[2 * B + b] * bb;
                }
                double tq = trans * q;
                c0 += tq * sigmoid(e0);
                c1 += tq * sigmoid(e1);
                c2 += tq * sigmoid(e2);
                wsum += tq;
            }
            trans *= a;
            if (eps_t > 0.0 && trans < eps_t) break;
        }
        wsum += trans;
        rgb_out[3 * r + 0] = c0 + trans * bg[0];
        rgb_out[3 * r + 1] = c1 + trans * bg[1];
        rgb_out[3 * r + 2] = c2 + trans * bg[2];
        tfin_out[r] = trans;
        wsum_out[r] = wsum;
    }
}

/* _kernels.py:227-324: forward with saves, then reverse sweep. */
void oracle_grad(const float* sigma, const float* sh, int64_t sh_stride, int basis_count,
                 const double* dirs, const double* targets, int64_t n_rays,
                 const int64_t* offsets, const int64_t* seg_leaf, const double* seg_delta,
                 const double* bg, double eps_t, double grad_scale,
                 double* seg_q, double* seg_dsig, double* seg_w, double* seg_trans,
                 double* seg_col, double* basis_out, double* rgb_out, double* tfin_out,
                 double* wsum_out, double* loss_out) {
    int degree = degree_for_basis(basis_count);
    int B = basis_count;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t r = 0; r < n_rays; ++r) {
        int64_t lo = offsets[r], hi = offsets[r + 1];
        double* basis = basis_out + r * B;
        eval_basis(degree, dirs[3 * r], dirs[3 * r + 1], dirs[3 * r + 2], basis);
        double trans = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0, wsum = 0.0;
        int64_t used = hi - lo;
        for (int64_t i = 0; i < hi - lo; ++i) {
            int64_t s = lo + i;
            int64_t node = seg_leaf[s];
            double sg = (double)sigma[node];
            double a = exp(-sg * seg_delta[s]);
            double q = 1.0 - a;
            const float* row = sh + node * sh_stride;
            double e0 = 0.0, e1 = 0.0, e2 = 0.0;
            for (int b = 0; b < B; ++b) {
                double bb = basis[b];
                e0 += (double)row[b] * bb;
                e1 += (double)row[B + b] * bb;
                e2 += (double)row[2 * B + b] * bb;
            }
            double col0 = sigmoid(e0), col1 = sigmoid(e1), col2 = sigmoid(e2);
            seg_trans[s] = trans;
            seg_q[s] = q;
            seg_col[3 * s + 0] = col0;
            seg_col[3 * s + 1] = col1;
            seg_col[3 * s + 2] = col2;
            double tq = trans * q;
            c0 += tq * col0;
            c1 += tq * col1;
            c2 += tq * col2;
            wsum += tq;
            trans *= a;
            if (eps_t > 0.0 && trans < eps_t) { used = i + 1; break; }
        }
        for (int64_t i = used; i < hi - lo; ++i) {
            int64_t s = lo + i;
            seg_q[s] = 0.0;
            seg_dsig[s] = 0.0;
            seg_w[3 * s + 0] = 0.0;
            seg_w[3 * s + 1] = 0.0;
            seg_w[3 * s + 2] = 0.0;
        }
        double tfin = trans;
        wsum += tfin;
        c0 += tfin * bg[0];
        c1 += tfin * bg[1];
        c2 += tfin * bg[2];
        rgb_out[3 * r + 0] = c0;
        rgb_out[3 * r + 1] = c1;
        rgb_out[3 * r + 2] = c2;
        tfin_out[r] = tfin;
        wsum_out[r] = wsum;
        double r0 = c0 - targets[3 * r + 0];
        double r1 = c1 - targets[3 * r + 1];
        double r2 = c2 - targets[3 * r + 2];
        loss_out[r] = r0 * r0 + r1 * r1 + r2 * r2;
        double g0 = grad_scale * r0, g1 = grad_scale * r1, g2 = grad_scale * r2;
        double suf0 = tfin * bg[0], suf1 = tfin * bg[1], suf2 = tfin * bg[2];
        for (int64_t i = used - 1; i >= 0; --i) {
            int64_t s = lo + i;
            double ti = seg_trans[s];
            double q = seg_q[s];
            double a = 1.0 - q;
            double col0 = seg_col[3 * s + 0], col1 = seg_col[3 * s + 1], col2 = seg_col[3 * s + 2];
            double tnext = ti * a;
            seg_dsig[s] = seg_delta[s] * (g0 * (tnext * col0 - suf0)
                                          + g1 * (tnext * col1 - suf1)
                                          + g2 * (tnext * col2 - suf2));
            double tq = ti * q;
            suf0 += tq * col0;
            suf1 += tq * col1;
            suf2 += tq * col2;
            seg_w[3 * s + 0] = g0 * tq * col0 * (1.0 - col0);
            seg_w[3 * s + 1] = g1 * tq * col1 * (1.0 - col1);
            seg_w[3 * s + 2] = g2 * tq * col2 * (1.0 - col2);
        }
    }
}

/* _kernels.py:327-346: serial per-leaf reduction in global segment order. */
void oracle_scatter(const int64_t* offsets, int64_t n_rays, const int64_t* seg_leaf,
                    const double* seg_q, const double* seg_dsig, const double* seg_w,
                    const double* basis_out, int basis_count, int64_t gsh_stride,
                    double* grad_sigma, double* grad_sh, double* signal, uint8_t* touched) {
    int B = basis_count;
    for (int64_t r = 0; r < n_rays; ++r) {
        for (int64_t s = offsets[r]; s < offsets[r + 1]; ++s) {
            int64_t node = seg_leaf[s];
            touched[node] = 1;
            grad_sigma[node] += seg_dsig[s];
            signal[node] += seg_q[s];
            double w0 = seg_w[3 * s], w1 = seg_w[3 * s + 1], w2 = seg_w[3 * s + 2];
            if (w0 != 0.0 || w1 != 0.0 || w2 != 0.0) {
                double* g = grad_sh + node * gsh_stride;
                for (int b = 0; b < B; ++b) {
                    double bb = basis_out[r * B + b];
                    g[b] += w0 * bb;
                    g[B + b] += w1 * bb;
                    g[2 * B + b] += w2 * bb;
                }
            }
        }
    }
}

/* North-star extras with no reference counterpart, DEFINED here on the
 * reference's own segment lists (render.py:105-124) and compositing order
 * (_kernels.py:189-224): per ray the expected termination depth
 * sum_i T_i Q_i (t_i + delta_i / 2); per leaf the sum and the max over
 * composited (pre-cut, crossing segment included) segments of the
 * compositing weight T_i Q_i.  Serial in ray-major order (like the scatter).
 * Any output may be NULL. */
void oracle_weights(const float* sigma, const int64_t* offsets, int64_t n_rays, const int64_t* seg_leaf,
                    const double* seg_t, const double* seg_delta, double eps, double* depth,
                    double* weight_sum, double* weight_max) {
    for (int64_t r = 0; r < n_rays; ++r) {
        double trans = 1.0, dep = 0.0;
        for (int64_t s = offsets[r]; s < offsets[r + 1]; ++s) {
            double a = exp(-(double)sigma[seg_leaf[s]] * seg_delta[s]);
            double q = 1.0 - a;
            double w = trans * q;
            if (q > 0.0) {
                dep += w * (seg_t[s] + 0.5 * seg_delta[s]);
                if (weight_sum) weight_sum[seg_leaf[s]] += w;
                if (weight_max && w > weight_max[seg_leaf[s]]) weight_max[seg_leaf[s]] = w;
            }
            trans *= a;
            if (eps > 0.0 && trans < eps) break;
        }
        if (depth) depth[r] = dep;
    }
}

/* Thread count of the OpenMP loops (the CPU baseline's 1-thread figure). */
void oracle_set_threads(int n) {
#ifdef _OPENMP
    extern void omp_set_num_threads(int);
    omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* glibc exp over an array (the reference's exp: Numba lowers np.exp to the
 * libm call).  Checker for the kernels' exp_ref. */
void oracle_exp(const double* x, double* y, int64_t n) {
    for (int64_t i = 0; i < n; ++i) y[i] = exp(x[i]);
}
