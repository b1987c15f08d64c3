/*
 * srwcr_oracle.c -- plain, slow, fp64 CPU oracle for the spatially region-weighted
 * correlation ratio (SRWCR) and its analytic gradient, arXiv 1804.05061
 * (Gong et al., "Non-rigid image registration using spatially region-weighted
 * correlation ratio and GPU-acceleration").  Citations "P:NNN" are lines of the
 * paper text; readings where the paper is silent or garbled are the
 * numbered items c1..c18 of SURVEY.md section 8(c), restated in DESIGN.md section 3.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the correctness reference for the CUDA
 * path.  Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * --impl reference) may load it.  It shares no code, header, table or constant
 * generator with paper_1804_05061_b200/ (the product), and neither includes the
 * other.
 *
 * Two routes, both fp64, both in this file so each checks the other:
 *   (1) LITERAL route -- the paper's definition as written: the dense 3-D joint
 *       histogram of Eq 3 with the Parzen window of Eq 5 and the
 *       B-spline spatial weight of Eq 7; marginals Eq 4; regional
 *       statistics Eq 10; the value by the loops of Table I
 *       (P:149-172); dD/dM(y) by Eq 27 as printed; the chain rule of
 *       Eq 16 with the Jacobian of Eq 17.
 * Both routes take the orientation: the moving image as the
 * estimated image B (0) or as the model image A (1, Eq 20-21, App. II).
 *   (2) MOMENT route -- the exact algebraic rewrite of SURVEY.md Appendix A
 *       (weighted counts N, Parzen moments S, Q per region and fixed bin), the
 *       combine of SURVEY 8(a) a7 and the per-voxel derivative a8.
 *   (3) the bending energy C_p of Eq 1 (reading c19), per
 *       voxel from B-spline second-derivative tensor products.
 *
 * Geometry (SURVEY 8 "Conventions", readings c14-c16):
 *   volumes x-fastest [Nz][Ny][Nx]; Nz == 1 means 2-D.
 *   control lattice spacing delta (voxels, fp64); nodes per axis
 *       G = floor((N-1)/delta) + 4; voxel i has taps floor(i/delta) + {0,1,2,3}
 *       with weights beta_l(t), t = i/delta - floor(i/delta)   (Eq 17, shifted +1)
 *   spatial lattice: k cells per axis, Delta = N/k (fp64 division), K = k+3
 *       regions per axis, taps floor(i/Delta) + {0..3} (Eq 7).  k = 0 (and the
 *       z axis in 2-D) is a degenerate axis: K = 4 regions, base 0, weights
 *       (1,0,0,0); regions 1..3 on that axis carry zero mass.
 *   params: displacements in voxels, SoA [ndim][Gz][Gy][Gx] (Gz = 1 in 2-D).
 * Rounding: compile with -ffp-contract=off.  All arithmetic fp64, except that
 * normalized intensities are rounded to fp32 exactly as stated in c1 of DESIGN.md.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int64_t n[3];       /* Nx, Ny, Nz */
    int32_t L;          /* maximal intensity bin L_eps; bins 0..L */
    int32_t nthreads;   /* OpenMP threads (<= 0: library default) */
    double  delta[3];   /* control-lattice spacing in voxels */
    int64_t kcells[3];  /* spatial cells per axis (0: degenerate axis) */
    double  eps_mass;   /* region retained iff N_r/Z > eps_mass   (reading c12) */
    double  eps_sigma;  /* ... and sigma_r^2 > eps_sigma (bin^2)  (reading c12) */
    int32_t orientation;/* 0: moving image is the estimated image B (Eq 18-19);
                           1: moving image is the model image A (Eq 20-21, App. II) */
} orc_cfg;

/* ------------------------------------------------------------------ geometry */

static int ndim_of(const orc_cfg *c) { return c->n[2] == 1 ? 2 : 3; }

static int axis_degenerate_spatial(const orc_cfg *c, int ax) {
    return c->kcells[ax] <= 0 || (ax == 2 && c->n[2] == 1);
}

/* nodes per axis of the control lattice, regions per axis of the spatial lattice */
void orc_derived(const orc_cfg *c, int64_t G[3], int64_t K[3]) {
    for (int ax = 0; ax < 3; ++ax) {
        if (ax == 2 && c->n[2] == 1) G[ax] = 1;
        else G[ax] = (int64_t)floor((double)(c->n[ax] - 1) / c->delta[ax]) + 4;
        K[ax] = axis_degenerate_spatial(c, ax) ? 4 : c->kcells[ax] + 3;
    }
}

/* Eq 8: cubic B-spline pieces beta_0..beta_3 at t in [0,1). */
void orc_beta(double t, double w[4]) {
    w[0] = (1.0 - t) * (1.0 - t) * (1.0 - t) / 6.0;
    w[1] = (3.0 * t * t * t - 6.0 * t * t + 4.0) / 6.0;
    w[2] = (-3.0 * t * t * t + 3.0 * t * t + 3.0 * t + 1.0) / 6.0;
    w[3] = t * t * t / 6.0;
}

/* taps of voxel index i on a lattice of the given spacing (Eq 17 indices) */
void orc_taps(int64_t i, double spacing, int degenerate, int64_t *base, double w[4]) {
    if (degenerate) {
        *base = 0; w[0] = 1.0; w[1] = 0.0; w[2] = 0.0; w[3] = 0.0;
        return;
    }
    double s = (double)i / spacing;
    double fl = floor(s);
    *base = (int64_t)fl;
    orc_beta(s - fl, w);
}

static void ctrl_taps(const orc_cfg *c, int ax, int64_t i, int64_t *b, double w[4]) {
    orc_taps(i, c->delta[ax], ax == 2 && c->n[2] == 1, b, w);
}
static void spat_taps(const orc_cfg *c, int ax, int64_t i, int64_t *b, double w[4]) {
    int deg = axis_degenerate_spatial(c, ax);
    double Delta = deg ? 1.0 : (double)c->n[ax] / (double)c->kcells[ax];
    orc_taps(i, Delta, deg, b, w);
}

/* ------------------------------------------------------- normalization */

/* v' = (float)(((double)v - lo) * ((double)L / (hi - lo))), clamped to [0, L];
 * lo/hi = volume min/max; a constant volume maps to 0.  (reading c1 / S:51-59) */
void orc_normalize(const float *v, int64_t n, int32_t L, float *out) {
    double lo = INFINITY, hi = -INFINITY;
    for (int64_t i = 0; i < n; ++i) {
        double x = (double)v[i];
        if (x < lo) lo = x;
        if (x > hi) hi = x;
    }
    if (!(hi > lo)) {
        for (int64_t i = 0; i < n; ++i) out[i] = 0.0f;
        return;
    }
    double scale = (double)L / (hi - lo);
    for (int64_t i = 0; i < n; ++i) {
        float f = (float)(((double)v[i] - lo) * scale);
        if (f < 0.0f) f = 0.0f;
        if (f > (float)L) f = (float)L;
        out[i] = f;
    }
}

/* ------------------------------------------------------------ Parzen (Eq 5) */

/* h(t), Eq 5 */
double orc_parzen(double t) {
    double a = fabs(t);
    if (a < 0.5) return -1.8 * a * a - 0.1 * a + 1.0;
    if (a < 1.0) return 1.8 * a * a - 3.7 * a + 1.9;
    return 0.0;
}

/* h'(t) = dh/dt.  At the kinks t in {0, -1, +1} (h is C0 there) the two-sided
 * average is used: h'(0) = 0, h'(+-1) = -+0.05 (reading c4). */
double orc_parzen_deriv(double t) {
    double a = fabs(t), s = t < 0.0 ? -1.0 : 1.0;
    if (t == 0.0) return 0.0;
    if (a < 0.5) return s * (-3.6 * a - 0.1);
    if (a < 1.0) return s * (3.6 * a - 3.7);
    if (a == 1.0) return s * -0.05;
    return 0.0;
}

/* ------------------------------------------------ FFD transform (Eq 17) */

static inline int64_t node_index(const int64_t G[3], int64_t gx, int64_t gy, int64_t gz) {
    return (gz * G[1] + gy) * G[0] + gx;
}

/* u(x) = sum over the 4x4x4 supporting nodes of beta_l beta_m beta_n phi */
void orc_displacement(const orc_cfg *c, const double *params, int64_t x, int64_t y, int64_t z,
                      double u[3]) {
    int64_t G[3], K[3];
    orc_derived(c, G, K);
    int nd = ndim_of(c);
    int64_t nodes = G[0] * G[1] * G[2];
    int64_t bx, by, bz;
    double wx[4], wy[4], wz[4];
    ctrl_taps(c, 0, x, &bx, wx);
    ctrl_taps(c, 1, y, &by, wy);
    ctrl_taps(c, 2, z, &bz, wz);
    u[0] = u[1] = u[2] = 0.0;
    for (int n = 0; n < 4; ++n) {
        if (wz[n] == 0.0) continue;
        for (int m = 0; m < 4; ++m) {
            if (wy[m] == 0.0) continue;
            for (int l = 0; l < 4; ++l) {
                if (wx[l] == 0.0) continue;
                double w = wx[l] * wy[m] * wz[n];
                int64_t s = node_index(G, bx + l, by + m, bz + n);
                for (int comp = 0; comp < nd; ++comp) u[comp] += w * params[comp * nodes + s];
            }
        }
    }
}

/* --------------------------------------- backward warping + trilinear */

/* m = M^(T(x)) by trilinear interpolation (reading c1), sample position clamped
 * per axis to [0, N-1] (c2); cell = min(floor(y), N-2); grad = analytic gradient
 * of the interpolant, 0 along clamped axes (c3).  Nz == 1: bilinear. */
void orc_sample(const orc_cfg *c, const float *M, const double yin[3], double *m, double g[3]) {
    int64_t cell[3];
    double t[3];
    int clamped[3];
    for (int ax = 0; ax < 3; ++ax) {
        double N1 = (double)(c->n[ax] - 1);
        double y = yin[ax];
        clamped[ax] = (y < 0.0 || y > N1);
        if (y < 0.0) y = 0.0;
        if (y > N1) y = N1;
        if (c->n[ax] == 1) { cell[ax] = 0; t[ax] = 0.0; continue; }
        int64_t fl = (int64_t)floor(y);
        if (fl > c->n[ax] - 2) fl = c->n[ax] - 2;
        cell[ax] = fl;
        t[ax] = y - (double)fl;
    }
    int64_t nx = c->n[0], nxy = c->n[0] * c->n[1];
    int64_t dx = c->n[0] > 1 ? 1 : 0, dy = c->n[1] > 1 ? nx : 0, dz = c->n[2] > 1 ? nxy : 0;
    const float *b = M + cell[2] * nxy + cell[1] * nx + cell[0];
    double c000 = b[0], c100 = b[dx], c010 = b[dy], c110 = b[dy + dx];
    double c001 = b[dz], c101 = b[dz + dx], c011 = b[dz + dy], c111 = b[dz + dy + dx];
    double tx = t[0], ty = t[1], tz = t[2];
    /* nested lerps a + t (b - a) */
    double e00 = c000 + tx * (c100 - c000), e10 = c010 + tx * (c110 - c010);
    double e01 = c001 + tx * (c101 - c001), e11 = c011 + tx * (c111 - c011);
    double f0 = e00 + ty * (e10 - e00), f1 = e01 + ty * (e11 - e01);
    *m = f0 + tz * (f1 - f0);
    /* partial derivatives of the trilinear polynomial w.r.t. the sample position */
    double gx = (1 - ty) * (1 - tz) * (c100 - c000) + ty * (1 - tz) * (c110 - c010) +
                (1 - ty) * tz * (c101 - c001) + ty * tz * (c111 - c011);
    double gy = (1 - tx) * (1 - tz) * (c010 - c000) + tx * (1 - tz) * (c110 - c100) +
                (1 - tx) * tz * (c011 - c001) + tx * tz * (c111 - c101);
    double gz = (1 - tx) * (1 - ty) * (c001 - c000) + tx * (1 - ty) * (c101 - c100) +
                (1 - tx) * ty * (c011 - c010) + tx * ty * (c111 - c110);
    g[0] = (clamped[0] || c->n[0] == 1) ? 0.0 : gx;
    g[1] = (clamped[1] || c->n[1] == 1) ? 0.0 : gy;
    g[2] = (clamped[2] || c->n[2] == 1) ? 0.0 : gz;
}

/* T(x) then sample: per voxel of z-slab [z0, z1): m and its spatial gradient */
void orc_warp(const orc_cfg *c, const float *M, const double *params, int64_t z0, int64_t z1,
              double *m_out, double *g_out) {
    int64_t nx = c->n[0], ny = c->n[1];
    for (int64_t z = z0; z < z1; ++z)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t x = 0; x < nx; ++x) {
                double u[3], p[3], m, g[3];
                orc_displacement(c, params, x, y, z, u);
                p[0] = (double)x + u[0]; p[1] = (double)y + u[1]; p[2] = (double)z + u[2];
                orc_sample(c, M, p, &m, g);
                int64_t i = ((z - z0) * ny + y) * nx + x;
                m_out[i] = m;
                if (g_out) { g_out[3 * i] = g[0]; g_out[3 * i + 1] = g[1]; g_out[3 * i + 2] = g[2]; }
            }
}

static int nthreads_of(const orc_cfg *c) {
#ifdef _OPENMP
    return c->nthreads > 0 ? c->nthreads : omp_get_max_threads();
#else
    (void)c;
    return 1;
#endif
}

/* ===================================================== (1) LITERAL route === */

/* Eq 3 without the 1/Z factor: P[r][a][b] = sum_x w(r,x) h(a-A(x)) h(b-B(x)) with
 * (A, B) = (F, M(T(x))) in orientation 0 and (M(T(x)), F) in orientation 1,
 * accumulated over the voxels of z-slab [z0, z1).  Dense (L+1)^2 table per region.
 * OpenMP over z with per-thread tables merged in thread order. */
void orc_joint_hist(const orc_cfg *c, const float *F, const float *M, const double *params,
                    int64_t z0, int64_t z1, double *P) {
    int64_t G[3], K[3];
    orc_derived(c, G, K);
    int L = c->L, B = L + 1;
    int64_t R = K[0] * K[1] * K[2], tab = R * B * B;
    int nt = nthreads_of(c);
    double *priv = (double *)calloc((size_t)nt * (size_t)tab, sizeof(double));
    int64_t nx = c->n[0], ny = c->n[1];
#pragma omp parallel num_threads(nt)
    {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        double *T = priv + (size_t)tid * (size_t)tab;
        double *ha = (double *)malloc(sizeof(double) * B), *hb = (double *)malloc(sizeof(double) * B);
#pragma omp for schedule(static)
        for (int64_t z = z0; z < z1; ++z)
            for (int64_t y = 0; y < ny; ++y)
                for (int64_t x = 0; x < nx; ++x) {
                    double u[3], p[3], m, g[3];
                    orc_displacement(c, params, x, y, z, u);
                    p[0] = (double)x + u[0]; p[1] = (double)y + u[1]; p[2] = (double)z + u[2];
                    orc_sample(c, M, p, &m, g);
                    double f = (double)F[(z * ny + y) * nx + x];
                    /* a: model image A, b: estimated image B */
                    const double va = c->orientation ? m : f, vb = c->orientation ? f : m;
                    for (int a = 0; a < B; ++a) ha[a] = orc_parzen((double)a - va);
                    for (int b = 0; b < B; ++b) hb[b] = orc_parzen((double)b - vb);
                    int64_t sbx, sby, sbz;
                    double wx[4], wy[4], wz[4];
                    spat_taps(c, 0, x, &sbx, wx);
                    spat_taps(c, 1, y, &sby, wy);
                    spat_taps(c, 2, z, &sbz, wz);
                    for (int n = 0; n < 4; ++n)
                        for (int mm = 0; mm < 4; ++mm)
                            for (int l = 0; l < 4; ++l) {
                                double w = wx[l] * wy[mm] * wz[n];  /* Eq 7 */
                                if (w == 0.0) continue;
                                int64_t r = ((sbz + n) * K[1] + (sby + mm)) * K[0] + (sbx + l);
                                double *Pr = T + r * B * B;
                                for (int a = 0; a < B; ++a) {
                                    if (ha[a] == 0.0) continue;
                                    double wa = w * ha[a];
                                    for (int b = 0; b < B; ++b)
                                        if (hb[b] != 0.0) Pr[a * B + b] += wa * hb[b];
                                }
                            }
                }
        free(ha);
        free(hb);
    }
    memset(P, 0, sizeof(double) * (size_t)tab);
    for (int t = 0; t < nt; ++t)
        for (int64_t i = 0; i < tab; ++i) P[i] += priv[(size_t)t * (size_t)tab + i];
    free(priv);
}

/* Table I lines 4-18 on the unnormalized joint histogram P.
 * Outputs (arrays may be NULL):
 *   reg[r*6 + {0..5}] = {p(r), sigma_r^2, mu_r, 1-CR_r ("cr" of Table I), retained, Z}
 *   mura[r*B + a]     = mu_r(a) (0 where p_r(a) = 0)
 * Returns E = D (Eq 9) summed over retained regions (reading c12). */
double orc_value_table1(const orc_cfg *c, const double *P, double *reg, double *mura) {
    int64_t G[3], K[3];
    orc_derived(c, G, K);
    int L = c->L, B = L + 1;
    int64_t R = K[0] * K[1] * K[2];
    double Z = 0.0;
    for (int64_t i = 0; i < R * B * B; ++i) Z += P[i];   /* Z = sum p~ (c17) */
    double E = 0.0;                                       /* line 4 */
    double *pra = (double *)malloc(sizeof(double) * B), *prb = (double *)malloc(sizeof(double) * B);
    double *mua = (double *)malloc(sizeof(double) * B);
    for (int64_t r = 0; r < R; ++r) {                     /* line 5 */
        const double *Pr = P + r * B * B;
        double pr = 0.0;                                  /* Eq 4: p(r) */
        for (int i = 0; i < B * B; ++i) pr += Pr[i] / Z;
        double sig2 = 0.0, mu = 0.0, cr = 0.0;
        int retained = 0;
        for (int a = 0; a < B; ++a) { pra[a] = 0.0; prb[a] = 0.0; mua[a] = 0.0; }
        if (pr > c->eps_mass) {
            /* line 6: marginals p_r(a), p_r(b) (Eq 4) with p_r(a,b) = p(a,b,r)/p(r) */
            for (int a = 0; a < B; ++a)
                for (int b = 0; b < B; ++b) {
                    double pab = (Pr[a * B + b] / Z) / pr;
                    pra[a] += pab;
                    prb[b] += pab;
                }
            /* line 7: sigma_r^2 of the estimated image (Eq 10) */
            double e2 = 0.0;
            for (int b = 0; b < B; ++b) { mu += (double)b * prb[b]; e2 += (double)b * (double)b * prb[b]; }
            sig2 = e2 - mu * mu;
            /* lines 8-10: mu_r(a) (Eq 10) */
            for (int a = 0; a < B; ++a) {
                if (pra[a] == 0.0) continue;
                double s = 0.0;
                for (int b = 0; b < B; ++b) s += (double)b * ((Pr[a * B + b] / Z) / pr);
                mua[a] = s / pra[a];
            }
            if (sig2 > c->eps_sigma) {
                retained = 1;
                /* lines 11-16 */
                for (int a = 0; a < B; ++a)
                    for (int b = 0; b < B; ++b) {
                        double pab = (Pr[a * B + b] / Z) / pr;
                        if (pab == 0.0) continue;
                        cr += ((double)b * (double)b - mua[a] * mua[a]) * pab / sig2;
                    }
                E += pr * cr;                             /* line 17 */
            }
        }
        if (reg) {
            reg[r * 6 + 0] = pr; reg[r * 6 + 1] = sig2; reg[r * 6 + 2] = mu;
            reg[r * 6 + 3] = cr; reg[r * 6 + 4] = (double)retained; reg[r * 6 + 5] = Z;
        }
        if (mura)
            for (int a = 0; a < B; ++a) mura[r * B + a] = mua[a];
    }
    free(pra);
    free(prb);
    free(mua);
    return E;
}

/* dD/dM(y) by Eq 27 as printed, per voxel of z-slab [z0, z1):
 *   (1/Z) sum_r sum_a sum_b [((1-CR_r)(b^2 - 2 b mu_r) + 2 b mu_r(a) - b^2) / sigma_r^2]
 *         * w(r,x) h(a - F(x)) h'(kappa),  kappa = b - M(T(x))          (reading c7)
 * over retained r.  The b-sum runs over -1..L+1: the virtual bins -1 and L+1 enter
 * the derivative only, and only when m is exactly 0 or L (reading c4). */
void orc_dDdm_eq27(const orc_cfg *c, const float *F, const float *M, const double *params,
                   const double *reg, const double *mura, int64_t z0, int64_t z1, double *out) {
    int64_t G[3], K[3];
    orc_derived(c, G, K);
    int L = c->L, B = L + 1;
    int64_t nx = c->n[0], ny = c->n[1];
    int nt = nthreads_of(c);
#pragma omp parallel for schedule(static) num_threads(nt)
    for (int64_t z = z0; z < z1; ++z)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t x = 0; x < nx; ++x) {
                double u[3], p[3], m, g[3];
                orc_displacement(c, params, x, y, z, u);
                p[0] = (double)x + u[0]; p[1] = (double)y + u[1]; p[2] = (double)z + u[2];
                orc_sample(c, M, p, &m, g);
                double f = (double)F[(z * ny + y) * nx + x];
                int64_t sbx, sby, sbz;
                double wx[4], wy[4], wz[4];
                spat_taps(c, 0, x, &sbx, wx);
                spat_taps(c, 1, y, &sby, wy);
                spat_taps(c, 2, z, &sbz, wz);
                double acc = 0.0, Z = reg[5];
                for (int n = 0; n < 4; ++n)
                    for (int mm = 0; mm < 4; ++mm)
                        for (int l = 0; l < 4; ++l) {
                            double w = wx[l] * wy[mm] * wz[n];
                            if (w == 0.0) continue;
                            int64_t r = ((sbz + n) * K[1] + (sby + mm)) * K[0] + (sbx + l);
                            if (reg[r * 6 + 4] == 0.0) continue;
                            double sig2 = reg[r * 6 + 1], mur = reg[r * 6 + 2], omcr = reg[r * 6 + 3];
                            for (int a = 0; a < B; ++a) {
                                double ha = orc_parzen((double)a - f);
                                if (ha == 0.0) continue;
                                double mua = mura[r * B + a];
                                for (int b = -1; b <= L + 1; ++b) {
                                    double hp = orc_parzen_deriv((double)b - m);
                                    if (hp == 0.0) continue;
                                    double bb = (double)b;
                                    double num = omcr * (bb * bb - 2.0 * bb * mur) + 2.0 * bb * mua - bb * bb;
                                    acc += num / sig2 * w * ha * hp;
                                }
                            }
                        }
                out[((z - z0) * ny + y) * nx + x] = acc / Z;
            }
}

/* dD/dM(y) for the moving image as the model image A: Eq 21 / Eq 31,
 *   (1/Z) sum_r sum_a sum_b [(2b - mu_r(a)) mu_r(a) / sigma_r^2] w(r,x) h(b - F(x)) h'(a - M(T(x)))
 * over retained r (sigma_r^2 is F's, static in this orientation).  The a-sum runs over
 * -1..L+1 (h' is nonzero at |a - m| = 1 only for integer m, reading c4).  Reading c23:
 * a bin a with p_r(a) = 0 (and the virtual bins -1, L+1) takes mu_r(a) = g1(F(x)) =
 * sum_b b h(b - F(x)), the limit of mu_r(a) as the voxel's own mass enters the bin, so
 * the derivative is that of the function D (central differences agree). */
void orc_dDdm_eq31(const orc_cfg *c, const float *F, const float *M, const double *params, const double *P,
                   const double *reg, const double *mura, int64_t z0, int64_t z1, double *out) {
    int64_t G[3], K[3];
    orc_derived(c, G, K);
    int L = c->L, B = L + 1;
    int64_t nx = c->n[0], ny = c->n[1];
    int nt = nthreads_of(c);
#pragma omp parallel for schedule(static) num_threads(nt)
    for (int64_t z = z0; z < z1; ++z)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t x = 0; x < nx; ++x) {
                double u[3], p[3], m, g[3];
                orc_displacement(c, params, x, y, z, u);
                p[0] = (double)x + u[0]; p[1] = (double)y + u[1]; p[2] = (double)z + u[2];
                orc_sample(c, M, p, &m, g);
                double f = (double)F[(z * ny + y) * nx + x];
                double g1f = 0.0;
                for (int b = 0; b < B; ++b) g1f += (double)b * orc_parzen((double)b - f);
                int64_t sbx, sby, sbz;
                double wx[4], wy[4], wz[4];
                spat_taps(c, 0, x, &sbx, wx);
                spat_taps(c, 1, y, &sby, wy);
                spat_taps(c, 2, z, &sbz, wz);
                double acc = 0.0, Z = reg[5];
                for (int n = 0; n < 4; ++n)
                    for (int mm = 0; mm < 4; ++mm)
                        for (int l = 0; l < 4; ++l) {
                            double w = wx[l] * wy[mm] * wz[n];
                            if (w == 0.0) continue;
                            int64_t r = ((sbz + n) * K[1] + (sby + mm)) * K[0] + (sbx + l);
                            if (reg[r * 6 + 4] == 0.0) continue;
                            double sig2 = reg[r * 6 + 1];
                            for (int a = -1; a <= L + 1; ++a) {
                                double hp = orc_parzen_deriv((double)a - m);
                                if (hp == 0.0) continue;
                                double pa = 0.0;
                                if (a >= 0 && a <= L)
                                    for (int b = 0; b < B; ++b) pa += P[(r * B + a) * B + b];
                                double mua = pa > 0.0 ? mura[r * B + a] : g1f;
                                for (int b = 0; b < B; ++b) {
                                    double hb = orc_parzen((double)b - f);
                                    if (hb == 0.0) continue;
                                    acc += (2.0 * b - mua) * mua / sig2 * w * hb * hp;
                                }
                            }
                        }
                out[((z - z0) * ny + y) * nx + x] = acc / Z;
            }
}

/* Eq 16 with the Jacobian of Eq 17:
 *   dD/dphi_{s,c} += sum_x dD/dM(y) * d_c M(y) * beta_l(eta) beta_m(gamma) beta_n(tau)
 * over the voxels of z-slab [z0, z1); grad is SoA [ndim][nodes] and is ADDED to. */
void orc_grad_chain(const orc_cfg *c, const float *M, const double *params, const double *dDdm,
                    int64_t z0, int64_t z1, double *grad) {
    int64_t G[3], K[3];
    orc_derived(c, G, K);
    int nd = ndim_of(c);
    int64_t nodes = G[0] * G[1] * G[2], nx = c->n[0], ny = c->n[1];
    int nt = nthreads_of(c);
    double *priv = (double *)calloc((size_t)nt * (size_t)(nd * nodes), sizeof(double));
#pragma omp parallel num_threads(nt)
    {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        double *T = priv + (size_t)tid * (size_t)(nd * nodes);
#pragma omp for schedule(static)
        for (int64_t z = z0; z < z1; ++z)
            for (int64_t y = 0; y < ny; ++y)
                for (int64_t x = 0; x < nx; ++x) {
                    double u[3], p[3], m, g[3];
                    orc_displacement(c, params, x, y, z, u);
                    p[0] = (double)x + u[0]; p[1] = (double)y + u[1]; p[2] = (double)z + u[2];
                    orc_sample(c, M, p, &m, g);
                    double d = dDdm[((z - z0) * ny + y) * nx + x];
                    if (d == 0.0) continue;
                    int64_t bx, by, bz;
                    double wx[4], wy[4], wz[4];
                    ctrl_taps(c, 0, x, &bx, wx);
                    ctrl_taps(c, 1, y, &by, wy);
                    ctrl_taps(c, 2, z, &bz, wz);
                    for (int n = 0; n < 4; ++n) {
                        if (wz[n] == 0.0) continue;
                        for (int mm = 0; mm < 4; ++mm) {
                            if (wy[mm] == 0.0) continue;
                            for (int l = 0; l < 4; ++l) {
                                if (wx[l] == 0.0) continue;
                                double jac = wx[l] * wy[mm] * wz[n];   /* Eq 17 */
                                int64_t s = node_index(G, bx + l, by + mm, bz + n);
                                for (int comp = 0; comp < nd; ++comp) T[comp * nodes + s] += d * g[comp] * jac;
                            }
                        }
                    }
                }
    }
    for (int t = 0; t < nt; ++t)
        for (int64_t i = 0; i < nd * nodes; ++i) grad[i] += priv[(size_t)t * (size_t)(nd * nodes) + i];
    free(priv);
}

/* full literal evaluation: D and (if grad != NULL) dD/dPhi, SoA [ndim][nodes] */
double orc_eval_literal(const orc_cfg *c, const float *F, const float *M, const double *params,
                        double *grad) {
    int64_t G[3], K[3];
    orc_derived(c, G, K);
    int B = c->L + 1;
    int64_t R = K[0] * K[1] * K[2], nvox = c->n[0] * c->n[1] * c->n[2];
    double *P = (double *)malloc(sizeof(double) * (size_t)(R * B * B));
    double *reg = (double *)malloc(sizeof(double) * (size_t)(R * 6));
    double *mura = (double *)malloc(sizeof(double) * (size_t)(R * B));
    orc_joint_hist(c, F, M, params, 0, c->n[2], P);
    double D = orc_value_table1(c, P, reg, mura);
    if (grad) {
        int64_t nodes = G[0] * G[1] * G[2];
        double *dd = (double *)malloc(sizeof(double) * (size_t)nvox);
        if (c->orientation) orc_dDdm_eq31(c, F, M, params, P, reg, mura, 0, c->n[2], dd);
        else orc_dDdm_eq27(c, F, M, params, reg, mura, 0, c->n[2], dd);
        memset(grad, 0, sizeof(double) * (size_t)(ndim_of(c) * nodes));
        orc_grad_chain(c, M, params, dd, 0, c->n[2], grad);
        free(dd);
    }
    free(P);
    free(reg);
    free(mura);
    return D;
}

/* ====================================================== (2) MOMENT route === */

/* w1(f) = h(1 - f): weight of the upper of the two active bins (Eq 5) */
static double w1_of(double f) {
    return f < 0.5 ? 0.1 * f + 1.8 * f * f : -1.8 * f * f + 3.7 * f - 0.9;
}
static double w1_deriv(double f) { return f < 0.5 ? 0.1 + 3.6 * f : 3.7 - 3.6 * f; }

/* bin split of an intensity v in [0, L]: n = min(floor v, L-1), f = v - n (reading c5) */
static void bin_split(double v, int L, int *n, double *f) {
    int k = (int)floor(v);
    if (k > L - 1) k = L - 1;
    if (k < 0) k = 0;
    *n = k;
    *f = v - (double)k;
}

/* N[r][a] = sum w_r h_a(A), S[r][a] = sum w_r h_a(A) g1(B), Q[r][a] = sum w_r h_a(A) g2(B)
 * with g1 = n + w1(f) = sum_b b h(b-B), g2 = n^2 + (2n+1) w1(f) = sum_b b^2 h(b-B)
 * (SURVEY Appendix A), over z-slab [z0, z1); (A, B) = (F, M(T)) in orientation 0 and
 * (M(T), F) in orientation 1 (then N, S are dynamic and sum_a Q[r][a] = Q_r is static).
 * Any of N, S, Q may be NULL. */
void orc_moments(const orc_cfg *c, const float *F, const float *M, const double *params,
                 int64_t z0, int64_t z1, double *N, double *S, double *Q) {
    int64_t G[3], K[3];
    orc_derived(c, G, K);
    int L = c->L, B = L + 1;
    int64_t R = K[0] * K[1] * K[2], tab = R * B;
    int nt = nthreads_of(c);
    double *priv = (double *)calloc((size_t)nt * 3 * (size_t)tab, sizeof(double));
    int64_t nx = c->n[0], ny = c->n[1];
#pragma omp parallel num_threads(nt)
    {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        double *TN = priv + (size_t)tid * 3 * (size_t)tab, *TS = TN + tab, *TQ = TS + tab;
#pragma omp for schedule(static)
        for (int64_t z = z0; z < z1; ++z)
            for (int64_t y = 0; y < ny; ++y)
                for (int64_t x = 0; x < nx; ++x) {
                    double u[3], p[3], m, g[3];
                    orc_displacement(c, params, x, y, z, u);
                    p[0] = (double)x + u[0]; p[1] = (double)y + u[1]; p[2] = (double)z + u[2];
                    orc_sample(c, M, p, &m, g);
                    /* the model image A gives the bin a0 and its two Parzen weights, the
                     * estimated image B the moments g1, g2 (orientation: A = F or A = M) */
                    const double f = (double)F[(z * ny + y) * nx + x];
                    int a0, n;
                    double fa, fm;
                    bin_split(c->orientation ? m : f, L, &a0, &fa);
                    bin_split(c->orientation ? f : m, L, &n, &fm);
                    double h1 = w1_of(fa), h0 = 1.0 - h1;
                    double w1m = w1_of(fm);
                    double g1 = (double)n + w1m, g2 = (double)n * (double)n + (2.0 * n + 1.0) * w1m;
                    int64_t sbx, sby, sbz;
                    double wx[4], wy[4], wz[4];
                    spat_taps(c, 0, x, &sbx, wx);
                    spat_taps(c, 1, y, &sby, wy);
                    spat_taps(c, 2, z, &sbz, wz);
                    for (int nn = 0; nn < 4; ++nn)
                        for (int mm = 0; mm < 4; ++mm)
                            for (int l = 0; l < 4; ++l) {
                                double w = wx[l] * wy[mm] * wz[nn];
                                if (w == 0.0) continue;
                                int64_t r = ((sbz + nn) * K[1] + (sby + mm)) * K[0] + (sbx + l);
                                int64_t i0 = r * B + a0;
                                TN[i0] += w * h0; TN[i0 + 1] += w * h1;
                                TS[i0] += w * h0 * g1; TS[i0 + 1] += w * h1 * g1;
                                TQ[i0] += w * h0 * g2; TQ[i0 + 1] += w * h1 * g2;
                            }
                }
    }
    double *outs[3] = {N, S, Q};
    for (int k = 0; k < 3; ++k) {
        if (!outs[k]) continue;
        memset(outs[k], 0, sizeof(double) * (size_t)tab);
        for (int t = 0; t < nt; ++t)
            for (int64_t i = 0; i < tab; ++i) outs[k][i] += priv[((size_t)t * 3 + k) * (size_t)tab + i];
    }
    free(priv);
}

/* per region N_r, S_r, Q_r; T_r = Q_r - S_r^2/N_r;
 * V_r = Q_r - sum_{a: N_ra>0} S_ra^2/N_ra; D = (1/Z) sum_{retained} N_r V_r / T_r.
 * Coefficients for the derivative (zero for non-retained r):
 *   alpha_r = CR_r/sigma_r^2, beta_r = (1-CR_r) mu_r/sigma_r^2, gamma_ra = mu_r(a)/sigma_r^2.
 * reg[r*6 + ...] as orc_value_table1.  Returns D; *Zout = Z. */
double orc_combine(const orc_cfg *c, const double *N, const double *S, const double *Q,
                   double *alpha, double *beta, double *gamma, double *reg, double *Zout) {
    int64_t G[3], K[3];
    orc_derived(c, G, K);
    int B = c->L + 1;
    int64_t R = K[0] * K[1] * K[2];
    double Z = 0.0;
    for (int64_t i = 0; i < R * B; ++i) Z += N[i];
    double D = 0.0;
    for (int64_t r = 0; r < R; ++r) {
        double Nr = 0.0, Sr = 0.0, Qr = 0.0, sumS2N = 0.0;
        for (int a = 0; a < B; ++a) {
            double n = N[r * B + a];
            Nr += n; Sr += S[r * B + a]; Qr += Q[r * B + a];
            if (n > 0.0) sumS2N += S[r * B + a] * S[r * B + a] / n;
        }
        double pr = Nr / Z, sig2 = 0.0, mu = 0.0, omcr = 0.0;
        int retained = 0;
        if (pr > c->eps_mass) {
            double Tr = Qr - Sr * Sr / Nr, Vr = Qr - sumS2N;
            sig2 = Tr / Nr;
            mu = Sr / Nr;
            if (sig2 > c->eps_sigma) {
                retained = 1;
                omcr = Vr / Tr;
                D += Nr * Vr / Tr;
            }
        }
        if (alpha) alpha[r] = retained ? (1.0 - omcr) / sig2 : 0.0;
        if (beta) beta[r] = retained ? omcr * mu / sig2 : 0.0;
        if (gamma)
            for (int a = 0; a < B; ++a) {
                double n = N[r * B + a];
                gamma[r * B + a] = (retained && n > 0.0) ? (S[r * B + a] / n) / sig2 : 0.0;
            }
        if (reg) {
            reg[r * 6 + 0] = pr; reg[r * 6 + 1] = sig2; reg[r * 6 + 2] = mu;
            reg[r * 6 + 3] = omcr; reg[r * 6 + 4] = (double)retained; reg[r * 6 + 5] = Z;
        }
    }
    if (Zout) *Zout = Z;
    return D / Z;
}

/* dD/dm = (g1'/Z) [c2 A~ - 2 G~ + 2 B~] with
 *   A~ = sum_r w_r alpha_r, B~ = sum_r w_r beta_r,
 *   G~ = sum_r w_r (h_a0 gamma_{r,a0} + h_a0+1 gamma_{r,a0+1}),
 *   g1' = w1'(f), c2 = 2n+1 for fractional m; at integer m: g1' = 0.1, c2 = 2m (c4).
 * Per voxel of z-slab [z0, z1) into out (may be NULL); if grad != NULL the chain
 * rule of Eq 16-17 is ADDED into grad. */
void orc_grad_moments(const orc_cfg *c, const float *F, const float *M, const double *params,
                      const double *alpha, const double *beta, const double *gamma, double Z,
                      int64_t z0, int64_t z1, double *out, double *grad) {
    int64_t G[3], K[3];
    orc_derived(c, G, K);
    int L = c->L, B = L + 1, nd = ndim_of(c);
    int64_t nodes = G[0] * G[1] * G[2], nx = c->n[0], ny = c->n[1];
    int nt = nthreads_of(c);
    double *priv = grad ? (double *)calloc((size_t)nt * (size_t)(nd * nodes), sizeof(double)) : NULL;
#pragma omp parallel num_threads(nt)
    {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        double *T = priv ? priv + (size_t)tid * (size_t)(nd * nodes) : NULL;
#pragma omp for schedule(static)
        for (int64_t z = z0; z < z1; ++z)
            for (int64_t y = 0; y < ny; ++y)
                for (int64_t x = 0; x < nx; ++x) {
                    double u[3], p[3], m, g[3];
                    orc_displacement(c, params, x, y, z, u);
                    p[0] = (double)x + u[0]; p[1] = (double)y + u[1]; p[2] = (double)z + u[2];
                    orc_sample(c, M, p, &m, g);
                    int a0, n;
                    double fa, fm;
                    bin_split((double)F[(z * ny + y) * nx + x], L, &a0, &fa);
                    bin_split(m, L, &n, &fm);
                    double h1 = w1_of(fa), h0 = 1.0 - h1;
                    double g1p, c2;
                    if (m == floor(m)) { g1p = 0.1; c2 = 2.0 * m; }
                    else { g1p = w1_deriv(fm); c2 = 2.0 * n + 1.0; }
                    int64_t sbx, sby, sbz;
                    double wx[4], wy[4], wz[4];
                    spat_taps(c, 0, x, &sbx, wx);
                    spat_taps(c, 1, y, &sby, wy);
                    spat_taps(c, 2, z, &sbz, wz);
                    double At = 0.0, Bt = 0.0, Gt = 0.0;
                    for (int nn = 0; nn < 4; ++nn)
                        for (int mm = 0; mm < 4; ++mm)
                            for (int l = 0; l < 4; ++l) {
                                double w = wx[l] * wy[mm] * wz[nn];
                                if (w == 0.0) continue;
                                int64_t r = ((sbz + nn) * K[1] + (sby + mm)) * K[0] + (sbx + l);
                                At += w * alpha[r];
                                Bt += w * beta[r];
                                Gt += w * (h0 * gamma[r * B + a0] + h1 * gamma[r * B + a0 + 1]);
                            }
                    double d = g1p / Z * (c2 * At - 2.0 * Gt + 2.0 * Bt);
                    if (out) out[((z - z0) * ny + y) * nx + x] = d;
                    if (!T || d == 0.0) continue;
                    int64_t bx, by, bz;
                    double cx[4], cy[4], cz[4];
                    ctrl_taps(c, 0, x, &bx, cx);
                    ctrl_taps(c, 1, y, &by, cy);
                    ctrl_taps(c, 2, z, &bz, cz);
                    for (int nn = 0; nn < 4; ++nn) {
                        if (cz[nn] == 0.0) continue;
                        for (int mm = 0; mm < 4; ++mm) {
                            if (cy[mm] == 0.0) continue;
                            for (int l = 0; l < 4; ++l) {
                                if (cx[l] == 0.0) continue;
                                double jac = cx[l] * cy[mm] * cz[nn];
                                int64_t s = node_index(G, bx + l, by + mm, bz + nn);
                                for (int comp = 0; comp < nd; ++comp) T[comp * nodes + s] += d * g[comp] * jac;
                            }
                        }
                    }
                }
    }
    if (grad) {
        for (int t = 0; t < nt; ++t)
            for (int64_t i = 0; i < nd * nodes; ++i) grad[i] += priv[(size_t)t * (size_t)(nd * nodes) + i];
        free(priv);
    }
}

/* Orientation 1 (moving image as the model image A; Eq 20-21, App. II Eq 28-31), moment
 * form: with mu_ra = S_ra/N_ra and psi_ra(g) = (mu_ra^2 - 2 mu_ra g)/sigma_r^2 (and, reading
 * c23, psi = -g^2/sigma_r^2 for an empty or virtual bin a), g = g1(F(x)):
 *   dD/dm = (1/Z) sum_r w_r sum_a (d h_a(m)/dm) psi_ra(g)
 * with d h_n/dm = -w1'(f), d h_{n+1}/dm = +w1'(f) for fractional m and, at integer m = k,
 * the two-sided average -0.05 (bin k-1), +0.05 (bin k+1) (reading c4).  gamma and reg as
 * orc_combine (gamma_ra = mu_ra/sigma_r^2), N for the empty-bin test.  Per voxel of the
 * slab into out (nullable); if grad != NULL the chain rule of Eq 16-17 is ADDED. */
void orc_grad_moments_A(const orc_cfg *c, const float *F, const float *M, const double *params,
                        const double *N, const double *gamma, const double *reg, double Z,
                        int64_t z0, int64_t z1, double *out, double *grad) {
    int64_t G[3], K[3];
    orc_derived(c, G, K);
    int L = c->L, B = L + 1, nd = ndim_of(c);
    int64_t nodes = G[0] * G[1] * G[2], nx = c->n[0], ny = c->n[1];
    int nt = nthreads_of(c);
    double *priv = grad ? (double *)calloc((size_t)nt * (size_t)(nd * nodes), sizeof(double)) : NULL;
#pragma omp parallel num_threads(nt)
    {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        double *T = priv ? priv + (size_t)tid * (size_t)(nd * nodes) : NULL;
#pragma omp for schedule(static)
        for (int64_t z = z0; z < z1; ++z)
            for (int64_t y = 0; y < ny; ++y)
                for (int64_t x = 0; x < nx; ++x) {
                    double u[3], p[3], m, g[3];
                    orc_displacement(c, params, x, y, z, u);
                    p[0] = (double)x + u[0]; p[1] = (double)y + u[1]; p[2] = (double)z + u[2];
                    orc_sample(c, M, p, &m, g);
                    int nF, n;
                    double fF, fm;
                    bin_split((double)F[(z * ny + y) * nx + x], L, &nF, &fF);
                    const double gF = (double)nF + w1_of(fF);
                    bin_split(m, L, &n, &fm);
                    int ab[2];
                    double dh[2];
                    if (m == floor(m)) { ab[0] = (int)m - 1; ab[1] = (int)m + 1; dh[0] = -0.05; dh[1] = 0.05; }
                    else { ab[0] = n; ab[1] = n + 1; dh[0] = -w1_deriv(fm); dh[1] = w1_deriv(fm); }
                    int64_t sbx, sby, sbz;
                    double wx[4], wy[4], wz[4];
                    spat_taps(c, 0, x, &sbx, wx);
                    spat_taps(c, 1, y, &sby, wy);
                    spat_taps(c, 2, z, &sbz, wz);
                    double acc = 0.0;
                    for (int nn = 0; nn < 4; ++nn)
                        for (int mm = 0; mm < 4; ++mm)
                            for (int l = 0; l < 4; ++l) {
                                double w = wx[l] * wy[mm] * wz[nn];
                                if (w == 0.0) continue;
                                int64_t r = ((sbz + nn) * K[1] + (sby + mm)) * K[0] + (sbx + l);
                                if (reg[r * 6 + 4] == 0.0) continue;
                                const double sig2 = reg[r * 6 + 1];
                                for (int k = 0; k < 2; ++k) {
                                    const int a = ab[k];
                                    double psi;
                                    if (a < 0 || a > L || N[r * B + a] <= 0.0) psi = -gF * gF / sig2;
                                    else {
                                        const double mu = gamma[r * B + a] * sig2;
                                        psi = (mu * mu - 2.0 * mu * gF) / sig2;
                                    }
                                    acc += w * dh[k] * psi;
                                }
                            }
                    const double d = acc / Z;
                    if (out) out[((z - z0) * ny + y) * nx + x] = d;
                    if (!T || d == 0.0) continue;
                    int64_t bx, by, bz;
                    double cx[4], cy[4], cz[4];
                    ctrl_taps(c, 0, x, &bx, cx);
                    ctrl_taps(c, 1, y, &by, cy);
                    ctrl_taps(c, 2, z, &bz, cz);
                    for (int nn = 0; nn < 4; ++nn) {
                        if (cz[nn] == 0.0) continue;
                        for (int mm = 0; mm < 4; ++mm) {
                            if (cy[mm] == 0.0) continue;
                            for (int l = 0; l < 4; ++l) {
                                if (cx[l] == 0.0) continue;
                                double jac = cx[l] * cy[mm] * cz[nn];
                                int64_t s = node_index(G, bx + l, by + mm, bz + nn);
                                for (int comp = 0; comp < nd; ++comp) T[comp * nodes + s] += d * g[comp] * jac;
                            }
                        }
                    }
                }
    }
    if (grad) {
        for (int t = 0; t < nt; ++t)
            for (int64_t i = 0; i < nd * nodes; ++i) grad[i] += priv[(size_t)t * (size_t)(nd * nodes) + i];
        free(priv);
    }
}

/* full moment-route evaluation */
double orc_eval_moments(const orc_cfg *c, const float *F, const float *M, const double *params,
                        double *grad) {
    int64_t G[3], K[3];
    orc_derived(c, G, K);
    int B = c->L + 1, nd = ndim_of(c);
    int64_t R = K[0] * K[1] * K[2], nodes = G[0] * G[1] * G[2];
    double *N = (double *)malloc(sizeof(double) * (size_t)(R * B));
    double *S = (double *)malloc(sizeof(double) * (size_t)(R * B));
    double *Q = (double *)malloc(sizeof(double) * (size_t)(R * B));
    double *al = (double *)malloc(sizeof(double) * (size_t)R), *be = (double *)malloc(sizeof(double) * (size_t)R);
    double *ga = (double *)malloc(sizeof(double) * (size_t)(R * B));
    double *reg = (double *)malloc(sizeof(double) * (size_t)(R * 6));
    orc_moments(c, F, M, params, 0, c->n[2], N, S, Q);
    double Z;
    double D = orc_combine(c, N, S, Q, al, be, ga, reg, &Z);
    if (grad) {
        memset(grad, 0, sizeof(double) * (size_t)(nd * nodes));
        if (c->orientation) orc_grad_moments_A(c, F, M, params, N, ga, reg, Z, 0, c->n[2], NULL, grad);
        else orc_grad_moments(c, F, M, params, al, be, ga, Z, 0, c->n[2], NULL, grad);
    }
    free(N); free(S); free(Q); free(al); free(be); free(ga); free(reg);
    return D;
}

/* ============================================ (3) bending energy C_p (F1) === */

/* First and second derivatives of the Eq 8 pieces with respect to t. */
static void beta_d1(double t, double w[4]) {
    w[0] = -(1.0 - t) * (1.0 - t) / 2.0;
    w[1] = (3.0 * t * t - 4.0 * t) / 2.0;
    w[2] = (-3.0 * t * t + 2.0 * t + 1.0) / 2.0;
    w[3] = t * t / 2.0;
}
static void beta_d2(double t, double w[4]) {
    w[0] = 1.0 - t;
    w[1] = 3.0 * t - 2.0;
    w[2] = -3.0 * t + 1.0;
    w[3] = t;
}

/* Derivative-order-p tap weights of voxel i on the control lattice of axis ax,
 * with respect to the voxel coordinate (d/di = (1/delta) d/dt).  The 2-D z axis
 * is constant: weights (1,0,0,0) for p = 0 and 0 for p >= 1. */
static void ctrl_taps_d(const orc_cfg *c, int ax, int64_t i, int64_t *b, double w[3][4]) {
    double t;
    if (ax == 2 && c->n[2] == 1) {
        *b = 0;
        for (int p = 0; p < 3; ++p)
            for (int k = 0; k < 4; ++k) w[p][k] = (p == 0 && k == 0) ? 1.0 : 0.0;
        return;
    }
    double s = (double)i / c->delta[ax];
    double fl = floor(s);
    *b = (int64_t)fl;
    t = s - fl;
    orc_beta(t, w[0]);
    beta_d1(t, w[1]);
    beta_d2(t, w[2]);
    double d = c->delta[ax];
    for (int k = 0; k < 4; ++k) {
        w[1][k] /= d;
        w[2][k] /= d * d;
    }
}

/* Bending energy of the FFD, the constraint C_p of Eq 1 (form of
 * Rueckert et al. [26], reading c19):
 *   C_p = (1/V) sum_x sum_c [ u_c,xx^2 + u_c,yy^2 + u_c,zz^2
 *                             + 2 u_c,xy^2 + 2 u_c,xz^2 + 2 u_c,yz^2 ]
 * over every voxel x of the volume (V voxels) and displacement component c, with
 * derivatives in voxel coordinates (u in voxels); in 2-D only the x,y terms.
 * Each second derivative is the tensor product of Eq 8 derivative weights (Eq 17
 * taps).  grad (nullable, zeroed here) receives dC_p/dphi.  Written per voxel:
 * plain and slow. */
double orc_bending(const orc_cfg *c, const double *params, double *grad) {
    int64_t G[3], K[3];
    orc_derived(c, G, K);
    int nd = ndim_of(c);
    int64_t nodes = G[0] * G[1] * G[2];
    double V = (double)c->n[0] * (double)c->n[1] * (double)c->n[2];
    /* the six (ordered-pair-folded) terms: derivative orders per axis, weight */
    static const int ord[6][3] = {{2, 0, 0}, {0, 2, 0}, {0, 0, 2}, {1, 1, 0}, {1, 0, 1}, {0, 1, 1}};
    static const double tw[6] = {1.0, 1.0, 1.0, 2.0, 2.0, 2.0};
    int use[6];
    for (int t = 0; t < 6; ++t) use[t] = nd == 3 || ord[t][2] == 0;
    if (grad) memset(grad, 0, sizeof(double) * (size_t)(nd * nodes));
    double E = 0.0;
    for (int64_t z = 0; z < c->n[2]; ++z)
        for (int64_t y = 0; y < c->n[1]; ++y)
            for (int64_t x = 0; x < c->n[0]; ++x) {
                int64_t bx, by, bz;
                double wx[3][4], wy[3][4], wz[3][4];
                ctrl_taps_d(c, 0, x, &bx, wx);
                ctrl_taps_d(c, 1, y, &by, wy);
                ctrl_taps_d(c, 2, z, &bz, wz);
                int nzt = nd == 3 ? 4 : 1;
                for (int comp = 0; comp < nd; ++comp) {
                    double h[6] = {0, 0, 0, 0, 0, 0};
                    for (int n = 0; n < nzt; ++n)
                        for (int m = 0; m < 4; ++m)
                            for (int l = 0; l < 4; ++l) {
                                double phi = params[comp * nodes + node_index(G, bx + l, by + m, bz + n)];
                                for (int t = 0; t < 6; ++t)
                                    if (use[t])
                                        h[t] += wx[ord[t][0]][l] * wy[ord[t][1]][m] * wz[ord[t][2]][n] * phi;
                            }
                    for (int t = 0; t < 6; ++t)
                        if (use[t]) E += tw[t] * h[t] * h[t];
                    if (!grad) continue;
                    for (int n = 0; n < nzt; ++n)
                        for (int m = 0; m < 4; ++m)
                            for (int l = 0; l < 4; ++l) {
                                double s = 0.0;
                                for (int t = 0; t < 6; ++t)
                                    if (use[t])
                                        s += 2.0 * tw[t] * h[t] * wx[ord[t][0]][l] * wy[ord[t][1]][m] * wz[ord[t][2]][n];
                                grad[comp * nodes + node_index(G, bx + l, by + m, bz + n)] += s / V;
                            }
                }
            }
    return E / V;
}
