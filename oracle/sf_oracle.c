/*
 * sf_oracle.c -- plain, slow, single-threaded CPU oracle of the structure-flow
 * filter's per-frame predictor-update loop (Adarve & Mahony, arXiv 2406.18031).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA library under paper_2406_18031_b200/;
 * the only thing both sides consume in common is the seeded input data produced
 * by sfgen/ (grid geometry, brightness, depth, run parameters).
 *
 * Compiled twice (see oracle/build.py):
 *   liboracle_f32.so  -DOR_F32   every value and every decision in IEEE float32;
 *                                this is the parity oracle, because the paper fixes
 *                                no precision and the discontinuous decisions
 *                                (dominant flow, upwind side, rho one-sided
 *                                difference) must be taken in the kernel's precision.
 *   liboracle_f64.so  (default)  the same algorithm in float64; pins the float32
 *                                build's rounding drift.
 * Build flags: -O2 -ffp-contract=off (no implicit FMA); every fused multiply-add
 * is an explicit fma() call, written where the formula is "a*b + c".
 *
 * Notation follows the paper; line numbers cite /root/reference/PAPER.md.
 * Readings of ambiguous passages are numbered as in DESIGN.md section 3
 * ("Readings"); the arithmetic order below IS the definition the CUDA path
 * reproduces.
 *
 * Parity status: every function below is pinned by tests/test_oracle_*.py
 * (pins.py: the H = 1 filter; eval.py, pyramid.py, map.py, imu.py: the NEXT rows)
 * except the full multi-frame trajectories on scenes with occlusions and an active
 * flow clamp (H = 1 and the H = 2 pyramid), which are pinned only by invariants,
 * closed-form special cases, f32-vs-f64 agreement and accuracy against the
 * rendered ground truth ("What the pins leave open").
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef OR_F32
typedef float real;
#define FMA fmaf
#define FABS fabsf
#define FMIN fminf
#define FMAX fmaxf
#else
typedef double real;
#define FMA fma
#define FABS fabs
#define FMIN fmin
#define FMAX fmax
#endif
#define R(x) ((real)(x))

#define OR_FLAG_CLAMPED 1u   /* |u_hat| exceeded max_flow and was clamped (reading 12) */
#define OR_FLAG_NONFINITE 2u /* a non-finite value appeared in the inputs Y or the state */
#define OR_FLAG_CFL 4u       /* clamp disabled and dt*|u_hat| > 1 (eq:numerical_stability) */

#define OR_DOM_LARGEST 0
#define OR_DOM_PRINTED 1

/* Run parameters, a fixed C layout independent of `real`. */
typedef struct {
    int32_t H, W;
    int32_t N;                      /* substeps, N = ceil(max_flow) (L684-689)           */
    int32_t smooth_iters;           /* S, 5x5 box passes after the solve (L590, L796)    */
    int32_t dominant_rule;          /* OR_DOM_LARGEST (reading 1) or OR_DOM_PRINTED       */
    int32_t clamp_advection;        /* 1: clamp u_hat to +-max_flow (reading 12)          */
    int32_t input_is_inverse_depth; /* 0: depth lambda in metres (L463); 1: rho given     */
    int32_t pad;
    double max_flow;
    double sigma;    /* source-term weight per pass (reading 2; 0.5)                     */
    double gamma[5]; /* gamma1..gamma5 (L556-559, L613-616)                               */
    int32_t imu;     /* 1: add the inertial source terms of eq:hflow_conservation (NEXT #4)  */
    int32_t pad2;
    double omega[3]; /* camera angular velocity Omega, rad per frame (camera frame)          */
    double accel[3]; /* camera linear acceleration a_c, per frame^2 (camera frame)           */
} or_params;

static inline int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* <a, x> accumulated x, then y, then z: fma(a.z, x.z, fma(a.y, x.y, a.x * x.x)). */
static inline real dot3(const real* a, const real* x) { return FMA(a[2], x[2], FMA(a[1], x[1], a[0] * x[0])); }

/* ------------------------------------------------------------------ geometry
 * Per-grid working geometry geo[p][10] = (s, e1, e2, d2) from the Spherepix input
 * (s, b1, b2, ds) (L406-437):  e_k = b_k / ds  (so that Phi = (1/ds) B^T w = (e1.w, e2.w),
 * eq:oflow_numeric L639-642, reading 5), d2 = ds * ds.
 */
void or_geometry(int H, int W, const float* g10, real* geo)
{
    for (long p = 0; p < (long)H * W; ++p) {
        const float* g = g10 + 10 * p;
        real* o = geo + 10 * p;
        real ds = R(g[9]);
        for (int a = 0; a < 3; ++a) {
            o[a] = R(g[a]);
            o[3 + a] = R(g[3 + a]) / ds;
            o[6 + a] = R(g[6 + a]) / ds;
        }
        o[9] = ds * ds;
    }
}

/* ------------------------------------------------------------------ predict (P1-P5)
 * One transport pass along one axis for all pixels (Jacobi: every read is a pre-pass value).
 *   axis 0 = column pass (beta_1, neighbours (i, j+-1), e = e1), L663-673;
 *   axis 1 = row pass    (beta_2, neighbours (i+-1, j), e = e2), L674-683 (reading 3).
 * For each pixel p:
 *   u_p  = <e_p, w_p>                                    optical flow in px, eq:oflow_numeric
 *   u_hat = dominant(u_{p-}, u_{p+})                      L643-650 (reading 1)
 *   u_hat = clamp(u_hat, -U, U)                           reading 12
 *   D(f) = f_p - f_{p-} if u_hat > 0 else f_{p+} - f_p    upwind operator, L652-658, table
 *   f*_p = f_p - dt [ u_hat D(f) + f_p sigma <s_p, w_p> ] for f in (w.x, w.y, w.z, rho), L665-669
 * with replicate (clamp-to-edge) neighbours at the border (reading 10).
 * Arithmetic: t = fma(u_hat, D, f * (sigma*sw)); f* = fma(-dt, t, f).
 */
static unsigned pass(const or_params* P, const real* geo, int axis, const real* w, const real* rho, real* wo,
                     real* rhoo, real* u)
{
    const int H = P->H, W = P->W;
    const real U = R(P->max_flow), sigma = R(P->sigma), dt = R(1) / R(P->N);
    unsigned flags = 0;
    for (long p = 0; p < (long)H * W; ++p) u[p] = dot3(geo + 10 * p + 3 + 3 * axis, w + 3 * p);
    for (int i = 0; i < H; ++i) {
        for (int j = 0; j < W; ++j) {
            const long p = (long)i * W + j;
            long pm, pp;
            if (axis == 0) {
                pm = (long)i * W + clampi(j - 1, 0, W - 1);
                pp = (long)i * W + clampi(j + 1, 0, W - 1);
            } else {
                pm = (long)clampi(i - 1, 0, H - 1) * W + j;
                pp = (long)clampi(i + 1, 0, H - 1) * W + j;
            }
            const real um = u[pm], up = u[pp];
            real uh;
            if (P->dominant_rule == OR_DOM_PRINTED)
                uh = (FABS(up) - FABS(um) > R(0)) ? um : up; /* as printed: delta^c |u| > 0 -> u_{j-1} */
            else
                uh = (FABS(um) > FABS(up)) ? um : up; /* largest magnitude, ties -> u_{j+1} */
            if (P->clamp_advection) {
                if (FABS(uh) > U) flags |= OR_FLAG_CLAMPED;
                uh = FMIN(FMAX(uh, -U), U);
            } else if (dt * FABS(uh) > R(1)) {
                flags |= OR_FLAG_CFL;
            }
            const real sw = dot3(geo + 10 * p, w + 3 * p); /* <s, w^n> at p */
            const real q = sigma * sw;
            real f[4] = {w[3 * p], w[3 * p + 1], w[3 * p + 2], rho[p]};
            real fm[4] = {w[3 * pm], w[3 * pm + 1], w[3 * pm + 2], rho[pm]};
            real fp[4] = {w[3 * pp], w[3 * pp + 1], w[3 * pp + 2], rho[pp]};
            real out[4];
            for (int c = 0; c < 4; ++c) {
                const real D = (uh > R(0)) ? (f[c] - fm[c]) : (fp[c] - f[c]);
                out[c] = FMA(-dt, FMA(uh, D, f[c] * q), f[c]);
            }
            wo[3 * p] = out[0];
            wo[3 * p + 1] = out[1];
            wo[3 * p + 2] = out[2];
            rhoo[p] = out[3];
        }
    }
    return flags;
}

/* Inertial source terms (NEXT #4; eq:hflow_conservation L341-345 with eq:totaldev_hflow and
 * a_w, L258-280): the paper drops -Omega x w + a_w (eq:assumption L505-514); with them
 *   dw/dt = ... - Omega x w + a_w,  a_w = rho a_c - Omega x (w + Omega x s)
 *         = ... + rho a_c - 2 Omega x w - Omega x (Omega x s)       (rho has no source term).
 * Reading 32: one explicit Euler stage per substep after the row pass, on the post-pass fields:
 *   c1 = Omega x s, c2 = Omega x c1, c3 = Omega x w   (cross(a,b)_x = fma(a_y, b_z, -(a_z b_y)), cyclic)
 *   f_a = fma(rho, a_c,a, -fma(2, c3_a, c2_a));  w_a = fma(dt, f_a, w_a). */
static inline void cross3(const real* a, const real* b, real* c)
{
    c[0] = FMA(a[1], b[2], -(a[2] * b[1]));
    c[1] = FMA(a[2], b[0], -(a[0] * b[2]));
    c[2] = FMA(a[0], b[1], -(a[1] * b[0]));
}

static void imu_stage(const or_params* P, const real* geo, real* w, const real* rho)
{
    const real dt = R(1) / R(P->N);
    const real om[3] = {R(P->omega[0]), R(P->omega[1]), R(P->omega[2])};
    const real ac[3] = {R(P->accel[0]), R(P->accel[1]), R(P->accel[2])};
    for (long p = 0; p < (long)P->H * P->W; ++p) {
        real c1[3], c2[3], c3[3];
        cross3(om, geo + 10 * p, c1);
        cross3(om, c1, c2);
        cross3(om, w + 3 * p, c3);
        for (int a = 0; a < 3; ++a) {
            const real f = FMA(rho[p], ac[a], -FMA(R(2), c3[a], c2[a]));
            w[3 * p + a] = FMA(dt, f, w[3 * p + a]);
        }
    }
}

/* Prediction k -> k+ (L501-523, numerical scheme L662-683): exactly N substeps
 * (reading 4), each a column pass then a row pass (then the inertial stage when enabled).
 * In place on (w, rho). */
unsigned or_predict(const or_params* P, const real* geo, real* w, real* rho)
{
    const long n = (long)P->H * P->W;
    real* w2 = malloc(sizeof(real) * 3 * n);
    real* r2 = malloc(sizeof(real) * n);
    real* u = malloc(sizeof(real) * n);
    unsigned flags = 0;
    for (int s = 0; s < P->N; ++s) {
        flags |= pass(P, geo, 0, w, rho, w2, r2, u);
        flags |= pass(P, geo, 1, w2, r2, w, rho, u);
        if (P->imu) imu_stage(P, geo, w, rho);
    }
    free(w2);
    free(r2);
    free(u);
    return flags;
}

/* ------------------------------------------------------------------ update models (U1, U2)
 * Brightness model (L442-457, eq:img_model, eq:img_gradient).  The 5x5 Gaussian-weighted
 * LS fit of Y_q ~ Yhat_p + beta . (q - p) (reading 7: offset q - p) has, because
 * sum g = 1, sum g k = 0, sum g k^2 = 1 for g = [1,4,6,4,1]/16, the closed form
 *   Yhat = (g x g) * Y,  beta1 = (g along i) x (h along j) * Y,  beta2 = (h along i) x (g along j) * Y
 * with h_k = k g_k = [-1,-2,0,2,1]/8, taps in offset order k = -2..2, as separable 1-D
 * convolutions (L452).  Horizontal pass first, then vertical; replicate border.
 * Each 1-D tap sum: acc = k_{-2} x_{-2}; acc = fma(k_t, x_t, acc) for t = -1..2.
 * Lift (eq:img_gradient, reading 5): ghat = ds B beta = d2 (e1 beta1 + e2 beta2),
 * per component  ghat_a = d2 * fma(e2_a, beta2, e1_a * beta1).
 */
static const double G5[5] = {0.0625, 0.25, 0.375, 0.25, 0.0625};
static const double H5[5] = {-0.125, -0.25, 0.0, 0.25, 0.125};

static void conv_h(int H, int W, const real* k5, const real* x, real* out)
{
    for (int i = 0; i < H; ++i)
        for (int j = 0; j < W; ++j) {
            const real* row = x + (long)i * W;
            real acc = k5[0] * row[clampi(j - 2, 0, W - 1)];
            for (int t = 1; t < 5; ++t) acc = FMA(k5[t], row[clampi(j + t - 2, 0, W - 1)], acc);
            out[(long)i * W + j] = acc;
        }
}

static void conv_v(int H, int W, const real* k5, const real* x, real* out)
{
    for (int i = 0; i < H; ++i)
        for (int j = 0; j < W; ++j) {
            real acc = k5[0] * x[(long)clampi(i - 2, 0, H - 1) * W + j];
            for (int t = 1; t < 5; ++t) acc = FMA(k5[t], x[(long)clampi(i + t - 2, 0, H - 1) * W + j], acc);
            out[(long)i * W + j] = acc;
        }
}

void or_brightness_model(int H, int W, const float* Y, const real* geo, real* yhat, real* beta1, real* beta2,
                         real* ghat)
{
    const long n = (long)H * W;
    real g[5], h[5];
    for (int t = 0; t < 5; ++t) {
        g[t] = R(G5[t]);
        h[t] = R(H5[t]);
    }
    real* y = malloc(sizeof(real) * n);
    real* hg = malloc(sizeof(real) * n);
    real* hh = malloc(sizeof(real) * n);
    for (long p = 0; p < n; ++p) y[p] = R(Y[p]);
    conv_h(H, W, g, y, hg);
    conv_h(H, W, h, y, hh);
    conv_v(H, W, g, hg, yhat);
    conv_v(H, W, g, hh, beta1);
    conv_v(H, W, h, hg, beta2);
    for (long p = 0; p < n; ++p) {
        const real* e1 = geo + 10 * p + 3;
        const real* e2 = geo + 10 * p + 6;
        const real d2 = geo[10 * p + 9];
        for (int a = 0; a < 3; ++a) ghat[3 * p + a] = d2 * FMA(e2[a], beta2[p], e1[a] * beta1[p]);
    }
    free(y);
    free(hg);
    free(hh);
}

/* Inverse-depth model (L460-499, eq:dominant_b1/b2, table:diff_operators, eq:inv_depth_gradient).
 *   valid = isfinite(lambda) && lambda > 0;  rhohat = 1 / lambda  (eq:inv_depth, lambda_ref = 1 m, L173)
 *   per axis: d+ = rho_{p+} - rho_p, d- = rho_p - rho_{p-};  beta_rho = d+ if |d+| <= |d-| else d-
 *   (reading 14: an invalid neighbour's difference drops out; both invalid -> 0; invalid p -> 0)
 *   drho = d2 * fma(e2, beta_rho2, e1 * beta_rho1)   (lift as for ghat, reading 5)
 */
static real pick_side(const real* rh, const unsigned char* v, long p, long pm, long pp)
{
    if (!v[p]) return R(0);
    const int hp = v[pp], hm = v[pm];
    const real dp = rh[pp] - rh[p];
    const real dm = rh[p] - rh[pm];
    if (hp && hm) return (FABS(dp) <= FABS(dm)) ? dp : dm;
    if (hp) return dp;
    if (hm) return dm;
    return R(0);
}

void or_invdepth_model(int H, int W, const float* depth, int is_inverse, const real* geo, real* rhohat,
                       unsigned char* valid, real* beta_r1, real* beta_r2, real* drho)
{
    const long n = (long)H * W;
    for (long p = 0; p < n; ++p) {
        const real x = R(depth[p]);
        const int ok = is_inverse ? (isfinite(x) && x >= R(0)) : (isfinite(x) && x > R(0));
        valid[p] = (unsigned char)ok;
        rhohat[p] = ok ? (is_inverse ? x : R(1) / x) : R(0);
    }
    for (int i = 0; i < H; ++i)
        for (int j = 0; j < W; ++j) {
            const long p = (long)i * W + j;
            const real b1 =
                pick_side(rhohat, valid, p, (long)i * W + clampi(j - 1, 0, W - 1), (long)i * W + clampi(j + 1, 0, W - 1));
            const real b2 =
                pick_side(rhohat, valid, p, (long)clampi(i - 1, 0, H - 1) * W + j, (long)clampi(i + 1, 0, H - 1) * W + j);
            beta_r1[p] = b1;
            beta_r2[p] = b2;
            const real* e1 = geo + 10 * p + 3;
            const real* e2 = geo + 10 * p + 6;
            const real d2 = geo[10 * p + 9];
            for (int a = 0; a < 3; ++a) drho[3 * p + a] = d2 * FMA(e2[a], b2, e1[a] * b1);
        }
}

/* ------------------------------------------------------------------ update solve (U3)
 * Per-pixel regularised LS (L552-588, eq:cost_top, eq:img_cost_top, eq:invdepth_cost_top,
 * eq:LS_update), with E_t = w - w^{k+} (reading 8) and P(s) dropped (reading 16):
 *   E_Y = ghat . w + cY,  E_rho = m . w + crho,  E_t = w - wp
 *   A = g3 I + g1 ghat ghat^T + g2 m m^T,   b = g3 wp - g1 cY ghat - g2 crho m
 * A is SPD (lambda_min >= g3 > 0); solved by LDL^T without pivoting (reading 17):
 *   entries  A_ab = fma(g2 m_a, m_b, (g1 g_a) g_b),  A_aa += g3
 *            b_a  = fma(-(g2 m_a), crho, fma(-(g1 g_a), cY, g3 wp_a))
 *   factor   r0 = 1/A00; l10 = A10 r0; l20 = A20 r0; d1 = fma(-l10, A10, A11); r1 = 1/d1;
 *            t = fma(-l20, A10, A21); l21 = t r1; d2 = fma(-l21, t, fma(-l20, A20, A22)); r2 = 1/d2
 *   forward  y1 = fma(-l10, b0, b1); y2 = fma(-l21, y1, fma(-l20, b0, b2))
 *   back     x2 = y2 r2; x1 = fma(-l21, x2, y1 r1); x0 = fma(-l20, x2, fma(-l10, x1, b0 r0))
 */
static void ls_solve(const real* g, const real* m, real cY, real cr, const real* wp, real g1, real g2, real g3,
                     real* x)
{
    real g1g[3], g2m[3], A[3][3], b[3];
    for (int a = 0; a < 3; ++a) {
        g1g[a] = g1 * g[a];
        g2m[a] = g2 * m[a];
    }
    for (int a = 0; a < 3; ++a)
        for (int c = 0; c <= a; ++c) A[a][c] = FMA(g2m[a], m[c], g1g[a] * g[c]);
    for (int a = 0; a < 3; ++a) {
        A[a][a] = A[a][a] + g3;
        b[a] = FMA(-g2m[a], cr, FMA(-g1g[a], cY, g3 * wp[a]));
    }
    const real r0 = R(1) / A[0][0];
    const real l10 = A[1][0] * r0, l20 = A[2][0] * r0;
    const real d1 = FMA(-l10, A[1][0], A[1][1]);
    const real r1 = R(1) / d1;
    const real t = FMA(-l20, A[1][0], A[2][1]);
    const real l21 = t * r1;
    const real d2 = FMA(-l21, t, FMA(-l20, A[2][0], A[2][2]));
    const real r2 = R(1) / d2;
    const real y1 = FMA(-l10, b[0], b[1]);
    const real y2 = FMA(-l21, y1, FMA(-l20, b[0], b[2]));
    x[2] = y2 * r2;
    x[1] = FMA(-l21, x[2], y1 * r1);
    x[0] = FMA(-l20, x[2], FMA(-l10, x[1], b[0] * r0));
}

/* Batch entry point for the L1 pin: n independent pixel systems; gam = (g1, g2, g3). */
void or_ls_solve_batch(long n, const real* g, const real* m, const real* cY, const real* cr, const real* wp,
                       const double* gam, real* out)
{
    for (long p = 0; p < n; ++p)
        ls_solve(g + 3 * p, m + 3 * p, cY[p], cr[p], wp + 3 * p, R(gam[0]), R(gam[1]), R(gam[2]), out + 3 * p);
}

/* ------------------------------------------------------------------ smoothing (U4)
 * "average smoothing filter of size 5x5" applied S times to w after the solve (L590, L796,
 * reading 13): each iteration a horizontal 5-sum (left to right, replicate border), then a
 * vertical 5-sum (top to bottom), then division by 25.
 */
void or_smooth(int H, int W, int S, real* w)
{
    const long n = (long)H * W;
    real* t = malloc(sizeof(real) * 3 * n);
    for (int it = 0; it < S; ++it) {
        for (int i = 0; i < H; ++i)
            for (int j = 0; j < W; ++j)
                for (int a = 0; a < 3; ++a) {
                    real acc = w[3 * ((long)i * W + clampi(j - 2, 0, W - 1)) + a];
                    for (int k = -1; k <= 2; ++k) acc = acc + w[3 * ((long)i * W + clampi(j + k, 0, W - 1)) + a];
                    t[3 * ((long)i * W + j) + a] = acc;
                }
        for (int i = 0; i < H; ++i)
            for (int j = 0; j < W; ++j)
                for (int a = 0; a < 3; ++a) {
                    real acc = t[3 * ((long)clampi(i - 2, 0, H - 1) * W + j) + a];
                    for (int k = -1; k <= 2; ++k) acc = acc + t[3 * ((long)clampi(i + k, 0, H - 1) * W + j) + a];
                    w[3 * ((long)i * W + j) + a] = acc / R(25);
                }
    }
    free(t);
}

/* ------------------------------------------------------------------ update (U1-U6)
 * k+ -> k+1 (L546-621).  State (w, rho, yhat) holds frame k on entry and k+1 on exit;
 * (wp, rhop) is the prediction k+.  Temporal references are yhat^k (L564) and rho^k (L572),
 * reading 9.  init != 0: first frame (L750): w = 0, rho = rhohat (0 where invalid), yhat = Yhat.
 * Fusion (L609-621): rho = rho^{k+} + kappa (rhohat - rho^{k+}), kappa = g4/(g4+g5), 0 where invalid,
 * computed as fma(kappa, rhohat - rhop, rhop).
 */
unsigned or_update(const or_params* P, const real* geo, const float* Y, const float* depth, const real* wp,
                   const real* rhop, real* w, real* rho, real* yhat, int init)
{
    const int H = P->H, W = P->W;
    const long n = (long)H * W;
    unsigned flags = 0;
    real* yh1 = malloc(sizeof(real) * n);
    real* b1 = malloc(sizeof(real) * n);
    real* b2 = malloc(sizeof(real) * n);
    real* ghat = malloc(sizeof(real) * 3 * n);
    real* rh = malloc(sizeof(real) * n);
    real* br1 = malloc(sizeof(real) * n);
    real* br2 = malloc(sizeof(real) * n);
    real* drho = malloc(sizeof(real) * 3 * n);
    unsigned char* valid = malloc(n);
    for (long p = 0; p < n; ++p)
        if (!isfinite(Y[p])) flags |= OR_FLAG_NONFINITE;
    or_brightness_model(H, W, Y, geo, yh1, b1, b2, ghat);
    or_invdepth_model(H, W, depth, P->input_is_inverse_depth, geo, rh, valid, br1, br2, drho);
    if (init) {
        for (long p = 0; p < n; ++p) {
            w[3 * p] = w[3 * p + 1] = w[3 * p + 2] = R(0);
            rho[p] = rh[p];
            yhat[p] = yh1[p];
        }
    } else {
        const real g1 = R(P->gamma[0]), g2v = R(P->gamma[1]), g3 = R(P->gamma[2]);
        const real kap = R(P->gamma[3]) / (R(P->gamma[3]) + R(P->gamma[4]));
        real* wls = malloc(sizeof(real) * 3 * n);
        for (long p = 0; p < n; ++p) {
            const real* s = geo + 10 * p;
            const real d2 = geo[10 * p + 9];
            const real d2r = d2 * rh[p];
            real m[3];
            for (int a = 0; a < 3; ++a) m[a] = FMA(d2r, s[a], drho[3 * p + a]);
            const real cY = d2 * (yh1[p] - yhat[p]);
            const real cr = d2 * (rh[p] - rho[p]);
            ls_solve(ghat + 3 * p, m, cY, cr, wp + 3 * p, g1, valid[p] ? g2v : R(0), g3, wls + 3 * p);
        }
        or_smooth(H, W, P->smooth_iters, wls);
        for (long p = 0; p < n; ++p) {
            for (int a = 0; a < 3; ++a) w[3 * p + a] = wls[3 * p + a];
            const real kappa = valid[p] ? kap : R(0);
            rho[p] = FMA(kappa, rh[p] - rhop[p], rhop[p]);
            yhat[p] = yh1[p];
        }
        free(wls);
    }
    for (long p = 0; p < n; ++p)
        if (!isfinite(w[3 * p]) || !isfinite(w[3 * p + 1]) || !isfinite(w[3 * p + 2]) || !isfinite(rho[p]))
            flags |= OR_FLAG_NONFINITE;
    free(yh1);
    free(b1);
    free(b2);
    free(ghat);
    free(rh);
    free(br1);
    free(br2);
    free(drho);
    free(valid);
    return flags;
}

/* One frame k -> k+1: predict (P1-P5) then update (U1-U6), Fig. 3a (L385, L397-401).
 * init != 0 runs only the first-frame initialisation.  If wp_out/rhop_out are non-NULL the
 * prediction (w^{k+}, rho^{k+}) is copied there. */
unsigned or_step(const or_params* P, const real* geo, const float* Y, const float* depth, real* w, real* rho,
                 real* yhat, int init, real* wp_out, real* rhop_out)
{
    const long n = (long)P->H * P->W;
    if (init) return or_update(P, geo, Y, depth, NULL, NULL, w, rho, yhat, 1);
    real* wp = malloc(sizeof(real) * 3 * n);
    real* rp = malloc(sizeof(real) * n);
    memcpy(wp, w, sizeof(real) * 3 * n);
    memcpy(rp, rho, sizeof(real) * n);
    unsigned flags = or_predict(P, geo, wp, rp);
    if (wp_out) memcpy(wp_out, wp, sizeof(real) * 3 * n);
    if (rhop_out) memcpy(rhop_out, rp, sizeof(real) * n);
    flags |= or_update(P, geo, Y, depth, wp, rp, w, rho, yhat, 0);
    free(wp);
    free(rp);
    return flags;
}

int or_real_bytes(void) { return (int)sizeof(real); }

/* ------------------------------------------------------------------ evaluation outputs (NEXT #3)
 * Tangent flow (eq:tangent_flow, L736-743) and normal flow (eq:normal_flow, L744-747), in pixels:
 *   sw = <s, w>;  t = P(s) w = w - s sw  (eq:tmatrix L124-128):  t_a = fma(-s_a, sw, w_a)
 *   w_perp = B^T P(s) w / ds, evaluated as (e1 . t, e2 . t) with the filter's e_k = b_k / ds
 *            (reading 23: B^T/ds is the same linear map the filter uses for the optical flow,
 *             eq:oflow_numeric L639-642, reading 5)
 *   w_par  = sw / ds
 * g10 supplies the raw pixel separation ds (Spherepix input, L437); geo the filter's (s, e1, e2).
 */
void or_flow_px(long n, const float* g10, const real* geo, const real* w, real* tangent, real* normal)
{
    for (long p = 0; p < n; ++p) {
        const real* g = geo + 10 * p;
        const real* wp = w + 3 * p;
        const real ds = R(g10[10 * p + 9]);
        const real sw = dot3(g, wp);
        real t[3];
        for (int a = 0; a < 3; ++a) t[a] = FMA(-g[a], sw, wp[a]);
        if (tangent) {
            tangent[2 * p] = dot3(g + 3, t);
            tangent[2 * p + 1] = dot3(g + 6, t);
        }
        if (normal) normal[p] = sw / ds;
    }
}

/* RMSE (eq:RMSE_vel, L727-730) and AAE (L731-734) of w against the ground truth w_gt, per pixel:
 *   d_a = (w_gt_a - w_a) / ds;   rmse = sqrt(fma(d_z, d_z, fma(d_y, d_y, d_x d_x)))   [px/frame, real]
 *   AAE in double (an evaluation metric, not a filter decision; float32 would floor it at ~0.02 deg):
 *   a = w_gt / ds, b = w / ds (px/frame, reading 22: Barron's homogeneous form, squared norms)
 *   c = (1 + a.b) / (sqrt(1 + a.a) sqrt(1 + b.b)), clamped to [-1, 1];  aae = acos(c) * 180/pi
 * (dot products in dot3 order, explicit fma; every double op IEEE-rounded).  sums[0] += rmse and
 * sums[1] += aae over the n pixels, in pixel order, in double.
 */
static inline double ddot3(const double* a, const double* x) { return fma(a[2], x[2], fma(a[1], x[1], a[0] * x[0])); }

void or_eval(long n, const float* g10, const real* wgt, const real* w, real* rmse, double* aae_cos, double* aae_deg,
             double* sums)
{
    double s0 = 0.0, s1 = 0.0;
    for (long p = 0; p < n; ++p) {
        const real ds = R(g10[10 * p + 9]);
        real d[3];
        double a[3], b[3];
        for (int k = 0; k < 3; ++k) {
            d[k] = (wgt[3 * p + k] - w[3 * p + k]) / ds;
            a[k] = (double)wgt[3 * p + k] / (double)g10[10 * p + 9];
            b[k] = (double)w[3 * p + k] / (double)g10[10 * p + 9];
        }
#ifdef OR_F32
        const real e = sqrtf(dot3(d, d));
#else
        const real e = sqrt(dot3(d, d));
#endif
        double c = (1.0 + ddot3(a, b)) / (sqrt(1.0 + ddot3(a, a)) * sqrt(1.0 + ddot3(b, b)));
        c = fmin(fmax(c, -1.0), 1.0);
        const double ang = acos(c) * (180.0 / 3.14159265358979323846);
        if (rmse) rmse[p] = e;
        if (aae_cos) aae_cos[p] = c;
        if (aae_deg) aae_deg[p] = ang;
        s0 += (double)e;
        s1 += ang;
    }
    if (sums) {
        sums[0] += s0;
        sums[1] += s1;
    }
}

/* ================================================================== H = 2 pyramid (NEXT #1)
 * Two levels (L358-404, Fig. 3): the top level h = 2 runs the H = 1 filter above on the
 * half-resolution grid with down-sampled measurements; the bottom level h = 1 keeps the
 * increment state (dw, rho) (L362-366), transports (w, dw, rho, Y) by the reconstructed flow w
 * (L525-536, eq:hflow_propagation_low .. eq:img_propagation_low; numerical scheme L662-683),
 * updates dw by the increment LS (eq:cost_bottom, L592-607) and reconstructs
 * w = up(w^2) + dw (eq:hflow_reconstruction, L368-372).  Readings 24-30:
 *   24  down-sampling (unspecified): 2x2 mean, Y2 = ((Y00 + Y01) + (Y10 + Y11)) * 0.25;
 *       depth likewise when all four samples are valid, else invalid (NaN).
 *   25  up-sampling: bilinear at the fine pixel centres (coarse coordinate (i - 1/2)/2), weights
 *       (3/4, 1/4), replicate border: h_r = fma(wc1, X[r][c1], X[r][c0] * wc0) per coarse row r,
 *       then up = fma(wr1, h_r1, h_r0 * wr0).
 *   26  the bottom level transports rho by the reconstructed flow w^h (L531 prints w^H).
 *   27  the bottom-level dilation terms use sigma <s, w> like the top level (reading 2); Y has
 *       none (eq:img_propagation_low).
 *   28  the bottom update uses rho^{k+} and Yhat^{k+} (the transported fields) as printed
 *       (L597-600), the prior dw^{k+} (L601), then S_1 box iterations on dw and the rho fusion.
 *   29  per-level parameters: N_1 = ceil(max_flow), N_2 = ceil(max_flow / 2) (flows halve on the
 *       half grid), smoothing [S_1, S_2] = [2, 4] (Table 3 caption, L803-811).
 *   30  first frame: top level as H = 1; bottom dw = 0, rho = rhohat, Yhat = Yhat(Y), w = up(0) + 0.
 * Bottom-level state per pixel: F[8] = (w.x, w.y, w.z, dw.x, dw.y, dw.z, rho, Yhat).
 */
void or_down2(int H, int W, const float* Y, const float* depth, int is_inverse, float* Y2, float* D2)
{
    const int Hc = H / 2, Wc = W / 2;
    for (int I = 0; I < Hc; ++I)
        for (int J = 0; J < Wc; ++J) {
            const long a = (long)(2 * I) * W + 2 * J, b = a + W;
            const long o = (long)I * Wc + J;
            if (Y2) Y2[o] = ((Y[a] + Y[a + 1]) + (Y[b] + Y[b + 1])) * 0.25f;
            if (D2) {
                const float d[4] = {depth[a], depth[a + 1], depth[b], depth[b + 1]};
                int ok = 1;
                for (int k = 0; k < 4; ++k)
                    ok &= is_inverse ? (isfinite(d[k]) && d[k] >= 0.0f) : (isfinite(d[k]) && d[k] > 0.0f);
                D2[o] = ok ? ((d[0] + d[1]) + (d[2] + d[3])) * 0.25f : NAN;
            }
        }
}

/* Bilinear 2x up-sampling of a coarse [Hc][Wc][3] field to [2Hc][2Wc][3] (reading 25). */
void or_up2(int Hc, int Wc, const real* X, real* out)
{
    const int H = 2 * Hc, W = 2 * Wc;
    for (int i = 0; i < H; ++i) {
        const int I = i >> 1;
        const int r0 = (i & 1) ? I : clampi(I - 1, 0, Hc - 1), r1 = (i & 1) ? clampi(I + 1, 0, Hc - 1) : I;
        const real wr0 = (i & 1) ? R(0.75) : R(0.25), wr1 = (i & 1) ? R(0.25) : R(0.75);
        for (int j = 0; j < W; ++j) {
            const int J = j >> 1;
            const int c0 = (j & 1) ? J : clampi(J - 1, 0, Wc - 1), c1 = (j & 1) ? clampi(J + 1, 0, Wc - 1) : J;
            const real wc0 = (j & 1) ? R(0.75) : R(0.25), wc1 = (j & 1) ? R(0.25) : R(0.75);
            for (int a = 0; a < 3; ++a) {
                const real h0 = FMA(wc1, X[3 * ((long)r0 * Wc + c1) + a], X[3 * ((long)r0 * Wc + c0) + a] * wc0);
                const real h1 = FMA(wc1, X[3 * ((long)r1 * Wc + c1) + a], X[3 * ((long)r1 * Wc + c0) + a] * wc0);
                out[3 * ((long)i * W + j) + a] = FMA(wr1, h1, h0 * wr0);
            }
        }
    }
}

/* One bottom-level transport pass (axis as in pass()): the dominant flow from the reconstructed
 * w, then for c = 0..6 f* = fma(-dt, fma(u_hat, D, f * (sigma <s,w>)), f) and for Yhat (c = 7)
 * f* = fma(-dt, u_hat * D, f). */
static unsigned pass_low(const or_params* P, const real* geo, int axis, const real* F, real* Fo, real* u)
{
    const int H = P->H, W = P->W;
    const real U = R(P->max_flow), sigma = R(P->sigma), dt = R(1) / R(P->N);
    unsigned flags = 0;
    for (long p = 0; p < (long)H * W; ++p) u[p] = dot3(geo + 10 * p + 3 + 3 * axis, F + 8 * p);
    for (int i = 0; i < H; ++i)
        for (int j = 0; j < W; ++j) {
            const long p = (long)i * W + j;
            long pm, pp;
            if (axis == 0) {
                pm = (long)i * W + clampi(j - 1, 0, W - 1);
                pp = (long)i * W + clampi(j + 1, 0, W - 1);
            } else {
                pm = (long)clampi(i - 1, 0, H - 1) * W + j;
                pp = (long)clampi(i + 1, 0, H - 1) * W + j;
            }
            const real um = u[pm], up = u[pp];
            real uh;
            if (P->dominant_rule == OR_DOM_PRINTED)
                uh = (FABS(up) - FABS(um) > R(0)) ? um : up;
            else
                uh = (FABS(um) > FABS(up)) ? um : up;
            if (P->clamp_advection) {
                if (FABS(uh) > U) flags |= OR_FLAG_CLAMPED;
                uh = FMIN(FMAX(uh, -U), U);
            } else if (dt * FABS(uh) > R(1)) {
                flags |= OR_FLAG_CFL;
            }
            const real q = sigma * dot3(geo + 10 * p, F + 8 * p);
            for (int c = 0; c < 8; ++c) {
                const real f = F[8 * p + c];
                const real D = (uh > R(0)) ? (f - F[8 * pm + c]) : (F[8 * pp + c] - f);
                Fo[8 * p + c] = (c < 7) ? FMA(-dt, FMA(uh, D, f * q), f) : FMA(-dt, uh * D, f);
            }
        }
    return flags;
}

/* The two-level filter state. */
typedef struct {
    or_params top, low;          /* per-level parameters (reading 29) */
    const real* geo2;            /* [Hc][Wc][10] working geometry of the top level */
    const real* geo1;            /* [H][W][10] of the bottom level */
    real *w2, *rho2, *yhat2;     /* top level state */
    real* F;                     /* bottom level [H][W][8] */
} or_pyr;

/* One frame of the H = 2 filter (init != 0: first frame).  Y, depth: [H][W] full resolution.
 * scratch: Y2, D2 [Hc][Wc] float.  Returns the flags of both levels. */
unsigned or_pyr_step(const or_pyr* S, const float* Y, const float* depth, float* Y2, float* D2, int init)
{
    const or_params* P = &S->low;
    const int H = P->H, W = P->W, Hc = S->top.H, Wc = S->top.W;
    const long n = (long)H * W;
    unsigned flags = 0;
    or_down2(H, W, Y, depth, P->input_is_inverse_depth, Y2, D2);
    flags |= or_step(&S->top, S->geo2, Y2, D2, S->w2, S->rho2, S->yhat2, init, NULL, NULL);

    real* yh1 = malloc(sizeof(real) * n);
    real* b1 = malloc(sizeof(real) * n);
    real* b2 = malloc(sizeof(real) * n);
    real* ghat = malloc(sizeof(real) * 3 * n);
    real* rh = malloc(sizeof(real) * n);
    real* br1 = malloc(sizeof(real) * n);
    real* br2 = malloc(sizeof(real) * n);
    real* drho = malloc(sizeof(real) * 3 * n);
    unsigned char* valid = malloc(n);
    real* up = malloc(sizeof(real) * 3 * n);
    real* F = S->F;
    for (long p = 0; p < n; ++p)
        if (!isfinite(Y[p])) flags |= OR_FLAG_NONFINITE;
    or_brightness_model(H, W, Y, S->geo1, yh1, b1, b2, ghat);
    or_invdepth_model(H, W, depth, P->input_is_inverse_depth, S->geo1, rh, valid, br1, br2, drho);
    if (init) {
        for (long p = 0; p < n; ++p) {
            for (int c = 3; c < 6; ++c) F[8 * p + c] = R(0);
            F[8 * p + 6] = rh[p];
            F[8 * p + 7] = yh1[p];
        }
    } else {
        /* prediction [P_[]] (L525-536): N_1 substeps, column pass then row pass */
        real* F2 = malloc(sizeof(real) * 8 * n);
        real* u = malloc(sizeof(real) * n);
        for (int s = 0; s < P->N; ++s) {
            flags |= pass_low(P, S->geo1, 0, F, F2, u);
            flags |= pass_low(P, S->geo1, 1, F2, F, u);
        }
        free(F2);
        free(u);
        /* update [dU] (L592-607): solve for dw with prior dw^{k+}, references Yhat^{k+}, rho^{k+} */
        const real g1 = R(P->gamma[0]), g2v = R(P->gamma[1]), g3 = R(P->gamma[2]);
        const real kap = R(P->gamma[3]) / (R(P->gamma[3]) + R(P->gamma[4]));
        real* dw = malloc(sizeof(real) * 3 * n);
        for (long p = 0; p < n; ++p) {
            const real* s = S->geo1 + 10 * p;
            const real d2 = s[9];
            const real d2r = d2 * rh[p];
            real m[3];
            for (int a = 0; a < 3; ++a) m[a] = FMA(d2r, s[a], drho[3 * p + a]);
            const real cY = d2 * (yh1[p] - F[8 * p + 7]);
            const real cr = d2 * (rh[p] - F[8 * p + 6]);
            ls_solve(ghat + 3 * p, m, cY, cr, F + 8 * p + 3, g1, valid[p] ? g2v : R(0), g3, dw + 3 * p);
        }
        or_smooth(H, W, P->smooth_iters, dw);
        for (long p = 0; p < n; ++p) {
            for (int a = 0; a < 3; ++a) F[8 * p + 3 + a] = dw[3 * p + a];
            const real kappa = valid[p] ? kap : R(0);
            F[8 * p + 6] = FMA(kappa, rh[p] - F[8 * p + 6], F[8 * p + 6]);
            F[8 * p + 7] = yh1[p];
        }
        free(dw);
    }
    /* reconstruction [R] (eq:hflow_reconstruction): w = up(w^2) + dw */
    or_up2(Hc, Wc, S->w2, up);
    for (long p = 0; p < n; ++p)
        for (int a = 0; a < 3; ++a) F[8 * p + a] = up[3 * p + a] + F[8 * p + 3 + a];
    for (long p = 0; p < n; ++p)
        for (int c = 0; c < 7; ++c)
            if (!isfinite(F[8 * p + c])) flags |= OR_FLAG_NONFINITE;
    free(yh1);
    free(b1);
    free(b2);
    free(ghat);
    free(rh);
    free(br1);
    free(br2);
    free(drho);
    free(valid);
    free(up);
    return flags;
}

/* Flat-argument entry point for the Python binding. */
unsigned or_pyr_step_flat(const or_params* top, const or_params* low, const real* geo2, const real* geo1, real* w2,
                          real* rho2, real* yhat2, real* F, const float* Y, const float* depth, float* Y2, float* D2,
                          int init)
{
    or_pyr S = {*top, *low, geo2, geo1, w2, rho2, yhat2, F};
    return or_pyr_step(&S, Y, depth, Y2, D2, init);
}

/* Bottom-level prediction alone (for the pins): N substeps of pass_low on F [H][W][8], in place. */
unsigned or_predict_low(const or_params* P, const real* geo, real* F)
{
    const long n = (long)P->H * P->W;
    real* F2 = malloc(sizeof(real) * 8 * n);
    real* u = malloc(sizeof(real) * n);
    unsigned flags = 0;
    for (int s = 0; s < P->N; ++s) {
        flags |= pass_low(P, geo, 0, F, F2, u);
        flags |= pass_low(P, geo, 1, F2, F, u);
    }
    free(F2);
    free(u);
    return flags;
}

/* ================================================================== Spherepix input mapping (NEXT #2)
 * The measurements reach the filter on the Spherepix grid (L409); the paper's timed region
 * includes "the time required to map image and depth measurements onto the spherepix image"
 * (L785) but does not give the operator.  Reading 31: a pinhole camera with
 * intrinsics K = (fx, fy, cx, cy) (pixel centres at integer coordinates) and rotation Rcg
 * (grid -> camera, row-major 3x3); per grid pixel, in float32:
 *   t = Rcg s (row r: dot3(R_r, s));  xn = t.x / t.z, yn = t.y / t.z;
 *   u = fma(fx, xn, cx), v = fma(fy, yn, cy)            (camera pixel coordinates)
 *   brightness: (u, v) clamped to [0, Wc-1] x [0, Hc-1]; j0 = floor(u), i0 = floor(v),
 *     b = u - j0, a = v - i0, j1 = min(j0+1, Wc-1), i1 = min(i0+1, Hc-1);
 *     r0 = fma(b, Y[i0][j1] - Y[i0][j0], Y[i0][j0]), r1 = fma(b, Y[i1][j1] - Y[i1][j0], Y[i1][j0]),
 *     Y_grid = fma(a, r1 - r0, r0)
 *   depth (the camera gives z-depth): invalid (NaN) if t.z <= 0, (u, v) outside the image's
 *     pixel footprint [-1/2, Wc - 1/2] x [-1/2, Hc - 1/2] or any of the four samples invalid
 *     (not finite or <= 0); else z = the same bilinear form at the clamped position and
 *     lambda = z / t.z (range along s, since |s| = 1 and the point is lambda t).
 * t.z <= 0 also gives the brightness of the clamped position of (0, 0).
 */
void or_map_inputs(long n, const float* g10, const float* Rcg, const float* K, int Hc, int Wc, const float* Ycam,
                   const float* Zcam, float* Y, float* D)
{
    const float fx = K[0], fy = K[1], cx = K[2], cy = K[3];
    for (long p = 0; p < n; ++p) {
        const float* s = g10 + 10 * p;
        float t[3];
        for (int r = 0; r < 3; ++r) t[r] = fmaf(Rcg[3 * r + 2], s[2], fmaf(Rcg[3 * r + 1], s[1], Rcg[3 * r] * s[0]));
        const int front = t[2] > 0.0f;
        float u = 0.0f, v = 0.0f;
        if (front) {
            u = fmaf(fx, t[0] / t[2], cx);
            v = fmaf(fy, t[1] / t[2], cy);
        }
        const int inside = front && u >= -0.5f && u <= (float)Wc - 0.5f && v >= -0.5f && v <= (float)Hc - 0.5f;
        const float uc = fminf(fmaxf(u, 0.0f), (float)(Wc - 1)), vc = fminf(fmaxf(v, 0.0f), (float)(Hc - 1));
        const int j0 = (int)floorf(uc), i0 = (int)floorf(vc);
        const int j1 = j0 + 1 < Wc ? j0 + 1 : Wc - 1, i1 = i0 + 1 < Hc ? i0 + 1 : Hc - 1;
        const float b = uc - (float)j0, a = vc - (float)i0;
        const long q00 = (long)i0 * Wc + j0, q01 = (long)i0 * Wc + j1, q10 = (long)i1 * Wc + j0, q11 = (long)i1 * Wc + j1;
        {
            const float r0 = fmaf(b, Ycam[q01] - Ycam[q00], Ycam[q00]);
            const float r1 = fmaf(b, Ycam[q11] - Ycam[q10], Ycam[q10]);
            Y[p] = fmaf(a, r1 - r0, r0);
        }
        const float z00 = Zcam[q00], z01 = Zcam[q01], z10 = Zcam[q10], z11 = Zcam[q11];
        const int zok = isfinite(z00) && z00 > 0.0f && isfinite(z01) && z01 > 0.0f && isfinite(z10) && z10 > 0.0f &&
                        isfinite(z11) && z11 > 0.0f;
        if (inside && zok) {
            const float r0 = fmaf(b, z01 - z00, z00);
            const float r1 = fmaf(b, z11 - z10, z10);
            D[p] = fmaf(a, r1 - r0, r0) / t[2];
        } else {
            D[p] = NAN;
        }
    }
}
