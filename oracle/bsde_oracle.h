/*
 * bsde_oracle.h -- CPU oracle for the multistep BSDE scheme of Kapllani & Teng,
 * "Multistep schemes for solving BSDEs on GPU" (arXiv 1909.13560).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant generator with the CUDA product path
 * (paper_1909_13560_b200/csrc, include/bsde.h).
 *
 * The oracle follows the paper step by step (PAPER.md = /root/reference/PAPER.md):
 *   grids                 PAPER.md:91 (Delta t), :334-337, :367-371 (box, balance rule)
 *   Gauss-Hermite         Eq. 21
 *   weights gamma         Tables 1-2, PAPER.md:235-269 (b == gamma, R1)
 *   spatial spline        not-a-knot cubic, tensor product for d>=2, Thomas algorithm
 *                         (R5, R14)
 *   clamping              PAPER.md:385 ("take the values on the boundaries")
 *   cell location         PAPER.md:391-392 (int((X-x_min)/dx))
 *   backward sweep        Eq. 20; z first, then y by Picard
 *                         (p = 30 fixed)
 *   forward SDE           Eq. 1, by "the Euler-Scheme"
 *   2-D bicubic           PAPER.md:406: first / mixed derivatives by 4th-order finite
 *                         differences, 16 coefficients per cell by a 16x16 mat-vec
 * Every function below cites the passage it follows.
 */
#ifndef BSDE_ORACLE_H
#define BSDE_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* status codes (oracle-local) */
enum { ORC_OK = 0, ORC_ERR_ARG = 1, ORC_ERR_RESOURCE = 2, ORC_ERR_SINGULAR = 3,
       ORC_ERR_DOMAIN = 4, ORC_ERR_STATE = 7, ORC_ERR_UNSUPPORTED = 8 };

/* driver ids: f(t, y, z) in the paper's convention -dy = f dt - z dW (Eq. 2) */
enum { ORC_DRV_ZERO = 0,       /* f = 0                                                */
       ORC_DRV_AFFINE = 1,     /* f = p0 y + sum_k p[1+k] z_k + p4  (Ex.3/4/5, P7 pin)   */
       ORC_DRV_EX1 = 2,        /* f = -y^3 + 5/2 y^2 - 3/2 y           (Eq. 22)          */
       ORC_DRV_EX2 = 3,        /* Eq. 24                                                 */
       ORC_DRV_DIFF_RATES = 4  /* f = -(r y + sum th_k z_k) + (R-r) max(sum pi_k z_k - y, 0)
                                  p0=r, p1=R, p2..4=theta_k, p5..7=pi_k  (R21) */ };

/* terminal ids: g(w) at W_T = w, in W-space (R20) */
enum { ORC_TERM_CONST = 0,     /* g = p0                                                 */
       ORC_TERM_POLY = 1,      /* g = prod_a (p[4a] + p[4a+1] w_a + p[4a+2] w_a^2 + p[4a+3] w_a^3) */
       ORC_TERM_LOGISTIC = 2,  /* g = logistic(sum_a w_a / sqrt(d) + T)   (Eq. 22 for d=1) */
       ORC_TERM_EX2 = 3,       /* g = ln(sin w + 3) exp(T^2)               (Eq. 24)        */
       ORC_TERM_CALL_W = 4,    /* S = p0 exp((p2 - p3^2/2) T + p3 w), g = (S - p1)^+ (Eq. 30/32) */
       ORC_TERM_SIN_SUM = 5,   /* g = sin(sum_a w_a + T)                   (Eq. 34)        */
       ORC_TERM_EXCHANGE_W = 6,/* S_k = p[k] exp((p[2+k] - s_k^2/2) T + (A w)_k), s=(p4,p5), rho=p6,
                                  g = (S_1 - S_2)^+                        (Eq. 36)        */
       ORC_TERM_GEO_BASKET_W = 7,/* S_k = p[k] exp((p4 - s_k^2/2) T + s_k w_k), s_k = p[5+k],
                                  G = (prod S_k)^(1/d), g = (G - p3)^+    (BASELINE cfg 5) */
       ORC_TERM_CALL_X = 8     /* forward-SDE payoff in the state x: g = (x_0 - p1)^+        */ };

/* forward process X of Eq. 1, diagonal diffusion, parameters sp;
   sp[9..11] = X_0 = x_0, the evaluation point of the solution (y_0, z_0) */
enum { ORC_SDE_BROWNIAN = 0,   /* a = 0, b = 1: X = W (Eq. 2)                              */
       ORC_SDE_GBM = 1,        /* a_k = sp[k] x_k, b_k = sp[3+k] x_k                       */
       ORC_SDE_OU = 2          /* a_k = sp[k] (sp[3+k] - x_k), b_k = sp[6+k]               */ };

/* spatial interpolation of a layer */
enum { ORC_INTERP_SPLINE = 0,  /* tensor not-a-knot cubic spline (Thomas)                  */
       ORC_INTERP_BICUBIC = 1  /* d = 2: FD (4th order) derivatives + 16-coefficient bicubic */ };

typedef struct {
  int32_t d;                 /* 1..3 */
  double  t0, T;
  int32_t N;
  int32_t Ky, Kz;            /* 1..6 */
  int32_t L;                 /* Gauss-Hermite nodes per axis, 1..64 */
  int64_t npts[3];           /* points per axis incl. both ends; 0 -> balance rule */
  double  xlo[3], xhi[3];
  int32_t r;                 /* balance rule interpolation order (4) */
  int32_t driver_id;   double dp[12];
  int32_t terminal_id; double tp[12];
  int32_t picard_max;  double picard_tol;   /* tol <= 0: exactly picard_max iterations */
  int32_t bootstrap;         /* 0: closed-form initial layers; 1: one-step scheme (K=1) */
  int32_t bootstrap_substeps;
  int32_t smoothing;         /* 0 off, 1 cell average at the payoff kink (R11) */
  int32_t nthreads;          /* OpenMP threads; 0 -> runtime default */
  int32_t sde_id;            /* ORC_SDE_*; 0: X = W */
  double  sp[12];
  int32_t interp;            /* ORC_INTERP_* */
} orc_config;

typedef struct orc_ctx orc_ctx;

/* ---- building blocks (exposed for the pin tests) ---- */
int  orc_gauss_hermite(int L, double* nodes, double* weights);           /* Eq. 21 */
int  orc_gamma(int K, int which /*0: Table 1 (y), 1: Table 2 (z)*/, double* g /*K+1*/);
int64_t orc_balance_npts(double width, double dt, int Ky, int Kz, int r);
int  orc_spline_moments(const double* F, int64_t P, double dx, double* M); /* Thomas, not-a-knot */
double orc_spline_eval(const double* F, const double* M, int64_t P, double xlo, double dx, double X);
int  orc_thomas(int64_t n, const double* a, const double* b, const double* c, const double* r, double* x);
int  orc_terminal(const orc_config* cfg, const double* w, double* y, double* z);
int  orc_exact(const orc_config* cfg, double t, const double* w, double* y, double* z);
double orc_driver(const orc_config* cfg, double t, double y, const double* z);
/* weights of the derivative at offset 0 of the degree-4 interpolant through the 5 nodes
   offsets[0..4] (unit spacing): exact for polynomials of degree <= 4 */
int  orc_fd_weights(const int* offsets, double* w);
/* 4th-order first derivative of a line of P >= 5 samples with spacing h (central in the
   interior, one-sided within 2 nodes of the ends) */
int  orc_fd_deriv(const double* f, int64_t P, double h, double* df);

/* ---- the solver ---- */
int  orc_create(const orc_config* cfg, orc_ctx** out);
int  orc_step(orc_ctx* ctx);                          /* one backward step n+1 -> n (Eq. 20) */
int  orc_solve(orc_ctx* ctx, double* y0, double* z0); /* to n = 0, then the evaluation point */
int  orc_level(const orc_ctx* ctx);
int  orc_get_layer(const orc_ctx* ctx, int field, double* dst, int64_t count);
int  orc_get_picard_counts(const orc_ctx* ctx, int32_t* dst, int64_t count);
int  orc_query_grid(const orc_ctx* ctx, int64_t* npts, double* dx);
/* one step from the current state at selected flat point indices, without advancing:
   out[(field) * count + s] for s < count, fields y, z_1..z_d */
int  orc_step_points(orc_ctx* ctx, int64_t count, const int64_t* idx, double* out, int32_t* picard);
/* value of the spline of the newest layer at an arbitrary point (all fields) */
int  orc_eval_newest(orc_ctx* ctx, const double* x, double* out);
void orc_destroy(orc_ctx* ctx);
const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
