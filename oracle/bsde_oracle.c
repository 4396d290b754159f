/*
 * bsde_oracle.c -- plain, slow, obviously-correct CPU oracle of the multistep
 * BSDE scheme (Kapllani & Teng, arXiv 1909.13560).
 *
 * TEST INFRASTRUCTURE ONLY (see bsde_oracle.h).  Compiled with
 *   gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC
 * (no FMA contraction, no fast-math).  OpenMP only over independent grid
 * points with a static schedule; every per-point loop is sequential in a fixed
 * order, so results do not depend on the thread count.
 *
 * Representation: the spatial spline of a layer is kept as values F plus
 * second-derivative "moments" M along each axis (tensor product for d >= 2),
 * i.e. NOT as B-spline coefficients, so the GPU's representation is
 * cross-checked.  Splines are solved by the Thomas algorithm.  Every
 * interpolation is a direct evaluation at X = x_i + sqrt(2 j dt) a_Lambda,
 * with per-coordinate clamping and int((X - x_min)/dx) cell location; no
 * stencil table is used.
 *
 * Parity pins: see tests/test_oracle_*.py and DESIGN.md section "Oracle pins".
 */
#include "bsde_oracle.h"
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <stdarg.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_PI 3.14159265358979323846264338327950288

static __thread char g_err[512];
static int fail(int code, const char* fmt, ...) {
  va_list ap; va_start(ap, fmt); vsnprintf(g_err, sizeof g_err, fmt, ap); va_end(ap);
  return code;
}
const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------- */
/* Gauss-Hermite rule, Eq. 21: nodes a_l are the roots of the
 * physicists' Hermite polynomial H_L, weights for the weight function e^{-a^2}.
 * Newton iteration on the orthonormal three-term recurrence in long double.   */
int orc_gauss_hermite(int L, double* nodes, double* weights) {
  if (L < 1 || L > 64) return fail(ORC_ERR_ARG, "L=%d outside 1..64", L);
  long double x[64], w[64];
  const long double pim4 = 0.7511255444649425l; /* pi^{-1/4} */
  long double z = 0.0l, z1, p1, p2, p3, pp = 0.0l;
  long double r[64];  /* r[i]: i-th largest root */
  int m = (L + 1) / 2;
  for (int i = 0; i < m; ++i) {
    /* initial guesses (asymptotic estimates of the largest roots, then extrapolation) */
    if (i == 0) z = sqrtl((long double)(2 * L + 1)) - 1.85575l * powl((long double)(2 * L + 1), -0.16667l);
    else if (i == 1) z = z - 1.14l * powl((long double)L, 0.426l) / z;
    else if (i == 2) z = 1.86l * z - 0.86l * r[0];
    else if (i == 3) z = 1.91l * z - 0.91l * r[1];
    else z = 2.0l * z - r[i - 2];
    for (int it = 0; it < 200; ++it) {
      p1 = pim4; p2 = 0.0l;
      for (int j = 1; j <= L; ++j) {
        p3 = p2; p2 = p1;
        p1 = z * sqrtl(2.0l / j) * p2 - sqrtl((long double)(j - 1) / j) * p3;
      }
      pp = sqrtl(2.0l * L) * p2;
      z1 = z;
      z = z1 - p1 / pp;
      if (fabsl(z - z1) <= 1e-19l * (1.0l + fabsl(z))) break;
    }
    r[i] = z;
    x[i] = z; x[L - 1 - i] = -z;
    w[i] = 2.0l / (pp * pp); w[L - 1 - i] = w[i];
  }
  if (L % 2 == 1) x[L / 2] = 0.0l;
  /* ascending order */
  for (int i = 0; i < L; ++i) { nodes[i] = (double)x[L - 1 - i]; weights[i] = (double)w[L - 1 - i]; }
  return ORC_OK;
}

/* Gauss-Legendre rule on [-1,1] (used only by the terminal smoothing, R11). */
static void gauss_legendre(int n, double* x, double* w) {
  for (int i = 0; i < (n + 1) / 2; ++i) {
    long double z = cosl(ORC_PI * (i + 0.75l) / (n + 0.5l)), z1, p1, p2, p3, pp = 1;
    for (int it = 0; it < 100; ++it) {
      p1 = 1.0l; p2 = 0.0l;
      for (int j = 1; j <= n; ++j) { p3 = p2; p2 = p1; p1 = ((2.0l * j - 1) * z * p2 - (j - 1.0l) * p3) / j; }
      pp = n * (z * p1 - p2) / (z * z - 1.0l);
      z1 = z; z = z1 - p1 / pp;
      if (fabsl(z - z1) < 1e-19l) break;
    }
    x[i] = (double)(-z); x[n - 1 - i] = (double)z;
    w[i] = w[n - 1 - i] = (double)(2.0l / ((1.0l - z * z) * pp * pp));
  }
}

/* ------------------------------------------------------------------------- */
/* Weights gamma: Table 1 (gamma^{Ky}_{Ky,j}) for the y-equation
 * and Table 2 (gamma^1_{Kz,j}) for the z-equation; Eq. 20 writes
 * them as b (R1).  Exact rationals as printed.                      */
int orc_gamma(int K, int which, double* g) {
  static const int ny[6][7] = {{1, 1}, {1, 2, 1}, {1, 3, 3, 1}, {1, 1, 1, 1, 1},
                               {41, 19, 107, 107, 19, 41}, {19, 3, 15, 4, 15, 3, 19}};
  static const int dy[6][7] = {{2, 2}, {6, 3, 6}, {8, 8, 8, 8}, {12, 3, 6, 3, 12},
                               {600, 75, 600, 600, 75, 600}, {336, 14, 112, 21, 112, 14, 336}};
  static const int nz[6][7] = {{1, 1}, {5, 2, -1}, {3, 19, -5, 1}, {35, 5, -13, 1, -1},
                               {131, 151, -103, 37, -1, 1}, {163, 47, -129, 3, -37, 1, -1}};
  static const int dz[6][7] = {{2, 2}, {12, 3, 12}, {8, 24, 24, 24}, {96, 6, 48, 12, 96},
                               {360, 180, 360, 360, 45, 360}, {448, 56, 448, 28, 1344, 168, 1344}};
  if (K < 1 || K > 6) return fail(ORC_ERR_ARG, "K=%d outside 1..6 (Tables 1-2)", K);
  for (int j = 0; j <= K; ++j)
    g[j] = which == 0 ? (double)ny[K - 1][j] / dy[K - 1][j] : (double)nz[K - 1][j] / dz[K - 1][j];
  return ORC_OK;
}

/* Balance rule: (dx)^r = (dt)^{q+1}.  Reading R3:
 * q = min{Ky+1, Kz, 3}, M = 2 ceil(X/dx) intervals on [-X, X], M+1 points.    */
int64_t orc_balance_npts(double width, double dt, int Ky, int Kz, int r) {
  int q = Ky + 1; if (Kz < q) q = Kz; if (3 < q) q = 3;
  double dxs = pow(dt, (double)(q + 1) / (double)r);
  double half = 0.5 * width;
  double cnt = half / dxs;
  int64_t c = (int64_t)ceil(cnt - 1e-9 * cnt);
  return 2 * c + 1;
}

/* ------------------------------------------------------------------------- */
/* Thomas algorithm for a tridiagonal system a_i x_{i-1} + b_i x_i + c_i x_{i+1} = r_i. */
int orc_thomas(int64_t n, const double* a, const double* b, const double* c, const double* r, double* x) {
  double* cp = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  if (!cp) return fail(ORC_ERR_RESOURCE, "oom");
  double beta = b[0];
  if (beta == 0.0) { free(cp); return fail(ORC_ERR_SINGULAR, "zero pivot"); }
  x[0] = r[0] / beta;
  for (int64_t i = 1; i < n; ++i) {
    cp[i - 1] = c[i - 1] / beta;
    beta = b[i] - a[i] * cp[i - 1];
    if (beta == 0.0) { free(cp); return fail(ORC_ERR_SINGULAR, "zero pivot"); }
    x[i] = (r[i] - a[i] * x[i - 1]) / beta;
  }
  for (int64_t i = n - 2; i >= 0; --i) x[i] -= cp[i] * x[i + 1];
  free(cp);
  return ORC_OK;
}

/* Not-a-knot cubic spline on a uniform line (reading R5): moments M_i = s''(x_i).
 * Interior rows M_{i-1} + 4 M_i + M_{i+1} = 6 (F_{i-1} - 2F_i + F_{i+1}) / dx^2,
 * not-a-knot M_0 = 2M_1 - M_2 and M_{P-1} = 2M_{P-2} - M_{P-3} (third derivative
 * continuous at x_1 and x_{P-2}); substituted, rows 1 and P-2 read 6 M = rhs.
 * Strided line: element i is F[i*fs], M[i*ms].  work: 4*P doubles.            */
static int line_moments(const double* F, int64_t fs, int64_t P, double dx, double* M, int64_t ms, double* work) {
  if (P < 4) return fail(ORC_ERR_ARG, "not-a-knot spline needs >= 4 points (P=%lld)", (long long)P);
  int64_t n = P - 2;
  double *a = work, *b = work + n, *c = work + 2 * n, *r = work + 3 * n;
  double inv = 6.0 / (dx * dx);
  for (int64_t k = 0; k < n; ++k) {
    int64_t i = k + 1;
    r[k] = inv * (F[(i - 1) * fs] - 2.0 * F[i * fs] + F[(i + 1) * fs]);
    a[k] = 1.0; b[k] = 4.0; c[k] = 1.0;
  }
  a[0] = 0.0; b[0] = 6.0; c[0] = 0.0;
  a[n - 1] = 0.0; b[n - 1] = 6.0; c[n - 1] = 0.0;
  double* x = (double*)malloc(sizeof(double) * (size_t)n);
  if (!x) return fail(ORC_ERR_RESOURCE, "oom");
  int st = orc_thomas(n, a, b, c, r, x);
  if (st) { free(x); return st; }
  for (int64_t k = 0; k < n; ++k) M[(k + 1) * ms] = x[k];
  M[0] = 2.0 * x[0] - x[1];
  M[(P - 1) * ms] = 2.0 * x[n - 1] - x[n - 2];
  free(x);
  return ORC_OK;
}

int orc_spline_moments(const double* F, int64_t P, double dx, double* M) {
  double* w = (double*)malloc(sizeof(double) * 4 * (size_t)(P > 4 ? P : 4));
  if (!w) return fail(ORC_ERR_RESOURCE, "oom");
  int st = line_moments(F, 1, P, dx, M, 1, w);
  free(w);
  return st;
}

/* clamp (reading R6) and locate the cell (R7) */
static inline int64_t locate(double X, double xlo, double xhi, double dx, int64_t P, double* t) {
  if (X < xlo) X = xlo;
  if (X > xhi) X = xhi;
  int64_t c = (int64_t)floor((X - xlo) / dx);
  if (c > P - 2) c = P - 2;
  if (c < 0) c = 0;
  *t = (X - (xlo + (double)c * dx)) / dx;
  return c;
}

/* cubic spline on a cell, t in [0,1]:
 * s = (1-t) F_c + t F_{c+1} + dx^2/6 [((1-t)^3 - (1-t)) M_c + (t^3 - t) M_{c+1}]  */
static inline void basis(double t, double dx, double* phi, double* psi) {
  double u = 1.0 - t, h2 = dx * dx / 6.0;
  phi[0] = u; phi[1] = t;
  psi[0] = h2 * (u * u * u - u); psi[1] = h2 * (t * t * t - t);
}

double orc_spline_eval(const double* F, const double* M, int64_t P, double xlo, double dx, double X) {
  double t, phi[2], psi[2];
  double xhi = xlo + (double)(P - 1) * dx;
  int64_t c = locate(X, xlo, xhi, dx, P, &t);
  basis(t, dx, phi, psi);
  return phi[0] * F[c] + phi[1] * F[c + 1] + psi[0] * M[c] + psi[1] * M[c + 1];
}

/* ------------------------------------------------------------------------- */
/* Problems: drivers f and terminal conditions g in W-space. */
static double logistic(double s) { return 1.0 / (1.0 + exp(-s)); }
static double ncdf(double x) { return 0.5 * erfc(-x / sqrt(2.0)); }

double orc_driver(const orc_config* cfg, double t, double y, const double* z) {
  const double* p = cfg->dp;
  int d = cfg->d;
  switch (cfg->driver_id) {
    case ORC_DRV_ZERO: return 0.0;
    case ORC_DRV_AFFINE: {                               /* Ex. 3 Eq. 29/30, Ex. 4 Eq. 34, Ex. 5 Eq. 36 */
      double f = p[0] * y;
      for (int k = 0; k < d; ++k) f += p[1 + k] * z[k];
      return f + p[4];
    }
    case ORC_DRV_EX1: return -y * y * y + 2.5 * y * y - 1.5 * y;   /* Eq. 22 */
    case ORC_DRV_EX2: {                                  /* Eq. 24 */
      double e = exp(t * t), ei = exp(-t * t);
      return 0.5 * (e - 4.0 * t * y - 3.0 * exp(t * t - y * ei) + z[0] * z[0] * ei);
    }
    case ORC_DRV_DIFF_RATES: {                           /* DESIGN.md R21 */
      double lin = p[0] * y, hold = 0.0;
      for (int k = 0; k < d; ++k) { lin += p[2 + k] * z[k]; hold += p[5 + k] * z[k]; }
      double b = hold - y;
      return -lin + (p[1] - p[0]) * (b > 0.0 ? b : 0.0);
    }
  }
  return NAN;
}

/* kink argument for the payoffs (S - K)^+ type: returns the signed argument */
static double payoff_arg(const orc_config* cfg, const double* w) {
  const double* p = cfg->tp;
  double T = cfg->T;
  switch (cfg->terminal_id) {
    case ORC_TERM_CALL_W: return p[0] * exp((p[2] - 0.5 * p[3] * p[3]) * T + p[3] * w[0]) - p[1];
    case ORC_TERM_EXCHANGE_W: {
      double s1 = p[4], s2 = p[5], rho = p[6];
      double aw1 = s1 * w[0], aw2 = rho * s2 * w[0] + s2 * sqrt(1.0 - rho * rho) * w[1];
      return p[0] * exp((p[2] - 0.5 * s1 * s1) * T + aw1) - p[1] * exp((p[3] - 0.5 * s2 * s2) * T + aw2);
    }
    case ORC_TERM_GEO_BASKET_W: {
      double lg = 0.0;
      for (int k = 0; k < cfg->d; ++k) lg += log(p[k]) + (p[4] - 0.5 * p[5 + k] * p[5 + k]) * T + p[5 + k] * w[k];
      return exp(lg / cfg->d) - p[3];
    }
  }
  return 0.0;
}

/* terminal condition y_T = g(W_T), z_T = grad g (Eq. 2, Eq. 4 z = grad u) */
int orc_terminal(const orc_config* cfg, const double* w, double* y, double* z) {
  const double* p = cfg->tp;
  int d = cfg->d;
  double T = cfg->T;
  for (int k = 0; k < d; ++k) z[k] = 0.0;
  switch (cfg->terminal_id) {
    case ORC_TERM_CONST: *y = p[0]; return ORC_OK;
    case ORC_TERM_POLY: {
      double fac[3], der[3];
      for (int a = 0; a < d; ++a) {
        double x = w[a];
        const double* c = p + 4 * a;
        fac[a] = c[0] + c[1] * x + c[2] * x * x + c[3] * x * x * x;
        der[a] = c[1] + 2.0 * c[2] * x + 3.0 * c[3] * x * x;
      }
      double prod = 1.0;
      for (int a = 0; a < d; ++a) prod *= fac[a];
      *y = prod;
      for (int a = 0; a < d; ++a) {
        double q = der[a];
        for (int b = 0; b < d; ++b) if (b != a) q *= fac[b];
        z[a] = q;
      }
      return ORC_OK;
    }
    case ORC_TERM_LOGISTIC: {
      double s = 0.0;
      for (int a = 0; a < d; ++a) s += w[a];
      s = s / sqrt((double)d) + T;
      double g = logistic(s);
      *y = g;
      for (int a = 0; a < d; ++a) z[a] = g * (1.0 - g) / sqrt((double)d);
      return ORC_OK;
    }
    case ORC_TERM_EX2: {
      double e = exp(T * T);
      *y = log(sin(w[0]) + 3.0) * e;
      z[0] = e * cos(w[0]) / (sin(w[0]) + 3.0);
      return ORC_OK;
    }
    case ORC_TERM_CALL_W: {
      double S = p[0] * exp((p[2] - 0.5 * p[3] * p[3]) * T + p[3] * w[0]);
      *y = S > p[1] ? S - p[1] : 0.0;
      z[0] = S > p[1] ? p[3] * S : 0.0;
      return ORC_OK;
    }
    case ORC_TERM_SIN_SUM: {
      double s = T;
      for (int a = 0; a < d; ++a) s += w[a];
      *y = sin(s);
      for (int a = 0; a < d; ++a) z[a] = cos(s);
      return ORC_OK;
    }
    case ORC_TERM_EXCHANGE_W: {
      if (d != 2) return fail(ORC_ERR_ARG, "exchange payoff needs d=2");
      double s1 = p[4], s2 = p[5], rho = p[6];
      double a21 = rho * s2, a22 = s2 * sqrt(1.0 - rho * rho);
      double S1 = p[0] * exp((p[2] - 0.5 * s1 * s1) * T + s1 * w[0]);
      double S2 = p[1] * exp((p[3] - 0.5 * s2 * s2) * T + a21 * w[0] + a22 * w[1]);
      if (S1 > S2) {
        *y = S1 - S2;
        z[0] = s1 * S1 - a21 * S2;   /* A^T (S1, -S2) */
        z[1] = -a22 * S2;
      } else *y = 0.0;
      return ORC_OK;
    }
    case ORC_TERM_GEO_BASKET_W: {
      double lg = 0.0;
      for (int k = 0; k < d; ++k) lg += log(p[k]) + (p[4] - 0.5 * p[5 + k] * p[5 + k]) * T + p[5 + k] * w[k];
      double G = exp(lg / d);
      if (G > p[3]) {
        *y = G - p[3];
        for (int k = 0; k < d; ++k) z[k] = G * p[5 + k] / d;
      } else *y = 0.0;
      return ORC_OK;
    }
    case ORC_TERM_CALL_X: {          /* payoff in the state variable of Eq. 1: g(x) = (x_0 - K)^+ */
      if (w[0] > p[1]) { *y = w[0] - p[1]; z[0] = 1.0; } else *y = 0.0;
      return ORC_OK;                 /* z = grad g here; fill_layer applies b (z = b^T grad u) */
    }
  }
  return fail(ORC_ERR_ARG, "unknown terminal id %d", cfg->terminal_id);
}

/* Black-Scholes price/delta*S with dividend yield q (Eq. 31 with delta in d1, reading R13) */
static void bs_call(double S, double K, double r, double q, double sig, double tau, double* V, double* SdV) {
  if (tau <= 0.0) { *V = S > K ? S - K : 0.0; *SdV = S > K ? S : 0.0; return; }
  double st = sig * sqrt(tau);
  double d1 = (log(S / K) + (r - q + 0.5 * sig * sig) * tau) / st, d2 = d1 - st;
  *V = S * exp(-q * tau) * ncdf(d1) - K * exp(-r * tau) * ncdf(d2);
  *SdV = S * exp(-q * tau) * ncdf(d1);
}

/* closed-form solutions (y, z) = (u, grad u)(t, w) used for the K-1 initial layers
 * (reading R9) -- Eq. 23, Eq. 25, Eq. 31, Eq. 35, Eq. 37 and DESIGN.md R21.     */
int orc_exact(const orc_config* cfg, double t, const double* w, double* y, double* z) {
  const double* p = cfg->tp;
  const double* q = cfg->dp;
  int d = cfg->d;
  double T = cfg->T, tau = T - t;
  int tid = cfg->terminal_id, did = cfg->driver_id;
  for (int k = 0; k < d; ++k) z[k] = 0.0;
  if (cfg->sde_id != ORC_SDE_BROWNIAN && !(tid == ORC_TERM_CONST && did == ORC_DRV_ZERO))
    return fail(ORC_ERR_UNSUPPORTED, "no closed form for a forward-SDE problem: use bootstrap = 1");
  if (tau == 0.0) return orc_terminal(cfg, w, y, z);
  if (tid == ORC_TERM_CONST && (did == ORC_DRV_ZERO || (did == ORC_DRV_AFFINE && q[1] == 0 && q[2] == 0 && q[3] == 0))) {
    double a = did == ORC_DRV_ZERO ? 0.0 : q[0], c0 = did == ORC_DRV_ZERO ? 0.0 : q[4];
    *y = a != 0.0 ? (p[0] + c0 / a) * exp(a * tau) - c0 / a : p[0] + c0 * tau;
    return ORC_OK;
  }
  if (tid == ORC_TERM_POLY && (did == ORC_DRV_ZERO || (did == ORC_DRV_AFFINE && q[1] == 0 && q[2] == 0 && q[3] == 0 && q[4] == 0))) {
    double a = did == ORC_DRV_ZERO ? 0.0 : q[0];
    double fac[3], der[3];
    for (int ax = 0; ax < d; ++ax) {           /* E[poly(x + sqrt(tau) N)] per axis */
      double x = w[ax];
      const double* c = p + 4 * ax;
      fac[ax] = c[0] + c[1] * x + c[2] * (x * x + tau) + c[3] * (x * x * x + 3.0 * tau * x);
      der[ax] = c[1] + 2.0 * c[2] * x + 3.0 * c[3] * (x * x + tau);
    }
    double e = exp(a * tau), prod = 1.0;
    for (int ax = 0; ax < d; ++ax) prod *= fac[ax];
    *y = e * prod;
    for (int ax = 0; ax < d; ++ax) {
      double v = der[ax];
      for (int b = 0; b < d; ++b) if (b != ax) v *= fac[b];
      z[ax] = e * v;
    }
    return ORC_OK;
  }
  if (tid == ORC_TERM_LOGISTIC && did == ORC_DRV_EX1) {  /* Eq. 23 */
    double s = 0.0;
    for (int a = 0; a < d; ++a) s += w[a];
    s = s / sqrt((double)d) + t;
    double g = logistic(s);
    *y = g;
    for (int a = 0; a < d; ++a) z[a] = g * (1.0 - g) / sqrt((double)d);
    return ORC_OK;
  }
  if (tid == ORC_TERM_EX2 && did == ORC_DRV_EX2) {        /* Eq. 25 */
    double e = exp(t * t);
    *y = log(sin(w[0]) + 3.0) * e;
    z[0] = e * cos(w[0]) / (sin(w[0]) + 3.0);
    return ORC_OK;
  }
  if (tid == ORC_TERM_CALL_W && (did == ORC_DRV_AFFINE || did == ORC_DRV_DIFF_RATES) && d == 1) {  /* Eq. 31 */
    double S0 = p[0], K = p[1], mu = p[2], sig = p[3];
    double r, th;
    if (did == ORC_DRV_AFFINE) { r = -q[0]; th = -q[1]; }
    else { r = q[0]; th = q[2]; }
    double del = th * sig - mu + r;
    double rate = did == ORC_DRV_AFFINE ? r : q[1];
    double S = S0 * exp((mu - 0.5 * sig * sig) * t + sig * w[0]);
    double V, SdV;
    bs_call(S, K, rate, del, sig, tau, &V, &SdV);
    *y = V; z[0] = sig * SdV;
    return ORC_OK;
  }
  if (tid == ORC_TERM_SIN_SUM && did == ORC_DRV_AFFINE) {  /* Eq. 35 */
    double s = t;
    for (int a = 0; a < d; ++a) s += w[a];
    *y = sin(s);
    for (int a = 0; a < d; ++a) z[a] = cos(s);
    return ORC_OK;
  }
  if (tid == ORC_TERM_EXCHANGE_W && did == ORC_DRV_AFFINE && d == 2) {  /* Eq. 37 (Margrabe) */
    double s1 = p[4], s2 = p[5], rho = p[6];
    double a21 = rho * s2, a22 = s2 * sqrt(1.0 - rho * rho);
    double S1 = p[0] * exp((p[2] - 0.5 * s1 * s1) * t + s1 * w[0]);
    double S2 = p[1] * exp((p[3] - 0.5 * s2 * s2) * t + a21 * w[0] + a22 * w[1]);
    double st = sqrt(s1 * s1 + s2 * s2 - 2.0 * rho * s1 * s2);
    double sq = st * sqrt(tau);
    double d1 = (log(S1 / S2) + 0.5 * st * st * tau) / sq, d2 = d1 - sq;
    double n1 = ncdf(d1), n2 = ncdf(d2);
    *y = S1 * n1 - S2 * n2;
    z[0] = s1 * S1 * n1 - a21 * S2 * n2;
    z[1] = -a22 * S2 * n2;
    return ORC_OK;
  }
  if (tid == ORC_TERM_GEO_BASKET_W && did == ORC_DRV_DIFF_RATES) {  /* DESIGN.md R21 */
    double lg = 0.0, ss = 0.0;
    for (int k = 0; k < d; ++k) {
      lg += log(p[k]) + (p[4] - 0.5 * p[5 + k] * p[5 + k]) * t + p[5 + k] * w[k];
      ss += p[5 + k] * p[5 + k];
    }
    double G = exp(lg / d);
    double sg = sqrt(ss) / d;
    double qg = ss / (2.0 * d) - 0.5 * sg * sg;
    double V, GdV;
    bs_call(G, p[3], q[1], qg, sg, tau, &V, &GdV);
    *y = V;
    for (int k = 0; k < d; ++k) z[k] = GdV * p[5 + k] / d;
    return ORC_OK;
  }
  return fail(ORC_ERR_UNSUPPORTED, "no closed form for terminal %d with driver %d", tid, did);
}

/* Terminal smoothing ("cf. Kreiss"; reading R11, parity unpinned):
 * at grid points whose cell [x - dx/2, x + dx/2]^d meets the payoff kink, y^N is the
 * cell average of g and z^N the gradient of the cell average (difference of face
 * averages).  d = 1 call: closed-form integral; otherwise tensor Gauss-Legendre, 16
 * nodes per axis.                                                                  */
#define SMOOTH_GL 16
static int kink_in_cell(const orc_config* cfg, const double* x, const double* h) {
  int d = cfg->d, pos = 0, neg = 0;
  for (int m = 0; m < (1 << d); ++m) {
    double c[3];
    for (int a = 0; a < d; ++a) c[a] = x[a] + ((m >> a) & 1 ? 0.5 : -0.5) * h[a];
    double v = payoff_arg(cfg, c);
    if (v > 0.0) pos = 1; else if (v < 0.0) neg = 1; else { pos = 1; neg = 1; }
  }
  return pos && neg;
}
static double call_avg(const orc_config* cfg, double lo, double hi) {
  const double* p = cfg->tp;
  double T = cfg->T, a = (p[2] - 0.5 * p[3] * p[3]) * T, s = p[3];
  double wk = (log(p[1] / p[0]) - a) / s;
  if (hi <= wk) return 0.0;
  double l = lo > wk ? lo : wk;
  return (p[0] * exp(a) * (exp(s * hi) - exp(s * l)) / s - p[1] * (hi - l)) / (hi - lo);
}
static double payoff_val(const orc_config* cfg, const double* w) {
  double y, z[3];
  orc_terminal(cfg, w, &y, z);
  return y;
}
/* average of g over the box prod_a [lo_a, hi_a] with axis `fixed` (if >= 0) pinned to lo */
static double box_avg(const orc_config* cfg, const double* lo, const double* hi, int fixed,
                      const double* gx, const double* gw) {
  int d = cfg->d;
  int n[3], tot = 1;
  for (int a = 0; a < d; ++a) { n[a] = (a == fixed) ? 1 : SMOOTH_GL; tot *= n[a]; }
  double acc = 0.0;
  for (int m = 0; m < tot; ++m) {
    int rem = m;
    double w[3], wt = 1.0;
    for (int a = d - 1; a >= 0; --a) {
      int k = rem % n[a]; rem /= n[a];
      if (a == fixed) { w[a] = lo[a]; }
      else {
        w[a] = 0.5 * (lo[a] + hi[a]) + 0.5 * (hi[a] - lo[a]) * gx[k];
        wt *= 0.5 * gw[k];
      }
    }
    acc += wt * payoff_val(cfg, w);
  }
  return acc;
}
static void smooth_point(const orc_config* cfg, const double* x, const double* h, double* y, double* z) {
  int d = cfg->d;
  if (d == 1 && cfg->terminal_id == ORC_TERM_CALL_W) {
    *y = call_avg(cfg, x[0] - 0.5 * h[0], x[0] + 0.5 * h[0]);
    double wp = x[0] + 0.5 * h[0], wm = x[0] - 0.5 * h[0];
    z[0] = (payoff_val(cfg, &wp) - payoff_val(cfg, &wm)) / h[0];
    return;
  }
  double gx[SMOOTH_GL], gw[SMOOTH_GL];
  gauss_legendre(SMOOTH_GL, gx, gw);
  double lo[3], hi[3];
  for (int a = 0; a < d; ++a) { lo[a] = x[a] - 0.5 * h[a]; hi[a] = x[a] + 0.5 * h[a]; }
  *y = box_avg(cfg, lo, hi, -1, gx, gw);
  for (int a = 0; a < d; ++a) {
    double lo2[3], hi2[3];
    memcpy(lo2, lo, sizeof lo2); memcpy(hi2, hi, sizeof hi2);
    lo2[a] = hi[a];
    double up = box_avg(cfg, lo2, hi2, a, gx, gw);
    lo2[a] = lo[a];
    double dn = box_avg(cfg, lo2, hi2, a, gx, gw);
    z[a] = (up - dn) / h[a];
  }
}
static int kinked(int tid) {
  return tid == ORC_TERM_CALL_W || tid == ORC_TERM_EXCHANGE_W || tid == ORC_TERM_GEO_BASKET_W;
}

/* ------------------------------------------------------------------------- */
/* Forward SDE of Eq. 1, diagonal: drift a_k(x) and diffusion b_k(x). */
static void sde_coef(const orc_config* cfg, int k, double x, double* a, double* b) {
  const double* q = cfg->sp;
  switch (cfg->sde_id) {
    case ORC_SDE_GBM: *a = q[k] * x; *b = q[3 + k] * x; return;
    case ORC_SDE_OU: *a = q[k] * (q[3 + k] - x); *b = q[6 + k]; return;
  }
  *a = 0.0; *b = 1.0;
}

/* ------------------------------------------------------------------------- */
/* 4th-order finite differences ("finite difference schemes of the fourth order
 * of accuracy (central, forward and backward)").  The weights of the derivative at offset 0 of
 * the degree-4 interpolating polynomial through the 5 nodes `off` are the solution of
 * sum_k w_k off_k^m = [m == 1], m = 0..4 (the definition, solved by Gaussian elimination).   */
int orc_fd_weights(const int* off, double* w) {
  double A[5][6];
  for (int m = 0; m < 5; ++m) {
    for (int k = 0; k < 5; ++k) {
      double v = 1.0;
      for (int e = 0; e < m; ++e) v *= (double)off[k];
      A[m][k] = v;
    }
    A[m][5] = m == 1 ? 1.0 : 0.0;
  }
  for (int c = 0; c < 5; ++c) {
    int piv = c;
    for (int r = c + 1; r < 5; ++r) if (fabs(A[r][c]) > fabs(A[piv][c])) piv = r;
    if (A[piv][c] == 0.0) return fail(ORC_ERR_SINGULAR, "fd weights: repeated offsets");
    for (int k = 0; k < 6; ++k) { double t = A[c][k]; A[c][k] = A[piv][k]; A[piv][k] = t; }
    for (int r = 0; r < 5; ++r) {
      if (r == c) continue;
      double f = A[r][c] / A[c][c];
      for (int k = c; k < 6; ++k) A[r][k] -= f * A[c][k];
    }
  }
  for (int k = 0; k < 5; ++k) w[k] = A[k][5] / A[k][k];
  return ORC_OK;
}

/* first derivative of a line: central 5-point stencil (-2..2) in the interior, one-sided
 * 5-point stencils at the two nodes nearest each end (0..4, -1..3 and mirrored) */
static int fd_line(const double* f, int64_t fs, int64_t P, double h, double* df, int64_t ds) {
  static const int offs[5][5] = {{0, 1, 2, 3, 4}, {-1, 0, 1, 2, 3}, {-2, -1, 0, 1, 2}, {-3, -2, -1, 0, 1}, {-4, -3, -2, -1, 0}};
  double w[5][5];
  if (P < 5) return fail(ORC_ERR_ARG, "4th-order differences need >= 5 nodes (P=%lld)", (long long)P);
  for (int s = 0; s < 5; ++s) { int e = orc_fd_weights(offs[s], w[s]); if (e) return e; }
  for (int64_t i = 0; i < P; ++i) {
    int s = i == 0 ? 0 : (i == 1 ? 1 : (i == P - 2 ? 3 : (i == P - 1 ? 4 : 2)));
    double acc = 0.0;
    for (int k = 0; k < 5; ++k) acc += w[s][k] * f[(i + offs[s][k]) * fs];
    df[i * ds] = acc / h;
  }
  return ORC_OK;
}

int orc_fd_deriv(const double* f, int64_t P, double h, double* df) { return fd_line(f, 1, P, h, df, 1); }

/* ------------------------------------------------------------------------- */
/* Solver state.  A layer's spline is stored as 2^d arrays per field:
 * D[mask] = moments along every axis in `mask` applied to the values (tensor
 * product, successive 1-D Thomas passes), D[0] = values.                      */
typedef struct { double* D[8]; double* bic; } field_spline;   /* bic: 16 coefficients per cell (interp 1) */
typedef struct { field_spline f[4]; } layer_spline;

struct orc_ctx {
  orc_config cfg;
  int d, F, K, Ky, Kz, L, N;
  int64_t P[3], npts, stride[3];
  double dx[3], dt;
  double gh_a[64], gh_w[64];
  double gy[7], gz[7];
  double binv[16][16];    /* bicubic: Hermite data (16 corner values) -> power coefficients */
  layer_spline* ring;     /* K slots; level m lives in slot m % K */
  double* values;         /* F * npts, newest level */
  int32_t* picard;        /* npts */
  int level;              /* index n of the newest computed level */
};

static void coords(const orc_ctx* c, int64_t idx, double* x) {
  for (int a = c->d - 1; a >= 0; --a) {
    int64_t i = idx % c->P[a]; idx /= c->P[a];
    x[a] = c->cfg.xlo[a] + (double)i * c->dx[a];
  }
}

static int alloc_spline(orc_ctx* c, layer_spline* s) {
  memset(s, 0, sizeof *s);
  const int bic = c->cfg.interp == ORC_INTERP_BICUBIC;
  for (int f = 0; f < c->F; ++f) {
    for (int m = 0; m < (bic ? 1 : (1 << c->d)); ++m) {
      s->f[f].D[m] = (double*)malloc(sizeof(double) * (size_t)c->npts);
      if (!s->f[f].D[m]) return fail(ORC_ERR_RESOURCE, "oom: %lld points", (long long)c->npts);
    }
    if (bic) {
      s->f[f].bic = (double*)malloc(sizeof(double) * 16 * (size_t)((c->P[0] - 1) * (c->P[1] - 1)));
      if (!s->f[f].bic) return fail(ORC_ERR_RESOURCE, "oom: bicubic coefficients");
    }
  }
  return ORC_OK;
}
static void free_spline(orc_ctx* c, layer_spline* s) {
  for (int f = 0; f < 4; ++f) {
    for (int m = 0; m < 8; ++m) free(s->f[f].D[m]);
    free(s->f[f].bic);
  }
  (void)c;
}

/* The paper's 2-D interpolation: first and mixed derivatives by 4th-order finite
 * differences (f_xy = the axis-1 difference of f_x), then per cell the 16 coefficients
 * a_mn of p(t0, t1) = sum a_mn t0^m t1^n on the unit cell by the 16x16 matrix-vector product
 * binv * (f, f_x h0, f_y h1, f_xy h0 h1 at the 4 corners).                                   */
static void bicubic_matrix(double binv[16][16]) {
  /* A[r][k]: condition r = 4 q + corner (q: value, d/dt0, d/dt1, d2/dt0dt1; corner = c0 + 2 c1)
     applied to the monomial k = 4 m + n (t0^m t1^n); binv = A^{-1} by Gauss-Jordan */
  double A[16][32];
  for (int q = 0; q < 4; ++q)
    for (int cr = 0; cr < 4; ++cr) {
      const int r = 4 * q + cr, c0 = cr & 1, c1 = cr >> 1;
      for (int m = 0; m < 4; ++m)
        for (int n = 0; n < 4; ++n) {
          const int dm = (q == 1 || q == 3), dn = (q == 2 || q == 3);
          double v = 0.0;
          if (m >= dm && n >= dn) {
            v = (dm ? m : 1) * (dn ? n : 1);
            for (int e = 0; e < m - dm; ++e) v *= c0;
            for (int e = 0; e < n - dn; ++e) v *= c1;
          }
          A[r][4 * m + n] = v;
        }
      for (int k = 0; k < 16; ++k) A[r][16 + k] = k == r ? 1.0 : 0.0;
    }
  for (int col = 0; col < 16; ++col) {
    int piv = col;
    for (int r = col + 1; r < 16; ++r) if (fabs(A[r][col]) > fabs(A[piv][col])) piv = r;
    for (int k = 0; k < 32; ++k) { double t = A[col][k]; A[col][k] = A[piv][k]; A[piv][k] = t; }
    const double d = A[col][col];
    for (int k = 0; k < 32; ++k) A[col][k] /= d;
    for (int r = 0; r < 16; ++r) {
      if (r == col || A[r][col] == 0.0) continue;
      const double f = A[r][col];
      for (int k = 0; k < 32; ++k) A[r][k] -= f * A[col][k];
    }
  }
  for (int i = 0; i < 16; ++i) for (int k = 0; k < 16; ++k) binv[i][k] = A[i][16 + k];
}

static int build_bicubic(orc_ctx* c, const double* vals, layer_spline* s) {
  const int64_t P0 = c->P[0], P1 = c->P[1], n = c->npts;
  const double h0 = c->dx[0], h1 = c->dx[1];
  double* fx = (double*)malloc(sizeof(double) * (size_t)n);
  double* fy = (double*)malloc(sizeof(double) * (size_t)n);
  double* fxy = (double*)malloc(sizeof(double) * (size_t)n);
  int e = (fx && fy && fxy) ? ORC_OK : fail(ORC_ERR_RESOURCE, "oom");
  for (int f = 0; f < c->F && !e; ++f) {
    const double* F = vals + (size_t)f * n;
    memcpy(s->f[f].D[0], F, sizeof(double) * (size_t)n);
    for (int64_t j = 0; j < P1 && !e; ++j) e = fd_line(F + j, P1, P0, h0, fx + j, P1);      /* d/dx_0 */
    for (int64_t i = 0; i < P0 && !e; ++i) e = fd_line(F + i * P1, 1, P1, h1, fy + i * P1, 1);   /* d/dx_1 */
    for (int64_t i = 0; i < P0 && !e; ++i) e = fd_line(fx + i * P1, 1, P1, h1, fxy + i * P1, 1);
    if (e) break;
    for (int64_t i = 0; i < P0 - 1; ++i)
      for (int64_t j = 0; j < P1 - 1; ++j) {
        double v[16];
        for (int cr = 0; cr < 4; ++cr) {
          const int64_t idx = (i + (cr & 1)) * P1 + j + (cr >> 1);
          v[cr] = F[idx];
          v[4 + cr] = fx[idx] * h0;
          v[8 + cr] = fy[idx] * h1;
          v[12 + cr] = fxy[idx] * h0 * h1;
        }
        double* a = s->f[f].bic + 16 * (i * (P1 - 1) + j);
        for (int k = 0; k < 16; ++k) {
          double acc = 0.0;
          for (int r = 0; r < 16; ++r) acc += c->binv[k][r] * v[r];
          a[k] = acc;
        }
      }
  }
  free(fx); free(fy); free(fxy);
  return e;
}

/* moments along axis a of src into dst, for every line of the tensor grid */
static int axis_pass(orc_ctx* c, const double* src, double* dst, int a) {
  int64_t P = c->P[a], st = c->stride[a];
  int64_t nlines = c->npts / P;
  int err = ORC_OK;
  int nt = c->cfg.nthreads;
#pragma omp parallel num_threads(nt > 0 ? nt : omp_get_max_threads())
  {
    double* work = (double*)malloc(sizeof(double) * 4 * (size_t)P);
#pragma omp for schedule(static)
    for (int64_t l = 0; l < nlines; ++l) {
      /* line l: index decomposition with axis a removed */
      int64_t outer = l / st, inner = l % st;
      int64_t base = outer * st * P + inner;
      int e = work ? line_moments(src + base, st, P, c->dx[a], dst + base, st, work) : ORC_ERR_RESOURCE;
      if (e) {
#pragma omp critical
        err = e;
      }
    }
    free(work);
  }
  return err;
}

static int build_spline(orc_ctx* c, const double* vals, layer_spline* s) {
  int d = c->d;
  if (c->cfg.interp == ORC_INTERP_BICUBIC) return build_bicubic(c, vals, s);
  for (int f = 0; f < c->F; ++f) {
    memcpy(s->f[f].D[0], vals + (size_t)f * c->npts, sizeof(double) * (size_t)c->npts);
    for (int m = 1; m < (1 << d); ++m) {
      int a = 31 - __builtin_clz((unsigned)m);        /* highest axis in mask */
      int e = axis_pass(c, s->f[f].D[m & ~(1 << a)], s->f[f].D[m], a);
      if (e) return e;
    }
  }
  return ORC_OK;
}

/* evaluate all fields of a layer spline at X (clamped per coordinate) */
static void eval_spline(const orc_ctx* c, const layer_spline* s, const double* X, double* out) {
  int d = c->d;
  int64_t cell[3];
  double phi[3][2], psi[3][2];
  if (c->cfg.interp == ORC_INTERP_BICUBIC) {        /* clamp, locate, Horner on the cell's cubic */
    double t[2];
    for (int a = 0; a < 2; ++a) cell[a] = locate(X[a], c->cfg.xlo[a], c->cfg.xhi[a], c->dx[a], c->P[a], &t[a]);
    for (int f = 0; f < c->F; ++f) {
      const double* A = s->f[f].bic + 16 * (cell[0] * (c->P[1] - 1) + cell[1]);
      double acc = 0.0;
      for (int m = 3; m >= 0; --m) {
        double row = 0.0;
        for (int n = 3; n >= 0; --n) row = row * t[1] + A[4 * m + n];
        acc = acc * t[0] + row;
      }
      out[f] = acc;
    }
    return;
  }
  for (int a = 0; a < d; ++a) {
    double t;
    double xhi = c->cfg.xhi[a];
    cell[a] = locate(X[a], c->cfg.xlo[a], xhi, c->dx[a], c->P[a], &t);
    basis(t, c->dx[a], phi[a], psi[a]);
  }
  for (int f = 0; f < c->F; ++f) {
    double acc = 0.0;
    for (int corner = 0; corner < (1 << d); ++corner) {
      int64_t idx = 0;
      for (int a = 0; a < d; ++a) idx += (cell[a] + ((corner >> a) & 1)) * c->stride[a];
      for (int m = 0; m < (1 << d); ++m) {
        double wgt = 1.0;
        for (int a = 0; a < d; ++a) {
          int k = (corner >> a) & 1;
          wgt *= ((m >> a) & 1) ? psi[a][k] : phi[a][k];
        }
        acc += wgt * s->f[f].D[m][idx];
      }
    }
    out[f] = acc;
  }
}

/* One point of Eq. 20 with Eq. 21 expectations.  lv[j-1] is the spline of level n+j.
 * Returns the Picard iteration count.                                             */
static int point_step(const orc_ctx* c, const layer_spline* const* lv, int K, int Ky, int Kz,
                      const double* gy, const double* gz, double dt, double tn,
                      const double* x, double* out) {
  int d = c->d, L = c->L;
  double Ez[7][3], Ef[7], EfdW[7][3], Ey = 0.0;
  memset(Ez, 0, sizeof Ez); memset(Ef, 0, sizeof Ef); memset(EfdW, 0, sizeof EfdW);
  double norm = pow(ORC_PI, -0.5 * d);
  int ntap = 1;
  for (int a = 0; a < d; ++a) ntap *= L;
  for (int j = 1; j <= K; ++j) {
    double sj = sqrt(2.0 * j * dt);
    double tj = tn + j * dt;
    for (int tap = 0; tap < ntap; ++tap) {   /* Lambda in lexicographic order */
      int lam[3], rem = tap;
      for (int a = d - 1; a >= 0; --a) { lam[a] = rem % L; rem /= L; }
      double wL = norm, X[3], dW[3], v[4];
      for (int a = 0; a < d; ++a) {
        wL *= c->gh_w[lam[a]];
        dW[a] = sj * c->gh_a[lam[a]];
        if (c->cfg.sde_id == ORC_SDE_BROWNIAN) X[a] = x[a] + dW[a];
        else {                     /* one Euler step of size j dt of Eq. 1 */
          double aa, bb;
          sde_coef(&c->cfg, a, x[a], &aa, &bb);
          X[a] = x[a] + aa * (j * dt) + bb * dW[a];
        }
      }
      eval_spline(c, lv[j - 1], X, v);
      double f = orc_driver(&c->cfg, tj, v[0], v + 1);
      for (int a = 0; a < d; ++a) {
        Ez[j][a] += wL * v[1 + a];
        EfdW[j][a] += wL * f * dW[a];
      }
      Ef[j] += wL * f;
      if (j == Ky) Ey += wL * v[0];
    }
  }
  /* z: second line of Eq. 20 solved for z^n (explicit) */
  double z[3];
  for (int a = 0; a < d; ++a) {
    double s = Ez[1][a];
    for (int j = 1; j <= Kz; ++j) s += gz[j] * (EfdW[j][a] - Ez[j][a]);
    z[a] = s / gz[0];
  }
  /* y: first line of Eq. 20, implicit, by Picard iteration from y = E[y^{n+Ky}] */
  double rhs = 0.0;
  for (int j = 1; j <= Ky; ++j) rhs += gy[j] * Ef[j];
  rhs = Ey + Ky * dt * rhs;
  double y = Ey, coef = Ky * dt * gy[0];
  int it = 0;
  for (it = 1; it <= c->cfg.picard_max; ++it) {
    double yn = rhs + coef * orc_driver(&c->cfg, tn, y, z);
    double dy = fabs(yn - y);
    y = yn;
    if (c->cfg.picard_tol > 0.0 && dy <= c->cfg.picard_tol) break;
  }
  if (it > c->cfg.picard_max) it = c->cfg.picard_max;
  out[0] = y;
  for (int a = 0; a < d; ++a) out[1 + a] = z[a];
  return it;
}

/* full-grid step with K_loc levels (lv) into c->values */
static int grid_step(orc_ctx* c, const layer_spline* const* lv, int K, int Ky, int Kz,
                     const double* gy, const double* gz, double dt, double tn) {
  int nt = c->cfg.nthreads, bad = 0;
  int64_t badidx = -1;
#pragma omp parallel for schedule(static) num_threads(nt > 0 ? nt : omp_get_max_threads())
  for (int64_t i = 0; i < c->npts; ++i) {
    double x[3], out[4];
    coords(c, i, x);
    int it = point_step(c, lv, K, Ky, Kz, gy, gz, dt, tn, x, out);
    c->picard[i] = it;
    for (int f = 0; f < c->F; ++f) {
      c->values[(size_t)f * c->npts + i] = out[f];
      if (!isfinite(out[f])) {
#pragma omp critical
        { bad = 1; badidx = i; }
      }
    }
  }
  if (bad) return fail(ORC_ERR_DOMAIN, "non-finite value at t=%g point %lld", tn, (long long)badidx);
  return ORC_OK;
}

/* layer from the terminal condition (m = N) or the closed form (reading R9) */
static int fill_layer(orc_ctx* c, int m, double* vals) {
  double t = c->cfg.t0 + m * c->dt;
  int err = ORC_OK;
  int nt = c->cfg.nthreads;
  int smooth = (m == c->N) && c->cfg.smoothing && kinked(c->cfg.terminal_id);
#pragma omp parallel for schedule(static) num_threads(nt > 0 ? nt : omp_get_max_threads())
  for (int64_t i = 0; i < c->npts; ++i) {
    double x[3], y, z[3];
    coords(c, i, x);
    int e;
    if (m == c->N) {
      e = orc_terminal(&c->cfg, x, &y, z);
      if (!e && smooth && kink_in_cell(&c->cfg, x, c->dx)) smooth_point(&c->cfg, x, c->dx, &y, z);
      if (c->cfg.sde_id != ORC_SDE_BROWNIAN)          /* z = b^T grad u for Eq. 1 */
        for (int a = 0; a < c->d; ++a) { double aa, bb; sde_coef(&c->cfg, a, x[a], &aa, &bb); z[a] *= bb; }
    } else e = orc_exact(&c->cfg, t, x, &y, z);
    if (e) {
#pragma omp critical
      err = e;
    }
    vals[i] = y;
    for (int a = 0; a < c->d; ++a) vals[(size_t)(1 + a) * c->npts + i] = z[a];
  }
  return err;
}

int orc_create(const orc_config* cfg, orc_ctx** out) {
  *out = NULL;
  if (cfg->d < 1 || cfg->d > 3) return fail(ORC_ERR_ARG, "d=%d outside 1..3", cfg->d);
  if (cfg->Ky < 1 || cfg->Ky > 6 || cfg->Kz < 1 || cfg->Kz > 6) return fail(ORC_ERR_ARG, "Ky/Kz outside 1..6");
  if (cfg->L < 1 || cfg->L > 64) return fail(ORC_ERR_ARG, "L outside 1..64");
  if (!(cfg->T > cfg->t0)) return fail(ORC_ERR_ARG, "T <= t0");
  int K = cfg->Ky > cfg->Kz ? cfg->Ky : cfg->Kz;
  if (cfg->N < K) return fail(ORC_ERR_ARG, "N=%d < K=%d", cfg->N, K);
  if (cfg->picard_max < 1) return fail(ORC_ERR_ARG, "picard_max < 1");
  orc_ctx* c = (orc_ctx*)calloc(1, sizeof *c);
  if (!c) return fail(ORC_ERR_RESOURCE, "oom");
  c->cfg = *cfg;
  c->d = cfg->d; c->F = 1 + cfg->d; c->K = K; c->Ky = cfg->Ky; c->Kz = cfg->Kz;
  c->L = cfg->L; c->N = cfg->N;
  c->dt = (cfg->T - cfg->t0) / cfg->N;
  c->npts = 1;
  for (int a = 0; a < c->d; ++a) {
    if (!(cfg->xhi[a] > cfg->xlo[a])) { free(c); return fail(ORC_ERR_ARG, "empty box on axis %d", a); }
    int64_t P = cfg->npts[a];
    if (P == 0) P = orc_balance_npts(cfg->xhi[a] - cfg->xlo[a], c->dt, cfg->Ky, cfg->Kz, cfg->r > 0 ? cfg->r : 4);
    if (P < 4) { free(c); return fail(ORC_ERR_ARG, "P=%lld < 4 on axis %d", (long long)P, a); }
    c->P[a] = P;
    c->dx[a] = (cfg->xhi[a] - cfg->xlo[a]) / (double)(P - 1);
    c->npts *= P;
  }
  c->stride[c->d - 1] = 1;
  for (int a = c->d - 2; a >= 0; --a) c->stride[a] = c->stride[a + 1] * c->P[a + 1];
  if (cfg->interp == ORC_INTERP_BICUBIC) {
    if (c->d != 2) { free(c); return fail(ORC_ERR_ARG, "bicubic interpolation is 2-D (PAPER.md:406)"); }
    if (c->P[0] < 5 || c->P[1] < 5) { free(c); return fail(ORC_ERR_ARG, "bicubic: >= 5 points per axis"); }
    bicubic_matrix(c->binv);
  }
  int e = orc_gauss_hermite(c->L, c->gh_a, c->gh_w);
  if (!e) e = orc_gamma(c->Ky, 0, c->gy);
  if (!e) e = orc_gamma(c->Kz, 1, c->gz);
  if (e) { free(c); return e; }
  c->ring = (layer_spline*)calloc((size_t)K, sizeof(layer_spline));
  c->values = (double*)malloc(sizeof(double) * (size_t)c->F * (size_t)c->npts);
  c->picard = (int32_t*)calloc((size_t)c->npts, sizeof(int32_t));
  if (!c->ring || !c->values || !c->picard) { orc_destroy(c); return fail(ORC_ERR_RESOURCE, "oom"); }
  for (int k = 0; k < K; ++k)
    if ((e = alloc_spline(c, &c->ring[k]))) { orc_destroy(c); return e; }

  /* K initial layers N, N-1, ..., N-K+1 */
  e = fill_layer(c, c->N, c->values);
  if (!e) e = build_spline(c, c->values, &c->ring[c->N % K]);
  if (e) { orc_destroy(c); return e; }
  c->level = c->N;
  if (K > 1 && cfg->bootstrap == 1) {
    /* one-step scheme (K=1) with S_b sub-steps per coarse interval (reading R9) */
    int Sb = cfg->bootstrap_substeps > 0 ? cfg->bootstrap_substeps : 1;
    double g1y[2], g1z[2];
    orc_gamma(1, 0, g1y); orc_gamma(1, 1, g1z);
    layer_spline tmp;
    if ((e = alloc_spline(c, &tmp))) { orc_destroy(c); return e; }
    const layer_spline* src = &c->ring[c->N % K];
    double db = c->dt / Sb;
    for (int m = c->N - 1; m >= c->N - K + 1 && !e; --m) {
      for (int s = Sb - 1; s >= 0 && !e; --s) {
        double tn = cfg->t0 + m * c->dt + s * db;
        const layer_spline* lv[1] = {src};
        e = grid_step(c, lv, 1, 1, 1, g1y, g1z, db, tn);
        if (!e) e = build_spline(c, c->values, s == 0 ? &c->ring[m % K] : &tmp);
        src = s == 0 ? &c->ring[m % K] : &tmp;
      }
      c->level = m;
    }
    free_spline(c, &tmp);
  } else {
    for (int m = c->N - 1; m >= c->N - K + 1 && !e; --m) {
      e = fill_layer(c, m, c->values);
      if (!e) e = build_spline(c, c->values, &c->ring[m % K]);
      c->level = m;
    }
  }
  if (e) { orc_destroy(c); return e; }
  for (int64_t i = 0; i < c->npts; ++i) c->picard[i] = 0;
  *out = c;
  return ORC_OK;
}

int orc_step(orc_ctx* c) {
  if (c->level <= 0) return fail(ORC_ERR_STATE, "already at n=0");
  int n = c->level - 1;
  const layer_spline* lv[6];
  for (int j = 1; j <= c->K; ++j) lv[j - 1] = &c->ring[(n + j) % c->K];
  int e = grid_step(c, lv, c->K, c->Ky, c->Kz, c->gy, c->gz, c->dt, c->cfg.t0 + n * c->dt);
  if (e) return e;
  /* the new level replaces level n+K in the ring */
  e = build_spline(c, c->values, &c->ring[n % c->K]);
  if (e) return e;
  c->level = n;
  return ORC_OK;
}

int orc_eval_newest(orc_ctx* c, const double* x, double* out) {
  eval_spline(c, &c->ring[c->level % c->K], x, out);
  return ORC_OK;
}

int orc_solve(orc_ctx* c, double* y0, double* z0) {
  while (c->level > 0) {
    int e = orc_step(c);
    if (e) return e;
  }
  /* evaluation point x = 0 (reading R4): the grid point if the grid has one, else the spline;
     forward-SDE problems: X_0 = x_0 = sp[9..11] (Eq. 1), by the spline of layer 0            */
  int on_grid = c->cfg.sde_id == ORC_SDE_BROWNIAN;
  int64_t idx = 0;
  for (int a = 0; a < c->d; ++a) {
    if (!(c->cfg.xlo[a] == -c->cfg.xhi[a] && (c->P[a] % 2) == 1)) on_grid = 0;
    idx += ((c->P[a] - 1) / 2) * c->stride[a];
  }
  double out[4];
  if (on_grid) {
    for (int f = 0; f < c->F; ++f) out[f] = c->values[(size_t)f * c->npts + idx];
  } else {
    double x[3] = {0, 0, 0};
    if (c->cfg.sde_id != ORC_SDE_BROWNIAN) for (int a = 0; a < c->d; ++a) x[a] = c->cfg.sp[9 + a];
    orc_eval_newest(c, x, out);
  }
  *y0 = out[0];
  for (int a = 0; a < c->d; ++a) z0[a] = out[1 + a];
  return ORC_OK;
}

int orc_level(const orc_ctx* c) { return c->level; }

int orc_get_layer(const orc_ctx* c, int field, double* dst, int64_t count) {
  if (field < 0 || field >= c->F) return fail(ORC_ERR_ARG, "field %d", field);
  if (count != c->npts) return fail(ORC_ERR_ARG, "count %lld != %lld", (long long)count, (long long)c->npts);
  memcpy(dst, c->values + (size_t)field * c->npts, sizeof(double) * (size_t)count);
  return ORC_OK;
}

int orc_get_picard_counts(const orc_ctx* c, int32_t* dst, int64_t count) {
  if (count != c->npts) return fail(ORC_ERR_ARG, "count mismatch");
  memcpy(dst, c->picard, sizeof(int32_t) * (size_t)count);
  return ORC_OK;
}

int orc_query_grid(const orc_ctx* c, int64_t* npts, double* dx) {
  for (int a = 0; a < 3; ++a) { npts[a] = a < c->d ? c->P[a] : 1; dx[a] = a < c->d ? c->dx[a] : 0.0; }
  return ORC_OK;
}

int orc_step_points(orc_ctx* c, int64_t count, const int64_t* idx, double* out, int32_t* picard) {
  if (c->level <= 0) return fail(ORC_ERR_STATE, "already at n=0");
  int n = c->level - 1;
  const layer_spline* lv[6];
  for (int j = 1; j <= c->K; ++j) lv[j - 1] = &c->ring[(n + j) % c->K];
  int nt = c->cfg.nthreads;
  double tn = c->cfg.t0 + n * c->dt;
#pragma omp parallel for schedule(static) num_threads(nt > 0 ? nt : omp_get_max_threads())
  for (int64_t s = 0; s < count; ++s) {
    double x[3], v[4];
    coords(c, idx[s], x);
    int it = point_step(c, lv, c->K, c->Ky, c->Kz, c->gy, c->gz, c->dt, tn, x, v);
    for (int f = 0; f < c->F; ++f) out[(size_t)f * count + s] = v[f];
    if (picard) picard[s] = it;
  }
  return ORC_OK;
}

void orc_destroy(orc_ctx* c) {
  if (!c) return;
  if (c->ring) {
    for (int k = 0; k < c->K; ++k) free_spline(c, &c->ring[k]);
    free(c->ring);
  }
  free(c->values);
  free(c->picard);
  free(c);
}
