// problems.cuh -- drivers f, terminal conditions g and closed-form solutions on the
// device (W-space, R20).  Drivers are template functors so the fused
// quadrature kernel is specialised per driver (no device function pointers).
#pragma once
#include <cuda_runtime.h>
#include "bsde_internal.h"

namespace bsde {

enum { DRV_ZERO = 0, DRV_AFFINE = 1, DRV_EX1 = 2, DRV_EX2 = 3, DRV_DIFF = 4 };
enum { TRM_CONST = 0, TRM_POLY = 1, TRM_LOGISTIC = 2, TRM_EX2 = 3, TRM_CALL = 4, TRM_SIN = 5,
       TRM_EXCHANGE = 6, TRM_GEO = 7, TRM_CALLX = 8 };
enum { SDE_BROWNIAN = 0, SDE_GBM = 1, SDE_OU = 2 };

// diffusion coefficient b_a(x) of the forward SDE (diagonal; bsde.h bsde_sde_id): the terminal
// layer of a forward-SDE problem is z_T = b(x) grad g(x) (z = b^T grad u)
__device__ inline double sde_diffusion(const Problem& pb, int a, double x) {
  if (pb.sde_id == SDE_GBM) return pb.sp[3 + a] * x;
  if (pb.sde_id == SDE_OU) return pb.sp[6 + a];
  return 1.0;
}

// ---------------------------------------------------------------- drivers f(t, y, z)
template <int DRV, int D> struct Driver;

template <int D> struct Driver<DRV_ZERO, D> {
  __device__ explicit Driver(const double*) {}
  __device__ void at(double) {}
  __device__ double operator()(double, const double*) const { return 0.0; }
};

// f = p0 y + sum_k p[1+k] z_k + p4  (Black-Scholes Eq. 29/30, Ex. 4 Eq. 34, Ex. 5 Eq. 36)
template <int D> struct Driver<DRV_AFFINE, D> {
  double a, b[D], c;
  __device__ explicit Driver(const double* p) {
    a = p[0];
#pragma unroll
    for (int k = 0; k < D; ++k) b[k] = p[1 + k];
    c = p[4];
  }
  __device__ void at(double) {}
  __device__ double operator()(double y, const double* z) const {
    double f = fma(a, y, c);
#pragma unroll
    for (int k = 0; k < D; ++k) f = fma(b[k], z[k], f);
    return f;
  }
};

// f = -y^3 + 5/2 y^2 - 3/2 y  (Eq. 22)
template <int D> struct Driver<DRV_EX1, D> {
  __device__ explicit Driver(const double*) {}
  __device__ void at(double) {}
  __device__ double operator()(double y, const double*) const {
    return y * fma(y, fma(-y, 1.0, 2.5), -1.5);
  }
};

// f = 1/2 (e^{t^2} - 4 t y - 3 e^{t^2 - y e^{-t^2}} + z^2 e^{-t^2})  (Eq. 24, d = 1)
template <int D> struct Driver<DRV_EX2, D> {
  double t, tt, E, Ei;
  __device__ explicit Driver(const double*) : t(0), tt(0), E(1), Ei(1) {}
  __device__ void at(double tm) { t = tm; tt = tm * tm; E = exp(tt); Ei = exp(-tt); }
  __device__ double operator()(double y, const double* z) const {
    return 0.5 * (E - 4.0 * t * y - 3.0 * exp(tt - y * Ei) + z[0] * z[0] * Ei);
  }
};

// f = -(r y + sum th_k z_k) + (R - r) max(sum pi_k z_k - y, 0)  (R21)
template <int D> struct Driver<DRV_DIFF, D> {
  double r, hRmr, th[D], pi[D];
  __device__ explicit Driver(const double* p) {
    r = p[0];
    hRmr = 0.5 * (p[1] - p[0]);                    // (R - r) / 2: exact scaling
#pragma unroll
    for (int k = 0; k < D; ++k) { th[k] = p[2 + k]; pi[k] = p[5 + k]; }
  }
  __device__ void at(double) {}
  __device__ double operator()(double y, const double* z) const {
    double lin = r * y, hold = -y;
#pragma unroll
    for (int k = 0; k < D; ++k) { lin = fma(th[k], z[k], lin); hold = fma(pi[k], z[k], hold); }
    // (R - r) max(hold, 0) = ((R - r) / 2) (hold + |hold|): hold + |hold| = 2 max(hold, 0) and the
    // halving are exact, so the product is the same rounding of (R - r) max(hold, 0) as before
    // (one DADD with an |.| operand modifier, no DMUL)
    return fma(hRmr, hold + fabs(hold), -lin);
  }
};

// ---------------------------------------------------------------- Picard solve of Eq. 20
// y = rhs + c f(t_n, y, z^n) by Picard iteration from y0 = E[y^{n+Ky}] (Eq. 20 line 1,
// PAPER.md:343-345, 377-378): exactly pmax iterations (p = 30; R8), or
// until |y^(k) - y^(k-1)| <= tol when tol > 0.  Two exact shortcuts leave the loop early without
// changing the result bit for bit: at a fixed point (y^(k) == y^(k-1)) every later iterate is
// y^(k); on a period-2 cycle (y^(k) == y^(k-2), rounding oscillation between two doubles) the
// iterate pmax is y^(k) or y^(k-1) by parity (and |dy| stays the same, so tol cannot be met
// later).  count: the iteration count the scheme defines (pmax, or the tolerance exit);
// executed: += the iterations actually evaluated.
template <class Fn>
__device__ __forceinline__ double picard_solve(const Fn& f, double y0, double rhs, double c, int pmax, double tol,
                                               int& count, unsigned& executed) {
  double y = y0, yprev = nan("");
  int it;
  for (it = 1; it <= pmax; ++it) {
    const double yn = fma(c, f(y), rhs);
    const double dy = fabs(yn - y);
    const bool fixed = (yn == y), cycle2 = (yn == yprev);
    yprev = y;
    y = yn;
    ++executed;
    if (tol > 0.0 && dy <= tol) break;
    if (fixed) { it = pmax; break; }
    if (cycle2) {
      if ((pmax - it) & 1) y = yprev;
      it = pmax;
      break;
    }
  }
  count = it > pmax ? pmax : it;
  return y;
}

// ---------------------------------------------------------------- terminal g, grad g
__device__ inline double logistic_d(double s) { return 1.0 / (1.0 + exp(-s)); }

__device__ inline double payoff_argument(const Problem& pb, const double* w) {
  const double* p = pb.tp;
  const double T = pb.T;
  if (pb.terminal_id == TRM_CALL) return p[0] * exp((p[2] - 0.5 * p[3] * p[3]) * T + p[3] * w[0]) - p[1];
  if (pb.terminal_id == TRM_EXCHANGE) {
    const double s1 = p[4], s2 = p[5], rho = p[6];
    const double e1 = (p[2] - 0.5 * s1 * s1) * T + s1 * w[0];
    const double e2 = (p[3] - 0.5 * s2 * s2) * T + rho * s2 * w[0] + s2 * sqrt(1.0 - rho * rho) * w[1];
    return p[0] * exp(e1) - p[1] * exp(e2);
  }
  if (pb.terminal_id == TRM_GEO) {
    double lg = 0.0;
    for (int k = 0; k < pb.d; ++k) lg += log(p[k]) + (p[4] - 0.5 * p[5 + k] * p[5 + k]) * T + p[5 + k] * w[k];
    return exp(lg / pb.d) - p[3];
  }
  return 0.0;
}

__device__ inline void terminal_eval(const Problem& pb, const double* w, double& y, double* z) {
  const double* p = pb.tp;
  const int d = pb.d;
  const double T = pb.T;
  for (int k = 0; k < d; ++k) z[k] = 0.0;
  switch (pb.terminal_id) {
    case TRM_CONST: y = p[0]; return;
    case TRM_POLY: {
      double v[kMaxD], dv[kMaxD];
      for (int a = 0; a < d; ++a) {
        const double x = w[a];
        const double* c = p + 4 * a;
        v[a] = c[0] + x * (c[1] + x * (c[2] + x * c[3]));
        dv[a] = c[1] + x * (2.0 * c[2] + 3.0 * c[3] * x);
      }
      double prod = 1.0;
      for (int a = 0; a < d; ++a) prod *= v[a];
      y = prod;
      for (int a = 0; a < d; ++a) {
        double q = dv[a];
        for (int b = 0; b < d; ++b) if (b != a) q *= v[b];
        z[a] = q;
      }
      return;
    }
    case TRM_LOGISTIC: {
      double s = 0.0;
      for (int a = 0; a < d; ++a) s += w[a];
      const double g = logistic_d(s / sqrt((double)d) + T);
      y = g;
      for (int a = 0; a < d; ++a) z[a] = g * (1.0 - g) / sqrt((double)d);
      return;
    }
    case TRM_EX2: {
      const double e = exp(T * T), sn = sin(w[0]);
      y = log(sn + 3.0) * e;
      z[0] = e * cos(w[0]) / (sn + 3.0);
      return;
    }
    case TRM_CALL: {
      const double S = p[0] * exp((p[2] - 0.5 * p[3] * p[3]) * T + p[3] * w[0]);
      y = S > p[1] ? S - p[1] : 0.0;
      z[0] = S > p[1] ? p[3] * S : 0.0;
      return;
    }
    case TRM_SIN: {
      double s = T;
      for (int a = 0; a < d; ++a) s += w[a];
      y = sin(s);
      const double c = cos(s);
      for (int a = 0; a < d; ++a) z[a] = c;
      return;
    }
    case TRM_EXCHANGE: {
      const double s1 = p[4], s2 = p[5], rho = p[6];
      const double a21 = rho * s2, a22 = s2 * sqrt(1.0 - rho * rho);
      const double S1 = p[0] * exp((p[2] - 0.5 * s1 * s1) * T + s1 * w[0]);
      const double S2 = p[1] * exp((p[3] - 0.5 * s2 * s2) * T + a21 * w[0] + a22 * w[1]);
      if (S1 > S2) { y = S1 - S2; z[0] = s1 * S1 - a21 * S2; z[1] = -a22 * S2; }
      else y = 0.0;
      return;
    }
    case TRM_GEO: {
      double lg = 0.0;
      for (int k = 0; k < d; ++k) lg += log(p[k]) + (p[4] - 0.5 * p[5 + k] * p[5 + k]) * T + p[5 + k] * w[k];
      const double G = exp(lg / d);
      if (G > p[3]) { y = G - p[3]; for (int k = 0; k < d; ++k) z[k] = G * p[5 + k] / d; }
      else y = 0.0;
      return;
    }
    case TRM_CALLX: {                      // (x_0 - K)^+ in the state variable; grad g only
      y = w[0] > p[1] ? w[0] - p[1] : 0.0;
      z[0] = w[0] > p[1] ? 1.0 : 0.0;
      return;
    }
  }
  y = nan("");
}

// Black-Scholes call with dividend yield q: price and S*dV/dS (Eq. 31, reading R13)
__device__ inline void bs_call_d(double S, double K, double r, double q, double sig, double tau, double& V, double& SdV) {
  const double st = sig * sqrt(tau);
  const double d1 = (log(S / K) + (r - q + 0.5 * sig * sig) * tau) / st;
  const double d2 = d1 - st;
  SdV = S * exp(-q * tau) * normcdf(d1);
  V = SdV - K * exp(-r * tau) * normcdf(d2);
}

// Closed-form solution (u, grad u)(t, w) for the supported (terminal, driver) pairs.
// Returns false if the pair has none (the host refuses closed-form initial layers then).
__device__ inline bool exact_eval(const Problem& pb, double t, const double* w, double& y, double* z) {
  const double* p = pb.tp;
  const double* q = pb.dp;
  const int d = pb.d;
  const double tau = pb.T - t;
  for (int k = 0; k < d; ++k) z[k] = 0.0;
  const int tid = pb.terminal_id, did = pb.driver_id;
  if (tid == TRM_CONST) {
    const double a = did == DRV_AFFINE ? q[0] : 0.0, c0 = did == DRV_AFFINE ? q[4] : 0.0;
    y = a != 0.0 ? (p[0] + c0 / a) * exp(a * tau) - c0 / a : p[0] + c0 * tau;
    return true;
  }
  if (tid == TRM_POLY) {
    const double a = did == DRV_AFFINE ? q[0] : 0.0;
    double v[kMaxD], dv[kMaxD];
    for (int ax = 0; ax < d; ++ax) {       // E[p(x + sqrt(tau) N)] per axis
      const double x = w[ax];
      const double* c = p + 4 * ax;
      v[ax] = c[0] + c[1] * x + c[2] * (x * x + tau) + c[3] * x * (x * x + 3.0 * tau);
      dv[ax] = c[1] + 2.0 * c[2] * x + 3.0 * c[3] * (x * x + tau);
    }
    const double e = exp(a * tau);
    double prod = e;
    for (int ax = 0; ax < d; ++ax) prod *= v[ax];
    y = prod;
    for (int ax = 0; ax < d; ++ax) {
      double g = e * dv[ax];
      for (int b = 0; b < d; ++b) if (b != ax) g *= v[b];
      z[ax] = g;
    }
    return true;
  }
  if (tid == TRM_LOGISTIC && did == DRV_EX1) {      // Eq. 23
    double s = 0.0;
    for (int a = 0; a < d; ++a) s += w[a];
    const double g = logistic_d(s / sqrt((double)d) + t);
    y = g;
    for (int a = 0; a < d; ++a) z[a] = g * (1.0 - g) / sqrt((double)d);
    return true;
  }
  if (tid == TRM_EX2 && did == DRV_EX2) {           // Eq. 25
    const double e = exp(t * t), sn = sin(w[0]);
    y = log(sn + 3.0) * e;
    z[0] = e * cos(w[0]) / (sn + 3.0);
    return true;
  }
  if (tid == TRM_CALL && (did == DRV_AFFINE || did == DRV_DIFF) && d == 1) {   // Eq. 31
    const double S0 = p[0], K = p[1], mu = p[2], sig = p[3];
    const double r = did == DRV_AFFINE ? -q[0] : q[0];
    const double th = did == DRV_AFFINE ? -q[1] : q[2];
    const double rate = did == DRV_AFFINE ? r : q[1];
    const double del = th * sig - mu + r;
    const double S = S0 * exp((mu - 0.5 * sig * sig) * t + sig * w[0]);
    double V, SdV;
    bs_call_d(S, K, rate, del, sig, tau, V, SdV);
    y = V; z[0] = sig * SdV;
    return true;
  }
  if (tid == TRM_SIN && did == DRV_AFFINE) {        // Eq. 35
    double s = t;
    for (int a = 0; a < d; ++a) s += w[a];
    y = sin(s);
    for (int a = 0; a < d; ++a) z[a] = cos(s);
    return true;
  }
  if (tid == TRM_EXCHANGE && did == DRV_AFFINE && d == 2) {   // Eq. 37 (Margrabe)
    const double s1 = p[4], s2 = p[5], rho = p[6];
    const double a21 = rho * s2, a22 = s2 * sqrt(1.0 - rho * rho);
    const double S1 = p[0] * exp((p[2] - 0.5 * s1 * s1) * t + s1 * w[0]);
    const double S2 = p[1] * exp((p[3] - 0.5 * s2 * s2) * t + a21 * w[0] + a22 * w[1]);
    const double sv = sqrt(s1 * s1 + s2 * s2 - 2.0 * rho * s1 * s2), sq = sv * sqrt(tau);
    const double d1 = (log(S1 / S2) + 0.5 * sv * sv * tau) / sq, d2 = d1 - sq;
    const double n1 = normcdf(d1), n2 = normcdf(d2);
    y = S1 * n1 - S2 * n2;
    z[0] = s1 * S1 * n1 - a21 * S2 * n2;
    z[1] = -a22 * S2 * n2;
    return true;
  }
  if (tid == TRM_GEO && did == DRV_DIFF) {          // DESIGN.md R21
    double lg = 0.0, ss = 0.0;
    for (int k = 0; k < d; ++k) {
      lg += log(p[k]) + (p[4] - 0.5 * p[5 + k] * p[5 + k]) * t + p[5 + k] * w[k];
      ss += p[5 + k] * p[5 + k];
    }
    const double G = exp(lg / d), sg = sqrt(ss) / d, qg = ss / (2.0 * d) - 0.5 * sg * sg;
    double V, GdV;
    bs_call_d(G, p[3], q[1], qg, sg, tau, V, GdV);
    y = V;
    for (int k = 0; k < d; ++k) z[k] = GdV * p[5 + k] / d;
    return true;
  }
  y = nan("");
  return false;
}

}  // namespace bsde
