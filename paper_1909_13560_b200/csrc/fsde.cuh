// fsde.cuh -- decoupled FBSDE with a general forward diffusion (Eq. 1; included
// by kernels.cu).  "The developed schemes can be applied also for solving (1), where the general
// Markovian diffusion X_t can be approximated, e.g., by using the Euler-Scheme":
// from grid point x_i the level-j sample of the forward process is one Euler step of size j dt
// driven by the same Gauss-Hermite increment as Eq. 21,
//     X^{i,j}_Lambda = x_i + a(x_i) j dt + b(x_i) sqrt(2 j dt) a_Lambda        (per axis, diagonal b),
// and Eq. 20 is unchanged (z is the BSDE's z = b^T grad u, dW_{t_{n+j}} = sqrt(2 j dt) a_Lambda).
// The shift now depends on x_i, so the stencil is not translation-invariant: every (point, level,
// node) locates its own cell, theta = u - floor(u) and B-spline basis (the paper's per-point
// location formula), clamped at the box.
#pragma once

// drift a and diagonal diffusion b of the forward SDE at x (bsde_sde_id; Problem::sp)
template <int SDE>
__device__ __forceinline__ void sde_coef(const double* sp, int a, double x, double& drift, double& diff) {
  if (SDE == SDE_GBM) { drift = sp[a] * x; diff = sp[3 + a] * x; }
  else if (SDE == SDE_OU) { drift = sp[a] * (sp[3 + a] - x); diff = sp[6 + a]; }
  else { drift = 0.0; diff = 1.0; }
}

// cubic B-spline basis at theta in [0, 1] (the same basis as the host's tap tables)
__device__ __forceinline__ void bspline4(double t, double* B) {
  const double u = 1.0 - t, t2 = t * t, t3 = t2 * t;
  B[0] = u * u * u * (1.0 / 6.0);
  B[1] = fma(3.0, t3, fma(-6.0, t2, 4.0)) * (1.0 / 6.0);
  B[2] = fma(-3.0, t3, fma(3.0, t2, fma(3.0, t, 1.0))) * (1.0 / 6.0);
  B[3] = t3 * (1.0 / 6.0);
}

// One thread per grid point: K levels x L^D nodes, each sample located individually.
template <int D, int DRV, int SDE>
__global__ void __launch_bounds__(256) quad_fsde(StepArgs s, Grid g, Problem pb) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= g.npts) return;
  double x[D], drift[D], diff[D];
  {
    int64_t r = p;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
      const int64_t i = r % g.P[a];
      r /= g.P[a];
      x[a] = g.xlo[a] + (double)i * g.dx[a];
      sde_coef<SDE>(pb.sp, a, x[a], drift[a], diff[a]);
    }
  }
  Driver<DRV, D> drv(pb.dp);
  const int L = s.L;
  double Az[D], Af = 0.0, Ay = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) Az[a] = 0.0;
  int ntap = 1;
#pragma unroll
  for (int a = 0; a < D; ++a) ntap *= L;
  for (int j = 1; j <= s.K; ++j) {
    drv.at(s.t_level[j - 1]);
    const double* C = s.ring + (int64_t)s.slot[j - 1] * s.slot_elems;
    const double czj = s.czj[j - 1], gzj = s.gzj[j - 1], gyj = s.gyj[j - 1];
    const bool yj = (j == s.Ky);
    const double jdt = (double)j * s.dt;          // the step's dt (bootstrap: the sub-step)
    const AxisTap* tj = axis_taps(s.tap_off) + (j - 1) * D * L;
    for (int tap = 0; tap < ntap; ++tap) {
      int lam[D];
      {
        int r = tap;
#pragma unroll
        for (int a = D - 1; a >= 0; --a) { lam[a] = r % L; r /= L; }
      }
      int64_t cell[D];
      double B[D][4];
      double w = 1.0, sa[D];
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const AxisTap& t = tj[a * L + lam[a]];
        const double X = fmin(fmax(fma(diff[a], t.s, fma(drift[a], jdt, x[a])), g.xlo[a]), g.xhi[a]);
        const double u = (X - g.xlo[a]) / g.dx[a];
        int64_t c = (int64_t)floor(u);
        c = c > g.P[a] - 2 ? g.P[a] - 2 : (c < 0 ? 0 : c);
        bspline4(u - (double)c, B[a]);
        cell[a] = c;                       // storage index of c_{cell-1}
        w *= t.w;
        sa[a] = t.s;
      }
      const double yh = gather<D>(C, g.cstride, cell, B);
      double zh[D];
#pragma unroll
      for (int a = 0; a < D; ++a) zh[a] = gather<D>(C + (int64_t)(1 + a) * g.cfield, g.cstride, cell, B);
      const double f = drv(yh, zh);
      const double wf = w * f;
#pragma unroll
      for (int a = 0; a < D; ++a) Az[a] += w * czj * zh[a] + gzj * sa[a] * wf;
      Af = fma(gyj, wf, Af);
      if (yj) Ay = fma(w, yh, Ay);
    }
  }
  epilogue<DRV, D>(s, p, g.npts, Ay, Af, Az, pb.dp);
}

template <int D, int DRV, int SDE>
static cudaError_t launch_fsde_t(const StepArgs& s, const Grid& g, const Problem& pb, cudaStream_t st) {
  const int T = 256;
  quad_fsde<D, DRV, SDE><<<(unsigned)((g.npts + T - 1) / T), T, 0, st>>>(s, g, pb);
  return cudaGetLastError();
}

template <int D, int SDE>
static cudaError_t launch_fsde_d(const StepArgs& s, const Grid& g, const Problem& pb, cudaStream_t st) {
  switch (pb.driver_id) {
    case DRV_ZERO: return launch_fsde_t<D, DRV_ZERO, SDE>(s, g, pb, st);
    case DRV_AFFINE: return launch_fsde_t<D, DRV_AFFINE, SDE>(s, g, pb, st);
    case DRV_EX1: return launch_fsde_t<D, DRV_EX1, SDE>(s, g, pb, st);
    case DRV_DIFF: return launch_fsde_t<D, DRV_DIFF, SDE>(s, g, pb, st);
  }
  return cudaErrorInvalidValue;
}

template <int SDE>
static cudaError_t launch_fsde_s(const StepArgs& s, const Grid& g, const Problem& pb, cudaStream_t st) {
  switch (g.d) {
    case 1: return launch_fsde_d<1, SDE>(s, g, pb, st);
    case 2: return launch_fsde_d<2, SDE>(s, g, pb, st);
    case 3: return launch_fsde_d<3, SDE>(s, g, pb, st);
  }
  return cudaErrorInvalidValue;
}

// quadrature + z + Picard of one step of a forward-SDE problem (the spline of level n+1 is
// built by launch_spline before it, exactly as for X = W)
cudaError_t launch_fsde_step(const StepArgs& s, const Grid& g, const Problem& pb, cudaStream_t st) {
  switch (pb.sde_id) {
    case SDE_GBM: return launch_fsde_s<SDE_GBM>(s, g, pb, st);
    case SDE_OU: return launch_fsde_s<SDE_OU>(s, g, pb, st);
  }
  return cudaErrorInvalidValue;
}
