// bicubic.cuh -- the paper's own 2-D interpolation (included by kernels.cu):
// "bicubic interpolation ... We need to calculate 16 coefficients for each point.  Based on the
// bicubic interpolation idea, we need the first and mixed derivatives.  These are approximated
// using finite difference schemes of the fourth order of accuracy (central, forward and
// backward)."
//
// B200 form.  The 16 power-form coefficients of a cell are a fixed linear map of the Hermite
// data (f, h0 f_x, h1 f_y, h0 h1 f_xy) at its 4 corners, so a ring slot keeps the 4 Hermite
// arrays per field in the value layout (4 doubles per node instead of 16 per cell) and the
// interpolant at (theta0, theta1) in cell (c0, c1) is evaluated directly as
//     sum_{a,b in {0,1}} sum_{u,v in {0,1}} H_{u,a}(theta0) H_{v,b}(theta1) D_{uv}[c0 + a][c1 + b]
// with the cubic Hermite basis H_{0,0} = 2t^3 - 3t^2 + 1, H_{0,1} = -2t^3 + 3t^2,
// H_{1,0} = t^3 - 2t^2 + t, H_{1,1} = t^3 - t^2 (the same surface as the paper's 16x16 mat-vec).
// The uniform grid makes (q, theta) of every Gauss-Hermite node translation-invariant, so the
// Hermite weights of a tap come from the constant tap table (AxisTap::B holds H00, H10, H01, H11
// for interp = FD-bicubic); a clamped tap (outside the box) is the boundary node's
// value.
#pragma once

// 4th-order first-derivative stencils (Fornberg): central (1, -8, 0, 8, -1)/12 and the one-sided
// rows at the two nodes nearest each end
__device__ __forceinline__ double fd4(const double* f, int64_t st, int64_t i, int64_t P) {
  const double inv12 = 1.0 / 12.0;
  if (i >= 2 && i <= P - 3)
    return (f[(i - 2) * st] - 8.0 * f[(i - 1) * st] + 8.0 * f[(i + 1) * st] - f[(i + 2) * st]) * inv12;
  if (i == 0)
    return (-25.0 * f[0] + 48.0 * f[st] - 36.0 * f[2 * st] + 16.0 * f[3 * st] - 3.0 * f[4 * st]) * inv12;
  if (i == 1)
    return (-3.0 * f[0] - 10.0 * f[st] + 18.0 * f[2 * st] - 6.0 * f[3 * st] + f[4 * st]) * inv12;
  if (i == P - 2)
    return (3.0 * f[(P - 1) * st] + 10.0 * f[(P - 2) * st] - 18.0 * f[(P - 3) * st] + 6.0 * f[(P - 4) * st] -
            f[(P - 5) * st]) * inv12;
  return (25.0 * f[(P - 1) * st] - 48.0 * f[(P - 2) * st] + 36.0 * f[(P - 3) * st] - 16.0 * f[(P - 4) * st] +
          3.0 * f[(P - 5) * st]) * inv12;
}

// pass 1: D0 = f, D1 = h0 f_x (axis 0), D2 = h1 f_y (axis 1) of every field; one thread per node
// (differences in grid units: h f' = the stencil applied to samples)
__global__ void hermite_pass1(const double* __restrict__ values, double* slot, Grid g, int F) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= g.npts) return;
  const int64_t P0 = g.P[0], P1 = g.P[1], i = p / P1, j = p % P1;
  for (int f = 0; f < F; ++f) {
    const double* v = values + (int64_t)f * g.npts;
    double* D = slot + (int64_t)f * g.cfield;
    D[p] = v[p];
    D[g.npts + p] = fd4(v + j, P1, i, P0);
    D[2 * g.npts + p] = fd4(v + i * P1, 1, j, P1);
  }
}
// pass 2: D3 = h0 h1 f_xy = the axis-1 difference of D1 ("composing the x then y stencils")
__global__ void hermite_pass2(double* slot, Grid g, int F) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= g.npts) return;
  const int64_t P1 = g.P[1], i = p / P1, j = p % P1;
  for (int f = 0; f < F; ++f) {
    double* D = slot + (int64_t)f * g.cfield;
    D[3 * g.npts + p] = fd4(D + g.npts + i * P1, 1, j, P1);
  }
}

cudaError_t launch_hermite(const Grid& g, const double* values, int F, double* slot, cudaStream_t st,
                           int64_t* launches) {
  const int T = 256;
  const unsigned nb = (unsigned)((g.npts + T - 1) / T);
  hermite_pass1<<<nb, T, 0, st>>>(values, slot, g, F);
  hermite_pass2<<<nb, T, 0, st>>>(slot, g, F);
  if (launches) *launches += 2;
  return cudaGetLastError();
}

// the bicubic surface of one field at cell (c0, c1) with the Hermite weights H0[4], H1[4]
// (order H00, H10, H01, H11 = value/left, slope/left, value/right, slope/right)
__device__ __forceinline__ double bicubic_at(const double* __restrict__ D, int64_t npts, int64_t P1, int64_t c0,
                                             int64_t c1, const double* H0, const double* H1) {
  double v = 0.0;
#pragma unroll
  for (int a = 0; a < 2; ++a) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const double w0 = H0[2 * a + u];               // node c0 + a, data kind u along axis 0
      // data kind (u along axis 0, w along axis 1) -> array u + 2 w: 0 f, 1 h0 f_x, 2 h1 f_y, 3 h0 h1 f_xy
      double row = 0.0;
#pragma unroll
      for (int b = 0; b < 2; ++b) {
#pragma unroll
        for (int w = 0; w < 2; ++w) {
          const int kind = u + 2 * w;
          row = fma(H1[2 * b + w], __ldg(D + (int64_t)kind * npts + (c0 + a) * P1 + c1 + b), row);
        }
      }
      v = fma(w0, row, v);
    }
  }
  return v;
}

// boundary handling of a tap: inside, cell c with the tap's Hermite weights; outside the box the
// coordinate is clamped to the edge node (value weight 1 at that node)
__device__ __forceinline__ int64_t herm_cell(int64_t c, int64_t P, const double* Hin, double* H) {
  if (c < 0) { H[0] = 1.0; H[1] = 0.0; H[2] = 0.0; H[3] = 0.0; return 0; }
  if (c >= P - 1) { H[0] = 0.0; H[1] = 0.0; H[2] = 1.0; H[3] = 0.0; return P - 2; }
  H[0] = Hin[0]; H[1] = Hin[1]; H[2] = Hin[2]; H[3] = Hin[3];
  return c;
}

// one thread per grid point: K levels x L^2 taps on the bicubic surfaces of every field
template <int DRV>
__global__ void __launch_bounds__(256) quad_bicubic(StepArgs s, Grid g, Problem pb) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= g.npts) return;
  const int64_t P0 = g.P[0], P1 = g.P[1], i0 = p / P1, i1 = p % P1;
  Driver<DRV, 2> drv(pb.dp);
  const int L = s.L;
  double Az[2] = {0.0, 0.0}, Af = 0.0, Ay = 0.0;
  for (int j = 1; j <= s.K; ++j) {
    drv.at(s.t_level[j - 1]);
    const double* C = s.ring + (int64_t)s.slot[j - 1] * s.slot_elems;
    const double czj = s.czj[j - 1], gzj = s.gzj[j - 1], gyj = s.gyj[j - 1];
    const bool yj = (j == s.Ky);
    const AxisTap* tj = axis_taps(s.tap_off) + (j - 1) * 2 * L;
    for (int l0 = 0; l0 < L; ++l0) {
      const AxisTap& t0 = tj[l0];
      double H0[4];
      const int64_t c0 = herm_cell(i0 + t0.q, P0, t0.B, H0);
      for (int l1 = 0; l1 < L; ++l1) {
        const AxisTap& t1 = tj[L + l1];
        double H1[4];
        const int64_t c1 = herm_cell(i1 + t1.q, P1, t1.B, H1);
        const double w = t0.w * t1.w;
        const double yh = bicubic_at(C, g.npts, P1, c0, c1, H0, H1);
        double zh[2];
        zh[0] = bicubic_at(C + g.cfield, g.npts, P1, c0, c1, H0, H1);
        zh[1] = bicubic_at(C + 2 * g.cfield, g.npts, P1, c0, c1, H0, H1);
        const double f = drv(yh, zh);
        const double wf = w * f;
        Az[0] += w * czj * zh[0] + gzj * t0.s * wf;
        Az[1] += w * czj * zh[1] + gzj * t1.s * wf;
        Af = fma(gyj, wf, Af);
        if (yj) Ay = fma(w, yh, Ay);
      }
    }
  }
  epilogue<DRV, 2>(s, p, g.npts, Ay, Af, Az, pb.dp);
}

cudaError_t launch_bicubic_step(const StepArgs& s, const Grid& g, const Problem& pb, cudaStream_t st) {
  const int T = 256;
  const unsigned nb = (unsigned)((g.npts + T - 1) / T);
  switch (pb.driver_id) {
    case DRV_ZERO: quad_bicubic<DRV_ZERO><<<nb, T, 0, st>>>(s, g, pb); break;
    case DRV_AFFINE: quad_bicubic<DRV_AFFINE><<<nb, T, 0, st>>>(s, g, pb); break;
    case DRV_EX1: quad_bicubic<DRV_EX1><<<nb, T, 0, st>>>(s, g, pb); break;
    case DRV_DIFF: quad_bicubic<DRV_DIFF><<<nb, T, 0, st>>>(s, g, pb); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// the bicubic surfaces of the newest level at one point (clamped; the evaluation point)
__global__ void eval_bicubic_kernel(Grid g, const double* slot, int F, double x0, double x1, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double x[2] = {x0, x1};
  int64_t cell[2];
  double H[2][4];
  for (int a = 0; a < 2; ++a) {
    const double X = fmin(fmax(x[a], g.xlo[a]), g.xhi[a]);
    const double u = (X - g.xlo[a]) / g.dx[a];
    int64_t c = (int64_t)floor(u);
    c = c > g.P[a] - 2 ? g.P[a] - 2 : (c < 0 ? 0 : c);
    const double t = u - (double)c, t2 = t * t, t3 = t2 * t;
    H[a][0] = 2.0 * t3 - 3.0 * t2 + 1.0;
    H[a][1] = t3 - 2.0 * t2 + t;
    H[a][2] = -2.0 * t3 + 3.0 * t2;
    H[a][3] = t3 - t2;
    cell[a] = c;
  }
  for (int f = 0; f < F; ++f) out[f] = bicubic_at(slot + (int64_t)f * g.cfield, g.npts, g.P[1], cell[0], cell[1], H[0], H[1]);
}

cudaError_t launch_eval_bicubic(const Grid& g, const double* slot, int F, const double* x, double* out, cudaStream_t st) {
  eval_bicubic_kernel<<<1, 32, 0, st>>>(g, slot, F, x[0], x[1], out);
  return cudaGetLastError();
}
