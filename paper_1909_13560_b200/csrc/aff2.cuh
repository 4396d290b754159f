// aff2.cuh -- d = 2 step for affine drivers (f = a y + b . z + c: Black-Scholes-type Ex. 3 / 5,
// Ex. 4, f = 0), included by kernels.cu.  SURVEY §8(f) item 2.
//
// For an affine f the per-tap driver commutes with the quadrature sum (Eq. 21):
//   E_j[f(y^, z^)]        = a E_j[y^] + b . E_j[z^] + c W_j
//   E_j[f(y^, z^) dW_k]   = a E_j[y^ dW_k] + b . E_j[z^ dW_k] + c S_jk
// (W_j, S_jk: the quadrature sums of 1 and dW_k), and every E_j[u^ ...] of a tensor-product
// spline u^ with the tensor Gauss-Hermite rule is separable: per axis, the L clamped 4-term
// B-spline stencils weighted by w_l (or w_l s_l) collapse into one
// 1-D operator.  So a level costs two 1-D passes per field instead of L^2 taps:
//   (A) aff_axis0: H_u^0 = sum_l w_l B(l) C_u,  H_u^s = sum_l w_l s_l B(l) C_u  along axis 0
//       (rows of coefficients, every storage column);
//   (B) aff_axis1: E[u] = sum_m w_m B(m) H_u^0, E[u dW_1] = sum_m w_m s_m B(m) H_u^0,
//       E[u dW_0] = sum_m w_m B(m) H_u^s along axis 1, combined with the scheme weights into
//       the per-point sums Az_0, Az_1, Af, Ay of Eq. 20 (the same sums the per-tap kernels
//       accumulate), then epilogue_zy2 (z explicit, y by Picard).
// The result equals the per-tap quadrature up to rounding (exact algebra).
#pragma once

constexpr int kA0Rows = 8;      // aff_axis0: consecutive rows per thread
constexpr int kA1Pts = 4;       // aff_axis1: consecutive points per thread (axis 1)

// (A) one level, one field (blockIdx.z): H[f][0|1][i0 - own0][e] for the owned rows i0 and the
// storage columns e < P1 + 3
__global__ void __launch_bounds__(128) aff_axis0(const double* __restrict__ C, double* __restrict__ H, Grid g,
                                                 int tap_off, int j, int L) {
  const int64_t cs0 = g.cstride[0];
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= g.P[1] + 3) return;
  const int f = blockIdx.z;
  const int64_t r0 = g.own0 + (int64_t)blockIdx.y * kA0Rows;     // first local row of this thread
  const AxisTap* t0 = axis_taps(tap_off) + (size_t)(j - 1) * 2 * L;
  const double* Cf = C + (int64_t)f * g.cfield + e;
  double h[kA0Rows], hs[kA0Rows];
#pragma unroll
  for (int r = 0; r < kA0Rows; ++r) { h[r] = 0.0; hs[r] = 0.0; }
  for (int l = 0; l < L; ++l) {
    const AxisTap& t = t0[l];
    const double w = t.w, ws = t.w * t.s;
    const int64_t c0 = r0 + g.off0 + t.q;                           // global cell of row r0
    if (c0 >= 0 && c0 + kA0Rows - 1 <= g.Pg0 - 2) {                  // no clamping: 11 rows
      double v[kA0Rows + 3];
      const double* p = Cf + (c0 - g.off0) * cs0;
#pragma unroll
      for (int k = 0; k < kA0Rows + 3; ++k) v[k] = __ldg(p + k * cs0);
#pragma unroll
      for (int r = 0; r < kA0Rows; ++r) {
        const double u = fma(t.B[0], v[r], fma(t.B[1], v[r + 1], fma(t.B[2], v[r + 2], t.B[3] * v[r + 3])));
        h[r] = fma(w, u, h[r]);
        hs[r] = fma(ws, u, hs[r]);
      }
    } else {
#pragma unroll
      for (int r = 0; r < kA0Rows; ++r) {
        double Bt[4];
        const int64_t cell = clamp_cell(c0 + r, g.Pg0, t.B, Bt) - g.off0;
        const double* p = Cf + cell * cs0;
        const double u = fma(Bt[0], __ldg(p), fma(Bt[1], __ldg(p + cs0), fma(Bt[2], __ldg(p + 2 * cs0),
                                                                             Bt[3] * __ldg(p + 3 * cs0))));
        h[r] = fma(w, u, h[r]);
        hs[r] = fma(ws, u, hs[r]);
      }
    }
  }
  const int64_t plane = g.nown0 * cs0;
  double* H0 = H + (int64_t)(2 * f) * plane + e;
  double* Hs = H0 + plane;
#pragma unroll
  for (int r = 0; r < kA0Rows; ++r) {
    const int64_t i = r0 + r - g.own0;
    if (i < g.nown0) {
      H0[i * cs0] = h[r];
      Hs[i * cs0] = hs[r];
    }
  }
}

// (B) one level: the axis-1 operators on H for kA1Pts consecutive points of an owned row, the
// affine combination and the scheme weights of level j, added to acc[4][owned points]
// (Az_0, Az_1, Af, Ay; stored at the first level)
template <int DRV>
__global__ void __launch_bounds__(128) aff_axis1(StepArgs s, Grid g, Problem pb, const double* __restrict__ H,
                                                 double* __restrict__ acc, int j, int first) {
  const int64_t P1 = g.P[1], cs0 = g.cstride[0];
  const int64_t i1 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kA1Pts;
  if (i1 >= P1) return;
  const int64_t i = blockIdx.y;                                    // owned row (relative to own0)
  const int L = s.L;
  const AxisTap* t0 = axis_taps(s.tap_off) + (size_t)(j - 1) * 2 * L;
  const AxisTap* t1 = t0 + L;
  // affine coefficients (f = a y + b . z + c; DRV_ZERO: all 0) and the quadrature sums of 1
  // and of dW_0, dW_1 over the level's tensor rule
  double a = 0.0, b0 = 0.0, b1 = 0.0, cc = 0.0;
  if (DRV == DRV_AFFINE) { a = pb.dp[0]; b0 = pb.dp[1]; b1 = pb.dp[2]; cc = pb.dp[4]; }
  double W0 = 0.0, S0 = 0.0, W1 = 0.0, S1 = 0.0;
  for (int l = 0; l < L; ++l) {
    W0 += t0[l].w; S0 += t0[l].w * t0[l].s;
    W1 += t1[l].w; S1 += t1[l].w * t1[l].s;
  }
  const double czj = s.czj[j - 1], gzj = s.gzj[j - 1], gyj = s.gyj[j - 1];
  const double yj = (j == s.Ky) ? 1.0 : 0.0;
  const int64_t plane = g.nown0 * cs0;
  double az0[kA1Pts], az1[kA1Pts], af[kA1Pts], ay[kA1Pts];
#pragma unroll
  for (int p = 0; p < kA1Pts; ++p) {
    af[p] = gyj * cc * W0 * W1;
    az0[p] = gzj * cc * S0 * W1;
    az1[p] = gzj * cc * W0 * S1;
    ay[p] = 0.0;
  }
#pragma unroll
  for (int f = 0; f < 3; ++f) {
    const double* H0 = H + (int64_t)(2 * f) * plane + i * cs0;
    const double* Hs = H0 + plane;
    double E[kA1Pts], E1[kA1Pts], E0[kA1Pts];        // E[u], E[u dW_1], E[u dW_0]
#pragma unroll
    for (int p = 0; p < kA1Pts; ++p) { E[p] = 0.0; E1[p] = 0.0; E0[p] = 0.0; }
    for (int m = 0; m < L; ++m) {
      const AxisTap& t = t1[m];
      const double w = t.w, ws = t.w * t.s;
      const int64_t c0 = i1 + t.q;
      if (c0 >= 0 && c0 + kA1Pts - 1 <= P1 - 2) {
        double v[kA1Pts + 3], vs[kA1Pts + 3];
#pragma unroll
        for (int k = 0; k < kA1Pts + 3; ++k) { v[k] = __ldg(H0 + c0 + k); vs[k] = __ldg(Hs + c0 + k); }
#pragma unroll
        for (int p = 0; p < kA1Pts; ++p) {
          const double u = fma(t.B[0], v[p], fma(t.B[1], v[p + 1], fma(t.B[2], v[p + 2], t.B[3] * v[p + 3])));
          const double us = fma(t.B[0], vs[p], fma(t.B[1], vs[p + 1], fma(t.B[2], vs[p + 2], t.B[3] * vs[p + 3])));
          E[p] = fma(w, u, E[p]);
          E1[p] = fma(ws, u, E1[p]);
          E0[p] = fma(w, us, E0[p]);
        }
      } else {
#pragma unroll
        for (int p = 0; p < kA1Pts; ++p) {
          double Bt[4];
          const int64_t cell = clamp_cell(c0 + p, P1, t.B, Bt);
          const double u = fma(Bt[0], __ldg(H0 + cell), fma(Bt[1], __ldg(H0 + cell + 1),
                               fma(Bt[2], __ldg(H0 + cell + 2), Bt[3] * __ldg(H0 + cell + 3))));
          const double us = fma(Bt[0], __ldg(Hs + cell), fma(Bt[1], __ldg(Hs + cell + 1),
                                fma(Bt[2], __ldg(Hs + cell + 2), Bt[3] * __ldg(Hs + cell + 3))));
          E[p] = fma(w, u, E[p]);
          E1[p] = fma(ws, u, E1[p]);
          E0[p] = fma(w, us, E0[p]);
        }
      }
    }
    // field f's share of the sums (f = 0: y, f = 1, 2: z_0, z_1)
    const double kf = f == 0 ? a : (f == 1 ? b0 : b1);
#pragma unroll
    for (int p = 0; p < kA1Pts; ++p) {
      af[p] = fma(gyj * kf, E[p], af[p]);
      az0[p] = fma(gzj * kf, E0[p], az0[p]);
      az1[p] = fma(gzj * kf, E1[p], az1[p]);
      if (f == 0) ay[p] = yj * E[p];
      if (f == 1) az0[p] = fma(czj, E[p], az0[p]);
      if (f == 2) az1[p] = fma(czj, E[p], az1[p]);
    }
  }
  const int64_t nown = g.nown0 * P1;
#pragma unroll
  for (int p = 0; p < kA1Pts; ++p) {
    if (i1 + p >= P1) break;
    const int64_t o = i * P1 + i1 + p;
    if (first) {
      acc[o] = az0[p]; acc[nown + o] = az1[p]; acc[2 * nown + o] = af[p]; acc[3 * nown + o] = ay[p];
    } else {
      acc[o] += az0[p]; acc[nown + o] += az1[p]; acc[2 * nown + o] += af[p]; acc[3 * nown + o] += ay[p];
    }
  }
}

// z explicit (Eq. 20 line 2), y by Picard (Eq. 20 line 1) from the level sums
template <int DRV>
__global__ void epilogue_zy2(StepArgs s, Grid g, Problem pb, const double* __restrict__ acc) {
  const int64_t nown = g.nown0 * g.P[1];
  const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= nown) return;
  const double inv_gz0 = 1.0 / s.gz0;
  Driver<DRV, 2> dn(pb.dp);
  dn.at(s.tn);
  const double z[2] = {acc[o] * inv_gz0, acc[nown + o] * inv_gz0};
  const double af = acc[2 * nown + o], ay = acc[3 * nown + o];
  const double rhs = fma(s.ky_dt, af, ay);
  double y = ay;
  int it;
  for (it = 1; it <= s.picard_max; ++it) {
    const double yn = fma(s.ky_dt_gy0, dn(y, z), rhs);
    const double dy = fabs(yn - y);
    const bool fixed = (yn == y);
    y = yn;
    if (s.picard_tol > 0.0 && dy <= s.picard_tol) break;
    if (fixed) { it = s.picard_max; break; }
  }
  if (it > s.picard_max) it = s.picard_max;
  const int64_t pidx = g.own0 * g.P[1] + o;                 // local value index
  s.values[pidx] = y;
  s.values[g.npts + pidx] = z[0];
  s.values[2 * g.npts + pidx] = z[1];
  s.picard[pidx] = it;
  if (!isfinite(y) || !isfinite(z[0]) || !isfinite(z[1])) atomicMin(s.bad, (unsigned long long)pidx);
}

template <int DRV>
static cudaError_t launch_aff2_t(const StepArgs& s, const Grid& g, const Problem& pb, double* H, double* acc,
                                 cudaStream_t st, int64_t* launches) {
  const dim3 ga((unsigned)((g.P[1] + 3 + 127) / 128), (unsigned)((g.nown0 + kA0Rows - 1) / kA0Rows), 3);
  const dim3 gb((unsigned)((g.P[1] + 128 * kA1Pts - 1) / (128 * kA1Pts)), (unsigned)g.nown0);
  for (int j = 1; j <= s.K; ++j) {
    const double* C = s.ring + (int64_t)s.slot[j - 1] * s.slot_elems;
    aff_axis0<<<ga, 128, 0, st>>>(C, H, g, s.tap_off, j, s.L);
    aff_axis1<DRV><<<gb, 128, 0, st>>>(s, g, pb, H, acc, j, j == 1 ? 1 : 0);
    if (launches) *launches += 2;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  const int64_t nown = g.nown0 * g.P[1];
  epilogue_zy2<DRV><<<(unsigned)((nown + 255) / 256), 256, 0, st>>>(s, g, pb, acc);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

// one d = 2 step of an affine-driver problem: K x (axis-0 pass + axis-1 pass) + epilogue.  H
// holds 2 x 3 x (owned rows) x cstride[0] doubles, acc 4 x (owned points)
cudaError_t launch_aff2(const StepArgs& s, const Grid& g, const Problem& pb, double* H, double* acc, cudaStream_t st,
                        int64_t* launches) {
  switch (pb.driver_id) {
    case DRV_ZERO: return launch_aff2_t<DRV_ZERO>(s, g, pb, H, acc, st, launches);
    case DRV_AFFINE: return launch_aff2_t<DRV_AFFINE>(s, g, pb, H, acc, st, launches);
  }
  return cudaErrorInvalidValue;
}
