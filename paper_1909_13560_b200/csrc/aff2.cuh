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
//   (B) aff_rows:  E[u] = sum_m w_m B(m) H_u^0, E[u dW_1] = sum_m w_m s_m B(m) H_u^0,
//       E[u dW_0] = sum_m w_m B(m) H_u^s along axis 1, combined with the scheme weights into
//       the per-point sums Az_0, Az_1, Af, Ay of Eq. 20 (the same sums the per-tap kernels
//       accumulate) over all levels in registers, then z explicit and y by Picard.
// The result equals the per-tap quadrature up to rounding (exact algebra).
#pragma once

constexpr int kA0Rows = 8;      // aff_axis0: consecutive rows per thread
constexpr int kA1Pts = 5;       // aff_rows: consecutive points per thread (axis 1; odd: conflict-free LDS.64)

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
    if (c0 >= 0 && c0 + kA0Rows - 1 <= g.Pg0 - 2) {                  // no clamping: kA0Rows + 3 rows
      double v[kA0Rows + 3];             // (kA0Rows + 3) row loads for kA0Rows outputs
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

// (B) all levels: for kA1Pts consecutive points of an owned row (a CTA: one row, kA1TX
// columns) the axis-1 operators on H of every (level, field), the affine combination and the
// scheme weights, accumulated in registers; then z explicit (Eq. 20 line 2) and y by Picard
// (Eq. 20 line 1).  The H rows of each (level, field) -- both kinds, the tile's column window
// -- arrive in shared memory by bulk copies, one (level, field) ahead.
constexpr int kA1Thr = 64;
constexpr int kA1TX = kA1Thr * kA1Pts;
template <int DRV>
__global__ void __launch_bounds__(kA1Thr) aff_rows(StepArgs s, Grid g, Problem pb, const double* __restrict__ H,
                                                   int WC) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* const buf = reinterpret_cast<double*>(smem_raw);        // [2 stages][2 kinds][WC]
  uint64_t* const bar = reinterpret_cast<uint64_t*>(buf + 4 * (size_t)WC);
  const int64_t P1 = g.P[1], cs0 = g.cstride[0];
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * kA1TX;
  const int64_t i1 = x0 + tid * kA1Pts;                            // this thread's first point
  const int64_t i = blockIdx.y;                                    // owned row (relative to own0)
  const int L = s.L, K = s.K;
  const int64_t plane = g.nown0 * cs0, level = 6 * plane;
  double a = 0.0, b0 = 0.0, b1 = 0.0, cc = 0.0;
  if (DRV == DRV_AFFINE) { a = pb.dp[0]; b0 = pb.dp[1]; b1 = pb.dp[2]; cc = pb.dp[4]; }

  auto window = [&](int j, int& wv, int& s0, int& n) {             // storage columns of level j
    const AxisTap* t1 = axis_taps(s.tap_off) + ((size_t)(j - 1) * 2 + 1) * L;
    const int wa = x0 + t1[0].q;
    wv = wa - (wa & 1);
    const int we = x0 + kA1TX - 1 + t1[L - 1].q + 3;
    s0 = max(wv, 0);
    const int s1 = min(we, (int)P1 + 2);
    n = ((s1 - s0 + 1) + 1) & ~1;
  };
  auto issue = [&](int pr, int stage) {                            // thread 0: pair pr = (j - 1) * 3 + f
    const int j = pr / 3 + 1, f = pr % 3;
    int wv, s0, n;
    window(j, wv, s0, n);
    const double* src = H + (int64_t)(j - 1) * level + (int64_t)(2 * f) * plane + i * cs0 + s0;
    double* dst = buf + (size_t)stage * 2 * WC + (s0 - wv);
    const uint32_t bytes = (uint32_t)(n * sizeof(double));
    mbar_expect_tx(&bar[stage], 2 * bytes);
    bulk_g2s(dst, src, bytes, &bar[stage]);
    bulk_g2s(dst + WC, src + plane, bytes, &bar[stage]);
  };
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int npairs = 3 * K;
  if (tid == 0) {
    issue(0, 0);
    if (npairs > 1) issue(1, 1);
  }
  uint32_t ph[2] = {0, 0};

  double az0[kA1Pts], az1[kA1Pts], af[kA1Pts], ay[kA1Pts];
#pragma unroll
  for (int p = 0; p < kA1Pts; ++p) { az0[p] = 0.0; az1[p] = 0.0; af[p] = 0.0; ay[p] = 0.0; }
  for (int pr = 0; pr < npairs; ++pr) {
    const int j = pr / 3 + 1, f = pr % 3, stage = pr & 1;
    const AxisTap* t0 = axis_taps(s.tap_off) + (size_t)(j - 1) * 2 * L;
    const AxisTap* t1 = t0 + L;
    int wv, s0, n;
    window(j, wv, s0, n);
    const double czj = s.czj[j - 1], gzj = s.gzj[j - 1], gyj = s.gyj[j - 1];
    if (f == 0) {     // the constant term of f: c W_j, c S_jk (quadrature sums of 1 and dW_k)
      double W0 = 0.0, S0 = 0.0, W1 = 0.0, S1 = 0.0;
      for (int l = 0; l < L; ++l) {
        W0 += t0[l].w; S0 += t0[l].w * t0[l].s;
        W1 += t1[l].w; S1 += t1[l].w * t1[l].s;
      }
#pragma unroll
      for (int p = 0; p < kA1Pts; ++p) {
        af[p] = fma(gyj * cc, W0 * W1, af[p]);
        az0[p] = fma(gzj * cc, S0 * W1, az0[p]);
        az1[p] = fma(gzj * cc, W0 * S1, az1[p]);
      }
    }
    mbar_wait(&bar[stage], ph[stage]);
    ph[stage] ^= 1u;
    const double* B0 = buf + (size_t)stage * 2 * WC - wv;          // B0[col] = H^0[row][col]
    const double* Bs = B0 + WC;
    double E[kA1Pts], E1[kA1Pts], E0[kA1Pts];
#pragma unroll
    for (int p = 0; p < kA1Pts; ++p) { E[p] = 0.0; E1[p] = 0.0; E0[p] = 0.0; }
    if (i1 < P1) {
      for (int m = 0; m < L; ++m) {
        const AxisTap& t = t1[m];
        const double w = t.w, ws = t.w * t.s;
        const int64_t c0 = i1 + t.q;
        if (c0 >= 0 && c0 + kA1Pts - 1 <= P1 - 2) {
          double v[kA1Pts + 3], vs[kA1Pts + 3];
#pragma unroll
          for (int k = 0; k < kA1Pts + 3; ++k) { v[k] = B0[c0 + k]; vs[k] = Bs[c0 + k]; }
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
            const double u = fma(Bt[0], B0[cell], fma(Bt[1], B0[cell + 1], fma(Bt[2], B0[cell + 2], Bt[3] * B0[cell + 3])));
            const double us = fma(Bt[0], Bs[cell], fma(Bt[1], Bs[cell + 1], fma(Bt[2], Bs[cell + 2], Bt[3] * Bs[cell + 3])));
            E[p] = fma(w, u, E[p]);
            E1[p] = fma(ws, u, E1[p]);
            E0[p] = fma(w, us, E0[p]);
          }
        }
      }
    }
    // the stage is free: stream the pair two ahead into it
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0 && pr + 2 < npairs) issue(pr + 2, stage);
    // field f's share of the sums (f = 0: y, f = 1, 2: z_0, z_1)
    const double kf = f == 0 ? a : (f == 1 ? b0 : b1);
    const double yj = (j == s.Ky) ? 1.0 : 0.0;
#pragma unroll
    for (int p = 0; p < kA1Pts; ++p) {
      af[p] = fma(gyj * kf, E[p], af[p]);
      az0[p] = fma(gzj * kf, E0[p], az0[p]);
      az1[p] = fma(gzj * kf, E1[p], az1[p]);
      if (f == 0) ay[p] = fma(yj, E[p], ay[p]);
      if (f == 1) az0[p] = fma(czj, E[p], az0[p]);
      if (f == 2) az1[p] = fma(czj, E[p], az1[p]);
    }
  }
  // ---- epilogue: z explicit (Eq. 20 line 2), y by Picard (Eq. 20 line 1)
  const double inv_gz0 = 1.0 / s.gz0;
  Driver<DRV, 2> dn(pb.dp);
  dn.at(s.tn);
#pragma unroll
  for (int p = 0; p < kA1Pts; ++p) {
    if (i1 + p >= P1) break;
    const double z[2] = {az0[p] * inv_gz0, az1[p] * inv_gz0};
    const double rhs = fma(s.ky_dt, af[p], ay[p]);
    int it;
    unsigned ex = 0;
    const double y = picard_solve([&](double v) { return dn(v, z); }, ay[p], rhs, s.ky_dt_gy0, s.picard_max,
                                  s.picard_tol, it, ex);
    const int64_t pidx = (g.own0 + i) * P1 + i1 + p;               // local value index
    s.values[pidx] = y;
    s.values[g.npts + pidx] = z[0];
    s.values[2 * g.npts + pidx] = z[1];
    s.picard[pidx] = it;
    if (!isfinite(y) || !isfinite(z[0]) || !isfinite(z[1])) atomicMin(s.bad, bad_key(s.n, pidx));
  }
}

// the widest axis-1 column window of aff_rows over the levels (doubles, even)
int aff2_window(const AxisTap* host_taps, int K, int L) {
  int span = 0;
  for (int j = 1; j <= K; ++j) {
    const AxisTap* t1 = host_taps + ((size_t)(j - 1) * 2 + 1) * L;
    span = span > t1[L - 1].q - t1[0].q ? span : t1[L - 1].q - t1[0].q;
  }
  return (kA1TX + span + 6 + 2 + 1) & ~1;
}
size_t aff2_smem(int WC) { return (size_t)4 * WC * sizeof(double) + 16; }

template <int DRV>
static cudaError_t launch_aff2_t(const StepArgs& s, const Grid& g, const Problem& pb, double* H, int WC,
                                 cudaStream_t st, int64_t* launches) {
  const dim3 ga((unsigned)((g.P[1] + 3 + 127) / 128), (unsigned)((g.nown0 + kA0Rows - 1) / kA0Rows), 3);
  const int64_t level = 6 * g.nown0 * g.cstride[0];
  for (int j = 1; j <= s.K; ++j) {
    const double* C = s.ring + (int64_t)s.slot[j - 1] * s.slot_elems;
    aff_axis0<<<ga, 128, 0, st>>>(C, H + (int64_t)(j - 1) * level, g, s.tap_off, j, s.L);
    if (launches) *launches += 1;
  }
  const dim3 gb((unsigned)((g.P[1] + kA1TX - 1) / kA1TX), (unsigned)g.nown0);
  aff_rows<DRV><<<gb, kA1Thr, aff2_smem(WC), st>>>(s, g, pb, H, WC);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

// one d = 2 step of an affine-driver problem: K axis-0 passes + one aff_rows launch.  H holds
// K x 2 x 3 x (owned rows) x cstride[0] doubles
cudaError_t launch_aff2(const StepArgs& s, const Grid& g, const Problem& pb, double* H, int WC, cudaStream_t st,
                        int64_t* launches) {
  if (aff2_smem(WC) > 220 * 1024) return cudaErrorInvalidConfiguration;
  switch (pb.driver_id) {
    case DRV_ZERO: return launch_aff2_t<DRV_ZERO>(s, g, pb, H, WC, st, launches);
    case DRV_AFFINE: return launch_aff2_t<DRV_AFFINE>(s, g, pb, H, WC, st, launches);
  }
  return cudaErrorInvalidValue;
}

static cudaError_t set_attr_aff2() {
  cudaError_t e = cudaFuncSetAttribute(aff_rows<DRV_ZERO>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(aff_rows<DRV_AFFINE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  return e;
}
