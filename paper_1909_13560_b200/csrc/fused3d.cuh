// fused3d.cuh -- the d = 3 quadrature path (included by kernels.cu, which owns the constant
// tap arena).  The hot kernels of BASELINE cfg 5.
//
// The tensor-product B-spline value at a tap (l0, l1, l2) is separable:
//   u(x + s) = sum_c B_c(l2) sum_b B_b(l1) A_l0[i0][c1 + b][c2 + c],
//   A_l0[i0][y][x] = sum_a B_a(l0) C[c0(i0) + a][y][x]
// so per level j
//   (1) `axis0_pass` builds the L planes-stacks A_l0 (one streaming pass over the level's
//       coefficients per node, axis-0 clamping folded into the per-plane basis);
//   (2) `quad3d` treats every plane i0 as a 2-D problem with quad2d's structure: for each
//       (l0, l1) a "row pass" contracts TY + 3 axis-1 lines of A_l0 into TY shared-memory rows
//       (7 loads per 4 outputs; the raw lines stream in by bulk copies one pair ahead, behind
//       the previous pair's column pass), then the L axis-2 nodes are evaluated on those rows
//       (4 FMA per field per point), the driver is applied and the folded weights accumulated;
//       partial sums of the levels are kept in `acc` (5 per point) between launches;
//   (3) `epilogue_zy` forms z (Eq. 20 line 2) and solves y by Picard (Eq. 20 line 1).
// Exact algebra: per tap 4 FMA per field instead of the direct 64-term tricubic stencil
// (DESIGN.md §4).  Axis-1 clamping is per row in the row pass, axis-2 clamping uses the
// virtual-window extension of the 1-D and 2-D kernels.
// The differential-rates driver (cfg 5) runs decomposed by default: its nonlinearity depends on
// the single combination U = pi.z - y, so (1') `axis0_u_lin` builds plane stacks of U alone and
// quad3d<DRV_DIFF, 1> interpolates only U per tap; the affine remainder's expectations are
// separable (`lin_axis`, `lin_axis2s`, below).
#pragma once

constexpr int k3TY = 4;            // tile rows (axis 1)
constexpr int k3R = 3;             // points per thread along axis 2 (odd: conflict-free LDS.64)
constexpr int k3NT = 256;          // threads per CTA
constexpr int k3TX = k3NT / k3TY * k3R;   // 192 tile columns (axis 2)
constexpr int k3F = 4;             // fields y, z_0, z_1, z_2
constexpr int k3Acc = 5;           // accumulators per point: Az_0..2, Af, Ay

// (1) A[l][f][i0][e] = sum_a Bt_a(l, i0) C[f][crow(l, i0) + a][e] over the plane elements e
__global__ void axis0_pass(const double* __restrict__ C, double* __restrict__ A, Grid g, int tap_off, int j, int L) {
  const int64_t plane = g.cstride[0];
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= plane) return;
  const int64_t i0 = g.own0 + blockIdx.y;          // owned local plane (quad3d reads only these)
  const int l = blockIdx.z;
  const AxisTap& ta = axis_taps(tap_off)[(size_t)(j - 1) * 3 * L + l];
  double Bt[4];
  const int64_t crow = clamp_cell(i0 + g.off0 + ta.q, g.Pg0, ta.B, Bt) - g.off0;
  const int64_t P0 = g.P[0];
#pragma unroll
  for (int f = 0; f < k3F; ++f) {
    const double* c = C + (int64_t)f * g.cfield + crow * plane + e;
    const double v = fma(Bt[0], __ldcg(c), fma(Bt[1], __ldcg(c + plane), fma(Bt[2], __ldcg(c + 2 * plane),
                                                                              Bt[3] * __ldcg(c + 3 * plane))));
    A[(((int64_t)l * k3F + f) * P0 + i0) * plane + e] = v;
  }
}

// (1') decomposed driver: the plane stacks of U = sum_f uc_f C_f together with the axis-0
// operators of the affine part.  A thread owns one plane element and 8 consecutive planes and
// loops over the L axis-0 nodes; the level's coefficient rows stream by (11 per node for 8
// planes, every row feeding the outputs whose 4-row stencil covers it), and one pass writes
// the U stacks (per node) and the six node-summed arrays Lf (plain, s-weighted), z_0..2, y.
__global__ void __launch_bounds__(128) axis0_u_lin(const double* __restrict__ C, double* __restrict__ A,
                                                   double* __restrict__ W0, Grid g, int tap_off, int j, int L,
                                                   double4 uc, double4 lc) {
  constexpr int RA = 8;
  const int64_t plane = g.cstride[0];
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= plane) return;
  const int64_t i0 = g.own0 + (int64_t)blockIdx.y * RA;          // first (owned) local plane
  const int64_t P0 = g.P[0], iend = g.own0 + g.nown0;
  const AxisTap* t0 = axis_taps(tap_off) + (size_t)(j - 1) * 3 * L;
  const double* Ce = C + e;
  double lp[RA], ls[RA], z0[RA], z1[RA], z2[RA], yy[RA];
#pragma unroll
  for (int r = 0; r < RA; ++r) { lp[r] = 0.0; ls[r] = 0.0; z0[r] = 0.0; z1[r] = 0.0; z2[r] = 0.0; yy[r] = 0.0; }
  for (int l = 0; l < L; ++l) {
    const AxisTap& t = t0[l];
    const double w = t.w, ws = t.w * t.s;
    const int64_t c0 = i0 + g.off0 + t.q;                          // global cell of plane i0
    double u[RA];
#pragma unroll
    for (int r = 0; r < RA; ++r) u[r] = 0.0;
    // row k contributes B_a(theta) to output r = k - a; for a clamped output its own 4 rows
    auto feed = [&](int r, double b, const double* c) {
      const double f0 = __ldg(c), f1 = __ldg(c + g.cfield), f2 = __ldg(c + 2 * g.cfield), f3 = __ldg(c + 3 * g.cfield);
      const double U = fma(uc.x, f0, fma(uc.y, f1, fma(uc.z, f2, uc.w * f3)));
      const double Lf = fma(lc.x, f0, fma(lc.y, f1, fma(lc.z, f2, lc.w * f3)));
      const double bw = b * w, bs = b * ws;
      u[r] = fma(b, U, u[r]);
      lp[r] = fma(bw, Lf, lp[r]); ls[r] = fma(bs, Lf, ls[r]);
      z0[r] = fma(bw, f1, z0[r]); z1[r] = fma(bw, f2, z1[r]); z2[r] = fma(bw, f3, z2[r]); yy[r] = fma(bw, f0, yy[r]);
    };
    if (c0 >= 0 && c0 + RA - 1 <= g.Pg0 - 2) {
      const double* c = Ce + (c0 - g.off0) * plane;
#pragma unroll
      for (int k = 0; k < RA + 3; ++k)
#pragma unroll
        for (int a = 0; a < 4; ++a)
          if (k - a >= 0 && k - a < RA) feed(k - a, t.B[a], c + k * plane);
    } else {
#pragma unroll
      for (int r = 0; r < RA; ++r) {
        double Bt[4];
        const int64_t cell = clamp_cell(c0 + r, g.Pg0, t.B, Bt) - g.off0;
#pragma unroll
        for (int a = 0; a < 4; ++a) feed(r, Bt[a], Ce + (cell + a) * plane);
      }
    }
#pragma unroll
    for (int r = 0; r < RA; ++r)
      if (i0 + r < iend) A[((int64_t)l * P0 + i0 + r) * plane + e] = u[r];
  }
  // the affine part's axis-0 arrays for the owned planes: [Lf, Lf s0, z_0, z_1, z_2, y][owned][plane]
  const int64_t arr = g.nown0 * plane;
#pragma unroll
  for (int r = 0; r < RA; ++r) {
    const int64_t i = i0 + r - g.own0;
    if (i < 0 || i >= g.nown0) continue;
    double* o = W0 + i * plane + e;
    o[0] = lp[r]; o[arr] = ls[r]; o[2 * arr] = z0[r]; o[3 * arr] = z1[r]; o[4 * arr] = z2[r]; o[5 * arr] = yy[r];
  }
}

// (2) one level of taps for a 4 x 192 tile of plane i0 (own rows only).  NF = 4: every field
// interpolated per tap and the driver applied; NF = 1 (decomposed differential-rates driver,
// f = -(r y + th.z) + (R - r) max(U, 0)): only U per tap and only the nonlinear part
// g = (R - r) max(U, 0) accumulated (the affine part is separable: lin_axis / lin_axis2s below)
template <int DRV, int NF>
__global__ void __launch_bounds__(k3NT, 2) quad3d(StepArgs s, Grid g, Problem pb, int WC, const double* __restrict__ A,
                                                  double* __restrict__ acc, int j, int first) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* const Rw = reinterpret_cast<double*>(smem_raw);     // [4 fields][TY rows][WC]
  const int tid = threadIdx.x;
  const int r = tid / (k3NT / k3TY), lb = tid % (k3NT / k3TY);
  const int64_t P1 = g.P[1], P2 = g.P[2];
  const int64_t plane = g.cstride[0], cs1 = g.cstride[1];
  const int x0 = blockIdx.x * k3TX;
  const int64_t y0 = (int64_t)blockIdx.y * k3TY;
  const int64_t i0 = g.own0 + blockIdx.z;                       // local plane
  const int L = s.L;
  const int cx0 = x0 + lb * k3R;
  const int64_t yrow = y0 + r;
  const bool rowok = yrow < P1;
  const AxisTap* t0 = axis_taps(s.tap_off) + (size_t)(j - 1) * 3 * L;
  const AxisTap* t1 = t0 + L;
  const AxisTap* t2 = t1 + L;
  const int64_t Afield = g.P[0] * plane;

  Driver<DRV, 3> drv(pb.dp);
  drv.at(s.t_level[j - 1]);
  const double Rmr = pb.dp[1] - pb.dp[0];          // NF = 1: (R - r) of the differential-rates driver
  const double czj = s.czj[j - 1], gzj = s.gzj[j - 1], gyj = s.gyj[j - 1];
  const bool yj = (j == s.Ky);
  double Az[3][k3R], Af[k3R], Ay[k3R];
#pragma unroll
  for (int q = 0; q < k3R; ++q) { Az[0][q] = 0.0; Az[1][q] = 0.0; Az[2][q] = 0.0; Af[q] = 0.0; Ay[q] = 0.0; }

  // column (axis-2) window of this level: storage columns [wv, we] (wv even)
  const int qmin2 = t2[0].q, qmax2 = t2[L - 1].q;
  const int wa = x0 + qmin2;
  const int wv = wa - (wa & 1);
  const int we = x0 + k3TX - 1 + qmax2 + 3;
  const int nwin = we - wv + 1;
  const int s0 = max(wv, 0), s1 = min(we, (int)P2 + 2);        // real columns
  const bool left = wv < 0, right = we > P2 + 2;

  // raw axis-1 rows of the current (l0, l1) pair: storage rows c0 .. c0 + TY + 2 of plane i0
  // of A_l0, columns [s0, s0 + nraw), all fields; streamed by bulk copies one pair ahead
  double* const raw = Rw + (size_t)NF * k3TY * WC;              // [4 fields][TY + 3][WC]
  uint64_t* const bar = reinterpret_cast<uint64_t*>(raw + (size_t)NF * (k3TY + 3) * WC);
  const int nraw = ((s1 - s0 + 1) + 1) & ~1;
  auto first_row = [&](int l1) -> int64_t {
    const int64_t c = y0 + t1[l1].q;
    return c < 0 ? 0 : (c > P1 - 1 ? P1 - 1 : c);
  };
  auto issue_rows = [&](int l0, int l1) {        // thread 0
    const double* Al = A + (int64_t)l0 * NF * Afield + i0 * plane + s0;
    const int64_t c0 = first_row(l1);
    const int nrows = (int)(P1 + 3 - c0 < k3TY + 3 ? P1 + 3 - c0 : k3TY + 3);
    const uint32_t bytes = (uint32_t)(nraw * sizeof(double));
    mbar_expect_tx(bar, bytes * nrows * NF);
    for (int f = 0; f < NF; ++f)
      for (int a = 0; a < nrows; ++a)
        bulk_g2s(raw + ((size_t)f * (k3TY + 3) + a) * WC, Al + (int64_t)f * Afield + (c0 + a) * cs1, bytes, bar);
  };
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) issue_rows(0, 0);
  uint32_t phase = 0;

  for (int l0 = 0; l0 < L; ++l0) {
    const AxisTap& ta = t0[l0];
    for (int l1 = 0; l1 < L; ++l1) {
      const AxisTap& tb = t1[l1];
      // ---- row pass: Rw[f][r'][k] = sum_b B_b A_l0[f][i0][row(r') + b][wv + k], r' < TY, from
      // the raw rows; clamped rows (cells < 0 or >= P1 - 1) take the boundary basis
      // (1/6, 2/3, 1/6, 0) at cell 0 / P1 - 1
      {
        const int64_t cy = y0 + tb.q;                 // cell of tile row 0
        const int64_t c0 = cy < 0 ? 0 : (cy > P1 - 1 ? P1 - 1 : cy);   // = first_row(l1)
        const bool consecutive = cy >= 0 && cy + k3TY - 1 <= P1 - 2;
        mbar_wait(bar, phase);
        phase ^= 1u;
        // (field, column) items spread evenly over the threads (NF x ncol items)
        const int ncol = s1 - s0 + 1;
        int f = 0, k = tid;
        while (k >= ncol) { k -= ncol; ++f; }
        for (; f < NF; k += k3NT) {
          while (k >= ncol) { k -= ncol; ++f; }
          if (f >= NF) break;
          {
            const double* rc = raw + (size_t)f * (k3TY + 3) * WC + k;
            double* out = Rw + (size_t)f * k3TY * WC + (s0 - wv) + k;
            if (consecutive) {
              double cin[k3TY + 3];
#pragma unroll
              for (int a = 0; a < k3TY + 3; ++a) cin[a] = rc[a * WC];
#pragma unroll
              for (int rr = 0; rr < k3TY; ++rr)
                out[rr * WC] =
                    fma(tb.B[0], cin[rr], fma(tb.B[1], cin[rr + 1], fma(tb.B[2], cin[rr + 2], tb.B[3] * cin[rr + 3])));
            } else {
#pragma unroll
              for (int rr = 0; rr < k3TY; ++rr) {
                double Bt[4];
                const int64_t cr = clamp_cell(cy + rr, P1, tb.B, Bt) - c0;
                const double* q = rc + cr * WC;
                out[rr * WC] = fma(Bt[0], q[0], fma(Bt[1], q[WC], fma(Bt[2], q[2 * WC], Bt[3] * q[3 * WC])));
              }
            }
          }
        }
        // the raw rows are free: stream the next pair's while this pair's columns are evaluated
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
          const int n1 = l1 + 1 < L ? l1 + 1 : 0, n0 = l1 + 1 < L ? l0 : l0 + 1;
          if (n0 < L) issue_rows(n0, n1);
        }
      }
      // ---- axis-2 boundary: clamped values of every row, virtual window entries
      double bl[NF], br[NF];
#pragma unroll
      for (int f = 0; f < NF; ++f) { bl[f] = 0.0; br[f] = 0.0; }
      if (left || right) {
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          const double* row = Rw + (f * k3TY + r) * WC;
          if (left) bl[f] = (1.0 / 6.0) * row[-wv] + (2.0 / 3.0) * row[1 - wv] + (1.0 / 6.0) * row[2 - wv];
          if (right)
            br[f] = (1.0 / 6.0) * row[P2 - 1 - wv] + (2.0 / 3.0) * row[P2 - wv] + (1.0 / 6.0) * row[P2 + 1 - wv];
        }
        // virtual window entries of every row (one warp per row, no index division); they
        // are disjoint from the real entries the boundary values are read from
        const int nleft = left ? -wv : 0, kright = right ? (int)P2 + 3 - wv : nwin;
        for (int fr = tid >> 5; fr < NF * k3TY; fr += k3NT / 32) {
          double* row = Rw + fr * WC;
          const int ln = tid & 31;
          if (left) {
            const double v = (1.0 / 6.0) * row[-wv] + (2.0 / 3.0) * row[1 - wv] + (1.0 / 6.0) * row[2 - wv];
            for (int k = ln; k < nleft; k += 32) row[k] = v;
          }
          if (right) {
            const double v = (1.0 / 6.0) * row[P2 - 1 - wv] + (2.0 / 3.0) * row[P2 - wv] + (1.0 / 6.0) * row[P2 + 1 - wv];
            for (int k = kright + ln; k < nwin; k += 32) row[k] = v;
          }
        }
        __syncthreads();
      }
      // ---- column pass over the axis-2 nodes
      const double W01 = ta.w * tb.w;
      const double Wcz = W01 * czj, Wgz = W01 * gzj, Wgy = W01 * gyj;
      const double sa = ta.s, sb = tb.s;
      const int rel0 = cx0 - wv;
      // NF = 1: sums over the axis-2 nodes of w_m g' and w_m s_m g' (g' = U + |U| = 2 max(U, 0)),
      // scaled once per (l0, l1) pair below
      double Sg[k3R], Sgs[k3R];
#pragma unroll
      for (int p = 0; p < k3R; ++p) { Sg[p] = 0.0; Sgs[p] = 0.0; }
      for (int m = 0; m < L; ++m) {
        const AxisTap& tc = t2[m];
        const int q = tc.q;
        double v[NF][k3R];
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          const double* rp = Rw + (f * k3TY + r) * WC + rel0 + q;
          double c[k3R + 3];
#pragma unroll
          for (int k = 0; k < k3R + 3; ++k) c[k] = rp[k];
#pragma unroll
          for (int p = 0; p < k3R; ++p)
            v[f][p] = fma(tc.B[0], c[p], fma(tc.B[1], c[p + 1], fma(tc.B[2], c[p + 2], tc.B[3] * c[p + 3])));
        }
        const int cb = cx0 + q, ce = cb + k3R - 1;
        if ((left || right) && ((left && cb <= -1 && ce >= -3) || (right && cb <= P2 + 2 && ce >= P2 - 1))) {
#pragma unroll
          for (int p = 0; p < k3R; ++p) {
            const int cell = cb + p;
            if (cell >= -3 && cell <= -1) {
#pragma unroll
              for (int f = 0; f < NF; ++f) v[f][p] = bl[f];
            }
            if (cell >= P2 - 1 && cell <= P2 + 2) {
#pragma unroll
              for (int f = 0; f < NF; ++f) v[f][p] = br[f];
            }
          }
        }
        const double wm = tc.w;
        const double wcz = Wcz * wm, wgy = Wgy * wm, wg = Wgz * wm;
        const double wgz0 = wg * sa, wgz1 = wg * sb, wgz2 = wg * tc.s;
        if constexpr (NF == k3F) {
#pragma unroll
          for (int p = 0; p < k3R; ++p) {
            const double zz[3] = {v[1 % NF][p], v[2 % NF][p], v[3 % NF][p]};
            const double f = drv(v[0][p], zz);
            Az[0][p] = fma(wcz, v[1 % NF][p], fma(wgz0, f, Az[0][p]));
            Az[1][p] = fma(wcz, v[2 % NF][p], fma(wgz1, f, Az[1][p]));
            Az[2][p] = fma(wcz, v[3 % NF][p], fma(wgz2, f, Az[2][p]));
            Af[p] = fma(wgy, f, Af[p]);
          }
          if (yj) {
            const double wy = W01 * wm;
#pragma unroll
            for (int p = 0; p < k3R; ++p) Ay[p] = fma(wy, v[0][p], Ay[p]);
          }
        } else {
          // only the nonlinear part g = (R - r) max(U, 0) of the decomposed driver
          const double wms = wm * tc.s;
#pragma unroll
          for (int p = 0; p < k3R; ++p) {
            const double u = v[0][p];
            const double g2 = u + fabs(u);                 // 2 max(U, 0)
            Sg[p] = fma(wm, g2, Sg[p]);
            Sgs[p] = fma(wms, g2, Sgs[p]);
          }
          (void)wcz; (void)wgy; (void)wgz0; (void)wgz1; (void)wgz2;
        }
      }
      if constexpr (NF == 1) {             // the pair's share: weights W01 w_m, dW factors s_a, s_b, s_m
        const double h = 0.5 * Rmr;
        const double cg0 = Wgz * sa * h, cg1 = Wgz * sb * h, cg2 = Wgz * h, cgy = Wgy * h;
#pragma unroll
        for (int p = 0; p < k3R; ++p) {
          Az[0][p] = fma(cg0, Sg[p], Az[0][p]);
          Az[1][p] = fma(cg1, Sg[p], Az[1][p]);
          Az[2][p] = fma(cg2, Sgs[p], Az[2][p]);
          Af[p] = fma(cgy, Sg[p], Af[p]);
        }
      }
      __syncthreads();                     // Rw is rewritten by the next row pass
    }
  }
  // ---- partial sums of this level
  if (!rowok) return;
  const int64_t nown = g.nown0 * P1 * P2;
#pragma unroll
  for (int p = 0; p < k3R; ++p) {
    const int64_t col = cx0 + p;
    if (col >= P2) break;
    const int64_t o = ((int64_t)blockIdx.z * P1 + yrow) * P2 + col;     // index among the owned points
    const double vals[k3Acc] = {Az[0][p], Az[1][p], Az[2][p], Af[p], Ay[p]};
#pragma unroll
    for (int a = 0; a < k3Acc; ++a) {
      double* dst = acc + (int64_t)a * nown + o;
      *dst = first ? vals[a] : *dst + vals[a];
    }
  }
}

// (3) z explicit (Eq. 20 line 2), y by Picard (Eq. 20 line 1) from the accumulated sums
template <int DRV>
__global__ void epilogue_zy3(StepArgs s, Grid g, Problem pb, const double* __restrict__ acc) {
  const int64_t nown = g.nown0 * g.P[1] * g.P[2];
  const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= nown) return;
  const double inv_gz0 = 1.0 / s.gz0;
  Driver<DRV, 3> dn(pb.dp);
  dn.at(s.tn);
  const double z[3] = {acc[o] * inv_gz0, acc[nown + o] * inv_gz0, acc[2 * nown + o] * inv_gz0};
  const double af = acc[3 * nown + o], ay = acc[4 * nown + o];
  const double rhs = fma(s.ky_dt, af, ay);
  int it;
  unsigned ex = 0;
  const double y = picard_solve([&](double v) { return dn(v, z); }, ay, rhs, s.ky_dt_gy0, s.picard_max,
                                s.picard_tol, it, ex);
  const int64_t pidx = g.own0 * g.P[1] * g.P[2] + o;       // local value index
  s.values[pidx] = y;
  s.values[g.npts + pidx] = z[0];
  s.values[2 * g.npts + pidx] = z[1];
  s.values[3 * g.npts + pidx] = z[2];
  s.picard[pidx] = it;
  if (!isfinite(y) || !isfinite(z[0]) || !isfinite(z[1]) || !isfinite(z[2])) atomicMin(s.bad, bad_key(s.n, pidx));
}

// shared memory of quad3d for a column-window width WC (doubles)
size_t fused3d_smem(int WC, int nf) { return (size_t)nf * (2 * k3TY + 3) * WC * sizeof(double) + 16; }

// the widest axis-2 window over the levels: TX + (q_max - q_min) on axis 2 + 4 + 2
int fused3d_window(const AxisTap* host_taps, int K, int L) {
  int span = 0;
  for (int j = 1; j <= K; ++j) {
    const AxisTap* t2 = host_taps + ((size_t)(j - 1) * 3 + 2) * L;
    span = span > t2[L - 1].q - t2[0].q ? span : t2[L - 1].q - t2[0].q;
  }
  return (k3TX + span + 6 + 1) & ~1;            // even: 16-byte aligned raw rows
}

// ---------------------------------------------------------------- decomposed driver (d = 3)
// For f = -(r y + th.z) + (R - r) max(U, 0), U = pi.z - y (differential rates), the affine part
// Lf = -(r y + th.z) is a fixed linear combination of the fields, so its expectations -- and
// those of z_k and y -- are separable tensor operators (as in aff2.cuh): per level
//   E[Lf], E[Lf dW_k] (k = 0..2), E[z_k], E[y]
// by one strided pass per axis (lin_axis: axes 0 and 1, 8 rows per thread) and one contiguous
// pass that also adds the scheme-weighted sums to acc (lin_axis2s).  quad3d<DRV_DIFF, 1> adds
// the nonlinear part.  Exact algebra (interpolation is linear in the data).
struct LinAxis {
  const double* X; int64_t xb, xr, xf; int nf; double coef[4];   // input rows: sum_f coef_f X_f
  double* Yp; double* Ys; int64_t yb, yr;                         // outputs (plain, s-weighted or null)
  int64_t ncols, nout, ibase, off, Pg;                            // columns, output rows, clamping
  int tap_off, j, a, L;                                           // taps of level j, axis a (d = 3)
};
template <int NFI>     // input fields combined per row (compile time: the row loads issue together)
__global__ void __launch_bounds__(128) lin_axis(LinAxis p) {
  constexpr int RA = 8;
  const int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= p.ncols) return;
  const int64_t b = blockIdx.z, i0 = (int64_t)blockIdx.y * RA;
  const AxisTap* tp = axis_taps(p.tap_off) + ((size_t)(p.j - 1) * 3 + p.a) * p.L;
  const double* Xb = p.X + b * p.xb + col;
  auto row = [&](int64_t r) {          // sum_f coef_f X_f[b][r][col]
    double v = 0.0;
#pragma unroll
    for (int f = 0; f < NFI; ++f) v = fma(p.coef[f], __ldg(Xb + f * p.xf + r * p.xr), v);
    return v;
  };
  double h[RA], hs[RA];
#pragma unroll
  for (int r = 0; r < RA; ++r) { h[r] = 0.0; hs[r] = 0.0; }
  for (int l = 0; l < p.L; ++l) {
    const AxisTap& t = tp[l];
    const double w = t.w, ws = t.w * t.s;
    const int64_t c0 = p.ibase + i0 + p.off + t.q;                 // global cell of output row i0
    if (c0 >= 0 && c0 + RA - 1 <= p.Pg - 2) {
      double v[RA + 3];
#pragma unroll
      for (int k = 0; k < RA + 3; ++k) v[k] = row(c0 - p.off + k);
#pragma unroll
      for (int r = 0; r < RA; ++r) {
        const double u = fma(t.B[0], v[r], fma(t.B[1], v[r + 1], fma(t.B[2], v[r + 2], t.B[3] * v[r + 3])));
        h[r] = fma(w, u, h[r]);
        hs[r] = fma(ws, u, hs[r]);
      }
    } else {
#pragma unroll
      for (int r = 0; r < RA; ++r) {
        double Bt[4];
        const int64_t cell = clamp_cell(c0 + r, p.Pg, t.B, Bt) - p.off;
        const double u = fma(Bt[0], row(cell), fma(Bt[1], row(cell + 1), fma(Bt[2], row(cell + 2), Bt[3] * row(cell + 3))));
        h[r] = fma(w, u, h[r]);
        hs[r] = fma(ws, u, hs[r]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < RA; ++r) {
    if (i0 + r >= p.nout) break;
    p.Yp[b * p.yb + (i0 + r) * p.yr + col] = h[r];
    if (p.Ys) p.Ys[b * p.yb + (i0 + r) * p.yr + col] = hs[r];
  }
}

// the contiguous axis (2) of the 7 axis-1 outputs [owned planes (stride cstride[0])][P1][cs1] and
// the level's scheme-weighted sums added to acc: Az_k += czj E[z_k] + gzj E[Lf dW_k],
// Af += gyj E[Lf], Ay += [j == Ky] E[y]  (arrays: 0 Lf_pp, 1 Lf_p s1, 2 Lf_s0 p, 3..5 z_k, 6 y).
// One row (i0, i1) x 192 columns per 64-thread CTA; the tile's column window of the 7 rows
// arrives in shared memory by bulk copies.
constexpr int kL2Thr = 64, kL2R = 3, kL2TX = kL2Thr * kL2R;
__global__ void __launch_bounds__(kL2Thr) lin_axis2s(StepArgs s, Grid g, const double* __restrict__ X, int64_t astride,
                                                    double* __restrict__ acc, int j, int WC) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* const buf = reinterpret_cast<double*>(smem_raw);          // [7][WC]
  uint64_t* const bar = reinterpret_cast<uint64_t*>(buf + 7 * (size_t)WC);
  const int64_t P1 = g.P[1], P2 = g.P[2], cs1 = g.cstride[1];
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * kL2TX;
  const int64_t i2 = x0 + tid * kL2R;
  const int64_t i1 = blockIdx.y, i0 = blockIdx.z;
  const int L = s.L;
  const AxisTap* tp = axis_taps(s.tap_off) + ((size_t)(j - 1) * 3 + 2) * L;
  const bool yj = (j == s.Ky);
  const int wa = x0 + tp[0].q;
  const int wv = wa - (wa & 1);
  const int we = x0 + kL2TX - 1 + tp[L - 1].q + 3;
  const int s0 = max(wv, 0), s1 = min(we, (int)P2 + 2);
  const int n = ((s1 - s0 + 1) + 1) & ~1;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    const int na = yj ? 7 : 6;
    const uint32_t bytes = (uint32_t)(n * sizeof(double));
    mbar_expect_tx(bar, bytes * na);
    const double* src = X + i0 * g.cstride[0] + i1 * cs1 + s0;
    for (int k = 0; k < na; ++k) bulk_g2s(buf + (size_t)k * WC + (s0 - wv), src + k * astride, bytes, bar);
  }
  __syncthreads();
  mbar_wait(bar, 0);
  if (i2 >= P2) return;
  double E[8][kL2R];                      // Lf, Lf dW2, Lf dW1, Lf dW0, z0, z1, z2, y
#pragma unroll
  for (int k = 0; k < 8; ++k)
#pragma unroll
    for (int q = 0; q < kL2R; ++q) E[k][q] = 0.0;
  for (int m = 0; m < L; ++m) {
    const AxisTap& t = tp[m];
    const double w = t.w, ws = t.w * t.s;
    const int64_t c0 = i2 + t.q;
#pragma unroll
    for (int k = 0; k < 7; ++k) {
      if (k == 6 && !yj) continue;
      const double* xr = buf + (size_t)k * WC - wv;                 // xr[col] = X_k[i0][i1][col]
      double u[kL2R];
      if (c0 >= 0 && c0 + kL2R - 1 <= P2 - 2) {
        double v[kL2R + 3];
#pragma unroll
        for (int q = 0; q < kL2R + 3; ++q) v[q] = xr[c0 + q];
#pragma unroll
        for (int q = 0; q < kL2R; ++q) u[q] = fma(t.B[0], v[q], fma(t.B[1], v[q + 1], fma(t.B[2], v[q + 2], t.B[3] * v[q + 3])));
      } else {
#pragma unroll
        for (int q = 0; q < kL2R; ++q) {
          double Bt[4];
          const int64_t cell = clamp_cell(c0 + q, P2, t.B, Bt);
          u[q] = fma(Bt[0], xr[cell], fma(Bt[1], xr[cell + 1], fma(Bt[2], xr[cell + 2], Bt[3] * xr[cell + 3])));
        }
      }
#pragma unroll
      for (int q = 0; q < kL2R; ++q) {
        if (k == 0) { E[0][q] = fma(w, u[q], E[0][q]); E[1][q] = fma(ws, u[q], E[1][q]); }
        else E[k + 1][q] = fma(w, u[q], E[k + 1][q]);
      }
    }
  }
  const double czj = s.czj[j - 1], gzj = s.gzj[j - 1], gyj = s.gyj[j - 1];
  const int64_t nown = g.nown0 * P1 * P2;
#pragma unroll
  for (int q = 0; q < kL2R; ++q) {
    if (i2 + q >= P2) break;
    const int64_t o = (i0 * P1 + i1) * P2 + i2 + q;
    acc[o] += czj * E[4][q] + gzj * E[3][q];
    acc[nown + o] += czj * E[5][q] + gzj * E[2][q];
    acc[2 * nown + o] += czj * E[6][q] + gzj * E[1][q];
    acc[3 * nown + o] += gyj * E[0][q];
    if (yj) acc[4 * nown + o] += E[7][q];
  }
}

// the affine part of a level after its axis-0 arrays (axis0_u_lin: Lf, Lf s0, z_0..2, y in W0):
// axis 1 (7 arrays into W1), axis 2 + accumulation; arrays of (owned planes) x cstride[0]
static cudaError_t launch_lin3(const StepArgs& s, const Grid& g, const Problem& pb, double* W0, double* W1,
                               double* acc, int j, int WC, cudaStream_t st, int64_t* launches) {
  const int64_t plane = g.cstride[0], cs1 = g.cstride[1], P1 = g.P[1], P2 = g.P[2];
  const int64_t arr = g.nown0 * plane;                 // one array of W0 / W1
  const bool yj = (j == s.Ky);
  (void)pb;
  // axis 1: batch = owned plane, rows = axis-1 coefficient rows, columns = cs1
  auto ax1 = [&](const double* x, double* yp, double* ys) {
    LinAxis p{};
    p.X = x; p.xb = plane; p.xr = cs1; p.xf = 0; p.nf = 1; p.coef[0] = 1.0;
    p.Yp = yp; p.Ys = ys; p.yb = plane; p.yr = cs1;
    p.ncols = cs1; p.nout = P1; p.ibase = 0; p.off = 0; p.Pg = P1;
    p.tap_off = s.tap_off; p.j = j; p.a = 1; p.L = s.L;
    const dim3 gr((unsigned)((cs1 + 127) / 128), (unsigned)((P1 + 7) / 8), (unsigned)g.nown0);
    lin_axis<1><<<gr, 128, 0, st>>>(p);
  };
  ax1(W0, W1, W1 + arr);                               // Lf_pp, Lf_p s1
  ax1(W0 + arr, W1 + 2 * arr, nullptr);                // Lf_s0 p
  for (int k = 0; k < 3; ++k) ax1(W0 + (2 + k) * arr, W1 + (3 + k) * arr, nullptr);
  if (yj) ax1(W0 + 5 * arr, W1 + 6 * arr, nullptr);
  // 64 threads x 3 points: 512 columns split 192 + 192 + 128; the tile's window of the 7 rows in
  // shared memory (bulk copies)
  static_assert(kL2TX == k3TX, "lin_axis2s shares quad3d's column window width");
  const dim3 g2((unsigned)((P2 + kL2TX - 1) / kL2TX), (unsigned)P1, (unsigned)g.nown0);
  lin_axis2s<<<g2, kL2Thr, (size_t)7 * WC * sizeof(double) + 16, st>>>(s, g, W1, arr, acc, j, WC);
  if (launches) *launches += 4 + (yj ? 1 : 0) + 1;
  return cudaGetLastError();
}

template <int DRV, int NF>
static cudaError_t launch_step3d_t(const StepArgs& s, const Grid& g, const Problem& pb, int WC, double* A,
                                   double* acc, cudaStream_t st, int64_t* launches) {
  const size_t smem = fused3d_smem(WC, NF);
  const int64_t plane = g.cstride[0];
  const double4 uc = make_double4(-1.0, pb.dp[5], pb.dp[6], pb.dp[7]);     // U = pi.z - y (NF = 1)
  const double4 lc = make_double4(-pb.dp[0], -pb.dp[2], -pb.dp[3], -pb.dp[4]);   // Lf = -(r y + th.z)
  for (int j = 1; j <= s.K; ++j) {
    const double* C = s.ring + (int64_t)s.slot[j - 1] * s.slot_elems;
    if constexpr (NF == 1) {
      // owned planes only (a slab rank's halo planes feed the stencil rows, never a stack)
      dim3 gu((unsigned)((plane + 127) / 128), (unsigned)((g.nown0 + 7) / 8), 1);
      double* W0 = A + (int64_t)s.L * g.P[0] * plane + (int64_t)(j - 1) * 6 * g.nown0 * plane;
      axis0_u_lin<<<gu, 128, 0, st>>>(C, A, W0, g, s.tap_off, j, s.L, uc, lc);
    } else {
      dim3 ga((unsigned)((plane + 255) / 256), (unsigned)g.nown0, (unsigned)s.L);
      axis0_pass<<<ga, 256, 0, st>>>(C, A, g, s.tap_off, j, s.L);
    }
    dim3 gq((unsigned)((g.P[2] + k3TX - 1) / k3TX), (unsigned)((g.P[1] + k3TY - 1) / k3TY), (unsigned)g.nown0);
    quad3d<DRV, NF><<<gq, k3NT, smem, st>>>(s, g, pb, WC, A, acc, j, j == 1 ? 1 : 0);
    if (launches) *launches += 2;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (NF == 1) {       // the affine part: axes 1 and 2 of every level's axis-0 arrays
    double* W0 = A + (int64_t)s.L * g.P[0] * plane;
    double* W1 = W0 + (int64_t)s.K * 6 * g.nown0 * plane;
    for (int j = 1; j <= s.K; ++j) {
      cudaError_t e = launch_lin3(s, g, pb, W0 + (int64_t)(j - 1) * 6 * g.nown0 * plane, W1, acc, j, WC, st, launches);
      if (e != cudaSuccess) return e;
    }
  }
  const int64_t nown = g.nown0 * g.P[1] * g.P[2];
  epilogue_zy3<DRV><<<(unsigned)((nown + 255) / 256), 256, 0, st>>>(s, g, pb, acc);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

// one d = 3 step: K x (axis-0 pass + quad3d) + epilogue; A holds L x 4 plane stacks of the
// local slab, acc 5 x (owned points) doubles
cudaError_t launch_step3d(const StepArgs& s, const Grid& g, const Problem& pb, int WC, double* A, double* acc,
                          int decompose, cudaStream_t st, int64_t* launches) {
  if (fused3d_smem(WC, k3F) > 112 * 1024) return cudaErrorInvalidConfiguration;
  switch (pb.driver_id) {
    case DRV_ZERO: return launch_step3d_t<DRV_ZERO, k3F>(s, g, pb, WC, A, acc, st, launches);
    case DRV_AFFINE: return launch_step3d_t<DRV_AFFINE, k3F>(s, g, pb, WC, A, acc, st, launches);
    case DRV_EX1: return launch_step3d_t<DRV_EX1, k3F>(s, g, pb, WC, A, acc, st, launches);
    case DRV_DIFF:
      return decompose ? launch_step3d_t<DRV_DIFF, 1>(s, g, pb, WC, A, acc, st, launches)
                       : launch_step3d_t<DRV_DIFF, k3F>(s, g, pb, WC, A, acc, st, launches);
  }
  return cudaErrorInvalidValue;
}

static cudaError_t set_attr_3d() {
  cudaError_t e = cudaFuncSetAttribute(quad3d<DRV_ZERO, k3F>, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(quad3d<DRV_AFFINE, k3F>, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(quad3d<DRV_EX1, k3F>, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(quad3d<DRV_DIFF, k3F>, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(quad3d<DRV_DIFF, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
  return e;
}
