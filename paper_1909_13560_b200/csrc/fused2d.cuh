// fused2d.cuh -- the d = 2 fused quadrature kernel (included by kernels.cu, which owns
// the constant tap arena).  The hot kernel of BASELINE cfg 4.
//
// The tensor-product B-spline value at a tap (lambda, mu) is separable:
//   u(x + s) = sum_b B_b(theta_mu) Rw_lambda[c2 + b],  Rw_lambda[k] = sum_a B_a(theta_lambda) C[c1 + a][k]
// so for every level j and axis-0 node lambda a CTA first interpolates its TY coefficient
// rows along axis 0 once ("row pass", 4 FMA per column of the window, both fields' rows
// read from L2 with 7 loads per 4 outputs), then evaluates the L axis-1 nodes mu on the
// shared-memory rows (4 FMA per field per point).  Exact algebra, 2.7x fewer FMAs than the
// direct 16-term tensor stencil at L = 8.
//
// Tile: TY = 4 rows x TX = 64 R columns; thread (r, lb) owns R = 5 consecutive points of
// row r (odd stride: conflict-free LDS.64).  Axis-1 clamping uses the same
// virtual extension as the 1-D kernel: window columns outside [0, P1+2] hold the clamped
// boundary value of the row and the straddling cells take it directly.  Axis-0 clamping is
// per row in the row pass.  Two CTAs per SM overlap one CTA's row pass loads with the
// other's column pass.
#pragma once

constexpr int k2TY = 4;            // tile rows
constexpr int k2R = 3;             // points per thread along axis 1 (odd: conflict-free LDS.64)
constexpr int k2NT = 512;          // threads per CTA (one CTA per SM: 16 warps)
constexpr int k2TX = k2NT / k2TY * k2R;   // 384 tile columns

template <int DRV>
__global__ void __launch_bounds__(k2NT, 1) quad2d(StepArgs s, Grid g, Problem pb, int WC) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* const Rw = reinterpret_cast<double*>(smem_raw);     // [3 fields][TY rows][WC]
  const int tid = threadIdx.x;
  const int r = tid / (k2NT / k2TY), lb = tid % (k2NT / k2TY);
  const int64_t P0g = g.Pg0, P1 = g.P[1];
  const int x0 = blockIdx.x * k2TX;
  const int64_t yl0 = g.own0 + (int64_t)blockIdx.y * k2TY;        // local first row of the tile
  const int64_t yown_end = g.own0 + g.nown0;
  const int L = s.L, K = s.K;
  const int cx0 = x0 + lb * k2R;                                   // thread's first column
  const int64_t yrow = yl0 + r;                                    // thread's row (local)
  const bool rowok = yrow < yown_end;
  const double inv_gz0 = 1.0 / s.gz0;

  Driver<DRV, 2> drv(pb.dp);
  double Az1[k2R], Az2[k2R], Af[k2R], Ay[k2R];
#pragma unroll
  for (int q = 0; q < k2R; ++q) { Az1[q] = 0.0; Az2[q] = 0.0; Af[q] = 0.0; Ay[q] = 0.0; }

  // raw axis-0 rows of the current (level, node) pair: local storage rows first .. first + TY + 2,
  // columns [s0, s0 + nraw) of the level's window, all fields; streamed by bulk copies one pair
  // ahead, behind the previous pair's column pass
  double* const raw = Rw + (size_t)3 * k2TY * WC;                // [3 fields][TY + 3][WC]
  uint64_t* const bar = reinterpret_cast<uint64_t*>(raw + (size_t)3 * (k2TY + 3) * WC);
  const int64_t P0loc = g.P[0];
  auto window = [&](int j, int& wv, int& we) {
    const AxisTap* t1 = axis_taps(s.tap_off) + ((size_t)(j - 1) * 2 + 1) * L;
    const int wa = x0 + t1[0].q;
    wv = wa - (wa & 1);
    we = x0 + k2TX - 1 + t1[L - 1].q + 3;
  };
  auto first_row = [&](int j, int l) -> int64_t {      // local storage row of raw row 0
    const int64_t c = yl0 + g.off0 + axis_taps(s.tap_off)[(size_t)(j - 1) * 2 * L + l].q;
    return (c < 0 ? 0 : (c > P0g - 1 ? P0g - 1 : c)) - g.off0;
  };
  auto issue_rows = [&](int j, int l) {                 // thread 0
    int wv, we;
    window(j, wv, we);
    const int s0 = max(wv, 0), s1 = min(we, (int)P1 + 2);
    const int nraw = ((s1 - s0 + 1) + 1) & ~1;
    const double* Cb = s.ring + (int64_t)s.slot[j - 1] * s.slot_elems + s0;
    const int64_t c0 = first_row(j, l);
    const int nrows = (int)(P0loc + 3 - c0 < k2TY + 3 ? P0loc + 3 - c0 : k2TY + 3);
    const uint32_t bytes = (uint32_t)(nraw * sizeof(double));
    mbar_expect_tx(bar, bytes * nrows * 3);
    for (int f = 0; f < 3; ++f)
      for (int a = 0; a < nrows; ++a)
        bulk_g2s(raw + ((size_t)f * (k2TY + 3) + a) * WC, Cb + (int64_t)f * g.cfield + (c0 + a) * g.cstride[0], bytes,
                 bar);
  };
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) issue_rows(1, 0);
  uint32_t phase = 0;

  for (int j = 1; j <= K; ++j) {
    const AxisTap* t0 = axis_taps(s.tap_off) + (j - 1) * 2 * L;     // axis 0 nodes
    const AxisTap* t1 = t0 + L;                                      // axis 1 nodes
    drv.at(s.t_level[j - 1]);
    const double czj = s.czj[j - 1], gzj = s.gzj[j - 1], gyj = s.gyj[j - 1];
    const bool yj = (j == s.Ky);
    // column window of this level: storage columns [wv, we] (wv even)
    int wv, we;
    window(j, wv, we);
    const int nwin = we - wv + 1;
    const int s0 = max(wv, 0), s1 = min(we, (int)P1 + 2);          // real columns
    const bool left = wv < 0, right = we > P1 + 2;
    for (int l = 0; l < L; ++l) {
      const AxisTap& ta = t0[l];
      // ---- row pass: Rw[f][r'][k] = sum_a B_a C[f][row(r') + a][wv + k], r' < TY, from the raw
      // rows; clamped rows (global cells < 0 or >= P0 - 1) take the boundary basis
      {
        const int64_t cy = yl0 + g.off0 + ta.q;                       // global cell of tile row 0
        const int64_t c0 = (cy < 0 ? 0 : (cy > P0g - 1 ? P0g - 1 : cy)) - g.off0;   // = first_row(j, l)
        const bool consecutive = cy >= 0 && cy + k2TY - 1 <= P0g - 2;
        mbar_wait(bar, phase);
        phase ^= 1u;
        // (field, column) items spread evenly over the threads (3 x ncol items)
        const int ncol = s1 - s0 + 1;
        int f = 0, k = tid;
        while (k >= ncol) { k -= ncol; ++f; }
        for (; f < 3; k += k2NT) {
          while (k >= ncol) { k -= ncol; ++f; }
          if (f >= 3) break;
          {
            const double* rc = raw + (size_t)f * (k2TY + 3) * WC + k;
            double* out = Rw + (size_t)f * k2TY * WC + (s0 - wv) + k;
            if (consecutive) {
              double cin[k2TY + 3];
#pragma unroll
              for (int a = 0; a < k2TY + 3; ++a) cin[a] = rc[a * WC];
#pragma unroll
              for (int rr = 0; rr < k2TY; ++rr)
                out[rr * WC] =
                    fma(ta.B[0], cin[rr], fma(ta.B[1], cin[rr + 1], fma(ta.B[2], cin[rr + 2], ta.B[3] * cin[rr + 3])));
            } else {
#pragma unroll
              for (int rr = 0; rr < k2TY; ++rr) {
                double Bt[4];
                const int64_t cr = clamp_cell(cy + rr, P0g, ta.B, Bt) - g.off0 - c0;
                const double* q = rc + cr * WC;
                out[rr * WC] = fma(Bt[0], q[0], fma(Bt[1], q[WC], fma(Bt[2], q[2 * WC], Bt[3] * q[3 * WC])));
              }
            }
          }
        }
        // the raw rows are free: stream the next pair's behind this pair's column pass
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
          if (l + 1 < L) issue_rows(j, l + 1);
          else if (j + 1 <= K) issue_rows(j + 1, 0);
        }
      }
      // ---- axis-1 boundary: clamped values of every row, virtual window entries
      double bl[3] = {0, 0, 0}, br[3] = {0, 0, 0};     // this thread's row
      if (left || right) {
#pragma unroll
        for (int f = 0; f < 3; ++f) {
          const double* row = Rw + (f * k2TY + r) * WC;
          if (left) bl[f] = (1.0 / 6.0) * row[-wv] + (2.0 / 3.0) * row[1 - wv] + (1.0 / 6.0) * row[2 - wv];
          if (right)
            br[f] = (1.0 / 6.0) * row[P1 - 1 - wv] + (2.0 / 3.0) * row[P1 - wv] + (1.0 / 6.0) * row[P1 + 1 - wv];
        }
        // virtual window entries of every row (one warp per row, no index division); they
        // are disjoint from the real entries the boundary values are read from
        const int nleft = left ? -wv : 0, kright = right ? (int)P1 + 3 - wv : nwin;
        for (int fr = tid >> 5; fr < 3 * k2TY; fr += k2NT / 32) {
          double* row = Rw + fr * WC;
          const int ln = tid & 31;
          if (left) {
            const double v = (1.0 / 6.0) * row[-wv] + (2.0 / 3.0) * row[1 - wv] + (1.0 / 6.0) * row[2 - wv];
            for (int k = ln; k < nleft; k += 32) row[k] = v;
          }
          if (right) {
            const double v = (1.0 / 6.0) * row[P1 - 1 - wv] + (2.0 / 3.0) * row[P1 - wv] + (1.0 / 6.0) * row[P1 + 1 - wv];
            for (int k = kright + ln; k < nwin; k += 32) row[k] = v;
          }
        }
        __syncthreads();
      }
      // ---- column pass over the axis-1 nodes
      const double wl = ta.w, sl = ta.s;
      const double Wcz = wl * czj, Wgz1 = wl * gzj * sl, Wgz = wl * gzj, Wgy = wl * gyj;
      const double* ry = Rw + (0 * k2TY + r) * WC;
      const double* rz1 = Rw + (1 * k2TY + r) * WC;
      const double* rz2 = Rw + (2 * k2TY + r) * WC;
      const int rel0 = cx0 - wv;
      for (int m = 0; m < L; ++m) {
        const AxisTap& tb = t1[m];
        const int q = tb.q;
        double yv[k2R], z1v[k2R], z2v[k2R];
        {
          double c[k2R + 3];
#pragma unroll
          for (int k = 0; k < k2R + 3; ++k) c[k] = ry[rel0 + q + k];
#pragma unroll
          for (int p = 0; p < k2R; ++p)
            yv[p] = fma(tb.B[0], c[p], fma(tb.B[1], c[p + 1], fma(tb.B[2], c[p + 2], tb.B[3] * c[p + 3])));
#pragma unroll
          for (int k = 0; k < k2R + 3; ++k) c[k] = rz1[rel0 + q + k];
#pragma unroll
          for (int p = 0; p < k2R; ++p)
            z1v[p] = fma(tb.B[0], c[p], fma(tb.B[1], c[p + 1], fma(tb.B[2], c[p + 2], tb.B[3] * c[p + 3])));
#pragma unroll
          for (int k = 0; k < k2R + 3; ++k) c[k] = rz2[rel0 + q + k];
#pragma unroll
          for (int p = 0; p < k2R; ++p)
            z2v[p] = fma(tb.B[0], c[p], fma(tb.B[1], c[p + 1], fma(tb.B[2], c[p + 2], tb.B[3] * c[p + 3])));
        }
        const int cb = cx0 + q, ce = cb + k2R - 1;
        if ((left || right) && ((left && cb <= -1 && ce >= -3) || (right && cb <= P1 + 2 && ce >= P1 - 1))) {
#pragma unroll
          for (int p = 0; p < k2R; ++p) {
            const int cell = cb + p;
            if (cell >= -3 && cell <= -1) { yv[p] = bl[0]; z1v[p] = bl[1]; z2v[p] = bl[2]; }
            if (cell >= P1 - 1 && cell <= P1 + 2) { yv[p] = br[0]; z1v[p] = br[1]; z2v[p] = br[2]; }
          }
        }
        const double wm = tb.w;
        const double wcz = Wcz * wm, wgz1 = Wgz1 * wm, wgz2 = Wgz * (wm * tb.s), wgy = Wgy * wm;
#pragma unroll
        for (int p = 0; p < k2R; ++p) {
          const double zz[2] = {z1v[p], z2v[p]};
          const double f = drv(yv[p], zz);
          Az1[p] = fma(wcz, z1v[p], fma(wgz1, f, Az1[p]));
          Az2[p] = fma(wcz, z2v[p], fma(wgz2, f, Az2[p]));
          Af[p] = fma(wgy, f, Af[p]);
        }
        if (yj) {
          const double wy = wl * wm;
#pragma unroll
          for (int p = 0; p < k2R; ++p) Ay[p] = fma(wy, yv[p], Ay[p]);
        }
      }
      __syncthreads();                     // Rw is rewritten by the next row pass
    }
  }
  // ---- epilogue: z explicit (Eq. 20 line 2), y by Picard (Eq. 20 line 1)
  if (!rowok) return;
  Driver<DRV, 2> dn(pb.dp);
  dn.at(s.tn);
#pragma unroll
  for (int p = 0; p < k2R; ++p) {
    const int64_t col = cx0 + p;
    if (col >= P1) break;
    const double z[2] = {Az1[p] * inv_gz0, Az2[p] * inv_gz0};
    const double rhs = fma(s.ky_dt, Af[p], Ay[p]);
    int it;
    unsigned ex = 0;
    const double y = picard_solve([&](double v) { return dn(v, z); }, Ay[p], rhs, s.ky_dt_gy0, s.picard_max,
                                  s.picard_tol, it, ex);
    const int64_t pidx = yrow * P1 + col;
    s.values[pidx] = y;
    s.values[g.npts + pidx] = z[0];
    s.values[2 * g.npts + pidx] = z[1];
    s.picard[pidx] = it;
    if (!isfinite(y) || !isfinite(z[0]) || !isfinite(z[1])) atomicMin(s.bad, bad_key(s.n, pidx));
  }
}

// shared memory of quad2d for a column-window width WC (doubles)
size_t fused2d_smem(int WC) { return (size_t)3 * (2 * k2TY + 3) * WC * sizeof(double) + 16; }

// the widest column window over the levels: TX + (q_max - q_min) on axis 1 + 4 + 2
int fused2d_window(const AxisTap* host_taps, int K, int L) {
  int span = 0;
  for (int j = 1; j <= K; ++j) {
    const AxisTap* t1 = host_taps + ((size_t)(j - 1) * 2 + 1) * L;
    span = span > t1[L - 1].q - t1[0].q ? span : t1[L - 1].q - t1[0].q;
  }
  return (k2TX + span + 6 + 1) & ~1;            // even: 16-byte aligned raw rows
}

template <int DRV>
static cudaError_t launch_quad2d_t(const StepArgs& s, const Grid& g, const Problem& pb, int WC, cudaStream_t st) {
  const size_t smem = fused2d_smem(WC);
  dim3 grid((unsigned)((g.P[1] + k2TX - 1) / k2TX), (unsigned)((g.nown0 + k2TY - 1) / k2TY));
  quad2d<DRV><<<grid, k2NT, smem, st>>>(s, g, pb, WC);
  return cudaGetLastError();
}

cudaError_t launch_quad2d(const StepArgs& s, const Grid& g, const Problem& pb, int WC, cudaStream_t st) {
  if (fused2d_smem(WC) > 220 * 1024) return cudaErrorInvalidConfiguration;
  switch (pb.driver_id) {
    case DRV_ZERO: return launch_quad2d_t<DRV_ZERO>(s, g, pb, WC, st);
    case DRV_AFFINE: return launch_quad2d_t<DRV_AFFINE>(s, g, pb, WC, st);
    case DRV_EX1: return launch_quad2d_t<DRV_EX1>(s, g, pb, WC, st);
    case DRV_DIFF: return launch_quad2d_t<DRV_DIFF>(s, g, pb, WC, st);
  }
  return cudaErrorInvalidValue;
}

static cudaError_t set_attr_2d() {
  cudaError_t e = cudaFuncSetAttribute(quad2d<DRV_ZERO>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(quad2d<DRV_AFFINE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(quad2d<DRV_EX1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(quad2d<DRV_DIFF>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  return e;
}
