// fused1d_small.cuh -- the d = 1 latency path (included by kernels.cu after fused1d.cuh): the
// whole backward sweep of a small grid (BASELINE cfg 1: P = 256) in ONE launch of ONE CTA.
//
// A small 1-D problem has microseconds of work per step, so launch latency and the per-step
// hand-offs of the multi-CTA kernels dominate it (round 1: 136 launches for cfg 1's 31 steps).
// Here every level the sweep needs -- the K coefficient lines of the ring, the new values and
// the spline scratch -- stays in shared memory for the whole sweep, and each step is
//   (1) Eq. 20 at every grid point: levels 1..K x L nodes on the translation-invariant stencil
//       (taps in constant memory), clamped at the box through the lines'
//       virtual boundary entries, z explicit, y by Picard (Eq. 20, p = 30);
//   (2) the not-a-knot spline of the new level on the whole line: the
//       odd-extension right-hand side and 5 constant-coefficient PCR levels (the same
//       construction as spline_pass / pass 2 of quad1d_fused), written into the level's
//       shared-memory ring slot with its virtual boundary entries;
// separated by CTA barriers only.  At the end the final values, Picard counts and the newest
// coefficient line go to global memory.
#pragma once

struct Small1D {
  Grid g;
  double* ring;              // global ring: slot m % RS holds level m (storage 0 = c_{-1})
  int64_t slot_elems, cfield, cpad;
  int RS, K, Ky, L;
  int tap1_off;
  int n0, nsteps, cur;       // first level computed, number of steps, current value buffer
  double t0, dt, gz0, ky_dt, ky_dt_gy0, picard_tol;
  int picard_max;
  double* vbuf[2];
  int32_t* picard;
  unsigned long long* bad;
  unsigned long long* picard_exec;
  double dp[12];
  double alpha[kPcrLevels];
  double inv_b;
};

// shared memory: RS x 2 coefficient lines of CW = P + 3 + 2 cpad doubles, the values (2 P),
// two PCR arrays (2 x 2 WA)
__host__ __device__ inline int small1d_wa(int P) { return (P + 2) + 8 + 2 * kPcrHalo; }
size_t small1d_smem(int P, int cpad, int RS) {
  const size_t cw = (size_t)P + 3 + 2 * (size_t)cpad;
  return sizeof(double) * ((size_t)RS * 2 * cw + 2 * (size_t)P + 4 * (size_t)small1d_wa(P));
}

// rhs of the odd periodic extension about nodes 1 and P-2 at any c index k (rhs_fold of
// fused1d.cuh with a full modulo: short lines fold several times across the PCR extent)
__device__ __forceinline__ double rhs_fold_any(const double* F, int P, int k, double m1, double mP2) {
  const int period = 2 * (P - 3);
  int u = (k - 1) % period;
  if (u < 0) u += period;
  if (u == 0 || u == P - 3) return 0.0;
  int i;
  double sgn;
  if (u < P - 3) { i = 1 + u; sgn = 1.0; }
  else { i = 1 + period - u; sgn = -1.0; }
  double r = 6.0 * (F[i - 1] - 2.0 * F[i] + F[i + 1]);
  if (i == 2) r -= m1;
  if (i == P - 3) r -= mP2;
  return sgn * r;
}

template <int DRV>
__global__ void __launch_bounds__(256, 1) quad1d_small(const __grid_constant__ Small1D a) {
  extern __shared__ __align__(16) double sm1[];
  const int P = (int)a.g.P[0], cpad = (int)a.cpad;
  const int CW = P + 3 + 2 * cpad, WA = small1d_wa(P), H = kPcrHalo;
  double* const CS = sm1;                                     // [slot][field][CW], storage s at cpad + s
  double* const V = CS + (size_t)a.RS * 2 * CW;               // [2][P]
  double* const T0 = V + 2 * P;                               // [2][WA]
  double* const T1 = T0 + 2 * WA;
  const int tid = threadIdx.x, NT = blockDim.x;
  auto line = [&](int slot, int f) { return CS + ((size_t)slot * 2 + f) * CW + cpad; };   // storage index 0
  // the K input levels n0+1..n0+K from the global ring
  for (int j = 1; j <= a.K; ++j) {
    const int slot = (a.n0 + j) % a.RS;
    for (int f = 0; f < 2; ++f) {
      const double* src = a.ring + (int64_t)slot * a.slot_elems + (int64_t)f * a.cfield - cpad;
      double* dst = line(slot, f) - cpad;
      for (int i = tid; i < CW; i += NT) dst[i] = src[i];
    }
  }
  __syncthreads();
  const Tap1D* const taps = taps1d(a.tap1_off);
  const int base = -1 - 4 - H;                               // PCR extent [base, base + WA) of c indices
  unsigned pexec = 0;
  Driver<DRV, 1> drv(a.dp), dn(a.dp);
  for (int it = 0; it < a.nsteps; ++it) {
    const int n = a.n0 - it;
    const double tn = a.t0 + n * a.dt;
    dn.at(tn);
    // (1) Eq. 20 at every point
    for (int p = tid; p < P; p += NT) {
      double Az = 0.0, Af = 0.0, Ay = 0.0;
      for (int j = a.K; j >= 1; --j) {
        const int slot = (n + j) % a.RS;
        const double* cy = line(slot, 0);
        const double* cz = line(slot, 1);
        const double y0b = cy[-1], z0b = cz[-1], y1b = cy[P + 3], z1b = cz[P + 3];   // clamped boundary values
        drv.at(a.t0 + (n + j) * a.dt);
        const bool yj = (j == a.Ky);
        const Tap1D* tj = taps + (j - 1) * a.L;
        for (int l = 0; l < a.L; ++l) {
          const Tap1D& t = tj[l];
          const int cell = p + t.q;                           // storage cell .. cell + 3
          double yh, zh;
          if (cell >= -3 && cell <= -1) { yh = y0b; zh = z0b; }
          else if (cell >= P - 1 && cell <= P + 2) { yh = y1b; zh = z1b; }
          else {
            yh = fma(t.B[0], cy[cell], fma(t.B[1], cy[cell + 1], fma(t.B[2], cy[cell + 2], t.B[3] * cy[cell + 3])));
            zh = fma(t.B[0], cz[cell], fma(t.B[1], cz[cell + 1], fma(t.B[2], cz[cell + 2], t.B[3] * cz[cell + 3])));
          }
          const double f = drv(yh, &zh);
          Az = fma(t.wcz, zh, fma(t.wgz, f, Az));
          Af = fma(t.wgy, f, Af);
          if (yj) Ay = fma(t.wy, yh, Ay);
        }
      }
      // z (Eq. 20 line 2, explicit) then y by Picard from E[y^{n+Ky}] (Eq. 20 line 1)
      const double z = Az / a.gz0;
      const double rhs = fma(a.ky_dt, Af, Ay);
      int itp;
      const double y = picard_solve([&](double v) { return dn(v, &z); }, Ay, rhs, a.ky_dt_gy0, a.picard_max,
                                    a.picard_tol, itp, pexec);
      V[p] = y;
      V[P + p] = z;
      a.picard[p] = itp;
      if (!isfinite(y) || !isfinite(z)) atomicMin(a.bad, bad_key(n, p));
    }
    __syncthreads();
    // (2) not-a-knot spline of level n into its ring slot: odd-extension rhs, 5 PCR levels
    const double m1_0 = V[0] - 2.0 * V[1] + V[2], m1_1 = V[P] - 2.0 * V[P + 1] + V[P + 2];
    const double mP2_0 = V[P - 3] - 2.0 * V[P - 2] + V[P - 1];
    const double mP2_1 = V[2 * P - 3] - 2.0 * V[2 * P - 2] + V[2 * P - 1];
    for (int p = tid; p < WA; p += NT) {
      const int k = base + p;
      if (k >= 2 && k <= P - 3) {                           // interior row: no fold (no modulo)
        double r0 = 6.0 * (V[k - 1] - 2.0 * V[k] + V[k + 1]);
        double r1 = 6.0 * (V[P + k - 1] - 2.0 * V[P + k] + V[P + k + 1]);
        if (k == 2) { r0 -= m1_0; r1 -= m1_1; }
        if (k == P - 3) { r0 -= mP2_0; r1 -= mP2_1; }
        T0[p] = r0;
        T0[WA + p] = r1;
      } else {
        T0[p] = rhs_fold_any(V, P, k, m1_0, mP2_0);
        T0[WA + p] = rhs_fold_any(V + P, P, k, m1_1, mP2_1);
      }
    }
    __syncthreads();
    const double* A = T0;
    double* B = T1;
#pragma unroll
    for (int l = 0; l < kPcrLevels; ++l) {
      const int sh = 1 << l;
      const double a1 = a.alpha[l];
      for (int p = tid; p < WA; p += NT) {
#pragma unroll
        for (int f = 0; f < 2; ++f) {
          const double* Af_ = A + f * WA;
          const double lft = p - sh >= 0 ? Af_[p - sh] : 0.0;
          const double rgt = p + sh < WA ? Af_[p + sh] : 0.0;
          B[f * WA + p] = Af_[p] - a1 * (lft + rgt);
        }
      }
      __syncthreads();
      const double* t = A;
      A = B;
      B = const_cast<double*>(t);
    }
    const int slot = n % a.RS;
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      const double* Fw = V + f * P;
      const double m1 = f ? m1_1 : m1_0, mP2 = f ? mP2_1 : mP2_0;
      const double* Am = A + f * WA;
      auto mt = [&](int k) { return Am[k - base] * a.inv_b; };
      auto mk = [&](int k) -> double {
        if (k == 1) return m1;
        if (k == P - 2) return mP2;
        if (k == 0) return 2.0 * m1 - (P - 2 == 2 ? mP2 : mt(2));
        if (k == P - 1) return 2.0 * mP2 - (P - 3 == 1 ? m1 : mt(P - 3));
        return mt(k);
      };
      auto coef = [&](int k) -> double {
        if (k >= 2 && k <= P - 3) return Fw[k] - mt(k) * (1.0 / 6.0);
        if (k >= 0 && k < P) return Fw[k] - mk(k) * (1.0 / 6.0);
        if (k < 0) {
          const double c0 = Fw[0] - mk(0) * (1.0 / 6.0), c1 = Fw[1] - m1 * (1.0 / 6.0);
          return 6.0 * Fw[0] - 4.0 * c0 - c1;
        }
        const double cl = Fw[P - 1] - mk(P - 1) * (1.0 / 6.0);
        const double cm = Fw[P - 2] - mP2 * (1.0 / 6.0);
        return 6.0 * Fw[P - 1] - 4.0 * cl - cm;
      };
      double* c = line(slot, f);
      for (int k = -1 + tid; k <= P; k += NT) c[k + 1] = coef(k);
      c[P + 2] = 0.0;                                         // zero pad c_{P+1}
      // virtual boundary entries: s(x_0) = (c_{-1} + 4 c_0 + c_1)/6 and s(x_{P-1}) (only the
      // threads that write them evaluate them)
      if (tid < cpad) {
        const double v0 = (1.0 / 6.0) * coef(-1) + (2.0 / 3.0) * coef(0) + (1.0 / 6.0) * coef(1);
        const double v1 = (1.0 / 6.0) * coef(P - 2) + (2.0 / 3.0) * coef(P - 1) + (1.0 / 6.0) * coef(P);
        for (int i = tid; i < cpad; i += NT) {
          c[-1 - i] = v0;
          c[P + 3 + i] = v1;
        }
      }
    }
    __syncthreads();
  }
  // results: the newest values, the newest coefficient line
  double* vo = a.vbuf[(a.cur + a.nsteps) & 1];
  for (int i = tid; i < 2 * P; i += NT) vo[i] = V[i];
  const int slot = (a.n0 - a.nsteps + 1) % a.RS;
  for (int f = 0; f < 2; ++f) {
    double* dst = a.ring + (int64_t)slot * a.slot_elems + (int64_t)f * a.cfield - cpad;
    const double* src = line(slot, f) - cpad;
    for (int i = tid; i < CW; i += NT) dst[i] = src[i];
  }
  const unsigned ex = __reduce_add_sync(0xffffffffu, pexec);
  if ((tid & 31) == 0 && ex && a.picard_exec) atomicAdd(a.picard_exec, (unsigned long long)ex);
}

template <int DRV>
static cudaError_t launch_small_t(const Small1D& a, size_t smem, cudaStream_t st) {
  static bool attr = false;     // opt in to > 48 KB once per process (per device for multi-GPU hosts)
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(quad1d_small<DRV>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  quad1d_small<DRV><<<1, 256, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_small1d(Small1D& a, int driver_id, cudaStream_t st) {
  pcr_constants(a.alpha, &a.inv_b);
  const size_t smem = small1d_smem((int)a.g.P[0], (int)a.cpad, a.RS);
  switch (driver_id) {
    case DRV_ZERO: return launch_small_t<DRV_ZERO>(a, smem, st);
    case DRV_AFFINE: return launch_small_t<DRV_AFFINE>(a, smem, st);
    case DRV_EX1: return launch_small_t<DRV_EX1>(a, smem, st);
    case DRV_EX2: return launch_small_t<DRV_EX2>(a, smem, st);
    case DRV_DIFF: return launch_small_t<DRV_DIFF>(a, smem, st);
  }
  return cudaErrorInvalidValue;
}

// the remaining sweep of a context: levels n0, n0-1, ..., n0-nsteps+1 (host.cu bsde_solve)
cudaError_t launch_small_sweep(const StepArgs& s, const Grid& g, const Problem& pb, int n0, int nsteps, int cur,
                               double t0, double dt, double* v0, double* v1, cudaStream_t st) {
  Small1D a{};
  a.g = g;
  a.ring = const_cast<double*>(s.ring);
  a.slot_elems = s.slot_elems;
  a.cfield = s.cfield;
  a.cpad = s.cpad;
  a.RS = s.ring_slots;
  a.K = s.K;
  a.Ky = s.Ky;
  a.L = s.L;
  a.tap1_off = s.tap1_off;
  a.n0 = n0;
  a.nsteps = nsteps;
  a.cur = cur;
  a.t0 = t0;
  a.dt = dt;
  a.gz0 = s.gz0;
  a.ky_dt = s.ky_dt;
  a.ky_dt_gy0 = s.ky_dt_gy0;
  a.picard_tol = s.picard_tol;
  a.picard_max = s.picard_max;
  a.vbuf[0] = v0;
  a.vbuf[1] = v1;
  a.picard = s.picard;
  a.bad = s.bad;
  a.picard_exec = s.picard_exec;
  for (int k = 0; k < 12; ++k) a.dp[k] = pb.dp[k];
  return launch_small1d(a, pb.driver_id, st);
}
