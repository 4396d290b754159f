// kernels.cu -- sm_100a fp64 kernels of the multistep BSDE solver.
//
//   layer_kernel      terminal layer y^N = g, z^N = grad g (+ smoothing, R11)
//                     and closed-form initial layers (R9)
//   spline_pass       not-a-knot cubic spline -> B-spline coefficients along one axis,
//                     batched constant-matrix tridiagonal solve by PCR in shared memory
//                     ("two linear systems", north_star (1))
//   quad_generic      fused Gauss-Hermite quadrature (Eq. 21) of spline-interpolated
//                     values + z (Eq. 20 line 2) + Picard y (Eq. 20 line 1), any d
//   quad1d_fused      d = 1: level-1 spline (PCR) + quadrature on shared-memory windows
//                     streamed by cp.async.bulk + z + Picard, one kernel per step (cfg 2)
//   eval_kernel       spline of the newest level at one point (the evaluation point)
#include <climits>
#include <cstdlib>
#include <algorithm>
#include <cstdio>
#include <cuda_runtime.h>
#include "bsde_internal.h"
#include "problems.cuh"

namespace bsde {

// ------------------------------------------------------------------ constant arena
// Byte arena of tap tables (AxisTap for the generic kernel, Tap1D for the fused 1-D
// kernel); each context owns 16-byte aligned ranges (host.cu allocator).
constexpr int kArenaBytes = 63 * 1024;
__constant__ __align__(16) unsigned char c_arena[kArenaBytes];
__constant__ double c_gl_x[kSmoothGL], c_gl_w[kSmoothGL];

cudaError_t upload_arena(const void* data, int bytes, int offset, cudaStream_t st) {
  if (offset < 0 || offset + bytes > kArenaBytes) return cudaErrorInvalidValue;
  return cudaMemcpyToSymbolAsync(c_arena, data, bytes, offset, cudaMemcpyHostToDevice, st);
}
int arena_capacity_bytes() { return kArenaBytes; }
__device__ __forceinline__ const AxisTap* axis_taps(int off) { return reinterpret_cast<const AxisTap*>(c_arena + off); }
__device__ __forceinline__ const Tap1D* taps1d(int off) { return reinterpret_cast<const Tap1D*>(c_arena + off); }
cudaError_t upload_gl(const double* x, const double* w, cudaStream_t st) {
  cudaError_t e = cudaMemcpyToSymbolAsync(c_gl_x, x, sizeof(double) * kSmoothGL, 0, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return e;
  return cudaMemcpyToSymbolAsync(c_gl_w, w, sizeof(double) * kSmoothGL, 0, cudaMemcpyHostToDevice, st);
}

// ------------------------------------------------------------------ layers
__device__ inline void grid_coords(const Grid& g, int64_t p, double* x) {
  for (int a = g.d - 1; a >= 0; --a) {
    const int64_t i = p % g.P[a] + (a == 0 ? g.off0 : 0);      // global index
    p /= g.P[a];
    x[a] = g.xlo[a] + (double)i * g.dx[a];
  }
}

// cell average of g over prod [lo_a, hi_a], axis `fixed` pinned at lo (GL16 tensor rule)
__device__ double smooth_box(const Problem& pb, const double* lo, const double* hi, int fixed) {
  const int d = pb.d;
  int n[kMaxD];
  int tot = 1;
  for (int a = 0; a < d; ++a) { n[a] = a == fixed ? 1 : kSmoothGL; tot *= n[a]; }
  double acc = 0.0;
  for (int m = 0; m < tot; ++m) {
    int rem = m;
    double w[kMaxD], wt = 1.0;
    for (int a = d - 1; a >= 0; --a) {
      const int k = rem % n[a];
      rem /= n[a];
      if (a == fixed) w[a] = lo[a];
      else {
        w[a] = 0.5 * (lo[a] + hi[a]) + 0.5 * (hi[a] - lo[a]) * c_gl_x[k];
        wt *= 0.5 * c_gl_w[k];
      }
    }
    double y, z[kMaxD];
    terminal_eval(pb, w, y, z);
    acc += wt * y;
  }
  return acc;
}

__global__ void layer_kernel(Problem pb, Grid g, double t, int terminal, double* values) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= g.npts) return;
  const int d = g.d;
  double x[kMaxD], y, z[kMaxD];
  grid_coords(g, p, x);
  if (terminal) {
    terminal_eval(pb, x, y, z);
    const int kinked = pb.terminal_id == TRM_CALL || pb.terminal_id == TRM_EXCHANGE || pb.terminal_id == TRM_GEO;
    if (pb.smoothing && kinked) {
      int pos = 0, neg = 0;
      for (int m = 0; m < (1 << d); ++m) {
        double c[kMaxD];
        for (int a = 0; a < d; ++a) c[a] = x[a] + (((m >> a) & 1) ? 0.5 : -0.5) * g.dx[a];
        const double v = payoff_argument(pb, c);
        if (v > 0.0) pos = 1;
        else if (v < 0.0) neg = 1;
        else { pos = 1; neg = 1; }
      }
      if (pos && neg) {
        if (d == 1 && pb.terminal_id == TRM_CALL) {
          // closed-form average of (S0 e^{a + s w} - K)^+ over the cell
          const double* q = pb.tp;
          const double a = (q[2] - 0.5 * q[3] * q[3]) * pb.T, s = q[3];
          const double lo = x[0] - 0.5 * g.dx[0], hi = x[0] + 0.5 * g.dx[0];
          const double wk = (log(q[1] / q[0]) - a) / s;
          const double l = lo > wk ? lo : wk;
          y = hi <= wk ? 0.0 : (q[0] * exp(a) * (exp(s * hi) - exp(s * l)) / s - q[1] * (hi - l)) / (hi - lo);
          double yp, ym, zz[kMaxD];
          double wp = hi, wm = lo;
          terminal_eval(pb, &wp, yp, zz);
          terminal_eval(pb, &wm, ym, zz);
          z[0] = (yp - ym) / g.dx[0];
        } else {
          double lo[kMaxD], hi[kMaxD];
          for (int a = 0; a < d; ++a) { lo[a] = x[a] - 0.5 * g.dx[a]; hi[a] = x[a] + 0.5 * g.dx[a]; }
          y = smooth_box(pb, lo, hi, -1);
          for (int a = 0; a < d; ++a) {
            double lo2[kMaxD], hi2[kMaxD];
            for (int b = 0; b < d; ++b) { lo2[b] = lo[b]; hi2[b] = hi[b]; }
            lo2[a] = hi[a];
            const double up = smooth_box(pb, lo2, hi2, a);
            lo2[a] = lo[a];
            const double dn = smooth_box(pb, lo2, hi2, a);
            z[a] = (up - dn) / g.dx[a];
          }
        }
      }
    }
    if (pb.sde_id != SDE_BROWNIAN)           // z = b^T grad u (forward-SDE problems, Eq. 1)
      for (int a = 0; a < d; ++a) z[a] *= sde_diffusion(pb, a, x[a]);
  } else {
    exact_eval(pb, t, x, y, z);
  }
  values[p] = y;
  for (int a = 0; a < d; ++a) values[(int64_t)(1 + a) * g.npts + p] = z[a];
}

cudaError_t launch_layer(const Problem& pb, const Grid& g, double t, bool terminal, double* values, cudaStream_t st) {
  const int T = 256;
  const int64_t nb = (g.npts + T - 1) / T;
  layer_kernel<<<(unsigned)nb, T, 0, st>>>(pb, g, t, terminal ? 1 : 0, values);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ spline pass (PCR)
struct PassArgs {
  const double* src;   // value index 0 of batch (0,0)
  double* dst;         // storage index 0 (k = -1) of batch (0,0)
  int64_t P;           // line length
  int64_t s_line, d_line;
  int64_t nb0, nb1;    // batch extents (nb1 inner)
  int64_t s_b0, s_b1, d_b0, d_b1;
  int32_t TS;          // outputs per tile
  double alpha[kPcrLevels];
  double inv_b;
  // Dirichlet fold nodes of the moment system: the unknown rows are fa+1 .. fb-1 and the
  // moments at fa, fb are known -- from the not-a-knot end rows at a global line end (nak = 1:
  // fa = 1 / fb = P - 2, outputs extend to the ghosts), or 0 at a slab interface (nak = 0,
  // SPIKE local solve).  Outputs k in [out_lo, out_hi].
  int64_t fa, fb, out_lo, out_hi;
  int32_t nak_a, nak_b;
  // slab interface: the local moments of the first / last unknown row of every line
  // (edge[side * e_side + b0 * e_b0 + b1]), null otherwise
  double* edge;
  int64_t e_side, e_b0;
};
// the default not-a-knot line of P values (outputs c_{-1} .. c_P)
inline void pass_defaults(PassArgs& pa) {
  pa.fa = 1; pa.fb = pa.P - 2; pa.out_lo = -1; pa.out_hi = pa.P;
  pa.nak_a = 1; pa.nak_b = 1; pa.edge = nullptr;
}

// One spline pass: LANES lines per CTA (1: lines along the contiguous axis; > 1: adjacent
// lines of a strided axis, coalesced across the lanes), a tile of TS outputs per line.  The
// line's values window is staged in shared memory first (every global element read once,
// coalesced), then the odd-extension RHS, 5 PCR levels in 3 passes on zero-padded arrays (no
// bounds checks) and the coefficients c = F - m/6 with the not-a-knot end entries, all from
// shared memory; the output is written once.
constexpr int kSplZP = 16;        // zero pad of the PCR arrays: the widest pass reads p +- 16
template <int LANES>
__global__ void spline_pass(PassArgs a) {
  extern __shared__ double sm[];
  const int H = kPcrHalo;
  const int lane = LANES > 1 ? threadIdx.x % LANES : 0;
  const int worker = threadIdx.x / LANES, nworkers = blockDim.x / LANES;
  const int64_t b1 = LANES > 1 ? (int64_t)blockIdx.y * LANES + lane : blockIdx.y;
  const bool valid = b1 < a.nb1;
  const int64_t b0 = blockIdx.z;
  const int64_t P = a.P;
  const double* F = a.src + b0 * a.s_b0 + (valid ? b1 : 0) * a.s_b1;
  double* out = a.dst + b0 * a.d_b0 + (valid ? b1 : 0) * a.d_b1;
  const int64_t sl = a.s_line;
  const int64_t k0 = a.out_lo + (int64_t)blockIdx.x * a.TS;
  const int64_t k1 = min(k0 + (int64_t)a.TS, a.out_hi + 1);
  const int64_t base = k0 - 3 - H;
  const int W = a.TS + 6 + 2 * H;
  const int WZ = W + 2 * kSplZP;
  // staged values F[lo_v .. hi_v] (every index the tile and the folded end rows touch)
  const int64_t lo_v = max(base - 3, (int64_t)0), hi_v = min(base + W + 2, P - 1);
  const int NV = W + 8;
  double* Fs = sm;                                          // [NV][LANES]
  double* A = sm + (size_t)NV * LANES + kSplZP * LANES;     // [WZ][LANES], data at [0, W)
  double* B = A + (size_t)WZ * LANES;
#pragma unroll 8
  for (int64_t k = lo_v + worker; k <= hi_v; k += nworkers)       // several loads in flight per thread
    Fs[(k - lo_v) * LANES + lane] = valid ? F[k * sl] : 0.0;
  for (int i = worker; i < kSplZP; i += nworkers) {        // zero pads of both PCR arrays
    A[(-1 - i) * LANES + lane] = 0.0;
    A[(W + i) * LANES + lane] = 0.0;
    B[(-1 - i) * LANES + lane] = 0.0;
    B[(W + i) * LANES + lane] = 0.0;
  }
  __syncthreads();
  auto Fv = [&](int64_t k) { return Fs[(k - lo_v) * LANES + lane]; };
  // known moments at the fold nodes: the not-a-knot end rows (where this tile reaches them), or
  // 0 at a slab interface
  const int64_t fa = a.fa, fb = a.fb;
  const double ma = a.nak_a && lo_v == 0 ? Fv(0) - 2.0 * Fv(1) + Fv(2) : 0.0;
  const double mb = a.nak_b && hi_v == P - 1 ? Fv(P - 3) - 2.0 * Fv(P - 2) + Fv(P - 1) : 0.0;
  for (int p = worker; p < W; p += nworkers) {
    const int64_t k = base + p;
    double r;
    if (k > fa && k < fb) {
      r = 6.0 * (Fv(k - 1) - 2.0 * Fv(k) + Fv(k + 1));
      if (k == fa + 1) r -= ma;
      if (k == fb - 1) r -= mb;
    } else {                                                // odd periodic extension (images)
      const int64_t period = 2 * (fb - fa);
      int64_t u = (k - fa) % period;
      if (u < 0) u += period;
      if (u == 0 || u == fb - fa) {
        r = 0.0;
      } else {
        int64_t i;
        double sgn;
        if (u < fb - fa) { i = fa + u; sgn = 1.0; }
        else { i = fa + period - u; sgn = -1.0; }
        r = 6.0 * (Fv(i - 1) - 2.0 * Fv(i) + Fv(i + 1));
        if (i == fa + 1) r -= ma;
        if (i == fb - 1) r -= mb;
        r *= sgn;
      }
    }
    A[p * LANES + lane] = r;
  }
  __syncthreads();
  // constant-coefficient PCR, two levels per pass where possible:
  //   u = r - a1 (r[-s] + r[+s]),   v = u - a2 (u[-2s] + u[+2s])
#pragma unroll
  for (int l = 0; l < kPcrLevels; l += 2) {
    const int sh = 1 << l;
    const double a1 = a.alpha[l];
    if (l + 1 < kPcrLevels) {
      const double a2 = a.alpha[l + 1];
      for (int p = worker; p < W; p += nworkers) {
        auto at = [&](int q) { return A[q * LANES + lane]; };
        const double cm1 = at(p - sh), cp1 = at(p + sh), cm2 = at(p - 2 * sh), cp2 = at(p + 2 * sh);
        const double cm3 = at(p - 3 * sh), cp3 = at(p + 3 * sh);
        const double u0 = at(p) - a1 * (cm1 + cp1);
        const double um = cm2 - a1 * (cm3 + cm1);
        const double up = cp2 - a1 * (cp1 + cp3);
        B[p * LANES + lane] = u0 - a2 * (um + up);
      }
    } else {
      for (int p = worker; p < W; p += nworkers)
        B[p * LANES + lane] = A[p * LANES + lane] - a1 * (A[(p - sh) * LANES + lane] + A[(p + sh) * LANES + lane]);
    }
    __syncthreads();
    double* t = A; A = B; B = t;
  }
  if (!valid) return;
  const double ib = a.inv_b;
  auto mt = [&](int64_t k) { return A[(k - base) * LANES + lane] * ib; };
  // moments of the not-a-knot end rows: m_fa, m_fb known, m_0 = 2 m_1 - m_2, m_{P-1} likewise
  auto mk = [&](int64_t k) -> double {
    if (k == fa) return ma;
    if (k == fb) return mb;
    if (k == fa - 1) return 2.0 * ma - (fa + 1 == fb ? mb : mt(fa + 1));
    if (k == fb + 1) return 2.0 * mb - (fb - 1 == fa ? ma : mt(fb - 1));
    return mt(k);
  };
  for (int64_t k = k0 + worker; k < k1; k += nworkers) {
    double c;
    if (k > fa && k < fb) c = Fv(k) - mt(k) * (1.0 / 6.0);
    else if (k >= 0 && k < P) c = Fv(k) - mk(k) * (1.0 / 6.0);
    else if (k < 0) {
      const double c0 = Fv(0) - mk(0) * (1.0 / 6.0), c1 = Fv(1) - ma * (1.0 / 6.0);
      c = 6.0 * Fv(0) - 4.0 * c0 - c1;
    } else {
      const double cl = Fv(P - 1) - mk(P - 1) * (1.0 / 6.0), cm = Fv(P - 2) - mb * (1.0 / 6.0);
      c = 6.0 * Fv(P - 1) - 4.0 * cl - cm;
    }
    out[(k + 1) * a.d_line] = c;
  }
  // SPIKE: the local moments next to the slab interfaces (the reduced system's right-hand side)
  if (a.edge != nullptr && worker == 0) {
    double* e = a.edge + b0 * a.e_b0 + b1;
    if (!a.nak_a && fa + 1 >= k0 && fa + 1 < k1) e[0] = mt(fa + 1);
    if (!a.nak_b && fb - 1 >= k0 && fb - 1 < k1) e[a.e_side] = mt(fb - 1);
  }
}

// Recursive-filter spline pass (r2): the same moment system as spline_pass, solved
// with the factorisation (1, 4, 1) = (-1/rho)(1 - rho z^-1)(1 - rho z), rho = sqrt(3) - 2:
//   u_k = r_k + rho u_{k-1} (causal),  v_k = u_k + rho v_{k+1} (anti-causal),  m = -rho v.
// A CTA owns 32 adjacent lines (lane = line) and a tile of NR = 16 S rows (warp = segment of S
// rows); each segment filters its rows in registers from a zero start, the segment carries are
// chained through shared memory (C_w = e_{w-1} + rho^S C_{w-1}), and the local results are
// corrected by rho^(j+1) C_w (exact: the filters are linear).  The tile starts and ends kRfH = 32
// rows beyond its outputs (the zero start there is the truncation |rho|^32 = 5e-19, the PCR
// pass's coupling bound).  Per element: 3 FMA-class ops for the right-hand side, 2 for the
// filters, 2 for the fix-ups, 1 for c = F - m/6 -- against ~25 for five PCR levels.  STRIDED:
// the lines are adjacent in memory (32 lines = one 256-byte row); else each line is contiguous and
// the tile is transposed through shared memory on the way in and out.
constexpr int kRfH = 32;
constexpr int kRfSeg = 16;             // segments (warps) per CTA
constexpr int kRfT = 32 * kRfSeg;      // threads per CTA
template <int S, bool STRIDED>
__global__ void __launch_bounds__(kRfT, 2) spline_rf(PassArgs a) {
  constexpr int NR = kRfSeg * S;       // tile rows
  constexpr int LD = 33;               // shared-memory pitch (lines + 1: conflict-free transposes)
  extern __shared__ double sm[];
  double* const Fs = sm;                                   // [NR + 2][LD]: rows kb - 1 .. kb + NR
  double* const E = Fs + (size_t)(NR + 2) * LD;            // [kRfSeg][32] segment carries
  double* const Me = E + kRfSeg * 32;                      // [2][32] m at rows fa + 1, fb - 1
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int P = (int)a.P;
  const int k0 = (int)a.out_lo + (int)blockIdx.x * a.TS;
  const int k1 = min(k0 + a.TS, (int)a.out_hi + 1);
  const int kb = k0 - kRfH;                                // first tile row
  const int64_t lb = (int64_t)blockIdx.y * 32;             // first line (b1)
  const int nl = (int)min((int64_t)32, a.nb1 - lb);        // lines of this CTA
  const int lo_v = max(kb - 1, 0), hi_v = min(kb + NR, P - 1);   // staged rows
  const int nv = hi_v - lo_v + 1;
  const double* src = a.src + (int64_t)blockIdx.z * a.s_b0;
  double* dst = a.dst + (int64_t)blockIdx.z * a.d_b0;
  // ---- stage F[lo_v .. hi_v] of the 32 lines (row k of the line at Fs[(k - kb + 1) * LD + line])
  {
    double* const F0 = Fs + (lo_v - kb + 1) * LD;
    if (STRIDED) {
      const double* sp = src + (int64_t)lo_v * a.s_line + lb;
      for (int i = threadIdx.x; i < nv * 32; i += kRfT) {
        const int r = i >> 5, l = i & 31;
        F0[r * LD + l] = l < nl ? __ldg(sp + (int64_t)r * a.s_line + l) : 0.0;
      }
    } else {
      const double* sp = src + lb * a.s_b1 + (int64_t)lo_v * a.s_line;
      for (int l = w; l < 32; l += kRfSeg) {               // warp per line, lanes along it
        const double* q = sp + (int64_t)l * a.s_b1;
        for (int r = lane; r < nv; r += 32) F0[r * LD + l] = l < nl ? __ldg(q + (int64_t)r * a.s_line) : 0.0;
      }
    }
  }
  __syncthreads();
  const double* const Fl = Fs + (1 - kb) * LD + lane;      // Fl[k * LD] = F_k of this lane's line
  auto Fv = [&](int k) { return Fl[k * LD]; };
  const int fa = (int)a.fa, fb = (int)a.fb;
  const double ma = a.nak_a && lo_v == 0 ? Fv(0) - 2.0 * Fv(1) + Fv(2) : 0.0;
  const double mb = a.nak_b && hi_v == P - 1 ? Fv(P - 3) - 2.0 * Fv(P - 2) + Fv(P - 1) : 0.0;
  auto rhs = [&](int k) -> double {                        // odd periodic extension (images)
    const int period = 2 * (fb - fa);
    int u = (k - fa) % period;
    if (u < 0) u += period;
    if (u == 0 || u == fb - fa) return 0.0;
    const int i = u < fb - fa ? fa + u : fa + period - u;
    double r = 6.0 * (Fv(i - 1) - 2.0 * Fv(i) + Fv(i + 1));
    if (i == fa + 1) r -= ma;
    if (i == fb - 1) r -= mb;
    return u < fb - fa ? r : -r;
  };
  const double rho = -0.26794919243112270;                // sqrt(3) - 2
  const int s0 = kb + w * S;                               // this segment's first row
  const bool interior = s0 - 1 > fa && s0 + S < fb;        // every row direct (no fold, no end row)
  // ---- causal filter of the segment from a zero start
  double x[S];
  {
    double u = 0.0;
    if (interior) {
      double fm = Fv(s0 - 1), f0 = Fv(s0);
#pragma unroll
      for (int j = 0; j < S; ++j) {
        const double fp = Fv(s0 + j + 1);
        u = fma(rho, u, 6.0 * (fm - 2.0 * f0 + fp));
        x[j] = u;
        fm = f0;
        f0 = fp;
      }
    } else {
#pragma unroll
      for (int j = 0; j < S; ++j) {
        u = fma(rho, u, rhs(s0 + j));
        x[j] = u;
      }
    }
    E[w * 32 + lane] = u;
  }
  __syncthreads();
  double rs = rho;                                         // rho^S
#pragma unroll
  for (int j = 1; j < S; ++j) rs *= rho;
  {
    double C = 0.0;                                        // true u of row s0 - 1
    for (int q = 0; q < w; ++q) C = fma(rs, C, E[q * 32 + lane]);
    double pw = rho, v = 0.0;
#pragma unroll
    for (int j = 0; j < S; ++j) { x[j] = fma(pw, C, x[j]); pw *= rho; }
    // ---- anti-causal filter from a zero end
#pragma unroll
    for (int j = S - 1; j >= 0; --j) { v = fma(rho, v, x[j]); x[j] = v; }
  }
  __syncthreads();                                         // E is reused for the backward carries
  E[w * 32 + lane] = x[0];
  __syncthreads();
  {
    double D = 0.0;                                        // true v of row s0 + S
    for (int q = kRfSeg - 1; q > w; --q) D = fma(rs, D, E[q * 32 + lane]);
    double pw = rho;
#pragma unroll
    for (int j = S - 1; j >= 0; --j) { x[j] = -rho * fma(pw, D, x[j]); pw *= rho; }   // m
  }
  if (!interior) {
#pragma unroll
    for (int j = 0; j < S; ++j) {
      if (s0 + j == fa + 1) Me[lane] = x[j];
      if (s0 + j == fb - 1) Me[32 + lane] = x[j];
    }
  }
  __syncthreads();                                         // Me complete; Fs still holds F
  const double ib6 = 1.0 / 6.0;
  const double mfa1 = Me[lane], mfb1 = Me[32 + lane];
  // the not-a-knot end rows k <= fa, k >= fb and the ghosts (m_fa, m_fb known, m_0 = 2 m_1 - m_2,
  // c_{-1} = 6 F_0 - 4 c_0 - c_1): computed now, written with the rest
  double ev[3] = {0.0, 0.0, 0.0};
  int ek[3] = {INT_MIN, INT_MIN, INT_MIN};
  if (!interior) {
    int ne = 0;
    for (int t = 0; t < 6; ++t) {
      const bool left = t < 3;
      if (left ? !a.nak_a : !a.nak_b) continue;
      const int k = left ? fa - 2 + t : fb + (t - 3);      // -1, 0, 1 | P-2, P-1, P
      if (k < s0 || k >= s0 + S || k < k0 || k >= k1 || ne >= 3) continue;
      const double m0 = 2.0 * ma - (fa + 1 == fb ? mb : mfa1), mP1 = 2.0 * mb - (fb - 1 == fa ? ma : mfb1);
      double c;
      if (k == fa) c = Fv(fa) - ma * ib6;
      else if (k == fb) c = Fv(fb) - mb * ib6;
      else if (k == 0) c = Fv(0) - m0 * ib6;
      else if (k == P - 1) c = Fv(P - 1) - mP1 * ib6;
      else if (k < 0) c = 6.0 * Fv(0) - 4.0 * (Fv(0) - m0 * ib6) - (Fv(1) - ma * ib6);
      else c = 6.0 * Fv(P - 1) - 4.0 * (Fv(P - 1) - mP1 * ib6) - (Fv(P - 2) - mb * ib6);
      ev[ne] = c;
      ek[ne] = k;
      ++ne;
    }
  }
#pragma unroll
  for (int j = 0; j < S; ++j) x[j] = Fv(s0 + j) - x[j] * ib6;   // c = F - m/6 (rows fa < k < fb)
  const bool valid = lane < nl;
  const int klo = max(k0, max(s0, fa + 1)), khi = min(k1, min(s0 + S, fb));   // direct output rows
  if (STRIDED) {
    if (valid) {
      double* dl = dst + lb + lane;
#pragma unroll
      for (int j = 0; j < S; ++j)
        if (s0 + j >= klo && s0 + j < khi) dl[(int64_t)(s0 + j + 1) * a.d_line] = x[j];
      for (int t = 0; t < 3; ++t)
        if (ek[t] != INT_MIN) dl[(int64_t)(ek[t] + 1) * a.d_line] = ev[t];
    }
  } else {
    __syncthreads();                                       // every F read is done: Fs -> output tile
    double* const Ol = Fs + (1 - kb) * LD + lane;
#pragma unroll
    for (int j = 0; j < S; ++j)
      if (s0 + j >= klo && s0 + j < khi) Ol[(s0 + j) * LD] = x[j];
    for (int t = 0; t < 3; ++t)
      if (ek[t] != INT_MIN) Ol[ek[t] * LD] = ev[t];
    __syncthreads();
    const int no = k1 - k0;
    double* const dp = dst + lb * a.d_b1 + (int64_t)(k0 + 1) * a.d_line;
    const double* const Op = Fs + (k0 - kb + 1) * LD;
    for (int l = w; l < nl; l += kRfSeg) {
      double* q = dp + (int64_t)l * a.d_b1;
      for (int r = lane; r < no; r += 32) q[(int64_t)r * a.d_line] = Op[r * LD + l];
    }
  }
  if (a.edge != nullptr && valid && w == 0) {
    double* e = a.edge + (int64_t)blockIdx.z * a.e_b0 + lb + lane;
    if (!a.nak_a && fa + 1 >= k0 && fa + 1 < k1) e[0] = mfa1;
    if (!a.nak_b && fb - 1 >= k0 && fb - 1 < k1) e[a.e_side] = mfb1;
  }
}
constexpr int kRfS = 20;                 // rows per segment: tiles of 320 rows, 256 outputs
static size_t spline_rf_smem() { return ((size_t)(kRfSeg * kRfS + 2) * 33 + kRfSeg * 32 + 64) * sizeof(double); }

// shared memory of one spline_pass CTA
static size_t spline_smem(int TS, int lanes) {
  const int W = TS + 6 + 2 * kPcrHalo;
  return ((size_t)(W + 8) + 2 * (size_t)(W + 2 * kSplZP)) * lanes * sizeof(double);
}

// PCR constants of the infinite (1,4,1) Toeplitz system, long double on the host
void pcr_constants(double* alpha, double* inv_b) {
  long double av = 1.0L, bv = 4.0L;
  for (int l = 0; l < kPcrLevels; ++l) {
    alpha[l] = (double)(av / bv);
    const long double an = -av * av / bv, bn = bv - 2.0L * av * av / bv;
    av = an; bv = bn;
  }
  *inv_b = (double)(1.0L / bv);
}

static cudaError_t run_pass(PassArgs pa, bool strided, cudaStream_t st, int64_t* launches) {
  pcr_constants(pa.alpha, &pa.inv_b);
  const int64_t n = pa.out_hi - pa.out_lo + 1;             // outputs per line (default c_{-1} .. c_P)
  // many lines: the recursive-filter pass (32 lines per CTA; strided lines must be adjacent)
  if (pa.nb1 >= 32 && (!strided || (pa.s_b1 == 1 && pa.d_b1 == 1))) {
    constexpr int TSr = kRfSeg * kRfS - 2 * kRfH;
    const int64_t nt = (n + TSr - 1) / TSr;
    pa.TS = (int)((n + nt - 1) / nt);
    dim3 grid((unsigned)nt, (unsigned)((pa.nb1 + 31) / 32), (unsigned)pa.nb0);
    if (strided) spline_rf<kRfS, true><<<grid, kRfT, spline_rf_smem(), st>>>(pa);
    else spline_rf<kRfS, false><<<grid, kRfT, spline_rf_smem(), st>>>(pa);
    ++*launches;
    return cudaGetLastError();
  }
  // (PCR) short contiguous lines go 4 lines per CTA, one tile per line: one 256-thread CTA per
  // short line spends its time in barriers and launch overhead
  const bool short_lines = !strided && n <= 1024 && pa.nb1 >= 4;
  if (strided || short_lines) {
    // 4 adjacent lines per CTA (32-byte coalesced row segments: 6 CTAs per SM instead of 3
    // with 8 lines; cfg 4 step 4.76 -> 4.66 ms), tiles of ~256 outputs (halo 27 %)
    constexpr int LN = 4;
    const int64_t nt = short_lines ? 1 : (n + 255) / 256;
    pa.TS = (int)((n + nt - 1) / nt);
    dim3 grid((unsigned)nt, (unsigned)((pa.nb1 + LN - 1) / LN), (unsigned)pa.nb0);
    spline_pass<LN><<<grid, 256, spline_smem(pa.TS, LN), st>>>(pa);
  } else {
    // one line per CTA, tiles of ~2048 outputs (balanced; halo 3 %), or spread over the SMs
    // when there is a single long line
    int64_t nt = (n + 2047) / 2048;
    if (pa.nb0 * pa.nb1 == 1 && n > 4096) nt = (n + 511) / 512;
    pa.TS = (int)((n + nt - 1) / nt);
    dim3 grid((unsigned)nt, (unsigned)pa.nb1, (unsigned)pa.nb0);
    spline_pass<1><<<grid, 256, spline_smem(pa.TS, 1), st>>>(pa);
  }
  ++*launches;
  return cudaGetLastError();
}

// Tensor-product spline of F fields of `values` (value layout) into a ring slot
// (coefficient layout): pass along axis 0, then 1, ....
// d = 1: the virtual boundary entries of every field of a freshly built slot (Grid::cpad)
__global__ void pad_fill_1d(double* slot, int64_t cfield, int64_t P, int64_t cpad) {
  double* c = slot + (int64_t)blockIdx.x * cfield;          // storage 0 of field blockIdx.x
  const double f0 = (1.0 / 6.0) * c[0] + (2.0 / 3.0) * c[1] + (1.0 / 6.0) * c[2];
  const double f1 = (1.0 / 6.0) * c[P - 1] + (2.0 / 3.0) * c[P] + (1.0 / 6.0) * c[P + 1];
  for (int64_t i = threadIdx.x; i < cpad; i += blockDim.x) {
    c[-1 - i] = f0;
    c[P + 3 + i] = f1;
  }
}

cudaError_t launch_spline(const Grid& g, const double* values, int F, double* slot, double* tmp0, double* tmp1,
                          cudaStream_t st, int64_t* launches) {
  const int d = g.d;
  for (int f = 0; f < F; ++f) {
    const double* vsrc = values + (int64_t)f * g.npts;
    double* cdst = slot + (int64_t)f * g.cfield;
    const double* src = vsrc;
    bool src_is_values = true;
    for (int ax = 0; ax < d; ++ax) {
      double* dst = (ax == d - 1) ? cdst : (ax % 2 == 0 ? tmp0 : tmp1);
      PassArgs pa{};
      pa.P = g.P[ax];
      pass_defaults(pa);
      // batch axes: all axes except ax, at most two; the last remaining one is "inner"
      int bax[2], nbx = 0;
      for (int b = 0; b < d; ++b) if (b != ax) bax[nbx++] = b;
      int64_t n[2] = {1, 1}, ss[2] = {0, 0}, ds[2] = {0, 0};
      int64_t soff = 0, doff = 0;
      for (int t = 0; t < nbx; ++t) {
        const int b = bax[t];
        const bool done = b < ax;                 // already spline-transformed -> ghosts included
        n[t] = done ? g.P[b] + 2 : g.P[b];
        ss[t] = src_is_values ? g.vstride[b] : g.cstride[b];
        ds[t] = g.cstride[b];
        if (!done) {
          if (!src_is_values) soff += g.cstride[b];   // value index 0 -> storage index 1
          doff += g.cstride[b];
        }
      }
      // line axis offsets: source value index 0 (storage 1 in coefficient layout)
      if (!src_is_values) soff += g.cstride[ax];
      pa.src = src + soff;
      pa.dst = dst + doff;
      pa.s_line = src_is_values ? g.vstride[ax] : g.cstride[ax];
      pa.d_line = g.cstride[ax];
      if (nbx == 0) { pa.nb0 = 1; pa.nb1 = 1; }
      else if (nbx == 1) { pa.nb0 = 1; pa.nb1 = n[0]; pa.s_b1 = ss[0]; pa.d_b1 = ds[0]; }
      else { pa.nb0 = n[0]; pa.s_b0 = ss[0]; pa.d_b0 = ds[0]; pa.nb1 = n[1]; pa.s_b1 = ss[1]; pa.d_b1 = ds[1]; }
      const bool strided = ax != d - 1;
      cudaError_t e = run_pass(pa, strided, st, launches);
      if (e != cudaSuccess) return e;
      src = dst;
      src_is_values = false;
    }
  }
  if (d == 1 && g.cpad > 0) {
    pad_fill_1d<<<F, 256, 0, st>>>(slot, g.cfield, g.P[0], g.cpad);
    if (launches) ++*launches;
    return cudaGetLastError();
  }
  return cudaSuccess;
}

// ------------------------------------------------------------------ SPIKE (slab partition)
// North_star's "spline solves along the partitioned axis are ... all-gathered" (SURVEY §8(e)
// option 1): rank p solves the axis-0 moment system on its own rows with zero
// coupling to its neighbours (Dirichlet m = 0 at rows r0 - 1 and r1, method of images), emits
// the local moments of its first / last row, the edges of every rank are all-gathered, and the
// true moments are m = m_loc + m(r0 - 1) S^L + m(r1) S^R with the closed-form spike vectors of
// the constant (1, 4, 1) matrix, S^L_k = (rho^{k+1} - rho^{2n+1-k}) / (1 - rho^{2n+2}),
// rho = sqrt(3) - 2.  The interface moments solve a 2 (R - 1) system whose inverse is the same
// for every line (host, long double); the correction is linear, so it is applied to the final
// tensor coefficients: Delta c(k, .) = -(S^L_k XL + S^R_k XR) / 6 with XL, XR the tensor splines
// of the interface moments along axes 1 .. d-1.
__global__ void spike_reduce(SpikeArgs a) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int f = blockIdx.y;
  if (e >= a.plane) return;
  const int64_t rs = (int64_t)a.F * 2 * a.plane;        // rank stride of gath
  const double* G = a.gath + (int64_t)f * 2 * a.plane + e;
  double xl = 0.0, xr = 0.0;
  for (int i = 0; i + 1 < a.R; ++i) {
    const double b = G[(int64_t)i * rs + a.plane];      // last row of rank i
    const double c = G[(int64_t)(i + 1) * rs];          // first row of rank i + 1
    xl = fma(a.wL[2 * i], b, fma(a.wL[2 * i + 1], c, xl));
    xr = fma(a.wR[2 * i], b, fma(a.wR[2 * i + 1], c, xr));
  }
  a.X[((int64_t)f * 2) * a.plane + e] = xl;
  a.X[((int64_t)f * 2 + 1) * a.plane + e] = xr;
}
cudaError_t launch_spike_reduce(const SpikeArgs& a, cudaStream_t st) {
  dim3 grid((unsigned)((a.plane + 255) / 256), (unsigned)a.F);
  spike_reduce<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

// Delta c of the corrected rows: unknown rows [row_lo, row_lo + n) (local), and where a side is a
// global not-a-knot end its two outer rows: m_0 = 2 m_1 - m_2 with m_1 fixed by the data, so
// Delta c_0 = Delta m_2 / 6 and the ghost c_{-1} = 6 F_0 - 4 c_0 - c_1 moves by -4 Delta c_0
// (mirrored at the right end)
__global__ void spike_correct(double* slot, int64_t cfield, int64_t cs0, const double* XC, int64_t plane_c,
                              const double* sLR, int64_t row_lo, int64_t n, int nak_a, int nak_b, int F) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= plane_c) return;
  const int64_t t = blockIdx.y;              // 0 .. n-1 unknown rows, n .. n+3 the not-a-knot extras
  int64_t row, srow;                         // corrected row; row whose Delta m it takes
  double scale;                              // Delta c = scale * Delta m(srow)
  if (t < n) { row = row_lo + t; srow = t; scale = -1.0 / 6.0; }
  else {
    const int x = (int)(t - n);
    if (x < 2) {
      if (!nak_a) return;
      row = row_lo - 2 - x; srow = 0; scale = x == 0 ? 1.0 / 6.0 : -4.0 / 6.0;     // rows 0, -1
    } else {
      if (!nak_b) return;
      row = row_lo + n + 1 + (x - 2); srow = n - 1; scale = x == 2 ? 1.0 / 6.0 : -4.0 / 6.0;   // P-1, P
    }
  }
  const double sl = sLR[srow], sr = sLR[n + srow];
  for (int f = 0; f < F; ++f) {
    const double xl = XC[((int64_t)f * 2) * plane_c + e], xr = XC[((int64_t)f * 2 + 1) * plane_c + e];
    double* c = slot + (int64_t)f * cfield + (row + 1) * cs0 + e;
    *c = fma(scale, fma(sl, xl, sr * xr), *c);
  }
}
cudaError_t launch_spike_correct(double* slot, int64_t cfield, int64_t cs0, const double* XC, int64_t plane_c,
                                 const double* sLR, int64_t row_lo, int64_t n, int nak_a, int nak_b, int F,
                                 cudaStream_t st) {
  dim3 grid((unsigned)((plane_c + 255) / 256), (unsigned)(n + 4));
  spike_correct<<<grid, 256, 0, st>>>(slot, cfield, cs0, XC, plane_c, sLR, row_lo, n, nak_a, nak_b, F);
  return cudaGetLastError();
}

// The local part of a slab rank's tensor spline (SPIKE): the axis-0 pass over the owned rows
// with Dirichlet folds at the interfaces (edges -> edge[F][2][plane]), then the passes along the
// other axes over the owned rows (+ the ghost rows at a global end) only.
cudaError_t launch_spline_slab(const Grid& g, const double* values, int F, double* slot, double* tmp0, double* tmp1,
                               bool first, bool last, double* edge, cudaStream_t st, int64_t* launches) {
  const int d = g.d;
  const int64_t own0 = g.own0, nown = g.nown0, P0 = g.P[0];
  const int64_t plane = g.npts / P0;
  // axis-0 rows the later passes cover (local, -1 = ghost)
  const int64_t rlo = first ? -1 : own0, rhi = last ? P0 : own0 + nown - 1;
  for (int f = 0; f < F; ++f) {
    const double* vsrc = values + (int64_t)f * g.npts;
    double* cdst = slot + (int64_t)f * g.cfield;
    const double* src = vsrc;
    bool src_is_values = true;
    for (int ax = 0; ax < d; ++ax) {
      double* dst = (ax == d - 1) ? cdst : (ax % 2 == 0 ? tmp0 : tmp1);
      PassArgs pa{};
      pa.P = g.P[ax];
      pass_defaults(pa);
      int bax[2], nbx = 0;
      for (int b = 0; b < d; ++b) if (b != ax) bax[nbx++] = b;
      int64_t n[2] = {1, 1}, ss[2] = {0, 0}, ds[2] = {0, 0};
      int64_t soff = 0, doff = 0;
      for (int t = 0; t < nbx; ++t) {
        const int b = bax[t];
        const bool done = b < ax;
        n[t] = done ? g.P[b] + 2 : g.P[b];
        ss[t] = src_is_values ? g.vstride[b] : g.cstride[b];
        ds[t] = g.cstride[b];
        if (!done) {
          if (!src_is_values) soff += g.cstride[b];
          doff += g.cstride[b];
        }
        if (b == 0 && done) {                   // axis 0 transformed: only rows [rlo, rhi]
          n[t] = rhi - rlo + 1;
          soff += (rlo + 1) * ss[t];
          doff += (rlo + 1) * ds[t];
        }
      }
      if (!src_is_values) soff += g.cstride[ax];
      pa.src = src + soff;
      pa.dst = dst + doff;
      pa.s_line = src_is_values ? g.vstride[ax] : g.cstride[ax];
      pa.d_line = g.cstride[ax];
      if (nbx == 0) { pa.nb0 = 1; pa.nb1 = 1; }
      else if (nbx == 1) { pa.nb0 = 1; pa.nb1 = n[0]; pa.s_b1 = ss[0]; pa.d_b1 = ds[0]; }
      else { pa.nb0 = n[0]; pa.s_b0 = ss[0]; pa.d_b0 = ds[0]; pa.nb1 = n[1]; pa.s_b1 = ss[1]; pa.d_b1 = ds[1]; }
      if (ax == 0) {
        pa.nak_a = first ? 1 : 0;
        pa.nak_b = last ? 1 : 0;
        pa.fa = first ? 1 : own0 - 1;
        pa.fb = last ? P0 - 2 : own0 + nown;
        pa.out_lo = first ? -1 : own0;
        pa.out_hi = last ? P0 : own0 + nown - 1;
        pa.edge = edge + (int64_t)f * 2 * plane;
        pa.e_side = plane;
        pa.e_b0 = nbx == 2 ? n[1] : 0;
      }
      cudaError_t e = run_pass(pa, ax != d - 1, st, launches);
      if (e != cudaSuccess) return e;
      src = dst;
      src_is_values = false;
    }
  }
  return cudaSuccess;
}

// ------------------------------------------------------------------ interpolation helpers
// per-axis cell and basis with boundary clamping (R6):
// outside the box the coordinate is clamped, i.e. the spline is evaluated at the
// boundary knot: cell 0 / P-1 with theta = 0 -> B = (1/6, 2/3, 1/6, 0).
__device__ inline int64_t clamp_cell(int64_t c, int64_t P, const double* Bin, double* B) {
  if (c < 0 || c >= P - 1) {
    B[0] = 1.0 / 6.0; B[1] = 2.0 / 3.0; B[2] = 1.0 / 6.0; B[3] = 0.0;
    return c < 0 ? 0 : P - 1;
  }
  B[0] = Bin[0]; B[1] = Bin[1]; B[2] = Bin[2]; B[3] = Bin[3];
  return c;
}

template <int D>
__device__ inline double gather(const double* __restrict__ C, const int64_t* cs, const int64_t* cell,
                                const double (*B)[4]) {
  if (D == 1) {
    const double* c = C + cell[0];
    return B[0][0] * __ldg(c) + B[0][1] * __ldg(c + 1) + B[0][2] * __ldg(c + 2) + B[0][3] * __ldg(c + 3);
  } else if (D == 2) {
    double v = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < 4; ++k0) {
      const double* c = C + (cell[0] + k0) * cs[0] + cell[1];
      const double row = B[1][0] * __ldg(c) + B[1][1] * __ldg(c + 1) + B[1][2] * __ldg(c + 2) + B[1][3] * __ldg(c + 3);
      v = fma(B[0][k0], row, v);
    }
    return v;
  } else {
    double v = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < 4; ++k0) {
      double pl = 0.0;
#pragma unroll
      for (int k1 = 0; k1 < 4; ++k1) {
        const double* c = C + (cell[0] + k0) * cs[0] + (cell[1] + k1) * cs[1] + cell[2];
        const double row = B[2][0] * __ldg(c) + B[2][1] * __ldg(c + 1) + B[2][2] * __ldg(c + 2) + B[2][3] * __ldg(c + 3);
        pl = fma(B[1][k1], row, pl);
      }
      v = fma(B[0][k0], pl, v);
    }
    return v;
  }
}

// Epilogue shared by all quadrature kernels: z (Eq. 20 line 2, explicit) then y by
// Picard iteration on Eq. 20 line 1 starting from E[y^{n+Ky}] (R8, R18).
template <int DRV, int D>
__device__ inline void epilogue(const StepArgs& s, int64_t p, int64_t npts, double Ay, double Af, const double* Az,
                                const double* dp) {
  Driver<DRV, D> drv(dp);
  drv.at(s.tn);
  double z[D];
#pragma unroll
  for (int a = 0; a < D; ++a) z[a] = Az[a] / s.gz0;
  const double rhs = fma(s.ky_dt, Af, Ay);
  int it;
  unsigned ex = 0;
  const double y = picard_solve([&](double v) { return drv(v, z); }, Ay, rhs, s.ky_dt_gy0, s.picard_max,
                                s.picard_tol, it, ex);
  s.values[p] = y;
  bool bad = !isfinite(y);
#pragma unroll
  for (int a = 0; a < D; ++a) {
    s.values[(int64_t)(1 + a) * npts + p] = z[a];
    bad |= !isfinite(z[a]);
  }
  s.picard[p] = it;
  if (bad) atomicMin(s.bad, bad_key(s.n, p));
}

// ------------------------------------------------------------------ generic fused kernel
// One thread per grid point; for level j and node tuple Lambda the tap is the
// translation-invariant stencil (q_Lambda, theta_Lambda) of PAPER.md:391-392.
template <int D, int DRV>
__global__ void __launch_bounds__(256) quad_generic(StepArgs s, Grid g, Problem pb) {
  // owned points only: rows [own0, own0 + nown0) of the (possibly partitioned) axis 0
  int64_t rowlen = 1;
#pragma unroll
  for (int a = 1; a < D; ++a) rowlen *= g.P[a];
  const int64_t q0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q0 >= g.nown0 * rowlen) return;
  const int64_t p = g.own0 * rowlen + q0;           // local linear index
  int64_t idx[D];
  {
    int64_t r = p;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) { idx[a] = r % g.P[a]; r /= g.P[a]; }
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
        if (a == 0)   // clamp at the global box, then back to local storage rows
          cell[a] = clamp_cell(idx[a] + g.off0 + t.q, g.Pg0, t.B, B[a]) - g.off0;
        else
          cell[a] = clamp_cell(idx[a] + t.q, g.P[a], t.B, B[a]);
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

// ------------------------------------------------------------------ 1-D fused step kernel
#include "fused1d.cuh"
#include "fused1d_small.cuh"

// ------------------------------------------------------------------ 2-D fused quadrature kernel
#include "fused2d.cuh"
#include "fused3d.cuh"
#include "aff2.cuh"
#include "fsde.cuh"
#include "bicubic.cuh"

template <int D, int DRV>
static cudaError_t launch_generic(const StepArgs& s, const Grid& g, const Problem& pb, cudaStream_t st) {
  const int T = 256;
  const int64_t nown = g.npts / g.P[0] * g.nown0;
  const int64_t nb = (nown + T - 1) / T;
  quad_generic<D, DRV><<<(unsigned)nb, T, 0, st>>>(s, g, pb);
  return cudaGetLastError();
}

template <int D>
static cudaError_t dispatch_generic(const StepArgs& s, const Grid& g, const Problem& pb, cudaStream_t st) {
  switch (pb.driver_id) {
    case DRV_ZERO: return launch_generic<D, DRV_ZERO>(s, g, pb, st);
    case DRV_AFFINE: return launch_generic<D, DRV_AFFINE>(s, g, pb, st);
    case DRV_EX1: return launch_generic<D, DRV_EX1>(s, g, pb, st);
    case DRV_EX2: return launch_generic<D, DRV_EX2>(s, g, pb, st);
    case DRV_DIFF: return launch_generic<D, DRV_DIFF>(s, g, pb, st);
  }
  return cudaErrorInvalidValue;
}

// generic fused quadrature kernel (any d); the spline of level n+1 is built by
// launch_spline before it
cudaError_t launch_generic_step(const StepArgs& s, const Grid& g, const Problem& pb, cudaStream_t st) {
  switch (g.d) {
    case 1: return dispatch_generic<1>(s, g, pb, st);
    case 2: return dispatch_generic<2>(s, g, pb, st);
    case 3: return dispatch_generic<3>(s, g, pb, st);
  }
  return cudaErrorInvalidValue;
}

// opt in to > 48 KB dynamic shared memory on the current device (called per context)
cudaError_t init_device_attributes() {
  const int lim = 200 * 1024;
  cudaError_t e = cudaFuncSetAttribute(spline_pass<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(spline_pass<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(spline_rf<kRfS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(spline_rf<kRfS, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  if (e == cudaSuccess) e = set_attr_drv<DRV_ZERO>();
  if (e == cudaSuccess) e = set_attr_drv<DRV_AFFINE>();
  if (e == cudaSuccess) e = set_attr_drv<DRV_EX1>();
  if (e == cudaSuccess) e = set_attr_drv<DRV_EX2>();
  if (e == cudaSuccess) e = set_attr_drv<DRV_DIFF>();
  if (e == cudaSuccess) e = set_attr_2d();
  if (e == cudaSuccess) e = set_attr_3d();
  if (e == cudaSuccess) e = set_attr_aff2();
  return e;
}

// ------------------------------------------------------------------ evaluation point
__global__ void eval_kernel(Grid g, const double* slot, int F, double x0, double x1, double x2, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double x[3] = {x0, x1, x2};
  int64_t cell[kMaxD];
  double B[kMaxD][4];
  for (int a = 0; a < g.d; ++a) {
    double X = fmin(fmax(x[a], g.xlo[a]), g.xhi[a]);
    const double u = (X - g.xlo[a]) / g.dx[a];
    const int64_t Pa = a == 0 ? g.Pg0 : g.P[a];
    int64_t c = (int64_t)floor(u);
    if (c > Pa - 2) c = Pa - 2;
    if (c < 0) c = 0;
    const double t = u - (double)c;
    if (a == 0) c -= g.off0;                       // local storage row (the owner evaluates)
    B[a][0] = (1.0 - t) * (1.0 - t) * (1.0 - t) / 6.0;
    B[a][1] = (3.0 * t * t * t - 6.0 * t * t + 4.0) / 6.0;
    B[a][2] = (-3.0 * t * t * t + 3.0 * t * t + 3.0 * t + 1.0) / 6.0;
    B[a][3] = t * t * t / 6.0;
    cell[a] = c;
  }
  for (int f = 0; f < F; ++f) {
    const double* C = slot + (int64_t)f * g.cfield;
    double v = 0.0;
    if (g.d == 1) v = gather<1>(C, g.cstride, cell, B);
    else if (g.d == 2) v = gather<2>(C, g.cstride, cell, B);
    else v = gather<3>(C, g.cstride, cell, B);
    out[f] = v;
  }
}

cudaError_t launch_eval(const Grid& g, const double* slot, int F, const double* x, double* out, cudaStream_t st) {
  eval_kernel<<<1, 32, 0, st>>>(g, slot, F, x[0], g.d > 1 ? x[1] : 0.0, g.d > 2 ? x[2] : 0.0, out);
  return cudaGetLastError();
}

}  // namespace bsde

namespace bsde {
// FP64 peak probe: 16 independent DFMA chains per thread (enough ILP to cover the DFMA
// latency at 8 warps per SM partition), results folded into one store so nothing is dead
__global__ void __launch_bounds__(256) fp64_peak_kernel(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;     // practically never taken; keeps the chains live
}

cudaError_t measure_fp64_peak(int device, int iters, double* tflops, double* ms_out) {
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return e;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  double* out = nullptr;
  if ((e = cudaMalloc(&out, sizeof(double))) != cudaSuccess) return e;
  const int blocks = nsm * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fp64_peak_kernel<<<blocks, threads>>>(out, iters / 10 + 1, 0.999999, 1e-7);   // warm-up (clocks up)
  cudaEventRecord(e0);
  fp64_peak_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  e = cudaEventSynchronize(e1);
  float ms = 0.f;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (e != cudaSuccess) return e;
  const double flops = 2.0 * 16.0 * (double)iters * blocks * threads;
  *tflops = flops / (ms * 1e-3) / 1e12;
  *ms_out = ms;
  return cudaSuccess;
}
}  // namespace bsde
