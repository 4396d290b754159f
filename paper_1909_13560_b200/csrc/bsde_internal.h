// bsde_internal.h -- data structures shared by the host runtime (host.cu) and the
// kernels (kernels.cu) of the B200 multistep BSDE solver.  Not part of the ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bsde {

constexpr int kMaxD = 3;
constexpr int kMaxK = 6;
constexpr int kMaxL = 64;
constexpr int kPcrLevels = 5;       // PCR levels of the constant (1,4,1) system; coupling
                                    // after 5 levels: a5/b5 = 5.0e-19
constexpr int kPcrHalo = (1 << kPcrLevels) - 1;   // 31
// (r2) pass 2 of the fused 1-D kernel: the recursive filter on globally aligned segments of kP2Seg
// rows, carries over kP2Q segments (|rho|^(7 x 6) = 1e-24); its window reaches at most kP2Halo
// rows beyond the outputs
constexpr int kP2Seg = 7, kP2Q = 6;
constexpr int kP2Halo = kP2Seg * (kP2Q + 1);       // 49
constexpr int kSmoothGL = 16;       // Gauss-Legendre nodes per axis for d >= 2 smoothing

// One entry of a per-level, per-axis tap table (translation-invariant stencil,
// PAPER.md:391-392): node l of level j shifts every grid point by
// s = sqrt(2 j dt) a_l = (q + theta) dx.
struct AxisTap {
  int32_t q;          // integer cell offset floor(s/dx)
  int32_t pad;
  double B[4];        // cubic B-spline basis at theta: (1-t)^3/6, (3t^3-6t^2+4)/6, ...
  double w;           // omega_l / sqrt(pi)
  double s;           // Brownian increment sqrt(2 j dt) a_l
};

// Per-(level, node) record of the fused 1-D kernel: the stencil (q, B) of AxisTap and the
// scheme weights folded in on the host: wcz = w ([j==1] - gz_j), wgz = w gz_j s,
// wgy = w gy_j, wy = w [j == Ky] (Eq. 20 with Eq. 21).
struct Tap1D {
  int32_t q;
  int32_t pad;
  double B[4];
  double wcz, wgz, wgy, wy;
};

struct Problem {
  int32_t d;
  int32_t driver_id, terminal_id;
  int32_t smoothing;
  double dp[12];
  double tp[12];
  double T, t0, dt;
  int32_t N;
  int32_t sde_id;          // forward SDE (bsde_sde_id; 0: X = W)
  double sp[12];           // its parameters
};

struct Grid {
  int32_t d;
  int64_t P[kMaxD];        // points per axis
  double xlo[kMaxD], xhi[kMaxD], dx[kMaxD];
  int64_t vstride[kMaxD];  // value layout strides (row-major, last axis contiguous)
  int64_t cstride[kMaxD];  // coefficient layout strides (extent P+3 per axis, storage k+1)
  int64_t npts;            // product of P
  int64_t cfield;          // elements of one coefficient field (incl. padding)
  // slab partition along axis 0 (d >= 2, nranks > 1): P[0] is the local extended slab,
  // local row 0 is global row off0, owned rows are local [own0, own0 + nown0); the global
  // axis-0 extent Pg0 is what clamping sees.  One rank: off0 = own0 = 0, nown0 = Pg0 = P[0].
  int64_t off0, Pg0, own0, nown0;
  // d = 1: every coefficient line carries cpad virtual entries on each side (storage -cpad..-1
  // and P+3..P+2+cpad) holding the clamped boundary values s(x_0), s(x_{P-1}) of that level
  // (PAPER.md:385), so the fused kernel's windows need no boundary fill; 0 for d >= 2
  int64_t cpad;
};

// Per-step parameters of the fused quadrature / z / Picard kernel (Eq. 20).
struct StepArgs {
  const double* ring;      // coefficient ring base
  int64_t slot_elems;      // elements per ring slot (F * cfield)
  int64_t cfield, cpad;    // the context's Grid::cfield / Grid::cpad (batched problems may differ)
  int32_t slot[kMaxK];     // ring slot of level n+j, j = 1..K (index j-1); the generic path
                           // rebuilds slot[0] from values_in at the start of the step
  int32_t slot_out;        // fused 1-D path: ring slot that receives the spline of the new
                           // level n (-1: none)
  double t_level[kMaxK];   // t_{n+j}
  double czj[kMaxK];       // coefficient of E[z^{n+j}] in z^n*gz0: [j==1] - gz_j
  double gzj[kMaxK];       // gz_j (0 for j > Kz): coefficient of E[f dW]
  double gyj[kMaxK];       // gy_j (0 for j > Ky): coefficient of E[f]
  int32_t K, Ky, Kz, L;
  int32_t ring_slots;      // RS: level m lives in ring slot m % RS
  int32_t tap_off;         // byte offset of the AxisTap table (K x d x L) in the constant arena
  int32_t tap1_off;        // byte offset of the Tap1D table (K x L, d = 1) in the constant arena
  double gz0, ky_dt_gy0, ky_dt, tn;
  double dt;               // step size of this step (the bootstrap's sub-step size inside bsde_setup)
  int32_t picard_max;
  double picard_tol;
  const double* values_in; // level n+1 values (input of the level-1 spline)
  double* values;          // out: F * npts (level n)
  int32_t* picard;         // out: npts
  unsigned long long* bad; // first non-finite output: min of bad_key(n, point) (bsde_internal.h)
  int32_t n;               // index of the level this step computes (ring_mode 0 launches)
  unsigned long long* picard_exec;   // optional: + the Picard iterations executed (fused 1-D kernel)
  unsigned long long* phase_ns;  // optional (debug): per-CTA %globaltimer stamps of the fused kernel
};

// Non-finite diagnostic key: the sweep runs n = N-K .. 0, so the smallest key is the first
// (largest n) non-finite point; decoded by the host (bsde_last_error names n, i, t, x, y, z).
constexpr int kBadShift = 40;
__host__ __device__ inline unsigned long long bad_key(int n, long long point) {
  return ((unsigned long long)(0xFFFFFu - (unsigned)n) << kBadShift) | (unsigned long long)point;
}

// Geometry of the fused 1-D step kernel (kernels.cu, quad1d_fused).
struct Fused1D {
  int variant;               // index into the instantiated (R, C, threads, unroll) table
  int TP;                    // points per CTA
  int WMAX;                  // doubles per field buffer in shared memory
  int WP;                    // doubles per PCR scratch array (own-tile spline)
  int WS;                    // doubles of the pass-2 spline scratch (values window + 2 PCR arrays)
  int TK;                    // doubles of the shared-memory tap table (K x L Tap1D)
  int sep;                   // 1: the spline scratch has its own shared memory (the next round's
                             // first windows stream in during pass 2); 0: it overlays the buffers
  double alpha[kPcrLevels];  // PCR elimination ratios
  double inv_b;              // 1 / b after the last PCR level
};

// Launch parameters of the fused kernel.  All CTAs of a launch are co-resident
// (cooperative launch); CTAs synchronise only with the neighbours they exchange data
// with, through per-CTA progress flags:
//   done_flag[b] = it + 1  once CTA b wrote its tile of the level-n values (pass 1 of step it)
//   ring_flag[b] = it + 1  once CTA b wrote its tile of the level-n coefficients (pass 2)
struct Persist1D {
  int n0, nsteps, ring_mode, cur;
  double t0, dt;
  double* vbuf[2];
  unsigned* ring_flag;
  unsigned* done_flag;
  int D[kMaxK + 1];  // D[j]: CTA distance of level j's window (j >= 1); D[0]: values halo of phase A
  int DK;            // max of D
  int nowait;        // debug build only (-DBSDE_DEBUG, BSDE_DEBUG_NOWAIT): skip every flag wait -- wrong results, busy time only
  int nopad;         // debug build only (-DBSDE_DEBUG, BSDE_DEBUG_NOPAD): skip the edge CTAs' pad fill -- wrong results
};

// One problem of a fused launch and the launch itself.  All problems of a launch share the
// grid, the driver template and the CTA geometry; each has its own levels, taps, ring, value
// buffers and progress flags.  CTAs run the problems' steps round-robin (step it of problem
// 0, 1, ..., then step it + 1), so a problem's neighbour waits overlap the other problems'
// work.  A single solve is a batch of one.
constexpr int kMaxRanks = 16;
struct SpikeArgs {
  const double* gath;        // [R][F][2][plane] edges of every rank (side 0: first row, 1: last)
  double* X;                 // [F][2][plane] this rank's m(r0 - 1), m(r1) (0 at global ends)
  int64_t plane;             // values per axis-0 row (value layout)
  int F, R;
  // xL = sum_j wL[j] rhs_j, xR = sum_j wR[j] rhs_j; rhs_{2i} = last-row edge of rank i,
  // rhs_{2i+1} = first-row edge of rank i + 1 (i = 0 .. R-2)
  double wL[2 * kMaxRanks], wR[2 * kMaxRanks];
};

constexpr int kMaxBatch = 8;
constexpr int kFlagCap = 8192;   // progress flags per kind and context (the workspace holds 2 x kFlagCap)
struct FusedProb {
  StepArgs s;
  Persist1D pp;
  double dp[12];       // driver parameters
};

}  // namespace bsde
