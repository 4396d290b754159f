// host.cu -- C ABI (include/bsde.h) and host runtime of the B200 multistep BSDE solver.
//
// Setup (steps 1-2 of the algorithm) runs on the host: grids and the
// balance rule, the Gauss-Hermite rule (Eq. 21), the weight rows (Tables 1-2), the
// translation-invariant tap tables uploaded to constant memory.
// Everything that touches grid data (terminal/initial layers, spline builds, the
// backward sweep of Eq. 20) runs in the kernels of kernels.cu.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>

#include "../../include/bsde.h"
#include "bsde_internal.h"

namespace bsde {
cudaError_t upload_arena(const void* data, int bytes, int offset, cudaStream_t st);
int arena_capacity_bytes();
cudaError_t upload_gl(const double* x, const double* w, cudaStream_t st);
cudaError_t launch_layer(const Problem& pb, const Grid& g, double t, bool terminal, double* values, cudaStream_t st);
cudaError_t launch_spline(const Grid& g, const double* values, int F, double* slot, double* tmp0, double* tmp1,
                          cudaStream_t st, int64_t* launches);
cudaError_t launch_generic_step(const StepArgs& s, const Grid& g, const Problem& pb, cudaStream_t st);
bool fused1d_geometry(const Grid& g, int K, int L, int qspan_max, int nsm, int variant, Fused1D& fz,
                      int& threads, int& blocks, size_t& smem);
int fused1d_num_variants();
int fused1d_alt_variant();
cudaError_t launch_fused1d_steps(const StepArgs& s, const Grid& g, const Problem& pb, const Fused1D& fz, int n0,
                                 int nsteps, int ring_mode, int cur, double t0, double dt, double* v0, double* v1,
                                 unsigned* flags, const int* D, int DK, int threads, int blocks, size_t smem,
                                 cudaStream_t st);
int fused1d_blocks_per_sm(int variant, size_t smem);
size_t fused1d_smem(Fused1D& fz);
cudaError_t measure_fp64_peak(int device, int iters, double* tflops, double* ms_out);
cudaError_t launch_fused1d_batch(const FusedProb* probs, int nprob, const Grid& g, const Fused1D& fz, int driver_id,
                                 int threads, int blocks, size_t smem, cudaStream_t st, const int* group,
                                 const int* gcta, const int* gns, int ngroup);
cudaError_t launch_eval(const Grid& g, const double* slot, int F, const double* x, double* out, cudaStream_t st);
cudaError_t init_device_attributes();
cudaError_t launch_quad2d(const StepArgs& s, const Grid& g, const Problem& pb, int WC, cudaStream_t st);
cudaError_t launch_aff2(const StepArgs& s, const Grid& g, const Problem& pb, double* H, int WC, cudaStream_t st,
                        int64_t* launches);
int aff2_window(const AxisTap* host_taps, int K, int L);
size_t aff2_smem(int WC);
int fused2d_window(const AxisTap* host_taps, int K, int L);
size_t fused2d_smem(int WC);
int fused3d_window(const AxisTap* host_taps, int K, int L);
size_t fused3d_smem(int WC, int nf);
struct Small1D;
size_t small1d_smem(int P, int cpad, int RS);
cudaError_t launch_small_sweep(const StepArgs& s, const Grid& g, const Problem& pb, int n0, int nsteps, int cur, double t0,
                               double dt, double* v0, double* v1, cudaStream_t st);
cudaError_t launch_fsde_step(const StepArgs& s, const Grid& g, const Problem& pb, cudaStream_t st);
cudaError_t launch_hermite(const Grid& g, const double* values, int F, double* slot, cudaStream_t st, int64_t* launches);
cudaError_t launch_bicubic_step(const StepArgs& s, const Grid& g, const Problem& pb, cudaStream_t st);
cudaError_t launch_eval_bicubic(const Grid& g, const double* slot, int F, const double* x, double* out, cudaStream_t st);
cudaError_t launch_step3d(const StepArgs& s, const Grid& g, const Problem& pb, int WC, double* A, double* acc,
                          int decompose, cudaStream_t st, int64_t* launches);
cudaError_t launch_spike_reduce(const SpikeArgs& a, cudaStream_t st);
cudaError_t launch_spike_correct(double* slot, int64_t cfield, int64_t cs0, const double* XC, int64_t plane_c,
                                 const double* sLR, int64_t row_lo, int64_t n, int nak_a, int nak_b, int F,
                                 cudaStream_t st);
cudaError_t launch_spline_slab(const Grid& g, const double* values, int F, double* slot, double* tmp0, double* tmp1,
                               bool first, bool last, double* edge, cudaStream_t st, int64_t* launches);
}  // namespace bsde

using namespace bsde;

// ------------------------------------------------------------------ errors
static thread_local std::string g_setup_error;

struct bsde_ctx {
  bsde_config cfg{};
  Problem pb{};
  Grid g{};
  int d = 1, F = 2, K = 1, Ky = 1, Kz = 1, L = 1, N = 1;
  double dt = 0;
  int level = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  char* ws = nullptr;
  size_t ws_bytes = 0;
  bool own_ws = false;
  double* vbuf[2] = {nullptr, nullptr};   // ping-pong value buffers, F * npts each
  int cur = 0;                  // vbuf[cur] holds the newest level
  int fused_variant = 0;        // fused 1-D kernel variant (kernel_variant = 10 + v)
  bool small_ok = false;        // d = 1 latency path: the whole sweep in one single-CTA launch
  int wc2 = 0, boot_wc2 = 0;    // 2-D / 3-D fused kernel column window (0: use the generic kernel)
  int wca = 0;                  // d = 2 affine path column window (0: not used)
  int nsm = 148;
  double* ring = nullptr;       // (RS + 1) * F * cfield ; slot RS = scratch
  int RS = 3;                   // ring slots: K + 2 (level m in slot m % RS; the 2 spare slots let the
                                // fused kernel's CTAs run up to 2 steps apart without write-after-read hazards)
  double* tmp0 = nullptr;       // cfield
  double* tmp1 = nullptr;       // cfield
  double* a3 = nullptr;         // d = 3 fused path: L x F plane stacks of one level (axis0_pass)
  double* acc3 = nullptr;       // d = 3 fused path: 5 partial sums per owned point
  int32_t* picard = nullptr;    // npts
  unsigned long long* bad = nullptr;
  unsigned* barrier = nullptr;  // grid-barrier counter of the persistent fused kernel
  double* dres = nullptr;       // 8 doubles
  int tap_off = -1, tap1_off = -1, tap_count = 0;        // byte offsets in the constant arena
  int boot_tap_off = -1, boot_tap1_off = -1;
  int qspan = 0, qspan1 = 0, boot_qspan = 0, boot_qspan1 = 0;
  struct Geo {
    bool ok = false;
    bool single = false;          // the one-tile-per-CTA launch is co-resident
    Fused1D fz{};
    int threads = 0, blocks = 0;
    int D[kMaxK + 1] = {};        // D[j]: CTA distance of level j's window; D[0]: values halo
    int DK = 1;                   // max over levels
    size_t smem = 0;
  } geo, boot_geo;
  double gy[7]{}, gz[7]{};
  double gh_a[kMaxL]{}, gh_w[kMaxL]{};
  std::vector<AxisTap> taps;    // host copy of the main table (K * d * L)
  int64_t launches = 0;
  unsigned long long* phase_ns = nullptr;   // debug: BSDE_PHASE_TIMING=1
  // slab partition (d >= 2): global rows [r0, r1) owned, halo rows exchanged per step
  int nranks = 1, rank = 0;
  int64_t P0g = 0, r0 = 0, r1 = 0, lo_e = 0, hi_e = 0, halo = 0;
  ncclComm_t comm = nullptr;        // multi-process mode (nccl_unique_id given)
  bool grouped = false;             // in-process group mode (bsde_group_*)
  // SPIKE slab spline (cfg.slab_spline = 0, nranks > 1): per ring slot the edge
  // moments [F][2][plane] of the local axis-0 solve; the all-gathered edges [R][F][2][plane]; the
  // interface moments X [F][2][plane] and their tensor splines XC [F][2][plane_c]; the spike
  // vectors S^L, S^R of the own unknown rows [row_lo, row_lo + spk_n) (local)
  bool spike = false;
  double *edge = nullptr, *gath = nullptr, *xs = nullptr, *xc = nullptr, *xtmp = nullptr, *slr = nullptr;
  int64_t plane_v = 0, plane_c = 0, spk_n = 0, spk_row_lo = 0;
  SpikeArgs spk{};
  Grid gplane{};                    // the axes 1 .. d-1 grid of the interface planes
  std::vector<double> h_slr;
  unsigned pending = 0;             // in-process group: ring slots whose interface correction is due
  bool prebuilt = false;            // in-process group: the newest level's spline is built (group step)
  bool rs_ready = false;            // in-process group: the scratch slot holds the corrected newest level
  std::string err;
  bool closed_form = true;
  // timing: host-clock setup time; CUDA-event stage timers (bootstrap always, the others with
  // cfg.timing = 1), accumulated until the next bsde_solve collects them
  double t_setup = 0;
  bool in_setup = false;              // bootstrap steps inside bsde_setup count as t_bootstrap_s only
  struct Stage { int kind; cudaEvent_t a, b; };
  std::vector<Stage> stages;
  std::vector<cudaEvent_t> ev_free;
  double t_stage[4] = {0, 0, 0, 0};   // 0 spline, 1 quadrature, 2 comm, 3 bootstrap
};

enum { ST_SPLINE = 0, ST_QUAD = 1, ST_COMM = 2, ST_BOOT = 3 };

static bsde_status set_err(bsde_ctx* c, bsde_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  else g_setup_error = buf;
  return st;
}

#define CU(call)                                                                              \
  do {                                                                                        \
    cudaError_t _e = (call);                                                                  \
    if (_e != cudaSuccess) return set_err(c, BSDE_ERR_CUDA, "%s: %s (%s:%d)", #call,         \
                                          cudaGetErrorString(_e), __FILE__, __LINE__);        \
  } while (0)

// ------------------------------------------------------------------ stage timers
static cudaEvent_t tmark(bsde_ctx* c) {
  cudaEvent_t e = nullptr;
  if (!c->ev_free.empty()) { e = c->ev_free.back(); c->ev_free.pop_back(); }
  else if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
  cudaEventRecord(e, c->stream);
  return e;
}
static void tstage(bsde_ctx* c, int kind, cudaEvent_t a) {
  if (!a) return;
  cudaEvent_t b = tmark(c);
  if (b) c->stages.push_back({kind, a, b});
}
// after the stream has been synchronised: accumulate and recycle the events
static void tcollect(bsde_ctx* c) {
  for (auto& st : c->stages) {
    float ms = 0;
    if (cudaEventElapsedTime(&ms, st.a, st.b) == cudaSuccess) c->t_stage[st.kind] += ms * 1e-3;
    c->ev_free.push_back(st.a);
    c->ev_free.push_back(st.b);
  }
  c->stages.clear();
}
static void tfree(bsde_ctx* c) {
  for (auto& st : c->stages) { c->ev_free.push_back(st.a); c->ev_free.push_back(st.b); }
  c->stages.clear();
  for (cudaEvent_t e : c->ev_free) cudaEventDestroy(e);
  c->ev_free.clear();
}

// ------------------------------------------------------------------ constant-arena allocator
namespace {
struct Arena {
  std::mutex mu;
  std::vector<std::pair<int, int>> used;   // (offset, count)
};
Arena g_arena[64];

int arena_alloc(int dev, int count) {        // count in bytes, 16-byte granularity
  count = (count + 15) & ~15;
  if (dev < 0 || dev >= 64) return -1;
  Arena& a = g_arena[dev];
  std::lock_guard<std::mutex> lk(a.mu);
  std::sort(a.used.begin(), a.used.end());
  int pos = 0;
  for (auto& u : a.used) {
    if (u.first - pos >= count) break;
    pos = (u.first + u.second + 15) & ~15;
  }
  if (pos + count > arena_capacity_bytes()) return -1;
  a.used.push_back({pos, count});
  return pos;
}
void arena_free(int dev, int off) {
  if (dev < 0 || dev >= 64 || off < 0) return;
  Arena& a = g_arena[dev];
  std::lock_guard<std::mutex> lk(a.mu);
  for (size_t i = 0; i < a.used.size(); ++i)
    if (a.used[i].first == off) { a.used.erase(a.used.begin() + i); return; }
}

// ------------------------------------------------------------------ numerics of the setup
// Weight rows as printed: Table 1 (y, gamma^{Ky}_{Ky,j}) and Table 2 (z, gamma^1_{Kz,j}),
// PAPER.md:235-269; Eq. 20's b is read as gamma (R1).
const long double kTab1[6][7] = {
    {1.0L / 2, 1.0L / 2},
    {1.0L / 6, 2.0L / 3, 1.0L / 6},
    {1.0L / 8, 3.0L / 8, 3.0L / 8, 1.0L / 8},
    {1.0L / 12, 1.0L / 3, 1.0L / 6, 1.0L / 3, 1.0L / 12},
    {41.0L / 600, 19.0L / 75, 107.0L / 600, 107.0L / 600, 19.0L / 75, 41.0L / 600},
    {19.0L / 336, 3.0L / 14, 15.0L / 112, 4.0L / 21, 15.0L / 112, 3.0L / 14, 19.0L / 336}};
const long double kTab2[6][7] = {
    {1.0L / 2, 1.0L / 2},
    {5.0L / 12, 2.0L / 3, -1.0L / 12},
    {3.0L / 8, 19.0L / 24, -5.0L / 24, 1.0L / 24},
    {35.0L / 96, 5.0L / 6, -13.0L / 48, 1.0L / 12, -1.0L / 96},
    {131.0L / 360, 151.0L / 180, -103.0L / 360, 37.0L / 360, -1.0L / 45, 1.0L / 360},
    {163.0L / 448, 47.0L / 56, -129.0L / 448, 3.0L / 28, -37.0L / 1344, 1.0L / 168, -1.0L / 1344}};

// Gauss-Hermite rule (Eq. 21): nodes are the eigenvalues of the Jacobi matrix of the
// Hermite weight e^{-x^2} (diagonal 0, off-diagonal sqrt(k/2)), found by Sturm-sequence
// bisection in long double; weights by the Christoffel function 1 / sum_k p_k(a)^2 of
// the orthonormal Hermite polynomials.
int sturm_count(int L, long double x) {   // eigenvalues < x
  int cnt = 0;
  long double q = -x;                     // d_1 - x, d = 0
  if (q < 0) ++cnt;
  for (int k = 1; k < L; ++k) {
    const long double b2 = (long double)k / 2.0L;
    if (q == 0) q = 1e-4000L;
    q = -x - b2 / q;
    if (q < 0) ++cnt;
  }
  return cnt;
}

void hermite_rule_compute(int L, double* a, double* w);
// the rule of each L is computed once per process (the long-double bisection costs ~0.7 ms at
// L = 32: a large share of a small problem's time to solution)
void hermite_rule(int L, double* a, double* w) {
  static std::mutex mu;
  static std::vector<double> cache[kMaxL + 1];
  std::lock_guard<std::mutex> lk(mu);
  std::vector<double>& c = cache[L];
  if (c.empty()) {
    c.resize(2 * (size_t)L);
    hermite_rule_compute(L, c.data(), c.data() + L);
  }
  std::copy(c.begin(), c.begin() + L, a);
  std::copy(c.begin() + L, c.end(), w);
}
void hermite_rule_compute(int L, double* a, double* w) {
  const long double bound = sqrtl(2.0L * L) + 2.0L;
  for (int i = 0; i < L; ++i) {           // i-th smallest eigenvalue
    long double lo = -bound, hi = bound;
    for (int it = 0; it < 200; ++it) {
      const long double mid = 0.5L * (lo + hi);
      if (mid == lo || mid == hi) break;
      if (sturm_count(L, mid) > i) hi = mid; else lo = mid;
    }
    long double x = 0.5L * (lo + hi);
    if (L % 2 == 1 && i == L / 2) x = 0.0L;
    // Christoffel weight
    const long double pim4 = 0.75112554446494248285870300477622L;   // pi^{-1/4}
    long double pm = 0.0L, p = pim4, sum = p * p;
    for (int k = 1; k < L; ++k) {
      const long double pn = (sqrtl(2.0L) * x * p - sqrtl((long double)(k - 1)) * pm) / sqrtl((long double)k);
      pm = p; p = pn;
      sum += p * p;
    }
    a[i] = (double)x;
    w[i] = (double)(1.0L / sum);
  }
  // exact symmetry
  for (int i = 0; i < L / 2; ++i) {
    const double m = 0.5 * (a[L - 1 - i] - a[i]);
    a[i] = -m; a[L - 1 - i] = m;
    const double ww = 0.5 * (w[i] + w[L - 1 - i]);
    w[i] = ww; w[L - 1 - i] = ww;
  }
}

// Gauss-Legendre rule on [-1, 1] for the d >= 2 smoothing (R11): Newton on
// P_n from Tricomi's initial guesses, long double.
void legendre_rule(int n, double* x, double* w) {
  for (int i = 0; i < n; ++i) {
    long double z = -cosl(3.14159265358979323846264338327950288L * (4.0L * (i + 1) - 1.0L) / (4.0L * n + 2.0L));
    long double dp = 1.0L;
    for (int it = 0; it < 60; ++it) {
      long double p0 = 1.0L, p1 = z;
      for (int k = 2; k <= n; ++k) {
        const long double p2 = ((2.0L * k - 1.0L) * z * p1 - (k - 1.0L) * p0) / k;
        p0 = p1; p1 = p2;
      }
      dp = n * (z * p1 - p0) / (z * z - 1.0L);
      const long double dz = p1 / dp;
      z -= dz;
      if (fabsl(dz) < 1e-20L) break;
    }
    x[i] = (double)z;
    w[i] = (double)(2.0L / ((1.0L - z * z) * dp * dp));
  }
}

// balance rule with reading R3: q = min(Ky+1, Kz, 3), M = 2 ceil(X/dx)
int64_t balanced_points(double width, double dt, int Ky, int Kz, int r) {
  const int q = std::min(std::min(Ky + 1, Kz), 3);
  const long double dxs = powl((long double)dt, (long double)(q + 1) / (long double)r);
  const long double cnt = 0.5L * (long double)width / dxs;
  const int64_t half = (int64_t)ceill(cnt * (1.0L - 1e-12L));
  return 2 * half + 1;
}

// B-spline basis of a shift theta in [0, 1)
void bspline_basis(long double t, double* B) {
  const long double u = 1.0L - t;
  B[0] = (double)(u * u * u / 6.0L);
  B[1] = (double)((3.0L * t * t * t - 6.0L * t * t + 4.0L) / 6.0L);
  B[2] = (double)((-3.0L * t * t * t + 3.0L * t * t + 3.0L * t + 1.0L) / 6.0L);
  B[3] = (double)(t * t * t / 6.0L);
}

// cubic Hermite basis at theta (FD-bicubic interpolation, bicubic.cuh): H00, H10, H01, H11
void hermite_basis(long double t, double* H) {
  const long double t2 = t * t, t3 = t2 * t;
  H[0] = (double)(2.0L * t3 - 3.0L * t2 + 1.0L);
  H[1] = (double)(t3 - 2.0L * t2 + t);
  H[2] = (double)(-2.0L * t3 + 3.0L * t2);
  H[3] = (double)(t3 - t2);
}

// tap table of levels 1..K for step dt: X = x_i + s, s = sqrt(2 j dt) a_l
void build_taps(const bsde_ctx* c, int K, double dt, std::vector<AxisTap>& out, int* qspan, int* qspan1) {
  const int d = c->d, L = c->L;
  out.assign((size_t)K * d * L, AxisTap{});
  const long double rpi = 1.0L / sqrtl(3.14159265358979323846264338327950288L);
  int span = 0;
  for (int j = 1; j <= K; ++j)
    for (int a = 0; a < d; ++a) {
      for (int l = 0; l < L; ++l) {
        AxisTap& t = out[((size_t)(j - 1) * d + a) * L + l];
        const long double s = sqrtl(2.0L * j * (long double)dt) * (long double)c->gh_a[l];
        const long double u = s / (long double)c->g.dx[a];
        const long double q = floorl(u);
        t.q = (int32_t)q;
        if (c->cfg.interp == BSDE_INTERP_FD_BICUBIC) hermite_basis(u - q, t.B);
        else bspline_basis(u - q, t.B);
        t.w = (double)((long double)c->gh_w[l] * rpi);
        t.s = (double)s;
      }
      span = std::max(span, out[((size_t)(j - 1) * d + a) * L + L - 1].q - out[((size_t)(j - 1) * d + a) * L].q);
    }
  if (qspan) *qspan = span;
  if (qspan1) *qspan1 = out[(size_t)(L - 1)].q - out[0].q;    // level 1, axis 0
}

// fused 1-D records: stencil of level j / node l with the scheme weights folded in
std::vector<Tap1D> build_tap1d(const std::vector<AxisTap>& t, int K, int L, int Ky, int Kz, const double* gy,
                               const double* gz) {
  std::vector<Tap1D> out((size_t)K * L);
  for (int j = 1; j <= K; ++j) {
    const long double gzj = j <= Kz ? gz[j] : 0.0L, gyj = j <= Ky ? gy[j] : 0.0L;
    const long double czj = (j == 1 ? 1.0L : 0.0L) - gzj;
    for (int l = 0; l < L; ++l) {
      const AxisTap& a = t[(size_t)(j - 1) * L + l];
      Tap1D& r = out[(size_t)(j - 1) * L + l];
      r.q = a.q;
      r.pad = 0;
      for (int k = 0; k < 4; ++k) r.B[k] = a.B[k];
      const long double w = a.w;
      r.wcz = (double)(w * czj);
      r.wgz = (double)(w * gzj * (long double)a.s);
      r.wgy = (double)(w * gyj);
      r.wy = j == Ky ? a.w : 0.0;
    }
  }
  return out;
}

// CTA distances of the fused kernel's neighbour waits; the fused path needs all CTAs
// co-resident (one per SM) and <= 8192 CTAs of flags
void set_distances(bsde_ctx* c, const std::vector<AxisTap>& t, int K, bsde_ctx::Geo& geo) {
  if (!geo.ok) return;
  const int L = c->L, TP = geo.fz.TP;
  auto reach = [&](int j) {
    const int qa = -t[(size_t)(j - 1) * L].q, qb = t[(size_t)(j - 1) * L + L - 1].q;
    return std::max(qa, qb) + 4;
  };
  geo.D[0] = (kP2Halo + 6 + TP - 1) / TP;     // values halo of the pass-2 own-tile spline
  int dk = geo.D[0];
  for (int j = 1; j <= K; ++j) {
    geo.D[j] = (reach(j) + TP - 1) / TP;
    dk = std::max(dk, geo.D[j]);
  }
  geo.DK = dk;
  const int per_sm = fused1d_blocks_per_sm(geo.fz.variant, geo.smem);
  if (geo.blocks > 8192) geo.ok = false;
  // one tile per CTA (bsde_step, bsde_solve) needs every CTA co-resident; a batch partitions the
  // tiles over fewer CTAs (bsde_solve_batch checks its own co-residency)
  geo.single = geo.blocks <= c->nsm * per_sm;
}

// balanced rows of rank r out of R
inline void rank_rows(int64_t P0, int R, int r, int64_t& r0, int64_t& r1) {
  r0 = (int64_t)r * P0 / R;
  r1 = (int64_t)(r + 1) * P0 / R;
}

// slab partition of axis 0 (host only): owned rows, halo = axis-0 quadrature reach + cubic
// support + PCR decay rows, extended slab [lo_e, hi_e)
bsde_status plan_partition(bsde_ctx* c) {
  if (c->nranks <= 1) {
    c->r0 = 0; c->r1 = c->P0g; c->lo_e = 0; c->hi_e = c->P0g; c->halo = 0;
    return BSDE_OK;
  }
  int reach = 0;
  for (int j = 1; j <= c->K; ++j)
    for (int l = 0; l < c->L; ++l) {
      const int q = c->taps[((size_t)(j - 1) * c->d + 0) * c->L + l].q;
      reach = std::max(reach, q < 0 ? -q : q);
    }
  // SPIKE: the final coefficients are exchanged, reach + 3 rows (the 4-row stencil of the farthest
  // tap); the redundant-halo ablation re-solves the axis-0 spline over the halo: + PCR decay
  c->halo = c->cfg.slab_spline == 0 ? reach + 3 : reach + 3 + kPcrHalo + 6;
  for (int r = 0; r < c->nranks; ++r) {
    int64_t a, b;
    rank_rows(c->P0g, c->nranks, r, a, b);
    if (b - a < c->halo)
      return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "slab of rank %d has %lld rows < halo %lld: use fewer ranks", r,
                     (long long)(b - a), (long long)c->halo);
  }
  rank_rows(c->P0g, c->nranks, c->rank, c->r0, c->r1);
  c->lo_e = std::max<int64_t>(0, c->r0 - c->halo);
  c->hi_e = std::min<int64_t>(c->P0g, c->r1 + c->halo);
  return BSDE_OK;
}

bool closed_form_supported(const bsde_config& cfg) {
  const int t = cfg.terminal_id, f = cfg.driver_id, d = cfg.d;
  const double* q = cfg.driver_params;
  if (cfg.sde_id != BSDE_SDE_BROWNIAN)        // forward SDE: only the constant solution is known
    return t == BSDE_TERM_CONST && f == BSDE_DRV_ZERO;
  if (t == BSDE_TERM_CONST) return f == BSDE_DRV_ZERO || (f == BSDE_DRV_AFFINE && q[1] == 0 && q[2] == 0 && q[3] == 0);
  if (t == BSDE_TERM_POLY)
    return f == BSDE_DRV_ZERO || (f == BSDE_DRV_AFFINE && q[1] == 0 && q[2] == 0 && q[3] == 0 && q[4] == 0);
  if (t == BSDE_TERM_LOGISTIC) return f == BSDE_DRV_EX1;
  if (t == BSDE_TERM_EX2) return f == BSDE_DRV_EX2 && d == 1;
  if (t == BSDE_TERM_CALL_W) return (f == BSDE_DRV_AFFINE || f == BSDE_DRV_DIFF_RATES) && d == 1;
  if (t == BSDE_TERM_SIN_SUM) return f == BSDE_DRV_AFFINE;
  if (t == BSDE_TERM_EXCHANGE_W) return f == BSDE_DRV_AFFINE && d == 2;
  if (t == BSDE_TERM_GEO_BASKET_W) return f == BSDE_DRV_DIFF_RATES;
  return false;
}

bsde_status validate(const bsde_config* cfg, bsde_ctx* c) {
  if (!cfg) return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "cfg is NULL");
  if (cfg->struct_size != sizeof(bsde_config))
    return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "struct_size %u != sizeof(bsde_config) %zu", cfg->struct_size,
                   sizeof(bsde_config));
  if (cfg->d < 1 || cfg->d > 3) return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "d=%d outside 1..3", cfg->d);
  if (cfg->m != 1) return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "m=%d: only m=1 is supported", cfg->m);
  if (cfg->Ky < 1 || cfg->Ky > 6 || cfg->Kz < 1 || cfg->Kz > 6)
    return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "Ky=%d Kz=%d outside 1..6 (Tables 1-2)", cfg->Ky, cfg->Kz);
  if (cfg->L < 1 || cfg->L > kMaxL) return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "L=%d outside 1..64", cfg->L);
  if (!(cfg->T > cfg->t0)) return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "T <= t0");
  const int K = std::max(cfg->Ky, cfg->Kz);
  if (cfg->N < K) return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "N=%d < K=%d", cfg->N, K);
  if (cfg->picard_max < 1) return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "picard_max < 1");
  if (cfg->driver_id < 0 || cfg->driver_id > 4) return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "driver_id");
  if (cfg->terminal_id < 0 || cfg->terminal_id > 8) return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "terminal_id");
  if (cfg->sde_id < 0 || cfg->sde_id > 2) return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "sde_id %d outside 0..2", cfg->sde_id);
  if (cfg->terminal_id == BSDE_TERM_CALL_X && cfg->sde_id == BSDE_SDE_BROWNIAN)
    return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "terminal CALL_X is a payoff of a forward SDE: set sde_id");
  if (cfg->sde_id != BSDE_SDE_BROWNIAN && cfg->driver_id == BSDE_DRV_EX2)
    return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "the Ex. 2 driver is defined for X = W only");
  if (cfg->sde_id != BSDE_SDE_BROWNIAN && cfg->nranks > 1)
    return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "forward-SDE problems run on one rank");
  if (cfg->sde_id != BSDE_SDE_BROWNIAN && cfg->smoothing)
    return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "terminal smoothing is defined for X = W payoffs only (R11)");
  if (cfg->interp < 0 || cfg->interp > 1) return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "interp %d outside 0..1", cfg->interp);
  if (cfg->slab_spline < 0 || cfg->slab_spline > 1)
    return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "slab_spline %d outside 0..1", cfg->slab_spline);
  if (cfg->nranks > kMaxRanks) return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "nranks %d > %d", cfg->nranks, kMaxRanks);
  if (cfg->interp == BSDE_INTERP_FD_BICUBIC && (cfg->d != 2 || cfg->sde_id != BSDE_SDE_BROWNIAN || cfg->nranks > 1))
    return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "FD-bicubic interpolation is the paper's 2-D scheme: d = 2, X = W, one rank");
  if (cfg->driver_id == BSDE_DRV_EX2 && cfg->d != 1) return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "EX2 driver is 1-D");
  if (cfg->terminal_id == BSDE_TERM_EXCHANGE_W && cfg->d != 2)
    return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "exchange payoff needs d=2");
  if (cfg->nranks > 1 && cfg->d < 2)
    return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "nranks > 1 needs d >= 2 (1-D runs as replicas, DESIGN.md)");
  if (cfg->nranks > 1 && (cfg->rank < 0 || cfg->rank >= cfg->nranks))
    return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "rank %d outside 0..%d", cfg->rank, cfg->nranks - 1);
  // an in-process group refreshes halos only in bsde_group_step: the one-step bootstrap inside
  // bsde_setup would build slab splines from stale halo rows
  if (cfg->nranks > 1 && cfg->nccl_unique_id == nullptr && cfg->bootstrap == 1 && std::max(cfg->Ky, cfg->Kz) > 1)
    return set_err(c, BSDE_ERR_INVALID_ARGUMENT,
                   "in-process slab groups need closed-form initial layers (bootstrap = 0) or K = 1; "
                   "the NCCL multi-process mode supports the bootstrap");
  for (int a = 0; a < cfg->d; ++a) {
    if (!(cfg->xhi[a] > cfg->xlo[a])) return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "empty box on axis %d", a);
    if (cfg->npts[a] != 0 && cfg->npts[a] < 4)
      return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "npts[%d]=%lld < 4 (not-a-knot needs 4 points)", a,
                     (long long)cfg->npts[a]);
    if (cfg->interp == BSDE_INTERP_FD_BICUBIC && cfg->npts[a] != 0 && cfg->npts[a] < 6)
      return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "npts[%d]=%lld < 6 (4th-order one-sided differences need 5 nodes "
                     "on a side of every node)", a, (long long)cfg->npts[a]);
  }
  if (cfg->bootstrap == 0 && K > 1 && !closed_form_supported(*cfg))
    return set_err(c, BSDE_ERR_INVALID_ARGUMENT,
                   "no closed form for terminal %d with driver %d: use bootstrap=1", cfg->terminal_id, cfg->driver_id);
  return BSDE_OK;
}

void fill_grid(const bsde_config* cfg, Grid& g, double dt) {
  g.d = cfg->d;
  g.npts = 1;
  for (int a = 0; a < 3; ++a) { g.P[a] = 1; g.xlo[a] = 0; g.xhi[a] = 0; g.dx[a] = 0; }
  for (int a = 0; a < cfg->d; ++a) {
    int64_t P = cfg->npts[a];
    if (P == 0) P = balanced_points(cfg->xhi[a] - cfg->xlo[a], dt, cfg->Ky, cfg->Kz, cfg->r > 0 ? cfg->r : 4);
    g.P[a] = P;
    g.xlo[a] = cfg->xlo[a];
    g.xhi[a] = cfg->xhi[a];
    g.dx[a] = (cfg->xhi[a] - cfg->xlo[a]) / (double)(P - 1);
    g.npts *= P;
  }
  const int d = cfg->d;
  g.vstride[d - 1] = 1;
  for (int a = d - 2; a >= 0; --a) g.vstride[a] = g.vstride[a + 1] * g.P[a + 1];
  // coefficient layout: extent P+3 per axis (c_{-1} .. c_{P+1}); last axis padded to 4
  const int64_t lastQ = ((g.P[d - 1] + 3 + 3) / 4) * 4;
  g.cstride[d - 1] = 1;
  int64_t ext = lastQ;
  for (int a = d - 2; a >= 0; --a) { g.cstride[a] = ext; ext *= g.P[a] + 3; }
  g.cfield = ext;
  g.cpad = 0;
  if (d == 1) {
    // the largest quadrature reach in cells (largest Hermite zero < sqrt(2L+1)) + slack
    const int K = std::max(cfg->Ky, cfg->Kz);
    const double reach = std::sqrt(2.0 * K * dt) * std::sqrt(2.0 * cfg->L + 1.0) / g.dx[0];
    g.cpad = ((int64_t)std::ceil(reach) + 8 + 1) & ~(int64_t)1;
    g.cfield += 2 * g.cpad;
  }
  for (int a = d; a < 3; ++a) { g.vstride[a] = 0; g.cstride[a] = 0; }
  if (cfg->interp == BSDE_INTERP_FD_BICUBIC) g.cfield = 4 * g.npts;   // f, h0 f_x, h1 f_y, h0 h1 f_xy
  g.off0 = 0;
  g.Pg0 = g.P[0];
  g.own0 = 0;
  g.nown0 = g.P[0];
}

// restrict a global grid to the local extended slab [lo_e, hi_e) of axis 0, owned [r0, r1)
void localize_grid(Grid& g, int64_t lo_e, int64_t hi_e, int64_t r0, int64_t r1) {
  const int d = g.d;
  const int64_t Pg0 = g.P[0];
  g.P[0] = hi_e - lo_e;
  g.npts = 1;
  for (int a = 0; a < d; ++a) g.npts *= g.P[a];
  g.vstride[d - 1] = 1;
  for (int a = d - 2; a >= 0; --a) g.vstride[a] = g.vstride[a + 1] * g.P[a + 1];
  const int64_t lastQ = ((g.P[d - 1] + 3 + 3) / 4) * 4;
  g.cstride[d - 1] = 1;
  int64_t ext = lastQ;
  for (int a = d - 2; a >= 0; --a) { g.cstride[a] = ext; ext *= g.P[a] + 3; }
  g.cfield = ext;
  g.off0 = lo_e;
  g.Pg0 = Pg0;
  g.own0 = r0 - lo_e;
  g.nown0 = r1 - r0;
}



// the d = 2 affine-driver path (aff2.cuh) is the default for f = 0 and
// affine f; kernel_variant 2 keeps the per-tap fused kernel
bool use_aff2(const bsde_config* cfg) {
  return cfg->d == 2 && cfg->kernel_variant == 0 && (cfg->driver_id == 0 || cfg->driver_id == 1) &&
         cfg->interp == BSDE_INTERP_SPLINE && cfg->sde_id == BSDE_SDE_BROWNIAN;
}
// the d = 3 fused path (plane stacks) serves X = W problems
bool use_fused3d(const bsde_config* cfg) {
  return (cfg->kernel_variant == 0 || cfg->kernel_variant == 2) && cfg->sde_id == BSDE_SDE_BROWNIAN;
}

struct Layout {
  size_t values, ring, tmp0, tmp1, a3, acc3, picard, bad, barrier, dres, spike, total;
};
// values: 2 ping-pong buffers of F * npts (the fused 1-D step reads level n+1 while
// other CTAs write level n)

// fused3d: the d = 3 fused path's per-level plane stacks (L x F x local planes) and the
// 5 partial sums per owned point; aff2: the d = 2 affine path's axis-0 operators of every
// level (K x 2 x F x owned rows, in the a3 region)
Layout layout(const Grid& g, int F, int K, int nodes, bool fused3d, bool aff2, int R = 1, bool spike = false) {
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  Layout L{};
  size_t off = 0;
  L.values = off; off += 2 * al(sizeof(double) * F * g.npts);
  L.ring = off; off += al(sizeof(double) * (size_t)(K + 3) * F * g.cfield);
  L.tmp0 = off; off += g.d >= 2 ? al(sizeof(double) * g.cfield) : 0;
  L.tmp1 = off; off += g.d >= 3 ? al(sizeof(double) * g.cfield) : 0;
  const bool f3 = g.d == 3 && fused3d, a2 = g.d == 2 && aff2;
  L.a3 = off;
  // d = 3: L x F plane stacks, or (decomposed differential-rates driver) L single-field stacks
  // + the 6 K + 7 arrays of its separable affine part
  off += f3 ? al(sizeof(double) * (size_t)std::max(nodes * F, nodes + 6 * K + 7) * g.P[0] * g.cstride[0])
            : (a2 ? al(sizeof(double) * 2 * (size_t)F * K * g.nown0 * g.cstride[0]) : 0);
  L.acc3 = off;
  off += f3 ? al(sizeof(double) * 5 * (size_t)g.nown0 * g.P[1] * g.P[2])
            : 0;
  L.picard = off; off += al(sizeof(int32_t) * g.npts);
  L.bad = off; off += 256;
  L.barrier = off; off += al(sizeof(unsigned) * 2 * kFlagCap);  // fused-kernel progress flags (ring, done)
  L.dres = off; off += 256;
  L.spike = off;
  if (spike && g.d >= 2) {            // edges per slot, gathered edges, X, XC, scratch, spike vectors
    const size_t pv = (size_t)(g.npts / g.P[0]), pc = (size_t)g.cstride[0];
    off += al(sizeof(double) * (size_t)(K + 3) * F * 2 * pv) + al(sizeof(double) * (size_t)R * F * 2 * pv) +
           al(sizeof(double) * F * 2 * pv) + al(sizeof(double) * F * 2 * pc) + al(sizeof(double) * pc) +
           al(sizeof(double) * 2 * (size_t)(g.P[0] + 4));
  }
  L.total = off;
  return L;
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

bsde_status exchange_nccl(bsde_ctx* c);
bsde_status finish_level(bsde_ctx* c, int slot);

// SPIKE edge moments of ring slot `slot`
static double* edge_slot(const bsde_ctx* c, int slot) { return c->edge + (int64_t)slot * c->F * 2 * c->plane_v; }

// interpolant of the newest values into ring slot `slot`: tensor not-a-knot spline (B-spline
// coefficients), or the Hermite data of the FD-bicubic surfaces (interp = 1)
cudaError_t build_level(bsde_ctx* c, int slot) {
  double* dst = c->ring + (int64_t)slot * c->F * c->g.cfield;
  if (c->cfg.interp == BSDE_INTERP_FD_BICUBIC)
    return launch_hermite(c->g, c->vbuf[c->cur], c->F, dst, c->stream, &c->launches);
  if (c->spike)          // the local part of the SPIKE solve; finish_level applies the correction
    return launch_spline_slab(c->g, c->vbuf[c->cur], c->F, dst, c->tmp0, c->tmp1, c->rank == 0,
                              c->rank == c->nranks - 1, edge_slot(c, slot), c->stream, &c->launches);
  return launch_spline(c->g, c->vbuf[c->cur], c->F, dst, c->tmp0, c->tmp1, c->stream, &c->launches);
}

// One step of the scheme (Eq. 20) from the newest values (level n+1) and the ring slots of
// levels n+2..n+K: slots[0] receives the spline of the newest values.  Output -> the other
// value buffer, which becomes the newest.
bsde_status run_step(bsde_ctx* c, int Kl, int Kyl, int Kzl, const double* gyl, const double* gzl, double dtl,
                     double tn, const int* slots, int slot_out, int tap_off, int tap1_off, const bsde_ctx::Geo& geo,
                     int variant, int wc2 = 0) {
  StepArgs s{};
  s.slot_out = slot_out;
  s.ring = c->ring;
  s.slot_elems = (int64_t)c->F * c->g.cfield;
  s.cfield = c->g.cfield;
  s.cpad = c->g.cpad;
  for (int j = 1; j <= Kl; ++j) {
    s.slot[j - 1] = slots[j - 1];
    s.t_level[j - 1] = tn + j * dtl;
    const double gzj = j <= Kzl ? gzl[j] : 0.0;
    s.gzj[j - 1] = gzj;
    s.czj[j - 1] = (j == 1 ? 1.0 : 0.0) - gzj;
    s.gyj[j - 1] = j <= Kyl ? gyl[j] : 0.0;
  }
  s.K = Kl; s.Ky = Kyl; s.Kz = Kzl; s.L = c->L;
  s.ring_slots = c->RS;
  s.tap_off = tap_off;
  s.tap1_off = tap1_off;
  s.gz0 = gzl[0];
  s.ky_dt = Kyl * dtl;
  s.ky_dt_gy0 = Kyl * dtl * gyl[0];
  s.tn = tn;
  s.dt = dtl;
  s.picard_max = c->cfg.picard_max;
  s.picard_tol = c->cfg.picard_tol;
  s.values_in = c->vbuf[c->cur];
  s.values = c->vbuf[c->cur ^ 1];
  s.picard = c->picard;
  s.bad = c->bad;
  s.phase_ns = c->phase_ns;
  s.n = (int)std::floor((tn - c->cfg.t0) / c->dt + 0.5);      // level index (bootstrap: nearest level)
  const bool timing = c->cfg.timing != 0 && !c->in_setup;
  cudaError_t e;
  if (c->d == 1 && (variant == 0 || variant >= 10) && geo.ok && geo.single && tap1_off >= 0 && c->pb.sde_id == 0) {
    cudaEvent_t t0 = timing ? tmark(c) : nullptr;            // spline fused into the kernel
    e = launch_fused1d_steps(s, c->g, c->pb, geo.fz, 0, 1, 0, c->cur, 0.0, 0.0, c->vbuf[0], c->vbuf[1], c->barrier,
                             geo.D, geo.DK, geo.threads, geo.blocks, geo.smem, c->stream);
    ++c->launches;
    if (timing) tstage(c, ST_QUAD, t0);
  } else {
    cudaEvent_t t0 = timing ? tmark(c) : nullptr;
    e = c->prebuilt ? cudaSuccess : build_level(c, slots[0]);
    if (timing) tstage(c, ST_SPLINE, t0);
    if (e == cudaSuccess && !c->prebuilt) {
      const bsde_status fs = finish_level(c, slots[0]);        // SPIKE interface correction (NCCL)
      if (fs) return fs;
    }
    cudaEvent_t t1 = timing ? tmark(c) : nullptr;
    if (e == cudaSuccess) {
      if (c->pb.sde_id != 0)                                   // forward SDE: per-point Euler samples
        e = launch_fsde_step(s, c->g, c->pb, c->stream);
      else if (c->cfg.interp == BSDE_INTERP_FD_BICUBIC)        // the paper's 2-D interpolation
        e = launch_bicubic_step(s, c->g, c->pb, c->stream);
      else if (c->d == 2 && variant == 0 && c->a3 && c->wca > 0 && (c->pb.driver_id == 0 || c->pb.driver_id == 1))
        e = launch_aff2(s, c->g, c->pb, c->a3, c->wca, c->stream, &c->launches);
      else if (c->d == 2 && (variant == 0 || variant == 2) && wc2 > 0 && c->pb.driver_id != 3)
        e = launch_quad2d(s, c->g, c->pb, wc2, c->stream);
      else if (c->d == 3 && (variant == 0 || variant == 2) && wc2 > 0 && c->pb.driver_id != 3 && c->a3 && c->acc3)
        e = launch_step3d(s, c->g, c->pb, wc2, c->a3, c->acc3, variant == 0 && c->pb.driver_id == 4, c->stream,
                          &c->launches);
      else
        e = launch_generic_step(s, c->g, c->pb, c->stream);
      ++c->launches;
    }
    if (timing) tstage(c, ST_QUAD, t1);
  }
  if (e != cudaSuccess) return set_err(c, BSDE_ERR_CUDA, "step kernels: %s", cudaGetErrorString(e));
  c->cur ^= 1;
  return exchange_nccl(c);      // no-op for one rank and for in-process groups (bsde_group_step)
}

// halo rows of the newest values between slab neighbours (d >= 2, nranks > 1)
struct HaloPlan {
  int64_t send_lo_off, send_lo_rows;   // to rank-1: local row offset / rows
  int64_t recv_lo_off, recv_lo_rows;   // from rank-1
  int64_t send_hi_off, send_hi_rows;   // to rank+1
  int64_t recv_hi_off, recv_hi_rows;   // from rank+1
};
// rows of a halo of h rows (clipped to the grid); SPIKE exchanges 1 row of values (the
// second difference of the interface rows) and h = halo rows of final coefficients
HaloPlan halo_plan(const bsde_ctx* c, int64_t h) {
  HaloPlan p{};
  if (c->rank > 0) {
    p.recv_lo_rows = std::min<int64_t>(h, c->r0);                // my rows [r0 - rows, r0)
    p.recv_lo_off = c->r0 - p.recv_lo_rows - c->lo_e;
    p.send_lo_off = c->r0 - c->lo_e;
    p.send_lo_rows = std::min<int64_t>(c->P0g - c->r0, h);      // rank-1's rows [r0, r0 + rows)
  }
  if (c->rank < c->nranks - 1) {
    p.recv_hi_off = c->r1 - c->lo_e;
    p.recv_hi_rows = std::min<int64_t>(h, c->P0g - c->r1);      // my rows [r1, r1 + rows)
    p.send_hi_rows = std::min<int64_t>(c->r1, h);               // rank+1's rows [r1 - rows, r1)
    p.send_hi_off = c->r1 - p.send_hi_rows - c->lo_e;
  }
  return p;
}
// the values halo exchanged after every step
HaloPlan halo_plan(const bsde_ctx* c) { return halo_plan(c, c->spike ? 1 : c->halo); }

int64_t row_len(const bsde_ctx* c) { return c->g.npts / c->g.P[0]; }

bsde_status exchange_nccl(bsde_ctx* c) {
  if (c->nranks <= 1 || c->grouped) return BSDE_OK;
  cudaEvent_t t0 = c->cfg.timing && !c->in_setup ? tmark(c) : nullptr;
  const HaloPlan hp = halo_plan(c);
  const int64_t rl = row_len(c);
  double* v = c->vbuf[c->cur];
  ncclResult_t nr = ncclGroupStart();
  for (int f = 0; f < c->F && nr == ncclSuccess; ++f) {
    double* b = v + (int64_t)f * c->g.npts;
    if (c->rank > 0) {
      nr = ncclSend(b + hp.send_lo_off * rl, (size_t)(hp.send_lo_rows * rl), ncclDouble, c->rank - 1, c->comm, c->stream);
      if (nr == ncclSuccess)
        nr = ncclRecv(b + hp.recv_lo_off * rl, (size_t)(hp.recv_lo_rows * rl), ncclDouble, c->rank - 1, c->comm, c->stream);
    }
    if (c->rank < c->nranks - 1 && nr == ncclSuccess) {
      nr = ncclSend(b + hp.send_hi_off * rl, (size_t)(hp.send_hi_rows * rl), ncclDouble, c->rank + 1, c->comm, c->stream);
      if (nr == ncclSuccess)
        nr = ncclRecv(b + hp.recv_hi_off * rl, (size_t)(hp.recv_hi_rows * rl), ncclDouble, c->rank + 1, c->comm, c->stream);
    }
  }
  ncclResult_t ne = ncclGroupEnd();
  tstage(c, ST_COMM, t0);
  if (nr != ncclSuccess || ne != ncclSuccess)
    return set_err(c, BSDE_ERR_COMM, "halo exchange: %s", ncclGetErrorString(nr != ncclSuccess ? nr : ne));
  return BSDE_OK;
}

// ------------------------------------------------------------------ SPIKE slab spline (§7)
// unknown-row range of rank p's axis-0 moment system (global rows): Dirichlet fold nodes fa, fb
static void spike_folds(int64_t P0g, int R, int p, int64_t& fa, int64_t& fb) {
  int64_t r0, r1;
  rank_rows(P0g, R, p, r0, r1);
  fa = p == 0 ? 1 : r0 - 1;
  fb = p == R - 1 ? P0g - 2 : r1;
}
// S^L_k of a system of n unknown rows: the response at row k to a unit moment at the left fold
static long double spike_sl(int64_t n, int64_t k) {
  const long double rho = sqrtl(3.0L) - 2.0L;
  return (powl(rho, (long double)(k + 1)) - powl(rho, (long double)(2 * n + 1 - k))) /
         (1.0L - powl(rho, (long double)(2 * n + 2)));
}
bsde_status spike_setup(bsde_ctx* c, char* base) {
  const Grid& g = c->g;
  const int R = c->nranks, F = c->F, p = c->rank;
  if (R > kMaxRanks) return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "SPIKE: nranks %d > %d", R, kMaxRanks);
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  c->plane_v = g.npts / g.P[0];
  c->plane_c = g.cstride[0];
  const size_t pv = (size_t)c->plane_v, pc = (size_t)c->plane_c;
  char* q = base;
  c->edge = (double*)q; q += al(sizeof(double) * (size_t)(c->K + 3) * F * 2 * pv);
  c->gath = (double*)q; q += al(sizeof(double) * (size_t)R * F * 2 * pv);
  c->xs = (double*)q; q += al(sizeof(double) * F * 2 * pv);
  c->xc = (double*)q; q += al(sizeof(double) * F * 2 * pc);
  c->xtmp = (double*)q; q += al(sizeof(double) * pc);
  c->slr = (double*)q;
  // the reduced system of the 2 (R - 1) interface moments u_i = m(r1_i - 1), v_i = m(r1_i):
  //   u_i - sA_i v_i - sB_i u_{i-1} = (last-row edge of rank i)
  //   v_i - sA_{i+1} u_i - sB_{i+1} v_{i+1} = (first-row edge of rank i + 1)
  // sA = S^L[0] = S^R[n-1], sB = S^L[n-1] = S^R[0]; the same matrix for every line: invert it once
  const int M = 2 * (R - 1);
  std::vector<long double> sA(R), sB(R), A((size_t)M * M, 0.0L), Inv((size_t)M * M, 0.0L);
  for (int r = 0; r < R; ++r) {
    int64_t fa, fb;
    spike_folds(c->P0g, R, r, fa, fb);
    const int64_t n = fb - fa - 1;
    if (n < 2) return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "SPIKE: rank %d has %lld unknown rows", r, (long long)n);
    sA[r] = spike_sl(n, 0);
    sB[r] = spike_sl(n, n - 1);
  }
  for (int i = 0; i < R - 1; ++i) {
    A[(size_t)(2 * i) * M + 2 * i] = 1.0L;
    A[(size_t)(2 * i) * M + 2 * i + 1] = -sA[i];
    if (i > 0) A[(size_t)(2 * i) * M + 2 * (i - 1)] = -sB[i];
    A[(size_t)(2 * i + 1) * M + 2 * i + 1] = 1.0L;
    A[(size_t)(2 * i + 1) * M + 2 * i] = -sA[i + 1];
    if (i + 1 < R - 1) A[(size_t)(2 * i + 1) * M + 2 * (i + 1) + 1] = -sB[i + 1];
  }
  for (int i = 0; i < M; ++i) Inv[(size_t)i * M + i] = 1.0L;
  for (int k = 0; k < M; ++k) {                   // Gauss-Jordan with partial pivoting
    int piv = k;
    for (int i = k + 1; i < M; ++i)
      if (fabsl(A[(size_t)i * M + k]) > fabsl(A[(size_t)piv * M + k])) piv = i;
    for (int j = 0; j < M; ++j) {
      std::swap(A[(size_t)k * M + j], A[(size_t)piv * M + j]);
      std::swap(Inv[(size_t)k * M + j], Inv[(size_t)piv * M + j]);
    }
    const long double dk = A[(size_t)k * M + k];
    for (int j = 0; j < M; ++j) { A[(size_t)k * M + j] /= dk; Inv[(size_t)k * M + j] /= dk; }
    for (int i = 0; i < M; ++i) {
      if (i == k) continue;
      const long double m = A[(size_t)i * M + k];
      if (m == 0.0L) continue;
      for (int j = 0; j < M; ++j) { A[(size_t)i * M + j] -= m * A[(size_t)k * M + j]; Inv[(size_t)i * M + j] -= m * Inv[(size_t)k * M + j]; }
    }
  }
  c->spk = SpikeArgs{};
  c->spk.gath = c->gath;
  c->spk.X = c->xs;
  c->spk.plane = c->plane_v;
  c->spk.F = F;
  c->spk.R = R;
  for (int j = 0; j < M; ++j) {
    c->spk.wL[j] = p > 0 ? (double)Inv[(size_t)(2 * (p - 1)) * M + j] : 0.0;      // m(r0 - 1) = u_{p-1}
    c->spk.wR[j] = p < R - 1 ? (double)Inv[(size_t)(2 * p + 1) * M + j] : 0.0;    // m(r1) = v_p
  }
  // own spike vectors, local rows [row_lo, row_lo + n)
  int64_t fa, fb;
  spike_folds(c->P0g, R, p, fa, fb);
  c->spk_n = fb - fa - 1;
  c->spk_row_lo = fa + 1 - c->lo_e;
  c->h_slr.assign((size_t)2 * c->spk_n, 0.0);
  for (int64_t k = 0; k < c->spk_n; ++k) {
    c->h_slr[(size_t)k] = (double)spike_sl(c->spk_n, k);
    c->h_slr[(size_t)(c->spk_n + k)] = (double)spike_sl(c->spk_n, c->spk_n - 1 - k);
  }
  cudaError_t e = cudaMemcpyAsync(c->slr, c->h_slr.data(), sizeof(double) * c->h_slr.size(), cudaMemcpyHostToDevice,
                                  c->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(c->xc, 0, sizeof(double) * F * 2 * pc, c->stream);   // pads stay 0
  if (e != cudaSuccess) return set_err(c, BSDE_ERR_CUDA, "SPIKE setup: %s", cudaGetErrorString(e));
  // the interface planes: a (d-1)-dimensional grid of axes 1 .. d-1 (same coefficient layout as a
  // slot's axis-0 row)
  Grid& gp = c->gplane;
  gp = Grid{};
  gp.d = g.d - 1;
  gp.npts = 1;
  for (int a = 0; a < 3; ++a) { gp.P[a] = 1; gp.vstride[a] = 0; gp.cstride[a] = 0; }
  for (int a = 0; a < gp.d; ++a) {
    gp.P[a] = g.P[a + 1];
    gp.xlo[a] = g.xlo[a + 1]; gp.xhi[a] = g.xhi[a + 1]; gp.dx[a] = g.dx[a + 1];
    gp.npts *= gp.P[a];
  }
  gp.vstride[gp.d - 1] = 1;
  for (int a = gp.d - 2; a >= 0; --a) gp.vstride[a] = gp.vstride[a + 1] * gp.P[a + 1];
  for (int a = 0; a < gp.d; ++a) gp.cstride[a] = g.cstride[a + 1];
  gp.cfield = c->plane_c;
  gp.cpad = 0;
  gp.off0 = 0; gp.Pg0 = gp.P[0]; gp.own0 = 0; gp.nown0 = gp.P[0];
  return BSDE_OK;
}

// X = the interface moments of this rank from the gathered edges, their splines XC, the
// correction of the slot's coefficients (one rank; the gather is done)
static cudaError_t spike_apply(bsde_ctx* c, int slot) {
  cudaError_t e = launch_spike_reduce(c->spk, c->stream);
  ++c->launches;
  if (e == cudaSuccess) e = launch_spline(c->gplane, c->xs, 2 * c->F, c->xc, c->xtmp, nullptr, c->stream, &c->launches);
  if (e != cudaSuccess) return e;
  double* dst = c->ring + (int64_t)slot * c->F * c->g.cfield;
  e = launch_spike_correct(dst, c->g.cfield, c->g.cstride[0], c->xc, c->plane_c, c->slr, c->spk_row_lo, c->spk_n,
                           c->rank == 0, c->rank == c->nranks - 1, c->F, c->stream);
  ++c->launches;
  return e;
}

// halo rows of ring slot `slot`'s final coefficients (SPIKE): local rows [r0 - h, r0) from
// rank - 1 and [r1, r1 + h) from rank + 1 (coefficient storage row = local row + 1)
bsde_status exchange_coef_nccl(bsde_ctx* c, int slot) {
  const HaloPlan hp = halo_plan(c, c->halo);
  const int64_t rl = c->g.cstride[0];
  double* v = c->ring + (int64_t)slot * c->F * c->g.cfield + rl;      // storage row 1 = local row 0
  ncclResult_t nr = ncclGroupStart();
  for (int f = 0; f < c->F && nr == ncclSuccess; ++f) {
    double* b = v + (int64_t)f * c->g.cfield;
    if (c->rank > 0) {
      nr = ncclSend(b + hp.send_lo_off * rl, (size_t)(hp.send_lo_rows * rl), ncclDouble, c->rank - 1, c->comm, c->stream);
      if (nr == ncclSuccess)
        nr = ncclRecv(b + hp.recv_lo_off * rl, (size_t)(hp.recv_lo_rows * rl), ncclDouble, c->rank - 1, c->comm, c->stream);
    }
    if (c->rank < c->nranks - 1 && nr == ncclSuccess) {
      nr = ncclSend(b + hp.send_hi_off * rl, (size_t)(hp.send_hi_rows * rl), ncclDouble, c->rank + 1, c->comm, c->stream);
      if (nr == ncclSuccess)
        nr = ncclRecv(b + hp.recv_hi_off * rl, (size_t)(hp.recv_hi_rows * rl), ncclDouble, c->rank + 1, c->comm, c->stream);
    }
  }
  ncclResult_t ne = ncclGroupEnd();
  if (nr != ncclSuccess || ne != ncclSuccess)
    return set_err(c, BSDE_ERR_COMM, "coefficient halo exchange: %s", ncclGetErrorString(nr != ncclSuccess ? nr : ne));
  return BSDE_OK;
}

// the interface correction of a freshly built slot: NCCL ranks all-gather the edges and finish
// now; an in-process group member defers it to the group (bsde_group_step)
bsde_status finish_level(bsde_ctx* c, int slot) {
  if (!c->spike) return BSDE_OK;
  if (c->grouped) {
    c->pending |= 1u << slot;
    return BSDE_OK;
  }
  cudaEvent_t t0 = c->cfg.timing && !c->in_setup ? tmark(c) : nullptr;
  const size_t cnt = (size_t)c->F * 2 * c->plane_v;
  ncclResult_t nr = ncclAllGather(edge_slot(c, slot), c->gath, cnt, ncclDouble, c->comm, c->stream);
  if (nr != ncclSuccess) return set_err(c, BSDE_ERR_COMM, "edge all-gather: %s", ncclGetErrorString(nr));
  tstage(c, ST_COMM, t0);
  cudaError_t e = spike_apply(c, slot);
  if (e != cudaSuccess) return set_err(c, BSDE_ERR_CUDA, "SPIKE correction: %s", cudaGetErrorString(e));
  cudaEvent_t t1 = c->cfg.timing && !c->in_setup ? tmark(c) : nullptr;
  bsde_status st = exchange_coef_nccl(c, slot);
  tstage(c, ST_COMM, t1);
  return st;
}

bsde_status spline_into(bsde_ctx* c, int slot) {
  cudaError_t e = build_level(c, slot);
  if (e != cudaSuccess) return set_err(c, BSDE_ERR_CUDA, "spline kernel: %s", cudaGetErrorString(e));
  return finish_level(c, slot);
}

void release(bsde_ctx* c) {
  if (!c) return;
  int dev = c->cfg.device;
  if (c->tap_off >= 0) arena_free(dev, c->tap_off);
  if (c->tap1_off >= 0) arena_free(dev, c->tap1_off);
  if (c->boot_tap_off >= 0) arena_free(dev, c->boot_tap_off);
  if (c->boot_tap1_off >= 0) arena_free(dev, c->boot_tap1_off);
  if (c->own_ws && c->ws) cudaFreeAsync(c->ws, c->stream);
  if (c->phase_ns) cudaFree(c->phase_ns);
  tfree(c);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}
}  // namespace

extern "C" {
static bsde_status bsde_eval_internal(bsde_ctx* c, const double* x, double* out);
}

// The evaluation point x = 0 (reading R4): the grid value if 0 is a grid node, else the
// spline of the newest level at 0.  With a slab partition the rank owning the cell of x = 0
// computes it; NCCL ranks then share it with an all-reduce (zeros elsewhere).
// Leaves out[] on the host (synchronises c->stream).
bsde_status eval_point(bsde_ctx* c, double* out) {
  for (int f = 0; f < 4; ++f) out[f] = 0.0;
  if (c->pb.sde_id != 0) {                 // forward SDE: X_0 = x_0 (Eq. 1), one rank (validate)
    return bsde_eval_internal(c, c->pb.sp + 9, out);
  }
  bool on_grid = true;
  for (int a = 0; a < c->d; ++a)
    if (!(c->g.xlo[a] == -c->g.xhi[a] && ((a == 0 ? c->P0g : c->g.P[a]) % 2) == 1)) on_grid = false;
  // global axis-0 row of the point (node or cell)
  const double u0 = (0.0 - c->g.xlo[0]) / c->g.dx[0];
  int64_t row = on_grid ? (c->P0g - 1) / 2 : std::min<int64_t>(std::max<int64_t>((int64_t)floor(u0), 0), c->P0g - 2);
  const bool owner = row >= c->r0 && row < c->r1;
  // SPIKE: the newest level's spline is a collective of every rank (NCCL), or built by the group
  const bool spike_rs = c->spike && !on_grid;
  if (spike_rs && !c->grouped) {
    bsde_status st = spline_into(c, c->RS);
    if (st) return st;
  }
  if (spike_rs && c->grouped && !c->rs_ready)
    return set_err(c, BSDE_ERR_STATE, "slab group member: the evaluation spline is built by bsde_group_solve");
  if (owner) {
    if (on_grid) {
      int64_t idx = (row - c->lo_e) * c->g.vstride[0];
      for (int a = 1; a < c->d; ++a) idx += ((c->g.P[a] - 1) / 2) * c->g.vstride[a];
      for (int f = 0; f < c->F; ++f) {
        cudaError_t e = cudaMemcpyAsync(&out[f], c->vbuf[c->cur] + (int64_t)f * c->g.npts + idx, sizeof(double),
                                        cudaMemcpyDeviceToHost, c->stream);
        if (e != cudaSuccess) return set_err(c, BSDE_ERR_CUDA, "read-back: %s", cudaGetErrorString(e));
      }
    } else {
      const double x[3] = {0, 0, 0};
      if (!spike_rs) {
        bsde_status st = spline_into(c, c->RS);               // newest level -> scratch slot
        if (st) return st;
      }
      cudaError_t e = c->cfg.interp == BSDE_INTERP_FD_BICUBIC
                          ? launch_eval_bicubic(c->g, c->ring + (int64_t)c->RS * c->F * c->g.cfield, c->F, x, c->dres, c->stream)
                          : launch_eval(c->g, c->ring + (int64_t)c->RS * c->F * c->g.cfield, c->F, x, c->dres, c->stream);
      ++c->launches;
      if (e == cudaSuccess) e = cudaMemcpyAsync(out, c->dres, sizeof(double) * c->F, cudaMemcpyDeviceToHost, c->stream);
      if (e != cudaSuccess) return set_err(c, BSDE_ERR_CUDA, "eval: %s", cudaGetErrorString(e));
    }
  }
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return set_err(c, BSDE_ERR_CUDA, "sync: %s", cudaGetErrorString(e));
  if (c->comm) {
    cudaError_t ce = cudaMemcpyAsync(c->dres, out, sizeof(double) * 4, cudaMemcpyHostToDevice, c->stream);
    ncclResult_t nr = ncclAllReduce(c->dres, c->dres, 4, ncclDouble, ncclSum, c->comm, c->stream);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(out, c->dres, sizeof(double) * 4, cudaMemcpyDeviceToHost, c->stream);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(c->stream);
    if (nr != ncclSuccess) return set_err(c, BSDE_ERR_COMM, "all-reduce of y0: %s", ncclGetErrorString(nr));
    if (ce != cudaSuccess) return set_err(c, BSDE_ERR_CUDA, "y0: %s", cudaGetErrorString(ce));
  }
  return BSDE_OK;
}

// in-process slab group (nranks contexts driven by one host thread, possibly on one GPU):
// copy halo rows of the newest values from the neighbours' buffers
bsde_status group_exchange(bsde_ctx** cs, int n) {
  for (int r = 0; r < n; ++r) {
    cudaSetDevice(cs[r]->cfg.device);
    cudaError_t e = cudaStreamSynchronize(cs[r]->stream);
    if (e != cudaSuccess) return set_err(cs[r], BSDE_ERR_CUDA, "group sync: %s", cudaGetErrorString(e));
  }
  for (int r = 0; r < n; ++r) {
    bsde_ctx* c = cs[r];
    const HaloPlan hp = halo_plan(c);
    const int64_t rl = row_len(c);
    cudaSetDevice(c->cfg.device);
    cudaEvent_t t0 = c->cfg.timing && !c->in_setup ? tmark(c) : nullptr;
    for (int side = 0; side < 2; ++side) {
      const int nbr = side == 0 ? r - 1 : r + 1;
      if (nbr < 0 || nbr >= n) continue;
      bsde_ctx* o = cs[nbr];
      const HaloPlan ho = halo_plan(o);
      const int64_t rows = side == 0 ? hp.recv_lo_rows : hp.recv_hi_rows;
      const int64_t dst_off = side == 0 ? hp.recv_lo_off : hp.recv_hi_off;
      const int64_t src_off = side == 0 ? ho.send_hi_off : ho.send_lo_off;
      const int64_t src_rows = side == 0 ? ho.send_hi_rows : ho.send_lo_rows;
      if (rows != src_rows) return set_err(c, BSDE_ERR_COMM, "halo plan mismatch (%lld vs %lld rows)", (long long)rows,
                                           (long long)src_rows);
      for (int f = 0; f < c->F; ++f) {
        double* dst = c->vbuf[c->cur] + (int64_t)f * c->g.npts + dst_off * rl;
        const double* src = o->vbuf[o->cur] + (int64_t)f * o->g.npts + src_off * rl;
        cudaError_t e = cudaMemcpyPeerAsync(dst, c->cfg.device, src, o->cfg.device, sizeof(double) * rows * rl, c->stream);
        if (e != cudaSuccess) return set_err(c, BSDE_ERR_CUDA, "halo copy: %s", cudaGetErrorString(e));
      }
    }
    tstage(c, ST_COMM, t0);
  }
  for (int r = 0; r < n; ++r) {
    cudaSetDevice(cs[r]->cfg.device);
    cudaError_t e = cudaStreamSynchronize(cs[r]->stream);
    if (e != cudaSuccess) return set_err(cs[r], BSDE_ERR_CUDA, "group sync: %s", cudaGetErrorString(e));
  }
  return BSDE_OK;
}

static bsde_status group_sync(bsde_ctx** cs, int n) {
  for (int r = 0; r < n; ++r) {
    cudaSetDevice(cs[r]->cfg.device);
    cudaError_t e = cudaStreamSynchronize(cs[r]->stream);
    if (e != cudaSuccess) return set_err(cs[r], BSDE_ERR_CUDA, "group sync: %s", cudaGetErrorString(e));
  }
  return BSDE_OK;
}

// SPIKE interface correction of ring slot `slot` across an in-process group: gather every
// member's edge moments (peer copies), correct each member's slot, then copy the coefficient
// halo rows from the neighbours
bsde_status group_finish(bsde_ctx** cs, int n, int slot) {
  bsde_status st = group_sync(cs, n);
  if (st) return st;
  for (int r = 0; r < n; ++r) {
    bsde_ctx* c = cs[r];
    cudaSetDevice(c->cfg.device);
    const size_t cnt = (size_t)c->F * 2 * c->plane_v;
    for (int q = 0; q < n; ++q) {
      cudaError_t e = cudaMemcpyPeerAsync(c->gath + (int64_t)q * cnt, c->cfg.device, edge_slot(cs[q], slot),
                                          cs[q]->cfg.device, sizeof(double) * cnt, c->stream);
      if (e != cudaSuccess) return set_err(c, BSDE_ERR_CUDA, "edge gather: %s", cudaGetErrorString(e));
    }
    cudaError_t e = spike_apply(c, slot);
    if (e != cudaSuccess) return set_err(c, BSDE_ERR_CUDA, "SPIKE correction: %s", cudaGetErrorString(e));
  }
  if ((st = group_sync(cs, n))) return st;
  for (int r = 0; r < n; ++r) {
    bsde_ctx* c = cs[r];
    const HaloPlan hp = halo_plan(c, c->halo);
    const int64_t rl = c->g.cstride[0];
    cudaSetDevice(c->cfg.device);
    for (int side = 0; side < 2; ++side) {
      const int nbr = side == 0 ? r - 1 : r + 1;
      if (nbr < 0 || nbr >= n) continue;
      bsde_ctx* o = cs[nbr];
      const HaloPlan ho = halo_plan(o, o->halo);
      const int64_t rows = side == 0 ? hp.recv_lo_rows : hp.recv_hi_rows;
      const int64_t dst_off = side == 0 ? hp.recv_lo_off : hp.recv_hi_off;
      const int64_t src_off = side == 0 ? ho.send_hi_off : ho.send_lo_off;
      const int64_t src_rows = side == 0 ? ho.send_hi_rows : ho.send_lo_rows;
      if (rows != src_rows)
        return set_err(c, BSDE_ERR_COMM, "coefficient halo plan mismatch (%lld vs %lld rows)", (long long)rows,
                       (long long)src_rows);
      for (int f = 0; f < c->F; ++f) {
        double* dst = c->ring + (int64_t)slot * c->F * c->g.cfield + (int64_t)f * c->g.cfield + (1 + dst_off) * rl;
        const double* src = o->ring + (int64_t)slot * o->F * o->g.cfield + (int64_t)f * o->g.cfield + (1 + src_off) * rl;
        cudaError_t e = cudaMemcpyPeerAsync(dst, c->cfg.device, src, o->cfg.device, sizeof(double) * rows * rl, c->stream);
        if (e != cudaSuccess) return set_err(c, BSDE_ERR_CUDA, "coefficient halo copy: %s", cudaGetErrorString(e));
      }
    }
  }
  for (int r = 0; r < n; ++r) cs[r]->pending &= ~(1u << slot);
  return group_sync(cs, n);
}

// ------------------------------------------------------------------ ABI
extern "C" {

bsde_status bsde_query_workspace(const bsde_config* cfg, size_t* bytes) {
  bsde_ctx* c = nullptr;
  bsde_status st = validate(cfg, c);
  if (st) return st;
  const int K = std::max(cfg->Ky, cfg->Kz);
  Grid g{};
  fill_grid(cfg, g, (cfg->T - cfg->t0) / cfg->N);
  *bytes = layout(g, 1 + cfg->d, K, cfg->L, use_fused3d(cfg), use_aff2(cfg), cfg->nranks,
                  cfg->nranks > 1 && cfg->slab_spline == 0).total;
  return BSDE_OK;
}

bsde_status bsde_setup(const bsde_config* cfg, void* d_workspace, size_t bytes, bsde_ctx** out) {
  const double t_start = now_s();
  if (out) *out = nullptr;
  if (!out) return set_err(nullptr, BSDE_ERR_INVALID_ARGUMENT, "out is NULL");
  bsde_status st = validate(cfg, nullptr);
  if (st) return st;
  bsde_ctx* c = new (std::nothrow) bsde_ctx();
  if (!c) return set_err(nullptr, BSDE_ERR_RESOURCE_LIMIT, "host allocation failed");
  c->cfg = *cfg;
  c->d = cfg->d;
  c->F = 1 + cfg->d;
  c->Ky = cfg->Ky;
  c->Kz = cfg->Kz;
  c->K = std::max(cfg->Ky, cfg->Kz);
  c->RS = c->K + 2;
  c->L = cfg->L;
  c->N = cfg->N;
  c->dt = (cfg->T - cfg->t0) / cfg->N;
  fill_grid(cfg, c->g, c->dt);
  c->pb.d = c->d;
  c->pb.driver_id = cfg->driver_id;
  c->pb.terminal_id = cfg->terminal_id;
  c->pb.smoothing = cfg->smoothing;
  for (int k = 0; k < 12; ++k) { c->pb.dp[k] = cfg->driver_params[k]; c->pb.tp[k] = cfg->terminal_params[k]; }
  c->pb.T = cfg->T;
  c->pb.t0 = cfg->t0;
  c->pb.sde_id = cfg->sde_id;
  for (int k = 0; k < 12; ++k) c->pb.sp[k] = cfg->sde_params[k];
  c->pb.dt = c->dt;
  c->pb.N = cfg->N;
  for (int j = 0; j <= c->Ky; ++j) c->gy[j] = (double)kTab1[c->Ky - 1][j];
  for (int j = 0; j <= c->Kz; ++j) c->gz[j] = (double)kTab2[c->Kz - 1][j];
  hermite_rule(c->L, c->gh_a, c->gh_w);

  auto fail = [&](bsde_status s) {
    g_setup_error = c->err;
    release(c);
    return s;
  };
  // tap tables (global grid spacing), then the slab partition of axis 0 (d >= 2, nranks > 1)
  build_taps(c, c->K, c->dt, c->taps, &c->qspan, &c->qspan1);
  c->nranks = cfg->nranks > 1 ? cfg->nranks : 1;
  c->rank = c->nranks > 1 ? cfg->rank : 0;
  c->P0g = c->g.P[0];
  if ((st = plan_partition(c))) return fail(st);
  if (c->nranks > 1) {
    localize_grid(c->g, c->lo_e, c->hi_e, c->r0, c->r1);
    c->grouped = cfg->nccl_unique_id == nullptr;
  }
  cudaError_t ce = cudaSetDevice(cfg->device);
  if (ce != cudaSuccess) { set_err(c, BSDE_ERR_CUDA, "cudaSetDevice(%d): %s", cfg->device, cudaGetErrorString(ce)); return fail(BSDE_ERR_CUDA); }
  {   // kernel attributes: once per device and process (they are per-function device state)
    static std::mutex mu;
    static bool done[64] = {};
    std::lock_guard<std::mutex> lk(mu);
    const int dv = cfg->device >= 0 && cfg->device < 64 ? cfg->device : 0;
    ce = done[dv] ? cudaSuccess : init_device_attributes();
    if (ce == cudaSuccess) done[dv] = true;
  }
  if (ce != cudaSuccess) { set_err(c, BSDE_ERR_CUDA, "kernel attributes: %s", cudaGetErrorString(ce)); return fail(BSDE_ERR_CUDA); }
  if (cfg->stream) c->stream = (cudaStream_t)cfg->stream;
  else {
    ce = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (ce != cudaSuccess) { set_err(c, BSDE_ERR_CUDA, "stream: %s", cudaGetErrorString(ce)); return fail(BSDE_ERR_CUDA); }
    c->own_stream = true;
  }
  if (c->nranks > 1 && !c->grouped) {
    ncclUniqueId id;
    memcpy(&id, cfg->nccl_unique_id, sizeof id);
    ncclResult_t nr = ncclCommInitRank(&c->comm, c->nranks, id, c->rank);
    if (nr != ncclSuccess) {
      set_err(c, BSDE_ERR_COMM, "ncclCommInitRank: %s", ncclGetErrorString(nr));
      return fail(BSDE_ERR_COMM);
    }
  }
  // memory
  c->spike = c->nranks > 1 && cfg->slab_spline == 0 && c->d >= 2;
  Layout lay = layout(c->g, c->F, c->K, c->L, use_fused3d(cfg), use_aff2(cfg), c->nranks, c->spike);
  if (d_workspace) {
    if (bytes < lay.total) {
      set_err(c, BSDE_ERR_RESOURCE_LIMIT, "workspace of %zu bytes < required %zu", bytes, lay.total);
      return fail(BSDE_ERR_RESOURCE_LIMIT);
    }
    c->ws = (char*)d_workspace;
    c->ws_bytes = bytes;
  } else {
    // stream-ordered allocation from the device's default pool: a setup after a destroy reuses
    // the freed block without a device synchronisation (small problems are setup-bound)
    ce = cudaMallocAsync((void**)&c->ws, lay.total, c->stream);
    if (ce != cudaSuccess) {
      set_err(c, BSDE_ERR_RESOURCE_LIMIT, "cudaMalloc(%zu) failed: %s (grid %lld points)", lay.total,
              cudaGetErrorString(ce), (long long)c->g.npts);
      cudaGetLastError();
      return fail(BSDE_ERR_RESOURCE_LIMIT);
    }
    c->own_ws = true;
    c->ws_bytes = lay.total;
  }
  c->vbuf[0] = (double*)(c->ws + lay.values);
  c->vbuf[1] = c->vbuf[0] + (lay.ring - lay.values) / (2 * sizeof(double));
  c->ring = (double*)(c->ws + lay.ring) + c->g.cpad;      // storage 0 of slot 0, field 0
  c->tmp0 = (double*)(c->ws + lay.tmp0);
  c->tmp1 = (double*)(c->ws + lay.tmp1);
  c->a3 = lay.a3 != lay.acc3 ? (double*)(c->ws + lay.a3) : nullptr;
  c->acc3 = lay.acc3 != lay.picard ? (double*)(c->ws + lay.acc3) : nullptr;
  c->picard = (int32_t*)(c->ws + lay.picard);
  c->bad = (unsigned long long*)(c->ws + lay.bad);
  c->barrier = (unsigned*)(c->ws + lay.barrier);
  c->dres = (double*)(c->ws + lay.dres);
  if (c->spike) {
    if ((st = spike_setup(c, c->ws + lay.spike))) return fail(st);
  }
#ifdef BSDE_DEBUG
  if (getenv("BSDE_PHASE_TIMING")) {      // debug build only: per-CTA phase stamps of the fused 1-D kernel
    if (cudaMalloc((void**)&c->phase_ns, (size_t)8 * 32 * 600 * 1100) != cudaSuccess) c->phase_ns = nullptr;
    else cudaMemset(c->phase_ns, 0, (size_t)8 * 32 * 600 * 1100);
  }
#endif
  // zero the whole ring once: the padding entry c_{P+1} of every line is read with weight 0
  ce = cudaMemsetAsync(c->ring - c->g.cpad, 0, sizeof(double) * (size_t)(c->RS + 1) * c->F * c->g.cfield, c->stream);
  if (ce == cudaSuccess) ce = cudaMemsetAsync(c->picard, 0, sizeof(int32_t) * c->g.npts, c->stream);
  if (ce == cudaSuccess) ce = cudaMemsetAsync(c->bad, 0xff, sizeof(unsigned long long), c->stream);
  // both value buffers: halo rows of a slab are defined before the first exchange
  if (ce == cudaSuccess) ce = cudaMemsetAsync(c->vbuf[0], 0, sizeof(double) * (size_t)c->F * c->g.npts, c->stream);
  if (ce == cudaSuccess) ce = cudaMemsetAsync(c->vbuf[1], 0, sizeof(double) * (size_t)c->F * c->g.npts, c->stream);
  if (ce != cudaSuccess) { set_err(c, BSDE_ERR_CUDA, "memset: %s", cudaGetErrorString(ce)); return fail(BSDE_ERR_CUDA); }

  // tap tables -> constant arena
  if (cfg->kernel_variant >= 10) c->fused_variant = cfg->kernel_variant - 10;
  cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, cfg->device);
  if (c->d == 2) {
    c->wc2 = fused2d_window(c->taps.data(), c->K, c->L);
    if (fused2d_smem(c->wc2) > 220 * 1024) c->wc2 = 0;
    c->wca = aff2_window(c->taps.data(), c->K, c->L);
    if (aff2_smem(c->wca) > 220 * 1024) c->wca = 0;
  }
  if (c->d == 3) {
    c->wc2 = fused3d_window(c->taps.data(), c->K, c->L);
    if (fused3d_smem(c->wc2, 4) > 112 * 1024) c->wc2 = 0;
  }
  if (c->d == 1 && cfg->sde_id == BSDE_SDE_BROWNIAN) {
    c->geo.ok = fused1d_geometry(c->g, c->K, c->L, c->qspan, c->nsm, c->fused_variant, c->geo.fz,
                                 c->geo.threads, c->geo.blocks, c->geo.smem);
    set_distances(c, c->taps, c->K, c->geo);
    if (cfg->kernel_variant == 0 && c->geo.ok && !c->geo.single) {
      // the default's one-tile-per-CTA launch does not fit (long lines): the two-CTA-per-SM variant
      c->fused_variant = fused1d_alt_variant();
      c->geo = bsde_ctx::Geo{};
      c->geo.ok = fused1d_geometry(c->g, c->K, c->L, c->qspan, c->nsm, c->fused_variant, c->geo.fz,
                                   c->geo.threads, c->geo.blocks, c->geo.smem);
      set_distances(c, c->taps, c->K, c->geo);
    }
  }
  if (cfg->sde_id != BSDE_SDE_BROWNIAN || cfg->interp != BSDE_INTERP_SPLINE) { c->wc2 = 0; c->wca = 0; }
  // small 1-D grids (no fused geometry): the single-CTA whole-sweep kernel when its shared
  // memory (every ring line + the spline scratch) fits
  if (c->d == 1 && cfg->sde_id == BSDE_SDE_BROWNIAN && !c->geo.ok && cfg->kernel_variant == 0 && c->g.P[0] >= 16 &&
      small1d_smem((int)c->g.P[0], (int)c->g.cpad, c->RS) <= 200 * 1024)
    c->small_ok = true;
  c->tap_count = (int)c->taps.size();
  {
    const int bytes = (int)(sizeof(AxisTap) * c->taps.size());
    c->tap_off = arena_alloc(cfg->device, bytes);
    if (c->tap_off < 0) {
      set_err(c, BSDE_ERR_RESOURCE_LIMIT, "constant tap arena full (%d bytes needed)", bytes);
      return fail(BSDE_ERR_RESOURCE_LIMIT);
    }
    ce = upload_arena(c->taps.data(), bytes, c->tap_off, c->stream);
    if (ce == cudaSuccess && c->d == 1) {
      std::vector<Tap1D> t1 = build_tap1d(c->taps, c->K, c->L, c->Ky, c->Kz, c->gy, c->gz);
      const int b1 = (int)(sizeof(Tap1D) * t1.size());
      c->tap1_off = arena_alloc(cfg->device, b1);
      if (c->tap1_off >= 0) ce = upload_arena(t1.data(), b1, c->tap1_off, c->stream);
      else c->geo.ok = false;               // no room: generic kernel
    }
    if (ce != cudaSuccess) { set_err(c, BSDE_ERR_CUDA, "taps: %s", cudaGetErrorString(ce)); return fail(BSDE_ERR_CUDA); }
  }
  if (cfg->smoothing && c->d >= 2) {      // the Gauss-Legendre cell rule of the d >= 2 smoothing (R11)
    double gx[kSmoothGL], gw[kSmoothGL];
    legendre_rule(kSmoothGL, gx, gw);
    ce = upload_gl(gx, gw, c->stream);
    if (ce != cudaSuccess) { set_err(c, BSDE_ERR_CUDA, "GL: %s", cudaGetErrorString(ce)); return fail(BSDE_ERR_CUDA); }
  }

  // K initial layers N, N-1, ..., N-K+1
  const int K = c->K, N = c->N;
  ce = launch_layer(c->pb, c->g, cfg->T, true, c->vbuf[c->cur], c->stream);
  ++c->launches;
  if (ce != cudaSuccess) { set_err(c, BSDE_ERR_CUDA, "layer: %s", cudaGetErrorString(ce)); return fail(BSDE_ERR_CUDA); }
  if ((st = spline_into(c, N % c->RS))) return fail(st);
  c->level = N;
  cudaEvent_t tb0 = tmark(c);                  // device time of the K-1 initial layers (t_bootstrap_s)
  c->in_setup = true;
  if (K > 1 && cfg->bootstrap == 1) {
    // one-step scheme (K = 1) on S_b sub-steps per coarse interval (reading R9)
    const int Sb = cfg->bootstrap_substeps > 0 ? cfg->bootstrap_substeps : 1;
    const double db = c->dt / Sb;
    std::vector<AxisTap> bt;
    build_taps(c, 1, db, bt, &c->boot_qspan, &c->boot_qspan1);
    if (c->d == 1 && cfg->sde_id == BSDE_SDE_BROWNIAN) {
      c->boot_geo.ok = fused1d_geometry(c->g, 1, c->L, c->boot_qspan, c->nsm, c->fused_variant,
                                        c->boot_geo.fz, c->boot_geo.threads, c->boot_geo.blocks, c->boot_geo.smem);
      set_distances(c, bt, 1, c->boot_geo);
    }
    if (c->d == 2) {
      c->boot_wc2 = fused2d_window(bt.data(), 1, c->L);
      if (fused2d_smem(c->boot_wc2) > 220 * 1024) c->boot_wc2 = 0;
    }
    if (c->d == 3) {
      c->boot_wc2 = fused3d_window(bt.data(), 1, c->L);
      if (fused3d_smem(c->boot_wc2, 4) > 112 * 1024) c->boot_wc2 = 0;
    }
    const double g1[2] = {0.5, 0.5};
    {
      const int bytes = (int)(sizeof(AxisTap) * bt.size());
      c->boot_tap_off = arena_alloc(cfg->device, bytes);
      if (c->boot_tap_off < 0) {
        set_err(c, BSDE_ERR_RESOURCE_LIMIT, "constant tap arena full (bootstrap)");
        return fail(BSDE_ERR_RESOURCE_LIMIT);
      }
      ce = upload_arena(bt.data(), bytes, c->boot_tap_off, c->stream);
      if (ce == cudaSuccess && c->d == 1) {
        std::vector<Tap1D> t1 = build_tap1d(bt, 1, c->L, 1, 1, g1, g1);
        const int b1 = (int)(sizeof(Tap1D) * t1.size());
        c->boot_tap1_off = arena_alloc(cfg->device, b1);
        if (c->boot_tap1_off >= 0) ce = upload_arena(t1.data(), b1, c->boot_tap1_off, c->stream);
      }
      if (ce != cudaSuccess) { set_err(c, BSDE_ERR_CUDA, "taps: %s", cudaGetErrorString(ce)); return fail(BSDE_ERR_CUDA); }
    }
    for (int m = N - 1; m >= N - K + 1; --m) {
      for (int s = Sb - 1; s >= 0; --s) {
        const double tn = cfg->t0 + m * c->dt + s * db;
        const int slots[1] = {c->RS};                        // scratch slot
        // the fused 1-D kernel reads the spline of its input level from the ring: build it
        if (c->d == 1 && c->boot_geo.ok && c->boot_geo.single && (st = spline_into(c, c->RS))) return fail(st);
        if ((st = run_step(c, 1, 1, 1, g1, g1, db, tn, slots, -1, c->boot_tap_off, c->boot_tap1_off, c->boot_geo,
                           cfg->kernel_variant, c->boot_wc2)))
          return fail(st);
      }
      if ((st = spline_into(c, m % c->RS))) return fail(st);
      c->level = m;
    }
  } else {
    for (int m = N - 1; m >= N - K + 1; --m) {
      ce = launch_layer(c->pb, c->g, cfg->t0 + m * c->dt, false, c->vbuf[c->cur], c->stream);
      ++c->launches;
      if (ce != cudaSuccess) { set_err(c, BSDE_ERR_CUDA, "layer: %s", cudaGetErrorString(ce)); return fail(BSDE_ERR_CUDA); }
      if ((st = spline_into(c, m % c->RS))) return fail(st);
      c->level = m;
    }
  }
  tstage(c, ST_BOOT, tb0);
  c->in_setup = false;
  ce = cudaMemsetAsync(c->picard, 0, sizeof(int32_t) * c->g.npts, c->stream);
  if (ce != cudaSuccess) { set_err(c, BSDE_ERR_CUDA, "memset: %s", cudaGetErrorString(ce)); return fail(BSDE_ERR_CUDA); }
  c->t_setup = now_s() - t_start;
  *out = c;
  return BSDE_OK;
}

static bsde_status step_internal(bsde_ctx* c) {
  if (c->level <= 0) return set_err(c, BSDE_ERR_STATE, "already at n = 0");
  cudaSetDevice(c->cfg.device);
  const int n = c->level - 1;
  int slots[kMaxK];
  for (int j = 1; j <= c->K; ++j) slots[j - 1] = (n + j) % c->RS;   // ring slot of level n+j
  bsde_status st = run_step(c, c->K, c->Ky, c->Kz, c->gy, c->gz, c->dt, c->cfg.t0 + n * c->dt, slots, n % c->RS, c->tap_off,
                            c->tap1_off, c->geo, c->cfg.kernel_variant, c->wc2);
  if (st) return st;
  c->level = n;
  return BSDE_OK;
}

bsde_status bsde_step(bsde_ctx* c) {
  if (!c) return set_err(nullptr, BSDE_ERR_INVALID_ARGUMENT, "ctx is NULL");
  if (c->grouped && c->nranks > 1)
    return set_err(c, BSDE_ERR_STATE, "member of an in-process slab group: use bsde_group_step (halo refresh)");
  return step_internal(c);
}

// device non-finite flag: the first (largest n) non-finite point, with (n, i, t_n, x_i) and the
// y, z values the newest level holds there
static bsde_status check_bad(bsde_ctx* c) {
  unsigned long long bad = 0;
  cudaError_t e = cudaMemcpyAsync(&bad, c->bad, sizeof bad, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return set_err(c, BSDE_ERR_CUDA, "sync: %s", cudaGetErrorString(e));
  if (bad == ~0ULL) return BSDE_OK;
  const int n = (int)(0xFFFFFu - (unsigned)(bad >> kBadShift));
  const int64_t p = (int64_t)(bad & ((1ULL << kBadShift) - 1));
  double x[3] = {0, 0, 0}, v[4] = {0, 0, 0, 0};
  int64_t q = p;
  for (int a = c->d - 1; a >= 0; --a) {
    const int64_t i = q % c->g.P[a] + (a == 0 ? c->g.off0 : 0);
    q /= c->g.P[a];
    x[a] = c->g.xlo[a] + (double)i * c->g.dx[a];
  }
  for (int f = 0; f < c->F && p < c->g.npts; ++f)
    cudaMemcpy(&v[f], c->vbuf[c->cur] + (int64_t)f * c->g.npts + p, sizeof(double), cudaMemcpyDeviceToHost);
  return set_err(c, BSDE_ERR_NUMERICAL_DOMAIN,
                 "non-finite y or z: first at level n = %d (t = %.6g), point i = %lld (x = %.6g, %.6g, %.6g); the newest "
                 "level (n = %d) holds y = %g, z = (%g, %g, %g) there", n, c->cfg.t0 + n * c->dt, (long long)p, x[0], x[1],
                 x[2], c->level, v[0], v[1], v[2], v[3]);
}

// device counter of the Picard iterations the fused 1-D kernel executes (in the dres area)
static unsigned long long* pexec_counter(const bsde_ctx* c) {
  return reinterpret_cast<unsigned long long*>(c->dres + 16);
}

// StepArgs of a persistent fused launch (ring_mode 1: the kernel derives the per-step slots,
// times and value buffers from Persist1D)
static StepArgs persistent_args(const bsde_ctx* c) {
  StepArgs s{};
  s.ring = c->ring;
  s.slot_elems = (int64_t)c->F * c->g.cfield;
  s.cfield = c->g.cfield;
  s.cpad = c->g.cpad;
  s.K = c->K; s.Ky = c->Ky; s.Kz = c->Kz; s.L = c->L;
  s.ring_slots = c->RS;
  s.tap_off = c->tap_off;
  s.tap1_off = c->tap1_off;
  s.gz0 = c->gz[0];
  s.ky_dt = c->Ky * c->dt;
  s.ky_dt_gy0 = c->Ky * c->dt * c->gy[0];
  s.picard_max = c->cfg.picard_max;
  s.picard_tol = c->cfg.picard_tol;
  s.picard = c->picard;
  s.bad = c->bad;
  s.phase_ns = c->phase_ns;
  s.picard_exec = pexec_counter(c);
  return s;
}

static void fill_result(bsde_ctx* c, bsde_result* res, const double out[4], double t_sweep, double t_call,
                        int64_t steps) {
  memset(res, 0, sizeof *res);
  res->y0 = out[0];
  for (int a = 0; a < c->d; ++a) res->z0[a] = out[1 + a];
  res->t_setup_s = c->t_setup;
  res->t_sweep_s = t_sweep;
  res->t_total_s = c->t_setup + t_call;
  res->updates = c->g.nown0 * row_len(c) * steps;
  res->picard_max_used = c->cfg.picard_max;
  res->picard_iters = -1;
  tcollect(c);                                   // the stream is synchronised by now
  res->t_spline_s = c->t_stage[ST_SPLINE];
  res->t_quad_s = c->t_stage[ST_QUAD];
  res->t_comm_s = c->t_stage[ST_COMM];
  res->t_bootstrap_s = c->t_stage[ST_BOOT];
  c->t_stage[ST_SPLINE] = c->t_stage[ST_QUAD] = c->t_stage[ST_COMM] = 0.0;   // per call
}

bsde_status bsde_solve(bsde_ctx* c, bsde_result* res) {
  if (!c) return set_err(nullptr, BSDE_ERR_INVALID_ARGUMENT, "ctx is NULL");
  if (c->grouped && c->nranks > 1) return set_err(c, BSDE_ERR_STATE, "in-process slab group: use bsde_group_solve");
  cudaSetDevice(c->cfg.device);
  const double t0 = now_s();
  cudaEvent_t e0, e1;
  if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess)
    return set_err(c, BSDE_ERR_CUDA, "event create");
  cudaEventRecord(e0, c->stream);
  int64_t steps = 0;
  bsde_status st = BSDE_OK;
  // d = 1 fused path: all remaining steps in one cooperative (persistent) launch
  const bool fused = c->d == 1 && (c->cfg.kernel_variant == 0 || c->cfg.kernel_variant >= 10) && c->geo.ok &&
                     c->geo.single && c->tap1_off >= 0;
  int64_t pexec = -1;
  bool read_pexec = false;
  if (c->small_ok && c->level >= 1) {                  // latency path: one single-CTA launch
    const StepArgs s = persistent_args(c);
    const int ns = c->level;
    cudaEvent_t tq = c->cfg.timing ? tmark(c) : nullptr;
    cudaMemsetAsync(pexec_counter(c), 0, sizeof(unsigned long long), c->stream);
    cudaError_t e = launch_small_sweep(s, c->g, c->pb, c->level - 1, ns, c->cur, c->cfg.t0, c->dt, c->vbuf[0],
                                       c->vbuf[1], c->stream);
    ++c->launches;
    tstage(c, ST_QUAD, tq);
    if (e != cudaSuccess) st = set_err(c, BSDE_ERR_CUDA, "small sweep kernel: %s", cudaGetErrorString(e));
    else {
      c->cur ^= (ns & 1);
      c->level = 0;
      steps = ns;
      read_pexec = true;                               // after the sweep's end event
    }
  } else if (fused && c->level >= 2) {
    const StepArgs s = persistent_args(c);
    const int ns = c->level;
    cudaMemsetAsync(pexec_counter(c), 0, sizeof(unsigned long long), c->stream);
    cudaEvent_t tq = c->cfg.timing ? tmark(c) : nullptr;
    cudaError_t e = launch_fused1d_steps(s, c->g, c->pb, c->geo.fz, c->level - 1, ns, 1, c->cur, c->cfg.t0, c->dt, c->vbuf[0],
                               c->vbuf[1], c->barrier, c->geo.D, c->geo.DK, c->geo.threads, c->geo.blocks,
                               c->geo.smem, c->stream);
    ++c->launches;
    tstage(c, ST_QUAD, tq);
    if (e != cudaSuccess) st = set_err(c, BSDE_ERR_CUDA, "persistent step kernel: %s", cudaGetErrorString(e));
    else {
      c->cur ^= (ns & 1);
      c->level = 0;
      steps = ns;
      read_pexec = true;
    }
  }
  while (st == BSDE_OK && c->level > 0) {
    if ((st = step_internal(c))) break;
    ++steps;
  }
  cudaEventRecord(e1, c->stream);                      // the sweep's device time ends here
  if (read_pexec) {                                    // executed Picard iterations (one read-back)
    unsigned long long v = 0;
    if (cudaMemcpyAsync(&v, pexec_counter(c), sizeof v, cudaMemcpyDeviceToHost, c->stream) == cudaSuccess &&
        cudaStreamSynchronize(c->stream) == cudaSuccess)
      pexec = (int64_t)v;
  }
  if (st) { cudaEventDestroy(e0); cudaEventDestroy(e1); return st; }
  if ((st = check_bad(c))) { cudaEventDestroy(e0); cudaEventDestroy(e1); return st; }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  // the evaluation point is a collective in the NCCL mode: every rank takes part
  if (res || c->comm) {
    double out[4] = {0, 0, 0, 0};
    if ((st = eval_point(c, out))) return st;
    cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return set_err(c, BSDE_ERR_CUDA, "sync: %s", cudaGetErrorString(e));
    if (res) {
      fill_result(c, res, out, ms * 1e-3, now_s() - t0, steps);
      res->picard_iters = pexec;
    }
  }
  return BSDE_OK;
}

// CTA distances of the fused kernel's neighbour waits for CTAs owning `tile` points (the
// problem-partitioned batch: a range of ns tiles per CTA)
static void distances_for(const bsde_ctx* c, int tile, int* D, int& DK) {
  const int L = c->L;
  for (int j = 0; j <= kMaxK; ++j) D[j] = 0;
  D[0] = (kP2Halo + 6 + tile - 1) / tile;
  int dk = D[0];
  for (int j = 1; j <= c->K; ++j) {
    const int qa = -c->taps[(size_t)(j - 1) * L].q, qb = c->taps[(size_t)(j - 1) * L + L - 1].q;
    D[j] = (std::max(qa, qb) + 4 + tile - 1) / tile;
    dk = std::max(dk, D[j]);
  }
  DK = dk;
}

// Problem-partitioned plan of a batch (fused1d.cuh FusedBatch::part): the problems form groups;
// group g gets gcta[g] CTAs, each serving the group's problems round robin on a range of gns[g]
// tiles.  The fixed costs of a (CTA, problem, step) -- the spline pass, the hand-offs -- are paid
// for fewer CTAs than round robin, and within a group of >= 2 problems a problem's neighbour waits
// overlap the other problem's work.  Cost model of a group's (CTA, step) in units of one
// tile-level: sum_{i in g} steps_i (ns (K_i a + b) + c); the plan minimises the slowest group's
// time subject to sum gcta <= slots (binary search on that time).  Returns false if none fits.
static bool plan_batch_groups(int n, const int* K, const int* steps, const int* group, int ngroup, int tiles, int slots,
                              int nsmax, int* gcta, int* gns, double* t_pred = nullptr) {
  // (r2) calibrated on the 12-warp default's per-round timeline (scripts/batch_timeline.py): a tile
  // costs ~2.4 us per level + ~4.7 us fixed (epilogue, window start, its share of the pass-2
  // spline), a round ~3.6 us more (flag waits)
  const double a = 1.0, b = 2.0, c = 1.5;
  auto cost = [&](int gi, int s) {
    double t = 0.0;
    for (int i = 0; i < n; ++i)
      if (group[i] == gi) t += (double)steps[i] * (s * (K[i] * a + b) + c);
    return t;
  };
  auto fit = [&](double T, int* nc, int* nsv) {
    int tot = 0;
    for (int gi = 0; gi < ngroup; ++gi) {
      int s = 0;
      for (int t = nsmax; t >= 1; --t)
        if (cost(gi, t) <= T) { s = t; break; }
      if (s == 0) return false;
      nc[gi] = (tiles + s - 1) / s;
      nsv[gi] = (tiles + nc[gi] - 1) / nc[gi];           // balanced tiles per CTA
      tot += nc[gi];
    }
    return tot <= slots;
  };
  double lo = 0.0, hi = 0.0;
  for (int gi = 0; gi < ngroup; ++gi) hi = std::max(hi, cost(gi, nsmax));
  hi *= 4.0;
  int nc[kMaxBatch], nsv[kMaxBatch];
  if (!fit(hi, nc, nsv)) return false;
  for (int it = 0; it < 60; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (fit(mid, nc, nsv)) hi = mid; else lo = mid;
  }
  fit(hi, gcta, gns);
  if (t_pred) {                      // the plan's predicted time: its slowest group
    double m = 0.0;
    for (int gi = 0; gi < ngroup; ++gi) m = std::max(m, cost(gi, gns[gi]));
    *t_pred = m;
  }
  return true;
}

bsde_status bsde_solve_batch(bsde_ctx* const* cs, int32_t n, bsde_result* res) {
  return bsde_solve_batch_mode(cs, n, 0, res);
}

bsde_status bsde_solve_batch_mode(bsde_ctx* const* cs, int32_t n, int32_t mode, bsde_result* res) {
  if (mode < 0 || (mode > 5 && (mode < 11 || mode > 19)))
    return set_err(nullptr, BSDE_ERR_INVALID_ARGUMENT, "batch: mode %d outside 0..5, 11..19", mode);
  if (!cs || n < 1 || n > kMaxBatch) return set_err(nullptr, BSDE_ERR_INVALID_ARGUMENT, "batch: need 1..%d contexts", kMaxBatch);
  for (int i = 0; i < n; ++i)
    if (!cs[i]) return set_err(nullptr, BSDE_ERR_INVALID_ARGUMENT, "batch: ctx %d is NULL", i);
  bsde_ctx* c0 = cs[0];
  for (int i = 0; i < n; ++i) {
    const bsde_ctx* c = cs[i];
    for (int j = 0; j < i; ++j)
      if (cs[j] == c) return set_err(c0, BSDE_ERR_INVALID_ARGUMENT, "batch: ctx %d repeated", i);
    const bool fused = c->d == 1 && (c->cfg.kernel_variant == 0 || c->cfg.kernel_variant >= 10) && c->geo.ok &&
                       c->tap1_off >= 0;
    if (!fused || c->nranks > 1 || c->grouped)
      return set_err(c0, BSDE_ERR_INVALID_ARGUMENT, "batch: ctx %d is not a one-rank d = 1 fused-kernel context", i);
    if (c->cfg.device != c0->cfg.device || c->g.P[0] != c0->g.P[0] || c->g.xlo[0] != c0->g.xlo[0] ||
        c->g.xhi[0] != c0->g.xhi[0] || c->pb.driver_id != c0->pb.driver_id)
      return set_err(c0, BSDE_ERR_INVALID_ARGUMENT, "batch: ctx %d differs in device, grid or driver", i);
    if (c->geo.fz.variant != c0->geo.fz.variant || c->geo.threads != c0->geo.threads || c->geo.blocks != c0->geo.blocks)
      return set_err(c0, BSDE_ERR_INVALID_ARGUMENT, "batch: ctx %d has another fused-kernel geometry", i);
  }
  cudaSetDevice(c0->cfg.device);
  // common geometry: the largest buffers of the batch
  Fused1D fz = c0->geo.fz;
  for (int i = 1; i < n; ++i) {
    const Fused1D& f = cs[i]->geo.fz;
    fz.WMAX = std::max(fz.WMAX, f.WMAX);
    fz.WP = std::max(fz.WP, f.WP);
    fz.WS = std::max(fz.WS, f.WS);
    fz.TK = std::max(fz.TK, f.TK);
  }
  // problem-partitioned modes (groups of problems on their own CTAs) when a plan fits, else
  // round robin.  mode 2: pairs (smallest K with largest K, ...); modes 0, 3 and 11..19: one
  // problem per group (11..19: mode - 10 tiles per CTA, ablation).  Measured on cfg 2 (K = 1..6):
  // round robin 20.9-22.2 ms, pairs 17.6-18.2 ms, one problem per group 16.9-17.2 ms.
  int group[kMaxBatch], gcta[kMaxBatch], gns[kMaxBatch], ngroup = 0, pblocks = 0;
  bool part = false;
  Fused1D fzp = fz;
  size_t smem_p = 0;
  if (mode != 1 && (n >= 2 || mode >= 2)) {
    const int TP = fz.TP, P = (int)c0->g.P[0];
    const int mb = fused1d_blocks_per_sm(fz.variant, fused1d_smem(fzp));
    // tiles per CTA: bounded by the pass-2 window (its folded end rows) and by shared memory
    int nsmax = std::max(1, std::min(9, (P - 2 * kP2Halo - 256) / (2 * TP)));
    while (nsmax > 1) {
      Fused1D t = fz;
      t.WP = ((nsmax * TP + 2 + 2 * kP2Halo + 8) + 1) & ~1;
      t.WS = 6 * t.WP + 16;
      if (fused1d_smem(t) > 0) break;
      --nsmax;
    }
    int Kv[kMaxBatch], st[kMaxBatch];
    for (int i = 0; i < n; ++i) { Kv[i] = cs[i]->K; st[i] = cs[i]->level; }
    auto pair_groups = [&]() {                       // pairs by K rank: (1st, last), (2nd, 2nd last), ...
      int idx[kMaxBatch];
      for (int i = 0; i < n; ++i) idx[i] = i;
      std::stable_sort(idx, idx + n, [&](int x, int y) { return Kv[x] < Kv[y]; });
      ngroup = 0;
      for (int r = 0; r < n; ++r) {
        const int pr = std::min(r, n - 1 - r);
        group[idx[r]] = pr;
        ngroup = std::max(ngroup, pr + 1);
      }
    };
    if (mode == 0 && n >= 4 && mb > 0) {
      // auto: pairs when the cost model predicts them faster than one problem per group (the
      // one-CTA-per-SM default leaves too few CTAs for six separate groups to balance)
      int g1[kMaxBatch], c1[kMaxBatch], s1[kMaxBatch], c2[kMaxBatch], s2[kMaxBatch];
      for (int i = 0; i < n; ++i) g1[i] = i;
      double t1 = 0.0, t2 = 0.0;
      const bool ok1 = plan_batch_groups(n, Kv, st, g1, n, c0->geo.blocks, c0->nsm * mb, nsmax, c1, s1, &t1);
      pair_groups();
      const bool ok2 = plan_batch_groups(n, Kv, st, group, ngroup, c0->geo.blocks, c0->nsm * mb, nsmax, c2, s2, &t2);
      if (!ok2 || (ok1 && t1 <= t2)) {
        for (int i = 0; i < n; ++i) group[i] = i;
        ngroup = n;
      }
    } else if (mode == 2) {
      pair_groups();
    } else if ((mode == 4 || mode == 5) && n > mode - 2) {   // the m = mode - 2 smallest K share a group
      const int m = mode - 2;
      int idx[kMaxBatch];
      for (int i = 0; i < n; ++i) idx[i] = i;
      std::stable_sort(idx, idx + n, [&](int x, int y) { return Kv[x] < Kv[y]; });
      for (int r = 0; r < n; ++r) group[idx[r]] = r < m ? 0 : r - m + 1;
      ngroup = n - m + 1;
    } else {
      for (int i = 0; i < n; ++i) group[i] = i;
      ngroup = n;
    }
    bool planned = false;
    if (mode >= 11) {
      planned = true;
      for (int gi = 0; gi < ngroup; ++gi) {
        gns[gi] = std::min(mode - 10, nsmax);
        gcta[gi] = (c0->geo.blocks + gns[gi] - 1) / gns[gi];
        gns[gi] = (c0->geo.blocks + gcta[gi] - 1) / gcta[gi];
      }
    } else {
      planned = mb > 0 && plan_batch_groups(n, Kv, st, group, ngroup, c0->geo.blocks, c0->nsm * mb, nsmax, gcta, gns);
    }
    if (planned) {
      int nsm_ = 1;
      for (int gi = 0; gi < ngroup; ++gi) { nsm_ = std::max(nsm_, gns[gi]); pblocks += gcta[gi]; }
      fzp.WP = ((nsm_ * TP + 2 + 2 * kP2Halo + 8) + 1) & ~1;   // pass-2 window of a CTA's range
      fzp.WS = 6 * fzp.WP + 16;
      smem_p = fused1d_smem(fzp);
      part = smem_p > 0 && pblocks <= c0->nsm * fused1d_blocks_per_sm(fzp.variant, smem_p) && pblocks <= kFlagCap;
    }
  }
  if (mode >= 2 && !part)
    return set_err(c0, BSDE_ERR_RESOURCE_LIMIT, "batch: no problem-partitioned plan fits (shared memory / co-residency)");
  if (part) fz = fzp;
  const size_t smem = part ? smem_p : fused1d_smem(fz);
  if (smem == 0) return set_err(c0, BSDE_ERR_RESOURCE_LIMIT, "batch: the level windows do not fit in shared memory");
  const int per_sm = fused1d_blocks_per_sm(fz.variant, smem);
  const int blocks = part ? pblocks : c0->geo.blocks;
  if (blocks > c0->nsm * per_sm)
    return set_err(c0, BSDE_ERR_RESOURCE_LIMIT, "batch: %d CTAs with %zu B of shared memory are not co-resident", blocks, smem);
  const double t0 = now_s();
  cudaEvent_t e0, e1;
  if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess)
    return set_err(c0, BSDE_ERR_CUDA, "event create");
  // order the launch after every context's queued work
  for (int i = 1; i < n; ++i)
    if (cs[i]->stream != c0->stream) {
      cudaEvent_t ev;
      cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      cudaEventRecord(ev, cs[i]->stream);
      cudaStreamWaitEvent(c0->stream, ev, 0);
      cudaEventDestroy(ev);
    }
  for (int i = 0; i < n; ++i) cudaMemsetAsync(pexec_counter(cs[i]), 0, sizeof(unsigned long long), c0->stream);
  cudaEventRecord(e0, c0->stream);
  FusedProb probs[kMaxBatch];
  int64_t steps[kMaxBatch];
  for (int i = 0; i < n; ++i) {
    bsde_ctx* c = cs[i];
    FusedProb& fp = probs[i];
    fp = FusedProb{};
    fp.s = persistent_args(c);
    fp.pp.n0 = c->level - 1;
    fp.pp.nsteps = c->level;
    fp.pp.ring_mode = 1;
    fp.pp.cur = c->cur;
    fp.pp.t0 = c->cfg.t0;
    fp.pp.dt = c->dt;
    fp.pp.vbuf[0] = c->vbuf[0];
    fp.pp.vbuf[1] = c->vbuf[1];
    fp.pp.ring_flag = c->barrier;
    if (part) {
      fp.pp.done_flag = c->barrier + kFlagCap;
      distances_for(c, gns[group[i]] * fz.TP, fp.pp.D, fp.pp.DK);
    } else {
      fp.pp.done_flag = c->barrier + c->geo.blocks;
      for (int j = 0; j <= kMaxK; ++j) fp.pp.D[j] = c->geo.D[j];
      fp.pp.DK = c->geo.DK;
    }
    for (int k = 0; k < 12; ++k) fp.dp[k] = c->pb.dp[k];
    steps[i] = c->level;
  }
  cudaError_t e = launch_fused1d_batch(probs, n, c0->g, fz, c0->pb.driver_id, c0->geo.threads, blocks, smem,
                                       c0->stream, part ? group : nullptr, part ? gcta : nullptr, part ? gns : nullptr,
                                       part ? ngroup : 0);
  cudaEventRecord(e1, c0->stream);
  if (e != cudaSuccess) {
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return set_err(c0, BSDE_ERR_CUDA, "batch kernel: %s", cudaGetErrorString(e));
  }
  for (int i = 0; i < n; ++i) {
    bsde_ctx* c = cs[i];
    ++c->launches;
    c->cur ^= (int)(steps[i] & 1);
    c->level = 0;
    if (c->stream != c0->stream) cudaStreamWaitEvent(c->stream, e1, 0);
  }
  e = cudaEventSynchronize(e1);
  float ms = 0;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (e != cudaSuccess) return set_err(c0, BSDE_ERR_CUDA, "batch kernel: %s", cudaGetErrorString(e));
  for (int i = 0; i < n; ++i) {
    bsde_status st = check_bad(cs[i]);
    if (st) return st;
    if (res) {
      double out[4] = {0, 0, 0, 0};
      if ((st = eval_point(cs[i], out))) return st;
      e = cudaStreamSynchronize(cs[i]->stream);
      if (e != cudaSuccess) return set_err(cs[i], BSDE_ERR_CUDA, "sync: %s", cudaGetErrorString(e));
      fill_result(cs[i], &res[i], out, ms * 1e-3, now_s() - t0, steps[i]);
      res[i].batch_ctas = part ? gcta[group[i]] : blocks;
      res[i].batch_tiles = part ? gns[group[i]] : 1;
      unsigned long long v = 0;
      if (cudaMemcpy(&v, pexec_counter(cs[i]), sizeof v, cudaMemcpyDeviceToHost) == cudaSuccess)
        res[i].picard_iters = (int64_t)v;
    }
  }
  return BSDE_OK;
}

bsde_status bsde_level(const bsde_ctx* c, int32_t* n_out) {
  if (!c || !n_out) return BSDE_ERR_INVALID_ARGUMENT;
  *n_out = c->level;
  return BSDE_OK;
}

bsde_status bsde_get_layer(const bsde_ctx* cc, int32_t field, double* host_dst, int64_t count) {
  bsde_ctx* c = const_cast<bsde_ctx*>(cc);
  if (!c || !host_dst) return BSDE_ERR_INVALID_ARGUMENT;
  if (field < 0 || field >= c->F) return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "field %d outside 0..%d", field, c->F - 1);
  const int64_t own = c->g.nown0 * row_len(c);
  if (count != own) return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "count %lld != %lld", (long long)count, (long long)own);
  cudaSetDevice(c->cfg.device);
  CU(cudaMemcpyAsync(host_dst, c->vbuf[c->cur] + (int64_t)field * c->g.npts + c->g.own0 * row_len(c),
                     sizeof(double) * count, cudaMemcpyDeviceToHost,
                     c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return BSDE_OK;
}

bsde_status bsde_get_picard_counts(const bsde_ctx* cc, int32_t* host_dst, int64_t count) {
  bsde_ctx* c = const_cast<bsde_ctx*>(cc);
  if (!c || !host_dst) return BSDE_ERR_INVALID_ARGUMENT;
  if (count != c->g.nown0 * row_len(c)) return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "count mismatch");
  cudaSetDevice(c->cfg.device);
  CU(cudaMemcpyAsync(host_dst, c->picard + c->g.own0 * row_len(c), sizeof(int32_t) * count, cudaMemcpyDeviceToHost,
                     c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return BSDE_OK;
}

bsde_status bsde_query_grid(const bsde_ctx* c, int64_t npts[3], double dx[3]) {
  if (!c) return BSDE_ERR_INVALID_ARGUMENT;
  for (int a = 0; a < 3; ++a) {
    npts[a] = a < c->d ? (a == 0 ? c->P0g : c->g.P[a]) : 1;
    dx[a] = a < c->d ? c->g.dx[a] : 0.0;
  }
  return BSDE_OK;
}

bsde_status bsde_query_partition(const bsde_ctx* c, int64_t* own_lo, int64_t* own_hi, int64_t* halo) {
  if (!c) return BSDE_ERR_INVALID_ARGUMENT;
  if (own_lo) *own_lo = c->r0;
  if (own_hi) *own_hi = c->r1;
  if (halo) *halo = c->halo;
  return BSDE_OK;
}

bsde_status bsde_query_partition_cfg(const bsde_config* cfg, int64_t out[5]) {
  bsde_status st = validate(cfg, nullptr);
  if (st) return st;
  bsde_ctx c;
  c.cfg = *cfg;
  c.d = cfg->d; c.F = 1 + cfg->d; c.Ky = cfg->Ky; c.Kz = cfg->Kz; c.K = std::max(cfg->Ky, cfg->Kz);
  c.L = cfg->L; c.N = cfg->N;
  c.dt = (cfg->T - cfg->t0) / cfg->N;
  fill_grid(cfg, c.g, c.dt);
  hermite_rule(c.L, c.gh_a, c.gh_w);
  build_taps(&c, c.K, c.dt, c.taps, &c.qspan, &c.qspan1);
  c.nranks = cfg->nranks > 1 ? cfg->nranks : 1;
  c.rank = c.nranks > 1 ? cfg->rank : 0;
  c.P0g = c.g.P[0];
  if ((st = plan_partition(&c))) { g_setup_error = c.err; return st; }
  out[0] = c.r0; out[1] = c.r1; out[2] = c.halo; out[3] = c.lo_e; out[4] = c.hi_e;
  return BSDE_OK;
}

bsde_status bsde_nccl_unique_id(void* out, size_t bytes) {
  if (!out || bytes < sizeof(ncclUniqueId)) return set_err(nullptr, BSDE_ERR_INVALID_ARGUMENT, "need %zu bytes", sizeof(ncclUniqueId));
  ncclUniqueId id;
  ncclResult_t nr = ncclGetUniqueId(&id);
  if (nr != ncclSuccess) return set_err(nullptr, BSDE_ERR_COMM, "ncclGetUniqueId: %s", ncclGetErrorString(nr));
  memcpy(out, &id, sizeof id);
  return BSDE_OK;
}

bsde_status bsde_group_step(bsde_ctx** cs, int32_t n) {
  if (!cs || n < 1) return set_err(nullptr, BSDE_ERR_INVALID_ARGUMENT, "empty group");
  for (int r = 0; r < n; ++r)
    if (!cs[r] || cs[r]->rank != r || cs[r]->nranks != n || (n > 1 && !cs[r]->grouped))
      return set_err(nullptr, BSDE_ERR_INVALID_ARGUMENT, "group member %d is not rank %d of %d (in-process mode)", r, r, n);
  if (n > 1 && cs[0]->spike) {
    if (cs[0]->level <= 0) return set_err(cs[0], BSDE_ERR_STATE, "already at n = 0");
    // initial levels built in bsde_setup, then the newest level: SPIKE correction across the group
    for (int slot = 0; slot <= cs[0]->RS; ++slot)
      if (cs[0]->pending & (1u << slot)) {
        bsde_status st = group_finish(cs, n, slot);
        if (st) return st;
      }
    const int slot = cs[0]->level % cs[0]->RS;
    for (int r = 0; r < n; ++r) {
      cudaSetDevice(cs[r]->cfg.device);
      cudaError_t e = build_level(cs[r], slot);
      if (e != cudaSuccess) return set_err(cs[r], BSDE_ERR_CUDA, "spline kernel: %s", cudaGetErrorString(e));
    }
    bsde_status st = group_finish(cs, n, slot);
    if (st) return st;
    for (int r = 0; r < n; ++r) {
      cs[r]->prebuilt = true;
      st = step_internal(cs[r]);
      cs[r]->prebuilt = false;
      if (st) return st;
    }
    return group_exchange(cs, n);
  }
  for (int r = 0; r < n; ++r) {
    bsde_status st = step_internal(cs[r]);
    if (st) return st;
  }
  return n > 1 ? group_exchange(cs, n) : BSDE_OK;
}

bsde_status bsde_group_solve(bsde_ctx** cs, int32_t n, bsde_result* res) {
  if (!cs || n < 1) return set_err(nullptr, BSDE_ERR_INVALID_ARGUMENT, "empty group");
  const double t0 = now_s();
  int64_t steps = 0;
  while (cs[0]->level > 0) {
    bsde_status st = bsde_group_step(cs, n);
    if (st) return st;
    ++steps;
  }
  double out[4] = {0, 0, 0, 0};
  if (n > 1 && cs[0]->spike) {                 // the newest level's corrected spline in the scratch slot
    for (int r = 0; r < n; ++r) {
      cudaSetDevice(cs[r]->cfg.device);
      cudaError_t e = build_level(cs[r], cs[r]->RS);
      if (e != cudaSuccess) return set_err(cs[r], BSDE_ERR_CUDA, "spline kernel: %s", cudaGetErrorString(e));
    }
    bsde_status st = group_finish(cs, n, cs[0]->RS);
    if (st) return st;
    for (int r = 0; r < n; ++r) cs[r]->rs_ready = true;
  }
  for (int r = 0; r < n; ++r) {
    cudaSetDevice(cs[r]->cfg.device);
    bsde_status st = check_bad(cs[r]);
    if (st == BSDE_OK) {
      double o[4];
      st = eval_point(cs[r], o);
      for (int f = 0; f < 4 && st == BSDE_OK; ++f) out[f] += o[f];
    }
    if (st) {
      for (int q = 0; q < n; ++q) cs[q]->rs_ready = false;
      return st;
    }
  }
  for (int r = 0; r < n; ++r) cs[r]->rs_ready = false;
  if (res) {
    fill_result(cs[0], res, out, 0.0, 0.0, steps);
    for (int r = 1; r < n; ++r) {                    // stage times: the slowest rank
      tcollect(cs[r]);
      res->t_spline_s = std::max(res->t_spline_s, cs[r]->t_stage[ST_SPLINE]);
      res->t_quad_s = std::max(res->t_quad_s, cs[r]->t_stage[ST_QUAD]);
      res->t_comm_s = std::max(res->t_comm_s, cs[r]->t_stage[ST_COMM]);
      cs[r]->t_stage[ST_SPLINE] = cs[r]->t_stage[ST_QUAD] = cs[r]->t_stage[ST_COMM] = 0.0;
    }
    res->y0 = out[0];
    for (int a = 0; a < cs[0]->d; ++a) res->z0[a] = out[1 + a];
    double tset = 0;
    for (int r = 0; r < n; ++r) tset = std::max(tset, cs[r]->t_setup);
    res->t_setup_s = tset;
    res->t_sweep_s = now_s() - t0;               // host clock: the group synchronises every step
    res->t_total_s = tset + res->t_sweep_s;
    int64_t pts = 0;
    for (int r = 0; r < n; ++r) pts += cs[r]->g.nown0 * row_len(cs[r]);
    res->updates = pts * steps;
    res->picard_max_used = cs[0]->cfg.picard_max;
  }
  return BSDE_OK;
}

bsde_status bsde_query_taps(const bsde_ctx* cc, int32_t level, int32_t axis, int32_t* q, double* basis4, double* w,
                            double* dw) {
  bsde_ctx* c = const_cast<bsde_ctx*>(cc);
  if (!c) return BSDE_ERR_INVALID_ARGUMENT;
  if (level < 1 || level > c->K || axis < 0 || axis >= c->d)
    return set_err(c, BSDE_ERR_INVALID_ARGUMENT, "level %d / axis %d out of range", level, axis);
  for (int l = 0; l < c->L; ++l) {
    const AxisTap& t = c->taps[((size_t)(level - 1) * c->d + axis) * c->L + l];
    if (q) q[l] = t.q;
    if (basis4) for (int k = 0; k < 4; ++k) basis4[4 * l + k] = t.B[k];
    if (w) w[l] = t.w;
    if (dw) dw[l] = t.s;
  }
  return BSDE_OK;
}

bsde_status bsde_eval(bsde_ctx* c, const double* x, double* out) {
  if (!c || !x || !out) return BSDE_ERR_INVALID_ARGUMENT;
  return bsde_eval_internal(c, x, out);
}

static bsde_status bsde_eval_internal(bsde_ctx* c, const double* x, double* out) {
  cudaSetDevice(c->cfg.device);
  if (c->spike && c->grouped)
    return set_err(c, BSDE_ERR_STATE, "bsde_eval on a SPIKE slab-group member (the spline spans the group)");
  double xx[3] = {0, 0, 0};
  for (int a = 0; a < c->d; ++a) xx[a] = x[a];
  bsde_status st = spline_into(c, c->RS);                        // newest level -> scratch slot
  if (st) return st;
  CU(c->cfg.interp == BSDE_INTERP_FD_BICUBIC
         ? launch_eval_bicubic(c->g, c->ring + (int64_t)c->RS * c->F * c->g.cfield, c->F, xx, c->dres, c->stream)
         : launch_eval(c->g, c->ring + (int64_t)c->RS * c->F * c->g.cfield, c->F, xx, c->dres, c->stream));
  ++c->launches;
  CU(cudaMemcpyAsync(out, c->dres, sizeof(double) * c->F, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return BSDE_OK;
}

bsde_status bsde_layer_device_ptr(const bsde_ctx* c, int32_t field, const double** dptr) {
  if (!c || !dptr || field < 0 || field >= c->F) return BSDE_ERR_INVALID_ARGUMENT;
  *dptr = c->vbuf[c->cur] + (int64_t)field * c->g.npts;
  return BSDE_OK;
}

bsde_status bsde_measure_fp64_peak(int32_t device, int32_t iters, double* tflops, double* ms) {
  if (!tflops || !ms || iters < 1) return set_err(nullptr, BSDE_ERR_INVALID_ARGUMENT, "fp64 peak: bad arguments");
  const cudaError_t e = measure_fp64_peak(device, iters, tflops, ms);
  if (e != cudaSuccess) return set_err(nullptr, BSDE_ERR_CUDA, "fp64 peak: %s", cudaGetErrorString(e));
  return BSDE_OK;
}

bsde_status bsde_kernel_launches(const bsde_ctx* c, int64_t* count) {
  if (!c || !count) return BSDE_ERR_INVALID_ARGUMENT;
  *count = c->launches;
  return BSDE_OK;
}

#ifdef BSDE_DEBUG
// debug build only (not in bsde.h, not in the product library): per-CTA phase stamps of the
// last fused step
int bsde_internal_phase_times(const bsde_ctx* c, unsigned long long* host, int n) {
  if (!c || !c->phase_ns) return 1;
  cudaStreamSynchronize(c->stream);
  return cudaMemcpy(host, c->phase_ns, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost) != cudaSuccess;
}
#endif

const char* bsde_last_error(const bsde_ctx* c) { return c ? c->err.c_str() : g_setup_error.c_str(); }

void bsde_destroy(bsde_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->cfg.device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  release(c);
}

}  // extern "C"
