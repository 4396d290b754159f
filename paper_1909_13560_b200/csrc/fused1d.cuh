// fused1d.cuh -- the d = 1 fused step kernel (included by kernels.cu, which owns the
// constant tap arena).  This is the hot kernel of BASELINE cfg 2.
//
// One CTA per tile of TP consecutive points (TP = 32 * NT/(32 C) * R, about P / #SMs).
// Per backward step t_{n+1} -> t_n (Eq. 20):
//  (1) the not-a-knot spline of the level-(n+1) values on the CTA's own tile is solved by
//      constant-coefficient PCR in shared memory (tile + 31-point decay halo, DESIGN.md
//      "spline"; the values arrive by cp.async.bulk) and written to the ring slot of n+1.
//  (2) levels K..1: windows of B-spline coefficients c[lo+q_min-1 .. hi+q_max+2] are
//      streamed from the ring by cp.async.bulk (one elected thread, mbarrier completion),
//      double-buffered against the computation of the previous level.
//  (3) each warp owns one chunk of Gauss-Hermite nodes (lambda = chunk, chunk + C, ...) and
//      each lane R consecutive points (odd R: conflict-free 8-byte smem access); every
//      lane of a warp reads the same tap (q, B, weights) from constant memory
//      (the translation-invariant stencil of PAPER.md:391-392).
//  (4) the C partial sums per point are reduced in a fixed order in smem and the
//      epilogue (z explicit, y by Picard, Eq. 20) writes level n.
// All CTAs of a launch are co-resident (cooperative launch) and synchronise with their
// neighbours only, through per-CTA progress flags; bsde_solve runs all remaining steps in
// one launch (persistent), bsde_step one step per launch.  Levels are processed K..1 so the
// wait for the neighbours' level-(n+1) coefficients is hidden behind levels K..2.
#pragma once
#include <type_traits>

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
}
// bulk shared -> global copy (bulk-group completion)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void bulk_wait() { asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory"); }
template <int N> __device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(smem_addr(bar)), "r"(phase) : "memory");
  } while (!done);
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// per-CTA phase stamps: a debug build only (-DBSDE_DEBUG); the product library compiles them out
#ifdef BSDE_DEBUG
#define PHASE_STAMP(i)                                                                          \
  do {                                                                                          \
    if (s.phase_ns != nullptr && threadIdx.x == 0)                                              \
      s.phase_ns[((size_t)it_stamp * gridDim.x + blockIdx.x) * 32 + (i)] = gtimer();              \
  } while (0)
#define DBG_FLAG(x) (x)
#else
#define PHASE_STAMP(i) do { (void)it_stamp; } while (0)
#define DBG_FLAG(x) 0
#endif
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// span [wv, we] (storage indices, wv even) of the window of a level whose node offsets
// are [qmin, qmax], for the tile [lo, hi): cells lo+qmin .. hi-1+qmax, 4 coefficients each
__device__ __forceinline__ void level_span(int qmin, int qmax, int lo, int hi, int& wv, int& we) {
  const int a = lo + qmin;
  wv = a - (a & 1);
  we = hi - 1 + qmax + 3;
}

// shared-memory header: 4 mbarriers @0, the flag marks @64, the window spans @256, the
// problems' parameters @1024
constexpr int kFusedHdr = (int)((1024 + kMaxBatch * sizeof(FusedProb) + 127) & ~(size_t)127);
// rhs_tilde (kernels.cu) for the rows near the line ends that the fused kernel's PCR extent
// reaches (|k| and |k - P| below the 2 (P - 3) period): the same odd extension, folded
// without a 64-bit modulo
__device__ __forceinline__ double rhs_fold(const double* F, int P, int k, double m1, double mP2) {
  const int period = 2 * (P - 3);
  int u = k - 1;
  if (u < 0) u += period;
  if (u >= period) u -= period;
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

// Persist1D, FusedProb: bsde_internal.h
struct FusedBatch {
  Fused1D fz;
  Grid g;
  const unsigned char* arena;   // global address of the constant tap arena (bulk-copy source)
  int nprob, max_steps;
  FusedProb prob[kMaxBatch];
  // problem-partitioned mode (part = 1): the problems form groups (contiguous in prob[]); the
  // CTAs [gcta0[g], gcta0[g+1]) serve group g's problems [gp0[g], gp0[g+1]) round robin, each
  // CTA a range of gns[g] consecutive tiles of TP points (sub-tiles of pass 1) whose spline is
  // built in one pass 2; round-robin mode (part = 0): every CTA serves every problem on one tile
  int part, ngroup;
  int gp0[kMaxBatch + 1], gcta0[kMaxBatch + 1];
  int gns[kMaxBatch];
};

__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// warp 0 waits until flag[b'] >= target for all CTAs b' within distance D of b (one lane per
// flag, so a satisfied wait costs one round trip); returns the smallest value it observed
// (warp-uniform), a lower bound of every flag in the range from then on (flags only grow)
__device__ __forceinline__ unsigned wait_neighbours_warp(const unsigned* flag, int b, int D, int nb, unsigned target) {
  const int lane = threadIdx.x & 31;
  const int a = max(0, b - D), e = min(nb - 1, b + D);
  unsigned seen = 0xffffffffu;
  for (int q0 = a; q0 <= e; q0 += 32) {
    const int q = q0 + lane;
    // first an acquire read (one round trip when the flags are already set), then relaxed
    // polling (no L1 invalidation) and a final acquire
    unsigned v = q <= e ? ld_acquire(flag + q) : 0xffffffffu;
    if (!__all_sync(0xffffffffu, v >= target)) {
      bool ok = v >= target;
      while (!__all_sync(0xffffffffu, ok)) {
        __nanosleep(32);
        if (!ok) ok = ld_relaxed(flag + q) >= target;
      }
      v = q <= e ? ld_acquire(flag + q) : 0xffffffffu;   // synchronises with the release
    }
    seen = min(seen, __reduce_min_sync(0xffffffffu, v));
  }
  __syncwarp();
  if (lane == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
  return seen;
}

// Progress marks of a problem's neighbour flags (shared memory, touched by one warp at a time):
// mk[0] = a lower bound of the flags within the short distance Dn of that flag kind (ring
// flags: D[1], the newest level's window; done flags: D[0], the values halo), mk[1] = a lower
// bound within DK.  Flags only grow, so a wait whose target is covered costs nothing.
__device__ __forceinline__ void wait_flags(const unsigned* flag, unsigned* mk, int b, int D, int DK, int nb,
                                           unsigned target) {
  if (mk[1] >= target || (D < DK && mk[0] >= target)) return;
  const unsigned seen = wait_neighbours_warp(flag, b, D, nb, target);
  if ((threadIdx.x & 31) == 0) {
    if (D >= DK) mk[1] = seen;
    mk[0] = max(mk[0], seen);          // every short-range wait of a kind uses that kind's Dn <= D
  }
  __syncwarp();
}

// warp 0: one read of every problem's flags of one kind within DK, raising the marks; a
// problem whose DK range is wider than a warp keeps its marks (its waits poll).  The loads
// are relaxed so that all problems' reads are in flight together (a chain of acquire loads
// would cost one round trip each); one acquire fence afterwards orders every later access
// of the CTA (after the barrier that follows) behind them.
template <int KIND>   // 0: ring flags (short range D[1]), 1: done flags (short range D[0])
__device__ __forceinline__ void refresh_marks(const FusedProb* prob, int nprob, int it, unsigned* marks, int b, int nb,
                                              int pf, int pl) {
  const int lane = threadIdx.x & 31;
  unsigned v[kMaxBatch];
#pragma unroll
  for (int ip = 0; ip < kMaxBatch; ++ip) {
    v[ip] = 0xffffffffu;
    if (ip < nprob && it < prob[ip].pp.nsteps && ip >= pf && ip < pl) {
      const Persist1D& pp = prob[ip].pp;
      const int q = b - pp.DK + lane;
      if (2 * pp.DK + 1 <= 32 && lane <= 2 * pp.DK && q >= 0 && q < nb)
        v[ip] = ld_relaxed((KIND ? pp.done_flag : pp.ring_flag) + q);
    }
  }
#pragma unroll
  for (int ip = 0; ip < kMaxBatch; ++ip) {
    if (ip >= nprob || it >= prob[ip].pp.nsteps || 2 * prob[ip].pp.DK + 1 > 32 || ip < pf || ip >= pl) continue;
    const Persist1D& pp = prob[ip].pp;
    const int Dn = KIND ? pp.D[0] : pp.D[1];
    const int d = lane - pp.DK;
    const unsigned mK = __reduce_min_sync(0xffffffffu, v[ip]);
    const unsigned mN = __reduce_min_sync(0xffffffffu, (d >= -Dn && d <= Dn) ? v[ip] : 0xffffffffu);
    if (lane == 0) {
      unsigned* mk = marks + 4 * ip + 2 * KIND;
      mk[0] = max(mk[0], mN);
      mk[1] = max(mk[1], mK);
    }
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  __syncwarp();
  if (lane == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ring slot of level n+j (j = 1..K) of a problem at round it
__device__ __forceinline__ int level_slot(const FusedProb& fp, int it, int j) {
  return fp.pp.ring_mode ? (fp.pp.n0 - it + j) % fp.s.ring_slots : fp.s.slot[j - 1];
}

// bulk-load the window of level j of problem fp into dst (lane 0 of the calling warp): the
// whole window [wv, we] (the virtual boundary entries live in the line's pads, Grid::cpad),
// even-aligned for the bulk copy
__device__ __forceinline__ void issue_window(const FusedProb& fp, const int* sp, int it, int j, double* dst, int WM,
                                             uint64_t* bar, int lo, int hi) {
  if ((threadIdx.x & 31) != 0) return;
  int wv, we;
  level_span(sp[2 * (j - 1)], sp[2 * (j - 1) + 1], lo, hi, wv, we);
  const int s1 = (we + 2) & ~1;
  const uint32_t bytes = (uint32_t)((s1 - wv) * sizeof(double));
  const double* Cf = fp.s.ring + (int64_t)level_slot(fp, it, j) * fp.s.slot_elems;
  // the flags may have been acquired by another warp (before a CTA barrier): order this
  // thread's async-proxy reads behind them
  asm volatile("fence.proxy.async.global;" ::: "memory");
  mbar_expect_tx(bar, 2 * bytes);
  bulk_g2s(dst, Cf + wv, bytes, bar);
  bulk_g2s(dst + WM, Cf + fp.s.cfield + wv, bytes, bar);
}

// Level n+j was written by pass 2 of round it-j by the CTAs within D[j]: levels >= 2 are
// covered by the ring flags of round it-2 within DK, level 1 needs round it-1 within D[1].
__device__ __forceinline__ void ring_wait(const FusedProb& fp, unsigned* mk, int it, int j, int bid, int nb) {
  if (it == 0 || DBG_FLAG(fp.pp.nowait)) return;
  const Persist1D& pp = fp.pp;
  if (j == 1) wait_flags(pp.ring_flag, mk, bid, pp.D[1], pp.DK, nb, (unsigned)it);
  else if (it >= 2) wait_flags(pp.ring_flag, mk, bid, pp.DK, pp.DK, nb, (unsigned)(it - 1));
}

// the first one or two windows of a problem's step it (levels K and K-1 into buffers 0 and 1;
// warp 0), skipping the `have` already in flight
__device__ __forceinline__ void start_windows(const FusedProb& fp, const int* sp, unsigned* mk, int it, int have,
                                              double* buf0, double* buf1, int WM, uint64_t* bar, int lo, int hi,
                                              int bid, int nb) {
  const int K = fp.s.K;
  for (int w = have; w < min(2, K); ++w) {
    ring_wait(fp, mk, it, K - w, bid, nb);
    issue_window(fp, sp, it, K - w, w ? buf1 : buf0, WM, &bar[w], lo, hi);
  }
}

// the problem's Tap1D table (K x L) from the arena into shared memory (lane 0 of warp 0)
__device__ __forceinline__ void issue_taps(const FusedProb& fp, const unsigned char* arena, Tap1D* dst, uint64_t* bar) {
  if ((threadIdx.x & 31) != 0) return;
  const uint32_t bytes = (uint32_t)(((size_t)fp.s.K * fp.s.L * sizeof(Tap1D) + 15) & ~(size_t)15);
  mbar_expect_tx(bar, bytes);
  bulk_g2s(dst, arena + fp.s.tap1_off, bytes, bar);
}

// the same for step it of a problem issued one round early (at the end of pass 1 of round
// it-1, streaming in during pass 2): only levels >= 2, whose ring data is from round it-2 or
// older (level 1 is written by that pass 2); returns the number of windows issued
__device__ __forceinline__ int start_windows_ahead(const FusedProb& fp, const int* sp, unsigned* mk, int it,
                                                   double* buf0, double* buf1, int WM, uint64_t* bar, int lo, int hi,
                                                   int bid, int nb) {
  const int K = fp.s.K;
  int w = 0;
  for (; w < 2 && K - w >= 2; ++w) {
    ring_wait(fp, mk, it, K - w, bid, nb);
    issue_window(fp, sp, it, K - w, w ? buf1 : buf0, WM, &bar[w], lo, hi);
  }
  return w;
}

template <int DRV, int R, int C, int NT, int MB>
__global__ void __launch_bounds__(NT, MB) quad1d_fused(const __grid_constant__ FusedBatch bt) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // 0/1: level buffers (full), 2: values tile, 3: taps, 4/5: level buffers released by every warp
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  const Fused1D& fz = bt.fz;
  const Grid& g = bt.g;
  const int WM = fz.WMAX, WP = fz.WP;
  double* const buf0 = reinterpret_cast<double*>(smem_raw + kFusedHdr);
  double* const buf1 = buf0 + 2 * WM;
  // spline scratch of pass 2: values window Fs (2 x (WP + 8)) and the PCR arrays T0, T1
  // (2 x WP each), behind the level buffers (fz.sep) or overlaying them (free after the
  // epilogue)
  double* const Fs = buf0 + (fz.sep ? 4 * WM : 0);
  // the current problem's tap table (bulk-copied one problem ahead) and window spans
  Tap1D* const tsm = reinterpret_cast<Tap1D*>(buf0 + 4 * WM + (fz.sep ? fz.WS : 0));
  int* const spans = reinterpret_cast<int*>(smem_raw + 256);     // [problem][level][qmin, qmax]
  FusedProb* const PB = reinterpret_cast<FusedProb*>(smem_raw + 1024);
  double* const T0 = Fs + 2 * (WP + 8);
  double* const T1 = T0 + 2 * WP;
  constexpr int NWPG = NT / (32 * C);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int chunk = warp / NWPG, pg = warp % NWPG;
  const int P = (int)g.P[0];
  const int TP = fz.TP;
  // this CTA: its problems [pf, pl) (part mode: its group's; else every problem), its index bid
  // among the nb CTAs that serve them (the index of its progress flags), its range [clo, chi) of
  // nsub tiles
  int pf = 0, pl = bt.nprob, bid = blockIdx.x, nb = gridDim.x, nsub = 1;
  if (bt.part) {
    int gi = 0;
    while (gi + 1 < bt.ngroup && (int)blockIdx.x >= bt.gcta0[gi + 1]) ++gi;
    pf = bt.gp0[gi];
    pl = bt.gp0[gi + 1];
    bid = blockIdx.x - bt.gcta0[gi];
    nb = bt.gcta0[gi + 1] - bt.gcta0[gi];
    nsub = bt.gns[gi];
  }
  const int clo = bid * nsub * TP;
  const int chi = min(clo + nsub * TP, P);
  const int nunit_sub = (chi - clo + TP - 1) / TP;   // non-empty tiles of the range
  int lo = clo;                                      // the current tile [lo, hi) (pass 1)
  int hi = min(lo + TP, chi);
  const int li0 = (pg * 32 + lane) * R;              // first local point of this lane
  bool active = lo + li0 < hi;
  // coefficients this CTA owns (c indices k = storage - 1) and the pass-2 window around them:
  // the globally aligned segments [sa, sb] of kP2Seg rows, kP2Q beyond the outputs on each side
  const int k0 = clo == 0 ? -1 : clo, k1 = chi == P ? P + 1 : chi;
  auto fdiv = [](int x) { return x >= 0 ? x / kP2Seg : -((-x + kP2Seg - 1) / kP2Seg); };
  const int sa = fdiv(k0) - kP2Q, sb = fdiv(k1 - 1) + kP2Q;
  const int base = sa * kP2Seg;
  const int Wa = (sb - sa + 1) * kP2Seg;
  // values window [va, vb] of both fields (clamped to the grid); the grid is long enough
  // (fused1d_geometry) that every folded index of the odd extension lands inside it
  const int va = max(base - 3, 0), vb = min(base + Wa + 2, P - 1);
  const int va0 = va & ~1;                                   // field 0 start, even
  const int va1 = (int)((((int64_t)P + va) & ~(int64_t)1) - P);  // field 1 start (P + va1 even)
  const int publisher = NT - 32;  // thread that releases the flags (the last warp pays the fence)

  // progress marks of the neighbours' flags, 4 per problem: ring (short range, DK), done
  // (short range, DK); see wait_flags
  unsigned* const marks = reinterpret_cast<unsigned*>(smem_raw + 64);
  unsigned long long* const pcnt = reinterpret_cast<unsigned long long*>(smem_raw + 192);   // per problem
  if (tid < kMaxBatch) pcnt[tid] = 0;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    mbar_init(&bar[3], 1);
    mbar_init(&bar[4], NT / 32);
    mbar_init(&bar[5], NT / 32);
    fence_mbar_init();
    for (int i = 0; i < 4 * kMaxBatch; ++i) marks[i] = 0;
  }
  // the problems' parameters in shared memory (indexed accesses to the kernel parameter
  // would go through the small constant cache)
  {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(bt.prob);
    uint32_t* dst = reinterpret_cast<uint32_t*>(PB);
    for (int i = tid; i < bt.nprob * (int)(sizeof(FusedProb) / 4); i += NT) dst[i] = src[i];
  }
  for (int i = tid; i < bt.nprob * kMaxK; i += NT) {
    const FusedProb& fp = bt.prob[i / kMaxK];
    const int j = i % kMaxK;
    if (j < fp.s.K) {
      const Tap1D* tj = taps1d(fp.s.tap1_off) + j * fp.s.L;
      spans[2 * i] = tj[0].q;
      spans[2 * i + 1] = tj[fp.s.L - 1].q;
    }
  }
  grid_dep_wait();            // previous kernel in the stream has completed
  __syncthreads();
  uint32_t ph[6] = {0, 0, 0, 0, 0, 0};
  unsigned pexec = 0;         // Picard iterations this thread executed (current problem-step, or the launch)
  unsigned pexec1 = 0;        // ... for the CTA's second problem (pairs: no shared-memory atomics per unit)
  int prefetched = 0;         // windows of the current problem already in flight
  // the warp that issues the next problem's copies during the epilogue: the last warp, which has
  // the fewest epilogue points (none when TP <= NT - 32; (r2) one per lane instead of two in the
  // 12-warp default), not warp 0 with its flag waits.  It touches the flag marks only between CTA
  // barriers that separate it from warp 0's waits.
  const int iw = NT / 32 - 1;
  bool taps_in = false;       // its tap table is in flight
  // work units of a round: round-robin mode one per problem (the CTA's tile), part mode one per
  // tile of the CTA's range (its one problem)
  // (problem-major: every tile of a problem, then the next problem of the group)
  const int nunits = (pl - pf) * nunit_sub;
  int it_end = 0;
  for (int ip = pf; ip < pl; ++ip) it_end = max(it_end, PB[ip].pp.nsteps);
  auto unit_prob = [&](int u) { return pf + u / nunit_sub; };
  auto unit_lo = [&](int u) { return clo + (u % nunit_sub) * TP; };

  const bool multi = pl - pf > 1;
  for (int it = 0; it < it_end; ++it) {
#ifdef BSDE_DEBUG
    for (int ip = pf; ip < pl; ++ip) {   // round start of every problem of the group (debug timeline)
      const int it_stamp = it;
      const StepArgs& s = PB[ip].s;
      PHASE_STAMP(20);
    }
#endif
    // ================= pass 1: levels K..1, z and Picard of step it of every problem / tile
    // one relaxed read of every problem's flags + one acquire fence serve all problems' waits of
    // the pass; a CTA with a single problem waits with per-flag acquire loads instead (no fence)
    if (warp == 0 && it > 0 && multi) refresh_marks<0>(PB, bt.nprob, it, marks, bid, nb, pf, pl);
    for (int un = 0; un < nunits; ++un) {
      const int ip = unit_prob(un);
      const FusedProb& fp = PB[ip];
      const Persist1D& pp = fp.pp;
      if (it >= pp.nsteps) continue;
      lo = unit_lo(un);
      hi = min(lo + TP, chi);
      active = lo + li0 < hi;
      const StepArgs& s = fp.s;
      const int it_stamp = it;
      PHASE_STAMP(0);
      const int L = s.L, K = s.K;
      const Tap1D* const tap0 = tsm;
      const int* const sp = spans + 2 * kMaxK * ip;
      double tlev[kMaxK];
      double tn;
      double* vout;
      if (pp.ring_mode) {
        const int n = pp.n0 - it;
#pragma unroll
        for (int j = 1; j <= kMaxK; ++j) tlev[j - 1] = pp.t0 + (n + j) * pp.dt;
        tn = pp.t0 + n * pp.dt;
        vout = pp.vbuf[(pp.cur + it + 1) & 1];
      } else {
#pragma unroll
        for (int j = 0; j < kMaxK; ++j) tlev[j] = s.t_level[j];
        tn = s.tn;
        vout = s.values;
      }
      // windows of levels K and K-1 (unless prefetched during the previous problem's
      // epilogue); later levels are issued behind the computation.  (No CTA barrier here:
      // the previous pass ended with one; the other warps wait on the mbarriers.)
      if (warp == 0) {
        if (!taps_in) issue_taps(fp, bt.arena, tsm, &bar[3]);
        start_windows(fp, spans + 2 * kMaxK * ip, marks + 4 * ip, it, prefetched, buf0, buf1, WM, bar, lo, hi, bid,
                      nb);
      }
      prefetched = 0;
      taps_in = false;
      mbar_wait(&bar[3], ph[3]);
      ph[3] ^= 1u;
      PHASE_STAMP(1);

      Driver<DRV, 1> drv(fp.dp);
      double Az[R], Af[R], Ay[R];
#pragma unroll
      for (int r = 0; r < R; ++r) { Az[r] = 0.0; Af[r] = 0.0; Ay[r] = 0.0; }
      // one level of taps on the window in buffer b.  The window spans storage indices
      // [wv, we] (wv even); entries outside the real range [0, P+2] are filled with the
      // clamped boundary values F_0 / F_{P-1}, so every tap uses the same
      // 4-term B-spline stencil; the cells whose stencil straddles the boundary
      // ([-3, -1] and [P-1, P+2]) are clamped cells and get the boundary value directly.
      auto level = [&](int j, int b) {
        const Tap1D* tj = tap0 + (j - 1) * L;
        int wv, we;
        level_span(sp[2 * (j - 1)], sp[2 * (j - 1) + 1], lo, hi, wv, we);
        mbar_wait(&bar[b], ph[b]);
        ph[b] ^= 1u;
        double* const wy = b ? buf1 : buf0;
        double* const wz = wy + WM;
        // clamped boundary values s(x_0) = (c_{-1} + 4 c_0 + c_1)/6 and s(x_{P-1}): the
        // virtual entries of the window (from the line's pads)
        const bool left = wv < 0, right = we > P + 2;
        const double fy0 = left ? wy[0] : 0.0, fz0 = left ? wz[0] : 0.0;
        const double fy1 = right ? wy[we - wv] : 0.0, fz1 = right ? wz[we - wv] : 0.0;
        drv.at(tlev[j - 1]);
        const bool yj = (j == s.Ky);
        const int cl0 = lo + li0;                      // lane's first point
        // ... relative to the window (q = 0); a lane past a ragged tile's end reads the tile's
        // first point's stencils instead (its sums are never stored), so the tap loop has no
        // per-lane branch
        const int rel0 = (active ? cl0 : lo) - wv;
        // EDGE: the tile's stencils may straddle the box boundary (edge CTAs only); YJ: this
        // level also feeds E[y^{n+Ky}].  Specialised so that the interior tap loop is
        // branch-free and consecutive taps interleave.
        auto tap_loop = [&](auto edge_c, auto yj_c) {
          constexpr bool EDGE = decltype(edge_c)::value;
          constexpr bool YJ = decltype(yj_c)::value;
#pragma unroll 2
          for (int l = chunk; l < L; l += C) {
            const Tap1D& t = tj[l];
            const int q = t.q;
            double yh[R], zh[R];
            {
              // the R 4-term stencils of consecutive points, coefficient-major: every loaded
              // coefficient feeds up to 4 independent FMA chains at once (y and z interleaved), so
              // few registers stay live and the chains overlap
              const double* py = wy + (rel0 + q);
              const double* pz = wz + (rel0 + q);
              const double B0 = t.B[0], B1 = t.B[1], B2 = t.B[2], B3 = t.B[3];
#pragma unroll
              for (int k = 0; k < R + 3; ++k) {
                const double cy = py[k], cz = pz[k];
                if (k < R) { yh[k] = B0 * cy; zh[k] = B0 * cz; }
                if (k - 1 >= 0 && k - 1 < R) { yh[k - 1] = fma(B1, cy, yh[k - 1]); zh[k - 1] = fma(B1, cz, zh[k - 1]); }
                if (k - 2 >= 0 && k - 2 < R) { yh[k - 2] = fma(B2, cy, yh[k - 2]); zh[k - 2] = fma(B2, cz, zh[k - 2]); }
                if (k - 3 >= 0 && k - 3 < R) { yh[k - 3] = fma(B3, cy, yh[k - 3]); zh[k - 3] = fma(B3, cz, zh[k - 3]); }
              }
            }
            if (EDGE) {
              const int cb = cl0 + q, ce = cb + R - 1;     // lane's cells
              if ((left && cb <= -1 && ce >= -3) || (right && cb <= P + 2 && ce >= P - 1)) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                  const int cell = cb + r;
                  if (cell >= -3 && cell <= -1) { yh[r] = fy0; zh[r] = fz0; }
                  if (cell >= P - 1 && cell <= P + 2) { yh[r] = fy1; zh[r] = fz1; }
                }
              }
            }
            const double wcz = t.wcz, wgz = t.wgz, wgy = t.wgy;
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const double f = drv(yh[r], &zh[r]);
              Az[r] = fma(wcz, zh[r], fma(wgz, f, Az[r]));
              Af[r] = fma(wgy, f, Af[r]);
            }
            if (YJ) {
              const double wy_ = t.wy;
#pragma unroll
              for (int r = 0; r < R; ++r) Ay[r] = fma(wy_, yh[r], Ay[r]);
            }
          }
        };
        using T_ = std::true_type;
        using F_ = std::false_type;
        if (left || right) { if (yj) tap_loop(T_{}, T_{}); else tap_loop(T_{}, F_{}); }
        else { if (yj) tap_loop(F_{}, T_{}); else tap_loop(F_{}, F_{}); }
      };

      // levels K, ..., 1, double-buffered: level j-2 streams in while level j is computed
      for (int j = K; j >= 1; --j) {
        const int b = (K - j) & 1;
        level(j, b);
        if (j <= 6) PHASE_STAMP(1 + j);
        if (j - 2 >= 1) {                     // refill this buffer with level j-2
          // (r2) every warp releases the buffer on an mbarrier and goes on to level j-1; only warp 0
          // waits for all of them before it issues the copy (no CTA barrier per level)
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&bar[4 + b]);
          if (warp == 0) {
            mbar_wait(&bar[4 + b], ph[4 + b]);
            ph[4 + b] ^= 1u;
            if (j - 2 == 1) ring_wait(fp, marks + 4 * ip, it, 1, bid, nb);
            issue_window(fp, sp, it, j - 2, b ? buf1 : buf0, WM, &bar[b], lo, hi);
          }
        }
      }
      // reduction over node chunks (fixed order) and epilogue.  (r2) With a separate spline scratch
      // large enough (idle in pass 1) the partial sums go there: the level buffers need no barrier
      // of their own before the next unit's copies (one CTA barrier less per tile)
      const bool red_sep = fz.sep && fz.WS >= 3 * C * TP;
      if (!red_sep) __syncthreads();
      else asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      double* red = red_sep ? Fs : buf0;
      if (active) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          double* q = red + (chunk * TP + li0 + r) * 3;
          q[0] = Az[r];
          q[1] = Af[r];
          q[2] = Ay[r];
        }
      }
      __syncthreads();
      PHASE_STAMP(8);
      // the sums of this thread's points (TP = 32 NWPG R <= U NT, U = ceil(R / C)) into registers, so
      // the level buffers are free during the epilogue
      constexpr int U = (R + C - 1) / C;
      double az[U], af[U], ay[U];
#pragma unroll
      for (int u = 0; u < U; ++u) { az[u] = 0.0; af[u] = 0.0; ay[u] = 0.0; }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int t = tid + u * NT;
        if (t < hi - lo) {
#pragma unroll
          for (int c = 0; c < C; ++c) {
            const double* q = red + (c * TP + t) * 3;
            az[u] += q[0];
            af[u] += q[1];
            ay[u] += q[2];
          }
        }
      }
      // the next problem's first windows stream in during this epilogue
      if (!red_sep) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
      }
      PHASE_STAMP(16);
      {
        // the next unit of this round (next problem, or next tile of the range)
        int uq = un + 1;
        while (uq < nunits && it >= PB[unit_prob(uq)].pp.nsteps) ++uq;
        if (uq < nunits) {
          const int iq = unit_prob(uq);
          const int lq = unit_lo(uq), hq = min(lq + TP, chi);
          if (warp == iw) {
            issue_taps(PB[iq], bt.arena, tsm, &bar[3]);
            start_windows(PB[iq], spans + 2 * kMaxK * iq, marks + 4 * iq, it, 0, buf0, buf1, WM, bar, lq, hq,
                          bid, nb);
          }
          prefetched = 2;
          taps_in = true;
        } else {
          // last unit of the round: the tap table of the first unit of the next round (with a
          // separate spline scratch its windows of levels >= 2 follow at the start of pass 2,
          // off the critical path of this epilogue)
          uq = 0;
          while (uq < nunits && it + 1 >= PB[unit_prob(uq)].pp.nsteps) ++uq;
          if (uq < nunits) {
            const int iq = unit_prob(uq);
            if (warp == iw) issue_taps(PB[iq], bt.arena, tsm, &bar[3]);
            prefetched = fz.sep ? min(2, max(0, PB[iq].s.K - 1)) : 0;   // what pass 2 issues
            taps_in = true;
          }
        }
      }
      PHASE_STAMP(17);
      const double inv_gz0 = 1.0 / s.gz0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int t = tid + u * NT;
        if (t >= hi - lo) continue;
        // z: Eq. 20 line 2 (explicit); y: Eq. 20 line 1 by Picard from E[y^{n+Ky}]
        Driver<DRV, 1> dn(fp.dp);
        dn.at(tn);
        const double z = az[u] * inv_gz0;
        const double rhs = fma(s.ky_dt, af[u], ay[u]);
        int itp;
        const double y = picard_solve([&](double v) { return dn(v, &z); }, ay[u], rhs, s.ky_dt_gy0, s.picard_max,
                                      s.picard_tol, itp, pexec);
        const int p = lo + t;
        vout[p] = y;
        vout[P + p] = z;
        s.picard[p] = itp;
        if (!isfinite(y) || !isfinite(z)) atomicMin(s.bad, bad_key(pp.ring_mode ? pp.n0 - it : s.n, p));
      }
      PHASE_STAMP(18);
      if (multi && ip != pf) {   // executed Picard iterations per problem (the roofline's executed work):
                                 // the CTA's first two problems count in registers and flush once at
                                 // the end, any further one per unit
        if (ip == pf + 1) {
          pexec1 += pexec;
        } else {
          const unsigned ex = __reduce_add_sync(0xffffffffu, pexec);
          if (lane == 0 && ex) atomicAdd(pcnt + ip, (unsigned long long)ex);
        }
        pexec = 0;
      }
      // generic-proxy accesses of the level buffers before later bulk copies into them
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      PHASE_STAMP(9);
      // the problem's level n is complete on this CTA after its last unit
      if (tid == publisher && un % nunit_sub == nunit_sub - 1) st_release(pp.done_flag + bid, (unsigned)it + 1);
    }

    // ================= pass 2: spline of every problem's new level n on this CTA's tile
    if (fz.sep && warp == iw && iw != 0) {
      // the next round's first unit: its windows of levels >= 2 (ring data of round it-1 or
      // older) stream into the level buffers during this pass (ring marks only: warp 0 touches
      // the done marks)
      int uq = 0;
      while (uq < nunits && it + 1 >= PB[unit_prob(uq)].pp.nsteps) ++uq;
      if (uq < nunits) {
        const int iq = unit_prob(uq);
        const int lq = unit_lo(uq), hq = min(lq + TP, chi);
        start_windows_ahead(PB[iq], spans + 2 * kMaxK * iq, marks + 4 * iq, it + 1, buf0, buf1, WM, bar, lq, hq, bid,
                            nb);
      }
    }
    if (warp == 0) {
      if (multi) refresh_marks<1>(PB, bt.nprob, it, marks, bid, nb, pf, pl);
      if (fz.sep && iw == 0) {      // no point-free warp: warp 0 issues the windows itself
        int uq = 0;
        while (uq < nunits && it + 1 >= PB[unit_prob(uq)].pp.nsteps) ++uq;
        if (uq < nunits) {
          const int iq = unit_prob(uq);
          const int lq = unit_lo(uq), hq = min(lq + TP, chi);
          start_windows_ahead(PB[iq], spans + 2 * kMaxK * iq, marks + 4 * iq, it + 1, buf0, buf1, WM, bar, lq, hq,
                              bid, nb);
        }
      }
    }
    for (int ip = 0; ip < bt.nprob; ++ip) {
      const FusedProb& fp = PB[ip];
      const Persist1D& pp = fp.pp;
      if (it >= pp.nsteps || ip < pf || ip >= pl) continue;
      const StepArgs& s = fp.s;
      const int it_stamp = it;
      int slot_out;
      const double* vn;
      if (pp.ring_mode) {
        slot_out = (pp.n0 - it) % s.ring_slots;
        vn = pp.vbuf[(pp.cur + it + 1) & 1];
      } else {
        slot_out = s.slot_out;
        vn = s.values;
      }
      if (slot_out < 0) continue;
      PHASE_STAMP(10);
      // the CTAs within D[0] wrote their level-n values (done flag it+1); the CTAs within DK
      // finished pass 1 of round it-2, the last reader of ring slot n (level n + K + 2)
      if (warp == 0 && !DBG_FLAG(pp.nowait)) {
        unsigned* mk = marks + 4 * ip + 2;
        if (it >= 2) wait_flags(pp.done_flag, mk, bid, pp.DK, pp.DK, nb, (unsigned)(it - 1));
        wait_flags(pp.done_flag, mk, bid, pp.D[0], pp.DK, nb, (unsigned)it + 1);
      }
      __syncthreads();
      PHASE_STAMP(11);
      if (tid == 0) {
        const uint32_t n0b = (uint32_t)((((vb + 1 - va0) + 1) & ~1) * sizeof(double));
        const uint32_t n1b = (uint32_t)((((vb + 1 - va1) + 1) & ~1) * sizeof(double));
        mbar_expect_tx(&bar[2], n0b + n1b);
        bulk_g2s(Fs, vn + va0, n0b, &bar[2]);
        bulk_g2s(Fs + (WP + 8), vn + ((int64_t)P + va1), n1b, &bar[2]);
      }
      const double* Fw0 = Fs - va0;                 // Fw[k] = F[k] for k in [va, vb]
      const double* Fw1 = Fs + (WP + 8) - va1;
      mbar_wait(&bar[2], ph[2]);
      ph[2] ^= 1u;
      PHASE_STAMP(12);
      // m_1 and m_{P-2} (not-a-knot end rows), only where the window reaches the ends
      double m1_0 = 0.0, m1_1 = 0.0, mP2_0 = 0.0, mP2_1 = 0.0;
      if (va == 0) {
        m1_0 = Fw0[0] - 2.0 * Fw0[1] + Fw0[2];
        m1_1 = Fw1[0] - 2.0 * Fw1[1] + Fw1[2];
      }
      if (vb == P - 1) {
        mP2_0 = Fw0[P - 3] - 2.0 * Fw0[P - 2] + Fw0[P - 1];
        mP2_1 = Fw1[P - 3] - 2.0 * Fw1[P - 2] + Fw1[P - 1];
      }
      for (int p = tid; p < Wa; p += NT) {
        const int k = base + p;
        double r0, r1;
        if (k >= 2 && k <= P - 3) {
          r0 = 6.0 * (Fw0[k - 1] - 2.0 * Fw0[k] + Fw0[k + 1]);
          r1 = 6.0 * (Fw1[k - 1] - 2.0 * Fw1[k] + Fw1[k + 1]);
          if (k == 2) { r0 -= m1_0; r1 -= m1_1; }
          if (k == P - 3) { r0 -= mP2_0; r1 -= mP2_1; }
        } else {
          r0 = rhs_fold(Fw0, P, k, m1_0, mP2_0);
          r1 = rhs_fold(Fw1, P, k, m1_1, mP2_1);
        }
        T0[p] = r0;
        T0[WP + p] = r1;
      }
      __syncthreads();
      PHASE_STAMP(13);
      // (r2) the moment system of both fields by the recursive filter of spline_rf (kernels.cu),
      // (1,4,1) = (-1/rho)(1 - rho z^-1)(1 - rho z): half of the CTA per field, segments of kP2Seg
      // rows aligned to the global grid (segment g = rows [7g, 7g + 7)), each filtered from a zero
      // start, the carries combined over the kP2Q previous / next segments (|rho|^42 = 1e-24).
      // Every output is the same arithmetic on the same data in every CTA schedule (bitwise
      // identical batch modes); m in place of the right-hand side
      {
        constexpr double rho = -0.26794919243112270;        // sqrt(3) - 2
        constexpr int NH = NT / 2, S = kP2Seg;
        const int f = tid >= NH, lt = tid - (f ? NH : 0);
        const int nseg = Wa / S;
        double* const X = T0 + f * WP;
        double* const Ec = T1 + f * WP;                      // forward segment ends
        double* const Fc = Ec + nseg;                        // backward segment starts
        double rs = 1.0;
#pragma unroll
        for (int j = 0; j < S; ++j) rs *= rho;
        // (the segment in registers: its loads issue together, the filter chains run at FMA latency)
        for (int sg = lt; sg < nseg; sg += NH) {
          double* xp = X + sg * S;
          double x[S];
#pragma unroll
          for (int j = 0; j < S; ++j) x[j] = xp[j];
          double u = 0.0;
#pragma unroll
          for (int j = 0; j < S; ++j) { u = fma(rho, u, x[j]); x[j] = u; }
#pragma unroll
          for (int j = 0; j < S; ++j) xp[j] = x[j];
          Ec[sg] = u;
        }
        __syncthreads();
        for (int sg = lt; sg < nseg; sg += NH) {
          double* xp = X + sg * S;
          double e[kP2Q];                                     // the kP2Q previous segment ends
#pragma unroll
          for (int q = 0; q < kP2Q; ++q) e[q] = sg - kP2Q + q >= 0 ? Ec[sg - kP2Q + q] : 0.0;
          double x[S];
#pragma unroll
          for (int j = 0; j < S; ++j) x[j] = xp[j];
          double C = 0.0;                                    // u of the row before the segment
#pragma unroll
          for (int q = 0; q < kP2Q; ++q)
            if (sg - kP2Q + q >= 0) C = fma(rs, C, e[q]);
          double pw = rho;
#pragma unroll
          for (int j = 0; j < S; ++j) { x[j] = fma(pw, C, x[j]); pw *= rho; }
          double v = 0.0;
#pragma unroll
          for (int j = S - 1; j >= 0; --j) { v = fma(rho, v, x[j]); x[j] = v; }
#pragma unroll
          for (int j = 0; j < S; ++j) xp[j] = x[j];
          Fc[sg] = v;
        }
        __syncthreads();
        for (int sg = lt; sg < nseg; sg += NH) {
          double* xp = X + sg * S;
          double e[kP2Q];                                     // the kP2Q next segment starts
#pragma unroll
          for (int q = 0; q < kP2Q; ++q) e[q] = sg + kP2Q - q < nseg ? Fc[sg + kP2Q - q] : 0.0;
          double x[S];
#pragma unroll
          for (int j = 0; j < S; ++j) x[j] = xp[j];
          double D = 0.0;                                    // v of the row after the segment
#pragma unroll
          for (int q = 0; q < kP2Q; ++q)
            if (sg + kP2Q - q < nseg) D = fma(rs, D, e[q]);
          double pw = rho;
#pragma unroll
          for (int j = S - 1; j >= 0; --j) { x[j] = -rho * fma(pw, D, x[j]); pw *= rho; }
#pragma unroll
          for (int j = 0; j < S; ++j) xp[j] = x[j];
        }
        __syncthreads();
      }
      const double* A = T0;
      PHASE_STAMP(14);
      const double ib = 1.0;                                 // m itself (the PCR form had a scale)
      double* ringn = const_cast<double*>(s.ring) + (int64_t)slot_out * s.slot_elems;
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        const double* Fw = f ? Fw1 : Fw0;
        const double m1 = f ? m1_1 : m1_0, mP2 = f ? mP2_1 : mP2_0;
        const double* Am = A + f * WP;
        auto mt = [&](int k) { return Am[k - base] * ib; };
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
        double* rf = ringn + (int64_t)f * s.cfield;
        for (int k = k0 + tid; k < k1; k += NT) rf[k + 1] = coef(k);
        // edge CTAs: the line's virtual boundary entries, the clamped boundary values
        // s(x_0) = (c_{-1} + 4 c_0 + c_1)/6 and s(x_{P-1}), from shared memory
        // edge CTAs: the line's virtual boundary entries, the clamped boundary values
        // s(x_0) = (c_{-1} + 4 c_0 + c_1)/6 and s(x_{P-1}), from shared memory
        // (16-byte stores: the pad [-cpad, 0) is 16-byte aligned, cpad even; the right pad
        // starts at P + 3, its odd-aligned head and tail take 8-byte stores)
        if (k0 == -1 && !DBG_FLAG(pp.nopad)) {
          const double v = (1.0 / 6.0) * coef(-1) + (2.0 / 3.0) * coef(0) + (1.0 / 6.0) * coef(1);
          double2* q = reinterpret_cast<double2*>(rf - s.cpad);
          for (int i = tid; i < (int)(s.cpad >> 1); i += NT) q[i] = make_double2(v, v);
        }
        if (k1 == P + 1 && !DBG_FLAG(pp.nopad)) {
          const double v = (1.0 / 6.0) * coef(P - 2) + (2.0 / 3.0) * coef(P - 1) + (1.0 / 6.0) * coef(P);
          double* r0 = rf + P + 3;
          const int h = (int)((reinterpret_cast<uintptr_t>(r0) >> 3) & 1);     // 1: odd-aligned start
          const int n2 = (int)((s.cpad - h) >> 1);
          double2* q = reinterpret_cast<double2*>(r0 + h);
          for (int i = tid; i < n2; i += NT) q[i] = make_double2(v, v);
          if (tid == 0 && h) r0[0] = v;
          if (tid == 1 && h + 2 * n2 < s.cpad) r0[s.cpad - 1] = v;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      PHASE_STAMP(15);
      // publish the CTA's ring stores: a gpu-scope release by one thread after the CTA
      // barrier (cumulative over the CTA's stores)
      if (tid == publisher) st_release(pp.ring_flag + bid, (unsigned)it + 1);
    }
  }
  if (pl > pf) {
    const unsigned ex = __reduce_add_sync(0xffffffffu, pexec);
    if (lane == 0 && ex) atomicAdd(pcnt + pf, (unsigned long long)ex);
    if (multi) {
      const unsigned ex1 = __reduce_add_sync(0xffffffffu, pexec1);
      if (lane == 0 && ex1) atomicAdd(pcnt + pf + 1, (unsigned long long)ex1);
    }
  }
  __syncthreads();
  if (tid < bt.nprob && PB[tid].s.picard_exec != nullptr && pcnt[tid] != 0) atomicAdd(PB[tid].s.picard_exec, pcnt[tid]);
}

// instantiated (R, C, NT, MB = CTAs per SM) variants of the fused kernel; index 0 is the default
// (r2) index 0 = 12 warps in 3 point groups x 4 node chunks, one CTA per SM (cfg 2 batch 16.6 ->
// 15.4 ms against the round-1 default, now index 7: 8 chunks x 1 group, two CTAs per SM)
#define BSDE_FUSED_VARIANTS(X) X(0, 7, 4, 384, 1) X(1, 7, 8, 512, 1) X(2, 5, 4, 384, 1) X(3, 3, 4, 640, 1) X(4, 7, 4, 256, 1) X(5, 5, 4, 256, 2) X(6, 7, 4, 256, 2) \
  X(7, 7, 8, 256, 2)
struct FusedVariant { int R, C, NT, MB; };
constexpr int kFusedAltVariant = 7;   // when index 0's one-tile-per-CTA launch is not co-resident
static const FusedVariant kVariants[] = {
#define BSDE_V_ROW(i, R, C, NT, MB) {R, C, NT, MB},
    BSDE_FUSED_VARIANTS(BSDE_V_ROW)
#undef BSDE_V_ROW
};
constexpr int kNumVariants = sizeof(kVariants) / sizeof(kVariants[0]);
int fused1d_num_variants() { return kNumVariants; }
int fused1d_alt_variant() { return kFusedAltVariant; }

// shared memory of the fused kernel for fz's buffer sizes: the spline scratch gets its own
// region when it fits (fz.sep = 1), else it overlays the level buffers; 0 if neither fits
size_t fused1d_smem(Fused1D& fz) {
  const size_t limit = kVariants[fz.variant].MB == 1 ? 220 * 1024 : 112 * 1024;
  const size_t sep = kFusedHdr + ((size_t)4 * fz.WMAX + fz.WS + fz.TK) * sizeof(double);
  const int wo = std::max(fz.WMAX, (fz.WS + 3) / 4);
  const size_t ovl = kFusedHdr + ((size_t)4 * wo + fz.TK) * sizeof(double);
  fz.sep = sep <= limit;
  if (fz.sep) return sep;
  if (ovl > limit) return 0;
  fz.WMAX = (wo + 1) & ~1;
  return kFusedHdr + ((size_t)4 * fz.WMAX + fz.TK) * sizeof(double);
}

bool fused1d_geometry(const Grid& g, int K, int L, int qspan_max, int nsm, int variant, Fused1D& fz, int& threads,
                      int& blocks, size_t& smem) {
  if (variant < 0 || variant >= kNumVariants) return false;
  const FusedVariant v = kVariants[variant];
  const int64_t P = g.P[0];
  if (P >= (1ll << 30) || P < 8) return false;
  const int nwpg = v.NT / (32 * v.C);
  fz.variant = variant;
  fz.TP = 32 * nwpg * v.R;
  // the pass-2 values window must contain every folded index of the odd extension
  if (P < 2 * fz.TP + 2 * kP2Halo + 256) return false;     // small grids: generic kernels
  threads = v.NT;
  blocks = (int)((P + fz.TP - 1) / fz.TP);
  fz.WP = ((fz.TP + 2 + 2 * kP2Halo + 8) + 1) & ~1;          // pass-2 window of the own tile (+ slack)
  int wm = fz.TP + qspan_max + 4 + 2;                        // level window
  const int wr = (3 * v.C * fz.TP + 3) / 4;                  // reduction (overlays buf0/buf1)
  if (wr > wm) wm = wr;
  fz.WMAX = (wm + 1) & ~1;
  fz.WS = 6 * fz.WP + 16;                                    // pass-2 spline scratch
  fz.TK = ((int)((size_t)K * L * sizeof(Tap1D) / sizeof(double)) + 1) & ~1;   // tap table
  smem = fused1d_smem(fz);
  (void)K; (void)L; (void)nsm;
  return smem > 0;
}

void pcr_constants(double* alpha, double* inv_b);

template <int DRV, int R, int C, int NT, int MB>
static cudaError_t launch_fused1d(FusedBatch& bt, int threads, int blocks, size_t smem, cudaStream_t st) {
  pcr_constants(bt.fz.alpha, &bt.fz.inv_b);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;     // neighbour flags need all CTAs co-resident
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, quad1d_fused<DRV, R, C, NT, MB>, bt);
}

template <int DRV>
static cudaError_t launch_fused1d_v(FusedBatch& bt, int threads, int blocks, size_t smem, cudaStream_t st) {
  switch (bt.fz.variant) {
#define BSDE_V_CASE(i, R, C, NT, MB) \
    case i: return launch_fused1d<DRV, R, C, NT, MB>(bt, threads, blocks, smem, st);
    BSDE_FUSED_VARIANTS(BSDE_V_CASE)
#undef BSDE_V_CASE
  }
  return cudaErrorInvalidValue;
}

template <int DRV>
static cudaError_t set_attr_drv() {
  cudaError_t e = cudaSuccess;
#define BSDE_V_ATTR(i, R, C, NT, MB)                                                                   \
  if (e == cudaSuccess)                                                                               \
    e = cudaFuncSetAttribute(quad1d_fused<DRV, R, C, NT, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             MB == 1 ? 220 * 1024 : 112 * 1024);
  BSDE_FUSED_VARIANTS(BSDE_V_ATTR)
#undef BSDE_V_ATTR
  return e;
}

// blocks per SM the fused kernel can keep resident (for the cooperative launch)
int fused1d_blocks_per_sm(int variant, size_t smem) {
  int nb = 0;
  cudaError_t e = cudaErrorInvalidValue;
  switch (variant) {
#define BSDE_V_OCC(i, R, C, NT, MB) \
    case i: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, quad1d_fused<DRV_DIFF, R, C, NT, MB>, NT, smem); break;
    BSDE_FUSED_VARIANTS(BSDE_V_OCC)
#undef BSDE_V_OCC
  }
  return e == cudaSuccess ? nb : 0;
}

// one cooperative launch over nprob problems (round-robin steps); the progress flags of
// every problem (pp.ring_flag, 2 x blocks) are cleared first
cudaError_t launch_fused1d_batch(const FusedProb* probs, int nprob, const Grid& g, const Fused1D& fz, int driver_id,
                                 int threads, int blocks, size_t smem, cudaStream_t st, const int* group,
                                 const int* gcta, const int* gns, int ngroup) {
  if (nprob < 1 || nprob > kMaxBatch) return cudaErrorInvalidValue;
  thread_local static FusedBatch bt;     // ~6 KB: kept off the stack
  bt = FusedBatch{};
  bt.fz = fz;
  bt.g = g;
  bt.part = group != nullptr;
  {
    void* a = nullptr;
    cudaError_t e = cudaGetSymbolAddress(&a, c_arena);
    if (e != cudaSuccess) return e;
    bt.arena = static_cast<const unsigned char*>(a);
  }
  bt.nprob = nprob;
  bt.max_steps = 0;
  // problems with more levels first: the first problem of a round then has windows of levels
  // >= 2 that stream in during the previous round's pass 2 (a stable order; each problem's
  // arithmetic does not depend on it)
  // (part mode: group-major, each group's problems contiguous)
  int order[kMaxBatch];
  for (int i = 0; i < nprob; ++i) order[i] = i;
  std::stable_sort(order, order + nprob, [&](int a, int b) {
    if (group && group[a] != group[b]) return group[a] < group[b];
    return probs[a].s.K > probs[b].s.K;
  });
  int tot = 0;
  if (bt.part) {
    bt.ngroup = ngroup;
    for (int gi = 0; gi < ngroup; ++gi) {
      bt.gcta0[gi] = tot;
      bt.gns[gi] = gns[gi];
      tot += gcta[gi];
    }
    bt.gcta0[ngroup] = tot;
    int k = 0;
    for (int gi = 0; gi <= ngroup; ++gi) {
      while (k < nprob && group[order[k]] < gi) ++k;
      bt.gp0[gi] = k;
    }
  }
  for (int i = 0; i < nprob; ++i) {
    bt.prob[i] = probs[order[i]];
    if (bt.prob[i].pp.nsteps > bt.max_steps) bt.max_steps = bt.prob[i].pp.nsteps;
#ifdef BSDE_DEBUG
    if (getenv("BSDE_DEBUG_NOWAIT")) bt.prob[i].pp.nowait = 1;   // timing experiments only: wrong results
    if (getenv("BSDE_DEBUG_NOPAD")) bt.prob[i].pp.nopad = 1;
#endif
    // ring flags at [0, n), done flags behind them (round-robin: n = blocks; part: 8192)
    const size_t nf = bt.part ? 2 * (size_t)kFlagCap : 2 * (size_t)blocks;
    cudaError_t e = cudaMemsetAsync(probs[i].pp.ring_flag, 0, sizeof(unsigned) * nf, st);
    if (e != cudaSuccess) return e;
  }
  if (bt.part && tot != blocks) return cudaErrorInvalidValue;
  switch (driver_id) {
    case DRV_ZERO: return launch_fused1d_v<DRV_ZERO>(bt, threads, blocks, smem, st);
    case DRV_AFFINE: return launch_fused1d_v<DRV_AFFINE>(bt, threads, blocks, smem, st);
    case DRV_EX1: return launch_fused1d_v<DRV_EX1>(bt, threads, blocks, smem, st);
    case DRV_EX2: return launch_fused1d_v<DRV_EX2>(bt, threads, blocks, smem, st);
    case DRV_DIFF: return launch_fused1d_v<DRV_DIFF>(bt, threads, blocks, smem, st);
  }
  return cudaErrorInvalidValue;
}

// nsteps consecutive steps (ring_mode 1: levels n0, n0-1, ...) or one step with StepArgs'
// fields (ring_mode 0); one cooperative launch either way
cudaError_t launch_fused1d_steps(const StepArgs& s, const Grid& g, const Problem& pb, const Fused1D& fz, int n0,
                                 int nsteps, int ring_mode, int cur, double t0, double dt, double* v0, double* v1,
                                 unsigned* flags, const int* D, int DK, int threads, int blocks, size_t smem,
                                 cudaStream_t st) {
  FusedProb fp{};
  fp.s = s;
  fp.pp.n0 = n0;
  fp.pp.nsteps = nsteps;
  fp.pp.ring_mode = ring_mode;
  fp.pp.cur = cur;
  fp.pp.t0 = t0;
  fp.pp.dt = dt;
  fp.pp.vbuf[0] = v0;
  fp.pp.vbuf[1] = v1;
  fp.pp.ring_flag = flags;
  fp.pp.done_flag = flags + blocks;
  for (int j = 0; j <= kMaxK; ++j) fp.pp.D[j] = D[j];
  fp.pp.DK = DK;
  for (int i = 0; i < 12; ++i) fp.dp[i] = pb.dp[i];
  return launch_fused1d_batch(&fp, 1, g, fz, pb.driver_id, threads, blocks, smem, st, nullptr, nullptr, nullptr, 0);
}
