/*
 * bsde.h -- C ABI of the B200-native multistep BSDE solver
 * (Kapllani & Teng, "Multistep schemes for solving backward stochastic
 *  differential equations on GPU", arXiv 1909.13560).
 *
 * One context solves one decoupled BSDE (Eq. 2)
 *     -dy_t = f(t, y_t, z_t) dt - z_t dW_t,   y_T = g(W_T),
 * backward in time with the fully discrete multistep scheme of Eq. 20
 * on a uniform tensor grid of a truncated box
 * (PAPER.md:334-337, 367-371).  Conditional expectations are Gauss-Hermite
 * quadratures of spline-interpolated values (Eq. 21); z^n is
 * explicit, y^n is solved by Picard iteration (p = 30 at
 * PAPER.md:493).  All numerical work runs in hand-written sm_100a fp64 kernels.
 *
 * Conventions
 *  - No C++ exception crosses this boundary; every call returns bsde_status.
 *  - Host pointers are plain host memory; device pointers are CUDA device memory
 *    of cfg.device.  The library never frees memory it did not allocate.
 *  - Layout of a layer (bsde_get_layer): fp64, row-major over the d axes (the last
 *    axis contiguous), npts[0]*...*npts[d-1] values; field 0 = y, field k = z_k.
 *  - A context is used from one host thread.  Calls are stream-ordered on
 *    cfg.stream (or a library-owned stream); bsde_step does not synchronise.
 *  - Determinism: results are bitwise identical across runs for a fixed config.
 */
#ifndef BSDE_H
#define BSDE_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BSDE_OK = 0,
  BSDE_ERR_INVALID_ARGUMENT = 1, /* config outside the documented ranges; nothing allocated */
  BSDE_ERR_RESOURCE_LIMIT = 2,   /* device memory / workspace / constant arena too small   */
  BSDE_ERR_SINGULAR = 3,         /* reserved (the spline matrix is never singular)          */
  BSDE_ERR_NUMERICAL_DOMAIN = 4, /* a non-finite y or z was produced (details: last_error)  */
  BSDE_ERR_CUDA = 5,             /* a CUDA runtime error (message in last_error)            */
  BSDE_ERR_COMM = 6,             /* an NCCL failure of the multi-GPU halo exchange          */
  BSDE_ERR_STATE = 7             /* e.g. bsde_step at n == 0                                */
} bsde_status;

/* Driver f(t, y, z) in the paper's sign convention -dy = f dt - z dW (Eq. 2).
 * Parameters p = driver_params. */
typedef enum {
  BSDE_DRV_ZERO = 0,       /* f = 0                                                        */
  BSDE_DRV_AFFINE = 1,     /* f = p0 y + sum_k p[1+k] z_k + p4 : Black-Scholes Eq. 29/30,
                              Ex. 4 Eq. 34 (p = 1, -1/2, -1/2), exchange Eq. 36             */
  BSDE_DRV_EX1 = 2,        /* f = -y^3 + 5/2 y^2 - 3/2 y          (Eq. 22)   */
  BSDE_DRV_EX2 = 3,        /* f = 1/2 (e^{t^2} - 4 t y - 3 e^{t^2 - y e^{-t^2}} + z^2 e^{-t^2})
                                                                  (Eq. 24)   */
  BSDE_DRV_DIFF_RATES = 4  /* f = -(r y + sum_k th_k z_k) + (R - r) max(sum_k pi_k z_k - y, 0)
                              p0 = r (lending), p1 = R (borrowing), p2..4 = th_k, p5..7 = pi_k
                              (wealth equation Eq. 28 with a borrowing rate; R21) */
} bsde_driver_id;

/* Terminal condition g(w), w = W_T, in W-space (R20); z_T = grad g (Eq. 4). */
typedef enum {
  BSDE_TERM_CONST = 0,        /* g = p0                                                    */
  BSDE_TERM_POLY = 1,         /* g = prod_a (p[4a] + p[4a+1] w_a + p[4a+2] w_a^2 + p[4a+3] w_a^3) */
  BSDE_TERM_LOGISTIC = 2,     /* g = 1/(1 + exp(-(sum_a w_a/sqrt(d) + T)))  (Eq. 22 for d=1)*/
  BSDE_TERM_EX2 = 3,          /* g = ln(sin w + 3) e^{T^2}                      (Eq. 24)   */
  BSDE_TERM_CALL_W = 4,       /* S = p0 exp((p2 - p3^2/2) T + p3 w), g = (S - p1)^+ (Eq. 30, 32) */
  BSDE_TERM_SIN_SUM = 5,      /* g = sin(sum_a w_a + T)                         (Eq. 34)   */
  BSDE_TERM_EXCHANGE_W = 6,   /* S_k = p[k] exp((p[2+k] - s_k^2/2) T + (A w)_k), s = (p4, p5),
                                 rho = p6, A = [[s1, 0], [rho s2, s2 sqrt(1-rho^2)]],
                                 g = (S_1 - S_2)^+                               (Eq. 36)   */
  BSDE_TERM_GEO_BASKET_W = 7, /* S_k = p[k] exp((p4 - s_k^2/2) T + s_k w_k), s_k = p[5+k],
                                 G = (prod_k S_k)^{1/d}, g = (G - p3)^+     (BASELINE cfg 5) */
  BSDE_TERM_CALL_X = 8        /* forward-SDE problems (sde_id != 0): g(x) = (x_0 - p1)^+ in the
                                 state variable x = X_T itself (e.g. a stock price)          */
} bsde_terminal_id;

/* Forward process X of the FBSDE (Eq. 1): dX = a(X) dt + b(X) dW with a
 * diagonal b, approximated by one Euler step per level ("e.g. by using the Euler-Scheme",
 * PAPER.md:50): from grid point x_i the level-j sample is
 *     X = x_i + a(x_i) j dt + b(x_i) sqrt(2 j dt) a_Lambda        (per axis k),
 * so the stencil is no longer translation-invariant (per-point cell location).
 * z is the BSDE's z = b^T grad u; the terminal layer is z_T = b(x) grad g(x).
 * Parameters p = sde_params; p[9..11] = X_0 = x_0 is the evaluation point of (y_0, z_0)
 * (the spline of layer 0 there).  sde_id 0 is Eq. 2 (X = W) and uses the stencil kernels. */
typedef enum {
  BSDE_SDE_BROWNIAN = 0,      /* a = 0, b = 1 (X = W, Eq. 2)                                 */
  BSDE_SDE_GBM = 1,           /* a_k = p[k] x_k, b_k = p[3+k] x_k (geometric Brownian motion) */
  BSDE_SDE_OU = 2             /* a_k = p[k] (p[3+k] - x_k), b_k = p[6+k] (Ornstein-Uhlenbeck)  */
} bsde_sde_id;

/* Spatial interpolation of the levels. */
typedef enum {
  BSDE_INTERP_SPLINE = 0,     /* tensor-product not-a-knot cubic spline (north_star; R14)     */
  BSDE_INTERP_FD_BICUBIC = 1  /* d = 2 only: the paper's bicubic interpolation with first and
                                 mixed derivatives by 4th-order finite differences (central,
                                 one-sided within 2 nodes of the box edge)      */
} bsde_interp_id;

typedef struct {
  uint32_t struct_size;      /* caller sets sizeof(bsde_config) (ABI versioning)          */
  int32_t  d;                /* Brownian dimension, 1..3                                  */
  int32_t  m;                /* solution dimension, must be 1                             */
  double   t0, T;            /* time interval; dt = (T - t0)/N, t_n = t0 + n dt */
  int32_t  N;                /* time steps, N >= max(Ky, Kz)                               */
  int32_t  Ky, Kz;           /* multistep levels, 1..6 (Tables 1-2)     */
  int32_t  L;                /* Gauss-Hermite nodes per axis, 1..64 (Eq. 21)              */
  int64_t  npts[3];          /* grid points per axis incl. both ends, >= 4; 0 -> balance rule
                                M = 2 ceil(X/dx), dx = dt^{(q+1)/r}, q = min(Ky+1, Kz, 3),
                                npts = M + 1 (R3)              */
  double   xlo[3], xhi[3];   /* truncated box in W-space                    */
  int32_t  r;                /* balance-rule interpolation order (0 -> 4)                  */
  int32_t  driver_id;   double driver_params[12];
  int32_t  terminal_id; double terminal_params[12];
  int32_t  picard_max;       /* Picard iterations (30)                       */
  double   picard_tol;       /* <= 0: exactly picard_max iterations (R8)          */
  int32_t  bootstrap;        /* 0: closed-form initial layers; 1: one-step scheme (K = 1) with
                                bootstrap_substeps sub-steps per interval */
  int32_t  bootstrap_substeps;
  int32_t  smoothing;        /* 1: cell-average the kinked payoff at the terminal layer
                                (R11)                          */
  int32_t  nranks, rank;     /* slab partition along axis 0 (d >= 2); 1/0 for one GPU.  Rank r
                                owns rows [r P0/R, (r+1) P0/R) and keeps `halo` extra rows on
                                each side: reach + 3 rows of coefficients (SPIKE, slab_spline
                                = 0) or reach + 3 + 37 rows of values (slab_spline = 1),
                                exchanged every step.  With SPIKE and NCCL,
                                bsde_eval / bsde_solve are collectives (every rank calls)     */
  const void* nccl_unique_id;/* nranks > 1: 128-byte ncclUniqueId from bsde_nccl_unique_id()
                                (multi-process, one rank per GPU, halos by NCCL send/recv), or
                                NULL for an in-process group driven by bsde_group_step/solve */
  void*    stream;           /* cudaStream_t to run on; NULL -> library-owned stream        */
  int32_t  device;           /* CUDA device ordinal                                         */
  int32_t  kernel_variant;   /* 0: auto (fastest available; d = 2 with f = 0 or affine f:
                                the separable affine path), 1: generic reference kernels;
                                2 (d = 2): the per-tap fused 2-D kernel for every driver;
                                10 + v (d = 1): fused kernel variant v; any other value
                                selects the generic kernels                               */
  int32_t  interp;           /* interpolation, a bsde_interp_id value; 0 = tensor spline   */
  int32_t  sde_id;           /* forward SDE, a bsde_sde_id value; 0 = X = W                */
  double   sde_params[12];
  int32_t  timing;           /* 1: per-stage CUDA-event timers (t_spline_s, t_quad_s, t_comm_s
                                of bsde_result); 0: only setup / bootstrap / sweep times   */
  int32_t  slab_spline;      /* nranks > 1: the axis-0 spline across slab interfaces.
                                0 (default): SPIKE -- each rank solves its own rows with zero
                                coupling, the 2 edge moments per line and rank are all-gathered,
                                the 2 (R-1) interface system is solved (same inverse for every
                                line) and the spike-vector correction applied; the halo is
                                reach + 3 rows of final coefficients.
                                1 (ablation): the axis-0 spline is re-solved redundantly over a
                                values halo of reach + 3 + 37 rows (PCR decay, 5e-19)        */
} bsde_config;

typedef struct {
  double  y0, z0[3];         /* solution at t0 and x = 0 (grid value if x = 0 is a grid point,
                                else the spline of layer 0 at 0; R4)             */
  double  t_setup_s;         /* bsde_setup wall time (host clock; includes the bootstrap)   */
  double  t_sweep_s;         /* backward sweep of this call (CUDA events on the stream)    */
  double  t_total_s;         /* t_setup_s + wall time of this call incl. result read-back   */
  int64_t updates;           /* points this rank owns * sweep steps performed by this call  */
  int32_t picard_max_used;
  double  t_bootstrap_s;     /* device time of the K-1 initial layers (closed form or the
                                one-step bootstrap), CUDA events inside bsde_setup          */
  double  t_spline_s;        /* cfg.timing = 1: device time of the spline builds of this call
                                (0 where the spline is fused into the quadrature kernel:
                                the d = 1 persistent kernel)                                */
  double  t_quad_s;          /* cfg.timing = 1: quadrature + z + Picard kernels             */
  double  t_comm_s;          /* cfg.timing = 1: halo exchange (NCCL or peer copies)         */
  int64_t picard_iters;      /* Picard iterations executed by the sweep of this call (all
                                points; the d = 1 persistent kernel counts them, -1 otherwise).
                                The kernel leaves the loop at an exact fixed point, where the
                                remaining iterations of the fixed count p are identities     */
  int32_t batch_ctas;        /* bsde_solve_batch*: CTAs that stepped this problem            */
  int32_t batch_tiles;       /* ... and tiles (of TP points) per CTA (1: round robin)         */
} bsde_result;

typedef struct bsde_ctx bsde_ctx;

/* Device bytes the context needs (values, coefficient ring of K levels, scratch).
 * Errors: INVALID_ARGUMENT for an invalid config.                                      */
bsde_status bsde_query_workspace(const bsde_config* cfg, size_t* bytes);

/* Validate, build grids / Gauss-Hermite rule / weight rows / tap tables, allocate (or
 * adopt the caller's d_workspace of `bytes` >= bsde_query_workspace; caller-owned, must
 * outlive the context), compute the K initial layers and their splines.  On return the
 * newest level is N-K+1.  On failure nothing stays allocated and *out = NULL.          */
bsde_status bsde_setup(const bsde_config* cfg, void* d_workspace, size_t bytes, bsde_ctx** out);

/* One backward step n+1 -> n (Eq. 20): fused quadrature/z/Picard kernel, then the
 * spline build of the new level into the ring slot of level n+K.  Asynchronous.
 * Errors: STATE at n == 0 and for a member of an in-process slab group (use
 * bsde_group_step, which also refreshes the halos); CUDA on a launch failure.          */
bsde_status bsde_step(bsde_ctx* ctx);

/* Remaining steps to n = 0, then the evaluation point; synchronises the stream and
 * checks the device non-finite flag (NUMERICAL_DOMAIN; last_error names the level n, the
 * point index i, t_n, x_i and the y, z found there).  res may be NULL.  Multi-process
 * NCCL ranks (nranks > 1 with an nccl_unique_id) always run the evaluation-point
 * all-reduce, so every rank must call bsde_solve; res may differ per rank.             */
bsde_status bsde_solve(bsde_ctx* ctx, bsde_result* res);

/* Batched solve of n (1..8) independent d = 1 problems on one device: the remaining steps
 * of every context run in ONE persistent launch whose CTAs execute the problems' steps
 * round-robin (step it of problems 0..n-1, then step it+1), so each problem's neighbour
 * waits overlap the other problems' arithmetic.  Requirements (else INVALID_ARGUMENT,
 * nothing launched): distinct contexts, one rank, d = 1, same device, grid (P, xlo, xhi)
 * and driver id, the fused kernel available to every context with the same variant;
 * RESOURCE_LIMIT if the combined shared-memory footprint cannot be
 * co-resident.  The launch is issued on ctxs[0]'s stream,
 * ordered after the other contexts' streams and before their later work (event joins).
 * res: n results or NULL; t_sweep_s is the batch's device time (the same in every result),
 * updates the context's own.  Synchronises ctxs[0]'s stream; NUMERICAL_DOMAIN as for
 * bsde_solve (first failing context).                                                 */
bsde_status bsde_solve_batch(bsde_ctx* const* ctxs, int32_t n, bsde_result* res);

/* bsde_solve_batch with an explicit CTA schedule.  mode 0: auto (= bsde_solve_batch: mode 2 or 3,
 * whichever the calibrated cost model predicts faster, when a plan fits, else round robin); 1: round robin (every CTA steps every
 * problem on one tile of TP points); 2: paired problem-partitioned (the problems are paired by K
 * rank -- smallest with largest -- and each pair gets its own CTAs, which step the pair's two
 * problems round robin on a range of consecutive tiles whose spline is built in one pass; the
 * CTAs per pair come from a cost model so that all pairs finish together); 3: the same with one
 * problem per group; RESOURCE_LIMIT from modes 2, 3 if no plan fits.  The arithmetic of every
 * point is the same in every mode (bitwise identical results).
 * mode 11..19 (ablation): one problem per group, mode - 10 tiles per CTA.                    */
bsde_status bsde_solve_batch_mode(bsde_ctx* const* ctxs, int32_t n, int32_t mode, bsde_result* res);

/* index n of the newest level                                                         */
bsde_status bsde_level(const bsde_ctx* ctx, int32_t* n_out);

/* Copy field (0 = y, k = z_k) of the newest level to host memory; count = the points this
 * rank owns (all points for one rank).                                                 */
bsde_status bsde_get_layer(const bsde_ctx* ctx, int32_t field, double* host_dst, int64_t count);

/* Picard iteration count per point of the newest level (0 for initial layers).         */
bsde_status bsde_get_picard_counts(const bsde_ctx* ctx, int32_t* host_dst, int64_t count);

/* Grid actually used: points per axis and dx (axes >= d report 1 and 0).              */
bsde_status bsde_query_grid(const bsde_ctx* ctx, int64_t npts[3], double dx[3]);

/* Tap table of level j (1..K) on `axis`: for each node l < L the cell offset q, the 4
 * cubic B-spline basis weights at theta, the Gauss-Hermite weight w/sqrt(pi) and the
 * Brownian increment sqrt(2 j dt) a_l (Eq. 21).  Host arrays of L,
 * 4L, L, L entries.                                                                   */
bsde_status bsde_query_taps(const bsde_ctx* ctx, int32_t level, int32_t axis, int32_t* q,
                            double* basis4, double* w, double* dw);

/* Values of all fields of the newest level's spline at the host point x[d] (clamped to
 * the box).  out[1+d] host.                                                           */
bsde_status bsde_eval(bsde_ctx* ctx, const double* x, double* out);

/* Device pointer of field `field` of the newest level (npts contiguous doubles, valid
 * until the next bsde_step).                                                          */
bsde_status bsde_layer_device_ptr(const bsde_ctx* ctx, int32_t field, const double** dptr);

/* Slab partition of this rank: owned global rows [own_lo, own_hi) of axis 0 and the halo
 * width (0 for one rank).  bsde_get_layer / bsde_get_picard_counts return the owned rows.  */
bsde_status bsde_query_partition(const bsde_ctx* ctx, int64_t* own_lo, int64_t* own_hi, int64_t* halo);

/* Host only (no device needed): the partition a config would get: out = {own_lo, own_hi,
 * halo, slab_lo, slab_hi} (global rows of axis 0).  INVALID_ARGUMENT if a slab is thinner
 * than the halo.                                                                        */
bsde_status bsde_query_partition_cfg(const bsde_config* cfg, int64_t out[5]);

/* A fresh NCCL unique id (rank 0 calls it and broadcasts the bytes, e.g. with
 * torch.distributed); out must hold >= 128 bytes.                                      */
bsde_status bsde_nccl_unique_id(void* out, size_t bytes);

/* In-process slab group: ctxs[r] is rank r of n (nccl_unique_id == NULL), all at the same
 * level.  One backward step on every rank, then the halo copy between neighbours
 * (cudaMemcpyPeer; ranks may share a GPU).  Synchronises the ranks' streams.           */
bsde_status bsde_group_step(bsde_ctx** ctxs, int32_t n);

/* Remaining steps of an in-process group to n = 0 and the evaluation point (from the
 * owning rank).  res may be NULL.                                                      */
bsde_status bsde_group_solve(bsde_ctx** ctxs, int32_t n, bsde_result* res);

/* Number of kernels launched by this context so far.                                  */
bsde_status bsde_kernel_launches(const bsde_ctx* ctx, int64_t* count);

/* Measured FP64 peak of `device` (the denominator of the roofline in DESIGN.md §5):
 * a kernel of independent DFMA chains (16 per thread, 8 warps per CTA, 8 CTAs per SM) is
 * timed with CUDA events over `iters` chain steps after one warm-up launch.  Outputs the
 * sustained rate in TFLOP/s (DFMA = 2 flops) and the kernel time in ms.  Not thread-safe
 * with respect to other work on the device (it owns the device while it runs).          */
bsde_status bsde_measure_fp64_peak(int32_t device, int32_t iters, double* tflops, double* ms);

/* Message of the last failing call on ctx (owned by ctx; valid until the next call), or
 * of the last failing bsde_setup/bsde_query_workspace when ctx == NULL (thread-local). */
const char* bsde_last_error(const bsde_ctx* ctx);

/* Release library-owned memory and streams; never the caller's workspace.              */
void bsde_destroy(bsde_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* BSDE_H */
