#!/usr/bin/env python
"""Benchmark of the multistep BSDE hot path on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], "cfg 2"): 1-D call under different borrowing /
lending rates, P = 2^16 grid points on [-16, 16] (W-space), N = 256 time steps,
L = 16 Gauss-Hermite nodes, K = Ky = Kz = 1..6.  One bench *step* is the backward
sweep n = N-K .. 0 (Eq. 20) of all six K; updates = P * (N - K + 1) summed over K.
The six sweeps run in one persistent launch (bsde_solve_batch: CTAs execute the problems'
steps round-robin).  Setup (grids, tap tables, the K closed-form initial layers and their
splines) is outside the device-timed region; the e2e number includes it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun): 1-D has no data-path exchange ("replicas only"), each rank
solves the same workload on its own GPU; value = all ranks' updates / max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "grid-point·time-step updates/s (fp64) + time-to-solution at fixed error vs host oracle"
UNIT = "updates/s"
KS = [1, 2, 3, 4, 5, 6]
# Algorithmic FP64 flops per point-step of the fused kernel:
#   per tap: 2 fields x 4 FMA (16) + driver diff-rates (8) + accumulations (6)   = 30
#   per point: K*L taps, + 2 per tap at j = Ky (E[y]), Picard 30 x (8 + 2)       = 300
#   spline of the new level: 2 fields x 21                                       = 42
FLOP_TAP, FLOP_PICARD, FLOP_SPLINE = 30, 300, 42


def flops_per_point_step(K, L=16):
    return K * L * FLOP_TAP + L * 2 + FLOP_PICARD + FLOP_SPLINE


def peak_fp64_tflops(sm_mhz=1965.0, nsm=148):
    # B200: 64 FP64 FMA per clock per SM (B200_PROFILING.md / SURVEY A.4), 2 flops per FMA
    return nsm * 64 * 2 * sm_mhz * 1e6 / 1e12


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws > 1:
        import torch.distributed as dist
        if not dist.is_initialized():
            dist.init_process_group("nccl" if os.environ.get("BENCH_BACKEND", "nccl") == "nccl" else "gloo")
        return dist, dist.get_rank(), ws
    return None, 0, 1


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, dev):
        self.dev = dev
        self.p = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None
        time.sleep(0.25)
        return self

    def __exit__(self, *exc):
        self.rows = []
        if self.p is None:
            return
        self.p.terminate()
        try:
            out, _ = self.p.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
            out, _ = self.p.communicate()
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        smax = max(float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit())
        names = ["active", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for nm, v in zip(names[1:], r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        load = [float(r[0]) for r in self.rows if r[2] and float(r[2] or 0) > 200.0] or sm
        load.sort()
        return {"sm_mhz": load[len(load) // 2] if load else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def flush_l2(torch, buf):
    buf.add_(1.0)        # 512 MiB write > 126 MB L2


def run_ours(args):
    import numpy as np
    import torch
    from paper_1909_13560_b200 import Solver, solve_batch, workloads as W, query_workspace
    dist, rank, world = _dist()
    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    ts = torch.cuda.Stream()          # a real stream (handle 0 would make the library create its own)
    torch.cuda.set_stream(ts)
    stream = ts.cuda_stream
    specs = {K: W.cfg2(K) for K in KS}
    ws = {K: torch.empty(query_workspace(specs[K]), dtype=torch.uint8, device="cuda") for K in KS}
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def one_step():
        """Set up the six contexts (untimed), flush L2, then the six sweeps in ONE persistent
        launch (bsde_solve_batch, device-timed with CUDA events on `stream`)."""
        ss = [Solver(specs[K], device=dev, stream=stream, workspace=ws[K]) for K in KS]
        n0 = [s.kernel_launches for s in ss]
        flush_l2(torch, flush)
        torch.cuda.synchronize()
        res = solve_batch(ss)
        t = res[0].t_sweep_s
        upd = sum(r.updates for r in res)
        # one batched launch is counted by every context; the rest are the y0 evaluations
        launches = 1 + sum(s.kernel_launches - a - 1 for s, a in zip(ss, n0))
        y0 = {K: (r.y0, r.z0[0]) for K, r in zip(KS, res)}
        for s in ss:
            s.close()
        return t, upd, launches, y0

    for _ in range(args.warmup):
        one_step()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    times, upds, launches = [], 0, 0
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            t, u, nl, y0 = one_step()
            times.append(t)
            upds += u
            launches += nl
    torch.cuda.synchronize()
    elapsed = sum(times)
    if dist:
        tt = torch.tensor([elapsed], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed = float(tt.item())
    value = upds * world / elapsed

    # ---- the dominant kernel is quad1d_fused: ONE persistent launch per bench step runs all
    # six sweeps (round-robin over the problems).  Its average duration is the CUDA-event time
    # of the launches of the timed region (recorded on `stream` inside bsde_solve_batch).
    launch_s = elapsed / args.steps
    fl = sum(flops_per_point_step(K) * 65536 * (256 - K + 1) for K in KS)
    clocks = clk.summary()
    peak = peak_fp64_tflops(1965.0)
    achieved = fl / launch_s / 1e12
    traffic = None
    try:   # dram__bytes_read.sum + dram__bytes_write.sum (MB) per launch, from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "round1", "ncu_quad1d_fused_batch_summary.json")) as fh:
            prof = json.load(fh)
        traffic = (float(prof["dram__bytes_read.sum"]) + float(prof["dram__bytes_write.sum"])) * 1e6
    except (OSError, KeyError, ValueError):
        pass
    roof = {"bound": "alu", "achieved": round(achieved, 3), "peak": round(peak, 2), "unit": "TFLOP/s",
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "traffic_note": "DRAM bytes per launch (six sweeps; state is L2-resident) from ncu --set full",
            "kernel": "quad1d_fused<DRV_DIFF>: one launch = the 6 sweeps K=1..6 (1521 steps)",
            "flops_per_launch": fl, "launch_us": round(launch_s * 1e6, 3),
            "peak_note": "FP64 pipe: 148 SM x 64 DFMA/clk x 2 x 1965 MHz (derived; DESIGN.md Roofline)"}
    try:   # the same denominator measured: a DFMA-chain kernel of the library (bsde_measure_fp64_peak)
        from paper_1909_13560_b200 import measure_fp64_peak
        mp = measure_fp64_peak(dev)
        roof["peak_measured"] = {"value": round(mp["tflops"], 2), "unit": "TFLOP/s",
                                 "frac_of_measured": round(achieved / mp["tflops"], 4),
                                 "note": "16 independent DFMA chains/thread, 8 x 256-thread CTAs per SM"}
    except Exception as exc:  # noqa: BLE001 -- reported, never fatal for the bench line
        roof["peak_measured"] = {"error": str(exc)}

    # ---- e2e: setup (host config -> device) + sweep + final layers device -> host, host clock
    host = np.empty(65536, dtype=np.float64)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_upd, h2d, d2h = 0, 0, 0
    for _ in range(args.steps):
        ss = [Solver(specs[K], device=dev, stream=stream, workspace=ws[K]) for K in KS]
        res = solve_batch(ss)
        for K, s, r in zip(KS, ss, res):
            s.layer(0, out=host)
            s.layer(1, out=host)
            e2e_upd += r.updates
            h2d += K * 16 * 72 + 2 * 16 * 8 + 1024          # tap table + GL rule + config/params
            d2h += 2 * 65536 * 8 + 32                        # y, z of layer 0 + y0/z0
            s.close()
    torch.cuda.synchronize()
    e2e_t = time.perf_counter() - t0
    if dist:
        tt = torch.tensor([e2e_t], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_t = float(tt.item())
    e2e = {"value": e2e_upd * world / e2e_t, "unit": UNIT, "h2d_bytes_per_step": h2d // args.steps,
           "d2h_bytes_per_step": d2h // args.steps,
           "note": "6 x bsde_setup + bsde_solve_batch + bsde_get_layer(y, z) per K, host wall clock"}

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": elapsed / args.steps * 1e3, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": "cfg2: 1-D differential-rates call, P=65536, N=256, L=16, K=1..6 (one step = the six sweeps in one bsde_solve_batch launch)",
                      "global_batch": 65536 * world, "seq_len": 256, "parallelism": f"replicas{world}",
                      "l2": "flushed (512 MiB write) before every step; the six sweeps' state (~50 MiB) is L2-resident by design"},
           "roofline": roof, "e2e": e2e, "gpu_launches": launches // max(args.steps, 1),
           "clocks": clocks,
           "accuracy": {str(K): {"y0": y0[K][0], "z0": y0[K][1]} for K in KS},
           "reference_solution": list(W.reference_solution(specs[1])[:1]) + [W.reference_solution(specs[1])[1][0]]}
    if rank == 0 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args)
    if rank == 0 and not args.no_tts:
        out["tts"] = tts_sweep(dev)
    if rank == 0 and world == 1 and not args.no_d23:
        out["d23_configs"] = d23_configs(dev, stream)
    if rank == 0:
        print(json.dumps(out))
    if dist:
        dist.barrier()
        dist.destroy_process_group()


TTS_NS = [16, 32, 64, 128, 256, 512, 1024]
TTS_EPS = {"ex1": [1e-6, 1e-8, 1e-10, 1e-12], "ex2": [1e-6, 1e-8]}


def tts_sweep(dev, oracle_budget_s=90.0):
    """Time-to-solution at fixed error (BASELINE metric): for Ex. 1 and Ex. 2
    (closed forms y0 = 1/2, ln 3) on the (K, N) grid K = 1..6 x N = 16..1024 (L = 32, balanced
    grid), the smallest wall time from bsde_setup to bsde_solve's return among runs with
    |y0 - y_exact| <= eps.  The oracle is timed on the same runs (identical y0 by parity), the
    two cheapest qualifying (K, N) per eps, within a bounded budget."""
    from paper_1909_13560_b200 import Solver, workloads as W
    out = {}
    for prob in ("ex1", "ex2"):
        mk = W.ex1 if prob == "ex1" else W.ex2
        exact = W.reference_solution(mk(1, 16))[0]
        with Solver(mk(3, 64), device=dev) as s:          # warm-up (context, caches)
            s.solve()
        runs = []
        for K in range(1, 7):
            for N in TTS_NS:
                if N < K + 1:
                    continue
                spec = mk(K, N)
                t0 = time.perf_counter()
                try:
                    with Solver(spec, device=dev) as s:
                        r = s.solve()
                        P = s.shape[0]
                except Exception:                          # e.g. a non-finite solution (unstable K, N)
                    continue
                t = time.perf_counter() - t0
                runs.append({"K": K, "N": N, "P": P, "s": t, "err": abs(r.y0 - exact),
                             "work": P * (N - K + 1) * K})
        res = {}
        for eps in TTS_EPS[prob]:
            ok = [r for r in runs if r["err"] <= eps]
            if not ok:
                res[f"{eps:g}"] = {"gpu": None, "note": "no (K, N) of the grid reaches this error"}
                continue
            best = min(ok, key=lambda r: r["s"])
            res[f"{eps:g}"] = {"gpu": {"s": best["s"], "K": best["K"], "N": best["N"], "P": best["P"],
                                       "err": best["err"]},
                               "candidates": sorted(ok, key=lambda r: r["work"])[:2]}
        out[prob] = res
    # the oracle on the cheapest qualifying runs
    import oracle
    nthreads = os.cpu_count() or 1
    spent = 0.0
    for prob, res in out.items():
        mk = W.ex1 if prob == "ex1" else W.ex2
        for eps, e in res.items():
            cands = e.pop("candidates", [])
            best = None
            for c in cands:
                est = c["work"] * 32 * 40e-9 / nthreads              # ~40 ns per tap per core
                if spent + est > oracle_budget_s:
                    continue
                t0 = time.perf_counter()
                o = oracle.Oracle(mk(c["K"], c["N"]), nthreads=nthreads)
                y0, _ = o.solve()
                o.close()
                t = time.perf_counter() - t0
                spent += t
                if best is None or t < best["s"]:
                    best = {"s": t, "K": c["K"], "N": c["N"], "err": abs(y0 - W.reference_solution(mk(1, 16))[0])}
            e["oracle"] = best if best is not None else "not measured (budget)"
    return {"grid": "K=1..6 x N=16..1024, L=32, balanced P (SURVEY A.1), wall time setup+solve",
            "oracle_cores": nthreads, "results": out}


# algorithmic FP64 flops per point-step of the d >= 2 configs (separable evaluation, FMA = 2;
# DESIGN.md §5): per tap F x 4 FMA (last axis) + the staged row/plane passes' share + driver +
# accumulation, K L^d taps, + Picard + spline passes
FLOPS_CFG4 = 4 * 64 * (24 + 3 + 6 + 10) + 2 * 64 + 30 * 8 + 3 * 2 * 21
FLOPS_CFG5 = 3 * 512 * (32 + 4 + 18 + 14) + 2 * 512 + 30 * 22 + 4 * 3 * 21
# cfg 4 through the affine separable path (aff2.cuh): per level and field an axis-0 operator
# (L x (4 interpolation + 2 accumulation) FMA per output) and three axis-1 operators (L x (8 + 3)
# FMA per point) + the combination (6 FMA); Picard 30 x 4 FMA; splines as above
FLOPS_CFG4_AFF = 2 * (4 * 3 * (6 * 8 + 11 * 8 + 6) + 30 * 4) + 3 * 2 * 21
# cfg 5 through the decomposed differential-rates path: per level the per-tap part on U alone
# (L^3 x (4 interpolation FMA + 1 add for 2 max(U, 0) + 2 accumulation FMA; the pair weights
# are applied once per (l0, l1)) + row-pass and plane-stack shares) and the separable affine
# part (3 axis passes over 5 / 6 / 7 arrays); Picard 30 x 22; splines 4 fields x 3 axes x 21
FLOPS_CFG5_DEC = 3 * (13 * 512 + 683 + 320 + 197 * 8 + 12) + 30 * 22 + 4 * 3 * 21


def d23_configs(dev, stream):
    """cfg 4 and cfg 5 at their full sizes: device time of backward steps (after one warm-up
    step) through bsde_step, with the FP64 fraction of the derived peak.  Setup untimed."""
    import torch
    from paper_1909_13560_b200 import Solver, workloads as W
    out = {}
    for name, spec, steps, fl, kv in (("cfg4", W.cfg4(), 3, FLOPS_CFG4_AFF, 0),
                                      ("cfg4_per_tap", W.cfg4(), 3, FLOPS_CFG4, 2),
                                      ("cfg5", W.basket_3d(3, 64, 8, P=512), 2, FLOPS_CFG5_DEC, 0),
                                      ("cfg5_per_tap", W.basket_3d(3, 64, 8, P=512), 2, FLOPS_CFG5, 2)):
        with Solver(spec, device=dev, stream=stream, kernel_variant=kv) as s:
            npts = 1
            for n in s.shape:
                npts *= n
            s.step()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(steps):
                s.step()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / steps
        ups = npts / (ms * 1e-3)
        out[name] = {"workload": spec["name"], "points": npts, "ms_per_step": ms, "updates_per_s": ups,
                     "path": {0: "default" + (" (affine separable, aff2.cuh)" if name == "cfg4"
                                              else " (decomposed driver: quad3d on U + separable affine part)"),
                              2: "per-tap " + ("quad2d" if name.startswith("cfg4") else "quad3d")}[kv],
                     "flops_per_point_step": fl, "tflops": fl * ups / 1e12,
                     "frac_fp64_peak": fl * ups / 1e12 / peak_fp64_tflops(1965.0)}
    return out


def _oracle_sample(max_seconds=15.0, steps_per_K=120, nthreads=None):
    """Time the oracle (as it stands) on a bounded sample of cfg 2: steps_per_K backward
    steps of each K after its (untimed) setup."""
    import oracle
    from paper_1909_13560_b200 import workloads as W
    nthreads = nthreads or os.cpu_count() or 1
    tot_t, tot_u = 0.0, 0
    for K in KS:
        o = oracle.Oracle(W.cfg2(K), nthreads=nthreads)
        for _ in range(steps_per_K):
            t0 = time.perf_counter()
            o.step()
            tot_t += time.perf_counter() - t0
            tot_u += 65536
            if tot_t > max_seconds:
                break
        o.close()
    return tot_u / tot_t, tot_u, tot_t, nthreads


def cpu_baseline(args):
    v, u, t, nt = _oracle_sample()
    v1, u1, t1, _ = _oracle_sample(max_seconds=5.0, steps_per_K=4, nthreads=1)
    return {"value": v, "unit": UNIT, "cores": nt, "kind": "oracle",
            "sample": f"cfg2, up to 120 backward steps per K=1..6 after untimed setup, capped at 15 s "
                      f"({u} updates in {t:.2f} s)",
            "one_thread": {"value": v1, "unit": UNIT, "cores": 1,
                           "sample": f"cfg2, 4 backward steps per K=1..6 ({u1} updates in {t1:.2f} s); "
                                     "comparable to the paper's serial CPU baseline (PAPER.md:458)"}}


def run_reference(args):
    dist, rank, world = _dist()
    if rank != 0:
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return
    for _ in range(args.warmup):
        _oracle_sample(max_seconds=3.0, steps_per_K=1)
    vals, us, ts = [], 0, 0.0
    for _ in range(args.steps):
        v, u, t, nt = _oracle_sample(max_seconds=8.0, steps_per_K=4)
        vals.append(v)
        us += u
        ts += t
    value = us / ts
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ts / args.steps * 1e3, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": {"workload": "cfg2: 1-D differential-rates call, P=65536, N=256, L=16, K=1..6",
                      "global_batch": 65536, "seq_len": 256, "parallelism": "host cores (OpenMP)"},
           "cpu_baseline": {"value": value, "unit": UNIT, "kind": "oracle", "cores": os.cpu_count(),
                            "sample": "each step: 4 backward steps of each K=1..6 of cfg2 (setup untimed)"},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tts", action="store_true", help="skip the time-to-solution sweep")
    ap.add_argument("--no-d23", action="store_true", help="skip the cfg 4 / cfg 5 step timings")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
