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
P_CFG2, N_CFG2, L_CFG2 = 65536, 256, 16


def survey_ops(K, L, d, F_f, p=30.0):
    """Algorithmic FP64 work per point-step, SURVEY.md §8(d) as written (FMA = 1 op):
    K L^d (F 4^d + F_f + 2d + 1) + p (F_f + 2) + 2 K d + 10 F,  F = 1 + d.
    F_f: FP64 ops of one driver evaluation (differential rates 1-D: 5)."""
    F = 1 + d
    return K * L ** d * (F * 4 ** d + F_f + 2 * d + 1) + p * (F_f + 2) + 2 * K * d + 10 * F


def fp64_pipe_peak(sm_mhz=1965.0, nsm=148):
    """FP64 pipe ops/s (FMA = 1 op): 148 SM x 64 DFMA lanes per clock (B200_PROFILING.md: 148 SMs,
    1965 MHz max; the 64 DFMA/clk/SM of sm_100 confirmed by ncu's
    sm__sass_thread_inst_executed_op_dfma_pred_on.avg.peak_sustained), in units of 1e12."""
    return nsm * 64 * sm_mhz * 1e6 / 1e12


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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
        pexec = sum(r.picard_iters for r in res)
        # one batched launch is counted by every context; the rest are the y0 evaluations
        launches = 1 + sum(s.kernel_launches - a - 1 for s, a in zip(ss, n0))
        y0 = {K: (r.y0, r.z0[0]) for K, r in zip(KS, res)}
        for s in ss:
            s.close()
        return t, upd, launches, y0, pexec

    for _ in range(args.warmup):
        one_step()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    times, upds, launches, pexecs = [], 0, 0, 0
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            t, u, nl, y0, pe = one_step()
            times.append(t)
            upds += u
            launches += nl
            pexecs += pe
    torch.cuda.synchronize()
    elapsed = sum(times)
    if dist:
        tt = torch.tensor([elapsed], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed = float(tt.item())
    value = upds * world / elapsed

    # ---- roofline of the dominant kernel, quad1d_fused: ONE persistent launch per bench step runs
    # all six sweeps (round-robin over the problems); its average duration is the CUDA-event time of
    # the launches of the timed region (recorded on `stream` inside bsde_solve_batch).  Algorithmic
    # work: SURVEY §8(d)'s per-point-step FP64 op count as written (FMA = 1 op, p = 30 Picard
    # iterations, differential-rates driver F_f = 5) x the point-steps of one launch.
    launch_s = elapsed / args.steps
    pts = {K: P_CFG2 * (N_CFG2 - K + 1) for K in KS}
    ops = sum(survey_ops(K, L_CFG2, 1, 5) * pts[K] for K in KS)
    p_exec = pexecs / max(args.steps, 1) / sum(pts.values())          # mean executed Picard iterations
    ops_exec = sum(survey_ops(K, L_CFG2, 1, 5, p=p_exec) * pts[K] for K in KS)
    clocks = clk.summary()
    peak = fp64_pipe_peak(1965.0)
    achieved = ops / launch_s / 1e12
    traffic = None
    prof = _load_profile("ncu_quad1d_fused_batch_summary.json")
    if prof:   # dram__bytes_read.sum + dram__bytes_write.sum per launch, from the committed ncu --set full capture
        traffic = _dram_bytes(prof)
    roof = {"bound": "alu", "achieved": round(achieved, 3), "peak": round(peak, 3), "unit": "TFLOP/s",
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "unit_note": "FP64-pipe ops/s, FMA = 1 op (SURVEY §8(d) convention); peak = 148 SM x 64 DFMA lanes/clk "
                         "x 1965 MHz (B200_PROFILING.md SM count and max clock; no FP64 figure in MEASURED_PEAKS.json)",
            "kernel": "quad1d_fused<DRV_DIFF>: one launch = the 6 sweeps K=1..6 (1521 steps)",
            "ops_per_launch": ops, "launch_us": round(launch_s * 1e6, 3),
            "ops_formula": "K L (F 4 + F_f + 2d + 1) + p (F_f + 2) + 2 K d + 10 F, d=1, F=2, F_f=5, L=16, p=30",
            "executed_picard": {"mean_iterations": round(p_exec, 3),
                                "frac": round(ops_exec / launch_s / 1e12 / peak, 4),
                                "note": "the same formula with p = the Picard iterations the kernel executed "
                                        "(it leaves the loop at an exact fixed point; bsde_result.picard_iters)"},
            "traffic_note": "DRAM bytes per launch (the state is L2-resident) from ncu --set full, profiles/round2"}
    if clocks.get("sm_mhz"):
        roof["frac_at_sampled_clock"] = round(achieved / fp64_pipe_peak(float(clocks["sm_mhz"])), 4)
    try:   # the same denominator measured: a DFMA-chain kernel of the library (bsde_measure_fp64_peak)
        from paper_1909_13560_b200 import measure_fp64_peak
        mp = measure_fp64_peak(dev)
        roof["peak_measured"] = {"value": round(mp["tflops"] / 2, 3), "unit": "T op/s (FMA = 1)",
                                 "frac_of_measured": round(achieved / (mp["tflops"] / 2), 4),
                                 "note": "16 independent DFMA chains/thread, 8 x 256-thread CTAs per SM"}
    except Exception as exc:  # noqa: BLE001 -- reported, never fatal for the bench line
        roof["peak_measured"] = {"error": str(exc)}

    # ---- e2e: setup (host config -> device) + sweep + final layers device -> host, host clock
    host = np.empty(P_CFG2, dtype=np.float64)
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
            d2h += 2 * P_CFG2 * 8 + 32                      # y, z of layer 0 + y0/z0
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
                      "global_batch": P_CFG2 * world, "seq_len": N_CFG2, "parallelism": f"replicas{world}",
                      "l2": "flushed (512 MiB write) before every step; the six sweeps' state (~50 MiB) is L2-resident by design"},
           "roofline": roof, "e2e": e2e, "gpu_launches": launches // max(args.steps, 1),
           "clocks": clocks,
           "accuracy": {str(K): {"y0": y0[K][0], "z0": y0[K][1],
                                 "note": "K >= 3 at P = 2^16, L = 16 is linearly unstable (DESIGN.md R25); see cfg2_stable"}
                        for K in KS},
           "reference_solution": list(W.reference_solution(specs[1])[:1]) + [W.reference_solution(specs[1])[1][0]]}
    if rank == 0 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args)
    if rank == 0 and world == 1:
        out["cfg2_stable"] = cfg2_stable(dev, stream)
        out["cfg1_latency"] = cfg1_latency(dev, stream)
    if rank == 0 and not args.no_tts:
        out["tts"] = tts_sweep(dev)
    if rank == 0 and world == 1 and not args.no_d23:
        out["d23_configs"] = d23_configs(dev, stream)
    if rank == 0:
        print(json.dumps(out))
    if dist:
        dist.barrier()
        dist.destroy_process_group()


PROFILE_DIRS = ("round2", "round1")


def _load_profile(name):
    for d in PROFILE_DIRS:
        try:
            with open(os.path.join(ROOT, "profiles", d, name)) as fh:
                return json.load(fh)
        except (OSError, ValueError):
            continue
    return None


def _dram_bytes(prof):
    """dram__bytes_read.sum + dram__bytes_write.sum of an ncu summary, in bytes."""
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    try:
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(prof[k]) * scale.get(prof.get(k + ".unit", "byte"), 1.0)
        return tot
    except (KeyError, ValueError):
        return None


def cfg2_stable(dev, stream):
    """The stable companion of cfg 2 (R25): the same problem at P = 16385 (stable for
    every K with L = 16), all six sweeps in one batched launch: throughput and accuracy per K."""
    from paper_1909_13560_b200 import Solver, solve_batch, workloads as W
    P = 16385
    specs = [dict(W.diff_rates(K, N=N_CFG2, P=P), name=f"cfg2_stable_K{K}") for K in KS]
    ref = W.reference_solution(specs[0])
    best, acc = None, None
    for _ in range(3):
        ss = [Solver(sp, device=dev, stream=stream) for sp in specs]
        res = solve_batch(ss)
        t = res[0].t_sweep_s
        if best is None or t < best[0]:
            best = (t, sum(r.updates for r in res))
            acc = {str(K): {"y0_err": abs(r.y0 - ref[0]), "z0_err": abs(r.z0[0] - ref[1][0])} for K, r in zip(KS, res)}
        for s in ss:
            s.close()
    return {"workload": "cfg2 shape at P=16385 (stable for all K, DESIGN.md R25), N=256, L=16, K=1..6 batched",
            "ms": best[0] * 1e3, "updates_per_s": best[1] / best[0], "accuracy": acc}


def cfg1_latency(dev, stream):
    """BASELINE cfg 1 (Black-Scholes, P=256, K=2, N=32, L=8) as a latency path: device time of
    the sweep (bsde_solve) and wall time of setup + solve, best of 5."""
    from paper_1909_13560_b200 import Solver, workloads as W
    spec = W.cfg1()
    sweep, wall = 1e9, 1e9
    for _ in range(5):
        t0 = time.perf_counter()
        with Solver(spec, device=dev, stream=stream) as s:
            r = s.solve()
            launches = s.kernel_launches
        wall = min(wall, time.perf_counter() - t0)
        sweep = min(sweep, r.t_sweep_s)
    return {"workload": spec["name"], "sweep_us": sweep * 1e6, "setup_plus_solve_ms": wall * 1e3,
            "kernel_launches": launches, "y0": r.y0}


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


# Per-kernel rooflines of the d >= 2 configs (committed ncu --set full summaries, profiles/round2):
# FP64-pipe kernels report ncu's sm__pipe_fp64_cycles_active (the executed FP64 work per cycle),
# HBM kernels their algorithmic bytes (8 B read + 8 B write per point, field and pass) / duration
# against MEASURED_PEAKS.json's copy bandwidth.
D23_KERNELS = {
    "cfg4": [("aff_rows", "ncu_aff_rows_cfg4_summary.json", "alu"),
             ("spline_rf<strided>", "ncu_spline_rf_strided_cfg4_summary.json", "hbm"),
             ("spline_rf<contiguous>", "ncu_spline_rf_contig_cfg4_summary.json", "hbm")],
    "cfg5": [("quad3d<DRV_DIFF,1>", "ncu_quad3d_dec_cfg5_summary.json", "alu"),
             ("spline_rf<strided>", "ncu_spline_rf_strided_cfg5_summary.json", "hbm"),
             ("spline_rf<contiguous>", "ncu_spline_rf_contig_cfg5_summary.json", "hbm")],
}


def _hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        return 6650.0, "B200_PROFILING.md fallback"


def kernel_rooflines(cfg, points):
    out = []
    hbm, hbm_src = _hbm_peak()
    for kname, fname, bound in D23_KERNELS.get(cfg, []):
        prof = _load_profile(fname)
        if not prof:
            out.append({"kernel": kname, "profile": None, "note": f"profiles/round2/{fname} not captured"})
            continue
        dur = float(prof["gpu__time_duration.sum"]) * {"ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3,
                                                         "ns": 1e-9, "nsecond": 1e-9}.get(prof.get("gpu__time_duration.sum.unit", "ms"), 1e-3)
        ent = {"kernel": kname, "launch_us": dur * 1e6, "traffic": _dram_bytes(prof), "profile": fname}
        if bound == "alu":
            pct = float(prof["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"])
            ent.update({"bound": "alu", "frac": round(pct / 100.0, 4), "unit": "TFLOP/s",
                        "peak": round(fp64_pipe_peak(), 3),
                        "achieved": round(pct / 100.0 * fp64_pipe_peak(), 3),
                        "note": "executed FP64-pipe utilisation of the launch (ncu sm__pipe_fp64_cycles_active, "
                                "FMA = 1 op)"})
        else:
            alg = points * 16.0                       # 8 B read + 8 B write per point of one field-pass
            ach = alg / dur / 1e9
            ent.update({"bound": "hbm", "unit": "GB/s", "achieved": round(ach, 1), "peak": hbm,
                        "frac": round(ach / hbm, 4), "peak_source": hbm_src,
                        "note": "algorithmic bytes of one field-pass (16 B per point) / ncu duration"})
        out.append(ent)
    return out


def d23_configs(dev, stream):
    """cfg 4 and cfg 5 at their full sizes: device time of backward steps (after one warm-up
    step) through bsde_step, the survey's direct-stencil op count per point-step over that time,
    and the per-kernel rooflines of the committed ncu captures.  Setup untimed."""
    import torch
    from paper_1909_13560_b200 import Solver, workloads as W
    out = {}
    runs = (("cfg4", W.cfg4(), 3, 0, 3, "default: affine separable path (aff2.cuh)"),
            ("cfg4_per_tap", W.cfg4(), 3, 2, 3, "per-tap quad2d"),
            ("cfg4_fd_bicubic", dict(W.cfg4(), interp="fd_bicubic"), 1, 0, 3,
             "the paper's FD-bicubic interpolation (bicubic.cuh, one thread per point)"),
            ("cfg5", W.basket_3d(3, 64, 8, P=512), 2, 0, 9, "default: decomposed driver (quad3d on U + separable affine part)"),
            ("cfg5_per_tap", W.basket_3d(3, 64, 8, P=512), 1, 2, 9, "per-tap quad3d"))
    for name, spec, steps, kv, F_f, path in runs:
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
        d = spec["d"]
        K = max(spec["Ky"], spec["Kz"])
        ops = survey_ops(K, spec["L"], d, F_f)
        out[name] = {"workload": spec["name"], "points": npts, "ms_per_step": ms, "updates_per_s": ups, "path": path,
                     "survey_ops_per_point_step": ops,
                     "survey_ops_frac": round(ops * ups / 1e12 / fp64_pipe_peak(), 4),
                     "survey_ops_note": "SURVEY §8(d) direct-stencil op count / step time / FP64-pipe peak; the "
                                        "separable paths execute fewer ops than the direct form (can exceed 1)"}
        if name in D23_KERNELS:
            out[name]["kernels"] = kernel_rooflines(name, npts)
    return out


ORACLE_STEPS_PER_K = 8      # one oracle sample: 8 backward steps of each K = 1..6 of cfg 2 (setup untimed)


def oracle_sample(nthreads=None, steps_per_K=ORACLE_STEPS_PER_K):
    """ONE sampling protocol for both arms: the oracle (as it stands, OpenMP over all host cores)
    on a bounded sample of the cfg 2 workload -- steps_per_K backward steps of each K after its
    (untimed) setup.  Returns (updates, seconds, threads)."""
    import oracle
    from paper_1909_13560_b200 import workloads as W
    nthreads = nthreads or os.cpu_count() or 1
    tot_t, tot_u = 0.0, 0
    for K in KS:
        o = oracle.Oracle(W.cfg2(K), nthreads=nthreads)
        t0 = time.perf_counter()
        for _ in range(steps_per_K):
            o.step()
        tot_t += time.perf_counter() - t0
        tot_u += P_CFG2 * steps_per_K
        o.close()
    return tot_u, tot_t, nthreads


def _sample_text(n):
    return (f"{n} sample(s) of {ORACLE_STEPS_PER_K} backward steps of each K=1..6 of cfg2 (P=65536, L=16) after "
            f"untimed setup; host CPU: {cpu_model()}")


def cpu_baseline(args, budget_s=10.0):
    us, ts, n, nt = 0, 0.0, 0, 1
    while ts < budget_s or n < 1:
        u, t, nt = oracle_sample()
        us, ts, n = us + u, ts + t, n + 1
    u1, t1, _ = oracle_sample(nthreads=1, steps_per_K=1)
    return {"value": us / ts, "unit": UNIT, "cores": nt, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": _sample_text(n) + f" ({us} updates in {ts:.2f} s)",
            "one_thread": {"value": u1 / t1, "unit": UNIT, "cores": 1,
                           "sample": f"1 backward step of each K, 1 thread ({u1} updates in {t1:.2f} s); comparable "
                                     "to the paper's serial CPU baseline (PAPER.md:458)"}}


def run_reference(args):
    """--impl reference: the oracle, as it stands, on the host cores; each bench step is one
    oracle sample (the protocol of cpu_baseline) of the same cfg 2 workload."""
    dist, rank, world = _dist()
    if rank != 0:
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return
    for _ in range(args.warmup):
        oracle_sample(steps_per_K=1)
    us, ts, nt = 0, 0.0, 1
    for _ in range(args.steps):
        u, t, nt = oracle_sample()
        us += u
        ts += t
    value = us / ts
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ts / args.steps * 1e3, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": {"workload": "cfg2: 1-D differential-rates call, P=65536, N=256, L=16, K=1..6",
                      "global_batch": P_CFG2, "seq_len": N_CFG2, "parallelism": "host cores (OpenMP)"},
           "cpu_baseline": {"value": value, "unit": UNIT, "kind": "oracle", "cores": nt, "cpu_model": cpu_model(),
                            "sample": _sample_text(args.steps)},
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
