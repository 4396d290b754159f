"""Extract the metrics DESIGN.md / bench.py cite from an ncu report into a JSON summary.
usage: python scripts/ncu_summary.py X.ncu-rep out.json [kernel-regex]"""
import csv, io, json, re, subprocess, sys
KEYS = ["gpu__time_duration.sum", "sm__cycles_active.avg", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]
rep, out = sys.argv[1], sys.argv[2]
pat = re.compile(sys.argv[3]) if len(sys.argv) > 3 else None
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, units = rows[0], rows[1]
res = {}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    if pat and not pat.search(name):
        continue
    d = {}
    for i, h in enumerate(hdr):
        if h in KEYS or h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            d[h] = r[i]
            if units[i]:
                d[h + ".unit"] = units[i]
    res[name[:60]] = d
    break
json.dump(res[next(iter(res))] if len(res) == 1 else res, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in list(res.values())[0].items() if not k.endswith(".unit")}, indent=0)[:2500])
