ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_cfg5_dec.csv python scripts/step_probe.py cfg5 1 0 512 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/launches_cfg5_dec.csv")))
hdr = None
agg = collections.defaultdict(lambda: collections.defaultdict(float)); cnt = collections.Counter()
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if not hdr or len(r) != len(hdr): continue
    d = dict(zip(hdr, r)); k = d["Kernel Name"].split("(")[0][:40]
    try: v = float(d["Metric Value"].replace(",", ""))
    except ValueError: continue
    agg[k][d["Metric Name"]] += v; cnt[(k, d["Metric Name"])] += 1
for k, m in agg.items():
    n = cnt[(k, "gpu__time_duration.sum")]
    print(k, "launches", n, "total_ms", round(m["gpu__time_duration.sum"] / 1e6, 3), {mm: round(v / max(cnt[(k, mm)], 1), 3) for mm, v in m.items() if mm != "gpu__time_duration.sum"})
PY
