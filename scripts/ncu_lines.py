"""Aggregate an ncu source page (--print-source=cuda,sass --csv) to per-source-line stall samples.
usage: ncu -i X.ncu-rep --page source --csv --print-source=cuda,sass > x.csv; python ncu_lines.py x.csv [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
out = []
fname = "?"
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0]:
        continue
    try:
        samp = int(r[4])
    except (ValueError, IndexError):
        continue
    stalls = {}
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                v = int(r[i])
            except ValueError:
                continue
            if v:
                stalls[h[6:]] = v
    top = sorted(stalls.items(), key=lambda x: -x[1])[:4]
    out.append((samp, fname, r[0], r[1].strip()[:70], top))
tot = sum(o[0] for o in out)
print("total samples", tot)
for s, f, ln, src, top in sorted(out, key=lambda o: -o[0])[:N]:
    print(f"{100*s/tot:5.1f}% {f}:{ln:>4} {src:70s} {' '.join(f'{k}={v}' for k, v in top)}")
