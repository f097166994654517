"""Top SASS instructions by warp-stall samples from an ncu report (profiling aid).
  python tools/ncu_sass_hot.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
data = []
tot = 0
for r in rows[1:]:
    if len(r) < len(h):
        continue
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    tot += s
    data.append((s, r))
data.sort(key=lambda x: -x[0])
print(f"total samples {tot}")
for s, r in data[:top]:
    st = sorted(((int(r[ix[k]] or 0), k[6:]) for k in stalls), reverse=True)[:3]
    print(f"{100.0 * s / tot:5.1f}% {r[ix['Source']].strip()[:60]:60s} exec={r[ix['Instructions Executed']]:>10s} " +
          " ".join(f"{k}={v}" for v, k in st if v))
