"""Warp-stall samples aggregated by CUDA source line (file:line) from an ncu report
(profiling aid; needs -lineinfo and --import-source).  python tools/ncu_line_hot.py rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
res = []
fname = "?"
hdr = None
for line in out.splitlines():
    if line.startswith('"File Path"'):
        fname = next(csv.reader(io.StringIO(line)))[1].rsplit("/", 1)[-1]
        continue
    if line.startswith('"Line No"'):
        hdr = next(csv.reader(io.StringIO(line)))
        continue
    if hdr is None or line.startswith('"Function Name"'):
        continue
    r = next(csv.reader(io.StringIO(line)))
    if len(r) < len(hdr) or not r[0]:
        continue
    ix = {k: i for i, k in enumerate(hdr) if k}
    num = lambda x: int(x) if x.strip().lstrip("-").isdigit() else 0
    s = num(r[4])
    stalls = sorted(((num(r[i]), k[6:]) for k, i in ix.items() if k.startswith("stall_") and "Not Issued" not in k), reverse=True)[:3]
    res.append((s, f"{fname}:{r[0]}", r[1].strip()[:70], num(r[7]), stalls))
tot = sum(x[0] for x in res) or 1
res.sort(key=lambda x: -x[0])
print(f"total samples {tot}")
for s, loc, src, ex, st in res[:top]:
    print(f"{100.0 * s / tot:5.1f}% {loc:22s} {src:70s} inst={ex:>11d} " + " ".join(f"{k}={v}" for v, k in st if v))
