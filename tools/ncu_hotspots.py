"""Per-source-line hotspots of an ncu report (profiling aid).

  ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
  python tools/ncu_hotspots.py src.csv [top]

Prints the source lines with the most warp-stall samples, their share, executed
instructions and the two largest stall reasons."""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    out = []
    hdr = None
    fname = ""
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr) or r[2] != "-":
            continue
        d = dict(zip(hdr, r))
        try:
            smp = int(d["Warp Stall Sampling (All Samples)"])
        except ValueError:
            continue
        stalls = sorted(((int(d[k]), k) for k in hdr if k.startswith("stall_") and "Not Issued" not in k
                         and d[k].isdigit()), reverse=True)[:2]
        out.append((smp, fname, int(d["Line No"]), r[1].strip()[:70], d["Instructions Executed"], stalls))
    tot = sum(o[0] for o in out) or 1
    for smp, f, ln, src, ins, st in sorted(out, reverse=True)[:top]:
        print(f"{f[:14]:>14}:{ln:<5} {100.0 * smp / tot:5.1f}% inst={ins:>11}  {src:<70} "
              + " ".join(f"{k}={v}" for v, k in st))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
