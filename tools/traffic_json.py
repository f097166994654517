"""DRAM traffic of one solver launch, from an ncu metrics CSV (profiling aid).

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
      -k regex:smo_ -c 1 --csv --log-file t.csv python tools/one_solve.py W2
  python tools/traffic_json.py t.csv W2 profiles/traffic_W2.json

bench.py reads the JSON as the roofline's "traffic" (per launch = one whole solve)."""
import csv
import json
import sys


def main(src, workload, out, iterations=None):
    vals, kernel = {}, None
    with open(src) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    for r in csv.DictReader(lines):
        kernel = r.get("Kernel Name", kernel)
        name, unit, v = r.get("Metric Name"), r.get("Metric Unit"), r.get("Metric Value", "").replace(",", "")
        try:
            x = float(v)
        except ValueError:
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
                 "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6, "s": 1e3, "second": 1e3}.get(unit, 1)
        vals[name] = x * scale
    rd, wr = vals.get("dram__bytes_read.sum", 0.0), vals.get("dram__bytes_write.sum", 0.0)
    short = kernel.split("(")[0].replace("void ", "").replace("svmk::", "").replace(" ", "") if kernel else None
    res = {"kernel": short, "workload": workload, "dram_bytes_per_launch": int(rd + wr),
           "iterations": int(iterations) if iterations else None,
           "dram_bytes_per_iter": (rd + wr) / int(iterations) if iterations else None,
           "dram_read": int(rd), "dram_write": int(wr), "duration_ms": vals.get("gpu__time_duration.sum"),
           "note": "ncu --metrics dram__bytes_{read,write}.sum of one solver launch (the given iterations)", "source": src}
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main(*sys.argv[1:5])
