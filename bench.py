"""bench.py -- SVM train time-to-converge on B200 (BASELINE.json metric), one JSON line.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload W5]

Headline workload: W5 (BASELINE.json configs[4], the "1/2/4/8 GPUs" scaling config,
n = 1,000,000, d = 256, RBF).  `value` = the time-to-converge of the SMO solve (seconds,
lower is better) on inputs already resident in HBM, measured with CUDA events on the
launching stream, max over ranks.

Steps.  One W5 solve is ~4*10^5 SMO iterations (~1 minute), so a step is one contiguous
window of that solve: the library runs the solve as K persistent launches of
ceil(T / K) iterations each (svm_params.iters_per_launch; T = the trajectory's iteration
count, deterministic), and the timed region -- barrier + synchronize on
both sides -- is the whole solve from device-resident X to alpha and b: validation,
staging (a1), the K launches (a2-a7) and finalisation (a10).  `value` = the sum of the K
windows = time-to-converge; `ms_per_step` = value / K.  The W warm-up steps are the first
W windows of a separate solve (same launch configuration).  Small workloads (--workload
W1..W3) instead time K whole solves (`value` = their mean).

`e2e` = the same solve through the host C-ABI call (svm_train_ex, host buffers, H2D of X
and y and D2H of alpha inside the timed region).  Extra keys: the batched prediction of
the 1M held-out rows on the tensor cores (a11), the time-to-converge of W2-W4, the
projected-GD trainer, and the CPU oracle timed on a bounded sample (`cpu_baseline`).

N > 1 is launched by torchrun (one process per GPU): the rows are sharded and every
iteration exchanges per-CTA candidate records over NVLink (strong scaling: the problem
is fixed).  --impl reference times the CPU oracle (oracle/) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SVM train time-to-converge (s) & SMO iters/s at 1/2/4/8 B200; kernel-row HBM GB/s"

# Iteration counts of the deterministic trajectories (the oracle and the GPU
# take the same steps).  Used only to size the windows of a step; if a solve takes a
# different count, the number of launches (reported as `launches`) differs from K.
PLAN_ITERS = {"W1": 150, "W2": 42790, "W3": 11659, "W4": 133952, "W5": 411469}
WINDOWED = ("W4", "W5")


def peaks():
    """(HBM GB/s, bf16 dense TF/s, kind) from the driver-written MEASURED_PEAKS.json."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), float(p.get("bf16_tflops", 2250.0)), "measured"
    except Exception:
        return 6650.0, 2250.0, "fallback"


def cpu_model() -> str:
    try:
        out = subprocess.check_output(["lscpu"], timeout=10).decode()
        for ln in out.splitlines():
            if ln.startswith("Model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


class Clocks:
    """Samples SM clocks and throttle reasons during the timed region (NVML in-process;
    B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _nvml_row(self, pynvml, h):
        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        bits = [0x8, 0x40, 0x20, 0x4]       # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
        return [str(self.index), str(sm), str(mx), str(pw), hex(r)] + \
               ["Active" if r & b else "Not Active" for b in bits]

    def __enter__(self):
        def run():
            nv = None
            try:
                import pynvml
                pynvml.nvmlInit()
                nv = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index))
            except Exception:
                nv = None
            while not self._stop.is_set():
                try:
                    if nv is not None:
                        self.rows.append(self._nvml_row(*nv))
                    else:
                        out = subprocess.check_output(
                            ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                             "--format=csv,noheader,nounits"], timeout=5).decode().strip()
                        self.rows.append([c.strip() for c in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.5)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def oracle_sample(w, X, y, budget_s: float, iters_total: int):
    """Time the oracle as it stands on the head of this workload's trajectory, about
    budget_s seconds of CPU work; returns (iters/s, iterations run, threads)."""
    from oracle import oracle as O
    t0 = time.perf_counter()
    O.train(X, y, w.C, w.kernel, w.gamma, w.tol, max_iter=2)
    probe = max(time.perf_counter() - t0, 1e-6) / 2
    k = int(max(2, min(iters_total, budget_s / probe)))
    t0 = time.perf_counter()
    r = O.train(X, y, w.C, w.kernel, w.gamma, w.tol, max_iter=k)
    dt = time.perf_counter() - t0
    return r.iterations / dt, r.iterations, O.num_threads()


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    """The CPU oracle (the tier's reference arm), as it stands, on the bench workload:
    each step times a bounded sample of its trajectory (~args.ref_budget s, capped so
    the whole run stays within a few minutes); value = the time-to-converge projected
    from the sampled iteration rate."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from gen import workloads as W
    w = W.get(args.workload)
    X, y = w.train()
    iters = PLAN_ITERS.get(w.name)
    budget = min(args.ref_budget, 150.0 / max(1, args.steps + args.warmup))
    per_step = []
    k_iters = 0
    threads = 1
    for s in range(args.warmup + args.steps):
        ips, k, threads = oracle_sample(w, X, y, budget, iters or 10 ** 9)
        if s >= args.warmup:
            per_step.append(ips)
            k_iters = k
    ips = statistics.mean(per_step)
    value = (iters / ips) if iters else None
    sample = (f"first {k_iters} SMO iterations of {w.name} (n={w.n}) per step on {threads} host threads "
              f"({cpu_model()}); time-to-converge projected to the trajectory's {iters} iterations")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * value / args.steps if value else None, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{w.name}: {w.config}", "n": w.n, "d": w.d},
        "smo_iters_per_s": ips,
        "cpu_baseline": {"value": value, "unit": "s", "cores": threads, "kind": "oracle",
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2311_14908_b200 as S
    from gen import workloads as W

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook (SVMB200_BENCH_HOSTCOMM=1): several ranks on the GPUs there are (possibly
    # one), bootstrapped over gloo + svm_comm_init_host instead of NCCL, to exercise the N > 1
    # path of this script where NCCL refuses to run (two ranks on one device)
    hostcomm = os.environ.get("SVMB200_BENCH_HOSTCOMM") == "1"
    if hostcomm:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cdev = torch.device("cpu") if hostcomm else dev       # the collectives' device
    if world > 1:
        if hostcomm:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    S.lib()
    hbm, bf16, peak_kind = peaks()
    w = W.get(args.workload)
    X, y = w.train()
    n, d = X.shape
    blocks = S.shard_rows(n, world)
    lo, hi = blocks[rank]
    stream = torch.cuda.current_stream()
    Xd_full = torch.from_numpy(X).to(dev)
    yd_full = torch.from_numpy(y).to(dev)
    Xl = Xd_full[lo:hi].contiguous() if world > 1 else Xd_full
    yl = yd_full[lo:hi].contiguous() if world > 1 else yd_full
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > L2 (126 MB)
    comm = None
    if world > 1:
        if hostcomm:
            comm = S.svm_comm_init_host(rank, world, local)
        else:
            from paper_2311_14908_b200.dist import broadcast_uid
            uid = broadcast_uid(S.svm_comm_unique_id() if rank == 0 else None, dev)
            comm = S.svm_comm_init(rank, world, uid, local)

    windowed = (w.name in WINDOWED or args.windowed) and w.name in PLAN_ITERS
    window = math.ceil(PLAN_ITERS[w.name] / args.steps) if windowed else 0

    def train(**kw):
        if world == 1:
            return S.svm_train_dev(Xd_full, yd_full, w.C, w.kernel, w.gamma, w.tol, stream=stream, **kw)
        return S.svm_train_shard(comm, Xl, yl, lo, n, w.C, w.kernel, w.gamma, w.tol, stream=stream, **kw)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def gmax(v):
        if world > 1:
            from paper_2311_14908_b200.dist import max_over_ranks
            return max_over_ranks(v, cdev)
        return v

    # ---- warm-up: the first W windows of a solve (windowed) / W whole solves
    if windowed:
        if args.warmup > 0:
            train(iters_per_launch=window, max_iter=args.warmup * window)
    else:
        for _ in range(args.warmup):
            train()
    barrier()

    # ---- timed: one solve in K windows (windowed) / K whole solves
    launches0 = S.kernel_launches()
    infos = []
    with Clocks(local) as clk:
        flush.fill_(1.0)                               # L2 flush before the timed region
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        if windowed:
            e0.record(stream)
            r = train(iters_per_launch=window)
            e1.record(stream)
            infos.append(r["info"])
            barrier()
            t_total = e0.elapsed_time(e1) * 1e-3
            t_step = t_total / args.steps
        else:
            ts = []
            for k in range(args.steps):
                flush.fill_(float(k))                  # L2 flush between steps
                e0.record(stream)
                r = train()
                e1.record(stream)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e-3)
                infos.append(r["info"])
            barrier()
            t_total = statistics.mean(ts)
            t_step = t_total
    our_launches = S.kernel_launches() - launches0
    plan = S.last_plan()
    info = infos[-1]
    iters = info["iterations"]
    value = gmax(t_total)
    step_ms = gmax(t_step) * 1e3                       # (collectives: every rank, before the rank-0 block)
    solve_s = gmax(statistics.mean(i["seconds_solve"] for i in infos))
    alpha_last, b_last = r["alpha"], r["b"]

    # ---- roofline of the dominant kernel, the persistent solver launch (~98% of the step):
    # algorithmic bytes per iteration (miss path) n_r (4 d_p + 25) -- the
    # fp32 X rows, f read + write, the status byte -- times the iterations of one launch,
    # over the average launch duration (device events around the launch loop / launches).
    n_r = hi - lo
    d_p = (d + 3) // 4 * 4
    bytes_iter = n_r * (4 * d_p + 25)
    per_launch_s = info["seconds_solve"] / max(1, info["launches"])
    it_per_launch = iters / max(1, info["launches"])
    achieved = bytes_iter * it_per_launch / per_launch_s / 1e9
    traffic = None
    traffic_note = None
    tp = os.path.join(ROOT, "profiles", f"traffic_{w.name}.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            if tj.get("kernel", "").split("<")[0] == plan.get("kernel", "").split("<")[0]:
                if tj.get("dram_bytes_per_iter"):
                    traffic = int(tj["dram_bytes_per_iter"] * it_per_launch)
                    traffic_note = (f"ncu dram__bytes_read.sum + dram__bytes_write.sum per iteration "
                                    f"({tj['dram_bytes_per_iter']:.4g} B, {tj.get('iterations')} iterations "
                                    f"captured, {tj.get('source')}) x iterations per launch")
                else:
                    traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic, "peak_kind": peak_kind, "kernel": plan.get("kernel"),
                "bytes_per_iter": bytes_iter, "iters_per_launch": it_per_launch,
                "launch_ms": per_launch_s * 1e3}
    if traffic:
        roofline["frac_measured_traffic"] = traffic / per_launch_s / 1e9 / hbm
        roofline["traffic_note"] = traffic_note
    hbm_eff = None
    if plan.get("mode") == "binary-resident":
        # X resident in shared memory as bit rows: no HBM stream; the POPC pipe of the SMs the
        # solver occupies bounds the row pass
        Wd = (d + 31) // 32
        sms = int(plan.get("ctas_per_rank", 1)) * int(plan.get("ranks", 1))
        mhz = clk.summary().get("sm_mhz") or 1965.0
        popc_iter = n_r * 2 * Wd
        alu_ach = popc_iter * it_per_launch / per_launch_s / 1e9
        alu_peak = 16 * sms * mhz * 1e6 / 1e9
        hbm_eff = dict(roofline, effective=True,
                       note="fp32-equivalent algorithmic bytes; served from shared memory as bit rows")
        roofline = {"bound": "alu", "pipe": "POPC, 16/clk/SM x %d SMs x %.0f MHz" % (sms, mhz),
                    "achieved": alu_ach, "peak": alu_peak, "unit": "Gpopc/s", "frac": alu_ach / alu_peak,
                    "frac_whole_chip": alu_ach / (16 * 148 * mhz * 1e6 / 1e9),
                    "traffic": traffic, "kernel": plan.get("kernel"), "ops_per_iter": popc_iter,
                    "latency_bound": True}

    # ---- e2e: the same solve through the host C-ABI (host X / y, H2D + D2H timed)
    e2e = None
    if world == 1 and not args.no_e2e:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rr = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, iters_per_launch=window)
        e2e_s = time.perf_counter() - t0
        e2e = {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": int(n * d * 4 + n),
               "d2h_bytes_per_step": int(n * 8),
               "api": "svm_train_ex (host pointers: X, y in; alpha, b out)",
               "iterations": rr["info"]["iterations"], "seconds_h2d": rr["info"].get("seconds_h2d")}
    elif world > 1 and not args.no_e2e:
        Xh = torch.from_numpy(X[lo:hi]).pin_memory()
        yh = torch.from_numpy(y[lo:hi]).pin_memory()
        ah = torch.empty(hi - lo, dtype=torch.float64).pin_memory()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        Xl.copy_(Xh, non_blocking=True); yl.copy_(yh, non_blocking=True)
        rr = train(iters_per_launch=window)
        ah.copy_(rr["alpha"], non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e = {"value": gmax(e0.elapsed_time(e1) * 1e-3), "unit": "s",
               "h2d_bytes_per_step": int((hi - lo) * (d * 4 + 1)), "d2h_bytes_per_step": int((hi - lo) * 8),
               "api": "svm_train_shard (pinned host -> device copies in the timed region)"}

    # ---- time-to-converge of the other configs (one warm + one timed whole solve each)
    others = None
    if world == 1 and not args.no_others:
        others = []
        for name, extra in (("W2", {}), ("W3", {}), ("W4", {}), ("W3", {"wss": 2})):
            if name == w.name and not extra:
                continue
            wo = W.get(name)
            Xo, yo = wo.train()
            Xo_d, yo_d = torch.from_numpy(Xo).to(dev), torch.from_numpy(yo).to(dev)
            S.svm_train_dev(Xo_d, yo_d, wo.C, wo.kernel, wo.gamma, wo.tol, stream=stream, **extra)
            flush.fill_(2.0)
            torch.cuda.synchronize()
            a0 = torch.cuda.Event(enable_timing=True); a1 = torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            ro = S.svm_train_dev(Xo_d, yo_d, wo.C, wo.kernel, wo.gamma, wo.tol, stream=stream, **extra)
            a1.record(stream)
            torch.cuda.synchronize()
            po = S.last_plan()
            it_o = ro["info"]["iterations"]
            ent = {"workload": f"{wo.name}: {wo.config}", "wss": extra.get("wss", 1),
                   "time_to_converge_s": a0.elapsed_time(a1) * 1e-3,
                   "iterations": it_o, "us_per_iter": 1e6 * ro["info"]["seconds_solve"] / max(1, it_o),
                   "converged": ro["info"]["converged"], "plan": po,
                   "cache_hits": ro["info"].get("cache_hits"), "cache_misses": ro["info"].get("cache_misses")}
            dpo = (wo.d + 3) // 4 * 4
            b_fp32 = wo.n * (4 * dpo + 25)
            ent["hbm_fp32_equivalent_gbs"] = b_fp32 * it_o / ro["info"]["seconds_solve"] / 1e9
            others.append(ent)
            del Xo_d, yo_d
            torch.cuda.empty_cache()

    # ---- projected-gradient dual trainer on W2: K built once in HBM,
    # every epoch one pass over it (k_gd_epoch, HBM-bound GEMV + fused update)
    gd = None
    if world == 1 and not args.no_gd:
        wg = W.get("W2")
        Xg, yg = wg.train()
        Xg_d, yg_d = torch.from_numpy(Xg).to(dev), torch.from_numpy(yg).to(dev)
        ng = Xg.shape[0]
        ep = 30
        S.svm_train_gd_dev(Xg_d, yg_d, wg.C, wg.kernel, wg.gamma, 1e-4, 2, stream=stream)      # warm
        g10 = S.svm_train_gd_dev(Xg_d, yg_d, wg.C, wg.kernel, wg.gamma, 1e-4, 10, stream=stream)["info"]
        gi = S.svm_train_gd_dev(Xg_d, yg_d, wg.C, wg.kernel, wg.gamma, 1e-4, ep, stream=stream)["info"]
        per_epoch = (gi["seconds_epochs"] - g10["seconds_epochs"]) / (ep - 10)
        gbytes = 8 * ng * ng + 40 * ng
        gd = {"workload": "W2", "epochs": ep, "lr": 1e-4, "seconds_gram": gi["seconds_gram"],
              "ms_per_epoch": 1e3 * per_epoch, "objective": gi["objective"],
              "roofline": {"bound": "hbm", "kernel": "k_gd_epoch", "achieved": gbytes / per_epoch / 1e9,
                           "peak": hbm, "unit": "GB/s", "frac": gbytes / per_epoch / 1e9 / hbm,
                           "peak_kind": peak_kind, "bytes_per_epoch": gbytes,
                           "note": "a read-only stream of K; the measured peak is a copy (read + write) "
                                   "figure, which a pure read stream can exceed"}}
        del Xg_d, yg_d

    # ---- batched prediction (a11) of the held-out rows on the tensor cores (tcgen05 3xTF32):
    # each rank predicts its share of the test rows against the whole model's SVs.  (Last:
    # its ~2.6 GB workspace left in the memory pool made the whole-solve times of the other
    # configs above pay fresh mappings, W3 0.094 -> 0.80 s, profiles/r2s3h.)
    predict = None
    if not args.no_predict:
        if world > 1:
            from paper_2311_14908_b200.dist import gather_rows
            alpha_full = gather_rows(alpha_last.contiguous().to(cdev), blocks, cdev).to(dev)
        else:
            alpha_full = alpha_last
        Xsv, coef, _ = S.svm_support_vectors_dev(Xd_full, yd_full, alpha_full, stream=stream)
        Xt, _ = w.test(args.predict_rows if args.predict_rows >= 0 else None)
        m = Xt.shape[0]
        mt = -(-m // world)
        tl, th = min(m, rank * mt), min(m, (rank + 1) * mt)
        Xt_d = torch.from_numpy(Xt[tl:th]).to(dev).contiguous()
        del Xt
        # warm with the full shape: the workspace (packed operands, ~2 GB) then comes from the
        # memory pool instead of a first-time mapping inside the timed launch
        S.svm_predict_dev(Xsv, coef, b_last, w.kernel, w.gamma, Xt_d, stream=stream, mode=1)
        barrier()
        p0 = torch.cuda.Event(enable_timing=True); p1 = torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        S.svm_predict_dev(Xsv, coef, b_last, w.kernel, w.gamma, Xt_d, stream=stream, mode=1)
        p1.record(stream)
        barrier()
        tp_s = gmax(p0.elapsed_time(p1) * 1e-3)
        nsv = int(coef.shape[0])
        flops = 2.0 * m * nsv * d
        tf32_peak = bf16 * 0.5            # nominal TF32 : BF16 dense ratio (1.1 : 2.25 PF), no TF32 measured peak
        # context: cuBLAS's own TF32 GEMM rate on this box (8192^3, the tensor pipe as a library drives it)
        ga = torch.randn(8192, 8192, device=dev)
        gb = torch.randn(8192, 8192, device=dev)
        tf32_prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = True
        with torch.cuda.stream(stream):
            for _ in range(3):
                ga @ gb
            g0 = torch.cuda.Event(enable_timing=True); g1 = torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            for _ in range(10):
                ga @ gb
            g1.record(stream)
        stream.synchronize()
        torch.backends.cuda.matmul.allow_tf32 = tf32_prev
        cublas_tf32 = 10 * 2.0 * 8192 ** 3 / (g0.elapsed_time(g1) * 1e-3) / 1e12
        del ga, gb
        predict = {"rows": m, "n_sv": nsv, "seconds": tp_s,
                   "mode": "tcgen05 kind::tf32 3xTF32, 128 x 256 accumulator tiles + fp64/fp32 split-exp epilogue",
                   "cublas_tf32_tflops": cublas_tf32,
                   "frac_of_cublas_tf32": 3 * flops / tp_s / 1e12 / cublas_tf32,
                   "roofline": {"bound": "tensor", "achieved": 3 * flops / tp_s / 1e12, "peak": tf32_peak,
                                "unit": "TFLOP/s", "frac": 3 * flops / tp_s / 1e12 / tf32_peak,
                                "algorithmic_tflops": flops / tp_s / 1e12,
                                "peak_kind": f"{peak_kind} bf16 x 0.5 (nominal TF32/BF16 ratio)",
                                "note": "achieved counts the 3 TF32 MMA passes issued (hi*hi + hi*lo + lo*hi)"},
                   "exp_per_s": m * nsv / tp_s}
        del Xt_d, Xsv, coef

    line = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            ips, k_it, thr = oracle_sample(w, X, y, args.cpu_budget, iters)
            cpu = {"value": iters / ips, "unit": "s", "cores": thr, "kind": "oracle", "cpu_model": cpu_model(),
                   "sample": f"first {k_it} SMO iterations of {w.name} (n={n}) on {thr} host threads "
                             f"({ips:.2f} iters/s); time-to-converge projected to the {iters} iterations "
                             f"of the identical trajectory"}
        line = {
            "metric": METRIC, "value": value, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{w.name}: {w.config}", "n": n, "d": d,
                       "kernel": "rbf" if w.kernel else "linear", "gamma": w.gamma, "C": w.C, "tol": w.tol,
                       "step": (f"one window of {window} SMO iterations of the solve (iters_per_launch); "
                                f"value = the K windows = the whole solve" if windowed else "one whole solve"),
                       "parallelism": f"rows sharded over {world} GPU(s)",
                       "l2": "X (1 GB) larger than L2; L2 flushed (256 MB write) before the timed region"
                             if windowed else "flushed between steps (256 MB write)"},
            "iterations": iters,
            "converged": info["converged"],
            "launches": info["launches"],
            "smo_iters_per_s": iters / value,
            "us_per_iter": 1e6 * solve_s / max(iters, 1),
            "solve_s": solve_s,
            "kernel_row_gbs": achieved,
            "roofline": roofline,
            "roofline_hbm_effective": hbm_eff,
            "predict": predict,
            "others": others,
            "gd": gd,
            "plan": plan,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": our_launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        S.svm_comm_destroy(comm)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="W5")
    ap.add_argument("--predict-rows", type=int, default=-1)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--ref-budget", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-predict", action="store_true")
    ap.add_argument("--no-others", action="store_true", help="skip the W2-W4 time-to-converge entries")
    ap.add_argument("--no-gd", action="store_true", help="skip the projected-GD trainer measurement")
    ap.add_argument("--windowed", action="store_true", help="time one solve in K windows for any workload")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
