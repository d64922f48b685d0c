#!/usr/bin/env python3
"""Benchmark of the B200 Boys-function evaluator (driver contract: one JSON line).

Default workload (--config cfg1 = BASELINE.json configs[1], the configuration
the metric is quoted on): F_0..F_32 for 1e8 uniform x in [0,100] per GPU, SoA
output, FP64.  The metric is quoted "at kmax=8/32": the default line also
carries `secondary.k8`, the same batch at kmax = 8 timed the same way.  A "step" is one pass of the hot path (boysfn_eval_device) over
that batch; x is the splitmix64 stream of boysfn_generate_uniform (seed 2), rank
r taking global indices [r*N, (r+1)*N) -- weak scaling, no collective on the
data path (the only NCCL calls are the timing barrier and the max-over-ranks
reduction).  Other named configs (--config NAME; the default one-GPU line also
carries each of them, device side only, under `configs`):
  cfg0       configs[0]: 1e6 uniform x in [0,50], k = 8, AoS; the CPU side is the
             reference API on ONE thread (cpu_baseline, --impl reference)
  cfg2       configs[2]: 1e8 x clustered at the region boundaries, k = 0..32 sweep
  cfg3       configs[3]: 1e9 log-uniform x in [1e-12, 1e4], k = 16, AoS (fits HBM)
  cfg4       configs[4]: 1e10 x in total, sharded over the GPUs (strong scaling),
             k = 16 by default (--k 4/16/32), streamed
  northstar  1e9 uniform x in [0,100], k = 32, SoA, streamed through a reused
             1e8-x output buffer (264 GB of F per step > HBM)

Reported beside `value` (device-resident, CUDA events on the launching stream):
  e2e          same metric through the reference-facing host API
               (boys_batch_many -> boysfn_eval_host), page-locked host buffers from
               boysfn_host_alloc, H2D of x and D2H of all F values inside the
               timed region; e2e_pageable: the reference's own calling
               convention (plain pageable numpy buffers, AoS)
  roofline     algorithmic bytes per launch (8 B read + 8(k+1) B written per x)
               / mean launch time, against MEASURED_PEAKS.json hbm_gbs; traffic
               from the committed ncu capture (profiles/ncu_summary.json);
               roofline.fp64: algorithmic flops of the step (SURVEY 8(a) counts,
               the step's own region mix) against the measured DFMA peak
  step_ms      min/median/max per timed step and the worst host enqueue time
               (the steps are queued behind a short device spin outside the
               timed interval, so host hiccups cannot idle the GPU inside it)
  cpu_baseline the unmodified reference (oracle/_ref) on all host cores (one
               for cfg0) over the timed batch itself (up to 1e8 x; rank 0, N=1)
  accuracy     max |F - oracle| and |F - reference| on a strided sample READ BACK
               FROM THE TIMED OUTPUT (the last launch's buffer), region C
               checked bit for bit
  configs      (default run, one GPU) cfg0, cfg2, cfg3, northstar and cfg4 on
               the device: value, ms per step, HBM roofline fraction and
               accuracy, each after 3 untimed steps (--no-secondary skips them)

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config NAME]

With --gpus N > 1 and no torchrun environment, bench.py re-launches itself as
`python -m torch.distributed.run --nproc-per-node N` (127.0.0.1 rendezvous),
one rank per GPU.  --dry-run: the same launch over gloo on CPU, no kernels
(tests the launcher).
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Boys values/sec (F_k·x) at kmax=8/32, 1/2/4/8 B200; %FP64/HBM roofline; max abs err"
UNIT = "values/s"

CONFIGS = {
    "cfg0": dict(workload="configs[0]: F_0..F_8 for 1e6 uniform x in [0,50], AoS (the reference API's layout); "
                          "CPU side single-thread through the reference API",
                 n=1_000_000, k=8, layout="aos", dist="uniform", lo=0.0, hi=50.0, seed=1, chunk=None, cpu_threads=1),
    "cfg1": dict(workload="configs[1]: F_0..F_32 for 1e8 uniform x in [0,100] per B200, SoA output, FP64",
                 n=100_000_000, k=32, layout="soa", dist="uniform", lo=0.0, hi=100.0, seed=2, chunk=None),
    "cfg3": dict(workload="configs[3]: ERI-like F_0..F_16 for 1e9 log-uniform x in [1e-12,1e4] per B200, AoS",
                 n=1_000_000_000, k=16, layout="aos", dist="loguniform", lo=-12.0, hi=4.0, seed=4, chunk=None),
    "cfg2": dict(workload="configs[2]: region-boundary stress, 1e8 x clustered at 0+/x0/x1 and mixed per warp, "
                          "kmax 0..32 sweep (one launch per k per step), SoA",
                 n=100_000_000, k=32, ks=list(range(33)), layout="soa", dist="boundary", lo=0.0, hi=0.0, seed=3,
                 chunk=None),
    "cfg4": dict(workload="configs[4]: 1e10 uniform x in [0,100] sharded across the GPUs (strong scaling), "
                          "k=16 (--k 4/16/32), SoA, each shard streamed through a reused 1e8-x output buffer",
                 n=10_000_000_000, k=16, layout="soa", dist="uniform", lo=0.0, hi=100.0, seed=5,
                 chunk=100_000_000, strong=True),
    "northstar": dict(workload="north star: F_0..F_32 for 1e9 uniform x in [0,100] per B200, SoA, streamed "
                               "through a reused 1e8-x output buffer (264 GB of F per step > HBM)",
                      n=1_000_000_000, k=32, layout="soa", dist="uniform", lo=0.0, hi=100.0, seed=2,
                      chunk=100_000_000),
}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg1", choices=sorted(CONFIGS))
    ap.add_argument("--n", type=float, default=None, help="override x values per GPU")
    ap.add_argument("--k", type=int, default=None, help="override kmax")
    ap.add_argument("--ks", default=None, help="override a sweep's orders, e.g. 0,1,2 (diagnostics)")
    ap.add_argument("--layout", default=None, choices=["soa", "aos"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-accuracy", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="launcher test: gloo ranks on CPU, no kernels")
    a = ap.parse_args()
    a.warmup = max(a.warmup, 3)
    cfg = dict(CONFIGS[a.config])
    if a.n is not None:
        cfg["n"] = int(a.n)
    if a.k is not None:
        cfg["k"] = a.k
    if a.ks is not None:
        cfg["ks"] = [int(v) for v in a.ks.split(",")]
        cfg["k"] = max(cfg["ks"])
    if a.layout is not None:
        cfg["layout"] = a.layout
    a.cfg = cfg
    return a


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(cfg):
    """DRAM bytes per launch from the committed ncu --set full capture, when it
    was taken on this workload (profiles/ncu_summary.json)."""
    if cfg.get("ks"):
        return None  # a sweep has no single dominant launch
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            s = json.load(f)
        e = s["launches"].get("%s_k%d" % (cfg["layout"], cfg["k"]))
        if e and e.get("n", cfg["n"]) == (cfg["chunk"] or cfg["n"]):
            return e["dram_bytes_per_launch"]
    except Exception:
        pass
    return None


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML from a
    background thread during the timed region.  Only the two cheap queries are
    polled: an `nvidia-smi --query-gpu=... -lms 20` subprocess perturbed the
    timed kernels (one step in ~5 ran 25% slow with it, none without)."""
    REASONS = {  # NVML clocks-event reason bits
        "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

    def __init__(self, device_index, period_s=0.01):
        self.dev = device_index
        self.period = period_s
        self.rows = []
        self.stop_flag = threading.Event()
        self.t = None

    def start(self):
        if os.environ.get("BENCH_NO_CLOCKS"):  # diagnostics: timing without the sampler
            return
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.dev)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception:
            return

        def run():
            while not self.stop_flag.is_set():
                try:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.rows.append((sm, rs))
                except Exception:
                    pass
                self.stop_flag.wait(self.period)
        self.t = threading.Thread(target=run, daemon=True)
        self.t.start()

    def stop(self):
        if self.t is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        self.stop_flag.set()
        self.t.join(timeout=2)
        sm = [r[0] for r in self.rows]
        reasons = sorted({name for _, rs in self.rows for name, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.rows), "source": "NVML, 10 ms"}


def generate(pkg, x, cfg, offset):
    if cfg["dist"] == "uniform":
        pkg.generate_uniform(x, cfg["seed"], cfg["lo"], cfg["hi"], offset=offset)
    elif cfg["dist"] == "boundary":
        pkg.generate_boundary(x, cfg["seed"], offset=offset)
    else:
        pkg.generate_loguniform(x, cfg["seed"], cfg["lo"], cfg["hi"], offset=offset)


def cpu_reference(xs, k, threads, min_seconds=2.0, out=None, warm=True):
    """The unmodified reference (oracle/_ref, else the C restatement) on
    `threads` host threads over xs, repeated until min_seconds elapsed (at
    least one pass; warm: one untimed pass first, for the page faults).
    Returns (values/s, kind, passes, seconds)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import pyoracle
    if out is None or out.size < xs.size * (k + 1):
        out = np.empty(xs.size * (k + 1))
    out = out[: xs.size * (k + 1)]
    if pyoracle.Ref.available():
        ref, kind = pyoracle.Ref(), "reference"
        if threads > 1:
            run = lambda: ref.boys_batch_many_mt(xs, k, threads, out=out)  # noqa: E731
        else:  # the reference's own entry point, one call on one thread
            run = lambda: ref.boys_batch_many(xs, k, out=out)  # noqa: E731
    else:
        port, kind = pyoracle.Port(), "port"
        run = lambda: port.boys_batch_many(xs, k, threads=threads)  # noqa: E731
    if warm:
        run()
    passes, t0 = 0, time.perf_counter()
    while True:
        run()
        passes += 1
        el = time.perf_counter() - t0
        if el >= min_seconds:
            break
    return passes * xs.size * (k + 1) / el, kind, passes, el


def host_workload(cfg, m):
    """The first m x of the workload on the host, for the reference arm (no
    device there): the uniform and boundary streams bit for bit as the device
    generates them (up to an ulp in the boundary stream's 10^-s offsets), the
    log-uniform law with the host's exp10 (ulp-level differences only)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    port = pyoracle.Port()
    if cfg["dist"] == "uniform":
        return port.gen_uniform(m, cfg["seed"], cfg["lo"], cfg["hi"])
    if cfg["dist"] == "boundary":
        return port.gen_boundary(m, cfg["seed"])
    return port.gen_loguniform(m, cfg["seed"], cfg["lo"], cfg["hi"])


def cpu_threads(cfg):
    return cfg.get("cpu_threads") or os.cpu_count() or 1


# Largest batch the CPU side evaluates per step: configs[1]'s whole 1e8-x batch
# (0.8 s per pass on 16 host cores); the 1e9/1e10-x configs time their first
# 1e8 x (same stream, same law) and say so.
CPU_MAX_X = 100_000_000


def run_reference_arm(args):
    """--impl reference: the unmodified reference boys_batch_many on the host
    cores, each step one pass over the workload's batch (capped at CPU_MAX_X;
    a sweep config at 1e7 x per order)."""
    cfg, k = args.cfg, args.cfg["k"]
    threads = cpu_threads(cfg)
    ks = cfg.get("ks") or [k]
    n_sample = min(cfg["n"], CPU_MAX_X if len(ks) == 1 else 10_000_000)
    xs = host_workload(cfg, n_sample)
    import numpy as np
    out = np.empty(n_sample * (max(ks) + 1))
    vals = []
    kind = "reference"
    for i in range(args.warmup + args.steps):
        t_all, values = 0.0, 0
        for kk in ks:
            v, kind, passes, el = cpu_reference(xs, kk, threads, min_seconds=0.0, out=out, warm=i == 0)
            t_all += el
            values += passes * n_sample * (kk + 1)
        if i >= args.warmup:
            vals.append(values / t_all)
    value = statistics.mean(vals)
    same = n_sample == cfg["n"]
    sample = ("each step: one pass of boys_batch_many over %s x of the workload stream (%s), k=%s, AoS, "
              "%d host thread%s" % ("all %d" % n_sample if same else "the first %d of %d" % (n_sample, cfg["n"]),
                                    cfg["dist"], "0..32" if len(ks) > 1 else k, threads, "" if threads == 1 else "s"))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": 0, "launched_with_gpus": args.gpus, "host_threads": threads,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * n_sample * sum(kk + 1 for kk in ks) / value, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["workload"], "name": args.config, "kmax": k, "layout": "aos (reference API)",
                   "n_per_step": n_sample, "same_batch_as_device_arm": same, "parallelism": "host threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def fp64_roofline(pkg, x, ks, step_s):
    """The FP64 side of the roofline: FP64-pipe lane-ops of the step over its
    time, against the measured DFMA peak (tools/fp64_peak.cu).  The ops per x
    are MEASURED per (region, k) -- ncu sm__inst_executed_pipe_fp64 of the
    default kernels on single-region batches (tools/fp64_pipe_table.py,
    profiles/r02_fp64_pipe_ops.json: divisions, exp, sqrt, classification and
    store-side FP64 work included) -- weighted with this step's region counts.
    MUFU (RCP64H/RSQ64H) runs on the XU pipe and is reported beside it."""
    import torch
    t = pkg.embedded_default()
    na = nab = 0
    for c in range(0, x.numel(), 1 << 27):  # chunked: configs[4] holds 1e10 x
        xc = x[c:c + (1 << 27)]
        na += int(torch.count_nonzero(xc < t.x0).item())
        nab += int(torch.count_nonzero(xc < t.x1).item())
    nb = nab - na
    nc = x.numel() - nab
    try:
        with open(os.path.join(ROOT, "profiles", "r01_fp64_peak.json")) as f:
            peak_tflops, kind = float(json.load(f)["fp64_tflops"]), "measured (tools/fp64_peak.cu)"
    except Exception:
        peak_tflops, kind = 37.2, "nominal (148 SMs x 64 DFMA/clk x 1.965 GHz x 2)"
    res = {"region_counts": [na, nb, nc], "peak_kind": kind}
    try:
        with open(os.path.join(ROOT, "profiles", "r02_fp64_pipe_ops.json")) as f:
            tab = json.load(f)["per_k"]
    except Exception:
        tab = None
    if tab is not None:
        ops = sum(na * tab[str(k)]["A"]["fp64"] + nb * tab[str(k)]["B"]["fp64"] + nc * tab[str(k)]["C"]["fp64"]
                  for k in ks)
        xu = sum(na * tab[str(k)]["A"]["xu"] + nb * tab[str(k)]["B"]["xu"] + nc * tab[str(k)]["C"]["xu"]
                 for k in ks)
        peak_ops = peak_tflops * 1e12 / 2  # DFMA lane-ops/s
        achieved = ops / step_s
        res.update({"achieved": achieved / 1e12, "peak": peak_ops / 1e12, "unit": "T fp64-pipe lane-ops/s",
                    "frac": achieved / peak_ops, "fp64_pipe_ops_per_step": ops, "xu_ops_per_step": xu,
                    "ops_source": "profiles/r02_fp64_pipe_ops.json (ncu, per region and k)"})
    return res


def accuracy_from_output(x, out, c0, c1, k, layout, m=20000):
    """max |F - oracle| and |F - reference| over m x strided through the last
    launch's batch x[c0:c1], with F READ BACK from that launch's output buffer
    (the timed output itself); region C compared bit for bit."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import torch
    import pyoracle
    cn = c1 - c0
    m = min(m, cn)
    j = torch.arange(m, device=x.device, dtype=torch.int64) * (cn // m)
    xs = x[c0:c1][j].cpu().numpy()
    R = k + 1
    if layout == "soa":  # out[l*cn + j]
        idx = torch.arange(R, device=x.device, dtype=torch.int64)[None, :] * cn + j[:, None]
    else:  # out[j*R + l]
        idx = j[:, None] * R + torch.arange(R, device=x.device, dtype=torch.int64)[None, :]
    g = out[idx.reshape(-1)].view(m, R).cpu().numpy()
    port = pyoracle.Port()
    hp = port.hp(xs, k)
    ref = port.boys_batch_many(xs, k)
    inC = xs >= port.x1
    mism = int(np.count_nonzero(g[inC].view(np.uint64) != ref[inC].view(np.uint64)))
    return {"max_abs_err_vs_oracle": float(np.abs(g - hp).max()),
            "max_abs_dev_vs_reference": float(np.abs(g - ref).max()),
            "region_c_bit_mismatches": mism, "region_c_values_checked": int(inC.sum()) * R,
            "eps_tol": 5e-14,
            "sample": "%d x strided over the last timed launch (global x [%d, %d), k=%d), F read back from the "
                      "timed output buffer" % (m, c0, c1, k)}


def time_device(pkg, x, k, out, layout, pieces, steps, warmup, stream):
    """Mean device ms per step of eval_device over `pieces` (CUDA events on
    the launching stream, after warm-up)."""
    import torch
    from paper_2512_10059_b200 import dist as D

    def step():
        for c0, c1 in pieces:
            pkg.eval_device(x[c0:c1], k, out[: (c1 - c0) * (k + 1)], layout=layout)
    for _ in range(warmup):
        step()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    D.barrier()
    torch.cuda.synchronize()
    torch.cuda._sleep(int(0.02 * 2e9))
    ev0.record(stream)
    for _ in range(steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    D.barrier()
    return D.max_over_ranks(ev0.elapsed_time(ev1)) / steps


def run_other_configs(args, pkg, dev, stream, hbm):
    """The other BASELINE configurations, device side only, in the default
    run (one GPU): so the driver's own run carries a line for each, not only
    the builder's `--config NAME` runs.  Each: the config's own x (device
    generator), W = 3 untimed steps, then K steps timed with CUDA events on
    the launching stream; accuracy read back from the last timed launch."""
    import torch
    res = {}
    for name, steps in (("cfg0", 20), ("cfg2", 3), ("cfg3", 5), ("northstar", 3), ("cfg4", 2)):
        cfg = CONFIGS[name]
        n, layout = cfg["n"], cfg["layout"]
        ks = cfg.get("ks") or [cfg["k"]]
        chunk = min(cfg["chunk"] or n, n)
        x = torch.empty(n, dtype=torch.float64, device=dev)
        generate(pkg, x, cfg, 0)
        out = torch.empty(chunk * (max(ks) + 1), dtype=torch.float64, device=dev)
        pieces = [(c, min(n, c + chunk)) for c in range(0, n, chunk)]

        def step():
            for kk in ks:
                for c0, c1 in pieces:
                    pkg.eval_device(x[c0:c1], kk, out[: (c1 - c0) * (kk + 1)], layout=layout)
        for _ in range(3):
            step()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(int(0.02 * 2e9))
        e0.record(stream)
        for _ in range(steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1) / steps
        alg = n * sum(8 + 8 * (kk + 1) for kk in ks)
        entry = {"workload": cfg["workload"], "value": n * sum(kk + 1 for kk in ks) / (ms * 1e-3), "unit": UNIT,
                 "ms_per_step": ms, "steps": steps, "warmup": 3, "launches_per_step": len(ks) * len(pieces),
                 "roofline": {"bound": "hbm", "achieved": alg / (ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                              "frac": alg / (ms * 1e-3) / 1e9 / hbm}}
        if not args.no_accuracy:
            a = accuracy_from_output(x, out, pieces[-1][0], pieces[-1][1], ks[-1], layout, m=5000)
            entry["accuracy"] = {k_: a[k_] for k_ in ("max_abs_err_vs_oracle", "max_abs_dev_vs_reference",
                                                       "region_c_bit_mismatches", "sample")}
        res[name] = entry
        del x, out
        torch.cuda.empty_cache()
    return res


def run_b200(args, world, rank, local):
    import torch
    import paper_2512_10059_b200 as pkg
    from paper_2512_10059_b200 import dist as D

    if world != args.gpus:
        raise SystemExit("bench.py: --gpus %d but %d rank(s) started" % (args.gpus, world))
    cfg = args.cfg
    n_total = cfg["n"]
    if cfg.get("strong"):  # total work fixed, contiguous near-equal shards
        begin, end = D.strong_shard(n_total, world, rank)
        n = end - begin
    else:  # per-GPU work fixed
        begin, n = D.weak_shard(n_total, rank)[0], n_total
    k, layout = cfg["k"], cfg["layout"]
    chunk = min(cfg["chunk"] or n, n)
    dev = torch.device("cuda", local if world > 1 else 0)
    x = torch.empty(n, dtype=torch.float64, device=dev)
    generate(pkg, x, cfg, begin)
    ks = cfg.get("ks") or [k]
    out = torch.empty(chunk * (max(ks) + 1), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    pieces = [(c, min(n, c + chunk)) for c in range(0, n, chunk)]
    launch_ev = {}

    def step(record=False):
        for kk in ks:
            for c0, c1 in pieces:
                if record:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                pkg.eval_device(x[c0:c1], kk, out[: (c1 - c0) * (kk + 1)], layout=layout)
                if record:
                    e1 = torch.cuda.Event(enable_timing=True)
                    e1.record(stream)
                    launch_ev.setdefault(kk, []).append((e0, e1))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    sampler = ClockSampler(dev.index if world == 1 else local)
    sampler.start()
    time.sleep(0.1)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    D.barrier()
    torch.cuda.synchronize(dev)
    launches0 = pkg.kernel_launch_count()
    # Hold the stream in a short spin (outside the timed region) while the host
    # enqueues all timed steps, so a host-side hiccup cannot leave the GPU idle
    # between steps and inflate the device-timed interval.
    # (~3 ms of device time per launch to enqueue covers the host's worst
    # observed per-step enqueue time, GIL hand-offs to the clock sampler included)
    torch.cuda._sleep(int(min(2.0, 0.02 + 0.003 * args.steps * len(pieces) * len(ks)) * 2e9))
    ev[0].record(stream)
    host_ms = []
    for s in range(args.steps):
        h0 = time.perf_counter()
        step(record=len(ks) > 1)
        ev[s + 1].record(stream)
        host_ms.append((time.perf_counter() - h0) * 1e3)
    torch.cuda.synchronize(dev)
    D.barrier()
    launches = pkg.kernel_launch_count() - launches0
    clocks = sampler.stop()
    total_ms = D.max_over_ranks(ev[0].elapsed_time(ev[-1]))
    per_step = [ev[s].elapsed_time(ev[s + 1]) for s in range(args.steps)]
    step_stats = {"min": min(per_step), "median": statistics.median(per_step), "max": max(per_step),
                  "host_enqueue_max": max(host_ms)}
    ms_step = total_ms / args.steps
    # whole-job throughput: every rank's values over the slowest rank's time
    value = (n_total if cfg.get("strong") else world * n) * sum(kk + 1 for kk in ks) / (ms_step * 1e-3)

    # accuracy first, from the buffer the last timed launch wrote
    acc = None
    if rank == 0 and not args.no_accuracy:
        acc = accuracy_from_output(x, out, pieces[-1][0], pieces[-1][1], ks[-1], layout)

    hbm, peak_kind = peaks()
    alg_bytes = chunk * (8 + 8 * (k + 1))
    if len(ks) > 1:  # sweep: algorithmic bytes of the whole step over its time
        alg_bytes = sum(n * (8 + 8 * (kk + 1)) for kk in ks)
        mean_launch_s = statistics.mean(per_step) * 1e-3
    else:
        mean_launch_s = statistics.mean(per_step) * 1e-3 / len(pieces)
    achieved = alg_bytes / mean_launch_s / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": ncu_traffic(cfg), "peak_kind": peak_kind,
                "algorithmic_bytes_per_launch": alg_bytes,
                "note": "per x: 8 B read + 8*(k+1) B written; %d launch(es) per step" % len(pieces)}
    roofline["fp64"] = fp64_roofline(pkg, x, ks, ms_step * 1e-3)

    per_k = None
    if len(ks) > 1:
        per_k = {}
        for kk, evs in launch_ev.items():
            ms = statistics.median(a.elapsed_time(b) for a, b in evs)
            gbs = n * (8 + 8 * (kk + 1)) / (ms * 1e-3) / 1e9
            per_k[kk] = {"values_per_s": n * (kk + 1) / (ms * 1e-3), "ms": ms, "hbm_frac": gbs / hbm}

    # the other half of "kmax=8/32": the same batch at kmax = 8, timed the same way
    secondary = None
    if args.config == "cfg1" and not args.no_secondary and len(ks) == 1:
        k2 = 8
        ms2 = time_device(pkg, x, k2, out, layout, pieces, args.steps, args.warmup, stream)
        v2 = world * n * (k2 + 1) / (ms2 * 1e-3)
        a2 = chunk * (16 + 8 * k2) / (ms2 * 1e-3 / len(pieces)) / 1e9
        secondary = {"k8": {"kmax": k2, "value": v2, "unit": UNIT, "ms_per_step": ms2,
                            "roofline": {"bound": "hbm", "achieved": a2, "peak": hbm, "unit": "GB/s",
                                         "frac": a2 / hbm},
                            "config": "same x and layout as the main line, kmax = 8"}}

    del out
    torch.cuda.empty_cache()
    e2e = e2e_pageable = None
    host_out = None
    if not args.no_e2e and len(ks) == 1:
        try:
            e2e = run_e2e(args, x, world, pinned=True)
        except Exception as exc:  # e.g. pinned host memory exhausted; the device line still stands
            e2e = {"value": None, "unit": UNIT, "error": "%s: %s" % (type(exc).__name__, exc)}
        try:
            e2e_pageable, host_out = run_e2e(args, x, world, pinned=False)
        except Exception as exc:
            e2e_pageable = {"value": None, "unit": UNIT, "error": "%s: %s" % (type(exc).__name__, exc)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = cpu_threads(cfg)
        m = min(n, CPU_MAX_X if len(ks) == 1 else 10_000_000)
        xs = x[:m].cpu().numpy()  # the exact doubles the GPU evaluated
        t_all = v_all = 0.0
        for kk in ks:  # time-weighted over the sweep (one k unless cfg2)
            v, kind, passes, el = cpu_reference(xs, kk, threads, min_seconds=2.0 / len(ks), out=host_out)
            t_all += el
            v_all += v * el
        cpu = {"value": v_all / t_all, "unit": UNIT, "cores": threads, "kind": kind,
               "same_batch": m == n,
               "sample": "%s x of the timed batch, k in %s, AoS, %d thread%s, %.2f s"
                         % ("all %d" % m if m == n else "the first %d of %d" % (m, n),
                            "0..%d" % max(ks) if len(ks) > 1 else str(k), threads, "" if threads == 1 else "s",
                            t_all)}
    host_out = None

    # the other BASELINE configurations, device side (default run, one GPU)
    others = None
    if args.config == "cfg1" and not args.no_secondary and world == 1 and args.n is None and args.k is None:
        del x
        torch.cuda.empty_cache()
        others = run_other_configs(args, pkg, dev, stream, hbm)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if cfg.get("strong") else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["workload"], "name": args.config, "n_per_gpu": n, "n_total": n_total
                       if cfg.get("strong") else n * world, "kmax": k,
                       "layout": layout,
                       "x": "%s [%g,%g] splitmix64 seed %d, global index offset rank*N"
                            % (cfg["dist"], cfg["lo"], cfg["hi"], cfg["seed"]),
                       "l2": ("inputs+outputs %.1f GB per launch >> 126 MB L2 (no flush needed)" % (alg_bytes / 1e9))
                       if alg_bytes > 1e9 else "inputs+outputs %.2f GB per launch" % (alg_bytes / 1e9),
                       "parallelism": "dp%d (independent shards, no collective)" % world},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "e2e_pageable": e2e_pageable,
            "gpu_launches": launches, "clocks": clocks, "accuracy": acc, "step_ms": step_stats,
        }
        if secondary is not None:
            line["secondary"] = secondary
        if others is not None:
            line["configs"] = others
        if per_k is not None:
            line["per_k"] = per_k
        print(json.dumps(line), flush=True)


def run_e2e(args, x_dev, world, pinned=True):
    """Same metric through the host API (boys_batch_many -> boysfn_eval_host):
    host x -> device -> host F, every step.  pinned: buffers from
    boysfn_host_alloc (pkg.host_empty), the main layout; else plain pageable
    numpy arrays in AoS, the reference's own calling convention (eval.hpp:43-45).
    The full batch when its output fits host RAM comfortably (configs[0]/[1]),
    else the first 1e8 x (n_per_step says which)."""
    import numpy as np
    import paper_2512_10059_b200 as pkg
    from paper_2512_10059_b200 import dist as D
    cfg = args.cfg
    k = cfg["k"]
    layout = cfg["layout"] if pinned else "aos"
    # host output per rank: 26 GB at 1e8 x, k=32 -- one rank gets the full
    # batch, N ranks share the host's RAM (1/N of the batch each, >= 1e7)
    n = min(cfg["n"], 100_000_000 if world == 1 else max(10_000_000, 100_000_000 // world))
    if pinned:
        xs, out = pkg.host_empty(n), pkg.host_empty(n * (k + 1))
    else:
        xs, out = np.empty(n), np.empty(n * (k + 1))
    xs[:] = x_dev[:n].cpu().numpy()
    tables = pkg.embedded_default()
    pkg.boys_batch_many(xs, k, tables, out, layout=layout)  # warm (pipeline buffers, first touch)
    D.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        pkg.boys_batch_many(xs, k, tables, out, layout=layout)
    el = time.perf_counter() - t0
    D.barrier()
    el = D.max_over_ranks(el)
    v = world * n * (k + 1) * args.e2e_steps / el
    res = {"value": v, "unit": UNIT, "h2d_bytes_per_step": n * 8, "d2h_bytes_per_step": n * (k + 1) * 8,
           "steps": args.e2e_steps, "n_per_step": n,
           "api": "boys_batch_many -> boysfn_eval_host (%s)" % (
               "page-locked buffers from boysfn_host_alloc" if pinned else
               "plain pageable numpy buffers: the reference's calling convention"),
           "layout": layout}
    if pinned:
        return res
    return res, out  # the pageable output array is reused by the CPU baseline


def run_dry(args, world, rank):
    """--dry-run: the multi-rank launch and the max-over-ranks timing plumbing
    over gloo on CPU, no kernels; rank 0 prints one line."""
    from paper_2512_10059_b200 import dist as D
    if world != args.gpus:
        raise SystemExit("bench.py: --gpus %d but %d rank(s) started" % (args.gpus, world))
    D.barrier()
    t = D.max_over_ranks(float(rank + 1))
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "max_over_ranks": t, "metric": METRIC}), flush=True)


def relaunch(args):
    """Re-run this command under torchrun with --gpus ranks (one per GPU)."""
    import socket
    import subprocess
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


def main():
    args = parse_args()
    under_launcher = "WORLD_SIZE" in os.environ
    if args.gpus > 1 and not under_launcher and (args.impl == "b200" or args.dry_run):
        sys.exit(relaunch(args))
    rank = int(os.environ.get("RANK", "0"))
    from paper_2512_10059_b200 import dist as D
    if args.dry_run:
        world, rank, _ = D.init("gloo")
        try:
            run_dry(args, world, rank)
        finally:
            D.finalize()
        return
    if args.impl == "reference":
        if rank == 0:  # the other ranks exit 0 without work
            run_reference_arm(args)
        return
    world, rank, local = D.init("nccl")
    try:
        run_b200(args, world, rank, local)
    finally:
        D.finalize()


if __name__ == "__main__":
    main()
