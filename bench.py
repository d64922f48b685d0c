#!/usr/bin/env python3
"""Benchmark of the B200 Boys-function evaluator (driver contract: one JSON line).

Default workload (--config cfg1 = BASELINE.json configs[1], the configuration
the metric is quoted on): F_0..F_32 for 1e8 uniform x in [0,100] per GPU, SoA
output, FP64.  A "step" is one pass of the hot path (boysfn_eval_device) over
that batch; x is the splitmix64 stream of boysfn_generate_uniform (seed 2), rank
r taking global indices [r*N, (r+1)*N) -- weak scaling, no collective on the
data path (the only NCCL calls are the timing barrier and the max-over-ranks
reduction).  Other named configs (reported in DESIGN.md, not the driver's line):
  cfg2       configs[2]: 1e8 x clustered at the region boundaries, k = 0..32 sweep
  cfg3       configs[3]: 1e9 log-uniform x in [1e-12, 1e4], k = 16, AoS (fits HBM)
  cfg4       configs[4]: 1e10 x in total, sharded over the GPUs (strong scaling),
             k = 16 by default (--k 4/16/32), streamed
  northstar  1e9 uniform x in [0,100], k = 32, SoA, streamed through a reused
             1e8-x output buffer (264 GB of F per step > HBM)

Reported beside `value` (device-resident, CUDA events on the launching stream):
  e2e          same metric through the reference-facing host API
               (boys_batch_many -> boysfn_eval_host), pinned host buffers, H2D of
               x and D2H of all F values inside the timed region
  roofline     algorithmic bytes per launch (8 B read + 8(k+1) B written per x)
               / mean launch time, against MEASURED_PEAKS.json hbm_gbs; traffic
               from the committed ncu capture (profiles/ncu_summary.json);
               roofline.fp64: algorithmic flops of the step (SURVEY 8(a) counts,
               the step's own region mix) against the measured DFMA peak
  step_ms      min/median/max per timed step and the worst host enqueue time
               (the steps are queued behind a short device spin outside the
               timed interval, so host hiccups cannot idle the GPU inside it)
  cpu_baseline the unmodified reference (oracle/_ref) on all host cores over a
               bounded sample of the same stream (rank 0, N=1 only)
  accuracy     max |F - oracle| on a sample (binary128 oracle, oracle/boys_hp.c)

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config NAME]
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
    ap.add_argument("--layout", default=None, choices=["soa", "aos"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-accuracy", action="store_true")
    a = ap.parse_args()
    a.warmup = max(a.warmup, 3)
    cfg = dict(CONFIGS[a.config])
    if a.n is not None:
        cfg["n"] = int(a.n)
    if a.k is not None:
        cfg["k"] = a.k
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


def cpu_reference(xs, k, threads, min_seconds=2.0):
    """The unmodified reference (oracle/_ref, else the C restatement) on
    `threads` host threads over xs (a bounded sample of the workload stream),
    repeated until min_seconds elapsed.  Returns (values/s, kind, passes, seconds)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import pyoracle
    if pyoracle.Ref.available():
        ref, kind = pyoracle.Ref(), "reference"
        run = lambda out: ref.boys_batch_many_mt(xs, k, threads, out=out)  # noqa: E731
    else:
        port, kind = pyoracle.Port(), "port"
        run = lambda out: port.boys_batch_many(xs, k, threads=threads)  # noqa: E731
    out = np.empty(xs.size * (k + 1))
    run(out)  # warm (page faults)
    passes, t0 = 0, time.perf_counter()
    while True:
        run(out)
        passes += 1
        el = time.perf_counter() - t0
        if el >= min_seconds:
            break
    return passes * xs.size * (k + 1) / el, kind, passes, el


def reference_sample(cfg, m):
    """The first m x of the workload on the host, for the reference arm (no
    device there): the uniform stream bit-identical to the device's; the
    log-uniform law with the host's exp10 (ulp-level differences only)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    port = pyoracle.Port()
    if cfg["dist"] == "uniform":
        return port.gen_uniform(m, cfg["seed"], cfg["lo"], cfg["hi"])
    if cfg["dist"] == "boundary":  # same clustering law on the host
        import numpy as np
        rng = np.random.default_rng(cfg["seed"])
        b = np.array([0.0, port.x0, port.x1])[rng.integers(0, 3, m)]
        mode = rng.integers(0, 3, m)
        j = rng.integers(-64, 65, m).astype(np.float64)
        ulp = np.where(b == 0.0, 5e-324, np.spacing(np.maximum(b, 1e-300)))
        v = np.where(mode == 0, b + j * ulp,
                     np.where(mode == 1, b + rng.choice([-1.0, 1.0], m) * 10.0 ** -rng.uniform(1, 15, m),
                              b + rng.uniform(-1, 1, m)))
        return np.abs(v)
    u = port.gen_uniform(m, cfg["seed"], 0.0, 1.0)
    return 10.0 ** (cfg["lo"] + (cfg["hi"] - cfg["lo"]) * u)


def run_reference_arm(args):
    cfg, k = args.cfg, args.cfg["k"]
    threads = os.cpu_count() or 1
    n_sample = min(cfg["n"], 4_000_000)
    xs = reference_sample(cfg, n_sample)
    ks = cfg.get("ks") or [k]
    vals = []
    kind = "reference"
    for i in range(args.warmup + args.steps):
        t_all, v_all = 0.0, 0.0
        for kk in ks:
            v, kind, passes, el = cpu_reference(xs, kk, threads, min_seconds=0.5 / len(ks))
            t_all += el
            v_all += v * el
        if i >= args.warmup:
            vals.append(v_all / t_all)
    value = statistics.mean(vals)
    sample = ("each step: passes over the first %d x of the workload stream until >= 0.5 s, k=%d, AoS, "
              "%d threads" % (n_sample, k, threads))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * n_sample * (k + 1) / value, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["workload"], "kmax": k, "layout": "aos (reference API)",
                   "n_per_step": n_sample, "parallelism": "host threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def fp64_roofline(pkg, x, ks, step_s):
    """The FP64 side of the roofline: algorithmic
    flops of the step -- per x, A: 2(n_k+m_k)+1+[k>0](2+3k), B: 25+3k,
    C: 3+2k (a mul+add pair counts 2; div, sqrt, exp count 1), with the
    step's own region counts -- over the step time, against the measured DFMA
    peak (tools/fp64_peak.cu)."""
    import torch
    t = pkg.embedded_default()
    na = nab = 0
    for c in range(0, x.numel(), 1 << 27):  # chunked: configs[4] holds 1e10 x
        xc = x[c:c + (1 << 27)]
        na += int(torch.count_nonzero(xc < t.x0).item())
        nab += int(torch.count_nonzero(xc < t.x1).item())
    nb = nab - na
    nc = x.numel() - nab
    flops = 0
    for k in ks:
        ra = t.r_A[k]
        flops += na * (2 * (ra.degree_n() + ra.degree_m()) + 1 + (2 + 3 * k if k > 0 else 0))
        flops += nb * (25 + 3 * k) + nc * (3 + 2 * k)
    try:
        with open(os.path.join(ROOT, "profiles", "r01_fp64_peak.json")) as f:
            peak, kind = float(json.load(f)["fp64_tflops"]), "measured (tools/fp64_peak.cu)"
    except Exception:
        peak, kind = 37.2, "nominal (148 SMs x 64 DFMA/clk x 1.965 GHz x 2)"
    achieved = flops / step_s / 1e12
    return {"achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "peak_kind": kind,
            "algorithmic_flops_per_step": flops, "region_counts": [na, nb, nc]}


def accuracy_sample(x_dev, k, layout):
    """max |gpu - oracle| and |gpu - reference| on a strided sample."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import torch
    import pyoracle
    import paper_2512_10059_b200 as pkg
    n = x_dev.numel()
    m = min(20000, n)
    idx = torch.arange(m, device=x_dev.device, dtype=torch.int64) * (n // m)
    xs = x_dev[idx].contiguous()
    out = torch.empty(m * (k + 1), dtype=torch.float64, device=x_dev.device)
    pkg.eval_device(xs, k, out, layout=layout)
    g = out.view(k + 1, m).T.cpu().numpy() if layout == "soa" else out.view(m, k + 1).cpu().numpy()
    port = pyoracle.Port()
    xh = xs.cpu().numpy()
    hp = port.hp(xh, k)
    ref = port.boys_batch_many(xh, k)
    return {"max_abs_err_vs_oracle": float(np.abs(g - hp).max()),
            "max_abs_dev_vs_reference": float(np.abs(g - ref).max()),
            "eps_tol": 5e-14, "sample": "%d x strided over the timed batch, all orders 0..%d" % (m, k)}


def run_b200(args, world, rank, local):
    import torch
    import paper_2512_10059_b200 as pkg
    from paper_2512_10059_b200 import dist as D

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
    out = torch.empty(chunk * (k + 1), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    pieces = [(c, min(n, c + chunk)) for c in range(0, n, chunk)]
    ks = cfg.get("ks") or [k]
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

    e2e = None
    if not args.no_e2e and len(ks) == 1:
        try:
            e2e = run_e2e(args, x, world)
        except Exception as exc:  # e.g. pinned host memory exhausted; the device line still stands
            e2e = {"value": None, "unit": UNIT, "error": "%s: %s" % (type(exc).__name__, exc)}

    acc = None
    if rank == 0 and not args.no_accuracy:
        acc = accuracy_sample(x, k, layout)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        m = min(n, 4_000_000)
        xs = x[:m].cpu().numpy()  # the exact doubles the GPU evaluated
        t_all = v_all = 0.0
        for kk in ks:  # time-weighted over the sweep (one k unless cfg2)
            v, kind, passes, el = cpu_reference(xs, kk, threads, min_seconds=2.0 / len(ks))
            t_all += el
            v_all += v * el
        cpu = {"value": v_all / t_all, "unit": UNIT, "cores": threads, "kind": kind,
               "sample": "first %d x of the timed batch, k in %s, AoS, %d threads, %.2f s"
                         % (m, "0..%d" % max(ks) if len(ks) > 1 else str(k), threads, t_all)}

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
                       "l2": "inputs+outputs %.1f GB per launch >> 126 MB L2 (no flush needed)" % (alg_bytes / 1e9),
                       "parallelism": "dp%d (independent shards, no collective)" % world},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks, "accuracy": acc, "step_ms": step_stats,
        }
        if per_k is not None:
            line["per_k"] = per_k
        print(json.dumps(line), flush=True)


def run_e2e(args, x_dev, world):
    """Same metric through the host API: pinned host x -> device -> pinned host F.
    The full batch when its output fits comfortably in host RAM (cfg1), else
    the first 1e8 x (n_per_step says which)."""
    import torch
    import paper_2512_10059_b200 as pkg
    from paper_2512_10059_b200 import dist as D
    cfg = args.cfg
    k, layout = cfg["k"], cfg["layout"]
    # pinned host output per rank: 26 GB at 1e8 x, k=32 -- one rank gets the
    # full batch, N ranks share the host's RAM (1/N of the batch each, >= 1e7)
    n = min(cfg["n"], 100_000_000 if world == 1 else max(10_000_000, 100_000_000 // world))
    hx = torch.empty(n, dtype=torch.float64, pin_memory=True)
    hx.copy_(x_dev[:n])
    hout = torch.empty(n * (k + 1), dtype=torch.float64, pin_memory=True)
    xs, out = hx.numpy(), hout.numpy()
    tables = pkg.embedded_default()
    pkg.boys_batch_many(xs, k, tables, out, layout=layout)  # warm (pipeline buffers)
    D.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        pkg.boys_batch_many(xs, k, tables, out, layout=layout)
    el = time.perf_counter() - t0
    D.barrier()
    el = D.max_over_ranks(el)
    v = world * n * (k + 1) * args.e2e_steps / el
    return {"value": v, "unit": UNIT, "h2d_bytes_per_step": n * 8, "d2h_bytes_per_step": n * (k + 1) * 8,
            "steps": args.e2e_steps, "n_per_step": n,
            "api": "boys_batch_many -> boysfn_eval_host (pinned host buffers)", "layout": layout}


def main():
    args = parse_args()
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank == 0:  # the other ranks exit 0 without work
            run_reference_arm(args)
        return
    from paper_2512_10059_b200 import dist as D
    world, rank, local = D.init("nccl")
    try:
        run_b200(args, world, rank, local)
    finally:
        D.finalize()


if __name__ == "__main__":
    main()
