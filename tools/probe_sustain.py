"""Per-launch timing under different launch cadences (development aid):
isolated launches (idle gap before each) vs back-to-back trains, with NVML
SM clock / power samples, to separate kernel speed from sustained-load effects.

    python tools/probe_sustain.py soa:8 aos:blocktmabin:8 soa:32     (layout[:path]:k)
"""
import os
import statistics
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_10059_b200 as pkg  # noqa: E402


def sampler(rows, stop):
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    while not stop.is_set():
        rows.append((time.perf_counter(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                     pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                     pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        stop.wait(0.005)


def main():
    n = 100_000_000
    specs = [s.split(":") for s in sys.argv[1:]] or [["soa", "8"]]
    specs = [(s[0], s[1] if len(s) == 3 else "", s[-1]) for s in specs]
    kmax = max(int(s[2]) for s in specs)
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    pkg.generate_uniform(x, 2, 0.0, 100.0)
    out = torch.empty(n * (kmax + 1), dtype=torch.float64, device="cuda")
    rows, stop = [], threading.Event()
    th = threading.Thread(target=sampler, args=(rows, stop), daemon=True)
    th.start()
    for lay, path, ks in specs:
        k = int(ks)
        os.environ.pop("BOYSFN_SOA_PATH", None)
        os.environ.pop("BOYSFN_AOS_PATH", None)
        if path:
            os.environ["BOYSFN_SOA_PATH" if lay == "soa" else "BOYSFN_AOS_PATH"] = path
        o = out[: n * (k + 1)]
        for _ in range(3):
            pkg.eval_device(x, k, o, layout=lay)
        torch.cuda.synchronize()
        # isolated
        iso = []
        for _ in range(10):
            time.sleep(0.05)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            pkg.eval_device(x, k, o, layout=lay)
            b.record()
            b.synchronize()
            iso.append(a.elapsed_time(b))
        # trains
        for train in (10, 200):
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(train + 1)]
            time.sleep(0.1)
            t0 = time.perf_counter()
            evs[0].record()
            for j in range(train):
                pkg.eval_device(x, k, o, layout=lay)
                evs[j + 1].record()
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            per = [evs[j].elapsed_time(evs[j + 1]) for j in range(train)]
            win = [r for r in rows if t0 <= r[0] <= t1]
            print("%s:%s k=%d train=%d  first %.3f  median %.3f  last %.3f  min %.3f ms | isolated median %.3f | "
                  "sm_mhz med %s  power max %.0f W  reasons %s" % (
                      lay, path, k, train, per[0], statistics.median(per), per[-1], min(per), statistics.median(iso),
                      statistics.median([r[1] for r in win]) if win else None,
                      max([r[2] for r in win]) if win else 0, sorted({hex(r[3]) for r in win})), flush=True)
    stop.set()


if __name__ == "__main__":
    main()
