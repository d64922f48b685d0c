"""FP64-pipe instructions per x by region and order, measured (development aid).

    ncu --metrics sm__inst_executed_pipe_fp64.sum,sm__inst_executed_pipe_xu.sum,smsp__inst_executed.sum \
        --clock-control none -k regex:boys_eval --csv --log-file gpurun_out/fp64.csv python tools/fp64_pipe_table.py run
    python tools/fp64_pipe_table.py table gpurun_out/fp64.csv profiles/r02_fp64_pipe_ops.json

`run` evaluates, for k = 0..32 and each region, one batch of x drawn only from
that region (A: [0, x0), B: [x0, x1), C: [x1, 100)) through the default
eval_device path (SoA), so each launch's counters are that region's cost.
`table` turns the launch list into warp-instruction counts per x:
fp64 = FP64-pipe lane-ops per x (DFMA/DMUL/DADD/DSETP/...), xu = MUFU
(RCP64H/RSQ64H) per x, all = all instructions per x.  bench.py's
roofline.fp64 weights these with the step's own region counts.
"""
import csv
import json
import os
import sys

N = 1 << 22
REGIONS = ("A", "B", "C")


def run():
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2512_10059_b200 as pkg
    t = pkg.embedded_default()
    bounds = {"A": (0.0, t.x0), "B": (t.x0, t.x1), "C": (t.x1, 100.0)}
    out = torch.empty(N * 33, dtype=torch.float64, device="cuda")
    xs = {}
    for r in REGIONS:
        x = torch.empty(N, dtype=torch.float64, device="cuda")
        pkg.generate_uniform(x, 11, *bounds[r])
        x.clamp_(min=bounds[r][0])
        x[x >= bounds[r][1]] = bounds[r][0]  # half-open: x < hi
        xs[r] = x
    for k in range(33):
        for r in REGIONS:
            pkg.eval_device(xs[r], k, out[: N * (k + 1)], layout="soa")
    torch.cuda.synchronize()


def table(csv_path, out_path):
    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 10]
    hdr = rows[0]
    ci = {h: i for i, h in enumerate(hdr)}
    launches = {}
    for r in rows[1:]:
        if "boys_eval" not in r[ci["Kernel Name"]]:
            continue
        lid = int(r[ci["ID"]])
        v = float(r[ci["Metric Value"]].replace(",", ""))
        launches.setdefault(lid, {})[r[ci["Metric Name"]]] = v
    ids = sorted(launches)
    assert len(ids) == 33 * 3, len(ids)
    tab = {}
    for j, lid in enumerate(ids):
        k, reg = divmod(j, 3)
        m = launches[lid]
        tab.setdefault(str(k), {})[REGIONS[reg]] = {
            "fp64": 32 * m["sm__inst_executed_pipe_fp64.sum"] / N,
            "xu": 32 * m["sm__inst_executed_pipe_xu.sum"] / N,
            "all": 32 * m["smsp__inst_executed.sum"] / N}
    with open(out_path, "w") as f:
        json.dump({"source": "ncu launch counters, %d x per launch drawn from one region, default SoA path" % N,
                   "unit": "warp instructions x 32 / x (lane-ops per x)", "per_k": tab}, f, indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run()
    else:
        table(sys.argv[2], sys.argv[3])
