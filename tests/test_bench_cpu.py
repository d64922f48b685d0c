"""bench.py's launcher and reference arm on CPU (no GPU): `--gpus N` starts N
ranks by itself (torchrun, gloo in --dry-run) and exactly one JSON line comes
out; the reference arm times the reference on the host alone."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*argv, timeout=300):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *argv], capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    return lines


def test_gpus_n_self_launches_n_ranks_one_line():
    for n in (2, 3):
        lines = _run("--gpus", str(n), "--dry-run")
        assert len(lines) == 1, lines
        d = json.loads(lines[0])
        assert d["n_gpus"] == n and d["dry_run"] is True
        assert d["max_over_ranks"] == float(n)  # rank r reported r+1: the max came from the last rank


def test_reference_arm_cfg0_single_thread():
    lines = _run("--impl", "reference", "--config", "cfg0", "--steps", "2", "--warmup", "3")
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 0 and d["host_threads"] == 1
    assert d["cpu_baseline"]["cores"] == 1 and d["config"]["same_batch_as_device_arm"] is True
    assert d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0
