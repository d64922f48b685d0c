"""Every output path (per-warp SoA / AoS-transpose, block-tile LSU and TMA,
region-binned kernels) computes each value with the same arithmetic routine, so
all must agree BIT FOR BIT with one another -- on ragged sizes around the 32-x
tile, 128-x block and 512-x chunk edges and for every order 0..32.  The default
selection is covered by test_gpu_parity.py against the oracle."""
import os

import numpy as np
import pytest

import paper_2512_10059_b200 as pkg

pytestmark = pytest.mark.gpu

PATHS = [("soa", "warp"), ("soa", "block"), ("soa", "binned"), ("soa", "blocktma"), ("soa", "blocktmabin"),
         ("aos", "xpose"), ("aos", "binned"), ("aos", "blocktma"), ("aos", "blocktmabin"),
         ("soa", "blockbulk"), ("soa", "blockbulkw"), ("soa", "blockbulkw3")]


def run(torch, x, k, lay, path, monkeypatch):
    monkeypatch.setenv("BOYSFN_SOA_PATH" if lay == "soa" else "BOYSFN_AOS_PATH", path)
    n = x.numel()
    out = torch.full((n * (k + 1),), float("nan"), dtype=torch.float64, device="cuda")
    pkg.eval_device(x, k, out, layout=lay)
    torch.cuda.synchronize()
    monkeypatch.delenv("BOYSFN_SOA_PATH", raising=False)
    monkeypatch.delenv("BOYSFN_AOS_PATH", raising=False)
    return out.view(k + 1, n).T.contiguous() if lay == "soa" else out.view(n, k + 1)


@pytest.mark.parametrize("n", [1, 31, 33, 127, 128, 129, 511, 513, 4099, 200_003])
def test_all_paths_bit_identical(cuda, monkeypatch, n):
    torch = cuda
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    pkg.generate_uniform(x, 100 + n, 0.0, 45.0)
    ks = range(33) if n in (129, 4099) else (0, 1, 3, 4, 7, 8, 9, 11, 15, 16, 19, 31, 32)
    for k in ks:
        ref = run(torch, x, k, "soa", "warp", monkeypatch).view(torch.int64)
        for lay, path in PATHS[1:]:
            got = run(torch, x, k, lay, path, monkeypatch).view(torch.int64)
            assert torch.equal(got, ref), (n, k, lay, path)


def test_all_paths_report_first_bad(cuda, port, monkeypatch):
    torch = cuda
    xs = port.gen_uniform(5000, 3, 0.0, 30.0)
    xs[4321] = np.inf
    xs[777] = -3.0
    x = torch.from_numpy(xs).cuda()
    for k in (0, 4, 8, 16):
        for lay, path in PATHS:
            monkeypatch.setenv("BOYSFN_SOA_PATH" if lay == "soa" else "BOYSFN_AOS_PATH", path)
            fb = torch.full((1,), -1, dtype=torch.int64, device="cuda")
            out = torch.empty(xs.size * (k + 1), dtype=torch.float64, device="cuda")
            pkg.eval_device(x, k, out, layout=lay, first_bad=fb)
            monkeypatch.delenv("BOYSFN_SOA_PATH", raising=False)
            monkeypatch.delenv("BOYSFN_AOS_PATH", raising=False)
            assert int(fb.item()) == 777, (k, lay, path)


@pytest.mark.parametrize("n", [1_000_003, 3_000_001])
def test_block_paths_static_and_claimed_schedules(cuda, monkeypatch, n):
    """Batches around the block-TMA kernels' static/claimed schedule switch
    (<= 16 tiles per block: static) agree bit for bit with the per-warp path."""
    torch = cuda
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    pkg.generate_uniform(x, 7 + n, 0.0, 60.0)
    for k in (0, 7, 8, 16, 32):
        ref = run(torch, x, k, "soa", "warp", monkeypatch).view(torch.int64)
        for lay, path in (("soa", "blocktma"), ("soa", "blocktmabin"), ("soa", "blockbulk"), ("soa", "blockbulkw"), ("soa", "blockbulkw3"),
                          ("aos", "blocktma"), ("aos", "blocktmabin"), ("aos", "")):
            got = run(torch, x, k, lay, path, monkeypatch).view(torch.int64)
            assert torch.equal(got, ref), (n, k, lay, path)
