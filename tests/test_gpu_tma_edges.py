"""The TMA store paths at their edges: SoA with an odd ld (any odd n with the
default ld = n) or an 8-B-aligned output (per-row 1D bulk copies,
kStoreSoABlockBulk*), a last tile ending at an odd n (the tensor store clips
only at 16-B granularity, so that tile goes out by LSU), and batches above the
int32 tensor-coordinate range (split launches with a global first-bad
index).  Bit-identical to the per-warp LSU path; padding columns untouched."""
import pytest

import paper_2512_10059_b200 as pkg

pytestmark = pytest.mark.gpu


def _soa(torch, x, k, out, ld, path, monkeypatch):
    if path:
        monkeypatch.setenv("BOYSFN_SOA_PATH", path)
    pkg.eval_device(x, k, out, layout="soa", ld=ld)
    torch.cuda.synchronize()
    monkeypatch.delenv("BOYSFN_SOA_PATH", raising=False)


@pytest.mark.parametrize("n", [4099, 100_001, 257])
def test_soa_tma_odd_ld_and_misaligned_out(cuda, monkeypatch, n):
    torch = cuda
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    pkg.generate_uniform(x, 17, 0.0, 60.0)
    for k in (0, 1, 7, 8, 13, 16, 31, 32):
        ref = torch.empty((k + 1) * n, dtype=torch.float64, device="cuda")
        _soa(torch, x, k, ref, n, "warp", monkeypatch)
        ref = ref.view(k + 1, n).view(torch.int64)
        for path in ("blocktma", "blocktmabin", "blockbulk", "blockbulkw", "blockbulkw3", None):
            for shift, ld in ((0, n), (1, n), (0, n + 1), (1, n + 3), (1, n + 2)):
                buf = torch.full((shift + (k + 1) * ld,), float("nan"), dtype=torch.float64, device="cuda")
                out = buf[shift:]
                _soa(torch, x, k, out, ld, path, monkeypatch)
                got = out.view(k + 1, ld)[:, :n].contiguous().view(torch.int64)
                assert torch.equal(got, ref), (n, k, path, shift, ld)
                if ld > n:  # the padding columns are untouched
                    assert torch.isnan(out.view(k + 1, ld)[:, n:]).all(), (n, k, path, shift, ld)


@pytest.mark.parametrize("n", [4099, 257])
def test_generic_tma_odd_n_padded_ld(cuda, monkeypatch, n):
    """The run-time-k kernel's SoA tensor store (forced with BOYSFN_GENERIC=3)
    at an odd n inside an even, padded ld: no element past n is written."""
    torch = cuda
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    pkg.generate_uniform(x, 19, 0.0, 60.0)
    for k in (3, 8):
        ref = torch.empty((k + 1) * n, dtype=torch.float64, device="cuda")
        _soa(torch, x, k, ref, n, "warp", monkeypatch)
        ld = n + 5
        out = torch.full(((k + 1) * ld,), float("nan"), dtype=torch.float64, device="cuda")
        monkeypatch.setenv("BOYSFN_GENERIC", "3")
        pkg.eval_device(x, k, out, layout="soa", ld=ld)
        torch.cuda.synchronize()
        monkeypatch.delenv("BOYSFN_GENERIC", raising=False)
        o = out.view(k + 1, ld)
        assert torch.equal(o[:, :n].contiguous().view(torch.int64), ref.view(k + 1, n).view(torch.int64)), k
        assert torch.isnan(o[:, n:]).all(), k


def test_soa_tma_above_int32_coordinates(cuda, monkeypatch):
    """2^31 + 1e6 x through the tensor-store kernel (forced at k = 0 to keep the
    output at 17 GB): split launches, the same values as the LSU kernel on
    strided samples, the first bad index reported in the global numbering."""
    torch = cuda
    n = (1 << 31) + 1_000_000
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    pkg.generate_uniform(x, 21, 0.0, 50.0)
    bad = (1 << 31) + 5
    x[bad] = -1.0
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    fb = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    monkeypatch.setenv("BOYSFN_SOA_PATH", "blocktma")
    pkg.eval_device(x, 0, out, layout="soa", first_bad=fb)
    torch.cuda.synchronize()
    monkeypatch.delenv("BOYSFN_SOA_PATH", raising=False)
    assert int(fb.item()) == bad
    idx = torch.cat([torch.arange(0, n, 9973, device="cuda"), torch.arange(n - 70000, n, device="cuda"),
                     torch.arange((1 << 31) - 70000, (1 << 31) + 70000, device="cuda")])
    idx = idx[idx != bad]
    xs = x[idx].contiguous()
    ref = torch.empty_like(xs)
    _soa(torch, xs, 0, ref, xs.numel(), "warp", monkeypatch)
    assert torch.equal(out[idx].view(torch.int64), ref.view(torch.int64))
    del x, out
    torch.cuda.empty_cache()


def test_aos_padded_tma_above_int32_coordinates(cuda, monkeypatch):
    """The padded AoS stage's 2D tensor store (rows of 4 doubles, k = 3) at
    2^31 + 1e6 x: split launches, values equal to the LSU kernel's on strided
    samples and around the split, the first bad index global (86 GB)."""
    torch = cuda
    n = (1 << 31) + 1_000_000
    k = 3
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    pkg.generate_uniform(x, 22, 0.0, 50.0)
    bad = (1 << 31) + 9
    x[bad] = float("nan")
    out = torch.empty(n * (k + 1), dtype=torch.float64, device="cuda")
    fb = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    monkeypatch.setenv("BOYSFN_AOS_PATH", "blocktma")
    pkg.eval_device(x, k, out, layout="aos", first_bad=fb)
    torch.cuda.synchronize()
    monkeypatch.delenv("BOYSFN_AOS_PATH", raising=False)
    assert int(fb.item()) == bad
    split = (1 << 31) - (1 << 20)  # kTmaMaxX
    idx = torch.cat([torch.arange(0, n, 9973, device="cuda"), torch.arange(n - 70000, n, device="cuda"),
                     torch.arange(split - 70000, split + 70000, device="cuda")])
    idx = idx[idx != bad]
    xs = x[idx].contiguous()
    m = xs.numel()
    ref = torch.empty(m * (k + 1), dtype=torch.float64, device="cuda")
    _soa(torch, xs, k, ref, m, "warp", monkeypatch)
    got = out.view(n, k + 1)[idx]
    assert torch.equal(got.contiguous().view(torch.int64), ref.view(k + 1, m).T.contiguous().view(torch.int64))
    del x, out
    torch.cuda.empty_cache()
