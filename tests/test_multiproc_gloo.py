"""CPU multi-process tests (gloo, world_size 2) of the multi-GPU plumbing in
paper_2512_10059_b200/dist.py: shards are disjoint and cover the batch, the
global-index-keyed stream makes the union of shards bit-identical to one
process's input (and hence its output), and the timing reduction is the max
over ranks.  The Boys evaluation inside each rank is the CPU oracle here --
this exercises the host-side sharding only (the kernels never communicate)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port_no, n_per, k, result_dir):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no), WORLD_SIZE=str(world),
                      RANK=str(rank), LOCAL_RANK=str(rank))
    import torch
    import torch.distributed as dist
    import pyoracle
    from paper_2512_10059_b200 import dist as D
    w, r, _ = D.init("gloo")
    assert (w, r) == (world, rank)
    port = pyoracle.Port()
    b, e = D.weak_shard(n_per, rank)
    xs = port.gen_uniform(e - b, 2, 0.0, 100.0, offset=b)
    f = port.boys_batch_many(xs, k)
    np.save(os.path.join(result_dir, "x%d.npy" % rank), xs)
    np.save(os.path.join(result_dir, "f%d.npy" % rank), f)
    # strong shards: gather the ranges
    rng = torch.tensor(D.strong_shard(1001, world, rank), dtype=torch.int64)
    allr = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allr, rng)
    np.save(os.path.join(result_dir, "r%d.npy" % rank), torch.stack(allr).numpy())
    D.barrier()
    m = D.max_over_ranks(10.0 + rank)
    np.save(os.path.join(result_dir, "m%d.npy" % rank), np.array([m]))
    D.finalize()


@pytest.mark.timeout(300)
def test_two_rank_sharding_gloo(tmp_path, port):
    world, n_per, k = 2, 5000, 8
    mp.start_processes(_worker, args=(world, _free_port(), n_per, k, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    xs = np.concatenate([np.load(tmp_path / ("x%d.npy" % r)) for r in range(world)])
    fs = np.concatenate([np.load(tmp_path / ("f%d.npy" % r)) for r in range(world)])
    single_x = port.gen_uniform(world * n_per, 2, 0.0, 100.0)
    assert np.array_equal(xs.view(np.uint64), single_x.view(np.uint64))
    assert np.array_equal(fs.view(np.uint64), port.boys_batch_many(single_x, k).view(np.uint64))
    ranges = np.load(tmp_path / "r0.npy")
    assert ranges[0, 0] == 0 and ranges[-1, 1] == 1001
    assert all(ranges[i, 1] == ranges[i + 1, 0] for i in range(world - 1))
    assert [float(np.load(tmp_path / ("m%d.npy" % r))[0]) for r in range(world)] == [11.0, 11.0]
