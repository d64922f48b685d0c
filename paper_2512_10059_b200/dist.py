"""Multi-GPU plumbing: one process per GPU, independent shards, no data-path
collective (every x is independent: eval.cpp:92-95).

torch.distributed carries only the timing barrier and the max-over-ranks
reduction; the Boys kernels never communicate.  The synthetic stream is keyed
by the GLOBAL index (boysfn_generate_uniform's offset), so the union of the
shards is bit-for-bit the single-GPU input whatever the world size.
"""
import os


def env_world():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def weak_shard(n_per_rank, rank):
    """Weak scaling: rank r owns global indices [r*n, (r+1)*n)."""
    return rank * n_per_rank, (rank + 1) * n_per_rank


def strong_shard(n_total, world, rank):
    """Strong scaling: contiguous near-equal ranges covering [0, n_total)."""
    base, extra = divmod(n_total, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def init(backend="nccl"):
    """Initialise the process group from the torchrun environment (127.0.0.1
    rendezvous is the caller's MASTER_ADDR); no-op for a single process."""
    import torch
    import torch.distributed as dist
    world, rank, local = env_world()
    if world > 1 and not dist.is_initialized():
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    elif world == 1 and backend == "nccl" and torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def barrier():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


def max_over_ranks(value):
    """Max of a per-rank float (device-timed durations): the job finishes when
    the slowest rank does."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def finalize():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()
