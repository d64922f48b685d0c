"""D2H copy-engine experiments (development aid): 2 GiB into pinned memory as
one copy, 8 chunks on one stream, 8 chunks on 2/3 streams, 2 halves concurrently."""
import torch


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        a.record()
        fn()
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


n = (2 << 30) // 8
d = torch.empty(n, dtype=torch.float64, device="cuda")
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
streams = [torch.cuda.Stream() for _ in range(3)]


def chunks(ns, nchunks=8):
    c = n // nchunks
    def f():
        for i in range(nchunks):
            s = streams[i % ns]
            with torch.cuda.stream(s):
                h[i * c:(i + 1) * c].copy_(d[i * c:(i + 1) * c], non_blocking=True)
    return f


def one():
    h.copy_(d, non_blocking=True)


for name, fn in (("one 2 GiB copy", one), ("8 chunks, 1 stream", chunks(1)), ("8 chunks, 2 streams", chunks(2)),
                 ("8 chunks, 3 streams", chunks(3)), ("2 halves, 2 streams", chunks(2, 2)),
                 ("32 chunks, 2 streams", chunks(2, 32))):
    ms = timed(fn)
    print("%-24s %.1f GB/s" % (name, (2 << 30) / ms / 1e6), flush=True)
