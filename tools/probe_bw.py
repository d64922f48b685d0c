"""Bandwidth ceilings for a write-dominated kernel (development aid).

Times, with CUDA events after warm-up: a pure device write (fill_) and a copy
over buffers the size of one bench step, so the Boys kernel's fraction of
MEASURED_PEAKS.json's copy figure can be read against the write-only ceiling.
"""
import torch


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e-3


def main():
    n = 100_000_000 * 33
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    t = timeit(lambda: out.fill_(1.0))
    print("fill_  %.1f GB  %.3f ms  %.0f GB/s (write only)" % (n * 8 / 1e9, t * 1e3, n * 8 / t / 1e9))
    src = torch.empty(n // 2, dtype=torch.float64, device="cuda")
    dst = torch.empty(n // 2, dtype=torch.float64, device="cuda")
    t = timeit(lambda: dst.copy_(src))
    print("copy_  %.1f GB  %.3f ms  %.0f GB/s (read+write)" % (n * 8 / 1e9, t * 1e3, n * 8 / t / 1e9))


if __name__ == "__main__":
    main()
