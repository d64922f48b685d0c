"""cudaHostRegister cost vs staging for pageable host output (development aid):
time register + D2H + unregister of pageable chunks against D2H into pinned
staging + memcpy, at several chunk sizes."""
import ctypes
import time

import numpy as np
import torch


def main():
    import os
    lib = None
    for name in ("libcudart.so.12", "libcudart.so"):
        try:
            lib = ctypes.CDLL(name)
            break
        except OSError:
            continue
    if lib is None:
        import glob
        import torch as _t
        cands = glob.glob(os.path.join(os.path.dirname(_t.__file__), "lib", "libcudart*.so*")) + \
            glob.glob("/usr/local/cuda/lib64/libcudart.so*")
        lib = ctypes.CDLL(cands[0])
    reg, unreg = lib.cudaHostRegister, lib.cudaHostUnregister
    reg.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint]
    unreg.argtypes = [ctypes.c_void_p]
    total = 4 << 30
    out = np.empty(total // 8)
    out[:] = 1.0  # touch
    dev = torch.empty(total // 8, dtype=torch.float64, device="cuda")
    for chunk_mb in (32, 128, 512):
        cb = chunk_mb << 20
        n = total // cb
        torch.cuda.synchronize()
        t = time.perf_counter()
        tr = 0.0
        for c in range(n):
            view = out[c * cb // 8:(c + 1) * cb // 8]
            t0 = time.perf_counter()
            assert reg(view.ctypes.data, cb, 0) == 0
            tr += time.perf_counter() - t0
            torch.from_numpy(view).copy_(dev[c * cb // 8:(c + 1) * cb // 8])
            t0 = time.perf_counter()
            assert unreg(view.ctypes.data) == 0
            tr += time.perf_counter() - t0
        el = time.perf_counter() - t
        print("register+D2H+unregister chunk %4d MB: %.1f GB/s total (register+unregister %.1f%% of time)"
              % (chunk_mb, total / el / 1e9, 100 * tr / el), flush=True)
    pin = torch.empty(128 << 17, dtype=torch.float64, pin_memory=True)
    t = time.perf_counter()
    for c in range(total // (128 << 20)):
        pin.copy_(dev[c * (128 << 17):(c + 1) * (128 << 17)])
        np.copyto(out[c * (128 << 17):(c + 1) * (128 << 17)], pin.numpy())
    el = time.perf_counter() - t
    print("serial staging 128 MB (D2H pinned + 1-thread memcpy): %.1f GB/s" % (total / el / 1e9))


if __name__ == "__main__":
    main()
