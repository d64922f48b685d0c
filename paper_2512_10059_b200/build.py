"""In-tree build of libboysfn_b200.so (sm_100a) and the test programs.

    python -m paper_2512_10059_b200.build          # or __graft_entry__.build()

nvcc cross-compiles for sm_100a without a GPU.  Outputs stay in the tree
(paper_2512_10059_b200/_lib/, build/) so they travel to the GPU box with the
gpurun snapshot; they are git-ignored.  cudart is linked statically and the
static archive's symbols are kept local, so the library never binds to the
libcudart that torch happens to have loaded.
"""
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
CPP = os.path.join(PKG, "cpp")
OBJ = os.path.join(ROOT, "build", "obj")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libboysfn_b200.so")
SHIM_TEST = os.path.join(ROOT, "build", "shim_test")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-Xptxas", "-v", "--expt-relaxed-constexpr"]
CXX_FLAGS = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra"]

CU_SOURCES = ["kernels_soa.cu", "kernels_aos_xpose.cu", "kernels_soa_block.cu", "kernels_soa_binned.cu",
              "kernels_aos_binned.cu",
              "kernels_soa_block_tma.cu", "kernels_aos_block_tma.cu", "kernels_soa_block_tma_bin.cu",
              "kernels_aos_block_tma_bin.cu", "kernels_soa_block_bulk.cu", "kernels_soa_block_bulk_w.cu", "kernels_soa_block_bulk_w3.cu", "kernels_region.cu", "kernels_generic.cu", "alg2.cu", "verify.cu",
              "gen_scan.cu",
              "capi.cu"]
CPP_SOURCES = ["shim_tables.cpp", "shim_eval.cpp"]


def _run(cmd, log=None):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        with open(log, "w") as f:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n%s\n%s%s" % (" ".join(cmd), r.stdout, r.stderr[-8000:]))
    return r


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h", ".inc"))]
    hs += [os.path.join(ROOT, "include", "boysfn_b200.h")]
    hs += [os.path.join(CPP, "include", "boysfn", f) for f in ("eval.hpp", "tables.hpp", "verify.hpp")]
    return hs


def build_library(force=False, verbose=True, variant=None, defines=()):
    """variant/defines: an experimental build into _lib/variants/<variant>/
    (selected at run time with BOYSFN_LIB); the product build has neither."""
    global OBJ, LIB
    if variant:
        OBJ = os.path.join(ROOT, "build", "obj_" + variant)
        LIB = os.path.join(LIBDIR, "variants", variant, "libboysfn_b200.so")
        os.makedirs(os.path.dirname(LIB), exist_ok=True)
    extra = ["-D" + d for d in defines]
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    hdrs = _headers()
    jobs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src + ".o")
        if force or _stale(o, [s] + hdrs):
            jobs.append(([NVCC] + NVCC_FLAGS + extra + ["-c", s, "-o", o], os.path.join(OBJ, src + ".ptxas.log")))
    for src in CPP_SOURCES:
        s = os.path.join(CPP, "src", src)
        o = os.path.join(OBJ, src + ".o")
        if force or _stale(o, [s] + hdrs):
            jobs.append((["g++"] + CXX_FLAGS + ["-I", os.path.join(CPP, "include"), "-c", s, "-o", o], None))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        list(ex.map(lambda j: _run(*j), jobs))
    objs = [os.path.join(OBJ, s + ".o") for s in CU_SOURCES + CPP_SOURCES]
    if force or jobs or _stale(LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs +
             ["-Xlinker", "--exclude-libs,ALL", "-Xlinker", "-Bsymbolic", "-lrt", "-lpthread", "-ldl"])
        if verbose:
            print("built", LIB)
    return LIB


def build_shim_test(force=False):
    src = os.path.join(ROOT, "tests", "cpp", "shim_test.cpp")
    if not os.path.exists(src):
        return None
    if force or _stale(SHIM_TEST, [src, LIB] + _headers()):
        _run(["g++"] + CXX_FLAGS[:2] + ["-I", os.path.join(CPP, "include"), "-I",
                                        os.path.join(ROOT, "oracle"), src, "-o", SHIM_TEST,
                                        "-L", LIBDIR, "-lboysfn_b200", "-Wl,-rpath," + LIBDIR,
                                        "-L", os.path.join(ROOT, "oracle", "_build"), "-lboys_oracle",
                                        "-Wl,-rpath," + os.path.join(ROOT, "oracle", "_build")])
    return SHIM_TEST


GEN = os.path.join(LIBDIR, "boysfn_gen")
GEN_SOURCES = ["special.cpp", "minimax.cpp", "gen_main.cpp"]


def build_gen(force=False):
    """The native table generator (binary128 minimax exchange and Walsh search,
    GPU extremum scan through the C ABI)."""
    srcs = [os.path.join(CPP, "src", "gen", f) for f in GEN_SOURCES]
    hdrs = [os.path.join(CPP, "include", "boysfn_gen", "minimax.hpp")] + [
        os.path.join(CPP, "include", "boysfn", f) for f in ("tables.hpp", "verify.hpp")]
    if force or _stale(GEN, srcs + hdrs + [LIB]):
        _run(["g++", "-std=gnu++20", "-O2", "-Wall", "-Wextra", "-I", os.path.join(CPP, "include")] + srcs +
             ["-o", GEN, "-L", LIBDIR, "-lboysfn_b200", "-Wl,-rpath,$ORIGIN", "-lquadmath", "-lpthread"])
    return GEN


def build_oracle():
    """The test-only checkers (oracle/Makefile): always the C restatement, plus
    the compiled reference where /root/reference exists."""
    _run(["make", "-s", "-C", os.path.join(ROOT, "oracle")])


def build_all(force=False):
    build_oracle()
    build_library(force=force)
    build_shim_test(force=force)
    build_gen(force=force)


if __name__ == "__main__":
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        build_library(force=True, variant=sys.argv[i + 1], defines=sys.argv[i + 2:])
    else:
        build_all(force="--force" in sys.argv)
