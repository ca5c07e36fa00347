"""Build libturbosat.so in-tree with nvcc for sm_100a (no JIT, no torch ext).

    python -m paper_2511_07737_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libturbosat.so")
def _nccl_include() -> str:
    """Directory of nccl.h: the NCCL wheel PyTorch ships (nvidia.nccl), any
    nvidia/nccl/include on sys.path, $NCCL_HOME/include or the system headers
    (the library itself is dlopen'ed at run time)."""
    cands = []
    try:
        import nvidia.nccl
        cands += [os.path.join(p, "include") for p in nvidia.nccl.__path__]
    except Exception:
        pass
    cands += [os.path.join(p, "nvidia", "nccl", "include") for p in sys.path if p]
    if os.environ.get("NCCL_HOME"):
        cands.append(os.path.join(os.environ["NCCL_HOME"], "include"))
    cands += ["/usr/include", "/usr/local/include", "/usr/local/cuda/include"]
    for c in cands:
        if os.path.exists(os.path.join(c, "nccl.h")):
            return c
    raise RuntimeError("nccl.h not found (install the nvidia-nccl wheel or set NCCL_HOME)")


NCCL_INC = _nccl_include()
SOURCES = ["capi.cu", "launch.cu", "k_clause.cu", "k_misc.cu", "k_update.cu", "k_update_blk.cu", "k_dense.cu", "k_fp64.cu", "k_shard.cu", "comm.cpp", "host_cnf.cpp", "host_cdcl.cpp", "host_gen.cpp"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",                      # canonical arithmetic: no implicit FMA contraction
    "-Xcompiler", "-fPIC,-O2,-ffp-contract=off",
    "-Xptxas", "-v",
    "-I", os.path.join(ROOT, "include"),
    "-I", NCCL_INC,
]
LINK_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "--shared", "-cudart", "static", "-ldl"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "turbosat.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines: tuple = ()) -> str:
    """Compile libturbosat.so.  `out`/`defines` build an experimental
    variant next to it (e.g. -DTSAT_VARIANT=1); bench/tests pick one with the
    TSAT_LIB environment variable."""
    if out is None and not defines and not force and not _stale():
        return LIB
    import tempfile
    from concurrent.futures import ThreadPoolExecutor
    nvcc = os.environ.get("NVCC", "nvcc")
    dst = out or LIB
    tmp = dst + f".tmp{os.getpid()}"
    with tempfile.TemporaryDirectory(prefix="tsat_build_") as bd:
        def compile_one(src):           # one nvcc per translation unit, in parallel
            obj = os.path.join(bd, src + ".o")
            cmd = [nvcc, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", "-o", obj, os.path.join(CSRC, src)]
            return obj, subprocess.run(cmd, capture_output=True, text=True)
        with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
            results = list(ex.map(compile_one, SOURCES))
        for _, r in results:
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError("nvcc failed building libturbosat.so")
            if verbose:
                sys.stderr.write(r.stderr)
        r = subprocess.run([nvcc, *LINK_FLAGS, "-o", tmp, *[o for o, _ in results]], capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed linking libturbosat.so")
    os.replace(tmp, dst)
    return dst


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
