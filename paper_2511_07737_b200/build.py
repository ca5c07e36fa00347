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
    """nccl.h of the NCCL PyTorch ships (the library itself is dlopen'ed)."""
    try:
        import nvidia.nccl
        return os.path.join(list(nvidia.nccl.__path__)[0], "include")
    except Exception:
        return "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/include"


NCCL_INC = _nccl_include()
SOURCES = ["capi.cu", "launch.cu", "k_clause.cu", "k_misc.cu", "k_update.cu", "k_shard.cu", "comm.cpp", "host_cnf.cpp"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",                      # canonical arithmetic: no implicit FMA contraction
    "-Xcompiler", "-fPIC,-O2,-ffp-contract=off",
    "-Xptxas", "-v",
    "--shared",
    "-cudart", "static",
    "-I", os.path.join(ROOT, "include"),
    "-I", NCCL_INC,
    "-ldl",
]


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
    nvcc = os.environ.get("NVCC", "nvcc")
    dst = out or LIB
    tmp = dst + f".tmp{os.getpid()}"
    cmd = [nvcc, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-o", tmp, *[os.path.join(CSRC, s) for s in SOURCES]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libturbosat.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, dst)
    return dst


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
