"""paper_2511_07737_b200 - B200-native (sm_100a) TurboSAT batched
differentiable SAT step (arXiv 2511.07737) behind a C-ABI library.

    from paper_2511_07737_b200 import Solver
    s = Solver(device=0)
    s.load_dimacs(open("f.cnf", "rb").read())
    s.init_batch(N_global=4096, seed=1)
    info = s.step(30)            # 30 iterations, one CUDA graph
    unsat = s.query_unsat()

The package holds only the hot path: ``csrc/`` (kernels + C-ABI runtime),
``binding.py`` (ctypes marshalling) and ``build.py`` (nvcc, sm_100a).
"""
from .binding import (  # noqa: F401
    LIB_PATH,
    Solver,
    StepInfo,
    TsatError,
    cdcl_portfolio,
    cdcl_solve,
    config_default,
    gen_industrial,
    gen_planted,
    load_library,
    nccl_unique_id,
    parse_dimacs,
    verify_model,
    write_dimacs,
)

__all__ = ["Solver", "StepInfo", "TsatError", "cdcl_portfolio", "cdcl_solve", "config_default", "load_library", "nccl_unique_id",
           "parse_dimacs", "LIB_PATH", "gen_planted", "gen_industrial", "write_dimacs",
           "verify_model"]
