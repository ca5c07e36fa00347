"""CPU-side tests of the C-ABI library: it loads, exports every symbol that
include/turbosat.h declares, and its host-only logic (DIMACS parser, defaults)
behaves per SPEC S:41-49.  No compute calls (no GPU here)."""
import ctypes as ct
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2511_07737_b200 import build
    build.build()
    from paper_2511_07737_b200 import binding
    return binding.load_library()


def _declared():
    txt = open(os.path.join(ROOT, "include", "turbosat.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(tsat_[a-z_0-9]+)\s*\(", txt)))


def test_exports_every_declared_symbol(lib):
    names = _declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n


def test_binding_covers_every_symbol():
    from paper_2511_07737_b200 import binding
    assert set(_declared()) == set(binding._SIGS)


def test_library_is_sm100a():
    """The shared library carries sm_100a SASS (cuobjdump)."""
    import shutil
    import subprocess
    from paper_2511_07737_b200 import LIB_PATH
    if not shutil.which("cuobjdump"):
        pytest.skip("no cuobjdump")
    out = subprocess.run(["cuobjdump", "--list-elf", LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_config_defaults(lib):
    from paper_2511_07737_b200 import config_default
    c = config_default()
    assert (c.tau, c.normalize, c.beta1, c.beta2, c.eps, c.weight_decay) == (1.0, 1, 0.9, 0.999, 1e-8, 1e-2)
    assert (c.lr0, c.lr_min, c.decay_factor, c.decay_every, c.restart_every) == (0.1, 1e-15, 10.0, 30, 360)
    assert c.noise_sigma == 0.0 and c.eps_norm == 1e-8
    assert lib.tsat_status_string(2) == b"TSAT_E_PARSE"


def _parse(text):
    from paper_2511_07737_b200 import parse_dimacs
    return parse_dimacs(text.encode() if isinstance(text, str) else text)


def test_parse_paper_example():
    """the Fig. 1 instance, clause 2 = (x3 v x4)."""
    info = _parse("c fig 1\np cnf 4 5\n1 2 0\n3 4 0\n-1 -3 0\n-2 4 0\n1 -4 0\n")
    assert (info.V, info.C, info.nnz, info.K) == (4, 5, 10, 2)
    assert info.n_warnings == 0 and info.has_empty == 0


def test_parse_dedup_tautology_empty_and_warnings():
    info = _parse("p cnf 2 1\n1 1 -2 0\n")                 # S:49 duplicate literal
    assert (info.nnz, info.n_duplicates) == (2, 1)
    info = _parse("p cnf 2 2\n1 -1 2 0\n0\n")              # tautology kept, empty clause kept
    assert info.n_tautologies == 1 and info.has_empty == 1 and info.C == 2
    info = _parse("p cnf 3 5\n1 2 0\n-3 0\n")              # header/body mismatch: warning
    assert info.C == 2 and info.header_C == 5 and info.n_warnings == 1
    info = _parse("p cnf 3 1\n1 2\n 3 0\n")                 # clause over two lines
    assert (info.C, info.nnz) == (1, 3)
    info = _parse("p cnf 3 1\n1 2 3")                       # missing final 0: warning
    assert info.C == 1 and info.n_warnings == 1


@pytest.mark.parametrize("text", [
    "p cnf x 1\n1 0\n",            # malformed header
    "p dnf 2 1\n1 0\n",
    "1 2 0\n",                      # clause before header
    "p cnf 2 1\n1 -0 2 0\n",        # -0 inside a clause
    "p cnf 2 1\n3 0\n",             # variable > V
    "p cnf 2 1\n1 a 0\n",           # non-integer token
    "c only a comment\n",           # no header
])
def test_parse_errors(text):
    from paper_2511_07737_b200 import TsatError
    with pytest.raises(TsatError) as ei:
        _parse(text)
    assert ei.value.name == "TSAT_E_PARSE"


def test_parse_clause_length_limit():
    """K <= 15 is supported (KB = 16 bins); longer clauses are TSAT_E_RANGE."""
    from paper_2511_07737_b200 import TsatError
    info = _parse("p cnf 15 1\n" + " ".join(str(i) for i in range(1, 16)) + " 0\n")
    assert info.K == 15
    with pytest.raises(TsatError) as ei:
        _parse("p cnf 16 1\n" + " ".join(str(i) for i in range(1, 17)) + " 0\n")
    assert ei.value.name == "TSAT_E_RANGE"


def test_parse_roundtrip_generated():
    """DIMACS written by tsat_synth parses back to the same sizes."""
    from tsat_synth import industrial_cnf, planted_ksat, to_dimacs
    for cnf in (planted_ksat(300, 1260, 3, 4), industrial_cnf(400, 1500, 2)):
        info = _parse(to_dimacs(cnf, "roundtrip"))
        assert (info.V, info.C, info.nnz, info.K) == (cnf.V, cnf.C, cnf.nnz, cnf.K)
        assert info.n_warnings == 0 and info.n_duplicates == 0


def test_solver_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2511_07737_b200 import Solver
    with pytest.raises(RuntimeError):
        Solver(0)
