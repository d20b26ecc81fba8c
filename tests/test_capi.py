"""CPU tests of the C-ABI boundary: the library loads, exports exactly what include/ddelm_gpu.h
declares, and fails loudly (no CPU fallback) when there is no CUDA device."""
import ctypes as C
import os
import re

import pytest

import paper_2503_10032_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ddelm_gpu.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ddelm_gpu_\w+)\s*\(", text)))


def test_header_matches_python_exports():
    assert header_symbols() == sorted(P.EXPORTS)


def test_library_exports_every_header_symbol():
    L = P.load_library()
    for name in header_symbols():
        assert hasattr(L, name), name
    assert b"sm_100a" in L.ddelm_gpu_version()


def test_struct_layouts_match_header(tmp_path):
    """Compile a C probe against the header: the ctypes mirrors must have the same layout."""
    import subprocess
    src = tmp_path / "probe.c"
    src.write_text('''#include <stdio.h>
#include <stddef.h>
#include "ddelm_gpu.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu\\n", sizeof(ddelm_desc), sizeof(ddelm_report),
         offsetof(ddelm_desc, seed), offsetof(ddelm_desc, rank_tol), offsetof(ddelm_report, total_seconds));
  return 0;
}
''')
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    vals = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert vals == [C.sizeof(P._Desc), C.sizeof(P._Report), P._Desc.seed.offset,
                    P._Desc.rank_tol.offset, P._Report.total_seconds.offset]


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device error path")
def test_no_device_fails_loudly():
    with pytest.raises(RuntimeError, match="no CUDA device|CUDA"):
        P.Workspace("poisson_sinpi", 2, 10, 64, 8.0, 1)


def test_invalid_arguments_mirror_reference():
    with pytest.raises(ValueError):
        P.make_problem("no_such_problem")
    with pytest.raises(ValueError):
        P.ddelm_nn_solve(None, 1.5)
    with pytest.raises(ValueError):
        P.SolverOptions(flux_variant="bogus") and P.Workspace("poisson_sinpi", 2, 10, 64, 8.0, 1,
                                                              P.SolverOptions(flux_variant="bogus"))


FACADE_BIN = os.path.join(ROOT, "paper_2503_10032_b200", "ddelm_solve")


def test_cpp_facade_builds_and_links():
    """examples/ddelm_solve.cpp uses only include/ddelm_b200/solvers.hpp (the reference-shaped
    C++ API) over the C-ABI; it is built by the package Makefile."""
    import subprocess
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2503_10032_b200", "csrc")], check=True)
    assert os.access(FACADE_BIN, os.X_OK)


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device error path")
def test_cpp_facade_fails_loudly_without_device():
    import subprocess
    out = subprocess.run([FACADE_BIN], capture_output=True, text=True)
    assert out.returncode == 2 and "no CUDA device" in out.stderr
    bad = subprocess.run([FACADE_BIN, "bogus=1"], capture_output=True, text=True)
    assert bad.returncode == 3
    bad = subprocess.run([FACADE_BIN, "cg_blocks=dense"], capture_output=True, text=True)
    assert bad.returncode == 3 and "cg_blocks" in bad.stderr


def test_problem_catalogue_matches_header():
    """make_problem's names (problems.cpp:132-188 + C4's addition) map onto the C enumerants."""
    import re
    import paper_2503_10032_b200 as P
    h = open(os.path.join(ROOT, "include", "ddelm_gpu.h")).read()
    enums = {m.group(1).lower(): int(m.group(2)) for m in re.finditer(r"DDELM_([A-Z0-9_]+) = (\d+)", h)
             if not m.group(1).startswith(("METHOD", "FLUX", "OK", "ERR"))}
    assert enums == P.PROBLEMS
    with pytest.raises(ValueError):
        P.make_problem("heat_equation")
    with pytest.raises(ValueError):
        P.make_problem("poisson_grf", P.ProblemParams(alpha=-1.0))
    assert P.make_problem("varcoef_poisson").params.rho_seed == 3  # problems.hpp:64-68 defaults


def test_every_config_has_a_golden():
    """Every named workload is pinned by an oracle fixture (tools/make_goldens.py)."""
    import paper_2503_10032_b200 as P
    missing = [n for n in P.CONFIGS if not os.path.exists(os.path.join(ROOT, "tests", "golden", f"{n}.npz"))]
    assert not missing, missing
