"""CPU tests of the C-ABI boundary (include/lpsg.h) without compute calls.

* liblpsg.so loads and exports every function include/lpsg.h declares.
* Argument validation and error codes behave as documented.
* On a machine without a GPU the solver fails loudly (LPSG_CUDA_ERROR): there
  is no CPU fallback anywhere in the product.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT, gpu_available


def _declared():
    text = open(os.path.join(ROOT, "include", "lpsg.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lpsg_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("lpsg_create", "lpsg_solve", "lpsg_get_x", "lpsg_destroy",
                 "lpsg_two_phase_solve", "lpsg_set_observer", "lpsg_last_error",
                 "lpsg_price", "lpsg_compute_direction", "lpsg_ratio_test",
                 "lpsg_select_leaving", "lpsg_pivot_update", "lpsg_generate"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1803_04378_b200 import _lib
    lib = _lib.load()
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding covers every declared symbol
    bound = {s[0] for s in _lib.SIGNATURES}
    assert set(_declared()) <= bound


def test_library_is_sm100a_only():
    """The fatbin carries sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess
    from paper_1803_04378_b200 import _lib
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_config_defaults_match_reference():
    """SolverConfig defaults (solver.hpp:35-45)."""
    from paper_1803_04378_b200 import _lib
    lib = _lib.load()
    c = _lib.Config()
    lib.lpsg_config_default(C.byref(c))
    assert (c.opt_tol, c.pivot_tol, c.feas_tol, c.ratio_tie_tol) == (1e-7, 1e-9, 1e-7, 1e-9)
    assert c.max_iter == 0 and c.anticycle == 0


def test_config_struct_layout_and_public_fields():
    """The ctypes mirror of lpsg_config matches the C struct (every field at
    the C offset: a mismatch would shift memory_budget / reinvert_every), and
    the public Python config carries the reference's fields plus the opt-in
    modes, not the perf-experiment knobs (those live only in the
    -DLPSG_EXPERIMENTS build)."""
    import dataclasses
    import os
    import subprocess
    import tempfile
    from paper_1803_04378_b200 import SolverConfig, _lib
    names = {f.name for f in dataclasses.fields(SolverConfig)}
    for must in ("opt_tol", "pivot_tol", "feas_tol", "ratio_tie_tol", "max_iter", "anticycle",
                 "kernel", "workers", "observer", "observer_rows", "memory_budget", "reinvert_every"):
        assert must in names
    for gone in ("experiment", "debug_flags", "use_graphs"):
        assert gone not in names
    src = ('#include <stddef.h>\n#include <stdio.h>\n#include "lpsg.h"\n'
           'int main(void){printf("%zu %zu %zu %zu\\n", sizeof(lpsg_config), '
           'offsetof(lpsg_config, peer), offsetof(lpsg_config, reinvert_every), '
           'offsetof(lpsg_config, memory_budget)); return 0;}\n')
    with tempfile.TemporaryDirectory() as d:
        with open(os.path.join(d, "t.c"), "w") as f:
            f.write(src)
        exe = os.path.join(d, "t")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), os.path.join(d, "t.c"), "-o", exe],
                       check=True)
        got = [int(v) for v in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    C_ = _lib.Config
    assert got == [C.sizeof(C_), C_.peer.offset, C_.reinvert_every.offset, C_.memory_budget.offset]


def test_null_arguments_are_rejected():
    from paper_1803_04378_b200 import _lib
    lib = _lib.load()
    assert lib.lpsg_create(None, None, None) == 4  # LPSG_INVALID_ARGUMENT
    assert b"null" in lib.lpsg_last_error()
    assert lib.lpsg_solve(None, None) == 4


def test_empty_problem_is_an_error():
    import paper_1803_04378_b200 as P
    lp = P.StandardFormLP(0, 0, np.zeros((0, 0)), np.zeros(0), np.zeros(0), np.zeros(0, np.uint8))
    with pytest.raises((P.DegenerateSpec, P.CudaError)):
        P.two_phase_solve(lp)


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback_without_gpu():
    import paper_1803_04378_b200 as P
    lp = P.generate(P.GenSpec(8, 12, seed=1))
    with pytest.raises(P.CudaError, match="no CUDA device"):
        P.two_phase_solve(lp)
    assert P.device_count() == 0
