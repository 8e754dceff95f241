"""GPU test of the C++ drop-in: one binary (oracle/_ref/dropin_check, built by
oracle/Makefile from oracle/dropin_check.cpp) links the unmodified reference
and lpsg through include/lpsg.hpp, solves the same lps::StandardFormLP with
both and compares them pivot for pivot and bit for bit."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
EXE = os.path.join(ROOT, "oracle", "_ref", "dropin_check")


@pytest.mark.skipif(not os.path.exists(EXE), reason="dropin_check not built (needs the reference)")
@pytest.mark.parametrize("args", [("64", "128", "0", "2"), ("256", "512", "1", "1"),
                                  ("128", "256", "2", "5"), ("300", "500", "0", "9")])
def test_cxx_dropin_matches_reference(args):
    r = subprocess.run([EXE, *args], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.startswith("PASS"), r.stdout + r.stderr
