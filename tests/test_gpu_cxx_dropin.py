"""GPU test of the C++ drop-in: one binary (oracle/_ref/dropin_check, built by
oracle/Makefile from oracle/dropin_check.cpp) links the unmodified reference
and lpsg through include/lpsg.hpp, solves the same lps::StandardFormLP with
both and compares them pivot for pivot and bit for bit: the whole basis at
every observer call, tableau rows through IterationView::row (`rows`), and
the step API driven by hand (`steps=N`: price, compute_direction,
ratio_test, select_leaving, pivot_update and the Figure-1 accessors); `parts=P`
runs both libraries under a memory budget of ~P row partitions (the
reference's own Case 2 against lpsg's, case_used compared too) and `naive`
both in KernelMode::naive."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
EXE = os.path.join(ROOT, "oracle", "_ref", "dropin_check")


@pytest.mark.skipif(not os.path.exists(EXE), reason="dropin_check not built (needs the reference)")
@pytest.mark.parametrize("args", [("64", "128", "0", "2", "steps=40"), ("256", "512", "1", "1"),
                                  ("128", "256", "2", "5", "steps=60"), ("300", "500", "0", "9"),
                                  ("40", "80", "0", "3", "rows"), ("48", "64", "2", "7", "rows"),
                                  ("96", "160", "1", "4", "rows", "steps=30"),
                                  # the reference's own Case 2 and naive kernel mode against lpsg's
                                  ("128", "256", "2", "5", "parts=3"), ("96", "160", "1", "4", "rows", "parts=4"),
                                  ("64", "128", "0", "2", "naive", "steps=20"),
                                  ("200", "300", "2", "9", "parts=2", "naive")])
def test_cxx_dropin_matches_reference(args):
    r = subprocess.run([EXE, *args], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.startswith("PASS"), r.stdout + r.stderr
