"""CPU test: the C++ shim (include/lpsg.hpp) compiles beside the reference's
own headers and links against liblpsg.so (no compute: no GPU here)."""
import os
import shutil
import subprocess

import pytest

from conftest import ROOT

SRC = r'''
#include <vector>
#include "lpsg.hpp"
struct LP { int m, n_total; std::vector<double> A, b, c; std::vector<int> col_kind; };
int main() {
    LP lp{1, 2, {1.0, 1.0}, {1.0}, {-1.0, 0.0}, {0, 1}};
    try { lpsg::two_phase_solve(lp); } catch (const lpsg::CudaError&) { return 0; }
    catch (...) { return 3; }
    return lpsg_device_count() > 0 ? 0 : 4;
}
'''


@pytest.mark.skipif(shutil.which("g++") is None, reason="no g++")
def test_cxx_shim_compiles_and_links(tmp_path):
    from paper_1803_04378_b200 import _lib
    _lib.load()
    src = tmp_path / "shim.cpp"
    src.write_text(SRC)
    exe = tmp_path / "shim"
    libdir = os.path.dirname(_lib.LIB_PATH)
    r = subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"), str(src), "-o",
                        str(exe), "-L", libdir, "-llpsg", f"-Wl,-rpath,{libdir}"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
