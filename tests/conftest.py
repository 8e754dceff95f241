"""Shared fixtures. `-m "not gpu"` runs everywhere; `-m gpu` needs a B200."""
import glob
import os
import sys

# P2P shards that share one GPU (tests/test_gpu_sharded.py) need one hardware
# work queue per shard stream; the CUDA runtime reads this when the context is
# created, so it is set before anything touches CUDA (the library itself never
# sets it: include/lpsg.h lpsg_solve_sharded).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import numpy as np  # noqa: E402
import pytest  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def golden_names():
    return sorted(os.path.splitext(os.path.basename(p))[0]
                  for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz")))


class Golden:
    """One reference run: the LP, the reference's report and per-pivot trace."""

    def __init__(self, name):
        self.name = name
        z = np.load(os.path.join(GOLDEN_DIR, name + ".npz"), allow_pickle=False)
        self.z = z
        self.m, self.n_total = int(z["m"]), int(z["n_total"])
        self.status = int(z["status"])
        self.objective = float(z["objective"])
        self.x = z["x"]
        self.p1, self.p2 = int(z["iterations_phase1"]), int(z["iterations_phase2"])
        self.trace = z["trace"]
        self.trace_len = int(z["trace_len"])
        self.digest = str(z["digest"])
        self.max_iter = int(z["cfg_max_iter"])
        self.anticycle = int(z["cfg_anticycle"])
        self.pivot_tol = float(z["cfg_pivot_tol"])
        self.kernel = int(z["cfg_kernel"]) if "cfg_kernel" in z.files else 0  # 1: KernelMode::naive
        self.spec = tuple(int(v) for v in z["spec"]) if "spec" in z.files else None

    def arrays(self, generate=None):
        """(A, b, c, col_kind). Generated fixtures are re-drawn with `generate`
        (rows, cols, seed, form) -> object with A, b, c, col_kind."""
        z = self.z
        if self.spec is not None:
            rows, cols, form, seed, _ = self.spec
            lp = generate(rows, cols, seed, form)
            return lp.A, lp.b, lp.c, lp.col_kind
        A = np.zeros((self.m, self.n_total))
        A[z["A_rows"], z["A_cols"]] = z["A_vals"]
        return A, z["b"], z["c"], z["col_kind"]

    def config_kwargs(self):
        return dict(max_iter=self.max_iter, anticycle="none" if self.anticycle else "tabu",
                    pivot_tol=self.pivot_tol, kernel="naive" if self.kernel else "cached")


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Port, build
    if not os.path.exists(os.path.join(ROOT, "oracle", "_build", "liblps_port.so")):
        build(ref=False)
    return Port()


def gpu_available():
    try:
        import paper_1803_04378_b200 as p
        return p.device_count() > 0
    except Exception:
        return False
