"""Bench-harness compatibility (reference bench.hpp / bench.cpp): CSV schema,
round trip, tpi / speedup errors. CPU-only except the suite run."""
import math

import pytest

import paper_1803_04378_b200.harness as H


def test_csv_header_matches_reference_schema():
    # bench.hpp:40-43, verbatim
    assert H.CSV_HEADER == ("instance,status,objective,iterations_p1,iterations_p2,total_seconds,"
                            "tpi_seconds,case,device_reads,device_writes,h2d_bytes,d2h_bytes,"
                            "reference_seconds,speedup")


def test_csv_round_trip():
    rows = [H.BenchRow("gen_8000x16000", "Optimal", 633.766187425, 9510, 12093, 1.99, 9.2e-5,
                       "InCore", 10, 20, 30, 40, 168.5, 84.67),
            H.BenchRow("bad.mps", "ParseError")]
    text = H.write_csv(rows)
    back = H.read_csv(text)
    assert H.write_csv(back) == text
    assert back[0].objective == float("%.6g" % 633.766187425)
    assert back[1].reference_seconds is None and back[1].speedup is None


def test_tpi_and_speedup_rules():
    assert H.tpi(2.0, 4) == 0.5
    with pytest.raises(H.ZeroIterations):
        H.tpi(1.0, 0)
    assert H.speedup(10.0, 2.0) == 5.0
    with pytest.raises(H.NonPositiveTime, match=r"^speedup: t_par must be positive, got 0\.000000$"):
        H.speedup(1.0, 0.0)  # std::to_string formatting (bench.cpp:16-17)
    assert H.status_name(H.SolveStatus.optimal) == "Optimal"
    assert H.status_name(H.SolveStatus.iteration_limit) == "IterationLimit"


def test_read_csv_rejects_bad_header():
    with pytest.raises(H.Error):
        H.read_csv("a,b\n")


@pytest.mark.gpu
def test_run_suite_rows():
    import paper_1803_04378_b200 as P
    rows = H.run_suite([("c1", P.GenSpec(256, 512, seed=1, form=P.Form.le_max)),
                        ("tiny", P.GenSpec(20, 40, seed=1))], runs=2,
                       reference=lambda lp: 1.0)
    assert [r.status for r in rows] == ["Optimal", "Optimal"]
    assert rows[0].iterations_p2 == 824 and rows[0].case_used == "InCore"
    assert rows[0].speedup == pytest.approx(1.0 / rows[0].total_seconds)
    assert math.isclose(rows[0].tpi_seconds, rows[0].total_seconds / 824)
    assert H.read_csv(H.write_csv(rows))[0].iterations_p2 == 824


@pytest.mark.gpu
def test_run_suite_mps_and_parse_error(tmp_path):
    """MPS instances go through load_mps and report the recovered objective
    (bench.cpp:191-195); an unreadable instance is a ParseError row with a NaN
    objective (bench.cpp:160-168)."""
    import os
    import numpy as np
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "mps")
    z = np.load(os.path.join(here, "production.npz"))
    bad = tmp_path / "bad.mps"
    bad.write_text("NAME X\nFOO\n")
    rows = H.run_suite([("prod", os.path.join(here, "production.mps")), ("bad", str(bad))])
    assert rows[0].status == "Optimal"
    assert rows[0].objective == float(z["objective_recovered"])
    assert rows[1].status == "ParseError" and math.isnan(rows[1].objective)
