"""Wire formats and run artifacts (controls.cpp:20-45,183-288; tools/main.cpp:94-200): byte
layouts checked against hand-packed bytes, round trips, and the error behaviour."""
import json
import struct

import numpy as np
import pytest

from paper_1603_01237_b200 import ism as I
from paper_1603_01237_b200 import wire as W


def test_control_binary_layout_and_round_trip():
    g = I.TimeGrid(0.25, 0.125, 3)
    u = np.array([[1.0, 2.0, 3.0], [-1.0, 0.5, 7.0]])
    b = W.write_control_binary(u, g)
    # u32 C, u64 steps, f64 t0, f64 dt, channel-major samples (controls.cpp:229-236)
    assert b[:28] == struct.pack("<IQdd", 2, 3, 0.25, 0.125)
    assert struct.unpack("<6d", b[28:]) == (1.0, 2.0, 3.0, -1.0, 0.5, 7.0)
    u2, g2 = W.read_control_binary(b)
    assert np.array_equal(u2, u) and g2 == g
    with pytest.raises(RuntimeError):
        W.read_control_binary(b[:-1])


def test_matrix_and_vector_binary():
    m = np.array([[1 + 2j, 3 - 1j], [0.5j, -2.0]])
    b = W.write_matrix_binary(m)
    assert b[:16] == struct.pack("<QQ", 2, 2)
    # column-major (re, im) pairs (controls.cpp:248-256)
    assert struct.unpack("<8d", b[16:]) == (1.0, 2.0, 0.0, 0.5, 3.0, -1.0, -2.0, 0.0)
    assert np.array_equal(W.read_matrix_binary(b), m)
    v = np.array([1 - 1j, 2j])
    assert np.array_equal(W.read_vector_binary(W.write_vector_binary(v)), v)


def test_control_csv():
    g = I.TimeGrid(0.0, 0.5, 2)
    u = np.array([[0.1, 1.0 / 3.0]])
    text = W.write_control_csv(u, g)
    assert text.splitlines()[0] == "t,u_1"
    assert text.splitlines()[1] == "0.25,0.10000000000000001"
    assert np.array_equal(W.read_control_csv(text, g), u)
    with pytest.raises(RuntimeError):
        W.read_control_csv("x,u_1\n", g)


def test_run_artifacts(tmp_path):
    from tests import oracle_api as O
    p, u = O.dense_fixture(2400)
    run = O.ism_run(p, u, I.IsmConfig(subintervals=2, max_outer=3, eta=0.0), I.SolverSpec(step_size=0.4))[0]
    W.write_run_artifacts(tmp_path, p, run, {"preset": "fixture"})
    lines = (tmp_path / "iterations.jsonl").read_text().splitlines()
    assert len(lines) == 4 and json.loads(lines[0])["iteration"] == 0 and "error" not in json.loads(lines[0])
    assert "error" in json.loads(lines[1])
    s = json.loads((tmp_path / "summary.json").read_text())
    assert s["format_version"] == 1 and s["result"]["iterations"] == 3 and s["problem"]["steps"] == p.grid.steps
    assert np.allclose(W.read_control_csv((tmp_path / "control.csv").read_text(), p.grid), run.control,
                       rtol=0, atol=0)


def test_kat7_efficiency_formulas_and_csv():
    # acceptance_main.cpp:541-575 (criterion 10) and runtime_test.cpp:143-170, exact strings
    from paper_1603_01237_b200 import ism as I
    from paper_1603_01237_b200 import wire as W

    def record_with(objectives, times):
        r = I.RunRecord()
        r.iterations = [I.IterationStat(iteration=k, objective=o, device_seconds=t)
                        for k, (o, t) in enumerate(zip(objectives, times))]
        return r

    serial = record_with([0.0, 0.2, 0.5, 1.0], [249.25] * 4)
    eight = record_with([0.4, 1.0], [62.5, 62.5])
    stuck = record_with([0.1, 0.2], [10.0, 10.0])
    rows = W.efficiency_table([(1, serial), (8, eight), (16, stuck)], 1.0, 0.25)
    assert len(rows) == 3
    assert rows[0].reached and rows[0].t_seconds == 997.0 and rows[0].speedup == 1.0
    assert rows[0].efficiency_percent == 100.0
    assert rows[1].reached and rows[1].t_seconds == 125.0 and rows[1].speedup == 997.0 / 125.0
    assert rows[1].efficiency_percent == 100.0 * (997.0 / 125.0) / 8.0
    assert not rows[2].reached
    assert W.format_percent(rows[1].efficiency_percent) == "99.7%"
    assert W.format_percent(rows[0].efficiency_percent) == "100.0%"
    assert W.efficiency_csv(rows) == ("N,t_seconds,speedup,efficiency\n"
                                      "1,997.000000,1.000000,100.0%\n"
                                      "8,125.000000,7.976000,99.7%\n"
                                      "16,,,unreached\n")
    a = W.EfficiencyRow(1, 8.0, 1.0, 100.0, True)
    b = W.EfficiencyRow(2, 2.5, 3.2, 160.0, True)
    c = W.EfficiencyRow(4)
    assert W.efficiency_csv([a, b, c]) == ("N,t_seconds,speedup,efficiency\n"
                                           "1,8.000000,1.000000,100.0%\n"
                                           "2,2.500000,3.200000,160.0%\n"
                                           "4,,,unreached\n")
    assert W.format_percent(12.34) == "12.3%" and W.format_percent(99.96) == "100.0%"
    assert W.format_percent(0.0) == "0.0%"
    try:
        W.efficiency_table([(2, eight)], 1.0, 0.25)
    except ValueError:
        pass
    else:
        raise AssertionError("an N=1 run is required")
