"""The reference CLI's generate/run subcommands on the device path
(_lib/rkmf_b200_bench, csrc/cli.cpp + csrc/sweep.cpp), after
proj/tests/test_cli.cpp and acceptance.cpp:545-582 (c14: byte-identical CSV
across reruns with timing off)."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2503_22631_b200", "_lib", "rkmf_b200_bench")
HEADER = ("method,n,m_or_totalm,cycle,matvecs,rel_error,update_norm,kappa_W,leftmost_ritz_re,"
          "elapsed_ms,note")


def _cli(*args, cwd=None):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600, cwd=cwd)


def _cfg(tmp_path, name, obj):
    p = tmp_path / name
    p.write_text(json.dumps(obj))
    return str(p)


def test_generate_writes_the_baseline_problem(rk, tmp_path):
    cfg = _cfg(tmp_path, "gen.json", {"problem": {"kind": "baseline", "config": "cfg4", "N": 9},
                                      "output": str(tmp_path / "p")})
    r = _cli("generate", "--config", cfg)
    assert r.returncode == 0, r.stderr
    from paper_2503_22631_b200 import configs
    P = configs.build("cfg4", 9)
    rp, ci, v, n, nc = rk.load_matrix_market(str(tmp_path / "p.mtx"))
    assert np.array_equal(rp, P.row_ptr) and np.array_equal(ci, P.col_idx)
    assert np.array_equal(v, P.values)
    assert np.array_equal(rk.load_vector(str(tmp_path / "p.b.txt")), P.b)


@pytest.mark.parametrize("obj,msg", [
    ({}, "missing 'problem'"),
    ({"problem": {"kind": "membrane"}}, "unknown problem kind"),
    ({"problem": {"kind": "baseline", "config": "cfg9"}}, "unknown baseline config"),
    ({"problem": {"kind": "baseline", "config": "cfg1", "N": 8,
                  "function": {"kind": "phi1_neg"}}}, "not on the device path"),
    ({"problem": {"kind": "external", "matrix": "/nonexistent.mtx", "rhs": "x",
                  "function": {"kind": "exp_neg", "t": 1.0}}}, "cannot open"),
])
def test_configuration_errors_exit_1(tmp_path, obj, msg):
    r = _cli("run", "--config", _cfg(tmp_path, "bad.json", obj))
    assert r.returncode == 1 and msg in r.stderr, r.stderr


def test_usage_errors_exit_1(tmp_path):
    assert _cli().returncode == 1
    assert _cli("run").returncode == 1
    assert _cli("spectrum", "--config", "x").returncode == 1
    r = _cli("run", "--config", "/nonexistent.json")
    assert r.returncode == 1 and "cannot open config" in r.stderr


@pytest.mark.gpu
def test_run_sweep_csv_is_deterministic(tmp_path):
    methods = [{"name": "restart-rand", "m_r": 30, "d": 120, "zeta": 8, "tol": 1e-10,
                "k_max": 6, "seed": 1},
               {"name": "restart", "m_r": 30, "tol": 1e-10, "k_max": 6},
               {"name": "rand", "m": 40},
               {"name": "sfom", "m": 40},
               {"name": "restart-rand", "m_r": 30, "d": 10, "k_max": 2}]
    cfg = {"problem": {"kind": "baseline", "config": "cfg1", "N": 64},
           "methods": methods, "reference": {"mode": "restart-highm"}}
    c = _cfg(tmp_path, "run.json", cfg)
    a, b = str(tmp_path / "a.csv"), str(tmp_path / "b.csv")
    r1 = _cli("run", "--config", c, "--output", a)
    r2 = _cli("run", "--config", c, "--output", b)
    assert r1.returncode == 0 and r2.returncode == 0, r1.stderr + r2.stderr
    ta, tb = open(a).read(), open(b).read()
    assert ta == tb  # byte-identical (acceptance c14)
    lines = ta.splitlines()
    assert lines[0] == HEADER
    rows = [ln.split(",") for ln in lines[1:]]
    rr = [r for r in rows if r[0] == "restart-rand" and r[3] != "0"]
    rc = [r for r in rows if r[0] == "restart"]
    assert len(rr) >= 1 and len(rc) >= 1
    # per-cycle rows: total_m grows by m_r, rel_error against the high-m reference
    assert [int(r[2]) for r in rr] == [30 * (i + 1) for i in range(len(rr))]
    assert float(rr[-1][5]) <= 1e-8 and float(rc[-1][5]) <= 1e-8
    # kappa_W and the leftmost Ritz value are filled (restart.cpp:101,103)
    assert all(float(r[7]) >= 1.0 for r in rr)
    # "rand" = the first cycle of restart-rand with d = 4 m: one row, cycle 0
    shot = [r for r in rows if r[0] == "rand"]
    assert len(shot) == 1 and shot[0][2] == "40" and shot[0][3] == "0" and shot[0][4] == "40"
    assert shot[0][10] == "" and float(shot[0][5]) < 1.0 and float(shot[0][7]) >= 1.0
    # the unsupported one-shot method and the failing cell: one NaN row each with a note
    one = [r for r in rows if r[0] == "sfom"]
    assert len(one) == 1 and one[0][5] == "nan" and "one-shot" in one[0][10]
    bad = [r for r in rows if r[0] == "restart-rand" and r[3] == "0"]
    assert len(bad) == 1 and bad[0][10] != ""


@pytest.mark.gpu
def test_run_external_problem_and_timing(rk, tmp_path):
    from paper_2503_22631_b200 import configs
    P = configs.build("cfg2", 12)
    rk.save_matrix_market((P.row_ptr, P.col_idx, P.values), str(tmp_path / "m.mtx"))
    rk.save_vector(P.b, str(tmp_path / "b.txt"))
    cfg = {"problem": {"kind": "external", "matrix": str(tmp_path / "m.mtx"),
                       "rhs": str(tmp_path / "b.txt"),
                       "function": {"kind": "exp_neg", "t": P.t}},
           "methods": [{"name": "restart-rand", "m_r": 20, "d": 80, "zeta": 8, "tol": P.tol,
                        "k_max": 20, "seed": 1}],
           "timing": True}
    r = _cli("run", "--config", _cfg(tmp_path, "ext.json", cfg))
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert lines[0] == HEADER and len(lines) >= 2
    assert "timing restart-rand: basis build" in r.stderr
    assert float(lines[-1].split(",")[9]) > 0.0  # elapsed_ms with timing on
