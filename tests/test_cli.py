"""Command-line front end (tools/slablu_gpu_main.cpp), following the
reference's CLI tests (proj/tests/test_cli.cpp): config validation and exit codes (host only),
--dump-config as a fixed point, report schema of solve / bench, verify."""
import csv
import io
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2211_07572_b200", "slablu_gpu")
HEADER = ("N,n1,n2,b,kappa,T_factor_stage1_s,T_factor_stage2_s,T_solve_s,M_factor_scalars,relerr_res,"
          "relerr_true,hbs_max_rank,seed")


def cli():
    if not os.path.exists(CLI):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2211_07572_b200", "csrc")], check=True)
    return CLI


def run(args, cfg=None, tmp=None):
    if cfg is not None:
        path = os.path.join(tmp, "cfg.json")
        with open(path, "w") as fh:
            fh.write(cfg if isinstance(cfg, str) else json.dumps(cfg))
        args = args + ["--config", path]
    return subprocess.run([cli()] + args, capture_output=True, text=True, timeout=600)


@pytest.mark.parametrize("cfg,msg", [
    ({"problem": "poisson", "n1": 32, "n2": 32, "bogus": 1}, "unknown config key"),
    ({"problem": "poisson", "n1": 32, "n2": 32, "b": 4, "c": 0.5}, "exactly one of 'b' and 'c'"),
    ({"problem": "helmholtz_const", "n1": 32, "n2": 32}, "exactly one of 'kappa' and 'ppw'"),
    ({"problem": "poisson", "n1": 32, "n2": 32, "ppw": 10}, "apply only to Helmholtz"),
    ({"problem": "poisson", "n1": 16, "n2": 32}, "n1 >= n2 >= 2"),
    ({"problem": "poisson", "n2": 32}, "needs 'n1' and 'n2'"),
    ({"problem": "laplace", "n1": 8, "n2": 8}, "must be one of"),
    ("{not json", "not valid JSON"),
])
def test_config_errors_exit_1(tmp_path, cfg, msg):  # test_cli.cpp config validation, exit code 1
    r = run(["solve"], cfg, str(tmp_path))
    assert r.returncode == 1, r.stderr
    assert msg in r.stderr


def test_bench_config_errors(tmp_path):
    r = run(["bench"], {"problem": "poisson", "n1": 8, "n2": 8}, str(tmp_path))
    assert r.returncode == 1 and "sweep_n2" in r.stderr
    r = run(["bench"], {"problem": "poisson", "sweep_n2": [16], "aspect": 0.5}, str(tmp_path))
    assert r.returncode == 1 and "aspect" in r.stderr


def test_usage_errors():
    assert subprocess.run([cli()], capture_output=True).returncode == 1
    assert subprocess.run([cli(), "frobnicate"], capture_output=True).returncode == 1
    assert subprocess.run([cli(), "verify", "--quick", "--full"], capture_output=True).returncode == 1


def test_dump_config_fixed_point(tmp_path):  # test_cli.cpp:274-312 (written before the run)
    d1, d2 = tmp_path / "d1.json", tmp_path / "d2.json"
    cfg = {"problem": "helmholtz_varcoef", "n1": 24, "n2": 16, "ppw": 12, "seed": 3}
    run(["solve", "--dump-config", str(d1)], cfg, str(tmp_path))
    resolved = json.loads(d1.read_text())
    assert resolved["c"] == 0.6 and resolved["compression"] == "auto" and resolved["seed"] == 3
    run(["solve", "--dump-config", str(d2)], d1.read_text(), str(tmp_path))
    assert json.loads(d2.read_text()) == resolved


@pytest.mark.gpu
def test_solve_csv_and_json(tmp_path):
    r = run(["solve"], {"problem": "poisson", "n1": 32, "n2": 32, "b": 4}, str(tmp_path))
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[0] == HEADER
    row = next(csv.DictReader(io.StringIO(r.stdout)))
    assert int(row["N"]) == 1024 and int(row["b"]) == 4
    assert abs(float(row["relerr_true"]) / 4.961321e-04 - 1) < 1e-4   # test_driver.cpp:247-252
    out = tmp_path / "o.json"
    r = run(["solve", "--format", "json", "--output", str(out), "--seed", "7"],
            {"problem": "helmholtz_const", "n1": 40, "n2": 32, "kappa": 9.0}, str(tmp_path))
    assert r.returncode == 0, r.stderr
    j = json.loads(out.read_text())
    assert set(j) == set(HEADER.split(",")) and j["seed"] == 7 and j["relerr_res"] < 1e-10


@pytest.mark.gpu
def test_bench_rows_and_failed_row(tmp_path):
    r = run(["bench"], {"problem": "poisson", "sweep_n2": [16, 32], "b": 4}, str(tmp_path))
    assert r.returncode == 0, r.stderr
    rows = list(csv.DictReader(io.StringIO(r.stdout)))
    assert [int(x["n2"]) for x in rows] == [16, 32] and all(x["status"] == "ok" for x in rows)
    # a row that fails keeps its place with the error in the status column (driver.hpp:305-319)
    r = run(["bench", "--format", "json"], {"problem": "helmholtz_const", "sweep_n2": [16, 4200], "kappa": 5.0,
                                            "b": 4}, str(tmp_path))
    assert r.returncode == 0, r.stderr
    js = [json.loads(x) for x in r.stdout.strip().splitlines()]
    assert js[0]["status"] == "ok" and js[1]["status"].startswith("error")


@pytest.mark.gpu
def test_verify_passes():
    r = subprocess.run([cli(), "verify"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "verification: 4/4 checks passed" in r.stdout
