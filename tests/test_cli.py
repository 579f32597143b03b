"""The GPU command line (paper_1802_03433_b200/cli.py), mirroring the
reference's CLI tests (tests/test_cli.cpp): output lines, files, exit codes
(usage 2, runtime 1) and the bench CSV column contract. Usage errors and
codegen run on CPU; assemble / solve / bench need the GPU."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_cli(args, cwd):
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run([sys.executable, "-m", "paper_1802_03433_b200.cli"] + args, cwd=cwd, env=env,
                       capture_output=True, text=True, timeout=600)
    return r.returncode, r.stdout, r.stderr


@pytest.mark.parametrize("args,needle", [
    (["assemble", "--f", "sin(x"], "parse error"),            # test_cli.cpp:55-58
    (["assemble", "--f", "x+t"], "'t'"),                      # :59-63
    (["assemble", "--no-such-option"], "unrecognized"),
    # out of the hot-path scope: a usage error, not a silent fallback
    (["assemble", "--layout", "dense"], "invalid choice"),
    (["mesh", "3"], "invalid choice"),
])
def test_usage_errors_exit_2(tmp_path, args, needle):
    code, _, err = run_cli(args, tmp_path)
    assert code == 2 and needle in err


def test_codegen_deterministic(tmp_path):
    """test_cli.cpp:93-110: two runs byte-identical, no unresolved
    placeholders, a listing entry for every bilinear (i, j) and linear i."""
    r1 = run_cli(["codegen", "--n", "4", "--out-source", "cg1.cu", "--out-ir", "cg1.ir"], tmp_path)
    r2 = run_cli(["codegen", "--n", "4", "--out-source", "cg2.cu", "--out-ir", "cg2.ir"], tmp_path)
    assert r1[0] == 0 and r2[0] == 0
    src = (tmp_path / "cg1.cu").read_text()
    assert src == (tmp_path / "cg2.cu").read_text() and "{{" not in src
    ir = (tmp_path / "cg1.ir").read_text()
    assert ir == (tmp_path / "cg2.ir").read_text()
    for i in range(3):
        for j in range(3):
            assert f"program bilinear_{i}_{j}\n" in ir
        assert f"program linear_{i}\n" in ir


@pytest.mark.gpu
def test_assemble_reports_and_exports(tmp_path):
    """test_cli.cpp:45-53, plus the exported system equals the reference
    library's (oracle/_ref) on the same mesh and form, <= 1e-12 normwise."""
    code, out, err = run_cli(["assemble", "--n", "4", "--out-matrix", "cli_A.mtx", "--out-vector", "cli_b.mtx"],
                             tmp_path)
    assert code == 0, err
    assert "N: 25" in out and "MAX_NZ: 7" in out and "wall_ms:" in out and "nnz: 137" in out
    A = (tmp_path / "cli_A.mtx").read_text()
    b = (tmp_path / "cli_b.mtx").read_text()
    assert A.startswith("%%MatrixMarket matrix coordinate real general\n25 25 137\n")
    assert b.startswith("%%MatrixMarket matrix array real general\n25 1\n")
    import pyoracle as po
    from conftest import normwise
    xy, conn = po.unit_square_mesh(4)
    rp, ci = po.build_pattern(conn, xy.shape[0])
    ov, ob = po.assemble("demo2d", 2, 1, 3, xy, conn, conn, rp, ci)
    vals = np.array([float(l.split()[2]) for l in A.splitlines()[2:]])
    bv = np.array([float(l) for l in b.splitlines()[2:]])
    assert normwise(vals, ov) <= 1e-12 and normwise(bv, ob) <= 1e-12


@pytest.mark.gpu
def test_solve_manufactured_cosine(tmp_path):
    """test_cli.cpp:75-91: converged, 0 < l2_error < 1e-2 at n=16."""
    pi = "3.14159265358979312"
    code, out, err = run_cli(["solve", "--sigma", "1,0,0,1", "--lambda", "1",
                              "--f", f"(2*{pi}^2+1)*cos({pi}*x)*cos({pi}*y)", "--n", "16",
                              "--exact", f"cos({pi}*x)*cos({pi}*y)", "--tol", "1e-10"], tmp_path)
    assert code == 0, err
    assert "converged: yes" in out
    err_l2 = float(out.split("l2_error:")[1].split()[0])
    assert 0.0 < err_l2 < 1e-2


@pytest.mark.gpu
def test_bench_csv_contract(tmp_path):
    """test_cli.cpp:121-139: header, 8 columns per row; one GPU row per size."""
    code, out, err = run_cli(["bench", "--sizes", "4,8", "--repeats", "1", "--csv", "cli_bench.csv"], tmp_path)
    assert code == 0, err
    lines = (tmp_path / "cli_bench.csv").read_text().splitlines()
    assert lines[0] == "n,nodes,elements,evaluator,mode,workers,median_ms,speedup_vs_interpreted"
    rows = [l for l in lines[1:] if l]
    assert len(rows) == 2 and all(l.count(",") == 7 for l in rows)
    assert rows[0].split(",")[:6] == ["4", "25", "32", "nvrtc", "gpu", "1"]
