"""The command-line drop-in (paper_1703_06155_b200/h2lu_gpu) against the
reference CLI's own smoke test (proj/tests/cli_smoke.sh): build -> factor ->
rhs -> solve -> bench, exit codes 0 / 2 / 3; the files it writes are read back
by the CPU oracle's H2LU v1 reader and its solution checked against the
oracle's."""
import json
import os
import subprocess

import numpy as np
import pytest

import pyoracle as O
from helpers import rel

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_1703_06155_b200", "h2lu_gpu")


def run(*args, cwd=None):
    return subprocess.run([BIN, *args], capture_output=True, text=True, cwd=cwd, timeout=600)


def test_help_rhs_and_input_errors(tmp_path):
    assert run("--help").returncode == 0
    r = run("rhs", "--n", "600", "--seed", "7", "--out", "b.vec", "--json", cwd=tmp_path)
    assert r.returncode == 0 and json.loads(r.stdout)["n"] == 600
    r2 = run("rhs", "--n", "600", "--seed", "3", "--out", "b2.vec", cwd=tmp_path)
    assert r2.returncode == 0
    assert open(tmp_path / "b.vec", "rb").read() != open(tmp_path / "b2.vec", "rb").read()
    # the seeded vector is the reference CLI's (mt19937_64 + normal_distribution, h2lu_cli.cpp:181-191)
    assert np.array_equal(O.load_vector(tmp_path / "b.vec"), O.rhs(600, 7))
    assert run("build", "--geometry", "torus", "--n", "100", "--out", "t.h2", cwd=tmp_path).returncode == 2
    assert run("build", "--no-such-flag", cwd=tmp_path).returncode == 2
    assert run("factor", "--in", "x").returncode == 2  # --out missing
    assert run("bogus").returncode == 2


@pytest.mark.gpu
def test_cli_smoke_and_oracle_parity(tmp_path):
    w = str(tmp_path)
    assert run("build", "--geometry", "rod", "--n", "600", "--eps-h2", "1e-6", "--shift", "2", "--out", "m.h2", cwd=w).returncode == 0
    assert os.path.getsize(tmp_path / "m.h2") > 0
    r = run("factor", "--in", "m.h2", "--eps-fill-in", "1e-8", "--out", "m.chain", "--json", cwd=w)
    assert r.returncode == 0, r.stderr
    fj = json.loads(r.stdout)
    assert fj["n"] == 600 and len(fj["levels"]) >= 1
    assert run("rhs", "--n", "600", "--seed", "7", "--out", "b.vec", cwd=w).returncode == 0
    r = run("solve", "--chain", "m.chain", "--rhs", "b.vec", "--matrix", "m.h2", "--out", "x.vec", "--json", cwd=w)
    assert r.returncode == 0, r.stderr
    sj = json.loads(r.stdout)
    assert sj["n"] == 600 and sj["residual"] < 1e-6
    assert run("solve", "--chain", "m.chain", "--rhs", "b.vec", "--out", "x2.vec", cwd=w).returncode == 0
    assert open(tmp_path / "x.vec", "rb").read() == open(tmp_path / "x2.vec", "rb").read()  # deterministic
    # the oracle reads the CLI's files: same matrix, same chain -> same solution
    A = O.load_h2(tmp_path / "m.h2")
    ch = O.load_chain(tmp_path / "m.chain")
    och = A.factorize(1e-8)
    b = O.load_vector(tmp_path / "b.vec")
    x = O.load_vector(tmp_path / "x.vec")
    t = O.Tree(np.stack([np.arange(600.0), np.zeros(600), np.zeros(600)], axis=1), 25)
    perm = t.perm
    xt = och.solve(b[perm])
    xo = np.zeros_like(xt)
    xo[perm] = xt
    assert rel(x, xo) < 1e-9
    xl = ch.solve(b[perm])
    assert rel(xl[np.argsort(perm)], x) < 1e-12
    r = run("bench", "--geometry", "rod", "--sizes", "200,400", "--eps-h2", "1e-4", "--eps-fill-in", "1e-4", "--shift", "2", "--csv", "bench.csv",
            "--json", cwd=w)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert len(lines) == 2 and len(open(tmp_path / "bench.csv").read().strip().splitlines()) == 3
    for ln in lines:
        rec = json.loads(ln)
        assert rec["geometry"] == "rod" and rec["residual"] < 1e-2
    assert run("solve", "--chain", "missing.chain", "--rhs", "b.vec", "--out", "y.vec", cwd=w).returncode == 2
    open(tmp_path / "bad.h2", "w").write("garbage\n")
    assert run("factor", "--in", "bad.h2", "--eps-fill-in", "1e-8", "--out", "z.chain", cwd=w).returncode == 2
