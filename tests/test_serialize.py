"""H2LU v1 container (proj/include/h2lu/serialize.hpp:27-353) on both sides:
the product's writer / reader (libh2g, device handles) against the oracle's
restatement, in both directions, plus the reference's corruption checks
(proj/tests/test_serialize.cpp: bad magic, wrong kind, truncation)."""
import os

import numpy as np
import pytest

import paper_1703_06155_b200 as h2g
import pyoracle as O
from helpers import rel, rod_problem, vie_problem


def test_vector_round_trip_both_ways(tmp_path):
    v = np.arange(7) - 0.5j * np.arange(7)
    h2g.save_vector(tmp_path / "a.bin", v)
    assert np.array_equal(O.load_vector(tmp_path / "a.bin"), v)
    O.save_vector(tmp_path / "b.bin", 3 * v)
    assert np.array_equal(h2g.load_vector(tmp_path / "b.bin"), 3 * v)
    raw = open(tmp_path / "a.bin", "rb").read()
    assert raw[:12] == b"H2LU\x01\x00\x00\x00\x03\x00\x00\x00" and len(raw) == 12 + 8 + 16 * 7


def test_vector_corruption_rejected(tmp_path):
    v = np.ones(4, np.complex128)
    h2g.save_vector(tmp_path / "v.bin", v)
    raw = open(tmp_path / "v.bin", "rb").read()
    open(tmp_path / "t.bin", "wb").write(raw[:-8])
    with pytest.raises(h2g.InvalidInputError, match="truncated"):
        h2g.load_vector(tmp_path / "t.bin")
    open(tmp_path / "m.bin", "wb").write(b"XXXX" + raw[4:])
    with pytest.raises(h2g.InvalidInputError, match="magic"):
        h2g.load_vector(tmp_path / "m.bin")
    A = rod_problem(64, 1e-6, leaf=16)
    O.save_h2(A, tmp_path / "h.bin")
    with pytest.raises(h2g.InvalidInputError, match="kind"):
        h2g.load_vector(tmp_path / "h.bin")
    with pytest.raises(h2g.InvalidInputError):
        h2g.load_vector(tmp_path / "missing.bin")


def test_oracle_container_round_trip_bitwise(tmp_path):
    A = rod_problem(256, 1e-10, leaf=32)
    ch = A.factorize(1e-12)
    O.save_h2(A, tmp_path / "a.h2")
    O.save_chain(ch, tmp_path / "a.chain")
    B = O.load_h2(tmp_path / "a.h2")
    ch2 = O.load_chain(tmp_path / "a.chain")
    b = O.rhs(256, 3)
    assert np.array_equal(B.matvec(b), A.matvec(b))
    assert np.array_equal(ch2.solve(b), ch.solve(b))
    assert ch2.hash() == ch.hash()


def with_tree(A, leaf):
    arr = A.arrays()
    arr["points_tree"] = A.tree.points
    arr["perm"] = A.tree.perm
    arr["leafsize"] = leaf
    return arr


@pytest.mark.gpu
def test_gpu_matrix_save_load_against_oracle(tmp_path):
    A, K = vie_problem(16, 0.5, 32, 1e-4)
    G = h2g.H2Matrix.upload(with_tree(A, 32))
    G.save(tmp_path / "g.h2")
    B = O.load_h2(tmp_path / "g.h2")  # the oracle reads the GPU's file
    x = O.rhs(A.n, 5)
    assert rel(B.matvec(x), A.matvec(x)) < 1e-14
    O.save_h2(A, tmp_path / "o.h2")  # the GPU reads the oracle's file
    G2 = h2g.H2Matrix.load(tmp_path / "o.h2")
    d1, d2 = G.download(), G2.download()
    for k in ("basis_data", "coupling_data", "dense_data", "adm_pairs", "split_pairs", "leaf_pairs", "cluster_begin", "cluster_end", "perm"):
        assert np.array_equal(d1[k], d2[k]), k
    assert h2g.factorize(G2, 1e-4).hash() == h2g.factorize(G, 1e-4).hash()


@pytest.mark.gpu
def test_gpu_chain_save_load_against_oracle(tmp_path):
    A = rod_problem(256, 1e-10, leaf=32)
    och = A.factorize(1e-12)
    G = h2g.H2Matrix.upload(with_tree(A, 32))
    gch = h2g.factorize(G, 1e-12)
    b = O.rhs(256, 11)
    xg = gch.solve(b)
    # GPU chain -> file -> oracle
    h2g.save_chain(gch, tmp_path / "g.chain")
    och2 = O.load_chain(tmp_path / "g.chain")
    assert rel(och2.solve(b), xg) < 1e-12
    ro = {(r["level"], r["cluster"]): r["rank_after"] for r in och.all_records()}
    rf = {(r["level"], r["cluster"]): r["rank_after"] for r in och2.all_records()}
    assert ro == rf
    # oracle chain -> file -> GPU (solved on the device)
    O.save_chain(och, tmp_path / "o.chain")
    lch = h2g.load_chain(tmp_path / "o.chain")
    assert lch.n == 256 and lch.root_size == och.root_size
    assert rel(lch.solve(b), och.solve(b)) < 1e-12
    # GPU round trip
    rch = h2g.load_chain(tmp_path / "g.chain")
    assert rel(rch.solve(b), xg) < 1e-12
    assert [l["rank_sum_after"] for l in rch.levels()] == [l["rank_sum_after"] for l in gch.levels()]


@pytest.mark.gpu
def test_gpu_chain_load_vie_multi_rhs(tmp_path):
    A, K = vie_problem(16, 0.5, 32, 1e-4)
    G = h2g.H2Matrix.upload(with_tree(A, 32))
    gch = h2g.factorize(G, 1e-4)
    h2g.save_chain(gch, tmp_path / "g.chain")
    rch = h2g.load_chain(tmp_path / "g.chain")
    B = np.stack([O.rhs(A.n, 1234 + c) for c in range(3)], axis=1)
    assert rel(rch.solve(B), gch.solve(B)) < 1e-12
