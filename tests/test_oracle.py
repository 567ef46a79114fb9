"""Pins the CPU oracle (oracle/, a restatement of the reference h2lu hot path)
against every known-answer test the reference's own suite holds for the path
(proj/tests/test_factorization.cpp, test_solve.cpp, test_dense_kernels.cpp,
acceptance_main.cpp). The reference ships no golden vectors, so
these property/known-answer tests are the pin."""
import numpy as np
import pytest

import pyoracle as O
from paper_1703_06155_b200.geometry import rod_points, slab_points, cube_points


def rod_h2(n, eps, eta=1.0, leaf=25, shift=2.0):
    t = O.Tree(rod_points(n), leaf)
    b = O.Blocks(t, eta)
    return O.H2(b, O.laplace(shift), eps)


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


# ---------------------------------------------------------------- dense kernels
def test_partial_lu_2x2_exact():  # test_dense_kernels.cpp:94-104
    L, U = O.partial_lu(np.array([[2.0, 1.0], [1.0, 2.0]]))
    assert L[0, 0] == 1 and L[1, 0] == 0.5 and L[0, 1] == 0
    assert U[0, 0] == 2 and U[0, 1] == 1 and U[1, 1] == 1.5 and U[1, 0] == 0


def test_partial_lu_multiplies_back():  # :106-118
    rng = np.random.default_rng(11)
    F = rng.normal(size=(20, 20)) + 1j * rng.normal(size=(20, 20)) + 10 * np.eye(20)
    L, U = O.partial_lu(F)
    assert np.abs(L @ U - F).max() < 1e-10 * np.abs(F).max()
    assert np.all(np.diag(L) == 1) and np.all(np.triu(L, 1) == 0) and np.all(np.tril(U, -1) == 0)


def test_partial_lu_singular_pivot():  # :120-131
    with pytest.raises(O.SingularPivotError) as ei:
        O.partial_lu(np.array([[0.0, 1.0], [1.0, 0.0]]))
    assert ei.value.pivot_index == 0 and ei.value.pivot_magnitude == 0.0


def _rand_orth(m, k, seed):
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.normal(size=(m, k)) + 1j * rng.normal(size=(m, k)))
    return q


def test_unitary_completion():  # :63-92
    assert np.allclose(O.unitary_completion(np.zeros((5, 0))), np.eye(5))
    assert O.unitary_completion(_rand_orth(4, 4, 5)).shape == (4, 0)
    for s in (1, 2, 3):
        V = _rand_orth(10, 4, s)
        P = O.unitary_completion(V)
        Q = np.hstack([P, V])
        assert np.abs(Q.conj().T @ Q - np.eye(10)).max() < 1e-12
        assert np.abs(P.conj().T @ V).max() < 1e-12
    with pytest.raises(O.InvalidInputError):
        O.unitary_completion(2.0 * _rand_orth(6, 2, 9))


def test_truncated_row_basis_exact_rank():
    rng = np.random.default_rng(3)
    X = (rng.normal(size=(12, 3)) + 1j * rng.normal(size=(12, 3))) @ (rng.normal(size=(3, 40)) + 0j)
    U = O.truncated_row_basis(X, 1e-10)
    assert U.shape[1] == 3
    assert np.abs(U.conj().T @ U - np.eye(3)).max() < 1e-12
    assert np.linalg.norm(X - U @ (U.conj().T @ X)) < 1e-10 * np.linalg.norm(X)


# ------------------------------------------------------------- factorization
def test_stepwise_dense_elimination_oracle():  # test_factorization.cpp:36-95
    t = O.Tree(rod_points(256), 32)
    b = O.Blocks(t, 1.0)
    assert b.l0 == 2
    A = O.H2(b, O.laplace(2.0), 1e-12)
    r = A.test_stepwise(1e-14)
    assert r["worst"] < 1e-10
    assert r["stop_level"] == 2 and r["root_size"] > 0
    assert r["root_err"] < 1e-10
    assert r["eliminated"] == 256 - r["root_size"] and r["eliminated"] > 128
    assert r["orth"] < 1e-12 and r["unitary"] < 1e-12


def test_stepwise_colored_schedule_is_exact_too():
    A = O.H2(O.Blocks(O.Tree(rod_points(256), 32)), O.laplace(2.0), 1e-12)
    r = A.test_stepwise(1e-14, O.SCHEDULE_COLORED)
    assert r["worst"] < 1e-10


def test_stepwise_interior_first_schedule_is_exact_too():
    """The north_star's subtree split as an elimination order (interior
    clusters of the 8 level-3 subtrees first, then the boundary): still an
    exact factorization of the represented matrix (stepwise dense oracle)."""
    from paper_1703_06155_b200.geometry import cube_points

    A = O.H2(O.Blocks(O.Tree(cube_points(512), 8)), O.laplace(2.0), 1e-10)
    r = A.test_stepwise(1e-12, O.SCHEDULE_INTERIOR_FIRST)
    assert r["worst"] < 1e-10
    ch_ref, ch_if = A.factorize(1e-12), A.factorize(1e-12, schedule=O.SCHEDULE_INTERIOR_FIRST)
    b = O.rhs(512, 4)
    assert np.linalg.norm(ch_if.solve(b) - ch_ref.solve(b)) / np.linalg.norm(ch_ref.solve(b)) < 1e-8


def test_replay_reproduces_matrix():  # :97-104
    A = rod_h2(128, 1e-8, 1.0, 16)
    for eps in (1e-6, 1e-10):
        ch = A.factorize(eps)
        assert ch.level(0)["ledger_blocks"] > 0
        assert ch.replay_error(A) < 100 * eps


def test_fill_bounds():  # :106-122
    t = O.Tree(rod_points(256), 32)
    b = O.Blocks(t, 1.0)
    A = O.H2(b, O.laplace(2.0), 1e-6)
    ch = A.factorize(1e-8)
    adm, _, _ = b.counts()
    for li in range(ch.num_levels):
        lv = ch.level(li)
        cap = b.csp(lv["level"]) ** 2
        for r in ch.records(li):
            assert r["fill_targets"] <= cap
            assert r["rank_before"] <= r["rank_after"] <= r["bsize"]
            assert r["eliminated"] == r["bsize"] - r["rank_after"]
        assert lv["ledger_blocks"] <= adm[lv["level"]]


def test_fill_free_bases_bit_identical():  # :124-145
    pts = np.vstack([rod_points(50), rod_points(50) + np.array([1000.0, 0, 0])])
    t = O.Tree(pts, 25)
    b = O.Blocks(t, 1.0)
    assert b.l0 == 1
    A = O.H2(b, O.laplace(2.0), 1e-8)
    r = A.test_fill_free_bits(1e-8)
    assert r["same_bits"] and r["ledger"] == 0 and not r["growth"]
    assert A.factorize(1e-8).replay_error(A) < 1e-12


def test_diagonal_kernel_stops_early():  # :147-160
    t = O.Tree(rod_points(400), 25)
    b = O.Blocks(t, 1.0)
    assert b.l0 == 2 and t.depth == 4
    A = O.H2(b, O.zero(2.0), 1e-8)
    ch = A.factorize(1e-8)
    assert ch.level(0)["eliminated"] == 400
    assert ch.root_size == 0 and ch.stop_level == 3
    assert all(r["eliminated"] == r["bsize"] for r in ch.records(0))
    bb = O.rhs(400, 9)
    assert np.linalg.norm(ch.solve(bb) - bb / 2) < 1e-14 * np.linalg.norm(bb)  # test_solve.cpp:104-113


def test_no_admissible_is_dense_lu():  # :162-171
    A = rod_h2(50, 1e-8)
    assert A.blocks.l0 == -1
    ch = A.factorize(1e-8)
    assert ch.num_levels == 0 and ch.stop_level == A.tree.depth + 1 and ch.root_size == 50
    L, U = ch.root()
    Z = A.dense_shadow()
    assert np.linalg.norm(L @ U - Z) < 1e-12 * np.linalg.norm(Z)


def test_single_leaf():  # :173-179
    A = rod_h2(20, 1e-8)
    ch = A.factorize(1e-8)
    assert ch.num_levels == 0 and ch.root_size == 20
    assert ch.replay_error(A) < 1e-13


def test_stop_level_override():  # :181-196
    A = rod_h2(128, 1e-8, 1.0, 16)
    L = A.tree.depth
    assert A.blocks.l0 == 2
    leaf = A.factorize(1e-8, stop_level=L)
    assert leaf.stop_level == L and leaf.num_levels == 1
    assert leaf.replay_error(A) < 100 * 1e-8
    full = A.factorize(1e-8, stop_level=2)
    assert full.root_size < leaf.root_size
    for bad in (1, L + 1):
        with pytest.raises(O.InvalidInputError):
            A.factorize(1e-8, stop_level=bad)


def test_deterministic():  # :198-225
    A = rod_h2(128, 1e-8, 1.0, 16)
    assert A.factorize(1e-7).hash() == A.factorize(1e-7).hash()


def test_singular_pivot_reports_cluster_and_level():  # :227-239
    t = O.Tree(rod_points(100), 25)
    A = O.H2(O.Blocks(t, 1.0), O.zero(0.0), 1e-10)
    with pytest.raises(O.SingularPivotError) as ei:
        A.factorize(1e-8)
    assert ei.value.cluster >= 0 and ei.value.level == t.depth


def test_input_not_modified():  # :241-254
    A = rod_h2(128, 1e-8, 1.0, 16)
    before = A.export()
    A.factorize(1e-6)
    after = A.export()
    for k in before:
        assert np.array_equal(before[k], after[k])


def test_carried_fill_embeds_one_level_up():  # :256-297
    t = O.Tree(rod_points(64), 8)
    b = O.Blocks(t, 1.0)
    assert b.l0 == 2
    A = O.H2(b, O.laplace(2.0), 1e-10)
    r = A.test_carried_embed()
    assert r["shadow_err"] < 1e-12
    assert r["carried_empty"] and r["ledger_found"]
    assert r["quad_err"] < 1e-12 and r["rest_norm"] == 0.0


# -------------------------------------------------------------------- solve
def test_solve_vs_dense_shadow():  # test_solve.cpp:40-47
    A = rod_h2(200, 1e-10)
    ch = A.factorize(1e-12)
    b = O.rhs(200, 11)
    assert rel(ch.solve(b), A.shadow_solve(b)) < 1e-10


def test_substitutions_vs_replayed_factors():  # :49-62
    A = rod_h2(128, 1e-8, 1.0, 16)
    ch = A.factorize(1e-10)
    L, U = ch.replay_factors()
    b = O.rhs(128, 3)
    y = ch.forward(b)
    assert rel(y, np.linalg.solve(L, b)) < 1e-11
    x = ch.backward(y)
    assert rel(x, np.linalg.solve(U, y)) < 1e-11


def test_helmholtz_solve():  # :64-73
    t = O.Tree(rod_points(200), 25)
    A = O.H2(O.Blocks(t, 1.0), O.helmholtz(0.3, 2.0), 1e-10)
    ch = A.factorize(1e-12)
    b = O.rhs(200, 5)
    assert rel(ch.solve(b), A.shadow_solve(b)) < 1e-9


def test_solve_vs_kernel_dense_oracle():  # :75-85
    t = O.Tree(rod_points(300), 25)
    K = O.laplace(2.0)
    A = O.H2(O.Blocks(t, 1.0), K, 1e-8)
    ch = A.factorize(1e-8)
    b = O.rhs(300, 23)
    assert rel(ch.solve(b), t.dense_solve(K, b)) < 100 * 2e-8


def test_linearity_zero_alias_inplace():  # :87-131
    A = rod_h2(128, 1e-8, 1.0, 16)
    ch = A.factorize(1e-8)
    a, c = O.rhs(128, 1), O.rhs(128, 2)
    al, be = 0.7 - 1.3j, -0.2 + 0.5j
    lhs = ch.solve(al * a + be * c)
    r = al * ch.solve(a) + be * ch.solve(c)
    assert np.linalg.norm(lhs - r) <= 1e-12 * (np.linalg.norm(r) + 1)
    assert np.array_equal(ch.apply_inverse(a), ch.solve(a))
    z = rod_h2(100, 1e-8).factorize(1e-8).solve(np.zeros(100))
    assert np.linalg.norm(z) == 0.0


def test_solve_validates_rhs():  # :133-140
    ch = rod_h2(100, 1e-8).factorize(1e-8)
    with pytest.raises(O.InvalidInputError):
        ch.solve(O.rhs(99, 1))
    bad = O.rhs(100, 1)
    bad[3] = np.nan
    with pytest.raises(O.NonFiniteError):
        ch.solve(bad)


# --------------------------------------------------------------- acceptance
@pytest.mark.parametrize("kernel", [O.laplace(2.0), O.helmholtz(0.5, 2.0)])
def test_acceptance_oracle_equivalence(kernel):  # acceptance_main.cpp:53-82
    for n in (100, 200, 400):
        t = O.Tree(rod_points(n), 25)
        A = O.H2(O.Blocks(t, 1.0), kernel, 1e-6)
        ch = A.factorize(1e-8)
        b = O.rhs(n, n)
        assert rel(ch.solve(b), t.dense_solve(kernel, b)) < 1e-4


def test_acceptance_accuracy_knob():  # acceptance_main.cpp:120-145
    t = O.Tree(rod_points(3200), 25)
    A = O.H2(O.Blocks(t, 1.0), O.laplace(2.0), 1e-10)
    b = O.rhs(3200, 1234)
    res = []
    for eps in (1e-3, 1e-5, 1e-7):
        x = A.factorize(eps).solve(b)
        res.append(A.relative_residual(x, b))
    assert res[0] > res[1] > res[2]
    assert A.relative_residual(A.factorize(1e-4).solve(b), b) <= 1e-2


@pytest.mark.parametrize("geom", ["rod", "slab", "cube"])
def test_acceptance_fill_targets_bounded(geom):  # acceptance_main.cpp:245-274
    pts = {"rod": rod_points(800), "slab": slab_points(900), "cube": cube_points(1000)}[geom]
    t = O.Tree(pts, 25)
    b = O.Blocks(t, 1.0)
    A = O.H2(b, O.laplace(2.0), 1e-6)
    ch = A.factorize(1e-6)
    adm, _, _ = b.counts()
    for li in range(ch.num_levels):
        lv = ch.level(li)
        for r in ch.records(li):
            assert r["fill_targets"] <= b.csp(lv["level"]) ** 2
        assert lv["ledger_blocks"] <= adm[lv["level"]]


def test_rhs_generator_reference_convention():
    """mt19937_64 + libstdc++ normal_distribution, cxd(g(rng), g(rng))."""
    v = O.rhs(4, 1234)
    assert v.dtype == np.complex128 and np.all(np.isfinite(v))
    assert np.array_equal(v, O.rhs(4, 1234)) and not np.array_equal(v, O.rhs(4, 1235))
