"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same H² input (oracle-built, uploaded through h2g_matrix_upload).

Tolerances (north_star): per-cluster ranks within +-1, solution within
10*eps of the oracle's, residual within 2x the oracle's; at tight eps the
factorizations agree to ~1e-10."""
import numpy as np
import pytest

import paper_1703_06155_b200 as h2g
import pyoracle as O
from helpers import ranks_by_cluster, rel, replay_gpu_chain, rod_problem, vie_problem

pytestmark = pytest.mark.gpu


def upload(A):
    return h2g.H2Matrix.upload(A.arrays())


def compare_chains(och, gch, rank_tol=0):
    assert och.stop_level == gch.stop_level
    ro, rg = ranks_by_cluster(och.all_records()), ranks_by_cluster(gch.all_records())
    assert ro.keys() == rg.keys()
    worst = max(abs(ro[k] - rg[k]) for k in ro) if ro else 0
    assert worst <= rank_tol, worst
    return worst


def test_rod_tight_eps_matches_oracle():
    A = rod_problem(256, 1e-12, leaf=32)
    och = A.factorize(1e-14)
    G = upload(A)
    gch = h2g.factorize(G, 1e-14)
    compare_chains(och, gch, 0)
    for lo, lg in zip(och.levels(), gch.levels()):
        for k in ("level", "rank_sum_before", "rank_sum_after", "eliminated", "ledger_blocks", "perm_len", "active_after"):
            assert lo[k] == lg[k], (k, lo, lg)
    assert och.root_size == gch.root_size
    b = O.rhs(256, 11)
    xo, xg = och.solve(b), gch.solve(b)
    assert rel(xg, xo) < 1e-10
    assert rel(xg, A.shadow_solve(b)) < 1e-10


def test_rod_substitutions_and_aliases():
    """test_solve.cpp:49-62 on the GPU chain: forward/backward apply the
    inverses of the replayed factors; the replay reproduces the matrix
    (verify.hpp:94-99, test_factorization.cpp:97-104)."""
    A = rod_problem(128, 1e-8, leaf=16)
    gch = h2g.factorize(upload(A), 1e-10)
    Lf, Uf = replay_gpu_chain(gch)
    Z = A.dense_shadow()
    assert np.linalg.norm(Lf @ Uf - Z) / np.linalg.norm(Z) < 100 * 1e-10
    b = O.rhs(128, 3)
    y = gch.forward(b)
    assert rel(y, np.linalg.solve(Lf, b)) < 1e-11
    assert rel(gch.backward(y), np.linalg.solve(Uf, y)) < 1e-11
    x = gch.solve(b)
    assert np.array_equal(gch.apply_inverse(b), x)
    assert rel(gch.apply_inverse_explicit(b), x) < 1e-12
    y = b.copy()
    h2g.solve_in_place(gch, y)
    assert np.array_equal(y, x)
    a, c = O.rhs(128, 1), O.rhs(128, 2)
    al, be = 0.7 - 1.3j, -0.2 + 0.5j
    lhs = gch.solve(al * a + be * c)
    r = al * gch.solve(a) + be * gch.solve(c)
    assert np.linalg.norm(lhs - r) <= 1e-12 * (np.linalg.norm(r) + 1)
    assert np.linalg.norm(gch.solve(np.zeros(128))) == 0.0


def test_multi_rhs_matches_columnwise():
    A = rod_problem(200, 1e-10)
    gch = h2g.factorize(upload(A), 1e-12)
    B = np.stack([O.rhs(200, s) for s in range(8)], axis=1)
    X = gch.apply_inverse(B)
    for j in range(8):
        assert rel(X[:, j], gch.solve(B[:, j])) < 1e-13
    Xe = gch.apply_inverse_explicit(B)
    assert rel(Xe, X) < 1e-12


@pytest.mark.parametrize("smem_kb,part_gb", [("24", None), ("6", "0")])
def test_rhs_groups_side_by_side_match_columnwise(monkeypatch, smem_kb, part_gb):
    """More right-hand sides than one shared-memory chunk holds run as groups
    side by side in one launch per level (grid y, own counters per group):
    bit-identical to the groups run one after the other, and equal to the
    column-by-column solves (solve.hpp:43-83 is column-independent)."""
    A, _ = vie_problem(16, 0.5, 32, 1e-4)
    gch = h2g.factorize(upload(A), 1e-4)
    n = A.n
    B = np.stack([O.rhs(n, 100 + s) for s in range(21)], axis=1)
    # a few columns per group -> several groups, ragged last one; second case: one
    # column per group -> 21 groups in two forward waves (16 + 5), backward waves of
    # one group (no room for more gathered-partials buffers)
    monkeypatch.setenv("H2G_SOLVE_SMEM_KB", smem_kb)
    if part_gb is not None:
        monkeypatch.setenv("H2G_SOLVE_PART_GB", part_gb)
    for fn in (gch.apply_inverse, gch.apply_inverse_explicit):
        monkeypatch.setenv("H2G_SOLVE_GROUPS", "1")
        X = fn(B)
        monkeypatch.setenv("H2G_SOLVE_GROUPS", "0")
        Xs = fn(B)
        assert np.array_equal(X, Xs)
        monkeypatch.setenv("H2G_SOLVE_GROUPS", "1")
        for j in (0, 7, 20):
            assert rel(X[:, j], fn(B[:, j])) < 1e-12


@pytest.mark.parametrize("refine_below", [None, "1e-4"])
def test_vie_config1_geometry_eps_1e6(monkeypatch, refine_below):
    """eps = 1e-6 (the tight end of config 4's sweep) on the config-1 geometry
    against the oracle: with the step-0 truncation decided on the Gram alone
    (default for eps >= 3e-7) and with the Rayleigh-Ritz refinement forced
    (H2G_REFINE_BELOW=1e-4), h2_matrix.hpp:279-290 / factorization.hpp:295-298."""
    if refine_below:
        monkeypatch.setenv("H2G_REFINE_BELOW", refine_below)
    eps = 1e-6
    A, _ = vie_problem(16, 0.5, 32, eps)
    och = A.factorize(eps)
    gch = h2g.factorize(upload(A), eps)
    compare_chains(och, gch, rank_tol=1)
    b = O.rhs(A.n, 1234)
    xo, xg = och.solve(b), gch.solve(b)
    assert rel(xg, xo) <= 10 * eps
    assert A.relative_residual(xg, b) <= 2 * A.relative_residual(xo, b)


def test_helmholtz_rod():
    A = rod_problem(200, 1e-10, kernel=O.helmholtz(0.3, 2.0))
    gch = h2g.factorize(upload(A), 1e-12)
    b = O.rhs(200, 5)
    assert rel(gch.solve(b), A.shadow_solve(b)) < 1e-9


@pytest.mark.parametrize("schedule", ["reference", "colored", "interior-first"])
def test_vie_config1_parity(schedule):
    """BASELINE config 1 (16^3 VIE cube, leaf 32, eps 1e-4) against the oracle
    run in the same elimination order."""
    A, K = vie_problem(16, 0.5, 32, 1e-4)
    eps = 1e-4
    sched = {"reference": O.SCHEDULE_REFERENCE, "colored": O.SCHEDULE_COLORED, "interior-first": O.SCHEDULE_INTERIOR_FIRST}[schedule]
    och = A.factorize(eps, schedule=sched)
    gch = h2g.factorize(upload(A), eps, schedule=schedule)
    compare_chains(och, gch, rank_tol=1)
    perm = A.tree.perm
    b = O.rhs(A.n, 1234)[perm]
    xo, xg = och.solve(b), gch.solve(b)
    assert rel(xg, xo) <= 10 * eps
    ro, rg = A.relative_residual(xo, b), A.relative_residual(xg, b)
    assert rg <= 2 * ro + 1e-14


def test_deterministic_and_input_untouched():
    A = rod_problem(128, 1e-8, leaf=16)
    G = upload(A)
    before = G.download()
    h1 = h2g.factorize(G, 1e-7).hash()
    h2 = h2g.factorize(G, 1e-7).hash()
    assert h1 == h2
    after = G.download()
    for k in before:
        assert np.array_equal(before[k], after[k]), k


def test_singular_pivot_reports_cluster_and_level():
    A = rod_problem(100, 1e-10, kernel=O.zero(0.0))
    with pytest.raises(h2g.SingularPivotError) as ei:
        h2g.factorize(upload(A), 1e-8)
    assert ei.value.cluster >= 0 and ei.value.level == A.tree.depth


def test_diagonal_kernel_early_stop():
    A = rod_problem(400, 1e-8, kernel=O.zero(2.0))
    gch = h2g.factorize(upload(A), 1e-8)
    assert gch.level(0)["eliminated"] == 400 and gch.root_size == 0 and gch.stop_level == 3
    b = O.rhs(400, 9)
    assert np.linalg.norm(gch.solve(b) - b / 2) < 1e-14 * np.linalg.norm(b)


def test_no_admissible_and_single_leaf():
    for n in (50, 20):
        A = rod_problem(n, 1e-8)
        gch = h2g.factorize(upload(A), 1e-8)
        assert gch.num_levels == 0 and gch.root_size == n
        L, U = gch.root()
        Z = A.dense_shadow()
        assert np.linalg.norm(L @ U - Z) < 1e-12 * np.linalg.norm(Z)


def test_input_validation():
    A = rod_problem(128, 1e-8, leaf=16)
    G = upload(A)
    with pytest.raises(h2g.InvalidInputError):
        h2g.factorize(G, 0.0)
    for bad in (1, A.tree.depth + 1):
        with pytest.raises(h2g.InvalidInputError):
            h2g.factorize(G, 1e-8, stop_level_override=bad)
    ch = h2g.factorize(G, 1e-8)
    with pytest.raises(h2g.InvalidInputError):
        ch.solve(O.rhs(127, 1))
    bad = O.rhs(128, 1)
    bad[3] = np.nan
    with pytest.raises(h2g.NonFiniteError):
        ch.solve(bad)


def test_gpu_matvec_matches_oracle():
    A, K = vie_problem(16, 0.5, 32, 1e-4)
    G = upload(A)
    x = O.rhs(A.n, 7)
    assert rel(G.matvec(x), A.matvec(x)) < 1e-12


@pytest.mark.parametrize("extra", [1, 2, "depth"])
def test_stop_level_override_paints_root(extra):
    """factorize(A, eps, stop_level_override) above l0: the root is painted
    from dense blocks, admissible couplings of this and coarser levels
    expanded to the root level, and the ledger / carried fill-in
    (factorization.hpp:204-234, 636-651); GPU against the oracle."""
    A = rod_problem(400, 1e-10, leaf=25)
    och_default = A.factorize(1e-10)
    l0 = och_default.stop_level
    stop = A.tree.depth if extra == "depth" else min(l0 + extra, A.tree.depth)
    och = A.factorize(1e-10, stop_level=stop)
    gch = h2g.factorize(upload(A), 1e-10, stop_level_override=stop)
    assert gch.stop_level == och.stop_level == stop
    assert gch.root_size == och.root_size > 0
    compare_chains(och, gch, 0)
    b = O.rhs(400, 21)
    xo, xg = och.solve(b), gch.solve(b)
    assert rel(xg, xo) < 1e-9
    assert rel(xg, A.shadow_solve(b)) < 1e-8


def test_vie_stop_override_matches_oracle():
    A, K = vie_problem(16, 0.5, 32, 1e-4)
    och0 = A.factorize(1e-4)
    stop = och0.stop_level + 1
    och = A.factorize(1e-4, stop_level=stop)
    gch = h2g.factorize(upload(A), 1e-4, stop_level_override=stop)
    assert gch.root_size == och.root_size
    compare_chains(och, gch, rank_tol=1)
    perm = A.tree.perm
    b = O.rhs(A.n, 77)[perm]
    xo, xg = och.solve(b), gch.solve(b)
    assert rel(xg, xo) <= 10 * 1e-4
    assert A.relative_residual(xg, b) <= 2 * A.relative_residual(xo, b) + 1e-14


def test_segmented_fill_and_streamed_chain_equal_resident(monkeypatch):
    """The large-configuration storage paths on a small input: segmented fill
    storage (compact cores, H2G_FILL_SEGMENTS) and the chain streamed to pinned
    host memory segment by segment (H2G_CHAIN_STREAM) run the same arithmetic as
    the resident layout, so the segmented + streamed chain equals the
    segmented + resident chain bit for bit, its records download the same, its
    container file round-trips, and the solve reads it from host memory."""
    A, _ = vie_problem(16, 0.5, 32, 1e-4)
    arrays = A.arrays()
    b = O.rhs(A.n, 21)
    ctx = h2g.Context.default()
    out = {}
    for mode, stream in (("resident", "0"), ("streamed", "1"), ("hostcores", "1")):
        monkeypatch.setenv("H2G_FILL_SEGMENTS", "4")
        monkeypatch.setenv("H2G_CHAIN_STREAM", stream)
        # third variant: the fill cores staged in pinned host memory (deposits over the host link, bulk return in the merge)
        monkeypatch.setenv("H2G_CORES_HOST", "1" if mode == "hostcores" else "0")
        ctx.clear_plans()
        G = h2g.H2Matrix.upload(arrays, ctx)
        ch = h2g.factorize(G, 1e-4)
        out[mode] = (ch, ch.hash(), ch.solve(b), ch.all_records(), G)
    monkeypatch.delenv("H2G_FILL_SEGMENTS")
    monkeypatch.delenv("H2G_CHAIN_STREAM")
    monkeypatch.delenv("H2G_CORES_HOST")
    ctx.clear_plans()
    assert out["resident"][1] == out["streamed"][1] == out["hostcores"][1]
    assert np.array_equal(out["resident"][2], out["streamed"][2])
    assert out["resident"][3] == out["streamed"][3]
    ch, G = out["streamed"][0], out["streamed"][4]
    Q0, L0, U0 = out["resident"][0].record_mats(0, 3)
    Q1, L1, U1 = ch.record_mats(0, 3)
    assert np.array_equal(Q0, Q1) and np.array_equal(L0, L1) and np.array_equal(U0, U1)
    # against the default storage (whole-level full blocks): same mathematics, different summation grouping
    ref = h2g.factorize(h2g.H2Matrix.upload(arrays, ctx), 1e-4)
    assert rel(out["streamed"][2], ref.solve(b)) <= 1e-3
    assert G.relative_residual(out["streamed"][2], b) <= 2 * G.relative_residual(ref.solve(b), b) + 1e-12


def test_large_block_eigensolver_path_is_bitwise_the_shared_memory_one(monkeypatch):
    """Blocks beyond ~420 rows keep the cluster's Gram columns in global memory
    (k_eig1c, reached at config 3's coarse levels); forced here on config 1's
    geometry, it must reproduce the shared-memory path bit for bit."""
    A, _ = vie_problem(16, 0.5, 32, 1e-4)
    G = upload(A)
    ref = h2g.factorize(G, 1e-4)
    monkeypatch.setenv("H2G_EIG_GLOBAL", "1")
    alt = h2g.factorize(G, 1e-4)
    monkeypatch.delenv("H2G_EIG_GLOBAL")
    assert ref.hash() == alt.hash()
