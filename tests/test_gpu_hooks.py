"""FactorizeHooks on the GPU path: the reference's stepwise dense-elimination
oracle (proj/tests/test_factorization.cpp:36-95) run against the device
state. A dense R is evolved by exact operations using the factorization's own
Qtilde (projection), an independent pivoted block elimination (elimination)
and the level permutation (merge); after every step the device state's
shadow (FactorState::shadow, painted from the device blocks) must equal R."""
import numpy as np
import pytest

import paper_1703_06155_b200 as h2g
from helpers import rod_problem

pytestmark = pytest.mark.gpu


def test_stepwise_dense_elimination_oracle_on_device():
    n = 256
    A = rod_problem(n, 1e-12, leaf=32)  # rod, leaf 32, Laplace shift 2, eps_h2 1e-12
    assert A.blocks.l0 == 2
    G = h2g.H2Matrix.upload(A.arrays())
    R = A.dense_shadow().copy()
    scale = np.linalg.norm(R)
    state = dict(R=R, worst=0.0, unit=0.0, steps=0)

    def gap(st):
        state["worst"] = max(state["worst"], np.linalg.norm(st.shadow() - state["R"]) / scale)
        state["steps"] += 1

    def after_basis_update(st, i):
        gap(st)  # extending a basis must not move the represented matrix

    def after_projection(st, i):
        c = st.cluster(i)
        assert c["rotated"]
        Q = st.qtilde(i)
        b, p = c["bsize"], c["pos"]
        state["unit"] = max(state["unit"], np.abs(Q.conj().T @ Q - np.eye(b)).max())
        Qf = np.eye(n, dtype=np.complex128)
        Qf[p:p + b, p:p + b] = Q
        state["R"] = Qf.conj().T @ state["R"] @ Qf.conj()
        gap(st)

    def after_elimination(st, i):
        c = st.cluster(i)
        e, p = c["eliminated"], c["pos"]
        R = state["R"]
        if e > 0:
            X = np.linalg.solve(R[p:p + e, p:p + e], R[p:p + e, :])  # independent pivoted elimination of the head
            R = R - R[:, p:p + e] @ X
            R[p:p + e, p:p + e] = np.eye(e)
            state["R"] = R
        gap(st)

    def after_merge(st):
        src = st.perm()
        P = np.zeros((n, n))
        P[np.arange(src.size), src] = 1.0
        for q in range(src.size, n):
            P[q, q] = 1.0
        state["R"] = P @ state["R"] @ P.T
        gap(st)

    ch = h2g.factorize_hooked(G, 1e-14, after_basis_update, after_projection, after_elimination, after_merge)
    assert state["steps"] > 3 * 8
    assert state["worst"] < 1e-10, state["worst"]
    assert state["unit"] < 1e-12
    assert ch.stop_level == 2 and ch.root_size > 0
    Lr, Ur = ch.root()
    r = ch.root_size
    assert np.linalg.norm(Lr @ Ur - state["R"][:r, :r]) < 1e-10 * scale
    elim = sum(l["eliminated"] for l in ch.levels())
    assert elim == n - r and elim > n // 2
    # the debug run is the reference order: same ranks as the batched run
    ref = h2g.factorize(G, 1e-14)
    assert [r["rank_after"] for r in ch.all_records()] == [r["rank_after"] for r in ref.all_records()]


def test_hook_exceptions_propagate():
    A = rod_problem(128, 1e-8, leaf=16)
    G = h2g.H2Matrix.upload(A.arrays())

    def boom(st, i):
        raise RuntimeError("from the hook")

    with pytest.raises(RuntimeError, match="from the hook"):
        h2g.factorize_hooked(G, 1e-8, after_projection=boom)
