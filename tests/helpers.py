"""Shared fixtures: identical seeded inputs for the oracle and the GPU path."""
import numpy as np

import pyoracle as O
from paper_1703_06155_b200.geometry import rod_points, vie_constants, vie_grid_points


def rod_problem(n, eps_h2, leaf=25, eta=1.0, kernel=None):
    kernel = kernel or O.laplace(2.0)
    t = O.Tree(rod_points(n), leaf)
    b = O.Blocks(t, eta)
    return O.H2(b, kernel, eps_h2)


def vie_problem(cells, side, leaf, eps):
    k0, scale, diag = vie_constants(cells, side)
    K = O.helmholtz(k0, diag, scale)
    t = O.Tree(vie_grid_points(cells, side), leaf)
    b = O.Blocks(t, 1.0)
    return O.H2(b, K, eps), K


def ranks_by_cluster(records):
    return {(r["level"], r["cluster"]): r["rank_after"] for r in records}


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def replay_gpu_chain(ch):
    """Explicit L, U of a downloaded GPU chain (verify.hpp:41-91 restated in
    numpy): L = prod_levels[prod_recs(Q_i L_i) P^T] L_root, U mirrored."""
    n = ch.n
    L = np.eye(n, dtype=np.complex128)
    levels = []
    for li in range(ch.num_levels):
        recs = ch.records(li)
        mats = []
        for ri, r in enumerate(recs):
            Q, L11, U11 = ch.record_mats(li, ri)
            Lb, Ub = ch.record_blocks(li, ri)
            mats.append((r, Q, L11, U11, Lb, Ub))
        levels.append((mats, ch.perm(li)))

    def emb_q(r, Q):
        M = np.eye(n, dtype=np.complex128)
        p, b = r["pos"], r["bsize"]
        M[p:p + b, p:p + b] = Q
        return M

    def emb_p(src):
        P = np.zeros((n, n))
        P[np.arange(len(src)), src] = 1.0
        for q in range(len(src), n):
            P[q, q] = 1.0
        return P

    for mats, src in levels:
        for r, Q, L11, U11, Lb, Ub in mats:
            E = np.eye(n, dtype=np.complex128)
            e, p = r["eliminated"], r["pos"]
            if e:
                E[p:p + e, p:p + e] = L11
                for pos, M in Lb:
                    E[pos:pos + M.shape[0], p:p + e] = M
            L = L @ emb_q(r, Q) @ E
        L = L @ emb_p(src).T
    Lr, Ur = ch.root()
    R = np.eye(n, dtype=np.complex128)
    R[: ch.root_size, : ch.root_size] = Lr
    L = L @ R
    U = np.eye(n, dtype=np.complex128)
    U[: ch.root_size, : ch.root_size] = Ur
    for mats, src in reversed(levels):
        U = U @ emb_p(src)
        for r, Q, L11, U11, Lb, Ub in reversed(mats):
            E = np.eye(n, dtype=np.complex128)
            e, p = r["eliminated"], r["pos"]
            if e:
                E[p:p + e, p:p + e] = U11
                for pos, M in Ub:
                    E[p:p + e, pos:pos + M.shape[1]] = M
            U = U @ E @ emb_q(r, Q).T
    return L, U
