// ORACLE — TEST INFRASTRUCTURE ONLY (see dense.hpp header).
// C ABI over the oracle for tests/ (ctypes), __graft_entry__.smoke() and the
// bench's cpu_baseline / --impl reference leg. Complex data is interleaved
// complex128, column-major, exactly the layout of the product C ABI
// (include/h2g.h).
#include <chrono>
#include <cstdio>
#include <random>

#include "factor.hpp"
#include "serialize.hpp"

using namespace h2o;

namespace {

thread_local std::string g_msg;
thread_local int64_t g_info[4] = {0, 0, -1, -1};
thread_local double g_pivmag = 0.0;

struct TreeH {
  std::shared_ptr<const ClusterTree> t;
};
struct BlocksH {
  std::shared_ptr<const BlockClusterTree> b;
};
struct H2H {
  H2Matrix A;
  KernelSpec K;
};
struct ChainH {
  FactorChain c;
};

int fail(int code, const std::string& m) {
  g_msg = m;
  g_info[0] = code;
  return code;
}

template <class F>
int guarded(F&& f) {
  try {
    g_info[0] = 0;
    f();
    return 0;
  } catch (const SingularPivotError& e) {
    g_info[1] = e.pivot_index;
    g_info[2] = e.cluster;
    g_info[3] = e.level;
    g_pivmag = e.pivot_magnitude;
    return fail(4, e.what());
  } catch (const InvalidInputError& e) {
    return fail(1, e.what());
  } catch (const SizeGuardError& e) {
    return fail(2, e.what());
  } catch (const NonFiniteError& e) {
    return fail(3, e.what());
  } catch (const UndefinedMetricError& e) {
    return fail(5, e.what());
  } catch (const ser::SerializationError& e) {
    return fail(6, e.what());
  } catch (const std::exception& e) {
    return fail(9, e.what());
  }
}

KernelSpec make_kernel(int kind, double kre, double kim, double sre, double sim, double dre, double dim) {
  KernelSpec K;
  K.kind = kind;
  K.wavenumber = cxd(kre, kim);
  K.scale = cxd(sre, sim);
  K.diag = cxd(dre, dim);
  return K;
}

Vec to_vec(const double* p, int64_t n) {
  Vec v(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) v[static_cast<size_t>(i)] = cxd(p[2 * i], p[2 * i + 1]);
  return v;
}
void from_vec(const Vec& v, double* p) {
  for (size_t i = 0; i < v.size(); ++i) p[2 * i] = v[i].real(), p[2 * i + 1] = v[i].imag();
}
void copy_mat(const Mat& M, double* out) { std::memcpy(out, M.d.data(), 16 * static_cast<size_t>(M.size())); }

uint64_t fnv(uint64_t h, const void* p, size_t n) {
  const unsigned char* c = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < n; ++i) h = (h ^ c[i]) * 1099511628211ull;
  return h;
}

}  // namespace

extern "C" {

int orc_last_error(char* buf, int len, int64_t* info, double* pivmag) {
  if (buf && len > 0) std::snprintf(buf, static_cast<size_t>(len), "%s", g_msg.c_str());
  if (info)
    for (int i = 0; i < 4; ++i) info[i] = g_info[i];
  if (pivmag) *pivmag = g_pivmag;
  return static_cast<int>(g_info[0]);
}

// Seeded complex-normal vector exactly as proj/tools/h2lu_cli.cpp:181-191
// (mt19937_64 + normal_distribution, cxd(g(rng), g(rng)) compiled by g++).
void orc_rhs(int64_t n, uint64_t seed, double* out) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> g;
  for (int64_t i = 0; i < n; ++i) {
    cxd v = cxd(g(rng), g(rng));
    out[2 * i] = v.real();
    out[2 * i + 1] = v.imag();
  }
}

void* orc_tree_new(const double* pts, int64_t n, int64_t leafsize) {
  TreeH* h = nullptr;
  guarded([&] {
    PointCloud P(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) P[static_cast<size_t>(i)] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    h = new TreeH{build_cluster_tree(P, leafsize)};
  });
  return h;
}
void orc_tree_free(void* h) { delete static_cast<TreeH*>(h); }
int orc_tree_depth(void* h) { return static_cast<TreeH*>(h)->t->depth; }
int64_t orc_tree_n(void* h) { return static_cast<TreeH*>(h)->t->n(); }
void orc_tree_perm(void* h, int64_t* out) {
  const auto& p = static_cast<TreeH*>(h)->t->perm;
  for (size_t i = 0; i < p.size(); ++i) out[i] = p[i];
}
void orc_tree_points(void* h, double* out) {
  const auto& p = static_cast<TreeH*>(h)->t->points;
  for (size_t i = 0; i < p.size(); ++i)
    for (int a = 0; a < 3; ++a) out[3 * i + static_cast<size_t>(a)] = p[i][static_cast<size_t>(a)];
}
void orc_tree_ranges(void* h, int64_t* begin, int64_t* end) {
  const auto& T = *static_cast<TreeH*>(h)->t;
  for (int i = 0; i < T.num_clusters(); ++i) begin[i] = T.cluster(i).begin, end[i] = T.cluster(i).end;
}

void* orc_blocks_new(void* tree, double eta) {
  BlocksH* h = nullptr;
  guarded([&] { h = new BlocksH{build_block_tree(static_cast<TreeH*>(tree)->t, eta)}; });
  return h;
}
void orc_blocks_free(void* h) { delete static_cast<BlocksH*>(h); }
int orc_blocks_l0(void* h) { return static_cast<BlocksH*>(h)->b->l0; }
int orc_blocks_csp(void* h, int level) { return static_cast<BlocksH*>(h)->b->csp(level); }
// counts: adm[depth+1], split[depth+1], then nleaf
void orc_blocks_counts(void* h, int64_t* adm, int64_t* split, int64_t* nleaf) {
  const auto& B = *static_cast<BlocksH*>(h)->b;
  for (size_t l = 0; l < B.admissible.size(); ++l) adm[l] = static_cast<int64_t>(B.admissible[l].size());
  for (size_t l = 0; l < B.split.size(); ++l) split[l] = static_cast<int64_t>(B.split[l].size());
  *nleaf = static_cast<int64_t>(B.inadmissible_leaf.size());
}
// kind 0 admissible, 1 split (per level), 2 inadmissible leaves (level ignored)
void orc_blocks_pairs(void* h, int kind, int level, int32_t* out) {
  const auto& B = *static_cast<BlocksH*>(h)->b;
  const std::vector<BlockPair>& v =
      kind == 0 ? B.admissible[static_cast<size_t>(level)] : kind == 1 ? B.split[static_cast<size_t>(level)] : B.inadmissible_leaf;
  for (size_t i = 0; i < v.size(); ++i) out[2 * i] = v[i].row, out[2 * i + 1] = v[i].col;
}

void* orc_h2_build(void* blocks, int kind, double kre, double kim, double sre, double sim, double dre, double dim, double eps_h2) {
  H2H* h = nullptr;
  guarded([&] {
    auto* hh = new H2H();
    hh->K = make_kernel(kind, kre, kim, sre, sim, dre, dim);
    try {
      hh->A = build_h2(hh->K, static_cast<BlocksH*>(blocks)->b, eps_h2);
    } catch (...) {
      delete hh;
      throw;
    }
    h = hh;
  });
  return h;
}
void orc_h2_free(void* h) { delete static_cast<H2H*>(h); }

// sizes: [num_clusters, basis_elems, num_adm, coupling_elems, num_leaf, dense_elems]
void orc_h2_sizes(void* h, int64_t* out) {
  const H2Matrix& A = static_cast<H2H*>(h)->A;
  int64_t be = 0, na = 0, ce = 0, de = 0;
  for (const auto& m : A.bases) be += m.size();
  for (const auto& lv : A.couplings)
    for (const auto& m : lv) na += 1, ce += m.size();
  for (const auto& m : A.dense_blocks) de += m.size();
  out[0] = static_cast<int64_t>(A.bases.size());
  out[1] = be;
  out[2] = na;
  out[3] = ce;
  out[4] = static_cast<int64_t>(A.dense_blocks.size());
  out[5] = de;
}

// Flat export in the layout of include/h2g.h (offsets in complex elements;
// couplings in level-major admissible order).
void orc_h2_export(void* h, int64_t* basis_rows, int64_t* basis_rank, int64_t* basis_off, double* basis_data, int64_t* coup_off,
                   double* coup_data, int64_t* dense_off, double* dense_data) {
  const H2Matrix& A = static_cast<H2H*>(h)->A;
  int64_t off = 0;
  for (size_t i = 0; i < A.bases.size(); ++i) {
    basis_rows[i] = A.bases[i].r;
    basis_rank[i] = A.bases[i].c;
    basis_off[i] = off;
    copy_mat(A.bases[i], basis_data + 2 * off);
    off += A.bases[i].size();
  }
  off = 0;
  size_t q = 0;
  for (const auto& lv : A.couplings)
    for (const auto& m : lv) {
      coup_off[q++] = off;
      copy_mat(m, coup_data + 2 * off);
      off += m.size();
    }
  off = 0;
  for (size_t i = 0; i < A.dense_blocks.size(); ++i) {
    dense_off[i] = off;
    copy_mat(A.dense_blocks[i], dense_data + 2 * off);
    off += A.dense_blocks[i].size();
  }
}

// Rebuild an oracle H2Matrix from flat arrays (e.g. a GPU-built matrix).
void* orc_h2_import(void* blocks, double eps_h2, const int64_t* basis_rows, const int64_t* basis_rank, const int64_t* basis_off,
                    const double* basis_data, const int64_t* coup_off, const double* coup_data, const int64_t* dense_off,
                    const double* dense_data) {
  H2H* h = nullptr;
  guarded([&] {
    auto* hh = new H2H();
    H2Matrix& A = hh->A;
    A.blocks = static_cast<BlocksH*>(blocks)->b;
    A.tree = A.blocks->tree;
    A.eps_h2 = eps_h2;
    const ClusterTree& T = *A.tree;
    A.bases.resize(static_cast<size_t>(T.num_clusters()));
    for (int i = 0; i < T.num_clusters(); ++i) {
      Mat M(basis_rows[i], basis_rank[i]);
      std::memcpy(M.d.data(), basis_data + 2 * basis_off[i], 16 * static_cast<size_t>(M.size()));
      A.bases[static_cast<size_t>(i)] = std::move(M);
    }
    size_t q = 0;
    A.couplings.resize(A.blocks->admissible.size());
    for (size_t l = 0; l < A.blocks->admissible.size(); ++l)
      for (const auto& p : A.blocks->admissible[l]) {
        Mat M(A.rank(p.row), A.rank(p.col));
        std::memcpy(M.d.data(), coup_data + 2 * coup_off[q++], 16 * static_cast<size_t>(M.size()));
        A.couplings[l].push_back(std::move(M));
      }
    const auto& lv = A.blocks->inadmissible_leaf;
    for (size_t i = 0; i < lv.size(); ++i) {
      Mat M(T.cluster(lv[i].row).size(), T.cluster(lv[i].col).size());
      std::memcpy(M.d.data(), dense_data + 2 * dense_off[i], 16 * static_cast<size_t>(M.size()));
      A.dense_blocks.push_back(std::move(M));
    }
    h = hh;
  });
  return h;
}

int orc_h2_rank(void* h, int id) { return static_cast<int>(static_cast<H2H*>(h)->A.rank(id)); }

int orc_h2_matvec(void* h, const double* x, double* y) {
  return guarded([&] {
    const H2Matrix& A = static_cast<H2H*>(h)->A;
    from_vec(A.matvec(to_vec(x, A.n())), y);
  });
}

int orc_h2_dense_shadow(void* h, double* out) {
  return guarded([&] { copy_mat(static_cast<H2H*>(h)->A.dense_shadow(), out); });
}

// Rows `rows` of the kernel matrix (tree order) times x: the dense sampled-row
// residual instrument of SURVEY §8d(ii).
int orc_kernel_rows_matvec(void* tree, int kind, double kre, double kim, double sre, double sim, double dre, double dim,
                           const int64_t* rows, int64_t nrows, const double* x, double* y) {
  return guarded([&] {
    const ClusterTree& T = *static_cast<TreeH*>(tree)->t;
    KernelSpec K = make_kernel(kind, kre, kim, sre, sim, dre, dim);
    const Index n = T.n();
    parallel_for(nrows, [&](int64_t q) {
      const Index r = rows[q];
      cxd s = 0.0;
      for (Index j = 0; j < n; ++j) {
        const cxd v = r == j ? K.diag : K.entry(T.points[static_cast<size_t>(r)], T.points[static_cast<size_t>(j)]);
        s += v * cxd(x[2 * j], x[2 * j + 1]);
      }
      y[2 * q] = s.real();
      y[2 * q + 1] = s.imag();
    });
  });
}

int orc_dense_solve(void* tree, int kind, double kre, double kim, double sre, double sim, double dre, double dim, const double* b,
                    double* x) {
  return guarded([&] {
    const ClusterTree& T = *static_cast<TreeH*>(tree)->t;
    from_vec(dense_oracle_solve(make_kernel(kind, kre, kim, sre, sim, dre, dim), T, to_vec(b, T.n())), x);
  });
}

// Dense solve of the H² dense shadow (PartialPivLU of A.dense_shadow()).
int orc_shadow_solve(void* h, const double* b, double* x) {
  return guarded([&] {
    const H2Matrix& A = static_cast<H2H*>(h)->A;
    Mat Z = A.dense_shadow();
    Mat B(A.n(), 1);
    for (Index i = 0; i < A.n(); ++i) B(i, 0) = cxd(b[2 * i], b[2 * i + 1]);
    Mat X = pivoted_lu_solve(Z, B);
    copy_mat(X, x);
  });
}

void* orc_factorize(void* h, double eps, int stop_level, int schedule, double* seconds) {
  ChainH* c = nullptr;
  guarded([&] {
    const H2Matrix& A = static_cast<H2H*>(h)->A;
    auto t0 = std::chrono::steady_clock::now();
    std::optional<int> stop;
    if (stop_level >= 0) stop = stop_level;
    FactorChain ch = factorize(A, eps, stop, nullptr, schedule);
    if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    c = new ChainH{std::move(ch)};
  });
  return c;
}
void orc_chain_free(void* c) { delete static_cast<ChainH*>(c); }

// [n, stop_level, root_size, num_levels, storage_bytes]
void orc_chain_info(void* c, int64_t* out) {
  const FactorChain& ch = static_cast<ChainH*>(c)->c;
  out[0] = ch.n;
  out[1] = ch.stop_level;
  out[2] = ch.root_size;
  out[3] = static_cast<int64_t>(ch.levels.size());
  out[4] = static_cast<int64_t>(ch.storage_bytes());
}
// [level, nrecs, rank_sum_before, rank_sum_after, eliminated, ledger_blocks, chain_bytes, perm_len, active_after]
void orc_chain_level(void* c, int li, int64_t* out) {
  const LevelBlock& lb = static_cast<ChainH*>(c)->c.levels[static_cast<size_t>(li)];
  out[0] = lb.level;
  out[1] = static_cast<int64_t>(lb.recs.size());
  out[2] = lb.diag.rank_sum_before;
  out[3] = lb.diag.rank_sum_after;
  out[4] = lb.diag.eliminated;
  out[5] = lb.diag.ledger_blocks;
  out[6] = static_cast<int64_t>(lb.diag.chain_bytes);
  out[7] = static_cast<int64_t>(lb.perm.src.size());
  out[8] = lb.perm.active_after;
}
// per record: [cluster, level, pos, bsize, eliminated, rank_before, rank_after, fill_targets, nLbar, nUbar]
void orc_chain_records(void* c, int li, int64_t* out) {
  const LevelBlock& lb = static_cast<ChainH*>(c)->c.levels[static_cast<size_t>(li)];
  for (size_t r = 0; r < lb.recs.size(); ++r) {
    const auto& R = lb.recs[r];
    int64_t* o = out + 10 * r;
    o[0] = R.cluster, o[1] = R.level, o[2] = R.pos, o[3] = R.bsize, o[4] = R.eliminated, o[5] = R.rank_before, o[6] = R.rank_after,
    o[7] = R.fill_targets, o[8] = static_cast<int64_t>(R.Lbar.size()), o[9] = static_cast<int64_t>(R.Ubar.size());
  }
}
void orc_chain_perm(void* c, int li, int64_t* out) {
  const auto& src = static_cast<ChainH*>(c)->c.levels[static_cast<size_t>(li)].perm.src;
  for (size_t i = 0; i < src.size(); ++i) out[i] = src[i];
}
void orc_chain_root(void* c, double* l, double* u) {
  const FactorChain& ch = static_cast<ChainH*>(c)->c;
  copy_mat(ch.root_l, l);
  copy_mat(ch.root_u, u);
}
// Qtilde (bsize^2), L11/U11 (e^2) of one record.
void orc_chain_record_mats(void* c, int li, int ri, double* q, double* l11, double* u11) {
  const auto& R = static_cast<ChainH*>(c)->c.levels[static_cast<size_t>(li)].recs[static_cast<size_t>(ri)];
  if (q) copy_mat(R.Qtilde, q);
  if (l11) copy_mat(R.L11, l11);
  if (u11) copy_mat(R.U11, u11);
}
// FNV-1a over every bit of the chain (determinism tests).
uint64_t orc_chain_hash(void* c) {
  const FactorChain& ch = static_cast<ChainH*>(c)->c;
  uint64_t h = 1469598103934665603ull;
  auto hm = [&](const Mat& m) {
    h = fnv(h, &m.r, 8);
    h = fnv(h, &m.c, 8);
    h = fnv(h, m.d.data(), 16 * m.d.size());
  };
  for (const auto& lb : ch.levels) {
    h = fnv(h, lb.perm.src.data(), 8 * lb.perm.src.size());
    for (const auto& r : lb.recs) {
      hm(r.Qtilde), hm(r.L11), hm(r.U11);
      for (const auto& b : r.Lbar) h = fnv(h, &b.pos, 8), hm(b.M);
      for (const auto& b : r.Ubar) h = fnv(h, &b.pos, 8), hm(b.M);
    }
  }
  hm(ch.root_l), hm(ch.root_u);
  return h;
}

// mode: 0 solve, 1 forward, 2 backward, 3 apply_inverse
int orc_solve(void* c, const double* b, int64_t nb, double* x, int mode) {
  return guarded([&] {
    const FactorChain& ch = static_cast<ChainH*>(c)->c;
    Vec v = to_vec(b, nb);
    if (mode == 0) v = solve(ch, v);
    else if (mode == 1) forward_substitute_in_place(ch, v);
    else if (mode == 2) backward_substitute_in_place(ch, v);
    else v = apply_inverse(ch, v);
    from_vec(v, x);
  });
}

int orc_replay(void* c, void* h, double* out) {
  return guarded([&] { *out = replay_dense_shadow(static_cast<ChainH*>(c)->c, static_cast<H2H*>(h)->A); });
}
// Explicit replayed L and U (n x n each).
int orc_replay_factors(void* c, double* L, double* U) {
  return guarded([&] {
    ReplayFactors f = replay_factors(static_cast<ChainH*>(c)->c);
    copy_mat(f.L, L);
    copy_mat(f.U, U);
  });
}

int orc_relative_residual(void* h, const double* x, const double* b, double* out) {
  return guarded([&] {
    const H2Matrix& A = static_cast<H2H*>(h)->A;
    *out = relative_residual(A, to_vec(x, A.n()), to_vec(b, A.n()));
  });
}

// Dense primitives for the dense-kernel tests (test_dense_kernels.cpp).
int orc_partial_lu(const double* F, int64_t n, double* L, double* U) {
  return guarded([&] {
    Mat M(n, n);
    std::memcpy(M.d.data(), F, 16 * static_cast<size_t>(n * n));
    auto lu = partial_lu(M);
    copy_mat(lu.first, L);
    copy_mat(lu.second, U);
  });
}
int orc_unitary_completion(const double* V, int64_t m, int64_t k, double* P) {
  return guarded([&] {
    Mat M(m, k);
    std::memcpy(M.d.data(), V, 16 * static_cast<size_t>(m * k));
    copy_mat(unitary_completion(M), P);
  });
}
// Returns rank r and fills U (m x r, caller sizes m*min(m,f)).
int orc_truncated_row_basis(const double* B, int64_t m, int64_t f, double eps, double floor, double* U, int64_t* r) {
  return guarded([&] {
    Mat M(m, f);
    std::memcpy(M.d.data(), B, 16 * static_cast<size_t>(m * f));
    Mat R = truncated_row_basis(M, eps, floor);
    *r = R.c;
    copy_mat(R, U);
  });
}

// -------------------------------------------------------------------------
// Reference test fixtures that need FactorState access, run in-process.

// test_factorization.cpp:36-95: the stepwise dense elimination oracle.
// out: [worst_gap, stop_level, root_size, elim_total, root_lu_err/scale, max_orth_defect, max_unitary_defect]
int orc_test_stepwise(void* h, double eps_fill, int schedule, double* out) {
  return guarded([&] {
    const H2Matrix& A = static_cast<H2H*>(h)->A;
    const Index n = A.n();
    Mat R = A.dense_shadow();
    const double scale = R.norm();
    double worst = 0.0, orth = 0.0, unit = 0.0;
    auto gap = [&](const FactorState& st) { worst = std::max(worst, (st.shadow() - R).norm() / scale); };
    FactorizeHooks hk;
    hk.after_basis_update = [&](const FactorState& st, int i) {
      const Mat& V = st.basis[static_cast<size_t>(i)];
      if (V.c > 0) orth = std::max(orth, (mul(V.adjoint(), V) - Mat::identity(V.c)).max_abs());
      gap(st);
    };
    hk.after_projection = [&](const FactorState& st, int i) {
      const EliminationRecord& rec = st.chain.levels.back().recs.back();
      if (rec.cluster != i) throw InvalidInputError("stepwise: record/cluster mismatch");
      unit = std::max(unit, (mul(rec.Qtilde.adjoint(), rec.Qtilde) - Mat::identity(rec.bsize)).max_abs());
      Mat Q = Mat::identity(n);
      Q.set_block(rec.pos, rec.pos, rec.Qtilde);
      R = mul(mul(Q.adjoint(), R), Q.conjugate());
      gap(st);
    };
    hk.after_elimination = [&](const FactorState& st, int i) {
      const EliminationRecord& rec = st.chain.levels.back().recs.back();
      if (rec.cluster != i) throw InvalidInputError("stepwise: record/cluster mismatch");
      const Index e = rec.eliminated, p = rec.pos;
      if (e > 0) {
        Mat X = pivoted_lu_solve(R.block(p, p, e, e), R.block(p, 0, e, n));
        R -= mul(R.block(0, p, n, e), X);
        R.set_block(p, p, Mat::identity(e));
      }
      gap(st);
    };
    hk.after_merge = [&](const FactorState& st) {
      const PermutationRecord& perm = st.chain.levels.back().perm;
      Mat P(n, n);
      for (size_t j = 0; j < perm.src.size(); ++j) P(static_cast<Index>(j), perm.src[j]) = 1.0;
      for (Index q = static_cast<Index>(perm.src.size()); q < n; ++q) P(q, q) = 1.0;
      R = mul(mul(P, R), P.transpose());
      gap(st);
    };
    FactorChain ch = factorize(A, eps_fill, std::nullopt, &hk, schedule);
    Index elim = 0;
    for (const auto& lb : ch.levels) elim += lb.diag.eliminated;
    double rerr = 0.0;
    if (ch.root_size > 0) rerr = (mul(ch.root_l, ch.root_u) - R.block(0, 0, ch.root_size, ch.root_size)).norm() / scale;
    out[0] = worst;
    out[1] = ch.stop_level;
    out[2] = static_cast<double>(ch.root_size);
    out[3] = static_cast<double>(elim);
    out[4] = rerr;
    out[5] = orth;
    out[6] = unit;
  });
}

// test_factorization.cpp:124-145: fill-free geometry keeps bases bit-identical.
// out: [all_bits_equal (0/1), ledger_total, any_rank_growth]
int orc_test_fill_free_bits(void* h, double eps_fill, double* out) {
  return guarded([&] {
    const H2Matrix& A = static_cast<H2H*>(h)->A;
    bool same = true;
    FactorizeHooks hk;
    hk.after_basis_update = [&](const FactorState& st, int i) {
      const Mat& V = st.basis[static_cast<size_t>(i)];
      const Mat& O = A.bases[static_cast<size_t>(i)];
      if (V.r != O.r || V.c != O.c || (V.size() && std::memcmp(V.d.data(), O.d.data(), 16 * V.d.size()) != 0)) same = false;
      if (st.kfin[static_cast<size_t>(i)] != O.c) same = false;
    };
    FactorChain ch = factorize(A, eps_fill, std::nullopt, &hk);
    Index ledger = 0;
    bool growth = false;
    for (const auto& lb : ch.levels) {
      ledger += lb.diag.ledger_blocks;
      for (const auto& r : lb.recs) growth = growth || r.rank_after != r.rank_before;
    }
    out[0] = same ? 1.0 : 0.0;
    out[1] = static_cast<double>(ledger);
    out[2] = growth ? 1.0 : 0.0;
  });
}

// test_factorization.cpp:256-297: carried fill on an ancestor-owned block
// embeds one level up. out: [shadow_err_rel, carried_empty, ledger_found, quad_err_rel, rest_norm]
int orc_test_carried_embed(void* h, double* out) {
  return guarded([&] {
    const H2Matrix& A = static_cast<H2H*>(h)->A;
    const ClusterTree& T = *A.tree;
    const BlockPair cover = A.blocks->admissible[2].front();
    const int j = T.cluster(cover.row).children[0];
    const int k = T.cluster(cover.col).children[0];
    FactorState st;
    st.init(A, 1e-13);
    std::mt19937_64 rng(7);
    std::normal_distribution<double> g;
    Mat F(st.bsz[static_cast<size_t>(j)], st.bsz[static_cast<size_t>(k)]);
    for (Index c = 0; c < F.c; ++c)
      for (Index r = 0; r < F.r; ++r) F(r, c) = cxd(g(rng), g(rng));
    st.carried.put(j, k, F);
    Mat expected = A.dense_shadow();
    expected.add_block(st.pos[static_cast<size_t>(j)], st.pos[static_cast<size_t>(k)], F);
    out[0] = (st.shadow() - expected).norm() / expected.norm();
    for (int i = T.level_begin(3); i < T.level_begin(3) + T.level_count(3); ++i) {
      step0_update_basis(st, i);
      const Mat& qt = step1_projection(st, i);
      step2_apply_projection(st, i, qt);
      step3_partial_eliminate(st, i);
    }
    const Mat vj = st.basis[static_cast<size_t>(j)], vk = st.basis[static_cast<size_t>(k)];
    const Index kj = st.kfin[static_cast<size_t>(j)], kk = st.kfin[static_cast<size_t>(k)];
    finish_level(st);
    merge_permute(st);
    out[1] = st.carried.empty() ? 1.0 : 0.0;
    const Mat* Lg = st.ledger.find(cover.row, cover.col);
    out[2] = Lg ? 1.0 : 0.0;
    if (Lg) {
      Mat quad = Lg->block(0, 0, kj, kk);
      out[3] = (quad - mul(mul(vj.adjoint(), F), vk.conjugate())).norm() / F.norm();
      Mat rest = *Lg;
      rest.zero_block(0, 0, kj, kk);
      out[4] = rest.norm();
    }
  });
}

}  // extern "C"

// ----------------------------------------------- H2LU v1 container (tests)
extern "C" {
// self-noise study: 1 = accumulate GEMM inner products last-to-first
void orc_set_gemm_order(int reverse) { gemm_order_flag() = reverse ? 1 : 0; }
// self-noise study: 1 = step-0 truncation through the Gram (Eq. 16-18)
void orc_set_truncation(int mode) { truncation_mode() = mode; }
int64_t orc_h2_n(void* h) { return static_cast<H2H*>(h)->A.n(); }
int orc_h2_save(void* h, const char* path) {
  return guarded([&] { ser::save_h2(path, static_cast<H2H*>(h)->A); });
}
void* orc_h2_load(const char* path) {
  H2H* out = nullptr;
  guarded([&] { out = new H2H{ser::load_h2(path), KernelSpec{}}; });
  return out;
}
int orc_chain_save(void* c, const char* path) {
  return guarded([&] { ser::save_chain(path, static_cast<ChainH*>(c)->c); });
}
void* orc_chain_load(const char* path) {
  ChainH* out = nullptr;
  guarded([&] { out = new ChainH{ser::load_chain(path)}; });
  return out;
}
int orc_vector_save(const char* path, const double* x, int64_t n) {
  return guarded([&] {
    std::vector<cxd> v(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) v[static_cast<size_t>(i)] = cxd(x[2 * i], x[2 * i + 1]);
    ser::save_vector(path, v);
  });
}
int orc_vector_load(const char* path, double* x, int64_t* n) {
  return guarded([&] {
    const auto v = ser::load_vector(path);
    if (x) {
      if (*n < static_cast<int64_t>(v.size())) throw InvalidInputError("vector_load: buffer too short");
      for (size_t i = 0; i < v.size(); ++i) x[2 * i] = v[i].real(), x[2 * i + 1] = v[i].imag();
    }
    *n = static_cast<int64_t>(v.size());
  });
}
}
