// ORACLE — TEST INFRASTRUCTURE ONLY (see dense.hpp header).
//
// Restatement of the level-by-level H² partial LU of
// proj/include/h2lu/factorization.hpp:19-653 and of the substitutions of
// proj/include/h2lu/solve.hpp:11-113. Differences from the reference, none of
// which changes the arithmetic performed on any block:
//   * block maps keep a per-column index so "every key touching cluster i" is
//     found without the whole-map scans of factorization.hpp:268-293, :345,
//     :404, :436 (iteration order is still the std::map key order);
//   * the within-level cluster order is a parameter (`ClusterOrder`). The
//     default is the reference's ascending heap id (factorization.hpp:618);
//     `colored` processes a greedy distance-1 colouring colour by colour, the
//     batched order the GPU `colored` schedule runs.
#pragma once

#include <functional>
#include <optional>
#include <set>

#include "h2.hpp"

namespace h2o {

struct EliminationRecord {  // factorization.hpp:22-44
  int cluster = -1, level = -1;
  Index pos = 0, bsize = 0, eliminated = 0, rank_before = 0, rank_after = 0, fill_targets = 0;
  Mat Qtilde, L11, U11;
  struct Block {
    Index pos = 0;
    Mat M;
  };
  std::vector<Block> Lbar, Ubar;
};

struct PermutationRecord {  // factorization.hpp:50-54
  int level = -1;
  std::vector<Index> src;
  Index active_after = 0;
};

struct LevelDiagnostics {  // factorization.hpp:56-63
  int level = -1;
  Index rank_sum_before = 0, rank_sum_after = 0, eliminated = 0, ledger_blocks = 0;
  size_t chain_bytes = 0;
};

struct LevelBlock {
  int level = -1;
  std::vector<EliminationRecord> recs;
  PermutationRecord perm;
  LevelDiagnostics diag;
};

struct FactorChain {  // factorization.hpp:76-98
  std::shared_ptr<const ClusterTree> tree;
  Index n = 0;
  int stop_level = 0;
  double eps_fill_in = 0.0;
  std::vector<LevelBlock> levels;
  Mat root_l, root_u;
  Index root_size = 0;
  size_t storage_bytes() const {
    size_t t = 16 * static_cast<size_t>(root_l.size() + root_u.size());
    for (const auto& lb : levels) {
      t += 8 * lb.perm.src.size();
      for (const auto& r : lb.recs) {
        t += 16 * static_cast<size_t>(r.Qtilde.size() + r.L11.size() + r.U11.size());
        for (const auto& b : r.Lbar) t += 16 * static_cast<size_t>(b.M.size());
        for (const auto& b : r.Ubar) t += 16 * static_cast<size_t>(b.M.size());
      }
    }
    return t;
  }
};

using Key = std::pair<int, int>;

// std::map keyed (row, col) plus a column index, so the keys touching one
// cluster come out in map order in O(touching) instead of O(map).
struct BlockMap {
  std::map<Key, Mat> m;
  std::map<int, std::set<int>> by_col;

  Mat* find(int r, int c) {
    auto it = m.find({r, c});
    return it == m.end() ? nullptr : &it->second;
  }
  const Mat* find(int r, int c) const {
    auto it = m.find({r, c});
    return it == m.end() ? nullptr : &it->second;
  }
  Mat& at(int r, int c) {
    auto it = m.find({r, c});
    if (it == m.end()) throw InvalidInputError("block map: missing key");
    return it->second;
  }
  Mat& put(int r, int c, Mat M) {
    by_col[c].insert(r);
    auto& slot = m[{r, c}];
    slot = std::move(M);
    return slot;
  }
  // Adds into an existing entry or creates it (deposit_fill try_emplace).
  void accumulate(int r, int c, const Mat& F) {
    auto it = m.find({r, c});
    if (it == m.end()) {
      put(r, c, F);
    } else {
      it->second += F;
    }
  }
  void clear() {
    m.clear();
    by_col.clear();
  }
  bool empty() const { return m.empty(); }
  size_t size() const { return m.size(); }
  // Keys with row == i or col == i, in lexicographic (row, col) order.
  std::vector<Key> touching(int i) const {
    std::vector<Key> out;
    auto cit = by_col.find(i);
    const std::set<int>* rows = cit == by_col.end() ? nullptr : &cit->second;
    if (rows)
      for (int r : *rows) {
        if (r >= i) break;
        out.emplace_back(r, i);
      }
    for (auto it = m.lower_bound({i, std::numeric_limits<int>::min()}); it != m.end() && it->first.first == i; ++it)
      out.push_back(it->first);
    if (rows)
      for (auto it = rows->upper_bound(i); it != rows->end(); ++it) out.emplace_back(*it, i);
    return out;
  }
};

// ------------------------------------------------------------- schedules
enum ScheduleKind { SCHEDULE_REFERENCE = 0, SCHEDULE_COLORED = 1, SCHEDULE_INTERIOR_FIRST = 3 };
constexpr int kInteriorParts = 8;  // the north_star's 8-GPU subtree split

// Greedy distance-1 colouring in ascending id over the dense-neighbour graph
// of one level; returns the cluster order (colour, id).
inline std::vector<int> colored_order(const std::vector<int>& ids, const std::vector<Key>& dense_keys) {
  std::map<int, std::set<int>> nb;
  for (const auto& k : dense_keys)
    if (k.first != k.second) {
      nb[k.first].insert(k.second);
      nb[k.second].insert(k.first);
    }
  std::map<int, int> color;
  for (int i : ids) {
    std::set<int> used;
    for (int x : nb[i]) {
      auto it = color.find(x);
      if (it != color.end()) used.insert(it->second);
    }
    int c = 0;
    while (used.count(c)) ++c;
    color[i] = c;
  }
  std::vector<int> order = ids;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return color[a] < color[b]; });
  return order;
}

// ----------------------------------------------------------- factor state
struct FactorState {  // factorization.hpp:115-251
  const H2Matrix* A = nullptr;
  double eps_fill_in = 0.0;
  int level = 0;
  Index active_len = 0;
  std::vector<Index> pos, bsz, kfin;
  std::vector<char> rotated;
  std::vector<Mat> basis, qtilde;
  BlockMap dense, ledger, carried, final_coupling;
  FactorChain chain;

  Index korig(int id) const { return A->rank(id); }

  void init(const H2Matrix& M, double eps) {
    A = &M;
    eps_fill_in = eps;
    const ClusterTree& T = *M.tree;
    level = T.depth;
    active_len = T.n();
    const size_t nc = static_cast<size_t>(T.num_clusters());
    pos.assign(nc, 0);
    bsz.assign(nc, 0);
    kfin.assign(nc, 0);
    rotated.assign(nc, 0);
    basis.assign(nc, Mat());
    qtilde.assign(nc, Mat());
    for (int id = T.level_begin(level); id < T.level_begin(level) + T.level_count(level); ++id) {
      const Cluster& c = T.cluster(id);
      pos[static_cast<size_t>(id)] = c.begin;
      bsz[static_cast<size_t>(id)] = c.size();
      kfin[static_cast<size_t>(id)] = korig(id);
      basis[static_cast<size_t>(id)] = M.bases[static_cast<size_t>(id)];
    }
    const auto& leaves = M.blocks->inadmissible_leaf;
    for (size_t q = 0; q < leaves.size(); ++q) dense.put(leaves[q].row, leaves[q].col, M.dense_blocks[q]);
    chain.tree = M.tree;
    chain.n = T.n();
    chain.eps_fill_in = eps;
  }

  LevelBlock& level_block() {
    if (chain.levels.empty() || chain.levels.back().level != level) {
      chain.levels.emplace_back();
      chain.levels.back().level = level;
      chain.levels.back().perm.level = level;
      chain.levels.back().diag.level = level;
    }
    return chain.levels.back();
  }

  void place_block(Mat& Z, int t, int s, Mat M) const {  // :177-188
    const size_t ut = static_cast<size_t>(t), us = static_cast<size_t>(s);
    if (rotated[ut]) {
      M = mul(qtilde[ut].adjoint(), M);
      M.zero_block(0, 0, bsz[ut] - kfin[ut], M.c);
    }
    if (rotated[us]) {
      M = mul(M, qtilde[us].conjugate());
      M.zero_block(0, 0, M.r, bsz[us] - kfin[us]);
    }
    Z.set_block(pos[ut], pos[us], M);
  }

  void expand_to_level(int id, const Mat& C, std::vector<std::pair<int, Mat>>& out) const {  // :192-201
    const Cluster& c = A->tree->cluster(id);
    if (c.level == level) {
      out.emplace_back(id, mul(basis[static_cast<size_t>(id)].left_cols(korig(id)), C));
      return;
    }
    const Mat& T = A->bases[static_cast<size_t>(id)];
    expand_to_level(c.children[0], mul(T.top_rows(korig(c.children[0])), C), out);
    expand_to_level(c.children[1], mul(T.bottom_rows(korig(c.children[1])), C), out);
  }

  void paint(Mat& Z) const {  // :207-234
    for (const auto& kv : dense.m)
      Z.set_block(pos[static_cast<size_t>(kv.first.first)], pos[static_cast<size_t>(kv.first.second)], kv.second);
    const auto& adm = A->blocks->admissible[static_cast<size_t>(level)];
    for (size_t q = 0; q < adm.size(); ++q) {
      const int t = adm[q].row, s = adm[q].col;
      Mat M = mul(mul(basis[static_cast<size_t>(t)].left_cols(korig(t)), A->couplings[static_cast<size_t>(level)][q]),
                  basis[static_cast<size_t>(s)].left_cols(korig(s)).transpose());
      if (const Mat* F = ledger.find(t, s)) M += *F;
      place_block(Z, t, s, std::move(M));
    }
    const int l0 = A->blocks->l0;
    if (l0 < 0) return;
    for (int la = l0; la < level; ++la) {
      const auto& coarse = A->blocks->admissible[static_cast<size_t>(la)];
      for (size_t q = 0; q < coarse.size(); ++q) {
        std::vector<std::pair<int, Mat>> rs, cs;
        expand_to_level(coarse[q].row, Mat::identity(korig(coarse[q].row)), rs);
        expand_to_level(coarse[q].col, Mat::identity(korig(coarse[q].col)), cs);
        const Mat& S = A->couplings[static_cast<size_t>(la)][q];
        for (const auto& u : rs)
          for (const auto& v : cs) {
            Mat M = mul(mul(u.second, S), v.second.transpose());
            if (const Mat* F = carried.find(u.first, v.first)) M += *F;
            place_block(Z, u.first, v.first, std::move(M));
          }
      }
    }
  }

  Mat shadow() const {
    Mat Z(A->n(), A->n());
    for (Index p = active_len; p < A->n(); ++p) Z(p, p) = 1.0;
    paint(Z);
    return Z;
  }
  Mat active_matrix() const {
    Mat Z(active_len, active_len);
    paint(Z);
    return Z;
  }
};

// Self-noise study only: the step-0 truncation through the Gram of the
// projected fill stack (the paper's Eq. 16-18 formulation, the one the GPU
// path uses) instead of QR(W^H) + Jacobi SVD (h2_matrix.hpp:279-285); same
// rule sigma > max(eps sigma_0, floor, 1e-300). 0 = reference form (default).
inline int& truncation_mode() {
  static int mode = 0;
  return mode;
}

inline Mat truncated_row_basis_gram(const Mat& W, double eps, double floor) {
  const Index m = W.r;
  if (m == 0 || W.c == 0) return Mat(m, 0);
  Mat G = mul(W, W.adjoint());
  SVDResult svd = jacobi_svd_left(G);  // PSD: singular values = eigenvalues
  if (svd.sigma.empty() || svd.sigma[0] <= 0.0) return Mat(m, 0);
  const double s0 = std::sqrt(svd.sigma[0]);
  const double thr = std::max({eps * s0, floor, 1e-300});
  Index r = 0;
  while (r < static_cast<Index>(svd.sigma.size()) && std::sqrt(std::max(svd.sigma[static_cast<size_t>(r)], 0.0)) > thr) ++r;
  return svd.U.left_cols(r);
}

// Step 0 (factorization.hpp:260-312).
inline Index step0_update_basis(FactorState& st, int i) {
  const size_t ui = static_cast<size_t>(i);
  Mat& V = st.basis[ui];
  const Index b = st.bsz[ui], k = V.c;
  st.kfin[ui] = k;
  std::vector<std::pair<const Mat*, bool>> parts;  // (block, transposed)
  Index cols = 0;
  for (const BlockMap* bm : {&st.ledger, &st.carried})
    for (const Key& key : bm->touching(i)) {
      const Mat* F = bm->find(key.first, key.second);
      if (key.first == i) parts.emplace_back(F, false), cols += F->c;
      if (key.second == i) parts.emplace_back(F, true), cols += F->r;
    }
  if (cols == 0 || k == b) return 0;
  Mat W(b, cols);
  Index at = 0;
  for (const auto& p : parts) {
    const Mat& F = *p.first;
    if (!p.second) {
      W.set_block(0, at, F);
      at += F.c;
    } else {
      W.set_block(0, at, F.transpose());
      at += F.r;
    }
  }
  double cmax = 0.0;
  for (Index j = 0; j < W.c; ++j) {
    double s = 0.0;
    for (Index r = 0; r < W.r; ++r) s += std::norm(W(r, j));
    cmax = std::max(cmax, std::sqrt(s));
  }
  const double floor = st.eps_fill_in * cmax;
  if (k > 0) W -= mul(V, mul(V.adjoint(), W));
  Mat add = truncation_mode() == 1 ? truncated_row_basis_gram(W, st.eps_fill_in, floor) : truncated_row_basis(W, st.eps_fill_in, floor);
  const Index r = std::min<Index>(add.c, b - k);
  if (r == 0) return 0;
  Mat vnew(b, k + r);
  vnew.set_block(0, 0, V);
  if (k > 0) {
    Mat a = add.left_cols(r);
    Mat polish = a - mul(V, mul(V.adjoint(), a));
    HouseholderQR qr(polish);
    vnew.set_block(0, k, qr.q_cols(r));
  } else {
    vnew.set_block(0, k, add.left_cols(r));
  }
  V = std::move(vnew);
  st.kfin[ui] = k + r;
  return r;
}

// Step 1 (factorization.hpp:317-339).
inline const Mat& step1_projection(FactorState& st, int i) {
  const size_t ui = static_cast<size_t>(i);
  const Mat& V = st.basis[ui];
  const Index b = st.bsz[ui];
  Mat qt(b, b);
  qt.set_block(0, 0, unitary_completion(V));
  qt.set_block(0, b - V.c, V);
  EliminationRecord rec;
  rec.cluster = i;
  rec.level = st.level;
  rec.pos = st.pos[ui];
  rec.bsize = b;
  rec.eliminated = b - V.c;
  rec.rank_before = st.korig(i);
  rec.rank_after = st.kfin[ui];
  rec.Qtilde = qt;
  st.qtilde[ui] = std::move(qt);
  LevelBlock& lb = st.level_block();
  lb.recs.push_back(std::move(rec));
  return lb.recs.back().Qtilde;
}

// Step 2 (factorization.hpp:344-350).
inline void step2_apply_projection(FactorState& st, int i, const Mat& Q) {
  const Mat QH = Q.adjoint(), Qc = Q.conjugate();
  const auto keys = st.dense.touching(i);
  std::vector<Mat*> blocks;
  for (const Key& key : keys) blocks.push_back(&st.dense.at(key.first, key.second));
  pool_for(static_cast<int64_t>(keys.size()), [&](int64_t q) {  // distinct blocks
    Mat& D = *blocks[static_cast<size_t>(q)];
    if (keys[static_cast<size_t>(q)].first == i) D = mul(QH, D);
    if (keys[static_cast<size_t>(q)].second == i) D = mul(D, Qc);
  });
  st.rotated[static_cast<size_t>(i)] = 1;
}

// deposit_fill (factorization.hpp:359-366): the lift of a rotated side ...
inline Mat lift_fill(const FactorState& st, int j, int k, Mat F) {
  const size_t uj = static_cast<size_t>(j), uk = static_cast<size_t>(k);
  if (st.rotated[uj]) F = mul(st.basis[uj], F.bottom_rows(st.kfin[uj]));
  if (st.rotated[uk]) F = mul(F.right_cols(st.kfin[uk]), st.basis[uk].transpose());
  return F;
}

// ... and the accumulation into the ledger (admissible at this level) or the
// carried map.
inline void deposit_fill(FactorState& st, int j, int k, Mat F) {
  F = lift_fill(st, j, k, std::move(F));
  BlockMap& target = contains_pair(st.A->blocks->admissible[static_cast<size_t>(st.level)], j, k) ? st.ledger : st.carried;
  target.accumulate(j, k, F);
}

// Step 3 (factorization.hpp:377-440).
inline void step3_partial_eliminate(FactorState& st, int i) {
  const size_t ui = static_cast<size_t>(i);
  LevelBlock& lb = st.level_block();
  if (lb.recs.empty() || lb.recs.back().cluster != i)
    throw InvalidInputError("step3_partial_eliminate: cluster " + std::to_string(i) + " has no open elimination record");
  EliminationRecord& rec = lb.recs.back();
  const Index b = st.bsz[ui], k = st.kfin[ui], e = b - k;
  rec.eliminated = e;
  if (e == 0) return;
  Mat& Dii = st.dense.at(i, i);
  try {
    auto lu = partial_lu(Dii.block(0, 0, e, e));
    rec.L11 = std::move(lu.first);
    rec.U11 = std::move(lu.second);
  } catch (const SingularPivotError& ex) {
    throw SingularPivotError(std::string(ex.what()) + " (cluster " + std::to_string(i) + ", level " + std::to_string(st.level) + ")",
                             ex.pivot_index, ex.pivot_magnitude, i, st.level);
  }
  std::vector<std::pair<int, Mat>> rows, cols;
  const auto keys = st.dense.touching(i);
  for (const Key& key : keys) {
    const Mat& D = *st.dense.find(key.first, key.second);
    if (key.first == i && key.second != i) cols.emplace_back(key.second, solve_unit_lower(rec.L11, D.top_rows(e)));
    if (key.second == i && key.first != i) rows.emplace_back(key.first, solve_right_upper(D.left_cols(e), rec.U11));
  }
  if (k > 0) {
    cols.emplace_back(i, solve_unit_lower(rec.L11, Dii.block(0, e, e, k)));
    rows.emplace_back(i, solve_right_upper(Dii.block(e, 0, k, e), rec.U11));
  }
  // Every (row, column) pair is a distinct target, so the products run in
  // parallel; the fill slots are created first (serially, in map order) and
  // each receives exactly one contribution from this cluster.
  const size_t nr = rows.size(), nc = cols.size();
  std::vector<Mat*> dense_t(nr * nc, nullptr), fill_t(nr * nc, nullptr);
  std::vector<char> fresh(nr * nc, 0);
  for (size_t a = 0; a < nr; ++a)
    for (size_t c = 0; c < nc; ++c) {
      const int j = rows[a].first, x = cols[c].first;
      if (Mat* T = st.dense.find(j, x)) {
        dense_t[a * nc + c] = T;
        continue;
      }
      BlockMap& target = contains_pair(st.A->blocks->admissible[static_cast<size_t>(st.level)], j, x) ? st.ledger : st.carried;
      Mat* slot = target.find(j, x);
      if (!slot) slot = &target.put(j, x, Mat()), fresh[a * nc + c] = 1;
      fill_t[a * nc + c] = slot;
    }
  pool_for(static_cast<int64_t>(nr * nc), [&](int64_t q) {
    const size_t a = static_cast<size_t>(q) / nc, c = static_cast<size_t>(q) % nc;
    const auto& rj = rows[a];
    const auto& cc = cols[c];
    Mat P = mul(rj.second, cc.second);
    if (Mat* T = dense_t[static_cast<size_t>(q)]) {
      const Index ro = rj.first == i ? e : 0, co = cc.first == i ? e : 0;
      T->add_block(ro, co, P, -1.0);
      return;
    }
    for (cxd& v : P.d) v = -v;
    Mat F = lift_fill(st, rj.first, cc.first, std::move(P));
    if (fresh[static_cast<size_t>(q)])
      *fill_t[static_cast<size_t>(q)] = std::move(F);
    else
      *fill_t[static_cast<size_t>(q)] += F;
  });
  rec.fill_targets = static_cast<Index>(rows.size() * cols.size());
  for (auto& rj : rows) rec.Lbar.push_back({st.pos[static_cast<size_t>(rj.first)] + (rj.first == i ? e : 0), std::move(rj.second)});
  for (auto& cc : cols) rec.Ubar.push_back({st.pos[static_cast<size_t>(cc.first)] + (cc.first == i ? e : 0), std::move(cc.second)});
  Dii.set_block(0, 0, Mat::identity(e));
  if (k > 0) {
    Dii.zero_block(0, e, e, k);
    Dii.zero_block(e, 0, k, e);
  }
  for (const Key& key : keys) {
    Mat& D = st.dense.at(key.first, key.second);
    if (key.first == i && key.second != i) D.zero_block(0, 0, e, D.c);
    if (key.second == i && key.first != i) D.zero_block(0, 0, D.r, e);
  }
}

// finish_level (factorization.hpp:445-475).
inline void finish_level(FactorState& st) {
  const auto& adm = st.A->blocks->admissible[static_cast<size_t>(st.level)];
  const auto& coup = st.A->couplings[static_cast<size_t>(st.level)];
  size_t absorbed = 0;
  std::vector<Mat> sfs(adm.size());
  pool_for(static_cast<int64_t>(adm.size()), [&](int64_t qq) {
    const size_t q = static_cast<size_t>(qq);
    const int t = adm[q].row, s = adm[q].col;
    const size_t ut = static_cast<size_t>(t), us = static_cast<size_t>(s);
    Mat sf(st.kfin[ut], st.kfin[us]);
    sf.set_block(0, 0, coup[q]);
    if (const Mat* F = st.ledger.find(t, s)) sf += mul(mul(st.basis[ut].adjoint(), *F), st.basis[us].conjugate());
    sfs[q] = std::move(sf);
  });
  for (size_t q = 0; q < adm.size(); ++q) {
    if (st.ledger.find(adm[q].row, adm[q].col)) ++absorbed;
    st.final_coupling.put(adm[q].row, adm[q].col, std::move(sfs[q]));
  }
  if (absorbed != st.ledger.size()) throw InvalidInputError("finish_level: ledger holds a key that is not admissible at this level");
  st.ledger.clear();
  st.level_block().diag.ledger_blocks = static_cast<Index>(absorbed);
  if (st.level > 0) {
    const ClusterTree& T = *st.A->tree;
    const int lp = st.level - 1;
    for (int t = T.level_begin(lp); t < T.level_begin(lp) + T.level_count(lp); ++t) {
      const Cluster& c = T.cluster(t);
      const int c1 = c.children[0], c2 = c.children[1];
      const Mat& Tr = st.A->bases[static_cast<size_t>(t)];
      Mat padded(st.kfin[static_cast<size_t>(c1)] + st.kfin[static_cast<size_t>(c2)], Tr.c);
      padded.set_block(0, 0, Tr.top_rows(st.korig(c1)));
      padded.set_block(st.kfin[static_cast<size_t>(c1)], 0, Tr.bottom_rows(st.korig(c2)));
      st.basis[static_cast<size_t>(t)] = std::move(padded);
    }
  }
}

// merge_permute (factorization.hpp:483-584).
inline void merge_permute(FactorState& st) {
  const ClusterTree& T = *st.A->tree;
  const int l = st.level, lp = l - 1;
  LevelBlock& lb = st.level_block();
  auto kf = [&](int id) { return st.kfin[static_cast<size_t>(id)]; };
  auto elim = [&](int id) { return st.bsz[static_cast<size_t>(id)] - kf(id); };
  PermutationRecord perm;
  perm.level = l;
  perm.src.reserve(static_cast<size_t>(st.active_len));
  for (int t = T.level_begin(lp); t < T.level_begin(lp) + T.level_count(lp); ++t) {
    const Cluster& c = T.cluster(t);
    for (int ch : {c.children[0], c.children[1]}) {
      const Index base = st.pos[static_cast<size_t>(ch)] + elim(ch);
      for (Index q = 0; q < kf(ch); ++q) perm.src.push_back(base + q);
    }
  }
  const Index active_new = static_cast<Index>(perm.src.size());
  for (int i = T.level_begin(l); i < T.level_begin(l) + T.level_count(l); ++i) {
    const Index base = st.pos[static_cast<size_t>(i)];
    for (Index q = 0; q < elim(i); ++q) perm.src.push_back(base + q);
  }
  if (static_cast<Index>(perm.src.size()) != st.active_len) throw InvalidInputError("merge_permute: active layout does not add up");
  perm.active_after = active_new;

  BlockMap ndense;
  for (const BlockPair& p : st.A->blocks->split[static_cast<size_t>(lp)]) {
    const Cluster& t = T.cluster(p.row);
    const Cluster& s = T.cluster(p.col);
    Mat D(kf(t.children[0]) + kf(t.children[1]), kf(s.children[0]) + kf(s.children[1]));
    Index ro = 0;
    for (int a : {t.children[0], t.children[1]}) {
      Index co = 0;
      for (int c : {s.children[0], s.children[1]}) {
        if (const Mat* S = st.final_coupling.find(a, c)) {
          D.set_block(ro, co, *S);
        } else {
          const Mat* Dd = st.dense.find(a, c);
          if (!Dd) throw InvalidInputError("merge_permute: child block is neither dense nor admissible");
          D.set_block(ro, co, Dd->block(elim(a), elim(c), kf(a), kf(c)));
        }
        co += kf(c);
      }
      ro += kf(a);
    }
    ndense.put(p.row, p.col, std::move(D));
  }

  BlockMap moved;
  std::vector<const std::pair<const Key, Mat>*> items;
  for (const auto& kv : st.carried.m) items.push_back(&kv);
  std::vector<Mat> projs(items.size());
  pool_for(static_cast<int64_t>(items.size()), [&](int64_t q) {
    const auto& kv = *items[static_cast<size_t>(q)];
    projs[static_cast<size_t>(q)] =
        mul(mul(st.basis[static_cast<size_t>(kv.first.first)].adjoint(), kv.second), st.basis[static_cast<size_t>(kv.first.second)].conjugate());
  });
  for (size_t q = 0; q < items.size(); ++q) {
    const auto& kv = *items[q];
    const int j = kv.first.first, c = kv.first.second;
    const int pj = T.cluster(j).parent, pc = T.cluster(c).parent;
    const Mat& proj = projs[q];
    const Cluster& cpj = T.cluster(pj);
    const Cluster& cpc = T.cluster(pc);
    const Index ro = j == cpj.children[0] ? 0 : kf(cpj.children[0]);
    const Index co = c == cpc.children[0] ? 0 : kf(cpc.children[0]);
    const Index bpj = kf(cpj.children[0]) + kf(cpj.children[1]);
    const Index bpc = kf(cpc.children[0]) + kf(cpc.children[1]);
    Mat* slot = moved.find(pj, pc);
    if (!slot) slot = &moved.put(pj, pc, Mat(bpj, bpc));
    slot->add_block(ro, co, proj);
  }
  st.carried.clear();
  for (auto& kv : moved.m) {
    if (contains_pair(st.A->blocks->admissible[static_cast<size_t>(lp)], kv.first.first, kv.first.second)) {
      st.ledger.put(kv.first.first, kv.first.second, std::move(kv.second));
    } else if (ndense.find(kv.first.first, kv.first.second)) {
      throw InvalidInputError("merge_permute: carried fill-in resurfaced on a dense block");
    } else {
      st.carried.put(kv.first.first, kv.first.second, std::move(kv.second));
    }
  }

  lb.diag.rank_sum_before = lb.diag.rank_sum_after = lb.diag.eliminated = 0;
  for (int i = T.level_begin(l); i < T.level_begin(l) + T.level_count(l); ++i) {
    lb.diag.rank_sum_before += st.korig(i);
    lb.diag.rank_sum_after += kf(i);
    lb.diag.eliminated += elim(i);
  }
  Index off = 0;
  for (int t = T.level_begin(lp); t < T.level_begin(lp) + T.level_count(lp); ++t) {
    const Cluster& c = T.cluster(t);
    st.pos[static_cast<size_t>(t)] = off;
    st.bsz[static_cast<size_t>(t)] = kf(c.children[0]) + kf(c.children[1]);
    off += st.bsz[static_cast<size_t>(t)];
    st.kfin[static_cast<size_t>(t)] = st.basis[static_cast<size_t>(t)].c;
  }
  if (off != active_new) throw InvalidInputError("merge_permute: parent layout does not match the permutation");
  st.dense = std::move(ndense);
  st.final_coupling.clear();
  lb.perm = std::move(perm);
  st.level = lp;
  st.active_len = active_new;
  lb.diag.chain_bytes = st.chain.storage_bytes();
}

struct FactorizeHooks {  // factorization.hpp:588-593
  std::function<void(const FactorState&, int)> after_basis_update, after_projection, after_elimination;
  std::function<void(const FactorState&)> after_merge;
};

inline std::vector<int> level_order(const FactorState& st, int l, int schedule) {
  const ClusterTree& T = *st.A->tree;
  std::vector<int> ids(static_cast<size_t>(T.level_count(l)));
  std::iota(ids.begin(), ids.end(), T.level_begin(l));
  if (schedule == SCHEDULE_COLORED) {
    std::vector<Key> keys;
    for (const auto& kv : st.dense.m) keys.push_back(kv.first);
    return colored_order(ids, keys);
  }
  if (schedule == SCHEDULE_INTERIOR_FIRST && T.level_count(l) >= kInteriorParts) {
    // interior clusters of the level-3 subtrees (all dense neighbours in the
    // same subtree) first, then the boundary clusters, each ascending
    int lp = 0;
    while ((1 << lp) < kInteriorParts) ++lp;
    const int first = T.level_begin(l), shift = l - lp;
    std::set<int> boundary;
    for (const auto& kv : st.dense.m) {
      const int a = kv.first.first - first, b = kv.first.second - first;
      if ((a >> shift) != (b >> shift)) boundary.insert(kv.first.first), boundary.insert(kv.first.second);
    }
    std::vector<int> order;
    for (int i : ids)
      if (!boundary.count(i)) order.push_back(i);
    for (int i : ids)
      if (boundary.count(i)) order.push_back(i);
    return order;
  }
  return ids;
}

// factorize (factorization.hpp:600-653) with the within-level order as data.
inline FactorChain factorize(const H2Matrix& A, double eps_fill_in, std::optional<int> stop_override = std::nullopt,
                             const FactorizeHooks* hooks = nullptr, int schedule = SCHEDULE_REFERENCE) {
  if (eps_fill_in <= 0.0) throw InvalidInputError("factorize: eps_fill_in must be positive");
  FactorState st;
  st.init(A, eps_fill_in);
  const int L = A.depth(), l0 = A.blocks->l0;
  int stop = L + 1;
  if (l0 >= 0) {
    stop = stop_override.value_or(l0);
    if (stop < l0 || stop > L)
      throw InvalidInputError("factorize: stop level " + std::to_string(stop) + " outside [" + std::to_string(l0) + ", " + std::to_string(L) + "]");
  }
  st.chain.stop_level = stop;
  for (int l = L; l >= stop; --l) {
    Index elim_total = 0;
    for (int i : level_order(st, l, schedule)) {
      step0_update_basis(st, i);
      if (hooks && hooks->after_basis_update) hooks->after_basis_update(st, i);
      const Mat& qt = step1_projection(st, i);
      step2_apply_projection(st, i, qt);
      if (hooks && hooks->after_projection) hooks->after_projection(st, i);
      step3_partial_eliminate(st, i);
      if (hooks && hooks->after_elimination) hooks->after_elimination(st, i);
      elim_total += st.bsz[static_cast<size_t>(i)] - st.kfin[static_cast<size_t>(i)];
    }
    finish_level(st);
    merge_permute(st);
    if (hooks && hooks->after_merge) hooks->after_merge(st);
    if (elim_total == 0 && l > stop) {
      st.chain.stop_level = l;
      break;
    }
  }
  Mat root = st.active_matrix();
  st.chain.root_size = root.r;
  if (root.r > 0) {
    try {
      auto lu = partial_lu(root);
      st.chain.root_l = std::move(lu.first);
      st.chain.root_u = std::move(lu.second);
    } catch (const SingularPivotError& ex) {
      throw SingularPivotError(std::string(ex.what()) + " (root block after level " + std::to_string(st.chain.stop_level) + ")",
                               ex.pivot_index, ex.pivot_magnitude, -1, st.chain.stop_level);
    }
  }
  return std::move(st.chain);
}

// ------------------------------------------------------------------- solve
// proj/include/h2lu/solve.hpp:11-113. Vectors in tree order.
using Vec = std::vector<cxd>;

inline void check_rhs(const FactorChain& ch, const Vec& b) {
  if (static_cast<Index>(b.size()) != ch.n)
    throw InvalidInputError("solve: right-hand side has length " + std::to_string(b.size()) + ", factorization expects " + std::to_string(ch.n));
  for (const cxd& v : b)
    if (!std::isfinite(v.real()) || !std::isfinite(v.imag())) throw NonFiniteError("solve: right-hand side contains non-finite entries");
}

inline void forward_substitute_in_place(const FactorChain& ch, Vec& y) {
  check_rhs(ch, y);
  Vec scratch;
  for (const LevelBlock& lb : ch.levels) {
    for (const EliminationRecord& rec : lb.recs) {
      Vec seg(y.begin() + rec.pos, y.begin() + rec.pos + rec.bsize), out(static_cast<size_t>(rec.bsize), 0.0);
      for (Index j = 0; j < rec.bsize; ++j)
        for (Index i = 0; i < rec.bsize; ++i) out[static_cast<size_t>(j)] += std::conj(rec.Qtilde(i, j)) * seg[static_cast<size_t>(i)];
      std::copy(out.begin(), out.end(), y.begin() + rec.pos);
      if (rec.eliminated == 0) continue;
      cxd* head = y.data() + rec.pos;
      for (Index p = 0; p < rec.eliminated; ++p)
        for (Index i = p + 1; i < rec.eliminated; ++i) head[i] -= rec.L11(i, p) * head[p];
      for (const auto& blk : rec.Lbar)
        for (Index j = 0; j < blk.M.c; ++j)
          for (Index i = 0; i < blk.M.r; ++i) y[static_cast<size_t>(blk.pos + i)] -= blk.M(i, j) * head[j];
    }
    scratch.resize(lb.perm.src.size());
    for (size_t j = 0; j < lb.perm.src.size(); ++j) scratch[j] = y[static_cast<size_t>(lb.perm.src[j])];
    std::copy(scratch.begin(), scratch.end(), y.begin());
  }
  if (ch.root_size > 0) {
    for (Index p = 0; p < ch.root_size; ++p)
      for (Index i = p + 1; i < ch.root_size; ++i) y[static_cast<size_t>(i)] -= ch.root_l(i, p) * y[static_cast<size_t>(p)];
  }
}

inline void backward_substitute_in_place(const FactorChain& ch, Vec& y) {
  check_rhs(ch, y);
  Vec scratch;
  if (ch.root_size > 0) {
    for (Index p = ch.root_size - 1; p >= 0; --p) {
      y[static_cast<size_t>(p)] /= ch.root_u(p, p);
      for (Index i = 0; i < p; ++i) y[static_cast<size_t>(i)] -= ch.root_u(i, p) * y[static_cast<size_t>(p)];
    }
  }
  for (auto lit = ch.levels.rbegin(); lit != ch.levels.rend(); ++lit) {
    scratch.assign(lit->perm.src.size(), 0.0);
    for (size_t j = 0; j < lit->perm.src.size(); ++j) scratch[static_cast<size_t>(lit->perm.src[j])] = y[j];
    std::copy(scratch.begin(), scratch.end(), y.begin());
    for (auto rit = lit->recs.rbegin(); rit != lit->recs.rend(); ++rit) {
      const EliminationRecord& rec = *rit;
      if (rec.eliminated > 0) {
        cxd* head = y.data() + rec.pos;
        for (const auto& blk : rec.Ubar)
          for (Index j = 0; j < blk.M.c; ++j)
            for (Index i = 0; i < blk.M.r; ++i) head[i] -= blk.M(i, j) * y[static_cast<size_t>(blk.pos + j)];
        for (Index p = rec.eliminated - 1; p >= 0; --p) {
          head[p] /= rec.U11(p, p);
          for (Index i = 0; i < p; ++i) head[i] -= rec.U11(i, p) * head[p];
        }
      }
      Vec seg(y.begin() + rec.pos, y.begin() + rec.pos + rec.bsize), out(static_cast<size_t>(rec.bsize), 0.0);
      for (Index j = 0; j < rec.bsize; ++j)
        for (Index i = 0; i < rec.bsize; ++i) out[static_cast<size_t>(i)] += std::conj(rec.Qtilde(i, j)) * seg[static_cast<size_t>(j)];
      std::copy(out.begin(), out.end(), y.begin() + rec.pos);
    }
  }
}

inline Vec solve(const FactorChain& ch, const Vec& b) {
  Vec x = b;
  forward_substitute_in_place(ch, x);
  backward_substitute_in_place(ch, x);
  return x;
}
inline Vec apply_inverse(const FactorChain& ch, const Vec& b) { return solve(ch, b); }

// ------------------------------------------------------------------ verify
// proj/include/h2lu/verify.hpp:14-99.
inline double vnorm(const Vec& v) {
  double s = 0.0;
  for (const cxd& x : v) s += std::norm(x);
  return std::sqrt(s);
}

inline double relative_residual(const H2Matrix& A, const Vec& x, const Vec& b) {
  if (static_cast<Index>(x.size()) != A.n() || static_cast<Index>(b.size()) != A.n())
    throw InvalidInputError("relative_residual: vector length does not match the matrix");
  const double nb = vnorm(b);
  if (nb == 0.0) throw UndefinedMetricError("relative_residual: right-hand side is zero");
  Vec r = A.matvec(x);
  for (size_t i = 0; i < r.size(); ++i) r[i] -= b[i];
  return vnorm(r) / nb;
}

struct ReplayFactors {
  Mat L, U;
};

inline ReplayFactors replay_factors(const FactorChain& ch, Index guard = 200) {
  const Index n = ch.n;
  if (n > guard) throw SizeGuardError("replay_factors: n = " + std::to_string(n) + " exceeds the replay guard " + std::to_string(guard));
  auto eq = [n](const EliminationRecord& r) {
    Mat Q = Mat::identity(n);
    Q.set_block(r.pos, r.pos, r.Qtilde);
    return Q;
  };
  auto el = [n](const EliminationRecord& r) {
    Mat L = Mat::identity(n);
    if (r.eliminated == 0) return L;
    L.set_block(r.pos, r.pos, r.L11);
    for (const auto& b : r.Lbar) L.set_block(b.pos, r.pos, b.M);
    return L;
  };
  auto eu = [n](const EliminationRecord& r) {
    Mat U = Mat::identity(n);
    if (r.eliminated == 0) return U;
    U.set_block(r.pos, r.pos, r.U11);
    for (const auto& b : r.Ubar) U.set_block(r.pos, b.pos, b.M);
    return U;
  };
  auto ep = [n](const PermutationRecord& p) {
    Mat P(n, n);
    for (size_t j = 0; j < p.src.size(); ++j) P(static_cast<Index>(j), p.src[j]) = 1.0;
    for (Index q = static_cast<Index>(p.src.size()); q < n; ++q) P(q, q) = 1.0;
    return P;
  };
  ReplayFactors out;
  out.L = Mat::identity(n);
  for (const LevelBlock& lb : ch.levels) {
    for (const auto& r : lb.recs) out.L = mul(mul(out.L, eq(r)), el(r));
    out.L = mul(out.L, ep(lb.perm).transpose());
  }
  Mat rl = Mat::identity(n);
  rl.set_block(0, 0, ch.root_l);
  out.L = mul(out.L, rl);
  Mat ru = Mat::identity(n);
  ru.set_block(0, 0, ch.root_u);
  out.U = ru;
  for (auto lit = ch.levels.rbegin(); lit != ch.levels.rend(); ++lit) {
    out.U = mul(out.U, ep(lit->perm));
    for (auto rit = lit->recs.rbegin(); rit != lit->recs.rend(); ++rit) out.U = mul(mul(out.U, eu(*rit)), eq(*rit).transpose());
  }
  return out;
}

inline double replay_dense_shadow(const FactorChain& ch, const H2Matrix& A, Index guard = 200) {
  if (A.n() != ch.n) throw InvalidInputError("replay_dense_shadow: chain and matrix sizes differ");
  ReplayFactors f = replay_factors(ch, guard);
  Mat Z = A.dense_shadow();
  return (mul(f.L, f.U) - Z).norm() / Z.norm();
}

inline Vec dense_oracle_solve(const KernelSpec& K, const ClusterTree& T, const Vec& b, Index guard = 4096) {
  if (T.n() > guard) throw SizeGuardError("dense_oracle_solve: n = " + std::to_string(T.n()) + " exceeds the dense guard " + std::to_string(guard));
  if (static_cast<Index>(b.size()) != T.n()) throw InvalidInputError("dense_oracle_solve: right-hand side length does not match the tree");
  Mat Z = assemble_dense(K, T);
  Mat B(T.n(), 1);
  for (Index i = 0; i < T.n(); ++i) B(i, 0) = b[static_cast<size_t>(i)];
  Mat X = pivoted_lu_solve(Z, B);
  if (!X.all_finite()) throw NonFiniteError("dense_oracle_solve: solution contains non-finite entries");
  return Vec(X.d.begin(), X.d.end());
}

}  // namespace h2o
