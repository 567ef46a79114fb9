// ORACLE — TEST INFRASTRUCTURE ONLY (see dense.hpp header).
//
// Restatement of the reference's H2LU v1 container for the oracle's types
// (proj/include/h2lu/serialize.hpp:27-353): header "H2LU" / version 1 /
// kind, little-endian raw fields, column-major complex128 matrices, trees as
// permutation + tree-order points + heap-order ranges with the partition
// recomputed on load (:204-206). Used by tests to exchange matrices and
// chains with the GPU path's writer / reader.
#pragma once

#include <cstdio>
#include <string>

#include "factor.hpp"

namespace h2o {
namespace ser {

constexpr uint32_t kMagic = 0x554C3248, kVersion = 1, kKindH2 = 1, kKindChain = 2, kKindVector = 3;
constexpr int64_t kGuard = int64_t(1) << 27;

struct SerializationError : std::runtime_error {
  explicit SerializationError(const std::string& m) : std::runtime_error("serialize: " + m) {}
};

struct W {
  std::FILE* f;
  explicit W(const std::string& p) : f(std::fopen(p.c_str(), "wb")) {
    if (!f) throw SerializationError("cannot open " + p + " for writing");
  }
  ~W() {
    if (f) std::fclose(f);
  }
  void raw(const void* p, size_t n) {
    if (n && std::fwrite(p, 1, n, f) != n) throw SerializationError("write failed");
  }
  template <class T>
  void v(T x) {
    raw(&x, sizeof x);
  }
  void mat(const Mat& m) {
    v<int64_t>(m.r);
    v<int64_t>(m.c);
    raw(m.d.data(), m.d.size() * sizeof(cxd));
  }
  void idx(const std::vector<Index>& a) {
    v<int64_t>(static_cast<int64_t>(a.size()));
    for (Index x : a) v<int64_t>(x);
  }
  void head(uint32_t kind) {
    v<uint32_t>(kMagic);
    v<uint32_t>(kVersion);
    v<uint32_t>(kind);
  }
  void tree(const ClusterTree& t) {  // serialize.hpp:121-132
    v<int64_t>(t.n());
    v<int32_t>(t.depth);
    v<int64_t>(t.leafsize);
    idx(t.perm);
    for (const Vec3& p : t.points)
      for (int a = 0; a < 3; ++a) v<double>(p[a]);
    for (const Cluster& c : t.clusters) v<int64_t>(c.begin), v<int64_t>(c.end);
  }
};

struct R {
  std::FILE* f;
  explicit R(const std::string& p) : f(std::fopen(p.c_str(), "rb")) {
    if (!f) throw SerializationError("cannot open " + p);
  }
  ~R() {
    if (f) std::fclose(f);
  }
  void raw(void* p, size_t n) {
    if (n && std::fread(p, 1, n, f) != n) throw SerializationError("truncated input");
  }
  template <class T>
  T v() {
    T x;
    raw(&x, sizeof x);
    return x;
  }
  int64_t count(const char* what) {
    const int64_t x = v<int64_t>();
    if (x < 0 || x > kGuard) throw SerializationError(std::string("implausible ") + what);
    return x;
  }
  Mat mat() {
    const int64_t r = count("matrix rows"), c = count("matrix cols");
    if (r > 0 && c > kGuard / r) throw SerializationError("implausible matrix size");
    Mat m(r, c);
    raw(m.d.data(), m.d.size() * sizeof(cxd));
    return m;
  }
  std::vector<Index> idx() {
    std::vector<Index> a(static_cast<size_t>(count("index vector length")));
    for (auto& x : a) x = v<int64_t>();
    return a;
  }
  void head(uint32_t kind) {
    if (v<uint32_t>() != kMagic) throw SerializationError("bad magic, not an h2lu file");
    const uint32_t ver = v<uint32_t>();
    if (ver != kVersion) throw SerializationError("unsupported version " + std::to_string(ver));
    const uint32_t k = v<uint32_t>();
    if (k != kind) throw SerializationError("file holds payload kind " + std::to_string(k) + ", expected " + std::to_string(kind));
  }
  std::shared_ptr<const ClusterTree> tree() {  // serialize.hpp:134-182
    auto T = std::make_shared<ClusterTree>();
    const Index n = count("point count");
    T->depth = v<int32_t>();
    T->leafsize = count("leafsize");
    if (n < 1 || T->leafsize < 1 || T->depth < 0 || T->depth > 48) throw SerializationError("malformed tree header");
    T->perm = idx();
    if (static_cast<Index>(T->perm.size()) != n) throw SerializationError("permutation length mismatch");
    std::vector<char> seen(static_cast<size_t>(n), 0);
    for (Index p : T->perm) {
      if (p < 0 || p >= n || seen[static_cast<size_t>(p)]) throw SerializationError("perm is not a permutation");
      seen[static_cast<size_t>(p)] = 1;
    }
    T->points.resize(static_cast<size_t>(n));
    for (auto& p : T->points)
      for (int a = 0; a < 3; ++a) p[a] = v<double>();
    const int nc = (2 << T->depth) - 1;
    T->clusters.resize(static_cast<size_t>(nc));
    int level = 0;
    for (int id = 0; id < nc; ++id) {
      if (id >= (2 << level) - 1) ++level;
      Cluster& c = T->clusters[static_cast<size_t>(id)];
      c.id = id;
      c.level = level;
      c.parent = id == 0 ? -1 : (id - 1) / 2;
      if (level < T->depth) c.children[0] = 2 * id + 1, c.children[1] = 2 * id + 2;
      c.begin = v<int64_t>();
      c.end = v<int64_t>();
      if (c.begin < 0 || c.begin > c.end || c.end > n) throw SerializationError("cluster range out of bounds");
      if (c.begin < c.end) {
        c.bbox.lo = c.bbox.hi = T->points[static_cast<size_t>(c.begin)];
        for (Index i = c.begin + 1; i < c.end; ++i)
          for (int a = 0; a < 3; ++a) {
            c.bbox.lo[a] = std::min(c.bbox.lo[a], T->points[static_cast<size_t>(i)][a]);
            c.bbox.hi[a] = std::max(c.bbox.hi[a], T->points[static_cast<size_t>(i)][a]);
          }
      }
    }
    if (T->clusters[0].begin != 0 || T->clusters[0].end != n) throw SerializationError("root range mismatch");
    for (const Cluster& c : T->clusters)
      if (!c.is_leaf()) {
        const Cluster& a = T->clusters[static_cast<size_t>(c.children[0])];
        const Cluster& b = T->clusters[static_cast<size_t>(c.children[1])];
        if (a.begin != c.begin || a.end != b.begin || b.end != c.end) throw SerializationError("children do not partition their parent");
      }
    return T;
  }
};

inline void save_h2(const std::string& path, const H2Matrix& A) {  // :186-196
  W w(path);
  w.head(kKindH2);
  w.tree(*A.tree);
  w.v<double>(A.blocks->eta);
  w.v<double>(A.eps_h2);
  w.v<int64_t>(A.shadow_guard);
  for (const Mat& b : A.bases) w.mat(b);
  for (const auto& lv : A.couplings)
    for (const Mat& S : lv) w.mat(S);
  for (const Mat& D : A.dense_blocks) w.mat(D);
}

inline H2Matrix load_h2(const std::string& path) {  // :198-243
  R r(path);
  r.head(kKindH2);
  H2Matrix A;
  A.tree = r.tree();
  const double eta = r.v<double>();
  if (!(eta > 0.0)) throw SerializationError("eta must be positive");
  A.blocks = build_block_tree(A.tree, eta);
  A.eps_h2 = r.v<double>();
  A.shadow_guard = r.count("shadow guard");
  const ClusterTree& T = *A.tree;
  A.bases.resize(static_cast<size_t>(T.num_clusters()));
  for (auto& b : A.bases) b = r.mat();
  for (int id = 0; id < T.num_clusters(); ++id) {
    const Cluster& c = T.cluster(id);
    const Index expect = c.is_leaf() ? c.size() : A.bases[static_cast<size_t>(c.children[0])].c + A.bases[static_cast<size_t>(c.children[1])].c;
    if (A.bases[static_cast<size_t>(id)].r != expect) throw SerializationError("basis rows inconsistent with tree");
  }
  A.couplings.resize(static_cast<size_t>(T.depth) + 1);
  for (int l = 0; l <= T.depth; ++l)
    for (const BlockPair& p : A.blocks->admissible[static_cast<size_t>(l)]) {
      Mat S = r.mat();
      if (S.r != A.rank(p.row) || S.c != A.rank(p.col)) throw SerializationError("coupling dims inconsistent with basis ranks");
      A.couplings[static_cast<size_t>(l)].push_back(std::move(S));
    }
  for (const BlockPair& p : A.blocks->inadmissible_leaf) {
    Mat D = r.mat();
    if (D.r != T.cluster(p.row).size() || D.c != T.cluster(p.col).size()) throw SerializationError("dense block dims inconsistent with tree");
    A.dense_blocks.push_back(std::move(D));
  }
  return A;
}

inline void save_chain(const std::string& path, const FactorChain& ch) {  // :245-284
  W w(path);
  w.head(kKindChain);
  w.tree(*ch.tree);
  w.v<int64_t>(ch.n);
  w.v<int32_t>(ch.stop_level);
  w.v<double>(ch.eps_fill_in);
  w.v<int64_t>(static_cast<int64_t>(ch.levels.size()));
  for (const LevelBlock& lb : ch.levels) {
    w.v<int32_t>(lb.level);
    w.v<int64_t>(static_cast<int64_t>(lb.recs.size()));
    for (const EliminationRecord& r : lb.recs) {
      w.v<int32_t>(r.cluster);
      w.v<int32_t>(r.level);
      for (Index f : {r.pos, r.bsize, r.eliminated, r.rank_before, r.rank_after, r.fill_targets}) w.v<int64_t>(f);
      w.mat(r.Qtilde);
      w.mat(r.L11);
      w.mat(r.U11);
      for (const auto* side : {&r.Lbar, &r.Ubar}) {
        w.v<int64_t>(static_cast<int64_t>(side->size()));
        for (const auto& b : *side) w.v<int64_t>(b.pos), w.mat(b.M);
      }
    }
    w.v<int32_t>(lb.perm.level);
    w.idx(lb.perm.src);
    w.v<int64_t>(lb.perm.active_after);
    w.v<int32_t>(lb.diag.level);
    for (Index f : {lb.diag.rank_sum_before, lb.diag.rank_sum_after, lb.diag.eliminated, lb.diag.ledger_blocks}) w.v<int64_t>(f);
    w.v<uint64_t>(lb.diag.chain_bytes);
  }
  w.mat(ch.root_l);
  w.mat(ch.root_u);
  w.v<int64_t>(ch.root_size);
}

inline FactorChain load_chain(const std::string& path) {  // :286-343
  R r(path);
  r.head(kKindChain);
  FactorChain ch;
  ch.tree = r.tree();
  ch.n = r.count("matrix size");
  if (ch.n != ch.tree->n()) throw SerializationError("chain size disagrees with its tree");
  ch.stop_level = r.v<int32_t>();
  ch.eps_fill_in = r.v<double>();
  const int64_t nl = r.count("level count");
  if (nl > ch.tree->depth + 1) throw SerializationError("more level blocks than tree levels");
  ch.levels.resize(static_cast<size_t>(nl));
  for (auto& lb : ch.levels) {
    lb.level = r.v<int32_t>();
    lb.recs.resize(static_cast<size_t>(r.count("record count")));
    for (auto& e : lb.recs) {
      e.cluster = r.v<int32_t>();
      e.level = r.v<int32_t>();
      for (Index* f : {&e.pos, &e.bsize, &e.eliminated, &e.rank_before, &e.rank_after, &e.fill_targets}) *f = r.v<int64_t>();
      e.Qtilde = r.mat();
      e.L11 = r.mat();
      e.U11 = r.mat();
      if (e.Qtilde.r != e.Qtilde.c || e.Qtilde.r != e.bsize || e.L11.r != e.eliminated || e.L11.r != e.L11.c || e.U11.r != e.U11.c ||
          e.U11.r != e.eliminated || e.eliminated > e.bsize || e.eliminated < 0)
        throw SerializationError("elimination record dims inconsistent");
      for (auto* side : {&e.Lbar, &e.Ubar}) {
        side->resize(static_cast<size_t>(r.count("off-diagonal block count")));
        for (auto& b : *side) {
          b.pos = r.v<int64_t>();
          b.M = r.mat();
          if (b.pos < 0 || b.pos >= ch.n) throw SerializationError("off-diagonal block out of range");
        }
      }
    }
    lb.perm.level = r.v<int32_t>();
    lb.perm.src = r.idx();
    lb.perm.active_after = r.v<int64_t>();
    for (Index s : lb.perm.src)
      if (s < 0 || s >= static_cast<Index>(lb.perm.src.size())) throw SerializationError("permutation entry out of range");
    lb.diag.level = r.v<int32_t>();
    for (Index* f : {&lb.diag.rank_sum_before, &lb.diag.rank_sum_after, &lb.diag.eliminated, &lb.diag.ledger_blocks}) *f = r.v<int64_t>();
    lb.diag.chain_bytes = r.v<uint64_t>();
  }
  ch.root_l = r.mat();
  ch.root_u = r.mat();
  ch.root_size = r.count("root size");
  if (ch.root_l.r != ch.root_size || ch.root_l.c != ch.root_size || ch.root_u.r != ch.root_size || ch.root_u.c != ch.root_size)
    throw SerializationError("root factor dims inconsistent");
  return ch;
}

inline void save_vector(const std::string& path, const std::vector<cxd>& x) {
  W w(path);
  w.head(kKindVector);
  w.v<int64_t>(static_cast<int64_t>(x.size()));
  w.raw(x.data(), x.size() * sizeof(cxd));
}

inline std::vector<cxd> load_vector(const std::string& path) {
  R r(path);
  r.head(kKindVector);
  std::vector<cxd> x(static_cast<size_t>(r.count("vector length")));
  r.raw(x.data(), x.size() * sizeof(cxd));
  return x;
}

}  // namespace ser
}  // namespace h2o
