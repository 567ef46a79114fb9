// ORACLE — TEST INFRASTRUCTURE ONLY (see dense.hpp header).
//
// Input stack of the reference restated: geometry + cluster tree
// (proj/include/h2lu/geometry.hpp, cluster_tree.hpp:71-118), block partition
// (block_tree.hpp:15-73), kernels (kernel.hpp:17-109, plus the complex
// diagonal the BASELINE VIE needs), and the algebraic H²
// construction (h2_matrix.hpp:29-375). Used to produce identical inputs for the
// oracle and the GPU path; construction is not on the hot path.
#pragma once

#include <array>
#include <map>
#include <memory>
#include <numeric>

#include <atomic>
#include <mutex>
#include <thread>

#include "dense.hpp"

namespace h2o {

// Deterministic parallel loop over independent items (no libgomp in this
// image): every item's arithmetic is identical to the serial loop.
template <class F>
inline void parallel_for(int64_t n, F&& f) {
  int nt = static_cast<int>(std::min<int64_t>(n, std::max(1u, std::thread::hardware_concurrency())));
  if (const char* e = std::getenv("H2O_THREADS")) nt = std::max(1, std::min(nt, std::atoi(e)));
  if (nt <= 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<int64_t> next{0};
  std::mutex mu;
  std::exception_ptr err;
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&] {
      for (int64_t i = next++; i < n; i = next++) {
        try {
          f(i);
        } catch (...) {
          std::lock_guard<std::mutex> g(mu);
          if (!err) err = std::current_exception();
        }
      }
    });
  for (auto& t : th) t.join();
  if (err) std::rethrow_exception(err);
}

using Vec3 = std::array<double, 3>;
using PointCloud = std::vector<Vec3>;

// ------------------------------------------------------------------ geometry
struct BoundingBox {
  Vec3 lo{0, 0, 0}, hi{0, 0, 0};
  double diameter() const {  // geometry.hpp:21
    const double x = hi[0] - lo[0], y = hi[1] - lo[1], z = hi[2] - lo[2];
    return std::sqrt(x * x + y * y + z * z);
  }
  int longest_axis() const {  // geometry.hpp:23-28
    const double e0 = hi[0] - lo[0], e1 = hi[1] - lo[1], e2 = hi[2] - lo[2];
    const double e[3] = {e0, e1, e2};
    int ax = 0;
    if (e[1] > e[0]) ax = 1;
    if (e[2] > e[ax]) ax = 2;
    return ax;
  }
};

inline double box_distance(const BoundingBox& a, const BoundingBox& b) {  // geometry.hpp:45-52
  double d2 = 0.0;
  for (int ax = 0; ax < 3; ++ax) {
    const double g = std::max({a.lo[ax] - b.hi[ax], b.lo[ax] - a.hi[ax], 0.0});
    d2 += g * g;
  }
  return std::sqrt(d2);
}

// --------------------------------------------------------------- cluster tree
struct Cluster {
  int id = -1, level = 0, parent = -1;
  int children[2] = {-1, -1};
  Index begin = 0, end = 0;
  BoundingBox bbox;
  Index size() const { return end - begin; }
  bool is_leaf() const { return children[0] < 0; }
};

// Heap-ordered uniform-depth binary tree (cluster_tree.hpp:31-118).
struct ClusterTree {
  PointCloud points;          // tree order
  std::vector<Index> perm;    // perm[tree index] = original index
  std::vector<Cluster> clusters;
  int depth = 0;
  Index leafsize = 0;
  Index n() const { return static_cast<Index>(points.size()); }
  const Cluster& cluster(int id) const { return clusters[static_cast<size_t>(id)]; }
  int num_clusters() const { return static_cast<int>(clusters.size()); }
  int level_begin(int l) const { return (1 << l) - 1; }
  int level_count(int l) const { return 1 << l; }
};

inline std::shared_ptr<const ClusterTree> build_cluster_tree(const PointCloud& pts, Index leafsize) {
  if (pts.empty()) throw InvalidInputError("build_cluster_tree: empty point cloud");
  if (leafsize < 1) throw InvalidInputError("build_cluster_tree: leafsize must be >= 1");
  auto T = std::make_shared<ClusterTree>();
  const Index n = static_cast<Index>(pts.size());
  int depth = 0;
  while ((n + (Index(1) << depth) - 1) / (Index(1) << depth) > leafsize) ++depth;
  T->depth = depth;
  T->leafsize = leafsize;
  T->perm.resize(static_cast<size_t>(n));
  std::iota(T->perm.begin(), T->perm.end(), Index(0));
  T->clusters.resize(static_cast<size_t>((2 << depth) - 1));
  auto& perm = T->perm;
  struct Item {
    int id, level;
    Index b, e;
  };
  std::vector<Item> stack{{0, 0, 0, n}};
  while (!stack.empty()) {
    const Item it = stack.back();
    stack.pop_back();
    Cluster& c = T->clusters[static_cast<size_t>(it.id)];
    c.id = it.id;
    c.level = it.level;
    c.parent = it.id == 0 ? -1 : (it.id - 1) / 2;
    c.begin = it.b;
    c.end = it.e;
    if (it.b < it.e) {
      c.bbox.lo = c.bbox.hi = pts[static_cast<size_t>(perm[static_cast<size_t>(it.b)])];
      for (Index i = it.b + 1; i < it.e; ++i) {
        const Vec3& p = pts[static_cast<size_t>(perm[static_cast<size_t>(i)])];
        for (int a = 0; a < 3; ++a) {
          c.bbox.lo[a] = std::min(c.bbox.lo[a], p[a]);
          c.bbox.hi[a] = std::max(c.bbox.hi[a], p[a]);
        }
      }
    }
    if (it.level == depth) continue;
    const int ax = c.bbox.longest_axis();
    const Index mid = it.b + (it.e - it.b + 1) / 2;
    std::nth_element(perm.begin() + it.b, perm.begin() + mid, perm.begin() + it.e, [&](Index a, Index b) {
      const double ca = pts[static_cast<size_t>(a)][ax], cb = pts[static_cast<size_t>(b)][ax];
      return ca < cb || (ca == cb && a < b);
    });
    c.children[0] = 2 * it.id + 1;
    c.children[1] = 2 * it.id + 2;
    stack.push_back({c.children[0], it.level + 1, it.b, mid});
    stack.push_back({c.children[1], it.level + 1, mid, it.e});
  }
  T->points.resize(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i) T->points[static_cast<size_t>(i)] = pts[static_cast<size_t>(perm[static_cast<size_t>(i)])];
  return T;
}

// ------------------------------------------------------------- block tree
struct BlockPair {
  int row = -1, col = -1;
};
inline bool pair_less(const BlockPair& a, const BlockPair& b) { return a.row < b.row || (a.row == b.row && a.col < b.col); }

inline bool is_admissible(const Cluster& t, const Cluster& s, double eta) {  // block_tree.hpp:15-18
  const double diam = std::max(t.bbox.diameter(), s.bbox.diameter());
  return diam < eta * box_distance(t.bbox, s.bbox);
}

struct BlockClusterTree {
  std::shared_ptr<const ClusterTree> tree;
  double eta = 1.0;
  std::vector<std::vector<BlockPair>> admissible, split;
  std::vector<BlockPair> inadmissible_leaf;
  std::vector<int> csp_level;
  int l0 = -1;
  int csp(int l) const { return csp_level[static_cast<size_t>(l)]; }
  int csp_max() const { return csp_level.empty() ? 0 : *std::max_element(csp_level.begin(), csp_level.end()); }
};

inline std::shared_ptr<const BlockClusterTree> build_block_tree(std::shared_ptr<const ClusterTree> tree, double eta) {
  if (eta <= 0.0) throw InvalidInputError("build_block_tree: eta must be positive");
  auto B = std::make_shared<BlockClusterTree>();
  B->tree = tree;
  B->eta = eta;
  const int depth = tree->depth;
  B->admissible.resize(static_cast<size_t>(depth) + 1);
  B->split.resize(static_cast<size_t>(depth) + 1);
  std::vector<BlockPair> stack{{0, 0}};
  while (!stack.empty()) {
    const BlockPair p = stack.back();
    stack.pop_back();
    const Cluster& t = tree->cluster(p.row);
    const Cluster& s = tree->cluster(p.col);
    if (is_admissible(t, s, eta)) {
      B->admissible[static_cast<size_t>(t.level)].push_back(p);
    } else if (t.is_leaf()) {
      B->inadmissible_leaf.push_back(p);
    } else {
      B->split[static_cast<size_t>(t.level)].push_back(p);
      for (int a = 1; a >= 0; --a)
        for (int b = 1; b >= 0; --b) stack.push_back({t.children[a], s.children[b]});
    }
  }
  for (auto& v : B->admissible) std::sort(v.begin(), v.end(), pair_less);
  for (auto& v : B->split) std::sort(v.begin(), v.end(), pair_less);
  std::sort(B->inadmissible_leaf.begin(), B->inadmissible_leaf.end(), pair_less);
  for (int l = 0; l <= depth; ++l)
    if (!B->admissible[static_cast<size_t>(l)].empty()) {
      B->l0 = l;
      break;
    }
  B->csp_level.assign(static_cast<size_t>(depth) + 1, 0);
  for (int l = 0; l <= depth; ++l) {
    std::map<int, int> per_row;
    for (const auto& p : B->admissible[static_cast<size_t>(l)]) ++per_row[p.row];
    for (const auto& p : B->split[static_cast<size_t>(l)]) ++per_row[p.row];
    if (l == depth)
      for (const auto& p : B->inadmissible_leaf) ++per_row[p.row];
    for (const auto& kv : per_row) B->csp_level[static_cast<size_t>(l)] = std::max(B->csp_level[static_cast<size_t>(l)], kv.second);
  }
  return B;
}

inline bool contains_pair(const std::vector<BlockPair>& v, int r, int c) {  // factorization.hpp:102-107
  auto it = std::lower_bound(v.begin(), v.end(), BlockPair{r, c}, pair_less);
  return it != v.end() && it->row == r && it->col == c;
}

// ---------------------------------------------------------------- kernels
// kernel.hpp:13-61, with the diagonal widened to complex:
//   off-diagonal = scale * f(r), f = 1/(4 pi r) (laplace) or
//   exp(-i k r)/(4 pi r) (helmholtz); diagonal (same index) = diag.
// kind "zero" is the reference's custom kernel returning 0.
enum KernelKind { KERNEL_LAPLACE = 0, KERNEL_HELMHOLTZ = 1, KERNEL_ZERO = 2 };

struct KernelSpec {
  int kind = KERNEL_LAPLACE;
  cxd wavenumber = 0.0;
  cxd scale = 1.0;
  cxd diag = 1.0;
  cxd entry(const Vec3& a, const Vec3& b) const {
    const double x = a[0] - b[0], y = a[1] - b[1], z = a[2] - b[2];
    const double r = std::sqrt(x * x + y * y + z * z);
    cxd v;
    switch (kind) {
      case KERNEL_LAPLACE:
        v = cxd(1.0 / (4.0 * M_PI * r), 0.0);
        break;
      case KERNEL_HELMHOLTZ:
        v = std::exp(cxd(0.0, -1.0) * wavenumber * r) / (4.0 * M_PI * r);
        break;
      default:
        return cxd(0.0, 0.0);
    }
    if (scale == cxd(1.0)) return v;
    return scale * v;
  }
};

// assemble_block (kernel.hpp:64-102) for index lists in tree order.
inline Mat assemble(const KernelSpec& K, const ClusterTree& T, const std::vector<Index>& rows, const std::vector<Index>& cols) {
  Mat Z(static_cast<Index>(rows.size()), static_cast<Index>(cols.size()));
  for (size_t j = 0; j < cols.size(); ++j) {
    const Index cj = cols[j];
    const Vec3& pn = T.points[static_cast<size_t>(cj)];
    for (size_t i = 0; i < rows.size(); ++i) {
      const Index ri = rows[i];
      const cxd v = ri == cj ? K.diag : K.entry(T.points[static_cast<size_t>(ri)], pn);
      if (!std::isfinite(v.real()) || !std::isfinite(v.imag()))
        throw NonFiniteError("kernel entry (" + std::to_string(ri) + "," + std::to_string(cj) + ") is not finite");
      Z(static_cast<Index>(i), static_cast<Index>(j)) = v;
    }
  }
  return Z;
}

inline std::vector<Index> range_idx(Index b, Index e) {
  std::vector<Index> v(static_cast<size_t>(e - b));
  std::iota(v.begin(), v.end(), b);
  return v;
}

inline Mat assemble_dense(const KernelSpec& K, const ClusterTree& T, Index guard = 20000) {
  if (T.n() > guard) throw SizeGuardError("assemble_dense: n=" + std::to_string(T.n()) + " exceeds guard " + std::to_string(guard));
  auto all = range_idx(0, T.n());
  return assemble(K, T, all, all);
}

// ---------------------------------------------------------------- H² matrix
struct H2Matrix {
  std::shared_ptr<const ClusterTree> tree;
  std::shared_ptr<const BlockClusterTree> blocks;
  double eps_h2 = 0.0;
  std::vector<Mat> bases;                 // by cluster id
  std::vector<std::vector<Mat>> couplings;  // [level][idx] aligned with admissible(level)
  std::vector<Mat> dense_blocks;          // aligned with inadmissible_leaf
  Index shadow_guard = 4000;

  Index n() const { return tree->n(); }
  int depth() const { return tree->depth; }
  Index rank(int id) const { return bases[static_cast<size_t>(id)].c; }

  Mat expand_basis(int id) const {  // h2_matrix.hpp:44-56
    const Cluster& c = tree->cluster(id);
    if (c.is_leaf()) return bases[static_cast<size_t>(id)];
    Mat E1 = expand_basis(c.children[0]), E2 = expand_basis(c.children[1]);
    const Mat& T = bases[static_cast<size_t>(id)];
    if (T.r != E1.c + E2.c) throw InvalidInputError("expand_basis: transfer rows do not match child ranks");
    Mat E(c.size(), T.c);
    E.set_block(0, 0, mul(E1, T.top_rows(E1.c)));
    E.set_block(E1.r, 0, mul(E2, T.bottom_rows(E2.c)));
    return E;
  }

  // h2_matrix.hpp:80-137 (upward transpose, couplings, downward, dense).
  std::vector<cxd> matvec(const std::vector<cxd>& x) const {
    if (static_cast<Index>(x.size()) != n()) throw InvalidInputError("matvec: dimension mismatch");
    const int L = depth();
    const int nc = tree->num_clusters();
    std::vector<std::vector<cxd>> xh(static_cast<size_t>(nc)), yh(static_cast<size_t>(nc));
    for (int l = L; l >= 0; --l) {
      for (int id = tree->level_begin(l); id < tree->level_begin(l) + tree->level_count(l); ++id) {
        const Cluster& c = tree->cluster(id);
        const Mat& B = bases[static_cast<size_t>(id)];
        std::vector<cxd> in;
        if (c.is_leaf()) {
          in.assign(x.begin() + c.begin, x.begin() + c.end);
        } else {
          in = xh[static_cast<size_t>(c.children[0])];
          const auto& x2 = xh[static_cast<size_t>(c.children[1])];
          in.insert(in.end(), x2.begin(), x2.end());
        }
        std::vector<cxd> out(static_cast<size_t>(B.c), 0.0);
        for (Index j = 0; j < B.c; ++j) {
          cxd s = 0.0;
          for (Index i = 0; i < B.r; ++i) s += B(i, j) * in[static_cast<size_t>(i)];
          out[static_cast<size_t>(j)] = s;
        }
        xh[static_cast<size_t>(id)] = std::move(out);
        yh[static_cast<size_t>(id)].assign(static_cast<size_t>(B.c), 0.0);
      }
    }
    for (int l = 0; l <= L; ++l) {
      const auto& adm = blocks->admissible[static_cast<size_t>(l)];
      for (size_t q = 0; q < adm.size(); ++q) {
        const Mat& S = couplings[static_cast<size_t>(l)][q];
        auto& y = yh[static_cast<size_t>(adm[q].row)];
        const auto& xx = xh[static_cast<size_t>(adm[q].col)];
        for (Index j = 0; j < S.c; ++j)
          for (Index i = 0; i < S.r; ++i) y[static_cast<size_t>(i)] += S(i, j) * xx[static_cast<size_t>(j)];
      }
    }
    std::vector<cxd> y(static_cast<size_t>(n()), 0.0);
    for (int l = 0; l <= L; ++l) {
      for (int id = tree->level_begin(l); id < tree->level_begin(l) + tree->level_count(l); ++id) {
        const Cluster& c = tree->cluster(id);
        const Mat& B = bases[static_cast<size_t>(id)];
        const auto& yv = yh[static_cast<size_t>(id)];
        if (yv.empty()) continue;
        std::vector<cxd> pushed(static_cast<size_t>(B.r), 0.0);
        for (Index j = 0; j < B.c; ++j)
          for (Index i = 0; i < B.r; ++i) pushed[static_cast<size_t>(i)] += B(i, j) * yv[static_cast<size_t>(j)];
        if (c.is_leaf()) {
          for (Index i = 0; i < B.r; ++i) y[static_cast<size_t>(c.begin + i)] += pushed[static_cast<size_t>(i)];
        } else {
          const Index k1 = rank(c.children[0]);
          auto& y1 = yh[static_cast<size_t>(c.children[0])];
          auto& y2 = yh[static_cast<size_t>(c.children[1])];
          for (Index i = 0; i < k1; ++i) y1[static_cast<size_t>(i)] += pushed[static_cast<size_t>(i)];
          for (Index i = k1; i < B.r; ++i) y2[static_cast<size_t>(i - k1)] += pushed[static_cast<size_t>(i)];
        }
      }
    }
    const auto& inadm = blocks->inadmissible_leaf;
    for (size_t q = 0; q < inadm.size(); ++q) {
      const Cluster& t = tree->cluster(inadm[q].row);
      const Cluster& s = tree->cluster(inadm[q].col);
      const Mat& D = dense_blocks[q];
      for (Index j = 0; j < D.c; ++j)
        for (Index i = 0; i < D.r; ++i) y[static_cast<size_t>(t.begin + i)] += D(i, j) * x[static_cast<size_t>(s.begin + j)];
    }
    return y;
  }

  Mat dense_shadow() const {  // h2_matrix.hpp:140-160
    if (n() > shadow_guard) throw SizeGuardError("dense_shadow: n=" + std::to_string(n()) + " exceeds guard " + std::to_string(shadow_guard));
    Mat Z(n(), n());
    for (int l = 0; l <= depth(); ++l) {
      const auto& adm = blocks->admissible[static_cast<size_t>(l)];
      for (size_t q = 0; q < adm.size(); ++q) {
        const Cluster& t = tree->cluster(adm[q].row);
        const Cluster& s = tree->cluster(adm[q].col);
        Z.set_block(t.begin, s.begin, mul(mul(expand_basis(adm[q].row), couplings[static_cast<size_t>(l)][q]), expand_basis(adm[q].col).transpose()));
      }
    }
    for (size_t q = 0; q < blocks->inadmissible_leaf.size(); ++q) {
      const Cluster& t = tree->cluster(blocks->inadmissible_leaf[q].row);
      const Cluster& s = tree->cluster(blocks->inadmissible_leaf[q].col);
      Z.set_block(t.begin, s.begin, dense_blocks[q]);
    }
    return Z;
  }

  size_t storage_bytes() const {
    size_t b = 0;
    for (const auto& m : bases) b += 16 * static_cast<size_t>(m.size());
    for (const auto& lv : couplings)
      for (const auto& m : lv) b += 16 * static_cast<size_t>(m.size());
    for (const auto& m : dense_blocks) b += 16 * static_cast<size_t>(m.size());
    return b + 8 * tree->perm.size();
  }
};

// h2_matrix.hpp:274-292 — left singular vectors of a wide block, truncated at
// sigma_j <= max(eps*sigma_0, floor, 1e-300); QR of B^H first when f > m.
inline Mat truncated_row_basis(const Mat& B, double eps, double floor = 0.0) {
  const Index m = B.r, f = B.c;
  if (m == 0 || f == 0) return Mat(m, 0);
  Mat RH;  // R^H, m x min(m,f)
  if (f > m) {
    HouseholderQR qr(B.adjoint());
    RH = qr.matrix_r().adjoint();
  } else {
    RH = B;
  }
  SVDResult svd = jacobi_svd_left(RH);
  if (svd.sigma.empty() || svd.sigma[0] == 0.0) return Mat(m, 0);
  const double thr = std::max({eps * svd.sigma[0], floor, 1e-300});
  Index r = 0;
  while (r < static_cast<Index>(svd.sigma.size()) && svd.sigma[static_cast<size_t>(r)] > thr) ++r;
  return svd.U.left_cols(r);
}

namespace detail {

struct IndexRange {
  Index b, e;
};

inline void merge_ranges(std::vector<IndexRange>& v) {
  std::sort(v.begin(), v.end(), [](const IndexRange& a, const IndexRange& b) { return a.b < b.b; });
  std::vector<IndexRange> out;
  for (const auto& r : v) {
    if (!out.empty() && out.back().e >= r.b)
      out.back().e = std::max(out.back().e, r.e);
    else
      out.push_back(r);
  }
  v.swap(out);
}

inline std::vector<Index> flatten(const std::vector<IndexRange>& v) {
  std::vector<Index> idx;
  for (const auto& r : v)
    for (Index i = r.b; i < r.e; ++i) idx.push_back(i);
  return idx;
}

// V_c^H Z[c, cols] through the nested basis (h2_matrix.hpp:237-250).
inline Mat project_rows(const H2Matrix& A, const KernelSpec& K, int id, const std::vector<Index>& cols) {
  const Cluster& c = A.tree->cluster(id);
  const Mat& B = A.bases[static_cast<size_t>(id)];
  if (c.is_leaf()) return mul(B.adjoint(), assemble(K, *A.tree, range_idx(c.begin, c.end), cols));
  Mat P1 = project_rows(A, K, c.children[0], cols), P2 = project_rows(A, K, c.children[1], cols);
  Mat st(P1.r + P2.r, P1.c);
  st.set_block(0, 0, P1);
  st.set_block(P1.r, 0, P2);
  return mul(B.adjoint(), st);
}

// Z[rows, c] conj(V_c) through the nested basis (h2_matrix.hpp:254-267).
inline Mat project_cols(const H2Matrix& A, const KernelSpec& K, int id, const std::vector<Index>& rows) {
  const Cluster& c = A.tree->cluster(id);
  const Mat& B = A.bases[static_cast<size_t>(id)];
  if (c.is_leaf()) return mul(assemble(K, *A.tree, rows, range_idx(c.begin, c.end)), B.conjugate());
  Mat P1 = project_cols(A, K, c.children[0], rows), P2 = project_cols(A, K, c.children[1], rows);
  Mat cat(P1.r, P1.c + P2.c);
  cat.set_block(0, 0, P1);
  cat.set_block(0, P1.c, P2);
  return mul(cat, B.conjugate());
}

}  // namespace detail

// h2_matrix.hpp:300-375. Clusters of one level are independent, so they are
// built in parallel (OpenMP) without changing any arithmetic.
inline H2Matrix build_h2(const KernelSpec& K, std::shared_ptr<const BlockClusterTree> blocks, double eps_h2) {
  if (eps_h2 <= 0.0) throw InvalidInputError("build_h2: eps_h2 must be positive");
  H2Matrix A;
  A.blocks = blocks;
  A.tree = blocks->tree;
  A.eps_h2 = eps_h2;
  const ClusterTree& T = *A.tree;
  const int L = T.depth;
  A.bases.resize(static_cast<size_t>(T.num_clusters()));

  struct Far {
    std::vector<detail::IndexRange> cols, rows;
  };
  std::vector<Far> far(static_cast<size_t>(T.num_clusters()));
  for (int l = 0; l <= L; ++l) {
    for (int id = T.level_begin(l); id < T.level_begin(l) + T.level_count(l); ++id) {
      const Cluster& c = T.cluster(id);
      if (c.parent >= 0) far[static_cast<size_t>(id)] = far[static_cast<size_t>(c.parent)];
    }
    for (const auto& p : blocks->admissible[static_cast<size_t>(l)]) {
      const Cluster& t = T.cluster(p.row);
      const Cluster& s = T.cluster(p.col);
      far[static_cast<size_t>(p.row)].cols.push_back({s.begin, s.end});
      far[static_cast<size_t>(p.col)].rows.push_back({t.begin, t.end});
    }
  }
  for (auto& f : far) {
    detail::merge_ranges(f.cols);
    detail::merge_ranges(f.rows);
  }

  for (int l = L; l >= 0; --l) {
    const int lb = T.level_begin(l), lc = T.level_count(l);
    parallel_for(lc, [&](int64_t q) {
        const int id = lb + static_cast<int>(q);
        const Cluster& c = T.cluster(id);
        auto scols = detail::flatten(far[static_cast<size_t>(id)].cols);
        auto srows = detail::flatten(far[static_cast<size_t>(id)].rows);
        const Index local = c.is_leaf() ? c.size() : A.rank(c.children[0]) + A.rank(c.children[1]);
        if ((scols.empty() && srows.empty()) || local == 0) {
          A.bases[static_cast<size_t>(id)] = Mat(local, 0);
          return;
        }
        const Index nc = static_cast<Index>(scols.size()), nr = static_cast<Index>(srows.size());
        Mat B(local, nc + nr);
        if (c.is_leaf()) {
          auto own = range_idx(c.begin, c.end);
          B.set_block(0, 0, assemble(K, T, own, scols));
          B.set_block(0, nc, assemble(K, T, srows, own).transpose());
        } else {
          const Index k1 = A.rank(c.children[0]);
          B.set_block(0, 0, detail::project_rows(A, K, c.children[0], scols));
          B.set_block(k1, 0, detail::project_rows(A, K, c.children[1], scols));
          B.set_block(0, nc, detail::project_cols(A, K, c.children[0], srows).transpose());
          B.set_block(k1, nc, detail::project_cols(A, K, c.children[1], srows).transpose());
        }
        A.bases[static_cast<size_t>(id)] = truncated_row_basis(B, eps_h2);
    });
  }

  A.couplings.resize(static_cast<size_t>(L) + 1);
  for (int l = 0; l <= L; ++l) {
    const auto& adm = blocks->admissible[static_cast<size_t>(l)];
    A.couplings[static_cast<size_t>(l)].resize(adm.size());
    parallel_for(static_cast<int64_t>(adm.size()), [&](int64_t q) {
      const Cluster& s = T.cluster(adm[static_cast<size_t>(q)].col);
      Mat P = detail::project_rows(A, K, adm[static_cast<size_t>(q)].row, range_idx(s.begin, s.end));
      A.couplings[static_cast<size_t>(l)][static_cast<size_t>(q)] = mul(P, A.expand_basis(adm[static_cast<size_t>(q)].col).conjugate());
    });
  }
  const auto& inadm = blocks->inadmissible_leaf;
  A.dense_blocks.resize(inadm.size());
  parallel_for(static_cast<int64_t>(inadm.size()), [&](int64_t q) {
    const Cluster& t = T.cluster(inadm[static_cast<size_t>(q)].row);
    const Cluster& s = T.cluster(inadm[static_cast<size_t>(q)].col);
    A.dense_blocks[static_cast<size_t>(q)] = assemble(K, T, range_idx(t.begin, t.end), range_idx(s.begin, s.end));
  });
  return A;
}

}  // namespace h2o
