// Host symbolic analysis, see plan.hpp.
#include "plan.hpp"

#include <climits>
#include <mutex>
#include <thread>
#include <cstdlib>
#include <map>

#include <algorithm>
#include <cmath>
#include <complex>
#include <random>
#include <numeric>
#include <stdexcept>

#include "../../include/h2g.h"

namespace h2g {

namespace {
bool pair_less(const Pair& a, const Pair& b) { return a.row < b.row || (a.row == b.row && a.col < b.col); }
}  // namespace

Structure structure_from_desc(const h2g_matrix_desc* d) {
  if (!d || d->n <= 0 || d->depth < 0 || d->depth > 24) throw std::invalid_argument("matrix desc: bad n/depth");
  Structure S;
  S.n = d->n;
  S.depth = d->depth;
  S.eta = d->eta;
  const int nc = S.num_clusters();
  S.begin.assign(d->cluster_begin, d->cluster_begin + nc);
  S.end.assign(d->cluster_end, d->cluster_end + nc);
  S.adm.resize(static_cast<size_t>(S.depth) + 1);
  S.split.resize(static_cast<size_t>(S.depth) + 1);
  S.adm_offset.assign(static_cast<size_t>(S.depth) + 2, 0);
  for (int l = 0; l <= S.depth; ++l) {
    for (int64_t q = d->adm_offsets[l]; q < d->adm_offsets[l + 1]; ++q) S.adm[static_cast<size_t>(l)].push_back({d->adm_pairs[2 * q], d->adm_pairs[2 * q + 1]});
    for (int64_t q = d->split_offsets[l]; q < d->split_offsets[l + 1]; ++q)
      S.split[static_cast<size_t>(l)].push_back({d->split_pairs[2 * q], d->split_pairs[2 * q + 1]});
    S.adm_offset[static_cast<size_t>(l) + 1] = d->adm_offsets[l + 1];
    if (!std::is_sorted(S.adm[static_cast<size_t>(l)].begin(), S.adm[static_cast<size_t>(l)].end(), pair_less) ||
        !std::is_sorted(S.split[static_cast<size_t>(l)].begin(), S.split[static_cast<size_t>(l)].end(), pair_less))
      throw std::invalid_argument("matrix desc: block pairs must be sorted by (row, col)");
  }
  for (int64_t q = 0; q < d->num_leaf_pairs; ++q) S.leaf.push_back({d->leaf_pairs[2 * q], d->leaf_pairs[2 * q + 1]});
  if (!std::is_sorted(S.leaf.begin(), S.leaf.end(), pair_less)) throw std::invalid_argument("matrix desc: leaf pairs must be sorted");
  for (int l = 0; l <= S.depth; ++l)
    if (!S.adm[static_cast<size_t>(l)].empty()) {
      S.l0 = l;
      break;
    }
  return S;
}

// ---------------------------------------------------------------------------
// Host tree + partition (cluster_tree.hpp:71-118, block_tree.hpp:30-73),
// used by h2g_matrix_build. Same splitting rule and tie-break (longest bbox
// axis, median index, coordinate then original index), same strict
// admissibility diam < eta * dist.
namespace {
struct Box {
  double lo[3], hi[3];
  double diameter() const {
    const double x = hi[0] - lo[0], y = hi[1] - lo[1], z = hi[2] - lo[2];
    return std::sqrt(x * x + y * y + z * z);
  }
};
double box_distance(const Box& a, const Box& b) {
  double d2 = 0.0;
  for (int ax = 0; ax < 3; ++ax) {
    const double g = std::max({a.lo[ax] - b.hi[ax], b.lo[ax] - a.hi[ax], 0.0});
    d2 += g * g;
  }
  return std::sqrt(d2);
}
}  // namespace

static void partition(Structure& S, const std::vector<Box>& box);

Structure build_structure(const double* pts, int64_t n, int64_t leafsize, double eta, std::vector<int64_t>* perm_out) {
  if (n <= 0) throw std::invalid_argument("build: empty point cloud");
  if (leafsize < 1) throw std::invalid_argument("build: leafsize must be >= 1");
  if (eta <= 0.0) throw std::invalid_argument("build: eta must be positive");
  Structure S;
  S.n = n;
  S.eta = eta;
  int depth = 0;
  while ((n + (int64_t(1) << depth) - 1) / (int64_t(1) << depth) > leafsize) ++depth;
  S.depth = depth;
  const int nc = S.num_clusters();
  S.begin.assign(static_cast<size_t>(nc), 0);
  S.end.assign(static_cast<size_t>(nc), 0);
  std::vector<Box> box(static_cast<size_t>(nc));
  std::vector<int64_t> perm(static_cast<size_t>(n));
  std::iota(perm.begin(), perm.end(), int64_t(0));
  struct Item {
    int id, level;
    int64_t b, e;
  };
  std::vector<Item> stack{{0, 0, 0, n}};
  while (!stack.empty()) {
    const Item it = stack.back();
    stack.pop_back();
    S.begin[static_cast<size_t>(it.id)] = it.b;
    S.end[static_cast<size_t>(it.id)] = it.e;
    Box& bx = box[static_cast<size_t>(it.id)];
    for (int a = 0; a < 3; ++a) bx.lo[a] = bx.hi[a] = 0.0;
    if (it.b < it.e) {
      for (int a = 0; a < 3; ++a) bx.lo[a] = bx.hi[a] = pts[3 * perm[static_cast<size_t>(it.b)] + a];
      for (int64_t i = it.b + 1; i < it.e; ++i)
        for (int a = 0; a < 3; ++a) {
          const double v = pts[3 * perm[static_cast<size_t>(i)] + a];
          bx.lo[a] = std::min(bx.lo[a], v);
          bx.hi[a] = std::max(bx.hi[a], v);
        }
    }
    if (it.level == depth) continue;
    const double e0 = bx.hi[0] - bx.lo[0], e1 = bx.hi[1] - bx.lo[1], e2 = bx.hi[2] - bx.lo[2];
    const double ext[3] = {e0, e1, e2};
    int ax = 0;
    if (ext[1] > ext[0]) ax = 1;
    if (ext[2] > ext[ax]) ax = 2;
    const int64_t mid = it.b + (it.e - it.b + 1) / 2;
    std::nth_element(perm.begin() + it.b, perm.begin() + mid, perm.begin() + it.e, [&](int64_t a, int64_t b) {
      const double ca = pts[3 * a + ax], cb = pts[3 * b + ax];
      return ca < cb || (ca == cb && a < b);
    });
    stack.push_back({2 * it.id + 1, it.level + 1, it.b, mid});
    stack.push_back({2 * it.id + 2, it.level + 1, mid, it.e});
  }
  partition(S, box);
  if (perm_out) *perm_out = std::move(perm);
  return S;
}

// Block partition of an existing tree (block_tree.hpp:15-73): strict
// admissibility max(diam) < eta * dist on the cluster bounding boxes.
static void partition(Structure& S, const std::vector<Box>& box) {
  const int depth = S.depth;
  const double eta = S.eta;
  S.adm.assign(static_cast<size_t>(depth) + 1, {});
  S.split.assign(static_cast<size_t>(depth) + 1, {});
  S.leaf.clear();
  auto level_of = [](int id) {
    int l = 0;
    while ((2 << l) - 1 <= id) ++l;
    return l;
  };
  std::vector<Pair> st{{0, 0}};
  while (!st.empty()) {
    const Pair p = st.back();
    st.pop_back();
    const Box& t = box[static_cast<size_t>(p.row)];
    const Box& s = box[static_cast<size_t>(p.col)];
    const int lt = level_of(p.row);
    if (std::max(t.diameter(), s.diameter()) < eta * box_distance(t, s)) {
      S.adm[static_cast<size_t>(lt)].push_back(p);
    } else if (lt == depth) {
      S.leaf.push_back(p);
    } else {
      S.split[static_cast<size_t>(lt)].push_back(p);
      for (int a = 1; a >= 0; --a)
        for (int b = 1; b >= 0; --b) st.push_back({2 * p.row + 1 + a, 2 * p.col + 1 + b});
    }
  }
  for (auto& v : S.adm) std::sort(v.begin(), v.end(), pair_less);
  for (auto& v : S.split) std::sort(v.begin(), v.end(), pair_less);
  std::sort(S.leaf.begin(), S.leaf.end(), pair_less);
  S.adm_offset.assign(static_cast<size_t>(depth) + 2, 0);
  for (int l = 0; l <= depth; ++l) S.adm_offset[static_cast<size_t>(l) + 1] = S.adm_offset[static_cast<size_t>(l)] + static_cast<int64_t>(S.adm[static_cast<size_t>(l)].size());
  S.l0 = -1;
  for (int l = 0; l <= depth; ++l)
    if (!S.adm[static_cast<size_t>(l)].empty()) {
      S.l0 = l;
      break;
    }
}

// Tree given (loaded from an H2LU file: ranges + tree-order points), partition
// recomputed exactly as load_h2 does (serialize.hpp:204-206).
Structure structure_from_tree(const double* pts_tree, int64_t n, int depth, const std::vector<int64_t>& begin, const std::vector<int64_t>& end,
                              double eta) {
  Structure S;
  S.n = n;
  S.depth = depth;
  S.eta = eta;
  S.begin = begin;
  S.end = end;
  const int nc = S.num_clusters();
  if ((int)begin.size() != nc || (int)end.size() != nc) throw std::invalid_argument("structure_from_tree: range arrays do not match the depth");
  std::vector<Box> box(static_cast<size_t>(nc));
  for (int id = 0; id < nc; ++id) {
    Box& bx = box[static_cast<size_t>(id)];
    for (int a = 0; a < 3; ++a) bx.lo[a] = bx.hi[a] = 0.0;
    const int64_t b = begin[static_cast<size_t>(id)], e = end[static_cast<size_t>(id)];
    if (b >= e) continue;
    for (int a = 0; a < 3; ++a) bx.lo[a] = bx.hi[a] = pts_tree[3 * b + a];
    for (int64_t i = b + 1; i < e; ++i)
      for (int a = 0; a < 3; ++a) {
        bx.lo[a] = std::min(bx.lo[a], pts_tree[3 * i + a]);
        bx.hi[a] = std::max(bx.hi[a], pts_tree[3 * i + a]);
      }
  }
  partition(S, box);
  return S;
}

// ---------------------------------------------------------------------------
std::vector<LevelSym> build_levels(const Structure& S, int stop) {
  std::vector<LevelSym> out;
  const int last = std::max(stop - 1, 0);
  const int L = S.depth;
  const bool no_levels = stop > L;  // no admissible blocks: root = leaf level
  const int lowest = no_levels ? L : last;
  for (int l = L; l >= lowest; --l) {
    LevelSym Y;
    Y.level = l;
    Y.nl = 1 << l;
    Y.first = Structure::first(l);
    const int nl = Y.nl, first = Y.first;
    const bool processed = !no_levels && l >= stop;
    const std::vector<Pair>& dp = (l == L) ? S.leaf : S.split[static_cast<size_t>(l)];
    Y.diag_blk.assign(static_cast<size_t>(nl), -1);
    for (size_t q = 0; q < dp.size(); ++q) {
      const int r = dp[q].row - first, c = dp[q].col - first;
      if (r < 0 || r >= nl || c < 0 || c >= nl) throw std::invalid_argument("dense pair outside its level");
      Y.drow.push_back(r);
      Y.dcol.push_back(c);
      Y.dense_of[int64_t(r) * nl + c] = static_cast<int>(q);
      if (r == c) Y.diag_blk[static_cast<size_t>(r)] = static_cast<int>(q);
    }
    for (int t = 0; t < nl; ++t)
      if (Y.diag_blk[static_cast<size_t>(t)] < 0) throw std::invalid_argument("cluster without a dense diagonal block");
    // R / C entries
    std::vector<std::vector<std::pair<int, int>>> R(static_cast<size_t>(nl)), Cc(static_cast<size_t>(nl));
    for (size_t q = 0; q < Y.drow.size(); ++q) {
      const int r = Y.drow[q], c = Y.dcol[q];
      if (r == c) continue;
      Cc[static_cast<size_t>(r)].push_back({c, static_cast<int>(q)});
      R[static_cast<size_t>(c)].push_back({r, static_cast<int>(q)});
    }
    Y.R_ptr.assign(1, 0);
    Y.C_ptr.assign(1, 0);
    for (int t = 0; t < nl; ++t) {
      auto& rr = R[static_cast<size_t>(t)];
      std::sort(rr.begin(), rr.end());
      for (auto& e : rr) Y.R_nb.push_back(e.first), Y.R_blk.push_back(e.second);
      Y.R_ptr.push_back(static_cast<int>(Y.R_nb.size()));
      auto& cc = Cc[static_cast<size_t>(t)];
      std::sort(cc.begin(), cc.end());
      for (auto& e : cc) Y.C_nb.push_back(e.first), Y.C_blk.push_back(e.second);
      Y.C_ptr.push_back(static_cast<int>(Y.C_nb.size()));
    }
    // fill targets
    std::vector<int64_t> keys;
    if (processed) {
      // every (row, column) neighbour pair of a cluster that is not dense;
      // clusters split over host threads (read-only lookups), merged below
      const int nt = std::max(1, std::min<int>(static_cast<int>(std::thread::hardware_concurrency()), nl / 64));
      std::vector<std::vector<int64_t>> part(static_cast<size_t>(nt));
      auto work = [&](int w) {
        std::vector<int64_t>& out_keys = part[static_cast<size_t>(w)];
        for (int m = w; m < nl; m += nt)
          for (int a = Y.R_ptr[static_cast<size_t>(m)]; a < Y.R_ptr[static_cast<size_t>(m) + 1]; ++a)
            for (int b = Y.C_ptr[static_cast<size_t>(m)]; b < Y.C_ptr[static_cast<size_t>(m) + 1]; ++b) {
              const int j = Y.R_nb[static_cast<size_t>(a)], c = Y.C_nb[static_cast<size_t>(b)];
              if (Y.dense_index(j, c) < 0) out_keys.push_back(int64_t(j) * nl + c);
            }
        std::sort(out_keys.begin(), out_keys.end());
        out_keys.erase(std::unique(out_keys.begin(), out_keys.end()), out_keys.end());
      };
      std::vector<std::thread> th;
      for (int w = 1; w < nt; ++w) th.emplace_back(work, w);
      work(0);
      for (auto& t : th) t.join();
      for (auto& v : part) keys.insert(keys.end(), v.begin(), v.end());
    }
    if (!out.empty()) {
      const LevelSym& P = out.back();  // level l+1
      for (size_t f = 0; f < P.frow.size(); ++f)
        if (P.fadm[f] < 0) {
          const int pj = P.frow[f] / 2, pc = P.fcol[f] / 2;
          if (Y.dense_index(pj, pc) >= 0) throw std::invalid_argument("merge_permute: carried fill-in resurfaced on a dense block");
          keys.push_back(int64_t(pj) * nl + pc);
        }
    }
    std::sort(keys.begin(), keys.end());
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    const auto& adm = S.adm[static_cast<size_t>(l)];
    for (int64_t k : keys) {
      const int r = static_cast<int>(k / nl), c = static_cast<int>(k % nl);
      const Pair hp{r + first, c + first};
      auto it = std::lower_bound(adm.begin(), adm.end(), hp, pair_less);
      const int ai = (it != adm.end() && it->row == hp.row && it->col == hp.col) ? static_cast<int>(it - adm.begin()) : -1;
      Y.fill_of[k] = static_cast<int>(Y.frow.size());
      Y.frow.push_back(r);
      Y.fcol.push_back(c);
      Y.fadm.push_back(ai);
      if (ai >= 0) ++Y.nledger;
    }
    // parent links of level l+1 carried fills
    if (!out.empty()) {
      LevelSym& P = out.back();
      P.carried_parent.assign(P.frow.size(), -1);
      for (size_t f = 0; f < P.frow.size(); ++f)
        if (P.fadm[f] < 0) P.carried_parent[f] = Y.fill_index(P.frow[f] / 2, P.fcol[f] / 2);
    }
    // step-0 gather lists: ledger keys touching t in map order, then carried
    {
      std::vector<std::vector<int>> by_row(static_cast<size_t>(nl)), by_col(static_cast<size_t>(nl));
      for (size_t f = 0; f < Y.frow.size(); ++f) {
        by_row[static_cast<size_t>(Y.frow[f])].push_back(static_cast<int>(f));
        by_col[static_cast<size_t>(Y.fcol[f])].push_back(static_cast<int>(f));
      }
      Y.G_ptr.assign(1, 0);
      for (int t = 0; t < nl; ++t) {
        for (int kind = 0; kind < 2; ++kind) {
          auto want = [&](int f) { return (Y.fadm[static_cast<size_t>(f)] >= 0) == (kind == 0); };
          // (x, t), x < t
          for (int f : by_col[static_cast<size_t>(t)])
            if (want(f) && Y.frow[static_cast<size_t>(f)] < t) Y.G_fill.push_back(f), Y.G_tr.push_back(1);
          // (t, y)
          for (int f : by_row[static_cast<size_t>(t)])
            if (want(f)) Y.G_fill.push_back(f), Y.G_tr.push_back(0);
          // (x, t), x > t
          for (int f : by_col[static_cast<size_t>(t)])
            if (want(f) && Y.frow[static_cast<size_t>(f)] > t) Y.G_fill.push_back(f), Y.G_tr.push_back(1);
        }
        Y.G_ptr.push_back(static_cast<int>(Y.G_fill.size()));
      }
    }
    out.push_back(std::move(Y));
  }
  if (!out.empty()) out.back().carried_parent.assign(out.back().frow.size(), -1);
  return out;
}

LevelSchedule build_schedule(const LevelSym& L, int kind) {
  const int nl = L.nl;
  std::vector<std::vector<int>> nb(static_cast<size_t>(nl));
  for (size_t q = 0; q < L.drow.size(); ++q) {
    const int r = L.drow[q], c = L.dcol[q];
    if (r == c) continue;
    nb[static_cast<size_t>(r)].push_back(c);
    nb[static_cast<size_t>(c)].push_back(r);
  }
  std::vector<int> key(static_cast<size_t>(nl), 0);
  std::vector<int> part_batch(static_cast<size_t>(kInteriorParts) + 1, 0);
  if (kind == H2G_SCHEDULE_COLORED) {
    std::vector<int> mark(static_cast<size_t>(nl) + 1, -1);
    for (int t = 0; t < nl; ++t) {
      for (int x : nb[static_cast<size_t>(t)])
        if (x < t) mark[static_cast<size_t>(key[static_cast<size_t>(x)])] = t;
      int c = 0;
      while (mark[static_cast<size_t>(c)] == t) ++c;
      key[static_cast<size_t>(t)] = c;
    }
  } else if (kind == H2G_SCHEDULE_SERIAL) {
    for (int t = 0; t < nl; ++t) key[static_cast<size_t>(t)] = t;  // one cluster per batch, ascending id
  } else if (kind == H2G_SCHEDULE_INTERIOR_FIRST && nl >= kInteriorParts) {
    // the north_star's subtree split (SURVEY §8e option 2): the level-3
    // subtrees are the parts; clusters whose dense neighbours all lie in
    // their own part go first (ascending id), the boundary clusters after
    // them (ascending id); batches are the dependency wavefronts of that order
    int lp = 0;
    while ((1 << lp) < kInteriorParts) ++lp;
    const int shift = L.level - lp;
    std::vector<int> pos(static_cast<size_t>(nl));
    std::vector<int> order;
    std::vector<char> interior(static_cast<size_t>(nl), 1);
    for (int t = 0; t < nl; ++t)
      for (int x : nb[static_cast<size_t>(t)])
        if ((x >> shift) != (t >> shift)) interior[static_cast<size_t>(t)] = 0;
    for (int pass = 1; pass >= 0; --pass)
      for (int t = 0; t < nl; ++t)
        if (interior[static_cast<size_t>(t)] == pass) pos[static_cast<size_t>(t)] = static_cast<int>(order.size()), order.push_back(t);
    for (int t : order) {
      int w = 0;
      for (int x : nb[static_cast<size_t>(t)])
        if (pos[static_cast<size_t>(x)] < pos[static_cast<size_t>(t)]) w = std::max(w, key[static_cast<size_t>(x)] + 1);
      key[static_cast<size_t>(t)] = w;
    }
  } else if (kind == H2G_SCHEDULE_SUBTREE && nl >= kInteriorParts) {
    // the interior-first split with subtree-pure batches: the interior
    // clusters of subtree 0 (wavefronts of their ascending-id order), then
    // subtree 1's, ..., then the boundary clusters (wavefronts again)
    int lp = 0;
    while ((1 << lp) < kInteriorParts) ++lp;
    const int shift = L.level - lp;
    std::vector<char> interior(static_cast<size_t>(nl), 1);
    for (int t = 0; t < nl; ++t)
      for (int x : nb[static_cast<size_t>(t)])
        if ((x >> shift) != (t >> shift)) interior[static_cast<size_t>(t)] = 0;
    int base = 0;
    for (int s = 0; s <= kInteriorParts; ++s) {
      part_batch[static_cast<size_t>(s)] = base;
      int top = base;
      for (int t = 0; t < nl; ++t) {
        const bool mine = s < kInteriorParts ? (interior[static_cast<size_t>(t)] && (t >> shift) == s) : !interior[static_cast<size_t>(t)];
        if (!mine) continue;
        int w = base;
        // earlier members of the same group with a lower id (interior
        // clusters of other subtrees are never neighbours; for the boundary
        // group every interior neighbour lies in an earlier batch already)
        for (int x : nb[static_cast<size_t>(t)]) {
          const bool same = s < kInteriorParts ? (interior[static_cast<size_t>(x)] && (x >> shift) == s) : !interior[static_cast<size_t>(x)];
          if (same && x < t) w = std::max(w, key[static_cast<size_t>(x)] + 1);
        }
        key[static_cast<size_t>(t)] = w;
        top = std::max(top, w + 1);
      }
      base = top;
    }
  } else {
    // dependency wavefronts of the ascending-id order: every lower-id
    // neighbour completes before t starts, no higher-id neighbour does.
    for (int t = 0; t < nl; ++t) {
      int w = 0;
      for (int x : nb[static_cast<size_t>(t)])
        if (x < t) w = std::max(w, key[static_cast<size_t>(x)] + 1);
      key[static_cast<size_t>(t)] = w;
    }
  }
  const int nb_batches = nl ? *std::max_element(key.begin(), key.end()) + 1 : 0;
  LevelSchedule S;
  S.order = key;
  S.part_batch = part_batch;
  std::vector<std::vector<int>> bat(static_cast<size_t>(nb_batches));
  for (int t = 0; t < nl; ++t) bat[static_cast<size_t>(key[static_cast<size_t>(t)])].push_back(t);
  S.batch_ptr.assign(1, 0);
  for (auto& b : bat) {
    for (int t : b) S.batch_cl.push_back(t);
    S.batch_ptr.push_back(static_cast<int>(S.batch_cl.size()));
  }
  return S;
}

std::vector<PartList> build_parts(const LevelSym& L, const LevelSchedule& sch, const LevelWork& W) {
  std::vector<PartList> parts(static_cast<size_t>(kInteriorParts));
  if (sch.part_batch.size() != static_cast<size_t>(kInteriorParts) + 1) return parts;
  for (int sp = 0; sp < kInteriorParts; ++sp) {
    PartList& PL = parts[static_cast<size_t>(sp)];
    std::vector<char> dm(L.drow.size(), 0), fm(L.frow.size(), 0);
    for (int bi = sch.part_batch[static_cast<size_t>(sp)]; bi < sch.part_batch[static_cast<size_t>(sp) + 1]; ++bi) {
      for (int p = sch.batch_ptr[static_cast<size_t>(bi)]; p < sch.batch_ptr[static_cast<size_t>(bi) + 1]; ++p) {
        const int t = sch.batch_cl[static_cast<size_t>(p)];
        PL.cl.push_back(t);
        dm[static_cast<size_t>(L.diag_blk[static_cast<size_t>(t)])] = 1;
      }
      for (int it = W.panel_ptr[static_cast<size_t>(bi)]; it < W.panel_ptr[static_cast<size_t>(bi) + 1]; ++it)
        dm[static_cast<size_t>(W.panel[static_cast<size_t>(it)].blk)] = 1;
      for (int q = W.schur_ptr[static_cast<size_t>(bi)]; q < W.schur_ptr[static_cast<size_t>(bi) + 1]; ++q) {
        const SchurTarget& T = W.schur[static_cast<size_t>(q)];
        ((T.kind & 1) ? fm : dm)[static_cast<size_t>(T.idx)] = 1;
      }
    }
    for (size_t q = 0; q < dm.size(); ++q)
      if (dm[q]) PL.dblk.push_back(static_cast<int>(q));
    for (size_t q = 0; q < fm.size(); ++q)
      if (fm[q]) PL.fblk.push_back(static_cast<int>(q));
  }
  return parts;
}

int fill_segments(int nbat, int requested) { return std::max(1, std::min(requested, nbat)); }

namespace {

// Best-fit interval allocator over one contiguous pool (element units).
class FrontAllocator {
 public:
  long long alloc(long long n) {
    auto it = by_size_.lower_bound(n);
    if (it == by_size_.end()) {
      const long long o = top_;
      top_ += n;
      return o;
    }
    const long long o = it->second, sz = it->first;
    by_size_.erase(it);
    by_off_.erase(o);
    if (sz > n) insert(o + n, sz - n);
    return o;
  }
  void release(long long o, long long n) {
    // coalesce with the neighbours
    auto nx = by_off_.lower_bound(o);
    if (nx != by_off_.end() && nx->first == o + n) {
      n += nx->second;
      erase(nx->first, nx->second);
    }
    auto pv = by_off_.lower_bound(o);
    if (pv != by_off_.begin()) {
      --pv;
      if (pv->first + pv->second == o) {
        o = pv->first;
        n += pv->second;
        erase(pv->first, pv->second);
      }
    }
    if (o + n == top_) {
      top_ = o;  // give the tail back
      return;
    }
    insert(o, n);
  }
  long long high() const { return high_; }
  void note() { high_ = std::max(high_, top_); }

 private:
  void insert(long long o, long long n) {
    by_off_[o] = n;
    by_size_.emplace(n, o);
  }
  void erase(long long o, long long n) {
    by_off_.erase(o);
    auto r = by_size_.equal_range(n);
    for (auto it = r.first; it != r.second; ++it)
      if (it->second == o) {
        by_size_.erase(it);
        break;
      }
  }
  long long top_ = 0, high_ = 0;
  std::map<long long, long long> by_off_;
  std::multimap<long long, long long> by_size_;
};

}  // namespace

FrontPlan build_front(const LevelSym& L, const LevelSchedule& sch, const LevelWork& W, const std::vector<int>& bsz, const std::vector<int>& init) {
  FrontPlan F;
  const int nbat = static_cast<int>(sch.batch_ptr.size()) - 1;
  const int K = W.fill_segments;
  F.K = K;
  F.seg_first_batch.assign(static_cast<size_t>(K) + 1, nbat);
  for (int b = nbat - 1; b >= 0; --b) F.seg_first_batch[static_cast<size_t>(fill_segment(b, nbat, K))] = b;
  const size_t nf = L.frow.size();
  // first / last batch depositing into each fill block
  std::vector<int> fd(nf, INT32_MAX), ld(nf, -1);
  for (int b = 0; b < nbat; ++b)
    for (int q = W.schur_ptr[static_cast<size_t>(b)]; q < W.schur_ptr[static_cast<size_t>(b) + 1]; ++q) {
      const SchurTarget& T = W.schur[static_cast<size_t>(q)];
      if ((T.kind & 1) == 0) continue;
      fd[static_cast<size_t>(T.idx)] = std::min(fd[static_cast<size_t>(T.idx)], b);
      ld[static_cast<size_t>(T.idx)] = std::max(ld[static_cast<size_t>(T.idx)], b);
    }
  F.foff.assign(nf, -1);
  F.zero_at.assign(static_cast<size_t>(K), {});
  F.collapse_at.assign(static_cast<size_t>(K), {});
  F.core_at.assign(static_cast<size_t>(K), {});
  std::vector<std::vector<int>> start(static_cast<size_t>(K)), stop(static_cast<size_t>(K));
  for (size_t f = 0; f < nf; ++f) {
    const int bc = std::max(sch.order[static_cast<size_t>(L.frow[f])], sch.order[static_cast<size_t>(L.fcol[f])]);
    const int s1 = fill_segment(bc, nbat, K);
    const bool in = !init.empty() && init[f];
    const bool full = in || (ld[f] >= 0 && fill_segment(fd[f], nbat, K) <= s1);
    const bool core_dep = ld[f] >= 0 && fill_segment(ld[f], nbat, K) > s1;
    if (full) {
      const int s0 = in ? 0 : fill_segment(fd[f], nbat, K);
      start[static_cast<size_t>(s0)].push_back(static_cast<int>(f));
      stop[static_cast<size_t>(s1)].push_back(static_cast<int>(f));
      F.collapse_at[static_cast<size_t>(s1)].push_back(static_cast<int>(f));
      F.full_elems_total += static_cast<long long>(bsz[static_cast<size_t>(L.frow[f])]) * bsz[static_cast<size_t>(L.fcol[f])];
    }
    if (full || core_dep) F.core_at[static_cast<size_t>(s1)].push_back(static_cast<int>(f));
  }
  FrontAllocator A;
  auto size_of = [&](int f) {
    return static_cast<long long>(bsz[static_cast<size_t>(L.frow[static_cast<size_t>(f)])]) * bsz[static_cast<size_t>(L.fcol[static_cast<size_t>(f)])];
  };
  for (int s = 0; s < K; ++s) {
    for (int f : start[static_cast<size_t>(s)]) {
      F.foff[static_cast<size_t>(f)] = A.alloc(size_of(f));
      if (s > 0) F.zero_at[static_cast<size_t>(s)].push_back(f);
    }
    A.note();
    for (int f : stop[static_cast<size_t>(s)]) A.release(F.foff[static_cast<size_t>(f)], size_of(f));
  }
  F.pool_elems = A.high();
  return F;
}

LevelWork build_work(const LevelSym& L, const LevelSchedule& sch, int segments) {
  LevelWork W;
  const int nbat = static_cast<int>(sch.batch_ptr.size()) - 1;
  const int K = fill_segments(nbat, segments);
  W.fill_segments = K;
  const auto& ord = sch.order;
  struct Tmp {
    int64_t key;  // kind, idx
    SchurContrib c;
  };
  struct STmp {
    int64_t seg;
    SolveContrib c;
  };
  std::vector<int> batch_of(static_cast<size_t>(L.nl), -1);
  for (int b = 0; b < nbat; ++b)
    for (int q = sch.batch_ptr[static_cast<size_t>(b)]; q < sch.batch_ptr[static_cast<size_t>(b) + 1]; ++q)
      batch_of[static_cast<size_t>(sch.batch_cl[static_cast<size_t>(q)])] = b;
  auto target_rc = [&](const SchurTarget& T) {
    if ((T.kind & 1) == 0) return std::make_pair(L.drow[static_cast<size_t>(T.idx)], L.dcol[static_cast<size_t>(T.idx)]);
    return std::make_pair(L.frow[static_cast<size_t>(T.idx)], L.fcol[static_cast<size_t>(T.idx)]);
  };
  // Batches are independent: ranges of batches are built on host threads and
  // concatenated in batch order (indices into the contribution lists shifted).
  auto build_range = [&](int b0, int b1, LevelWork& W) {
    W.panel_ptr.assign(1, 0);
    W.schur_ptr.assign(1, 0);
    W.fsolve_ptr.assign(1, 0);
    std::vector<Tmp> tmp;
    std::vector<STmp> stmp;
    std::vector<SchurTarget> bulk;
    for (int b = b0; b < b1; ++b) {
      const int p0 = sch.batch_ptr[static_cast<size_t>(b)], p1 = sch.batch_ptr[static_cast<size_t>(b) + 1];
      W.max_batch = std::max(W.max_batch, p1 - p0);
      tmp.clear();
      stmp.clear();
      for (int q = p0; q < p1; ++q) {
        const int t = sch.batch_cl[static_cast<size_t>(q)];
        const int ot = ord[static_cast<size_t>(t)];
        for (int e = L.C_ptr[static_cast<size_t>(t)]; e < L.C_ptr[static_cast<size_t>(t) + 1]; ++e) {
          const int c = L.C_nb[static_cast<size_t>(e)];
          W.panel.push_back({q - p0, 0, c, L.C_blk[static_cast<size_t>(e)], e, ord[static_cast<size_t>(c)] < ot ? 1 : 0});
        }
        for (int e = L.R_ptr[static_cast<size_t>(t)]; e < L.R_ptr[static_cast<size_t>(t) + 1]; ++e) {
          const int j = L.R_nb[static_cast<size_t>(e)];
          W.panel.push_back({q - p0, 1, j, L.R_blk[static_cast<size_t>(e)], e, ord[static_cast<size_t>(j)] < ot ? 1 : 0});
        }
        // Schur products rows x cols, self last (factorization.hpp:403-425)
        const int r0 = L.R_ptr[static_cast<size_t>(t)], r1 = L.R_ptr[static_cast<size_t>(t) + 1];
        const int c0 = L.C_ptr[static_cast<size_t>(t)], c1 = L.C_ptr[static_cast<size_t>(t) + 1];
        for (int a = r0; a <= r1; ++a) {
          const bool rself = a == r1;
          const int j = rself ? t : L.R_nb[static_cast<size_t>(a)];
          for (int e = c0; e <= c1; ++e) {
            const bool cself = e == c1;
            if (rself && cself) continue;  // D(t,t) corner: head kernel
            const int c = cself ? t : L.C_nb[static_cast<size_t>(e)];
            SchurContrib sc{t, rself ? -1 - t : a, cself ? -1 - t : e, 0};
            int kind, idx;
            if (rself) {
              kind = 0, idx = L.C_blk[static_cast<size_t>(e)];
            } else if (cself) {
              kind = 0, idx = L.R_blk[static_cast<size_t>(a)];
            } else {
              idx = L.dense_index(j, c);
              kind = 0;
              if (idx < 0) {
                kind = 1;
                idx = L.fill_index(j, c);
                if (idx < 0) throw std::logic_error("plan: Schur target neither dense nor fill");
                if (ord[static_cast<size_t>(j)] < ot) sc.flags |= 1;
                if (ord[static_cast<size_t>(c)] < ot) sc.flags |= 2;
              }
            }
            tmp.push_back({(int64_t(kind) << 40) | int64_t(idx), sc});
            ++W.schur_products;
          }
          // forward-solve Lbar targets (solve.hpp:51)
          stmp.push_back({rself ? -1 - int64_t(t) : int64_t(j), {t, rself ? -1 - t : a}});
        }
      }
      std::stable_sort(tmp.begin(), tmp.end(), [](const Tmp& x, const Tmp& y) { return x.key < y.key; });
      bulk.clear();
      int ncrit = 0;
      for (size_t i = 0; i < tmp.size();) {
        size_t j = i;
        while (j < tmp.size() && tmp[j].key == tmp[i].key) ++j;
        SchurTarget T{static_cast<int32_t>(tmp[i].key >> 40), static_cast<int32_t>(tmp[i].key & ((int64_t(1) << 40) - 1)),
                      static_cast<int32_t>(W.contrib.size()), static_cast<int32_t>(W.contrib.size() + (j - i))};
        const auto rc = target_rc(T);
        // fill target whose core already exists (both sides collapsed in an
        // earlier segment): deposit into the core, unlifted panels
        bool core = false;
        if (T.kind == 1) {
          const int bc = std::max(ord[static_cast<size_t>(rc.first)], ord[static_cast<size_t>(rc.second)]);
          core = fill_segment(b, nbat, K) > fill_segment(bc, nbat, K);
          if (core) T.kind |= 8;
        }
        for (size_t k = i; k < j; ++k) {
          SchurContrib cb = tmp[k].c;
          if (core) cb.flags = 0;
          W.contrib.push_back(cb);
        }
        // dense target whose row (column) cluster was eliminated in an earlier
        // batch: its first e rows (columns) are zero and stay zero (cleanup,
        // factorization.hpp:431-439), so the update there is exactly zero and
        // the kernel starts its tiles at e (bit 1: rows, bit 2: columns)
        if (T.kind == 0) {
          if (batch_of[static_cast<size_t>(rc.first)] < b) T.kind |= 2;
          if (batch_of[static_cast<size_t>(rc.second)] < b) T.kind |= 4;
        }
        if (batch_of[static_cast<size_t>(rc.first)] == b + 1 || batch_of[static_cast<size_t>(rc.second)] == b + 1) {
          W.schur.push_back(T);
          ++ncrit;
        } else {
          bulk.push_back(T);
        }
        i = j;
      }
      W.schur.insert(W.schur.end(), bulk.begin(), bulk.end());
      W.schur_crit.push_back(ncrit);
      std::stable_sort(stmp.begin(), stmp.end(), [](const STmp& x, const STmp& y) { return x.seg < y.seg; });
      for (size_t i = 0; i < stmp.size();) {
        size_t j = i;
        while (j < stmp.size() && stmp[j].seg == stmp[i].seg) ++j;
        SolveTarget T{static_cast<int32_t>(stmp[i].seg), static_cast<int32_t>(W.fcontrib.size()), static_cast<int32_t>(W.fcontrib.size() + (j - i))};
        for (size_t k = i; k < j; ++k) W.fcontrib.push_back(stmp[k].c);
        W.fsolve.push_back(T);
        i = j;
      }
      W.panel_ptr.push_back(static_cast<int32_t>(W.panel.size()));
      W.schur_ptr.push_back(static_cast<int32_t>(W.schur.size()));
      W.fsolve_ptr.push_back(static_cast<int32_t>(W.fsolve.size()));
    }
  };
  const int nt = std::max(1, std::min<int>(static_cast<int>(std::thread::hardware_concurrency()), nbat / 16));
  std::vector<LevelWork> part(static_cast<size_t>(nt));
  {
    std::vector<std::thread> th;
    std::exception_ptr failed;
    std::mutex fm;
    for (int w = 0; w < nt; ++w)
      th.emplace_back([&, w] {
        try {
          build_range(static_cast<int>(static_cast<int64_t>(nbat) * w / nt), static_cast<int>(static_cast<int64_t>(nbat) * (w + 1) / nt),
                      part[static_cast<size_t>(w)]);
        } catch (...) {
          std::lock_guard<std::mutex> g(fm);
          if (!failed) failed = std::current_exception();
        }
      });
    for (auto& t : th) t.join();
    if (failed) std::rethrow_exception(failed);
  }
  W.panel_ptr.assign(1, 0);
  W.schur_ptr.assign(1, 0);
  W.fsolve_ptr.assign(1, 0);
  for (LevelWork& P : part) {
    const int32_t po = static_cast<int32_t>(W.panel.size()), so = static_cast<int32_t>(W.schur.size()), co = static_cast<int32_t>(W.contrib.size());
    const int32_t fo = static_cast<int32_t>(W.fsolve.size()), fco = static_cast<int32_t>(W.fcontrib.size());
    for (size_t i = 1; i < P.panel_ptr.size(); ++i) W.panel_ptr.push_back(po + P.panel_ptr[i]);
    for (size_t i = 1; i < P.schur_ptr.size(); ++i) W.schur_ptr.push_back(so + P.schur_ptr[i]);
    for (size_t i = 1; i < P.fsolve_ptr.size(); ++i) W.fsolve_ptr.push_back(fo + P.fsolve_ptr[i]);
    W.panel.insert(W.panel.end(), P.panel.begin(), P.panel.end());
    for (SchurTarget T : P.schur) {
      T.c0 += co, T.c1 += co;
      W.schur.push_back(T);
    }
    W.contrib.insert(W.contrib.end(), P.contrib.begin(), P.contrib.end());
    W.schur_crit.insert(W.schur_crit.end(), P.schur_crit.begin(), P.schur_crit.end());
    for (SolveTarget T : P.fsolve) {
      T.c0 += fco, T.c1 += fco;
      W.fsolve.push_back(T);
    }
    W.fcontrib.insert(W.fcontrib.end(), P.fcontrib.begin(), P.fcontrib.end());
    W.max_batch = std::max(W.max_batch, P.max_batch);
    W.schur_products += P.schur_products;
  }
  return W;
}

}  // namespace h2g

// Seeded right-hand side exactly as proj/tools/h2lu_cli.cpp:181-191. Compiled
// by g++ (not nvcc) so cxd(g(rng), g(rng)) evaluates its arguments in the
// same order as the reference build.
extern "C" void h2g_random_rhs(int64_t n, uint64_t seed, double* out) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> g;
  for (int64_t i = 0; i < n; ++i) {
    std::complex<double> v = std::complex<double>(g(rng), g(rng));
    out[2 * i] = v.real();
    out[2 * i + 1] = v.imag();
  }
}
