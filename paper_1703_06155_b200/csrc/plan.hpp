// Host-side symbolic analysis of an H² factorization (the structural part of
// proj/include/h2lu/factorization.hpp, done once per matrix and schedule).
//
// The reference discovers structure on the fly by scanning std::maps for every
// cluster (factorization.hpp:268-293, :345, :404, :436). Here
// every level's structure — dense blocks, fill-in targets (ledger/carried),
// Schur target maps, merge maps — is derived once from the block partition,
// laid out as CSR arrays and uploaded; the device kernels only index them.
#pragma once

#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/h2g.h"

namespace h2g {

struct Pair {
  int row, col;
};

// Cluster tree + block partition, as described by h2g_matrix_desc.
struct Structure {
  int64_t n = 0;
  int depth = 0;
  double eta = 1.0;
  std::vector<int64_t> begin, end;          // [num_clusters]
  std::vector<std::vector<Pair>> adm, split;  // [depth+1], sorted (row, col)
  std::vector<Pair> leaf;                     // sorted
  std::vector<int64_t> adm_offset;            // global admissible index of (level, 0)
  int l0 = -1;
  int num_clusters() const { return (2 << depth) - 1; }
  static int first(int l) { return (1 << l) - 1; }
  int64_t num_adm() const { return adm_offset.empty() ? 0 : adm_offset.back(); }
};

// One level's static structure. Cluster ids are LOCAL (0..nl-1, heap id =
// first + local).
struct LevelSym {
  int level = 0, nl = 0, first = 0;
  // dense (inadmissible at this level) blocks, sorted (row, col)
  std::vector<int> drow, dcol, diag_blk;
  // row entries R(t): j with (j,t) dense, j != t, ascending j (the "rows"
  // list of factorization.hpp:403-408) and col entries C(t): c with (t,c)
  // dense, c != t, ascending (the "cols" list).
  std::vector<int> R_ptr, R_nb, R_blk, C_ptr, C_nb, C_blk;
  // fill targets (ledger: admissible at this level; carried: owned by a
  // coarser admissible ancestor), sorted (row, col)
  std::vector<int> frow, fcol, fadm;  // fadm = index into adm[level] or -1 (carried)
  int nledger = 0;
  // step-0 gather list per cluster (factorization.hpp:278-293 order: ledger
  // keys touching t in map order, then carried keys): fill index + transposed
  std::vector<int> G_ptr, G_fill;
  std::vector<uint8_t> G_tr;
  // carried fills -> parent fill index at level-1, and which child slots
  std::vector<int> carried_parent;  // [nfill], -1 for ledger
  // dense-pair and fill lookup
  std::unordered_map<int64_t, int> dense_of, fill_of;
  int dense_index(int r, int c) const {
    auto it = dense_of.find(int64_t(r) * nl + c);
    return it == dense_of.end() ? -1 : it->second;
  }
  int fill_index(int r, int c) const {
    auto it = fill_of.find(int64_t(r) * nl + c);
    return it == fill_of.end() ? -1 : it->second;
  }
};

// Parts of the interior-first schedule (the north_star's 8-GPU subtree split).
constexpr int kInteriorParts = 8;

// Processing order of one level: batches of mutually non-adjacent clusters.
struct LevelSchedule {
  std::vector<int> batch_ptr, batch_cl;  // local ids, ascending within a batch
  std::vector<int> order;                // [nl] batch index of each cluster
  // SUBTREE schedule: batches [part_batch[s], part_batch[s + 1]) eliminate
  // interior clusters of subtree s only; batches from part_batch[parts] on are
  // the boundary clusters (all batches, for the other schedules)
  std::vector<int> part_batch;           // [kInteriorParts + 1]
};

// Per-batch work lists (static for a schedule; sizes resolved on device).
struct PanelItem {
  int32_t q;      // slot of the cluster in its batch
  int32_t side;   // 0: column item D(t,c) (Ubar), 1: row item D(j,t) (Lbar)
  int32_t nb;     // neighbour local id
  int32_t blk;    // dense block index
  int32_t entry;  // C entry (side 0) or R entry (side 1) global index
  int32_t lift;   // neighbour eliminated earlier: also store the lifted panel
};

// Fill-in storage by segments (compact fill). A level's batches
// are cut into K contiguous segments. A fill block (j, c) is held in full
// (bsz_j x bsz_c, level-entry frames, as deposit_fill keeps it,
// factorization.hpp:359-366) only while a side still has its step 0 ahead:
// at the end of the segment holding max(batch(j), batch(c)) it is projected to
// its core V_j^H F conj(V_c) (kfin_j x kfin_c, the only form its later
// consumers read, :455 and :540), and deposits of later segments go straight
// to the core (the lifts through V_j / V_c cancel against the projection).
int fill_segments(int nbat, int requested);
inline int fill_segment(int b, int nbat, int K) { return nbat > 0 ? static_cast<int>(static_cast<int64_t>(b) * K / nbat) : 0; }

struct SchurTarget {
  int32_t kind;   // bit 0: 0 dense, 1 fill; bits 1/2 (dense): row / column cluster eliminated in an earlier batch;
                  // bit 3 (fill): deposit into the compact core (both sides already collapsed)
  int32_t idx;    // dense block / fill index
  int32_t c0, c1; // contribution range
};

struct SchurContrib {
  int32_t t;      // cluster local id
  int32_t r;      // R entry global index, or -1 - t for the self row
  int32_t c;      // C entry global index, or -1 - t for the self column
  int32_t flags;  // bit0: lifted row panel, bit1: lifted column panel
};

struct SolveTarget {
  int32_t seg;    // neighbour local id j (or -1 - m: retained tail of record m)
  int32_t c0, c1; // contribution range into SolveContrib
};
struct SolveContrib {
  int32_t m;      // record (cluster local id)
  int32_t entry;  // R entry global index, or -1 - m for self
};

struct LevelWork {
  std::vector<int32_t> panel_ptr;  // per batch
  std::vector<PanelItem> panel;
  std::vector<int32_t> schur_ptr;  // per batch
  // per batch: the first schur_crit[b] targets of batch b lie in a row or
  // column of a cluster of batch b+1 (applied in-line on the main stream);
  // the rest are deferred to the side stream, overlapping batch b+1
  std::vector<int32_t> schur_crit;
  std::vector<SchurTarget> schur;
  std::vector<SchurContrib> contrib;
  std::vector<int32_t> fsolve_ptr;  // per batch
  std::vector<SolveTarget> fsolve;
  std::vector<SolveContrib> fcontrib;
  int max_batch = 0;
  int fill_segments = 1;       // K of the fill storage plan (fill_segments)
  int64_t schur_products = 0;  // structural count (upper bound)
};

// Segment plan of one level's fill storage (see fill_segments): full-block
// offsets in a reused "front" pool (interval allocation over segments) and
// the per-segment lists the driver acts on.
struct FrontPlan {
  int K = 1;
  std::vector<int> seg_first_batch;             // [K + 1]
  std::vector<long long> foff;                  // per fill: element offset in the front pool, -1 = never held in full
  long long pool_elems = 0;
  std::vector<std::vector<int>> zero_at;        // per segment: full blocks whose storage starts there (zeroed first; s > 0)
  std::vector<std::vector<int>> collapse_at;    // per segment: full blocks projected to cores at its end
  std::vector<std::vector<int>> core_at;        // per segment: every core created at its end (collapsed + core-only)
  long long full_elems_total = 0;               // sum of all full blocks (what a non-segmented pool would hold)
};
// init[f] != 0: the block holds content at level entry (carried fill-in
// deposited by the merge of the finer level); may be empty.
FrontPlan build_front(const LevelSym& L, const LevelSchedule& sch, const LevelWork& W, const std::vector<int>& bsz, const std::vector<int>& init);

// Multi-GPU subtree partition (h2g_factorize_dist): what the interior phase of
// each of the kInteriorParts subtrees writes under the SUBTREE schedule - the
// clusters it eliminates (final ranks, chain records), the dense blocks it
// rotates / updates and the fill blocks it deposits into - read off the work
// lists of the subtree's batches. Lists of different subtrees are disjoint
// (an interior cluster's dense neighbours all lie in its own subtree).
struct PartList {
  std::vector<int> cl, dblk, fblk;
  size_t ints() const { return cl.size() + fblk.size(); }
};
std::vector<PartList> build_parts(const LevelSym& L, const LevelSchedule& sch, const LevelWork& W);

Structure structure_from_desc(const h2g_matrix_desc* d);
Structure build_structure(const double* pts, int64_t n, int64_t leafsize, double eta, std::vector<int64_t>* perm);
// Partition of a given tree (tree-order points and heap-order ranges).
Structure structure_from_tree(const double* pts_tree, int64_t n, int depth, const std::vector<int64_t>& begin, const std::vector<int64_t>& end,
                              double eta);

// Levels from depth down to (and including) `stop`.
std::vector<LevelSym> build_levels(const Structure& S, int stop);
LevelSchedule build_schedule(const LevelSym& L, int kind);
// segments: requested fill-storage segments K (1 = whole-level full blocks,
// collapsed at the level end)
LevelWork build_work(const LevelSym& L, const LevelSchedule& sch, int segments);

}  // namespace h2g
