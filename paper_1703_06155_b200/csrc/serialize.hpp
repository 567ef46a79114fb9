// H2LU v1 container (the reference's on-disk format,
// proj/include/h2lu/serialize.hpp:27-343): little-endian raw fields behind a
// 12-byte header (magic "H2LU", version 1, payload kind 1 = H2 matrix,
// 2 = factor chain, 3 = vector); matrices as (int64 rows, int64 cols,
// column-major complex128). Host-side reader / writer of plain data; api.cu
// moves it to and from the device handles.
#pragma once

#include <complex>
#include <cstdint>
#include <string>
#include <vector>

namespace h2g {
namespace io {

using cxd = std::complex<double>;

struct HMat {
  int64_t rows = 0, cols = 0;
  std::vector<cxd> data;  // column-major
};

// ClusterTree as serialized (serialize.hpp:121-182): permutation, points in
// tree order, per-cluster index ranges in heap order.
struct TreeData {
  int64_t n = 0;
  int32_t depth = 0;
  int64_t leafsize = 0;
  std::vector<int64_t> perm;    // tree index -> original index
  std::vector<double> points;   // 3 n, tree order
  std::vector<int64_t> begin, end;
};

struct MatrixFile {  // save_h2 / load_h2 (:186-243)
  TreeData tree;
  double eta = 1.0, eps_h2 = 0.0;
  int64_t shadow_guard = 4000;
  std::vector<HMat> bases;                   // per cluster, heap order
  std::vector<std::vector<HMat>> couplings;  // per level, admissible order
  std::vector<HMat> dense;                   // inadmissible-leaf order
};

struct OffBlock {
  int64_t pos = 0;
  HMat M;
};
struct RecordData {  // EliminationRecord (factorization.hpp:22-44)
  int32_t cluster = -1, level = -1;
  int64_t pos = 0, bsize = 0, eliminated = 0, rank_before = 0, rank_after = 0, fill_targets = 0;
  HMat Qtilde, L11, U11;
  std::vector<OffBlock> Lbar, Ubar;
};
struct LevelFile {
  int32_t level = 0;
  std::vector<RecordData> recs;
  int32_t perm_level = 0;
  std::vector<int64_t> src;
  int64_t active_after = 0;
  int32_t diag_level = 0;
  int64_t rank_sum_before = 0, rank_sum_after = 0, eliminated = 0, ledger_blocks = 0;
  uint64_t chain_bytes = 0;
};
struct ChainFile {  // save_chain / load_chain (:245-343)
  TreeData tree;
  int64_t n = 0;
  int32_t stop_level = 0;
  double eps_fill_in = 0.0;
  std::vector<LevelFile> levels;
  HMat root_l, root_u;
  int64_t root_size = 0;
};

// All throw std::runtime_error("serialize: ...") on malformed input (the
// reference's SerializationError) and std::invalid_argument on I/O failure.
void save_matrix(const std::string& path, const MatrixFile& m);
// Reads everything but the couplings (their count depends on the block
// partition, which the caller recomputes from the tree); then call
// read_couplings with the per-level admissible counts.
class MatrixReader {
 public:
  explicit MatrixReader(const std::string& path);
  ~MatrixReader();
  MatrixFile& head() { return m_; }  // tree, eta, eps_h2, shadow_guard, bases
  void read_rest(const std::vector<int64_t>& adm_per_level, int64_t num_leaf_pairs);
  MatrixFile take() { return std::move(m_); }

 private:
  struct Impl;
  Impl* p_;
  MatrixFile m_;
};

void save_chain(const std::string& path, const ChainFile& c);
ChainFile load_chain(const std::string& path);

void save_vector(const std::string& path, const std::vector<cxd>& v);
std::vector<cxd> load_vector(const std::string& path);

}  // namespace io
}  // namespace h2g
