// H2LU v1 reader / writer (format of proj/include/h2lu/serialize.hpp:27-343,
// restated for host data; see serialize.hpp).
#include "serialize.hpp"

#include <cstdio>
#include <cstring>
#include <stdexcept>

namespace h2g {
namespace io {

namespace {

constexpr uint32_t kMagic = 0x554C3248;  // "H2LU"
constexpr uint32_t kVersion = 1;
constexpr uint32_t kKindH2 = 1, kKindChain = 2, kKindVector = 3;
constexpr int64_t kDimGuard = int64_t(1) << 27;  // implausible counts fail with a message

[[noreturn]] void fail(const std::string& m) { throw std::runtime_error("serialize: " + m); }

class Out {
 public:
  explicit Out(const std::string& path) : f_(std::fopen(path.c_str(), "wb")) {
    if (!f_) throw std::invalid_argument("serialize: cannot open " + path + " for writing");
    std::setvbuf(f_, nullptr, _IOFBF, 1 << 22);
  }
  ~Out() {
    if (f_) std::fclose(f_);
  }
  void close() {
    const int rc = std::fclose(f_);
    f_ = nullptr;
    if (rc != 0) fail("write failed");
  }
  void bytes(const void* p, size_t n) {
    if (n && std::fwrite(p, 1, n, f_) != n) fail("write failed");
  }
  template <class T>
  void put(T v) {
    bytes(&v, sizeof v);
  }
  void mat(const HMat& m) {
    put<int64_t>(m.rows);
    put<int64_t>(m.cols);
    bytes(m.data.data(), m.data.size() * sizeof(cxd));
  }
  void index_vec(const std::vector<int64_t>& v) {
    put<int64_t>(static_cast<int64_t>(v.size()));
    bytes(v.data(), v.size() * sizeof(int64_t));
  }
  void header(uint32_t kind) {
    put<uint32_t>(kMagic);
    put<uint32_t>(kVersion);
    put<uint32_t>(kind);
  }
  void tree(const TreeData& t) {  // serialize.hpp:121-132
    put<int64_t>(t.n);
    put<int32_t>(t.depth);
    put<int64_t>(t.leafsize);
    index_vec(t.perm);
    bytes(t.points.data(), t.points.size() * sizeof(double));
    for (size_t id = 0; id < t.begin.size(); ++id) {
      put<int64_t>(t.begin[id]);
      put<int64_t>(t.end[id]);
    }
  }

 private:
  std::FILE* f_;
};

class In {
 public:
  explicit In(const std::string& path) : f_(std::fopen(path.c_str(), "rb")) {
    if (!f_) throw std::invalid_argument("serialize: cannot open " + path);
    std::setvbuf(f_, nullptr, _IOFBF, 1 << 22);
  }
  ~In() {
    if (f_) std::fclose(f_);
  }
  void bytes(void* p, size_t n) {
    if (n && std::fread(p, 1, n, f_) != n) fail("truncated input");
  }
  template <class T>
  T get() {
    T v;
    bytes(&v, sizeof v);
    return v;
  }
  int64_t count(const char* what) {
    const int64_t v = get<int64_t>();
    if (v < 0 || v > kDimGuard) fail(std::string("implausible ") + what);
    return v;
  }
  HMat mat() {
    HMat m;
    m.rows = count("matrix rows");
    m.cols = count("matrix cols");
    if (m.rows > 0 && m.cols > kDimGuard / m.rows) fail("implausible matrix size");
    m.data.resize(static_cast<size_t>(m.rows * m.cols));
    bytes(m.data.data(), m.data.size() * sizeof(cxd));
    return m;
  }
  std::vector<int64_t> index_vec() {
    std::vector<int64_t> v(static_cast<size_t>(count("index vector length")));
    bytes(v.data(), v.size() * sizeof(int64_t));
    return v;
  }
  void header(uint32_t kind) {
    if (get<uint32_t>() != kMagic) fail("bad magic, not an h2lu file");
    const uint32_t ver = get<uint32_t>();
    if (ver != kVersion) fail("unsupported version " + std::to_string(ver));
    const uint32_t k = get<uint32_t>();
    if (k != kind) fail("file holds payload kind " + std::to_string(k) + ", expected " + std::to_string(kind));
  }
  TreeData tree() {  // serialize.hpp:134-182 (validation included)
    TreeData t;
    t.n = count("point count");
    t.depth = get<int32_t>();
    t.leafsize = count("leafsize");
    if (t.n < 1 || t.leafsize < 1 || t.depth < 0 || t.depth > 48) fail("malformed tree header");
    t.perm = index_vec();
    if (static_cast<int64_t>(t.perm.size()) != t.n) fail("permutation length mismatch");
    std::vector<char> seen(static_cast<size_t>(t.n), 0);
    for (int64_t p : t.perm) {
      if (p < 0 || p >= t.n || seen[static_cast<size_t>(p)]) fail("perm is not a permutation");
      seen[static_cast<size_t>(p)] = 1;
    }
    t.points.resize(static_cast<size_t>(3 * t.n));
    bytes(t.points.data(), t.points.size() * sizeof(double));
    const int64_t nc = (int64_t(2) << t.depth) - 1;
    t.begin.resize(static_cast<size_t>(nc));
    t.end.resize(static_cast<size_t>(nc));
    for (int64_t id = 0; id < nc; ++id) {
      t.begin[static_cast<size_t>(id)] = get<int64_t>();
      t.end[static_cast<size_t>(id)] = get<int64_t>();
      if (t.begin[static_cast<size_t>(id)] < 0 || t.begin[static_cast<size_t>(id)] > t.end[static_cast<size_t>(id)] || t.end[static_cast<size_t>(id)] > t.n)
        fail("cluster range out of bounds");
    }
    if (t.begin[0] != 0 || t.end[0] != t.n) fail("root range mismatch");
    const int64_t inner = (int64_t(1) << t.depth) - 1;
    for (int64_t id = 0; id < inner; ++id) {
      const size_t a = static_cast<size_t>(2 * id + 1), b = a + 1, c = static_cast<size_t>(id);
      if (t.begin[a] != t.begin[c] || t.end[a] != t.begin[b] || t.end[b] != t.end[c]) fail("children do not partition their parent");
    }
    return t;
  }

 private:
  std::FILE* f_;
};

}  // namespace

// ------------------------------------------------------------------ matrix
void save_matrix(const std::string& path, const MatrixFile& m) {  // save_h2, serialize.hpp:186-196
  Out o(path);
  o.header(kKindH2);
  o.tree(m.tree);
  o.put<double>(m.eta);
  o.put<double>(m.eps_h2);
  o.put<int64_t>(m.shadow_guard);
  for (const HMat& b : m.bases) o.mat(b);
  for (const auto& lv : m.couplings)
    for (const HMat& S : lv) o.mat(S);
  for (const HMat& D : m.dense) o.mat(D);
  o.close();
}

struct MatrixReader::Impl {
  In in;
  explicit Impl(const std::string& p) : in(p) {}
};

MatrixReader::MatrixReader(const std::string& path) : p_(new Impl(path)) {  // load_h2, serialize.hpp:198-243
  In& in = p_->in;
  in.header(kKindH2);
  m_.tree = in.tree();
  m_.eta = in.get<double>();
  if (!(m_.eta > 0.0)) fail("eta must be positive");
  m_.eps_h2 = in.get<double>();
  m_.shadow_guard = in.count("shadow guard");
  const size_t nc = m_.tree.begin.size();
  m_.bases.resize(nc);
  for (auto& b : m_.bases) b = in.mat();
  const int64_t first_leaf = (int64_t(1) << m_.tree.depth) - 1;
  for (size_t id = 0; id < nc; ++id) {
    const int64_t expect = static_cast<int64_t>(id) >= first_leaf ? m_.tree.end[id] - m_.tree.begin[id]
                                                                  : m_.bases[2 * id + 1].cols + m_.bases[2 * id + 2].cols;
    if (m_.bases[id].rows != expect) fail("basis rows inconsistent with tree");
  }
}

MatrixReader::~MatrixReader() { delete p_; }

void MatrixReader::read_rest(const std::vector<int64_t>& adm_per_level, int64_t num_leaf_pairs) {
  In& in = p_->in;
  m_.couplings.assign(adm_per_level.size(), {});
  for (size_t l = 0; l < adm_per_level.size(); ++l) {
    m_.couplings[l].resize(static_cast<size_t>(adm_per_level[l]));
    for (auto& S : m_.couplings[l]) S = in.mat();
  }
  m_.dense.resize(static_cast<size_t>(num_leaf_pairs));
  for (auto& D : m_.dense) D = in.mat();
}

// ------------------------------------------------------------------- chain
void save_chain(const std::string& path, const ChainFile& c) {  // serialize.hpp:245-284
  Out o(path);
  o.header(kKindChain);
  o.tree(c.tree);
  o.put<int64_t>(c.n);
  o.put<int32_t>(c.stop_level);
  o.put<double>(c.eps_fill_in);
  o.put<int64_t>(static_cast<int64_t>(c.levels.size()));
  for (const LevelFile& lb : c.levels) {
    o.put<int32_t>(lb.level);
    o.put<int64_t>(static_cast<int64_t>(lb.recs.size()));
    for (const RecordData& r : lb.recs) {
      o.put<int32_t>(r.cluster);
      o.put<int32_t>(r.level);
      for (int64_t f : {r.pos, r.bsize, r.eliminated, r.rank_before, r.rank_after, r.fill_targets}) o.put<int64_t>(f);
      o.mat(r.Qtilde);
      o.mat(r.L11);
      o.mat(r.U11);
      for (const auto* side : {&r.Lbar, &r.Ubar}) {
        o.put<int64_t>(static_cast<int64_t>(side->size()));
        for (const OffBlock& b : *side) {
          o.put<int64_t>(b.pos);
          o.mat(b.M);
        }
      }
    }
    o.put<int32_t>(lb.perm_level);
    o.index_vec(lb.src);
    o.put<int64_t>(lb.active_after);
    o.put<int32_t>(lb.diag_level);
    for (int64_t f : {lb.rank_sum_before, lb.rank_sum_after, lb.eliminated, lb.ledger_blocks}) o.put<int64_t>(f);
    o.put<uint64_t>(lb.chain_bytes);
  }
  o.mat(c.root_l);
  o.mat(c.root_u);
  o.put<int64_t>(c.root_size);
  o.close();
}

ChainFile load_chain(const std::string& path) {  // serialize.hpp:286-343
  In in(path);
  in.header(kKindChain);
  ChainFile c;
  c.tree = in.tree();
  c.n = in.count("matrix size");
  if (c.n != c.tree.n) fail("chain size disagrees with its tree");
  c.stop_level = in.get<int32_t>();
  c.eps_fill_in = in.get<double>();
  const int64_t nlev = in.count("level count");
  if (nlev > c.tree.depth + 1) fail("more level blocks than tree levels");
  c.levels.resize(static_cast<size_t>(nlev));
  for (LevelFile& lb : c.levels) {
    lb.level = in.get<int32_t>();
    lb.recs.resize(static_cast<size_t>(in.count("record count")));
    for (RecordData& r : lb.recs) {
      r.cluster = in.get<int32_t>();
      r.level = in.get<int32_t>();
      for (int64_t* f : {&r.pos, &r.bsize, &r.eliminated, &r.rank_before, &r.rank_after, &r.fill_targets}) *f = in.get<int64_t>();
      r.Qtilde = in.mat();
      r.L11 = in.mat();
      r.U11 = in.mat();
      if (r.Qtilde.rows != r.Qtilde.cols || r.Qtilde.rows != r.bsize || r.L11.rows != r.eliminated || r.L11.rows != r.L11.cols ||
          r.U11.rows != r.U11.cols || r.U11.rows != r.eliminated || r.eliminated > r.bsize || r.eliminated < 0)
        fail("elimination record dims inconsistent");
      for (auto* side : {&r.Lbar, &r.Ubar}) {
        side->resize(static_cast<size_t>(in.count("off-diagonal block count")));
        for (OffBlock& b : *side) {
          b.pos = in.get<int64_t>();
          b.M = in.mat();
          if (b.pos < 0 || b.pos >= c.n) fail("off-diagonal block out of range");
        }
      }
    }
    lb.perm_level = in.get<int32_t>();
    lb.src = in.index_vec();
    lb.active_after = in.get<int64_t>();
    for (int64_t s : lb.src)
      if (s < 0 || s >= static_cast<int64_t>(lb.src.size())) fail("permutation entry out of range");
    lb.diag_level = in.get<int32_t>();
    for (int64_t* f : {&lb.rank_sum_before, &lb.rank_sum_after, &lb.eliminated, &lb.ledger_blocks}) *f = in.get<int64_t>();
    lb.chain_bytes = in.get<uint64_t>();
  }
  c.root_l = in.mat();
  c.root_u = in.mat();
  c.root_size = in.count("root size");
  if (c.root_l.rows != c.root_size || c.root_l.cols != c.root_size || c.root_u.rows != c.root_size || c.root_u.cols != c.root_size)
    fail("root factor dims inconsistent");
  return c;
}

// ------------------------------------------------------------------ vector
void save_vector(const std::string& path, const std::vector<cxd>& v) {  // serialize.hpp:345-348
  Out o(path);
  o.header(kKindVector);
  o.put<int64_t>(static_cast<int64_t>(v.size()));
  o.bytes(v.data(), v.size() * sizeof(cxd));
  o.close();
}

std::vector<cxd> load_vector(const std::string& path) {  // :350-353
  In in(path);
  in.header(kKindVector);
  std::vector<cxd> v(static_cast<size_t>(in.count("vector length")));
  in.bytes(v.data(), v.size() * sizeof(cxd));
  return v;
}

}  // namespace io
}  // namespace h2g
