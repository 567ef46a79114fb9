// C++ facade over the h2g C ABI with the reference h2lu hot-path API shape:
//   FactorChain factorize(const H2Matrix&, double eps_fill_in, std::optional<int> stop)
//   Vec solve(const FactorChain&, const Vec&), apply_inverse, solve_in_place,
//   forward_substitute, backward_substitute
// (proj/include/h2lu/factorization.hpp:600, solve.hpp:85-113) and the same
// exception types (types.hpp:18-47). Header-only; link libh2g.so.
//
// The reference's H2Matrix is Eigen-based; H2Desc below is the plain-array
// view of it that INTEGRATION.md shows how to fill from an h2lu::H2Matrix.
#pragma once

#include <complex>
#include <functional>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "h2g.h"

namespace h2lu_gpu {

using cxd = std::complex<double>;
using Vec = std::vector<cxd>;

struct InvalidInputError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct SizeGuardError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NonFiniteError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct SingularPivotError : std::runtime_error {
  int64_t pivot_index;
  double pivot_magnitude;
  int cluster, level;
  SingularPivotError(const std::string& m, int64_t i, double g, int c, int l)
      : std::runtime_error(m), pivot_index(i), pivot_magnitude(g), cluster(c), level(l) {}
};
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int rc, const h2g_error& e) {
  if (rc == H2G_OK) return;
  switch (rc) {
    case H2G_ERR_INVALID_INPUT:
      throw InvalidInputError(e.msg);
    case H2G_ERR_SIZE_GUARD:
      throw SizeGuardError(e.msg);
    case H2G_ERR_NON_FINITE:
      throw NonFiniteError(e.msg);
    case H2G_ERR_SINGULAR_PIVOT:
      throw SingularPivotError(e.msg, e.pivot_index, e.pivot_magnitude, e.cluster, e.level);
    default:
      throw DeviceError(e.msg);
  }
}

class Context {
 public:
  explicit Context(int device = 0) {
    h2g_error e{};
    h2g_context* c = nullptr;
    check(h2g_context_create(device, &c, &e), e);
    ctx_.reset(c, [](h2g_context* p) { h2g_context_destroy(p); });
  }
  h2g_context* get() const { return ctx_.get(); }

 private:
  std::shared_ptr<h2g_context> ctx_;
};

// Device-resident H2Matrix (immutable input of factorize).
class H2Matrix {
 public:
  H2Matrix(const Context& ctx, h2g_matrix* m) : ctx_(ctx), m_(m, [](h2g_matrix* p) { h2g_matrix_destroy(p); }) {
    int64_t s[8];
    h2g_matrix_sizes(m, s);
    n_ = s[0];
  }
  H2Matrix(const Context& ctx, const h2g_matrix_desc& d) : ctx_(ctx) {
    h2g_error e{};
    h2g_matrix* m = nullptr;
    check(h2g_matrix_upload(ctx.get(), &d, &m, &e), e);
    m_.reset(m, [](h2g_matrix* p) { h2g_matrix_destroy(p); });
    int64_t s[8];
    h2g_matrix_sizes(m, s);
    n_ = s[0];
  }
  // load_h2 (serialize.hpp:198-243) onto the device
  static H2Matrix load(const Context& ctx, const std::string& path) {
    h2g_error e{};
    h2g_matrix* m = nullptr;
    check(h2g_matrix_load(ctx.get(), path.c_str(), &m, &e), e);
    return H2Matrix(ctx, m);
  }
  int64_t n() const { return n_; }
  const h2g_matrix* get() const { return m_.get(); }
  const Context& ctx() const { return ctx_; }

 private:
  Context ctx_;
  std::shared_ptr<h2g_matrix> m_;
  int64_t n_ = 0;
};

class FactorChain {
 public:
  // The chain keeps its context alive (the C ABI reference-counts it too).
  FactorChain(h2g_chain* c, int64_t n, Context ctx) : ctx_(std::move(ctx)), c_(c, [](h2g_chain* p) { h2g_chain_destroy(p); }), n_(n) {}
  int64_t n() const { return n_; }
  h2g_chain* get() const { return c_.get(); }
  int stop_level() const { return info()[1]; }
  int64_t root_size() const { return info()[2]; }
  size_t storage_bytes() const { return static_cast<size_t>(info()[4]); }

 private:
  std::vector<int64_t> info() const {
    std::vector<int64_t> v(6);
    h2g_chain_info(c_.get(), v.data());
    return v;
  }
  Context ctx_;
  std::shared_ptr<h2g_chain> c_;
  int64_t n_;
};

// FactorState as a hook sees it (factorization.hpp:115-251).
class FactorState {
 public:
  explicit FactorState(const h2g_state* s) : s_(s) {}
  struct ClusterInfo {
    int64_t pos, bsize, rank, rotated, eliminated;
  };
  ClusterInfo cluster(int id) const {
    int64_t o[5];
    h2g_error e{};
    check(h2g_state_cluster(s_, id, o), e);
    return {o[0], o[1], o[2], o[3], o[4]};
  }
  // FactorState::shadow() (:240-245), n x n column-major
  std::vector<cxd> shadow() const {
    int64_t info[3];
    h2g_state_info(s_, info);
    std::vector<cxd> Z(static_cast<size_t>(info[2] * info[2]));
    h2g_error e{};
    const int rc = h2g_state_shadow(s_, reinterpret_cast<double*>(Z.data()));
    if (rc) {
      h2g_last_error(&e);
      check(rc, e);
    }
    return Z;
  }
  const h2g_state* get() const { return s_; }

 private:
  const h2g_state* s_;
};

// FactorizeHooks (factorization.hpp:588-593)
struct FactorizeHooks {
  std::function<void(const FactorState&, int)> after_basis_update, after_projection, after_elimination;
  std::function<void(const FactorState&)> after_merge;
};

inline FactorChain factorize(const H2Matrix& A, double eps_fill_in, std::optional<int> stop_level_override = std::nullopt,
                             int schedule = H2G_SCHEDULE_REFERENCE) {
  h2g_error e{};
  h2g_chain* c = nullptr;
  check(h2g_factorize(A.ctx().get(), A.get(), eps_fill_in, stop_level_override.value_or(-1), schedule, &c, &e), e);
  return FactorChain(c, A.n(), A.ctx());
}

// factorize run by one process per GPU (h2g_factorize_dist: the north_star's
// subtree partition). `exchange(buf, offsets, nranks)` must all-gather the
// per-rank parts of the device buffer (ncclBroadcast per part inside one
// group) and return 0; every rank gets the complete chain.
using Exchange = std::function<int(void* device_buf, const int64_t* offsets, int nranks)>;
inline FactorChain factorize_dist(const H2Matrix& A, double eps_fill_in, int rank, int nranks, const Exchange& exchange,
                                  std::optional<int> stop_level_override = std::nullopt) {
  h2g_dist d{};
  d.rank = rank;
  d.nranks = nranks;
  d.user = const_cast<Exchange*>(&exchange);
  d.exchange = [](void* u, void* buf, const int64_t* off, int32_t n) -> int {
    auto* f = static_cast<Exchange*>(u);
    return *f ? (*f)(buf, off, n) : 1;
  };
  h2g_error e{};
  h2g_chain* c = nullptr;
  check(h2g_factorize_dist(A.ctx().get(), A.get(), eps_fill_in, stop_level_override.value_or(-1), &d, &c, &e), e);
  return FactorChain(c, A.n(), A.ctx());
}

// factorize(A, eps, stop, hooks) (factorization.hpp:600-601): the device in
// debug mode (reference order, one cluster per step).
inline FactorChain factorize(const H2Matrix& A, double eps_fill_in, std::optional<int> stop_level_override, const FactorizeHooks* hooks) {
  if (!hooks) return factorize(A, eps_fill_in, stop_level_override);
  h2g_factorize_hooks h{};
  h.user = const_cast<FactorizeHooks*>(hooks);
  h.after_basis_update = [](void* u, const h2g_state* st, int32_t i) {
    auto* k = static_cast<FactorizeHooks*>(u);
    if (k->after_basis_update) k->after_basis_update(FactorState(st), i);
  };
  h.after_projection = [](void* u, const h2g_state* st, int32_t i) {
    auto* k = static_cast<FactorizeHooks*>(u);
    if (k->after_projection) k->after_projection(FactorState(st), i);
  };
  h.after_elimination = [](void* u, const h2g_state* st, int32_t i) {
    auto* k = static_cast<FactorizeHooks*>(u);
    if (k->after_elimination) k->after_elimination(FactorState(st), i);
  };
  h.after_merge = [](void* u, const h2g_state* st) {
    auto* k = static_cast<FactorizeHooks*>(u);
    if (k->after_merge) k->after_merge(FactorState(st));
  };
  h2g_error e{};
  h2g_chain* c = nullptr;
  check(h2g_factorize_hooked(A.ctx().get(), A.get(), eps_fill_in, stop_level_override.value_or(-1), &h, &c, &e), e);
  return FactorChain(c, A.n(), A.ctx());
}

// ---- H2LU v1 container (serialize.hpp:186-353)
inline void save_h2(const std::string& path, const H2Matrix& A) {
  h2g_error e{};
  check(h2g_matrix_save(A.get(), path.c_str(), &e), e);
}
inline void save_chain(const std::string& path, const FactorChain& c, const H2Matrix& source) {
  h2g_error e{};
  check(h2g_chain_save(c.get(), source.get(), path.c_str(), &e), e);
}
inline FactorChain load_chain(const Context& ctx, const std::string& path) {
  h2g_error e{};
  h2g_chain* c = nullptr;
  check(h2g_chain_load(ctx.get(), path.c_str(), &c, &e), e);
  int64_t info[6];
  h2g_chain_info(c, info);
  return FactorChain(c, info[0], ctx);
}
inline void save_vector(const std::string& path, const Vec& v) {
  h2g_error e{};
  check(h2g_vector_save(path.c_str(), reinterpret_cast<const double*>(v.data()), static_cast<int64_t>(v.size()), &e), e);
}
inline Vec load_vector(const std::string& path) {
  h2g_error e{};
  int64_t n = 0;
  check(h2g_vector_load(path.c_str(), nullptr, &n, &e), e);
  Vec v(static_cast<size_t>(n));
  check(h2g_vector_load(path.c_str(), reinterpret_cast<double*>(v.data()), &n, &e), e);
  return v;
}

inline Vec run(const FactorChain& ch, const Vec& b, int mode) {
  Vec x(b.size());
  h2g_error e{};
  check(h2g_solve(ch.get(), reinterpret_cast<const double*>(b.data()), reinterpret_cast<double*>(x.data()), static_cast<int64_t>(b.size()), 1,
                  mode, &e),
        e);
  return x;
}

inline Vec solve(const FactorChain& ch, const Vec& b) { return run(ch, b, H2G_SOLVE); }
inline Vec apply_inverse(const FactorChain& ch, const Vec& b) { return run(ch, b, H2G_APPLY_INVERSE); }
inline Vec forward_substitute(const FactorChain& ch, const Vec& b) { return run(ch, b, H2G_FORWARD); }
inline Vec backward_substitute(const FactorChain& ch, const Vec& y) { return run(ch, y, H2G_BACKWARD); }
inline void solve_in_place(const FactorChain& ch, Vec& b) {
  h2g_error e{};
  check(h2g_solve(ch.get(), reinterpret_cast<const double*>(b.data()), reinterpret_cast<double*>(b.data()), static_cast<int64_t>(b.size()), 1,
                  H2G_SOLVE, &e),
        e);
}

}  // namespace h2lu_gpu
