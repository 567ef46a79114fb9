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
  H2Matrix(const Context& ctx, const h2g_matrix_desc& d) : ctx_(ctx) {
    h2g_error e{};
    h2g_matrix* m = nullptr;
    check(h2g_matrix_upload(ctx.get(), &d, &m, &e), e);
    m_.reset(m, [](h2g_matrix* p) { h2g_matrix_destroy(p); });
    int64_t s[8];
    h2g_matrix_sizes(m, s);
    n_ = s[0];
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
  FactorChain(h2g_chain* c, int64_t n) : c_(c, [](h2g_chain* p) { h2g_chain_destroy(p); }), n_(n) {}
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
  std::shared_ptr<h2g_chain> c_;
  int64_t n_;
};

inline FactorChain factorize(const H2Matrix& A, double eps_fill_in, std::optional<int> stop_level_override = std::nullopt,
                             int schedule = H2G_SCHEDULE_REFERENCE) {
  h2g_error e{};
  h2g_chain* c = nullptr;
  check(h2g_factorize(A.ctx().get(), A.get(), eps_fill_in, stop_level_override.value_or(-1), schedule, &c, &e), e);
  return FactorChain(c, A.n());
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
