// ORACLE — TEST INFRASTRUCTURE ONLY.
// CPU restatement of the reference h2lu hot path, used by tests/, by
// __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference leg
// as the CHECKER. Nothing in paper_1703_06155_b200/ links or calls this code.
//
// Dense layer. The reference builds on Eigen 3 (unpinned, proj/CMakeLists.txt:13),
// which is absent from this image, so the primitives the hot path calls are
// restated here from their published algorithms:
//   * Householder QR (Eigen HouseholderQR convention: H = I - tau v v^H, v0 = 1,
//     beta = -sign(Re c0) |x|, Q = H_0^H H_1^H ...), used at
//     proj/include/h2lu/dense_kernels.hpp:62, h2_matrix.hpp:280, factorization.hpp:304
//   * a Jacobi SVD (one-sided Hestenes here; Eigen uses two-sided JacobiSVD,
//     proj/include/h2lu/h2_matrix.hpp:285). Singular values agree to rounding.
//   * unpivoted LU exactly as proj/include/h2lu/dense_kernels.hpp:70-93.
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pool.hpp"

namespace h2o {

using cxd = std::complex<double>;
using Index = int64_t;

// Error taxonomy of proj/include/h2lu/types.hpp:18-47.
struct InvalidInputError : std::runtime_error {
  explicit InvalidInputError(const std::string& m) : std::runtime_error(m) {}
};
struct SizeGuardError : std::runtime_error {
  explicit SizeGuardError(const std::string& m) : std::runtime_error(m) {}
};
struct NonFiniteError : std::runtime_error {
  explicit NonFiniteError(const std::string& m) : std::runtime_error(m) {}
};
struct UndefinedMetricError : std::runtime_error {
  explicit UndefinedMetricError(const std::string& m) : std::runtime_error(m) {}
};
struct SingularPivotError : std::runtime_error {
  Index pivot_index;
  double pivot_magnitude;
  int cluster;
  int level;
  SingularPivotError(const std::string& m, Index idx, double mag, int cl = -1, int lv = -1)
      : std::runtime_error(m), pivot_index(idx), pivot_magnitude(mag), cluster(cl), level(lv) {}
};

// Column-major complex128 matrix (same memory layout as Eigen::MatrixXcd).
struct Mat {
  Index r = 0, c = 0;
  std::vector<cxd> d;
  Mat() = default;
  Mat(Index rows, Index cols) : r(rows), c(cols), d(static_cast<size_t>(rows * cols)) {}
  Index rows() const { return r; }
  Index cols() const { return c; }
  Index size() const { return r * c; }
  cxd& operator()(Index i, Index j) { return d[static_cast<size_t>(i + j * r)]; }
  const cxd& operator()(Index i, Index j) const { return d[static_cast<size_t>(i + j * r)]; }
  cxd* col(Index j) { return d.data() + j * r; }
  const cxd* col(Index j) const { return d.data() + j * r; }

  static Mat identity(Index n) {
    Mat I(n, n);
    for (Index i = 0; i < n; ++i) I(i, i) = 1.0;
    return I;
  }
  static Mat identity(Index m, Index n) {
    Mat I(m, n);
    for (Index i = 0; i < std::min(m, n); ++i) I(i, i) = 1.0;
    return I;
  }
  Mat block(Index i0, Index j0, Index m, Index n) const {
    Mat B(m, n);
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i < m; ++i) B(i, j) = (*this)(i0 + i, j0 + j);
    return B;
  }
  void set_block(Index i0, Index j0, const Mat& B) {
    for (Index j = 0; j < B.c; ++j)
      for (Index i = 0; i < B.r; ++i) (*this)(i0 + i, j0 + j) = B(i, j);
  }
  // this[i0.., j0..] += alpha * B
  void add_block(Index i0, Index j0, const Mat& B, double alpha = 1.0) {
    for (Index j = 0; j < B.c; ++j)
      for (Index i = 0; i < B.r; ++i) (*this)(i0 + i, j0 + j) += alpha * B(i, j);
  }
  void zero_block(Index i0, Index j0, Index m, Index n) {
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i < m; ++i) (*this)(i0 + i, j0 + j) = 0.0;
  }
  Mat left_cols(Index n) const { return block(0, 0, r, n); }
  Mat right_cols(Index n) const { return block(0, c - n, r, n); }
  Mat top_rows(Index m) const { return block(0, 0, m, c); }
  Mat bottom_rows(Index m) const { return block(r - m, 0, m, c); }
  Mat adjoint() const {
    Mat T(c, r);
    for (Index j = 0; j < c; ++j)
      for (Index i = 0; i < r; ++i) T(j, i) = std::conj((*this)(i, j));
    return T;
  }
  Mat transpose() const {
    Mat T(c, r);
    for (Index j = 0; j < c; ++j)
      for (Index i = 0; i < r; ++i) T(j, i) = (*this)(i, j);
    return T;
  }
  Mat conjugate() const {
    Mat T(r, c);
    for (size_t q = 0; q < d.size(); ++q) T.d[q] = std::conj(d[q]);
    return T;
  }
  double squared_norm() const {
    double s = 0.0;
    for (const cxd& v : d) s += std::norm(v);
    return s;
  }
  double norm() const { return std::sqrt(squared_norm()); }
  double max_abs() const {
    double m = 0.0;
    for (const cxd& v : d) m = std::max(m, std::abs(v));
    return m;
  }
  bool all_finite() const {
    for (const cxd& v : d)
      if (!std::isfinite(v.real()) || !std::isfinite(v.imag())) return false;
    return true;
  }
  Mat& operator+=(const Mat& B) {
    for (size_t q = 0; q < d.size(); ++q) d[q] += B.d[q];
    return *this;
  }
  Mat& operator-=(const Mat& B) {
    for (size_t q = 0; q < d.size(); ++q) d[q] -= B.d[q];
    return *this;
  }
  Mat operator-(const Mat& B) const {
    Mat R = *this;
    R -= B;
    return R;
  }
  Mat operator+(const Mat& B) const {
    Mat R = *this;
    R += B;
    return R;
  }
  Mat scaled(cxd a) const {
    Mat R = *this;
    for (cxd& v : R.d) v *= a;
    return R;
  }
};

// Summation-order switch for the oracle self-noise study (H2O_GEMM_ORDER=reverse
// accumulates the inner dimension last-to-first, as a differently blocked BLAS
// would): the same algorithm with rounding-level differences. Default: forward.
inline int& gemm_order_flag() {
  static int flag = [] {
    const char* e = std::getenv("H2O_GEMM_ORDER");
    return e && std::string(e) == "reverse" ? 1 : 0;
  }();
  return flag;
}
inline bool gemm_reverse_k() { return gemm_order_flag() != 0; }

// C += alpha * A * B (all column-major, plain). A and C are split into real
// and imaginary planes so the inner loops are pure FMA streams, and four
// columns of C share every load of A.
inline void gemm_acc(Mat& C, const Mat& A, const Mat& B, double alpha = 1.0) {
  if (A.c != B.r || C.r != A.r || C.c != B.c) throw InvalidInputError("gemm: shape mismatch");
  const Index m = A.r, n = B.c, k = A.c;
  if (m == 0 || n == 0 || k == 0) return;
  std::vector<double> ar(static_cast<size_t>(m * k)), ai(static_cast<size_t>(m * k));
  for (Index q = 0; q < m * k; ++q) ar[static_cast<size_t>(q)] = A.d[static_cast<size_t>(q)].real(), ai[static_cast<size_t>(q)] = A.d[static_cast<size_t>(q)].imag();
  // Each group of four C columns is computed start to finish by one thread,
  // so the arithmetic is the same for any thread count.
  const bool reverse_k = gemm_reverse_k();
  auto panel = [&](Index j0) {
    std::vector<double> cr(static_cast<size_t>(m * 4), 0.0), ci(static_cast<size_t>(m * 4), 0.0);
    const Index nj = std::min<Index>(4, n - j0);
    for (Index pp = 0; pp < k; ++pp) {
      const Index p = reverse_k ? k - 1 - pp : pp;
      const double* xr = ar.data() + p * m;
      const double* xi = ai.data() + p * m;
      for (Index jj = 0; jj < nj; ++jj) {
        const cxd bv = B(p, j0 + jj);
        const double br = bv.real(), bi = bv.imag();
        if (br == 0.0 && bi == 0.0) continue;
        double* yr = cr.data() + jj * m;
        double* yi = ci.data() + jj * m;
        for (Index i = 0; i < m; ++i) {
          yr[i] += xr[i] * br - xi[i] * bi;
          yi[i] += xr[i] * bi + xi[i] * br;
        }
      }
    }
    for (Index jj = 0; jj < nj; ++jj) {
      cxd* cj = C.col(j0 + jj);
      for (Index i = 0; i < m; ++i) cj[i] += alpha * cxd(cr[static_cast<size_t>(jj * m + i)], ci[static_cast<size_t>(jj * m + i)]);
    }
  };
  const Index groups = (n + 3) / 4;
  if (groups > 1 && m * n * k >= (Index(1) << 20)) {
    pool_for(groups, [&](int64_t g) { panel(static_cast<Index>(g) * 4); });
  } else {
    for (Index g = 0; g < groups; ++g) panel(g * 4);
  }
}

inline Mat mul(const Mat& A, const Mat& B) {
  Mat C(A.r, B.c);
  gemm_acc(C, A, B);
  return C;
}

// ---------------------------------------------------------------- Householder
// Reflector for x (length m): H x = beta e0, H = I - tau v v^H, v = [1; ess].
struct Reflector {
  cxd tau = 0.0;
  double beta = 0.0;
};

inline Reflector make_householder(cxd* x, Index m) {
  Reflector h;
  const cxd c0 = x[0];
  double tail_sq = 0.0;
  for (Index i = 1; i < m; ++i) tail_sq += std::norm(x[i]);
  const double tiny = std::numeric_limits<double>::min();
  if (tail_sq <= tiny && c0.imag() * c0.imag() <= tiny) {
    h.tau = 0.0;
    h.beta = c0.real();
    for (Index i = 1; i < m; ++i) x[i] = 0.0;
  } else {
    double beta = std::sqrt(std::norm(c0) + tail_sq);
    if (c0.real() >= 0.0) beta = -beta;
    const cxd denom = c0 - beta;
    for (Index i = 1; i < m; ++i) x[i] /= denom;
    h.tau = std::conj((beta - c0) / beta);
    h.beta = beta;
  }
  return h;
}

// A[row0.., col0..col1) = (I - tau v v^H) A, v = [1; ess], len = #rows.
inline void apply_householder_left(Mat& A, Index row0, Index col0, Index col1, const cxd* ess, Index len, cxd tau) {
  if (tau == cxd(0.0)) return;
  auto one = [&](Index j) {
    cxd* a = A.col(j) + row0;
    cxd t = a[0];
    for (Index i = 1; i < len; ++i) t += std::conj(ess[i - 1]) * a[i];
    t *= tau;
    a[0] -= t;
    for (Index i = 1; i < len; ++i) a[i] -= ess[i - 1] * t;
  };
  // columns are independent: one thread per column, serial arithmetic
  if ((col1 - col0) > 1 && (col1 - col0) * len >= (Index(1) << 16)) {
    pool_for(col1 - col0, [&](int64_t j) { one(col0 + static_cast<Index>(j)); });
  } else {
    for (Index j = col0; j < col1; ++j) one(j);
  }
}

// Compact Householder QR of A (m x n): R in the upper triangle, reflectors
// below, tau per column.
struct HouseholderQR {
  Mat qr;
  std::vector<cxd> tau;
  explicit HouseholderQR(const Mat& A) : qr(A) {
    const Index m = qr.r, n = qr.c, s = std::min(m, n);
    tau.assign(static_cast<size_t>(s), 0.0);
    for (Index k = 0; k < s; ++k) {
      cxd* x = qr.col(k) + k;
      Reflector h = make_householder(x, m - k);
      tau[static_cast<size_t>(k)] = h.tau;
      x[0] = h.beta;
      apply_householder_left(qr, k, k + 1, n, x + 1, m - k, h.tau);
    }
  }
  // R (min(m,n) x n), upper triangular part.
  Mat matrix_r() const {
    const Index s = std::min(qr.r, qr.c);
    Mat R(s, qr.c);
    for (Index j = 0; j < qr.c; ++j)
      for (Index i = 0; i <= std::min(j, s - 1); ++i) R(i, j) = qr(i, j);
    return R;
  }
  // First `ncols` columns of Q = H_0^H H_1^H ... (m x ncols).
  Mat q_cols(Index ncols) const {
    const Index m = qr.r, s = std::min(qr.r, qr.c);
    Mat Q = Mat::identity(m, ncols);
    for (Index k = s - 1; k >= 0; --k)
      apply_householder_left(Q, k, 0, ncols, qr.col(k) + k + 1, m - k, std::conj(tau[static_cast<size_t>(k)]));
    return Q;
  }
};

// ------------------------------------------------------------------ Jacobi SVD
// Left singular vectors and singular values of a square-or-tall M by one-sided
// Jacobi on its columns: M V = U Sigma. Values sorted descending.
struct SVDResult {
  Mat U;                     // m x min(m, n)
  std::vector<double> sigma; // min(m, n), descending
};

inline SVDResult jacobi_svd_left(const Mat& Min) {
  Mat M = Min;
  const Index m = M.r, n = M.c;
  const double tol = 4.0 * std::numeric_limits<double>::epsilon();
  for (int sweep = 0; sweep < 80; ++sweep) {
    bool rotated = false;
    for (Index p = 0; p < n - 1; ++p) {
      for (Index q = p + 1; q < n; ++q) {
        cxd* mp = M.col(p);
        cxd* mq = M.col(q);
        double a = 0.0, b = 0.0;
        cxd g = 0.0;
        for (Index i = 0; i < m; ++i) {
          a += std::norm(mp[i]);
          b += std::norm(mq[i]);
          g += std::conj(mp[i]) * mq[i];
        }
        const double ga = std::abs(g);
        if (ga == 0.0 || ga <= tol * std::sqrt(a * b)) continue;
        rotated = true;
        const cxd ph = g / ga;  // e^{i phi}
        const double zeta = (b - a) / (2.0 * ga);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / std::sqrt(1.0 + t * t);
        const double sn = cs * t;
        for (Index i = 0; i < m; ++i) {
          const cxd xp = mp[i];
          const cxd xq = mq[i] * std::conj(ph);
          mp[i] = cs * xp - sn * xq;
          mq[i] = (sn * xp + cs * xq) * ph;
        }
      }
    }
    if (!rotated) break;
  }
  std::vector<double> nrm(static_cast<size_t>(n));
  for (Index j = 0; j < n; ++j) {
    double s = 0.0;
    for (Index i = 0; i < m; ++i) s += std::norm(M(i, j));
    nrm[static_cast<size_t>(j)] = std::sqrt(s);
  }
  std::vector<Index> order(static_cast<size_t>(n));
  for (Index j = 0; j < n; ++j) order[static_cast<size_t>(j)] = j;
  std::stable_sort(order.begin(), order.end(),
                   [&](Index x, Index y) { return nrm[static_cast<size_t>(x)] > nrm[static_cast<size_t>(y)]; });
  const Index s = std::min(m, n);
  SVDResult out;
  out.U = Mat(m, s);
  out.sigma.resize(static_cast<size_t>(s));
  for (Index q = 0; q < s; ++q) {
    const Index j = order[static_cast<size_t>(q)];
    const double sv = nrm[static_cast<size_t>(j)];
    out.sigma[static_cast<size_t>(q)] = sv;
    if (sv > 0.0)
      for (Index i = 0; i < m; ++i) out.U(i, q) = M(i, j) / sv;
  }
  return out;
}

// proj/include/h2lu/dense_kernels.hpp:51-65 — [V_perp V] unitary.
inline Mat unitary_completion(const Mat& V) {
  const Index m = V.r, k = V.c;
  if (k > m) throw InvalidInputError("unitary_completion: more columns than rows");
  if (k > 0) {
    Mat G = mul(V.adjoint(), V);
    double defect = 0.0;
    for (Index j = 0; j < k; ++j)
      for (Index i = 0; i < k; ++i) defect = std::max(defect, std::abs(G(i, j) - (i == j ? cxd(1.0) : cxd(0.0))));
    if (defect > 1e-10)
      throw InvalidInputError("unitary_completion: input columns are not orthonormal (defect " + std::to_string(defect) + ")");
  }
  if (k == 0) return Mat::identity(m);
  if (k == m) return Mat(m, 0);
  HouseholderQR qr(V);
  Mat Q = qr.q_cols(m);
  return Q.right_cols(m - k);
}

// proj/include/h2lu/dense_kernels.hpp:70-93 — unpivoted right-looking LU with
// the relative pivot test |piv| < tol * max|F|.
inline std::pair<Mat, Mat> partial_lu(const Mat& F, double pivot_tol = 1e-13) {
  if (F.r != F.c) throw InvalidInputError("partial_lu: matrix must be square");
  const Index n = F.r;
  Mat A = F;
  const double scale = n > 0 ? F.max_abs() : 0.0;
  if (n > 0 && scale == 0.0) throw SingularPivotError("partial_lu: zero matrix", 0, 0.0);
  for (Index k = 0; k < n; ++k) {
    const cxd piv = A(k, k);
    if (std::abs(piv) < pivot_tol * scale)
      throw SingularPivotError("partial_lu: pivot " + std::to_string(k) + " below tolerance", k, std::abs(piv));
    if (k + 1 < n) {
      for (Index i = k + 1; i < n; ++i) A(i, k) /= piv;
      for (Index j = k + 1; j < n; ++j) {
        const cxd u = A(k, j);
        for (Index i = k + 1; i < n; ++i) A(i, j) -= A(i, k) * u;
      }
    }
  }
  Mat L = Mat::identity(n), U(n, n);
  for (Index j = 0; j < n; ++j) {
    for (Index i = j + 1; i < n; ++i) L(i, j) = A(i, j);
    for (Index i = 0; i <= j; ++i) U(i, j) = A(i, j);
  }
  return {std::move(L), std::move(U)};
}

// X = L^{-1} B, L unit lower triangular.
inline Mat solve_unit_lower(const Mat& L, const Mat& B) {
  Mat X = B;
  const Index n = L.r;
  for (Index j = 0; j < X.c; ++j) {
    cxd* x = X.col(j);
    for (Index p = 0; p < n; ++p) {
      const cxd v = x[p];
      if (v == cxd(0.0)) continue;
      for (Index i = p + 1; i < n; ++i) x[i] -= L(i, p) * v;
    }
  }
  return X;
}

// X = U^{-1} B, U upper triangular.
inline Mat solve_upper(const Mat& U, const Mat& B) {
  Mat X = B;
  const Index n = U.r;
  for (Index j = 0; j < X.c; ++j) {
    cxd* x = X.col(j);
    for (Index p = n - 1; p >= 0; --p) {
      x[p] /= U(p, p);
      const cxd v = x[p];
      if (v == cxd(0.0)) continue;
      for (Index i = 0; i < p; ++i) x[i] -= U(i, p) * v;
    }
  }
  return X;
}

// X = B U^{-1}, U upper triangular (row-side solve of factorization.hpp:407).
inline Mat solve_right_upper(const Mat& B, const Mat& U) {
  Mat X = B;
  const Index n = U.r;
  for (Index j = 0; j < n; ++j) {
    cxd* xj = X.col(j);
    for (Index p = 0; p < j; ++p) {
      const cxd u = U(p, j);
      if (u == cxd(0.0)) continue;
      const cxd* xp = X.col(p);
      for (Index i = 0; i < X.r; ++i) xj[i] -= xp[i] * u;
    }
    const cxd piv = U(j, j);
    for (Index i = 0; i < X.r; ++i) xj[i] /= piv;
  }
  return X;
}

// Row-pivoted LU solve (verify.hpp:23-31 dense_oracle_solve; solve checks).
inline Mat pivoted_lu_solve(const Mat& Ain, const Mat& B) {
  if (Ain.r != Ain.c || B.r != Ain.r) throw InvalidInputError("pivoted_lu_solve: shape mismatch");
  Mat A = Ain, X = B;
  const Index n = A.r;
  for (Index k = 0; k < n; ++k) {
    Index p = k;
    double best = std::abs(A(k, k));
    for (Index i = k + 1; i < n; ++i)
      if (std::abs(A(i, k)) > best) best = std::abs(A(i, k)), p = i;
    if (p != k) {
      for (Index j = 0; j < n; ++j) std::swap(A(k, j), A(p, j));
      for (Index j = 0; j < X.c; ++j) std::swap(X(k, j), X(p, j));
    }
    const cxd piv = A(k, k);
    if (piv == cxd(0.0)) continue;
    for (Index i = k + 1; i < n; ++i) A(i, k) /= piv;
    for (Index j = k + 1; j < n; ++j) {
      const cxd u = A(k, j);
      if (u == cxd(0.0)) continue;
      for (Index i = k + 1; i < n; ++i) A(i, j) -= A(i, k) * u;
    }
  }
  Mat L = Mat::identity(n), U(n, n);
  for (Index j = 0; j < n; ++j) {
    for (Index i = j + 1; i < n; ++i) L(i, j) = A(i, j);
    for (Index i = 0; i <= j; ++i) U(i, j) = A(i, j);
  }
  return solve_upper(U, solve_unit_lower(L, X));
}

}  // namespace h2o
