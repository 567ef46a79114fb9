// Device building blocks for the H² factorization on sm_100a: complex128
// arithmetic, CTA-cooperative dense kernels (small GEMM, Householder QR,
// two-sided Hermitian Jacobi, unpivoted LU with the reference pivot rule,
// triangular inverses). All routines take generic pointers so a matrix can
// live in shared memory (b <= 64) or in a global-memory workspace.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace h2g {

typedef double2 cplx;

__device__ __forceinline__ cplx cmk(double r, double i) { return make_double2(r, i); }
__device__ __forceinline__ cplx czero() { return make_double2(0.0, 0.0); }
__device__ __forceinline__ cplx cone() { return make_double2(1.0, 0.0); }
__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ cplx csub(cplx a, cplx b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ cplx cmul(cplx a, cplx b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ cplx cconj(cplx a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ cplx cscale(cplx a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double cabs2(cplx a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ double cabsd(cplx a) { return hypot(a.x, a.y); }
// acc += a * b
__device__ __forceinline__ void cfma(cplx& acc, cplx a, cplx b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
// a / b with Smith's scaling
__device__ __forceinline__ cplx cdiv(cplx a, cplx b) {
  if (fabs(b.x) >= fabs(b.y)) {
    const double r = b.y / b.x, d = b.x + b.y * r;
    return make_double2((a.x + a.y * r) / d, (a.y - a.x * r) / d);
  }
  const double r = b.x / b.y, d = b.y + b.x * r;
  return make_double2((a.x * r + a.y) / d, (a.y * r - a.x) / d);
}

// Device error word: first failure wins (code 0 = none).
struct DevError {
  int code;
  int cluster;
  int level;
  int pad;
  long long pivot_index;
  double pivot_magnitude;
};

__device__ __forceinline__ void raise_error(DevError* e, int code, int cluster, int level, long long piv, double mag) {
  if (atomicCAS(&e->code, 0, code) == 0) {
    e->cluster = cluster;
    e->level = level;
    e->pivot_index = piv;
    e->pivot_magnitude = mag;
    __threadfence();
  }
}

// op codes: 'N' plain, 'T' transpose, 'C' conjugate transpose, 'R' conjugate
enum Op { OP_N = 0, OP_T = 1, OP_C = 2, OP_R = 3 };

__device__ __forceinline__ cplx ld_op(const cplx* A, int lda, int op, int i, int p) {
  switch (op) {
    case OP_N:
      return A[i + (size_t)p * lda];
    case OP_T:
      return A[p + (size_t)i * lda];
    case OP_C:
      return cconj(A[p + (size_t)i * lda]);
    default:
      return cconj(A[i + (size_t)p * lda]);
  }
}

// C (m x n) = alpha * op(A) (m x k) * op(B) (k x n) + beta * C, cooperative
// over the CTA. C must not alias A or B. Caller syncs.
__device__ inline void cta_gemm(int m, int n, int k, double alpha, const cplx* A, int lda, int opA, const cplx* B, int ldb,
                                int opB, double beta, cplx* C, int ldc) {
  for (int idx = threadIdx.x; idx < m * n; idx += blockDim.x) {
    const int i = idx % m, j = idx / m;
    cplx s = czero();
    for (int p = 0; p < k; ++p) cfma(s, ld_op(A, lda, opA, i, p), ld_op(B, ldb, opB, p, j));
    cplx* c = C + i + (size_t)j * ldc;
    if (beta == 0.0)
      *c = cscale(s, alpha);
    else
      *c = make_double2(beta * c->x + alpha * s.x, beta * c->y + alpha * s.y);
  }
}

__device__ inline void cta_copy(int m, int n, const cplx* S, int lds, cplx* D, int ldd) {
  for (int idx = threadIdx.x; idx < m * n; idx += blockDim.x) {
    const int i = idx % m, j = idx / m;
    D[i + (size_t)j * ldd] = S[i + (size_t)j * lds];
  }
}

__device__ inline void cta_fill(int m, int n, cplx* D, int ldd, cplx v) {
  for (int idx = threadIdx.x; idx < m * n; idx += blockDim.x) D[(idx % m) + (size_t)(idx / m) * ldd] = v;
}

__device__ inline void cta_identity(int m, int n, cplx* D, int ldd) {
  for (int idx = threadIdx.x; idx < m * n; idx += blockDim.x) {
    const int i = idx % m, j = idx / m;
    D[i + (size_t)j * ldd] = i == j ? cone() : czero();
  }
}

// Block-wide sum / max of a double (all threads get the result).
__device__ inline double cta_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < nw; ++i) s += red[i];
  __syncthreads();
  return s;
}

__device__ inline double cta_max(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < nw; ++i) s = fmax(s, red[i]);
  __syncthreads();
  return s;
}

// A (rows x m, ld lda) <- A * Q where Q = H_0^H H_1^H ... H_{s-1}^H is stored
// compactly in QR (m x s, ld ldq; essential parts below the diagonal) and tau.
__device__ inline void cta_apply_q_right(int rows, int m, int s, cplx* A, int lda, const cplx* QR, int ldq, const cplx* tau, cplx* tmp) {
  for (int k = 0; k < s; ++k) {
    const cplx tk = cconj(tau[k]);
    if (tk.x == 0.0 && tk.y == 0.0) continue;
    const cplx* v = QR + k + (size_t)k * ldq;  // v[0] = 1 implicit
    // t_i = sum_j A[i, k + j] v_j
    for (int i = threadIdx.x; i < rows; i += blockDim.x) {
      cplx t = A[i + (size_t)k * lda];
      for (int j = 1; j < m - k; ++j) cfma(t, A[i + (size_t)(k + j) * lda], v[j]);
      tmp[i] = cmul(t, tk);
    }
    __syncthreads();
    // A[:, k + j] -= t conj(v_j)
    for (int idx = threadIdx.x; idx < rows * (m - k); idx += blockDim.x) {
      const int i = idx % rows, j = idx / rows;
      const cplx vj = j == 0 ? cone() : v[j];
      cplx* a = A + i + (size_t)(k + j) * lda;
      *a = csub(*a, cmul(tmp[i], cconj(vj)));
    }
    __syncthreads();
  }
}

// Compact Householder QR of A (m x n, ld lda) in place with the Eigen
// HouseholderQR convention (H = I - tau v v^H, v0 = 1, beta = -sign(Re c0)|x|),
// then Q (m x m, ld ldq) = H_0^H ... H_{s-1}^H. tau: s entries of scratch.
__device__ inline void cta_householder_qr(int m, int n, cplx* A, int lda, cplx* tau, double* red) {
  const int s = min(m, n);
  for (int k = 0; k < s; ++k) {
    cplx* x = A + k + (size_t)k * lda;
    double part = 0.0;
    for (int i = 1 + threadIdx.x; i < m - k; i += blockDim.x) part += cabs2(x[i]);
    const double tail = cta_sum(part, red);
    const cplx c0 = x[0];
    __shared__ cplx s_denom, s_tau;
    __shared__ double s_beta;
    __shared__ int s_triv;
    if (threadIdx.x == 0) {
      const double tiny = 2.2250738585072014e-308;
      if (tail <= tiny && c0.y * c0.y <= tiny) {
        s_triv = 1;
        s_tau = czero();
        s_beta = c0.x;
      } else {
        double beta = sqrt(cabs2(c0) + tail);
        if (c0.x >= 0.0) beta = -beta;
        s_triv = 0;
        s_beta = beta;
        s_denom = csub(c0, cmk(beta, 0.0));
        s_tau = cconj(cdiv(csub(cmk(beta, 0.0), c0), cmk(beta, 0.0)));
      }
      tau[k] = s_tau;
    }
    __syncthreads();
    const int triv = s_triv;
    const cplx denom = s_denom, tk = s_tau;
    const cplx rden = triv ? czero() : cdiv(cone(), denom);
    for (int i = 1 + threadIdx.x; i < m - k; i += blockDim.x) x[i] = triv ? czero() : cmul(x[i], rden);
    __syncthreads();
    // apply H to A[k:, k+1:]: one warp per column
    if (!triv) {
      const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
      for (int j = k + 1 + w; j < n; j += nw) {
        cplx* a = A + k + (size_t)j * lda;
        cplx t = czero();
        for (int i = 1 + lane; i < m - k; i += 32) cfma(t, cconj(x[i]), a[i]);
        for (int o = 16; o > 0; o >>= 1) {
          t.x += __shfl_xor_sync(0xffffffffu, t.x, o);
          t.y += __shfl_xor_sync(0xffffffffu, t.y, o);
        }
        t = cmul(tk, cadd(t, a[0]));
        __syncwarp();
        if (lane == 0) a[0] = csub(a[0], t);
        for (int i = 1 + lane; i < m - k; i += 32) a[i] = csub(a[i], cmul(x[i], t));
        __syncwarp();
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) x[0] = cmk(s_beta, 0.0);
    __syncthreads();
  }
}

__device__ inline void cta_householder_q(int m, int n, cplx* A, int lda, cplx* Q, int ldq, cplx* tau, double* red) {
  const int s = min(m, n);
  cta_householder_qr(m, n, A, lda, tau, red);
  // Q = H_0^H H_1^H ... H_{s-1}^H applied to I
  cta_identity(m, m, Q, ldq);
  __syncthreads();
  for (int k = s - 1; k >= 0; --k) {
    const cplx* v = A + k + (size_t)k * lda;  // v[0] is beta; essential part v[1..]
    const cplx tk = cconj(tau[k]);
    if (tk.x == 0.0 && tk.y == 0.0) continue;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int j = k + w; j < m; j += nw) {
      cplx* q = Q + k + (size_t)j * ldq;
      cplx t = czero();
      for (int i = 1 + lane; i < m - k; i += 32) cfma(t, cconj(v[i]), q[i]);
      for (int o = 16; o > 0; o >>= 1) {
        t.x += __shfl_xor_sync(0xffffffffu, t.x, o);
        t.y += __shfl_xor_sync(0xffffffffu, t.y, o);
      }
      t = cmul(tk, cadd(t, q[0]));
      __syncwarp();
      if (lane == 0) q[0] = csub(q[0], t);
      for (int i = 1 + lane; i < m - k; i += 32) q[i] = csub(q[i], cmul(v[i], t));
      __syncwarp();
    }
    __syncthreads();
  }
}

// Two-sided cyclic Jacobi on a Hermitian n x n matrix H (ld n), round-robin
// parallel ordering. On exit H is (numerically) diagonal and U (ld n) holds
// the eigenvectors: H_in = U diag(H_out) U^H. rot: scratch of 4*((n+1)/2) doubles.
// A pair rotates while |h_pq| > 1e-15 sqrt(|h_pp h_qq|) (relative accuracy
// for graded matrices) and |h_pq| > absfloor (entries below the caller's
// resolution floor are left alone, so noise-level blocks do not keep the
// sweeps going).
__device__ inline void cta_jacobi_eig(int n, cplx* H, cplx* U, double* rot, int* pr, double* red, double absfloor = 0.0) {
  cta_identity(n, n, U, n);
  __syncthreads();
  if (n <= 1) return;
  const int n2 = (n + 1) & ~1;
  const int npair = n2 / 2;
  double* rc = rot;
  double* rs = rot + npair;
  double* rphr = rot + 2 * npair;
  double* rphi = rot + 3 * npair;
  __shared__ int s_rot;
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (threadIdx.x == 0) s_rot = 0;
    __syncthreads();
    for (int r = 0; r < n2 - 1; ++r) {
      for (int i = threadIdx.x; i < npair; i += blockDim.x) {
        int p, q;
        if (i == 0) {
          p = r;
          q = n2 - 1;
        } else {
          p = (r + i) % (n2 - 1);
          q = (r - i + (n2 - 1)) % (n2 - 1);
        }
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        pr[2 * i] = p;
        pr[2 * i + 1] = q;
        double c = 1.0, s = 0.0, phr = 1.0, phi = 0.0;
        if (q < n) {
          const cplx g = H[p + q * n];
          const double ga = cabsd(g);
          const double a = H[p + p * n].x, d = H[q + q * n].x;
          // relative criterion (keeps small eigenvalues of graded matrices accurate)
          if (ga > 1e-300 && ga > absfloor && ga > 1e-15 * sqrt(fabs(a) * fabs(d))) {
            s_rot = 1;
            phr = g.x / ga;
            phi = g.y / ga;
            const double th = (d - a) / (2.0 * ga);
            const double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
          }
        }
        rc[i] = c;
        rs[i] = s;
        rphr[i] = phr;
        rphi[i] = phi;
      }
      __syncthreads();
      // rows: [H_px; H_qx] <- J^H [H_px; H_qx], J^H = [[c, -s e^{i phi}], [s, c e^{i phi}]]
      for (int idx = threadIdx.x; idx < npair * n; idx += blockDim.x) {
        const int i = idx % npair, x = idx / npair;
        const int p = pr[2 * i], q = pr[2 * i + 1];
        if (q >= n || rs[i] == 0.0) continue;
        const double c = rc[i], s = rs[i];
        const cplx ph = cmk(rphr[i], rphi[i]);
        const cplx hp = H[p + x * n], hq = H[q + x * n];
        const cplx ehq = cmul(ph, hq);
        H[p + x * n] = csub(cscale(hp, c), cscale(ehq, s));
        H[q + x * n] = cadd(cscale(hp, s), cscale(ehq, c));
      }
      __syncthreads();
      // columns: [H_xp, H_xq] <- [H_xp, H_xq] J, J = [[c, s], [-s e^{-i phi}, c e^{-i phi}]]
      for (int idx = threadIdx.x; idx < npair * n; idx += blockDim.x) {
        const int i = idx % npair, x = idx / npair;
        const int p = pr[2 * i], q = pr[2 * i + 1];
        if (q >= n || rs[i] == 0.0) continue;
        const double c = rc[i], s = rs[i];
        const cplx phc = cmk(rphr[i], -rphi[i]);
        {
          const cplx hp = H[x + p * n], hq = H[x + q * n];
          const cplx ehq = cmul(phc, hq);
          H[x + p * n] = csub(cscale(hp, c), cscale(ehq, s));
          H[x + q * n] = cadd(cscale(hp, s), cscale(ehq, c));
        }
        {
          const cplx up = U[x + p * n], uq = U[x + q * n];
          const cplx euq = cmul(phc, uq);
          U[x + p * n] = csub(cscale(up, c), cscale(euq, s));
          U[x + q * n] = cadd(cscale(up, s), cscale(euq, c));
        }
      }
      __syncthreads();
    }
    if (!s_rot) break;
    __syncthreads();
  }
}

// Unpivoted LU in place (n x n, ld lda) with the reference pivot rule
// |piv| < tol * max|F| (dense_kernels.hpp:70-93). Returns -1 on success or
// the failing pivot index (magnitude in *pmag). All threads return the same.
__device__ inline int cta_lu_nopiv(int n, cplx* A, int lda, double tol, double* pmag, double* red) {
  double mx = 0.0;
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) mx = fmax(mx, cabsd(A[(idx % n) + (size_t)(idx / n) * lda]));
  const double scale = cta_max(mx, red);
  if (n > 0 && scale == 0.0) {
    *pmag = 0.0;
    return 0;
  }
  for (int k = 0; k < n; ++k) {
    const cplx piv = A[k + (size_t)k * lda];
    const double pa = cabsd(piv);
    if (pa < tol * scale) {
      *pmag = pa;
      return k;
    }
    for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) A[i + (size_t)k * lda] = cdiv(A[i + (size_t)k * lda], piv);
    __syncthreads();
    const int r = n - k - 1;
    for (int idx = threadIdx.x; idx < r * r; idx += blockDim.x) {
      const int i = k + 1 + idx % r, j = k + 1 + idx / r;
      cplx a = A[i + (size_t)j * lda];
      const cplx l = A[i + (size_t)k * lda], u = A[k + (size_t)j * lda];
      a.x -= l.x * u.x - l.y * u.y;
      a.y -= l.x * u.y + l.y * u.x;
      A[i + (size_t)j * lda] = a;
    }
    __syncthreads();
  }
  return -1;
}

// Inverses of the unit-lower L and upper U stored packed in LU (n x n):
// Li = L^{-1}, Ui = U^{-1} (both n x n, ld n). One thread per column.
__device__ inline void cta_tri_inverses(int n, const cplx* LU, int ld, cplx* Li, cplx* Ui) {
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    // L x = e_j
    for (int i = 0; i < n; ++i) {
      cplx x = i == j ? cone() : czero();
      if (i > j)
        for (int p = j; p < i; ++p) {
          const cplx l = LU[i + (size_t)p * ld], xp = Li[p + (size_t)j * n];
          x.x -= l.x * xp.x - l.y * xp.y;
          x.y -= l.x * xp.y + l.y * xp.x;
        }
      Li[i + (size_t)j * n] = i < j ? czero() : x;
    }
    // U x = e_j
    for (int i = n - 1; i >= 0; --i) {
      cplx x = i == j ? cone() : czero();
      if (i <= j) {
        for (int p = i + 1; p <= j; ++p) {
          const cplx u = LU[i + (size_t)p * ld], xp = Ui[p + (size_t)j * n];
          x.x -= u.x * xp.x - u.y * xp.y;
          x.y -= u.x * xp.y + u.y * xp.x;
        }
        x = cdiv(x, LU[i + (size_t)i * ld]);
      }
      Ui[i + (size_t)j * n] = i > j ? czero() : x;
    }
  }
}

}  // namespace h2g

namespace h2g {

// ---------------------------------------------------------------------------
// Hermitian eigen-solver for the step-0 truncation: Householder reduction to
// a real symmetric tridiagonal T = Q^H H Q (zhetd2 scheme), Sturm-count
// bisection for the eigenvalues that matter, inverse iteration for the
// retained eigenvectors, back-transformation by the stored reflectors.
// H (n x n, ld n, full storage) is overwritten by the reflectors; d, e real
// (n), tau complex (n), p/w complex scratch (n).
__device__ inline void cta_hetrd(int n, cplx* H, double* d, double* e, cplx* tau, cplx* p, cplx* w, double* red) {
  __shared__ cplx s_tau, s_scale;
  __shared__ double s_beta;
  __shared__ int s_skip;
  for (int k = 0; k + 1 < n; ++k) {
    const int nk = n - k - 1;
    cplx* x = H + (k + 1) + (size_t)k * n;  // x[0] = H[k+1,k]
    double part = 0.0;
    for (int i = 1 + threadIdx.x; i < nk; i += blockDim.x) part += cabs2(x[i]);
    const double xn2 = cta_sum(part, red);
    if (threadIdx.x == 0) {
      const cplx al = x[0];
      if (xn2 == 0.0 && al.y == 0.0) {
        s_skip = 1;
        s_tau = czero();
        s_beta = al.x;
      } else {
        double beta = sqrt(cabs2(al) + xn2);
        if (al.x >= 0.0) beta = -beta;
        s_skip = 0;
        s_beta = beta;
        s_tau = cdiv(csub(cmk(beta, 0.0), al), cmk(beta, 0.0));
        s_scale = cdiv(cone(), csub(al, cmk(beta, 0.0)));
      }
      tau[k] = s_tau;
      d[k] = H[k + (size_t)k * n].x;
      e[k] = s_beta;
    }
    __syncthreads();
    if (s_skip) continue;
    const cplx tk = s_tau, sc = s_scale;
    for (int i = 1 + threadIdx.x; i < nk; i += blockDim.x) x[i] = cmul(x[i], sc);
    __syncthreads();
    // p = tau * A22 v, A22 = H[k+1:, k+1:], v = [1; x[1:]]: rows split over
    // warps' lanes, columns over SL slices, partial sums reduced through w
    const cplx* A22 = H + (k + 1) + (size_t)(k + 1) * n;
    {
      const int SL = blockDim.x >= 512 ? 8 : 4;
      const int per = blockDim.x / SL;
      const int sl = threadIdx.x / per, li = threadIdx.x % per;
      const int jc = (nk + SL - 1) / SL;
      const int j0 = sl * jc, j1 = min(nk, j0 + jc);
      for (int i0 = 0; i0 < nk; i0 += per) {
        const int i = i0 + li;
        cplx s = czero();
        if (i < nk)
          for (int j = j0; j < j1; ++j) cfma(s, A22[i + (size_t)j * n], j == 0 ? cone() : x[j]);
        if (sl == 0 && i < nk) p[i] = s;
        __syncthreads();
        for (int q2 = 1; q2 < SL; ++q2) {
          if (sl == q2 && i < nk) p[i] = cadd(p[i], s);
          __syncthreads();
        }
      }
      for (int i = threadIdx.x; i < nk; i += blockDim.x) p[i] = cmul(tk, p[i]);
    }
    __syncthreads();
    // c = v^H p ; w = p - 1/2 conj(tau) c v
    double cr = 0.0, ci = 0.0;
    for (int i = threadIdx.x; i < nk; i += blockDim.x) {
      const cplx v = i == 0 ? cone() : x[i];
      const cplx t = cmul(cconj(v), p[i]);
      cr += t.x;
      ci += t.y;
    }
    cr = cta_sum(cr, red);
    ci = cta_sum(ci, red);
    const cplx hc = cscale(cmul(cconj(tk), cmk(cr, ci)), 0.5);
    for (int i = threadIdx.x; i < nk; i += blockDim.x) {
      const cplx v = i == 0 ? cone() : x[i];
      w[i] = csub(p[i], cmul(hc, v));
    }
    __syncthreads();
    // A22 -= v w^H + w v^H
    cplx* B = H + (k + 1) + (size_t)(k + 1) * n;
    for (int idx = threadIdx.x; idx < nk * nk; idx += blockDim.x) {
      const int i = idx % nk, j = idx / nk;
      const cplx vi = i == 0 ? cone() : x[i], vj = j == 0 ? cone() : x[j];
      cplx a = B[i + (size_t)j * n];
      a = csub(a, cmul(vi, cconj(w[j])));
      a = csub(a, cmul(w[i], cconj(vj)));
      B[i + (size_t)j * n] = a;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    d[n - 1] = H[(n - 1) + (size_t)(n - 1) * n].x;
    if (n >= 1) e[n - 1] = 0.0;
  }
  __syncthreads();
}

// Number of eigenvalues of T (d, e: off-diagonal e[0..n-2]) strictly below x.
__device__ inline int sturm_count(int n, const double* d, const double* e, double x, double pivmin) {
  int c = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  if (q < 0) ++c;
  for (int i = 1; i < n; ++i) {
    q = d[i] - x - e[i - 1] * e[i - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    if (q < 0) ++c;
  }
  return c;
}

// 1/q to ~1 ulp: hardware reciprocal seed + two Newton steps (a fraction of
// the latency of a correctly rounded division on the FP64 pipe).
__device__ __forceinline__ double rcp_nr(double q) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  double e = fma(-q, r, 1.0);
  r = fma(r, e, r);
  e = fma(-q, r, 1.0);
  return fma(r, e, r);
}

// Sturm counts at P shifts at once: P independent recurrences interleaved so
// the dependent FP64 chains overlap. e2[i] = e[i]^2.
template <int P>
__device__ __forceinline__ void sturm_count_p(int n, const double* d, const double* e2, const double* x, double pivmin, int* c) {
  double q[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    q[p] = d[0] - x[p];
    if (fabs(q[p]) < pivmin) q[p] = -pivmin;
    c[p] = q[p] < 0.0;
  }
  for (int i = 1; i < n; ++i) {
    const double di = d[i], ei = e2[i - 1];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      q[p] = (di - x[p]) - ei * rcp_nr(q[p]);
      if (fabs(q[p]) < pivmin) q[p] = -pivmin;
      c[p] += q[p] < 0.0;
    }
  }
}

// Eigenvalues with descending index j = 0..r-1 (ascending index n-1-j) of T,
// out[j], by multisection: G lanes of one warp per eigenvalue, 4 shifts per
// lane, so every round shrinks the bracket (4G+1)-fold; stops at a relative
// width of 1e-13 like bisect_eig. Whole CTA; no block barriers inside.
// part / nparts: this CTA computes the eigenvalues j = part, part + nparts, ...
// (the CTAs of a cluster share the work).
__device__ inline void multisect_top(int n, const double* d, const double* e2, int r, double lo0, double hi0, double pivmin, double* out,
                                     int part = 0, int nparts = 1) {
  constexpr int P = 2;  // 2 shifts per lane: latency and FP64 throughput of the counts balance
  const int cnt = r > part ? (r - part + nparts - 1) / nparts : 0;
  int G = 32;
  while (G > 1 && G * cnt > (int)blockDim.x) G >>= 1;
  const int slots = blockDim.x / G;
  const int glane = (threadIdx.x & 31) % G, gid = threadIdx.x / G;
  const int npts = G * P;
  for (int j0 = 0; j0 < cnt; j0 += slots) {
    const int jl = j0 + gid;
    const bool act = jl < cnt;
    const int j = part + nparts * jl;
    const int J = n - 1 - j;
    double lo = lo0, hi = hi0;
    bool done = !act;
    for (int it = 0; it < 200; ++it) {
      if (!done && hi - lo <= 1e-13 * fmax(fabs(lo), fabs(hi))) done = true;
      if (__all_sync(0xffffffffu, done)) break;
      double x[P];
      int c[P];
#pragma unroll
      for (int p = 0; p < P; ++p) x[p] = lo + (hi - lo) * (double)(glane * P + p + 1) / (double)(npts + 1);
      if (!done) {
        sturm_count_p<P>(n, d, e2, x, pivmin, c);
      } else {
#pragma unroll
        for (int p = 0; p < P; ++p) c[p] = n;
      }
      int below = 0;
#pragma unroll
      for (int p = 0; p < P; ++p) below += c[p] <= J;
      for (int o = G / 2; o > 0; o >>= 1) below += __shfl_xor_sync(0xffffffffu, below, o);
      if (!done) {
        const double nlo = below == 0 ? lo : lo + (hi - lo) * (double)below / (double)(npts + 1);
        const double nhi = below == npts ? hi : lo + (hi - lo) * (double)(below + 1) / (double)(npts + 1);
        if (nlo == lo && nhi == hi) done = true;
        lo = fmax(lo, nlo), hi = fmin(hi, nhi);
      }
    }
    if (act && glane == 0) out[j] = 0.5 * (lo + hi);
  }
}

// Eigenvalue with ascending index j of T by bisection on [lo, hi].
__device__ inline double bisect_eig(int n, const double* d, const double* e, int j, double lo, double hi, double pivmin) {
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    if (sturm_count(n, d, e, mid, pivmin) > j)
      hi = mid;
    else
      lo = mid;
    if (hi - lo <= 1e-13 * fmax(fabs(lo), fabs(hi))) break;
  }
  return 0.5 * (lo + hi);
}

// One inverse-iteration solve (T - lam I) y = z, tridiagonal LU with partial
// pivoting (dgtsv scheme); work: 4n doubles. Result overwrites z.
__device__ inline void tri_shift_solve(int n, const double* d, const double* e, double lam, double* z, double* wk, double tiny) {
  double* dl = wk;          // sub
  double* dd = wk + n;      // diag
  double* du = wk + 2 * n;  // super
  double* du2 = wk + 3 * n; // second super (fill-in)
  for (int i = 0; i < n; ++i) {
    dd[i] = d[i] - lam;
    du[i] = i + 1 < n ? e[i] : 0.0;
    dl[i] = i + 1 < n ? e[i] : 0.0;
    du2[i] = 0.0;
  }
  for (int i = 0; i + 1 < n; ++i) {
    if (fabs(dd[i]) >= fabs(dl[i])) {
      if (fabs(dd[i]) < tiny) dd[i] = dd[i] >= 0 ? tiny : -tiny;
      const double f = dl[i] / dd[i];
      dd[i + 1] -= f * du[i];
      z[i + 1] -= f * z[i];
      dl[i] = 0.0;
    } else {
      // swap rows i and i+1
      const double f = dd[i] / dl[i];
      dd[i] = dl[i];
      const double t = dd[i + 1];
      dd[i + 1] = du[i] - f * t;
      if (i + 2 < n) {
        du2[i] = du[i + 1];
        du[i + 1] = -f * du2[i];
      }
      du[i] = t;
      const double zt = z[i];
      z[i] = z[i + 1];
      z[i + 1] = zt - f * z[i + 1];
    }
  }
  if (fabs(dd[n - 1]) < tiny) dd[n - 1] = dd[n - 1] >= 0 ? tiny : -tiny;
  z[n - 1] /= dd[n - 1];
  if (n > 1) z[n - 2] = (z[n - 2] - du[n - 2] * z[n - 1]) / dd[n - 2];
  for (int i = n - 3; i >= 0; --i) z[i] = (z[i] - du[i] * z[i + 1] - du2[i] * z[i + 2]) / dd[i];
}

}  // namespace h2g

namespace h2g {

// ---------------------------------------------------------------------------
// CTA-cooperative tiled ZGEMM: C (m x n) = alpha op(A) op(B) + beta C over
// 64 x 64 output tiles, K staged 16 at a time through shared memory (sm must
// hold kTileSmemCplx complex), 4 x 4 complex register micro-tile per thread.
// Requires blockDim.x == 256. C must not alias A or B.
constexpr int kTileSmemCplx = 64 * 17 + 16 * 65;

__device__ inline void cta_gemm_tiled(int m, int n, int k, double alpha, const cplx* A, int lda, int opA, const cplx* B, int ldb, int opB,
                                      double beta, cplx* C, int ldc, cplx* sm) {
  cplx(*sA)[17] = reinterpret_cast<cplx(*)[17]>(sm);
  cplx(*sB)[65] = reinterpret_cast<cplx(*)[65]>(sm + 64 * 17);
  const int tr = threadIdx.x % 16, tc = threadIdx.x / 16;
  const bool a_rowmajor = opA == OP_T || opA == OP_C;  // consecutive p contiguous
  const bool b_rowmajor = opB == OP_N || opB == OP_R;  // consecutive p contiguous
  for (int r0 = 0; r0 < m; r0 += 64)
    for (int c0 = 0; c0 < n; c0 += 64) {
      cplx acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = czero();
      for (int k0 = 0; k0 < k; k0 += 16) {
        const int kk = min(16, k - k0);
        __syncthreads();
        for (int idx = threadIdx.x; idx < 64 * 16; idx += 256) {
          int i, p;
          if (a_rowmajor) p = idx % 16, i = idx / 16;
          else i = idx % 64, p = idx / 64;
          sA[i][p] = (p < kk && r0 + i < m) ? ld_op(A, lda, opA, r0 + i, k0 + p) : czero();
          int j, q;
          if (b_rowmajor) q = idx % 16, j = idx / 16;
          else j = idx % 64, q = idx / 64;
          sB[q][j] = (q < kk && c0 + j < n) ? ld_op(B, ldb, opB, k0 + q, c0 + j) : czero();
        }
        __syncthreads();
        for (int p = 0; p < kk; ++p) {
          cplx av[4], bv[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) av[a] = sA[tr * 4 + a][p];
#pragma unroll
          for (int b = 0; b < 4; ++b) bv[b] = sB[p][tc * 4 + b];
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) cfma(acc[a][b], av[a], bv[b]);
        }
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int i = r0 + tr * 4 + a, j = c0 + tc * 4 + b;
          if (i < m && j < n) {
            cplx* o = C + i + (size_t)j * ldc;
            const cplx v = acc[a][b];
            *o = beta == 0.0 ? cscale(v, alpha) : make_double2(beta * o->x + alpha * v.x, beta * o->y + alpha * v.y);
          }
        }
    }
  __syncthreads();
}

}  // namespace h2g

namespace h2g {

// ---------------------------------------------------------------------------
// 64 x 64 complex output tile, 128 threads, 8 x 4 register micro-tile per
// thread (rows tr + 8a, cols 4 tc + b: conflict-free shared reads), K staged
// 8 at a time, double-buffered. acc += op(A)[0:64, 0:k] op(B)[0:k, 0:64] with
// rows >= mv / cols >= nv treated as zero. A/B point at the tile origin.
// Measured 20 TFLOP/s on a 4096 x 4096 x 512 ZGEMM (tests/cuda/gemm_bench.cu).
// 3-stage k-slices (8 deep) of a TM x TM output tile computed by 128 threads;
// thread (tr, tc) = (tid % 8, tid / 8) owns rows tr + 8a (a < TM/8) and
// columns tc * (TM/16) + b.
// Rows padded by one complex: the cp.async writes of a k-major operand hit
// 8 consecutive k-rows, which would otherwise all start in the same bank.
template <int TM, int NST = 3>
struct TileSmem {
  cplx a[NST][8][TM + 1];
  cplx b[NST][8][TM + 1];
};
using Tile128Smem = TileSmem<64>;

__device__ __forceinline__ void cp_async16(void* smem, const void* g, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 16 : 0;  // src-size 0: zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(g), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }

// acc[tile row i][tile col j] += sum_p op(A)[i + ash, p] op(B)[p, j + bsh]
// (rows outside [0, am) / cols outside [0, bn) of op(A) / op(B) read as zero).
// Every operand form streams through a 3-stage cp.async pipeline (one 16-byte
// complex per cp.async, so transposed operands need no register staging);
// conjugation is applied when the k-slice is read from shared memory.
template <int TM, bool CA, bool CB>
__device__ __forceinline__ void tile_pipe(cplx (&acc)[TM / 8][TM / 16], TileSmem<TM>& S, const cplx* A, int lda, bool at, int ash, int am,
                                          const cplx* B, int ldb, bool bt, int bsh, int bn, int k) {
  constexpr int RM = TM / 8, RN = TM / 16;
  const int tr = threadIdx.x % 8, tc = threadIdx.x / 8;
  const int nk = (k + 7) / 8;
  __syncthreads();
  auto load = [&](int st, int kc) {
    const int k0 = kc * 8;
    for (int idx = threadIdx.x; idx < TM * 8; idx += 128) {
      // op(A)(i, p): column-major A[i + p lda] (N/R) or A[p + i lda] (T/C)
      int i, p;
      if (at) p = idx % 8, i = idx / 8;
      else i = idx % TM, p = idx / TM;
      const int ai = i + ash;
      const bool va = k0 + p < k && ai >= 0 && ai < am;
      const cplx* ga = at ? A + (k0 + p) + (size_t)ai * lda : A + ai + (size_t)(k0 + p) * lda;
      cp_async16(&S.a[st][p][i], va ? ga : A, va);
      // op(B)(q, j): B[q + j ldb] (N/R) or B[j + q ldb] (T/C)
      int j, q;
      if (bt) j = idx % TM, q = idx / TM;
      else q = idx % 8, j = idx / 8;
      const int bj = j + bsh;
      const bool vb = k0 + q < k && bj >= 0 && bj < bn;
      const cplx* gb = bt ? B + bj + (size_t)(k0 + q) * ldb : B + (k0 + q) + (size_t)bj * ldb;
      cp_async16(&S.b[st][q][j], vb ? gb : B, vb);
    }
    cp_async_commit();
  };
  for (int st = 0; st < 2; ++st) {
    if (st < nk) load(st, st);
    else cp_async_commit();
  }
  for (int kc = 0; kc < nk; ++kc) {
    asm volatile("cp.async.wait_group 1;");
    __syncthreads();
    const int st = kc % 3;
    if (kc + 2 < nk) load((kc + 2) % 3, kc + 2);
    else cp_async_commit();
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      cplx av[RM], bv[RN];
#pragma unroll
      for (int a = 0; a < RM; ++a) {
        av[a] = S.a[st][p][tr + 8 * a];
        if (CA) av[a].y = -av[a].y;
      }
#pragma unroll
      for (int b = 0; b < RN; ++b) {
        bv[b] = S.b[st][p][tc * RN + b];
        if (CB) bv[b].y = -bv[b].y;
      }
#pragma unroll
      for (int a = 0; a < RM; ++a)
#pragma unroll
        for (int b = 0; b < RN; ++b) cfma(acc[a][b], av[a], bv[b]);
    }
  }
  asm volatile("cp.async.wait_group 0;");
  __syncthreads();
}

// 64 x 64 complex tile on the FP64 tensor cores (DMMA m8n8k4): 4 warps, each
// a 32 x 32 warp tile of 4 x 4 m8n8 tiles with separate real / imaginary
// accumulators; the k-slices are the same cp.async stages as tile_pipe.
// Thread (g, tq) = (lane / 4, lane % 4) holds rows wr + 8 mi + g and columns
// wc + 8 ni + 2 tq + h of its warp tile.
struct Acc64 {
  double re[4][4][2], im[4][4][2];
};

__device__ __forceinline__ void acc64_zero(Acc64& c) {
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) c.re[a][b][0] = c.re[a][b][1] = c.im[a][b][0] = c.im[a][b][1] = 0.0;
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// f(i, j, v) for every accumulator element (i, j tile-local)
template <class F>
__device__ __forceinline__ void acc64_each(const Acc64& c, F&& f) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int wr = (warp % 2) * 32, wc = (warp / 2) * 32, g = lane / 4, tq = lane % 4;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) f(wr + mi * 8 + g, wc + ni * 8 + tq * 2 + h, make_double2(c.re[mi][ni][h], c.im[mi][ni][h]));
}

template <bool CA, bool CB>
__device__ __forceinline__ void tile_pipe_dmma(Acc64& acc, TileSmem<64>& S, const cplx* A, int lda, bool at, int ash, int am, const cplx* B,
                                               int ldb, bool bt, int bsh, int bn, int k) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int wr = (warp % 2) * 32, wc = (warp / 2) * 32, g = lane / 4, tq = lane % 4;
  const int nk = (k + 7) / 8;
  __syncthreads();
  auto load = [&](int st, int kc) {
    const int k0 = kc * 8;
    for (int idx = threadIdx.x; idx < 64 * 8; idx += 128) {
      int i, p;
      if (at) p = idx % 8, i = idx / 8;
      else i = idx % 64, p = idx / 64;
      const int ai = i + ash;
      const bool va = k0 + p < k && ai >= 0 && ai < am;
      const cplx* ga = at ? A + (k0 + p) + (size_t)ai * lda : A + ai + (size_t)(k0 + p) * lda;
      cp_async16(&S.a[st][p][i], va ? ga : A, va);
      int j, q;
      if (bt) j = idx % 64, q = idx / 64;
      else q = idx % 8, j = idx / 8;
      const int bj = j + bsh;
      const bool vb = k0 + q < k && bj >= 0 && bj < bn;
      const cplx* gb = bt ? B + bj + (size_t)(k0 + q) * ldb : B + (k0 + q) + (size_t)bj * ldb;
      cp_async16(&S.b[st][q][j], vb ? gb : B, vb);
    }
    cp_async_commit();
  };
  for (int st = 0; st < 2; ++st) {
    if (st < nk) load(st, st);
    else cp_async_commit();
  }
  for (int kc = 0; kc < nk; ++kc) {
    asm volatile("cp.async.wait_group 1;");
    __syncthreads();
    const int st = kc % 3;
    if (kc + 2 < nk) load((kc + 2) % 3, kc + 2);
    else cp_async_commit();
#pragma unroll
    for (int kk = 0; kk < 8; kk += 4) {
      cplx af[4], bf[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        af[mi] = S.a[st][kk + tq][wr + mi * 8 + g];
        if (CA) af[mi].y = -af[mi].y;
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        bf[ni] = S.b[st][kk + tq][wc + ni * 8 + g];
        if (CB) bf[ni].y = -bf[ni].y;
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
          dmma884(acc.re[mi][ni][0], acc.re[mi][ni][1], af[mi].x, bf[ni].x);
          dmma884(acc.re[mi][ni][0], acc.re[mi][ni][1], -af[mi].y, bf[ni].y);
          dmma884(acc.im[mi][ni][0], acc.im[mi][ni][1], af[mi].x, bf[ni].y);
          dmma884(acc.im[mi][ni][0], acc.im[mi][ni][1], af[mi].y, bf[ni].x);
        }
    }
  }
  asm volatile("cp.async.wait_group 0;");
  __syncthreads();
}

// One Schur contribution as the concatenated pipeline sees it: the tile's
// rows / columns of op(A) = A (arows x e, ld arows) and op(B) = B (e x bcols,
// ld e), shifted by ash / bsh; e = 0 marks a contribution that misses the tile.
struct SchurPanel {
  const cplx* A;
  const cplx* B;
  int arows, bcols, ash, bsh, e, pad;
};

// acc += sum over panels tab[0..n) of A_p B_p on the tile: ONE cp.async
// pipeline runs through the k-slices of all panels back to back (no ramp,
// drain or extra barrier per contribution; the loads of the next panel are in
// flight while the current one is multiplied). Slices are 8 deep, zero padded;
// the upper half of a slice is skipped when it holds no data (e <= 4 at the
// fine levels). kv: NST ints of shared memory. NST = 3 stages (2 for the
// target-prefetch variant of k_schur, which needs the shared memory).
// mlim / nlim: rows / columns of the tile inside the target; a warp skips the
// 8 x 8 blocks of its 32 x 32 share that lie outside (targets of ~100 rows
// would otherwise pay for 128).
template <int NST>
__device__ __forceinline__ void schur_pipe_dmma(Acc64& acc, TileSmem<64, NST>& S, const SchurPanel* tab, int n, int* kv, int mlim, int nlim) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int wr = (warp % 2) * 32, wc = (warp / 2) * 32, g = lane / 4, tq = lane % 4;
  const int mi_n = min(4, max(0, (mlim - wr + 7) / 8)), ni_n = min(4, max(0, (nlim - wc + 7) / 8));
  int total = 0;
  for (int p = 0; p < n; ++p) total += (tab[p].e + 7) / 8;
  if (total == 0) return;
  int li = 0, lk = 0, issued = 0;
  while (li < n && tab[li].e == 0) ++li;
  auto issue = [&]() {
    if (li < n) {
      const SchurPanel P = tab[li];
      const int st = issued % NST;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = threadIdx.x + u * 128;
        const int i = idx % 64, p = idx / 64;
        const int ai = i + P.ash;
        const bool va = lk + p < P.e && ai >= 0 && ai < P.arows;
        cp_async16(&S.a[st][p][i], va ? P.A + ai + (size_t)(lk + p) * P.arows : P.A, va);
        const int q = idx % 8, j = idx / 8;
        const int bj = j + P.bsh;
        const bool vb = lk + q < P.e && bj >= 0 && bj < P.bcols;
        cp_async16(&S.b[st][q][j], vb ? P.B + (lk + q) + (size_t)bj * P.e : P.B, vb);
      }
      if (threadIdx.x == 0) kv[st] = P.e - lk;
      lk += 8;
      if (lk >= P.e) {
        lk = 0;
        ++li;
        while (li < n && tab[li].e == 0) ++li;
      }
      ++issued;
    }
    cp_async_commit();
  };
  // NST - 1 slices in flight ahead of the one being multiplied
#pragma unroll
  for (int q = 0; q < NST - 1; ++q) issue();
  for (int s = 0; s < total; ++s) {
    if constexpr (NST == 4) asm volatile("cp.async.wait_group 2;");
    else if constexpr (NST == 3) asm volatile("cp.async.wait_group 1;");
    else asm volatile("cp.async.wait_group 0;");
    __syncthreads();
    issue();
    const int st = s % NST;
    const int nh = kv[st] > 4 ? 8 : 4;
    if (mi_n == 0 || ni_n == 0) continue;
    for (int kk = 0; kk < nh; kk += 4) {
      cplx af[4], bf[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) af[mi] = S.a[st][kk + tq][wr + mi * 8 + g];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) bf[ni] = S.b[st][kk + tq][wc + ni * 8 + g];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        if (mi >= mi_n) break;
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
          if (ni >= ni_n) break;
          dmma884(acc.re[mi][ni][0], acc.re[mi][ni][1], af[mi].x, bf[ni].x);
          dmma884(acc.re[mi][ni][0], acc.re[mi][ni][1], -af[mi].y, bf[ni].y);
          dmma884(acc.im[mi][ni][0], acc.im[mi][ni][1], af[mi].x, bf[ni].y);
          dmma884(acc.im[mi][ni][0], acc.im[mi][ni][1], af[mi].y, bf[ni].x);
        }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;");
  __syncthreads();
}

__device__ __forceinline__ void tile_acc_dmma(Acc64& acc, TileSmem<64>& S, const cplx* A, int lda, int opA, int ash, int am, const cplx* B, int ldb,
                                              int opB, int bsh, int bn, int k) {
  if (k <= 0) return;
  const bool at = opA == OP_T || opA == OP_C, bt = opB == OP_T || opB == OP_C;
  const bool ca = opA == OP_C || opA == OP_R, cb = opB == OP_C || opB == OP_R;
  if (!ca && !cb) tile_pipe_dmma<false, false>(acc, S, A, lda, at, ash, am, B, ldb, bt, bsh, bn, k);
  else if (ca && !cb) tile_pipe_dmma<true, false>(acc, S, A, lda, at, ash, am, B, ldb, bt, bsh, bn, k);
  else if (!ca && cb) tile_pipe_dmma<false, true>(acc, S, A, lda, at, ash, am, B, ldb, bt, bsh, bn, k);
  else tile_pipe_dmma<true, true>(acc, S, A, lda, at, ash, am, B, ldb, bt, bsh, bn, k);
}

// acc[tile row i][tile col j] += sum_p op(A)[i + ash, p] op(B)[p, j + bsh]
// (rows outside [0, am) / cols outside [0, bn) of op(A) / op(B) read as zero).
template <int TM>
__device__ __forceinline__ void tile_acc(cplx (&acc)[TM / 8][TM / 16], TileSmem<TM>& S, const cplx* A, int lda, int opA, int ash, int am,
                                         const cplx* B, int ldb, int opB, int bsh, int bn, int k) {
  if (k <= 0) return;
  const bool at = opA == OP_T || opA == OP_C, bt = opB == OP_T || opB == OP_C;
  const bool ca = opA == OP_C || opA == OP_R, cb = opB == OP_C || opB == OP_R;
  if (!ca && !cb) tile_pipe<TM, false, false>(acc, S, A, lda, at, ash, am, B, ldb, bt, bsh, bn, k);
  else if (ca && !cb) tile_pipe<TM, true, false>(acc, S, A, lda, at, ash, am, B, ldb, bt, bsh, bn, k);
  else if (!ca && cb) tile_pipe<TM, false, true>(acc, S, A, lda, at, ash, am, B, ldb, bt, bsh, bn, k);
  else tile_pipe<TM, true, true>(acc, S, A, lda, at, ash, am, B, ldb, bt, bsh, bn, k);
}

__device__ __forceinline__ void tile128_acc(cplx (&acc)[8][4], Tile128Smem& S, const cplx* A, int lda, int opA, int ash, int am, const cplx* B,
                                            int ldb, int opB, int bsh, int bn, int k) {
  tile_acc<64>(acc, S, A, lda, opA, ash, am, B, ldb, opB, bsh, bn, k);
}

}  // namespace h2g

namespace h2g {

// ---------------------------------------------------------------------------
// Blocked (panel 32) unpivoted LU in place, A n x n (ld lda). Same pivot rule
// and order of pivots as the right-looking reference (dense_kernels.hpp:70-93);
// trailing updates are tiled GEMMs. Returns -1 or the failing pivot index.
__device__ inline int cta_lu_blocked(int n, cplx* A, int lda, double tol, double* pmag, double* red, cplx* tile_sm) {
  double mx = 0.0;
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) mx = fmax(mx, cabsd(A[(idx % n) + (size_t)(idx / n) * lda]));
  const double scale = cta_max(mx, red);
  if (n > 0 && scale == 0.0) {
    *pmag = 0.0;
    return 0;
  }
  for (int j0 = 0; j0 < n; j0 += 32) {
    const int kb = min(32, n - j0), je = j0 + kb;
    for (int k = j0; k < je; ++k) {
      const cplx piv = A[k + (size_t)k * lda];
      const double pa = cabsd(piv);
      if (pa < tol * scale) {
        *pmag = pa;
        return k;
      }
      for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) A[i + (size_t)k * lda] = cdiv(A[i + (size_t)k * lda], piv);
      __syncthreads();
      const int nc = je - k - 1, nr = n - k - 1;
      for (int idx = threadIdx.x; idx < nr * nc; idx += blockDim.x) {
        const int i = k + 1 + idx % nr, j = k + 1 + idx / nr;
        cplx a = A[i + (size_t)j * lda];
        const cplx l = A[i + (size_t)k * lda], u = A[k + (size_t)j * lda];
        a.x -= l.x * u.x - l.y * u.y;
        a.y -= l.x * u.y + l.y * u.x;
        A[i + (size_t)j * lda] = a;
      }
      __syncthreads();
    }
    if (je < n) {
      // U12 = L11^{-1} A[j0:je, je:n] (unit lower), one thread per column
      for (int c = je + threadIdx.x; c < n; c += blockDim.x) {
        cplx* x = A + j0 + (size_t)c * lda;
        for (int i = 1; i < kb; ++i) {
          cplx s = x[i];
          for (int p = 0; p < i; ++p) {
            const cplx l = A[j0 + i + (size_t)(j0 + p) * lda];
            s.x -= l.x * x[p].x - l.y * x[p].y;
            s.y -= l.x * x[p].y + l.y * x[p].x;
          }
          x[i] = s;
        }
      }
      __syncthreads();
      cta_gemm_tiled(n - je, n - je, kb, -1.0, A + je + (size_t)j0 * lda, lda, OP_N, A + j0 + (size_t)je * lda, lda, OP_N, 1.0,
                     A + je + (size_t)je * lda, lda, tile_sm);
    }
  }
  return -1;
}

// X = L^{-1} for the unit-lower factor packed in LU (n x n, ld ldl); X ld ldx.
__device__ inline void cta_inv_unit_lower(int n, const cplx* LU, int ldl, cplx* X, int ldx, cplx* tile_sm) {
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) X[(idx % n) + (size_t)(idx / n) * ldx] = czero();
  __syncthreads();
  for (int j0 = 0; j0 < n; j0 += 32) {
    const int kb = min(32, n - j0), je = j0 + kb;
    if (j0 > 0) cta_gemm_tiled(kb, j0, j0, -1.0, LU + j0, ldl, OP_N, X, ldx, OP_N, 0.0, X + j0, ldx, tile_sm);
    for (int idx = threadIdx.x; idx < kb * kb; idx += blockDim.x) {
      const int i = idx % kb, c = idx / kb;
      X[j0 + i + (size_t)(j0 + c) * ldx] = i == c ? cone() : czero();
    }
    __syncthreads();
    for (int c = threadIdx.x; c < je; c += blockDim.x) {
      cplx* x = X + j0 + (size_t)c * ldx;
      for (int i = 1; i < kb; ++i) {
        cplx s = x[i];
        for (int p = 0; p < i; ++p) {
          const cplx l = LU[j0 + i + (size_t)(j0 + p) * ldl];
          s.x -= l.x * x[p].x - l.y * x[p].y;
          s.y -= l.x * x[p].y + l.y * x[p].x;
        }
        x[i] = s;
      }
    }
    __syncthreads();
  }
}

// Y = U^{-1} for the upper factor packed in LU; W: n x 32 scratch (ld n).
__device__ inline void cta_inv_upper(int n, const cplx* LU, int ldu, cplx* Y, int ldy, cplx* W, cplx* tile_sm) {
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) Y[(idx % n) + (size_t)(idx / n) * ldy] = czero();
  __syncthreads();
  for (int j0 = 0; j0 < n; j0 += 32) {
    const int kb = min(32, n - j0);
    // Y[J,J] = U_JJ^{-1}, one thread per column
    for (int c = threadIdx.x; c < kb; c += blockDim.x) {
      cplx* y = Y + j0 + (size_t)(j0 + c) * ldy;
      for (int i = c; i >= 0; --i) {
        cplx s = i == c ? cone() : czero();
        for (int p = i + 1; p <= c; ++p) {
          const cplx u = LU[j0 + i + (size_t)(j0 + p) * ldu];
          s.x -= u.x * y[p].x - u.y * y[p].y;
          s.y -= u.x * y[p].y + u.y * y[p].x;
        }
        y[i] = cdiv(s, LU[j0 + i + (size_t)(j0 + i) * ldu]);
      }
    }
    __syncthreads();
    if (j0 > 0) {
      cta_gemm_tiled(j0, kb, j0, 1.0, Y, ldy, OP_N, LU + (size_t)j0 * ldu, ldu, OP_N, 0.0, W, n, tile_sm);
      cta_gemm_tiled(j0, kb, kb, -1.0, W, n, OP_N, Y + j0 + (size_t)j0 * ldy, ldy, OP_N, 0.0, Y + (size_t)j0 * ldy, ldy, tile_sm);
    }
  }
}

}  // namespace h2g

namespace h2g {

// ---------------------------------------------------------------------------
// Blocked Householder QR (panels of 16 columns factored in shared memory,
// trailing columns updated with the panel's compact-WY form through tiled
// GEMMs). Same reflectors (Eigen convention) as cta_householder_qr.
// P: shared scratch of m x 16 complex; Tb: shared 16 x 16; W: global scratch
// of 16 x n complex (ld 16).
__device__ inline void cta_householder_qr_blocked(int m, int n, cplx* A, int lda, cplx* tau, double* red, cplx* tile_sm, cplx* P, cplx* Tb,
                                                  cplx* W, cplx* W2) {
  const int s = min(m, n);
  for (int j0 = 0; j0 < s; j0 += 16) {
    const int kb = min(16, s - j0), mr = m - j0;
    cta_copy(mr, kb, A + j0 + (size_t)j0 * lda, lda, P, mr);
    __syncthreads();
    cta_householder_qr(mr, kb, P, mr, tau + j0, red);
    cta_copy(mr, kb, P, mr, A + j0 + (size_t)j0 * lda, lda);
    __syncthreads();
    const int nt = n - j0 - kb;
    if (nt <= 0) continue;
    // Y (mr x kb, unit lower trapezoidal) in P; T (kb x kb) of Qp = H_0^H..H_{kb-1}^H = I - Y T Y^H
    for (int idx = threadIdx.x; idx < mr * kb; idx += blockDim.x) {
      const int i = idx % mr, j = idx / mr;
      if (i < j) P[idx] = czero();
      else if (i == j) P[idx] = cone();
    }
    __syncthreads();
    // S = Y^H Y (kb x kb) into Tb, then T in place column by column
    for (int idx = threadIdx.x; idx < kb * kb; idx += blockDim.x) {
      const int i = idx % kb, j = idx / kb;
      cplx v = czero();
      for (int p = max(i, j); p < mr; ++p) cfma(v, cconj(P[p + (size_t)i * mr]), P[p + (size_t)j * mr]);
      W2[idx] = v;  // S
    }
    __syncthreads();
    // T column by column, rows of a column in parallel
    for (int kk = 0; kk < kb; ++kk) {
      const cplx tk = cconj(tau[j0 + kk]);
      const int i = threadIdx.x;
      if (i < kk) {
        cplx v = czero();
        for (int j = i; j < kk; ++j) cfma(v, Tb[i + j * 16], W2[j + kk * kb]);
        Tb[i + kk * 16] = cmul(cmk(-tk.x, -tk.y), v);
      } else if (i == kk) {
        Tb[kk + kk * 16] = tk;
      } else if (i < kb) {
        Tb[i + kk * 16] = czero();
      }
      __syncthreads();
    }
    // A_trail <- Qp^H A_trail = A_trail - Y (T^H (Y^H A_trail))
    cplx* At = A + j0 + (size_t)(j0 + kb) * lda;
    cta_gemm_tiled(kb, nt, mr, 1.0, P, mr, OP_C, At, lda, OP_N, 0.0, W, 16, tile_sm);
    cta_gemm_tiled(kb, nt, kb, 1.0, Tb, 16, OP_C, W, 16, OP_N, 0.0, W2, 16, tile_sm);
    cta_gemm_tiled(mr, nt, kb, -1.0, P, mr, OP_N, W2, 16, OP_N, 1.0, At, lda, tile_sm);
  }
}

}  // namespace h2g
