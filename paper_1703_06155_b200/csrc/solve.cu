// Forward / backward substitution on the device (proj/include/h2lu/solve.hpp:
// 43-83), batch by batch in the factorization's elimination order. Vectors
// are n x nrhs column-major complex128 in tree order, updated in place.
#include <cooperative_groups.h>

#include <algorithm>
#include <map>
#include <tuple>
#include <mutex>
#include <stdexcept>

#include "solve.cuh"

namespace h2g {

// out = op(A) x for an n x n matrix A in global memory (op: N, R = conj, or
// C = conj-transpose), x / out n x nrhs in shared memory: one warp per output
// row with the lanes spread over the row's k range (many independent loads in
// flight), up to 8 right-hand sides per pass over A.
__device__ void warp_gemv(int n, int nrhs, const cplx* A, int lda, int op, const cplx* x, int ldx, cplx* out, long long ldo, int r0 = 0,
                          int r1 = -1) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  if (r1 < 0) r1 = n;  // output rows [r0, r1) only (a slab of the product)
  for (int c0 = 0; c0 < nrhs; c0 += 8) {
    const int nc = min(8, nrhs - c0);
    for (int i = r0 + warp; i < r1; i += nw) {
      cplx acc[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = czero();
      for (int p = lane; p < n; p += 32) {
        cplx av;
        if (op == OP_C) av = cconj(A[p + (size_t)i * lda]);
        else if (op == OP_R) av = cconj(A[i + (size_t)p * lda]);
        else av = A[i + (size_t)p * lda];
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c < nc) cfma(acc[c], av, x[p + (size_t)(c0 + c) * ldx]);
      }
      if (nc > 2) {
        // several columns: transposed butterfly. Every step halves the values
        // a lane carries (16 doubles -> 8 -> 4 -> 2 -> 1, then one plain step):
        // 16 double shuffles instead of 80, and the same summation tree as the
        // plain butterfly below (distance 16, 8, 4, 2, 1; IEEE addition is
        // commutative), so the results are bit-identical to it.
        double v[16];
#pragma unroll
        for (int c = 0; c < 8; ++c) v[2 * c] = acc[c].x, v[2 * c + 1] = acc[c].y;
#pragma unroll
        for (int h = 8, o = 16; h >= 1; h >>= 1, o >>= 1) {
          const bool up = (lane & o) != 0;
#pragma unroll
          for (int j = 0; j < h; ++j) {
            const double keep = up ? v[j + h] : v[j];
            const double send = up ? v[j] : v[j + h];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
        }
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
        // lane bits 16 / 8 / 4 / 2 selected halves of 8 / 4 / 2 / 1: value index = those bits
        const int idx = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
        if (!(lane & 1) && (idx >> 1) < nc) reinterpret_cast<double*>(out + i + (size_t)(c0 + (idx >> 1)) * ldo)[idx & 1] = v[0];
        continue;
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (c >= nc) break;
        double re = acc[c].x, im = acc[c].y;
        for (int o = 16; o > 0; o >>= 1) {
          re += __shfl_xor_sync(0xffffffffu, re, o);
          im += __shfl_xor_sync(0xffffffffu, im, o);
        }
        if (lane == 0) out[i + (size_t)(c0 + c) * ldo] = make_double2(re, im);
      }
    }
  }
}

// inner dimensions up to this run one thread per result entry in the many-RHS
// paths: every size by default (measured, profiles/r02_solve_smallk.txt);
// H2G_SOLVE_SMALLK overrides (0: the k-sliced form; read once per device)
__constant__ int kSmallK = 1 << 30;

// out = op(A) x for a column-major m x k matrix A (op: A or conj(A), no
// transpose), x k x nrhs (global or shared). Coalesced: thread t owns row
// i = t % m' of a chunk of m' <= blockDim rows and the k-slice p = g, g + G,
// ... with g = t / m', G = blockDim / m' groups; the G partial sums are
// reduced through shared memory in a fixed order (deterministic). subtract:
// out -= result instead of out = result. red: blockDim complex of shared.
__device__ void cta_gemv_n(int m, int k, int nrhs, const cplx* A, int lda, bool conjA, const cplx* x, long long ldx, cplx* out, long long ldo,
                           bool subtract, cplx* red) {
  if (nrhs >= 4 && k <= kSmallK) {
    // many right-hand sides: one thread per (row, column) entry of the result
    // (per row and 4 columns when that still fills the CTA), the whole k range
    // in registers -> no k-slices, no reduction barriers. Measured faster than
    // the k-sliced form below at every level (profiles/r02_solve_smallk.txt).
    if (m * ((nrhs + 3) / 4) >= (int)blockDim.x) {
      const int ncb = (nrhs + 3) / 4;
      for (int idx = threadIdx.x; idx < m * ncb; idx += blockDim.x) {
        const int i = idx % m, c0 = (idx / m) * 4, nc = min(4, nrhs - c0);
        const cplx* xc = x + (size_t)c0 * ldx;
        cplx acc[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[c] = czero();
#pragma unroll 2
        for (int p = 0; p < k; ++p) {
          cplx a = A[i + (size_t)p * lda];
          if (conjA) a.y = -a.y;
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (c < nc) cfma(acc[c], a, xc[p + (size_t)c * ldx]);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c < nc) {
            cplx* o = out + i + (size_t)(c0 + c) * ldo;
            *o = subtract ? csub(*o, acc[c]) : acc[c];
          }
      }
      __syncthreads();
      return;
    }
    for (int idx = threadIdx.x; idx < m * nrhs; idx += blockDim.x) {
      const int i = idx % m, c = idx / m;
      const cplx* xc = x + (size_t)c * ldx;
      cplx acc = czero();
      for (int p = 0; p < k; ++p) {
        cplx a = A[i + (size_t)p * lda];
        if (conjA) a.y = -a.y;
        cfma(acc, a, xc[p]);
      }
      cplx* o = out + i + (size_t)c * ldo;
      *o = subtract ? csub(*o, acc) : acc;
    }
    __syncthreads();
    return;
  }
  if (nrhs >= 4) {
    // many right-hand sides: the same (row, k-slice) threads, each A element
    // read once for up to 8 columns (8 accumulators), the k-slices reduced
    // through shared memory one column at a time
    for (int c0 = 0; c0 < nrhs; c0 += 8) {
      const int nc = min(8, nrhs - c0);
      for (int i0 = 0; i0 < m; i0 += blockDim.x) {
        const int mm = min(m - i0, (int)blockDim.x);
        const int G = max(1, (int)blockDim.x / mm);
        const int t = threadIdx.x, i = t % mm, g = t / mm;
        cplx acc[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = czero();
        if (g < G) {
#pragma unroll 2
          for (int p = g; p < k; p += G) {
            cplx a = A[(i0 + i) + (size_t)p * lda];
            if (conjA) a.y = -a.y;
#pragma unroll
            for (int c = 0; c < 8; ++c)
              if (c < nc) cfma(acc[c], a, x[p + (size_t)(c0 + c) * ldx]);
          }
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (c >= nc) break;
          __syncthreads();
          if (g < G) red[g * mm + i] = acc[c];
          __syncthreads();
          if (t < mm) {
            cplx s2 = red[t];
            for (int q = 1; q < G; ++q) s2 = cadd(s2, red[q * mm + t]);
            cplx* o = out + (i0 + t) + (size_t)(c0 + c) * ldo;
            *o = subtract ? csub(*o, s2) : s2;
          }
        }
      }
    }
    __syncthreads();
    return;
  }
  for (int i0 = 0; i0 < m; i0 += blockDim.x) {
    const int mm = min(m - i0, (int)blockDim.x);
    // k-slices: no more than k (a record with 2 eliminated rows would otherwise
    // have its 2 result threads add up 128 partials, 126 of them empty). A
    // further cap of 8 slices was measured slower (31.8 against 30.5 ms, config 2).
    const int G = max(1, min((int)blockDim.x / mm, k));
    const int t = threadIdx.x, i = t % mm, g = t / mm;
    for (int c = 0; c < nrhs; ++c) {
      cplx acc = czero();
      if (g < G) {
        const cplx* xc = x + (size_t)c * ldx;
#pragma unroll 4
        for (int p = g; p < k; p += G) {
          cplx a = A[(i0 + i) + (size_t)p * lda];
          if (conjA) a.y = -a.y;
          cfma(acc, a, xc[p]);
        }
      }
      __syncthreads();
      if (g < G) red[g * mm + i] = acc;
      __syncthreads();
      if (t < mm) {
        cplx s = red[t];
        for (int q = 1; q < G; ++q) s = cadd(s, red[q * mm + t]);
        cplx* o = out + (i0 + t) + (size_t)c * ldo;
        *o = subtract ? csub(*o, s) : s;
      }
    }
  }
  __syncthreads();
}

// seg <- Qt^H seg, then head <- L11^{-1} head (solve.hpp:47-50); one CTA per
// record.
__device__ void fwd_head_body(const SolveLevel& S, int t, cplx* y, long long ldy, int nrhs, int explicit_inv, unsigned char* smraw,
                              const cplx* pre = nullptr) {
  const int b = S.bsz[t], e = b - S.kfin[t];
  const long long p0 = S.pos[t];
  cplx* sS = reinterpret_cast<cplx*>(smraw);  // b x nrhs
  cplx* sO = sS + (size_t)b * nrhs;           // b x nrhs
  cplx* sR = sO + (size_t)b * nrhs;           // reduction scratch (blockDim)
  // pre == nullptr: rotate the segment here; else pre holds Qt^H seg already
  // (computed by the record's slab items, split records)
  if (pre) {
    for (int idx = threadIdx.x; idx < b * nrhs; idx += blockDim.x) sO[idx] = pre[p0 + (idx % b) + (idx / b) * ldy];
  } else {
    for (int idx = threadIdx.x; idx < b * nrhs; idx += blockDim.x) sS[idx] = y[p0 + (idx % b) + (idx / b) * ldy];
    __syncthreads();
    const cplx* Q = S.chain + S.Qt_off[t];
    warp_gemv(b, nrhs, Q, b, OP_C, sS, b, sO, b);
  }
  __syncthreads();
  if (e > 0) {
    if (explicit_inv) {
      const cplx* Li = S.chain + S.Linv_off[t];
      cta_gemv_n(e, e, nrhs, Li, e, false, sO, b, sS, b, false, sR);
      for (int idx = threadIdx.x; idx < e * nrhs; idx += blockDim.x) sO[(idx % e) + (idx / e) * b] = sS[(idx % e) + (idx / e) * b];
      __syncthreads();
    } else {
      const cplx* L = S.chain + S.L11_off[t];
      for (int p = 0; p < e; ++p) {
        for (int idx = threadIdx.x; idx < (e - p - 1) * nrhs; idx += blockDim.x) {
          const int i = p + 1 + idx % (e - p - 1), c = idx / (e - p - 1);
          const cplx l = L[i + (size_t)p * e], x = sO[p + c * b];
          cplx v = sO[i + c * b];
          v.x -= l.x * x.x - l.y * x.y;
          v.y -= l.x * x.y + l.y * x.x;
          sO[i + c * b] = v;
        }
        __syncthreads();
      }
    }
  }
  for (int idx = threadIdx.x; idx < b * nrhs; idx += blockDim.x) y[p0 + (idx % b) + (idx / b) * ldy] = sO[idx];
}

// Slab sl of ns of a split record's rotation: rows [r0, r1) of Qt^H seg into
// pre (the record's head item applies L11^{-1} once every slab has landed).
__device__ void fwd_slab_body(const SolveLevel& S, int t, int sl, int ns, const cplx* y, long long ldy, int nrhs, cplx* pre, unsigned char* smraw) {
  const int b = S.bsz[t];
  const long long p0 = S.pos[t];
  cplx* sS = reinterpret_cast<cplx*>(smraw);  // b x nrhs
  for (int idx = threadIdx.x; idx < b * nrhs; idx += blockDim.x) sS[idx] = y[p0 + (idx % b) + (idx / b) * ldy];
  __syncthreads();
  const int rows = (b + ns - 1) / ns, r0 = sl * rows, r1 = min(b, r0 + rows);
  warp_gemv(b, nrhs, S.chain + S.Qt_off[t], b, OP_C, sS, b, pre + p0, ldy, r0, r1);
}

// y[pos_j ...] -= sum_m Lbar(m, j) head_m (solve.hpp:51). Thread (i, g):
// row i of the target, slice g of every contribution's columns (coalesced
// column reads); contributions accumulate per thread, one fixed-order
// reduction at the end (deterministic).
__device__ void fwd_lbar_body(const SolveLevel& S, const SolveTargetD tg, const SolveContribD* contrib, cplx* y, long long ldy, int nrhs,
                              cplx* red) {
  int rows;
  long long base;
  if (tg.seg >= 0) {
    rows = S.bsz[tg.seg];
    base = S.pos[tg.seg];
  } else {
    const int m = -1 - tg.seg;
    rows = S.kfin[m];
    base = S.pos[m] + (S.bsz[m] - S.kfin[m]);
  }
  int ktot = 0;
  for (int ci = tg.c0; ci < tg.c1; ++ci) ktot += S.bsz[contrib[ci].m] - S.kfin[contrib[ci].m];
  if (nrhs >= 4 && ktot <= kSmallK) {
    // many right-hand sides: one thread per (row, column) entry (per row and
    // 4 columns when that still fills the CTA), contributions in order
    if (rows * ((nrhs + 3) / 4) >= (int)blockDim.x) {
      const int ncb = (nrhs + 3) / 4;
      for (int idx = threadIdx.x; idx < rows * ncb; idx += blockDim.x) {
        const int i = idx % rows, c0 = (idx / rows) * 4, nc = min(4, nrhs - c0);
        cplx acc[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[c] = czero();
        for (int ci = tg.c0; ci < tg.c1; ++ci) {
          const SolveContribD cb = contrib[ci];
          const int e = S.bsz[cb.m] - S.kfin[cb.m];
          const cplx* M = S.chain + (cb.entry >= 0 ? S.Lbar_off[cb.entry] : S.Lself_off[cb.m]) + i;
          const cplx* h = y + S.pos[cb.m] + (size_t)c0 * ldy;
#pragma unroll 2
          for (int p = 0; p < e; ++p) {
            const cplx mv = M[(size_t)p * rows];
#pragma unroll
            for (int c = 0; c < 4; ++c)
              if (c < nc) cfma(acc[c], mv, h[p + (size_t)c * ldy]);
          }
        }
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c < nc) {
            cplx* o = y + base + i + (size_t)(c0 + c) * ldy;
            *o = csub(*o, acc[c]);
          }
      }
      __syncthreads();
      return;
    }
    for (int idx = threadIdx.x; idx < rows * nrhs; idx += blockDim.x) {
      const int i = idx % rows, c = idx / rows;
      cplx acc = czero();
      for (int ci = tg.c0; ci < tg.c1; ++ci) {
        const SolveContribD cb = contrib[ci];
        const int e = S.bsz[cb.m] - S.kfin[cb.m];
        const cplx* M = S.chain + (cb.entry >= 0 ? S.Lbar_off[cb.entry] : S.Lself_off[cb.m]) + i;
        const cplx* h = y + S.pos[cb.m] + (size_t)c * ldy;
        for (int p = 0; p < e; ++p) cfma(acc, M[(size_t)p * rows], h[p]);
      }
      cplx* o = y + base + i + (size_t)c * ldy;
      *o = csub(*o, acc);
    }
    __syncthreads();
    return;
  }
  if (nrhs >= 4) {
    // many right-hand sides: the same (row, k-slice) threads with up to 8
    // columns per Lbar element, k-slices reduced one column at a time
    for (int c0 = 0; c0 < nrhs; c0 += 8) {
      const int nc = min(8, nrhs - c0);
      for (int i0 = 0; i0 < rows; i0 += blockDim.x) {
        const int mm = min(rows - i0, (int)blockDim.x);
        const int G = max(1, (int)blockDim.x / mm);
        const int t = threadIdx.x, i = t % mm, g = t / mm;
        cplx acc[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = czero();
        if (g < G) {
          for (int ci = tg.c0; ci < tg.c1; ++ci) {
            const SolveContribD cb = contrib[ci];
            const int e = S.bsz[cb.m] - S.kfin[cb.m];
            const cplx* M = S.chain + (cb.entry >= 0 ? S.Lbar_off[cb.entry] : S.Lself_off[cb.m]) + i0 + i;
            const cplx* h = y + S.pos[cb.m] + (size_t)c0 * ldy;
#pragma unroll 2
            for (int p = g; p < e; p += G) {
              const cplx mv = M[(size_t)p * rows];
#pragma unroll
              for (int c = 0; c < 8; ++c)
                if (c < nc) cfma(acc[c], mv, h[p + (size_t)c * ldy]);
            }
          }
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (c >= nc) break;
          __syncthreads();
          if (g < G) red[g * mm + i] = acc[c];
          __syncthreads();
          if (t < mm) {
            cplx s2 = red[t];
            for (int q = 1; q < G; ++q) s2 = cadd(s2, red[q * mm + t]);
            cplx* o = y + base + i0 + t + (size_t)(c0 + c) * ldy;
            *o = csub(*o, s2);
          }
        }
      }
    }
    __syncthreads();
    return;
  }
  for (int i0 = 0; i0 < rows; i0 += blockDim.x) {
    const int mm = min(rows - i0, (int)blockDim.x);
    const int G = max(1, min((int)blockDim.x / mm, ktot));  // ktot bounds every contribution's columns
    const int t = threadIdx.x, i = t % mm, g = t / mm;
    for (int c = 0; c < nrhs; ++c) {
      cplx acc = czero();
      if (g < G) {
        for (int ci = tg.c0; ci < tg.c1; ++ci) {
          const SolveContribD cb = contrib[ci];
          const int e = S.bsz[cb.m] - S.kfin[cb.m];
          const cplx* M = S.chain + (cb.entry >= 0 ? S.Lbar_off[cb.entry] : S.Lself_off[cb.m]) + i0 + i;
          const cplx* h = y + S.pos[cb.m] + (size_t)c * ldy;
#pragma unroll 4
          for (int p = g; p < e; p += G) cfma(acc, M[(size_t)p * rows], h[p]);
        }
      }
      __syncthreads();
      if (g < G) red[g * mm + i] = acc;
      __syncthreads();
      if (t < mm) {
        cplx s2 = red[t];
        for (int q = 1; q < G; ++q) s2 = cadd(s2, red[q * mm + t]);
        cplx* o = y + base + i0 + t + (size_t)c * ldy;
        *o = csub(*o, s2);
      }
    }
  }
  __syncthreads();
}

// Backward gather (solve.hpp:77): partial[q][c] = Ubar(m, c) y[pos_c ...]
// for one neighbour c of record m = batch[q] (the last slot is the self
// block), spread over CTAs so the chain blocks stream at full bandwidth.
__device__ void bwd_gather_to(const SolveLevel& S, int t, int c, const cplx* y, long long ldy, int nrhs, cplx* out, cplx* red) {
  const int b = S.bsz[t], kf = S.kfin[t], e = b - kf;
  const int nC = S.C_ptr[t + 1] - S.C_ptr[t];
  if (e == 0 || c > nC || (c == nC && kf == 0)) return;
  const cplx* M;
  const cplx* x;
  int cols;
  if (c < nC) {
    const int ent = S.C_ptr[t] + c, nb = S.C_nb[ent];
    cols = S.bsz[nb];
    M = S.chain + S.Ubar_off[ent];
    x = y + S.pos[nb];
  } else {
    cols = kf;
    M = S.chain + S.Uself_off[t];
    x = y + S.pos[t] + e;
  }
  cta_gemv_n(e, cols, nrhs, M, e, false, x, ldy, out, e, false, red);
}

__device__ void bwd_gather_body(const SolveLevel& S, int t, int q, int c, int nslot, const cplx* y, long long ldy, int nrhs, cplx* part,
                                long long pstride, cplx* red) {
  bwd_gather_to(S, t, c, y, ldy, nrhs, part + ((size_t)q * nslot + c) * pstride, red);
}

// Backward record (solve.hpp:73-81): head -= sum of the gathered partials (in
// neighbour order); U11 solve; seg <- conj(Qt) seg. One CTA per record.
// post != nullptr (split record): the segment before its rotation goes to
// post and the record's slab items apply conj(Qt).
__device__ void bwd_body(const SolveLevel& S, int t, cplx* y, long long ldy, int nrhs, int explicit_inv, const cplx* part0, long long slot_stride,
                         unsigned char* smraw, cplx* post = nullptr) {
  const int b = S.bsz[t], kf = S.kfin[t], e = b - kf;
  const long long p0 = S.pos[t];
  cplx* sS = reinterpret_cast<cplx*>(smraw);
  cplx* sO = sS + (size_t)b * nrhs;
  cplx* sR = sO + (size_t)b * nrhs;  // reduction scratch (blockDim)
  for (int idx = threadIdx.x; idx < b * nrhs; idx += blockDim.x) sS[idx] = y[p0 + (idx % b) + (idx / b) * ldy];
  __syncthreads();
  if (e > 0) {
    const int nC = S.C_ptr[t + 1] - S.C_ptr[t];
    const int nuse = nC + (kf > 0 ? 1 : 0);
    // head -= sum of the gathered partials: one warp per (row, rhs), lanes
    // over the neighbour slots, fixed shuffle tree
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
    for (int idx = warp; idx < e * nrhs; idx += nw) {
      const int i = idx % e, c = idx / e;
      cplx acc = czero();
      for (int u = lane; u < nuse; u += 32) acc = cadd(acc, part0[(size_t)u * slot_stride + i + (size_t)c * e]);
      double re = acc.x, im = acc.y;
      for (int o = 16; o > 0; o >>= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, o);
        im += __shfl_xor_sync(0xffffffffu, im, o);
      }
      if (lane == 0) sS[i + c * b] = csub(sS[i + c * b], make_double2(re, im));
    }
    __syncthreads();
    if (explicit_inv) {
      const cplx* Ui = S.chain + S.Uinv_off[t];
      cta_gemv_n(e, e, nrhs, Ui, e, false, sS, b, sO, b, false, sR);
      __syncthreads();
      for (int idx = threadIdx.x; idx < e * nrhs; idx += blockDim.x) sS[(idx % e) + (idx / e) * b] = sO[(idx % e) + (idx / e) * b];
      __syncthreads();
    } else {
      const cplx* U = S.chain + S.U11_off[t];
      for (int p = e - 1; p >= 0; --p) {
        for (int c = threadIdx.x; c < nrhs; c += blockDim.x) sS[p + c * b] = cdiv(sS[p + c * b], U[p + (size_t)p * e]);
        __syncthreads();
        for (int idx = threadIdx.x; idx < p * nrhs; idx += blockDim.x) {
          const int i = idx % p, c = idx / p;
          const cplx u = U[i + (size_t)p * e], x = sS[p + c * b];
          cplx v = sS[i + c * b];
          v.x -= u.x * x.x - u.y * x.y;
          v.y -= u.x * x.y + u.y * x.x;
          sS[i + c * b] = v;
        }
        __syncthreads();
      }
    }
  }
  if (post) {
    for (int idx = threadIdx.x; idx < b * nrhs; idx += blockDim.x) post[p0 + (idx % b) + (idx / b) * ldy] = sS[idx];
    return;
  }
  const cplx* Q = S.chain + S.Qt_off[t];
  cta_gemv_n(b, b, nrhs, Q, b, true, sS, b, sO, b, false, sR);
  for (int idx = threadIdx.x; idx < b * nrhs; idx += blockDim.x) y[p0 + (idx % b) + (idx / b) * ldy] = sO[idx];
}

// Slab sl of ns of a split record's backward rotation: rows [r0, r1) of
// conj(Qt) post -> y.
__device__ void bwd_slab_body(const SolveLevel& S, int t, int sl, int ns, cplx* y, long long ldy, int nrhs, const cplx* post, unsigned char* smraw) {
  const int b = S.bsz[t];
  const long long p0 = S.pos[t];
  cplx* sS = reinterpret_cast<cplx*>(smraw);
  cplx* sR = sS + 2 * (size_t)b * nrhs;
  for (int idx = threadIdx.x; idx < b * nrhs; idx += blockDim.x) sS[idx] = post[p0 + (idx % b) + (idx / b) * ldy];
  __syncthreads();
  const int rows = (b + ns - 1) / ns, r0 = sl * rows, r1 = min(b, r0 + rows);
  if (r1 > r0) cta_gemv_n(r1 - r0, b, nrhs, S.chain + S.Qt_off[t] + r0, b, true, sS, b, y + p0 + r0, ldy, false, sR);
}

// One persistent cooperative kernel per level and direction: the batches of
// the elimination order run back to back with grid-wide barriers between the
// record phase and the neighbour phase, instead of two launches per batch.
__global__ void __launch_bounds__(256) k_fwd_level(SolveLevel S, SolveSched P, cplx* y, long long ldy, int nrhs, int explicit_inv) {
  namespace cg = cooperative_groups;
  cg::grid_group g = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smraw[];
  for (int bi = 0; bi < P.nbat; ++bi) {
    const int p0 = P.batch_ptr[bi], nb = P.batch_ptr[bi + 1] - p0;
    for (int q = blockIdx.x; q < nb; q += gridDim.x) {
      fwd_head_body(S, P.batch_cl[p0 + q], y, ldy, nrhs, explicit_inv, smraw);
      __syncthreads();
    }
    g.sync();
    const int f0 = P.fs_ptr[bi], f1 = P.fs_ptr[bi + 1];
    for (int f = f0 + blockIdx.x; f < f1; f += gridDim.x) fwd_lbar_body(S, P.fs[f], P.fc, y, ldy, nrhs, reinterpret_cast<cplx*>(smraw));
    g.sync();
  }
}

__global__ void __launch_bounds__(256) k_bwd_level(SolveLevel S, SolveSched P, cplx* y, long long ldy, int nrhs, int explicit_inv, cplx* part,
                                                   long long pstride) {
  namespace cg = cooperative_groups;
  cg::grid_group g = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smraw[];
  for (int bi = P.nbat - 1; bi >= 0; --bi) {
    const int p0 = P.batch_ptr[bi], nb = P.batch_ptr[bi + 1] - p0;
    const int nslot = P.batch_maxc[bi] + 1;
    for (int it = blockIdx.x; it < nb * nslot; it += gridDim.x)
      bwd_gather_body(S, P.batch_cl[p0 + it / nslot], it / nslot, it % nslot, nslot, y, ldy, nrhs, part, pstride, reinterpret_cast<cplx*>(smraw));
    g.sync();
    for (int q = blockIdx.x; q < nb; q += gridDim.x) {
      bwd_body(S, P.batch_cl[p0 + q], y, ldy, nrhs, explicit_inv, part + (size_t)q * nslot * pstride, pstride, smraw);
      __syncthreads();
    }
    g.sync();
  }
}

// ------------------------------------------------------------ dataflow
// The substitutions as a dependency graph instead of batch-wide barriers:
// work items (records, neighbour targets / gather slots) are handed out in
// the elimination order by a global ticket, and every item waits only on the
// items it reads from (per-segment writer counters, record-done flags). An
// item depends only on items with smaller tickets, which are held by running
// CTAs, so the wait cannot deadlock; per-segment writers are serialised in a
// fixed order, so results are deterministic.
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) { asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }
// Spin until *p >= v; a wait longer than ~2 s means a broken schedule: the
// stall is reported through *fail (and the host raises) instead of hanging.
__device__ __forceinline__ bool wait_ge(const int* p, int v, int* fail) {
  if (ld_acquire(p) >= v) return true;
  const long long t0 = clock64();
  while (ld_acquire(p) < v) {
    __nanosleep(64);
    if (clock64() - t0 > 4000000000LL || *(volatile int*)fail) {
      atomicExch(fail, 1);
      return false;
    }
  }
  return true;
}
// after a wait by thread 0: its acquire load (gpu scope) followed by the block
// barrier orders the producers' stores before every thread's loads (the
// consumer half of the CUTLASS semaphore pattern)
__device__ __forceinline__ void acquire_all(const int*) { __syncthreads(); }
// publish: the block's stores are visible before the counter moves. The
// block barrier orders every thread's stores before thread 0's release store,
// which is cumulative at gpu scope (the CUTLASS semaphore pattern): no
// per-thread fence.
__device__ __forceinline__ void publish(int* p, int v) {
  __syncthreads();
  if (threadIdx.x == 0) st_release(p, v);
}
// same for a counter incremented by several items
__device__ __forceinline__ void publish_add(int* p) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(p, 1);
  }
}

// The chain data of an item (static) is pulled into L2 while the item still
// waits for its inputs, so the dependent part after the wait reads it at L2
// latency: one prefetch per 128-byte line, spread over the CTA.
__device__ __forceinline__ void cta_prefetch_l2(const void* p, size_t bytes) {
  const char* c = static_cast<const char*>(p);
  for (size_t o = (size_t)threadIdx.x * 128; o < bytes; o += (size_t)blockDim.x * 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(c + o));
}

// Records with large blocks are split: the b x b rotation, which sits on the
// dependency chain, is cut into row slabs handed to different CTAs (item code
// kSlabBase + 64 t + slab); the record's own item then only applies the
// triangular inverse (forward) or runs before the slabs (backward).
constexpr int kSlabBase = 1 << 30;

// Forward (solve.hpp:43-59). items: >= 0 record cluster t, < 0 target -1-f.
// cnt: [0] ticket, [1 + s] writers of segment s done, [1 + nl + t] slabs of record t done.
template <int NT>
__global__ void __launch_bounds__(NT) k_fwd_flow(SolveLevel S, SolveSched P, SolveFlow F, cplx* y, long long ldy, int nrhs, int explicit_inv,
                                                 int* cnt, int* fail, cplx* tmp, FlowGroups G) {
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ int s_item, s_ok;
  {
    // right-hand-side group blockIdx.y: its own columns, counters and ticket
    const int g = blockIdx.y;
    y += (size_t)g * G.rchunk * ldy;
    tmp += (size_t)g * G.rchunk * ldy;
    cnt += (size_t)g * G.cstride;
    nrhs = min(G.rchunk, nrhs - g * G.rchunk);
  }
  int* seg = cnt + 1;
  int* slab_done = cnt + 1 + S.nl;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(cnt, 1), s_ok = 1;
    __syncthreads();
    const int it = s_item;
    __syncthreads();
    if (it >= F.nf) return;
    const int code = F.f_items[it];
    if (code >= kSlabBase) {
      // slab of a split record's rotation: reads the segment once its earlier writers are done
      const int t = (code - kSlabBase) >> 6, sl = (code - kSlabBase) & 63, w = F.rec_widx[t];
      {
        const int b = S.bsz[t], ns = F.rec_ns_f[t], rows = (b + ns - 1) / ns, r0 = sl * rows;
        if (r0 < b) cta_prefetch_l2(S.chain + S.Qt_off[t] + (size_t)r0 * b, (size_t)min(rows, b - r0) * b * sizeof(cplx));
      }
      if (threadIdx.x == 0) s_ok = wait_ge(seg + t, w, fail);
      acquire_all(seg + t);
      if (!s_ok) return;
      fwd_slab_body(S, t, sl, F.rec_ns_f[t], y, ldy, nrhs, tmp, smraw);
      publish_add(slab_done + t);
    } else if (code >= 0) {
      const int t = code, w = F.rec_widx[t], ns = F.rec_ns_f[t];
      {
        const int b = S.bsz[t], e = b - S.kfin[t];
        if (!ns) cta_prefetch_l2(S.chain + S.Qt_off[t], (size_t)b * b * sizeof(cplx));
        if (e > 0) cta_prefetch_l2(S.chain + (explicit_inv ? S.Linv_off[t] : S.L11_off[t]), (size_t)e * e * sizeof(cplx));
      }
      if (F.pull) {
        // the updates of the earlier neighbours, applied here in the same
        // (batch) order the per-segment items would apply them
        for (int u = F.rec_fs_ptr[t]; u < F.rec_fs_ptr[t + 1]; ++u) {
          const SolveTargetD tg = P.fs[F.rec_fs[u]];
          if (threadIdx.x == 0)
            for (int ci = tg.c0; ci < tg.c1 && s_ok; ++ci) {
              const int m = P.fc[ci].m;
              s_ok = wait_ge(seg + m, F.rec_widx[m] + 1, fail);
            }
          acquire_all(seg + t);
          if (!s_ok) return;
          fwd_lbar_body(S, tg, P.fc, y, ldy, nrhs, reinterpret_cast<cplx*>(smraw));
        }
      }
      if (threadIdx.x == 0) s_ok = ns ? wait_ge(slab_done + t, ns, fail) : wait_ge(seg + t, w, fail);
      acquire_all(ns ? slab_done + t : seg + t);
      if (!s_ok) return;
      fwd_head_body(S, t, y, ldy, nrhs, explicit_inv, smraw, ns ? tmp : nullptr);
      publish(seg + t, w + 1);
    } else {
      const int f = -1 - code;
      const SolveTargetD tg = P.fs[f];
      const int sg = tg.seg >= 0 ? tg.seg : -1 - tg.seg;
      {
        const int rows = tg.seg >= 0 ? S.bsz[sg] : S.kfin[sg];
        for (int ci = tg.c0; ci < tg.c1; ++ci) {
          const SolveContribD cb = P.fc[ci];
          cta_prefetch_l2(S.chain + (cb.entry >= 0 ? S.Lbar_off[cb.entry] : S.Lself_off[cb.m]), (size_t)rows * (S.bsz[cb.m] - S.kfin[cb.m]) * sizeof(cplx));
        }
      }
      if (threadIdx.x == 0) {
        for (int ci = tg.c0; ci < tg.c1 && s_ok; ++ci) {
          const int m = P.fc[ci].m;
          s_ok = wait_ge(seg + m, F.rec_widx[m] + 1, fail);  // head of record m final
        }
        if (s_ok) s_ok = wait_ge(seg + sg, F.fs_widx[f], fail);  // earlier writers of the segment
      }
      acquire_all(seg + sg);
      if (!s_ok) return;
      fwd_lbar_body(S, tg, P.fc, y, ldy, nrhs, reinterpret_cast<cplx*>(smraw));
      publish(seg + sg, F.fs_widx[f] + 1);
    }
    __syncthreads();
  }
}

// Backward (solve.hpp:65-83). items: >= 0 record cluster m, < 0 gather slot
// -1-s. cnt: [0] ticket, [1 + m] slots of m done, [1 + nl + c] reads of c's
// retained part done, [1 + 2 nl + c] record c done (split: its slabs done),
// [1 + 3 nl + m] head of split record m done.
template <int NT>
__global__ void __launch_bounds__(NT) k_bwd_flow(SolveLevel S, SolveFlow F, cplx* y, long long ldy, int nrhs, int explicit_inv, cplx* part,
                                                 int* cnt, int* fail, cplx* tmp, FlowGroups G) {
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ int s_item, s_ok;
  {
    const int g = blockIdx.y;
    y += (size_t)g * G.rchunk * ldy;
    tmp += (size_t)g * G.rchunk * ldy;
    cnt += (size_t)g * G.cstride;
    part += (size_t)g * G.part_stride;
    nrhs = min(G.rchunk, nrhs - g * G.rchunk);
  }
  const int nl = S.nl;
  int* slots_done = cnt + 1;
  int* reads_done = cnt + 1 + nl;
  int* rec_done = cnt + 1 + 2 * nl;
  int* head_done = cnt + 1 + 3 * nl;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(cnt, 1), s_ok = 1;
    __syncthreads();
    const int it = s_item;
    __syncthreads();
    if (it >= F.nb) return;
    const int code = F.b_items[it];
    if (code >= kSlabBase) {
      const int m = (code - kSlabBase) >> 6, sl = (code - kSlabBase) & 63;
      if (threadIdx.x == 0) s_ok = wait_ge(head_done + m, 1, fail);  // (row slabs of Qt are strided: no prefetch)
      acquire_all(head_done + m);
      if (!s_ok) return;
      bwd_slab_body(S, m, sl, F.rec_ns_b[m], y, ldy, nrhs, tmp, smraw);
      publish_add(rec_done + m);
    } else if (code >= 0) {
      const int m = code;
      {
        const int b = S.bsz[m], e2 = b - S.kfin[m];
        if (e2 > 0) cta_prefetch_l2(S.chain + (explicit_inv ? S.Uinv_off[m] : S.U11_off[m]), (size_t)e2 * e2 * sizeof(cplx));
        if (!F.rec_ns_b[m]) cta_prefetch_l2(S.chain + S.Qt_off[m], (size_t)b * b * sizeof(cplx));
      }
      if (threadIdx.x == 0) {
        s_ok = wait_ge(slots_done + m, F.rec_nslot[m], fail);
        if (s_ok) s_ok = wait_ge(reads_done + m, F.reader_need[m], fail);  // nobody still reads the retained part
      }
      acquire_all(slots_done + m);
      if (!s_ok) return;
      const int e = S.bsz[m] - S.kfin[m];
      const int ns = F.rec_ns_b[m];
      bwd_body(S, m, y, ldy, nrhs, explicit_inv, part + (size_t)F.slot_off[F.rec_slot0[m]] * nrhs, (long long)e * nrhs, smraw, ns ? tmp : nullptr);
      publish(ns ? head_done + m : rec_done + m, 1);
    } else {
      const int sl = -1 - code;
      const int m = F.slot_m[sl], a = F.slot_c[sl];
      const int nC = S.C_ptr[m + 1] - S.C_ptr[m];
      const int c = a >= 0 ? S.C_nb[a] : -1;
      {
        const int e2 = S.bsz[m] - S.kfin[m];
        if (e2 > 0) cta_prefetch_l2(S.chain + (a >= 0 ? S.Ubar_off[a] : S.Uself_off[m]), (size_t)e2 * (a >= 0 ? S.bsz[c] : S.kfin[m]) * sizeof(cplx));
      }
      if (threadIdx.x == 0 && c >= 0 && F.slot_final[sl]) s_ok = wait_ge(rec_done + c, max(1, F.rec_ns_b[c]), fail);
      acquire_all(rec_done + (c >= 0 ? c : m));
      if (!s_ok) return;
      bwd_gather_to(S, m, a >= 0 ? a - S.C_ptr[m] : nC, y, ldy, nrhs, part + (size_t)F.slot_off[sl] * nrhs, reinterpret_cast<cplx*>(smraw));
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(slots_done + m, 1);
        if (c >= 0 && !F.slot_final[sl]) atomicAdd(reads_done + c, 1);
      }
    }
    __syncthreads();
  }
}

// (P v)[j] = v[src[j]] (gather, solve.hpp:18-23) or its inverse (scatter, :25-30).
__global__ void k_permute(const long long* src, long long len, const cplx* in, cplx* out, long long ldy, int nrhs, int scatter) {
  const long long total = len * nrhs;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total; idx += (long long)gridDim.x * blockDim.x) {
    const long long j = idx % len, c = idx / len;
    if (scatter)
      out[src[j] + c * ldy] = in[j + c * ldy];
    else
      out[j + c * ldy] = in[src[j] + c * ldy];
  }
}

__global__ void k_copy_cols(const cplx* in, cplx* out, long long len, long long ldy, int nrhs) {
  const long long total = len * nrhs;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total; idx += (long long)gridDim.x * blockDim.x) {
    const long long j = idx % len, c = idx / len;
    out[j + c * ldy] = in[j + c * ldy];
  }
}

// Dense root triangular solves (solve.hpp:55-58, :67-70); blocked by 64
// columns, one CTA.
__global__ void __launch_bounds__(512) k_root_trsv(const cplx* A, int n, cplx* y, long long ldy, int nrhs, int upper) {
  if (!upper) {
    for (int p = 0; p < n; ++p) {
      __syncthreads();
      for (int idx = threadIdx.x; idx < (n - p - 1) * nrhs; idx += blockDim.x) {
        const int i = p + 1 + idx % (n - p - 1), c = idx / (n - p - 1);
        const cplx l = A[i + (size_t)p * n], x = y[p + c * ldy];
        cplx v = y[i + c * ldy];
        v.x -= l.x * x.x - l.y * x.y;
        v.y -= l.x * x.y + l.y * x.x;
        y[i + c * ldy] = v;
      }
    }
  } else {
    for (int p = n - 1; p >= 0; --p) {
      __syncthreads();
      for (int c = threadIdx.x; c < nrhs; c += blockDim.x) y[p + c * ldy] = cdiv(y[p + c * ldy], A[p + (size_t)p * n]);
      __syncthreads();
      for (int idx = threadIdx.x; idx < p * nrhs; idx += blockDim.x) {
        const int i = idx % p, c = idx / p;
        const cplx u = A[i + (size_t)p * n], x = y[p + c * ldy];
        cplx v = y[i + c * ldy];
        v.x -= u.x * x.x - u.y * x.y;
        v.y -= u.x * x.y + u.y * x.x;
        y[i + c * ldy] = v;
      }
    }
  }
}

// Non-finite check of the right-hand side (solve.hpp:15).
__global__ void k_finite(const cplx* y, long long total, int* bad) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const cplx v = y[i];
    if (!isfinite(v.x) || !isfinite(v.y)) *bad = 1;
  }
}

// ----------------------------------------------------------------- launchers
static int cur_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

// Dynamic shared-memory opt-in, cached per (device, kernel).
static void smem_attr(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  std::lock_guard<std::mutex> g(mu);
  size_t& cur = done[{cur_device(), fn}];
  if (bytes > cur) {
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
      throw std::runtime_error("cudaFuncSetAttribute(MaxDynamicSharedMemorySize) failed");
    cur = bytes;
  }
}

// Co-resident grid for the cooperative level kernels (cached per device /
// kernel / smem).
template <class K>
static int coop_grid(K kernel, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, size_t>, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_tuple(cur_device(), (const void*)kernel, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int dev = 0, nsm = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, 256, smem);
  const int g = std::max(1, std::min(per, 2)) * nsm;
  if (per < 1) throw std::runtime_error("solve level kernel does not fit on an SM");
  cache[key] = g;
  return g;
}

void launch_fwd_level(const SolveLevel& S, const SolveSched& P, cplx* y, long long ldy, int nrhs, int explicit_inv, cudaStream_t s) {
  if (P.nbat <= 0) return;
  const size_t smem = 2 * (size_t)S.bmax * nrhs * sizeof(cplx) + 256 * sizeof(cplx);
  smem_attr((const void*)k_fwd_level, smem);
  const int grid = coop_grid(k_fwd_level, smem);
  SolveLevel Sv = S;
  SolveSched Pv = P;
  void* args[] = {&Sv, &Pv, &y, &ldy, &nrhs, &explicit_inv};
  const cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_fwd_level, grid, 256, args, smem, s);
  if (e != cudaSuccess) throw std::runtime_error(std::string("launch of k_fwd_level failed: ") + cudaGetErrorString(e));
}

void launch_bwd_level(const SolveLevel& S, const SolveSched& P, cplx* y, long long ldy, int nrhs, int explicit_inv, cplx* part, cudaStream_t s) {
  if (P.nbat <= 0) return;
  const size_t smem = 2 * (size_t)S.bmax * nrhs * sizeof(cplx) + 256 * sizeof(cplx);
  smem_attr((const void*)k_bwd_level, smem);
  const int grid = coop_grid(k_bwd_level, smem);
  long long pstride = (long long)S.bmax * nrhs;
  SolveLevel Sv = S;
  SolveSched Pv = P;
  void* args[] = {&Sv, &Pv, &y, &ldy, &nrhs, &explicit_inv, &part, &pstride};
  const cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_bwd_level, grid, 256, args, smem, s);
  if (e != cudaSuccess) throw std::runtime_error(std::string("launch of k_bwd_level failed: ") + cudaGetErrorString(e));
}

void launch_permute(const long long* src, long long len, cplx* y, cplx* tmp, long long ldy, int nrhs, int scatter, cudaStream_t s) {
  if (len <= 0) return;
  const int grid = (int)std::min<long long>(4096, (len * nrhs + 255) / 256);
  k_permute<<<grid, 256, 0, s>>>(src, len, y, tmp, ldy, nrhs, scatter);
  k_copy_cols<<<grid, 256, 0, s>>>(tmp, y, len, ldy, nrhs);
}

void launch_root_trsv(const cplx* A, int n, cplx* y, long long ldy, int nrhs, int upper, cudaStream_t s) {
  if (n > 0) k_root_trsv<<<1, 512, 0, s>>>(A, n, y, ldy, nrhs, upper);
}

void launch_finite(const cplx* y, long long total, int* bad, cudaStream_t s) {
  const int grid = (int)std::min<long long>(4096, (total + 255) / 256);
  if (total > 0) k_finite<<<grid, 256, 0, s>>>(y, total, bad);
}


static int flow_grid(const void* fn, int nt, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, size_t>, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_tuple(cur_device(), fn, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int dev = 0, nsm = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, nt, smem);
  if (per < 1) throw std::runtime_error("solve flow kernel does not fit on an SM");
  const int g = std::max(1, std::min(per, 2)) * nsm;
  cache[key] = g;
  return g;
}

// Right-hand-side groups (grid y): every group is an independent dataflow over
// its own columns, counters and ticket, so the groups' latency chains overlap.
// The x extent is cut so that all groups are resident together (CTAs are
// placed x-first: a full-width x would run the groups one after the other).
static void set_small_k_once() {
  const char* e = std::getenv("H2G_SOLVE_SMALLK");
  if (!e) return;
  static std::mutex mu;
  static std::map<int, bool> done;  // constant memory is per device
  std::lock_guard<std::mutex> lk(mu);
  bool& d = done[cur_device()];
  if (d) return;
  const int v = std::max(0, std::atoi(e));
  cudaMemcpyToSymbol(kSmallK, &v, sizeof v);
  d = true;
}
static int flow_ngroups(int nrhs, const FlowGroups& G) { return (nrhs + G.rchunk - 1) / G.rchunk; }
static int group_grid(int resident, int ng) { return std::max(1, (resident + ng - 1) / ng); }

// Threads per CTA of the dataflow kernels: a record's rotation (a b x b GEMV
// by one CTA) sits on the dependency chain, so the coarse levels with large
// blocks run wide CTAs. H2G_SOLVE_THREADS overrides (256 / 512 / 1024).
static int flow_threads(int bmax) {
  static const int forced = std::getenv("H2G_SOLVE_THREADS") ? std::atoi(std::getenv("H2G_SOLVE_THREADS")) : 0;
  if (forced == 256 || forced == 512 || forced == 1024) return forced;
  return bmax <= 48 ? 256 : (bmax <= 96 ? 512 : 1024);
}

template <int NT>
static void fwd_flow_nt(const SolveLevel& S, const SolveSched& P, const SolveFlow& F, cplx* y, long long ldy, int nrhs, int explicit_inv, int* cnt,
                        int* fail, cplx* tmp, const FlowGroups& G, cudaStream_t s) {
  const size_t smem = 2 * (size_t)S.bmax * std::min(nrhs, G.rchunk) * sizeof(cplx) + NT * sizeof(cplx);
  smem_attr((const void*)k_fwd_flow<NT>, smem);
  const int ng = flow_ngroups(nrhs, G);
  const int grid = std::min(group_grid(flow_grid((const void*)k_fwd_flow<NT>, NT, smem), ng), F.nf);
  k_fwd_flow<NT><<<dim3(grid, ng), NT, smem, s>>>(S, P, F, y, ldy, nrhs, explicit_inv, cnt, fail, tmp, G);
}

void launch_fwd_flow(const SolveLevel& S, const SolveSched& P, const SolveFlow& F, cplx* y, long long ldy, int nrhs, int explicit_inv, int* cnt,
                     int* fail, cplx* tmp, const FlowGroups& G, cudaStream_t s) {
  if (F.nf <= 0) return;
  set_small_k_once();
  cudaMemsetAsync(cnt, 0, ((size_t)(flow_ngroups(nrhs, G) - 1) * G.cstride + 2 * S.nl + 1) * sizeof(int), s);
  const int nt = flow_threads(S.bmax);
  if (nt == 256) fwd_flow_nt<256>(S, P, F, y, ldy, nrhs, explicit_inv, cnt, fail, tmp, G, s);
  else if (nt == 512) fwd_flow_nt<512>(S, P, F, y, ldy, nrhs, explicit_inv, cnt, fail, tmp, G, s);
  else fwd_flow_nt<1024>(S, P, F, y, ldy, nrhs, explicit_inv, cnt, fail, tmp, G, s);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("launch of k_fwd_flow failed: ") + cudaGetErrorString(e));
}

template <int NT>
static void bwd_flow_nt(const SolveLevel& S, const SolveFlow& F, cplx* y, long long ldy, int nrhs, int explicit_inv, cplx* part, int* cnt, int* fail,
                        cplx* tmp, const FlowGroups& G, cudaStream_t s) {
  const size_t smem = 2 * (size_t)S.bmax * std::min(nrhs, G.rchunk) * sizeof(cplx) + NT * sizeof(cplx);
  smem_attr((const void*)k_bwd_flow<NT>, smem);
  const int ng = flow_ngroups(nrhs, G);
  const int grid = std::min(group_grid(flow_grid((const void*)k_bwd_flow<NT>, NT, smem), ng), F.nb);
  k_bwd_flow<NT><<<dim3(grid, ng), NT, smem, s>>>(S, F, y, ldy, nrhs, explicit_inv, part, cnt, fail, tmp, G);
}

void launch_bwd_flow(const SolveLevel& S, const SolveFlow& F, cplx* y, long long ldy, int nrhs, int explicit_inv, cplx* part, int* cnt, int* fail,
                     cplx* tmp, const FlowGroups& G, cudaStream_t s) {
  if (F.nb <= 0) return;
  set_small_k_once();
  cudaMemsetAsync(cnt, 0, ((size_t)(flow_ngroups(nrhs, G) - 1) * G.cstride + 4 * S.nl + 1) * sizeof(int), s);
  const int nt = flow_threads(S.bmax);
  if (nt == 256) bwd_flow_nt<256>(S, F, y, ldy, nrhs, explicit_inv, part, cnt, fail, tmp, G, s);
  else if (nt == 512) bwd_flow_nt<512>(S, F, y, ldy, nrhs, explicit_inv, part, cnt, fail, tmp, G, s);
  else bwd_flow_nt<1024>(S, F, y, ldy, nrhs, explicit_inv, part, cnt, fail, tmp, G, s);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("launch of k_bwd_flow failed: ") + cudaGetErrorString(e));
}

}  // namespace h2g
