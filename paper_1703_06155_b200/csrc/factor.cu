// Level kernels of the B200 H² factorization. One batch = a set of mutually
// non-adjacent clusters of one level (plan.cpp); per batch four launches:
//   k_gram   step 0, part 1: Gram of the complement-projected fill-in stack
//   k_head   step 0, part 2 + step 1 + step 3a: truncation (Jacobi), Qtilde,
//            rotation of the diagonal block, unpivoted LU, self panels
//   panels   step 2 + step 3b (rotations, Lbar/Ubar, lift to the entry frame,
//            :359-362, :437-438) as k_gemm descriptors with e resolved on
//            the device from kfin, then k_mask
//   k_schur  step 3c: Schur products scattered to dense / fill-in targets
// Reference: proj/include/h2lu/factorization.hpp:260-440.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <set>
#include <mutex>
#include <stdexcept>
#include <string>

#include "factor.cuh"

namespace h2g {

namespace {

__device__ __forceinline__ cplx* blk(cplx* pool, int idx, int bmax) { return pool + (size_t)idx * bmax * bmax; }

// Workspace: shared memory if it fits, else a global slot per CTA.
struct Ws {
  cplx* p;
};

}  // namespace

// --------------------------------------------------------------------------
// Complement of the level-entry basis: Vp = Q[:, k:] from a Householder QR of
// V (b x korig); also the orthonormality guard of unitary_completion
// (dense_kernels.hpp:55-59).
__global__ void __launch_bounds__(256) k_complement(DevLevel L, cplx* gws) {
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ double red[32];
  const int t = blockIdx.x;
  const int b = L.bsz[t], k = L.korig[t], bm = L.bmax;
  cplx* ws = gws ? gws + (size_t)t * (2 * bm * bm + bm) : reinterpret_cast<cplx*>(smraw);
  cplx* A = ws;
  cplx* Q = ws + bm * bm;
  cplx* tau = ws + 2 * bm * bm;
  const cplx* V = L.V0 + (size_t)t * bm * bm;
  cplx* Vp = L.Vp + (size_t)t * bm * bm;
  if (k > 0) {
    double defect = 0.0;
    for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) {
      const int i = idx % k, j = idx / k;
      cplx s = czero();
      for (int p = 0; p < b; ++p) cfma(s, cconj(V[p + (size_t)i * b]), V[p + (size_t)j * b]);
      if (i == j) s.x -= 1.0;
      defect = fmax(defect, cabsd(s));
    }
    defect = cta_max(defect, red);
    if (defect > 1e-10) {
      if (threadIdx.x == 0) raise_error(L.err, 1, (1 << L.level) - 1 + t, L.level, -1, defect);
      return;
    }
  }
  if (k == b) return;
  if (k == 0) {
    cta_identity(b, b, Vp, b);
    return;
  }
  cta_copy(b, k, V, b, A, b);
  __syncthreads();
  cta_householder_q(b, k, A, b, Q, b, tau, red);
  cta_copy(b, b - k, Q + (size_t)k * b, b, Vp, b);
}

// H, U, then scratch for inverse iteration and the blocked QR
// H, U, aux (8 bm), X1, X2, Tm, Sm (bm^2 each), tau (bm)
__host__ __device__ inline size_t eig1_ws_cplx(int bm) { return (size_t)bm * bm * 6 + (size_t)bm * 9 + 16; }

// --------------------------------------------------------------------------
// Step 0, pass 1. The projected fill-in stack Y = Vp^H W (factorization.hpp:
// 278-296, Vp = complement of the level-entry basis) is reduced to partial
// Gram matrices by descriptor GEMMs (k_gemm); here the partials are summed,
// eigendecomposed (Jacobi) and truncated with the eps rule and floor of
// h2_matrix.hpp:287-290 / factorization.hpp:295. When the truncation
// threshold sits below ~1e-4 sigma_0 the Gram matrix cannot resolve it
// (sigma^2 meets the fp64 noise of ||G||), so a Rayleigh-Ritz refinement pass
// is requested: the stack is re-projected on the pass-1 directions
// (D1 = Vp U1) and eigendecomposed again (k_head), which resolves singular
// values down to ~eps_mach * sigma_0 like the reference's QR + SVD.
// Step 0, pass 1 on a 16-CTA thread-block cluster. The m x m Gram of the
// projected fill stack is distributed column-cyclically over the CTAs' shared
// memory (column c lives in CTA c % 16); the Householder tridiagonalization
// (zhetd2 scheme) runs with two cluster barriers per column: the owner of
// column k builds the reflector, every CTA forms its partial A v over its own
// columns, the partials are reduced through distributed shared memory and
// each CTA applies the rank-2 update to its own columns. CTA 0 then counts the
// eigenvalues above thr^2 (Sturm) and bisects the retained ones; vectors are
// formed by k_eigvec, the basis by k_eig1b. Threshold rule: factorization.hpp:
// 295-298 / h2_matrix.hpp:287-290.
constexpr int kHCmax = 16;

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}



// gH != nullptr: the cluster's Gram columns do not fit its shared memory
// (blocks beyond ~420 rows); each CTA then keeps its columns in global memory
// (gH, bmax^2 + 16 bmax per batch slot, L2 resident) and only the vectors in shared.
__global__ void __launch_bounds__(256) k_eig1c(DevLevel L, const int* batch_cl, int p0, cplx* gws, cplx* gH) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ double red[32];
  __shared__ int s_any;
  __shared__ cplx s_tau[2];
  __shared__ int s_skip[2];
  const int kHC = (int)cl.num_blocks();  // 1, 4, 8 or 16 CTAs per cluster
  const unsigned long long tm0 = (L.debug & 8) ? gtimer() : 0ull;
  unsigned long long tm1 = 0, tm2 = 0, tm3 = 0;
  const int rank = (int)cl.block_rank();
  const int q = blockIdx.x / kHC, p = p0 + q;
  const int t = batch_cl[q];
  const int b = L.bsz[t], k = L.korig[t], m = b - k, bm = L.bmax;
  const size_t bb = (size_t)bm * bm;
  cplx* ws = gws + (size_t)q * eig1_ws_cplx(bm);
  cplx* H = ws;  // reflectors out (m x m, ld m)
  double* aux = reinterpret_cast<double*>(ws + 2 * bb);
  const int ncl = (m + kHC - 1) / kHC;
  cplx* Hl = gH ? gH + (size_t)q * (bb + 16 * (size_t)bm) + (size_t)rank * m * ncl : reinterpret_cast<cplx*>(smraw);  // m x ncl local columns (col c = rank + kHC * jl)
  cplx* vbuf = gH ? reinterpret_cast<cplx*>(smraw) : Hl + (size_t)m * ncl;  // [2][m] reflector broadcast (owner)
  cplx* pbuf = vbuf + 2 * m;                  // [2][m] partial A v over own columns
  cplx* wfull = pbuf + 2 * m;                 // [2][m] reduced tau A v (each CTA its own copy)
  cplx* vv = wfull + 2 * m;                   // local copy of v (+ [m] next v, cluster path)
  if (threadIdx.x == 0) s_any = 0;
  __syncthreads();
  {
    int any = 0;
    for (int f = L.G_ptr[t] + threadIdx.x; f < L.G_ptr[t + 1]; f += blockDim.x) any |= L.fexists[L.G_fill[f]];
    if (any) s_any = 1;
  }
  __syncthreads();
  if (!s_any || m == 0) {
    // no fill-in: the basis stays (factorization.hpp:276)
    if (rank == 0 && threadIdx.x == 0) L.pass2[q] = 0, L.rank1[q] = 0, L.cmax[q] = 0.0, L.lam[(size_t)q * bm] = 0.0;
    return;  // uniform over the cluster
  }
  const int g0 = L.slot_g0[p], gn = L.slot_gn[p];
  __shared__ long long s_goff[128];
  for (int gb = 0; gb < gn; gb += 128) {
    const int gc = min(128, gn - gb);
    __syncthreads();
    for (int g = threadIdx.x; g < gc; g += blockDim.x) s_goff[g] = L.gram_off[g0 + gb + g];
    __syncthreads();
    for (int idx = threadIdx.x; idx < m * ncl; idx += blockDim.x) {
      const int i = idx % m, jl = idx / m, c = rank + kHC * jl;
      cplx s0 = gb ? Hl[idx] : czero(), s1 = czero(), s2 = czero(), s3 = czero();
      if (c < m) {
        const size_t e = i + (size_t)c * m;
        int g = 0;
        for (; g + 4 <= gc; g += 4) {
          s0 = cadd(s0, L.gram[s_goff[g] + e]);
          s1 = cadd(s1, L.gram[s_goff[g + 1] + e]);
          s2 = cadd(s2, L.gram[s_goff[g + 2] + e]);
          s3 = cadd(s3, L.gram[s_goff[g + 3] + e]);
        }
        for (; g < gc; ++g) s0 = cadd(s0, L.gram[s_goff[g] + e]);
      }
      Hl[idx] = cadd(cadd(s0, s1), cadd(s2, s3));
    }
  }
  if (L.debug & 8) tm1 = gtimer();
  // remote views of every CTA's partial / result buffers
  const cplx* rp[kHCmax];
#pragma unroll
  for (int rr = 0; rr < kHCmax; ++rr) {
    const int r2 = rr < kHC ? rr : 0;
    rp[rr] = cl.map_shared_rank(pbuf, r2);
  }
  cl.sync();
  if (kHC == 1 && m <= 64) {
    // small blocks, one CTA: warp 0 forms the reflector; the matvec runs as
    // (row, column-group) partials over all 256 threads, the rank-2 update
    // over all threads; four block barriers per column
    __shared__ int s_sk1[2];  // by column parity: a skipped column has no closing barrier
    __shared__ cplx s_tk1[2];
    cplx* vs = vbuf;       // v of the current column
    cplx* wsv = vbuf + m;  // w of the current column
    cplx* part = pbuf;     // [4][m] matvec partials (pbuf + wfull: 4m)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int kk = 0; kk + 1 < m; ++kk) {
      const int nk = m - kk - 1;
      cplx* x = Hl + (kk + 1) + (size_t)kk * m;
      if (warp == 0) {
        const cplx x0 = lane < nk ? x[lane] : czero();
        const cplx x1 = lane + 32 < nk ? x[lane + 32] : czero();
        double part2 = (lane >= 1 ? cabs2(x0) : 0.0) + cabs2(x1);
        for (int o = 16; o > 0; o >>= 1) part2 += __shfl_xor_sync(0xffffffffu, part2, o);
        const double xn2 = part2;
        const cplx al = make_double2(__shfl_sync(0xffffffffu, x0.x, 0), __shfl_sync(0xffffffffu, x0.y, 0));
        const bool skip = xn2 == 0.0 && al.y == 0.0;
        double beta = al.x;
        cplx tk = czero(), sc = czero();
        if (!skip) {
          beta = sqrt(cabs2(al) + xn2);
          if (al.x >= 0.0) beta = -beta;
          tk = cdiv(csub(cmk(beta, 0.0), al), cmk(beta, 0.0));
          sc = cdiv(cone(), csub(al, cmk(beta, 0.0)));
        }
        if (lane == 0) {
          aux[kk] = Hl[kk + (size_t)kk * m].x;  // d_k
          aux[bm + kk] = beta;                   // e_k
          reinterpret_cast<cplx*>(aux + 4 * bm)[kk] = tk;
          s_sk1[kk & 1] = skip;
          s_tk1[kk & 1] = tk;
        }
        if (!skip) {
          const cplx v0 = lane == 0 ? cone() : cmul(x0, sc), v1 = cmul(x1, sc);
          if (lane >= 1 && lane < nk) x[lane] = v0;
          if (lane + 32 < nk) x[lane + 32] = v1;
          if (lane < nk) vs[lane] = v0;
          if (lane + 32 < nk) vs[lane + 32] = v1;
        }
      }
      __syncthreads();
      if (s_sk1[kk & 1]) continue;  // uniform
      const cplx tk = s_tk1[kk & 1];
      const cplx* A22 = Hl + (kk + 1) + (size_t)(kk + 1) * m;
      {
        const int i = threadIdx.x & 63, g = threadIdx.x >> 6;
        if (i < nk) {
          cplx acc = czero();
          for (int j = g; j < nk; j += 4) cfma(acc, A22[i + (size_t)j * m], vs[j]);
          part[g * m + i] = acc;
        }
      }
      __syncthreads();
      // p = tau A22 v, c = v^H p (rows over the first two warps)
      cplx pi = czero();
      double cr = 0.0, ci = 0.0;
      if (threadIdx.x < 64) {
        const int i = threadIdx.x;
        if (i < nk) {
          pi = cmul(tk, cadd(cadd(part[i], part[m + i]), cadd(part[2 * m + i], part[3 * m + i])));
          const cplx tt = cmul(cconj(vs[i]), pi);
          cr = tt.x, ci = tt.y;
        }
        for (int o = 16; o > 0; o >>= 1) {
          cr += __shfl_xor_sync(0xffffffffu, cr, o);
          ci += __shfl_xor_sync(0xffffffffu, ci, o);
        }
        if (lane == 0) red[2 * warp] = cr, red[2 * warp + 1] = ci;
      }
      __syncthreads();
      if (threadIdx.x < 64 && (int)threadIdx.x < nk) {
        const cplx hc = cscale(cmul(cconj(tk), cmk(red[0] + red[2], red[1] + red[3])), 0.5);
        wsv[threadIdx.x] = csub(pi, cmul(hc, vs[threadIdx.x]));
      }
      __syncthreads();
      // rank-2 update of the trailing block: A22[i, j] -= v_i conj(w_j) + w_i conj(v_j)
      cplx* A22w = Hl + (kk + 1) + (size_t)(kk + 1) * m;
      for (int idx = threadIdx.x; idx < nk * nk; idx += blockDim.x) {
        const int i = idx % nk, j = idx / nk;
        cplx* a = A22w + i + (size_t)j * m;
        *a = csub(csub(*a, cmul(vs[i], cconj(wsv[j]))), cmul(wsv[i], cconj(vs[j])));
      }
      __syncthreads();
    }
    __syncthreads();
  } else {
  // One cluster barrier per column. Every CTA keeps the current reflector v
  // (and tau) itself: after the barrier that delivers the partials A v of
  // column kk, each CTA reduces w and v^H w, takes column kk+1 as its owner
  // published it before the barrier (pre-update copy), applies the rank-2
  // update of column kk to it and forms reflector kk+1 redundantly; the
  // owner also keeps it in its columns (the reflector output).
  cplx* pub = vbuf;            // [2][m] published next column (owner), rows kk+1..
  cplx* wb = wfull;            // [m] w (local)
  cplx* colb = wfull + m;      // [m] next column after the update (local)
  cplx* const vbase = vv;      // [2][m] reflectors by column parity (local)
  cplx* vn = vbase;            // where the next reflector goes
  // reflector of column kk from col[0 .. m-kk-1] = A[kk.., kk] (updated);
  // writes vn, s_tl, s_sk (aux from rank 0)
  // every thread forms the scalars itself from one block reduction (no
  // broadcast barrier); the partial sums alternate between two halves of red2
  __shared__ double red2[64];
  cplx r_tl = czero();
  auto reflector = [&](int kk, const cplx* col) {
    const int nk = m - kk - 1;
    double part = 0.0;
    for (int i = 1 + threadIdx.x; i < nk; i += blockDim.x) part += cabs2(col[1 + i]);
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    double* rb = red2 + 32 * (kk & 1);
    if ((threadIdx.x & 31) == 0) rb[threadIdx.x >> 5] = part;
    __syncthreads();
    double xn2 = 0.0;
    for (int u = 0; u < (int)(blockDim.x >> 5); ++u) xn2 += rb[u];
    const cplx al = col[1];
    const bool sk = xn2 == 0.0 && al.y == 0.0;
    double beta = al.x;
    cplx sc = czero();
    r_tl = czero();
    if (!sk) {
      beta = sqrt(cabs2(al) + xn2);
      if (al.x >= 0.0) beta = -beta;
      // tau = (beta - al) / beta, scale = 1 / (al - beta) (beta real)
      const double ib = 1.0 / beta;
      r_tl = cmk((beta - al.x) * ib, -al.y * ib);
      const double zx = al.x - beta, zy = al.y, iz = 1.0 / (zx * zx + zy * zy);
      sc = cmk(zx * iz, -zy * iz);
    }
    if (rank == 0 && threadIdx.x == 0) {
      aux[kk] = col[0].x;  // d_k
      aux[bm + kk] = beta; // e_k
      reinterpret_cast<cplx*>(aux + 4 * bm)[kk] = r_tl;
    }
    // skipped columns (tau = 0) use v = e_1: the update then subtracts zeros
    for (int i = threadIdx.x; i < nk; i += blockDim.x) vn[i] = i == 0 ? cone() : (sk ? czero() : cmul(col[1 + i], sc));
  };
  if (m > 1) {
    // column 0 lives in CTA 0 (Gram reduced and the cluster synchronised above)
    const cplx* c0 = gH ? gH + (size_t)q * (bb + 16 * (size_t)bm) : cl.map_shared_rank(Hl, 0);
    for (int i = threadIdx.x; i < m; i += blockDim.x) colb[i] = c0[i];
    __syncthreads();
    reflector(0, colb);
    __syncthreads();
  }
  for (int kk = 0; kk + 1 < m; ++kk) {
    const int buf = kk & 1;
    const int nk = m - kk - 1;
    // current reflector
    const cplx tk = r_tl;
    vv = vbase + (size_t)(kk & 1) * m;  // written by reflector(kk), visible since the last barrier
    vn = vbase + (size_t)((kk + 1) & 1) * m;
    // publish column kk+1 (rows kk+1..) before its update by column kk
    const int own1 = (kk + 1) % kHC;
    if (kk + 2 < m && rank == own1) {
      const cplx* src = Hl + (kk + 1) + (size_t)((kk + 1) / kHC) * m;
      for (int i = threadIdx.x; i < nk; i += blockDim.x) pub[(size_t)buf * m + i] = src[i];
    }
    // partial p over own columns c > kk (local rows kk+1 .. m-1)
    cplx* pb = pbuf + (size_t)buf * m;
    {
      const int jl0 = (kk + 1 - rank + kHC - 1) / kHC;  // first local column with c > kk
      for (int i = threadIdx.x; i < nk; i += blockDim.x) {
        cplx sacc = czero();
        for (int jl = max(jl0, 0); jl < ncl; ++jl) {
          const int c = rank + kHC * jl;
          if (c >= m) break;
          cfma(sacc, Hl[(kk + 1 + i) + (size_t)jl * m], vv[c - kk - 1]);
        }
        pb[i] = sacc;
      }
    }
    cl.sync();  // partials of column kk and the published column kk+1 ready
    // the owner stores reflector kk below the subdiagonal of its column kk
    // (nobody reads that column any more; earlier, other CTAs may still have
    // been copying it)
    if (rank == kk % kHC) {
      cplx* x = Hl + (kk + 1) + (size_t)(kk / kHC) * m;
      for (int i = 1 + threadIdx.x; i < nk; i += blockDim.x) x[i] = vv[i];
    }
    // w = tau * sum_r p_r (rank order), c = v^H w
    double dr = 0.0, di = 0.0;
    for (int i = threadIdx.x; i < nk; i += blockDim.x) {
      cplx parts[kHCmax];
#pragma unroll
      for (int rr = 0; rr < kHCmax; ++rr)
        if (rr < kHC) parts[rr] = rp[rr][(size_t)buf * m + i];
      cplx sacc = czero();
#pragma unroll
      for (int rr = 0; rr < kHCmax; ++rr)
        if (rr < kHC) sacc = cadd(sacc, parts[rr]);
      sacc = cmul(tk, sacc);
      wb[i] = sacc;
      const cplx tt = cmul(cconj(vv[i]), sacc);
      dr += tt.x;
      di += tt.y;
    }
    for (int o = 16; o > 0; o >>= 1) {
      dr += __shfl_xor_sync(0xffffffffu, dr, o);
      di += __shfl_xor_sync(0xffffffffu, di, o);
    }
    {
      const int wi = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
      if ((threadIdx.x & 31) == 0) red[wi] = dr, red[16 + wi] = di;
      __syncthreads();
      dr = 0.0, di = 0.0;
      for (int u = 0; u < nw; ++u) dr += red[u], di += red[16 + u];
    }
    // w = w - 1/2 conj(tau) c v
    const cplx hc = cscale(cmul(cconj(tk), cmk(dr, di)), 0.5);
    // next column: the published copy with this column's update (same
    // expression as the owner's own update below, so the copies agree)
    if (kk + 2 < m) {
      const cplx* pc = cl.map_shared_rank(pub, own1) + (size_t)buf * m;
      const cplx wc = csub(wb[0], cmul(hc, vv[0]));
      for (int i = threadIdx.x; i < nk; i += blockDim.x) {
        const cplx wi2 = csub(wb[i], cmul(hc, vv[i]));
        cplx av = pc[i];
        av = csub(av, cmul(vv[i], cconj(wc)));
        av = csub(av, cmul(wi2, cconj(vv[0])));
        colb[i] = av;
      }
    }
    // rank-2 update of own columns c > kk: A[i, c] -= v_i conj(w_c) + w_i conj(v_c)
    {
      const int jl0 = max((kk + 1 - rank + kHC - 1) / kHC, 0);
      const int ncols = ncl - jl0;
      for (int idx = threadIdx.x; idx < nk * ncols; idx += blockDim.x) {
        const int i = idx % nk, jl = jl0 + idx / nk;
        const int c = rank + kHC * jl;
        if (c >= m) continue;
        const int jc = c - kk - 1;
        const cplx wi2 = csub(wb[i], cmul(hc, vv[i])), wc = csub(wb[jc], cmul(hc, vv[jc]));
        cplx* a = Hl + (kk + 1 + i) + (size_t)jl * m;
        cplx av = *a;
        av = csub(av, cmul(vv[i], cconj(wc)));
        av = csub(av, cmul(wi2, cconj(vv[jc])));
        *a = av;
      }
    }
    __syncthreads();
    if (kk + 2 < m) reflector(kk + 1, colb);
    __syncthreads();
  }
  }  // cluster path
  if (L.debug & 8) tm2 = gtimer();
  // last diagonal, reflectors to global memory
  if (rank == (m - 1) % kHC && threadIdx.x == 0) {
    aux[m - 1] = Hl[(m - 1) + (size_t)((m - 1) / kHC) * m].x;
    aux[bm + m - 1] = 0.0;
  }
  for (int idx = threadIdx.x; idx < m * ncl; idx += blockDim.x) {
    const int i = idx % m, c = rank + kHC * (idx / m);
    if (c < m) H[i + (size_t)c * m] = Hl[idx];
  }
  cl.sync();
  // ---- every CTA (redundantly, identical results): spectrum edge and rank;
  // the retained eigenvalues are split over the CTAs of the cluster
  __shared__ double s_lo, s_hi, s_piv, s_s0, s_thr;
  __shared__ int s_r, s_need;
  double cm = 0.0;
  for (int c = threadIdx.x; c < L.slot_cn[p]; c += blockDim.x) cm = fmax(cm, L.colnorm[L.slot_c0[p] + c]);
  const double cmax = cta_max(cm, red);
  double* dg = reinterpret_cast<double*>(smraw);  // local columns no longer needed
  double* ed = dg + m;
  for (int i = threadIdx.x; i < m; i += blockDim.x) dg[i] = aux[i], ed[i] = aux[bm + i];
  __syncthreads();
  if (threadIdx.x == 0) {
    double lo = 0.0, hi = 0.0, emax = 0.0;
    for (int i = 0; i < m; ++i) {
      const double off = (i > 0 ? fabs(ed[i - 1]) : 0.0) + (i + 1 < m ? fabs(ed[i]) : 0.0);
      lo = i == 0 ? dg[i] - off : fmin(lo, dg[i] - off);
      hi = i == 0 ? dg[i] + off : fmax(hi, dg[i] + off);
      if (i + 1 < m) emax = fmax(emax, ed[i] * ed[i]);
    }
    const double span = fmax(hi - lo, 1e-300);
    lo -= 1e-14 * span;
    hi += 1e-14 * span;
    s_lo = lo, s_hi = hi;
    s_piv = 2.2250738585072014e-308 * fmax(1.0, emax);
  }
  __syncthreads();
  // largest eigenvalue by multisection: every thread tests one point of the
  // current bracket, so each round shrinks it (blockDim.x + 1)-fold (more
  // points per thread saturate the FP64 pipe without saving a round)
  double* e2 = ed + m;
  for (int i = threadIdx.x; i + 1 < m; i += blockDim.x) e2[i] = ed[i] * ed[i];
  {
    constexpr int P = 1;
    __shared__ double s_a, s_b;
    if (threadIdx.x == 0) s_a = s_lo, s_b = s_hi;
    __syncthreads();
    const int npts = blockDim.x * P;
    for (int round = 0; round < 12; ++round) {
      const double a = s_a, bnd = s_b;
      if (bnd - a <= 2e-16 * fmax(fabs(a), fabs(bnd))) break;
      double x[P];
      int c[P];
#pragma unroll
      for (int pp = 0; pp < P; ++pp) x[pp] = a + (bnd - a) * (double)(threadIdx.x * P + pp + 1) / (double)(npts + 1);
      sturm_count_p<P>(m, dg, e2, x, s_piv, c);  // #eigenvalues below x
      // points below which fewer than m eigenvalues lie (monotone in x)
      int below = 0;
#pragma unroll
      for (int pp = 0; pp < P; ++pp) below += __syncthreads_count(c[pp] < m);
      if (threadIdx.x == 0) {
        s_a = below == 0 ? a : a + (bnd - a) * (double)below / (double)(npts + 1);
        s_b = below == npts ? bnd : a + (bnd - a) * (double)(below + 1) / (double)(npts + 1);
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) s_s0 = 0.5 * (s_a + s_b);  // lmax (temporarily)
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double lo = s_lo, hi = s_hi, pivmin = s_piv;
    (void)lo;
    (void)hi;
    const double lmax = s_s0;
    const double s0 = sqrt(fmax(lmax, 0.0));
    const double thr = fmax(fmax(L.eps * s0, L.eps * cmax), 1e-300);
    int r = 0;
    if (s0 > 0.0) r = m - sturm_count(m, dg, ed, thr * thr, pivmin);
    s_r = max(0, min(r, m));
    s_lo = lo, s_hi = hi, s_piv = pivmin, s_s0 = s0, s_thr = thr;
    // the Gram resolves eigenvalues to ~eps_mach * lmax: below ~1e-4 sigma_0
    // the truncation needs the refinement pass (k_eig1_refine)
    s_need = s0 > 0.0 && (thr < L.refine_below * s0 || (L.debug & 4));  // debug bit 2: always refine
  }
  __syncthreads();
  const int r = s_r;
  if (L.debug & 8) tm3 = gtimer();
  if (!s_need) multisect_top(m, dg, e2, r, s_lo, s_hi, s_piv, aux + 2 * bm, rank, kHC);
  if (rank != 0) return;
  if ((L.debug & 8) && threadIdx.x == 0)
    printf("[h2g] eig1c-timing level %d cl %d kHC %d m %d r %d: gram %.1f us tridiag %.1f us lmax+rank %.1f us multisect %.1f us\n", L.level, t, kHC, m, r,
           (tm1 - tm0) * 1e-3, (tm2 - tm1) * 1e-3, (tm3 - tm2) * 1e-3, (gtimer() - tm3) * 1e-3);
  if (threadIdx.x == 0) {
    L.pass2[q] = s_need ? 2 : 0;  // 2: refinement requested
    L.rank1[q] = r;
    L.cmax[q] = cmax;
    L.lam[(size_t)q * bm] = s_s0;
    if (L.debug & 1) printf("[h2g] eig1 level %d cluster %d m %d cmax %.3e s0 %.3e thr %.3e r %d%s\n", L.level, t, m, cmax, s_s0, s_thr, r, s_need ? " (refine)" : "");
  }
}

// Rare path (thr < 1e-4 sigma_0, e.g. eps_fill < 1e-4): full Jacobi
// decomposition of the pass-1 Gram, D1 = Vp U1 sorted, then the
// Rayleigh-Ritz refinement pass in k_head.
__global__ void __launch_bounds__(256) k_eig1_refine(DevLevel L, const int* batch_cl, int p0, cplx* gws) {
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ double red[32];
  const int q = blockIdx.x, p = p0 + q;
  if (L.pass2[q] != 2) return;
  const int t = batch_cl[q];
  const int b = L.bsz[t], k = L.korig[t], m = b - k, bm = L.bmax;
  const size_t bb = (size_t)bm * bm;
  cplx* ws = gws + (size_t)q * eig1_ws_cplx(bm);
  cplx* H = ws;
  cplx* U = ws + bb;
  double* lam = reinterpret_cast<double*>(smraw);
  int* ord = reinterpret_cast<int*>(lam + bm);
  int* pr = ord + bm;
  double* rot = reinterpret_cast<double*>(pr + bm + 2);
  cplx* D1 = L.dir + (size_t)q * bb;
  const cplx* Vp = L.Vp + (size_t)t * bb;
  const int g0 = L.slot_g0[p], gn = L.slot_gn[p];
  for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x) {
    cplx s = czero();
    for (int g = 0; g < gn; ++g) s = cadd(s, L.gram[L.gram_off[g0 + g] + idx]);
    H[idx] = s;
  }
  double dmax = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) dmax = fmax(dmax, H[i + i * m].x);
  dmax = cta_max(dmax, red);
  __syncthreads();
  cta_jacobi_eig(m, H, U, rot, pr, red, 1e-17 * dmax);
  for (int i = threadIdx.x; i < m; i += blockDim.x) lam[i] = sqrt(fmax(H[i + i * m].x, 0.0));
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    int rk = 0;
    for (int j = 0; j < m; ++j) rk += (lam[j] > lam[i]) || (lam[j] == lam[i] && j < i);
    ord[rk] = i;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < b * m; idx += blockDim.x) {
    const int i = idx % b, j = idx / b;
    cplx v = czero();
    const int col = ord[j];
    for (int rr = 0; rr < m; ++rr) cfma(v, Vp[i + (size_t)rr * b], U[rr + col * m]);
    D1[i + (size_t)j * b] = v;
  }
  double* lout = L.lam + (size_t)q * bm;
  for (int i = threadIdx.x; i < m; i += blockDim.x) lout[i] = lam[ord[i]];
  __syncthreads();
  if (threadIdx.x == 0) {
    const double s0 = lam[ord[0]];
    const double thr = fmax(fmax(L.eps * s0, L.eps * L.cmax[q]), 1e-300);
    int rr = 0;
    while (rr < m && lam[ord[rr]] > thr) ++rr;
    L.pass2[q] = 1, L.rank1[q] = rr;
  }
}

// Eigenvectors of the retained eigenvalues: inverse iteration on T (thread 0,
// work arrays in shared memory; eigenvalues closer than 1e-8 ||T|| form a
// cluster handled by one CTA and Gram-Schmidt'ed against each other), then
// the back-transformation by the tridiagonalisation reflectors (whole CTA).
template <int kPer>  // entries of an eigenvector per lane: m <= 32 kPer
__global__ void __launch_bounds__(256) k_eigvec(DevLevel L, const int* batch_cl, cplx* gws, int wpc) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int q = blockIdx.x;
  if (L.pass2[q]) return;
  const int r = L.rank1[q];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.y * wpc + warp;  // one warp per retained eigenvector
  if ((int)blockIdx.y * wpc >= r) return;  // uniform over the CTA
  const int t = batch_cl[q];
  const int b = L.bsz[t], k = L.korig[t], m = b - k, bm = L.bmax;
  const size_t bb = (size_t)bm * bm;
  cplx* ws = gws + (size_t)q * eig1_ws_cplx(bm);
  const cplx* H = ws;
  cplx* U = ws + bb;
  const double* aux = reinterpret_cast<const double*>(ws + 2 * bb);
  const double* glam = aux + 2 * bm;
  const cplx* tau = reinterpret_cast<const cplx*>(aux + 4 * bm);
  double* dg = reinterpret_cast<double*>(smraw);
  double* ed = dg + m;
  for (int i = threadIdx.x; i < m; i += blockDim.x) dg[i] = aux[i], ed[i] = aux[bm + i];
  __syncthreads();
  // every warp stays for the staged back-transformation below; idle ones
  // (j >= r or beyond wpc) only help staging
  const bool act = j < r && warp < wpc;
  const unsigned long long tv0 = (L.debug & 8) ? gtimer() : 0ull;
  // per-warp work arrays: U factor (dd, du, du2, 1/dd), multipliers, pivots, z
  double* wk = ed + m + (size_t)min(warp, wpc - 1) * 7 * m;
  double* dd = wk;
  double* du = wk + m;
  double* du2 = wk + 2 * m;
  double* rdd = wk + 3 * m;
  double* fl = wk + 4 * m;
  double* z = wk + 5 * m;
  unsigned char* pv = reinterpret_cast<unsigned char*>(wk + 6 * m);
  if (act && lane == 0) {
    // inverse iteration from a per-eigenvalue pseudo-random start: (near-)
    // degenerate eigenvalues get independent vectors of their invariant
    // subspace; k_eig1b orthonormalises the retained set as a whole.
    // T - lam I = P L U is factored once (partial pivoting, tiny pivots
    // replaced as in tri_shift_solve) and reused for the three solves.
    double emax = 0.0;
    for (int i = 0; i + 1 < m; ++i) emax = fmax(emax, ed[i] * ed[i]);
    const double tiny = 2.2250738585072014e-308 * fmax(1.0, emax) * 1e10 + 1e-300;
    const double lam = glam[j];
    double dcur = dg[0] - lam;  // dd[i] while eliminating row i+1
    double dnext_e = m > 1 ? ed[0] : 0.0;  // du[i] (may be modified by a swap)
    for (int i = 0; i + 1 < m; ++i) {
      const double sub = ed[i];                     // dl[i]
      const double dn = dg[i + 1] - lam;            // dd[i+1] before elimination
      const double un = i + 2 < m ? ed[i + 1] : 0.0; // du[i+1]
      if (fabs(dcur) >= fabs(sub)) {
        if (fabs(dcur) < tiny) dcur = dcur >= 0 ? tiny : -tiny;
        const double f = sub * rcp_nr(dcur);
        dd[i] = dcur, du[i] = dnext_e, du2[i] = 0.0, fl[i] = f, pv[i] = 0;
        dcur = dn - f * dnext_e;
        dnext_e = un;
      } else {
        const double f = dcur * rcp_nr(sub);
        dd[i] = sub, du[i] = dn, du2[i] = un, fl[i] = f, pv[i] = 1;
        dcur = dnext_e - f * dn;
        dnext_e = -f * un;
      }
      rdd[i] = rcp_nr(dd[i]);
    }
    if (fabs(dcur) < tiny) dcur = dcur >= 0 ? tiny : -tiny;
    dd[m - 1] = dcur;
    rdd[m - 1] = 1.0 / dcur;
    for (int i = 0; i < m; ++i) {
      unsigned h = (unsigned)(i * 2654435761u) ^ (unsigned)((j + 1) * 40503u);
      h ^= h >> 13;
      h *= 0x5bd1e995u;
      h ^= h >> 15;
      z[i] = 1.0 + 0.5 * ((double)(h & 0xffff) / 65535.0 - 0.5);
    }
    for (int it = 0; it < 3; ++it) {
      // forward: the row operations of the factorization
      double zi = z[0];
      for (int i = 0; i + 1 < m; ++i) {
        const double zn = z[i + 1];
        if (!pv[i]) {
          z[i] = zi;
          zi = zn - fl[i] * zi;
        } else {
          z[i] = zn;
          zi = zi - fl[i] * zn;
        }
      }
      z[m - 1] = zi;
      // back substitution with U (two superdiagonals)
      double z1 = z[m - 1] * rdd[m - 1], z2 = 0.0;
      z[m - 1] = z1;
      double nrm = z1 * z1;
      for (int i = m - 2; i >= 0; --i) {
        const double zi2 = (z[i] - du[i] * z1 - du2[i] * z2) * rdd[i];
        z[i] = zi2;
        z2 = z1, z1 = zi2;
        nrm += zi2 * zi2;
      }
      const double inv = nrm > 0.0 ? 1.0 / sqrt(nrm) : 0.0;
      for (int i = 0; i < m; ++i) z[i] *= inv;
    }
  }
  __syncwarp();
  const unsigned long long tv1 = (L.debug & 8) ? gtimer() : 0ull;
  // back-transform y = Q z, Q = H_0 ... H_{m-2}: reflectors staged CH at a
  // time in shared memory by the whole CTA (coalesced), then every warp
  // streams its vector through them (lane owns entries lane, lane + 32, ...)
  constexpr int CH = 8;
  cplx* Hs = reinterpret_cast<cplx*>(dg + (size_t)(2 + 7 * wpc) * m + (((2 + 7 * wpc) * m) & 1));  // [CH][m]
  __shared__ cplx ts[CH];
  cplx y[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int i = lane + 32 * u;
    y[u] = (act && i < m) ? cmk(z[i], 0.0) : czero();
  }
  for (int k1 = m - 2; k1 >= 0; k1 -= CH) {
    const int k0 = max(0, k1 - CH + 1);
    __syncthreads();  // previous chunk consumed
    {
      // flattened (column, row) index so each thread has its loads in flight at once
      const int tot = (k1 - k0 + 1) * m;
      for (int base = 0; base < tot; base += 8 * (int)blockDim.x) {
        cplx tmp[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int idx = base + u * (int)blockDim.x + (int)threadIdx.x;
          const int c = k0 + idx / m, i = idx % m;
          tmp[u] = (idx < tot && i > 0 && i < m - c - 1) ? H[(c + 1) + i + (size_t)c * m] : cone();
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int idx = base + u * (int)blockDim.x + (int)threadIdx.x;
          if (idx < tot) Hs[idx] = tmp[u];
        }
      }
    }
    if (threadIdx.x <= k1 - k0) ts[threadIdx.x] = tau[k0 + threadIdx.x];
    __syncthreads();
    if (!act) continue;
    for (int kk = k1; kk >= k0; --kk) {
      const cplx tk = ts[kk - k0];
      if (tk.x == 0.0 && tk.y == 0.0) continue;
      const cplx* v = Hs + (size_t)(kk - k0) * m - (kk + 1);  // v[i] for global row i > kk
      double sr = 0.0, si = 0.0, sr2 = 0.0, si2 = 0.0;
      const int u0 = ((kk + 1) / 32) & ~1, u1 = (m + 31) / 32;  // warp-uniform live range
#pragma unroll
      for (int u = 0; u < kPer; u += 2) {
        if (u >= u1) break;
        if (u + 2 <= u0) continue;
        const int i = lane + 32 * u, i2 = i + 32;
        if (i > kk && i < m) {
          const cplx vc = cconj(v[i]);
          sr += vc.x * y[u].x - vc.y * y[u].y;
          si += vc.x * y[u].y + vc.y * y[u].x;
        }
        if (i2 > kk && i2 < m) {
          const cplx vc = cconj(v[i2]);
          sr2 += vc.x * y[u + 1].x - vc.y * y[u + 1].y;
          si2 += vc.x * y[u + 1].y + vc.y * y[u + 1].x;
        }
      }
      sr += sr2, si += si2;
      for (int o = 16; o > 0; o >>= 1) {
        sr += __shfl_xor_sync(0xffffffffu, sr, o);
        si += __shfl_xor_sync(0xffffffffu, si, o);
      }
      const cplx sc = cmul(tk, cmk(sr, si));
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        if (u >= u1) break;
        if (u < u0) continue;
        const int i = lane + 32 * u;
        if (i > kk && i < m) y[u] = csub(y[u], cmul(v[i], sc));
      }
    }
  }
  if (!act) return;
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int i = lane + 32 * u;
    if (i < m) U[i + (size_t)m * j] = y[u];
  }
  if ((L.debug & 8) && lane == 0 && j == 0)
    printf("[h2g] eigvec-timing level %d m %d r %d: inverse iteration %.1f us back-transform %.1f us\n", L.level, m, r, (tv1 - tv0) * 1e-3, (gtimer() - tv1) * 1e-3);
}

// D1 = Vp Qm with Qm = H_0^H ... H_{r-1}^H from a Householder QR of the
// retained eigenvectors U_r: [new | complement]. k_eig1b: blocked QR of U_r,
// the explicit reflectors Y and tau; k_eig1_apply: D1 row by row.
__global__ void __launch_bounds__(256) k_eig1b(DevLevel L, const int* batch_cl, cplx* gws) {
  __shared__ cplx tile_sm[kTileSmemCplx];
  __shared__ double red[32];
  __shared__ cplx tau[512];
  extern __shared__ __align__(16) unsigned char qsm[];
  const int q = blockIdx.x;
  if (L.pass2[q]) return;
  const int r = L.rank1[q];
  const int t = batch_cl[q];
  const int b = L.bsz[t], k = L.korig[t], m = b - k, bm = L.bmax;
  const size_t bb = (size_t)bm * bm;
  cplx* ws = gws + (size_t)q * eig1_ws_cplx(bm);
  cplx* U = ws + bb;
  if (r == 0 || m == 0) return;
  cplx* P = reinterpret_cast<cplx*>(qsm);  // m x 16 panel
  __shared__ cplx Tb[16 * 16];
  cplx* Wq = ws + 2 * bb + 4 * bm;
  cplx* Wq2 = Wq + (size_t)16 * r;
  cta_householder_qr_blocked(m, r, U, m, tau, red, tile_sm, P, Tb, Wq, Wq2);
  cplx* Y = ws;  // m x r explicit reflectors (H no longer needed)
  for (int idx = threadIdx.x; idx < m * r; idx += blockDim.x) {
    const int i = idx % m, jj = idx / m;
    Y[idx] = i < jj ? czero() : (i == jj ? cone() : U[i + (size_t)jj * m]);
  }
  cplx* tau_g = ws + 2 * bb + 4 * bm + 4 * bb;  // after X1, X2, Tm, Sm
  for (int i = threadIdx.x; i < r; i += blockDim.x) tau_g[i] = tau[i];
}

// The same QR on a thread-block cluster: the columns of U_r are spread
// column-cyclically over the CTAs' shared memory; per column the owner forms
// the reflector (one warp), publishes it, one cluster barrier, and every CTA
// applies it to its own later columns (a warp per column). Same reflector
// convention and outputs as k_eig1b (Y unit lower trapezoidal, tau).
// gU != nullptr: the local columns live in global memory (blocks too large
// for the cluster's shared memory, as in k_eig1c).
__global__ void __launch_bounds__(256) k_eig1b_cl(DevLevel L, const int* batch_cl, cplx* gws, cplx* gU) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smraw[];
  const int kHC = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  const int q = blockIdx.x / kHC;
  if (L.pass2[q]) return;  // uniform over the cluster
  const int r = L.rank1[q];
  const int t = batch_cl[q];
  const int b = L.bsz[t], k = L.korig[t], m = b - k, bm = L.bmax;
  if (r == 0 || m == 0) return;
  const size_t bb = (size_t)bm * bm;
  cplx* ws = gws + (size_t)q * eig1_ws_cplx(bm);
  const cplx* U = ws + bb;
  cplx* Y = ws;
  cplx* tau_g = ws + 2 * bb + 4 * bm + 4 * bb;
  const int ncl = (r + kHC - 1) / kHC;
  cplx* Ul = gU ? gU + (size_t)q * (bb + 16 * (size_t)bm) + (size_t)rank * m * ncl : reinterpret_cast<cplx*>(smraw);  // m x ncl, local column jl = global rank + kHC jl
  cplx* pubw = gU ? reinterpret_cast<cplx*>(smraw) : Ul + (size_t)m * ncl;  // [2][m] published reflector (owner), w[0] = 1
  cplx* wv = pubw + 2 * m;                    // local copy
  __shared__ cplx pubt[2];
  __shared__ cplx s_tk;
  for (int idx = threadIdx.x; idx < m * ncl; idx += blockDim.x) {
    const int i = idx % m, jl = idx / m, c = rank + kHC * jl;
    Ul[idx] = c < r ? U[i + (size_t)c * m] : czero();
  }
  cl.sync();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int s = min(m, r);
  for (int j = 0; j < s; ++j) {
    const int owner = j % kHC, buf = j & 1, mr = m - j;
    if (rank == owner && warp == 0) {
      cplx* x = Ul + j + (size_t)(j / kHC) * m;
      double part = 0.0;
      for (int i = 1 + lane; i < mr; i += 32) part += cabs2(x[i]);
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      const double tail = part;
      const cplx c0 = x[0];
      const double tiny = 2.2250738585072014e-308;
      const bool triv = tail <= tiny && c0.y * c0.y <= tiny;
      cplx tk = czero(), rden = czero();
      if (!triv) {
        double beta = sqrt(cabs2(c0) + tail);
        if (c0.x >= 0.0) beta = -beta;
        const cplx denom = csub(c0, cmk(beta, 0.0));
        tk = cconj(cdiv(csub(cmk(beta, 0.0), c0), cmk(beta, 0.0)));
        rden = cdiv(cone(), denom);
      }
      cplx* pw = pubw + (size_t)buf * m;
      for (int i = lane; i < mr; i += 32) {
        const cplx v = i == 0 ? cone() : (triv ? czero() : cmul(x[i], rden));
        if (i > 0) x[i] = v;
        pw[i] = v;
      }
      if (lane == 0) pubt[buf] = tk, tau_g[j] = tk;
    }
    if (kHC == 1) __syncthreads();  // single CTA: a block barrier suffices
    else cl.sync();                  // reflector j published
    const cplx* ow = cl.map_shared_rank(pubw, owner) + (size_t)buf * m;
    if (threadIdx.x == 0) s_tk = cl.map_shared_rank(pubt, owner)[buf];
    for (int i = threadIdx.x; i < mr; i += blockDim.x) wv[i] = ow[i];
    __syncthreads();
    const cplx tk = s_tk;
    if (tk.x != 0.0 || tk.y != 0.0) {
      // own columns c > j, a warp per column
      const int jl0 = (j + 1 - rank + kHC - 1) / kHC;
      for (int jl = max(jl0, 0) + warp; jl < ncl; jl += nw) {
        const int c = rank + kHC * jl;
        if (c >= r) break;
        cplx* a = Ul + j + (size_t)jl * m;
        cplx tt = czero();
        for (int i = 1 + lane; i < mr; i += 32) cfma(tt, cconj(wv[i]), a[i]);
        for (int o = 16; o > 0; o >>= 1) {
          tt.x += __shfl_xor_sync(0xffffffffu, tt.x, o);
          tt.y += __shfl_xor_sync(0xffffffffu, tt.y, o);
        }
        tt = cmul(tk, cadd(tt, a[0]));
        __syncwarp();
        if (lane == 0) a[0] = csub(a[0], tt);
        for (int i = 1 + lane; i < mr; i += 32) a[i] = csub(a[i], cmul(wv[i], tt));
        __syncwarp();
      }
    }
    __syncthreads();
  }
  cl.sync();  // nobody reads this CTA's published reflectors any more
  // Y (m x r): unit lower trapezoidal reflectors
  for (int idx = threadIdx.x; idx < m * ncl; idx += blockDim.x) {
    const int i = idx % m, jl = idx / m, c = rank + kHC * jl;
    if (c < r) Y[i + (size_t)c * m] = i < c ? czero() : (i == c ? cone() : Ul[idx]);
  }
}

// D1 = Vp H_0^H H_1^H ... H_{r-1}^H applied row by row: every row of D1 is
// transformed independently (d <- d - conj(tau_j) (d y_j) y_j^H), so one warp
// per row streams through the r reflectors with no block-wide barrier. This
// replaces the compact-WY chain (S = Y^H Y, T recurrence, three GEMMs).
template <int KP>  // columns per lane: m <= 32 KP
__global__ void __launch_bounds__(256) k_eig1_apply(DevLevel L, const int* batch_cl, const cplx* gws) {
  const int q = blockIdx.x;
  if (L.pass2[q]) return;
  const int t = batch_cl[q];
  const int b = L.bsz[t], k = L.korig[t], m = b - k, bm = L.bmax;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int row = blockIdx.y * (blockDim.x / 32) + warp;
  if (row >= b || m == 0) return;
  const size_t bb = (size_t)bm * bm;
  const int r = L.rank1[q];
  const cplx* ws = gws + (size_t)q * eig1_ws_cplx(bm);
  const cplx* Y = ws;                                    // m x r, unit lower trapezoidal
  const cplx* tau_g = ws + 2 * bb + 4 * bm + 4 * bb;
  const cplx* Vp = L.Vp + (size_t)t * bb;
  cplx* D1 = L.dir + (size_t)q * bb;
  cplx d[KP];
#pragma unroll
  for (int u = 0; u < KP; ++u) {
    const int c = lane + 32 * u;
    d[u] = c < m ? Vp[row + (size_t)c * b] : czero();
  }
  // reflector j + 1 is loaded (predicated, all loads in flight together)
  // while reflector j is applied
  cplx yn[KP];
  auto load = [&](int j) {
    const cplx* y = Y + (size_t)j * m;
#pragma unroll
    for (int u = 0; u < KP; ++u) {
      const int c = lane + 32 * u;
      yn[u] = (c < m && c >= j) ? y[c] : czero();
    }
  };
  if (r > 0) load(0);
  const int u1 = (m + 31) / 32;
  for (int j = 0; j < r; ++j) {
    cplx yv[KP];
#pragma unroll
    for (int u = 0; u < KP; ++u) yv[u] = yn[u];
    const cplx tj = tau_g[j];
    if (j + 1 < r) load(j + 1);
    const int u0 = j / 32;  // warp-uniform live range of the reflector
    double sr = 0.0, si = 0.0;
#pragma unroll
    for (int u = 0; u < KP; ++u) {
      if (u >= u1) break;
      if (u < u0) continue;
      sr += d[u].x * yv[u].x - d[u].y * yv[u].y;
      si += d[u].x * yv[u].y + d[u].y * yv[u].x;
    }
    for (int o = 16; o > 0; o >>= 1) {
      sr += __shfl_xor_sync(0xffffffffu, sr, o);
      si += __shfl_xor_sync(0xffffffffu, si, o);
    }
    const cplx f = cmul(cconj(tj), cmk(sr, si));
#pragma unroll
    for (int u = 0; u < KP; ++u) {
      if (u >= u1) break;
      if (u < u0) continue;
      d[u] = csub(d[u], cmul(f, cconj(yv[u])));
    }
  }
#pragma unroll
  for (int u = 0; u < KP; ++u) {
    const int c = lane + 32 * u;
    if (c < m) D1[row + (size_t)c * b] = d[u];
  }
}

// --------------------------------------------------------------------------
// Step 0 part 2 (truncation of the projected fill spectrum, eps rule and
// floor of factorization.hpp:295-298 / h2_matrix.hpp:287-290), step 1
// (Qtilde = [complement | V | new], :317-339), the rotation of D(t,t) (:345-347)
// and step 3a (unpivoted LU of the leading e x e block, :390-398; self panels
// and the self Schur product, :409-420; cleanup, :431-435).
__global__ void __launch_bounds__(256) k_head(DevLevel L, const int* batch_cl, int p0, cplx* gws) {
  __shared__ cplx sm[kTileSmemCplx];
  __shared__ double red[32];
  __shared__ int s_r;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int q = blockIdx.x, p = p0 + q;
  const int t = batch_cl[q];
  const int b = L.bsz[t], k = L.korig[t], m = b - k, bm = L.bmax;
  const size_t bb = (size_t)bm * bm;
  cplx* ws = gws + (size_t)q * 4 * bb;
  cplx* Hc = ws;          // pass-2 Gram (m x m)
  cplx* Uc = ws + bb;     // pass-2 eigenvectors
  cplx* T = ws + 3 * bb;  // temporaries
  double* lam = reinterpret_cast<double*>(smraw);
  int* ord = reinterpret_cast<int*>(lam + bm);
  int* pr = ord + bm;
  double* rot = reinterpret_cast<double*>(pr + bm + 2);

  const cplx* D1 = L.dir + (size_t)q * bb;
  for (int i = threadIdx.x; i < m; i += blockDim.x) ord[i] = i;
  if (threadIdx.x == 0) s_r = L.rank1[q];
  __syncthreads();
  const bool p2 = L.pass2[q] != 0;
  if (p2) {
    // pass 2: Gram of D1^H W (near-diagonal, graded), Jacobi with the relative criterion
    const int g0 = L.slot_g0[p], gn = L.slot_gn[p];
    for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x) {
      cplx s = czero();
      for (int g = 0; g < gn; ++g) s = cadd(s, L.gram[L.gram_off[g0 + g] + idx]);
      Hc[idx] = s;
    }
    __syncthreads();
    // pass 2 must resolve values near the pass-1 threshold (sigma^2 ~ thr^2)
    const double thr1 = fmax(L.eps * L.lam[(size_t)q * bm], L.eps * L.cmax[q]);
    cta_jacobi_eig(m, Hc, Uc, rot, pr, red, 1e-8 * thr1 * thr1);
    for (int i = threadIdx.x; i < m; i += blockDim.x) lam[i] = sqrt(fmax(Hc[i + i * m].x, 0.0));
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      int rk = 0;
      for (int j = 0; j < m; ++j) rk += (lam[j] > lam[i]) || (lam[j] == lam[i] && j < i);
      ord[rk] = i;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const double s0 = lam[ord[0]];
      int r = 0;
      if (s0 > 0.0) {
        const double thr = fmax(fmax(L.eps * s0, L.eps * L.cmax[q]), 1e-300);
        while (r < m && lam[ord[r]] > thr) ++r;
      }
      s_r = r;
      if (L.debug & 1) printf("[h2g] pass2 level %d cluster %d m %d s0 %.3e r %d\n", L.level, t, m, s0, r);
    }
    __syncthreads();
    // directions D1 Uc (b x m) into T
    cta_gemm_tiled(b, m, m, 1.0, D1, b, OP_N, Uc, m, OP_N, 0.0, T, b, sm);
  }
  const int r = s_r;
  const int kf = k + r, e = b - kf;
  if (threadIdx.x == 0) L.kfin[t] = kf;
  const cplx* Dir = p2 ? T : D1;

  // Qtilde = [Dir(:, ord[r:]) | V | Dir(:, ord[:r])] (factorization.hpp:300-333)
  cplx* Qt = L.chain + L.Qt_off[t];
  const cplx* V = L.V0 + (size_t)t * bb;
  for (int idx = threadIdx.x; idx < b * b; idx += blockDim.x) {
    const int i = idx % b, j = idx / b;
    cplx v;
    if (j >= e && j < e + k)
      v = V[i + (size_t)(j - e) * b];
    else
      v = Dir[i + (size_t)(j < e ? ord[r + j] : ord[j - e - k]) * b];
    Qt[i + (size_t)j * b] = v;
  }
  __syncthreads();
}

// Step 3a after the diagonal block was rotated (descriptor GEMMs between
// k_head and this kernel): blocked unpivoted LU of the leading e x e block
// with the 1e-13 relative pivot test (dense_kernels.hpp:70-93,
// factorization.hpp:390-398), blocked triangular inverses, self panels and the
// self Schur product (:409-420), head set to identity (:431-435).
__global__ void __launch_bounds__(256) k_head2(DevLevel L, const int* batch_cl, cplx* gws) {
  __shared__ cplx sm[kTileSmemCplx];
  __shared__ double red[32];
  const int q = blockIdx.x;
  const int t = batch_cl[q];
  const int b = L.bsz[t], kf = L.kfin[t], e = b - kf, bm = L.bmax;
  const size_t bb = (size_t)bm * bm;
  const int cid = (1 << L.level) - 1 + t;
  cplx* ws = gws + (size_t)q * 2 * bb;
  cplx* LU = ws;        // e x e (ld e)
  cplx* W = ws + bb;    // e x 32 scratch
  cplx* Dd = L.D + L.D_off[L.diag_blk[t]];  // rotated diagonal block (ld b)
  if (e == 0) return;
  cta_copy(e, e, Dd, b, LU, e);
  __syncthreads();
  double pmag = 0.0;
  const int fail = cta_lu_blocked(e, LU, e, 1e-13, &pmag, red, sm);
  if (fail >= 0) {
    if (threadIdx.x == 0) raise_error(L.err, 4, cid, L.level, fail, pmag);
    return;
  }
  __syncthreads();
  cplx* L11 = L.chain + L.L11_off[t];
  cplx* U11 = L.chain + L.U11_off[t];
  for (int idx = threadIdx.x; idx < e * e; idx += blockDim.x) {
    const int i = idx % e, j = idx / e;
    const cplx v = LU[idx];
    L11[idx] = i > j ? v : (i == j ? cone() : czero());
    U11[idx] = i <= j ? v : czero();
  }
  cplx* Li = L.chain + L.Linv_off[t];
  cplx* Ui = L.chain + L.Uinv_off[t];
  cta_inv_unit_lower(e, LU, e, Li, e, sm);
  cta_inv_upper(e, LU, e, Ui, e, W, sm);
  if (kf > 0) {
    cplx* Us = L.chain + L.Uself_off[t];  // e x kf, ld e
    cplx* Ls = L.chain + L.Lself_off[t];  // kf x e, ld kf
    cta_gemm_tiled(e, kf, e, 1.0, Li, e, OP_N, Dd + (size_t)e * b, b, OP_N, 0.0, Us, e, sm);
    cta_gemm_tiled(kf, e, e, 1.0, Dd + e, b, OP_N, Ui, e, OP_N, 0.0, Ls, kf, sm);
    cta_gemm_tiled(kf, kf, e, -1.0, Ls, kf, OP_N, Us, e, OP_N, 1.0, Dd + e + (size_t)e * b, b, sm);
  }
  for (int idx = threadIdx.x; idx < b * b; idx += blockDim.x) {
    const int i = idx % b, j = idx / b;
    if (i < e || j < e) Dd[i + (size_t)j * b] = (i == j) ? cone() : czero();
  }
}

// --------------------------------------------------------------------------
// Step 3a for large heads (e > 64) as a multi-CTA blocked LU on the extended
// matrix M = [[D, I_e], [I_e, 0]] (D the rotated b x b diagonal block, I_e
// identities on the first e rows / columns). Eliminating only the first e
// pivots right-looking gives, in place (factorization.hpp:390-420):
//   M[:e, :e] = L11 \ U11 (1e-13 relative pivot test, dense_kernels.hpp:70-93)
//   M[e:b, :e] = D21 U11^{-1} (Lself),   M[:e, e:b] = L11^{-1} D12 (Uself)
//   M[e:b, e:b] = D22 - Lself Uself (self Schur),
//   M[:e, b:b+e] = L11^{-1},            M[b:b+e, :e] = U11^{-1},
// so the triangular inverses and self panels come out of the same trailing
// GEMM updates. Per 32-wide panel: k_hlu_panel (diagonal block + row/column
// triangular solves) and k_hlu_update (trailing GEMM over every CTA).
__global__ void __launch_bounds__(256) k_hlu_prep(DevLevel L, const int* batch_cl, cplx* M0, int ldm, double* scale, int* fail) {
  __shared__ double red[32];
  const int q = blockIdx.x;
  const int t = batch_cl[q];
  const int b = L.bsz[t], e = b - L.kfin[t];
  if (e == 0) return;
  const int N = b + e;
  cplx* M = M0 + (size_t)q * ldm * ldm;
  const cplx* Dd = L.D + L.D_off[L.diag_blk[t]];
  double mx = 0.0;
  for (int idx = blockIdx.y * blockDim.x + threadIdx.x; idx < N * N; idx += gridDim.y * blockDim.x) {
    const int i = idx % N, j = idx / N;
    cplx v;
    if (i < b && j < b) {
      v = Dd[i + (size_t)j * b];
      if (i < e && j < e) mx = fmax(mx, cabsd(v));
    } else if (i < b) {
      v = (i == j - b) ? cone() : czero();
    } else {
      v = (i - b == j) ? cone() : czero();
    }
    M[i + (size_t)j * ldm] = v;
  }
  mx = cta_max(mx, red);
  if (threadIdx.x == 0) {
    atomicMax(reinterpret_cast<unsigned long long*>(scale + q), __double_as_longlong(mx));
    if (blockIdx.y == 0) fail[q] = 0;
  }
}

__global__ void __launch_bounds__(256) k_hlu_panel(DevLevel L, const int* batch_cl, cplx* M0, int ldm, const double* scale, int* fail, int j0,
                                                   cplx* Dg) {
  // grid (nb, NY): every CTA factors the 32 x 32 diagonal block itself
  // (identical results) and takes a share of the row / column triangular
  // solves; the factored block goes to Dg (k_hlu_update stores it into M, so
  // no CTA here can see it half-written)
  __shared__ cplx P[32][33];
  __shared__ cplx rinv[32];
  const int q = blockIdx.x;
  const int t = batch_cl[q];
  const int b = L.bsz[t], e = b - L.kfin[t];
  if (j0 >= e || fail[q]) return;
  const int kb = min(32, e - j0), N = b + e;
  cplx* M = M0 + (size_t)q * ldm * ldm;
  const double tol = 1e-13 * scale[q];
  for (int idx = threadIdx.x; idx < kb * kb; idx += blockDim.x) {
    const int i = idx % kb, j = idx / kb;
    P[i][j] = M[(j0 + i) + (size_t)(j0 + j) * ldm];
  }
  __syncthreads();
  for (int k = 0; k < kb; ++k) {
    const cplx piv = P[k][k];
    const double pa = cabsd(piv);
    if (pa < tol || (scale[q] == 0.0)) {
      if (threadIdx.x == 0 && blockIdx.y == 0) {
        raise_error(L.err, 4, (1 << L.level) - 1 + t, L.level, j0 + k, pa);
        fail[q] = 1;
      }
      return;  // uniform
    }
    const cplx rp = cdiv(cone(), piv);
    if (threadIdx.x == 0) rinv[k] = rp;
    for (int i = k + 1 + threadIdx.x; i < kb; i += blockDim.x) P[i][k] = cmul(P[i][k], rp);
    __syncthreads();
    for (int idx = threadIdx.x; idx < (kb - k - 1) * (kb - k - 1); idx += blockDim.x) {
      const int i = k + 1 + idx % (kb - k - 1), j = k + 1 + idx / (kb - k - 1);
      P[i][j] = csub(P[i][j], cmul(P[i][k], P[k][j]));
    }
    __syncthreads();
  }
  if (blockIdx.y == 0)
    for (int idx = threadIdx.x; idx < kb * kb; idx += blockDim.x) {
      const int i = idx % kb, j = idx / kb;
      Dg[(size_t)q * 1024 + i + 32 * j] = P[i][j];
    }
  // rows below the panel: x U = a (L21); columns right of it: L y = c (U12)
  const int rest = N - j0 - kb;
  for (int it = blockIdx.y * blockDim.x + threadIdx.x; it < 2 * rest; it += gridDim.y * blockDim.x) {
    cplx x[32];
    if (it < rest) {
      cplx* row = M + (j0 + kb + it) + (size_t)j0 * ldm;
#pragma unroll
      for (int k = 0; k < 32; ++k)
        if (k < kb) x[k] = row[(size_t)k * ldm];
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        if (k >= kb) break;
        cplx a0 = x[k], a1 = czero();
        int l = 0;
        for (; l + 1 < k; l += 2) {
          a0 = csub(a0, cmul(x[l], P[l][k]));
          a1 = csub(a1, cmul(x[l + 1], P[l + 1][k]));
        }
        if (l < k) a0 = csub(a0, cmul(x[l], P[l][k]));
        x[k] = cmul(cadd(a0, a1), rinv[k]);
        row[(size_t)k * ldm] = x[k];
      }
    } else {
      cplx* col = M + j0 + (size_t)(j0 + kb + it - rest) * ldm;
#pragma unroll
      for (int k = 0; k < 32; ++k)
        if (k < kb) x[k] = col[k];
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        if (k >= kb) break;
        cplx a0 = x[k], a1 = czero();
        int l = 0;
        for (; l + 1 < k; l += 2) {
          a0 = csub(a0, cmul(P[k][l], x[l]));
          a1 = csub(a1, cmul(P[k][l + 1], x[l + 1]));
        }
        if (l < k) a0 = csub(a0, cmul(P[k][l], x[l]));
        x[k] = cadd(a0, a1);
        col[k] = x[k];
      }
    }
  }
}

__global__ void __launch_bounds__(128, 3) k_hlu_update(DevLevel L, const int* batch_cl, cplx* M0, int ldm, const int* fail, int j0, const cplx* Dg) {
  extern __shared__ __align__(16) unsigned char tsm[];
  Tile128Smem& S = *reinterpret_cast<Tile128Smem*>(tsm);
  const int q = blockIdx.x;
  const int t = batch_cl[q];
  const int b = L.bsz[t], e = b - L.kfin[t];
  if (j0 >= e || fail[q]) return;
  const int kb = min(32, e - j0), N = b + e, c = j0 + kb, rest = N - c;
  const int nt = (rest + 63) / 64;
  cplx* M = M0 + (size_t)q * ldm * ldm;
  if (blockIdx.y == 0)  // the panel's factored diagonal block (read by nobody in this launch)
    for (int idx = threadIdx.x; idx < kb * kb; idx += blockDim.x) {
      const int i = idx % kb, j = idx / kb;
      M[(j0 + i) + (size_t)(j0 + j) * ldm] = Dg[(size_t)q * 1024 + i + 32 * j];
    }
  for (int tile = blockIdx.y; tile < nt * nt; tile += gridDim.y) {
    const int r0 = (tile % nt) * 64, c0 = (tile / nt) * 64;
    Acc64 acc;
    acc64_zero(acc);
    tile_acc_dmma(acc, S, M + c + (size_t)j0 * ldm, ldm, OP_N, r0, rest, M + j0 + (size_t)c * ldm, ldm, OP_N, c0, rest, kb);
    acc64_each(acc, [&](int ii, int jj, cplx v) {
      const int i = r0 + ii, j = c0 + jj;
      if (i < rest && j < rest) {
        cplx* o = M + (c + i) + (size_t)(c + j) * ldm;
        *o = csub(*o, v);
      }
    });
  }
}

__global__ void __launch_bounds__(256) k_hlu_finish(DevLevel L, const int* batch_cl, const cplx* M0, int ldm, const int* fail) {
  const int q = blockIdx.x;
  const int t = batch_cl[q];
  const int b = L.bsz[t], kf = L.kfin[t], e = b - kf;
  if (e == 0 || fail[q]) return;
  const cplx* M = M0 + (size_t)q * ldm * ldm;
  cplx* L11 = L.chain + L.L11_off[t];
  cplx* U11 = L.chain + L.U11_off[t];
  cplx* Li = L.chain + L.Linv_off[t];
  cplx* Ui = L.chain + L.Uinv_off[t];
  cplx* Us = L.chain + L.Uself_off[t];  // e x kf, ld e
  cplx* Ls = L.chain + L.Lself_off[t];  // kf x e, ld kf
  cplx* Dd = L.D + L.D_off[L.diag_blk[t]];
  const int stride = gridDim.y * blockDim.x;
  for (int idx = blockIdx.y * blockDim.x + threadIdx.x; idx < e * e; idx += stride) {
    const int i = idx % e, j = idx / e;
    const cplx v = M[i + (size_t)j * ldm];
    L11[idx] = i > j ? v : (i == j ? cone() : czero());
    U11[idx] = i <= j ? v : czero();
    Li[idx] = i >= j ? M[i + (size_t)(b + j) * ldm] : czero();
    Ui[idx] = i <= j ? M[(b + i) + (size_t)j * ldm] : czero();
  }
  for (int idx = blockIdx.y * blockDim.x + threadIdx.x; idx < e * kf; idx += stride) {
    const int i = idx % e, j = idx / e;
    Us[idx] = M[i + (size_t)(e + j) * ldm];
  }
  for (int idx = blockIdx.y * blockDim.x + threadIdx.x; idx < kf * e; idx += stride) {
    const int i = idx % kf, j = idx / kf;
    Ls[idx] = M[(e + i) + (size_t)j * ldm];
  }
  for (int idx = blockIdx.y * blockDim.x + threadIdx.x; idx < b * b; idx += stride) {
    const int i = idx % b, j = idx / b;
    Dd[i + (size_t)j * b] = (i < e || j < e) ? ((i == j) ? cone() : czero()) : M[i + (size_t)j * ldm];
  }
}

// --------------------------------------------------------------------------
// Step 3c: one CTA per target block (dense or fill-in); the contributions of
// every cluster of the batch that hits it are summed in a fixed order, then
// subtracted once (:414-425, deposit_fill :363-365). 64 x 64 output tiles,
// 4 x 4 complex micro-tile per thread, K staged through shared memory.
// PF (TM = 64, levels whose eliminated sizes are small): the launch is bound
// by the read-modify-write of the targets, not by the products, so the target
// tile is fetched into shared memory by cp.async at the start (64 KB in flight
// per CTA while the contribution tables and panels load) and the epilogue
// subtracts from the staged copy; two CTAs per SM instead of three.
// Target and panel descriptors of one batch, resolved once (one thread per
// target) instead of by every tile's CTA.
__global__ void __launch_bounds__(128) k_schur_resolve(DevLevel L, const SchurTargetD* targets, int ntargets, const SchurContribD* contrib,
                                                       RTarget* rt, RPanel* rp) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ntargets) return;
  const SchurTargetD tg = targets[i];
  RTarget R{};
  R.rs = R.cs = 0;
  R.ldo = -1;
  if ((tg.kind & 1) == 0) {
    const int j = L.drow[tg.idx], c = L.dcol[tg.idx];
    R.rows = L.bsz[j];
    R.cols = L.bsz[c];
    R.out = L.D + L.D_off[tg.idx];
    if (tg.kind & 2) R.rs = R.rows - L.kfin[j];
    if (tg.kind & 4) R.cs = R.cols - L.kfin[c];
  } else {
    const int j = L.frow[tg.idx], c = L.fcol[tg.idx];
    R.rows = L.bsz[j];
    R.cols = L.bsz[c];
    if (tg.kind & 8) {
      R.rs = R.rows - L.kfin[j];
      R.cs = R.cols - L.kfin[c];
      R.ldo = L.kfin[j];
      R.out = L.core_ptr[tg.idx] - R.rs - (size_t)R.cs * R.ldo;
    } else {
      R.out = L.F + L.F_off[tg.idx];
    }
  }
  if (R.ldo < 0) R.ldo = R.rows;
  rt[i] = R;
  for (int ci = tg.c0; ci < tg.c1; ++ci) {
    const SchurContribD cb = contrib[ci];
    const int t = cb.t;
    const int kf = L.kfin[t], e = L.bsz[t] - kf;
    RPanel P{};
    P.e = e;
    if (e > 0) {
      if (cb.r >= 0) {
        P.arows = L.bsz[L.R_nb[cb.r]];
        P.A = (cb.flags & 1) ? L.lift + L.liftL_off[cb.r] : L.chain + L.Lbar_off[cb.r];
        P.ro = 0;
      } else {
        P.arows = kf;
        P.A = L.chain + L.Lself_off[t];
        P.ro = e;
      }
      if (cb.c >= 0) {
        P.bcols = L.bsz[L.C_nb[cb.c]];
        P.B = (cb.flags & 2) ? L.lift + L.liftU_off[cb.c] : L.chain + L.Ubar_off[cb.c];
        P.co = 0;
      } else {
        P.bcols = kf;
        P.B = L.chain + L.Uself_off[t];
        P.co = e;
      }
    }
    rp[ci] = P;
  }
}

template <int TM, bool PF = false, int NSTAGE = 3>
__global__ void __launch_bounds__(128, PF ? 2 : 3) k_schur(DevLevel L, const SchurTargetD* targets, const SchurContribD* contrib,
                                                         const RTarget* rt, const RPanel* rp) {
  constexpr int RM = TM / 8, RN = TM / 16;  // DFMA micro-tile (TM < 64)
  extern __shared__ __align__(16) unsigned char tsm[];
  using Smem = TileSmem<TM, PF ? 2 : NSTAGE>;
  Smem& S = *reinterpret_cast<Smem*>(tsm);
  cplx(*Tt)[TM] = reinterpret_cast<cplx(*)[TM]>(tsm + sizeof(Smem));  // PF: target tile, [column][row]
  const SchurTargetD tg = targets[blockIdx.x];
  int rows, cols, rs = 0, cs = 0, ldo = -1;
  cplx* out;
  if (rt) {
    const RTarget R = rt[blockIdx.x];
    rows = R.rows, cols = R.cols, rs = R.rs, cs = R.cs, ldo = R.ldo, out = R.out;
  } else if ((tg.kind & 1) == 0) {
    const int j = L.drow[tg.idx], c = L.dcol[tg.idx];
    rows = L.bsz[j];
    cols = L.bsz[c];
    out = L.D + L.D_off[tg.idx];
    // rows / columns eliminated by an earlier batch receive exact zeros
    if (tg.kind & 2) rs = rows - L.kfin[j];
    if (tg.kind & 4) cs = cols - L.kfin[c];
  } else {
    const int j = L.frow[tg.idx], c = L.fcol[tg.idx];
    rows = L.bsz[j];
    cols = L.bsz[c];
    if (tg.kind & 8) {
      // compact core of a collapsed block: target rows / columns [e, b) of
      // the (rotated) panels land at [0, kfin) of the kfin_j x kfin_c core
      rs = rows - L.kfin[j];
      cs = cols - L.kfin[c];
      ldo = L.kfin[j];
      out = L.core_ptr[tg.idx] - rs - (size_t)cs * ldo;
    } else {
      out = L.F + L.F_off[tg.idx];
    }
  }
  if (ldo < 0) ldo = rows;
  const int ntr = (rows - rs + TM - 1) / TM, ntc = (cols - cs + TM - 1) / TM;
  if ((int)blockIdx.y >= ntr * ntc) return;
  const int r0 = rs + (blockIdx.y % ntr) * TM, c0 = cs + (blockIdx.y / ntr) * TM;
  if constexpr (PF) {
    for (int idx = threadIdx.x; idx < TM * TM; idx += 128) {
      const int i = idx % TM, j = idx / TM;
      const bool v = r0 + i < rows && c0 + j < cols;
      cp_async16(&Tt[j][i], v ? out + (r0 + i) + (size_t)(c0 + j) * ldo : out, v);
    }
    cp_async_commit();
  }
  Acc64 acc;
  cplx accs[TM == 64 ? 1 : RM][TM == 64 ? 1 : RN];
  if constexpr (TM == 64) {
    acc64_zero(acc);
  } else {
#pragma unroll
    for (int a = 0; a < RM; ++a)
#pragma unroll
      for (int b = 0; b < RN; ++b) accs[a][b] = czero();
  }
  bool touched = false;
  // one contribution resolved against this tile; returns its e (0: the
  // cluster eliminated nothing), use = false when it misses the tile
  auto resolve = [&](int ci, SchurPanel& P, bool& use) {
    if (rp) {
      const RPanel Q = rp[ci];
      use = false;
      if (Q.e == 0) return 0;
      P.A = Q.A, P.B = Q.B, P.arows = Q.arows, P.bcols = Q.bcols, P.e = Q.e;
      P.ash = r0 - Q.ro;
      P.bsh = c0 - Q.co;
      use = !(P.ash >= P.arows || P.bsh >= P.bcols || P.ash + TM <= 0 || P.bsh + TM <= 0);
      return Q.e;
    }
    const SchurContribD cb = contrib[ci];
    const int t = cb.t;
    const int kf = L.kfin[t], e = L.bsz[t] - kf;
    use = false;
    if (e == 0) return 0;
    int ro, co;
    if (cb.r >= 0) {
      P.arows = L.bsz[L.R_nb[cb.r]];
      P.A = (cb.flags & 1) ? L.lift + L.liftL_off[cb.r] : L.chain + L.Lbar_off[cb.r];
      ro = 0;
    } else {
      P.arows = kf;
      P.A = L.chain + L.Lself_off[t];
      ro = e;
    }
    if (cb.c >= 0) {
      P.bcols = L.bsz[L.C_nb[cb.c]];
      P.B = (cb.flags & 2) ? L.lift + L.liftU_off[cb.c] : L.chain + L.Ubar_off[cb.c];
      co = 0;
    } else {
      P.bcols = kf;
      P.B = L.chain + L.Uself_off[t];
      co = e;
    }
    // the contribution covers target rows [ro, ro+arows) x cols [co, co+bcols)
    P.ash = r0 - ro;
    P.bsh = c0 - co;
    P.e = e;
    use = !(P.ash >= P.arows || P.bsh >= P.bcols || P.ash + TM <= 0 || P.bsh + TM <= 0);
    return e;
  };
  if constexpr (TM == 64) {
    // all contributions of the target through one load pipeline (tables of
    // 16 panels resolved by 16 threads in parallel)
    __shared__ SchurPanel tab[16];
    __shared__ int s_kv[4], s_touched;
    if (threadIdx.x == 0) s_touched = 0;
    for (int cbase = tg.c0; cbase < tg.c1; cbase += 16) {
      const int nc = min(16, tg.c1 - cbase);
      __syncthreads();
      if ((int)threadIdx.x < nc) {
        SchurPanel P;
        bool use;
        const int e = resolve(cbase + threadIdx.x, P, use);
        if (e > 0) s_touched = 1;
        if (!use) P.A = nullptr, P.B = nullptr, P.arows = P.bcols = P.ash = P.bsh = 0, P.e = 0;
        P.pad = 0;
        tab[threadIdx.x] = P;
      }
      __syncthreads();
      schur_pipe_dmma(acc, S, tab, nc, s_kv, rows - r0, cols - c0);
    }
    __syncthreads();
    touched = s_touched != 0;
  } else {
    for (int ci = tg.c0; ci < tg.c1; ++ci) {
      SchurPanel P;
      bool use;
      if (resolve(ci, P, use) == 0) continue;
      touched = true;
      if (!use) continue;
      tile_acc<TM>(accs, S, P.A, P.arows, OP_N, P.ash, P.arows, P.B, P.e, OP_N, P.bsh, P.bcols, P.e);
    }
  }
  if constexpr (PF) {
    asm volatile("cp.async.wait_group 0;");
    __syncthreads();
  }
  // Epilogue: target -= acc. The target values of a row group are loaded
  // together before any store (the stores may alias later loads, so loads
  // interleaved with stores would serialise into one round trip each).
  if constexpr (TM == 64) {
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int wr = (warp % 2) * 32, wc = (warp / 2) * 32, g = lane / 4, tq = lane % 4;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int n0 = 0; n0 < 4; n0 += 2) {  // groups of 4 targets: bounded registers
        cplx old[2][2];
        bool ok[2][2];
        const int i = r0 + wr + mi * 8 + g;
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int ni = n0 + u, j = c0 + wc + ni * 8 + tq * 2 + h;
            ok[u][h] = i < rows && j < cols && (acc.re[mi][ni][h] != 0.0 || acc.im[mi][ni][h] != 0.0);
            if (ok[u][h]) old[u][h] = PF ? Tt[j - c0][i - r0] : out[i + (size_t)j * ldo];
          }
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (ok[u][h]) {
              const int ni = n0 + u, j = c0 + wc + ni * 8 + tq * 2 + h;
              out[i + (size_t)j * ldo] = make_double2(old[u][h].x - acc.re[mi][ni][h], old[u][h].y - acc.im[mi][ni][h]);
            }
      }
  } else {
    const int tr = threadIdx.x % 8, tc = threadIdx.x / 8;
    cplx old[RM][RN];
    bool ok[RM][RN];
#pragma unroll
    for (int a = 0; a < RM; ++a)
#pragma unroll
      for (int b = 0; b < RN; ++b) {
        const int i = r0 + tr + 8 * a, j = c0 + tc * RN + b;
        ok[a][b] = i < rows && j < cols && (accs[a][b].x != 0.0 || accs[a][b].y != 0.0);
        if (ok[a][b]) old[a][b] = out[i + (size_t)j * ldo];
      }
#pragma unroll
    for (int a = 0; a < RM; ++a)
#pragma unroll
      for (int b = 0; b < RN; ++b)
        if (ok[a][b]) {
          const int i = r0 + tr + 8 * a, j = c0 + tc * RN + b;
          out[i + (size_t)j * ldo] = csub(old[a][b], accs[a][b]);
        }
  }
  if ((tg.kind & 1) == 1 && touched && threadIdx.x == 0 && blockIdx.y == 0) L.fexists[tg.idx] = 1;
}

// --------------------------------------------------------------------------
// Descriptor-driven copy / GEMM (level boundaries: finish_level, merge_permute,
// root assembly, :445-584 and :637).
__global__ void __launch_bounds__(256) k_mask(const MaskDesc* descs) {
  const MaskDesc d = descs[blockIdx.x];
  const int e = d.e0 - *d.kf;
  for (int idx = blockIdx.y * blockDim.x + threadIdx.x; idx < d.m * d.n; idx += gridDim.y * blockDim.x) {
    const int i = idx % d.m, j = idx / d.m;
    const bool z = d.mode == 0 ? i < e : j < e;
    d.dst[i + (size_t)j * d.ld] = z ? czero() : d.src[i + (size_t)j * d.ld];
  }
}

// Largest column norm of a fill-in block as it enters W (F's columns, or
// F's rows for a transposed key): the floor of factorization.hpp:295.
__global__ void __launch_bounds__(256) k_colnorm(const NormDesc* descs) {
  __shared__ double red[32];
  const NormDesc d = descs[blockIdx.x];
  double mx = 0.0;
  if (!d.flag || *d.flag) {
    const int ncol = d.trans ? d.rows : d.cols, len = d.trans ? d.cols : d.rows;
    for (int j = threadIdx.x; j < ncol; j += blockDim.x) {
      double s = 0.0;
      for (int p = 0; p < len; ++p) s += cabs2(d.trans ? d.F[j + (size_t)p * d.rows] : d.F[p + (size_t)j * d.rows]);
      mx = fmax(mx, sqrt(s));
    }
  }
  mx = cta_max(mx, red);
  if (threadIdx.x == 0) *d.out = mx;
}

__global__ void __launch_bounds__(256) k_copy(const CopyDesc* descs) {
  const CopyDesc d = descs[blockIdx.x];
  for (int idx = threadIdx.x; idx < d.m * d.n; idx += blockDim.x) {
    const int i = idx % d.m, j = idx / d.m;
    const cplx v = d.src ? d.src[i + (size_t)j * d.lds] : czero();
    cplx* o = d.dst + i + (size_t)j * d.ldd;
    *o = d.accumulate ? cadd(*o, v) : v;
  }
}

template <int TM>
__global__ void __launch_bounds__(128, 3) k_gemm(const GemmDesc* descs) {
  constexpr int RM = TM / 8, RN = TM / 16;
  extern __shared__ __align__(16) unsigned char tsm[];
  TileSmem<TM>& S = *reinterpret_cast<TileSmem<TM>*>(tsm);
  GemmDesc d = descs[blockIdx.x];
  if (d.skipnz && *d.skipnz) return;
  if (d.dyn) {
    const int v = *d.dyn;
    d.m += d.mi * v, d.n += d.ni * v, d.k += d.ki * v;
    if (d.ldneg & 1) d.lda -= v;
    if (d.ldneg & 2) d.ldb -= v;
    if (d.ldneg & 4) d.ldc -= v;
  }
  const int ntr = (d.m + TM - 1) / TM, ntc = (d.n + TM - 1) / TM;
  const bool zero = (d.flag1 && !*d.flag1) || (d.flag2 && !*d.flag2);
  const int tr = threadIdx.x % 8, tc = threadIdx.x / 8;
  // each CTA walks the tiles blockIdx.y, blockIdx.y + gridDim.y, ...
  for (int tile = blockIdx.y; tile < ntr * ntc; tile += gridDim.y) {
    const int r0 = (tile % ntr) * TM, c0 = (tile / ntr) * TM;
    if constexpr (TM == 64) {
      Acc64 acc;
      acc64_zero(acc);
      if (!zero) tile_acc_dmma(acc, S, d.A, d.lda, d.opA, r0, d.m, d.B, d.ldb, d.opB, c0, d.n, d.k);
      acc64_each(acc, [&](int ii, int jj, cplx v) {
        const int i = r0 + ii, j = c0 + jj;
        if (i < d.m && j < d.n) {
          cplx* o = d.C + i + (size_t)j * d.ldc;
          *o = d.beta == 0.0 ? cscale(v, d.alpha) : make_double2(d.beta * o->x + d.alpha * v.x, d.beta * o->y + d.alpha * v.y);
        }
      });
      continue;
    }
    cplx acc[RM][RN];
#pragma unroll
    for (int a = 0; a < RM; ++a)
#pragma unroll
      for (int b = 0; b < RN; ++b) acc[a][b] = czero();
    if (!zero) tile_acc<TM>(acc, S, d.A, d.lda, d.opA, r0, d.m, d.B, d.ldb, d.opB, c0, d.n, d.k);
#pragma unroll
    for (int a = 0; a < RM; ++a)
#pragma unroll
      for (int b = 0; b < RN; ++b) {
        const int i = r0 + tr + 8 * a, j = c0 + tc * RN + b;
        if (i < d.m && j < d.n) {
          cplx* o = d.C + i + (size_t)j * d.ldc;
          const cplx v = acc[a][b];
          *o = d.beta == 0.0 ? cscale(v, d.alpha) : make_double2(d.beta * o->x + d.alpha * v.x, d.beta * o->y + d.alpha * v.y);
        }
      }
  }
}

// --------------------------------------------------------------------------
// Root: blocked right-looking unpivoted LU with the reference pivot rule
// (|piv| < 1e-13 max|A|, dense_kernels.hpp:74-79; factorization.hpp:637-651).
__global__ void k_absmax(const cplx* A, long long n2, double* out) {
  __shared__ double red[32];
  double m = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x) m = fmax(m, cabsd(A[i]));
  m = cta_max(m, red);
  if (threadIdx.x == 0) {
    unsigned long long* p = reinterpret_cast<unsigned long long*>(out);
    atomicMax(p, __double_as_longlong(m));  // non-negative doubles order like their bits
  }
}

__global__ void __launch_bounds__(256) k_lu_panel(cplx* A, int n, int k0, int kb, const double* scale, DevError* err) {
  // factor the tall panel A[k0:n, k0:k0+kb]
  const double sc = *scale;
  for (int kk = 0; kk < kb; ++kk) {
    const int k = k0 + kk;
    const cplx piv = A[k + (size_t)k * n];
    const double pa = cabsd(piv);
    if (pa < 1e-13 * sc || (sc == 0.0)) {
      if (threadIdx.x == 0) raise_error(err, 4, -1, -1, k, pa);
      return;
    }
    for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) A[i + (size_t)k * n] = cdiv(A[i + (size_t)k * n], piv);
    __syncthreads();
    const int nc = k0 + kb - k - 1;
    for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) {
      const cplx l = A[i + (size_t)k * n];
      for (int j = k + 1; j < k + 1 + nc; ++j) {
        const cplx u = A[k + (size_t)j * n];
        cplx a = A[i + (size_t)j * n];
        a.x -= l.x * u.x - l.y * u.y;
        a.y -= l.x * u.y + l.y * u.x;
        A[i + (size_t)j * n] = a;
      }
    }
    __syncthreads();
  }
}

__global__ void k_lu_trsm(cplx* A, int n, int k0, int kb) {
  // A[k0:k0+kb, j] <- L11^{-1} A[k0:k0+kb, j] for j >= k0+kb (unit lower)
  const int j = k0 + kb + blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  for (int i = 1; i < kb; ++i) {
    cplx s = A[k0 + i + (size_t)j * n];
    for (int p = 0; p < i; ++p) {
      const cplx l = A[k0 + i + (size_t)(k0 + p) * n], x = A[k0 + p + (size_t)j * n];
      s.x -= l.x * x.x - l.y * x.y;
      s.y -= l.x * x.y + l.y * x.x;
    }
    A[k0 + i + (size_t)j * n] = s;
  }
}

__global__ void __launch_bounds__(256) k_lu_update(cplx* A, int n, int k0, int kb) {
  extern __shared__ __align__(16) unsigned char smraw[];
  cplx(*sA)[33] = reinterpret_cast<cplx(*)[33]>(smraw);
  cplx(*sB)[65] = reinterpret_cast<cplx(*)[65]>(smraw + 64 * 33 * sizeof(cplx));
  const int base = k0 + kb;
  const int r0 = base + blockIdx.x * 64, c0 = base + blockIdx.y * 64;
  if (r0 >= n || c0 >= n) return;
  const int tr = threadIdx.x % 16, tc = threadIdx.x / 16;
  for (int idx = threadIdx.x; idx < 64 * 32; idx += blockDim.x) {
    const int i = idx % 64, p = idx / 64;
    sA[i][p] = (p < kb && r0 + i < n) ? A[r0 + i + (size_t)(k0 + p) * n] : czero();
    sB[p][i] = (p < kb && c0 + i < n) ? A[k0 + p + (size_t)(c0 + i) * n] : czero();
  }
  __syncthreads();
  cplx acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int bb = 0; bb < 4; ++bb) acc[a][bb] = czero();
  for (int p = 0; p < kb; ++p) {
    cplx av[4], bv[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) av[a] = sA[tr * 4 + a][p];
#pragma unroll
    for (int bb = 0; bb < 4; ++bb) bv[bb] = sB[p][tc * 4 + bb];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int bb = 0; bb < 4; ++bb) cfma(acc[a][bb], av[a], bv[bb]);
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int bb = 0; bb < 4; ++bb) {
      const int i = r0 + tr * 4 + a, j = c0 + tc * 4 + bb;
      if (i < n && j < n) {
        cplx* o = A + i + (size_t)j * n;
        *o = csub(*o, acc[a][bb]);
      }
    }
}

// ==========================================================================
// launchers
namespace {
size_t smem3(int bm) { return 3 * (size_t)bm * bm * sizeof(cplx); }
constexpr size_t kSmemCap = 220 * 1024;
}  // namespace

size_t head_smem_bytes(int bm) {
  // 3 matrices + lam/ord/pr/rot scratch
  return smem3(bm) + (size_t)bm * 8 + (size_t)bm * 4 + (size_t)(bm + 2) * 4 + 16 + (size_t)4 * (bm / 2 + 1) * 8 + 64;
}

static int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

// Opt in to the dynamic shared memory a launch needs (cached per device and
// kernel: the attribute is per device, a second GPU in the process needs its own).
static void set_smem(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  std::lock_guard<std::mutex> g(mu);
  size_t& cur = done[{current_device(), fn}];
  if (bytes > cur) {
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
      throw std::runtime_error("cudaFuncSetAttribute(MaxDynamicSharedMemorySize) failed");
    cur = bytes;
  }
}

// Non-portable cluster sizes (> 8 CTAs), opted in once per device and kernel.
static void allow_big_clusters(const void* fn) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  std::lock_guard<std::mutex> g(mu);
  if (done.insert({current_device(), fn}).second)
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
      throw std::runtime_error("cudaFuncSetAttribute(NonPortableClusterSizeAllowed) failed");
}

static int sync_debug() {
  static int v = std::getenv("H2G_SYNC") ? std::atoi(std::getenv("H2G_SYNC")) : 0;
  return v;
}

static void post_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && sync_debug()) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) throw std::runtime_error(std::string("launch of ") + what + " failed: " + cudaGetErrorString(e));
}

// Level scratch (complement / head / extended-LU workspaces). It is owned by
// the caller's level state (one allocation per context and level, stream
// ordered), never a process-wide buffer.
static size_t complement_bytes(int bm) { return 2 * (size_t)bm * bm * sizeof(cplx) + (size_t)bm * sizeof(cplx); }
static size_t hlu_ws_bytes(int bm, int nb) {
  const size_t ldm = 2 * (size_t)bm;
  return ldm * ldm * sizeof(cplx) * nb + (size_t)nb * 1024 * sizeof(cplx) + (size_t)nb * 16 + 64;
}

size_t level_scratch_bytes(int nl, int bm, int max_batch) {
  size_t need = 4 * (size_t)bm * bm * sizeof(cplx) * max_batch;  // k_head
  need = std::max(need, 2 * (size_t)bm * bm * sizeof(cplx) * max_batch);  // k_head2
  if (bm > 64) need = std::max(need, hlu_ws_bytes(bm, max_batch));  // k_hlu_* (e > 64 needs b > 64)
  if (complement_bytes(bm) > kSmemCap) need = std::max(need, complement_bytes(bm) * nl);
  return need;
}

static cplx* workspace(const DevLevel& L, size_t bytes) {
  if (!L.scratch || bytes > L.scratch_bytes)
    throw std::runtime_error("level scratch too small: " + std::to_string(bytes) + " bytes needed, " + std::to_string(L.scratch_bytes) + " allocated");
  return L.scratch;
}

void launch_complement(const DevLevel& L, cudaStream_t s) {
  const size_t need = complement_bytes(L.bmax);
  if (need <= kSmemCap) {
    set_smem((const void*)k_complement, need);
    k_complement<<<L.nl, 256, need, s>>>(L, nullptr); post_launch("k_complement");
  } else {
    cplx* ws = workspace(L, need * L.nl);
    k_complement<<<L.nl, 256, 0, s>>>(L, ws);
    post_launch("k_complement");
  }
}

size_t eig1_small_bytes(int bm) { return (size_t)(bm + 1) * 8 * 3 + (size_t)bm * 16 * 3 + (size_t)bm * 4 + (size_t)(bm + 2) * 4 + 16 + (size_t)4 * (bm / 2 + 1) * 8 + 64; }
size_t eig1_smem_bytes(int bm) { return eig1_ws_cplx(bm) * sizeof(cplx) + eig1_small_bytes(bm); }

size_t eig1_ws_bytes(int bmax) { return eig1_ws_cplx(bmax) * sizeof(cplx); }

void launch_eig1(const DevLevel& L, const int* batch_cl, int p0, int nb, int mmax, cudaStream_t s,
                 const std::function<void(int)>& phase) {
  cplx* ws = L.eigws;
  {
    // cluster size: small blocks fit one CTA's shared memory, large ones are
    // spread over 4 or 16 CTAs
    const int kHC = L.bmax <= 64 ? 1 : (L.bmax <= 128 ? 4 : (L.bmax <= 240 ? 8 : kHCmax));
    const int ncl = (L.bmax + kHC - 1) / kHC;
    size_t smem = (size_t)L.bmax * ncl * sizeof(cplx) + (size_t)L.bmax * sizeof(cplx) * 8 + 256;
    cplx* gH = nullptr;
    const char* force_g = std::getenv("H2G_EIG_GLOBAL");  // tests: take the large-block path on small inputs
    if (smem > kSmemCap || (force_g && std::atoi(force_g) && kHC > 1)) {
      // too large for the cluster's shared memory: Gram columns in global memory (level scratch, free until k_head)
      gH = workspace(L, (size_t)nb * ((size_t)L.bmax * L.bmax + 16 * (size_t)L.bmax) * sizeof(cplx));
      smem = (size_t)L.bmax * sizeof(cplx) * 8 + 256;
    }
    set_smem((const void*)k_eig1c, smem);
    allow_big_clusters((const void*)k_eig1c);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nb * kHC);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kHC;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, k_eig1c, L, batch_cl, p0, ws, gH);
    if (e != cudaSuccess) throw std::runtime_error(std::string("launch of k_eig1c failed: ") + cudaGetErrorString(e));
    post_launch("k_eig1c");
  }
  {
    const size_t small = (size_t)L.bmax * 8 + (size_t)L.bmax * 4 + (size_t)(L.bmax + 2) * 4 + 16 + (size_t)4 * (L.bmax / 2 + 1) * 8 + 64;
    // the refinement pass can only trigger when thr = eps max(s0, cmax) can
    // fall below 1e-4 s0, i.e. for eps < 1e-4 (k_eig1c)
    if (eig1_refine_possible(L)) {
      set_smem((const void*)k_eig1_refine, small);
      k_eig1_refine<<<nb, 256, small, s>>>(L, batch_cl, p0, ws);
      post_launch("k_eig1_refine");
    }
  }
  phase(1);
  if (mmax > 0) {
    if (mmax > 1024) throw std::runtime_error("k_eigvec: complement dimension > 1024");
    // one warp per eigenvector; shared: d, e (2 bmax) + 7 bmax doubles per warp
    // + the staged reflector chunk (8 x bmax complex)
    int wpc = 8;
    auto need = [&](int w) { return (size_t)(2 + 7 * w) * L.bmax * sizeof(double) + 8 * (size_t)L.bmax * sizeof(cplx) + 64; };
    while (wpc > 1 && need(wpc) > kSmemCap) --wpc;
    const size_t vsm = need(wpc);
    if (mmax <= 512) {
      set_smem((const void*)k_eigvec<16>, vsm);
      k_eigvec<16><<<dim3(nb, (mmax + wpc - 1) / wpc), 256, vsm, s>>>(L, batch_cl, ws, wpc);
    } else {
      set_smem((const void*)k_eigvec<32>, vsm);
      k_eigvec<32><<<dim3(nb, (mmax + wpc - 1) / wpc), 256, vsm, s>>>(L, batch_cl, ws, wpc);
    }
    post_launch("k_eigvec");
  }
  phase(2);
  {
    // QR of the retained vectors on a cluster (columns in distributed shared memory)
    const int kHC = L.bmax <= 64 ? 1 : (L.bmax <= 128 ? 4 : (L.bmax <= 240 ? 8 : kHCmax));
    const int ncl = (L.bmax + kHC - 1) / kHC;
    size_t smem = ((size_t)L.bmax * ncl + 3 * (size_t)L.bmax) * sizeof(cplx) + 64;
    cplx* gU = nullptr;
    const char* force_g = std::getenv("H2G_EIG_GLOBAL");
    if (smem > kSmemCap || (force_g && std::atoi(force_g) && kHC > 1)) {
      gU = workspace(L, (size_t)nb * ((size_t)L.bmax * L.bmax + 16 * (size_t)L.bmax) * sizeof(cplx));
      smem = 3 * (size_t)L.bmax * sizeof(cplx) + 64;
    }
    set_smem((const void*)k_eig1b_cl, smem);
    allow_big_clusters((const void*)k_eig1b_cl);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nb * kHC);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kHC;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, k_eig1b_cl, L, batch_cl, ws, gU);
    if (e != cudaSuccess) throw std::runtime_error(std::string("launch of k_eig1b_cl failed: ") + cudaGetErrorString(e));
    post_launch("k_eig1b_cl");
  }
  if (mmax > 1024) throw std::runtime_error("k_eig1_apply: complement dimension > 1024");
  const dim3 ga(nb, (L.bmax + 7) / 8);
  if (L.bmax <= 128)
    k_eig1_apply<4><<<ga, 256, 0, s>>>(L, batch_cl, ws);
  else if (L.bmax <= 256)
    k_eig1_apply<8><<<ga, 256, 0, s>>>(L, batch_cl, ws);
  else if (L.bmax <= 384)
    k_eig1_apply<12><<<ga, 256, 0, s>>>(L, batch_cl, ws);
  else if (L.bmax <= 512)
    k_eig1_apply<16><<<ga, 256, 0, s>>>(L, batch_cl, ws);
  else if (L.bmax <= 768)
    k_eig1_apply<24><<<ga, 256, 0, s>>>(L, batch_cl, ws);
  else
    k_eig1_apply<32><<<ga, 256, 0, s>>>(L, batch_cl, ws);
  post_launch("k_eig1_apply");
}

void launch_head(const DevLevel& L, const int* batch_cl, int p0, int nb, cudaStream_t s) {
  const int bm = L.bmax;
  const size_t small = (size_t)bm * 8 + (size_t)bm * 4 + (size_t)(bm + 2) * 4 + 16 + (size_t)4 * (bm / 2 + 1) * 8 + 64;
  set_smem((const void*)k_head, small);
  cplx* ws = workspace(L, 4 * (size_t)bm * bm * sizeof(cplx) * nb);
  k_head<<<nb, 256, small, s>>>(L, batch_cl, p0, ws);
  post_launch("k_head");
}

void launch_head2(const DevLevel& L, const int* batch_cl, int nb, int emax, cudaStream_t s) {
  if (emax > 64) {
    // multi-CTA extended LU (k_hlu_*); M per slot is (b + e)^2 <= (2 bmax)^2
    const int ldm = 2 * L.bmax;
    const size_t mbytes = (size_t)ldm * ldm * sizeof(cplx);
    char* ws = reinterpret_cast<char*>(workspace(L, hlu_ws_bytes(L.bmax, nb)));
    cplx* M0 = reinterpret_cast<cplx*>(ws);
    cplx* Dg = reinterpret_cast<cplx*>(ws + mbytes * nb);  // factored 32 x 32 diagonal blocks
    double* scale = reinterpret_cast<double*>(Dg + (size_t)nb * 1024);
    int* fail = reinterpret_cast<int*>(scale + nb);
    cudaMemsetAsync(scale, 0, (size_t)nb * sizeof(double), s);
    k_hlu_prep<<<dim3(nb, 16), 256, 0, s>>>(L, batch_cl, M0, ldm, scale, fail);
    post_launch("k_hlu_prep");
    set_smem((const void*)k_hlu_update, sizeof(Tile128Smem));
    const int nt = (ldm + 63) / 64;
    for (int j0 = 0; j0 < emax; j0 += 32) {
      k_hlu_panel<<<dim3(nb, (2 * ldm + 255) / 256), 256, 0, s>>>(L, batch_cl, M0, ldm, scale, fail, j0, Dg);
      post_launch("k_hlu_panel");
      k_hlu_update<<<dim3(nb, std::min(nt * nt, 64)), 128, sizeof(Tile128Smem), s>>>(L, batch_cl, M0, ldm, fail, j0, Dg);
      post_launch("k_hlu_update");
    }
    k_hlu_finish<<<dim3(nb, 16), 256, 0, s>>>(L, batch_cl, M0, ldm, fail);
    post_launch("k_hlu_finish");
    return;
  }
  cplx* ws = workspace(L, 2 * (size_t)L.bmax * L.bmax * sizeof(cplx) * nb);
  k_head2<<<nb, 256, 0, s>>>(L, batch_cl, ws);
  post_launch("k_head2");
}

void launch_mask(const MaskDesc* d, int n, cudaStream_t s) {
  if (n <= 0) return;
  k_mask<<<dim3(n, 8), 256, 0, s>>>(d);
  post_launch("k_mask");
}

void launch_colnorm(const NormDesc* d, int n, cudaStream_t s) {
  if (n <= 0) return;
  k_colnorm<<<n, 256, 0, s>>>(d);
  post_launch("k_colnorm");
}


void launch_schur_resolve(const DevLevel& L, const SchurTargetD* targets, int ntargets, const SchurContribD* contrib, RTarget* rt, RPanel* rp,
                          cudaStream_t s) {
  if (ntargets <= 0) return;
  k_schur_resolve<<<(ntargets + 127) / 128, 128, 0, s>>>(L, targets, ntargets, contrib, rt, rp);
  post_launch("k_schur_resolve");
}

void launch_schur(const DevLevel& L, const SchurTargetD* targets, int ntargets, const SchurContribD* contrib, cudaStream_t s, const RTarget* rt,
                  const RPanel* rp) {
  if (ntargets <= 0) return;
  static const int t32_bmax = std::getenv("H2G_SCHUR_T32_BMAX") ? std::atoi(std::getenv("H2G_SCHUR_T32_BMAX")) : 32;
  if (L.bmax <= t32_bmax) {
    // small blocks (leaf levels, e of a few columns): 32 x 32 DFMA tiles, the
    // target read-modify-write dominates and a 64 x 64 tensor tile would be 3/4 padding
    const int t32 = (L.bmax + 31) / 32;
    set_smem((const void*)k_schur<32>, sizeof(TileSmem<32>));
    k_schur<32><<<dim3(ntargets, t32 * t32), 128, sizeof(TileSmem<32>), s>>>(L, targets, contrib, rt, rp);
    post_launch("k_schur");
    return;
  }
  const int t = (L.bmax + 63) / 64;
  // small eliminated sizes (fine levels): bound by the targets' read-modify-write -> staged target tiles
  static const int pf_bmax = std::getenv("H2G_SCHUR_PF_BMAX") ? std::atoi(std::getenv("H2G_SCHUR_PF_BMAX")) : 0;
  if (L.bmax <= pf_bmax) {
    const size_t sm = sizeof(TileSmem<64, 2>) + 64 * 64 * sizeof(cplx);
    set_smem((const void*)k_schur<64, true>, sm);
    k_schur<64, true><<<dim3(ntargets, t * t), 128, sm, s>>>(L, targets, contrib, rt, rp);
    post_launch("k_schur");
    return;
  }
  static const int nst = std::getenv("H2G_SCHUR_STAGES") ? std::atoi(std::getenv("H2G_SCHUR_STAGES")) : 3;
  if (nst == 4) {
    set_smem((const void*)k_schur<64, false, 4>, sizeof(TileSmem<64, 4>));
    k_schur<64, false, 4><<<dim3(ntargets, t * t), 128, sizeof(TileSmem<64, 4>), s>>>(L, targets, contrib, rt, rp);
    post_launch("k_schur");
    return;
  }
  set_smem((const void*)k_schur<64>, sizeof(Tile128Smem));
  k_schur<64><<<dim3(ntargets, t * t), 128, sizeof(Tile128Smem), s>>>(L, targets, contrib, rt, rp);
  post_launch("k_schur");
}

__global__ void __launch_bounds__(256) k_move(const MoveDesc* descs) {
  const MoveDesc d = descs[blockIdx.x];
  for (long long i = (long long)blockIdx.y * blockDim.x + threadIdx.x; i < d.len; i += (long long)gridDim.y * blockDim.x) d.dst[i] = d.src[i];
}
__global__ void k_int_move(int* base, const int* idx, int n, int* packed, int scatter) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (scatter) base[idx[i]] = packed[i];
  else packed[i] = base[idx[i]];
}
void launch_move(const MoveDesc* d, int n, cudaStream_t s) {
  if (n > 0) k_move<<<dim3(n, 8), 256, 0, s>>>(d); post_launch("k_move");
}
void launch_int_move(int* base, const int* idx, int n, int* packed, int scatter, cudaStream_t s) {
  if (n > 0) k_int_move<<<(n + 255) / 256, 256, 0, s>>>(base, idx, n, packed, scatter); post_launch("k_int_move");
}

void launch_copy(const CopyDesc* d, int n, cudaStream_t s) {
  if (n > 0) k_copy<<<n, 256, 0, s>>>(d); post_launch("k_copy");
}

// maxdim: upper bound of max(m, n) over the descriptors (0: unknown). Small
// blocks run on 32 x 32 / 16 x 16 tiles instead of wasting a 64 x 64 tile.
template <int TM>
static void launch_gemm_tm(const GemmDesc* d, int n, cudaStream_t s, int maxdim, int cap = 16) {
  set_smem((const void*)k_gemm<TM>, sizeof(TileSmem<TM>));
  const int t = maxdim > 0 ? (maxdim + TM - 1) / TM : 1;
  k_gemm<TM><<<dim3(n, std::max(1, std::min(t * t, cap))), 128, sizeof(TileSmem<TM>), s>>>(d);
  post_launch("k_gemm");
}

void launch_gemm(const GemmDesc* d, int n, cudaStream_t s, int maxdim) {
  if (n <= 0) return;
  if (maxdim > 0 && maxdim <= 16)
    launch_gemm_tm<16>(d, n, s, maxdim);
  else if (maxdim > 0 && maxdim <= 32)
    launch_gemm_tm<32>(d, n, s, maxdim);
  else
    launch_gemm_tm<64>(d, n, s, maxdim);
}

int root_lu(cplx* A, int n, double tol, DevError* err, void* scratch, cudaStream_t s, long long* launches) {
  (void)tol;
  double* scale = reinterpret_cast<double*>(scratch);
  cudaMemsetAsync(scale, 0, sizeof(double), s);
  const long long n2 = (long long)n * n;
  k_absmax<<<(int)std::min<long long>(1024, (n2 + 255) / 256), 256, 0, s>>>(A, n2, scale);
  *launches += 1;
  for (int k0 = 0; k0 < n; k0 += 32) {
    const int kb = std::min(32, n - k0);
    k_lu_panel<<<1, 256, 0, s>>>(A, n, k0, kb, scale, err);
    post_launch("k_lu_panel");
    const int rest = n - k0 - kb;
    *launches += 1;
    if (rest > 0) {
      k_lu_trsm<<<(rest + 127) / 128, 128, 0, s>>>(A, n, k0, kb);
      dim3 g((rest + 63) / 64, (rest + 63) / 64);
      const int sm = (64 * 33 + 32 * 65) * (int)sizeof(cplx);
      set_smem((const void*)k_lu_update, sm);
      k_lu_update<<<g, 256, sm, s>>>(A, n, k0, kb);
      *launches += 2;
    }
  }
  return 0;
}

}  // namespace h2g
