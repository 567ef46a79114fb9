// Device H² construction and matvec.
//
// build_h2 (proj/include/h2lu/h2_matrix.hpp:300-375): bottom-up, every
// cluster's basis is the truncated left singular space (sigma_j >
// max(eps sigma_0, 1e-300), h2_matrix.hpp:287-290) of its far-field sample
// [Z(c, far cols) | Z(far rows, c)^T], projected through the children's
// expanded bases above the leaves (project_rows/project_cols, :237-267). On
// the device the sample is never materialised: kernel entries are generated
// tile by tile, projected (D^H Z) and folded into a Gram matrix whose
// Hermitian eigendecomposition (Jacobi) yields the left singular vectors.
// Couplings S = E_t^H Z(t,s) conj(E_s) (:354-365) and dense leaf blocks
// (:367-373) are generated the same way.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <stdexcept>

#include "build.cuh"
#include "factor.cuh"

namespace h2g {

namespace {

struct KernelD {
  int kind;
  double kr, ki, sr, si, dr, di;
};

__device__ __forceinline__ cplx kentry(const KernelD& K, const double* px, const double* py, const double* pz, long long i, long long j) {
  if (i == j) return cmk(K.dr, K.di);
  if (K.kind == H2G_KERNEL_ZERO) return czero();
  const double dx = px[i] - px[j], dy = py[i] - py[j], dz = pz[i] - pz[j];
  const double r = sqrt(dx * dx + dy * dy + dz * dz);
  const double inv = 1.0 / (4.0 * 3.141592653589793 * r);
  cplx v;
  if (K.kind == H2G_KERNEL_LAPLACE) {
    v = cmk(inv, 0.0);
  } else {
    // exp(-i k r), k = kr + i ki  ->  exp(ki r) (cos(kr r) - i sin(kr r))
    double s, c;
    sincos(K.kr * r, &s, &c);
    const double a = exp(K.ki * r) * inv;
    v = cmk(a * c, -a * s);
  }
  return cmul(cmk(K.sr, K.si), v);
}

constexpr int kTileSmem = 3 * 64 * 65 * 16;

struct FarItem {
  int q;          // cluster slot at this level
  int first_col;  // absolute tree index of the first column
  int ncols;      // <= 64, contiguous
  int part;       // partial slot of the cluster
};

struct BuildLevel {
  int bm;             // max local size (kloc)
  const long long* cbeg;  // per slot: first row (tree index)
  const int* csize;   // per slot: |c|
  const int* kloc;    // per slot: local dimension (|c| for leaves, k1 + k2 above)
  const long long* D_off;  // per slot: offset of D (|c| x kloc) in Dbuf (non-leaf), -1 for leaf
  const cplx* Dbuf;
  cplx* part;         // partial Grams, stride bm*bm
  int nparts;
  const double* px;
  const double* py;
  const double* pz;
  KernelD K;
};

// One CTA per (cluster slot, part, tile pair ta <= tb of the kloc x kloc
// Gram): Y_x = D(:, tile x)^H Z(c, cols) for the item's columns, G[ta, tb] +=
// Y_ta Y_tb^H; the mirrored tile is written as its conjugate transpose.
__device__ __forceinline__ void tile_pair(int pr, int& ta, int& tb) {
  ta = 0;
  while (pr > ta) pr -= ta + 1, ++ta;  // pairs (0,0) (0,1) (1,1) (0,2) ...: tb-major
  tb = ta;
  ta = pr;
}

__global__ void __launch_bounds__(256) k_far_gram(BuildLevel B, const FarItem* items, const int* item_ptr) {
  extern __shared__ __align__(16) unsigned char smraw[];
  cplx(*sZ)[65] = reinterpret_cast<cplx(*)[65]>(smraw);
  cplx(*sD)[65] = sZ + 64;
  const int q = blockIdx.x;  // one CTA per (cluster slot, part, tile pair)
  const int part = blockIdx.y;
  int ta, tb;
  tile_pair(blockIdx.z, ta, tb);
  const int kl = B.kloc[q], nr = B.csize[q];
  if (tb * 64 >= kl) return;
  const long long r0 = B.cbeg[q];
  const bool leaf = B.D_off[q] < 0;
  const bool same = ta == tb;
  const int tr = threadIdx.x % 16, tc = threadIdx.x / 16;
  cplx g[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) g[a][b] = czero();
  for (int it = item_ptr[q] + part; it < item_ptr[q + 1]; it += B.nparts) {
    const FarItem fi = items[it];
    cplx ya[4][4], yb[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) ya[a][b] = czero(), yb[a][b] = czero();
    for (int rc = 0; rc < nr; rc += 64) {
      const int rn = min(64, nr - rc);
      __syncthreads();
      for (int idx = threadIdx.x; idx < 64 * 64; idx += blockDim.x) {
        const int i = idx % 64, j = idx / 64;
        sZ[i][j] = (i < rn && j < fi.ncols) ? kentry(B.K, B.px, B.py, B.pz, r0 + rc + i, fi.first_col + j) : czero();
      }
      if (leaf) {
        // Y = Z directly (kloc = |c| <= 64, a single tile)
        __syncthreads();
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) ya[a][b] = sZ[tr * 4 + a][tc * 4 + b];
        continue;
      }
      const cplx* D = B.Dbuf + B.D_off[q];
      for (int pass = 0; pass < (same ? 1 : 2); ++pass) {
        const int c0 = (pass == 0 ? ta : tb) * 64;
        __syncthreads();
        for (int idx = threadIdx.x; idx < 64 * 64; idx += blockDim.x) {
          const int i = idx % 64, j = idx / 64;
          sD[i][j] = (i < rn && c0 + j < kl) ? D[rc + i + (size_t)(c0 + j) * nr] : czero();
        }
        __syncthreads();
        for (int p = 0; p < rn; ++p) {
          cplx dv[4], zv[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) dv[a] = cconj(sD[p][tr * 4 + a]);
#pragma unroll
          for (int b = 0; b < 4; ++b) zv[b] = sZ[p][tc * 4 + b];
          if (pass == 0) {
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
              for (int b = 0; b < 4; ++b) cfma(ya[a][b], dv[a], zv[b]);
          } else {
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
              for (int b = 0; b < 4; ++b) cfma(yb[a][b], dv[a], zv[b]);
          }
        }
      }
    }
    __syncthreads();
    // Y_ta into sZ, Y_tb into sD
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        sZ[tr * 4 + a][tc * 4 + b] = ya[a][b];
        sD[tr * 4 + a][tc * 4 + b] = same ? ya[a][b] : yb[a][b];
      }
    __syncthreads();
    // G += Y_ta Y_tb^H over the chunk's columns
    for (int p = 0; p < fi.ncols; ++p) {
      cplx av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = sZ[tr * 4 + a][p];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = cconj(sD[tc * 4 + b][p]);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) cfma(g[a][b], av[a], bv[b]);
    }
  }
  cplx* out = B.part + ((size_t)q * B.nparts + part) * B.bm * B.bm;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = ta * 64 + tr * 4 + a, j = tb * 64 + tc * 4 + b;
      if (i < kl && j < kl) {
        out[i + (size_t)j * kl] = g[a][b];
        if (!same) out[j + (size_t)i * kl] = cconj(g[a][b]);
      }
    }
}

// Per cluster: G = sum of parts (x mult), Jacobi eigendecomposition, eigen
// vectors sorted by descending value into U (kloc x kloc) and the rank.
__global__ void __launch_bounds__(256) k_far_eig(BuildLevel B, double mult, double eps, cplx* Uout, int* rank, cplx* gws) {
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ double red[32];
  const int q = blockIdx.x;
  const int n = B.kloc[q], bm = B.bm;
  // H, U in shared memory for small clusters, else in the global workspace
  cplx* H = gws ? gws + (size_t)q * 2 * bm * bm : reinterpret_cast<cplx*>(smraw);
  cplx* U = H + bm * bm;
  double* lam = gws ? reinterpret_cast<double*>(smraw) : reinterpret_cast<double*>(U + bm * bm);
  int* ord = reinterpret_cast<int*>(lam + bm);
  int* pr = ord + bm;
  double* rot = reinterpret_cast<double*>(pr + bm + 2);
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    cplx s = czero();
    for (int p = 0; p < B.nparts; ++p) s = cadd(s, B.part[((size_t)q * B.nparts + p) * bm * bm + idx]);
    H[idx] = cscale(s, mult);
  }
  __syncthreads();
  cta_jacobi_eig(n, H, U, rot, pr, red);
  for (int i = threadIdx.x; i < n; i += blockDim.x) lam[i] = sqrt(fmax(H[i + i * n].x, 0.0));
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int r = 0;
    for (int j = 0; j < n; ++j) r += (lam[j] > lam[i]) || (lam[j] == lam[i] && j < i);
    ord[r] = i;
  }
  __syncthreads();
  cplx* Uo = Uout + (size_t)q * bm * bm;
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    const int i = idx % n, j = idx / n;
    Uo[i + (size_t)j * n] = U[i + ord[j] * n];
  }
  if (threadIdx.x == 0) {
    int r = 0;
    const double s0 = n ? lam[ord[0]] : 0.0;
    if (s0 > 0.0) {
      const double thr = fmax(eps * s0, 1e-300);
      while (r < n && lam[ord[r]] > thr) ++r;
    }
    rank[q] = r;
  }
}

struct CoupItem {
  int pair;   // pair slot
  int rc;     // row chunk start (relative to t)
  int part;   // partial index
};

struct CoupLevel {
  const long long* tb;   // per pair: first row of t
  const long long* sb;   // per pair: first col of s
  const int* tn;
  const int* sn;
  const int* kt;
  const int* ks;
  const long long* Et_off;  // expanded basis of t (|t| x kt), ld |t|
  const long long* Es_off;
  const cplx* E;
  cplx* part;            // partial couplings (kt x ks), stride pstride
  long long pstride;
  const double* px;
  const double* py;
  const double* pz;
  KernelD K;
};

// One CTA per (pair, 64-row chunk of t, 64 x 64 tile (a, b) of S): X =
// Z(rows, s) conj(E_s(:, tile b)) then S_part(tile a, tile b) = E_t(rows, tile a)^H X.
__global__ void __launch_bounds__(256) k_coupling(CoupLevel C, const CoupItem* items, int ntb) {
  extern __shared__ __align__(16) unsigned char smraw[];
  cplx(*sZ)[65] = reinterpret_cast<cplx(*)[65]>(smraw);
  cplx(*sE)[65] = sZ + 64;
  cplx(*sX)[65] = sZ + 128;
  const CoupItem it = items[blockIdx.x];
  const int pq = it.pair;
  const int ta = blockIdx.y / ntb, tb = blockIdx.y % ntb;
  const int tn = C.tn[pq], sn = C.sn[pq], kt0 = C.kt[pq], ks0 = C.ks[pq];
  if (ta * 64 >= kt0 || tb * 64 >= ks0) return;
  const int kt = min(64, kt0 - ta * 64), ks = min(64, ks0 - tb * 64);
  const int rn = min(64, tn - it.rc);
  const long long r0 = C.tb[pq] + it.rc, c0 = C.sb[pq];
  const cplx* Et = C.E + C.Et_off[pq] + (size_t)ta * 64 * tn;
  const cplx* Es = C.E + C.Es_off[pq] + (size_t)tb * 64 * sn;
  const int tr = threadIdx.x % 16, tc = threadIdx.x / 16;
  cplx x[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) x[a][b] = czero();
  for (int cc = 0; cc < sn; cc += 64) {
    const int cn = min(64, sn - cc);
    __syncthreads();
    for (int idx = threadIdx.x; idx < 64 * 64; idx += blockDim.x) {
      const int i = idx % 64, j = idx / 64;
      sZ[i][j] = (i < rn && j < cn) ? kentry(C.K, C.px, C.py, C.pz, r0 + i, c0 + cc + j) : czero();
      sE[i][j] = (i < cn && j < ks) ? cconj(Es[cc + i + (size_t)j * sn]) : czero();
    }
    __syncthreads();
    for (int p = 0; p < cn; ++p) {
      cplx av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = sZ[tr * 4 + a][p];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = sE[p][tc * 4 + b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) cfma(x[a][b], av[a], bv[b]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) sX[tr * 4 + a][tc * 4 + b] = x[a][b];
  for (int idx = threadIdx.x; idx < 64 * 64; idx += blockDim.x) {
    const int i = idx % 64, j = idx / 64;  // sE <- Et(rows)^H : kt x rn
    sE[j][i] = (i < rn && j < kt) ? cconj(Et[it.rc + i + (size_t)j * tn]) : czero();
  }
  __syncthreads();
  cplx s[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) s[a][b] = czero();
  for (int p = 0; p < rn; ++p) {
    cplx av[4], bv[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) av[a] = sE[tr * 4 + a][p];
#pragma unroll
    for (int b = 0; b < 4; ++b) bv[b] = sX[p][tc * 4 + b];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) cfma(s[a][b], av[a], bv[b]);
  }
  cplx* out = C.part + (size_t)blockIdx.x * C.pstride;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = tr * 4 + a, j = tc * 4 + b;
      if (i < kt && j < ks) out[ta * 64 + i + (size_t)(tb * 64 + j) * kt0] = s[a][b];
    }
}

// S = sum of the pair's row-chunk partials (fixed order).
__global__ void k_coupling_reduce(const cplx* part, long long pstride, const int* item_ptr, const int* kt, const int* ks, const long long* out_off,
                                  cplx* out) {
  const int pq = blockIdx.x;
  const int n = kt[pq] * ks[pq];
  for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
    cplx s = czero();
    for (int it = item_ptr[pq]; it < item_ptr[pq + 1]; ++it) s = cadd(s, part[(size_t)it * pstride + idx]);
    out[out_off[pq] + idx] = s;
  }
}

// Dense leaf blocks Z(t, s) (kernel.hpp:64-83; diagonal entries = diag).
__global__ void k_dense(const long long* tb, const long long* sb, const int* tn, const int* sn, const long long* off, cplx* out, const double* px,
                        const double* py, const double* pz, KernelD K) {
  const int q = blockIdx.x;
  const int m = tn[q], n = sn[q];
  for (int idx = threadIdx.x; idx < m * n; idx += blockDim.x) {
    const int i = idx % m, j = idx / m;
    out[off[q] + idx] = kentry(K, px, py, pz, tb[q] + i, sb[q] + j);
  }
}

__global__ void k_finite_check(const cplx* a, long long n, int* bad) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (!isfinite(a[i].x) || !isfinite(a[i].y)) *bad = 1;
}

#define CKB(x)                                                                                                 \
  do {                                                                                                         \
    cudaError_t e_ = (x);                                                                                      \
    if (e_ != cudaSuccess) throw std::runtime_error(std::string("cuda: ") + #x + ": " + cudaGetErrorString(e_)); \
  } while (0)

template <class T>
T* dev_upload(const std::vector<T>& v, cudaStream_t s) {
  T* p = nullptr;
  CKB(cudaMallocAsync(&p, std::max<size_t>(v.size(), 1) * sizeof(T), s));
  if (!v.empty()) CKB(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  return p;
}

struct Range {
  int64_t b, e;
};

void merge_ranges(std::vector<Range>& v) {
  std::sort(v.begin(), v.end(), [](const Range& a, const Range& b) { return a.b < b.b; });
  std::vector<Range> out;
  for (const auto& r : v) {
    if (!out.empty() && out.back().e >= r.b)
      out.back().e = std::max(out.back().e, r.e);
    else
      out.push_back(r);
  }
  v.swap(out);
}

}  // namespace

BuildResult build_h2_device(const Structure& S, const double* points, const std::vector<int64_t>& perm, const h2g_kernel_spec& Ks,
                            double eps_h2, cudaStream_t st) {
  const int L = S.depth, nc = S.num_clusters();
  const int64_t n = S.n;
  KernelD K{Ks.kind, Ks.wavenumber_re, Ks.wavenumber_im, Ks.scale_re, Ks.scale_im, Ks.diag_re, Ks.diag_im};
  // points in tree order, structure-of-arrays
  std::vector<double> hx(n), hy(n), hz(n);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t o = perm[i];
    hx[i] = points[3 * o], hy[i] = points[3 * o + 1], hz[i] = points[3 * o + 2];
  }
  double* px = dev_upload(hx, st);
  double* py = dev_upload(hy, st);
  double* pz = dev_upload(hz, st);

  // far fields (h2_matrix.hpp:206-226)
  std::vector<std::vector<Range>> fcols(nc), frows(nc);
  for (int l = 0; l <= L; ++l) {
    for (int id = Structure::first(l); id < Structure::first(l + 1); ++id)
      if (id > 0) fcols[id] = fcols[(id - 1) / 2], frows[id] = frows[(id - 1) / 2];
    for (const auto& p : S.adm[l]) {
      fcols[p.row].push_back({S.begin[p.col], S.end[p.col]});
      frows[p.col].push_back({S.begin[p.row], S.end[p.row]});
    }
  }
  for (int id = 0; id < nc; ++id) merge_ranges(fcols[id]), merge_ranges(frows[id]);

  BuildResult R;
  R.basis_rows.assign(nc, 0);
  R.basis_rank.assign(nc, 0);
  std::vector<std::vector<std::complex<double>>> hbasis(nc);  // host copy of every basis (small)
  // expanded bases of the previous (finer) level: per cluster (|c| x r), device
  cplx* Eprev = nullptr;
  std::vector<long long> Eprev_off(nc, -1);

  std::vector<cplx*> to_free;
  std::vector<std::vector<std::complex<double>>> coup_level(L + 1);
  std::vector<long long> coup_local(S.num_adm(), 0);
  for (int l = L; l >= 0; --l) {
    const int f0 = Structure::first(l), cnt = 1 << l;
    std::vector<long long> cbeg(cnt), Doff(cnt, -1);
    std::vector<int> csize(cnt), kloc(cnt);
    std::vector<FarItem> items;
    std::vector<int> item_ptr(cnt + 1, 0);
    std::vector<char> active(cnt, 0), dup(cnt, 0);
    int bm = 1;
    long long dtop = 0;
    for (int q = 0; q < cnt; ++q) {
      const int id = f0 + q;
      cbeg[q] = S.begin[id];
      csize[q] = static_cast<int>(S.end[id] - S.begin[id]);
      const bool leaf = l == L;
      kloc[q] = leaf ? csize[q] : static_cast<int>(R.basis_rank[2 * id + 1] + R.basis_rank[2 * id + 2]);
      R.basis_rows[id] = kloc[q];
      const bool far = !(fcols[id].empty() && frows[id].empty());
      active[q] = far && kloc[q] > 0;
      if (active[q]) {
        bm = std::max(bm, kloc[q]);
        if (!leaf) Doff[q] = dtop, dtop += (long long)csize[q] * kloc[q];
        // sample columns: far cols, then far rows (symmetric kernel: Z(rows,c)^T = Z(c,rows))
        bool same = fcols[id].size() == frows[id].size();
        for (size_t i = 0; same && i < fcols[id].size(); ++i) same = fcols[id][i].b == frows[id][i].b && fcols[id][i].e == frows[id][i].e;
        dup[q] = same;
        for (int pass = 0; pass < (same ? 1 : 2); ++pass)
          for (const auto& r : (pass == 0 ? fcols[id] : frows[id]))
            for (int64_t c = r.b; c < r.e; c += 64) items.push_back({q, static_cast<int>(c), static_cast<int>(std::min<int64_t>(64, r.e - c)), 0});
      }
      item_ptr[q + 1] = static_cast<int>(items.size());
    }
    // mixed dup flags would need per-cluster multipliers; the sample is
    // symmetric for every cluster of a symmetric partition
    bool all_dup = true, any_active = false;
    for (int q = 0; q < cnt; ++q)
      if (active[q]) all_dup = all_dup && dup[q], any_active = true;
    if (!all_dup) {
      // rebuild without the duplicate shortcut
      items.clear();
      for (int q = 0; q < cnt; ++q) {
        const int id = f0 + q;
        if (active[q])
          for (int pass = 0; pass < 2; ++pass)
            for (const auto& r : (pass == 0 ? fcols[id] : frows[id]))
              for (int64_t c = r.b; c < r.e; c += 64) items.push_back({q, static_cast<int>(c), static_cast<int>(std::min<int64_t>(64, r.e - c)), 0});
        item_ptr[q + 1] = static_cast<int>(items.size());
      }
    }
    if (l == L && bm > 64) throw std::runtime_error("build_h2_device: leaf size > 64 not supported");
    const int T = (bm + 63) / 64;  // Gram tiles per side
    std::vector<int> rank(cnt, 0);
    cplx* Ubuf = nullptr;
    if (any_active) {
      // D = blockdiag(E_c1, E_c2) for non-leaf clusters (|c| x kloc)
      cplx* Dbuf = nullptr;
      if (l < L && dtop > 0) {
        CKB(cudaMallocAsync(&Dbuf, dtop * 16, st));
        CKB(cudaMemsetAsync(Dbuf, 0, dtop * 16, st));
        std::vector<CopyDesc> cd;
        for (int q = 0; q < cnt; ++q) {
          if (!active[q]) continue;
          const int id = f0 + q;
          const int c1 = 2 * id + 1, c2 = 2 * id + 2;
          const int n1 = static_cast<int>(S.end[c1] - S.begin[c1]);
          const int k1 = static_cast<int>(R.basis_rank[c1]), k2 = static_cast<int>(R.basis_rank[c2]);
          cplx* D = Dbuf + Doff[q];
          if (k1) cd.push_back({Eprev + Eprev_off[c1], D, n1, csize[q], n1, k1, 0, 0});
          if (k2) cd.push_back({Eprev + Eprev_off[c2], D + n1 + (size_t)k1 * csize[q], csize[q] - n1, csize[q], csize[q] - n1, k2, 0, 0});
        }
        CopyDesc* dcd = dev_upload(cd, st);
        launch_copy(dcd, static_cast<int>(cd.size()), st);
        to_free.push_back(reinterpret_cast<cplx*>(dcd));
      }
      const int nparts = 16;
      cplx* part = nullptr;
      CKB(cudaMallocAsync(&part, (size_t)cnt * nparts * bm * bm * 16, st));
      CKB(cudaMemsetAsync(part, 0, (size_t)cnt * nparts * bm * bm * 16, st));
      std::vector<int> kact(cnt);
      for (int q = 0; q < cnt; ++q) kact[q] = active[q] ? kloc[q] : 0;
      long long* dcb = dev_upload(cbeg, st);
      int* dcs = dev_upload(csize, st);
      int* dkl = dev_upload(kact, st);
      long long* ddo = dev_upload(Doff, st);
      FarItem* dit = dev_upload(items, st);
      int* dip = dev_upload(item_ptr, st);
      BuildLevel BL{bm, dcb, dcs, dkl, ddo, Dbuf, part, nparts, px, py, pz, K};
      CKB(cudaFuncSetAttribute((const void*)k_far_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileSmem));
      k_far_gram<<<dim3(cnt, nparts, T * (T + 1) / 2), 256, kTileSmem, st>>>(BL, dit, dip);
      CKB(cudaGetLastError());
      CKB(cudaMallocAsync(&Ubuf, (size_t)cnt * bm * bm * 16, st));
      int* drank = nullptr;
      CKB(cudaMallocAsync(&drank, cnt * 4, st));
      const size_t small = (size_t)bm * 8 + (size_t)bm * 4 + (size_t)(bm + 2) * 4 + 16 + (size_t)4 * (bm / 2 + 1) * 8 + 64;
      cplx* eigws = nullptr;
      size_t smem = 2 * (size_t)bm * bm * 16 + small;
      if (bm > 64) {
        CKB(cudaMallocAsync(&eigws, (size_t)cnt * 2 * bm * bm * 16, st));
        smem = small;
      }
      CKB(cudaFuncSetAttribute((const void*)k_far_eig, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_far_eig<<<cnt, 256, smem, st>>>(BL, all_dup ? 2.0 : 1.0, eps_h2, Ubuf, drank, eigws);
      if (eigws) cudaFreeAsync(eigws, st);
      CKB(cudaGetLastError());
      CKB(cudaMemcpyAsync(rank.data(), drank, cnt * 4, cudaMemcpyDeviceToHost, st));
      CKB(cudaStreamSynchronize(st));
      for (int q = 0; q < cnt; ++q)
        if (!active[q]) rank[q] = 0;
      for (void* p : {(void*)part, (void*)dcb, (void*)dcs, (void*)dkl, (void*)ddo, (void*)dit, (void*)dip, (void*)drank}) cudaFreeAsync(p, st);
      if (Dbuf) cudaFreeAsync(Dbuf, st);
    }
    // basis data to host (compact), expanded bases of this level
    std::vector<long long> Eoff(cnt, -1);
    long long etop = 0;
    for (int q = 0; q < cnt; ++q) {
      const int id = f0 + q;
      R.basis_rank[id] = rank[q];
      hbasis[id].assign((size_t)kloc[q] * rank[q], 0.0);
      if (rank[q]) {
        std::vector<std::complex<double>> tmp((size_t)kloc[q] * rank[q]);
        CKB(cudaMemcpyAsync(tmp.data(), Ubuf + (size_t)q * bm * bm, tmp.size() * 16, cudaMemcpyDeviceToHost, st));
        CKB(cudaStreamSynchronize(st));
        hbasis[id] = std::move(tmp);
      }
      Eoff[q] = etop;
      etop += (long long)csize[q] * rank[q];
    }
    cplx* Enew = nullptr;
    CKB(cudaMallocAsync(&Enew, std::max<long long>(etop, 1) * 16, st));
    {
      std::vector<GemmDesc> gd;
      std::vector<CopyDesc> cd;
      for (int q = 0; q < cnt; ++q) {
        if (!rank[q]) continue;
        const int id = f0 + q;
        const cplx* U = Ubuf + (size_t)q * bm * bm;  // kloc x kloc (first rank cols used)
        if (l == L) {
          cd.push_back({U, Enew + Eoff[q], kloc[q], csize[q], csize[q], rank[q], 0, 0});
        } else {
          const int c1 = 2 * id + 1, c2 = 2 * id + 2;
          const int n1 = static_cast<int>(S.end[c1] - S.begin[c1]), n2 = csize[q] - n1;
          const int k1 = static_cast<int>(R.basis_rank[c1]), k2 = static_cast<int>(R.basis_rank[c2]);
          cplx* E = Enew + Eoff[q];
          if (k1) gd.push_back({Eprev + Eprev_off[c1], U, E, n1, kloc[q], csize[q], n1, rank[q], k1, OP_N, OP_N, 1.0, 0.0});
          else cd.push_back({nullptr, E, 0, csize[q], n1, rank[q], 0, 0});
          if (k2) gd.push_back({Eprev + Eprev_off[c2], U + k1, E + n1, n2, kloc[q], csize[q], n2, rank[q], k2, OP_N, OP_N, 1.0, 0.0});
          else cd.push_back({nullptr, E + n1, 0, csize[q], n2, rank[q], 0, 0});
        }
      }
      CopyDesc* dcd = dev_upload(cd, st);
      GemmDesc* dgd = dev_upload(gd, st);
      launch_copy(dcd, static_cast<int>(cd.size()), st);
      launch_gemm(dgd, static_cast<int>(gd.size()), st);
      CKB(cudaGetLastError());
      CKB(cudaStreamSynchronize(st));
      cudaFreeAsync(dcd, st);
      cudaFreeAsync(dgd, st);
    }
    if (Ubuf) cudaFreeAsync(Ubuf, st);
    // couplings of this level: S = E_t^H Z(t,s) conj(E_s)
    if (Eprev) cudaFreeAsync(Eprev, st);
    Eprev = Enew;
    std::fill(Eprev_off.begin(), Eprev_off.end(), -1);
    for (int q = 0; q < cnt; ++q) Eprev_off[f0 + q] = Eoff[q];
    // couplings need E of this level only: compute now
    {
      const auto& adm = S.adm[l];
      if (!adm.empty()) {
        std::vector<long long> tb, sb, Et, Es, ooff;
        std::vector<int> tn, sn, kt, ks, iptr(1, 0);
        std::vector<CoupItem> items2;
        for (size_t p = 0; p < adm.size(); ++p) {
          const int t = adm[p].row, s = adm[p].col;
          tb.push_back(S.begin[t]);
          sb.push_back(S.begin[s]);
          tn.push_back(static_cast<int>(S.end[t] - S.begin[t]));
          sn.push_back(static_cast<int>(S.end[s] - S.begin[s]));
          kt.push_back(static_cast<int>(R.basis_rank[t]));
          ks.push_back(static_cast<int>(R.basis_rank[s]));
          Et.push_back(Eprev_off[t]);
          Es.push_back(Eprev_off[s]);
          if (kt.back() && ks.back())
            for (int rc = 0; rc < tn.back(); rc += 64) items2.push_back({static_cast<int>(p), rc, 0});
          iptr.push_back(static_cast<int>(items2.size()));
        }
        int kmx = 1;
        for (size_t p = 0; p < adm.size(); ++p) kmx = std::max(kmx, std::max(kt[p], ks[p]));
        const int ntk = (kmx + 63) / 64;
        const long long pstride = (long long)kmx * kmx;
        cplx* part = nullptr;
        CKB(cudaMallocAsync(&part, std::max<size_t>(items2.size(), 1) * pstride * 16, st));
        long long *dtb = dev_upload(tb, st), *dsb = dev_upload(sb, st), *dEt = dev_upload(Et, st), *dEs = dev_upload(Es, st);
        int *dtn = dev_upload(tn, st), *dsn = dev_upload(sn, st), *dkt = dev_upload(kt, st), *dks = dev_upload(ks, st), *dip = dev_upload(iptr, st);
        CoupItem* dit = dev_upload(items2, st);
        CoupLevel CLv{dtb, dsb, dtn, dsn, dkt, dks, dEt, dEs, Eprev, part, pstride, px, py, pz, K};
        CKB(cudaFuncSetAttribute((const void*)k_coupling, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileSmem));
        if (!items2.empty()) k_coupling<<<dim3(static_cast<int>(items2.size()), ntk * ntk), 256, kTileSmem, st>>>(CLv, dit, ntk);
        // compact output offsets (temporary buffer, then host)
        long long top = 0;
        for (size_t p = 0; p < adm.size(); ++p) ooff.push_back(top), top += (long long)kt[p] * ks[p];
        long long* doo = dev_upload(ooff, st);
        cplx* cout = nullptr;
        CKB(cudaMallocAsync(&cout, std::max<long long>(top, 1) * 16, st));
        k_coupling_reduce<<<static_cast<int>(adm.size()), 256, 0, st>>>(part, pstride, dip, dkt, dks, doo, cout);
        CKB(cudaGetLastError());
        std::vector<std::complex<double>> hc(std::max<long long>(top, 1));
        CKB(cudaMemcpyAsync(hc.data(), cout, top * 16, cudaMemcpyDeviceToHost, st));
        CKB(cudaStreamSynchronize(st));
        coup_level[l] = std::move(hc);
        for (size_t p = 0; p < adm.size(); ++p) coup_local[S.adm_offset[l] + p] = ooff[p];
        for (void* p : {(void*)part, (void*)dtb, (void*)dsb, (void*)dEt, (void*)dEs, (void*)dtn, (void*)dsn, (void*)dkt, (void*)dks, (void*)dip,
                        (void*)dit, (void*)doo, (void*)cout})
          cudaFreeAsync(p, st);
      }
    }
  }
  if (Eprev) cudaFreeAsync(Eprev, st);

  // ---- assemble compact device arrays
  R.basis_off.assign(nc, 0);
  long long btop = 0;
  for (int id = 0; id < nc; ++id) R.basis_off[id] = btop, btop += R.basis_rows[id] * R.basis_rank[id];
  R.basis_elems = btop;
  std::vector<std::complex<double>> hb(std::max<long long>(btop, 1));
  for (int id = 0; id < nc; ++id)
    if (!hbasis[id].empty()) std::memcpy(hb.data() + R.basis_off[id], hbasis[id].data(), hbasis[id].size() * 16);
  CKB(cudaMallocAsync(&R.basis, std::max<long long>(btop, 1) * 16, st));
  CKB(cudaMemcpyAsync(R.basis, hb.data(), btop * 16, cudaMemcpyHostToDevice, st));
  R.coup_off.assign(S.num_adm(), 0);
  long long ctop = 0;
  for (int l = 0; l <= L; ++l)
    for (size_t p = 0; p < S.adm[l].size(); ++p) {
      const int64_t g = S.adm_offset[l] + p;
      R.coup_off[g] = ctop;
      ctop += R.basis_rank[S.adm[l][p].row] * R.basis_rank[S.adm[l][p].col];
    }
  std::vector<std::complex<double>> hcp(std::max<long long>(ctop, 1));
  for (int l = 0; l <= L; ++l)
    for (size_t p = 0; p < S.adm[l].size(); ++p) {
      const int64_t g = S.adm_offset[l] + p;
      const long long sz = R.basis_rank[S.adm[l][p].row] * R.basis_rank[S.adm[l][p].col];
      if (sz) std::memcpy(hcp.data() + R.coup_off[g], coup_level[l].data() + coup_local[g], sz * 16);
    }
  R.coup_elems = ctop;
  CKB(cudaMallocAsync(&R.coup, std::max<long long>(ctop, 1) * 16, st));
  CKB(cudaMemcpyAsync(R.coup, hcp.data(), ctop * 16, cudaMemcpyHostToDevice, st));
  // dense leaf blocks
  {
    std::vector<long long> tb, sb, off;
    std::vector<int> tn, sn;
    long long top = 0;
    for (const auto& p : S.leaf) {
      tb.push_back(S.begin[p.row]);
      sb.push_back(S.begin[p.col]);
      tn.push_back(static_cast<int>(S.end[p.row] - S.begin[p.row]));
      sn.push_back(static_cast<int>(S.end[p.col] - S.begin[p.col]));
      off.push_back(top);
      top += (long long)tn.back() * sn.back();
    }
    R.dense_off.assign(off.begin(), off.end());
    R.dense_elems = top;
    CKB(cudaMallocAsync(&R.dense, std::max<long long>(top, 1) * 16, st));
    long long *dtb = dev_upload(tb, st), *dsb = dev_upload(sb, st), *doff = dev_upload(off, st);
    int *dtn = dev_upload(tn, st), *dsn = dev_upload(sn, st);
    if (!S.leaf.empty())
      k_dense<<<static_cast<int>(S.leaf.size()), 256, 0, st>>>(dtb, dsb, dtn, dsn, doff, reinterpret_cast<cplx*>(R.dense), px, py, pz, K);
    int* bad = nullptr;
    CKB(cudaMallocAsync(&bad, 4, st));
    CKB(cudaMemsetAsync(bad, 0, 4, st));
    if (top) k_finite_check<<<1024, 256, 0, st>>>(reinterpret_cast<cplx*>(R.dense), top, bad);
    int hbad = 0;
    CKB(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, st));
    CKB(cudaStreamSynchronize(st));
    for (void* p : {(void*)dtb, (void*)dsb, (void*)doff, (void*)dtn, (void*)dsn, (void*)bad}) cudaFreeAsync(p, st);
    if (hbad) throw std::invalid_argument("build_h2: kernel entry is not finite");
  }
  for (cplx* p : to_free) cudaFreeAsync(p, st);
  cudaFreeAsync(px, st);
  cudaFreeAsync(py, st);
  cudaFreeAsync(pz, st);
  CKB(cudaStreamSynchronize(st));
  return R;
}

// ---------------------------------------------------------------- matvec
void matvec_device(const Structure& S, const std::vector<int64_t>& basis_rows, const std::vector<int64_t>& basis_rank,
                   const std::vector<int64_t>& basis_off, const std::vector<int64_t>& coup_off, const std::vector<int64_t>& dense_off,
                   const cplx* basis, const cplx* coup, const cplx* dense, const double* x_host, double* y_host, int nrhs, cudaStream_t st) {
  const int L = S.depth, nc = S.num_clusters();
  const int64_t n = S.n;
  cplx *x = nullptr, *y = nullptr, *xh = nullptr, *yh = nullptr, *push = nullptr;
  std::vector<long long> hoff(nc);
  long long top = 0;
  for (int id = 0; id < nc; ++id) hoff[id] = top, top += basis_rank[id];
  long long ptop = 0;
  std::vector<long long> poff(nc);
  for (int id = 0; id < nc; ++id) poff[id] = ptop, ptop += basis_rows[id];
  CKB(cudaMallocAsync(&x, n * nrhs * 16, st));
  CKB(cudaMallocAsync(&y, n * nrhs * 16, st));
  CKB(cudaMallocAsync(&xh, std::max<long long>(top, 1) * nrhs * 16, st));
  CKB(cudaMallocAsync(&yh, std::max<long long>(top, 1) * nrhs * 16, st));
  CKB(cudaMallocAsync(&push, std::max<long long>(ptop, 1) * nrhs * 16, st));
  CKB(cudaMemcpyAsync(x, x_host, n * nrhs * 16, cudaMemcpyHostToDevice, st));
  CKB(cudaMemsetAsync(y, 0, n * nrhs * 16, st));
  CKB(cudaMemsetAsync(yh, 0, std::max<long long>(top, 1) * nrhs * 16, st));
  const int ldh = static_cast<int>(std::max<long long>(top, 1));
  std::vector<void*> tmp;
  auto run_g = [&](const std::vector<GemmDesc>& g) {
    if (g.empty()) return;
    GemmDesc* d = dev_upload(g, st);
    launch_gemm(d, static_cast<int>(g.size()), st);
    tmp.push_back(d);
  };
  auto run_c = [&](const std::vector<CopyDesc>& c) {
    if (c.empty()) return;
    CopyDesc* d = dev_upload(c, st);
    launch_copy(d, static_cast<int>(c.size()), st);
    tmp.push_back(d);
  };
  // upward: xhat = B^T x (plain transpose, h2_matrix.hpp:88-103)
  for (int l = L; l >= 0; --l) {
    std::vector<GemmDesc> g1, g2;
    for (int id = Structure::first(l); id < Structure::first(l + 1); ++id) {
      const int k = static_cast<int>(basis_rank[id]);
      if (!k) continue;
      const cplx* B = basis + basis_off[id];
      const int rows = static_cast<int>(basis_rows[id]);
      if (l == L) {
        g1.push_back({B, x + S.begin[id], xh + hoff[id], rows, (int)n, ldh, k, nrhs, rows, OP_T, OP_N, 1.0, 0.0});
      } else {
        const int c1 = 2 * id + 1, c2 = 2 * id + 2;
        const int k1 = static_cast<int>(basis_rank[c1]), k2 = static_cast<int>(basis_rank[c2]);
        if (k1) g1.push_back({B, xh + hoff[c1], xh + hoff[id], rows, ldh, ldh, k, nrhs, k1, OP_T, OP_N, 1.0, 0.0});
        if (k2) g2.push_back({B + k1, xh + hoff[c2], xh + hoff[id], rows, ldh, ldh, k, nrhs, k2, OP_T, OP_N, 1.0, k1 ? 1.0 : 0.0});
        if (!k1 && !k2) {
          std::vector<CopyDesc> z{{nullptr, xh + hoff[id], 0, ldh, k, nrhs, 0, 0}};
          run_c(z);
        }
      }
    }
    run_g(g1);
    run_g(g2);
  }
  // couplings: yhat[row] += S xhat[col], rounds by position within the row
  for (int l = 0; l <= L; ++l) {
    const auto& adm = S.adm[l];
    std::vector<std::vector<GemmDesc>> rounds;
    int prev = -1, r = 0;
    for (size_t p = 0; p < adm.size(); ++p) {
      r = adm[p].row == prev ? r + 1 : 0;
      prev = adm[p].row;
      const int kt = static_cast<int>(basis_rank[adm[p].row]), ks = static_cast<int>(basis_rank[adm[p].col]);
      if (!kt || !ks) continue;
      if ((int)rounds.size() <= r) rounds.resize(r + 1);
      rounds[r].push_back({coup + coup_off[S.adm_offset[l] + p], xh + hoff[adm[p].col], yh + hoff[adm[p].row], kt, ldh, ldh, kt, nrhs, ks, OP_N, OP_N,
                           1.0, 1.0});
    }
    for (auto& g : rounds) run_g(g);
  }
  // downward (h2_matrix.hpp:115-129)
  for (int l = 0; l <= L; ++l) {
    std::vector<GemmDesc> g;
    std::vector<CopyDesc> c;
    for (int id = Structure::first(l); id < Structure::first(l + 1); ++id) {
      const int k = static_cast<int>(basis_rank[id]);
      if (!k) continue;
      const cplx* B = basis + basis_off[id];
      const int rows = static_cast<int>(basis_rows[id]);
      if (l == L) {
        g.push_back({B, yh + hoff[id], y + S.begin[id], rows, ldh, (int)n, rows, nrhs, k, OP_N, OP_N, 1.0, 1.0});
      } else {
        const int pl = static_cast<int>(std::max<long long>(ptop, 1));
        g.push_back({B, yh + hoff[id], push + poff[id], rows, ldh, pl, rows, nrhs, k, OP_N, OP_N, 1.0, 0.0});
        const int c1 = 2 * id + 1, c2 = 2 * id + 2;
        const int k1 = static_cast<int>(basis_rank[c1]), k2 = static_cast<int>(basis_rank[c2]);
        if (k1) c.push_back({push + poff[id], yh + hoff[c1], pl, ldh, k1, nrhs, 1, 0});
        if (k2) c.push_back({push + poff[id] + k1, yh + hoff[c2], pl, ldh, k2, nrhs, 1, 0});
      }
    }
    run_g(g);
    run_c(c);
  }
  // dense leaf blocks, rounds by position within the row
  {
    std::vector<std::vector<GemmDesc>> rounds;
    int prev = -1, r = 0;
    for (size_t p = 0; p < S.leaf.size(); ++p) {
      r = S.leaf[p].row == prev ? r + 1 : 0;
      prev = S.leaf[p].row;
      const int t = S.leaf[p].row, s = S.leaf[p].col;
      const int m = static_cast<int>(S.end[t] - S.begin[t]), k = static_cast<int>(S.end[s] - S.begin[s]);
      if ((int)rounds.size() <= r) rounds.resize(r + 1);
      rounds[r].push_back({dense + dense_off[p], x + S.begin[s], y + S.begin[t], m, (int)n, (int)n, m, nrhs, k, OP_N, OP_N, 1.0, 1.0});
    }
    for (auto& g : rounds) run_g(g);
  }
  CKB(cudaGetLastError());
  CKB(cudaMemcpyAsync(y_host, y, n * nrhs * 16, cudaMemcpyDeviceToHost, st));
  CKB(cudaStreamSynchronize(st));
  for (void* p : tmp) cudaFreeAsync(p, st);
  for (void* p : {(void*)x, (void*)y, (void*)xh, (void*)yh, (void*)push}) cudaFreeAsync(p, st);
}

// ------------------------------------------------- sampled dense rows
// y[q] = sum_j Z(rows[q], j) x[j] with Z generated from the kernel (the
// north_star's dense sampled-row residual; the reference's
// assemble_block, kernel.hpp:64-102). One CTA per sampled row; each thread
// strides the columns, then a fixed-order tree reduction (deterministic).
__global__ void __launch_bounds__(256) k_rows_matvec(KernelD K, const double* px, const double* py, const double* pz, long long n,
                                                      const long long* rows, const cplx* x, int nrhs, long long ldx, cplx* y, long long ldy) {
  __shared__ cplx red[256];
  const long long r = rows[blockIdx.x];
  for (int c = 0; c < nrhs; ++c) {
    cplx s = czero();
    const cplx* xc = x + (size_t)c * ldx;
    for (long long j = threadIdx.x; j < n; j += blockDim.x) cfma(s, kentry(K, px, py, pz, r, j), xc[j]);
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
      if (threadIdx.x < w) red[threadIdx.x] = cadd(red[threadIdx.x], red[threadIdx.x + w]);
      __syncthreads();
    }
    if (threadIdx.x == 0) y[blockIdx.x + (size_t)c * ldy] = red[0];
    __syncthreads();
  }
}

void kernel_rows_matvec_device(const double* points_tree, int64_t n, const h2g_kernel_spec& Ks, const int64_t* rows, int64_t nrows,
                               const double* x_host, double* y_host, int nrhs, cudaStream_t st) {
  KernelD K{Ks.kind, Ks.wavenumber_re, Ks.wavenumber_im, Ks.scale_re, Ks.scale_im, Ks.diag_re, Ks.diag_im};
  std::vector<double> hx(n), hy(n), hz(n);
  for (int64_t i = 0; i < n; ++i) hx[i] = points_tree[3 * i], hy[i] = points_tree[3 * i + 1], hz[i] = points_tree[3 * i + 2];
  for (int64_t q = 0; q < nrows; ++q)
    if (rows[q] < 0 || rows[q] >= n) throw std::invalid_argument("kernel_rows_matvec: row index out of range");
  std::vector<long long> hr(rows, rows + nrows);
  double* px = dev_upload(hx, st);
  double* py = dev_upload(hy, st);
  double* pz = dev_upload(hz, st);
  long long* dr = dev_upload(hr, st);
  cplx *x = nullptr, *y = nullptr;
  CKB(cudaMallocAsync(&x, (size_t)n * nrhs * 16, st));
  CKB(cudaMallocAsync(&y, (size_t)std::max<int64_t>(nrows, 1) * nrhs * 16, st));
  CKB(cudaMemcpyAsync(x, x_host, (size_t)n * nrhs * 16, cudaMemcpyHostToDevice, st));
  if (nrows) k_rows_matvec<<<static_cast<unsigned>(nrows), 256, 0, st>>>(K, px, py, pz, n, dr, x, nrhs, n, y, nrows);
  CKB(cudaGetLastError());
  if (nrows) CKB(cudaMemcpyAsync(y_host, y, (size_t)nrows * nrhs * 16, cudaMemcpyDeviceToHost, st));
  CKB(cudaStreamSynchronize(st));
  for (void* p : {(void*)px, (void*)py, (void*)pz, (void*)dr, (void*)x, (void*)y}) cudaFreeAsync(p, st);
}

}  // namespace h2g
