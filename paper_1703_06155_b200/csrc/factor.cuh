// Device-side state of one tree level during the factorization and the
// launch entry points of the level kernels (factor.cu).
#pragma once

#include <functional>

#include "device.cuh"

namespace h2g {

struct DevLevel {
  int level;
  int nl;
  int bmax;
  double eps;
  // step 0: a truncation threshold below refine_below * sigma_0 takes the
  // Rayleigh-Ritz refinement pass (the Gram alone resolves sigma down to
  // ~sqrt(m eps_mach) sigma_0); H2G_REFINE_BELOW overrides
  double refine_below;
  const int* bsz;
  const int* pos;
  const int* korig;
  int* kfin;
  // dense blocks, packed (offset D_off[i], rows x cols, ld = rows)
  cplx* D;
  const long long* D_off;
  const int* drow;
  const int* dcol;
  const int* diag_blk;
  // fills, packed (offset F_off[i], ld = rows)
  cplx* F;
  const long long* F_off;
  int* fexists;
  const int* frow;
  const int* fcol;
  // neighbour lists
  const int* R_ptr;
  const int* R_nb;
  const int* C_ptr;
  const int* C_nb;
  const int* G_ptr;
  const int* G_fill;
  const unsigned char* G_tr;
  // level-entry basis V (b x korig) and its complement Vp (b x (b-korig)),
  // stride bmax^2, ld b
  const cplx* V0;
  cplx* Vp;
  // chain storage (complex elements)
  cplx* chain;
  const long long* Qt_off;
  const long long* L11_off;
  const long long* U11_off;
  const long long* Lbar_off;  // per R entry
  const long long* Ubar_off;  // per C entry
  const long long* Lself_off;
  const long long* Uself_off;
  // scratch
  cplx* lift;                 // lifted panels (packed: only entries whose neighbour was eliminated earlier)
  const long long* liftL_off; // per R entry, offset into lift (-1: not lifted)
  const long long* liftU_off; // per C entry
  const long long* Linv_off;  // L11^{-1}, U11^{-1} (e x e) in the chain
  const long long* Uinv_off;
  // step-0 per batch-slot data (indexed by the slot's global position p in
  // the level's batch order, or by the local slot q for scratch)
  const int* slot_g0;          // [p] first Gram partial of the slot
  const int* slot_gn;          // [p] number of partials
  const int* slot_c0;          // [p] first column-norm entry
  const int* slot_cn;          // [p] number of column-norm entries
  const cplx* gram;            // partial Grams (batch-relative offsets, m x m each)
  const long long* gram_off;   // [partial] offset into gram
  const double* colnorm;       // [entry] max column norm of one fill block
  cplx* dir;                   // [q] pass-1 directions D1 = Vp U1 sorted (b x m), stride bmax^2
  double* lam;                 // [q] pass-1 singular values (sorted desc), stride bmax
  int* pass2;                  // [q] 1 if the refinement pass runs
  int* rank1;                  // [q] pass-1 rank (used when pass2 == 0)
  double* cmax;                // [q]
  DevError* err;
  int debug;
  cplx* eigws;  // step-0 eigensolver workspace, eig1_ws_cplx(bmax) per batch slot
  cplx* const* core_ptr; // per fill: its compact core (kfin_j x kfin_c) once collapsed (SchurTarget kind bit 3)
  cplx* scratch;         // level scratch of the head / extended-LU / complement kernels
  size_t scratch_bytes;  // >= level_scratch_bytes(nl, bmax, max batch)
};

struct PanelItemD {
  int q, side, nb, blk, entry, lift;
};
struct SchurTargetD {
  int kind, idx, c0, c1;
};
struct SchurContribD {
  int t, r, c, flags;
};

// Descriptor-driven batched kernels used for merges, root assembly and paints
// (sizes known on the host at level boundaries).
struct CopyDesc {
  const cplx* src;  // nullptr: zero fill
  cplx* dst;
  int lds, ldd, m, n;
  int accumulate;   // dst += src
  int pad;
};
struct GemmDesc {
  const cplx* A;
  const cplx* B;
  cplx* C;
  int lda, ldb, ldc, m, n, k, opA, opB;
  double alpha, beta;
  const int* flag1;  // if set and *flag1 == 0 (or *flag2 == 0): op(A) op(B) counts as zero
  const int* flag2;
  // device-resolved sizes: m += mi * *dyn, n += ni * *dyn, k += ki * *dyn
  const int* dyn;
  int mi, ni, ki;
  int ldneg;  // bits 0/1/2: lda/ldb/ldc -= *dyn
  const int* skipnz;  // if set and *skipnz != 0: the descriptor is skipped (no write)
};
// Masked copy T -> D zeroing the eliminated rows (mode 0) or columns (mode
// 1) of a rotated neighbour block: e = e0 - *kf (cleanup, factorization.hpp:437-438).
struct MaskDesc {
  const cplx* src;
  cplx* dst;
  int ld, m, n, mode, e0, pad;
  const int* kf;
};
struct NormDesc {
  const cplx* F;
  int rows, cols, trans, pad;
  const int* flag;
  double* out;
};

// Multi-GPU exchange (h2g_factorize_dist): contiguous regions moved between
// the level pools and the exchange buffer, and indexed ints (kfin, fexists).
struct MoveDesc {
  const cplx* src;
  cplx* dst;
  long long len;
};
void launch_move(const MoveDesc* d, int n, cudaStream_t s);
// scatter = 0: packed[i] = base[idx[i]]; 1: base[idx[i]] = packed[i]
void launch_int_move(int* base, const int* idx, int n, int* packed, int scatter, cudaStream_t s);

// Bytes of DevLevel::scratch a level with nl clusters, bmax and the given
// largest batch needs.
size_t level_scratch_bytes(int nl, int bmax, int max_batch);
void launch_complement(const DevLevel& L, cudaStream_t s);
void launch_eig1(const DevLevel& L, const int* batch_cl, int p0, int nb, int mmax, cudaStream_t s,
                 const std::function<void(int)>& phase);
size_t eig1_ws_bytes(int bmax);
void launch_head(const DevLevel& L, const int* batch_cl, int p0, int nb, cudaStream_t s);
void launch_colnorm(const NormDesc* d, int n, cudaStream_t s);
void launch_mask(const MaskDesc* d, int n, cudaStream_t s);
// emax: upper bound of the batch's eliminated sizes (b - korig); > 64 takes
// the multi-CTA extended LU
void launch_head2(const DevLevel& L, const int* batch_cl, int nb, int emax, cudaStream_t s);
// Resolved Schur descriptors of one batch (k_schur_resolve, one thread per
// target): what a k_schur CTA would otherwise find through two chains of
// dependent index loads. rp is indexed by the global contribution index.
struct RTarget {
  cplx* out;
  int rows, cols, rs, cs, ldo, pad;
};
struct RPanel {
  const cplx* A;
  const cplx* B;
  int arows, bcols, ro, co, e, pad;
};
void launch_schur_resolve(const DevLevel& L, const SchurTargetD* targets, int ntargets, const SchurContribD* contrib, RTarget* rt, RPanel* rp,
                          cudaStream_t s);
// rt / rp: resolved descriptors of these targets (nullptr: resolved inside the kernel)
void launch_schur(const DevLevel& L, const SchurTargetD* targets, int ntargets, const SchurContribD* contrib, cudaStream_t s,
                  const RTarget* rt = nullptr, const RPanel* rp = nullptr);
void launch_copy(const CopyDesc* d, int n, cudaStream_t s);
// tiles: upper bound on 64 x 64 output tiles per descriptor (CTAs per desc, capped)
void launch_gemm(const GemmDesc* d, int n, cudaStream_t s, int maxdim = 0);
// Step-0 refinement pass (k_eig1_refine, pass-2 Gram) reachable only for eps < 1e-4.
// Default of DevLevel::refine_below. The Gram G = Y Y^H resolves singular
// values down to ~sqrt(c eps_mach) sigma_0 (c grows with the stack width): at
// eps >= 3e-7 the truncation is decided on the Gram alone (fast cluster
// eigensolver); tighter eps takes the one-CTA Jacobi + Rayleigh-Ritz pass,
// which matches the reference's QR + SVD resolution but is ~70x slower on
// 32^3 unknowns (profiles/r02_refine_switch.txt). H2G_REFINE_BELOW=1e-4
// restores the refinement for every eps < 1e-4.
constexpr double kRefineBelow = 3e-7;
inline bool eig1_refine_possible(const DevLevel& L) { return L.eps < L.refine_below || (L.debug & 4); }
void launch_zero_desc_flags(int* p, int n, cudaStream_t s);
int root_lu(cplx* A, int n, double tol, DevError* err, void* scratch, cudaStream_t s, long long* launches);
size_t head_smem_bytes(int bmax);

}  // namespace h2g
