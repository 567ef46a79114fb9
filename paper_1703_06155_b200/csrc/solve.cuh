// Device view of one level of a factor chain for the substitutions (solve.cu).
#pragma once

#include "device.cuh"

namespace h2g {

struct SolveLevel {
  int nl;
  int bmax;
  const int* bsz;
  const long long* pos;
  const int* kfin;
  const int* C_ptr;
  const int* C_nb;
  const cplx* chain;
  const long long* Qt_off;
  const long long* L11_off;
  const long long* U11_off;
  const long long* Linv_off;
  const long long* Uinv_off;
  const long long* Lbar_off;
  const long long* Ubar_off;
  const long long* Lself_off;
  const long long* Uself_off;
};

struct SolveTargetD {
  int seg, c0, c1;
};
struct SolveContribD {
  int m, entry;
};

void launch_fwd_head(const SolveLevel& S, const int* batch_cl, int nb, cplx* y, long long ldy, int nrhs, int explicit_inv, cudaStream_t s);
void launch_fwd_lbar(const SolveLevel& S, const SolveTargetD* t, int nt, const SolveContribD* c, cplx* y, long long ldy, int nrhs, cudaStream_t s);
void launch_bwd(const SolveLevel& S, const int* batch_cl, int nb, int maxc, cplx* y, long long ldy, int nrhs, int explicit_inv, cplx* part,
                cudaStream_t s);
void launch_permute(const long long* src, long long len, cplx* y, cplx* tmp, long long ldy, int nrhs, int scatter, cudaStream_t s);
void launch_root_trsv(const cplx* A, int n, cplx* y, long long ldy, int nrhs, int upper, cudaStream_t s);
void launch_finite(const cplx* y, long long total, int* bad, cudaStream_t s);

}  // namespace h2g
