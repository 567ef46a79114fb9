// Unit harness for the CTA-level dense routines of csrc/device.cuh: each
// entry point runs one routine in one CTA on host-provided data (test-only
// library libh2g_selftest.so; the product is libh2g.so).
#include <cuda_runtime.h>

#include "../../paper_1703_06155_b200/csrc/device.cuh"

using namespace h2g;

__global__ void kt_householder(cplx* A, int m, int k, cplx* Q, cplx* tau) {
  __shared__ double red[32];
  cta_householder_q(m, k, A, m, Q, m, tau, red);
}

__global__ void kt_jacobi(cplx* H, cplx* U, int n, double* rot, int* pr) {
  __shared__ double red[32];
  cta_jacobi_eig(n, H, U, rot, pr, red);
}

__global__ void kt_lu(cplx* A, int n, int* fail, double* mag, cplx* Li, cplx* Ui) {
  __shared__ double red[32];
  double pm = 0.0;
  const int f = cta_lu_nopiv(n, A, n, 1e-13, &pm, red);
  if (threadIdx.x == 0) *fail = f, *mag = pm;
  __syncthreads();
  if (f < 0) cta_tri_inverses(n, A, n, Li, Ui);
}

__global__ void kt_gemm(int m, int n, int k, const cplx* A, int lda, int opA, const cplx* B, int ldb, int opB, cplx* C) {
  cta_gemm(m, n, k, 1.0, A, lda, opA, B, ldb, opB, 0.0, C, m);
}

template <class T>
static T* up(const void* h, size_t bytes) {
  T* d = nullptr;
  cudaMalloc(&d, bytes ? bytes : 16);
  if (h && bytes) cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice);
  return d;
}

extern "C" {
int st_householder(double* V, int m, int k, double* Q) {
  cplx* dA = up<cplx>(V, (size_t)m * k * 16);
  cplx* dQ = up<cplx>(nullptr, (size_t)m * m * 16);
  cplx* dt = up<cplx>(nullptr, (size_t)(k + 1) * 16);
  kt_householder<<<1, 256>>>(dA, m, k, dQ, dt);
  cudaMemcpy(Q, dQ, (size_t)m * m * 16, cudaMemcpyDeviceToHost);
  cudaMemcpy(V, dA, (size_t)m * k * 16, cudaMemcpyDeviceToHost);
  cudaFree(dA), cudaFree(dQ), cudaFree(dt);
  return (int)cudaDeviceSynchronize();
}
int st_jacobi(double* H, int n, double* U) {
  cplx* dH = up<cplx>(H, (size_t)n * n * 16);
  cplx* dU = up<cplx>(nullptr, (size_t)n * n * 16);
  double* rot = up<double>(nullptr, (size_t)4 * (n / 2 + 1) * 8);
  int* pr = up<int>(nullptr, (size_t)(n + 2) * 4);
  kt_jacobi<<<1, 256>>>(dH, dU, n, rot, pr);
  cudaMemcpy(H, dH, (size_t)n * n * 16, cudaMemcpyDeviceToHost);
  cudaMemcpy(U, dU, (size_t)n * n * 16, cudaMemcpyDeviceToHost);
  cudaFree(dH), cudaFree(dU), cudaFree(rot), cudaFree(pr);
  return (int)cudaDeviceSynchronize();
}
int st_lu(double* A, int n, double* Li, double* Ui, int* fail, double* mag) {
  cplx* dA = up<cplx>(A, (size_t)n * n * 16);
  cplx* dL = up<cplx>(nullptr, (size_t)n * n * 16);
  cplx* dU = up<cplx>(nullptr, (size_t)n * n * 16);
  int* df = up<int>(nullptr, 4);
  double* dm = up<double>(nullptr, 8);
  kt_lu<<<1, 256>>>(dA, n, df, dm, dL, dU);
  cudaMemcpy(A, dA, (size_t)n * n * 16, cudaMemcpyDeviceToHost);
  cudaMemcpy(Li, dL, (size_t)n * n * 16, cudaMemcpyDeviceToHost);
  cudaMemcpy(Ui, dU, (size_t)n * n * 16, cudaMemcpyDeviceToHost);
  cudaMemcpy(fail, df, 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(mag, dm, 8, cudaMemcpyDeviceToHost);
  cudaFree(dA), cudaFree(dL), cudaFree(dU), cudaFree(df), cudaFree(dm);
  return (int)cudaDeviceSynchronize();
}
int st_gemm(int m, int n, int k, const double* A, int lda, int opA, const double* B, int ldb, int opB, double* C) {
  const size_t sa = (size_t)lda * (opA == 0 || opA == 3 ? k : m), sb = (size_t)ldb * (opB == 0 || opB == 3 ? n : k);
  cplx* dA = up<cplx>(A, sa * 16);
  cplx* dB = up<cplx>(B, sb * 16);
  cplx* dC = up<cplx>(nullptr, (size_t)m * n * 16);
  kt_gemm<<<1, 256>>>(m, n, k, dA, lda, opA, dB, ldb, opB, dC);
  cudaMemcpy(C, dC, (size_t)m * n * 16, cudaMemcpyDeviceToHost);
  cudaFree(dA), cudaFree(dB), cudaFree(dC);
  return (int)cudaDeviceSynchronize();
}
}
