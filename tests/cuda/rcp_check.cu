// Accuracy of rcp_nr (rcp.approx.ftz.f64 + 2 Newton steps) against 1.0 / q.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "../../paper_1703_06155_b200/csrc/device.cuh"
using namespace h2g;
__global__ void k(const double* q, double* err, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const double a = rcp_nr(q[i]), b = 1.0 / q[i];
    err[i] = fabs(a - b) / fabs(b);
  }
}
int main() {
  const int n = 1 << 20;
  double* h = (double*)malloc(n * 8);
  srand(1);
  for (int i = 0; i < n; ++i) {
    double m = (rand() + 1.0) / RAND_MAX, e = (rand() % 1200) - 600;
    h[i] = (i & 1 ? -1 : 1) * m * pow(2.0, e);
  }
  double *dq, *de;
  cudaMalloc(&dq, n * 8);
  cudaMalloc(&de, n * 8);
  cudaMemcpy(dq, h, n * 8, cudaMemcpyHostToDevice);
  k<<<n / 256, 256>>>(dq, de, n);
  cudaMemcpy(h, de, n * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < n; ++i) mx = fmax(mx, h[i]);
  printf("rcp_nr max relative error %.3e (ulp %.2f)\n", mx, mx / 2.220446049250313e-16);
  return 0;
}
