// multisect_top (grouped multisection) against bisect_eig on random
// tridiagonals of several sizes / retained counts.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../../paper_1703_06155_b200/csrc/device.cuh"
using namespace h2g;
__global__ void k(int n, int r, const double* d, const double* e, double lo, double hi, double piv, double* o1, double* o2) {
  __shared__ double sd[512], se[512], se2[512];
  for (int i = threadIdx.x; i < n; i += blockDim.x) sd[i] = d[i], se[i] = e[i], se2[i] = e[i] * e[i];
  __syncthreads();
  multisect_top(n, sd, se2, r, lo, hi, piv, o1);
  for (int j = threadIdx.x; j < r; j += blockDim.x) o2[j] = bisect_eig(n, sd, se, n - 1 - j, lo, hi, piv);
}
int main() {
  srand(3);
  int sizes[] = {5, 15, 31, 64, 100, 130, 200, 300};
  double worst = 0;
  for (int n : sizes)
    for (int r : {1, 3, 8, 17, 40, 100, 129, 250, 300}) {
      if (r > n) continue;
      std::vector<double> d(n), e(n, 0.0);
      for (int i = 0; i < n; ++i) d[i] = pow(10.0, -8.0 * rand() / RAND_MAX);
      for (int i = 0; i + 1 < n; ++i) e[i] = 1e-3 * (rand() / (double)RAND_MAX - 0.5);
      double lo = 1e300, hi = -1e300;
      for (int i = 0; i < n; ++i) {
        double off = (i ? fabs(e[i - 1]) : 0) + (i + 1 < n ? fabs(e[i]) : 0);
        lo = fmin(lo, d[i] - off), hi = fmax(hi, d[i] + off);
      }
      double *dd, *de, *o1, *o2;
      cudaMalloc(&dd, n * 8); cudaMalloc(&de, n * 8); cudaMalloc(&o1, n * 8); cudaMalloc(&o2, n * 8);
      cudaMemcpy(dd, d.data(), n * 8, cudaMemcpyHostToDevice);
      cudaMemcpy(de, e.data(), n * 8, cudaMemcpyHostToDevice);
      k<<<1, 256>>>(n, r, dd, de, lo, hi, 2.2250738585072014e-308, o1, o2);
      std::vector<double> a(r), b(r);
      cudaMemcpy(a.data(), o1, r * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(b.data(), o2, r * 8, cudaMemcpyDeviceToHost);
      double w = 0;
      for (int j = 0; j < r; ++j) w = fmax(w, fabs(a[j] - b[j]) / fmax(fabs(b[j]), 1e-300));
      printf("n %3d r %3d max rel diff %.3e  (top %.6e vs %.6e, last %.6e vs %.6e)\n", n, r, w, a[0], b[0], a[r - 1], b[r - 1]);
      worst = fmax(worst, w);
      cudaFree(dd); cudaFree(de); cudaFree(o1); cudaFree(o2);
    }
  printf("worst %.3e %s\n", worst, cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
