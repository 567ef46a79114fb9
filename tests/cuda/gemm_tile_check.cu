// Cross-check of the descriptor GEMM tile paths (k_gemm<32> over several
// tiles per descriptor vs k_gemm<64>) on every operand form; prints the
// largest relative difference per case. Build: see the Makefile rule in the
// commit message; run on a B200.
#include "../../paper_1703_06155_b200/csrc/factor.cu"

#include <cstdio>
#include <random>
#include <vector>

using namespace h2g;

int main() {
  std::mt19937_64 rng(7);
  std::normal_distribution<double> g;
  const int dims[3] = {64, 100, 235};
  const int ks[2] = {7, 150};
  double worst = 0.0;
  for (int opA = 0; opA < 4; ++opA)
    for (int opB = 0; opB < 4; ++opB)
      for (int m : dims)
        for (int n : dims)
          for (int k : ks)
            for (int beta = 0; beta < 2; ++beta) {
              const bool at = opA == OP_T || opA == OP_C, bt = opB == OP_T || opB == OP_C;
              const int lda = at ? k : m, ldb = bt ? n : k;
              const size_t na = (size_t)lda * (at ? m : k), nb = (size_t)ldb * (bt ? k : n), nc = (size_t)m * n;
              std::vector<double2> A(na), B(nb), C(nc);
              for (auto& v : A) v = make_double2(g(rng), g(rng));
              for (auto& v : B) v = make_double2(g(rng), g(rng));
              for (auto& v : C) v = make_double2(g(rng), g(rng));
              double2 *dA, *dB, *dC1, *dC2;
              GemmDesc* dd;
              cudaMalloc(&dA, na * 16);
              cudaMalloc(&dB, nb * 16);
              cudaMalloc(&dC1, nc * 16);
              cudaMalloc(&dC2, nc * 16);
              cudaMalloc(&dd, 2 * sizeof(GemmDesc));
              cudaMemcpy(dA, A.data(), na * 16, cudaMemcpyHostToDevice);
              cudaMemcpy(dB, B.data(), nb * 16, cudaMemcpyHostToDevice);
              cudaMemcpy(dC1, C.data(), nc * 16, cudaMemcpyHostToDevice);
              cudaMemcpy(dC2, C.data(), nc * 16, cudaMemcpyHostToDevice);
              GemmDesc d1{dA, dB, dC1, lda, ldb, m, m, n, k, opA, opB, 1.0, beta ? 1.0 : 0.0};
              GemmDesc d2 = d1;
              d2.C = dC2;
              cudaMemcpy(dd, &d1, sizeof(GemmDesc), cudaMemcpyHostToDevice);
              cudaMemcpy(dd + 1, &d2, sizeof(GemmDesc), cudaMemcpyHostToDevice);
              const int maxdim = std::max(m, n);
              const int t32 = (maxdim + 31) / 32;
              launch_gemm_tm<32>(dd, 1, 0, maxdim, t32 * t32);
              launch_gemm_tm<64>(dd + 1, 1, 0, maxdim);
              cudaDeviceSynchronize();
              std::vector<double2> C1(nc), C2(nc);
              cudaMemcpy(C1.data(), dC1, nc * 16, cudaMemcpyDeviceToHost);
              cudaMemcpy(C2.data(), dC2, nc * 16, cudaMemcpyDeviceToHost);
              double num = 0.0, den = 0.0;
              for (size_t i = 0; i < nc; ++i) {
                const double dx = C1[i].x - C2[i].x, dy = C1[i].y - C2[i].y;
                num += dx * dx + dy * dy;
                den += C2[i].x * C2[i].x + C2[i].y * C2[i].y;
              }
              const double rel = std::sqrt(num / (den + 1e-300));
              if (rel > 1e-12) std::printf("MISMATCH opA %d opB %d m %d n %d k %d beta %d rel %.3e\n", opA, opB, m, n, k, beta, rel);
              worst = std::max(worst, rel);
              cudaFree(dA), cudaFree(dB), cudaFree(dC1), cudaFree(dC2), cudaFree(dd);
            }
  std::printf("worst relative difference k_gemm<32> (multi-tile) vs k_gemm<64>: %.3e (%s)\n", worst, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
