// Device H² construction (build_h2, proj/include/h2lu/h2_matrix.hpp:300-375)
// and the compressed matvec (h2_matrix.hpp:80-137).
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "../../include/h2g.h"
#include "device.cuh"
#include "plan.hpp"

namespace h2g {

struct BuildResult {
  std::vector<int64_t> basis_rows, basis_rank, basis_off, coup_off, dense_off;
  int64_t basis_elems = 0, coup_elems = 0, dense_elems = 0;
  void* basis = nullptr;  // device, cudaMallocAsync on the stream
  void* coup = nullptr;
  void* dense = nullptr;
};

BuildResult build_h2_device(const Structure& S, const double* points, const std::vector<int64_t>& perm, const h2g_kernel_spec& K,
                            double eps_h2, cudaStream_t s);

void matvec_device(const Structure& S, const std::vector<int64_t>& basis_rows, const std::vector<int64_t>& basis_rank,
                   const std::vector<int64_t>& basis_off, const std::vector<int64_t>& coup_off, const std::vector<int64_t>& dense_off,
                   const cplx* basis, const cplx* coup, const cplx* dense, const double* x_host, double* y_host, int nrhs, cudaStream_t s);

// Dense kernel rows times x (tree order points, n x 3 row-major): the sampled
// dense residual of the north_star.
void kernel_rows_matvec_device(const double* points_tree, int64_t n, const h2g_kernel_spec& K, const int64_t* rows, int64_t nrows,
                               const double* x_host, double* y_host, int nrhs, cudaStream_t s);

}  // namespace h2g
