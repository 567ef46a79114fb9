// Micro-benchmark of CTA-tile ZGEMM variants on sm_100a (complex128):
// C (M x N) = A (M x K) B (K x N), one CTA per output tile, vs the FP64 peak.
#include <cstdio>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>

#include "../../paper_1703_06155_b200/csrc/device.cuh"

using namespace h2g;

// V1: the library's tile (64x64, 4x4 micro, sA[64][17] / sB[16][65]).
__global__ void __launch_bounds__(256) v1(int M, int N, int K, const cplx* A, const cplx* B, cplx* C) {
  __shared__ cplx sm[kTileSmemCplx];
  const int r0 = blockIdx.x * 64, c0 = blockIdx.y * 64;
  cta_gemm_tiled(min(64, M - r0), min(64, N - c0), K, 1.0, A + r0, M, OP_N, B + (size_t)c0 * K, K, OP_N, 0.0, C + r0 + (size_t)c0 * M, M, sm);
}

// V3: 64x64 tile, 128 threads, 8x4 micro-tile, k-major smem (sA[k][i], sB[k][j]),
// double-buffered K chunks of 16.
__global__ void __launch_bounds__(128) v3(int M, int N, int K, const cplx* A, const cplx* B, cplx* C) {
  __shared__ __align__(16) cplx sA[2][8][64];
  __shared__ __align__(16) cplx sB[2][8][64];
  const int r0 = blockIdx.x * 64, c0 = blockIdx.y * 64;
  const int tr = threadIdx.x % 8, tc = threadIdx.x / 8;  // rows tr*8.., cols tc*4..
  cplx acc[8][4];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = czero();
  auto load = [&](int buf, int k0) {
    for (int idx = threadIdx.x; idx < 64 * 8; idx += 128) {
      const int i = idx % 64, p = idx / 64;
      sA[buf][p][i] = (k0 + p < K) ? A[r0 + i + (size_t)(k0 + p) * M] : czero();
      const int q = idx % 8, j = idx / 8;
      sB[buf][q][j] = (k0 + q < K) ? B[k0 + q + (size_t)(c0 + j) * K] : czero();
    }
  };
  load(0, 0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < K; k0 += 8) {
    if (k0 + 8 < K) load(buf ^ 1, k0 + 8);
#pragma unroll 4
    for (int p = 0; p < 8; ++p) {
      cplx av[8], bv[4];
#pragma unroll
      for (int a = 0; a < 8; ++a) av[a] = sA[buf][p][tr * 8 + a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = sB[buf][p][tc * 4 + b];
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) cfma(acc[a][b], av[a], bv[b]);
    }
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) C[r0 + tr * 8 + a + (size_t)(c0 + tc * 4 + b) * M] = acc[a][b];
}

// V4: like V3 but the 8 rows of a thread are strided by 8 (tr + 8a) so a warp's
// A reads hit distinct banks, and B reads broadcast.
__global__ void __launch_bounds__(128) v4(int M, int N, int K, const cplx* A, const cplx* B, cplx* C) {
  __shared__ __align__(16) cplx sA[2][8][64];
  __shared__ __align__(16) cplx sB[2][8][64];
  const int r0 = blockIdx.x * 64, c0 = blockIdx.y * 64;
  const int tr = threadIdx.x % 8, tc = threadIdx.x / 8;
  cplx acc[8][4];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = czero();
  auto load = [&](int buf, int k0) {
    for (int idx = threadIdx.x; idx < 64 * 8; idx += 128) {
      const int i = idx % 64, p = idx / 64;
      sA[buf][p][i] = (k0 + p < K) ? A[r0 + i + (size_t)(k0 + p) * M] : czero();
      const int q = idx % 8, j = idx / 8;
      sB[buf][q][j] = (k0 + q < K) ? B[k0 + q + (size_t)(c0 + j) * K] : czero();
    }
  };
  load(0, 0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < K; k0 += 8) {
    if (k0 + 8 < K) load(buf ^ 1, k0 + 8);
#pragma unroll 4
    for (int p = 0; p < 8; ++p) {
      cplx av[8], bv[4];
#pragma unroll
      for (int a = 0; a < 8; ++a) av[a] = sA[buf][p][tr + 8 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = sB[buf][p][tc * 4 + b];
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) cfma(acc[a][b], av[a], bv[b]);
    }
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) C[r0 + tr + 8 * a + (size_t)(c0 + tc * 4 + b) * M] = acc[a][b];
}

// V5: DMMA (mma.sync m8n8k4 f64) on split real/imag planes. 64x64 CTA tile,
// 4 warps each 32x32 complex (4x4 m8n8 tiles), K chunks of 8 double-buffered.
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__global__ void __launch_bounds__(128) v5(int M, int N, int K, const cplx* A, const cplx* B, cplx* C) {
  __shared__ __align__(16) double sAr[2][8][64], sAi[2][8][64], sBr[2][8][64], sBi[2][8][64];
  const int r0 = blockIdx.x * 64, c0 = blockIdx.y * 64;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int wr = (warp % 2) * 32, wc = (warp / 2) * 32;
  const int g = lane / 4, tq = lane % 4;
  double re[4][4][2], im[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) re[a][b][0] = re[a][b][1] = im[a][b][0] = im[a][b][1] = 0.0;
  auto load = [&](int buf, int k0) {
    for (int idx = threadIdx.x; idx < 64 * 8; idx += 128) {
      const int i = idx % 64, p = idx / 64;
      const cplx a = (k0 + p < K) ? A[r0 + i + (size_t)(k0 + p) * M] : czero();
      sAr[buf][p][i] = a.x;
      sAi[buf][p][i] = a.y;
      const int q = idx % 8, j = idx / 8;
      const cplx bb = (k0 + q < K) ? B[k0 + q + (size_t)(c0 + j) * K] : czero();
      sBr[buf][q][j] = bb.x;
      sBi[buf][q][j] = bb.y;
    }
  };
  load(0, 0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < K; k0 += 8) {
    if (k0 + 8 < K) load(buf ^ 1, k0 + 8);
#pragma unroll
    for (int kk = 0; kk < 8; kk += 4) {
      double ar[4], ai[4], br[4], bi[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        ar[mi] = sAr[buf][kk + tq][wr + mi * 8 + g];
        ai[mi] = sAi[buf][kk + tq][wr + mi * 8 + g];
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        br[ni] = sBr[buf][kk + tq][wc + ni * 8 + g];
        bi[ni] = sBi[buf][kk + tq][wc + ni * 8 + g];
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
          dmma(re[mi][ni][0], re[mi][ni][1], ar[mi], br[ni]);
          dmma(re[mi][ni][0], re[mi][ni][1], -ai[mi], bi[ni]);
          dmma(im[mi][ni][0], im[mi][ni][1], ar[mi], bi[ni]);
          dmma(im[mi][ni][0], im[mi][ni][1], ai[mi], br[ni]);
        }
    }
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = r0 + wr + mi * 8 + g, col = c0 + wc + ni * 8 + tq * 2 + h;
        C[row + (size_t)col * M] = make_double2(re[mi][ni][h], im[mi][ni][h]);
      }
}

// V6: V4 + cp.async multi-stage (STG stages of K=8) staging, zero-fill via src-size 0.
__device__ __forceinline__ void cp16(void* smem, const void* g, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(g), "r"(sz));
}
template <int STG>
__global__ void __launch_bounds__(128) v6(int M, int N, int K, const cplx* A, const cplx* B, cplx* C) {
  extern __shared__ __align__(16) unsigned char raw[];
  cplx(*sA)[8][64] = reinterpret_cast<cplx(*)[8][64]>(raw);
  cplx(*sB)[8][64] = reinterpret_cast<cplx(*)[8][64]>(raw + STG * 8 * 64 * 16);
  const int r0 = blockIdx.x * 64, c0 = blockIdx.y * 64;
  const int tr = threadIdx.x % 8, tc = threadIdx.x / 8;
  cplx acc[8][4];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = czero();
  const int nk = (K + 7) / 8;
  auto load = [&](int st, int kc) {
    const int k0 = kc * 8;
    for (int idx = threadIdx.x; idx < 64 * 8; idx += 128) {
      const int i = idx % 64, p = idx / 64;
      const bool va = k0 + p < K;
      cp16(&sA[st][p][i], A + r0 + i + (size_t)(va ? k0 + p : 0) * M, va);
      const int q = idx % 8, j = idx / 8;
      const bool vb = k0 + q < K;
      cp16(&sB[st][q][j], B + (vb ? k0 + q : 0) + (size_t)(c0 + j) * K, vb);
    }
    asm volatile("cp.async.commit_group;");
  };
  for (int s = 0; s < STG - 1; ++s) {
    if (s < nk) load(s, s);
    else asm volatile("cp.async.commit_group;");
  }
  for (int kc = 0; kc < nk; ++kc) {
    asm volatile("cp.async.wait_group %0;" ::"n"(STG - 2));
    __syncthreads();
    const int st = kc % STG;
    const int nxt = kc + STG - 1;
    if (nxt < nk) load(nxt % STG, nxt);
    else asm volatile("cp.async.commit_group;");
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      cplx av[8], bv[4];
#pragma unroll
      for (int a = 0; a < 8; ++a) av[a] = sA[st][p][tr + 8 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = sB[st][p][tc * 4 + b];
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) cfma(acc[a][b], av[a], bv[b]);
    }
  }
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) C[r0 + tr + 8 * a + (size_t)(c0 + tc * 4 + b) * M] = acc[a][b];
}

// V7: DMMA m8n8k4 on interleaved complex k-slices staged by a 3-stage cp.async
// pipeline (padded rows); 4 warps, each a 32x32 complex warp tile (4x4 m8n8
// tiles, re/im accumulators).
template <int STG>
__global__ void __launch_bounds__(128) v7(int M, int N, int K, const cplx* A, const cplx* B, cplx* C) {
  extern __shared__ __align__(16) unsigned char raw[];
  cplx(*sA)[8][65] = reinterpret_cast<cplx(*)[8][65]>(raw);
  cplx(*sB)[8][65] = reinterpret_cast<cplx(*)[8][65]>(raw + STG * 8 * 65 * 16);
  const int r0 = blockIdx.x * 64, c0 = blockIdx.y * 64;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int wr = (warp % 2) * 32, wc = (warp / 2) * 32;
  const int g = lane / 4, tq = lane % 4;
  double re[4][4][2], im[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) re[a][b][0] = re[a][b][1] = im[a][b][0] = im[a][b][1] = 0.0;
  const int nk = (K + 7) / 8;
  auto load = [&](int st, int kc) {
    const int k0 = kc * 8;
    for (int idx = threadIdx.x; idx < 64 * 8; idx += 128) {
      const int i = idx % 64, p = idx / 64;
      const bool va = k0 + p < K;
      cp16(&sA[st][p][i], A + r0 + i + (size_t)(va ? k0 + p : 0) * M, va);
      const int q = idx % 8, j = idx / 8;
      const bool vb = k0 + q < K;
      cp16(&sB[st][q][j], B + (vb ? k0 + q : 0) + (size_t)(c0 + j) * K, vb);
    }
    asm volatile("cp.async.commit_group;");
  };
  for (int s = 0; s < STG - 1; ++s) {
    if (s < nk) load(s, s);
    else asm volatile("cp.async.commit_group;");
  }
  for (int kc = 0; kc < nk; ++kc) {
    asm volatile("cp.async.wait_group %0;" ::"n"(STG - 2));
    __syncthreads();
    const int st = kc % STG;
    const int nxt = kc + STG - 1;
    if (nxt < nk) load(nxt % STG, nxt);
    else asm volatile("cp.async.commit_group;");
#pragma unroll
    for (int kk = 0; kk < 8; kk += 4) {
      cplx af[4], bf[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) af[mi] = sA[st][kk + tq][wr + mi * 8 + g];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) bf[ni] = sB[st][kk + tq][wc + ni * 8 + g];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
          dmma(re[mi][ni][0], re[mi][ni][1], af[mi].x, bf[ni].x);
          dmma(re[mi][ni][0], re[mi][ni][1], -af[mi].y, bf[ni].y);
          dmma(im[mi][ni][0], im[mi][ni][1], af[mi].x, bf[ni].y);
          dmma(im[mi][ni][0], im[mi][ni][1], af[mi].y, bf[ni].x);
        }
    }
  }
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = r0 + wr + mi * 8 + g, col = c0 + wc + ni * 8 + tq * 2 + h;
        C[row + (size_t)col * M] = make_double2(re[mi][ni][h], im[mi][ni][h]);
      }
}

int main() {
  const int M = 4096, N = 4096, K = 512;
  cplx *A, *B, *C;
  cudaMalloc(&A, (size_t)M * K * 16);
  cudaMalloc(&B, (size_t)K * N * 16);
  cudaMalloc(&C, (size_t)M * N * 16);
  cudaMemset(A, 0, (size_t)M * K * 16);
  cudaMemset(B, 0, (size_t)K * N * 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaFuncSetAttribute((const void*)v1, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  dim3 g(M / 64, N / 64);
  const double flops = 8.0 * M * N * K;
  cudaFuncSetAttribute((const void*)v6<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 2 * 8 * 64 * 16);
  cudaFuncSetAttribute((const void*)v6<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 2 * 8 * 64 * 16);
  cudaFuncSetAttribute((const void*)v6<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 2 * 8 * 64 * 16);
  cudaFuncSetAttribute((const void*)v7<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 2 * 8 * 65 * 16);
  cudaFuncSetAttribute((const void*)v7<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 2 * 8 * 65 * 16);
  for (int v = 1; v <= 9; ++v) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (v == 1) v1<<<g, 256>>>(M, N, K, A, B, C);
      if (v == 2) v3<<<g, 128>>>(M, N, K, A, B, C);
      if (v == 3) v4<<<g, 128>>>(M, N, K, A, B, C);
      if (v == 4) v5<<<g, 128>>>(M, N, K, A, B, C);
      if (v == 5) v6<3><<<g, 128, 3 * 2 * 8 * 64 * 16>>>(M, N, K, A, B, C);
      if (v == 6) v6<4><<<g, 128, 4 * 2 * 8 * 64 * 16>>>(M, N, K, A, B, C);
      if (v == 7) v6<6><<<g, 128, 6 * 2 * 8 * 64 * 16>>>(M, N, K, A, B, C);
      if (v == 8) v7<3><<<g, 128, 3 * 2 * 8 * 65 * 16>>>(M, N, K, A, B, C);
      if (v == 9) v7<4><<<g, 128, 4 * 2 * 8 * 65 * 16>>>(M, N, K, A, B, C);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2) printf("variant %d: %.3f ms  %.2f TFLOP/s  (%s)\n", v, ms, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  // correctness: random A, B; compare v5 with v4
  {
    std::vector<double> h((size_t)M * K * 2), hb((size_t)K * N * 2);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)((i * 2654435761u) % 1000) / 1000.0 - 0.5;
    for (size_t i = 0; i < hb.size(); ++i) hb[i] = (double)((i * 40503u) % 997) / 997.0 - 0.5;
    cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(B, hb.data(), hb.size() * 8, cudaMemcpyHostToDevice);
    cplx* C2;
    cudaMalloc(&C2, (size_t)M * N * 16);
    v4<<<g, 128>>>(M, N, K, A, B, C);
    v7<3><<<g, 128, 3 * 2 * 8 * 65 * 16>>>(M, N, K, A, B, C2);
    std::vector<double> c1((size_t)M * N * 2), c2((size_t)M * N * 2);
    cudaMemcpy(c1.data(), C, c1.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(c2.data(), C2, c2.size() * 8, cudaMemcpyDeviceToHost);
    double md = 0, mx = 0;
    for (size_t i = 0; i < c1.size(); ++i) md = fmax(md, fabs(c1[i] - c2[i])), mx = fmax(mx, fabs(c1[i]));
    printf("v7 vs v4 max abs diff %.3e (max %.3e)\n", md, mx);
  }
  return 0;
}
