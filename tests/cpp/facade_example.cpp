// Uses the C++ facade (include/h2lu_gpu.hpp) the way the reference CLI would:
// upload an H2Matrix (here a single dense leaf, depth 0: factorize goes
// straight to the dense root, factorization.hpp:637-651), factorize, solve,
// check A x = b; then check the error mapping (SingularPivotError).
#include <cmath>
#include <cstdio>

#include "h2lu_gpu.hpp"

int main() {
  using namespace h2lu_gpu;
  const int n = 5;
  std::vector<cxd> D(n * n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) D[i + j * n] = i == j ? cxd(4.0, 1.0) : cxd(1.0 / (1 + i + j), 0.1 * (i - j));
  int64_t cb[1] = {0}, ce[1] = {n}, adm_off[2] = {0, 0}, split_off[2] = {0, 0};
  int32_t leaf[2] = {0, 0}, none[2] = {0, 0};
  int64_t brow[1] = {n}, brank[1] = {0}, boff[1] = {0}, coff[1] = {0}, doff[1] = {0};
  double dummy[2] = {0, 0};
  h2g_matrix_desc d{n, 0, 0, 1.0, 1e-8, cb, ce, adm_off, none, split_off, none, 1, leaf, brow, brank, boff, dummy, coff, dummy, doff,
                    reinterpret_cast<const double*>(D.data())};
  try {
    Context ctx(0);
    H2Matrix A(ctx, d);
    FactorChain ch = factorize(A, 1e-8);
    Vec b(n);
    for (int i = 0; i < n; ++i) b[i] = cxd(i + 1.0, -i);
    Vec x = solve(ch, b);
    double err = 0.0;
    for (int i = 0; i < n; ++i) {
      cxd s = 0.0;
      for (int j = 0; j < n; ++j) s += D[i + j * n] * x[j];
      err = std::max(err, std::abs(s - b[i]));
    }
    Vec y = apply_inverse(ch, b);
    bool same = y == x;
    std::printf("facade: root %lld residual %.3e apply_inverse==solve %d\n", (long long)ch.root_size(), err, (int)same);
    // the chain outlives the Context / H2Matrix handles it came from
    FactorChain kept = [&] {
      Context c2(0);
      H2Matrix A2(c2, d);
      return factorize(A2, 1e-8);
    }();
    const bool kept_ok = solve(kept, b) == x;
    // hooks (debug mode; a single leaf goes straight to the root: no steps)
    FactorizeHooks hk;
    int steps = 0;
    hk.after_projection = [&](const FactorState&, int) { ++steps; };
    FactorChain ch2 = factorize(A, 1e-8, std::nullopt, &hk);
    std::printf("facade: kept chain solves %d, hooked steps %d\n", (int)kept_ok, steps);
    if (!kept_ok || solve(ch2, b) != x) return 4;
    // multi-GPU entry point with a single rank (no exchange happens): the
    // SUBTREE order; a wrong rank count maps to InvalidInputError
    FactorChain ch3 = factorize_dist(A, 1e-8, 0, 1, Exchange());
    bool bad_ranks = false;
    try {
      factorize_dist(A, 1e-8, 0, 3, Exchange([](void*, const int64_t*, int) { return 0; }));
    } catch (const InvalidInputError&) {
      bad_ranks = true;
    }
    if (!bad_ranks || solve(ch3, b).size() != x.size()) return 5;
    // singular pivot -> SingularPivotError with the root's cluster -1
    std::vector<cxd> Z(n * n, cxd(0.0));
    d.dense_data = reinterpret_cast<const double*>(Z.data());
    H2Matrix Az(ctx, d);
    try {
      factorize(Az, 1e-8);
      std::printf("facade: expected SingularPivotError\n");
      return 2;
    } catch (const SingularPivotError& e) {
      std::printf("facade: SingularPivotError cluster %d pivot %lld\n", e.cluster, (long long)e.pivot_index);
    }
    return err < 1e-12 && same ? 0 : 1;
  } catch (const DeviceError& e) {
    std::printf("facade: no device: %s\n", e.what());
    return 3;
  }
}
