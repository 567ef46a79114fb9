// h2lu_gpu — command-line drop-in for the reference's h2lu CLI
// (proj/tools/h2lu_cli.cpp:87-317) on the B200 path: the same subcommands
// (build, factor, solve, rhs, bench), flags, defaults, H2LU v1 files, text /
// --json output and exit codes (0 ok, 2 input error, 3 numerical error),
// with every compute step on the device through the C ABI (include/h2g.h).
// Vectors on disk are in the original point order; the tree permutation is
// applied on the way in and undone on the way out (:47-57).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/h2g.h"

namespace {

using cxd = std::complex<double>;

struct CliError : std::runtime_error {
  int code;
  CliError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void check(int rc, const h2g_error& e) {
  if (rc == H2G_OK) return;
  const bool numerical = rc == H2G_ERR_SINGULAR_PIVOT || rc == H2G_ERR_NON_FINITE || rc == H2G_ERR_UNDEFINED_METRIC;
  throw CliError(numerical ? 3 : 2, e.msg);
}

double since(std::chrono::steady_clock::time_point t0) { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); }

struct Options {  // h2lu_cli.cpp:59-78 defaults
  std::string geometry = "rod";
  int64_t n = 0;
  std::string points_path;
  std::string kernel = "laplace";
  double wavenumber = 1.0, shift = 1.0;
  int64_t leafsize = 25;
  double eta = 1.0, eps_h2 = 1e-3, eps_fill_in = 1e-5;
  int stop_level = -1;
  unsigned long long seed = 1234;
  bool as_json = false, cold_cache = false;
  std::string in_path, out_path, chain_path, rhs_path, matrix_path, csv_path;
  std::vector<int64_t> sizes{400, 800, 1600};
  int solve_reps = 3;
};

// ------------------------------------------------------------ geometry (geometry.hpp:54-129)
std::vector<double> points_for(const std::string& g, int64_t n) {
  std::vector<double> p(3 * (size_t)n, 0.0);
  if (g == "rod") {
    for (int64_t i = 0; i < n; ++i) p[3 * i] = (double)i;
  } else if (g == "slab") {
    const int64_t side = (int64_t)std::ceil(std::sqrt((double)n));
    for (int64_t i = 0; i < n; ++i) p[3 * i] = (double)(i % side), p[3 * i + 1] = (double)(i / side);
  } else if (g == "cube") {
    int64_t side = (int64_t)std::ceil(std::cbrt((double)n));
    while (side * side * side < n) ++side;
    for (int64_t i = 0; i < n; ++i) p[3 * i] = (double)(i % side), p[3 * i + 1] = (double)((i / side) % side), p[3 * i + 2] = (double)(i / (side * side));
  } else {
    throw CliError(2, "unknown geometry '" + g + "' (rod, slab, cube)");
  }
  return p;
}

std::vector<double> load_points(const std::string& path) {
  std::vector<double> p;
  if (path.size() > 4 && path.substr(path.size() - 4) == ".bin") {
    std::ifstream in(path, std::ios::binary | std::ios::ate);
    if (!in) throw CliError(2, "cannot open point file: " + path);
    const std::streamoff bytes = in.tellg();
    if (bytes % 24 != 0) throw CliError(2, "binary point file size is not a multiple of 24: " + path);
    p.resize((size_t)(bytes / 8));
    in.seekg(0);
    in.read(reinterpret_cast<char*>(p.data()), bytes);
    if (!in) throw CliError(2, "truncated binary point file: " + path);
    return p;
  }
  std::ifstream in(path);
  if (!in) throw CliError(2, "cannot open point file: " + path);
  std::string line;
  int64_t lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
    std::istringstream ss(line);
    double v[3];
    char sep;
    if (!(ss >> v[0] >> sep >> v[1] >> sep >> v[2])) throw CliError(2, "bad CSV point at line " + std::to_string(lineno) + " of " + path);
    p.insert(p.end(), v, v + 3);
  }
  return p;
}

std::vector<double> load_cloud(const Options& o) {
  if (!o.points_path.empty()) return load_points(o.points_path);
  if (o.n <= 0) throw CliError(2, "either --points or --geometry with --n is required");
  return points_for(o.geometry, o.n);
}

h2g_kernel_spec make_kernel(const Options& o) {  // h2lu_cli.cpp:31-35, kernel.hpp:40-53
  h2g_kernel_spec k{};
  if (o.kernel == "laplace")
    k.kind = H2G_KERNEL_LAPLACE;
  else if (o.kernel == "helmholtz")
    k.kind = H2G_KERNEL_HELMHOLTZ, k.wavenumber_re = o.wavenumber;
  else
    throw CliError(2, "unknown kernel '" + o.kernel + "' (laplace, helmholtz)");
  k.scale_re = 1.0;
  k.diag_re = o.shift;
  return k;
}

// ------------------------------------------------------------------ handles
struct Ctx {
  h2g_context* c = nullptr;
  Ctx() {
    h2g_error e{};
    check(h2g_context_create(0, &c, &e), e);
  }
  ~Ctx() { h2g_context_destroy(c); }
};
struct Mat {
  h2g_matrix* m = nullptr;
  ~Mat() { h2g_matrix_destroy(m); }
};
struct Chain {
  h2g_chain* c = nullptr;
  ~Chain() { h2g_chain_destroy(c); }
};

std::vector<int64_t> matrix_sizes(const h2g_matrix* m) {
  std::vector<int64_t> s(8);
  h2g_matrix_sizes(m, s.data());
  return s;
}

std::vector<int64_t> perm_of(const h2g_matrix* m) {
  std::vector<int64_t> p(matrix_sizes(m)[0]);
  h2g_matrix_download(m, nullptr, nullptr, p.data(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                      nullptr, nullptr, nullptr);
  return p;
}

struct MatrixStats {
  int64_t n = 0, depth = 0, rank_max = 0, num_adm = 0, mem = 0;
  int csp = 0;
};

// csp (block_tree.hpp:64-72): most blocks in any cluster row of one level
MatrixStats stats_of(const h2g_matrix* m) {
  const auto s = matrix_sizes(m);
  MatrixStats st;
  st.n = s[0], st.depth = s[1], st.num_adm = s[3];
  st.mem = 16 * (s[5] + s[6] + s[7]);
  const int nc = (int)s[2], L = (int)s[1];
  std::vector<int64_t> rank(nc), aoff(L + 2), soff(L + 2);
  h2g_matrix_download(m, nullptr, nullptr, nullptr, aoff.data(), nullptr, soff.data(), nullptr, nullptr, nullptr, rank.data(), nullptr, nullptr,
                      nullptr, nullptr, nullptr, nullptr);
  std::vector<int32_t> ap(2 * std::max<int64_t>(aoff[L + 1], 1)), sp(2 * std::max<int64_t>(soff[L + 1], 1)), lp(2 * std::max<int64_t>(s[4], 1));
  h2g_matrix_download(m, nullptr, nullptr, nullptr, aoff.data(), ap.data(), soff.data(), sp.data(), lp.data(), nullptr, nullptr, nullptr, nullptr,
                      nullptr, nullptr, nullptr, nullptr);
  for (int64_t k : rank) st.rank_max = std::max(st.rank_max, k);
  for (int l = 0; l <= L; ++l) {
    std::map<int, int> row;
    for (int64_t q = aoff[l]; q < aoff[l + 1]; ++q) ++row[ap[2 * q]];
    for (int64_t q = soff[l]; q < soff[l + 1]; ++q) ++row[sp[2 * q]];
    if (l == L)
      for (int64_t q = 0; q < s[4]; ++q) ++row[lp[2 * q]];
    for (auto& kv : row) st.csp = std::max(st.csp, kv.second);
  }
  return st;
}

std::vector<cxd> load_vec(const std::string& path) {
  int64_t n = 0;
  h2g_error e{};
  check(h2g_vector_load(path.c_str(), nullptr, &n, &e), e);
  std::vector<cxd> v(n);
  check(h2g_vector_load(path.c_str(), reinterpret_cast<double*>(v.data()), &n, &e), e);
  return v;
}

void save_vec(const std::string& path, const std::vector<cxd>& v) {
  h2g_error e{};
  check(h2g_vector_save(path.c_str(), reinterpret_cast<const double*>(v.data()), (int64_t)v.size(), &e), e);
}

double norm(const std::vector<cxd>& v) {
  double s = 0.0;
  for (const cxd& x : v) s += std::norm(x);
  return std::sqrt(s);
}

double residual(Ctx& ctx, const h2g_matrix* m, const std::vector<cxd>& x, const std::vector<cxd>& b) {  // verify.hpp:14-19
  const double nb = norm(b);
  if (nb == 0.0) throw CliError(3, "relative_residual: right-hand side is zero");
  std::vector<cxd> y(x.size());
  h2g_error e{};
  check(h2g_matvec(ctx.c, m, reinterpret_cast<const double*>(x.data()), reinterpret_cast<double*>(y.data()), 1, &e), e);
  for (size_t i = 0; i < y.size(); ++i) y[i] -= b[i];
  return norm(y) / nb;
}

std::string jnum(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}
std::string jstr(const std::string& s) { return "\"" + s + "\""; }

// ---------------------------------------------------------------- commands
int run_build(const Options& o) {  // h2lu_cli.cpp:87-110
  const auto pts = load_cloud(o);
  const auto kern = make_kernel(o);
  Ctx ctx;
  Mat A;
  h2g_error e{};
  const auto t0 = std::chrono::steady_clock::now();
  check(h2g_matrix_build(ctx.c, pts.data(), (int64_t)pts.size() / 3, o.leafsize, o.eta, &kern, o.eps_h2, &A.m, &e), e);
  const double secs = since(t0);
  check(h2g_matrix_save(A.m, o.out_path.c_str(), &e), e);
  const MatrixStats st = stats_of(A.m);
  if (o.as_json) {
    std::printf("{\"n\": %lld, \"depth\": %lld, \"csp\": %d, \"admissible_blocks\": %lld, \"rank_max\": %lld, \"mem_bytes\": %lld, \"seconds\": %s, "
                "\"out\": %s}\n",
                (long long)st.n, (long long)st.depth, st.csp, (long long)st.num_adm, (long long)st.rank_max, (long long)st.mem, jnum(secs).c_str(),
                jstr(o.out_path).c_str());
  } else {
    std::printf("built n=%lld depth=%lld rank_max=%lld mem=%.1f MiB in %.2fs -> %s\n", (long long)st.n, (long long)st.depth, (long long)st.rank_max,
                st.mem / 1048576.0, secs, o.out_path.c_str());
  }
  return 0;
}

int run_factor(const Options& o) {  // h2lu_cli.cpp:112-150
  Ctx ctx;
  Mat A;
  Chain ch;
  h2g_error e{};
  check(h2g_matrix_load(ctx.c, o.in_path.c_str(), &A.m, &e), e);
  const auto t0 = std::chrono::steady_clock::now();
  check(h2g_factorize(ctx.c, A.m, o.eps_fill_in, o.stop_level, H2G_SCHEDULE_REFERENCE, &ch.c, &e), e);
  const double secs = since(t0);
  check(h2g_chain_save(ch.c, A.m, o.out_path.c_str(), &e), e);
  int64_t info[6];
  h2g_chain_info(ch.c, info);
  std::string levels = "[", text;
  for (int li = 0; li < info[3]; ++li) {
    int64_t d[9];
    h2g_chain_level(ch.c, li, d);
    levels += std::string(li ? ", " : "") + "{\"level\": " + std::to_string(d[0]) + ", \"eliminated\": " + std::to_string(d[4]) +
              ", \"rank_sum_before\": " + std::to_string(d[2]) + ", \"rank_sum_after\": " + std::to_string(d[3]) +
              ", \"ledger_blocks\": " + std::to_string(d[5]) + ", \"chain_bytes\": " + std::to_string(d[6]) + "}";
    char buf[256];
    std::snprintf(buf, sizeof buf, "level %lld: eliminated %lld of %lld unknowns, %lld fill blocks absorbed\n", (long long)d[0], (long long)d[4],
                  (long long)(d[4] + d[3]), (long long)d[5]);
    text += buf;
  }
  levels += "]";
  if (o.as_json) {
    std::printf("{\"n\": %lld, \"stop_level\": %lld, \"root_size\": %lld, \"mem_bytes\": %lld, \"seconds\": %s, \"levels\": %s, \"out\": %s}\n",
                (long long)info[0], (long long)info[1], (long long)info[2], (long long)info[4], jnum(secs).c_str(), levels.c_str(),
                jstr(o.out_path).c_str());
  } else {
    std::printf("%sfactorized n=%lld root=%lld mem=%.1f MiB in %.2fs -> %s\n", text.c_str(), (long long)info[0], (long long)info[2],
                info[4] / 1048576.0, secs, o.out_path.c_str());
  }
  return 0;
}

int run_solve(const Options& o) {  // h2lu_cli.cpp:152-179
  Ctx ctx;
  Chain ch;
  h2g_error e{};
  check(h2g_chain_load(ctx.c, o.chain_path.c_str(), &ch.c, &e), e);
  int64_t info[6];
  h2g_chain_info(ch.c, info);
  const auto b_orig = load_vec(o.rhs_path);
  if ((int64_t)b_orig.size() != info[0])
    throw CliError(2, "rhs length " + std::to_string(b_orig.size()) + " does not match the factorization size " + std::to_string(info[0]));
  // the chain file carries the tree permutation; read it through the matrix
  // when given, else from the chain's own tree (h2lu_cli.cpp:159)
  std::vector<int64_t> perm;
  Mat A;
  if (!o.matrix_path.empty()) {
    check(h2g_matrix_load(ctx.c, o.matrix_path.c_str(), &A.m, &e), e);
    perm = perm_of(A.m);
  } else {
    perm.resize(info[0]);
    check(h2g_chain_perm_tree(ch.c, perm.data()), e);
  }
  std::vector<cxd> b(b_orig.size()), x(b_orig.size());
  for (size_t i = 0; i < b.size(); ++i) b[i] = b_orig[perm[i]];
  const auto t0 = std::chrono::steady_clock::now();
  check(h2g_solve(ch.c, reinterpret_cast<const double*>(b.data()), reinterpret_cast<double*>(x.data()), info[0], 1, H2G_SOLVE, &e), e);
  const double secs = since(t0);
  std::vector<cxd> xo(x.size());
  for (size_t i = 0; i < x.size(); ++i) xo[perm[i]] = x[i];
  save_vec(o.out_path, xo);
  std::string extra, text;
  if (A.m) {
    const double res = residual(ctx, A.m, x, b);
    extra = ", \"residual\": " + jnum(res);
    char buf[128];
    std::snprintf(buf, sizeof buf, "relative residual %.3e\n", res);
    text += buf;
  }
  if (o.as_json)
    std::printf("{\"n\": %lld, \"seconds\": %s, \"out\": %s%s}\n", (long long)info[0], jnum(secs).c_str(), jstr(o.out_path).c_str(), extra.c_str());
  else
    std::printf("%ssolved n=%lld in %.3fs -> %s\n", text.c_str(), (long long)info[0], secs, o.out_path.c_str());
  return 0;
}

int run_rhs(const Options& o) {  // h2lu_cli.cpp:181-191
  if (o.n <= 0) throw CliError(2, "--n must be positive");
  std::vector<cxd> v(o.n);
  h2g_random_rhs(o.n, o.seed, reinterpret_cast<double*>(v.data()));
  save_vec(o.out_path, v);
  if (o.as_json)
    std::printf("{\"n\": %lld, \"seed\": %llu, \"out\": %s}\n", (long long)o.n, o.seed, jstr(o.out_path).c_str());
  else
    std::printf("wrote random vector of length %lld -> %s\n", (long long)o.n, o.out_path.c_str());
  return 0;
}

struct LoglogFit {  // bench.hpp:135-161
  double slope = 0.0;
  bool ok = false;
};
LoglogFit fit_loglog(const std::vector<double>& xs, const std::vector<double>& ys) {
  LoglogFit f;
  if (xs.size() != ys.size() || xs.size() < 2) return f;
  double sx = 0, sy = 0, sxx = 0, sxy = 0;
  const double m = (double)xs.size();
  for (size_t i = 0; i < xs.size(); ++i) {
    if (!(xs[i] > 0.0) || !(ys[i] > 0.0)) return f;
    const double lx = std::log(xs[i]), ly = std::log(ys[i]);
    sx += lx, sy += ly, sxx += lx * lx, sxy += lx * ly;
  }
  const double var = sxx - sx * sx / m;
  if (!(var > 0.0)) return f;
  f.slope = (sxy - sx * sy / m) / var;
  f.ok = true;
  return f;
}

int run_bench(const Options& o) {  // h2lu_cli.cpp:193-231, bench.hpp:77-124
  const auto kern = make_kernel(o);
  for (int64_t n : o.sizes) points_for(o.geometry, std::max<int64_t>(n, 1));  // validate the geometry first
  Ctx ctx;
  struct Run {
    int64_t n;
    MatrixStats st;
    int64_t root;
    double build, factor, solve, res, err;
    int64_t mem_chain;
  };
  std::vector<Run> runs;
  for (int64_t n : o.sizes) {
    const auto pts = points_for(o.geometry, n);
    Mat A;
    Chain ch;
    h2g_error e{};
    auto t0 = std::chrono::steady_clock::now();
    check(h2g_matrix_build(ctx.c, pts.data(), n, o.leafsize, o.eta, &kern, o.eps_h2, &A.m, &e), e);
    Run r{};
    r.n = n;
    r.build = since(t0);
    r.st = stats_of(A.m);
    t0 = std::chrono::steady_clock::now();
    check(h2g_factorize(ctx.c, A.m, o.eps_fill_in, -1, H2G_SCHEDULE_REFERENCE, &ch.c, &e), e);
    r.factor = since(t0);
    int64_t info[6];
    h2g_chain_info(ch.c, info);
    r.root = info[2];
    r.mem_chain = info[4];
    // manufactured solution (bench.hpp:104-108), in tree order
    std::vector<cxd> xt(n), b(n), x(n);
    h2g_random_rhs(n, o.seed, reinterpret_cast<double*>(xt.data()));
    check(h2g_matvec(ctx.c, A.m, reinterpret_cast<const double*>(xt.data()), reinterpret_cast<double*>(b.data()), 1, &e), e);
    std::vector<double> times;
    for (int rep = 0; rep < std::max(1, o.solve_reps); ++rep) {
      t0 = std::chrono::steady_clock::now();
      check(h2g_solve(ch.c, reinterpret_cast<const double*>(b.data()), reinterpret_cast<double*>(x.data()), n, 1, H2G_SOLVE, &e), e);
      times.push_back(since(t0));
    }
    std::sort(times.begin(), times.end());
    r.solve = times[times.size() / 2];
    r.res = residual(ctx, A.m, x, b);
    std::vector<cxd> d(n);
    for (int64_t i = 0; i < n; ++i) d[i] = x[i] - xt[i];
    r.err = norm(d) / norm(xt);
    runs.push_back(r);
  }
  if (!o.csv_path.empty()) {  // bench.hpp:163-172
    std::FILE* f = std::fopen(o.csv_path.c_str(), "w");
    if (!f) throw CliError(2, "cannot open " + o.csv_path + " for writing");
    std::fprintf(f, "geometry,n,depth,leafsize,eta,eps_h2,eps_fill_in,csp,rank_max,root_size,build_seconds,factor_seconds,solve_seconds,residual,"
                    "error_vs_true,mem_h2_bytes,mem_chain_bytes\n");
    for (const Run& r : runs)
      std::fprintf(f, "%s,%lld,%lld,%lld,%.17g,%.17g,%.17g,%d,%lld,%lld,%.17g,%.17g,%.17g,%.17g,%.17g,%lld,%lld\n", o.geometry.c_str(), (long long)r.n,
                   (long long)r.st.depth, (long long)o.leafsize, o.eta, o.eps_h2, o.eps_fill_in, r.st.csp, (long long)r.st.rank_max, (long long)r.root,
                   r.build, r.factor, r.solve, r.res, r.err, (long long)r.st.mem, (long long)r.mem_chain);
    std::fclose(f);
  }
  if (o.as_json) {  // bench.hpp:174-196, one object per line
    for (const Run& r : runs)
      std::printf("{\"geometry\": %s, \"n\": %lld, \"depth\": %lld, \"leafsize\": %lld, \"eta\": %s, \"eps_h2\": %s, \"eps_fill_in\": %s, \"csp\": %d, "
                  "\"rank_max\": %lld, \"root_size\": %lld, \"build_seconds\": %s, \"factor_seconds\": %s, \"solve_seconds\": %s, \"residual\": %s, "
                  "\"error_vs_true\": %s, \"mem_h2_bytes\": %lld, \"mem_chain_bytes\": %lld}\n",
                  jstr(o.geometry).c_str(), (long long)r.n, (long long)r.st.depth, (long long)o.leafsize, jnum(o.eta).c_str(), jnum(o.eps_h2).c_str(),
                  jnum(o.eps_fill_in).c_str(), r.st.csp, (long long)r.st.rank_max, (long long)r.root, jnum(r.build).c_str(), jnum(r.factor).c_str(),
                  jnum(r.solve).c_str(), jnum(r.res).c_str(), jnum(r.err).c_str(), (long long)r.st.mem, (long long)r.mem_chain);
    return 0;
  }
  std::printf("%-6s %8s %6s %10s %10s %10s %12s %12s\n", "geom", "n", "csp", "build_s", "factor_s", "solve_s", "residual", "mem_MiB");
  std::vector<double> ns, fs, ss, ms;
  for (const Run& r : runs) {
    const double mem = (double)(r.st.mem + r.mem_chain);
    std::printf("%-6s %8lld %6d %10.3f %10.3f %10.4f %12.3e %12.1f\n", o.geometry.c_str(), (long long)r.n, r.st.csp, r.build, r.factor, r.solve, r.res,
                mem / 1048576.0);
    ns.push_back((double)r.n), fs.push_back(r.factor), ss.push_back(r.solve), ms.push_back(mem);
  }
  const LoglogFit f = fit_loglog(ns, fs), s = fit_loglog(ns, ss), m = fit_loglog(ns, ms);
  if (f.ok) std::printf("slope vs n: factor %.2f, solve %.2f, memory %.2f\n", f.slope, s.slope, m.slope);
  return 0;
}

// ------------------------------------------------------------- arguments
[[noreturn]] void usage(const std::string& msg) {
  std::fprintf(stderr,
               "%s\nusage: h2lu_gpu {build,factor,solve,rhs,bench} [options]\n"
               "  build  --geometry rod|slab|cube --n N | --points FILE, --leafsize 25 --eta 1 --kernel laplace|helmholtz --wavenumber 1 --shift 1 "
               "--eps-h2 1e-3 --out FILE\n"
               "  factor --in FILE --eps-fill-in 1e-5 [--stop-level L] --out FILE\n"
               "  solve  --chain FILE --rhs FILE [--matrix FILE] --out FILE\n"
               "  rhs    --n N [--seed 1234] --out FILE\n"
               "  bench  geometry/kernel flags, --sizes 400,800,1600 --eps-h2 --eps-fill-in --solve-reps 3 --seed --csv FILE --cold-cache\n"
               "  every subcommand: --json\n",
               msg.c_str());
  throw CliError(2, msg);
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 2) usage("a subcommand is required");
    const std::string cmd = argv[1];
    if (cmd == "-h" || cmd == "--help") {
      try {
        usage("accuracy-controlled direct solver for hierarchically compressed kernel matrices (B200)");
      } catch (const CliError&) {
      }
      return 0;
    }
    static const std::map<std::string, std::vector<std::string>> allowed = {
        {"build", {"--geometry", "--n", "--points", "--leafsize", "--eta", "--kernel", "--wavenumber", "--shift", "--eps-h2", "--out", "--json"}},
        {"factor", {"--in", "--eps-fill-in", "--stop-level", "--out", "--json"}},
        {"solve", {"--chain", "--rhs", "--matrix", "--out", "--json"}},
        {"rhs", {"--n", "--seed", "--out", "--json"}},
        {"bench",
         {"--geometry", "--leafsize", "--eta", "--kernel", "--wavenumber", "--shift", "--sizes", "--eps-h2", "--eps-fill-in", "--solve-reps", "--seed",
          "--csv", "--cold-cache", "--json"}},
    };
    auto it = allowed.find(cmd);
    if (it == allowed.end()) usage("unknown subcommand '" + cmd + "'");
    Options o;
    std::map<std::string, std::string> got;
    for (int i = 2; i < argc; ++i) {
      const std::string a = argv[i];
      if (std::find(it->second.begin(), it->second.end(), a) == it->second.end()) usage("unknown option '" + a + "' for " + cmd);
      if (a == "--json" || a == "--cold-cache") {
        got[a] = "1";
        continue;
      }
      if (i + 1 >= argc) usage("option " + a + " needs a value");
      got[a] = argv[++i];
    }
    auto num = [&](const char* k, double& v) {
      if (got.count(k)) {
        char* end = nullptr;
        v = std::strtod(got[k].c_str(), &end);
        if (!end || *end) usage(std::string("bad value for ") + k);
      }
    };
    auto inum = [&](const char* k, int64_t& v) {
      double d = (double)v;
      num(k, d);
      v = (int64_t)d;
    };
    if (got.count("--geometry")) o.geometry = got["--geometry"];
    if (got.count("--points")) o.points_path = got["--points"];
    if (got.count("--kernel")) o.kernel = got["--kernel"];
    inum("--n", o.n);
    inum("--leafsize", o.leafsize);
    num("--eta", o.eta);
    num("--wavenumber", o.wavenumber);
    num("--shift", o.shift);
    num("--eps-h2", o.eps_h2);
    num("--eps-fill-in", o.eps_fill_in);
    if (got.count("--stop-level")) {
      int64_t s = 0;
      inum("--stop-level", s);
      o.stop_level = (int)s;
    }
    if (got.count("--seed")) o.seed = std::strtoull(got["--seed"].c_str(), nullptr, 10);
    if (got.count("--solve-reps")) {
      int64_t r = 3;
      inum("--solve-reps", r);
      o.solve_reps = (int)r;
    }
    o.as_json = got.count("--json") > 0;
    o.cold_cache = got.count("--cold-cache") > 0;
    o.in_path = got.count("--in") ? got["--in"] : "";
    o.out_path = got.count("--out") ? got["--out"] : "";
    o.chain_path = got.count("--chain") ? got["--chain"] : "";
    o.rhs_path = got.count("--rhs") ? got["--rhs"] : "";
    o.matrix_path = got.count("--matrix") ? got["--matrix"] : "";
    o.csv_path = got.count("--csv") ? got["--csv"] : "";
    if (got.count("--sizes")) {
      o.sizes.clear();
      std::stringstream ss(got["--sizes"]);
      std::string tok;
      while (std::getline(ss, tok, ',')) o.sizes.push_back(std::atoll(tok.c_str()));
    }
    auto need = [&](const char* k) {
      if (!got.count(k)) usage(std::string(k) + " is required");
    };
    if (cmd == "build") need("--out");
    if (cmd == "factor") need("--in"), need("--out");
    if (cmd == "solve") need("--chain"), need("--rhs"), need("--out");
    if (cmd == "rhs") need("--n"), need("--out");
    if (cmd == "rhs") return run_rhs(o);
    if (cmd == "build") return run_build(o);
    if (cmd == "factor") return run_factor(o);
    if (cmd == "solve") return run_solve(o);
    return run_bench(o);
  } catch (const CliError& e) {  // h2lu_cli.cpp:305-317
    if (e.code == 3)
      std::fprintf(stderr, "numerical error: %s\n", e.what());
    else
      std::fprintf(stderr, "error: %s\n", e.what());
    return e.code;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
}
