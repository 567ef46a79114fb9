// Host driver of the B200 H² factorize / solve: implements the C ABI of
// include/h2g.h. The level loop mirrors factorize()
// (proj/include/h2lu/factorization.hpp:600-653): per level, batches of
// clusters run the step kernels of factor.cu; at the level boundary the host
// reads back the final ranks (one small copy), finishes the level and merges
// to the parent (finish_level :445-475, merge_permute :483-584) with
// descriptor-driven batched copies/GEMMs; the remainder is LU-factored on the
// device (:637-651). There is no CPU fallback.
#include <atomic>
#include <thread>
#include <unistd.h>
#include <functional>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdlib>
#include <complex>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <unordered_map>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/h2g.h"
#include "build.cuh"
#include "factor.cuh"
#include "plan.hpp"
#include "serialize.hpp"
#include "solve.cuh"

using namespace h2g;

namespace {

// ------------------------------------------------------------------ errors
struct Error : std::runtime_error {
  int code;
  int cluster = -1, level = -1;
  long long pivot_index = -1;
  double pivot_magnitude = 0.0;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

thread_local h2g_error g_last{};

// NVTX range (header-only NVTX v3): factorize / level / merge / solve phases
// show up by name in Nsight timelines.
struct NvtxRange {
  explicit NvtxRange(const std::string& name) { nvtxRangePushA(name.c_str()); }
  ~NvtxRange() { nvtxRangePop(); }
};

void set_error(h2g_error* out, int code, const char* msg, int cluster = -1, int level = -1, long long piv = -1, double mag = 0.0) {
  h2g_error e{};
  e.code = code;
  e.cluster = cluster;
  e.level = level;
  e.pivot_index = piv;
  e.pivot_magnitude = mag;
  std::snprintf(e.msg, sizeof e.msg, "%s", msg);
  g_last = e;
  if (out) *out = e;
}

#define CK(x)                                                                                                   \
  do {                                                                                                          \
    cudaError_t e_ = (x);                                                                                       \
    if (e_ != cudaSuccess) throw Error(H2G_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));       \
  } while (0)

template <class F>
int guarded(h2g_error* err, F&& f) {
  try {
    f();
    if (err) *err = h2g_error{};
    return H2G_OK;
  } catch (const Error& e) {
    set_error(err, e.code, e.what(), e.cluster, e.level, e.pivot_index, e.pivot_magnitude);
    return e.code;
  } catch (const std::invalid_argument& e) {
    set_error(err, H2G_ERR_INVALID_INPUT, e.what());
    return H2G_ERR_INVALID_INPUT;
  } catch (const std::bad_alloc& e) {
    set_error(err, H2G_ERR_CUDA, "host out of memory");
    return H2G_ERR_CUDA;
  } catch (const std::exception& e) {
    set_error(err, H2G_ERR_INTERNAL, e.what());
    return H2G_ERR_INTERNAL;
  }
}

// ------------------------------------------------------------ device buffers
// Stream-ordered block cache in front of cudaMallocAsync. A factorize
// allocates and frees the same few hundred buffers (per-level chain arenas,
// Schur/fill pools, descriptor tables) every call; letting the driver pool
// grow and re-map them measured up to ~0.6 s of host stall per level. Freed
// blocks go back to a per-stream free list (reuse on the same stream is
// ordered after every earlier use) and are handed out again best-fit.
class BlockCache {
 public:
  static BlockCache& get() {
    static BlockCache* c = new BlockCache();  // leaked: outlives static destructors
    return *c;
  }
  static size_t round(size_t n) {
    const size_t g = n < (1u << 20) ? 512 : (2u << 20);
    return (n + g - 1) / g * g;
  }
  void add_stream(cudaStream_t s, int device) {
    std::lock_guard<std::mutex> g(mu_);
    live_[s] = device;
  }
  void remove_stream(cudaStream_t s) {
    std::lock_guard<std::mutex> g(mu_);
    auto& fl = free_[s];
    const int dev = live_.count(s) ? live_[s] : -1;
    for (auto& kv : fl) cudaFree(kv.second), cached_[dev] -= kv.first;
    free_.erase(s);
    live_.erase(s);
    spill_.erase(s);
  }
  // Out-of-memory hook of the factorization running on stream s (moves
  // finished chain levels to host memory); one per stream / context, so two
  // contexts never call each other's hook.
  void set_spill(cudaStream_t s, std::function<bool()> f) {
    std::lock_guard<std::mutex> g(mu_);
    if (f)
      spill_[s] = std::move(f);
    else
      spill_.erase(s);
  }
  void* alloc(size_t n, cudaStream_t s) {
    const size_t r = round(n);
    int dev = 0;
    cudaGetDevice(&dev);
    std::function<bool()> spill;
    {
      std::lock_guard<std::mutex> g(mu_);
      auto lv = live_.find(s);
      if (lv != live_.end()) {
        dev = lv->second;
        auto& fl = free_[s];
        auto it = fl.lower_bound(r);
        if (it != fl.end() && it->first <= r + r / 4 + (4u << 20)) {
          void* p = it->second;
          cached_[dev] -= it->first;
          fl.erase(it);
          return p;
        }
      }
      auto sp = spill_.find(s);
      if (sp != spill_.end()) spill = sp->second;
    }
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, r, s);
    if (e == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      trim(dev);
      e = cudaMallocAsync(&p, r, s);
      // still short: let the factorization on this stream move finished
      // chain levels to host memory, one at a time
      while (e == cudaErrorMemoryAllocation && spill && spill()) {
        cudaGetLastError();
        trim(dev);
        e = cudaMallocAsync(&p, r, s);
      }
    }
    if (e != cudaSuccess) throw Error(H2G_ERR_CUDA, std::string("device allocation of ") + std::to_string(n) + " bytes: " + cudaGetErrorString(e));
    std::lock_guard<std::mutex> g(mu_);
    size_[p] = r;
    return p;
  }
  void release(void* p, cudaStream_t s) {
    std::lock_guard<std::mutex> g(mu_);
    auto it = size_.find(p);
    auto lv = live_.find(s);
    if (it != size_.end() && lv != live_.end()) {
      free_[s].emplace(it->second, p);
      cached_[lv->second] += it->second;
      return;
    }
    if (it != size_.end()) size_.erase(it);
    if (s)
      cudaFree(p);  // owning stream already destroyed (context torn down first)
    else
      cudaFreeAsync(p, s);
  }
  // hand the cached blocks of one device back to the driver (out-of-memory retry)
  void trim(int dev) {
    std::lock_guard<std::mutex> g(mu_);
    for (auto& fs : free_) {
      auto lv = live_.find(fs.first);
      if (lv == live_.end() || lv->second != dev) continue;
      for (auto& kv : fs.second) {
        size_.erase(kv.second);
        cached_[dev] -= kv.first;
        cudaFreeAsync(kv.second, fs.first);
      }
      fs.second.clear();
      cudaStreamSynchronize(fs.first);
    }
    // and the pool's own reserve (release threshold is "keep everything")
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  }
  void trim() {
    int dev = 0;
    cudaGetDevice(&dev);
    trim(dev);
  }

  // device bytes a new allocation on the current device can still obtain:
  // driver-free memory, the pool's reserve and this device's cached blocks
  size_t headroom() {
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    size_t pool_spare = 0;
    int dev = 0;
    cudaMemPool_t pool;
    cudaGetDevice(&dev);
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t res = 0, used = 0;
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res);
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
      pool_spare = res > used ? res - used : 0;
    }
    std::lock_guard<std::mutex> g(mu_);
    return fr + pool_spare + cached_[dev];
  }

 private:
  std::mutex mu_;
  std::map<int, size_t> cached_;           // per device
  std::map<cudaStream_t, int> live_;       // stream -> device
  std::map<cudaStream_t, std::function<bool()>> spill_;
  std::map<cudaStream_t, std::multimap<size_t, void*>> free_;
  std::unordered_map<void*, size_t> size_;
};

struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), bytes(o.bytes), s(o.s) { o.p = nullptr, o.bytes = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p, bytes = o.bytes, s = o.s;
      o.p = nullptr, o.bytes = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void release() {
    if (p) BlockCache::get().release(p, s);
    p = nullptr;
    bytes = 0;
  }
  void alloc(size_t n, cudaStream_t st, bool zero = false) {
    release();
    s = st;
    bytes = n;
    if (n) {
      p = BlockCache::get().alloc(n, st);
      if (zero) CK(cudaMemsetAsync(p, 0, n, st));
    }
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Pinned, device-mapped host memory. Used only when a configuration does not
// fit in HBM (config 3: the level-12 -> 11 merge cores and the chains of
// finished levels); kernels read / write it in place over the host link.
// Process-wide cap on pinned staging memory (H2G_HOST_STAGING_GB; default:
// host RAM minus 20 GB, at least 75 % of it): past it a staging request fails
// as a device out-of-memory instead of exhausting the host.
std::atomic<size_t> g_pinned_bytes{0};
size_t pinned_cap() {
  static const size_t cap = [] {
    if (const char* e = std::getenv("H2G_HOST_STAGING_GB")) return (size_t)(std::atof(e) * 1e9);
    const long pages = sysconf(_SC_PHYS_PAGES), psz = sysconf(_SC_PAGE_SIZE);
    if (pages <= 0 || psz <= 0) return (size_t)96e9;
    const double ram = (double)pages * (double)psz;
    return (size_t)std::max(0.75 * ram, ram - 20e9);
  }();
  return cap;
}

// Pinning host memory costs ~0.45 s per GB on the B200 boxes (cudaHostAlloc at
// 2.2 GB/s, profiles/r02_pinned_alloc.txt), and the host-staged configurations
// pin and release hundreds of GB per factorization (fill cores of every
// level, chain chunks). Released buffers of >= 64 MB are kept and handed out
// again to requests they fit within 12 % (the host-staged fill cores use pages
// of one size, so a level's pages serve the next level); they still count against the
// staging cap and are given back to the system when the cap is near.
// Host staging of many similar pieces (fill cores, chain chunks) goes through
// pinned pages of one size, so the pages one level releases serve the next.
constexpr size_t kStagePage = size_t(2) << 30;

class PinnedCache {
 public:
  static PinnedCache& get() {
    static PinnedCache c;
    return c;
  }
  // a cached buffer of capacity in [n, 1.125 n + 16 MB], or nullptr
  void* take(size_t n, size_t* cap) {
    std::lock_guard<std::mutex> g(mu_);
    auto it = free_.lower_bound(n);
    if (it == free_.end() || it->first > n + n / 8 + (size_t(16) << 20)) return nullptr;
    void* p = it->second;
    *cap = it->first;
    free_.erase(it);
    return p;
  }
  void put(void* p, size_t cap) {
    std::lock_guard<std::mutex> g(mu_);
    free_.emplace(cap, p);
  }
  // give the largest cached buffer back to the system; false if none is left
  bool drop_one() {
    void* p = nullptr;
    size_t cap = 0;
    {
      std::lock_guard<std::mutex> g(mu_);
      if (free_.empty()) return false;
      auto it = std::prev(free_.end());
      p = it->second, cap = it->first;
      free_.erase(it);
    }
    cudaFreeHost(p);
    g_pinned_bytes -= cap;
    return true;
  }
  void clear() {
    while (drop_one()) {
    }
  }
  ~PinnedCache() {
    for (auto& kv : free_) cudaFreeHost(kv.second);  // process exit: errors after the runtime is gone are harmless
  }

 private:
  std::mutex mu_;
  std::multimap<size_t, void*> free_;
};

struct HBuf {
  void* p = nullptr;
  size_t bytes = 0;  // requested size
  size_t cap = 0;    // pinned capacity behind p (>= bytes when the buffer came from the cache)
  HBuf() = default;
  HBuf(const HBuf&) = delete;
  HBuf& operator=(const HBuf&) = delete;
  HBuf(HBuf&& o) noexcept : p(o.p), bytes(o.bytes), cap(o.cap) { o.p = nullptr, o.bytes = 0, o.cap = 0; }
  ~HBuf() { release(); }
  void release() {
    if (p) {
      if (cap >= (size_t(64) << 20)) {
        PinnedCache::get().put(p, cap);
      } else {
        cudaFreeHost(p);
        g_pinned_bytes -= cap;
      }
    }
    p = nullptr;
    bytes = cap = 0;
  }
  void alloc(size_t n) {
    release();
    const size_t want = std::max<size_t>(n, 16);
    if (void* q = PinnedCache::get().take(want, &cap)) {
      p = q;
      bytes = n;
      return;
    }
    while (g_pinned_bytes + want > pinned_cap() && PinnedCache::get().drop_one()) {
    }
    if (g_pinned_bytes + want > pinned_cap())
      throw Error(H2G_ERR_CUDA, std::string("out of memory: staging ") + std::to_string(n) + " bytes in pinned host memory would exceed the " +
                                    std::to_string(pinned_cap()) + "-byte cap (H2G_HOST_STAGING_GB)");
    cudaError_t e = cudaHostAlloc(&p, want, cudaHostAllocMapped | cudaHostAllocPortable);
    if (e != cudaSuccess) {
      cudaGetLastError();
      PinnedCache::get().clear();  // the system is short: cached buffers go back first
      e = cudaHostAlloc(&p, want, cudaHostAllocMapped | cudaHostAllocPortable);
    }
    if (e != cudaSuccess) {
      p = nullptr;
      cudaGetLastError();
      throw Error(H2G_ERR_CUDA, std::string("pinned host allocation of ") + std::to_string(n) + " bytes failed");
    }
    bytes = n;
    cap = want;
    g_pinned_bytes += want;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

template <class T>
void upload(DBuf& b, const std::vector<T>& v, cudaStream_t s) {
  b.alloc(std::max<size_t>(v.size(), 1) * sizeof(T), s);
  if (!v.empty()) CK(cudaMemcpyAsync(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
}

}  // namespace

// =============================================================== handles
// Per-kernel-class event timing (h2g_set_profiling).
struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  struct Rec {
    int cls;
    cudaEvent_t a, b;
    int level;
  };
  int cur_level = -1;
  std::vector<Rec> recs;
  int open_cls = -1;
  cudaEvent_t open_ev = nullptr;
  cudaEvent_t get() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
  void reset() {
    used = 0;
    recs.clear();
  }
  void begin(int cls, cudaStream_t s) {
    if (!on) return;
    open_cls = cls;
    open_ev = get();
    cudaEventRecord(open_ev, s);
  }
  void end(cudaStream_t s) {
    if (!on || open_cls < 0) return;
    cudaEvent_t b = get();
    cudaEventRecord(b, s);
    recs.push_back({open_cls, open_ev, b, cur_level});
    open_cls = -1;
  }
  ~Prof() {
    for (auto e : pool) cudaEventDestroy(e);
  }
};
enum { PC_COMPLEMENT = 0, PC_GRAM, PC_COLNORM, PC_EIG1, PC_HEAD, PC_PANEL, PC_SCHUR, PC_MERGE, PC_ROOT, PC_OTHER, PC_EIGVEC, PC_EIG1B, PC_N };

struct PlanCache {
  int stop = 0, schedule = 0;
  int segments = 1;  // fill storage segments K the work lists were built for
  Structure key;  // the structure the plan was built for (checked on a fingerprint hit)
  std::vector<LevelSym> levels;
  std::vector<LevelSchedule> sched;
  std::vector<LevelWork> work;
};

struct h2g_context {
  int device = 0;
  // Matrices and chains hold a reference: h2g_context_destroy only drops the
  // caller's, the context is torn down when the last user is gone (a chain
  // may outlive the handle it was factorized with).
  std::atomic<int> refs{1};
  // one factorize / solve at a time per context (they share its streams,
  // events and profiling state)
  std::recursive_mutex run_mu;
  // symbolic plans keyed by a fingerprint of the block structure, stop level
  // and schedule: a new matrix with the structure of an earlier one (same
  // geometry, new entries) reuses the plan (the two most recent are kept)
  std::mutex plan_mu;
  std::vector<std::pair<uint64_t, std::shared_ptr<PlanCache>>> plan_lru;
  cudaStream_t stream = nullptr;
  // Deferred Schur updates (targets not read by the next batch) run on a
  // lower-priority side stream, overlapping the next batch's step 0-3b.
  cudaStream_t side = nullptr;
  cudaEvent_t ev_crit = nullptr, ev_bulk = nullptr;
  Prof prof_side;
  // helper stream for small independent kernels of the main chain
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_aux0 = nullptr, ev_aux1 = nullptr;
  // device -> host copies of a streamed level's chain segments
  cudaStream_t copy = nullptr;
  Prof prof_aux;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  DevError* d_err = nullptr;
  int* d_flag = nullptr;
  Prof prof;
};

struct h2g_matrix {
  h2g_context* ctx = nullptr;
  Structure S;
  std::vector<int64_t> perm;
  std::vector<double> points_tree;  // n x 3, tree order (for the H2LU container); empty if unknown
  int64_t leafsize = 0;
  int64_t shadow_guard = 4000;      // carried through the H2LU container (h2_matrix.hpp:38)
  double eps_h2 = 0.0;
  std::vector<int64_t> basis_rows, basis_rank, basis_off, coup_off, dense_off;
  int64_t basis_elems = 0, coup_elems = 0, dense_elems = 0;
  DBuf basis, coup, dense;
  HBuf hdense;  // the dense blocks, moved to pinned host memory when HBM runs short (config 3)
  const cplx* dense_ptr() const { return hdense.p ? hdense.as<cplx>() : dense.as<cplx>(); }
  std::vector<std::shared_ptr<PlanCache>> plans;
  std::mutex mu;
};

struct ChainLevelHost {
  int level = 0;
  std::vector<int64_t> rec;  // 10 per record
  std::vector<int64_t> diag; // 9
  std::vector<int64_t> src;  // permutation
  // device-resident solve data
  DBuf arena;                // chain numeric data of this level
  HBuf harena;               // ... or here, once offloaded to pinned host memory
  const cplx* chain_ptr() const { return harena.p ? harena.as<cplx>() : arena.as<cplx>(); }
  size_t chain_bytes() const { return harena.p ? harena.bytes : arena.bytes; }
  DBuf meta;                 // packed int / offset arrays
  DBuf solve_meta;           // streamed level: the compact chain offsets the solve reads
  // streamed level until the end of the factorization: its Qt block and one
  // compact chunk per segment (on the device while HBM has room, else pinned
  // host memory), joined into one arena by assemble_streamed_chains
  struct Chunk {
    DBuf d;
    HBuf h;            // own pinned buffer (chunks beyond a staging page, chunks spilled later)
    char* hp = nullptr;  // or a range of one of hpages
    long long begin = 0, len = 0;  // compact element range
    const void* src() const { return d.p ? d.p : (hp ? static_cast<const void*>(hp) : h.p); }
  };
  std::vector<Chunk> chunks;
  std::vector<HBuf> hpages;  // pinned staging pages (kStagePage bytes) holding host-resident chunks, filled across segments
  char* hpage = nullptr;
  size_t hpage_used = 0;
  DBuf qchunk;
  long long compact_elems = 0;
  SolveLevel sl{};
  std::vector<int> batch_ptr, batch_maxc;
  const int* d_batch = nullptr;
  std::vector<int> fs_ptr;
  const SolveTargetD* d_fs = nullptr;
  const SolveContribD* d_fc = nullptr;
  DBuf sched_buf;     // batch_ptr | batch_maxc | fs_ptr on the device
  SolveSched sched{};
  DBuf flow_meta;     // dataflow solve schedule (k_fwd_flow / k_bwd_flow)
  SolveFlow flow{};
  size_t flow_part = 0;  // backward partials per rhs column (complex elements)
  size_t part_need = 0;  // backward partials per rhs column (complex elements)
  DBuf d_src;
  // host copies of sizes/offsets for downloads
  std::vector<int> bsz, kfin, korig, R_ptr, R_nb, C_ptr, C_nb;
  std::vector<long long> pos, Qt_off, L11_off, U11_off, Lbar_off, Ubar_off, Lself_off, Uself_off;
  std::vector<int> rec_cluster;  // local id per record (record order)
};

struct h2g_chain {
  h2g_context* ctx = nullptr;
  int64_t n = 0;
  int stop_level = 0;
  int schedule = 0;
  int depth = 0;
  double eps = 0.0;
  std::vector<std::unique_ptr<ChainLevelHost>> levels;
  int64_t root_size = 0;
  DBuf root;  // LU packed (n_root^2)
  DBuf ybuf, tmpbuf, partbuf, flowcnt;
  size_t storage_bytes = 0;
  std::vector<int64_t> tree_perm;  // tree index -> original index of the factorized matrix (empty: identity)
  double factor_ms = 0.0, solve_ms = 0.0;
  double dist_sent_bytes = 0.0, dist_total_bytes = 0.0, dist_exchange_s = 0.0;  // h2g_factorize_dist
  double plan_ms = 0.0;     // host symbolic plan (get_plan), outside factor_ms
  bool plan_built = false;  // false: reused from the matrix / context plan cache
  long long factor_launches = 0, solve_launches = 0;
  double factor_flops = 0.0, schur_flops = 0.0, solve_bytes = 0.0, schur_bytes = 0.0;
  double schur_flops_exec = 0.0, schur_bytes_exec = 0.0;  // k_schur work after the exact-zero skip
  double kms[PC_N] = {0}, kflops[PC_N] = {0}, kbytes[PC_N] = {0};
  // k_schur per level (profiling runs): level, executed flops, executed bytes, event ms
  std::map<int, std::array<double, 3>> schur_levels;
  long long klaunch[PC_N] = {0};
};

namespace {

std::string fmt(const char* f, long long a = 0, long long b = 0) {
  char buf[256];
  std::snprintf(buf, sizeof buf, f, a, b);
  return buf;
}

void check_device_error(h2g_context* ctx, int level_fallback) {
  DevError e{};
  CK(cudaMemcpyAsync(&e, ctx->d_err, sizeof e, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (e.code == 0) return;
  CK(cudaMemsetAsync(ctx->d_err, 0, sizeof(DevError), ctx->stream));
  if (e.code == H2G_ERR_SINGULAR_PIVOT) {
    Error x(H2G_ERR_SINGULAR_PIVOT, e.cluster >= 0 ? fmt("partial_lu: pivot %lld below tolerance (cluster %lld)", e.pivot_index, e.cluster)
                                                   : fmt("partial_lu: pivot %lld below tolerance (root block)", e.pivot_index));
    x.cluster = e.cluster;
    x.level = e.level >= 0 ? e.level : level_fallback;
    x.pivot_index = e.pivot_index;
    x.pivot_magnitude = e.pivot_magnitude;
    throw x;
  }
  Error x(e.code, e.code == 1 ? fmt("unitary_completion: input columns are not orthonormal (cluster %lld)", e.cluster)
                              : fmt("device error %lld at cluster %lld", e.code, e.cluster));
  x.cluster = e.cluster;
  x.level = e.level;
  throw x;
}

uint64_t structure_fingerprint(const Structure& S, int stop, int schedule) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](const void* p, size_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  };
  const int64_t hdr[5] = {S.n, S.depth, S.l0, stop, schedule};
  mix(hdr, sizeof(hdr));
  mix(&S.eta, sizeof(S.eta));
  mix(S.begin.data(), S.begin.size() * 8);
  mix(S.end.data(), S.end.size() * 8);
  for (const auto& v : S.adm) {
    const int64_t k = (int64_t)v.size();
    mix(&k, 8);
    mix(v.data(), v.size() * sizeof(Pair));
  }
  for (const auto& v : S.split) {
    const int64_t k = (int64_t)v.size();
    mix(&k, 8);
    mix(v.data(), v.size() * sizeof(Pair));
  }
  mix(S.leaf.data(), S.leaf.size() * sizeof(Pair));
  return h;
}

bool same_pairs(const std::vector<Pair>& a, const std::vector<Pair>& b) {
  if (a.size() != b.size()) return false;
  for (size_t i = 0; i < a.size(); ++i)
    if (a[i].row != b[i].row || a[i].col != b[i].col) return false;
  return true;
}

// Full structural equality behind the 64-bit fingerprint: a plan is only
// reused for an identical tree and partition.
bool same_structure(const Structure& a, const Structure& b) {
  if (a.n != b.n || a.depth != b.depth || a.eta != b.eta || a.l0 != b.l0 || a.begin != b.begin || a.end != b.end) return false;
  if (a.adm.size() != b.adm.size() || a.split.size() != b.split.size() || !same_pairs(a.leaf, b.leaf)) return false;
  for (size_t l = 0; l < a.adm.size(); ++l)
    if (!same_pairs(a.adm[l], b.adm[l])) return false;
  for (size_t l = 0; l < a.split.size(); ++l)
    if (!same_pairs(a.split[l], b.split[l])) return false;
  return true;
}

PlanCache* get_plan(h2g_matrix* M, int stop, int schedule, bool* built) {
  *built = false;
  std::lock_guard<std::mutex> g(M->mu);
  for (auto& p : M->plans)
    if (p->stop == stop && p->schedule == schedule) return p.get();
  const uint64_t fp = structure_fingerprint(M->S, stop, schedule);
  {
    std::lock_guard<std::mutex> g2(M->ctx->plan_mu);
    for (auto& e : M->ctx->plan_lru)
      if (e.first == fp && e.second->stop == stop && e.second->schedule == schedule && same_structure(e.second->key, M->S)) {
        M->plans.push_back(e.second);
        return M->plans.back().get();
      }
  }
  *built = true;
  auto P = std::make_shared<PlanCache>();
  P->key = M->S;
  P->stop = stop;
  P->schedule = schedule;
  P->levels = build_levels(M->S, stop);
  // fill storage: whole-level full blocks when the leaf level's fill pool
  // is small next to HBM (no segment syncs), else 16 segments (compact cores
  // once both sides have passed step 0); H2G_FILL_SEGMENTS overrides
  int segments = 1;
  if (const char* e = std::getenv("H2G_FILL_SEGMENTS")) {
    segments = std::max(1, std::atoi(e));
  } else if (!P->levels.empty()) {
    const LevelSym& Y0 = P->levels[0];
    const int first = Structure::first(Y0.level);
    double fill = 0.0;
    for (size_t f = 0; f < Y0.frow.size(); ++f)
      fill += 16.0 * (double)(M->S.end[first + Y0.frow[f]] - M->S.begin[first + Y0.frow[f]]) *
              (double)(M->S.end[first + Y0.fcol[f]] - M->S.begin[first + Y0.fcol[f]]);
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    if (fill > 0.15 * (double)tot) segments = 16;
    // the largest configurations: finer segments keep the fill front pool and
    // the chain halves of the coarse levels (blocks of 400-660 rows) small
    if (fill > 0.30 * (double)tot) segments = 64;
  }
  // the subtree partition exchanges whole fill blocks at the interior /
  // boundary border: whole-level storage (one collapse at the level end)
  if (schedule == H2G_SCHEDULE_SUBTREE) segments = 1;
  P->segments = segments;
  // schedules and work lists are independent per level: one host thread each
  size_t nfact = 0;
  for (const auto& L : P->levels)
    if (L.level >= stop && stop <= M->S.depth) ++nfact;
  P->sched.resize(nfact);
  P->work.resize(nfact);
  {
    std::vector<std::thread> th;
    std::exception_ptr failed;
    std::mutex fm;
    for (size_t i = 0; i < nfact; ++i)
      th.emplace_back([&, i] {
        try {
          P->sched[i] = build_schedule(P->levels[i], schedule);
          P->work[i] = build_work(P->levels[i], P->sched[i], segments);
        } catch (...) {
          std::lock_guard<std::mutex> g(fm);
          if (!failed) failed = std::current_exception();
        }
      });
    for (auto& t : th) t.join();
    if (failed) std::rethrow_exception(failed);
  }
  {
    std::lock_guard<std::mutex> g2(M->ctx->plan_mu);
    auto& lru = M->ctx->plan_lru;
    lru.insert(lru.begin(), {fp, P});
    if (lru.size() > 2) lru.pop_back();
  }
  M->plans.push_back(std::move(P));
  return M->plans.back().get();
}

// Packs host arrays into one device buffer; returns device pointers.
struct Packer {
  std::vector<char> host;
  template <class T>
  size_t add(const std::vector<T>& v) {
    size_t off = (host.size() + 15) & ~size_t(15);
    host.resize(off + std::max<size_t>(v.size(), 1) * sizeof(T));
    if (!v.empty()) std::memcpy(host.data() + off, v.data(), v.size() * sizeof(T));
    return off;
  }
  template <class T>
  size_t add_raw(const T* p, size_t n) {
    size_t off = (host.size() + 15) & ~size_t(15);
    host.resize(off + std::max<size_t>(n, 1) * sizeof(T));
    if (n) std::memcpy(host.data() + off, p, n * sizeof(T));
    return off;
  }
  void upload(DBuf& b, cudaStream_t s) {
    b.alloc(host.size() + 16, s);
    CK(cudaMemcpyAsync(b.p, host.data(), host.size(), cudaMemcpyHostToDevice, s));
  }
};

template <class T>
T* at(const DBuf& b, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(b.p) + off);
}


struct LevelData {
  // level-entry sizes
  std::vector<int> bsz, korig;
  std::vector<long long> pos;
  int bmax = 0;
  // dense blocks packed at their true sizes (bsz[row] x bsz[col]); fill
  // blocks in the segmented front pool (foff from the FrontPlan, -1 = never
  // held in full) or, for the root level, packed like the dense blocks
  std::vector<long long> doff, foff;
  FrontPlan front;
  bool has_front = false;
  std::vector<int> fex_host;  // fill blocks holding content at level entry
  DBuf D, F, fex, V0, Vp;
  long long foff_safe(size_t f) const { return foff[f] < 0 ? 0 : foff[f]; }
};

// Packed offsets of blocks (rows[i], cols[i]) with sizes bsz[.]; returns the total.
long long pack_offsets(const std::vector<int>& rows, const std::vector<int>& cols, const std::vector<int>& bsz, std::vector<long long>& off) {
  off.resize(rows.size());
  long long top = 0;
  for (size_t i = 0; i < rows.size(); ++i) off[i] = top, top += (long long)bsz[rows[i]] * bsz[cols[i]];
  return top;
}

}  // namespace

// Dataflow schedule of one level's substitutions (solve.cuh SolveFlow) from
// the batch schedule: items in the elimination order, writer indices per
// segment, gather slots per record. fs / fc: the per-batch forward targets.
void build_flow(ChainLevelHost& CL, int nl, const std::vector<int>& batch_ptr, const std::vector<int>& batch_cl, const std::vector<int>& fs_ptr,
                const std::vector<SolveTargetD>& fs, const std::vector<SolveContribD>& fc, cudaStream_t st) {
  const int nbat = (int)batch_ptr.size() - 1;
  std::vector<int> bat(nl, 0);
  for (int b = 0; b < nbat; ++b)
    for (int q = batch_ptr[b]; q < batch_ptr[b + 1]; ++q) bat[batch_cl[q]] = b;
  // records with large blocks: the rotation is cut into row slabs (32 rows of
  // Qt^H forward, 64 rows of conj(Qt) backward), each its own work item
  static const int split_min = std::getenv("H2G_SOLVE_SPLIT") ? std::atoi(std::getenv("H2G_SOLVE_SPLIT")) : 96;
  const int kSlabBase = 1 << 30;
  std::vector<int> rec_ns_f(nl, 0), rec_ns_b(nl, 0);
  if (split_min > 0)
    for (int t = 0; t < nl; ++t)
      if (CL.bsz[t] >= split_min) {
        rec_ns_f[t] = std::min(64, (CL.bsz[t] + 31) / 32);
        rec_ns_b[t] = std::min(64, (CL.bsz[t] + 63) / 64);
      }
  // fine levels: the forward updates of a not-yet-processed segment are
  // pulled by its own record (one dependent item per batch on the chain
  // instead of two, ~50 times fewer items); large blocks keep one item per
  // (segment, batch), which spreads the Lbar traffic over the CTAs
  static const int pull_max = std::getenv("H2G_SOLVE_PULL") ? std::atoi(std::getenv("H2G_SOLVE_PULL")) : 0;  // measured: no gain (the late record then applies ~50 updates in a row)
  int bmax_l = 1;
  for (int t = 0; t < nl; ++t) bmax_l = std::max(bmax_l, CL.bsz[t]);
  const int pull = (bmax_l <= pull_max && (split_min <= 0 || bmax_l < split_min)) ? 1 : 0;
  std::vector<std::vector<int>> rec_fs_l(pull ? nl : 0);
  // forward
  std::vector<int> f_items, rec_widx(nl, 0), fs_widx(fs.size(), 0), wcount(nl, 0);
  for (int b = 0; b < nbat; ++b) {
    for (int q = batch_ptr[b]; q < batch_ptr[b + 1]; ++q) {
      const int t = batch_cl[q];
      for (int sl = 0; sl < rec_ns_f[t]; ++sl) f_items.push_back(kSlabBase + t * 64 + sl);
    }
    for (int q = batch_ptr[b]; q < batch_ptr[b + 1]; ++q) {
      const int t = batch_cl[q];
      rec_widx[t] = wcount[t]++;
      f_items.push_back(t);
    }
    for (int f = fs_ptr[b]; f < fs_ptr[b + 1]; ++f) {
      if (pull && fs[f].seg >= 0 && bat[fs[f].seg] > b) {
        rec_fs_l[fs[f].seg].push_back(f);  // segment not processed yet: applied by its own record
        continue;
      }
      const int sg = fs[f].seg >= 0 ? fs[f].seg : -1 - fs[f].seg;
      fs_widx[f] = wcount[sg]++;
      f_items.push_back(-1 - f);
    }
  }
  std::vector<int> rec_fs_ptr(nl + 1, 0), rec_fs;
  for (int t = 0; t < nl; ++t) {
    if (pull) rec_fs.insert(rec_fs.end(), rec_fs_l[t].begin(), rec_fs_l[t].end());
    rec_fs_ptr[t + 1] = static_cast<int>(rec_fs.size());
  }
  // backward: per record its C entries then the self block
  std::vector<int> b_items, slot_m, slot_c, rec_slot0(nl, 0), rec_nslot(nl, 0), reader_need(nl, 0);
  std::vector<unsigned char> slot_final;
  std::vector<long long> slot_off;
  std::vector<int> slot_of_rec(nl, 0);
  long long poff = 0;
  for (int t = 0; t < nl; ++t) {
    const int e = CL.bsz[t] - CL.kfin[t];
    rec_slot0[t] = (int)slot_m.size();
    if (e > 0) {
      for (int a = CL.C_ptr[t]; a < CL.C_ptr[t + 1]; ++a) {
        const int c = CL.C_nb[a];
        slot_m.push_back(t), slot_c.push_back(a);
        const bool fin = bat[c] > bat[t];
        slot_final.push_back(fin ? 1 : 0);
        if (!fin) ++reader_need[c];
        slot_off.push_back(poff), poff += e;
      }
      if (CL.kfin[t] > 0) slot_m.push_back(t), slot_c.push_back(-1), slot_final.push_back(0), slot_off.push_back(poff), poff += e;
    }
    rec_nslot[t] = (int)slot_m.size() - rec_slot0[t];
  }
  for (int b = nbat - 1; b >= 0; --b) {
    for (int q = batch_ptr[b]; q < batch_ptr[b + 1]; ++q) {
      const int t = batch_cl[q];
      for (int u = 0; u < rec_nslot[t]; ++u) b_items.push_back(-1 - (rec_slot0[t] + u));
    }
    for (int q = batch_ptr[b]; q < batch_ptr[b + 1]; ++q) b_items.push_back(batch_cl[q]);
    for (int q = batch_ptr[b]; q < batch_ptr[b + 1]; ++q)
      for (int sl = 0; sl < rec_ns_b[batch_cl[q]]; ++sl) b_items.push_back(kSlabBase + batch_cl[q] * 64 + sl);
  }
  if (slot_off.empty()) slot_off.push_back(0);
  Packer pk;
  const size_t o_fi = pk.add(f_items), o_rw = pk.add(rec_widx), o_fw = pk.add(fs_widx), o_bi = pk.add(b_items), o_sm = pk.add(slot_m),
               o_sc = pk.add(slot_c), o_sf = pk.add(slot_final), o_so = pk.add(slot_off), o_r0 = pk.add(rec_slot0), o_rn = pk.add(rec_nslot),
               o_rd = pk.add(reader_need), o_nf = pk.add(rec_ns_f), o_nb = pk.add(rec_ns_b), o_fp = pk.add(rec_fs_ptr), o_ff = pk.add(rec_fs);
  pk.upload(CL.flow_meta, st);
  const DBuf& m = CL.flow_meta;
  CL.flow = SolveFlow{(int)f_items.size(), at<int>(m, o_fi), at<int>(m, o_rw), at<int>(m, o_fw), (int)b_items.size(), at<int>(m, o_bi),
                      at<int>(m, o_sm), at<int>(m, o_sc), at<unsigned char>(m, o_sf), at<long long>(m, o_so), at<int>(m, o_r0), at<int>(m, o_rn),
                      at<int>(m, o_rd), at<int>(m, o_nf), at<int>(m, o_nb), pull, at<int>(m, o_fp), at<int>(m, o_ff)};
  CL.flow_part = (size_t)std::max<long long>(poff, 1);
}

// ============================================== FactorizeHooks debug state
// What a hook sees (FactorState, factorization.hpp:115-251): the current
// level's device pools and the host bookkeeping of the driver.
struct h2g_state {
  h2g_context* ctx = nullptr;
  const h2g_matrix* M = nullptr;
  const LevelData* cur = nullptr;       // level pools (dense D, fill F, V0)
  const LevelSym* Y = nullptr;          // level structure
  int level = 0;
  const int* d_kfin = nullptr;          // device kfin (nullptr after a merge: kfin = korig)
  const std::vector<char>* rotated = nullptr;
  const std::vector<int>* elim = nullptr;  // eliminated count per cluster (0 until eliminated)
  const cplx* chain = nullptr;          // level chain arena (Qtilde)
  const std::vector<long long>* Qt_off = nullptr;
  const std::vector<int64_t>* perm_src = nullptr;  // after_merge: the permutation just applied
};

namespace {

using cx = std::complex<double>;

std::vector<cx> dl(const void* dev, size_t elems, cudaStream_t st) {
  std::vector<cx> h(elems);
  if (elems) CK(cudaMemcpyAsync(h.data(), dev, elems * 16, cudaMemcpyDefault, st));
  return h;
}

// FactorState::paint / shadow (factorization.hpp:177-245) from device blocks.
std::vector<cx> state_shadow(const h2g_state& S) {
  const h2g_matrix& M = *S.M;
  const Structure& T = M.S;
  const LevelData& cur = *S.cur;
  const LevelSym& Y = *S.Y;
  const int64_t n = T.n;
  if (n > 4096) throw Error(H2G_ERR_SIZE_GUARD, fmt("shadow: n = %lld exceeds the guard 4096", n));
  cudaStream_t st = S.ctx->stream;
  const int nl = Y.nl, l = S.level, first = Y.first;
  std::vector<int> kf(cur.korig);
  if (S.d_kfin) CK(cudaMemcpyAsync(kf.data(), S.d_kfin, nl * 4, cudaMemcpyDeviceToHost, st));
  const auto D = dl(cur.D.p, cur.D.bytes / 16, st);
  const auto F = dl(cur.F.p, cur.F.bytes / 16, st);
  std::vector<int> fex(Y.frow.size(), 0);
  if (!fex.empty()) CK(cudaMemcpyAsync(fex.data(), cur.fex.p, fex.size() * 4, cudaMemcpyDeviceToHost, st));
  const size_t bb = (size_t)cur.bmax * cur.bmax;
  const auto V0 = dl(cur.V0.p, cur.V0.bytes / 16, st);
  const auto B = dl(M.basis.p, M.basis_elems, st);
  const auto Cp = dl(M.coup.p, M.coup_elems, st);
  CK(cudaStreamSynchronize(st));
  std::vector<std::vector<cx>> Q(nl);
  for (int t = 0; t < nl; ++t)
    if ((*S.rotated)[t]) {
      Q[t] = dl(S.chain + (*S.Qt_off)[t], (size_t)cur.bsz[t] * cur.bsz[t], st);
      CK(cudaStreamSynchronize(st));
    }
  int64_t active = 0;
  for (int t = 0; t < nl; ++t) active = std::max<int64_t>(active, cur.pos[t] + cur.bsz[t]);
  std::vector<cx> Z((size_t)n * n, 0.0);
  for (int64_t p = active; p < n; ++p) Z[p + p * n] = 1.0;
  auto kor = [&](int id) { return (int)M.basis_rank[id]; };
  // place_block (:177-188): rotate a projected side and zero its eliminated part
  auto place = [&](int t, int s2, std::vector<cx> Mb) {
    const int bt = cur.bsz[t], bs = cur.bsz[s2];
    if ((*S.rotated)[t]) {
      std::vector<cx> R((size_t)bt * bs, 0.0);
      for (int j = 0; j < bs; ++j)
        for (int i = 0; i < bt; ++i) {
          cx a = 0.0;
          for (int p = 0; p < bt; ++p) a += std::conj(Q[t][p + (size_t)i * bt]) * Mb[p + (size_t)j * bt];
          R[i + (size_t)j * bt] = i < bt - kf[t] ? cx(0.0) : a;
        }
      Mb.swap(R);
    }
    if ((*S.rotated)[s2]) {
      std::vector<cx> R((size_t)bt * bs, 0.0);
      for (int j = 0; j < bs; ++j)
        for (int i = 0; i < bt; ++i) {
          cx a = 0.0;
          for (int p = 0; p < bs; ++p) a += Mb[i + (size_t)p * bt] * std::conj(Q[s2][p + (size_t)j * bs]);
          R[i + (size_t)j * bt] = j < bs - kf[s2] ? cx(0.0) : a;
        }
      Mb.swap(R);
    }
    for (int j = 0; j < bs; ++j)
      for (int i = 0; i < bt; ++i) Z[(cur.pos[t] + i) + (size_t)(cur.pos[s2] + j) * n] = Mb[i + (size_t)j * bt];
  };
  // dense blocks (in place on the device, already in their current frames)
  for (size_t q = 0; q < Y.drow.size(); ++q) {
    const int r = Y.drow[q], c = Y.dcol[q];
    for (int j = 0; j < cur.bsz[c]; ++j)
      for (int i = 0; i < cur.bsz[r]; ++i) Z[(cur.pos[r] + i) + (size_t)(cur.pos[c] + j) * n] = D[cur.doff[q] + i + (size_t)j * cur.bsz[r]];
  }
  // expanded level-entry bases of this level's clusters to an ancestor
  // level la (expand_to_level, :191-201): E (bsz_u x k_anc)
  auto expand = [&](int u, int la) {
    const int b = cur.bsz[u];
    std::vector<cx> E((size_t)b * kor(first + u));
    const int k0 = kor(first + u);
    for (int j = 0; j < k0; ++j)
      for (int i = 0; i < b; ++i) E[i + (size_t)j * b] = V0[u * bb + i + (size_t)j * b];
    int id = first + u, kc = k0;
    for (int lv = l; lv > la; --lv) {
      const int par = (id - 1) / 2, kp = kor(par);
      const int roff = (id == 2 * par + 1) ? 0 : kor(2 * par + 1);
      const int rows = (int)M.basis_rows[par];
      std::vector<cx> E2((size_t)b * kp, 0.0);
      for (int j = 0; j < kp; ++j)
        for (int p = 0; p < kc; ++p) {
          const cx tv = B[M.basis_off[par] + roff + p + (size_t)j * rows];
          for (int i = 0; i < b; ++i) E2[i + (size_t)j * b] += E[i + (size_t)p * b] * tv;
        }
      E.swap(E2);
      id = par, kc = kp;
    }
    return E;
  };
  auto fill_of = [&](int r, int c) {
    const int f = Y.fill_index(r, c);
    return (f >= 0 && fex[f] && cur.foff[f] >= 0) ? f : -1;
  };
  const int lmin = T.l0 >= 0 ? T.l0 : l + 1;
  for (int la = lmin; la <= l; ++la) {
    for (size_t pq = 0; pq < T.adm[la].size(); ++pq) {
      const int R = T.adm[la][pq].row, Cc = T.adm[la][pq].col;
      const int kr = kor(R), kc2 = kor(Cc);
      const cx* Sm = reinterpret_cast<const cx*>(Cp.data()) + M.coup_off[T.adm_offset[la] + pq];
      const int span = 1 << (l - la);
      const int u0 = ((R + 1) << (l - la)) - 1 - first, v0 = ((Cc + 1) << (l - la)) - 1 - first;
      for (int u = u0; u < u0 + span; ++u) {
        const auto Eu = expand(u, la);
        // X = Eu S (bsz_u x kc2)
        std::vector<cx> X((size_t)cur.bsz[u] * kc2, 0.0);
        for (int j = 0; j < kc2; ++j)
          for (int p = 0; p < kr; ++p) {
            const cx sv = Sm[p + (size_t)j * kr];
            for (int i = 0; i < cur.bsz[u]; ++i) X[i + (size_t)j * cur.bsz[u]] += Eu[i + (size_t)p * cur.bsz[u]] * sv;
          }
        for (int v = v0; v < v0 + span; ++v) {
          const auto Ev = expand(v, la);
          const int bu = cur.bsz[u], bv = cur.bsz[v];
          std::vector<cx> Mb((size_t)bu * bv, 0.0);
          for (int j = 0; j < bv; ++j)
            for (int p = 0; p < kc2; ++p) {
              const cx ev = Ev[j + (size_t)p * bv];
              for (int i = 0; i < bu; ++i) Mb[i + (size_t)j * bu] += X[i + (size_t)p * bu] * ev;
            }
          const int f = fill_of(u, v);
          if (f >= 0)
            for (int j = 0; j < bv; ++j)
              for (int i = 0; i < bu; ++i) Mb[i + (size_t)j * bu] += F[cur.foff[f] + i + (size_t)j * bu];
          place(u, v, std::move(Mb));
        }
      }
    }
  }
  return Z;
}

}  // namespace

// ================================================================ C ABI
extern "C" {

const char* h2g_version(void) { return "h2g 0.1 (sm_100a)"; }

int h2g_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int h2g_last_error(h2g_error* err) {
  if (err) *err = g_last;
  return g_last.code;
}

int h2g_context_create(int device, h2g_context** out, h2g_error* err) {
  return guarded(err, [&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) throw Error(H2G_ERR_CUDA, "no CUDA device available (h2g has no CPU fallback)");
    if (device < 0 || device >= n) throw Error(H2G_ERR_INVALID_INPUT, "bad device index");
    CK(cudaSetDevice(device));
    auto* c = new h2g_context();
    c->device = device;
    int prio_lo = 0, prio_hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    CK(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_hi));
    CK(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, prio_lo));
    CK(cudaEventCreateWithFlags(&c->ev_crit, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_bulk, cudaEventDisableTiming));
    CK(cudaStreamCreateWithPriority(&c->aux, cudaStreamNonBlocking, prio_hi));
    CK(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c->ev_aux0, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_aux1, cudaEventDisableTiming));
    BlockCache::get().add_stream(c->stream, device);
    CK(cudaEventCreate(&c->ev0));
    CK(cudaEventCreate(&c->ev1));
    CK(cudaMalloc(&c->d_err, sizeof(DevError)));
    CK(cudaMemset(c->d_err, 0, sizeof(DevError)));
    CK(cudaMalloc(&c->d_flag, 64));
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    *out = c;
  });
}

}  // extern "C"

static void context_teardown(h2g_context* ctx) {
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->side);
  cudaStreamSynchronize(ctx->stream);
  BlockCache::get().remove_stream(ctx->stream);
  cudaEventDestroy(ctx->ev_crit);
  cudaEventDestroy(ctx->ev_bulk);
  cudaStreamSynchronize(ctx->aux);
  cudaEventDestroy(ctx->ev_aux0);
  cudaEventDestroy(ctx->ev_aux1);
  cudaStreamDestroy(ctx->aux);
  if (ctx->copy) cudaStreamDestroy(ctx->copy);
  cudaStreamDestroy(ctx->side);
  cudaFree(ctx->d_err);
  cudaFree(ctx->d_flag);
  cudaEventDestroy(ctx->ev0);
  cudaEventDestroy(ctx->ev1);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
}

static void context_release(h2g_context* ctx) {
  if (ctx && --ctx->refs == 0) context_teardown(ctx);
}

extern "C" {

int h2g_context_destroy(h2g_context* ctx) {
  context_release(ctx);
  return H2G_OK;
}

int h2g_matrix_upload(h2g_context* ctx, const h2g_matrix_desc* d, h2g_matrix** out, h2g_error* err) {
  return guarded(err, [&] {
    if (!ctx || !d || !out) throw Error(H2G_ERR_INVALID_INPUT, "null argument");
    CK(cudaSetDevice(ctx->device));
    auto M = std::make_unique<h2g_matrix>();
    M->ctx = ctx;
    M->S = structure_from_desc(d);
    M->eps_h2 = d->eps_h2;
    const Structure& S = M->S;
    const int nc = S.num_clusters();
    M->basis_rows.assign(d->basis_rows, d->basis_rows + nc);
    M->basis_rank.assign(d->basis_rank, d->basis_rank + nc);
    M->basis_off.assign(d->basis_offset, d->basis_offset + nc);
    for (int id = 0; id < nc; ++id) {
      const bool leaf = id >= Structure::first(S.depth);
      const int64_t rows = leaf ? S.end[id] - S.begin[id] : M->basis_rank[2 * id + 1] + M->basis_rank[2 * id + 2];
      if (M->basis_rows[id] != rows) throw Error(H2G_ERR_INVALID_INPUT, fmt("basis of cluster %lld has %lld rows", id, M->basis_rows[id]));
      M->basis_elems = std::max<int64_t>(M->basis_elems, M->basis_off[id] + rows * M->basis_rank[id]);
    }
    const int64_t na = S.num_adm();
    M->coup_off.assign(d->coupling_offset, d->coupling_offset + na);
    for (int l = 0; l <= S.depth; ++l)
      for (size_t q = 0; q < S.adm[l].size(); ++q) {
        const int64_t g = S.adm_offset[l] + static_cast<int64_t>(q);
        M->coup_elems = std::max<int64_t>(M->coup_elems, M->coup_off[g] + M->basis_rank[S.adm[l][q].row] * M->basis_rank[S.adm[l][q].col]);
      }
    M->dense_off.assign(d->dense_offset, d->dense_offset + d->num_leaf_pairs);
    for (size_t q = 0; q < S.leaf.size(); ++q) {
      const auto& p = S.leaf[q];
      M->dense_elems = std::max<int64_t>(M->dense_elems, M->dense_off[q] + (S.end[p.row] - S.begin[p.row]) * (S.end[p.col] - S.begin[p.col]));
    }
    cudaStream_t s = ctx->stream;
    M->basis.alloc(std::max<int64_t>(M->basis_elems, 1) * 16, s);
    M->coup.alloc(std::max<int64_t>(M->coup_elems, 1) * 16, s);
    M->dense.alloc(std::max<int64_t>(M->dense_elems, 1) * 16, s);
    if (M->basis_elems) CK(cudaMemcpyAsync(M->basis.p, d->basis_data, M->basis_elems * 16, cudaMemcpyHostToDevice, s));
    if (M->coup_elems) CK(cudaMemcpyAsync(M->coup.p, d->coupling_data, M->coup_elems * 16, cudaMemcpyHostToDevice, s));
    if (M->dense_elems) CK(cudaMemcpyAsync(M->dense.p, d->dense_data, M->dense_elems * 16, cudaMemcpyHostToDevice, s));
    if (d->points_tree) M->points_tree.assign(d->points_tree, d->points_tree + 3 * S.n);
    if (d->perm) M->perm.assign(d->perm, d->perm + S.n);
    M->leafsize = d->leafsize;
    CK(cudaStreamSynchronize(s));
    ++ctx->refs;  // the matrix holds the context
    *out = M.release();
  });
}

int h2g_matrix_build(h2g_context* ctx, const double* points, int64_t n, int64_t leafsize, double eta, const h2g_kernel_spec* kernel,
                     double eps_h2, h2g_matrix** out, h2g_error* err) {
  return guarded(err, [&] {
    if (!ctx || !points || !kernel || !out) throw Error(H2G_ERR_INVALID_INPUT, "null argument");
    if (eps_h2 <= 0.0) throw Error(H2G_ERR_INVALID_INPUT, "build_h2: eps_h2 must be positive");
    CK(cudaSetDevice(ctx->device));
    auto M = std::make_unique<h2g_matrix>();
    M->ctx = ctx;
    M->S = build_structure(points, n, leafsize, eta, &M->perm);
    M->eps_h2 = eps_h2;
    M->leafsize = leafsize;
    M->points_tree.resize(3 * (size_t)n);
    for (int64_t i = 0; i < n; ++i)
      for (int a = 0; a < 3; ++a) M->points_tree[3 * i + a] = points[3 * M->perm[i] + a];
    BuildResult R = build_h2_device(M->S, points, M->perm, *kernel, eps_h2, ctx->stream);
    M->basis_rows = std::move(R.basis_rows);
    M->basis_rank = std::move(R.basis_rank);
    M->basis_off = std::move(R.basis_off);
    M->coup_off = std::move(R.coup_off);
    M->dense_off = std::move(R.dense_off);
    M->basis_elems = R.basis_elems;
    M->coup_elems = R.coup_elems;
    M->dense_elems = R.dense_elems;
    M->basis.p = R.basis;
    M->basis.s = ctx->stream;
    M->coup.p = R.coup;
    M->coup.s = ctx->stream;
    M->dense.p = R.dense;
    M->dense.s = ctx->stream;
    ++ctx->refs;  // the matrix holds the context
    *out = M.release();
  });
}

int h2g_matrix_destroy(h2g_matrix* m) {
  if (!m) return H2G_OK;
  h2g_context* ctx = m->ctx;
  cudaSetDevice(ctx->device);
  delete m;
  context_release(ctx);
  return H2G_OK;
}

int h2g_matrix_sizes(const h2g_matrix* m, int64_t* s) {
  if (!m || !s) return H2G_ERR_INVALID_INPUT;
  s[0] = m->S.n;
  s[1] = m->S.depth;
  s[2] = m->S.num_clusters();
  s[3] = m->S.num_adm();
  s[4] = static_cast<int64_t>(m->S.leaf.size());
  s[5] = m->basis_elems;
  s[6] = m->coup_elems;
  s[7] = m->dense_elems;
  return H2G_OK;
}

int h2g_matrix_download(const h2g_matrix* m, int64_t* cb, int64_t* ce, int64_t* perm, int64_t* adm_off, int32_t* adm_pairs, int64_t* split_off,
                        int32_t* split_pairs, int32_t* leaf_pairs, int64_t* basis_rows, int64_t* basis_rank, int64_t* basis_offset,
                        double* basis_data, int64_t* coupling_offset, double* coupling_data, int64_t* dense_offset, double* dense_data) {
  return guarded(nullptr, [&] {
    const Structure& S = m->S;
    const int nc = S.num_clusters();
    cudaStream_t s = m->ctx->stream;
    if (cb) std::copy(S.begin.begin(), S.begin.begin() + nc, cb);
    if (ce) std::copy(S.end.begin(), S.end.begin() + nc, ce);
    if (perm) {
      if (m->perm.empty())
        for (int64_t i = 0; i < S.n; ++i) perm[i] = i;
      else
        std::copy(m->perm.begin(), m->perm.end(), perm);
    }
    int64_t qa = 0, qs = 0;
    for (int l = 0; l <= S.depth; ++l) {
      if (adm_off) adm_off[l] = qa;
      if (split_off) split_off[l] = qs;
      for (const auto& p : S.adm[l]) {
        if (adm_pairs) adm_pairs[2 * qa] = p.row, adm_pairs[2 * qa + 1] = p.col;
        ++qa;
      }
      for (const auto& p : S.split[l]) {
        if (split_pairs) split_pairs[2 * qs] = p.row, split_pairs[2 * qs + 1] = p.col;
        ++qs;
      }
    }
    if (adm_off) adm_off[S.depth + 1] = qa;
    if (split_off) split_off[S.depth + 1] = qs;
    if (leaf_pairs)
      for (size_t q = 0; q < S.leaf.size(); ++q) leaf_pairs[2 * q] = S.leaf[q].row, leaf_pairs[2 * q + 1] = S.leaf[q].col;
    if (basis_rows) std::copy(m->basis_rows.begin(), m->basis_rows.end(), basis_rows);
    if (basis_rank) std::copy(m->basis_rank.begin(), m->basis_rank.end(), basis_rank);
    if (basis_offset) std::copy(m->basis_off.begin(), m->basis_off.end(), basis_offset);
    if (coupling_offset) std::copy(m->coup_off.begin(), m->coup_off.end(), coupling_offset);
    if (dense_offset) std::copy(m->dense_off.begin(), m->dense_off.end(), dense_offset);
    if (basis_data && m->basis_elems) CK(cudaMemcpyAsync(basis_data, m->basis.p, m->basis_elems * 16, cudaMemcpyDeviceToHost, s));
    if (coupling_data && m->coup_elems) CK(cudaMemcpyAsync(coupling_data, m->coup.p, m->coup_elems * 16, cudaMemcpyDeviceToHost, s));
    if (dense_data && m->dense_elems) CK(cudaMemcpyAsync(dense_data, m->dense_ptr(), m->dense_elems * 16, cudaMemcpyDefault, s));
    CK(cudaStreamSynchronize(s));
  });
}

int h2g_matvec(h2g_context* ctx, const h2g_matrix* m, const double* x, double* y, int32_t nrhs, h2g_error* err) {
  return guarded(err, [&] {
    if (!ctx || !m || !x || !y || nrhs < 1) throw Error(H2G_ERR_INVALID_INPUT, "matvec: bad arguments");
    CK(cudaSetDevice(ctx->device));
    matvec_device(m->S, m->basis_rows, m->basis_rank, m->basis_off, m->coup_off, m->dense_off, m->basis.as<cplx>(), m->coup.as<cplx>(),
                  m->dense_ptr(), x, y, nrhs, ctx->stream);
  });
}

int h2g_kernel_rows_matvec(h2g_context* ctx, const double* points_tree, int64_t n, const h2g_kernel_spec* kernel, const int64_t* rows,
                           int64_t nrows, const double* x, double* y, int32_t nrhs, h2g_error* err) {
  return guarded(err, [&] {
    if (!ctx || !points_tree || !kernel || (nrows && (!rows || !y)) || !x || n < 1 || nrows < 0 || nrhs < 1)
      throw Error(H2G_ERR_INVALID_INPUT, "kernel_rows_matvec: bad arguments");
    CK(cudaSetDevice(ctx->device));
    kernel_rows_matvec_device(points_tree, n, *kernel, rows, nrows, x, y, nrhs, ctx->stream);
  });
}

// ------------------------------------------------------------- factorize
}  // extern "C"

static int factorize_impl(h2g_context* ctx, const h2g_matrix* mc, double eps, int32_t stop_level, int32_t schedule, const h2g_factorize_hooks* hooks,
                          h2g_chain** out, h2g_error* err, const h2g_dist* dist = nullptr) {
  return guarded(err, [&] {
    if (!ctx || !mc || !out) throw Error(H2G_ERR_INVALID_INPUT, "null argument");
    if (!(eps > 0.0)) throw Error(H2G_ERR_INVALID_INPUT, "factorize: eps_fill_in must be positive");
    if (schedule != H2G_SCHEDULE_REFERENCE && schedule != H2G_SCHEDULE_COLORED && schedule != H2G_SCHEDULE_SERIAL &&
        schedule != H2G_SCHEDULE_INTERIOR_FIRST && schedule != H2G_SCHEDULE_SUBTREE)
      throw Error(H2G_ERR_INVALID_INPUT, "factorize: unknown schedule");
    if (hooks) schedule = H2G_SCHEDULE_SERIAL;  // debug mode: one cluster per step, reference order
    if (dist) {
      if (dist->nranks != 1 && dist->nranks != 2 && dist->nranks != 4 && dist->nranks != 8)
        throw Error(H2G_ERR_INVALID_INPUT, "factorize_dist: nranks must be 1, 2, 4 or 8 (the 8 level-3 subtrees are dealt to the ranks)");
      if (dist->rank < 0 || dist->rank >= dist->nranks) throw Error(H2G_ERR_INVALID_INPUT, "factorize_dist: rank outside [0, nranks)");
      if (dist->nranks > 1 && !dist->exchange) throw Error(H2G_ERR_INVALID_INPUT, "factorize_dist: exchange callback missing");
      schedule = H2G_SCHEDULE_SUBTREE;
    }
    std::lock_guard<std::recursive_mutex> run_lock(ctx->run_mu);
    CK(cudaSetDevice(ctx->device));
    NvtxRange nv_factor("h2g factorize");
    h2g_matrix* M = const_cast<h2g_matrix*>(mc);
    const Structure& S = M->S;
    const int L = S.depth, l0 = S.l0;
    int stop = L + 1;
    if (l0 >= 0) {
      stop = stop_level >= 0 ? stop_level : l0;
      if (stop < l0 || stop > L)
        throw Error(H2G_ERR_INVALID_INPUT, fmt("factorize: stop level %lld outside [l0, depth] = [%lld, depth]", stop, l0));
    }
    cudaStream_t st = ctx->stream;
    const auto tp0 = std::chrono::steady_clock::now();
    bool plan_built = false;
    PlanCache* P = get_plan(M, stop, schedule, &plan_built);
    const double plan_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - tp0).count();
    if (std::getenv("H2G_VERBOSE")) std::fprintf(stderr, "[h2g] plan %.3f s (%s)\n", plan_s, plan_built ? "built" : "cached");

    auto C = std::make_unique<h2g_chain>();
    C->ctx = ctx;
    C->n = S.n;
    C->stop_level = stop;
    C->schedule = schedule;
    C->depth = L;
    C->eps = eps;
    C->plan_ms = plan_s * 1e3;
    C->tree_perm = M->perm;
    C->plan_built = plan_built;
    CK(cudaMemsetAsync(ctx->d_err, 0, sizeof(DevError), st));
    ctx->prof.reset();
    ctx->prof_side.reset();
    ctx->prof_side.on = ctx->prof.on;
    ctx->prof_aux.reset();
    ctx->prof_aux.on = ctx->prof.on;
    CK(cudaEventRecord(ctx->ev0, st));
    long long launches = 0;
    double flops = 0.0, sflops = 0.0, sbytes = 0.0;

    // ---- leaf level entry state
    LevelData cur;
    {
      const int nl = 1 << L, first = Structure::first(L);
      cur.bsz.resize(nl);
      cur.korig.resize(nl);
      cur.pos.resize(nl);
      for (int t = 0; t < nl; ++t) {
        cur.bsz[t] = static_cast<int>(S.end[first + t] - S.begin[first + t]);
        cur.korig[t] = static_cast<int>(M->basis_rank[first + t]);
        cur.pos[t] = S.begin[first + t];
      }
      cur.bmax = std::max(1, *std::max_element(cur.bsz.begin(), cur.bsz.end()));
      const size_t bb = (size_t)cur.bmax * cur.bmax * 16;
      const LevelSym& Y = P->levels[0];
      const long long dtot = pack_offsets(Y.drow, Y.dcol, cur.bsz, cur.doff);
      cur.D.alloc(std::max<long long>(dtot, 1) * 16, st, true);
      cur.V0.alloc((size_t)nl * bb, st, true);
      std::vector<CopyDesc> cd;
      for (size_t q = 0; q < Y.drow.size(); ++q) {
        const int r = Y.drow[q], c = Y.dcol[q];
        cd.push_back({M->dense_ptr() + M->dense_off[q], cur.D.as<cplx>() + cur.doff[q], cur.bsz[r], cur.bsz[r], cur.bsz[r], cur.bsz[c], 0, 0});
      }
      for (int t = 0; t < nl; ++t)
        if (cur.korig[t] > 0)
          cd.push_back({M->basis.as<cplx>() + M->basis_off[first + t], at<cplx>(cur.V0, t * bb), cur.bsz[t], cur.bsz[t], cur.bsz[t], cur.korig[t], 0, 0});
      DBuf dd;
      upload(dd, cd, st);
      launch_copy(dd.as<CopyDesc>(), static_cast<int>(cd.size()), st);
      ++launches;
      cur.fex_host.assign(Y.frow.size(), 0);
      if (stop <= L) {
        cur.front = build_front(Y, P->sched[0], P->work[0], cur.bsz, {});
        cur.has_front = true;
        cur.foff = cur.front.foff;
        cur.F.alloc(std::max<long long>(cur.front.pool_elems, 1) * 16, st, true);
      } else {
        const long long ftot = pack_offsets(Y.frow, Y.fcol, cur.bsz, cur.foff);
        cur.F.alloc(std::max<long long>(ftot, 1) * 16, st, true);
      }
      cur.fex.alloc(std::max<size_t>(Y.frow.size(), 1) * 4, st, true);
      CK(cudaStreamSynchronize(st));
    }

    int li = 0;
    int last_level = L;  // level whose state is "cur" at the root
    // HBM budget: when the next allocation would not fit, finished levels'
    // chains move to pinned host memory (oldest first); the solve then reads
    // them over the host link (config 3 only; configs 1-2 never trigger this)
    const size_t kMargin = size_t(8) << 30;
    size_t offloaded = 0;
    auto offload_chain = [&](ChainLevelHost& X) {
      X.harena.alloc(X.arena.bytes);
      CK(cudaMemcpyAsync(X.harena.p, X.arena.p, X.arena.bytes, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      offloaded += X.arena.bytes;
      X.arena.release();
      X.sl.chain = X.harena.as<cplx>();
    };
    struct SpillGuard {
      cudaStream_t s;
      ~SpillGuard() { BlockCache::get().set_spill(s, nullptr); }
    } spill_guard{st};
    // the input's dense blocks are only read at the leaf-level entry (and by
    // the matvec); they are the second thing to leave HBM
    auto offload_dense = [&]() -> bool {
      if (M->hdense.p || !M->dense.p || M->dense_elems == 0) return false;
      M->hdense.alloc(M->dense_elems * 16);
      CK(cudaMemcpyAsync(M->hdense.p, M->dense.p, M->dense_elems * 16, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      M->dense.release();
      return true;
    };
    // one device chunk of a finished streamed level to pinned host memory
    auto offload_chunk = [&]() -> bool {
      for (auto& X : C->levels)
        for (auto& ck : X->chunks)
          if (ck.d.p) {
            ck.h.alloc(ck.d.bytes);
            CK(cudaMemcpyAsync(ck.h.p, ck.d.p, ck.d.bytes, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            offloaded += ck.d.bytes;
            ck.d.release();
            return true;
          }
      return false;
    };
    BlockCache::get().set_spill(st, [&]() -> bool {
      for (auto& X : C->levels)
        if (X->arena.p) {
          offload_chain(*X);
          return true;
        }
      if (offload_chunk()) return true;
      return offload_dense();
    });
    auto ensure = [&](size_t need, ChainLevelHost* extra) {
      if (BlockCache::get().headroom() >= need + kMargin) return;
      CK(cudaStreamSynchronize(st));
      BlockCache::get().trim();
      for (auto& X : C->levels) {
        if (BlockCache::get().headroom() >= need + kMargin) return;
        if (X->arena.p) offload_chain(*X), BlockCache::get().trim();
      }
      while (BlockCache::get().headroom() < need + kMargin && offload_chunk()) BlockCache::get().trim();
      if (extra && extra->arena.p && BlockCache::get().headroom() < need + kMargin) offload_chain(*extra), BlockCache::get().trim();
      if (BlockCache::get().headroom() < need + kMargin && offload_dense()) BlockCache::get().trim();
    };
    const int verbose = std::getenv("H2G_VERBOSE") ? std::atoi(std::getenv("H2G_VERBOSE")) : 0;
    auto wall = [] { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
    double tlev = wall();
    auto mark = [&](const char* what) {
      if (verbose >= 2) std::fprintf(stderr, "[h2g]   %-28s %.4f s\n", what, wall() - tlev);
    };
    std::vector<cplx*> core_ptr_h;  // per fill of the running level: its compact core (host copy of DevLevel::core_ptr)
    std::vector<DBuf> core_chunks;   // the cores, one chunk per segment; released after the merge
    std::vector<HBuf> core_hchunks;  // ... or in pinned host memory when HBM is short (pages of kCorePage bytes)
    const size_t kCorePage = kStagePage;
    char* core_page = nullptr;  // the page being filled (belongs to core_hchunks)
    size_t core_page_used = 0;
    if (stop <= L) {
      for (int l = L; l >= stop; --l, ++li) {
        NvtxRange nv_level("h2g level " + std::to_string(l));
        const LevelSym& Y = P->levels[li];
        const LevelSchedule& SC = P->sched[li];
        const LevelWork& W = P->work[li];
        const int nl = Y.nl;
        const int bm = cur.bmax;
        const size_t bb = (size_t)bm * bm;
        // ---- chain offsets (upper bound e <= b - korig)
        std::vector<long long> Qt_off(nl), L11_off(nl), U11_off(nl), Linv_off(nl), Uinv_off(nl), Lself_off(nl), Uself_off(nl);
        std::vector<long long> Lbar_off(Y.R_nb.size()), Ubar_off(Y.C_nb.size());
        long long top = 0;
        auto place = [&](int t) {  // everything of cluster t but Qt
          const long long b = cur.bsz[t], em = b - cur.korig[t];
          L11_off[t] = top, top += em * em;
          U11_off[t] = top, top += em * em;
          Linv_off[t] = top, top += em * em;
          Uinv_off[t] = top, top += em * em;
          Lself_off[t] = top, top += b * em;
          Uself_off[t] = top, top += b * em;
          for (int a = Y.R_ptr[t]; a < Y.R_ptr[t + 1]; ++a) Lbar_off[a] = top, top += (long long)cur.bsz[Y.R_nb[a]] * em;
          for (int a = Y.C_ptr[t]; a < Y.C_ptr[t + 1]; ++a) Ubar_off[a] = top, top += (long long)cur.bsz[Y.C_nb[a]] * em;
        };
        // Streamed chain (large segmented levels): only Qt, which later
        // clusters' lifts and the collapse read, stays on the device for the
        // whole level. Everything else of a cluster is read inside its own
        // batch only (and by the solve), so it is laid out in elimination
        // order, written to one of two device halves (segment parity) and
        // copied to the level's pinned host arena when its segment ends.
        // Logical layout (host arena, solve offsets): [all Qt | segment 0 | segment 1 | ...].
        const int stream_env = std::getenv("H2G_CHAIN_STREAM") ? std::atoi(std::getenv("H2G_CHAIN_STREAM")) : -1;  // 0 never, 1 always
        long long qtot = 0;
        for (int t = 0; t < nl; ++t) qtot += (long long)cur.bsz[t] * cur.bsz[t];
        bool streamed = false;
        if (cur.has_front && cur.front.K > 1 && !hooks && stream_env != 0) {
          long long ub = qtot;
          for (int t = 0; t < nl; ++t) {
            const long long b = cur.bsz[t], em = b - cur.korig[t];
            ub += 4 * em * em + 2 * b * em;
            for (int a = Y.R_ptr[t]; a < Y.R_ptr[t + 1]; ++a) ub += (long long)cur.bsz[Y.R_nb[a]] * em;
            for (int a = Y.C_ptr[t]; a < Y.C_ptr[t + 1]; ++a) ub += (long long)cur.bsz[Y.C_nb[a]] * em;
          }
          size_t fr = 0, tot = 0;
          cudaMemGetInfo(&fr, &tot);
          streamed = stream_env > 0 || (double)ub * 16 > 0.08 * (double)tot;
        }
        std::vector<long long> seg_begin, seg_len;  // streamed: logical start / length of every segment's part (elements)
        long long ring_half = 0;
        if (!streamed) {
          for (int t = 0; t < nl; ++t) {
            Qt_off[t] = top, top += (long long)cur.bsz[t] * cur.bsz[t];
            place(t);
          }
        } else {
          for (int t = 0; t < nl; ++t) Qt_off[t] = top, top += (long long)cur.bsz[t] * cur.bsz[t];
          const int Kc = cur.front.K;
          const int nbat1 = static_cast<int>(SC.batch_ptr.size()) - 1;
          for (int sg = 0; sg < Kc; ++sg) {
            seg_begin.push_back(top);
            for (int bi = cur.front.seg_first_batch[sg]; bi < cur.front.seg_first_batch[sg + 1] && bi < nbat1; ++bi)
              for (int p = SC.batch_ptr[bi]; p < SC.batch_ptr[bi + 1]; ++p) place(SC.batch_cl[p]);
            seg_len.push_back(top - seg_begin.back());
            ring_half = std::max(ring_half, seg_len.back());
          }
        }
        // offsets of the finished chain (host copies, solve). Resident level:
        // the device offsets. Streamed level: the compact layout [all Qt |
        // segment 0 | segment 1 | ...] with every block at its final size
        // (e = b - kfin instead of the bound b - korig), filled in as the
        // segments end.
        std::vector<long long> lQt(Qt_off), lL11(L11_off), lU11(U11_off), lLinv(Linv_off), lUinv(Uinv_off), lLself(Lself_off),
            lUself(Uself_off), lLbar(Lbar_off), lUbar(Ubar_off);
        const long long top_logical = top;
        long long compact_top = qtot;
        if (streamed) {
          std::vector<int> seg_of(nl, 0);
          for (int sg = 0; sg < cur.front.K; ++sg)
            for (int bi = cur.front.seg_first_batch[sg]; bi < cur.front.seg_first_batch[sg + 1] && bi + 1 < (int)SC.batch_ptr.size(); ++bi)
              for (int p = SC.batch_ptr[bi]; p < SC.batch_ptr[bi + 1]; ++p) seg_of[SC.batch_cl[p]] = sg;
          auto dev = [&](long long o, int sg) { return qtot + (long long)(sg & 1) * ring_half + (o - seg_begin[sg]); };
          for (int t = 0; t < nl; ++t) {
            const int sg = seg_of[t];
            L11_off[t] = dev(L11_off[t], sg), U11_off[t] = dev(U11_off[t], sg), Linv_off[t] = dev(Linv_off[t], sg);
            Uinv_off[t] = dev(Uinv_off[t], sg), Lself_off[t] = dev(Lself_off[t], sg), Uself_off[t] = dev(Uself_off[t], sg);
            for (int a = Y.R_ptr[t]; a < Y.R_ptr[t + 1]; ++a) Lbar_off[a] = dev(Lbar_off[a], sg);
            for (int a = Y.C_ptr[t]; a < Y.C_ptr[t + 1]; ++a) Ubar_off[a] = dev(Ubar_off[a], sg);
          }
          top = qtot + 2 * ring_half;  // the device allocation
        }
        mark("offsets");
        auto CL = std::make_unique<ChainLevelHost>();
        CL->level = l;
        // lifted panels (Qt_n Lbar / Ubar Qt_n^T for neighbours n eliminated
        // earlier, deposit_fill :359-366): packed, only the lifted entries
        std::vector<long long> liftL_off(Y.R_nb.size(), -1), liftU_off(Y.C_nb.size(), -1);
        // only panels that feed a fill-in target are lifted
        std::vector<char> needL(Y.R_nb.size(), 0), needU(Y.C_nb.size(), 0);
        for (const SchurContrib& cb : W.contrib) {
          if (cb.flags & 1) needL[cb.r] = 1;
          if (cb.flags & 2) needU[cb.c] = 1;
        }
        auto lifted = [&](const PanelItem& pi) { return pi.lift && (pi.side == 0 ? needU[pi.entry] : needL[pi.entry]); };
        // a lifted panel lives only through its own batch (written by the
        // panel GEMMs, read by that batch's Schur launches; the deferred
        // launch may still read it while the next batch writes its own), so
        // the buffer is two halves used by even / odd batches
        long long lhalf = 0;
        for (size_t bi = 0; bi + 1 < SC.batch_ptr.size(); ++bi) {
          long long lb = 0;
          for (int it = W.panel_ptr[bi]; it < W.panel_ptr[bi + 1]; ++it) {
            const PanelItem& pi = W.panel[it];
            if (!lifted(pi)) continue;
            const int t = SC.batch_cl[SC.batch_ptr[bi] + pi.q];
            const long long em = cur.bsz[t] - cur.korig[t];
            (pi.side == 0 ? liftU_off : liftL_off)[pi.entry] = lb;  // half-relative, rebased below
            lb += em * cur.bsz[pi.nb];
          }
          lhalf = std::max(lhalf, lb);
        }
        for (size_t bi = 1; bi + 1 < SC.batch_ptr.size(); bi += 2)
          for (int it = W.panel_ptr[bi]; it < W.panel_ptr[bi + 1]; ++it) {
            const PanelItem& pi = W.panel[it];
            if (lifted(pi)) (pi.side == 0 ? liftU_off : liftL_off)[pi.entry] += lhalf;
          }
        const long long ltop = 2 * lhalf;
        if (verbose)
          std::fprintf(stderr, "[h2g] level %d entry: chain arena %.2f GB, lifted panels %.2f GB, complements %.2f GB; device free %.2f GB\n", l,
                       top * 16 / 1e9, ltop * 16 / 1e9, (double)nl * bb * 16 / 1e9, BlockCache::get().headroom() / 1e9);
        ensure((size_t)(std::max<long long>(top, 1) + std::max<long long>(ltop, 1) + (long long)nl * bb) * 16 + (size_t(4) << 30), nullptr);
        CL->arena.alloc(std::max<long long>(top, 1) * 16, st);
        if (streamed) {
          if (verbose)
            std::fprintf(stderr, "[h2g] level %d: chain streamed to host memory: %.2f GB on the device (Qt %.2f GB + 2 x %.2f GB) instead of %.2f GB\n", l,
                         top * 16 / 1e9, qtot * 16 / 1e9, ring_half * 16 / 1e9, top_logical * 16 / 1e9);
        }
        DBuf lift;
        lift.alloc(std::max<long long>(ltop, 1) * 16, st);
        mark("chain allocated");
        // ---- per-level device metadata
        Packer pk;
        std::vector<int> posi(nl);
        std::vector<long long> posl(cur.pos.begin(), cur.pos.end());
        size_t o_bsz = pk.add(cur.bsz), o_korig = pk.add(cur.korig), o_pos = pk.add(posl);
        std::vector<int> kfin0(cur.korig);
        size_t o_kfin = pk.add(kfin0);
        size_t o_drow = pk.add(Y.drow), o_dcol = pk.add(Y.dcol), o_diag = pk.add(Y.diag_blk);
        std::vector<long long> foff_dev(cur.foff.size());
        for (size_t f = 0; f < foff_dev.size(); ++f) foff_dev[f] = cur.foff_safe(f);
        size_t o_doff = pk.add(cur.doff), o_foff = pk.add(foff_dev);
        size_t o_frow = pk.add(Y.frow), o_fcol = pk.add(Y.fcol);
        size_t o_Rp = pk.add(Y.R_ptr), o_Rn = pk.add(Y.R_nb), o_Cp = pk.add(Y.C_ptr), o_Cn = pk.add(Y.C_nb);
        size_t o_Gp = pk.add(Y.G_ptr), o_Gf = pk.add(Y.G_fill), o_Gt = pk.add(Y.G_tr);
        size_t o_Qt = pk.add(Qt_off), o_L11 = pk.add(L11_off), o_U11 = pk.add(U11_off), o_Li = pk.add(Linv_off), o_Ui = pk.add(Uinv_off);
        size_t o_Lb = pk.add(Lbar_off), o_Ub = pk.add(Ubar_off), o_Ls = pk.add(Lself_off), o_Us = pk.add(Uself_off);
        size_t o_lL = pk.add(liftL_off), o_lU = pk.add(liftU_off);

        size_t o_bat = pk.add(SC.batch_cl);
        size_t o_sch = pk.add_raw(reinterpret_cast<const SchurTargetD*>(W.schur.data()), W.schur.size());
        size_t o_con = pk.add_raw(reinterpret_cast<const SchurContribD*>(W.contrib.data()), W.contrib.size());
        size_t o_fs = pk.add_raw(reinterpret_cast<const SolveTargetD*>(W.fsolve.data()), W.fsolve.size());
        size_t o_fc = pk.add_raw(reinterpret_cast<const SolveContribD*>(W.fcontrib.data()), W.fcontrib.size());
        mark("meta packed");
        pk.upload(CL->meta, st);
        mark("meta uploaded");
        const DBuf& mt = CL->meta;
        cur.Vp.alloc((size_t)nl * bb * 16, st, true);
        // ---- step-0 projection / Gram work (static sizes: descriptor GEMMs)
        const int nslots = static_cast<int>(SC.batch_cl.size());
        const int nbat0 = static_cast<int>(SC.batch_ptr.size()) - 1;
        std::vector<int> slot_g0(nslots), slot_gn(nslots), slot_c0(nslots), slot_cn(nslots);
        std::vector<long long> gram_off;
        std::vector<int> a_ptr(1, 0), b_ptr(1, 0), n_ptr(1, 0);
        struct ADesc {
          int q, fi, tr, m, bx, col;
          long long yoff;
        };
        struct BDesc {
          int q, m, c0, cw;
          long long yoff, goff;
        };
        std::vector<ADesc> adesc;
        std::vector<BDesc> bdesc;
        std::vector<int> ndesc_f;  // fill index per colnorm entry
        long long ymax = 1, gmax = 1;
        // Gram partials: K split so that small Grams still spread over many CTAs
        static const int partw_env = std::getenv("H2G_GRAM_PARTW") ? std::atoi(std::getenv("H2G_GRAM_PARTW")) : 0;
        const int kPartW = partw_env > 0 ? partw_env : (bm <= 32 ? 128 : (bm <= 64 ? 256 : 512));
        for (int bi = 0; bi < nbat0; ++bi) {
          long long ytop = 0, gtop = 0;
          for (int p = SC.batch_ptr[bi]; p < SC.batch_ptr[bi + 1]; ++p) {
            const int q = p - SC.batch_ptr[bi];
            const int t = SC.batch_cl[p];
            const int b = cur.bsz[t], m = b - cur.korig[t];
            slot_c0[p] = static_cast<int>(ndesc_f.size());
            slot_g0[p] = static_cast<int>(gram_off.size());
            int w = 0;
            const long long yoff = ytop;
            for (int f = Y.G_ptr[t]; f < Y.G_ptr[t + 1]; ++f) {
              const int fi = Y.G_fill[f], tr = Y.G_tr[f];
              const int bx = tr ? cur.bsz[Y.frow[fi]] : cur.bsz[Y.fcol[fi]];
              ndesc_f.push_back(fi);
              if (m > 0) adesc.push_back({q, fi, tr, m, bx, w, yoff});
              w += bx;
            }
            slot_cn[p] = static_cast<int>(ndesc_f.size()) - slot_c0[p];
            if (m > 0) {
              ytop += (long long)m * w;
              for (int c0 = 0; c0 < w; c0 += kPartW) {
                bdesc.push_back({q, m, c0, std::min(kPartW, w - c0), yoff, gtop});
                gram_off.push_back(gtop);
                gtop += (long long)m * m;
              }
            }
            slot_gn[p] = static_cast<int>(gram_off.size()) - slot_g0[p];
          }
          ymax = std::max(ymax, ytop);
          gmax = std::max(gmax, gtop);
          a_ptr.push_back(static_cast<int>(adesc.size()));
          b_ptr.push_back(static_cast<int>(bdesc.size()));
          n_ptr.push_back(static_cast<int>(ndesc_f.size()));
        }
        DBuf ybuf, gbuf, cnbuf, dirbuf, lambuf, flagbuf, cmaxbuf;
        if (verbose)
          std::fprintf(stderr, "[h2g] level %d step-0 scratch: projected fill %.2f GB, Gram partials %.2f GB, directions %.2f GB; device free %.2f GB\n", l,
                       ymax * 16 / 1e9, gmax * 16 / 1e9, (double)std::max(1, W.max_batch) * bb * 16 / 1e9, BlockCache::get().headroom() / 1e9);
        ybuf.alloc(ymax * 16, st);
        gbuf.alloc(gmax * 16, st);
        cnbuf.alloc(std::max<size_t>(ndesc_f.size(), 1) * 8, st);
        const int mb = std::max(1, W.max_batch);
        dirbuf.alloc((size_t)mb * bb * 16, st);
        lambuf.alloc((size_t)mb * bm * 8, st);
        flagbuf.alloc((size_t)mb * 2 * 4, st, true);
        cmaxbuf.alloc((size_t)mb * 8, st);
        int* d_pass2 = flagbuf.as<int>();
        int* d_rank1 = d_pass2 + mb;
        std::vector<GemmDesc> gA1, gA2, gB1, gB2;
        std::vector<NormDesc> gN;
        gA1.reserve(adesc.size());
        gA2.reserve(adesc.size());
        {
          // cluster of each (batch, q): walk batches again
          size_t ai = 0, bi2 = 0;
          for (int bi = 0; bi < nbat0; ++bi) {
            for (; ai < (size_t)a_ptr[bi + 1]; ++ai) {
              const ADesc& a = adesc[ai];
              const int t = SC.batch_cl[SC.batch_ptr[bi] + a.q];
              const int b = cur.bsz[t];
              const int fr = cur.bsz[Y.frow[a.fi]];
              const cplx* F = cur.F.as<cplx>() + cur.foff_safe(a.fi);
              cplx* Cp = ybuf.as<cplx>() + a.yoff + (long long)a.m * a.col;
              const int* fx = cur.fex.as<int>() + a.fi;
              gA1.push_back({cur.Vp.as<cplx>() + (size_t)t * bb, F, Cp, b, fr, a.m, a.m, a.bx, b, OP_C, a.tr ? OP_T : OP_N, 1.0, 0.0, fx, nullptr});
              gA2.push_back({dirbuf.as<cplx>() + (size_t)a.q * bb, F, Cp, b, fr, a.m, a.m, a.bx, b, OP_C, a.tr ? OP_T : OP_N, 1.0, 0.0, fx, d_pass2 + a.q});
            }
            for (; bi2 < (size_t)b_ptr[bi + 1]; ++bi2) {
              const BDesc& d = bdesc[bi2];
              const cplx* Yp = ybuf.as<cplx>() + d.yoff + (long long)d.m * d.c0;
              cplx* G = gbuf.as<cplx>() + d.goff;
              gB1.push_back({Yp, Yp, G, d.m, d.m, d.m, d.m, d.m, d.cw, OP_N, OP_C, 1.0, 0.0, nullptr, nullptr});
              gB2.push_back({Yp, Yp, G, d.m, d.m, d.m, d.m, d.m, d.cw, OP_N, OP_C, 1.0, 0.0, d_pass2 + d.q, nullptr});
            }
          }
          for (size_t c = 0; c < ndesc_f.size(); ++c) {
            const int fi = ndesc_f[c];
            gN.push_back({cur.F.as<cplx>() + cur.foff_safe(fi), cur.bsz[Y.frow[fi]], cur.bsz[Y.fcol[fi]], 0, 0, cur.fex.as<int>() + fi, cnbuf.as<double>() + c});
          }
          // transposition flag of each colnorm entry
          size_t c = 0;
          for (int bi = 0; bi < nbat0; ++bi)
            for (int p = SC.batch_ptr[bi]; p < SC.batch_ptr[bi + 1]; ++p) {
              const int t = SC.batch_cl[p];
              for (int f = Y.G_ptr[t]; f < Y.G_ptr[t + 1]; ++f, ++c) gN[c].trans = Y.G_tr[f];
            }
        }
        // diagonal-block rotation Dii <- Qt^H Dii conj(Qt) as descriptor GEMMs (:345-347)
        DBuf rotbuf;
        rotbuf.alloc((size_t)mb * bb * 16, st);
        std::vector<GemmDesc> gR1, gR2;
        for (int bi = 0; bi < nbat0; ++bi)
          for (int p = SC.batch_ptr[bi]; p < SC.batch_ptr[bi + 1]; ++p) {
            const int q = p - SC.batch_ptr[bi], t = SC.batch_cl[p];
            const int b = cur.bsz[t];
            cplx* Tq = rotbuf.as<cplx>() + (size_t)q * bb;
            cplx* Dtt = cur.D.as<cplx>() + cur.doff[Y.diag_blk[t]];
            const cplx* Qt = CL->arena.as<cplx>() + Qt_off[t];
            gR1.push_back({Qt, Dtt, Tq, b, b, b, b, b, b, OP_C, OP_N, 1.0, 0.0, nullptr, nullptr});
            gR2.push_back({Tq, Qt, Dtt, b, b, b, b, b, b, OP_N, OP_R, 1.0, 0.0, nullptr, nullptr});
          }
        // step-0 eigensolver workspace (per batch slot)
        mark("gram descriptors built");
        DBuf eigws, scratch;
        eigws.alloc((size_t)mb * eig1_ws_bytes(bm), st);
        scratch.alloc(level_scratch_bytes(nl, bm, mb), st);
        // step 2/3b panels as descriptor GEMMs (device-resolved e = b - kfin):
        // column item D(t,c): T = Qt^H D, Ubar = L11^{-1} T[:e,:], lift = Ubar Qt_c^T, D = T (rows < e zeroed)
        // row item    D(j,t): T = D conj(Qt), Lbar = T[:,:e] U11^{-1}, lift = Qt_j Lbar, D = T (cols < e zeroed)
        std::vector<GemmDesc> gP1, gP2, gP3;
        std::vector<MaskDesc> gPM, gPC;
        std::vector<int> p3_ptr(1, 0);
        size_t pmax = 1;
        for (int bi = 0; bi < nbat0; ++bi) pmax = std::max<size_t>(pmax, W.panel_ptr[bi + 1] - W.panel_ptr[bi]);
        DBuf panbuf;
        if (verbose)
          std::fprintf(stderr, "[h2g] level %d panel scratch %.2f GB (%zu items), eigensolver workspace %.2f GB, level scratch %.2f GB; device free %.2f GB\n", l,
                       pmax * bb * 16 / 1e9, pmax, (double)mb * eig1_ws_bytes(bm) / 1e9, level_scratch_bytes(nl, bm, mb) / 1e9,
                       BlockCache::get().headroom() / 1e9);
        panbuf.alloc(pmax * bb * 16, st);
        DBuf dA1, dA2, dB1, dB2, dN, dR1, dR2, dP1, dP2, dP3, dPM, dPC;
        upload(dR1, gR1, st);
        upload(dR2, gR2, st);
        upload(dA1, gA1, st);
        upload(dA2, gA2, st);
        upload(dB1, gB1, st);
        upload(dB2, gB2, st);
        upload(dN, gN, st);
        Packer pk2;
        size_t o_sg0 = pk2.add(slot_g0), o_sgn = pk2.add(slot_gn), o_sc0 = pk2.add(slot_c0), o_scn = pk2.add(slot_cn), o_goff = pk2.add(gram_off);
        DBuf meta2;
        pk2.upload(meta2, st);

        DevLevel DL{};
        DL.level = l;
        DL.nl = nl;
        DL.bmax = bm;
        DL.eps = eps;
        DL.refine_below = std::getenv("H2G_REFINE_BELOW") ? std::atof(std::getenv("H2G_REFINE_BELOW")) : kRefineBelow;
        DL.bsz = at<int>(mt, o_bsz);
        DL.pos = at<int>(mt, o_pos);  // unused on device (long long copy kept for solve)
        DL.korig = at<int>(mt, o_korig);
        DL.kfin = at<int>(mt, o_kfin);
        DL.D = cur.D.as<cplx>();
        DL.D_off = at<long long>(mt, o_doff);
        DL.F_off = at<long long>(mt, o_foff);
        DL.drow = at<int>(mt, o_drow);
        DL.dcol = at<int>(mt, o_dcol);
        DL.diag_blk = at<int>(mt, o_diag);
        DL.F = cur.F.as<cplx>();
        DL.fexists = cur.fex.as<int>();
        DL.frow = at<int>(mt, o_frow);
        DL.fcol = at<int>(mt, o_fcol);
        DL.R_ptr = at<int>(mt, o_Rp);
        DL.R_nb = at<int>(mt, o_Rn);
        DL.C_ptr = at<int>(mt, o_Cp);
        DL.C_nb = at<int>(mt, o_Cn);
        DL.G_ptr = at<int>(mt, o_Gp);
        DL.G_fill = at<int>(mt, o_Gf);
        DL.G_tr = at<unsigned char>(mt, o_Gt);
        DL.V0 = cur.V0.as<cplx>();
        DL.Vp = cur.Vp.as<cplx>();
        DL.chain = CL->arena.as<cplx>();
        DL.Qt_off = at<long long>(mt, o_Qt);
        DL.L11_off = at<long long>(mt, o_L11);
        DL.U11_off = at<long long>(mt, o_U11);
        DL.Lbar_off = at<long long>(mt, o_Lb);
        DL.Ubar_off = at<long long>(mt, o_Ub);
        DL.Lself_off = at<long long>(mt, o_Ls);
        DL.Uself_off = at<long long>(mt, o_Us);
        DL.lift = lift.as<cplx>();
        DL.liftL_off = at<long long>(mt, o_lL);
        DL.liftU_off = at<long long>(mt, o_lU);
        DL.Linv_off = at<long long>(mt, o_Li);
        DL.Uinv_off = at<long long>(mt, o_Ui);
        DL.slot_g0 = at<int>(meta2, o_sg0);
        DL.slot_gn = at<int>(meta2, o_sgn);
        DL.slot_c0 = at<int>(meta2, o_sc0);
        DL.slot_cn = at<int>(meta2, o_scn);
        DL.gram = gbuf.as<cplx>();
        DL.gram_off = at<long long>(meta2, o_goff);
        DL.colnorm = cnbuf.as<double>();
        DL.dir = dirbuf.as<cplx>();
        DL.lam = lambuf.as<double>();
        DL.pass2 = d_pass2;
        DL.rank1 = d_rank1;
        DL.cmax = cmaxbuf.as<double>();
        DL.err = ctx->d_err;
        DL.debug = std::getenv("H2G_DEBUG") ? std::atoi(std::getenv("H2G_DEBUG")) : 0;
        DL.eigws = eigws.as<cplx>();
        DL.scratch = scratch.as<cplx>();
        DL.scratch_bytes = scratch.bytes;

        {
          cplx* chainb = CL->arena.as<cplx>();
          cplx* liftb = lift.as<cplx>();
          const int* kfd = DL.kfin;
          for (int bi = 0; bi < nbat0; ++bi) {
            for (int it = W.panel_ptr[bi]; it < W.panel_ptr[bi + 1]; ++it) {
              const PanelItem& pi = W.panel[it];
              const int t = SC.batch_cl[SC.batch_ptr[bi] + pi.q];
              const int b = cur.bsz[t], bn = cur.bsz[pi.nb];
              cplx* T = panbuf.as<cplx>() + (size_t)(it - W.panel_ptr[bi]) * bb;
              cplx* Dblk = cur.D.as<cplx>() + cur.doff[pi.blk];
              const cplx* Q = chainb + Qt_off[t];
              const cplx* Qn = chainb + Qt_off[pi.nb];
              GemmDesc r{}, pp{}, lf{};
              if (pi.side == 0) {  // D(t, c): b x bn
                r = {Q, Dblk, T, b, b, b, b, bn, b, OP_C, OP_N, 1.0, 0.0};
                // Ubar (e x bn, ld e) = L11^{-1} (e x e, ld e) T[:e, :]
                pp = {chainb + Linv_off[t], T, chainb + Ubar_off[pi.entry], b, b, b, b, bn, b, OP_N, OP_N, 1.0, 0.0};
                pp.dyn = kfd + t, pp.mi = -1, pp.ki = -1, pp.ldneg = 1 | 4;
                if (lifted(pi)) {
                  lf = {chainb + Ubar_off[pi.entry], Qn, liftb + liftU_off[pi.entry], b, bn, b, b, bn, bn, OP_N, OP_T, 1.0, 0.0};
                  lf.dyn = kfd + t, lf.mi = -1, lf.ldneg = 1 | 4;
                }
                gPM.push_back({T, Dblk, b, b, bn, 0, b, 0, kfd + t});
              } else {  // D(j, t): bn x b
                r = {Dblk, Q, T, bn, b, bn, bn, b, b, OP_N, OP_R, 1.0, 0.0};
                // Lbar (bn x e, ld bn) = T[:, :e] U11^{-1} (e x e, ld e)
                pp = {T, chainb + Uinv_off[t], chainb + Lbar_off[pi.entry], bn, b, bn, bn, b, b, OP_N, OP_N, 1.0, 0.0};
                pp.dyn = kfd + t, pp.ni = -1, pp.ki = -1, pp.ldneg = 2;
                if (lifted(pi)) {
                  lf = {Qn, chainb + Lbar_off[pi.entry], liftb + liftL_off[pi.entry], bn, bn, bn, bn, b, bn, OP_N, OP_N, 1.0, 0.0};
                  lf.dyn = kfd + t, lf.ni = -1;
                }
                gPM.push_back({T, Dblk, bn, bn, b, 1, b, 0, kfd + t});
              }
              gPC.push_back(gPM.back());
              gPC.back().e0 = 0;  // e = 0 - kfin <= 0: a plain copy (debug mode, after projection)
              gP1.push_back(r);
              gP2.push_back(pp);
              if (lifted(pi)) gP3.push_back(lf);
            }
            p3_ptr.push_back(static_cast<int>(gP3.size()));
          }
          upload(dP1, gP1, st);
          upload(dP2, gP2, st);
          upload(dP3, gP3, st);
          upload(dPM, gPM, st);
          if (hooks) upload(dPC, gPC, st);
        }
        mark("setup done");
        ctx->prof.cur_level = l;
        ctx->prof.begin(PC_COMPLEMENT, st);
        launch_complement(DL, st);
        ctx->prof.end(st);
        ++launches;
        ++C->klaunch[PC_COMPLEMENT];
        const int nbat = static_cast<int>(SC.batch_ptr.size()) - 1;
        const int* d_bat = at<int>(mt, o_bat);
        const SchurTargetD* d_sch = at<SchurTargetD>(mt, o_sch);
        const SchurContribD* d_con = at<SchurContribD>(mt, o_con);
        // ---- segmented fill storage (plan.hpp FrontPlan): full blocks are
        // zeroed when their storage interval starts and projected to their
        // compact cores Z = V_j^H F conj(V_c) (factorization.hpp:455, :540) at
        // the end of the segment in which the later side passed step 0
        const FrontPlan& FP = cur.front;
        const size_t nfill = Y.frow.size();
        core_ptr_h.assign(nfill, nullptr);
        core_chunks.clear();
        core_page = nullptr;
        DBuf core_tab, dzero;
        core_tab.alloc(std::max<size_t>(nfill, 1) * sizeof(cplx*), st, true);
        DL.core_ptr = core_tab.as<cplx*>();
        std::vector<int> zptr(1, 0);
        {
          std::vector<CopyDesc> zd;
          for (int sg = 0; sg < FP.K; ++sg) {
            for (int f : FP.zero_at[sg]) {
              const int rj = cur.bsz[Y.frow[f]], cc = cur.bsz[Y.fcol[f]];
              zd.push_back({nullptr, cur.F.as<cplx>() + cur.foff[f], rj, rj, rj, cc, 0, 0});
            }
            zptr.push_back(static_cast<int>(zd.size()));
          }
          upload(dzero, zd, st);
        }
        auto segment_end = [&](int sg) {
          CK(cudaStreamWaitEvent(st, ctx->ev_bulk, 0));  // deferred Schur updates land first
          std::vector<int> kf(nl);
          CK(cudaMemcpyAsync(kf.data(), DL.kfin, nl * 4, cudaMemcpyDeviceToHost, st));
          CK(cudaStreamSynchronize(st));
          const auto& cores = FP.core_at[sg];
          std::vector<long long> coff(cores.size());
          long long ctop = 0;
          for (size_t q = 0; q < cores.size(); ++q) coff[q] = ctop, ctop += (long long)kf[Y.frow[cores[q]]] * kf[Y.fcol[cores[q]]];
          if (ctop > 0) {
            ensure((size_t)ctop * 16, nullptr);
            cplx* base = nullptr;
            const char* force_host = std::getenv("H2G_CORES_HOST");  // tests: the HBM-short path on small inputs
            if (!(force_host && std::atoi(force_host)) && BlockCache::get().headroom() >= (size_t)ctop * 16 + kMargin) {
              core_chunks.emplace_back();
              core_chunks.back().alloc((size_t)ctop * 16, st, true);
              base = core_chunks.back().as<cplx>();
            } else {
              // HBM is short: this segment's cores live in pinned, device-mapped
              // host memory (written by the collapse and the later core
              // deposits, read once by the merge): pages of one size, filled
              // across segments, so that the pages a level releases serve the
              // next level as they are (pinning costs ~0.45 s per GB)
              for (size_t q = 0; q < cores.size(); ++q) {
                const size_t need = (size_t)kf[Y.frow[cores[q]]] * kf[Y.fcol[cores[q]]] * 16;
                if (need > kCorePage) {  // a single core beyond a page (never at the measured configurations)
                  core_hchunks.emplace_back();
                  core_hchunks.back().alloc(need);
                  CK(cudaMemsetAsync(core_hchunks.back().p, 0, need, st));
                  core_ptr_h[cores[q]] = core_hchunks.back().as<cplx>();
                  core_page = nullptr;
                  continue;
                }
                if (!core_page || core_page_used + need > kCorePage) {
                  core_hchunks.emplace_back();
                  core_hchunks.back().alloc(kCorePage);
                  CK(cudaMemsetAsync(core_hchunks.back().p, 0, kCorePage, st));
                  core_page = static_cast<char*>(core_hchunks.back().p);
                  core_page_used = 0;
                }
                core_ptr_h[cores[q]] = reinterpret_cast<cplx*>(core_page + core_page_used);
                core_page_used += need;
              }
            }
            if (base)
              for (size_t q = 0; q < cores.size(); ++q) core_ptr_h[cores[q]] = base + coff[q];
          }
          const cplx* chainp = CL->arena.as<cplx>();
          auto V = [&](int t) { return chainp + Qt_off[t] + (long long)(cur.bsz[t] - kf[t]) * cur.bsz[t]; };
          const auto& col = FP.collapse_at[sg];
          const long long kChunkX = (1LL << 30) / 16;
          DBuf xb, dg1, dg2;
          for (size_t q0 = 0; q0 < col.size();) {
            std::vector<GemmDesc> g1, g2;
            long long xt = 0;
            std::vector<long long> xo;
            size_t q1 = q0;
            for (; q1 < col.size(); ++q1) {
              const int f = col[q1], j = Y.frow[f], c = Y.fcol[f];
              const long long xn = (long long)kf[j] * cur.bsz[c];
              if (q1 > q0 && xt + xn > kChunkX) break;
              xo.push_back(xt);
              xt += xn;
            }
            xb.alloc((size_t)std::max<long long>(xt, 1) * 16, st);
            for (size_t q = q0; q < q1; ++q) {
              const int f = col[q], j = Y.frow[f], c = Y.fcol[f];
              if (!kf[j] || !kf[c]) continue;
              cplx* X = xb.as<cplx>() + xo[q - q0];
              const int* fx = cur.fex.as<int>() + f;
              g1.push_back({V(j), cur.F.as<cplx>() + cur.foff[f], X, cur.bsz[j], cur.bsz[j], kf[j], kf[j], cur.bsz[c], cur.bsz[j], OP_C, OP_N, 1.0, 0.0, fx, nullptr});
              g2.push_back({X, V(c), core_ptr_h[f], kf[j], cur.bsz[c], kf[j], kf[j], kf[c], cur.bsz[c], OP_N, OP_R, 1.0, 0.0, fx, nullptr});
            }
            upload(dg1, g1, st);
            upload(dg2, g2, st);
            ctx->prof.begin(PC_MERGE, st);
            launch_gemm(dg1.as<GemmDesc>(), static_cast<int>(g1.size()), st, bm);
            launch_gemm(dg2.as<GemmDesc>(), static_cast<int>(g2.size()), st, bm);
            ctx->prof.end(st);
            C->klaunch[PC_MERGE] += (!g1.empty()) + (!g2.empty());
            launches += (!g1.empty()) + (!g2.empty());
            q0 = q1;
          }
          CK(cudaMemcpyAsync(core_tab.p, core_ptr_h.data(), nfill * sizeof(cplx*), cudaMemcpyHostToDevice, st));
          CK(cudaStreamSynchronize(st));  // core_ptr_h is rewritten at the next segment end
          if (streamed && seg_len[sg] > 0) {
            // the segment's chain part is final (main and side streams have
            // drained) and its eliminated sizes are known: every block moves
            // to its compact place (the kernels already wrote it with its
            // final leading dimension), then the segment leaves the device
            CK(cudaStreamSynchronize(ctx->side));
            std::vector<MoveDesc> mv;
            const cplx* ringp = CL->arena.as<cplx>();
            const long long seg0 = compact_top;
            auto blockmv = [&](long long dev_off, long long len, long long& logical) {
              logical = compact_top;
              if (len > 0) mv.push_back({ringp + dev_off, reinterpret_cast<cplx*>((compact_top - seg0) * 16), len});
              compact_top += len;
            };
            for (int bi2 = FP.seg_first_batch[sg]; bi2 < FP.seg_first_batch[sg + 1]; ++bi2)
              for (int p = SC.batch_ptr[bi2]; p < SC.batch_ptr[bi2 + 1]; ++p) {
                const int t = SC.batch_cl[p];
                const long long b = cur.bsz[t], kft = kf[t], e = b - kft;
                blockmv(L11_off[t], e * e, lL11[t]);
                blockmv(U11_off[t], e * e, lU11[t]);
                blockmv(Linv_off[t], e * e, lLinv[t]);
                blockmv(Uinv_off[t], e * e, lUinv[t]);
                blockmv(Lself_off[t], kft * e, lLself[t]);
                blockmv(Uself_off[t], e * kft, lUself[t]);
                for (int a = Y.R_ptr[t]; a < Y.R_ptr[t + 1]; ++a) blockmv(Lbar_off[a], (long long)cur.bsz[Y.R_nb[a]] * e, lLbar[a]);
                for (int a = Y.C_ptr[t]; a < Y.C_ptr[t + 1]; ++a) blockmv(Ubar_off[a], (long long)cur.bsz[Y.C_nb[a]] * e, lUbar[a]);
              }
            const long long clen = compact_top - seg0;
            if (clen > 0) {
              if (BlockCache::get().headroom() >= (size_t)clen * 16 + kMargin) {
                ChainLevelHost::Chunk ck;
                ck.begin = seg0, ck.len = clen;
                ck.d.alloc((size_t)clen * 16, st);
                for (auto& d : mv) d.dst = ck.d.as<cplx>() + reinterpret_cast<long long>(d.dst) / 16;
                CL->chunks.push_back(std::move(ck));
              } else {
                // HBM is short: the segment goes to pinned host memory (mapped,
                // written by the kernel), block after block into the level's
                // staging pages; a page boundary starts a new chunk
                for (auto& d : mv) {
                  const long long rel = reinterpret_cast<long long>(d.dst) / 16;  // compact offset inside the segment
                  const size_t need = (size_t)d.len * 16;
                  if (need > kStagePage) throw Error(H2G_ERR_INTERNAL, "chain block larger than a staging page");
                  if (!CL->hpage || CL->hpage_used + need > kStagePage) {
                    CL->hpages.emplace_back();
                    CL->hpages.back().alloc(kStagePage);
                    CL->hpage = static_cast<char*>(CL->hpages.back().p);
                    CL->hpage_used = 0;
                    CL->chunks.emplace_back();
                    CL->chunks.back().begin = seg0 + rel;
                    CL->chunks.back().hp = CL->hpage;
                  } else if (CL->chunks.empty() || CL->chunks.back().hp == nullptr ||
                             CL->chunks.back().begin + CL->chunks.back().len != seg0 + rel) {
                    // first host block of this segment in a page already in use
                    CL->chunks.emplace_back();
                    CL->chunks.back().begin = seg0 + rel;
                    CL->chunks.back().hp = CL->hpage + CL->hpage_used;
                  }
                  d.dst = reinterpret_cast<cplx*>(CL->hpage + CL->hpage_used);
                  CL->hpage_used += need;
                  CL->chunks.back().len += d.len;
                }
              }
              DBuf dmv;
              upload(dmv, mv, st);
              launch_move(dmv.as<MoveDesc>(), static_cast<int>(mv.size()), st);
              CK(cudaStreamSynchronize(st));
              ++launches;
            }
          }
        };
        // ---- multi-GPU subtree partition (h2g_factorize_dist): what the
        // interior phase of every subtree writes, derived from the work lists
        // of its batches: final ranks and chain records of its clusters, the
        // dense blocks it rotates / updates, the fill blocks it deposits into
        std::vector<PartList> parts;
        const bool partitioned = dist && dist->nranks > 1;
        const int bnd0 = partitioned ? SC.part_batch[kInteriorParts] : 0;  // first boundary batch
        auto part_owner = [&](int sp) { return sp * dist->nranks / kInteriorParts; };
        auto batch_part = [&](int bi) {
          int sp = 0;
          while (sp + 1 < kInteriorParts && bi >= SC.part_batch[sp + 1]) ++sp;
          return sp;
        };
        if (partitioned && bnd0 > 0) {
          if (FP.K != 1) throw Error(H2G_ERR_INTERNAL, "factorize_dist: segmented fill storage in a partitioned level");
          parts = build_parts(Y, SC, W);
          for (const PartList& PL : parts)
            for (int q : PL.fblk)
              if (cur.foff[q] < 0) throw Error(H2G_ERR_INTERNAL, "factorize_dist: deposited fill block without storage");
        }
        bool exchanged = !(partitioned && bnd0 > 0);
        auto do_exchange = [&] {
          NvtxRange nv_x("h2g exchange level " + std::to_string(l));
          CK(cudaStreamWaitEvent(st, ctx->ev_bulk, 0));
          CK(cudaStreamSynchronize(ctx->side));
          CK(cudaStreamSynchronize(ctx->aux));
          // layout per rank: its subtrees in order, each [ints | pad to 16 B | complex regions]
          auto chain_end = [&](int t) { return t + 1 < nl ? Qt_off[t + 1] : top; };
          std::vector<int64_t> offs(dist->nranks + 1, 0);
          std::vector<size_t> part_off(kInteriorParts, 0);
          {
            size_t o = 0;
            int r = 0;
            for (int sp = 0; sp < kInteriorParts; ++sp) {
              while (r < part_owner(sp)) offs[++r] = static_cast<int64_t>(o);
              part_off[sp] = o;
              const PartList& PL = parts[sp];
              o += (PL.ints() * 4 + 15) / 16 * 16;
              for (int t : PL.cl) o += (size_t)(chain_end(t) - Qt_off[t]) * 16;
              for (int q : PL.dblk) o += (size_t)cur.bsz[Y.drow[q]] * cur.bsz[Y.dcol[q]] * 16;
              for (int q : PL.fblk) o += (size_t)cur.bsz[Y.frow[q]] * cur.bsz[Y.fcol[q]] * 16;
            }
            while (r < dist->nranks) offs[++r] = static_cast<int64_t>(o);
          }
          const size_t total = static_cast<size_t>(offs[dist->nranks]);
          if (total == 0) return;
          ensure(total, nullptr);
          DBuf xbuf, dmv, didx;
          xbuf.alloc(total, st);
          // descriptors: own subtrees pack (pool -> buffer), the others unpack
          std::vector<MoveDesc> mv_pack, mv_unpack;
          std::vector<int> idx_all;
          struct IntJob {
            int sp, which, i0, n;  // which: 0 kfin, 1 fexists
            size_t boff;
          };
          std::vector<IntJob> jobs;
          cplx* chainp = CL->arena.as<cplx>();
          for (int sp = 0; sp < kInteriorParts; ++sp) {
            const PartList& PL = parts[sp];
            const bool mine = part_owner(sp) == dist->rank;
            char* base = static_cast<char*>(xbuf.p) + part_off[sp];
            jobs.push_back({sp, 0, static_cast<int>(idx_all.size()), static_cast<int>(PL.cl.size()), part_off[sp]});
            idx_all.insert(idx_all.end(), PL.cl.begin(), PL.cl.end());
            jobs.push_back({sp, 1, static_cast<int>(idx_all.size()), static_cast<int>(PL.fblk.size()), part_off[sp] + PL.cl.size() * 4});
            idx_all.insert(idx_all.end(), PL.fblk.begin(), PL.fblk.end());
            cplx* bc = reinterpret_cast<cplx*>(base + (PL.ints() * 4 + 15) / 16 * 16);
            auto region = [&](cplx* pool, long long len) {
              if (len > 0) (mine ? mv_pack : mv_unpack).push_back(mine ? MoveDesc{pool, bc, len} : MoveDesc{bc, pool, len});
              bc += len;
            };
            for (int t : PL.cl) region(chainp + Qt_off[t], chain_end(t) - Qt_off[t]);
            for (int q : PL.dblk) region(cur.D.as<cplx>() + cur.doff[q], (long long)cur.bsz[Y.drow[q]] * cur.bsz[Y.dcol[q]]);
            for (int q : PL.fblk) region(cur.F.as<cplx>() + cur.foff[q], (long long)cur.bsz[Y.frow[q]] * cur.bsz[Y.fcol[q]]);
          }
          std::vector<MoveDesc> mv_all(mv_pack);
          mv_all.insert(mv_all.end(), mv_unpack.begin(), mv_unpack.end());
          upload(dmv, mv_all, st);
          upload(didx, idx_all, st);
          auto int_moves = [&](bool own, int scatter) {
            for (const IntJob& j : jobs) {
              if ((part_owner(j.sp) == dist->rank) != own) continue;
              int* basep = j.which == 0 ? DL.kfin : DL.fexists;
              launch_int_move(basep, didx.as<int>() + j.i0, j.n, reinterpret_cast<int*>(static_cast<char*>(xbuf.p) + j.boff), scatter, st);
            }
          };
          int_moves(true, 0);
          launch_move(dmv.as<MoveDesc>(), static_cast<int>(mv_pack.size()), st);
          CK(cudaStreamSynchronize(st));
          const double tx0 = wall();
          const int rc = dist->exchange(dist->user, xbuf.p, offs.data(), dist->nranks);
          if (rc != 0) throw Error(H2G_ERR_INTERNAL, fmt("factorize_dist: the exchange callback failed (code %lld) at level %lld", rc, l));
          C->dist_exchange_s += wall() - tx0;
          C->dist_sent_bytes += static_cast<double>(offs[dist->rank + 1] - offs[dist->rank]);
          C->dist_total_bytes += static_cast<double>(total);
          int_moves(false, 1);
          launch_move(dmv.as<MoveDesc>() + mv_pack.size(), static_cast<int>(mv_unpack.size()), st);
          CK(cudaStreamSynchronize(st));
          launches += 2 * kInteriorParts + 2;
          if (verbose)
            std::fprintf(stderr, "[h2g] level %d: rank %d/%d exchanged %.3f GB (own part %.3f GB), interior batches %d of %d\n", l, dist->rank,
                         dist->nranks, total / 1e9, (offs[dist->rank + 1] - offs[dist->rank]) / 1e9, bnd0, nbat);
        };
        auto maybe_exchange = [&](int next_bi) {
          if (!exchanged && next_bi >= bnd0) {
            exchanged = true;
            do_exchange();
          }
        };
        // resolved Schur descriptors (k_schur_resolve), two halves by batch
        // parity like the lifted panels; H2G_SCHUR_RESOLVE=0 resolves inside k_schur
        static const bool schur_resolve = !(std::getenv("H2G_SCHUR_RESOLVE") && std::atoi(std::getenv("H2G_SCHUR_RESOLVE")) == 0);
        std::vector<int> cbase(nbat, 0);
        int rt_max = 1, rp_max = 1;
        for (int bi = 0; bi < nbat; ++bi) {
          const int s0 = W.schur_ptr[bi], s1 = W.schur_ptr[bi + 1];
          int c_lo = INT32_MAX, c_hi = 0;
          for (int q = s0; q < s1; ++q) c_lo = std::min(c_lo, W.schur[q].c0), c_hi = std::max(c_hi, W.schur[q].c1);
          if (s1 > s0) {
            cbase[bi] = c_lo;
            rt_max = std::max(rt_max, s1 - s0);
            rp_max = std::max(rp_max, c_hi - c_lo);
          }
        }
        DBuf rtbuf, rpbuf;
        if (schur_resolve && !hooks) {
          rtbuf.alloc((size_t)2 * rt_max * sizeof(RTarget), st);
          rpbuf.alloc((size_t)2 * rp_max * sizeof(RPanel), st);
        }
        int prev_exec = -1;
        std::vector<char> rotated(nl, 0);
        std::vector<int> elimv(nl, 0);
        h2g_state hstate;
        hstate.ctx = ctx;
        hstate.M = M;
        hstate.cur = &cur;
        hstate.Y = &Y;
        hstate.level = l;
        hstate.d_kfin = nullptr;
        hstate.rotated = &rotated;
        hstate.elim = &elimv;
        hstate.chain = CL->arena.as<cplx>();
        hstate.Qt_off = &Qt_off;
        auto hook_sync = [&] {
          CK(cudaStreamSynchronize(st));
          check_device_error(ctx, l);
        };
        for (int bi = 0; bi < nbat; ++bi) {
          maybe_exchange(bi);
          if (partitioned && bi < bnd0 && part_owner(batch_part(bi)) != dist->rank) {
            // another rank's subtree: its results arrive with the exchange
            if (bi + 1 == nbat) {
              maybe_exchange(nbat);
              segment_end(0);
            }
            continue;
          }
          if (partitioned && prev_exec >= 0 && prev_exec != bi - 1) CK(cudaStreamWaitEvent(st, ctx->ev_bulk, 0));
          prev_exec = bi;
          const int p0 = SC.batch_ptr[bi], nb = SC.batch_ptr[bi + 1] - p0;
          const int sgi = fill_segment(bi, nbat, FP.K);
          if (sgi > 0 && bi == FP.seg_first_batch[sgi] && zptr[sgi + 1] > zptr[sgi]) {
            launch_copy(dzero.as<CopyDesc>() + zptr[sgi], zptr[sgi + 1] - zptr[sgi], st);
            ++launches;
          }
          const int na = a_ptr[bi + 1] - a_ptr[bi], nbd = b_ptr[bi + 1] - b_ptr[bi], nn = n_ptr[bi + 1] - n_ptr[bi];
          Prof& pf = ctx->prof;
          const int tl = bm;  // max GEMM dimension of this level's per-cluster products
          // column norms of the fill entering W on the helper stream, concurrent
          // with the projection / Gram GEMMs
          CK(cudaEventRecord(ctx->ev_aux0, st));
          CK(cudaStreamWaitEvent(ctx->aux, ctx->ev_aux0, 0));
          ctx->prof_aux.cur_level = l;
          ctx->prof_aux.begin(PC_COLNORM, ctx->aux);
          launch_colnorm(dN.as<NormDesc>() + n_ptr[bi], nn, ctx->aux);
          ctx->prof_aux.end(ctx->aux);
          CK(cudaEventRecord(ctx->ev_aux1, ctx->aux));
          pf.begin(PC_GRAM, st);
          launch_gemm(dA1.as<GemmDesc>() + a_ptr[bi], na, st, tl);
          launch_gemm(dB1.as<GemmDesc>() + b_ptr[bi], nbd, st, tl);
          pf.end(st);
          CK(cudaStreamWaitEvent(st, ctx->ev_aux1, 0));
          pf.begin(PC_EIG1, st);
          int mmax = 0;
          for (int pq = p0; pq < p0 + nb; ++pq) mmax = std::max(mmax, cur.bsz[SC.batch_cl[pq]] - cur.korig[SC.batch_cl[pq]]);
          launch_eig1(DL, d_bat + p0, p0, nb, mmax, st, [&](int ph) {
            pf.end(st);
            pf.begin(ph == 1 ? PC_EIGVEC : PC_EIG1B, st);
          });
          pf.end(st);
          const bool pass2_possible = eig1_refine_possible(DL);
          if (pass2_possible) {
            pf.begin(PC_GRAM, st);
            launch_gemm(dA2.as<GemmDesc>() + a_ptr[bi], na, st, tl);
            launch_gemm(dB2.as<GemmDesc>() + b_ptr[bi], nbd, st, tl);
            pf.end(st);
          }
          pf.begin(PC_HEAD, st);
          launch_head(DL, d_bat + p0, p0, nb, st);
          if (hooks) {  // debug mode (SERIAL schedule: the batch is one cluster)
            hook_sync();
            hstate.d_kfin = DL.kfin;
            if (hooks->after_basis_update) hooks->after_basis_update(hooks->user, &hstate, Y.first + SC.batch_cl[p0]);
          }
          launch_gemm(dR1.as<GemmDesc>() + p0, nb, st, tl);
          launch_gemm(dR2.as<GemmDesc>() + p0, nb, st, tl);
          if (hooks) {
            // step 2 in full before step 3: the rotated row / column blocks
            // land in D unmasked (the reference's state after projection)
            const int i0 = W.panel_ptr[bi], ni = W.panel_ptr[bi + 1] - i0;
            launch_gemm(dP1.as<GemmDesc>() + i0, ni, st, tl);
            launch_mask(dPC.as<MaskDesc>() + i0, ni, st);
            hook_sync();
            rotated[SC.batch_cl[p0]] = 1;
            if (hooks->after_projection) hooks->after_projection(hooks->user, &hstate, Y.first + SC.batch_cl[p0]);
          }
          launch_head2(DL, d_bat + p0, nb, mmax, st);
          pf.end(st);
          pf.begin(PC_PANEL, st);
          {
            const int i0 = W.panel_ptr[bi], ni = W.panel_ptr[bi + 1] - i0;
            if (!hooks) launch_gemm(dP1.as<GemmDesc>() + i0, ni, st, tl);
            launch_gemm(dP2.as<GemmDesc>() + i0, ni, st, tl);
            launch_gemm(dP3.as<GemmDesc>() + p3_ptr[bi], p3_ptr[bi + 1] - p3_ptr[bi], st, tl);
            launch_mask(dPM.as<MaskDesc>() + i0, ni, st);
          }
          pf.end(st);
          {
            // critical targets (rows/columns of the next batch) in-line, after
            // the previous batch's deferred targets have landed; the rest on
            // the side stream, overlapping the next batch
            const int s0 = W.schur_ptr[bi], ncr = W.schur_crit[bi], nbulk = W.schur_ptr[bi + 1] - s0 - ncr;
            if (bi > 0) CK(cudaStreamWaitEvent(st, ctx->ev_bulk, 0));
            RTarget* rtp = nullptr;
            RPanel* rpp = nullptr;
            pf.begin(PC_SCHUR, st);
            if (rtbuf.p && ncr + nbulk > 0) {
              rtp = rtbuf.as<RTarget>() + (size_t)(bi & 1) * rt_max;
              rpp = rpbuf.as<RPanel>() + (size_t)(bi & 1) * rp_max - cbase[bi];
              launch_schur_resolve(DL, d_sch + s0, ncr + nbulk, d_con, rtp, rpp, st);
              ++launches;
            }
            launch_schur(DL, d_sch + s0, ncr, d_con, st, rtp, rpp);
            pf.end(st);
            CK(cudaEventRecord(ctx->ev_crit, st));
            CK(cudaStreamWaitEvent(ctx->side, ctx->ev_crit, 0));
            ctx->prof_side.cur_level = l;
            ctx->prof_side.begin(PC_SCHUR, ctx->side);
            if (!(DL.debug & 16)) launch_schur(DL, d_sch + s0 + ncr, nbulk, d_con, ctx->side, rtp ? rtp + ncr : nullptr, rpp);  // debug 16: timing experiment only (wrong results)
            ctx->prof_side.end(ctx->side);
            CK(cudaEventRecord(ctx->ev_bulk, ctx->side));
            C->klaunch[PC_SCHUR] += (ncr > 0) + (nbulk > 0);
            launches += (ncr > 0) + (nbulk > 0);
          }
          C->klaunch[PC_GRAM] += (pass2_possible ? 2 : 1) * ((na > 0) + (nbd > 0));
          C->klaunch[PC_COLNORM] += nn > 0;
          C->klaunch[PC_EIG1] += 1 + pass2_possible;
          C->klaunch[PC_EIGVEC] += mmax > 0;
          C->klaunch[PC_EIG1B] += 2;
          const int nhead = 3 + (mmax > 64 ? 2 + 2 * ((mmax + 31) / 32) : 1);
          C->klaunch[PC_HEAD] += nhead;
          const int npl = W.panel_ptr[bi + 1] > W.panel_ptr[bi] ? 3 + (p3_ptr[bi + 1] > p3_ptr[bi]) : 0;
          C->klaunch[PC_PANEL] += npl;
          launches += 3 + pass2_possible + (mmax > 0) + nhead + (pass2_possible ? 2 : 1) * ((na > 0) + (nbd > 0)) + (nn > 0) + npl;
          if (hooks) {
            CK(cudaStreamWaitEvent(st, ctx->ev_bulk, 0));
            hook_sync();
            const int tcl = SC.batch_cl[p0];
            int kft = 0;
            CK(cudaMemcpy(&kft, DL.kfin + tcl, 4, cudaMemcpyDeviceToHost));
            elimv[tcl] = cur.bsz[tcl] - kft;
            if (hooks->after_elimination) hooks->after_elimination(hooks->user, &hstate, Y.first + tcl);
          }
          if (bi + 1 == FP.seg_first_batch[sgi + 1]) {
            maybe_exchange(bi + 1);
            segment_end(sgi);
          }
        }
        CK(cudaStreamWaitEvent(st, ctx->ev_bulk, 0));  // deferred Schur updates of the last batch
        const double t_launched = wall();
        CK(cudaGetLastError());
        check_device_error(ctx, l);
        if (verbose)
          std::fprintf(stderr,
                       "[h2g] level %d: nl %d bmax %d batches %d: host setup+launch %.3f s, device drain %.3f s; D %zu blocks %.2f GB, F %zu blocks "
                       "%.2f GB, chain %.2f GB\n",
                       l, nl, bm, nbat, t_launched - tlev, wall() - t_launched, Y.drow.size(), cur.D.bytes / 1e9, Y.frow.size(), cur.F.bytes / 1e9,
                       CL->arena.bytes / 1e9);
        // ---- read back final ranks and fill existence
        std::vector<int> kfin(nl), fex(Y.frow.size());
        CK(cudaMemcpyAsync(kfin.data(), DL.kfin, nl * 4, cudaMemcpyDeviceToHost, st));
        if (!fex.empty()) CK(cudaMemcpyAsync(fex.data(), DL.fexists, fex.size() * 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));

        mark("kfin read back");
        if (streamed) {
          // the halves are dead: Qt moves to its own buffer, the level's chain is
          // its compact chunks until the end of the factorization
          CL->qchunk.alloc((size_t)std::max<long long>(qtot, 1) * 16, st);
          CK(cudaMemcpyAsync(CL->qchunk.p, CL->arena.p, (size_t)qtot * 16, cudaMemcpyDeviceToDevice, st));
          CK(cudaStreamSynchronize(st));
          CL->arena.release();
          CL->compact_elems = compact_top;
          if (verbose) {
            double onhost = 0.0;
            for (const auto& ck : CL->chunks)
              if (!ck.d.p) onhost += (double)ck.len * 16;
            std::fprintf(stderr, "[h2g] level %d: chain %.2f GB at its final size (bound %.2f GB), %.2f GB of it in host memory\n", l,
                         compact_top * 16 / 1e9, top_logical * 16 / 1e9, onhost / 1e9);
          }
        }
        // level scratch is dead once the last batch has drained (keeps the
        // merge's peak memory down at config 3)
        lift.release();
        panbuf.release();
        ybuf.release();
        gbuf.release();
        dirbuf.release();
        rotbuf.release();
        eigws.release();
        scratch.release();
        const double sflops_lv0 = sflops, flops_lv0 = flops, sexec_lv0 = C->schur_flops_exec, sbexec_lv0 = C->schur_bytes_exec;
        // ---- records + diagnostics
        long long rsb = 0, rsa = 0, elim = 0, ledger = 0;
        std::vector<int> rec_order;
        if (schedule == H2G_SCHEDULE_REFERENCE) {
          for (int t = 0; t < nl; ++t) rec_order.push_back(t);
        } else {
          rec_order = SC.batch_cl;
        }
        size_t lvl_bytes = 0;
        for (int t : rec_order) {
          const int b = cur.bsz[t], kf = kfin[t], e = b - kf;
          const int nr = Y.R_ptr[t + 1] - Y.R_ptr[t], ncn = Y.C_ptr[t + 1] - Y.C_ptr[t];
          const int nlb = e > 0 ? nr + (kf > 0) : 0, nub = e > 0 ? ncn + (kf > 0) : 0;
          const int64_t r[10] = {Y.first + t, l, cur.pos[t], b, e, cur.korig[t], kf, e > 0 ? (int64_t)nlb * nub : 0, nlb, nub};
          CL->rec.insert(CL->rec.end(), r, r + 10);
          CL->rec_cluster.push_back(t);
          lvl_bytes += 16 * ((size_t)b * b + 2 * (size_t)e * e);
          if (e > 0) {
            for (int a = Y.R_ptr[t]; a < Y.R_ptr[t + 1]; ++a) lvl_bytes += 16 * (size_t)cur.bsz[Y.R_nb[a]] * e;
            for (int a = Y.C_ptr[t]; a < Y.C_ptr[t + 1]; ++a) lvl_bytes += 16 * (size_t)cur.bsz[Y.C_nb[a]] * e;
            if (kf > 0) lvl_bytes += 16 * 2 * (size_t)kf * e;
          }
          rsb += cur.korig[t];
          rsa += kf;
          elim += e;
          // algorithmic flops (SURVEY §8d F_factor)
          const double bd = b, ed = e, md = b - cur.korig[t];
          double gram_cols = 0;
          for (int f = Y.G_ptr[t]; f < Y.G_ptr[t + 1]; ++f)
            if (fex[Y.G_fill[f]]) gram_cols += Y.G_tr[f] ? cur.bsz[Y.frow[Y.G_fill[f]]] : cur.bsz[Y.fcol[Y.G_fill[f]]];
          flops += 8.0 * md * bd * gram_cols + 8.0 * md * md * gram_cols;  // Vp^H W and Y Y^H
          flops += 16.0 * bd * bd * bd;                                      // rotation of D(t,t)
          double rot = 0;
          for (int a = Y.R_ptr[t]; a < Y.R_ptr[t + 1]; ++a) rot += cur.bsz[Y.R_nb[a]];
          for (int a = Y.C_ptr[t]; a < Y.C_ptr[t + 1]; ++a) rot += cur.bsz[Y.C_nb[a]];
          flops += 8.0 * bd * bd * rot;  // step 2 on off-diagonal blocks
          if (e > 0) {
            flops += 8.0 / 3.0 * ed * ed * ed + 4.0 * ed * ed * (rot + 2.0 * kf);  // LU + TRSMs
            // Schur, SURVEY §8d algorithmic count: sum_j b_j * e * sum_c b_c
            // (incl. self rows/cols of kf), as the reference's GEMMs
            // (factorization.hpp:416-420) execute them
            double rows = kf, cols = kf;
            for (int a = Y.R_ptr[t]; a < Y.R_ptr[t + 1]; ++a) rows += cur.bsz[Y.R_nb[a]];
            for (int a = Y.C_ptr[t]; a < Y.C_ptr[t + 1]; ++a) cols += cur.bsz[Y.C_nb[a]];
            const double sch = 8.0 * rows * ed * cols;
            flops += sch;
            sflops += sch;
            // every target entry read + written once, panels read once
            sbytes += 16.0 * 2.0 * rows * cols + 16.0 * ed * (rows + cols);
          }
        }
        // Schur products actually executed by k_schur: per target and
        // contribution; rows / columns of a dense target whose cluster was
        // eliminated in an earlier batch receive exact zeros and are not
        // computed. Bytes: every target read + written once, panels read
        // once per target they feed.
        for (const SchurTarget& T : W.schur) {
          int rws, cls, rs = 0, cs = 0;
          if ((T.kind & 1) == 0) {
            const int j = Y.drow[T.idx], c = Y.dcol[T.idx];
            rws = cur.bsz[j], cls = cur.bsz[c];
            if (T.kind & 2) rs = cur.bsz[j] - kfin[j];
            if (T.kind & 4) cs = cur.bsz[c] - kfin[c];
          } else {
            const int j = Y.frow[T.idx], c = Y.fcol[T.idx];
            rws = cur.bsz[j], cls = cur.bsz[c];
            if (T.kind & 8) rs = cur.bsz[j] - kfin[j], cs = cur.bsz[c] - kfin[c];  // core deposit
          }
          bool any = false;
          for (int k = T.c0; k < T.c1; ++k) {
            const SchurContrib& cb = W.contrib[k];
            const int tc = cb.t, ec = cur.bsz[tc] - kfin[tc];
            if (ec == 0) continue;
            any = true;
            const int ro = cb.r >= 0 ? 0 : ec, ar = cb.r >= 0 ? cur.bsz[Y.R_nb[cb.r]] : kfin[tc];
            const int co = cb.c >= 0 ? 0 : ec, bc = cb.c >= 0 ? cur.bsz[Y.C_nb[cb.c]] : kfin[tc];
            const double rr = std::max(0, std::min(ro + ar, rws) - std::max(ro, rs));
            const double cc = std::max(0, std::min(co + bc, cls) - std::max(co, cs));
            C->schur_flops_exec += 8.0 * rr * ec * cc;
            C->schur_bytes_exec += 16.0 * ec * (rr + cc);
          }
          if (any) C->schur_bytes_exec += 32.0 * (double)(rws - rs) * (double)(cls - cs);
        }
        for (size_t f = 0; f < Y.frow.size(); ++f)
          if (Y.fadm[f] >= 0 && fex[f]) ++ledger;
        // collapse projections (segment ends)
        for (const auto& col : cur.front.collapse_at)
          for (int f : col)
            if (fex[f]) {
              const int a = Y.frow[f], c = Y.fcol[f];
              flops += 8.0 * kfin[a] * cur.bsz[a] * cur.bsz[c] + 8.0 * kfin[a] * cur.bsz[c] * kfin[c];
            }
        // ---- permutation (merge_permute :492-509)
        const int lp = l - 1;
        const int nlp = nl / 2;
        std::vector<long long> src;
        src.reserve(S.n);
        for (int P2 = 0; P2 < nlp; ++P2)
          for (int ch = 2 * P2; ch <= 2 * P2 + 1; ++ch) {
            const long long base = cur.pos[ch] + (cur.bsz[ch] - kfin[ch]);
            for (int q = 0; q < kfin[ch]; ++q) src.push_back(base + q);
          }
        const long long active_new = static_cast<long long>(src.size());
        for (int t = 0; t < nl; ++t)
          for (int q = 0; q < cur.bsz[t] - kfin[t]; ++q) src.push_back(cur.pos[t] + q);
        lvl_bytes += 8 * src.size();
        C->storage_bytes += lvl_bytes;
        CL->diag = {l, (int64_t)rec_order.size(), rsb, rsa, elim, ledger, (int64_t)C->storage_bytes, (int64_t)src.size(), active_new};
        CL->src.assign(src.begin(), src.end());
        upload(CL->d_src, CL->src, st);

        // ---- keep solve data
        CL->bsz = cur.bsz;
        CL->kfin = kfin;
        CL->korig = cur.korig;
        CL->pos = posl;
        CL->R_ptr = Y.R_ptr;
        CL->R_nb = Y.R_nb;
        CL->C_ptr = Y.C_ptr;
        CL->C_nb = Y.C_nb;
        CL->Qt_off = lQt;
        CL->L11_off = lL11;
        CL->U11_off = lU11;
        CL->Lbar_off = lLbar;
        CL->Ubar_off = lUbar;
        CL->Lself_off = lLself;
        CL->Uself_off = lUself;
        CL->batch_ptr = SC.batch_ptr;
        for (int bi = 0; bi + 1 < (int)SC.batch_ptr.size(); ++bi) {
          int mc = 0;
          for (int pq = SC.batch_ptr[bi]; pq < SC.batch_ptr[bi + 1]; ++pq) {
            const int tt = SC.batch_cl[pq];
            mc = std::max(mc, Y.C_ptr[tt + 1] - Y.C_ptr[tt]);
          }
          CL->batch_maxc.push_back(mc);
        }
        CL->d_batch = d_bat;
        CL->fs_ptr = W.fsolve_ptr;
        CL->d_fs = at<SolveTargetD>(mt, o_fs);
        CL->d_fc = at<SolveContribD>(mt, o_fc);
        {
          std::vector<int> sv(CL->batch_ptr);
          sv.insert(sv.end(), CL->batch_maxc.begin(), CL->batch_maxc.end());
          sv.insert(sv.end(), CL->fs_ptr.begin(), CL->fs_ptr.end());
          upload(CL->sched_buf, sv, st);
          const int nb1 = static_cast<int>(CL->batch_ptr.size());
          const int* base = CL->sched_buf.as<int>();
          CL->sched = {nb1 - 1, base, d_bat, base + nb1, base + nb1 + (nb1 - 1), CL->d_fs, CL->d_fc};
          for (int bi = 0; bi + 1 < nb1; ++bi)
            CL->part_need = std::max(CL->part_need, (size_t)(CL->batch_ptr[bi + 1] - CL->batch_ptr[bi]) * (CL->batch_maxc[bi] + 1) * bm);
        }
        CL->C_ptr = Y.C_ptr;
        CL->C_nb = Y.C_nb;
        CL->bsz = cur.bsz;
        CL->kfin = kfin;
        {
          std::vector<SolveTargetD> fsd(W.fsolve.size());
          std::vector<SolveContribD> fcd(W.fcontrib.size());
          for (size_t i = 0; i < fsd.size(); ++i) fsd[i] = {W.fsolve[i].seg, W.fsolve[i].c0, W.fsolve[i].c1};
          for (size_t i = 0; i < fcd.size(); ++i) fcd[i] = {W.fcontrib[i].m, W.fcontrib[i].entry};
          build_flow(*CL, nl, SC.batch_ptr, SC.batch_cl, W.fsolve_ptr, fsd, fcd, st);
        }
        SolveLevel& SL = CL->sl;
        SL.nl = nl;
        SL.bmax = bm;
        SL.bsz = DL.bsz;
        SL.pos = at<long long>(mt, o_pos);
        SL.kfin = DL.kfin;
        SL.C_ptr = DL.C_ptr;
        SL.C_nb = DL.C_nb;
        SL.chain = DL.chain;
        SL.Qt_off = DL.Qt_off;
        SL.L11_off = DL.L11_off;
        SL.U11_off = DL.U11_off;
        SL.Linv_off = DL.Linv_off;
        SL.Uinv_off = DL.Uinv_off;
        SL.Lbar_off = DL.Lbar_off;
        SL.Ubar_off = DL.Ubar_off;
        SL.Lself_off = DL.Lself_off;
        SL.Uself_off = DL.Uself_off;
        if (streamed) {
          // the solve reads the compact host arena
          Packer ps;
          const size_t q_Qt = ps.add(lQt), q_L11 = ps.add(lL11), q_U11 = ps.add(lU11), q_Li = ps.add(lLinv), q_Ui = ps.add(lUinv),
                       q_Lb = ps.add(lLbar), q_Ub = ps.add(lUbar), q_Ls = ps.add(lLself), q_Us = ps.add(lUself);
          ps.upload(CL->solve_meta, st);
          CK(cudaStreamSynchronize(st));
          const DBuf& sm2 = CL->solve_meta;
          SL.chain = nullptr;  // set by assemble_streamed_chains at the end of the factorization
          SL.Qt_off = at<long long>(sm2, q_Qt);
          SL.L11_off = at<long long>(sm2, q_L11);
          SL.U11_off = at<long long>(sm2, q_U11);
          SL.Linv_off = at<long long>(sm2, q_Li);
          SL.Uinv_off = at<long long>(sm2, q_Ui);
          SL.Lbar_off = at<long long>(sm2, q_Lb);
          SL.Ubar_off = at<long long>(sm2, q_Ub);
          SL.Lself_off = at<long long>(sm2, q_Ls);
          SL.Uself_off = at<long long>(sm2, q_Us);
        }
        // solve traffic (nrhs = 1): chain read (Qtilde twice) + vector
        C->solve_bytes += (double)lvl_bytes;
        for (int t = 0; t < nl; ++t) C->solve_bytes += 16.0 * (double)cur.bsz[t] * cur.bsz[t];  // second Qtilde pass
        C->solve_bytes += 4.0 * 16.0 * (double)S.n;

        C->schur_levels[l] = {C->schur_flops_exec - sexec_lv0, C->schur_bytes_exec - sbexec_lv0, 0.0};
        mark("records done");
        if (verbose)
          std::fprintf(stderr, "[h2g] level %d: algorithmic GFLOP total %.1f, Schur %.1f (executed %.1f)\n", l, (flops - flops_lv0) / 1e9,
                       (sflops - sflops_lv0) / 1e9, (C->schur_flops_exec - sexec_lv0) / 1e9);
        // ---- merge to level lp (finish_level + merge_permute)
        const LevelSym& YP = P->levels[li + 1];
        LevelData nxt;
        nxt.bsz.resize(nlp);
        nxt.korig.resize(nlp);
        nxt.pos.resize(nlp);
        long long off = 0;
        const int firstp = Structure::first(lp);
        for (int P2 = 0; P2 < nlp; ++P2) {
          nxt.bsz[P2] = kfin[2 * P2] + kfin[2 * P2 + 1];
          nxt.korig[P2] = static_cast<int>(M->basis_rank[firstp + P2]);
          nxt.pos[P2] = off;
          off += nxt.bsz[P2];
        }
        if (off != active_new) throw Error(H2G_ERR_INVALID_INPUT, "merge_permute: parent layout does not match the permutation");
        nxt.bmax = std::max(1, *std::max_element(nxt.bsz.begin(), nxt.bsz.end()));
        const size_t bbp = (size_t)nxt.bmax * nxt.bmax;
        const long long ndtot = pack_offsets(YP.drow, YP.dcol, nxt.bsz, nxt.doff);
        // Merge (finish_level :445-475 + merge_permute :483-584). Every fill
        // block that survives already sits in its compact core
        // Z = V_a^H F conj(V_c) (segment ends above), so the parent blocks are
        // assembled by copies: couplings / dense corners first, cores
        // accumulated on top (dst = pad(S) + Z).
        std::vector<CopyDesc> cd;  // dst pointers relative to nxt.D, fixed up after allocation
        struct PendingZ {
          int a, c, fi, kind;
          long long doff;  // element offset of the destination in nxt.D / nxt.F
          int ldd;
        };
        std::vector<PendingZ> pend;
        const auto& admL = S.adm[l];
        for (size_t pq = 0; pq < YP.drow.size(); ++pq) {
          const int Pr = YP.drow[pq], Pc = YP.dcol[pq];
          const long long dbase = nxt.doff[pq];
          const int ldd = nxt.bsz[Pr];
          for (int ia = 0; ia < 2; ++ia)
            for (int ic = 0; ic < 2; ++ic) {
              const int a = 2 * Pr + ia, c = 2 * Pc + ic;
              const int ro = ia ? kfin[2 * Pr] : 0, co = ic ? kfin[2 * Pc] : 0;
              const long long doff = dbase + ro + (long long)co * ldd;
              const int di = Y.dense_index(a, c);
              if (di >= 0) {
                const int ea = cur.bsz[a] - kfin[a], ec = cur.bsz[c] - kfin[c];
                if (kfin[a] && kfin[c]) {
                  cd.push_back({cur.D.as<cplx>() + cur.doff[di] + ea + (size_t)ec * cur.bsz[a], reinterpret_cast<cplx*>(doff * 16), cur.bsz[a], ldd, kfin[a], kfin[c], 0, 0});
                }
              } else {
                const Pair hp{a + Y.first, c + Y.first};
                auto it = std::lower_bound(admL.begin(), admL.end(), hp, [](const Pair& x, const Pair& y) { return x.row < y.row || (x.row == y.row && x.col < y.col); });
                if (it == admL.end() || it->row != hp.row || it->col != hp.col)
                  throw Error(H2G_ERR_INVALID_INPUT, "merge_permute: child block is neither dense nor admissible");
                const int64_t gi = S.adm_offset[l] + (it - admL.begin());
                const int ka = cur.korig[a], kc = cur.korig[c];
                if (ka && kc) {
                  cd.push_back({M->coup.as<cplx>() + M->coup_off[gi], reinterpret_cast<cplx*>(doff * 16), ka, ldd, ka, kc, 0, 0});
                }
                const int fi = Y.fill_index(a, c);
                if (fi >= 0 && fex[fi] && kfin[a] && kfin[c]) pend.push_back({a, c, fi, 0, doff, ldd});
              }
            }
        }
        // carried fill-in moves to the parent pair (content flags first: they
        // seed the next level's segment plan)
        std::vector<int> fexp(YP.frow.size(), 0);
        for (size_t f = 0; f < Y.frow.size(); ++f) {
          if (Y.fadm[f] >= 0 || !fex[f]) continue;
          const int pf = Y.carried_parent[f];
          if (pf < 0) throw Error(H2G_ERR_INTERNAL, "carried fill without a parent target");
          fexp[pf] = 1;
        }
        const bool next_factorized = lp >= stop;
        if (next_factorized) {
          nxt.front = build_front(YP, P->sched[li + 1], P->work[li + 1], nxt.bsz, fexp);
          nxt.has_front = true;
          nxt.foff = nxt.front.foff;
        }
        const long long nftot = next_factorized ? nxt.front.pool_elems : pack_offsets(YP.frow, YP.fcol, nxt.bsz, nxt.foff);
        for (size_t f = 0; f < Y.frow.size(); ++f) {
          if (Y.fadm[f] >= 0 || !fex[f]) continue;
          const int pf = Y.carried_parent[f];
          const int j = Y.frow[f], c = Y.fcol[f];
          if (!kfin[j] || !kfin[c]) continue;
          if (nxt.foff[pf] < 0) throw Error(H2G_ERR_INTERNAL, "carried fill has no storage at the next level");
          const int ro = (j & 1) ? kfin[j - 1] : 0, co = (c & 1) ? kfin[c - 1] : 0;
          const int ldd = nxt.bsz[YP.frow[pf]];
          pend.push_back({j, c, static_cast<int>(f), 1, nxt.foff[pf] + ro + (long long)co * ldd, ldd});
        }
        nxt.fex_host = fexp;
        for (const auto& pg : pend)
          if (!core_ptr_h[pg.fi]) throw Error(H2G_ERR_INTERNAL, "fill block with content has no core");
        // the level-l fill pool and scratch are dead
        cur.F.release();
        cur.fex.release();
        cur.Vp.release();
        mark("merge: fill pool released");
        // (1) parent dense blocks and padded transfers from the level-l dense
        // pool, which is then released before the parent fill pool exists
        ensure((size_t)(std::max<long long>(ndtot, 1) + (long long)nlp * bbp) * 16, CL.get());
        nxt.D.alloc(std::max<long long>(ndtot, 1) * 16, st, true);
        nxt.V0.alloc((size_t)nlp * bbp * 16, st, true);
        cplx* Dp = nxt.D.as<cplx>();
        for (size_t q = 0; q < cd.size(); ++q) cd[q].dst = Dp + reinterpret_cast<long long>(cd[q].dst) / 16;
        // padded transfers (finish_level :464-474)
        for (int P2 = 0; P2 < nlp; ++P2) {
          const int id = firstp + P2;
          const int k1 = cur.korig[2 * P2], k2 = cur.korig[2 * P2 + 1], kp = nxt.korig[P2];
          const int rows = static_cast<int>(M->basis_rows[id]);
          const cplx* T = M->basis.as<cplx>() + M->basis_off[id];
          cplx* dst = nxt.V0.as<cplx>() + (size_t)P2 * bbp;
          if (kp == 0) continue;
          if (k1) cd.push_back({T, dst, rows, nxt.bsz[P2], k1, kp, 0, 0});
          if (k2) cd.push_back({T + k1, dst + kfin[2 * P2], rows, nxt.bsz[P2], k2, kp, 0, 0});
        }
        DBuf dcd, dcz;
        upload(dcd, cd, st);
        ctx->prof.begin(PC_MERGE, st);
        launch_copy(dcd.as<CopyDesc>(), static_cast<int>(cd.size()), st);
        ctx->prof.end(st);
        cur.D.release();  // stream-ordered: reused only after the copies above
        mark("merge: dense blocks assembled");
        // (2) the parent fill pool; cores accumulate on top of the copies
        // (dst = pad(S) + Z). When HBM is short the device-resident cores
        // move to pinned host memory first (they are read once, below).
        {
          const size_t need = (size_t)std::max<long long>(nftot, 1) * 16 + YP.frow.size() * 4 + 16;
          ensure(need, CL.get());
          for (size_t ci = 0; ci < core_chunks.size() && BlockCache::get().headroom() < need + kMargin; ++ci) {
            DBuf& dch = core_chunks[ci];
            if (!dch.p) continue;
            core_hchunks.emplace_back();
            HBuf& hch = core_hchunks.back();
            hch.alloc(dch.bytes);
            CK(cudaMemcpyAsync(hch.p, dch.p, dch.bytes, cudaMemcpyDeviceToHost, st));
            const char* d0 = static_cast<const char*>(dch.p);
            for (auto& cp : core_ptr_h) {
              const char* q = reinterpret_cast<const char*>(cp);
              if (q >= d0 && q < d0 + dch.bytes) cp = reinterpret_cast<cplx*>(static_cast<char*>(hch.p) + (q - d0));
            }
            CK(cudaStreamSynchronize(st));
            dch.release();
            BlockCache::get().trim();
          }
        }
        nxt.F.alloc(std::max<long long>(nftot, 1) * 16, st, true);
        nxt.fex.alloc(std::max<size_t>(YP.frow.size(), 1) * 4, st, true);
        cplx* Fp = nxt.F.as<cplx>();
        std::vector<CopyDesc> cz;
        for (const auto& pg : pend) cz.push_back({core_ptr_h[pg.fi], (pg.kind ? Fp : Dp) + pg.doff, kfin[pg.a], pg.ldd, kfin[pg.a], kfin[pg.c], 1, 0});
        mark("merge descriptors built");
        // cores staged in pinned host memory come back chunk by chunk through
        // a device buffer (one bulk copy over the host link per chunk) instead
        // of being read element-wise by the copy kernel
        if (!core_hchunks.empty()) {
          size_t maxb = 0;
          for (auto& hch : core_hchunks) maxb = std::max(maxb, hch.bytes);
          DBuf stg;
          if (BlockCache::get().headroom() >= maxb + (kMargin >> 2)) stg.alloc(maxb, st);
          if (stg.p) {
            std::vector<CopyDesc> rest;
            std::vector<std::vector<CopyDesc>> grp(core_hchunks.size());
            for (const CopyDesc& d : cz) {
              const char* q = reinterpret_cast<const char*>(d.src);
              size_t hi = 0;
              for (; hi < core_hchunks.size(); ++hi) {
                const char* h0 = static_cast<const char*>(core_hchunks[hi].p);
                if (q >= h0 && q < h0 + core_hchunks[hi].bytes) break;
              }
              if (hi == core_hchunks.size()) {
                rest.push_back(d);
                continue;
              }
              CopyDesc r = d;
              r.src = reinterpret_cast<const cplx*>(static_cast<const char*>(stg.p) + (q - static_cast<const char*>(core_hchunks[hi].p)));
              grp[hi].push_back(r);
            }
            ctx->prof.begin(PC_MERGE, st);
            for (size_t hi = 0; hi < core_hchunks.size(); ++hi) {
              if (grp[hi].empty()) continue;
              CK(cudaMemcpyAsync(stg.p, core_hchunks[hi].p, core_hchunks[hi].bytes, cudaMemcpyHostToDevice, st));
              DBuf dg;
              upload(dg, grp[hi], st);
              launch_copy(dg.as<CopyDesc>(), static_cast<int>(grp[hi].size()), st);
              CK(cudaStreamSynchronize(st));  // the staging buffer is reused by the next chunk
              ++launches;
            }
            ctx->prof.end(st);
            cz.swap(rest);
          }
        }
        upload(dcz, cz, st);
        ctx->prof.begin(PC_MERGE, st);
        launch_copy(dcz.as<CopyDesc>(), static_cast<int>(cz.size()), st);
        ctx->prof.end(st);
        C->klaunch[PC_MERGE] += (!cd.empty()) + (!cz.empty());
        launches += (!cd.empty()) + (!cz.empty());
        if (!fexp.empty()) CK(cudaMemcpyAsync(nxt.fex.p, fexp.data(), fexp.size() * 4, cudaMemcpyHostToDevice, st));
        CK(cudaGetLastError());
        mark("merge launched");
        CK(cudaStreamSynchronize(st));  // temporaries die here
        size_t core_bytes = 0, core_host_bytes = 0;
        for (auto& ch : core_chunks) core_bytes += ch.bytes;
        for (auto& ch : core_hchunks) core_host_bytes += ch.bytes;
        core_chunks.clear();
        core_hchunks.clear();
        core_page = nullptr;

        if (verbose) {
          size_t fr = 0, tot = 0;
          cudaMemGetInfo(&fr, &tot);
          std::fprintf(stderr,
                       "[h2g] level %d: merge done at %.3f s; fill front pool %.2f GB (all full blocks %.2f GB, %d segments), cores %.2f GB "
                       "(+ %.2f GB host-staged), next D %.2f GB, next F %.2f GB; device free %.2f of %.2f GB\n",
                       l, wall() - tlev, cur.front.pool_elems * 16.0 / 1e9, cur.front.full_elems_total * 16.0 / 1e9, cur.front.K, core_bytes / 1e9,
                       core_host_bytes / 1e9,
                       nxt.D.bytes / 1e9, nxt.F.bytes / 1e9, fr / 1e9, tot / 1e9);
          std::fprintf(stderr, "[h2g] chains offloaded to host so far: %.2f GB\n", offloaded / 1e9);
        }
        tlev = wall();
        C->levels.push_back(std::move(CL));
        cur = std::move(nxt);
        last_level = lp;
        if (hooks && hooks->after_merge) {
          // the parent level's state (nothing projected yet); its structure
          // is the next plan level
          std::vector<char> rot0(cur.bsz.size(), 0);
          std::vector<int> el0(cur.bsz.size(), 0);
          std::vector<int64_t> src_used(C->levels.back()->src.begin(), C->levels.back()->src.end());
          h2g_state ms;
          ms.ctx = ctx;
          ms.M = M;
          ms.cur = &cur;
          ms.Y = &P->levels[li + 1];
          ms.level = lp;
          ms.d_kfin = nullptr;
          ms.rotated = &rot0;
          ms.elim = &el0;
          ms.perm_src = &src_used;
          CK(cudaStreamSynchronize(st));
          hooks->after_merge(hooks->user, &ms);
        }
        if (elim == 0 && l > stop) {
          C->stop_level = l;
          ++li;
          break;
        }
      }
    }

    // ---- root (factorization.hpp:637-651)
    {
      const int lv = last_level;
      const LevelSym* YR = nullptr;
      for (const auto& Y : P->levels)
        if (Y.level == lv) YR = &Y;
      if (!YR) throw Error(H2G_ERR_INTERNAL, "root level structure missing");
      long long nroot = 0;
      for (int b : cur.bsz) nroot += b;
      C->root_size = nroot;
      bool needs_paint = false;
      for (int la = std::max(l0, 0); la <= lv && l0 >= 0; ++la)
        if (!S.adm[la].empty()) needs_paint = true;
      if (nroot > 0) {
        C->root.alloc((size_t)nroot * nroot * 16, st, true);
        cplx* R0 = C->root.as<cplx>();
        const size_t bb = (size_t)cur.bmax * cur.bmax;
        std::vector<CopyDesc> cd;
        for (size_t q = 0; q < YR->drow.size(); ++q) {
          const int r = YR->drow[q], c = YR->dcol[q];
          if (!cur.bsz[r] || !cur.bsz[c]) continue;
          cd.push_back({cur.D.as<cplx>() + cur.doff[q], R0 + cur.pos[r] + (size_t)cur.pos[c] * nroot, cur.bsz[r], (int)nroot, cur.bsz[r], cur.bsz[c], 0, 0});
        }
        DBuf dcd;
        upload(dcd, cd, st);
        launch_copy(dcd.as<CopyDesc>(), static_cast<int>(cd.size()), st);
        ++launches;
        // paint (FactorState::paint, factorization.hpp:204-234): admissible
        // blocks of this level and of every coarser level >= l0, expanded
        // to this level's clusters (expand_to_level :191-201), plus the
        // ledger / carried fill-in held in F
        std::vector<DBuf> Ebuf;  // Ebuf[lv - la]: expanded bases per cluster at ancestor level la
        std::vector<std::vector<long long>> Eoff;
        if (needs_paint) {
          const int nlv = static_cast<int>(cur.bsz.size());
          const int flv = Structure::first(lv);
          const int lmin = std::max(l0, 0);
          auto anc = [&](int u, int la) { return ((flv + u + 1) >> (lv - la)) - 1; };  // heap id of u's ancestor at level la
          auto kor = [&](int id) { return static_cast<int>(M->basis_rank[id]); };
          Ebuf.resize(lv - lmin + 1);
          Eoff.resize(lv - lmin + 1);
          for (int la = lv - 1; la >= lmin; --la) {
            const int d = lv - la;
            long long top = 0;
            Eoff[d].resize(nlv);
            for (int u = 0; u < nlv; ++u) Eoff[d][u] = top, top += (long long)cur.bsz[u] * kor(anc(u, la));
            Ebuf[d].alloc(std::max<long long>(top, 1) * 16, st, true);
            std::vector<GemmDesc> ge;
            for (int u = 0; u < nlv; ++u) {
              const int a = anc(u, la), ch = anc(u, la + 1);
              const int ka = kor(a), kc = kor(ch), b = cur.bsz[u];
              if (!ka || !kc || !b) continue;
              const int roff = (ch == 2 * a + 1) ? 0 : kor(2 * a + 1);
              const cplx* T = M->basis.as<cplx>() + M->basis_off[a] + roff;
              const cplx* Ein = d == 1 ? cur.V0.as<cplx>() + (size_t)u * bb : Ebuf[d - 1].as<cplx>() + Eoff[d - 1][u];
              ge.push_back({Ein, T, Ebuf[d].as<cplx>() + Eoff[d][u], b, (int)M->basis_rows[a], b, b, ka, kc, OP_N, OP_N, 1.0, 0.0});
            }
            DBuf dge;
            upload(dge, ge, st);
            launch_gemm(dge.as<GemmDesc>(), static_cast<int>(ge.size()), st, 0);
            launches += !ge.empty();
          }
          auto Eptr = [&](int u, int la) -> const cplx* {
            return la == lv ? cur.V0.as<cplx>() + (size_t)u * bb : Ebuf[lv - la].as<cplx>() + Eoff[lv - la][u];
          };
          // X_u = E_u S (b_u x k_col), then root(u, v) = X_u E_v^T
          std::vector<GemmDesc> gx, gm;
          std::vector<long long> xoff;
          long long xtop = 0;
          struct Job {
            int u, la, kc, c0, nv;
            const cplx* S;
            int kr;
          };
          std::vector<Job> jobs;
          for (int la = lmin; la <= lv; ++la) {
            for (size_t pq = 0; pq < S.adm[la].size(); ++pq) {
              const int R = S.adm[la][pq].row, Cc = S.adm[la][pq].col;
              const int kr = kor(R), kc = kor(Cc);
              if (!kr || !kc) continue;
              const cplx* Sm = M->coup.as<cplx>() + M->coup_off[S.adm_offset[la] + pq];
              const int span = 1 << (lv - la);
              const int u0 = ((R + 1) << (lv - la)) - 1 - flv, v0 = ((Cc + 1) << (lv - la)) - 1 - flv;
              for (int u = u0; u < u0 + span; ++u) {
                if (!cur.bsz[u]) continue;
                jobs.push_back({u, la, kc, v0, span, Sm, kr});
                xoff.push_back(xtop);
                xtop += (long long)cur.bsz[u] * kc;
              }
            }
          }
          DBuf xbuf;
          xbuf.alloc(std::max<long long>(xtop, 1) * 16, st);
          for (size_t j = 0; j < jobs.size(); ++j) {
            const Job& J = jobs[j];
            const int b = cur.bsz[J.u];
            cplx* X = xbuf.as<cplx>() + xoff[j];
            gx.push_back({Eptr(J.u, J.la), J.S, X, b, J.kr, b, b, J.kc, J.kr, OP_N, OP_N, 1.0, 0.0});
            for (int v = J.c0; v < J.c0 + J.nv; ++v) {
              if (!cur.bsz[v]) continue;
              gm.push_back({X, Eptr(v, J.la), R0 + cur.pos[J.u] + (size_t)cur.pos[v] * nroot, b, cur.bsz[v], (int)nroot, b, cur.bsz[v], J.kc, OP_N,
                            OP_T, 1.0, 0.0});
            }
          }
          DBuf dgx, dgm;
          upload(dgx, gx, st);
          upload(dgm, gm, st);
          launch_gemm(dgx.as<GemmDesc>(), static_cast<int>(gx.size()), st, cur.bmax);
          launch_gemm(dgm.as<GemmDesc>(), static_cast<int>(gm.size()), st, cur.bmax);
          launches += (!gx.empty()) + (!gm.empty());
          // fill-in deltas (zero where no fill was deposited)
          std::vector<CopyDesc> cf;
          for (size_t f = 0; f < YR->frow.size(); ++f) {
            const int u = YR->frow[f], v = YR->fcol[f];
            if (!cur.bsz[u] || !cur.bsz[v]) continue;
            if (cur.foff[f] < 0 || (f < cur.fex_host.size() && !cur.fex_host[f])) continue;  // no content (segmented storage may be shared)
            cf.push_back({cur.F.as<cplx>() + cur.foff[f], R0 + cur.pos[u] + (size_t)cur.pos[v] * nroot, cur.bsz[u], (int)nroot, cur.bsz[u], cur.bsz[v], 1, 0});
          }
          DBuf dcf;
          upload(dcf, cf, st);
          launch_copy(dcf.as<CopyDesc>(), static_cast<int>(cf.size()), st);
          launches += !cf.empty();
          CK(cudaStreamSynchronize(st));
        }
        DBuf scratch;
        scratch.alloc(64, st);
        ctx->prof.begin(PC_ROOT, st);
        const long long l0c = launches;
        root_lu(C->root.as<cplx>(), static_cast<int>(nroot), 1e-13, ctx->d_err, scratch.p, st, &launches);
        ctx->prof.end(st);
        C->klaunch[PC_ROOT] += launches - l0c;
        C->kflops[PC_ROOT] += 8.0 / 3.0 * (double)nroot * nroot * nroot;
        C->kbytes[PC_ROOT] += 2.0 * 16.0 * (double)nroot * nroot;
        CK(cudaGetLastError());
        check_device_error(ctx, C->stop_level);
        flops += 8.0 / 3.0 * (double)nroot * nroot * nroot;
        C->storage_bytes += 2 * 16 * (size_t)nroot * nroot;
        C->solve_bytes += 16.0 * (double)nroot * nroot;
      }
    }
    // ---- the chain returns to HBM: with the level pools gone, levels that
    // were streamed or offloaded to host memory move back while they fit
    // (coarsest first), so the solve reads them at HBM speed
    {
      cur.D.release();
      cur.F.release();
      cur.V0.release();
      cur.Vp.release();
      cur.fex.release();
      // streamed levels: Qt block and chunks joined into one arena (HBM if it fits, else pinned host memory)
      for (auto it = C->levels.rbegin(); it != C->levels.rend(); ++it) {
        ChainLevelHost& X = **it;
        if (X.compact_elems == 0 || X.arena.p || X.harena.p) continue;
        CK(cudaStreamSynchronize(st));
        BlockCache::get().trim();
        const size_t bytes = (size_t)X.compact_elems * 16;
        char* base;
        if (BlockCache::get().headroom() >= bytes + (kMargin >> 2)) {
          X.arena.alloc(bytes, st);
          base = static_cast<char*>(X.arena.p);
        } else {
          X.harena.alloc(bytes);
          base = static_cast<char*>(X.harena.p);
        }
        CK(cudaMemcpyAsync(base, X.qchunk.p, X.qchunk.bytes, cudaMemcpyDefault, st));
        for (auto& ck : X.chunks)
          CK(cudaMemcpyAsync(base + (size_t)ck.begin * 16, ck.src(), (size_t)ck.len * 16, cudaMemcpyDefault, st));
        CK(cudaStreamSynchronize(st));
        X.chunks.clear();
        X.hpages.clear();
        X.hpage = nullptr;
        X.qchunk.release();
        X.sl.chain = reinterpret_cast<cplx*>(base);
      }
      double back = 0.0, kept = 0.0;
      bool synced = false;
      for (auto it = C->levels.rbegin(); it != C->levels.rend(); ++it) {
        ChainLevelHost& X = **it;
        if (!X.harena.p || X.arena.p) continue;
        if (!synced) {
          CK(cudaStreamSynchronize(st));
          BlockCache::get().trim();
          synced = true;
        }
        const size_t bytes = X.harena.bytes;
        if (BlockCache::get().headroom() < bytes + kMargin) {
          kept += bytes;
          continue;
        }
        X.arena.alloc(bytes, st);
        CK(cudaMemcpyAsync(X.arena.p, X.harena.p, bytes, cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
        X.sl.chain = X.arena.as<cplx>();
        X.harena.release();
        back += bytes;
      }
      if (verbose && (back > 0 || kept > 0))
        std::fprintf(stderr, "[h2g] chain levels moved back to HBM: %.2f GB; left in host memory: %.2f GB\n", back / 1e9, kept / 1e9);
    }
    CK(cudaEventRecord(ctx->ev1, st));
    CK(cudaEventSynchronize(ctx->ev1));
    if (verbose) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, ctx->device) == cudaSuccess) {
        uint64_t a = 0, b = 0, c = 0, d = 0;
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &a);
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemHigh, &b);
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &c);
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &d);
        std::fprintf(stderr, "[h2g] pool reserved %.2f GB (high %.2f), used %.2f GB (high %.2f)\n", a / 1e9, b / 1e9, c / 1e9, d / 1e9);
      }
    }
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    C->factor_ms = ms;
    C->factor_launches = launches;
    if (ctx->prof.on) {
      std::map<std::pair<int, int>, double> per;
      std::vector<Prof::Rec> all(ctx->prof.recs);
      all.insert(all.end(), ctx->prof_side.recs.begin(), ctx->prof_side.recs.end());
      all.insert(all.end(), ctx->prof_aux.recs.begin(), ctx->prof_aux.recs.end());
      for (const auto& r : all) {
        float e = 0.f;
        cudaEventElapsedTime(&e, r.a, r.b);
        C->kms[r.cls] += e;
        per[{r.level, r.cls}] += e;
        if (r.cls == PC_SCHUR && C->schur_levels.count(r.level)) C->schur_levels[r.level][2] += e;
      }
      if (verbose) {
        static const char* nm[PC_N] = {"complement", "gram", "colnorm", "eig1", "head", "panel", "schur", "merge", "root", "other", "eigvec", "eig1b"};
        for (const auto& kv : per) std::fprintf(stderr, "[h2g] level %d %-10s %9.2f ms\n", kv.first.first, nm[kv.first.second], kv.second);
      }
    }
    C->factor_flops = flops;
    C->schur_flops = sflops;
    C->schur_bytes = sbytes;
    C->kflops[PC_SCHUR] = sflops;
    C->kbytes[PC_SCHUR] = sbytes;
    ++ctx->refs;  // the chain holds the context
    *out = C.release();
  });
}

extern "C" {

int h2g_factorize(h2g_context* ctx, const h2g_matrix* m, double eps, int32_t stop_level, int32_t schedule, h2g_chain** out, h2g_error* err) {
  return factorize_impl(ctx, m, eps, stop_level, schedule, nullptr, out, err);
}

int h2g_factorize_hooked(h2g_context* ctx, const h2g_matrix* m, double eps, int32_t stop_level, const h2g_factorize_hooks* hooks, h2g_chain** out,
                         h2g_error* err) {
  return factorize_impl(ctx, m, eps, stop_level, H2G_SCHEDULE_SERIAL, hooks, out, err);
}

int h2g_factorize_dist(h2g_context* ctx, const h2g_matrix* m, double eps, int32_t stop_level, const h2g_dist* dist, h2g_chain** out, h2g_error* err) {
  if (!dist) {
    set_error(err, H2G_ERR_INVALID_INPUT, "factorize_dist: null dist");
    return H2G_ERR_INVALID_INPUT;
  }
  return factorize_impl(ctx, m, eps, stop_level, H2G_SCHEDULE_SUBTREE, nullptr, out, err, dist);
}

int h2g_partition_plan(const h2g_matrix_desc* d, int32_t stop_level, int32_t level, int64_t* counts, int32_t* batch_of, int32_t* part_batch,
                       int32_t* dense_part, int32_t* fill_part, int32_t* dense_rc, int32_t* fill_rc, h2g_error* err) {
  return guarded(err, [&] {
    if (!d || !counts) throw Error(H2G_ERR_INVALID_INPUT, "null argument");
    const Structure S = structure_from_desc(d);
    int stop = S.depth + 1;
    if (S.l0 >= 0) stop = stop_level >= 0 ? stop_level : S.l0;
    const std::vector<LevelSym> levels = build_levels(S, stop);
    const LevelSym* Y = nullptr;
    for (const auto& L : levels)
      if (L.level == level && L.level >= stop) Y = &L;
    if (!Y) throw Error(H2G_ERR_INVALID_INPUT, "partition_plan: level is not factorized");
    const LevelSchedule SC = build_schedule(*Y, H2G_SCHEDULE_SUBTREE);
    const LevelWork W = build_work(*Y, SC, 1);
    counts[0] = Y->nl;
    counts[1] = static_cast<int64_t>(SC.batch_ptr.size()) - 1;
    counts[2] = static_cast<int64_t>(Y->drow.size());
    counts[3] = static_cast<int64_t>(Y->frow.size());
    if (batch_of)
      for (int t = 0; t < Y->nl; ++t) batch_of[t] = SC.order[t];
    if (part_batch)
      for (int q = 0; q <= kInteriorParts; ++q) part_batch[q] = SC.part_batch[q];
    const std::vector<PartList> parts = build_parts(*Y, SC, W);
    auto mark = [&](int32_t* out, size_t n, bool fill) {
      if (!out) return;
      for (size_t q = 0; q < n; ++q) out[q] = -1;
      for (int sp = 0; sp < kInteriorParts; ++sp)
        for (int q : (fill ? parts[sp].fblk : parts[sp].dblk)) out[q] = out[q] == -1 ? sp : -2;  // -2: written by two subtrees (never)
    };
    mark(dense_part, Y->drow.size(), false);
    mark(fill_part, Y->frow.size(), true);
    if (dense_rc)
      for (size_t q = 0; q < Y->drow.size(); ++q) dense_rc[2 * q] = Y->drow[q], dense_rc[2 * q + 1] = Y->dcol[q];
    if (fill_rc)
      for (size_t q = 0; q < Y->frow.size(); ++q) fill_rc[2 * q] = Y->frow[q], fill_rc[2 * q + 1] = Y->fcol[q];
  });
}

int h2g_chain_dist_stats(const h2g_chain* c, double* out3) {
  if (!c || !out3) return H2G_ERR_INVALID_INPUT;
  out3[0] = c->dist_sent_bytes;
  out3[1] = c->dist_total_bytes;
  out3[2] = c->dist_exchange_s;
  return H2G_OK;
}

int h2g_chain_destroy(h2g_chain* c) {
  if (!c) return H2G_OK;
  h2g_context* ctx = c->ctx;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  delete c;
  context_release(ctx);
  return H2G_OK;
}

// ------------------------------------------------------------------ solve
static void solve_device_impl(h2g_chain* C, cplx* y, int64_t n, int nrhs, int mode) {
  NvtxRange nv_solve("h2g solve");
  h2g_context* ctx = C->ctx;
  cudaStream_t st = ctx->stream;
  if (n != C->n) throw Error(H2G_ERR_INVALID_INPUT, fmt("solve: right-hand side has length %lld, factorization expects %lld", n, C->n));
  if (nrhs < 1) throw Error(H2G_ERR_INVALID_INPUT, "solve: nrhs must be >= 1");
  CK(cudaMemsetAsync(ctx->d_flag, 0, 4, st));
  launch_finite(y, n * nrhs, ctx->d_flag, st);
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, ctx->d_flag, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (bad) throw Error(H2G_ERR_NON_FINITE, "solve: right-hand side contains non-finite entries");
  if ((size_t)n * nrhs * 16 > C->tmpbuf.bytes) C->tmpbuf.alloc((size_t)n * nrhs * 16, st);
  cplx* tmp = C->tmpbuf.as<cplx>();
  const bool fwd = mode != H2G_BACKWARD, bwd = mode != H2G_FORWARD;
  // The record heads apply the factorization's stored L11^{-1} / U11^{-1}
  // (GEMVs over the chain data) in every mode: the sequential triangular
  // substitution (solve.hpp:47-50, :73-81) costs one block barrier per
  // eliminated row on the critical path. Set H2G_SOLVE_TRIANGULAR=1 for the
  // substitution form.
  static const bool tri = std::getenv("H2G_SOLVE_TRIANGULAR") && std::atoi(std::getenv("H2G_SOLVE_TRIANGULAR"));
  const int expl = (mode == H2G_APPLY_INVERSE_EXPLICIT || !tri) ? 1 : 0;
  long long launches = 1;
  // right-hand sides per pass of the level kernels: 2 * bmax * rchunk
  // complex of shared memory per CTA stays under ~150 KB (measured: 96 / 150 / 200 KB give 895 / 765 / 777 ms for 64 RHS on config 2)
  int bmax_all = 1;
  for (auto& CLp : C->levels) bmax_all = std::max(bmax_all, CLp->sl.bmax);
  const int smem_kb = std::getenv("H2G_SOLVE_SMEM_KB") ? std::max(1, std::atoi(std::getenv("H2G_SOLVE_SMEM_KB"))) : 150;  // read per call (tests force several groups)
  const int rchunk = std::max(1, std::min(nrhs, (int)(((size_t)smem_kb * 1024) / (2 * 16 * (size_t)bmax_all))));
  // dataflow level kernels (per-item dependency counters) by default; the
  // batch-synchronous cooperative kernels with H2G_SOLVE_BATCHED=1
  static const bool batched = std::getenv("H2G_SOLVE_BATCHED") && std::atoi(std::getenv("H2G_SOLVE_BATCHED"));
  // H2G_SOLVE_GROUPS=0: the groups of right-hand sides one after the other (one launch each) instead of side by side
  const bool side_by_side = !(std::getenv("H2G_SOLVE_GROUPS") && !std::atoi(std::getenv("H2G_SOLVE_GROUPS")));
  FlowGroups fg{};
  constexpr int kWaveGroups = 16;
  // cap on the gathered-partials buffers of one backward wave (H2G_SOLVE_PART_GB)
  const size_t part_budget = (size_t)((std::getenv("H2G_SOLVE_PART_GB") ? std::max(0.0, std::atof(std::getenv("H2G_SOLVE_PART_GB"))) : 8.0) * 1073741824.0);
  {
    int nlmax = 1;
    for (auto& CLp : C->levels) nlmax = std::max(nlmax, CLp->sl.nl);
    // [0] stall flag, then one counter block per right-hand-side group
    fg.rchunk = rchunk;
    fg.cstride = 4 * nlmax + 2;
    fg.part_stride = 0;
    const size_t cb = (1 + (size_t)fg.cstride * ((nrhs + rchunk - 1) / rchunk)) * sizeof(int);
    if (cb > C->flowcnt.bytes) C->flowcnt.alloc(cb, st);
    CK(cudaMemsetAsync(C->flowcnt.p, 0, sizeof(int), st));
  }
  CK(cudaEventRecord(ctx->ev0, st));
  if (fwd) {
    for (auto& CLp : C->levels) {
      ChainLevelHost& CL = *CLp;
      if (!batched && side_by_side) {
        // waves of at most kWaveGroups groups (more groups than that only thin out each group's CTAs)
        for (int c0 = 0; c0 < nrhs; c0 += kWaveGroups * rchunk) {
          launch_fwd_flow(CL.sl, CL.sched, CL.flow, y + (size_t)c0 * n, n, std::min(kWaveGroups * rchunk, nrhs - c0), expl, C->flowcnt.as<int>() + 1,
                          C->flowcnt.as<int>(), tmp + (size_t)c0 * n, fg, st);
          ++launches;
        }
      } else
        for (int c0 = 0; c0 < nrhs; c0 += rchunk) {
          if (batched)
            launch_fwd_level(CL.sl, CL.sched, y + (size_t)c0 * n, n, std::min(rchunk, nrhs - c0), expl, st);
          else
            launch_fwd_flow(CL.sl, CL.sched, CL.flow, y + (size_t)c0 * n, n, std::min(rchunk, nrhs - c0), expl, C->flowcnt.as<int>() + 1,
                            C->flowcnt.as<int>(), tmp + (size_t)c0 * n, fg, st);
          ++launches;
        }
      launch_permute(CL.d_src.as<long long>(), static_cast<long long>(CL.src.size()), y, tmp, n, nrhs, 0, st);
      launches += 2;
    }
    if (C->root_size > 0) {
      launch_root_trsv(C->root.as<cplx>(), static_cast<int>(C->root_size), y, n, nrhs, 0, st);
      ++launches;
    }
  }
  if (bwd) {
    if (C->root_size > 0) {
      launch_root_trsv(C->root.as<cplx>(), static_cast<int>(C->root_size), y, n, nrhs, 1, st);
      ++launches;
    }
    for (auto it = C->levels.rbegin(); it != C->levels.rend(); ++it) {
      ChainLevelHost& CL = **it;
      launch_permute(CL.d_src.as<long long>(), static_cast<long long>(CL.src.size()), y, tmp, n, nrhs, 1, st);
      launches += 2;
      const bool grouped = !batched && side_by_side;
      const size_t per_group = (batched ? CL.part_need : CL.flow_part) * rchunk;
      // groups per wave: every group of a wave has its own gathered-partials
      // buffer, together at most part_budget (then kWaveGroups) of them
      const int wave = grouped ? (int)std::max<size_t>(1, std::min<size_t>({(size_t)kWaveGroups, (size_t)(nrhs + rchunk - 1) / rchunk,
                                                                             part_budget / std::max<size_t>(1, per_group * 16)}))
                               : 1;
      const size_t need = per_group * 16 * wave;
      if (need > C->partbuf.bytes) C->partbuf.alloc(need, st);
      if (grouped) {
        fg.part_stride = (long long)per_group;
        for (int c0 = 0; c0 < nrhs; c0 += wave * rchunk) {
          launch_bwd_flow(CL.sl, CL.flow, y + (size_t)c0 * n, n, std::min(wave * rchunk, nrhs - c0), expl, C->partbuf.as<cplx>(), C->flowcnt.as<int>() + 1,
                          C->flowcnt.as<int>(), tmp + (size_t)c0 * n, fg, st);
          ++launches;
        }
      } else
        for (int c0 = 0; c0 < nrhs; c0 += rchunk) {
          if (batched)
            launch_bwd_level(CL.sl, CL.sched, y + (size_t)c0 * n, n, std::min(rchunk, nrhs - c0), expl, C->partbuf.as<cplx>(), st);
          else
            launch_bwd_flow(CL.sl, CL.flow, y + (size_t)c0 * n, n, std::min(rchunk, nrhs - c0), expl, C->partbuf.as<cplx>(), C->flowcnt.as<int>() + 1,
                            C->flowcnt.as<int>(), tmp + (size_t)c0 * n, fg, st);
          ++launches;
        }
    }
  }
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->ev1, st));
  CK(cudaEventSynchronize(ctx->ev1));
  if (!batched) {
    int stalled = 0;
    CK(cudaMemcpy(&stalled, C->flowcnt.p, sizeof(int), cudaMemcpyDeviceToHost));
    if (stalled) throw Error(H2G_ERR_INTERNAL, "solve: a dataflow dependency wait stalled (schedule inconsistent with the chain)");
  }
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  C->solve_ms = ms;
  C->solve_launches = launches;
}

int h2g_solve_device(h2g_chain* c, double* x_dev, int64_t n, int32_t nrhs, int32_t mode, h2g_error* err) {
  return guarded(err, [&] {
    if (!c || !x_dev) throw Error(H2G_ERR_INVALID_INPUT, "null argument");
    std::lock_guard<std::recursive_mutex> run_lock(c->ctx->run_mu);
    CK(cudaSetDevice(c->ctx->device));
    solve_device_impl(c, reinterpret_cast<cplx*>(x_dev), n, nrhs, mode);
  });
}

int h2g_solve(h2g_chain* c, const double* b, double* x, int64_t n, int32_t nrhs, int32_t mode, h2g_error* err) {
  return guarded(err, [&] {
    if (!c || !b || !x) throw Error(H2G_ERR_INVALID_INPUT, "null argument");
    std::lock_guard<std::recursive_mutex> run_lock(c->ctx->run_mu);
    CK(cudaSetDevice(c->ctx->device));
    if (n != c->n) throw Error(H2G_ERR_INVALID_INPUT, fmt("solve: right-hand side has length %lld, factorization expects %lld", n, c->n));
    if (nrhs < 1) throw Error(H2G_ERR_INVALID_INPUT, "solve: nrhs must be >= 1");
    cudaStream_t st = c->ctx->stream;
    const size_t bytes = (size_t)n * nrhs * 16;
    if (bytes > c->ybuf.bytes) c->ybuf.alloc(bytes, st);
    CK(cudaMemcpyAsync(c->ybuf.p, b, bytes, cudaMemcpyHostToDevice, st));
    solve_device_impl(c, c->ybuf.as<cplx>(), n, nrhs, mode);
    CK(cudaMemcpyAsync(x, c->ybuf.p, bytes, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

// ------------------------------------------------------------- inspection
int h2g_chain_info(const h2g_chain* c, int64_t* info) {
  if (!c || !info) return H2G_ERR_INVALID_INPUT;
  info[0] = c->n;
  info[1] = c->stop_level;
  info[2] = c->root_size;
  info[3] = static_cast<int64_t>(c->levels.size());
  info[4] = static_cast<int64_t>(c->storage_bytes);
  info[5] = c->schedule;
  return H2G_OK;
}

int h2g_chain_level(const h2g_chain* c, int32_t li, int64_t* out) {
  if (!c || li < 0 || li >= (int)c->levels.size()) return H2G_ERR_INVALID_INPUT;
  std::copy(c->levels[li]->diag.begin(), c->levels[li]->diag.end(), out);
  return H2G_OK;
}

int h2g_chain_records(const h2g_chain* c, int32_t li, int64_t* out) {
  if (!c || li < 0 || li >= (int)c->levels.size()) return H2G_ERR_INVALID_INPUT;
  std::copy(c->levels[li]->rec.begin(), c->levels[li]->rec.end(), out);
  return H2G_OK;
}

int h2g_chain_perm(const h2g_chain* c, int32_t li, int64_t* src) {
  if (!c || li < 0 || li >= (int)c->levels.size()) return H2G_ERR_INVALID_INPUT;
  std::copy(c->levels[li]->src.begin(), c->levels[li]->src.end(), src);
  return H2G_OK;
}

int h2g_chain_record_mats(const h2g_chain* c, int32_t li, int32_t ri, double* q, double* l11, double* u11) {
  return guarded(nullptr, [&] {
    if (!c || li < 0 || li >= (int)c->levels.size()) throw Error(H2G_ERR_INVALID_INPUT, "bad level index");
    const ChainLevelHost& CL = *c->levels[li];
    if (ri < 0 || ri >= (int)CL.rec_cluster.size()) throw Error(H2G_ERR_INVALID_INPUT, "bad record index");
    const int t = CL.rec_cluster[ri];
    const int b = CL.bsz[t], e = b - CL.kfin[t];
    cudaStream_t st = c->ctx->stream;
    const cplx* base = CL.chain_ptr();
    if (q) CK(cudaMemcpyAsync(q, base + CL.Qt_off[t], (size_t)b * b * 16, cudaMemcpyDefault, st));
    if (l11 && e) CK(cudaMemcpyAsync(l11, base + CL.L11_off[t], (size_t)e * e * 16, cudaMemcpyDefault, st));
    if (u11 && e) CK(cudaMemcpyAsync(u11, base + CL.U11_off[t], (size_t)e * e * 16, cudaMemcpyDefault, st));
    CK(cudaStreamSynchronize(st));
  });
}

int h2g_chain_record_blocks_sizes(const h2g_chain* c, int32_t li, int32_t ri, int64_t* sizes4) {
  if (!c || li < 0 || li >= (int)c->levels.size()) return H2G_ERR_INVALID_INPUT;
  const ChainLevelHost& CL = *c->levels[li];
  if (ri < 0 || ri >= (int)CL.rec_cluster.size()) return H2G_ERR_INVALID_INPUT;
  const int t = CL.rec_cluster[ri];
  const int kf = CL.kfin[t], e = CL.bsz[t] - kf;
  int64_t nl = 0, nu = 0, el = 0, eu = 0;
  if (e > 0) {
    for (int a = CL.R_ptr[t]; a < CL.R_ptr[t + 1]; ++a) ++nl, el += (int64_t)CL.bsz[CL.R_nb[a]] * e;
    for (int a = CL.C_ptr[t]; a < CL.C_ptr[t + 1]; ++a) ++nu, eu += (int64_t)CL.bsz[CL.C_nb[a]] * e;
    if (kf > 0) ++nl, ++nu, el += (int64_t)kf * e, eu += (int64_t)kf * e;
  }
  sizes4[0] = nl, sizes4[1] = el, sizes4[2] = nu, sizes4[3] = eu;
  return H2G_OK;
}

int h2g_chain_record_blocks(const h2g_chain* c, int32_t li, int32_t ri, int64_t* lpos, int64_t* lrows, double* ldata, int64_t* upos, int64_t* ucols,
                            double* udata) {
  return guarded(nullptr, [&] {
    if (!c || li < 0 || li >= (int)c->levels.size()) throw Error(H2G_ERR_INVALID_INPUT, "bad level index");
    const ChainLevelHost& CL = *c->levels[li];
    if (ri < 0 || ri >= (int)CL.rec_cluster.size()) throw Error(H2G_ERR_INVALID_INPUT, "bad record index");
    const int t = CL.rec_cluster[ri];
    const int kf = CL.kfin[t], e = CL.bsz[t] - kf;
    if (e == 0) return;
    cudaStream_t st = c->ctx->stream;
    const cplx* base = CL.chain_ptr();
    size_t q = 0, off = 0;
    for (int a = CL.R_ptr[t]; a < CL.R_ptr[t + 1]; ++a, ++q) {
      const int j = CL.R_nb[a];
      lpos[q] = CL.pos[j];
      lrows[q] = CL.bsz[j];
      CK(cudaMemcpyAsync(ldata + 2 * off, base + CL.Lbar_off[a], (size_t)CL.bsz[j] * e * 16, cudaMemcpyDefault, st));
      off += (size_t)CL.bsz[j] * e;
    }
    if (kf > 0) {
      lpos[q] = CL.pos[t] + e;
      lrows[q] = kf;
      CK(cudaMemcpyAsync(ldata + 2 * off, base + CL.Lself_off[t], (size_t)kf * e * 16, cudaMemcpyDefault, st));
    }
    q = 0, off = 0;
    for (int a = CL.C_ptr[t]; a < CL.C_ptr[t + 1]; ++a, ++q) {
      const int cc = CL.C_nb[a];
      upos[q] = CL.pos[cc];
      ucols[q] = CL.bsz[cc];
      CK(cudaMemcpyAsync(udata + 2 * off, base + CL.Ubar_off[a], (size_t)CL.bsz[cc] * e * 16, cudaMemcpyDefault, st));
      off += (size_t)CL.bsz[cc] * e;
    }
    if (kf > 0) {
      upos[q] = CL.pos[t] + e;
      ucols[q] = kf;
      CK(cudaMemcpyAsync(udata + 2 * off, base + CL.Uself_off[t], (size_t)kf * e * 16, cudaMemcpyDefault, st));
    }
    CK(cudaStreamSynchronize(st));
  });
}

int h2g_chain_root(const h2g_chain* c, double* root_l, double* root_u) {
  return guarded(nullptr, [&] {
    if (!c) throw Error(H2G_ERR_INVALID_INPUT, "null chain");
    const int64_t r = c->root_size;
    if (r == 0) return;
    std::vector<std::complex<double>> A((size_t)r * r);
    CK(cudaMemcpyAsync(A.data(), c->root.p, (size_t)r * r * 16, cudaMemcpyDeviceToHost, c->ctx->stream));
    CK(cudaStreamSynchronize(c->ctx->stream));
    for (int64_t j = 0; j < r; ++j)
      for (int64_t i = 0; i < r; ++i) {
        const auto v = A[i + j * r];
        const std::complex<double> l = i > j ? v : (i == j ? 1.0 : 0.0);
        const std::complex<double> u = i <= j ? v : 0.0;
        if (root_l) root_l[2 * (i + j * r)] = l.real(), root_l[2 * (i + j * r) + 1] = l.imag();
        if (root_u) root_u[2 * (i + j * r)] = u.real(), root_u[2 * (i + j * r) + 1] = u.imag();
      }
  });
}

uint64_t h2g_chain_hash(const h2g_chain* c) {
  if (!c) return 0;
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](const void* p, size_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  };
  cudaStream_t st = c->ctx->stream;
  for (const auto& CL : c->levels) {
    mix(CL->src.data(), CL->src.size() * 8);
    mix(CL->rec.data(), CL->rec.size() * 8);
    std::vector<char> buf(CL->chain_bytes());
    if (cudaMemcpyAsync(buf.data(), CL->chain_ptr(), buf.size(), cudaMemcpyDefault, st) != cudaSuccess) return 0;
    cudaStreamSynchronize(st);
    // hash only the live parts of every record
    for (int t : CL->rec_cluster) {
      const int b = CL->bsz[t], kf = CL->kfin[t], e = b - kf;
      mix(buf.data() + CL->Qt_off[t] * 16, (size_t)b * b * 16);
      mix(buf.data() + CL->L11_off[t] * 16, (size_t)e * e * 16);
      mix(buf.data() + CL->U11_off[t] * 16, (size_t)e * e * 16);
      if (!e) continue;
      for (int a = CL->R_ptr[t]; a < CL->R_ptr[t + 1]; ++a) mix(buf.data() + CL->Lbar_off[a] * 16, (size_t)CL->bsz[CL->R_nb[a]] * e * 16);
      for (int a = CL->C_ptr[t]; a < CL->C_ptr[t + 1]; ++a) mix(buf.data() + CL->Ubar_off[a] * 16, (size_t)CL->bsz[CL->C_nb[a]] * e * 16);
      mix(buf.data() + CL->Lself_off[t] * 16, (size_t)kf * e * 16);
      mix(buf.data() + CL->Uself_off[t] * 16, (size_t)kf * e * 16);
    }
  }
  if (c->root_size) {
    std::vector<char> buf((size_t)c->root_size * c->root_size * 16);
    cudaMemcpyAsync(buf.data(), c->root.p, buf.size(), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    mix(buf.data(), buf.size());
  }
  return h;
}

int h2g_chain_timing(const h2g_chain* c, double* fms, double* sms, int64_t* fl, int64_t* sl) {
  if (!c) return H2G_ERR_INVALID_INPUT;
  if (fms) *fms = c->factor_ms;
  if (sms) *sms = c->solve_ms;
  if (fl) *fl = c->factor_launches;
  if (sl) *sl = c->solve_launches;
  return H2G_OK;
}

int h2g_chain_plan(const h2g_chain* c, double* plan_ms, int32_t* built) {
  if (!c) return H2G_ERR_INVALID_INPUT;
  if (plan_ms) *plan_ms = c->plan_ms;
  if (built) *built = c->plan_built ? 1 : 0;
  return H2G_OK;
}

int h2g_context_clear_plans(h2g_context* ctx) {
  if (!ctx) return H2G_ERR_INVALID_INPUT;
  std::lock_guard<std::mutex> g(ctx->plan_mu);
  ctx->plan_lru.clear();
  return H2G_OK;
}

int h2g_set_profiling(h2g_context* ctx, int32_t on) {
  if (!ctx) return H2G_ERR_INVALID_INPUT;
  ctx->prof.on = on != 0;
  return H2G_OK;
}

int h2g_chain_kernel_stats(const h2g_chain* c, int32_t cls, double* out) {
  if (!c || cls < 0 || cls >= PC_N || !out) return H2G_ERR_INVALID_INPUT;
  out[0] = c->kms[cls];
  out[1] = (double)c->klaunch[cls];
  out[2] = c->kflops[cls];
  out[3] = c->kbytes[cls];
  return H2G_OK;
}

int h2g_chain_schur_levels(const h2g_chain* c, int32_t* nlevels, double* out) {
  if (!c || !nlevels) return H2G_ERR_INVALID_INPUT;
  *nlevels = static_cast<int32_t>(c->schur_levels.size());
  if (out) {
    size_t q = 0;
    for (const auto& kv : c->schur_levels) {
      out[q++] = kv.first;
      for (double v : kv.second) out[q++] = v;
    }
  }
  return H2G_OK;
}

int h2g_chain_work(const h2g_chain* c, double* out) {
  if (!c || !out) return H2G_ERR_INVALID_INPUT;
  out[0] = c->factor_flops;
  out[1] = c->schur_flops;
  out[2] = c->solve_bytes;
  out[3] = c->schur_bytes;
  return H2G_OK;
}

int h2g_chain_schur_executed(const h2g_chain* c, double* out) {
  if (!c || !out) return H2G_ERR_INVALID_INPUT;
  out[0] = c->schur_flops_exec;
  out[1] = c->schur_bytes_exec;
  return H2G_OK;
}

}  // extern "C"

// =================================================== H2LU v1 container
namespace {

template <class F>
void io_guard(F&& f) {
  try {
    f();
  } catch (const Error&) {
    throw;
  } catch (const std::runtime_error& e) {  // serialize: malformed file (SerializationError)
    throw Error(H2G_ERR_INVALID_INPUT, e.what());
  }
}

io::TreeData tree_of(const h2g_matrix* m) {
  if (m->points_tree.empty() || m->leafsize < 1)
    throw Error(H2G_ERR_INVALID_INPUT, "save: the matrix does not know its points / leaf size (build it with h2g_matrix_build, or pass points_tree, "
                                       "perm and leafsize in the upload desc)");
  io::TreeData t;
  t.n = m->S.n;
  t.depth = m->S.depth;
  t.leafsize = m->leafsize;
  if (m->perm.empty()) {
    t.perm.resize(t.n);
    for (int64_t i = 0; i < t.n; ++i) t.perm[i] = i;
  } else {
    t.perm = m->perm;
  }
  t.points = m->points_tree;
  t.begin = m->S.begin;
  t.end = m->S.end;
  return t;
}

io::HMat hmat(int64_t r, int64_t c, const cplx* src_host) {
  io::HMat M;
  M.rows = r, M.cols = c;
  M.data.resize((size_t)(r * c));
  if (r * c) std::memcpy(M.data.data(), src_host, (size_t)(r * c) * 16);
  return M;
}

// Inverse of a unit-lower (lower = true) or upper e x e matrix, column-major.
std::vector<std::complex<double>> tri_inverse(const std::vector<std::complex<double>>& A, int e, bool lower) {
  std::vector<std::complex<double>> X((size_t)e * e, 0.0);
  for (int j = 0; j < e; ++j) {
    // solve A x = e_j
    std::vector<std::complex<double>> x(e, 0.0);
    x[j] = 1.0;
    if (lower) {
      for (int p = 0; p < e; ++p)
        for (int i = p + 1; i < e; ++i) x[i] -= A[i + (size_t)p * e] * x[p];
    } else {
      for (int p = e - 1; p >= 0; --p) {
        x[p] /= A[p + (size_t)p * e];
        for (int i = 0; i < p; ++i) x[i] -= A[i + (size_t)p * e] * x[p];
      }
    }
    for (int i = 0; i < e; ++i) X[i + (size_t)j * e] = x[i];
  }
  return X;
}

}  // namespace

extern "C" {

int h2g_matrix_save(const h2g_matrix* m, const char* path, h2g_error* err) {
  return guarded(err, [&] {
    if (!m || !path) throw Error(H2G_ERR_INVALID_INPUT, "null argument");
    CK(cudaSetDevice(m->ctx->device));
    io_guard([&] {
      const Structure& S = m->S;
      io::MatrixFile F;
      F.tree = tree_of(m);
      F.eta = S.eta;
      F.eps_h2 = m->eps_h2;
      F.shadow_guard = m->shadow_guard;
      cudaStream_t st = m->ctx->stream;
      std::vector<std::complex<double>> basis(m->basis_elems), coup(m->coup_elems), dense(m->dense_elems);
      if (m->basis_elems) CK(cudaMemcpyAsync(basis.data(), m->basis.p, m->basis_elems * 16, cudaMemcpyDeviceToHost, st));
      if (m->coup_elems) CK(cudaMemcpyAsync(coup.data(), m->coup.p, m->coup_elems * 16, cudaMemcpyDeviceToHost, st));
      if (m->dense_elems) CK(cudaMemcpyAsync(dense.data(), m->dense_ptr(), m->dense_elems * 16, cudaMemcpyDefault, st));
      CK(cudaStreamSynchronize(st));
      const int nc = S.num_clusters();
      F.bases.resize(nc);
      for (int id = 0; id < nc; ++id)
        F.bases[id] = hmat(m->basis_rows[id], m->basis_rank[id], reinterpret_cast<const cplx*>(basis.data() + m->basis_off[id]));
      F.couplings.resize(S.depth + 1);
      for (int l = 0; l <= S.depth; ++l)
        for (size_t q = 0; q < S.adm[l].size(); ++q) {
          const int64_t g = S.adm_offset[l] + (int64_t)q;
          F.couplings[l].push_back(hmat(m->basis_rank[S.adm[l][q].row], m->basis_rank[S.adm[l][q].col],
                                        reinterpret_cast<const cplx*>(coup.data() + m->coup_off[g])));
        }
      for (size_t q = 0; q < S.leaf.size(); ++q) {
        const auto& pr = S.leaf[q];
        F.dense.push_back(hmat(S.end[pr.row] - S.begin[pr.row], S.end[pr.col] - S.begin[pr.col], reinterpret_cast<const cplx*>(dense.data() + m->dense_off[q])));
      }
      io::save_matrix(path, F);
    });
  });
}

int h2g_matrix_load(h2g_context* ctx, const char* path, h2g_matrix** out, h2g_error* err) {
  return guarded(err, [&] {
    if (!ctx || !path || !out) throw Error(H2G_ERR_INVALID_INPUT, "null argument");
    io_guard([&] {
      io::MatrixReader R(path);
      io::MatrixFile& H = R.head();
      Structure S = structure_from_tree(H.tree.points.data(), H.tree.n, H.tree.depth, H.tree.begin, H.tree.end, H.eta);
      std::vector<int64_t> adm_count(S.depth + 1);
      for (int l = 0; l <= S.depth; ++l) adm_count[l] = (int64_t)S.adm[l].size();
      R.read_rest(adm_count, (int64_t)S.leaf.size());
      io::MatrixFile F = R.take();
      const int nc = S.num_clusters();
      // flatten into an upload descriptor
      std::vector<int64_t> brows(nc), brank(nc), boff(nc), coff, doff, aoff(S.depth + 2, 0), soff(S.depth + 2, 0);
      std::vector<int32_t> apairs, spairs, lpairs;
      std::vector<std::complex<double>> bdata, cdata, ddata;
      for (int id = 0; id < nc; ++id) {
        brows[id] = F.bases[id].rows;
        brank[id] = F.bases[id].cols;
        boff[id] = (int64_t)bdata.size();
        bdata.insert(bdata.end(), F.bases[id].data.begin(), F.bases[id].data.end());
      }
      for (int l = 0; l <= S.depth; ++l) {
        aoff[l + 1] = aoff[l] + (int64_t)S.adm[l].size();
        soff[l + 1] = soff[l] + (int64_t)S.split[l].size();
        for (size_t q = 0; q < S.adm[l].size(); ++q) {
          const auto& pr = S.adm[l][q];
          const io::HMat& C = F.couplings[l][q];
          if (C.rows != brank[pr.row] || C.cols != brank[pr.col]) throw std::runtime_error("serialize: coupling dims inconsistent with basis ranks");
          apairs.push_back(pr.row), apairs.push_back(pr.col);
          coff.push_back((int64_t)cdata.size());
          cdata.insert(cdata.end(), C.data.begin(), C.data.end());
        }
        for (const auto& pr : S.split[l]) spairs.push_back(pr.row), spairs.push_back(pr.col);
      }
      for (size_t q = 0; q < S.leaf.size(); ++q) {
        const auto& pr = S.leaf[q];
        const io::HMat& D = F.dense[q];
        if (D.rows != S.end[pr.row] - S.begin[pr.row] || D.cols != S.end[pr.col] - S.begin[pr.col])
          throw std::runtime_error("serialize: dense block dims inconsistent with tree");
        lpairs.push_back(pr.row), lpairs.push_back(pr.col);
        doff.push_back((int64_t)ddata.size());
        ddata.insert(ddata.end(), D.data.begin(), D.data.end());
      }
      h2g_matrix_desc d{};
      d.n = S.n;
      d.depth = S.depth;
      d.eta = S.eta;
      d.eps_h2 = F.eps_h2;
      d.cluster_begin = S.begin.data();
      d.cluster_end = S.end.data();
      d.adm_offsets = aoff.data();
      d.adm_pairs = apairs.data();
      d.split_offsets = soff.data();
      d.split_pairs = spairs.data();
      d.num_leaf_pairs = (int64_t)S.leaf.size();
      d.leaf_pairs = lpairs.data();
      d.basis_rows = brows.data();
      d.basis_rank = brank.data();
      d.basis_offset = boff.data();
      d.basis_data = reinterpret_cast<const double*>(bdata.data());
      d.coupling_offset = coff.data();
      d.coupling_data = reinterpret_cast<const double*>(cdata.data());
      d.dense_offset = doff.data();
      d.dense_data = reinterpret_cast<const double*>(ddata.data());
      d.points_tree = F.tree.points.data();
      d.perm = F.tree.perm.data();
      d.leafsize = F.tree.leafsize;
      h2g_error e2{};
      const int rc = h2g_matrix_upload(ctx, &d, out, &e2);
      if (rc) throw Error(rc, e2.msg);
      (*out)->shadow_guard = F.shadow_guard;
    });
  });
}

int h2g_chain_save(const h2g_chain* c, const h2g_matrix* source, const char* path, h2g_error* err) {
  return guarded(err, [&] {
    if (!c || !source || !path) throw Error(H2G_ERR_INVALID_INPUT, "null argument");
    if (source->S.n != c->n) throw Error(H2G_ERR_INVALID_INPUT, "save_chain: the chain and the matrix differ in size");
    CK(cudaSetDevice(c->ctx->device));
    io_guard([&] {
      io::ChainFile F;
      F.tree = tree_of(source);
      F.n = c->n;
      F.stop_level = c->stop_level;
      F.eps_fill_in = c->eps;
      cudaStream_t st = c->ctx->stream;
      for (const auto& CLp : c->levels) {
        const ChainLevelHost& CL = *CLp;
        std::vector<cplx> arena(CL.chain_bytes() / 16);
        if (!arena.empty()) CK(cudaMemcpyAsync(arena.data(), CL.chain_ptr(), arena.size() * 16, cudaMemcpyDefault, st));
        CK(cudaStreamSynchronize(st));
        io::LevelFile LF;
        LF.level = CL.level;
        const size_t nrec = CL.rec_cluster.size();
        for (size_t ri = 0; ri < nrec; ++ri) {
          const int64_t* r = CL.rec.data() + 10 * ri;
          const int t = CL.rec_cluster[ri];
          const int b = CL.bsz[t], kf = CL.kfin[t], e = b - kf;
          io::RecordData R;
          R.cluster = (int32_t)r[0];
          R.level = (int32_t)r[1];
          R.pos = r[2], R.bsize = r[3], R.eliminated = r[4], R.rank_before = r[5], R.rank_after = r[6], R.fill_targets = r[7];
          R.Qtilde = hmat(b, b, arena.data() + CL.Qt_off[t]);
          R.L11 = hmat(e, e, arena.data() + CL.L11_off[t]);
          R.U11 = hmat(e, e, arena.data() + CL.U11_off[t]);
          if (e > 0) {
            for (int a = CL.R_ptr[t]; a < CL.R_ptr[t + 1]; ++a)
              R.Lbar.push_back({CL.pos[CL.R_nb[a]], hmat(CL.bsz[CL.R_nb[a]], e, arena.data() + CL.Lbar_off[a])});
            if (kf > 0) R.Lbar.push_back({CL.pos[t] + e, hmat(kf, e, arena.data() + CL.Lself_off[t])});
            for (int a = CL.C_ptr[t]; a < CL.C_ptr[t + 1]; ++a)
              R.Ubar.push_back({CL.pos[CL.C_nb[a]], hmat(e, CL.bsz[CL.C_nb[a]], arena.data() + CL.Ubar_off[a])});
            if (kf > 0) R.Ubar.push_back({CL.pos[t] + e, hmat(e, kf, arena.data() + CL.Uself_off[t])});
          }
          LF.recs.push_back(std::move(R));
        }
        LF.perm_level = CL.level;
        LF.src = CL.src;
        LF.active_after = CL.diag[8];
        LF.diag_level = CL.level;
        LF.rank_sum_before = CL.diag[2], LF.rank_sum_after = CL.diag[3], LF.eliminated = CL.diag[4], LF.ledger_blocks = CL.diag[5];
        LF.chain_bytes = (uint64_t)CL.diag[6];
        F.levels.push_back(std::move(LF));
      }
      const int64_t r = c->root_size;
      F.root_size = r;
      F.root_l.rows = F.root_l.cols = F.root_u.rows = F.root_u.cols = r;
      if (r > 0) {
        std::vector<std::complex<double>> A((size_t)r * r);
        CK(cudaMemcpyAsync(A.data(), c->root.p, (size_t)r * r * 16, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        F.root_l.data.assign((size_t)r * r, 0.0);
        F.root_u.data.assign((size_t)r * r, 0.0);
        for (int64_t j = 0; j < r; ++j)
          for (int64_t i = 0; i < r; ++i) {
            const auto v = A[i + j * r];
            if (i > j) F.root_l.data[i + j * r] = v;
            else F.root_u.data[i + j * r] = v;
            if (i == j) F.root_l.data[i + j * r] = 1.0;
          }
      }
      io::save_chain(path, F);
    });
  });
}

int h2g_chain_load(h2g_context* ctx, const char* path, h2g_chain** out, h2g_error* err) {
  return guarded(err, [&] {
    if (!ctx || !path || !out) throw Error(H2G_ERR_INVALID_INPUT, "null argument");
    std::lock_guard<std::recursive_mutex> run_lock(ctx->run_mu);
    CK(cudaSetDevice(ctx->device));
    io_guard([&] {
      io::ChainFile F = io::load_chain(path);
      cudaStream_t st = ctx->stream;
      auto C = std::make_unique<h2g_chain>();
      C->ctx = ctx;
      C->n = F.n;
      C->stop_level = F.stop_level;
      C->schedule = H2G_SCHEDULE_REFERENCE;
      C->depth = F.tree.depth;
      C->eps = F.eps_fill_in;
      C->tree_perm = F.tree.perm;
      for (const io::LevelFile& LF : F.levels) {
        const int l = LF.level;
        if (l < 0 || l > F.tree.depth) throw std::runtime_error("serialize: level out of range");
        const int nl = 1 << l, first = Structure::first(l);
        auto CL = std::make_unique<ChainLevelHost>();
        CL->level = l;
        CL->bsz.assign(nl, 0);
        CL->kfin.assign(nl, 0);
        CL->korig.assign(nl, 0);
        CL->pos.assign(nl, 0);
        std::vector<int> rec_of(nl, -1);
        for (size_t ri = 0; ri < LF.recs.size(); ++ri) {
          const io::RecordData& R = LF.recs[ri];
          const int t = R.cluster - first;
          if (R.level != l || t < 0 || t >= nl || rec_of[t] >= 0) throw std::runtime_error("serialize: record cluster does not belong to its level");
          rec_of[t] = (int)ri;
          CL->bsz[t] = (int)R.bsize;
          CL->kfin[t] = (int)(R.bsize - R.eliminated);
          CL->korig[t] = (int)R.rank_before;
          CL->pos[t] = R.pos;
        }
        for (int t = 0; t < nl; ++t)
          if (rec_of[t] < 0) throw std::runtime_error("serialize: level block misses a cluster record");
        // segment start -> cluster (neighbour identification of the off-diagonal blocks)
        std::unordered_map<long long, int> seg_at;
        for (int t = 0; t < nl; ++t)
          if (CL->bsz[t] > 0) seg_at[CL->pos[t]] = t;
        auto seg_of = [&](int64_t pos) {
          auto it = seg_at.find(pos);
          if (it == seg_at.end()) throw std::runtime_error("serialize: off-diagonal block does not start a cluster segment");
          return it->second;
        };
        // neighbour lists (record order of the file = ascending cluster within
        // a block list, self last) and chain offsets
        CL->R_ptr.assign(1, 0);
        CL->C_ptr.assign(1, 0);
        std::vector<std::vector<int>> nbg(nl);
        for (int t = 0; t < nl; ++t) {
          const io::RecordData& R = LF.recs[rec_of[t]];
          const int b = CL->bsz[t], e = b - CL->kfin[t];
          for (const auto& blk : R.Lbar) {
            if (blk.pos >= R.pos && blk.pos < R.pos + b) continue;  // self block
            const int j = seg_of(blk.pos);
            if (blk.M.rows != CL->bsz[j] || blk.M.cols != e) throw std::runtime_error("serialize: Lbar block dims inconsistent");
            CL->R_nb.push_back(j);
            nbg[t].push_back(j), nbg[j].push_back(t);
          }
          CL->R_ptr.push_back((int)CL->R_nb.size());
          for (const auto& blk : R.Ubar) {
            if (blk.pos >= R.pos && blk.pos < R.pos + b) continue;
            const int c2 = seg_of(blk.pos);
            if (blk.M.cols != CL->bsz[c2] || blk.M.rows != e) throw std::runtime_error("serialize: Ubar block dims inconsistent");
            CL->C_nb.push_back(c2);
            nbg[t].push_back(c2), nbg[c2].push_back(t);
          }
          CL->C_ptr.push_back((int)CL->C_nb.size());
        }
        int bm = 1;
        for (int t = 0; t < nl; ++t) bm = std::max(bm, CL->bsz[t]);
        std::vector<long long> Qt(nl), L11(nl), U11(nl), Li(nl), Ui(nl), Ls(nl), Us(nl), Lb(CL->R_nb.size()), Ub(CL->C_nb.size());
        long long top = 0;
        for (int t = 0; t < nl; ++t) {
          const long long b = CL->bsz[t], kf = CL->kfin[t], e = b - kf;
          Qt[t] = top, top += b * b;
          L11[t] = top, top += e * e;
          U11[t] = top, top += e * e;
          Li[t] = top, top += e * e;
          Ui[t] = top, top += e * e;
          Ls[t] = top, top += kf * e;
          Us[t] = top, top += kf * e;
          for (int a = CL->R_ptr[t]; a < CL->R_ptr[t + 1]; ++a) Lb[a] = top, top += (long long)CL->bsz[CL->R_nb[a]] * e;
          for (int a = CL->C_ptr[t]; a < CL->C_ptr[t + 1]; ++a) Ub[a] = top, top += (long long)CL->bsz[CL->C_nb[a]] * e;
        }
        std::vector<std::complex<double>> arena((size_t)std::max<long long>(top, 1), 0.0);
        auto put = [&](long long off, const io::HMat& M) { std::copy(M.data.begin(), M.data.end(), arena.begin() + off); };
        for (int t = 0; t < nl; ++t) {
          const io::RecordData& R = LF.recs[rec_of[t]];
          const int b = CL->bsz[t], kf = CL->kfin[t], e = b - kf;
          put(Qt[t], R.Qtilde);
          if (e == 0) continue;
          put(L11[t], R.L11);
          put(U11[t], R.U11);
          const auto li = tri_inverse(R.L11.data, e, true), ui = tri_inverse(R.U11.data, e, false);
          std::copy(li.begin(), li.end(), arena.begin() + Li[t]);
          std::copy(ui.begin(), ui.end(), arena.begin() + Ui[t]);
          int ar = CL->R_ptr[t], ac = CL->C_ptr[t];
          for (const auto& blk : R.Lbar) {
            if (blk.pos >= R.pos && blk.pos < R.pos + b) {
              if (blk.M.rows != kf || blk.M.cols != e) throw std::runtime_error("serialize: self Lbar block dims inconsistent");
              put(Ls[t], blk.M);
            } else {
              put(Lb[ar++], blk.M);
            }
          }
          for (const auto& blk : R.Ubar) {
            if (blk.pos >= R.pos && blk.pos < R.pos + b) {
              if (blk.M.cols != kf || blk.M.rows != e) throw std::runtime_error("serialize: self Ubar block dims inconsistent");
              put(Us[t], blk.M);
            } else {
              put(Ub[ac++], blk.M);
            }
          }
        }
        // solve schedule: dependency wavefronts of the file's record order
        // over the neighbour graph (as build_schedule's reference mode)
        std::vector<int> key(nl, 0), order;
        for (const auto& R : LF.recs) order.push_back(R.cluster - first);
        std::vector<int> rank_in(nl);
        for (int q = 0; q < nl; ++q) rank_in[order[q]] = q;
        int nb_batches = 0;
        for (int t : order) {
          int w = 0;
          for (int x : nbg[t])
            if (rank_in[x] < rank_in[t]) w = std::max(w, key[x] + 1);
          key[t] = w;
          nb_batches = std::max(nb_batches, w + 1);
        }
        std::vector<std::vector<int>> bat(nb_batches);
        for (int t : order) bat[key[t]].push_back(t);
        std::vector<int> batch_ptr(1, 0), batch_cl, batch_maxc, fs_ptr(1, 0);
        std::vector<SolveTargetD> fs;
        std::vector<SolveContribD> fc;
        for (auto& bv : bat) {
          struct T2 {
            long long seg;
            SolveContribD c;
          };
          std::vector<T2> tmp;
          int mc = 0;
          for (int t : bv) {
            batch_cl.push_back(t);
            mc = std::max(mc, CL->C_ptr[t + 1] - CL->C_ptr[t]);
            for (int a = CL->R_ptr[t]; a < CL->R_ptr[t + 1]; ++a) tmp.push_back({CL->R_nb[a], {t, a}});
            tmp.push_back({-1 - (long long)t, {t, -1 - t}});
          }
          batch_ptr.push_back((int)batch_cl.size());
          batch_maxc.push_back(mc);
          std::stable_sort(tmp.begin(), tmp.end(), [](const T2& x, const T2& y) { return x.seg < y.seg; });
          for (size_t i = 0; i < tmp.size();) {
            size_t j = i;
            while (j < tmp.size() && tmp[j].seg == tmp[i].seg) ++j;
            fs.push_back({(int)tmp[i].seg, (int)fc.size(), (int)(fc.size() + (j - i))});
            for (size_t k = i; k < j; ++k) fc.push_back(tmp[k].c);
            i = j;
          }
          fs_ptr.push_back((int)fs.size());
        }
        // device data
        CL->arena.alloc((size_t)std::max<long long>(top, 1) * 16, st);
        CK(cudaMemcpyAsync(CL->arena.p, arena.data(), (size_t)std::max<long long>(top, 1) * 16, cudaMemcpyHostToDevice, st));
        Packer pk;
        size_t o_bsz = pk.add(CL->bsz), o_pos = pk.add(CL->pos), o_kfin = pk.add(CL->kfin), o_Cp = pk.add(CL->C_ptr), o_Cn = pk.add(CL->C_nb);
        size_t o_Qt = pk.add(Qt), o_L11 = pk.add(L11), o_U11 = pk.add(U11), o_Li = pk.add(Li), o_Ui = pk.add(Ui), o_Lb = pk.add(Lb), o_Ub = pk.add(Ub),
               o_Ls = pk.add(Ls), o_Us = pk.add(Us), o_bat = pk.add(batch_cl);
        size_t o_fs = pk.add_raw(fs.data(), fs.size()), o_fc = pk.add_raw(fc.data(), fc.size());
        pk.upload(CL->meta, st);
        const DBuf& mt = CL->meta;
        SolveLevel& SL = CL->sl;
        SL.nl = nl;
        SL.bmax = bm;
        SL.bsz = at<int>(mt, o_bsz);
        SL.pos = at<long long>(mt, o_pos);
        SL.kfin = at<int>(mt, o_kfin);
        SL.C_ptr = at<int>(mt, o_Cp);
        SL.C_nb = at<int>(mt, o_Cn);
        SL.chain = CL->arena.as<cplx>();
        SL.Qt_off = at<long long>(mt, o_Qt);
        SL.L11_off = at<long long>(mt, o_L11);
        SL.U11_off = at<long long>(mt, o_U11);
        SL.Linv_off = at<long long>(mt, o_Li);
        SL.Uinv_off = at<long long>(mt, o_Ui);
        SL.Lbar_off = at<long long>(mt, o_Lb);
        SL.Ubar_off = at<long long>(mt, o_Ub);
        SL.Lself_off = at<long long>(mt, o_Ls);
        SL.Uself_off = at<long long>(mt, o_Us);
        CL->batch_ptr = batch_ptr;
        CL->batch_maxc = batch_maxc;
        CL->d_batch = at<int>(mt, o_bat);
        CL->fs_ptr = fs_ptr;
        CL->d_fs = at<SolveTargetD>(mt, o_fs);
        CL->d_fc = at<SolveContribD>(mt, o_fc);
        {
          std::vector<int> sv(batch_ptr);
          sv.insert(sv.end(), batch_maxc.begin(), batch_maxc.end());
          sv.insert(sv.end(), fs_ptr.begin(), fs_ptr.end());
          upload(CL->sched_buf, sv, st);
          const int nb1 = (int)batch_ptr.size();
          const int* base = CL->sched_buf.as<int>();
          CL->sched = {nb1 - 1, base, CL->d_batch, base + nb1, base + nb1 + (nb1 - 1), CL->d_fs, CL->d_fc};
          for (int bi = 0; bi + 1 < nb1; ++bi)
            CL->part_need = std::max(CL->part_need, (size_t)(batch_ptr[bi + 1] - batch_ptr[bi]) * (batch_maxc[bi] + 1) * bm);
        }
        build_flow(*CL, nl, batch_ptr, batch_cl, fs_ptr, fs, fc, st);
        // host inspection copies
        CL->Qt_off = Qt, CL->L11_off = L11, CL->U11_off = U11, CL->Lbar_off = Lb, CL->Ubar_off = Ub, CL->Lself_off = Ls, CL->Uself_off = Us;
        for (size_t ri = 0; ri < LF.recs.size(); ++ri) {
          const io::RecordData& R = LF.recs[ri];
          const int t = R.cluster - first;
          const int e = (int)R.eliminated;
          const int nlb = e > 0 ? (CL->R_ptr[t + 1] - CL->R_ptr[t]) + (CL->kfin[t] > 0) : 0;
          const int nub = e > 0 ? (CL->C_ptr[t + 1] - CL->C_ptr[t]) + (CL->kfin[t] > 0) : 0;
          const int64_t rr[10] = {R.cluster, R.level, R.pos, R.bsize, R.eliminated, R.rank_before, R.rank_after, R.fill_targets, nlb, nub};
          CL->rec.insert(CL->rec.end(), rr, rr + 10);
          CL->rec_cluster.push_back(t);
        }
        CL->diag = {l, (int64_t)LF.recs.size(), LF.rank_sum_before, LF.rank_sum_after, LF.eliminated, LF.ledger_blocks, (int64_t)LF.chain_bytes,
                    (int64_t)LF.src.size(), LF.active_after};
        CL->src = LF.src;
        upload(CL->d_src, CL->src, st);
        C->storage_bytes = (size_t)LF.chain_bytes;
        C->levels.push_back(std::move(CL));
      }
      C->root_size = F.root_size;
      if (F.root_size > 0) {
        const int64_t r = F.root_size;
        std::vector<std::complex<double>> A((size_t)r * r);
        for (int64_t j = 0; j < r; ++j)
          for (int64_t i = 0; i < r; ++i) A[i + j * r] = i > j ? F.root_l.data[i + j * r] : F.root_u.data[i + j * r];
        C->root.alloc((size_t)r * r * 16, st);
        CK(cudaMemcpyAsync(C->root.p, A.data(), (size_t)r * r * 16, cudaMemcpyHostToDevice, st));
      }
      CK(cudaStreamSynchronize(st));
      ++ctx->refs;  // the chain holds the context
      *out = C.release();
    });
  });
}

int h2g_chain_perm_tree(const h2g_chain* c, int64_t* perm) {
  if (!c || !perm) return H2G_ERR_INVALID_INPUT;
  for (int64_t i = 0; i < c->n; ++i) perm[i] = c->tree_perm.empty() ? i : c->tree_perm[i];
  return H2G_OK;
}

int h2g_vector_save(const char* path, const double* data, int64_t n, h2g_error* err) {
  return guarded(err, [&] {
    if (!path || (n > 0 && !data) || n < 0) throw Error(H2G_ERR_INVALID_INPUT, "vector_save: bad arguments");
    io_guard([&] {
      std::vector<std::complex<double>> v((size_t)n);
      if (n) std::memcpy(v.data(), data, (size_t)n * 16);
      io::save_vector(path, v);
    });
  });
}

int h2g_vector_load(const char* path, double* data, int64_t* n, h2g_error* err) {
  return guarded(err, [&] {
    if (!path || !n) throw Error(H2G_ERR_INVALID_INPUT, "vector_load: bad arguments");
    io_guard([&] {
      const auto v = io::load_vector(path);
      if (data) {
        if (*n < (int64_t)v.size()) throw Error(H2G_ERR_INVALID_INPUT, "vector_load: buffer too short");
        std::memcpy(data, v.data(), v.size() * 16);
      }
      *n = (int64_t)v.size();
    });
  });
}

}  // extern "C"

extern "C" {

int h2g_state_info(const h2g_state* st, int64_t* info) {
  if (!st || !info) return H2G_ERR_INVALID_INPUT;
  int64_t active = 0;
  for (size_t t = 0; t < st->cur->bsz.size(); ++t) active = std::max<int64_t>(active, st->cur->pos[t] + st->cur->bsz[t]);
  info[0] = st->level;
  info[1] = active;
  info[2] = st->M->S.n;
  return H2G_OK;
}

int h2g_state_cluster(const h2g_state* st, int32_t cluster, int64_t* out) {
  return guarded(nullptr, [&] {
    if (!st || !out) throw Error(H2G_ERR_INVALID_INPUT, "null argument");
    const int t = cluster - st->Y->first;
    if (t < 0 || t >= st->Y->nl) throw Error(H2G_ERR_INVALID_INPUT, "state_cluster: cluster not on the current level");
    int kf = st->cur->korig[t];
    if (st->d_kfin) CK(cudaMemcpy(&kf, st->d_kfin + t, 4, cudaMemcpyDeviceToHost));
    out[0] = st->cur->pos[t];
    out[1] = st->cur->bsz[t];
    out[2] = kf;
    out[3] = (*st->rotated)[t];
    out[4] = (*st->elim)[t];
  });
}

int h2g_state_qtilde(const h2g_state* st, int32_t cluster, double* out) {
  return guarded(nullptr, [&] {
    if (!st || !out || !st->chain || !st->Qt_off) throw Error(H2G_ERR_INVALID_INPUT, "state_qtilde: no projection on this state");
    const int t = cluster - st->Y->first;
    if (t < 0 || t >= st->Y->nl) throw Error(H2G_ERR_INVALID_INPUT, "state_qtilde: cluster not on the current level");
    const int b = st->cur->bsz[t];
    CK(cudaMemcpy(out, st->chain + (*st->Qt_off)[t], (size_t)b * b * 16, cudaMemcpyDeviceToHost));
  });
}

int h2g_state_shadow(const h2g_state* st, double* out) {
  return guarded(nullptr, [&] {
    if (!st || !out) throw Error(H2G_ERR_INVALID_INPUT, "null argument");
    const auto Z = state_shadow(*st);
    std::memcpy(out, Z.data(), Z.size() * 16);
  });
}

int h2g_state_perm(const h2g_state* st, int64_t* src, int64_t* len) {
  if (!st || !len || !st->perm_src) return H2G_ERR_INVALID_INPUT;
  if (src) std::copy(st->perm_src->begin(), st->perm_src->end(), src);
  *len = (int64_t)st->perm_src->size();
  return H2G_OK;
}

}  // extern "C"
