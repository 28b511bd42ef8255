// rk_api.cu -- the C ABI (include/ranky_b200.h): argument checks with the
// reference's messages, exception -> status mapping, host <-> device marshaling.
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <unordered_map>

#include <unistd.h>

#include "rk_pipeline.cuh"

namespace rk {
thread_local uint64_t* g_launch_counter = nullptr;

void trim_pool(cudaStream_t s) {
  cudaStreamSynchronize(s);
  int dev = 0;
  cudaGetDevice(&dev);
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  cudaGetLastError();
}

namespace {
Tuning read_tuning() {
  Tuning t;
  auto flag = [](const char* name, char on) {
    const char* e = std::getenv(name);
    return e && e[0] == on;
  };
  auto num = [](const char* name, double def) {
    const char* e = std::getenv(name);
    return e ? std::strtod(e, nullptr) : def;
  };
  t.trace = flag("RK_TRACE", '1');
  t.hostprof = flag("RK_HOSTPROF", '1');
  t.meminfo_exact = flag("RK_MEMINFO", 'x');
  t.jacobi_gmax = (int)std::max(2.0, std::min(32.0, num("RK_JACOBI_GMAX", 16))) & ~1;
  t.jacobi_single_g = (int)num("RK_JACOBI_SINGLE_G", 8);
  if (const char* e = std::getenv("RK_JACOBI_WARP")) t.jacobi_warp = e[0] == '1' ? 1 : 0;
  if (const char* e = std::getenv("RK_JACOBI_SMEM")) t.jacobi_smem = e[0] == '1' ? 1 : 0;
  t.jacobi_smem_cl = (int)num("RK_JACOBI_SMEM_CL", 2);
  if (const char* e = std::getenv("RK_JACOBI_WIDE")) t.jacobi_wide = e[0] != '0';
  if (const char* e = std::getenv("RK_JACOBI_CARRY")) t.jacobi_carry = e[0] != '0';
  if (const char* e = std::getenv("RK_PRESENCE")) t.presence_csr = std::string(e) == "csr";
  if (const char* e = std::getenv("RK_SYRK")) t.syrk_block4 = std::string(e) != "tile";
  t.jacobi_check = num("RK_JACOBI_CHECK", -1.0);
  t.jacobi_cluster = (int)num("RK_JACOBI_CLUSTER", 0);
  t.jacobi_debug = std::getenv("RK_JACOBI_DEBUG") != nullptr;
  t.jacobi_q = (int)num("RK_JACOBI_Q", 0);
  t.jacobi_unroll = !flag("RK_JACOBI_UNROLL", '0');
  t.gram_pairs = flag("RK_GRAM_PAIRS", '1');
  t.diag_order = !flag("RK_DIAG_ORDER", '0');
  t.chol_right = flag("RK_CHOL", 'r');
  if (const char* e = std::getenv("RK_BLOCK_ROUTE")) t.householder_only = std::string(e) == "householder";
  t.precond = flag("RK_PRECOND", '1');
  t.precond_stop = (float)num("RK_PRECOND_STOP", 1e-5);
  t.spmm_warp = flag("RK_SPMM_WARP", '1');
  t.wide_reduce = !flag("RK_WIDE_REDUCE", '0');
  t.repair_speculate = !flag("RK_REPAIR_SPECULATE", '0');
  if (const char* e = std::getenv("RK_WIDE_ROWS")) t.wide_rows_pow2 = std::string(e) != "32";
  t.eig_merge = !flag("RK_EIG_MERGE", '0');
  t.spmm_tma = !flag("RK_SPMM_TMA", '0');
  if (const char* e = std::getenv("RK_APPLY_Q")) {
    t.apply_q_regs = std::string(e) == "regs";
    t.apply_q_wy = std::string(e) == "wy";
  }
  t.jacobi_chunk_mb = (uint64_t)num("RK_JACOBI_CHUNK_MB", 0);
  return t;
}
std::mutex g_tuning_mu;
Tuning g_tuning = read_tuning();
std::atomic<int> g_sms[64];
}  // namespace

const Tuning& tuning() { return g_tuning; }
void reload_tuning() {
  std::lock_guard<std::mutex> lk(g_tuning_mu);
  g_tuning = read_tuning();
}
int device_sms(int device) {
  if (device < 0 || device >= 64) fail(RK_INVALID_ARGUMENT, "device index");
  int v = g_sms[device].load(std::memory_order_relaxed);
  if (!v) {
    RK_CUDA_CHECK(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
    g_sms[device].store(v, std::memory_order_relaxed);
  }
  return v;
}

void trace_launch(const char* file, int line) {
  if (!tuning().trace) return;
  const auto t0 = std::chrono::steady_clock::now();
  const cudaError_t e = cudaDeviceSynchronize();
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  std::fprintf(stderr, "[rk trace] %s:%d %.3f ms %s\n", file, line, ms, cudaGetErrorString(e));
}
void* host_alloc_bytes(size_t bytes);

namespace {
struct ProfMark {
  const char* name;
  std::chrono::steady_clock::time_point t;
  cudaEvent_t ev;
};
thread_local std::vector<ProfMark> g_prof;
bool prof_on() { return tuning().hostprof; }
}  // namespace

void prof_mark(cudaStream_t s, const char* name) {
  if (!prof_on()) return;
  ProfMark m{name, std::chrono::steady_clock::now(), nullptr};
  cudaEventCreate(&m.ev);
  cudaEventRecord(m.ev, s);
  g_prof.push_back(m);
}

void prof_flush() {
  if (!prof_on() || g_prof.empty()) return;
  cudaEventSynchronize(g_prof.back().ev);
  std::fprintf(stderr, "[rk prof] %-28s %10s %10s\n", "segment (ends at mark)", "host ms", "device ms");
  for (size_t i = 1; i < g_prof.size(); ++i) {
    float dev = 0;
    cudaEventElapsedTime(&dev, g_prof[i - 1].ev, g_prof[i].ev);
    const double host = std::chrono::duration<double, std::milli>(g_prof[i].t - g_prof[i - 1].t).count();
    std::fprintf(stderr, "[rk prof] %-28s %10.3f %10.3f\n", g_prof[i].name, host, dev);
  }
  for (auto& m : g_prof) cudaEventDestroy(m.ev);
  g_prof.clear();
}

size_t device_free_bytes(Ctx& c, uint64_t want) {
  cudaMemPool_t pool;
  uint64_t used = 0, reserved = 0;
  const bool have_pool = cudaDeviceGetDefaultMemPool(&pool, c.device) == cudaSuccess &&
                         cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess &&
                         cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) == cudaSuccess;
  cudaGetLastError();
  const bool exact = tuning().meminfo_exact;
  if (have_pool && c.free_known && !exact) {
    // free now = free0 - (reserved - reserved0); the pool's reserved-but-unused part is ours too
    const int64_t est = (int64_t)c.free0 + (int64_t)c.reserved0 - (int64_t)used;
    if (est > 0 && (uint64_t)est >= want) return (size_t)est;
  }
  size_t fr = 0, tot = 0;
  RK_CUDA_CHECK(cudaMemGetInfo(&fr, &tot));
  if (have_pool) {
    c.free_known = true;
    c.free0 = fr;
    c.reserved0 = reserved;
    return fr + (reserved - std::min(used, reserved));
  }
  return fr;
}

thread_local PinnedArena* g_arena = nullptr;

CallScope::CallScope(Ctx* c) {
  cudaGetDevice(&prev_device);
  if (prev_device != c->device) RK_CUDA_CHECK(cudaSetDevice(c->device));
  prev_counter = g_launch_counter;
  g_launch_counter = &c->launches;
  PinnedArena& a = c->arena;
  if (!a.base) {
    constexpr size_t kArena = size_t(16) << 20;
    if (cudaMallocHost(reinterpret_cast<void**>(&a.base), kArena) == cudaSuccess) a.cap = kArena;
    else { a.base = nullptr; cudaGetLastError(); }
  }
  if (a.used) {  // the previous call's uploads must have been consumed before the rewind
    cudaStreamSynchronize(c->stream);
    a.used = 0;
  }
  prev_arena = g_arena;
  g_arena = &a;
}
CallScope::~CallScope() {
  g_arena = prev_arena;
  g_launch_counter = prev_counter;
  int cur = -1;
  cudaGetDevice(&cur);
  if (prev_device >= 0 && cur != prev_device) cudaSetDevice(prev_device);
}
}  // namespace rk

using namespace rk;

struct rk_ctx {
  Ctx c;
};
struct rk_dev_matrix {
  rk_ctx* owner;
  DevMatrix m;
};
struct DevOutputsImpl {
  rk_dev_outputs pub;
  DBuf<double> sigma, u, v;
  std::unique_ptr<DevMatrix> repaired;  // the matrix U, sigma, V reconstruct (null: the input)
};
struct rk_dev_shard {
  rk_ctx* owner;
  const rk_dev_matrix* a;
  Partition p;
  rk_method method;
  uint64_t seed;
  std::unique_ptr<DevMatrix> repaired;  // null: the input itself (no edges)
  const DevMatrix* rep() const { return repaired ? repaired.get() : &a->m; }
  // rk_dev_shard_factor_gram keeps the shard's block records for the TSQR
  // fallback (rk_dev_shard_tsqr)
  BlockStageResult blocks;
  std::vector<TreeLeaf> local;  // the shard's leaves, block indices relative to its first block
  bool has_records = false;
  RepairOut repair_out;         // the (whole-matrix) repair report
  uint64_t d_lo = 0;            // the shard's first block
};

namespace {

thread_local std::string g_error;
thread_local double g_residual = 0.0;

template <class F>
rk_status guarded(F&& body) {
  try {
    body();
    return RK_OK;
  } catch (const Error& e) {
    g_error = e.what();
    g_residual = e.residual;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_error = "host allocation failed";
    return RK_NOMEM;
  } catch (const std::exception& e) {
    g_error = e.what();
    return RK_RUNTIME;
  }
}

// Output buffers above 1 MiB are page-locked so device->host copies of V run at
// full PCIe rate. Page-locking is expensive (the OS pins every page), so freed
// pinned buffers go to a small cache keyed by size and are reused by the next
// call of the same shape; the registry lets rk_*_free release either kind.
std::mutex g_pinned_mu;
std::unordered_map<void*, size_t> g_pinned;          // live pinned buffers -> bytes
std::unordered_multimap<size_t, void*> g_pinned_free;  // cached for reuse
size_t g_pinned_cached = 0;
// up to a third of physical memory (at most 64 GiB): c3's full result (16 GiB of V +
// 1 GiB of records) is reused call after call instead of page-locked afresh each time
size_t pinned_cache_max() {
  static const size_t cap = [] {
    const long pages = sysconf(_SC_PHYS_PAGES), page = sysconf(_SC_PAGE_SIZE);
    const size_t phys = pages > 0 && page > 0 ? (size_t)pages * (size_t)page : (size_t(24) << 30);
    return std::min<size_t>(size_t(64) << 30, phys / 3);
  }();
  return cap;
}

template <class T>
T* host_alloc(size_t n) {
  const size_t bytes = (n ? n : 1) * sizeof(T);
  if (bytes >= (1u << 20)) {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    auto it = g_pinned_free.find(bytes);
    if (it != g_pinned_free.end()) {
      void* p = it->second;
      g_pinned_free.erase(it);
      g_pinned_cached -= bytes;
      g_pinned[p] = bytes;
      return static_cast<T*>(p);
    }
    void* p = nullptr;
    if (cudaMallocHost(&p, bytes) == cudaSuccess) {
      g_pinned[p] = bytes;
      return static_cast<T*>(p);
    }
    cudaGetLastError();
  }
  T* p = static_cast<T*>(std::malloc(bytes));
  if (!p) fail(RK_NOMEM, "host allocation failed");
  return p;
}

void host_free(void* p) {
  if (!p) return;
  {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    auto it = g_pinned.find(p);
    if (it != g_pinned.end()) {
      const size_t bytes = it->second;
      g_pinned.erase(it);
      if (g_pinned_cached + bytes <= pinned_cache_max()) {
        g_pinned_free.emplace(bytes, p);
        g_pinned_cached += bytes;
      } else {
        cudaFreeHost(p);
      }
      return;
    }
  }
  std::free(p);
}

template <class T>
T* host_copy(const T* d, size_t n, cudaStream_t s) {
  T* h = host_alloc<T>(n);
  if (n) RK_CUDA_CHECK(cudaMemcpyAsync(h, d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  return h;
}

void check_ctx(rk_ctx* ctx) {
  if (!ctx) fail(RK_INVALID_ARGUMENT, "rk_ctx is NULL");
}
void check_view(const rk_sparse_view* a) {
  if (!a) fail(RK_INVALID_ARGUMENT, "sparse view is NULL");
}

void report_to_host(const RepairOut& r, const Partition& p, rk_repair_report* out, cudaStream_t s) {
  std::memset(out, 0, sizeof *out);
  const uint64_t n = r.edges.n;
  out->n_edges = n;
  std::vector<uint32_t> b, rw, cl;
  std::vector<int32_t> mech;
  to_host(b, r.edges.block.get(), n, s);
  to_host(rw, r.edges.row.get(), n, s);
  to_host(cl, r.edges.col.get(), n, s);
  to_host(mech, r.edges.mech.get(), n, s);
  sync(s);
  out->block = host_alloc<uint64_t>(n);
  out->row = host_alloc<uint64_t>(n);
  out->col = host_alloc<uint64_t>(n);
  out->mechanism = host_alloc<int32_t>(n);
  for (uint64_t i = 0; i < n; ++i) {
    out->block[i] = b[i];
    out->row[i] = rw[i];
    out->col[i] = cl[i];
    out->mechanism[i] = mech[i];
  }
  out->n_blocks = p.blocks;
  out->lonely_counts = host_alloc<uint64_t>(p.blocks);
  for (uint64_t d = 0; d < p.blocks; ++d) out->lonely_counts[d] = r.lonely_counts[d];
  out->fallback_count = r.fallback;
}

// repair + the repaired matrix (null = unchanged input)
std::unique_ptr<DevMatrix> repair_and_apply(Ctx& c, const DevMatrix& a, const Partition& p, rk_method method,
                                            uint64_t seed, RepairOut& rep) {
  repair_device(a, p, method, seed, rep, c.stream);
  prof_mark(c.stream, "repair_device");
  if (rep.edges.n == 0) return nullptr;
  auto out = std::make_unique<DevMatrix>();
  apply_edges(a, rep.edges, *out, c.stream);
  return out;
}

[[noreturn]] void throw_block_failure(const BlockStageResult& b, uint64_t d_lo) {
  for (size_t i = 0; i < b.failures.size(); ++i)
    if (!b.failures[i].empty())
      fail(RK_RUNTIME, "block task " + std::to_string(d_lo + i) + " failed: " + b.failures[i]);
  fail(RK_RUNTIME, "block task failed");
}
bool any_failure(const BlockStageResult& b) {
  for (const auto& f : b.failures)
    if (!f.empty()) return true;
  return false;
}

// retained columns of recover_right_vectors (proxy.cpp:53-59)
std::vector<uint32_t> retained_of(const double* sigma, uint64_t n, double tol) {
  double smax = 0.0;
  for (uint64_t j = 0; j < n; ++j) smax = std::max(smax, sigma[j]);
  std::vector<uint32_t> ret;
  for (uint64_t j = 0; j < n; ++j)
    if (sigma[j] > tol * smax && sigma[j] > 0.0) ret.push_back((uint32_t)j);
  return ret;
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

struct FullRun {
  RepairOut rep;
  std::unique_ptr<DevMatrix> repaired;
  BlockStageResult blocks;
  MergeOut merge;
  DBuf<double> v;
  uint32_t r = 0;  // V columns
  // optional: the records' D2H into this host buffer, issued on c.copy right after
  // the block stage so it overlaps the merge and V (the caller waits on c.copy_ev[1])
  double* records_host = nullptr;
};

// repair -> blocks -> merge -> (V); everything device-resident
void full_run(Ctx& c, const DevMatrix& a, const Partition& p, rk_method method, uint64_t keep, uint64_t seed,
              uint32_t flags, uint64_t top_k, FullRun& fr, rk_timing* t) {
  cudaStream_t s = c.stream;
  const uint64_t launches0 = c.launches;
  cudaEvent_t ev0 = c.ev[3], ev1 = c.ev[4], ev2 = c.ev[5], ev3 = c.ev[6], ev4 = c.ev[7];
  // A full V (N x M doubles, 137 GB at c4: by far the call's largest buffer) is
  // taken from the pool first, while the previous call's block is still whole;
  // allocated after the block stage and the merge it often found the pool
  // fragmented and had to trim and map it again (c4: 0.1-0.4 s). With top_k (c5:
  // N x 64) it stays where it was: allocated early it only shrinks the block
  // stage's staging budget (c5 QR 98 -> 112 s)
  if ((flags & RK_WANT_V) && top_k == 0) {
    const uint64_t M = a.csr.rows;
    const uint64_t rmax = std::max<uint64_t>(1, top_k ? std::min<uint64_t>(top_k, M) : M);
    fr.v.alloc(a.csr.cols * rmax, s);
  }
  RK_NVTX("rk.full_svd");
  RK_CUDA_CHECK(cudaEventRecord(ev0, s));
  prof_mark(s, "start");
  {
    RK_NVTX("rk.repair");
    fr.repaired = repair_and_apply(c, a, p, method, seed, fr.rep);
  }
  prof_mark(s, "repair");
  const DevMatrix& rep = fr.repaired ? *fr.repaired : a;
  RK_CUDA_CHECK(cudaEventRecord(ev1, s));
  {
    RK_NVTX("rk.blocks");
    block_stage(c, rep, p, 0, p.blocks, keep, fr.blocks, nullptr);
  }
  if (any_failure(fr.blocks)) throw_block_failure(fr.blocks, 0);
  RK_CUDA_CHECK(cudaEventRecord(ev2, s));
  prof_mark(s, "blocks (end)");
  if (fr.records_host && fr.blocks.payload.n) {
    RK_CUDA_CHECK(cudaEventRecord(c.copy_ev[0], s));
    RK_CUDA_CHECK(cudaStreamWaitEvent(c.copy, c.copy_ev[0], 0));
    // in 32 MiB pieces: the merge's small result reads (effective columns, the kappa
    // guard, the bisection bounds) share the D2H engine and would otherwise queue
    // behind the whole 1 GiB transfer (c3: the SYRK segment waited 32 ms)
    const uint64_t total = fr.blocks.payload.n * sizeof(double), piece = 32ull << 20;
    for (uint64_t off = 0; off < total; off += piece)
      RK_CUDA_CHECK(cudaMemcpyAsync(reinterpret_cast<char*>(fr.records_host) + off,
                                    reinterpret_cast<const char*>(fr.blocks.payload.get()) + off,
                                    std::min(piece, total - off), cudaMemcpyDeviceToHost, c.copy));
    RK_CUDA_CHECK(cudaEventRecord(c.copy_ev[1], c.copy));
  }
  {
    RK_NVTX("rk.merge");
    merge_records(c, fr.blocks.payload.get(), fr.blocks.offset, fr.blocks.kept, (uint32_t)rep.csr.rows, fr.merge,
                  &fr.blocks.eff);
  }
  RK_CUDA_CHECK(cudaEventRecord(ev3, s));
  prof_mark(s, "merge (end)");
  if (!(flags & RK_WANT_RECORDS)) fr.blocks.payload.release();  // P is not an output: make room for V
  if (flags & RK_WANT_V) {
    RK_NVTX("rk.recover_v");
    const uint32_t k = fr.merge.k;
    const uint32_t kk = (top_k && top_k < k) ? (uint32_t)top_k : k;
    std::vector<double> sig;
    to_host(sig, fr.merge.sigma.get(), kk, s);
    sync(s);
    std::vector<uint32_t> ret = retained_of(sig.data(), kk, 1e-10);
    fr.r = (uint32_t)ret.size();
    if (fr.v.n < rep.csc.cols * (uint64_t)std::max<uint32_t>(fr.r, 1))
      fr.v.alloc(rep.csc.cols * (uint64_t)std::max<uint32_t>(fr.r, 1), s);
    if (fr.r) {
      DBuf<uint32_t> dret(fr.r, s);
      to_device(dret.get(), ret.data(), ret.size(), s);
      recover_v_device(rep.csc, fr.merge.u.get(), k, dret.get(), fr.merge.sigma.get(), fr.r, fr.v.get(), 0,
                       rep.csc.cols, s);
      sync(s);
    }
  }
  RK_CUDA_CHECK(cudaEventRecord(ev4, s));
  prof_mark(s, "V");
  sync(s);
  prof_flush();
  if (t) {
    std::memset(t, 0, sizeof *t);
    t->repair_ms = elapsed(ev0, ev1);
    t->blocks_ms = elapsed(ev1, ev2);
    t->merge_ms = elapsed(ev2, ev3);
    t->recover_ms = elapsed(ev3, ev4);
    t->total_ms = elapsed(ev0, ev4);
    t->qr_ms = fr.blocks.qr_ms;
    t->jacobi_ms = fr.blocks.jacobi_ms;
    t->jacobi_sweeps_max = fr.blocks.sweeps_max;
    t->jacobi_rotations = fr.blocks.rotations;
    t->kernel_launches = c.launches - launches0;
    t->jacobi_sweeps_sum = fr.blocks.sweeps_sum;
    t->qr_flops = fr.blocks.qr_flops;
    t->jacobi_flops = fr.blocks.jacobi_flops;
    t->merge_sweeps = fr.merge.sweeps;
    t->merge_rotations = fr.merge.rotations;
    t->merge_flops = fr.merge.flops;
  }
}

}  // namespace

void* rk::host_alloc_bytes(size_t bytes) { return host_alloc<char>(bytes); }

extern "C" {

const char* rk_last_error(void) { return g_error.c_str(); }
double rk_last_residual(void) { return g_residual; }
uint64_t rk_last_error_line(void) { return (uint64_t)g_residual; }

rk_status rk_load_matrix_market(rk_ctx* ctx, const char* path, rk_sparse* out) {
  return guarded([&] {
    check_ctx(ctx);
    if (!path || !out) fail(RK_INVALID_ARGUMENT, "NULL argument");
    std::memset(out, 0, sizeof *out);
    CallScope sc(&ctx->c);
    try {
      load_matrix_market(path, *out, ctx->c.stream);
    } catch (...) {
      rk_sparse_free(out);
      throw;
    }
  });
}

rk_status rk_save_matrix_market(const rk_sparse_view* a, const char* path) {
  return guarded([&] {
    check_view(a);
    if (!path) fail(RK_INVALID_ARGUMENT, "NULL argument");
    save_matrix_market(*a, path);
  });
}
void rk_reload_tuning(void) { reload_tuning(); }
uint32_t rk_build_flags(void) {
#ifdef RK_EXPERIMENTS
  return 1u;
#else
  return 0u;
#endif
}
int32_t rk_abi_version(void) { return RK_ABI_VERSION; }

rk_status rk_ctx_create(int32_t device, rk_ctx** out) {
  return guarded([&] {
    if (!out) fail(RK_INVALID_ARGUMENT, "out is NULL");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
      cudaGetLastError();
      fail(RK_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    }
    if (device < 0 || device >= n) fail(RK_INVALID_ARGUMENT, "device ordinal out of range");
    auto ctx = std::make_unique<rk_ctx>();
    Ctx& c = ctx->c;
    c.device = device;
    int prev = 0;
    cudaGetDevice(&prev);
    RK_CUDA_CHECK(cudaSetDevice(device));
    cudaDeviceProp prop;
    RK_CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
      fail(RK_CUDA, std::string("libranky_b200 is built for sm_100a; device is ") + prop.name);
    c.num_sms = prop.multiProcessorCount;
    c.smem_optin = prop.sharedMemPerBlockOptin;
    // keep freed blocks in the stream-ordered pool: repeated pipeline calls reuse
    // their buffers instead of paying cudaMalloc/cudaFree every step
    cudaMemPool_t pool;
    RK_CUDA_CHECK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t threshold = UINT64_MAX;
    RK_CUDA_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    RK_CUDA_CHECK(cudaStreamCreateWithFlags(&c.own, cudaStreamNonBlocking));
    c.stream = c.own;
    for (auto& ev : c.ev) RK_CUDA_CHECK(cudaEventCreate(&ev));
    cudaSetDevice(prev);
    *out = ctx.release();
  });
}

rk_status rk_ctx_destroy(rk_ctx* ctx) {
  if (!ctx) return RK_OK;
  cudaSetDevice(ctx->c.device);
  cudaStreamSynchronize(ctx->c.stream);
  for (auto& ev : ctx->c.ev) cudaEventDestroy(ev);
  if (ctx->c.side) {
    cudaStreamSynchronize(ctx->c.side);
    cudaStreamDestroy(ctx->c.side);
    for (auto& ev : ctx->c.side_ev) cudaEventDestroy(ev);
  }
  if (ctx->c.copy) {
    cudaStreamSynchronize(ctx->c.copy);
    cudaStreamDestroy(ctx->c.copy);
    for (auto& ev : ctx->c.copy_ev) cudaEventDestroy(ev);
  }
  if (ctx->c.arena.base) cudaFreeHost(ctx->c.arena.base);
  cudaStreamDestroy(ctx->c.own);
  delete ctx;
  return RK_OK;
}

rk_status rk_ctx_set_stream(rk_ctx* ctx, void* stream) {
  return guarded([&] {
    check_ctx(ctx);
    ctx->c.stream = stream ? static_cast<cudaStream_t>(stream) : ctx->c.own;
  });
}

rk_status rk_ctx_synchronize(rk_ctx* ctx) {
  return guarded([&] {
    check_ctx(ctx);
    CallScope sc(&ctx->c);
    sync(ctx->c.stream);
  });
}

uint64_t rk_ctx_kernel_launches(const rk_ctx* ctx) { return ctx ? ctx->c.launches : 0; }

void rk_host_free(void* p) { host_free(p); }

void rk_svd_free(rk_svd* s) {
  if (!s) return;
  host_free(s->u); host_free(s->sigma); host_free(s->v);
  std::memset(s, 0, sizeof *s);
}
void rk_repair_report_free(rk_repair_report* r) {
  if (!r) return;
  host_free(r->block); host_free(r->row); host_free(r->col); host_free(r->mechanism); host_free(r->lonely_counts);
  std::memset(r, 0, sizeof *r);
}
void rk_sparse_free(rk_sparse* s) {
  if (!s) return;
  host_free(s->entries);
  std::memset(s, 0, sizeof *s);
}
void rk_records_free(rk_records* r) {
  if (!r) return;
  host_free(r->kept); host_free(r->offset); host_free(r->payload);
  std::memset(r, 0, sizeof *r);
}
void rk_pipeline_result_free(rk_pipeline_result* r) {
  if (!r) return;
  rk_svd_free(&r->svd);
  rk_repair_report_free(&r->report);
  rk_sparse_free(&r->repaired);
  rk_records_free(&r->records);
}

rk_status rk_keyed_rng_next(rk_ctx* ctx, uint64_t n, uint64_t seed, const uint64_t* block, const uint64_t* row,
                            uint64_t draws, uint64_t* out) {
  return guarded([&] {
    check_ctx(ctx);
    CallScope sc(&ctx->c);
    cudaStream_t s = ctx->c.stream;
    if (!n || !draws) return;
    DBuf<uint64_t> db(n, s), dr(n, s), dout(n * draws, s);
    to_device(db.get(), block, n, s);
    to_device(dr.get(), row, n, s);
    rng_eval_device(n, seed, db.get(), dr.get(), draws, nullptr, dout.get(), s);
    RK_CUDA_CHECK(cudaMemcpyAsync(out, dout.get(), n * draws * 8, cudaMemcpyDeviceToHost, s));
    sync(s);
  });
}

rk_status rk_keyed_rng_below(rk_ctx* ctx, uint64_t n, uint64_t seed, const uint64_t* block, const uint64_t* row,
                             const uint64_t* bound, uint64_t* out) {
  return guarded([&] {
    check_ctx(ctx);
    CallScope sc(&ctx->c);
    cudaStream_t s = ctx->c.stream;
    if (!n) return;
    for (uint64_t i = 0; i < n; ++i)
      if (bound[i] == 0) fail(RK_INVALID_ARGUMENT, "KeyedRng::below: bound must be nonzero");
    DBuf<uint64_t> db(n, s), dr(n, s), dbd(n, s), dout(n, s);
    to_device(db.get(), block, n, s);
    to_device(dr.get(), row, n, s);
    to_device(dbd.get(), bound, n, s);
    rng_eval_device(n, seed, db.get(), dr.get(), 1, dbd.get(), dout.get(), s);
    RK_CUDA_CHECK(cudaMemcpyAsync(out, dout.get(), n * 8, cudaMemcpyDeviceToHost, s));
    sync(s);
  });
}

rk_status rk_find_lonely_rows(rk_ctx* ctx, const rk_sparse_view* a, uint64_t block_count, uint64_t d, uint64_t* out,
                              uint64_t* n_out) {
  return guarded([&] {
    check_ctx(ctx);
    check_view(a);
    CallScope sc(&ctx->c);
    Partition p = make_partition(a->cols, block_count);
    if (d >= block_count)
      fail(RK_OUT_OF_RANGE, "block index " + std::to_string(d) + " of " + std::to_string(block_count));
    DevMatrix m;
    upload_entries(*a, m, ctx->c.stream);
    std::vector<uint64_t> rows;
    lonely_rows_device(m, p, d, rows, ctx->c.stream);
    for (size_t i = 0; i < rows.size(); ++i) out[i] = rows[i];
    *n_out = rows.size();
  });
}

rk_status rk_repair(rk_ctx* ctx, const rk_sparse_view* a, uint64_t block_count, rk_method method, uint64_t seed,
                    rk_sparse* repaired, rk_repair_report* report) {
  return guarded([&] {
    check_ctx(ctx);
    check_view(a);
    CallScope sc(&ctx->c);
    Ctx& c = ctx->c;
    if ((int)method < 0 || (int)method > 3) fail(RK_INVALID_ARGUMENT, "bad repair method");
    Partition p = make_partition(a->cols, block_count);
    DevMatrix m;
    upload_entries(*a, m, c.stream);
    RepairOut rep;
    std::unique_ptr<DevMatrix> out = repair_and_apply(c, m, p, method, seed, rep);
    if (repaired) csr_to_entries_host(out ? out->csr : m.csr, *repaired, c.stream);
    if (report) report_to_host(rep, p, report, c.stream);
  });
}

rk_status rk_dense_svd(rk_ctx* ctx, uint64_t rows, uint64_t cols, const double* a, rk_svd* out) {
  return guarded([&] {
    check_ctx(ctx);
    if (!out) fail(RK_INVALID_ARGUMENT, "out is NULL");
    CallScope sc(&ctx->c);
    Ctx& c = ctx->c;
    std::memset(out, 0, sizeof *out);
    if (rows > 0xffffffffull || cols > 0xffffffffull) fail(RK_INVALID_ARGUMENT, "dense_svd: matrix too large");
    DBuf<double> da(rows * cols ? rows * cols : 1, c.stream);
    to_device(da.get(), a, rows * cols, c.stream);
    DenseSvdOut r;
    dense_svd_dev(c, da.get(), (uint32_t)rows, (uint32_t)cols, r);
    out->u_rows = rows;
    out->u_cols = r.k;
    out->n_sigma = r.k;
    out->has_v = 1;
    out->v_rows = cols;
    out->v_cols = r.k;
    out->u = host_copy(r.u.get(), rows * r.k, c.stream);
    out->sigma = host_copy(r.sigma.get(), r.k, c.stream);
    out->v = host_copy(r.v.get(), cols * r.k, c.stream);
    sync(c.stream);
  });
}

rk_status rk_block_svd(rk_ctx* ctx, const rk_sparse_view* block, uint64_t keep, rk_svd* out) {
  return guarded([&] {
    check_ctx(ctx);
    check_view(block);
    if (!out) fail(RK_INVALID_ARGUMENT, "out is NULL");
    CallScope sc(&ctx->c);
    Ctx& c = ctx->c;
    std::memset(out, 0, sizeof *out);
    if (keep == 0) fail(RK_INVALID_ARGUMENT, "block_svd: keep must be >= 1");
    const uint64_t M = block->rows, N = block->cols;
    if (M != 0 && (M * N) / M != N) fail(RK_INVALID_ARGUMENT, "dense_of: dimension overflow");
    if (M * N > (uint64_t(1) << 26))
      fail(RK_INVALID_ARGUMENT, "dense_of: " + std::to_string(M) + "x" + std::to_string(N) +
                                    " exceeds the densification cap");
    const uint64_t k_full = std::min(M, N);
    if (k_full == 0) {
      out->u_rows = M;
      out->u = host_alloc<double>(0);
      out->sigma = host_alloc<double>(0);
      return;
    }
    DevMatrix m;
    upload_entries(*block, m, c.stream);
    Partition p = make_partition(N, 1);
    BlockApiOut api;
    const uint64_t k = std::min(keep, k_full);
    api.u.alloc(M * k, c.stream);
    api.sigma.alloc(M, c.stream);
    api.deficient.alloc(M, c.stream);
    api.deficient.zero();
    BlockStageResult br;
    block_stage(c, m, p, 0, 1, keep, br, &api);
    if (!br.failures[0].empty()) {
      const std::string& f = br.failures[0];
      if (f.rfind("one-sided Jacobi", 0) == 0) fail(RK_CONVERGENCE, f, br.conv_residual);
      fail(RK_INVALID_ARGUMENT, f);
    }
    std::vector<uint8_t> def;
    to_host(def, api.deficient.get(), k, c.stream);
    sync(c.stream);
    bool any = false;
    for (uint8_t x : def) any |= x != 0;
    if (any) {
      DBuf<int> fl(1, c.stream);
      fl.zero();
      complete_columns_device(api.u.get(), (uint32_t)M, (uint32_t)k, api.deficient.get(), fl.get(), c.stream);
      int h = 0;
      RK_CUDA_CHECK(cudaMemcpyAsync(&h, fl.get(), sizeof h, cudaMemcpyDeviceToHost, c.stream));
      sync(c.stream);
      if (h) fail(RK_CONVERGENCE, "orthonormal completion has no independent direction (residual 0.000000)", 0.0);
      sign_rows(api.u.get(), (uint32_t)M, (uint32_t)k, nullptr, 0, c.stream);
    }
    out->u_rows = M;
    out->u_cols = k;
    out->n_sigma = k;
    out->u = host_copy(api.u.get(), M * k, c.stream);
    out->sigma = host_copy(api.sigma.get(), k, c.stream);
    sync(c.stream);
  });
}

rk_status rk_proxy_svd(rk_ctx* ctx, uint64_t rows, uint64_t total_cols, const double* proxy, uint64_t n_offsets,
                       const uint64_t* block_offsets, rk_svd* out) {
  if (n_offsets == 0 || !block_offsets || block_offsets[n_offsets - 1] != total_cols) {
    g_error = "proxy_svd: malformed block offsets";
    return RK_INVALID_ARGUMENT;
  }
  return rk_dense_svd(ctx, rows, total_cols, proxy, out);
}

rk_status rk_recover_right_vectors(rk_ctx* ctx, const rk_sparse_view* a, uint64_t u_rows, uint64_t u_cols,
                                   const double* u, uint64_t n_sigma, const double* sigma, double tol,
                                   rk_svd* out) {
  return guarded([&] {
    check_ctx(ctx);
    check_view(a);
    if (!out) fail(RK_INVALID_ARGUMENT, "out is NULL");
    CallScope sc(&ctx->c);
    Ctx& c = ctx->c;
    std::memset(out, 0, sizeof *out);
    if (u_rows != a->rows || u_cols != n_sigma)
      fail(RK_INVALID_ARGUMENT, "recover_right_vectors: factor shapes disagree");
    std::vector<uint32_t> ret = retained_of(sigma, n_sigma, tol);
    const uint32_t r = (uint32_t)ret.size();
    out->has_v = 1;
    out->v_rows = a->cols;
    out->v_cols = r;
    out->u = host_alloc<double>(0);
    out->sigma = host_alloc<double>(0);
    if (r == 0 || a->cols == 0) {
      out->v = host_alloc<double>(a->cols * r);
      return;
    }
    DevMatrix m;
    upload_entries(*a, m, c.stream);
    DBuf<double> du(u_rows * u_cols, c.stream), ds(n_sigma, c.stream), dv(a->cols * r, c.stream);
    DBuf<uint32_t> dret(r, c.stream);
    to_device(du.get(), u, u_rows * u_cols, c.stream);
    to_device(ds.get(), sigma, n_sigma, c.stream);
    to_device(dret.get(), ret.data(), r, c.stream);
    recover_v_device(m.csc, du.get(), (uint32_t)u_cols, dret.get(), ds.get(), r, dv.get(), 0, a->cols, c.stream);
    out->v = host_copy(dv.get(), a->cols * r, c.stream);
    sync(c.stream);
  });
}

rk_status rk_run_block_tasks(rk_ctx* ctx, const rk_sparse_view* a, uint64_t block_count, uint64_t keep,
                             rk_records* out) {
  return guarded([&] {
    check_ctx(ctx);
    check_view(a);
    if (!out) fail(RK_INVALID_ARGUMENT, "out is NULL");
    CallScope sc(&ctx->c);
    Ctx& c = ctx->c;
    std::memset(out, 0, sizeof *out);
    Partition p = make_partition(a->cols, block_count);
    DevMatrix m;
    upload_entries(*a, m, c.stream);
    BlockStageResult br;
    block_stage(c, m, p, 0, p.blocks, keep, br, nullptr);
    if (any_failure(br)) throw_block_failure(br, 0);
    out->n_records = p.blocks;
    out->rows = a->rows;
    out->kept = host_alloc<uint32_t>(p.blocks);
    out->offset = host_alloc<uint64_t>(p.blocks);
    for (uint64_t d = 0; d < p.blocks; ++d) {
      out->kept[d] = br.kept[d];
      out->offset[d] = br.offset[d];
    }
    out->payload = host_copy(br.payload.get(), br.payload.n, c.stream);
    sync(c.stream);
  });
}

rk_status rk_run_pipeline(rk_ctx* ctx, const rk_sparse_view* a, uint64_t block_count, rk_method method, uint64_t keep,
                          uint64_t seed, uint64_t workers, uint32_t flags, uint64_t top_k, rk_pipeline_result* out) {
  return guarded([&] {
    check_ctx(ctx);
    check_view(a);
    if (!out) fail(RK_INVALID_ARGUMENT, "out is NULL");
    CallScope sc(&ctx->c);
    Ctx& c = ctx->c;
    std::memset(out, 0, sizeof *out);
    if (workers == 0) fail(RK_INVALID_ARGUMENT, "workers must be >= 1");
    if ((int)method < 0 || (int)method > 3) fail(RK_INVALID_ARGUMENT, "bad repair method");
    Partition p = make_partition(a->cols, block_count);
    DevMatrix m;
    upload_entries(*a, m, c.stream);
    FullRun fr;
    double* rec_host = nullptr;
    if (flags & RK_WANT_RECORDS) {
      if (!c.copy) {
        RK_CUDA_CHECK(cudaStreamCreateWithFlags(&c.copy, cudaStreamNonBlocking));
        for (auto& ev : c.copy_ev) RK_CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      }
      // the records' size is known before the block stage: D blocks of M x k
      uint64_t tot = 0;
      for (uint64_t d = 0; d < p.blocks; ++d) {
        const uint64_t w = p.end(d) - p.begin(d), kf = std::min<uint64_t>(a->rows, w);
        tot += a->rows * (keep == 0 ? kf : std::min(keep, kf));
      }
      rec_host = host_alloc<double>(tot ? tot : 1);
      fr.records_host = rec_host;
    }
    struct RecGuard {  // the copy stream must be done before the payload is freed or on error
      Ctx& c;
      double*& p;
      ~RecGuard() {
        if (c.copy) cudaStreamSynchronize(c.copy);
        if (p) host_free(p);
      }
    } rec_guard{c, rec_host};
    full_run(c, m, p, method, keep, seed, flags, top_k, fr, &out->timing);
    cudaStream_t s = c.stream;
    const uint64_t M = a->rows;
    const uint32_t k = fr.merge.k;
    out->svd.u_rows = M;
    out->svd.u_cols = k;
    out->svd.n_sigma = k;
    RK_NVTX("rk.results_to_host");
    prof_mark(s, "out: start");
    out->svd.u = host_copy(fr.merge.u.get(), M * k, s);
    out->svd.sigma = host_copy(fr.merge.sigma.get(), k, s);
    if (flags & RK_WANT_V) {
      out->svd.has_v = 1;
      out->svd.v_rows = a->cols;
      out->svd.v_cols = fr.r;
      out->svd.v = host_copy(fr.v.get(), a->cols * (uint64_t)fr.r, s);
      prof_mark(s, "out: V D2H issued");
    }
    report_to_host(fr.rep, p, &out->report, s);
    prof_mark(s, "out: report");
    if (flags & RK_WANT_REPAIRED) csr_to_entries_host(fr.repaired ? fr.repaired->csr : m.csr, out->repaired, s);
    prof_mark(s, "out: repaired");
    if (flags & RK_WANT_RECORDS) {
      out->records.n_records = p.blocks;
      out->records.rows = M;
      out->records.kept = host_alloc<uint32_t>(p.blocks);
      out->records.offset = host_alloc<uint64_t>(p.blocks);
      for (uint64_t d = 0; d < p.blocks; ++d) {
        out->records.kept[d] = fr.blocks.kept[d];
        out->records.offset[d] = fr.blocks.offset[d];
      }
      if (fr.blocks.payload.n && fr.records_host) {
        RK_CUDA_CHECK(cudaStreamWaitEvent(s, c.copy_ev[1], 0));  // issued after the block stage
        out->records.payload = rec_host;
        rec_host = nullptr;  // owned by the result now
      } else {
        out->records.payload = host_copy(fr.blocks.payload.get(), fr.blocks.payload.n, s);
      }
    }
    sync(s);
    prof_mark(s, "out: records + sync");
    prof_flush();
  });
}

rk_status rk_dev_matrix_create(rk_ctx* ctx, const rk_sparse_view* a, rk_dev_matrix** out) {
  return guarded([&] {
    check_ctx(ctx);
    check_view(a);
    CallScope sc(&ctx->c);
    auto m = std::make_unique<rk_dev_matrix>();
    m->owner = ctx;
    upload_entries(*a, m->m, ctx->c.stream);
    sync(ctx->c.stream);
    *out = m.release();
  });
}

rk_status rk_dev_matrix_destroy(rk_dev_matrix* m) {
  if (!m) return RK_OK;
  return guarded([&] {
    CallScope sc(&m->owner->c);
    sync(m->owner->c.stream);
    delete m;
  });
}

uint64_t rk_dev_matrix_nnz(const rk_dev_matrix* m) { return m ? m->m.csr.nnz : 0; }

rk_status rk_dev_full_svd(rk_ctx* ctx, const rk_dev_matrix* a, uint64_t block_count, rk_method method, uint64_t keep,
                          uint64_t seed, uint32_t flags, uint64_t top_k, rk_dev_outputs** out, rk_timing* timing) {
  return guarded([&] {
    check_ctx(ctx);
    if (!a || !out) fail(RK_INVALID_ARGUMENT, "NULL argument");
    CallScope sc(&ctx->c);
    Ctx& c = ctx->c;
    Partition p = make_partition(a->m.csr.cols, block_count);
    FullRun fr;
    full_run(c, a->m, p, method, keep, seed, flags, top_k, fr, timing);
    auto o = std::make_unique<DevOutputsImpl>();
    o->pub.rows = a->m.csr.rows;
    o->pub.cols = a->m.csr.cols;
    o->pub.k_sigma = fr.merge.k;
    o->pub.k_v = fr.r;
    o->pub.n_edges = fr.rep.edges.n;
    o->sigma = std::move(fr.merge.sigma);
    o->u = std::move(fr.merge.u);
    o->v = std::move(fr.v);
    o->repaired = std::move(fr.repaired);
    o->pub.d_sigma = o->sigma.get();
    o->pub.d_u = o->u.get();
    o->pub.d_v = (flags & RK_WANT_V) ? o->v.get() : nullptr;
    *out = &o.release()->pub;
  });
}

rk_status rk_dev_outputs_free(rk_dev_outputs* o) {
  if (!o) return RK_OK;
  delete reinterpret_cast<DevOutputsImpl*>(o);
  return RK_OK;
}

uint32_t rk_crc32(const void* data, uint64_t size) { return size ? crc32_host(data, size) : 0u; }

rk_status rk_dev_crc32(rk_ctx* ctx, const void* d_data, const uint64_t* offsets, const uint64_t* lengths, uint64_t n,
                       uint32_t* crcs) {
  return guarded([&] {
    check_ctx(ctx);
    if (n && (!d_data || !offsets || !lengths || !crcs)) fail(RK_INVALID_ARGUMENT, "NULL argument");
    CallScope sc(&ctx->c);
    crc32_device(static_cast<const unsigned char*>(d_data), std::vector<uint64_t>(offsets, offsets + n),
                 std::vector<uint64_t>(lengths, lengths + n), crcs, ctx->c.stream);
  });
}

rk_status rk_write_block_record(uint32_t block_index, uint32_t rows, uint32_t kept, const double* payload,
                                const char* path) {
  return guarded([&] {
    if (!path) fail(RK_INVALID_ARGUMENT, "NULL argument");
    const uint64_t count = (uint64_t)rows * kept;
    if (count && !payload) fail(RK_INVALID_ARGUMENT, "block record payload size mismatch");
    write_record_file(block_index, rows, kept, payload, count ? crc32_host(payload, 8 * count) : 0u, path);
  });
}

rk_status rk_read_block_record(const char* path, uint32_t* block_index, uint32_t* rows, uint32_t* kept,
                               double** payload) {
  return guarded([&] {
    if (!path || !block_index || !rows || !kept || !payload) fail(RK_INVALID_ARGUMENT, "NULL argument");
    std::vector<double> p;
    read_record_file(path, *block_index, *rows, *kept, p);
    *payload = host_alloc<double>(p.size());
    if (!p.empty()) std::memcpy(*payload, p.data(), p.size() * sizeof(double));
  });
}

rk_status rk_write_records(rk_ctx* ctx, const rk_records* records, const char* path_prefix) {
  return guarded([&] {
    check_ctx(ctx);
    if (!records || !path_prefix) fail(RK_INVALID_ARGUMENT, "NULL argument");
    CallScope sc(&ctx->c);
    cudaStream_t s = ctx->c.stream;
    const uint64_t n = records->n_records, M = records->rows;
    std::vector<uint64_t> off(n), len(n);
    uint64_t total = 0;
    for (uint64_t d = 0; d < n; ++d) {
      off[d] = 8 * records->offset[d];
      len[d] = 8 * M * records->kept[d];
      total = std::max(total, off[d] + len[d]);
    }
    std::vector<uint32_t> crc(n, 0u);
    if (total) {
      DBuf<unsigned char> dev(total, s);
      RK_CUDA_CHECK(cudaMemcpyAsync(dev.get(), records->payload, total, cudaMemcpyHostToDevice, s));
      crc32_device(dev.get(), off, len, crc.data(), s);
    }
    for (uint64_t d = 0; d < n; ++d)
      write_record_file((uint32_t)d, (uint32_t)M, records->kept[d], records->payload + records->offset[d], crc[d],
                        std::string(path_prefix) + std::to_string(d) + ".rnky");
  });
}

rk_status rk_dev_residual(rk_ctx* ctx, const rk_dev_matrix* a, const rk_dev_outputs* out, double* residual,
                          double* a_norm) {
  return guarded([&] {
    check_ctx(ctx);
    if (!a || !out || !residual || !a_norm) fail(RK_INVALID_ARGUMENT, "NULL argument");
    if (!out->d_v) fail(RK_INVALID_ARGUMENT, "rk_dev_residual: the outputs carry no V (RK_WANT_V)");
    CallScope sc(&ctx->c);
    const auto* impl = reinterpret_cast<const DevOutputsImpl*>(out);
    const DevMatrix& m = impl->repaired ? *impl->repaired : a->m;
    if (m.csc.rows != out->rows || m.csc.cols != out->cols)
      fail(RK_INVALID_ARGUMENT, "rk_dev_residual: matrix and outputs differ in shape");
    double r2 = 0.0, a2 = 0.0;
    residual_device(m.csc, out->d_u, (uint32_t)out->k_sigma, out->d_sigma, (uint32_t)out->k_v, out->d_v,
                    ctx->c.num_sms, &r2, &a2, ctx->c.stream);
    *residual = std::sqrt(r2);
    *a_norm = std::sqrt(a2);
  });
}

// ---- RepairWorkspace (rk_workspace.cu) ----
struct rk_workspace {
  rk_ctx* owner;
  Workspace* w;
};

rk_status rk_workspace_create(rk_ctx* ctx, const rk_sparse_view* a, uint64_t block_count, rk_workspace** out) {
  return guarded([&] {
    check_ctx(ctx);
    check_view(a);
    if (!out) fail(RK_INVALID_ARGUMENT, "out is NULL");
    CallScope sc(&ctx->c);
    auto h = std::make_unique<rk_workspace>();
    h->owner = ctx;
    h->w = workspace_create(ctx->c, *a, block_count);
    *out = h.release();
  });
}

rk_status rk_workspace_destroy(rk_workspace* ws) {
  if (!ws) return RK_OK;
  return guarded([&] {
    CallScope sc(&ws->owner->c);
    workspace_destroy(ws->w);
    delete ws;
  });
}

rk_status rk_workspace_has_entry(rk_workspace* ws, uint64_t row, uint64_t col, int32_t* out) {
  return guarded([&] {
    if (!ws || !out) fail(RK_INVALID_ARGUMENT, "NULL argument");
    CallScope sc(&ws->owner->c);
    *out = workspace_has_entry(*ws->w, row, col) ? 1 : 0;
  });
}

rk_status rk_workspace_row_lonely_in_block(rk_workspace* ws, uint64_t d, uint64_t row, int32_t* out) {
  return guarded([&] {
    if (!ws || !out) fail(RK_INVALID_ARGUMENT, "NULL argument");
    CallScope sc(&ws->owner->c);
    std::vector<uint64_t> r;
    workspace_lonely(*ws->w, d, row, row + 1, r);
    *out = r.empty() ? 0 : 1;
  });
}

rk_status rk_workspace_lonely_rows(rk_workspace* ws, uint64_t d, uint64_t* rows_out, uint64_t* n_out) {
  return guarded([&] {
    if (!ws || !n_out) fail(RK_INVALID_ARGUMENT, "NULL argument");
    CallScope sc(&ws->owner->c);
    std::vector<uint64_t> r;
    workspace_lonely(*ws->w, d, 0, UINT64_MAX, r);
    if (!r.empty() && !rows_out) fail(RK_INVALID_ARGUMENT, "rows_out is NULL");
    std::copy(r.begin(), r.end(), rows_out);
    *n_out = r.size();
  });
}

rk_status rk_workspace_neighbor_columns(rk_workspace* ws, uint64_t d, uint64_t row, uint64_t* cols_out,
                                        uint64_t* n_out) {
  return guarded([&] {
    if (!ws || !n_out) fail(RK_INVALID_ARGUMENT, "NULL argument");
    CallScope sc(&ws->owner->c);
    std::vector<uint64_t> cols;
    workspace_neighbor_columns(*ws->w, d, row, cols);
    if (!cols.empty() && !cols_out) fail(RK_INVALID_ARGUMENT, "cols_out is NULL");
    std::copy(cols.begin(), cols.end(), cols_out);
    *n_out = cols.size();
  });
}

rk_status rk_workspace_insert(rk_workspace* ws, uint64_t row, uint64_t col) {
  return guarded([&] {
    if (!ws) fail(RK_INVALID_ARGUMENT, "NULL argument");
    CallScope sc(&ws->owner->c);
    workspace_insert(*ws->w, row, col);
  });
}

rk_status rk_workspace_to_matrix(rk_workspace* ws, rk_sparse* out) {
  return guarded([&] {
    if (!ws || !out) fail(RK_INVALID_ARGUMENT, "NULL argument");
    CallScope sc(&ws->owner->c);
    std::memset(out, 0, sizeof *out);
    workspace_to_matrix(*ws->w, *out);
  });
}

// ---- evaluation metrics (rk_eval.cu) ----
rk_status rk_dev_sigma_error(rk_ctx* ctx, const double* d_sigma_hat, uint64_t n_hat, const double* d_sigma_ref,
                             uint64_t n_ref, double* out) {
  return guarded([&] {
    check_ctx(ctx);
    if (!out || (n_hat && !d_sigma_hat) || (n_ref && !d_sigma_ref)) fail(RK_INVALID_ARGUMENT, "NULL argument");
    CallScope sc(&ctx->c);
    *out = sigma_error_device(d_sigma_hat, n_hat, d_sigma_ref, n_ref, ctx->c.stream);
  });
}

rk_status rk_dev_align_signs(rk_ctx* ctx, const double* d_u_hat, const double* d_u_ref, uint64_t rows, uint64_t cols,
                             const double* d_sigma_ref, uint64_t n_sigma, double* d_out) {
  return guarded([&] {
    check_ctx(ctx);
    if (rows * cols && (!d_u_hat || !d_u_ref || !d_out)) fail(RK_INVALID_ARGUMENT, "NULL argument");
    CallScope sc(&ctx->c);
    align_signs_device(ctx->c, d_u_hat, d_u_ref, rows, cols, d_sigma_ref, n_sigma, d_out);
    sync(ctx->c.stream);
  });
}

rk_status rk_dev_left_vector_error(rk_ctx* ctx, const double* d_u_hat, const double* d_u_ref, uint64_t rows,
                                   uint64_t cols, const double* d_sigma_ref, uint64_t n_sigma, double* out) {
  return guarded([&] {
    check_ctx(ctx);
    if (!out || (rows * cols && (!d_u_hat || !d_u_ref))) fail(RK_INVALID_ARGUMENT, "NULL argument");
    CallScope sc(&ctx->c);
    *out = left_vector_error_device(ctx->c, d_u_hat, d_u_ref, rows, cols, d_sigma_ref, n_sigma);
  });
}

rk_status rk_dev_numerical_rank(rk_ctx* ctx, const double* d_a, uint64_t rows, uint64_t cols, double tol,
                                uint64_t* out) {
  return guarded([&] {
    check_ctx(ctx);
    if (!out || (rows * cols && !d_a)) fail(RK_INVALID_ARGUMENT, "NULL argument");
    CallScope sc(&ctx->c);
    *out = numerical_rank_device(ctx->c, d_a, rows, cols, tol);
  });
}

rk_status rk_sigma_error(rk_ctx* ctx, const double* sigma_hat, uint64_t n_hat, const double* sigma_ref,
                         uint64_t n_ref, double* out) {
  return guarded([&] {
    check_ctx(ctx);
    if (!out || (n_hat && !sigma_hat) || (n_ref && !sigma_ref)) fail(RK_INVALID_ARGUMENT, "NULL argument");
    CallScope sc(&ctx->c);
    cudaStream_t s = ctx->c.stream;
    DBuf<double> a(n_hat + 1, s), b(n_ref + 1, s);
    to_device(a.get(), sigma_hat, n_hat, s);
    to_device(b.get(), sigma_ref, n_ref, s);
    *out = sigma_error_device(a.get(), n_hat, b.get(), n_ref, s);
  });
}

namespace {
void check_align_shapes(uint64_t n_sigma, uint64_t cols) {
  if (n_sigma && n_sigma != cols) fail(RK_INVALID_ARGUMENT, "align_signs: sigma length mismatch");
}
}  // namespace

rk_status rk_align_signs(rk_ctx* ctx, const double* u_hat, const double* u_ref, uint64_t rows, uint64_t cols,
                         const double* sigma_ref, uint64_t n_sigma, double* out) {
  return guarded([&] {
    check_ctx(ctx);
    if (rows * cols && (!u_hat || !u_ref || !out)) fail(RK_INVALID_ARGUMENT, "NULL argument");
    check_align_shapes(n_sigma, cols);
    CallScope sc(&ctx->c);
    cudaStream_t s = ctx->c.stream;
    const uint64_t n = rows * cols;
    DBuf<double> h(n + 1, s), r(n + 1, s), o(n + 1, s), sg(n_sigma + 1, s);
    to_device(h.get(), u_hat, n, s);
    to_device(r.get(), u_ref, n, s);
    to_device(sg.get(), sigma_ref, n_sigma, s);
    align_signs_device(ctx->c, h.get(), r.get(), rows, cols, n_sigma ? sg.get() : nullptr, n_sigma, o.get());
    if (n) RK_CUDA_CHECK(cudaMemcpyAsync(out, o.get(), n * sizeof(double), cudaMemcpyDeviceToHost, s));
    sync(s);
  });
}

rk_status rk_left_vector_error(rk_ctx* ctx, const double* u_hat, const double* u_ref, uint64_t rows, uint64_t cols,
                               const double* sigma_ref, uint64_t n_sigma, double* out) {
  return guarded([&] {
    check_ctx(ctx);
    if (!out || (rows * cols && (!u_hat || !u_ref))) fail(RK_INVALID_ARGUMENT, "NULL argument");
    check_align_shapes(n_sigma, cols);
    CallScope sc(&ctx->c);
    cudaStream_t s = ctx->c.stream;
    const uint64_t n = rows * cols;
    DBuf<double> h(n + 1, s), r(n + 1, s), sg(n_sigma + 1, s);
    to_device(h.get(), u_hat, n, s);
    to_device(r.get(), u_ref, n, s);
    to_device(sg.get(), sigma_ref, n_sigma, s);
    *out = left_vector_error_device(ctx->c, h.get(), r.get(), rows, cols, n_sigma ? sg.get() : nullptr, n_sigma);
  });
}

rk_status rk_numerical_rank(rk_ctx* ctx, const double* a, uint64_t rows, uint64_t cols, double tol, uint64_t* out) {
  return guarded([&] {
    check_ctx(ctx);
    if (!out || (rows * cols && !a)) fail(RK_INVALID_ARGUMENT, "NULL argument");
    CallScope sc(&ctx->c);
    cudaStream_t s = ctx->c.stream;
    DBuf<double> d(rows * cols + 1, s);
    to_device(d.get(), a, rows * cols, s);
    *out = numerical_rank_device(ctx->c, d.get(), rows, cols, tol);
  });
}

uint64_t rk_merge_tree_leaves(uint64_t rows, uint64_t cols, uint64_t block_count, uint64_t keep) {
  try {
    Partition p = make_partition(cols, block_count);
    std::vector<uint32_t> kept(block_count);
    for (uint64_t d = 0; d < block_count; ++d) {
      const uint64_t w = p.end(d) - p.begin(d), k_full = std::min(rows, w);
      kept[d] = (uint32_t)(keep == 0 ? k_full : std::min(keep, k_full));
    }
    return merge_leaves(kept, (uint32_t)rows).size();
  } catch (...) {
    return 0;
  }
}

}  // extern "C"

namespace {

// the shard's part of a sharded run: repair (whole matrix, redundantly), block
// stage of the leaves [leaf_lo, leaf_hi), then either the TSQR subtree factor
// (gram = false) or the Gram partial of the subtree (gram = true, records kept)
void shard_factor(rk_ctx* ctx, const rk_dev_matrix* a, uint64_t block_count, rk_method method, uint64_t keep,
                  uint64_t seed, uint64_t leaf_lo, uint64_t leaf_hi, double* d_out, rk_dev_shard** shard_out,
                  rk_timing* timing, bool gram, bool keep_records = false) {
  check_ctx(ctx);
  if (!a || !shard_out || !d_out) fail(RK_INVALID_ARGUMENT, "NULL argument");
  CallScope sc(&ctx->c);
  Ctx& c = ctx->c;
  cudaStream_t s = c.stream;
  const uint64_t launches0 = c.launches;
  const uint32_t M = (uint32_t)a->m.csr.rows;
  if (gram && !gram_merge_eligible(M))
    fail(RK_GRAM_REJECTED, "the merge's Gram route does not apply to " + std::to_string(M) + " rows");
  auto sh = std::make_unique<rk_dev_shard>();
  sh->owner = ctx;
  sh->a = a;
  sh->p = make_partition(a->m.csr.cols, block_count);
  sh->method = method;
  sh->seed = seed;
  // the tree's leaves from the per-block kept counts
  std::vector<uint32_t> kept(block_count);
  for (uint64_t d = 0; d < block_count; ++d) {
    const uint64_t w = sh->p.end(d) - sh->p.begin(d), k_full = std::min<uint64_t>(M, w);
    kept[d] = (uint32_t)(keep == 0 ? k_full : std::min(keep, k_full));
  }
  std::vector<TreeLeaf> leaves = merge_leaves(kept, M);
  if (leaf_lo >= leaf_hi || leaf_hi > leaves.size()) fail(RK_OUT_OF_RANGE, "leaf range outside the merge tree");
  RK_NVTX("rk.shard_factor");
  RK_CUDA_CHECK(cudaEventRecord(c.ev[3], s));
  sh->repaired = repair_and_apply(c, a->m, sh->p, method, seed, sh->repair_out);
  RK_CUDA_CHECK(cudaEventRecord(c.ev[4], s));
  const uint64_t d_lo = leaves[leaf_lo].r0, d_hi = leaves[leaf_hi - 1].r1;
  sh->d_lo = d_lo;
  BlockStageResult& br = sh->blocks;
  block_stage(c, *sh->rep(), sh->p, d_lo, d_hi, keep, br, nullptr);
  if (any_failure(br)) throw_block_failure(br, d_lo);
  RK_CUDA_CHECK(cudaEventRecord(c.ev[5], s));
  // leaves re-indexed to the shard's records
  sh->local.assign(leaves.begin() + leaf_lo, leaves.begin() + leaf_hi);
  for (TreeLeaf& L : sh->local) { L.r0 -= (uint32_t)d_lo; L.r1 -= (uint32_t)d_lo; }
  if (gram) {
    std::vector<std::pair<uint32_t, uint32_t>> lr;
    for (const TreeLeaf& L : sh->local) lr.push_back({L.r0, L.r1});
    leaf_gram_tree(br.payload.get(), br.offset, br.kept, M, lr, d_out, s, &br.eff);
    sh->has_records = true;
  } else {
    DBuf<double> R;
    merge_subtree(c, br.payload.get(), br.offset, br.kept, M, sh->local, 0, sh->local.size(), R, &br.eff);
    RK_CUDA_CHECK(cudaMemcpyAsync(d_out, R.get(), sizeof(double) * (uint64_t)M * M, cudaMemcpyDeviceToDevice, s));
    if (keep_records) sh->has_records = true;
    else br.payload.release();
  }
  RK_CUDA_CHECK(cudaEventRecord(c.ev[6], s));
  sync(s);
  if (timing) {
    std::memset(timing, 0, sizeof *timing);
    timing->repair_ms = elapsed(c.ev[3], c.ev[4]);
    timing->blocks_ms = elapsed(c.ev[4], c.ev[5]);
    timing->merge_ms = elapsed(c.ev[5], c.ev[6]);
    timing->total_ms = elapsed(c.ev[3], c.ev[6]);
    timing->qr_ms = br.qr_ms;
    timing->jacobi_ms = br.jacobi_ms;
    timing->jacobi_sweeps_max = br.sweeps_max;
    timing->jacobi_rotations = br.rotations;
    timing->kernel_launches = c.launches - launches0;
    timing->jacobi_sweeps_sum = br.sweeps_sum;
    timing->qr_flops = br.qr_flops;
    timing->jacobi_flops = br.jacobi_flops;
  }
  *shard_out = sh.release();
}

// V for the shard's columns from the finished merge, packaged as rk_dev_outputs
void shard_outputs(Ctx& c, const DevMatrix& rep, MergeOut& mo, uint32_t flags, uint64_t top_k, uint64_t col_lo,
                   uint64_t col_hi, rk_dev_outputs** out, rk_timing* timing, uint64_t launches0) {
  cudaStream_t s = c.stream;
  const uint32_t M = (uint32_t)rep.csr.rows;
  const uint64_t sweeps = mo.sweeps, rotations = mo.rotations;
  // the finish's share of the merge flops: the top of the tree's Jacobi (+ the
  // caller's Cholesky / combines, passed in mo.flops)
  const double merge_flops = mo.flops + jacobi_flops_of(sweeps, rotations, M, M);
  RK_CUDA_CHECK(cudaEventRecord(c.ev[4], s));
  auto o = std::make_unique<DevOutputsImpl>();
  uint32_t r = 0;
  if (flags & RK_WANT_V) {
    const uint32_t kk = (top_k && top_k < mo.k) ? (uint32_t)top_k : mo.k;
    std::vector<double> sig;
    to_host(sig, mo.sigma.get(), kk, s);
    sync(s);
    std::vector<uint32_t> ret = retained_of(sig.data(), kk, 1e-10);
    r = (uint32_t)ret.size();
    o->v.alloc((col_hi - col_lo) * (uint64_t)std::max<uint32_t>(r, 1), s);
    if (r) {
      DBuf<uint32_t> dret(r, s);
      to_device(dret.get(), ret.data(), r, s);
      recover_v_device(rep.csc, mo.u.get(), mo.k, dret.get(), mo.sigma.get(), r, o->v.get(), col_lo, col_hi, s);
      sync(s);
    }
  }
  RK_CUDA_CHECK(cudaEventRecord(c.ev[5], s));
  sync(s);
  o->pub.rows = M;
  o->pub.cols = col_hi - col_lo;
  o->pub.k_sigma = mo.k;
  o->pub.k_v = r;
  o->sigma = std::move(mo.sigma);
  o->u = std::move(mo.u);
  o->pub.d_sigma = o->sigma.get();
  o->pub.d_u = o->u.get();
  o->pub.d_v = (flags & RK_WANT_V) ? o->v.get() : nullptr;
  if (timing) {
    std::memset(timing, 0, sizeof *timing);
    timing->merge_ms = elapsed(c.ev[3], c.ev[4]);
    timing->recover_ms = elapsed(c.ev[4], c.ev[5]);
    timing->total_ms = elapsed(c.ev[3], c.ev[5]);
    timing->kernel_launches = c.launches - launches0;
    timing->merge_sweeps = sweeps;
    timing->merge_rotations = rotations;
    timing->merge_flops = merge_flops;
  }
  *out = &o.release()->pub;
}

}  // namespace

extern "C" {

rk_status rk_dev_shard_factor(rk_ctx* ctx, const rk_dev_matrix* a, uint64_t block_count, rk_method method,
                              uint64_t keep, uint64_t seed, uint64_t leaf_lo, uint64_t leaf_hi, double* d_root_out,
                              rk_dev_shard** shard_out, rk_timing* timing) {
  return guarded([&] {
    shard_factor(ctx, a, block_count, method, keep, seed, leaf_lo, leaf_hi, d_root_out, shard_out, timing, false);
  });
}

rk_status rk_dev_shard_factor_gram(rk_ctx* ctx, const rk_dev_matrix* a, uint64_t block_count, rk_method method,
                                   uint64_t keep, uint64_t seed, uint64_t leaf_lo, uint64_t leaf_hi,
                                   double* d_gram_out, rk_dev_shard** shard_out, rk_timing* timing) {
  return guarded([&] {
    shard_factor(ctx, a, block_count, method, keep, seed, leaf_lo, leaf_hi, d_gram_out, shard_out, timing, true);
  });
}

rk_status rk_dev_shard_tsqr(rk_ctx* ctx, rk_dev_shard* shard, double* d_root_out) {
  return guarded([&] {
    check_ctx(ctx);
    if (!shard || !d_root_out) fail(RK_INVALID_ARGUMENT, "NULL argument");
    if (!shard->has_records) fail(RK_INVALID_ARGUMENT, "the shard was not made by rk_dev_shard_factor_gram");
    CallScope sc(&ctx->c);
    Ctx& c = ctx->c;
    const uint32_t M = (uint32_t)shard->rep()->csr.rows;
    BlockStageResult& br = shard->blocks;
    DBuf<double> R;
    merge_subtree(c, br.payload.get(), br.offset, br.kept, M, shard->local, 0, shard->local.size(), R, &br.eff);
    RK_CUDA_CHECK(cudaMemcpyAsync(d_root_out, R.get(), sizeof(double) * (uint64_t)M * M, cudaMemcpyDeviceToDevice,
                                  c.stream));
    sync(c.stream);
  });
}

rk_status rk_dev_shard_finish_gram(rk_ctx* ctx, rk_dev_shard* shard, const double* d_grams, uint64_t n_roots,
                                   uint32_t flags, uint64_t top_k, uint64_t col_lo, uint64_t col_hi,
                                   rk_dev_outputs** out, rk_timing* timing) {
  return guarded([&] {
    check_ctx(ctx);
    if (!shard || !d_grams || !out || n_roots == 0) fail(RK_INVALID_ARGUMENT, "NULL argument");
    CallScope sc(&ctx->c);
    Ctx& c = ctx->c;
    cudaStream_t s = c.stream;
    const uint64_t launches0 = c.launches;
    const DevMatrix& rep = *shard->rep();
    const uint32_t M = (uint32_t)rep.csr.rows;
    if (col_hi > rep.csc.cols || col_lo > col_hi) fail(RK_OUT_OF_RANGE, "column range outside the matrix");
    RK_CUDA_CHECK(cudaEventRecord(c.ev[3], s));
    const uint64_t mm = (uint64_t)M * M;
    // the ranks' partials are aligned subtrees: finish the same pairwise tree
    DBuf<double> g(n_roots * mm, s);
    RK_CUDA_CHECK(cudaMemcpyAsync(g.get(), d_grams, sizeof(double) * n_roots * mm, cudaMemcpyDeviceToDevice, s));
    gram_tree_sum(g.get(), n_roots, M, s);
    const uint32_t cp = jacobi_cols_pad(M, M, false, c.smem_optin);
    DBuf<double> W((uint64_t)M * cp, s);
    W.zero();
    RK_CUDA_CHECK(cudaMemcpyAsync(W.get(), g.get(), sizeof(double) * mm, cudaMemcpyDeviceToDevice, s));
    g.release();
    MergeOut mo;
    if (!gram_merge(c, W, M, mo))
      fail(RK_GRAM_REJECTED, "the kappa guard rejected the merge's Gram route: rk_dev_shard_tsqr, all-gather, "
                             "rk_dev_shard_finish");
    mo.flops = (double)M * M * M / 3.0;  // the Cholesky of the summed Gram (its Jacobi: shard_outputs)
    shard_outputs(c, rep, mo, flags, top_k, col_lo, col_hi, out, timing, launches0);
  });
}

rk_status rk_dev_shard_finish(rk_ctx* ctx, rk_dev_shard* shard, const double* d_roots, uint64_t n_roots,
                              uint32_t flags, uint64_t top_k, uint64_t col_lo, uint64_t col_hi, rk_dev_outputs** out,
                              rk_timing* timing) {
  return guarded([&] {
    check_ctx(ctx);
    if (!shard || !d_roots || !out || n_roots == 0) fail(RK_INVALID_ARGUMENT, "NULL argument");
    CallScope sc(&ctx->c);
    Ctx& c = ctx->c;
    cudaStream_t s = c.stream;
    const uint64_t launches0 = c.launches;
    const DevMatrix& rep = *shard->rep();
    const uint32_t M = (uint32_t)rep.csr.rows;
    if (col_hi > rep.csc.cols || col_lo > col_hi) fail(RK_OUT_OF_RANGE, "column range outside the matrix");
    RK_CUDA_CHECK(cudaEventRecord(c.ev[3], s));
    std::vector<DBuf<double>> roots;
    for (uint64_t g = 0; g < n_roots; ++g) {
      roots.emplace_back((uint64_t)M * M, s);
      RK_CUDA_CHECK(cudaMemcpyAsync(roots.back().get(), d_roots + g * (uint64_t)M * M, sizeof(double) * M * M,
                                    cudaMemcpyDeviceToDevice, s));
    }
    MergeOut mo;
    merge_finish(c, roots, M, mo);
    shard_outputs(c, rep, mo, flags, top_k, col_lo, col_hi, out, timing, launches0);
  });
}

rk_status rk_dev_shard_destroy(rk_dev_shard* shard) {
  if (!shard) return RK_OK;
  return guarded([&] {
    CallScope sc(&shard->owner->c);
    sync(shard->owner->c.stream);
    delete shard;
  });
}

}  // extern "C"

// ===========================================================================
// Library-owned multi-GPU runs. One orchestration of the sharded protocol
// (DESIGN.md (e)) with three exchanges for its one collective (the all-gather of
// the ranks' M x M factors):
//   rk_multi_*                one process drives several devices: a host barrier,
//                             then every shard pulls the others' factors with peer
//                             copies (NVLink when peer access is available)
//   rk_dist_*                 one process per GPU: the library's own NCCL
//                             communicator (libnccl.so.2 opened at run time),
//                             ncclAllGather on the context's stream
//   rk_dev_sharded_full_svd   one process per GPU, the caller's all-gather (e.g.
//                             torch.distributed) as a callback
// Per rank: factor its leaves (Gram partial; the TSQR factor when the Gram route
// does not apply), exchange, finish; when the kappa guard rejects the summed Gram
// (identically on every rank) the TSQR factors are exchanged and finished instead.

#include <condition_variable>
#include <dlfcn.h>
#include <functional>
#include <thread>

#include <nccl.h>

namespace {

using Exchange = std::function<void(double* d_mine, double* d_all)>;  // all-gather of M*M doubles per rank

struct ShardPlan {
  uint64_t leaf_lo, leaf_hi, col_lo, col_hi;
};

ShardPlan plan_shard(uint64_t M, uint64_t cols, uint64_t D, uint64_t keep, int world, int rank) {
  Partition p = make_partition(cols, D);
  std::vector<uint32_t> kept(D);
  for (uint64_t d = 0; d < D; ++d) {
    const uint64_t w = p.end(d) - p.begin(d), k_full = std::min<uint64_t>(M, w);
    kept[d] = (uint32_t)(keep == 0 ? k_full : std::min(keep, k_full));
  }
  const std::vector<TreeLeaf> leaves = merge_leaves(kept, (uint32_t)M);
  const uint64_t n = leaves.size();
  if (world < 1 || (uint64_t)world > n || rank < 0 || rank >= world)
    fail(RK_INVALID_ARGUMENT, "cannot shard " + std::to_string(n) + " merge-tree leaves over " +
                                  std::to_string(world) + " ranks");
  const uint64_t per = n / world;
  ShardPlan sp;
  sp.leaf_lo = rank * per;
  sp.leaf_hi = rank + 1 == world ? n : (rank + 1) * per;
  sp.col_lo = p.begin(leaves[sp.leaf_lo].r0);
  sp.col_hi = p.end(leaves[sp.leaf_hi - 1].r1 - 1);
  return sp;
}

[[noreturn]] void rethrow_status(rk_status st) { fail(st, g_error); }
void chk(rk_status st) {
  if (st != RK_OK) rethrow_status(st);
}

struct RankRun {
  rk_dev_shard* shard = nullptr;
  rk_dev_outputs* out = nullptr;
  rk_timing tf{}, tfin{};
  ShardPlan plan{};
  ~RankRun() {
    if (out) rk_dev_outputs_free(out);
    if (shard) rk_dev_shard_destroy(shard);
  }
};

void sharded_run(rk_ctx* ctx, const rk_dev_matrix* a, uint64_t D, rk_method method, uint64_t keep, uint64_t seed,
                 uint32_t flags, uint64_t top_k, int world, int rank, const Exchange& ex, bool keep_records,
                 RankRun& r) {
  RK_NVTX("rk.sharded_run");
  const uint64_t M = a->m.csr.rows;
  r.plan = plan_shard(M, a->m.csr.cols, D, keep, world, rank);
  const uint64_t mm = M * M;
  DBuf<double> mine, all;
  {
    CallScope sc(&ctx->c);
    mine.alloc(mm ? mm : 1, ctx->c.stream);
    all.alloc(world * mm ? world * mm : 1, ctx->c.stream);
    sync(ctx->c.stream);
  }
  bool gram = gram_merge_eligible((uint32_t)M);
  try {
    shard_factor(ctx, a, D, method, keep, seed, r.plan.leaf_lo, r.plan.leaf_hi, mine.get(), &r.shard, &r.tf, gram,
                 keep_records);
  } catch (const Error& e) {
    if (e.code != RK_GRAM_REJECTED) throw;
    gram = false;
    shard_factor(ctx, a, D, method, keep, seed, r.plan.leaf_lo, r.plan.leaf_hi, mine.get(), &r.shard, &r.tf, false,
                 keep_records);
  }
  {
    RK_NVTX("rk.exchange");
    ex(mine.get(), all.get());
  }
  if (gram) {
    const rk_status st = rk_dev_shard_finish_gram(ctx, r.shard, all.get(), world, flags, top_k, r.plan.col_lo,
                                                  r.plan.col_hi, &r.out, &r.tfin);
    if (st != RK_GRAM_REJECTED) {
      chk(st);
      return;
    }
    chk(rk_dev_shard_tsqr(ctx, r.shard, mine.get()));
    ex(mine.get(), all.get());
  }
  chk(rk_dev_shard_finish(ctx, r.shard, all.get(), world, flags, top_k, r.plan.col_lo, r.plan.col_hi, &r.out,
                          &r.tfin));
}

void add_timing(rk_timing& t, const RankRun& r) {
  t.repair_ms = std::max(t.repair_ms, r.tf.repair_ms);
  t.blocks_ms = std::max(t.blocks_ms, r.tf.blocks_ms);
  t.merge_ms = std::max(t.merge_ms, r.tf.merge_ms + r.tfin.merge_ms);
  t.recover_ms = std::max(t.recover_ms, r.tfin.recover_ms);
  t.total_ms = std::max(t.total_ms, r.tf.total_ms + r.tfin.total_ms);
  t.qr_ms = std::max(t.qr_ms, (double)r.tf.qr_ms);
  t.jacobi_ms = std::max(t.jacobi_ms, (double)r.tf.jacobi_ms);
  t.jacobi_sweeps_max = std::max(t.jacobi_sweeps_max, r.tf.jacobi_sweeps_max);
  t.jacobi_rotations += r.tf.jacobi_rotations;
  t.kernel_launches += r.tf.kernel_launches + r.tfin.kernel_launches;
  t.jacobi_sweeps_sum += r.tf.jacobi_sweeps_sum;
  t.qr_flops += r.tf.qr_flops;
  t.jacobi_flops += r.tf.jacobi_flops;
  t.merge_sweeps = r.tfin.merge_sweeps;
  t.merge_rotations = r.tfin.merge_rotations;
  t.merge_flops = std::max(t.merge_flops, r.tfin.merge_flops);
}

// a host barrier that a failing shard can break (the others then fail too instead of waiting)
struct Barrier {
  std::mutex m;
  std::condition_variable cv;
  int n, count = 0;
  uint64_t gen = 0;
  bool broken = false;
  explicit Barrier(int n_) : n(n_) {}
  void wait() {
    std::unique_lock<std::mutex> lk(m);
    if (broken) fail(RK_RUNTIME, "another shard failed");
    const uint64_t g = gen;
    if (++count == n) {
      count = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    cv.wait(lk, [&] { return gen != g || broken; });
    if (gen == g) fail(RK_RUNTIME, "another shard failed");
  }
  void abort() {
    std::lock_guard<std::mutex> lk(m);
    broken = true;
    cv.notify_all();
  }
};

// ---- NCCL, opened at run time ----
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    if (!api.get_unique_id || !api.comm_init_rank || !api.all_gather || !api.comm_destroy || !api.error_string)
      err = "libnccl.so.2 lacks a required symbol";
  });
  if (!err.empty()) fail(RK_RUNTIME, err);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(RK_RUNTIME, std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace

struct rk_multi {
  std::vector<int> devices;
  std::vector<rk_ctx*> ctx;
};

struct rk_dist {
  rk_ctx* ctx = nullptr;
  ncclComm_t comm = nullptr;
  int world = 0, rank = 0;
};

extern "C" {

int32_t rk_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

rk_status rk_multi_create(const int32_t* devices, uint32_t n, rk_multi** out) {
  return guarded([&] {
    if (!devices || !n || !out) fail(RK_INVALID_ARGUMENT, "rk_multi_create: no devices");
    auto m = std::make_unique<rk_multi>();
    for (uint32_t g = 0; g < n; ++g) {
      rk_ctx* c = nullptr;
      const rk_status st = rk_ctx_create(devices[g], &c);
      if (st != RK_OK) {
        for (rk_ctx* x : m->ctx) rk_ctx_destroy(x);
        rethrow_status(st);
      }
      m->ctx.push_back(c);
      m->devices.push_back(devices[g]);
    }
    // peer access between distinct devices (the factor exchange then runs over NVLink)
    for (uint32_t i = 0; i < n; ++i)
      for (uint32_t j = 0; j < n; ++j) {
        const int a = devices[i], b = devices[j];
        int can = 0;
        if (a == b || cudaDeviceCanAccessPeer(&can, a, b) != cudaSuccess || !can) continue;
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(a);
        const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        cudaGetLastError();
        cudaSetDevice(prev);
      }
    *out = m.release();
  });
}

rk_status rk_multi_destroy(rk_multi* m) {
  if (!m) return RK_OK;
  for (rk_ctx* c : m->ctx) rk_ctx_destroy(c);
  delete m;
  return RK_OK;
}

rk_status rk_multi_run_pipeline(rk_multi* m, const rk_sparse_view* a, uint64_t block_count, rk_method method,
                                uint64_t keep, uint64_t seed, uint32_t flags, uint64_t top_k,
                                rk_pipeline_result* out) {
  return guarded([&] {
    if (!m || !out) fail(RK_INVALID_ARGUMENT, "NULL argument");
    check_view(a);
    std::memset(out, 0, sizeof *out);
    const int G = (int)m->ctx.size();
    const uint64_t M = a->rows;
    const uint64_t mm = M * M;
    std::vector<rk_dev_matrix*> dms(G, nullptr);
    std::vector<std::unique_ptr<RankRun>> runs(G);
    std::vector<double*> mines(G, nullptr);
    std::vector<rk_status> status(G, RK_OK);
    std::vector<std::string> errors(G);
    Barrier bar(G);
    auto worker = [&](int g) {
      try {
        rk_ctx* ctx = m->ctx[g];
        chk(rk_dev_matrix_create(ctx, a, &dms[g]));
        runs[g] = std::make_unique<RankRun>();
        Exchange ex = [&, g, ctx](double* mine, double* all) {
          mines[g] = mine;
          bar.wait();  // every shard's factor is written (each synchronized its stream)
          {
            CallScope sc(&ctx->c);
            for (int h = 0; h < G; ++h) {
              if (m->devices[h] == m->devices[g])
                RK_CUDA_CHECK(cudaMemcpyAsync(all + h * mm, mines[h], mm * 8, cudaMemcpyDeviceToDevice,
                                              ctx->c.stream));
              else
                RK_CUDA_CHECK(cudaMemcpyPeerAsync(all + h * mm, m->devices[g], mines[h], m->devices[h], mm * 8,
                                                  ctx->c.stream));
            }
            sync(ctx->c.stream);
          }
          bar.wait();  // nobody rewrites its factor (the TSQR fallback) while another copies it
        };
        sharded_run(ctx, dms[g], block_count, method, keep, seed, flags, top_k, G, g, ex,
                    (flags & RK_WANT_RECORDS) != 0, *runs[g]);
      } catch (const Error& e) {
        status[g] = e.code;
        errors[g] = e.what();
        bar.abort();
      } catch (const std::exception& e) {
        status[g] = RK_RUNTIME;
        errors[g] = e.what();
        bar.abort();
      }
    };
    std::vector<std::thread> th;
    for (int g = 0; g < G; ++g) th.emplace_back(worker, g);
    for (auto& t : th) t.join();
    auto cleanup = [&] {
      runs.clear();
      for (int g = 0; g < G; ++g)
        if (dms[g]) rk_dev_matrix_destroy(dms[g]);
    };
    for (int g = 0; g < G; ++g)
      if (status[g] != RK_OK && errors[g] != "another shard failed") {
        cleanup();
        fail(status[g], errors[g]);
      }
    for (int g = 0; g < G; ++g)
      if (status[g] != RK_OK) {
        cleanup();
        fail(status[g], errors[g]);
      }
    try {
      // host outputs: sigma, U from shard 0 (every shard holds the same), V rows and
      // records from their owners, copied concurrently on every device's stream
      RankRun& r0 = *runs[0];
      Ctx& c0 = m->ctx[0]->c;
      const rk_dev_outputs* o0 = r0.out;
      const uint64_t k = o0->k_sigma, r = o0->k_v;
      out->svd.u_rows = M;
      out->svd.u_cols = k;
      out->svd.n_sigma = k;
      {
        CallScope sc(&c0);
        out->svd.u = host_copy(o0->d_u, M * k, c0.stream);
        out->svd.sigma = host_copy(o0->d_sigma, k, c0.stream);
        report_to_host(r0.shard->repair_out, r0.shard->p, &out->report, c0.stream);
        if (flags & RK_WANT_REPAIRED) csr_to_entries_host(r0.shard->rep()->csr, out->repaired, c0.stream);
        sync(c0.stream);
      }
      if (flags & RK_WANT_V) {
        out->svd.has_v = 1;
        out->svd.v_rows = a->cols;
        out->svd.v_cols = r;
        out->svd.v = host_alloc<double>(a->cols * r);
      }
      std::vector<uint32_t> kept_all;
      std::vector<uint64_t> off_all;
      if (flags & RK_WANT_RECORDS) {
        const Partition p = make_partition(a->cols, block_count);
        for (uint64_t d = 0; d < block_count; ++d) {
          const uint64_t w = p.end(d) - p.begin(d), kf = std::min<uint64_t>(M, w);
          kept_all.push_back((uint32_t)(keep == 0 ? kf : std::min(keep, kf)));
        }
        uint64_t tot = 0;
        for (uint32_t kk : kept_all) {
          off_all.push_back(tot);
          tot += M * kk;
        }
        out->records.n_records = block_count;
        out->records.rows = M;
        out->records.kept = host_alloc<uint32_t>(block_count);
        out->records.offset = host_alloc<uint64_t>(block_count);
        std::copy(kept_all.begin(), kept_all.end(), out->records.kept);
        std::copy(off_all.begin(), off_all.end(), out->records.offset);
        out->records.payload = host_alloc<double>(tot ? tot : 1);
      }
      for (int g = 0; g < G; ++g) {
        RankRun& rr = *runs[g];
        Ctx& c = m->ctx[g]->c;
        CallScope sc(&c);
        if ((flags & RK_WANT_V) && r && rr.out->d_v)
          RK_CUDA_CHECK(cudaMemcpyAsync(out->svd.v + rr.plan.col_lo * r, rr.out->d_v,
                                        (rr.plan.col_hi - rr.plan.col_lo) * r * 8, cudaMemcpyDeviceToHost, c.stream));
        if (flags & RK_WANT_RECORDS) {
          const BlockStageResult& br = rr.shard->blocks;
          const uint64_t d0 = rr.shard->d_lo;
          if (!br.offset.empty()) {
            const uint64_t n = br.offset.back() + M * br.kept.back();
            RK_CUDA_CHECK(cudaMemcpyAsync(out->records.payload + off_all[d0], br.payload.get(), n * 8,
                                          cudaMemcpyDeviceToHost, c.stream));
          }
        }
      }
      for (int g = 0; g < G; ++g) {
        CallScope sc(&m->ctx[g]->c);
        sync(m->ctx[g]->c.stream);
        add_timing(out->timing, *runs[g]);
      }
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
}

rk_status rk_nccl_unique_id(uint8_t id_out[128]) {
  return guarded([&] {
    if (!id_out) fail(RK_INVALID_ARGUMENT, "NULL argument");
    ncclUniqueId id;
    nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    static_assert(sizeof id == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id_out, &id, 128);
  });
}

rk_status rk_dist_create(rk_ctx* ctx, int32_t world, int32_t rank, const uint8_t id[128], rk_dist** out) {
  return guarded([&] {
    check_ctx(ctx);
    if (!id || !out || world < 1 || rank < 0 || rank >= world) fail(RK_INVALID_ARGUMENT, "bad rank / world");
    CallScope sc(&ctx->c);
    auto d = std::make_unique<rk_dist>();
    d->ctx = ctx;
    d->world = world;
    d->rank = rank;
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    nccl_check(nccl().comm_init_rank(&d->comm, world, uid, rank), "ncclCommInitRank");
    *out = d.release();
  });
}

rk_status rk_dist_destroy(rk_dist* d) {
  if (!d) return RK_OK;
  return guarded([&] {
    if (d->comm) nccl().comm_destroy(d->comm);
    delete d;
  });
}

rk_status rk_dist_full_svd(rk_dist* d, const rk_dev_matrix* a, uint64_t block_count, rk_method method, uint64_t keep,
                           uint64_t seed, uint32_t flags, uint64_t top_k, rk_dev_outputs** out, rk_timing* timing,
                           uint64_t* col_lo, uint64_t* col_hi) {
  return guarded([&] {
    if (!d || !a || !out) fail(RK_INVALID_ARGUMENT, "NULL argument");
    const uint64_t mm = a->m.csr.rows * a->m.csr.rows;
    Exchange ex = [&](double* mine, double* all) {
      CallScope sc(&d->ctx->c);
      nccl_check(nccl().all_gather(mine, all, mm, ncclFloat64, d->comm, d->ctx->c.stream), "ncclAllGather");
      sync(d->ctx->c.stream);
    };
    RankRun r;
    sharded_run(d->ctx, a, block_count, method, keep, seed, flags, top_k, d->world, d->rank, ex, false, r);
    if (timing) {
      std::memset(timing, 0, sizeof *timing);
      add_timing(*timing, r);
    }
    if (col_lo) *col_lo = r.plan.col_lo;
    if (col_hi) *col_hi = r.plan.col_hi;
    *out = r.out;
    r.out = nullptr;
  });
}

rk_status rk_dev_sharded_full_svd(rk_ctx* ctx, const rk_dev_matrix* a, uint64_t block_count, rk_method method,
                                  uint64_t keep, uint64_t seed, uint32_t flags, uint64_t top_k, int32_t world,
                                  int32_t rank, rk_allgather_fn allgather, void* user, rk_dev_outputs** out,
                                  rk_timing* timing, uint64_t* col_lo, uint64_t* col_hi) {
  return guarded([&] {
    check_ctx(ctx);
    if (!a || !out || !allgather) fail(RK_INVALID_ARGUMENT, "NULL argument");
    const uint64_t mm = a->m.csr.rows * a->m.csr.rows;
    Exchange ex = [&](double* mine, double* all) {
      {
        CallScope sc(&ctx->c);
        sync(ctx->c.stream);
      }
      allgather(user, mine, all, mm);
    };
    RankRun r;
    sharded_run(ctx, a, block_count, method, keep, seed, flags, top_k, world, rank, ex, false, r);
    if (timing) {
      std::memset(timing, 0, sizeof *timing);
      add_timing(*timing, r);
    }
    if (col_lo) *col_lo = r.plan.col_lo;
    if (col_hi) *col_hi = r.plan.col_hi;
    *out = r.out;
    r.out = nullptr;
  });
}

}  // extern "C"
