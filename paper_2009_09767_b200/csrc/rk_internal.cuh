// rk_internal.cuh -- shared internals of libranky_b200 (not part of the ABI).
#pragma once

#include <nvtx3/nvToolsExt.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <cstring>
#include <string>
#include <vector>

#include "ranky_b200.h"

namespace rk {

// ---------------------------------------------------------------------------
// errors: internal C++ exceptions, mapped to rk_status at the C boundary

struct Error : std::runtime_error {
  rk_status code;
  double residual;
  Error(rk_status c, const std::string& what, double res = 0.0)
      : std::runtime_error(what), code(c), residual(res) {}
};

[[noreturn]] inline void fail(rk_status c, const std::string& what, double residual = 0.0) {
  throw Error(c, what, residual);
}

#define RK_CUDA_CHECK(expr)                                                                  \
  do {                                                                                      \
    cudaError_t rk_e_ = (expr);                                                             \
    if (rk_e_ != cudaSuccess)                                                               \
      ::rk::fail(RK_CUDA, std::string(#expr) + ": " + cudaGetErrorString(rk_e_));          \
  } while (0)

// launch bookkeeping: every kernel launch goes through RK_LAUNCH so the context
// can report how many of its kernels ran (bench.py "gpu_launches")
extern thread_local uint64_t* g_launch_counter;
// RK_TRACE=1: synchronize after every launch and log it to stderr (debugging hangs)
// Tuning and debug switches (RK_* environment variables).
// Read once per process on first use -- never on the hot path -- and re-read only by
// rk_reload_tuning() (tests flip them; no other API call may be in flight then).
// Defaults are the measured best.
struct Tuning {
  bool trace = false;             // RK_TRACE=1: synchronise and log every launch
  bool hostprof = false;          // RK_HOSTPROF=1: host/device segment times
  bool meminfo_exact = false;     // RK_MEMINFO=x: cudaMemGetInfo on every budget query
  int jacobi_gmax = 16;           // RK_JACOBI_GMAX: group-size cap
  int jacobi_single_g = 8;        // RK_JACOBI_SINGLE_G: the merge's group size
  int jacobi_warp = -1;           // RK_JACOBI_WARP=0/1 (-1: by shape)
  int jacobi_smem = -1;           // RK_JACOBI_SMEM=0/1: the shared-memory-resident Gram-assisted kernel (-1: batched blocks)
  int jacobi_smem_cl = 2;         // RK_JACOBI_SMEM_CL: its largest cluster (1, 2, 4, 8)
  bool jacobi_carry = true;       // RK_JACOBI_CARRY=0: the shared-memory kernel forms the full 16 x 16 Gram every step
  bool jacobi_wide = true;        // RK_JACOBI_WIDE=0: no wide pair-block kernel for >= 1024-row matrices
  double jacobi_check = -1.0;     // RK_JACOBI_CHECK: tail-check ratio (<0: by workload; 0 off)
  int jacobi_cluster = 0;         // RK_JACOBI_CLUSTER: cluster size override (0: planned)
  bool jacobi_debug = false;      // RK_JACOBI_DEBUG=1
  int jacobi_q = 0;               // RK_JACOBI_Q: lanes per pair override (0: planned)
  bool jacobi_unroll = true;      // RK_JACOBI_UNROLL=0: no compile-time group counts
  bool gram_pairs = false;        // RK_GRAM_PAIRS=1: row-pair Gram kernel (experiments build)
  bool diag_order = true;         // RK_DIAG_ORDER=0: no descending-diagonal ordering
  bool chol_right = false;        // RK_CHOL=r: right-looking Cholesky (experiments build)
  bool householder_only = false;  // RK_BLOCK_ROUTE=householder: no Gram route
  bool precond = false;           // RK_PRECOND=1: FP32-preconditioned Jacobi (experiments build)
  float precond_stop = 1e-5f;     // RK_PRECOND_STOP
  bool spmm_warp = false;         // RK_SPMM_WARP=1: warp-per-column V SpMM
  bool wide_reduce = true;        // RK_WIDE_REDUCE=0: wide blocks' Jacobi on X = T^T, not on its R
  bool presence_csr = false;      // RK_PRESENCE=csr: the rank check's flags by a thread per CSR entry (row search)
  bool syrk_block4 = true;        // RK_SYRK=tile: the merge's SYRK with one 8 x 8 tile per warp
  bool repair_speculate = true;   // RK_REPAIR_SPECULATE=0: the neighbor replay without speculated sets
  bool wide_rows_pow2 = true;     // RK_WIDE_ROWS=32: the reduced R's rows padded to multiples of 32
  bool eig_merge = true;          // RK_EIG_MERGE=0: the merge's Gram route by Cholesky + one-sided Jacobi
  bool spmm_tma = true;           // RK_SPMM_TMA=0: V rows by st.global instead of TMA bulk copies
  bool apply_q_regs = false;      // RK_APPLY_Q=regs: reflectors from L2 per step, not panels in shared memory
  bool apply_q_wy = true;         // RK_APPLY_Q=panel|regs: no compact-WY apply for factored jobs that kept T
  uint64_t jacobi_chunk_mb = 0;   // RK_JACOBI_CHUNK_MB: cap a batched Jacobi launch's matrices (0: one launch)
};
const Tuning& tuning();
void reload_tuning();
int device_sms(int device);  // cached per device

void trace_launch(const char* file, int line);

// NVTX stage ranges (nvtx3, header-only: free unless a tool such as nsys / ncu
// --nvtx is attached): RK_NVTX("rk.blocks") opens a range for the enclosing scope
struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
  NvtxScope(const NvtxScope&) = delete;
  NvtxScope& operator=(const NvtxScope&) = delete;
};
#define RK_NVTX_CAT2(a, b) a##b
#define RK_NVTX_CAT(a, b) RK_NVTX_CAT2(a, b)
#define RK_NVTX(name) ::rk::NvtxScope RK_NVTX_CAT(rk_nvtx_, __LINE__)(name)
#define RK_LAUNCH_CHECK()                                                                    \
  do {                                                                                      \
    if (::rk::g_launch_counter) ++*::rk::g_launch_counter;                                   \
    cudaError_t rk_e_ = cudaGetLastError();                                                 \
    if (rk_e_ != cudaSuccess)                                                               \
      ::rk::fail(RK_CUDA, std::string("kernel launch: ") + cudaGetErrorString(rk_e_));     \
    ::rk::trace_launch(__FILE__, __LINE__);                                                 \
  } while (0)

// ---------------------------------------------------------------------------
// stream-ordered device buffer

// synchronize `s` and release the device's pool memory that is not in use
void trim_pool(cudaStream_t s);

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(size_t count, cudaStream_t st) { alloc(count, st); }
  void alloc(size_t count, cudaStream_t st) {
    release();
    s = st;
    n = count;
    if (count) {
      cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), st);
      if (e == cudaErrorMemoryAllocation) {
        // the stream-ordered pool keeps freed blocks (release threshold = max); give
        // them back to the driver and retry once before reporting out-of-memory
        cudaGetLastError();
        trim_pool(st);
        e = cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), st);
      }
      if (e != cudaSuccess) {
        p = nullptr;
        n = 0;
        cudaGetLastError();
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        cudaGetLastError();
        fail(RK_NOMEM, std::string("device allocation of ") + std::to_string(count * sizeof(T)) +
                           " bytes failed: " + cudaGetErrorString(e) + " (device free " +
                           std::to_string(fr >> 20) + " of " + std::to_string(tot >> 20) + " MiB)");
      }
    }
  }
  void zero() {
    if (n) RK_CUDA_CHECK(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { release(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; s = o.s;
      o.p = nullptr; o.n = 0;
    }
    return *this;
  }
  T* get() const { return p; }
};

template <class T>
inline void to_host(std::vector<T>& dst, const T* src, size_t n, cudaStream_t s) {
  dst.resize(n);
  if (n) RK_CUDA_CHECK(cudaMemcpyAsync(dst.data(), src, n * sizeof(T), cudaMemcpyDeviceToHost, s));
}
// Pinned staging for the small host -> device uploads of an API call (job tables,
// pointer arrays). cudaMemcpyAsync from pageable memory waits for the stream, so
// every such upload would be a hidden host <-> device round trip; from the arena it
// is asynchronous. The arena belongs to the context and is rewound at the start of
// each call (after the previous call's uploads have been consumed).
struct PinnedArena {
  char* base = nullptr;
  size_t cap = 0, used = 0;
};
extern thread_local PinnedArena* g_arena;
template <class T>
inline void to_device(T* dst, const T* src, size_t n, cudaStream_t s) {
  if (!n) return;
  const size_t bytes = n * sizeof(T);
  PinnedArena* a = g_arena;
  if (a && a->base && a->used + bytes + 16 <= a->cap) {
    char* p = a->base + ((a->used + 15) & ~size_t(15));
    std::memcpy(p, src, bytes);
    a->used = (size_t)(p - a->base) + bytes;
    RK_CUDA_CHECK(cudaMemcpyAsync(dst, p, bytes, cudaMemcpyHostToDevice, s));
  } else {
    RK_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
  }
}
// RK_HOSTPROF=1: named marks (host wall clock + an event on the stream); prof_flush
// prints the host and device time of every segment between consecutive marks
void prof_mark(cudaStream_t s, const char* name);
void prof_flush();

inline void sync(cudaStream_t s) { RK_CUDA_CHECK(cudaStreamSynchronize(s)); }

inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// launch `kern` as clusters of `cluster` CTAs along x
inline void launch_cluster_kernel(const void* kern, unsigned grid, unsigned cluster, unsigned threads, size_t smem,
                                  cudaStream_t s, void** args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(threads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  RK_CUDA_CHECK(cudaLaunchKernelExC(&cfg, kern, args));
  RK_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// KeyedRng -- proj/src/rng.cpp:8-38, usable on host and device

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

struct KeyedRng {
  uint64_t state;
  __host__ __device__ __forceinline__ KeyedRng(uint64_t seed, uint64_t block, uint64_t row) {
    state = mix64(seed + 0x9e3779b97f4a7c15ull);
    state = mix64(state ^ (block + 0xbf58476d1ce4e5b9ull));
    state = mix64(state ^ (row + 0x94d049bb133111ebull));
  }
  __host__ __device__ __forceinline__ uint64_t next() {
    state += 0x9e3779b97f4a7c15ull;
    return mix64(state);
  }
  // unbiased: reject draws below 2^64 mod bound
  __host__ __device__ __forceinline__ uint64_t below(uint64_t bound) {
    const uint64_t threshold = (0 - bound) % bound;
    for (;;) {
      const uint64_t r = next();
      if (r >= threshold) return r % bound;
    }
  }
};

// ---------------------------------------------------------------------------
// column partition -- proj/src/partition.cpp:38-51: width floor(N/D), the last
// block absorbs the remainder

struct Partition {
  uint64_t n_cols = 0, blocks = 0, width = 0;
  __host__ __device__ uint64_t begin(uint64_t d) const { return d * width; }
  __host__ __device__ uint64_t end(uint64_t d) const { return d + 1 == blocks ? n_cols : (d + 1) * width; }
  __host__ __device__ uint64_t block_of(uint64_t col) const {
    uint64_t d = col / width;
    return d < blocks ? d : blocks - 1;
  }
};

inline Partition make_partition(uint64_t n_cols, uint64_t blocks) {
  if (blocks == 0 || blocks > n_cols)
    fail(RK_INVALID_ARGUMENT, "cannot split " + std::to_string(n_cols) + " columns into " +
                                  std::to_string(blocks) + " blocks");
  Partition p;
  p.n_cols = n_cols;
  p.blocks = blocks;
  p.width = n_cols / blocks;
  return p;
}

// ---------------------------------------------------------------------------
// device sparse matrix: CSR (row order) and CSC (column order), both with
// 64-bit offsets, 32-bit indices and FP64 values

struct DevCsr {
  uint64_t rows = 0, cols = 0, nnz = 0;
  DBuf<uint64_t> ptr;   // rows + 1
  DBuf<uint32_t> idx;   // column index
  DBuf<double> val;
};
struct DevCsc {
  uint64_t rows = 0, cols = 0, nnz = 0;
  DBuf<uint64_t> ptr;   // cols + 1
  DBuf<uint32_t> idx;   // row index, ascending within a column
  DBuf<double> val;
};

struct DevMatrix {
  DevCsr csr;
  DevCsc csc;
};

// ---------------------------------------------------------------------------
// context

struct Ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  size_t smem_optin = 227 * 1024;
  uint64_t launches = 0;
  cudaEvent_t ev[12] = {};  // [0..3] block stage, [3..7] pipeline stages, [8..11] spare
  PinnedArena arena;        // see to_device
  // device_free_bytes: cudaMemGetInfo at the first call, then tracked through the
  // stream-ordered pool's reservation
  bool free_known = false;
  size_t free0 = 0;
  uint64_t reserved0 = 0;
  // a second stream for result copies that overlap later stages (created on first use)
  cudaStream_t copy = nullptr;
  cudaEvent_t copy_ev[2] = {};
  // a side stream for independent launches of one stage (created on first use)
  cudaStream_t side = nullptr;
  cudaEvent_t side_ev[2] = {};
};

// free device memory for planning. Exact (cudaMemGetInfo, slow) at the first call
// and whenever the estimate is below `want` bytes; otherwise the first reading
// adjusted by the pool memory in use since then.
size_t device_free_bytes(Ctx& c, uint64_t want);

// RAII: activates the context's device and launch counter for one API call
struct CallScope {
  int prev_device = -1;
  uint64_t* prev_counter = nullptr;
  PinnedArena* prev_arena = nullptr;
  explicit CallScope(Ctx* c);
  ~CallScope();
};

// ---------------------------------------------------------------------------
// kernels & launchers (one .cu per group)

// rk_api.cu -- library-owned host output buffers (pinned above 1 MiB)
void* host_alloc_bytes(size_t bytes);

// rk_scan.cu -- exclusive prefix sums (deterministic)
void exclusive_scan_u64(const uint64_t* in, uint64_t* out, uint64_t n, cudaStream_t s);  // out has n+1
void exclusive_scan_u32to64(const uint32_t* in, uint64_t* out, uint64_t n, cudaStream_t s);

// rk_ingest.cu -- entries -> CSR, CSR -> CSC, CSC + edges -> repaired CSC/CSR
void upload_entries(const rk_sparse_view& a, DevMatrix& m, cudaStream_t s);
// stable device radix sort of host entries by (row, col) into host_sorted; dup_a / dup_b =
// the input positions of the first adjacent equal pair in sorted order (-1: none)
void sort_entries_device(const rk_entry* host_in, uint64_t n, rk_entry* host_sorted, int64_t* dup_a, int64_t* dup_b,
                         cudaStream_t s);
void csr_to_csc(const DevCsr& a, DevCsc& out, cudaStream_t s);
void csr_to_entries_host(const DevCsr& a, rk_sparse& out, cudaStream_t s);

struct DevEdges {  // repair edges in report order
  uint64_t n = 0;
  DBuf<uint32_t> block, row, col;
  DBuf<int32_t> mech;
};
void apply_edges(const DevMatrix& a, const DevEdges& e, DevMatrix& out, cudaStream_t s);

// rk_mm.cu: Matrix Market files
void load_matrix_market(const std::string& path, rk_sparse& out, cudaStream_t s);
void save_matrix_market(const rk_sparse_view& a, const std::string& path);

// rk_workspace.cu: RepairWorkspace's single-row API on the device
struct Workspace;
Workspace* workspace_create(Ctx& c, const rk_sparse_view& a, uint64_t block_count);
void workspace_destroy(Workspace* w);
bool workspace_has_entry(Workspace& w, uint64_t row, uint64_t col);
void workspace_lonely(Workspace& w, uint64_t d, uint64_t r_lo, uint64_t r_hi, std::vector<uint64_t>& out);
void workspace_neighbor_columns(Workspace& w, uint64_t d, uint64_t row, std::vector<uint64_t>& out);
void workspace_insert(Workspace& w, uint64_t row, uint64_t col);
void workspace_to_matrix(Workspace& w, rk_sparse& out);

// rk_repair.cu
struct RepairOut {
  DevEdges edges;
  std::vector<uint64_t> lonely_counts;
  uint64_t fallback = 0;
  uint64_t recomputed = 0;  // neighbor replay: steps whose speculated sets were invalidated
};
void repair_device(const DevMatrix& a, const Partition& p, rk_method method, uint64_t seed,
                   RepairOut& out, cudaStream_t s);
void lonely_rows_device(const DevMatrix& a, const Partition& p, uint64_t d, std::vector<uint64_t>& out,
                        cudaStream_t s);
void rng_eval_device(uint64_t n, uint64_t seed, const uint64_t* block, const uint64_t* row,
                     uint64_t draws, const uint64_t* bound, uint64_t* out, cudaStream_t s);

// rk_dense.cu -- QR, Jacobi, finalize, completion, apply_q (batched)
struct QrJob {        // one tall matrix, column-major, in place
  double* a;          // m x n, leading dimension lda
  uint64_t lda;
  uint32_t m, n;
  double* diag;       // n: R's diagonal
  double* beta;       // n: Householder betas (0 = identity)
  double* tmat;       // ceil(n/NB) * NB * NB: compact-WY T factors
  uint32_t split = 0; // > 0: [R_a; R_b] stacked triangles, R_a = rows [0, split) (split == n)
};
void qr_batched(const std::vector<QrJob>& jobs, cudaStream_t s, int sms);  // rk_qr.cu
uint32_t qr_max_rows();  // tallest matrix a panel can stage

// W := R^T (transpose=true) or R (false) from a factored QrJob; W is n x n col-major,
// zero-filled outside the triangle. rows: number of R rows (min(m, n)).
struct RJob {
  const double* a; uint64_t lda; const double* diag; uint32_t m, n;
  double* w; uint64_t ldw;
};
void r_extract_batched(const std::vector<RJob>& jobs, bool transpose, cudaStream_t s);

struct JacobiJob {    // one-sided Jacobi on the columns of w (rows x cols, col-major)
  double* w;          // rows x cols_pad, ldw = rows
  double* v;          // optional: cols x cols_pad accumulated rotations (col-major, ld = cols_pad) or null
  uint32_t rows, cols, cols_pad;
  double* alpha;      // cols_pad scratch
  uint64_t* stats;    // [0] sweeps, [1] rotations, [2] status (0 ok, 1 not converged), [3] residual bits, [4..7] scratch
  uint32_t gram_ok = 0;  // well-conditioned (kappa <= kappa_max): the Gram-assisted kernel may run it
  uint32_t rows_nz = 0;  // > 0: only the first rows_nz rows can be nonzero (a reduced R in a taller slot)
  uint32_t pre = 0;      // jacobi_smem_try already ran it: jacobi_batched only certifies
};
// latency: one latency-critical matrix (the merge) -- smaller groups, larger
// clusters. Never set for blocks: a block's rotation sequence (and with it its
// rounding) must not depend on how many blocks share the launch, so that the
// sharded path is bitwise identical for every rank count.
void jacobi_batched(std::vector<JacobiJob>& jobs, cudaStream_t s, int sms, size_t smem_optin, bool latency = false);
// the shared-memory-resident Gram-assisted kernel over a (heterogeneous) batch without V; true: every job ran
// (pre set) and jacobi_batched only has to certify. false: nothing was launched (a job does not fit, or switched off)
struct SideStream { cudaStream_t stream; cudaEvent_t fork, join; };  // optional: independent launches overlap the main stream's
bool jacobi_smem_try(std::vector<JacobiJob>& jobs, cudaStream_t s, size_t smem_optin, const SideStream* side);
bool jacobi_smem_fits(const JacobiJob& j, size_t smem_optin);  // a cluster's shared memory holds its staged matrix
// rk_precond.cu: FP32 Jacobi sweeps, then W <- W V with V the (Newton-Schulz
// orthogonalized) right singular vectors they give -- for gram_ok square jobs
bool precondition_eligible(const JacobiJob& j);
void precondition_fp32(std::vector<JacobiJob>& jobs, cudaStream_t s, int sms, size_t smem_optin, uint32_t g,
                       uint32_t G, int Q);
// RNKY records (rk_records.cu)
uint32_t crc32_host(const void* data, uint64_t size);
void crc32_device(const unsigned char* d_base, const std::vector<uint64_t>& off, const std::vector<uint64_t>& len,
                  uint32_t* h_crc, cudaStream_t s);
void write_record_file(uint32_t index, uint32_t rows, uint32_t kept, const double* payload, uint32_t crc,
                       const std::string& path);
void read_record_file(const std::string& path, uint32_t& index, uint32_t& rows, uint32_t& kept,
                      std::vector<double>& payload);
// ||A - U[:, :r] diag(sigma) V^T||_F^2 (exact, tile by tile) and ||A||_F^2
void residual_device(const DevCsc& a, const double* u, uint32_t ku, const double* sigma, uint32_t r, const double* v,
                     int sms, double* h_res2, double* h_a2, cudaStream_t s);

// finalize: sigma = column norms, stable descending sort, u = w/sigma, sign
// convention; optional payload (rows x k row-major, u*sigma) and U/sigma outputs
struct FinalJob {
  const double* w;    // rows x cols (ld = rows)
  uint32_t rows, cols, k;
  double* payload;    // rows x k row-major (nullable)
  double* u;          // rows x k row-major (nullable)
  double* sigma;      // k (nullable), descending
  double* sigma_all;  // cols (nullable): all singular values, descending
  uint32_t* order;    // cols scratch
  double* scratch;    // cols scratch
  const double* v_in; // optional cols x cols col-major rotations (ld = ldv) to permute into v_out
  uint64_t ldv;
  double* v_out;      // cols x k row-major (nullable)
  uint8_t* deficient; // k flags out (nullable): sigma <= kRankTol * sigma_max or zero
  const uint32_t* row_perm;  // nullable: W's row i is original row row_perm[i] (u / payload rows un-permuted)
};
void finalize_batched(const std::vector<FinalJob>& jobs, cudaStream_t s);
// deterministic orthonormal completion of flagged columns -- svd.cpp:150-201
void complete_columns_device(double* u_rowmajor, uint32_t rows, uint32_t cols, const uint8_t* deficient,
                             int* d_fail, cudaStream_t s);
// Jacobi planning: padded column count for rows x cols
uint32_t jacobi_cols_pad(uint32_t rows, uint32_t cols, bool with_v, size_t smem_optin);
// out (m x ncols col-major) = Q [x; 0] for a factored QrJob (svd.cpp:111-132)
void apply_q_device(const QrJob& qr, const double* x, uint32_t x_rows, uint32_t ncols, double* out,
                    cudaStream_t s);
struct ApplyQJob {    // out (qr.m x ncols col-major, ld qr.m) = Q [x; 0], x x_rows x ncols (ld x_rows)
  QrJob qr;
  const double* x;
  uint32_t x_rows, ncols;
  double* out;
  uint32_t wy_nb = 0;  // > 0: qr.tmat holds the compact-WY T factors of panels this wide (dense job)
};
// rk_qr.cu: the panel width qr_batched factors an h_max-row batch with; apply_q through the T factors
uint32_t qr_panel_nb(uint32_t h_max);
bool apply_q_wy_batched(const ApplyQJob* d_jobs, size_t n_jobs, uint32_t m_max, uint32_t c_max, uint32_t nb,
                        cudaStream_t s);
void apply_q_batched(const std::vector<ApplyQJob>& jobs, cudaStream_t s);

// rk_spmm.cu -- V = A^T U Sigma^-1 over the CSC
void recover_v_device(const DevCsc& a, const double* u, uint32_t u_cols, const uint32_t* retained,
                      const double* sigma, uint32_t r, double* v, uint64_t col_lo, uint64_t col_hi,
                      cudaStream_t s);

// rk_compact.cu -- per-block compaction of the sparse block into the tall
// factor input
struct BlockPlan {
  uint64_t block;
  uint32_t n_multi, n_single;  // compacted rows
  uint32_t n_rows;             // n_multi + n_single
  bool tall;                   // n_rows > M: QR first; else W = T^T directly
  uint64_t offset;             // doubles into the staging buffer
};
void compaction_counts(const DevMatrix& a, const Partition& p, uint64_t d_lo, uint64_t d_hi,
                       uint32_t* d_counts /* 2 * nblocks */, double* d_single /* nblocks * M */,
                       cudaStream_t s);
void compaction_fill(const DevMatrix& a, const Partition& p, const std::vector<BlockPlan>& plans,
                     uint64_t d_lo, const double* d_single, double* staging, cudaStream_t s);

}  // namespace rk
