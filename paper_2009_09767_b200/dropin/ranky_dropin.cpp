// ranky_dropin.cpp -- the reference's hot-path C++ API on the B200 C ABI.
//
// Compiled against the reference's own headers (proj/include/ranky/*.hpp, which
// a user of the reference already has) and linked IN PLACE OF the reference
// objects repair.o, svd.o, proxy.o and pipeline.o. Every numeric routine is a
// call into libranky_b200.so (include/ranky_b200.h); this file only converts the
// reference's value types to and from the C ABI's plain arrays and maps rk_status
// back onto the reference's exception types. See INTEGRATION.md.
//
// Replaced definitions (reference file:line):
//   repair.cpp:9-25    to_string / repair_method_from_string      (host, no arithmetic)
//   repair.cpp:27-40   RepairReport::to_log                       (host formatting)
//   repair.cpp:42-50   find_lonely_rows                           -> rk_find_lonely_rows
//   repair.cpp:162-216 repair                                     -> rk_repair
//   repair.cpp:218-223 rank_equal_probability                     (Eq. 5, host arithmetic)
//   svd.cpp:365-379    dense_svd                                  -> rk_dense_svd
//   svd.cpp:381-400    block_svd                                  -> rk_block_svd
//   proxy.cpp:8-38     build_proxy                                (host concatenation)
//   proxy.cpp:40-46    proxy_svd                                  -> rk_proxy_svd
//   proxy.cpp:48-72    recover_right_vectors                      -> rk_recover_right_vectors
//   pipeline.cpp:11-16 run_block_task                             -> rk_run_block_tasks
//   pipeline.cpp:18-59 proxy_from_records                         (host concatenation)
//   pipeline.cpp:61-121 run_pipeline                              -> rk_run_pipeline
//   repair.cpp:52-160  RepairWorkspace                            -> rk_workspace_* (device
//                      adjacency + inserted edges; the caller's KeyedRng draws on the host)
#include <algorithm>
#include <cstring>
#include <mutex>
#include <sstream>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "ranky/block_record.hpp"
#include "ranky/dense_matrix.hpp"
#include "ranky/errors.hpp"
#include "ranky/partition.hpp"
#include "ranky/pipeline.hpp"
#include "ranky/proxy.hpp"
#include "ranky/repair.hpp"
#include "ranky/sparse_matrix.hpp"
#include "ranky/svd.hpp"
#include "ranky_b200.h"

static_assert(sizeof(ranky::Entry) == sizeof(rk_entry), "ranky::Entry must match rk_entry");

namespace ranky {
namespace {

// The reference's functions are reentrant and may run concurrently (proj/src/pipeline.cpp
// runs run_block_task on a thread pool); an rk_ctx is not thread-safe (include/ranky_b200.h),
// so every calling thread gets its own context (own stream, pinned arena and launch
// counter), created on first use and destroyed when the thread exits.
struct ThreadContext {
  rk_ctx* ctx = nullptr;
  ~ThreadContext() {
    if (ctx) rk_ctx_destroy(ctx);
  }
};

rk_ctx* context() {
  thread_local ThreadContext tc;
  if (!tc.ctx) {
    int dev = 0;
    if (const char* e = std::getenv("RANKY_DEVICE")) dev = std::atoi(e);
    if (rk_ctx_create(dev, &tc.ctx) != RK_OK) {
      tc.ctx = nullptr;
      throw std::runtime_error(std::string("ranky B200 drop-in: ") + rk_last_error());
    }
  }
  return tc.ctx;
}

void check(rk_status st) {
  if (st == RK_OK) return;
  const std::string msg = rk_last_error();
  switch (st) {
    case RK_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case RK_OUT_OF_RANGE: throw std::out_of_range(msg);
    case RK_CONVERGENCE: {
      // ConvergenceError appends " (residual r)" itself: strip ours
      std::string what = msg;
      const auto pos = what.rfind(" (residual ");
      if (pos != std::string::npos) what = what.substr(0, pos);
      throw ConvergenceError(what, rk_last_residual());
    }
    default: throw std::runtime_error(msg);
  }
}

rk_sparse_view view_of(const SparseMatrix& a) {
  rk_sparse_view v;
  v.rows = a.rows();
  v.cols = a.cols();
  v.nnz = a.nnz();
  v.entries = reinterpret_cast<const rk_entry*>(a.entries().data());
  return v;
}

rk_method method_of(RepairMethod m) {
  switch (m) {
    case RepairMethod::kRandom: return RK_RANDOM;
    case RepairMethod::kNeighbor: return RK_NEIGHBOR;
    case RepairMethod::kNeighborRandom: return RK_NEIGHBOR_RANDOM;
    case RepairMethod::kNone: return RK_NONE;
  }
  throw std::invalid_argument("bad repair method");
}

void require_uniform(const BlockPartition& p) {
  const BlockPartition q = partition_columns(p.total_cols(), p.block_count());
  if (!(q == p)) throw std::invalid_argument("the B200 drop-in supports partitions made by partition_columns");
}

DenseMatrix dense_of_rows(uint64_t rows, uint64_t cols, const double* data) {
  return DenseMatrix(rows, cols, std::vector<double>(data, data + rows * cols));
}

SvdResult svd_of(const rk_svd& s) {
  SvdResult r;
  r.u = dense_of_rows(s.u_rows, s.u_cols, s.u);
  r.sigma.assign(s.sigma, s.sigma + s.n_sigma);
  if (s.has_v) r.v = dense_of_rows(s.v_rows, s.v_cols, s.v);
  return r;
}

SparseMatrix sparse_of_rk(const rk_sparse& s) {
  std::vector<Entry> e(s.nnz);
  if (s.nnz) std::memcpy(e.data(), s.entries, s.nnz * sizeof(Entry));
  return SparseMatrix(s.rows, s.cols, std::move(e));
}

RepairReport report_of(const rk_repair_report& r) {
  RepairReport rep;
  rep.added_edges.resize(r.n_edges);
  for (uint64_t i = 0; i < r.n_edges; ++i) {
    rep.added_edges[i].block = r.block[i];
    rep.added_edges[i].row = r.row[i];
    rep.added_edges[i].col = r.col[i];
    rep.added_edges[i].mechanism = r.mechanism[i] ? RepairMethod::kNeighbor : RepairMethod::kRandom;
  }
  rep.lonely_counts.assign(r.lonely_counts, r.lonely_counts + r.n_blocks);
  rep.fallback_count = r.fallback_count;
  return rep;
}

// RepairWorkspace's state lives in a device workspace (rk_workspace_*). The class
// layout is the reference's (repair.hpp:80-86: no destructor hook, no spare member),
// so the handle is kept in a registry keyed by the object's address: created by the
// constructor, replaced when a new workspace is constructed at the same address (the
// old object is then necessarily dead), released at exit. The reference members
// origin_ / partition_ are set as in repair.cpp:52-63; row_cols_ / col_rows_ stay
// empty (the adjacency is on the device). A copied workspace has no handle of its
// own and reports std::logic_error. Each workspace owns its context (any thread may
// use it; calls on one workspace must not overlap, as for the reference object).
// Handles still registered at exit are left to process teardown.
struct WsHandle {
  rk_ctx* ctx = nullptr;
  rk_workspace* ws = nullptr;
};
struct WorkspaceRegistry {
  std::mutex mu;
  std::unordered_map<const void*, WsHandle> map;
};
WorkspaceRegistry& registry() {
  static WorkspaceRegistry* r = new WorkspaceRegistry;  // never destroyed: see above
  return *r;
}
void release(WsHandle& h) {
  rk_workspace_destroy(h.ws);
  rk_ctx_destroy(h.ctx);
  h = WsHandle{};
}
rk_workspace* workspace_of(const void* self) {
  WorkspaceRegistry& r = registry();
  std::lock_guard<std::mutex> lk(r.mu);
  auto it = r.map.find(self);
  if (it == r.map.end())
    throw std::logic_error("RepairWorkspace: no device workspace for this object (copies are not supported)");
  return it->second.ws;
}

}  // namespace

// ---- repair.cpp ------------------------------------------------------------
std::string to_string(RepairMethod method) {
  switch (method) {
    case RepairMethod::kRandom: return "random";
    case RepairMethod::kNeighbor: return "neighbor";
    case RepairMethod::kNeighborRandom: return "neighbor-random";
    case RepairMethod::kNone: return "none";
  }
  throw std::invalid_argument("bad repair method");
}

RepairMethod repair_method_from_string(const std::string& name) {
  if (name == "random") return RepairMethod::kRandom;
  if (name == "neighbor") return RepairMethod::kNeighbor;
  if (name == "neighbor-random") return RepairMethod::kNeighborRandom;
  if (name == "none") return RepairMethod::kNone;
  throw std::invalid_argument("unknown repair method '" + name + "'");
}

std::string RepairReport::to_log() const {
  std::ostringstream out;
  for (const AddedEdge& e : added_edges)
    out << e.block << '\t' << e.row << '\t' << e.col << '\t' << to_string(e.mechanism) << '\n';
  out << "# lonely=";
  for (std::size_t d = 0; d < lonely_counts.size(); ++d) out << (d ? "," : "") << lonely_counts[d];
  out << " fallback=" << fallback_count << '\n';
  return out.str();
}

std::vector<std::size_t> find_lonely_rows(const SparseMatrix& a, const BlockPartition& p, std::size_t d) {
  require_uniform(p);
  if (p.total_cols() != a.cols()) throw std::invalid_argument("partition does not match matrix columns");
  (void)p.range(d);  // out_of_range as the reference
  const rk_sparse_view v = view_of(a);
  std::vector<uint64_t> out(a.rows() ? a.rows() : 1);
  uint64_t n = 0;
  check(rk_find_lonely_rows(context(), &v, p.block_count(), d, out.data(), &n));
  return std::vector<std::size_t>(out.begin(), out.begin() + n);
}

// ---- RepairWorkspace (repair.cpp:52-160) on rk_workspace_* ----------------------
RepairWorkspace::RepairWorkspace(const SparseMatrix& a, const BlockPartition& p) : origin_(&a), partition_(&p) {
  if (p.total_cols() != a.cols()) throw std::invalid_argument("partition does not match matrix columns");
  require_uniform(p);
  const rk_sparse_view v = view_of(a);
  WsHandle h;
  int dev = 0;
  if (const char* e = std::getenv("RANKY_DEVICE")) dev = std::atoi(e);
  check(rk_ctx_create(dev, &h.ctx));
  const rk_status st = rk_workspace_create(h.ctx, &v, p.block_count(), &h.ws);
  if (st != RK_OK) {
    rk_ctx_destroy(h.ctx);
    check(st);  // rk_last_error() still holds the create's message
  }
  WorkspaceRegistry& r = registry();
  std::lock_guard<std::mutex> lk(r.mu);
  auto it = r.map.find(this);
  if (it != r.map.end()) release(it->second);
  r.map[this] = h;
}

void RepairWorkspace::insert(std::size_t row, std::size_t col) { check(rk_workspace_insert(workspace_of(this), row, col)); }

std::size_t RepairWorkspace::apply_random(std::size_t d, std::size_t row, KeyedRng& rng) {
  const ColumnRange& range = partition_->range(d);
  const std::size_t col = range.begin + rng.below(range.width());
  insert(row, col);
  return col;
}

std::optional<std::size_t> RepairWorkspace::apply_neighbor(std::size_t d, std::size_t row, KeyedRng& rng) {
  const ColumnRange& range = partition_->range(d);
  std::vector<uint64_t> cols(range.width() ? range.width() : 1);
  uint64_t n = 0;
  check(rk_workspace_neighbor_columns(workspace_of(this), d, row, cols.data(), &n));
  if (n == 0) return std::nullopt;  // no draw on an empty set (repair.cpp:127)
  const std::size_t col = cols[rng.below(n)];
  insert(row, col);
  return col;
}

std::vector<std::size_t> RepairWorkspace::apply_neighbor_random(std::size_t d, std::size_t row, KeyedRng& rng) {
  std::vector<std::size_t> added;
  if (auto col = apply_neighbor(d, row, rng)) added.push_back(*col);
  const std::size_t random_col = apply_random(d, row, rng);
  if (added.empty() || added.front() != random_col) added.push_back(random_col);
  return added;
}

bool RepairWorkspace::has_entry(std::size_t row, std::size_t col) const {
  int32_t f = 0;
  check(rk_workspace_has_entry(workspace_of(this), row, col, &f));
  return f != 0;
}

bool RepairWorkspace::row_lonely_in_block(std::size_t d, std::size_t row) const {
  int32_t f = 0;
  check(rk_workspace_row_lonely_in_block(workspace_of(this), d, row, &f));
  return f != 0;
}

std::vector<std::size_t> RepairWorkspace::lonely_rows(std::size_t d) const {
  std::vector<uint64_t> rows(origin_->rows() ? origin_->rows() : 1);
  uint64_t n = 0;
  check(rk_workspace_lonely_rows(workspace_of(this), d, rows.data(), &n));
  return std::vector<std::size_t>(rows.begin(), rows.begin() + n);
}

SparseMatrix RepairWorkspace::to_matrix() const {
  rk_sparse rs{};
  const rk_status st = rk_workspace_to_matrix(workspace_of(this), &rs);
  if (st != RK_OK) {
    rk_sparse_free(&rs);
    check(st);
  }
  SparseMatrix m = sparse_of_rk(rs);
  rk_sparse_free(&rs);
  return m;
}

std::pair<SparseMatrix, RepairReport> repair(const SparseMatrix& a, const BlockPartition& p, RepairMethod method,
                                             std::uint64_t seed) {
  if (p.total_cols() != a.cols()) throw std::invalid_argument("partition does not match matrix columns");
  require_uniform(p);
  if (method == RepairMethod::kNone) {  // repair.cpp:167-168: the input unchanged, zero counts
    RepairReport rep;
    rep.lonely_counts.assign(p.block_count(), 0);
    return {a, rep};
  }
  const rk_sparse_view v = view_of(a);
  rk_sparse rs{};
  rk_repair_report rr{};
  const rk_status st = rk_repair(context(), &v, p.block_count(), method_of(method), seed, &rs, &rr);
  if (st != RK_OK) {
    rk_sparse_free(&rs);
    rk_repair_report_free(&rr);
    check(st);
  }
  std::pair<SparseMatrix, RepairReport> out{sparse_of_rk(rs), report_of(rr)};
  rk_sparse_free(&rs);
  rk_repair_report_free(&rr);
  return out;
}

double rank_equal_probability(std::size_t columns, std::size_t single_entry_rows) {
  if (columns == 0) throw std::invalid_argument("column count must be positive");
  if (single_entry_rows >= columns) return 0.0;
  return static_cast<double>(columns - single_entry_rows) / static_cast<double>(columns);
}

// ---- svd.cpp ---------------------------------------------------------------
SvdResult dense_svd(const DenseMatrix& a) {
  rk_svd s{};
  const rk_status st = rk_dense_svd(context(), a.rows(), a.cols(), a.values().data(), &s);
  if (st != RK_OK) {
    rk_svd_free(&s);
    check(st);
  }
  SvdResult r = svd_of(s);
  rk_svd_free(&s);
  return r;
}

SvdResult block_svd(const SparseMatrix& block, std::size_t keep) {
  const rk_sparse_view v = view_of(block);
  rk_svd s{};
  const rk_status st = rk_block_svd(context(), &v, keep, &s);
  if (st != RK_OK) {
    rk_svd_free(&s);
    check(st);
  }
  SvdResult r = svd_of(s);
  r.v.reset();
  rk_svd_free(&s);
  return r;
}

// ---- proxy.cpp -------------------------------------------------------------
ProxyMatrix build_proxy(std::span<const SvdResult> block_results, std::size_t rows) {
  std::size_t total = 0;
  for (const SvdResult& r : block_results) {
    if (r.u.rows() != rows)
      throw std::invalid_argument("build_proxy: block factor has " + std::to_string(r.u.rows()) +
                                  " rows, expected " + std::to_string(rows));
    if (r.u.cols() != r.sigma.size()) throw std::invalid_argument("build_proxy: U column count does not match sigma");
    total += r.sigma.size();
  }
  ProxyMatrix proxy;
  proxy.matrix = DenseMatrix(rows, total);
  std::size_t off = 0;
  for (const SvdResult& r : block_results) {
    proxy.block_offsets.push_back(off);
    for (std::size_t j = 0; j < r.sigma.size(); ++j)
      for (std::size_t i = 0; i < rows; ++i) proxy.matrix(i, off + j) = r.u(i, j) * r.sigma[j];
    off += r.sigma.size();
  }
  proxy.block_offsets.push_back(off);
  return proxy;
}

SvdResult proxy_svd(const ProxyMatrix& proxy) {
  std::vector<uint64_t> offs(proxy.block_offsets.begin(), proxy.block_offsets.end());
  rk_svd s{};
  const rk_status st = rk_proxy_svd(context(), proxy.matrix.rows(), proxy.matrix.cols(),
                                    proxy.matrix.values().data(), offs.size(), offs.data(), &s);
  if (st != RK_OK) {
    rk_svd_free(&s);
    check(st);
  }
  SvdResult r = svd_of(s);
  rk_svd_free(&s);
  return r;
}

DenseMatrix recover_right_vectors(const SparseMatrix& a, const DenseMatrix& u, std::span<const double> sigma,
                                  double tol) {
  const rk_sparse_view v = view_of(a);
  rk_svd s{};
  const rk_status st = rk_recover_right_vectors(context(), &v, u.rows(), u.cols(), u.values().data(), sigma.size(),
                                                sigma.data(), tol, &s);
  if (st != RK_OK) {
    rk_svd_free(&s);
    check(st);
  }
  DenseMatrix out = dense_of_rows(s.v_rows, s.v_cols, s.v);
  rk_svd_free(&s);
  return out;
}

// ---- pipeline.cpp ----------------------------------------------------------
BlockResultRecord run_block_task(const BlockTask& task) {
  const rk_sparse_view v = view_of(task.block);
  rk_records rec{};
  const rk_status st = rk_run_block_tasks(context(), &v, 1, task.keep, &rec);
  if (st != RK_OK) {
    rk_records_free(&rec);
    // the pool wraps the message with the block index; a lone task reports the kernel's error
    const std::string msg = rk_last_error();
    const std::string prefix = "block task 0 failed: ";
    if (st == RK_RUNTIME && msg.rfind(prefix, 0) == 0) {
      const std::string inner = msg.substr(prefix.size());
      if (inner.rfind("one-sided Jacobi", 0) == 0) throw ConvergenceError("one-sided Jacobi did not converge", 0.0);
      throw std::invalid_argument(inner);
    }
    check(st);
  }
  BlockResultRecord r;
  r.block_index = static_cast<std::uint32_t>(task.block_index);
  r.rows = static_cast<std::uint32_t>(rec.rows);
  r.kept = rec.kept[0];
  r.payload.assign(rec.payload, rec.payload + rec.rows * rec.kept[0]);
  rk_records_free(&rec);
  return r;
}

ProxyMatrix proxy_from_records(std::span<const BlockResultRecord> records, std::size_t rows) {
  std::vector<const BlockResultRecord*> ordered;
  for (const BlockResultRecord& r : records) ordered.push_back(&r);
  std::sort(ordered.begin(), ordered.end(),
            [](const BlockResultRecord* a, const BlockResultRecord* b) { return a->block_index < b->block_index; });
  for (std::size_t i = 1; i < ordered.size(); ++i)
    if (ordered[i - 1]->block_index == ordered[i]->block_index)
      throw std::invalid_argument("duplicate block record index " + std::to_string(ordered[i]->block_index));
  std::size_t total = 0;
  for (const BlockResultRecord* r : ordered) {
    if (r->rows != rows)
      throw std::invalid_argument("block record " + std::to_string(r->block_index) + " has " +
                                  std::to_string(r->rows) + " rows, expected " + std::to_string(rows));
    total += r->kept;
  }
  ProxyMatrix proxy;
  proxy.matrix = DenseMatrix(rows, total);
  std::size_t off = 0;
  for (const BlockResultRecord* r : ordered) {
    proxy.block_offsets.push_back(off);
    for (std::size_t i = 0; i < rows; ++i)
      for (std::size_t j = 0; j < r->kept; ++j) proxy.matrix(i, off + j) = r->payload[i * r->kept + j];
    off += r->kept;
  }
  proxy.block_offsets.push_back(off);
  return proxy;
}

// The devices run_pipeline spreads its blocks over: RANKY_DEVICES ("0,1,2,3"; a device
// may repeat). Unset (the default): one device, so results are bitwise the same for
// every `workers` as the reference promises (acceptance_main.cpp:211-250); the sharded
// merge agrees with the single-device one to the parity tolerance, and bitwise across
// shard counts whose leaves / shards is a power of two.
std::vector<int32_t> pipeline_devices() {
  std::vector<int32_t> d;
  if (const char* e = std::getenv("RANKY_DEVICES")) {
    std::string s(e);
    std::size_t pos = 0;
    while (pos < s.size()) {
      const std::size_t comma = s.find(',', pos);
      const std::string tok = s.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
      if (!tok.empty()) d.push_back(std::atoi(tok.c_str()));
      if (comma == std::string::npos) break;
      pos = comma + 1;
    }
  }
  return d;
}

struct ThreadMulti {
  std::vector<int32_t> devices;
  rk_multi* m = nullptr;
  ~ThreadMulti() {
    if (m) rk_multi_destroy(m);
  }
};

rk_multi* multi_for(const std::vector<int32_t>& devices) {
  thread_local ThreadMulti tm;
  if (!tm.m || tm.devices != devices) {
    if (tm.m) rk_multi_destroy(tm.m);
    tm.m = nullptr;
    check(rk_multi_create(devices.data(), (uint32_t)devices.size(), &tm.m));
    tm.devices = devices;
  }
  return tm.m;
}

PipelineResult run_pipeline(const SparseMatrix& a, std::size_t block_count, RepairMethod method, std::size_t keep,
                            std::uint64_t seed, std::size_t workers) {
  if (workers == 0) throw std::invalid_argument("workers must be >= 1");
  const rk_sparse_view v = view_of(a);
  rk_pipeline_result pr{};
  const std::vector<int32_t> devices = pipeline_devices();
  const uint64_t leaves = rk_merge_tree_leaves(a.rows(), a.cols(), block_count, keep);
  const bool multi = devices.size() > 1 && leaves >= devices.size();
  const rk_status st = multi ? rk_multi_run_pipeline(multi_for(devices), &v, block_count, method_of(method), keep,
                                                     seed, RK_WANT_REPAIRED | RK_WANT_RECORDS, 0, &pr)
                             : rk_run_pipeline(context(), &v, block_count, method_of(method), keep, seed, workers,
                                               RK_WANT_REPAIRED | RK_WANT_RECORDS, 0, &pr);
  if (st != RK_OK) {
    rk_pipeline_result_free(&pr);
    check(st);
  }
  PipelineResult out;
  out.svd = svd_of(pr.svd);
  out.svd.v.reset();  // right vectors are not part of the distributed result (pipeline.cpp:112)
  out.report = report_of(pr.report);
  out.repaired = sparse_of_rk(pr.repaired);
  out.partition = partition_columns(a.cols(), block_count);
  out.records.resize(pr.records.n_records);
  for (uint64_t d = 0; d < pr.records.n_records; ++d) {
    BlockResultRecord& r = out.records[d];
    r.block_index = static_cast<std::uint32_t>(d);
    r.rows = static_cast<std::uint32_t>(pr.records.rows);
    r.kept = pr.records.kept[d];
    const double* p = pr.records.payload + pr.records.offset[d];
    r.payload.assign(p, p + pr.records.rows * r.kept);
  }
  rk_pipeline_result_free(&pr);
  return out;
}

}  // namespace ranky
