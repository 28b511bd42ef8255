// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI wrapper around the *unmodified* reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It exposes
// the same or_result record as the C restatement so tests can run both
// oracles -- and the CUDA path -- on identical inputs. It adds no arithmetic
// of its own: every number comes from the reference routines named below.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <thread>
#include <exception>
#include <stdexcept>
#include <vector>

#include "or_result.h"
#include "ranky/block_record.hpp"
#include "ranky/dense_matrix.hpp"
#include "ranky/errors.hpp"
#include "ranky/matrix_market.hpp"
#include "ranky/metrics.hpp"
#include "ranky/partition.hpp"
#include "ranky/pipeline.hpp"
#include "ranky/proxy.hpp"
#include "ranky/repair.hpp"
#include "ranky/rng.hpp"
#include "ranky/sparse_matrix.hpp"
#include "ranky/svd.hpp"
#include "ranky/synth.hpp"

using namespace ranky;

namespace {

or_result* fresh() { return static_cast<or_result*>(std::calloc(1, sizeof(or_result))); }

template <class T>
T* copy_out(const T* src, std::size_t n) {
  T* dst = static_cast<T*>(std::malloc((n ? n : 1) * sizeof(T)));
  if (n) std::memcpy(dst, src, n * sizeof(T));
  return dst;
}

void fail(or_result* res, int code, const char* what) {
  res->status = code;
  std::snprintf(res->message, sizeof res->message, "%s", what);
}

// map C++ exceptions to the shared status codes
template <class F>
or_result* guarded(F&& body) {
  or_result* res = fresh();
  try {
    body(res);
  } catch (const ConvergenceError& e) {
    res->residual = e.residual();
    fail(res, OR_CONVERGE, e.what());
  } catch (const std::invalid_argument& e) {
    fail(res, OR_INVALID, e.what());
  } catch (const std::out_of_range& e) {
    fail(res, OR_RANGE, e.what());
  } catch (const std::exception& e) {
    fail(res, OR_RUNTIME, e.what());
  }
  return res;
}

SparseMatrix make_sparse(uint64_t rows, uint64_t cols, uint64_t nnz, const uint64_t* r,
                         const uint64_t* c, const double* v) {
  std::vector<Entry> entries(nnz);
  for (uint64_t i = 0; i < nnz; ++i) entries[i] = {r[i], c[i], v[i]};
  return SparseMatrix(rows, cols, std::move(entries));
}

void put_sparse(or_result* res, const SparseMatrix& m) {
  res->rows = m.rows();
  res->cols = m.cols();
  res->nnz = m.nnz();
  res->r = static_cast<uint64_t*>(std::malloc((m.nnz() ? m.nnz() : 1) * 8));
  res->c = static_cast<uint64_t*>(std::malloc((m.nnz() ? m.nnz() : 1) * 8));
  res->v = static_cast<double*>(std::malloc((m.nnz() ? m.nnz() : 1) * 8));
  std::size_t i = 0;
  for (const Entry& e : m.entries()) {
    res->r[i] = e.row;
    res->c[i] = e.col;
    res->v[i] = e.value;
    ++i;
  }
}

void put_report(or_result* res, const RepairReport& rep) {
  const std::size_t n = rep.added_edges.size();
  res->n_edges = n;
  res->e_block = static_cast<uint64_t*>(std::malloc((n ? n : 1) * 8));
  res->e_row = static_cast<uint64_t*>(std::malloc((n ? n : 1) * 8));
  res->e_col = static_cast<uint64_t*>(std::malloc((n ? n : 1) * 8));
  res->e_mech = static_cast<int32_t*>(std::malloc((n ? n : 1) * 4));
  for (std::size_t i = 0; i < n; ++i) {
    res->e_block[i] = rep.added_edges[i].block;
    res->e_row[i] = rep.added_edges[i].row;
    res->e_col[i] = rep.added_edges[i].col;
    res->e_mech[i] = rep.added_edges[i].mechanism == RepairMethod::kNeighbor ? 1 : 0;
  }
  res->n_blocks = rep.lonely_counts.size();
  std::vector<uint64_t> lc(rep.lonely_counts.begin(), rep.lonely_counts.end());
  res->lonely = copy_out(lc.data(), lc.size());
  res->fallback = rep.fallback_count;
}

void put_svd(or_result* res, const SvdResult& s) {
  res->u_rows = s.u.rows();
  res->u_cols = s.u.cols();
  res->u = copy_out(s.u.values().data(), s.u.values().size());
  res->n_sigma = s.sigma.size();
  res->sigma = copy_out(s.sigma.data(), s.sigma.size());
  res->has_v = s.v.has_value();
  if (s.v) {
    res->v_rows = s.v->rows();
    res->v_cols = s.v->cols();
    res->vm = copy_out(s.v->values().data(), s.v->values().size());
  }
}

RepairMethod method_of(int m) {
  switch (m) {
    case 0: return RepairMethod::kRandom;
    case 1: return RepairMethod::kNeighbor;
    case 2: return RepairMethod::kNeighborRandom;
    default: return RepairMethod::kNone;
  }
}

}  // namespace

extern "C" {

void ref_free(or_result* res) {
  if (!res) return;
  std::free(res->e_block); std::free(res->e_row); std::free(res->e_col); std::free(res->e_mech);
  std::free(res->lonely); std::free(res->r); std::free(res->c); std::free(res->v);
  std::free(res->u); std::free(res->sigma); std::free(res->vm);
  std::free(res->rec_kept); std::free(res->rec_payload);
  std::free(res);
}

void ref_rng_stream(uint64_t seed, uint64_t block, uint64_t row, uint64_t n, uint64_t* out) {
  KeyedRng g(seed, block, row);
  for (uint64_t i = 0; i < n; ++i) out[i] = g.next();
}

uint64_t ref_rng_below(uint64_t seed, uint64_t block, uint64_t row, uint64_t bound) {
  KeyedRng g(seed, block, row);
  return g.below(bound);
}

// synth_bipartite -- proj/src/synth.cpp:14-29
or_result* ref_synth_bipartite(uint64_t rows, uint64_t cols, double density, uint64_t seed) {
  return guarded([&](or_result* res) { put_sparse(res, synth_bipartite(rows, cols, density, seed)); });
}

// repair -- proj/src/repair.cpp:162-216
or_result* ref_repair(uint64_t rows, uint64_t cols, uint64_t nnz, const uint64_t* r,
                      const uint64_t* c, const double* v, uint64_t D, int method, uint64_t seed) {
  return guarded([&](or_result* res) {
    SparseMatrix a = make_sparse(rows, cols, nnz, r, c, v);
    BlockPartition p = partition_columns(cols, D);
    auto [repaired, report] = repair(a, p, method_of(method), seed);
    put_sparse(res, repaired);
    put_report(res, report);
  });
}

// find_lonely_rows -- proj/src/repair.cpp:42-50
uint64_t ref_find_lonely_rows(uint64_t rows, uint64_t cols, uint64_t nnz, const uint64_t* r,
                              const uint64_t* c, uint64_t D, uint64_t d, uint64_t* out) {
  std::vector<double> ones(nnz, 1.0);
  SparseMatrix a = make_sparse(rows, cols, nnz, r, c, ones.data());
  BlockPartition p = partition_columns(cols, D);
  auto lonely = find_lonely_rows(a, p, d);
  for (std::size_t i = 0; i < lonely.size(); ++i) out[i] = lonely[i];
  return lonely.size();
}

// dense_svd -- proj/src/svd.cpp:365-379
or_result* ref_dense_svd(uint64_t rows, uint64_t cols, const double* a) {
  return guarded([&](or_result* res) {
    DenseMatrix m(rows, cols, std::vector<double>(a, a + rows * cols));
    put_svd(res, dense_svd(m));
  });
}

// block_svd -- proj/src/svd.cpp:381-400
or_result* ref_block_svd(uint64_t rows, uint64_t cols, uint64_t nnz, const uint64_t* r,
                         const uint64_t* c, const double* v, uint64_t keep) {
  return guarded([&](or_result* res) {
    put_svd(res, block_svd(make_sparse(rows, cols, nnz, r, c, v), keep));
  });
}

// recover_right_vectors -- proj/src/proxy.cpp:48-72
or_result* ref_recover_right_vectors(uint64_t rows, uint64_t cols, uint64_t nnz, const uint64_t* r,
                                     const uint64_t* c, const double* v, const double* u,
                                     uint64_t u_rows, uint64_t u_cols, const double* sigma,
                                     uint64_t n_sigma, double tol) {
  return guarded([&](or_result* res) {
    SparseMatrix a = make_sparse(rows, cols, nnz, r, c, v);
    DenseMatrix um(u_rows, u_cols, std::vector<double>(u, u + u_rows * u_cols));
    DenseMatrix vm = recover_right_vectors(a, um, std::span<const double>(sigma, n_sigma), tol);
    res->has_v = 1;
    res->v_rows = vm.rows();
    res->v_cols = vm.cols();
    res->vm = copy_out(vm.values().data(), vm.values().size());
  });
}

// proxy_svd over records -- proj/src/pipeline.cpp:18-59 + proj/src/proxy.cpp:40-46
or_result* ref_proxy_svd_records(uint64_t rows, uint64_t n_records, const uint32_t* kept,
                                 const double* payload) {
  return guarded([&](or_result* res) {
    std::vector<BlockResultRecord> recs(n_records);
    std::size_t off = 0;
    for (uint64_t d = 0; d < n_records; ++d) {
      recs[d].block_index = static_cast<uint32_t>(d);
      recs[d].rows = static_cast<uint32_t>(rows);
      recs[d].kept = kept[d];
      recs[d].payload.assign(payload + off, payload + off + rows * kept[d]);
      off += rows * kept[d];
    }
    put_svd(res, proxy_svd(proxy_from_records(recs, rows)));
  });
}

// run_pipeline -- proj/src/pipeline.cpp:61-121; t_* fields carry the wall time
// of the whole call in t_blocks (the reference exposes no finer breakdown)
or_result* ref_run_pipeline(uint64_t rows, uint64_t cols, uint64_t nnz, const uint64_t* r,
                            const uint64_t* c, const double* v, uint64_t D, int method,
                            uint64_t keep, uint64_t seed, uint64_t workers) {
  return guarded([&](or_result* res) {
    SparseMatrix a = make_sparse(rows, cols, nnz, r, c, v);
    const auto t0 = std::chrono::steady_clock::now();
    PipelineResult pr = run_pipeline(a, D, method_of(method), keep, seed, workers);
    const auto t1 = std::chrono::steady_clock::now();
    res->t_blocks = std::chrono::duration<double>(t1 - t0).count();
    put_svd(res, pr.svd);
    put_report(res, pr.report);
    put_sparse(res, pr.repaired);
    res->n_records = pr.records.size();
    std::vector<uint32_t> kept(pr.records.size());
    std::size_t total = 0;
    for (std::size_t d = 0; d < pr.records.size(); ++d) {
      kept[d] = pr.records[d].kept;
      total += pr.records[d].payload.size();
    }
    res->rec_kept = copy_out(kept.data(), kept.size());
    res->rec_payload = static_cast<double*>(std::malloc((total ? total : 1) * 8));
    std::size_t off = 0;
    for (const auto& rec : pr.records) {
      std::memcpy(res->rec_payload + off, rec.payload.data(), rec.payload.size() * 8);
      off += rec.payload.size();
    }
  });
}

// run_pipeline + recover_right_vectors(repaired, U, sigma, kRankTol): the
// "full Ranky SVD" the benchmark times. Fills vm with V.
or_result* ref_full_svd(uint64_t rows, uint64_t cols, uint64_t nnz, const uint64_t* r,
                        const uint64_t* c, const double* v, uint64_t D, int method,
                        uint64_t keep, uint64_t seed, uint64_t workers, uint64_t top_k) {
  return guarded([&](or_result* res) {
    SparseMatrix a = make_sparse(rows, cols, nnz, r, c, v);
    const auto t0 = std::chrono::steady_clock::now();
    PipelineResult pr = run_pipeline(a, D, method_of(method), keep, seed, workers);
    const auto t1 = std::chrono::steady_clock::now();
    std::size_t k = pr.svd.sigma.size();
    if (top_k && top_k < k) k = top_k;
    DenseMatrix uk(pr.svd.u.rows(), k);
    for (std::size_t i = 0; i < uk.rows(); ++i)
      for (std::size_t j = 0; j < k; ++j) uk(i, j) = pr.svd.u(i, j);
    DenseMatrix vm = recover_right_vectors(pr.repaired, uk,
                                           std::span<const double>(pr.svd.sigma.data(), k), kRankTol);
    const auto t2 = std::chrono::steady_clock::now();
    res->t_blocks = std::chrono::duration<double>(t1 - t0).count();
    res->t_proxy = std::chrono::duration<double>(t2 - t1).count();
    put_svd(res, pr.svd);
    res->has_v = 1;
    res->v_rows = vm.rows();
    res->v_cols = vm.cols();
    res->vm = copy_out(vm.values().data(), vm.values().size());
  });
}

// crc32 / write_block_record -- proj/src/block_record.cpp:53-106
uint32_t ref_crc32(const void* data, uint64_t size) { return crc32(data, size); }

int ref_write_block_record(uint32_t index, uint32_t rows, uint32_t kept, const double* payload, const char* path) {
  try {
    BlockResultRecord r;
    r.block_index = index;
    r.rows = rows;
    r.kept = kept;
    r.payload.assign(payload, payload + (uint64_t)rows * kept);
    write_block_record(r, path);
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

// read_block_record: 0 ok (payload copied into out, rows*kept doubles), 1 RecordError, 2 other
int ref_read_block_record(const char* path, uint32_t* index, uint32_t* rows, uint32_t* kept, double* out,
                          uint64_t cap) {
  try {
    BlockResultRecord r = read_block_record(path);
    *index = r.block_index;
    *rows = r.rows;
    *kept = r.kept;
    for (uint64_t i = 0; i < r.payload.size() && i < cap; ++i) out[i] = r.payload[i];
    return 0;
  } catch (const RecordError&) {
    return 1;
  } catch (const std::exception&) {
    return 2;
  }
}

// ---- Matrix Market -- proj/src/matrix_market.cpp:38-132 ----
// load: res->matrix on success; status 6 (a ParseError) + message "... (line L)" and
// residual = L. (save: oracle/ref_mm_save.cpp, a separate process.)
or_result* ref_load_matrix_market(const char* path) {
  or_result* res = fresh();
  try {
    put_sparse(res, load_matrix_market(path));
  } catch (const ParseError& e) {
    res->residual = (double)e.line();
    fail(res, 6, e.what());
  } catch (const std::exception& e) {
    fail(res, OR_RUNTIME, e.what());
  }
  return res;
}
// ---- evaluation metrics -- proj/src/metrics.cpp:32-114 ----
double ref_sigma_error(const double* a, uint64_t na, const double* b, uint64_t nb) {
  return sigma_error(std::span<const double>(a, na), std::span<const double>(b, nb));
}
int ref_align_signs(const double* hat, const double* ref, uint64_t rows, uint64_t cols, const double* sigma,
                    uint64_t n_sigma, double* out) {
  try {
    DenseMatrix h(rows, cols, std::vector<double>(hat, hat + rows * cols));
    DenseMatrix r(rows, cols, std::vector<double>(ref, ref + rows * cols));
    DenseMatrix o = align_signs(h, r, std::span<const double>(sigma, n_sigma));
    std::memcpy(out, o.values().data(), rows * cols * sizeof(double));
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}
double ref_left_vector_error(const double* hat, const double* ref, uint64_t rows, uint64_t cols,
                             const double* sigma, uint64_t n_sigma) {
  DenseMatrix h(rows, cols, std::vector<double>(hat, hat + rows * cols));
  DenseMatrix r(rows, cols, std::vector<double>(ref, ref + rows * cols));
  return left_vector_error(h, r, std::span<const double>(sigma, n_sigma));
}
uint64_t ref_numerical_rank(const double* a, uint64_t rows, uint64_t cols, double tol) {
  return numerical_rank(DenseMatrix(rows, cols, std::vector<double>(a, a + rows * cols)), tol);
}

// ---- the reference arm's bounded sample (bench.py --impl reference) ----------
// run_pipeline (proj/src/pipeline.cpp:61-121) + recover_right_vectors
// (proj/src/proxy.cpp:48-72) are serial except the block-task pool, so their
// time is the sum of the stages below. Each stage calls the reference's own
// functions and is timed here with std::chrono around those calls only (no
// marshalling inside the timed regions). phase selects what runs:
//   phase & 1: repair in full (pipeline.cpp:70) ............ t[0]
//   phase & 2: block_view of the n sampled blocks .......... t[1]  (pipeline.cpp:73-75)
//              run_block_task over them on min(workers, n) threads pulling from an
//              atomic, as pipeline.cpp:79-101 does ........ t[2]
//   phase & 4: proxy_from_records + proxy_svd on the first n/2 and on all n
//              sampled records (proj/src/pipeline.cpp:18-59, proxy.cpp:40-46) ... t[3], t[4]
//              recover_right_vectors of the repaired matrix's first slice_cols
//              columns with that proxy's U, sigma ............................... t[5]
// t[6] = sum of the kept sigma count of the full-n proxy (its Σk), t[7] = the n/2 one's.
int ref_sampled_pipeline(uint64_t rows, uint64_t cols, uint64_t nnz, const uint64_t* r, const uint64_t* c,
                         const double* v, uint64_t D, int method, uint64_t keep, uint64_t seed, uint64_t workers,
                         const uint64_t* sample, uint64_t n, uint64_t slice_cols, int phase, double* t) {
  using clk = std::chrono::steady_clock;
  auto secs = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); };
  try {
    SparseMatrix a = make_sparse(rows, cols, nnz, r, c, v);
    BlockPartition p = partition_columns(a.cols(), D);
    auto t0 = clk::now();
    auto [repaired, report] = repair(a, p, method_of(method), seed);
    auto t1 = clk::now();
    if (phase & 1) t[0] = secs(t0, t1);
    if (!(phase & 6)) return 0;
    std::vector<BlockTask> tasks;
    t0 = clk::now();
    for (uint64_t i = 0; i < n; ++i) tasks.push_back({sample[i], block_view(repaired, p, sample[i]), keep});
    t1 = clk::now();
    t[1] = secs(t0, t1);
    std::vector<BlockResultRecord> recs(n);
    std::atomic<std::size_t> next{0};
    auto loop = [&] {
      for (;;) {
        const std::size_t i = next.fetch_add(1);
        if (i >= n) return;
        recs[i] = run_block_task(tasks[i]);
      }
    };
    const std::size_t pool = std::min<uint64_t>(workers, n);
    t0 = clk::now();
    {
      std::vector<std::thread> th;
      for (std::size_t i = 0; i < pool; ++i) th.emplace_back(loop);
      for (auto& x : th) x.join();
    }
    t1 = clk::now();
    t[2] = secs(t0, t1);
    if (!(phase & 4)) return 0;
    for (std::size_t i = 0; i < n; ++i) recs[i].block_index = static_cast<uint32_t>(i);
    const std::size_t half = std::max<std::size_t>(1, n / 2);
    double sk_half = 0, sk_all = 0;
    for (std::size_t i = 0; i < n; ++i) (i < half ? sk_half : sk_all) += recs[i].kept;
    sk_all += sk_half;
    t0 = clk::now();
    SvdResult s_half = proxy_svd(proxy_from_records(std::span<const BlockResultRecord>(recs.data(), half), rows));
    t1 = clk::now();
    t[4] = secs(t0, t1);
    t0 = clk::now();
    SvdResult s_all = proxy_svd(proxy_from_records(recs, rows));
    t1 = clk::now();
    t[3] = secs(t0, t1);
    t[6] = sk_all;
    t[7] = sk_half;
    const uint64_t sc = std::min<uint64_t>(slice_cols, cols);
    std::vector<Entry> es;
    for (const Entry& e : repaired.entries())
      if (e.col < sc) es.push_back(e);
    SparseMatrix slice(rows, sc, std::move(es));
    t0 = clk::now();
    DenseMatrix vm = recover_right_vectors(slice, s_all.u, s_all.sigma, kRankTol);
    t1 = clk::now();
    t[5] = secs(t0, t1);
    return vm.rows() == sc ? 0 : 1;
  } catch (const std::exception&) {
    return 2;
  }
}

}  // extern "C"
