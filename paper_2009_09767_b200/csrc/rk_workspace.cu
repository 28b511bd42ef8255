// rk_workspace.cu -- RepairWorkspace's single-row API on the device
// (proj/include/ranky/repair.hpp:56-87, proj/src/repair.cpp:52-160).
//
// The reference keeps a mutable CSR (row_cols_) and CSC (col_rows_) adjacency and
// inserts each repair edge into both. Here the workspace is the matrix's device
// CSR + CSC (immutable, as uploaded) plus an overlay of the inserted edges; every
// query sees base + overlay:
//
//   has_entry / row_lonely_in_block   binary search in the row's CSR segment + overlay scan
//   lonely_rows(d)                    one thread per row, flags compacted in row order
//   neighbor_columns(d, row)          the NeighborChecker's candidate set before the draw
//                                     (repair.cpp:107-130): candidate rows share a column
//                                     with `row` outside block d (the row itself included);
//                                     their columns inside block d, ascending, distinct.
//                                     Two bitmap passes (rows, then block columns) and an
//                                     ordered compaction -- the sort + unique of the reference.
//   insert(row, col)                  idempotent (repair.cpp:85-93): appended when absent
//   to_matrix()                       apply_edges: the base entries keep their values, the
//                                     inserted ones are 1.0 (repair.cpp:147-160)
//
// The draw itself (KeyedRng::below on the caller's generator) stays with the caller,
// exactly where the reference makes it: apply_neighbor = neighbor_columns, then
// cols[rng.below(n)] when n > 0 (no draw on an empty set), then insert.
#include <algorithm>
#include <memory>

#include "rk_internal.cuh"

namespace rk {
namespace {

constexpr int kWT = 256;

__device__ bool csr_has(const uint64_t* ptr, const uint32_t* idx, uint32_t row, uint32_t col) {
  uint64_t lo = ptr[row], hi = ptr[row + 1];
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (idx[mid] < col) lo = mid + 1; else hi = mid;
  }
  return lo < ptr[row + 1] && idx[lo] == col;
}

// any base entry of `row` in [b, e)
__device__ bool csr_any_in(const uint64_t* ptr, const uint32_t* idx, uint32_t row, uint32_t b, uint32_t e) {
  uint64_t lo = ptr[row], hi = ptr[row + 1];
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (idx[mid] < b) lo = mid + 1; else hi = mid;
  }
  return lo < ptr[row + 1] && idx[lo] < e;
}

__global__ void ws_has_entry(const uint64_t* ptr, const uint32_t* idx, const uint32_t* er, const uint32_t* ec,
                             uint64_t ne, uint32_t row, uint32_t col, int32_t* out) {
  if (blockIdx.x || threadIdx.x) return;
  bool f = csr_has(ptr, idx, row, col);
  for (uint64_t i = 0; i < ne && !f; ++i) f = er[i] == row && ec[i] == col;
  *out = f ? 1 : 0;
}

// flags[r] = 1 when row r has no entry (base or inserted) in [b, e)
__global__ void ws_lonely_flags(const uint64_t* ptr, const uint32_t* idx, const uint32_t* er, const uint32_t* ec,
                                uint64_t ne, uint32_t rows, uint32_t b, uint32_t e, uint32_t r_lo, uint32_t r_hi,
                                uint8_t* flags) {
  const uint64_t r = r_lo + blockIdx.x * (uint64_t)kWT + threadIdx.x;
  if (r >= r_hi) return;
  bool has = csr_any_in(ptr, idx, (uint32_t)r, b, e);
  for (uint64_t i = 0; i < ne && !has; ++i) has = er[i] == r && ec[i] >= b && ec[i] < e;
  flags[r - r_lo] = has ? 0 : 1;
}

__device__ __forceinline__ void set_bit(uint32_t* bits, uint32_t i) { atomicOr(&bits[i >> 5], 1u << (i & 31)); }
__device__ __forceinline__ bool get_bit(const uint32_t* bits, uint32_t i) { return (bits[i >> 5] >> (i & 31)) & 1u; }

// mark the rows of column c (base CSC + overlay) as candidates
__device__ void mark_column_rows(const uint64_t* cptr, const uint32_t* cidx, const uint32_t* er, const uint32_t* ec,
                                 uint64_t ne, uint32_t c, uint32_t* cand) {
  for (uint64_t k = cptr[c]; k < cptr[c + 1]; ++k) set_bit(cand, cidx[k]);
  for (uint64_t i = 0; i < ne; ++i)
    if (ec[i] == c) set_bit(cand, er[i]);
}

// candidates: rows sharing a column with `row` outside [b, e) (repair.cpp:108-114)
__global__ void ws_candidates(const uint64_t* ptr, const uint32_t* idx, const uint64_t* cptr, const uint32_t* cidx,
                              const uint32_t* er, const uint32_t* ec, uint64_t ne, uint32_t row, uint32_t b,
                              uint32_t e, uint32_t* cand) {
  const uint64_t n_base = ptr[row + 1] - ptr[row];
  for (uint64_t t = blockIdx.x * (uint64_t)kWT + threadIdx.x; t < n_base + ne; t += (uint64_t)gridDim.x * kWT) {
    uint32_t c;
    if (t < n_base) {
      c = idx[ptr[row] + t];
    } else {
      const uint64_t i = t - n_base;
      if (er[i] != row) continue;
      c = ec[i];
    }
    if (c >= b && c < e) continue;
    mark_column_rows(cptr, cidx, er, ec, ne, c, cand);
  }
}

// neighbor columns: candidates' columns inside [b, e) (repair.cpp:116-125), as bits over the block
__global__ void ws_block_columns(const uint64_t* ptr, const uint32_t* idx, const uint32_t* er, const uint32_t* ec,
                                 uint64_t ne, uint32_t rows, const uint32_t* cand, uint32_t b, uint32_t e,
                                 uint32_t* colbits) {
  const uint64_t m = blockIdx.x * (uint64_t)kWT + threadIdx.x;
  if (m >= rows || !get_bit(cand, (uint32_t)m)) return;
  uint64_t lo = ptr[m], hi = ptr[m + 1];
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (idx[mid] < b) lo = mid + 1; else hi = mid;
  }
  for (uint64_t k = lo; k < ptr[m + 1] && idx[k] < e; ++k) set_bit(colbits, idx[k] - b);
  for (uint64_t i = 0; i < ne; ++i)
    if (er[i] == m && ec[i] >= b && ec[i] < e) set_bit(colbits, ec[i] - b);
}

// ascending compaction of set bits (one CTA): out[rank] = b + bit index
__global__ void ws_compact_bits(const uint32_t* bits, uint32_t n_words, uint32_t base, uint64_t* out,
                                uint64_t* n_out) {
  __shared__ uint32_t s_run;
  if (threadIdx.x == 0) s_run = 0;
  __syncthreads();
  for (uint32_t w0 = 0; w0 < n_words; w0 += blockDim.x) {
    const uint32_t w = w0 + threadIdx.x;
    const uint32_t word = w < n_words ? bits[w] : 0u;
    const uint32_t cnt = __popc(word);
    // block-wide exclusive scan of cnt (warp scans + warp totals)
    uint32_t x = cnt;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    __shared__ uint32_t s_warp[32];
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint32_t v = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      s_warp[lane] = v;
    }
    __syncthreads();
    const uint32_t excl = s_run + (warp ? s_warp[warp - 1] : 0u) + x - cnt;
    uint32_t pos = excl, wd = word;
    while (wd) {
      const int bit = __ffs(wd) - 1;
      out[pos++] = (uint64_t)base + (uint64_t)w * 32 + bit;
      wd &= wd - 1;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) s_run += s_warp[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_out = s_run;
}

}  // namespace

struct Workspace {
  Ctx* c = nullptr;
  DevMatrix base;
  Partition p;
  uint64_t n_edges = 0, cap = 0;
  DBuf<uint32_t> er, ec;  // inserted edges (row, col), insertion order
};

Workspace* workspace_create(Ctx& c, const rk_sparse_view& a, uint64_t block_count) {
  auto w = std::make_unique<Workspace>();
  w->c = &c;
  w->p = make_partition(a.cols, block_count);
  upload_entries(a, w->base, c.stream);
  w->cap = 64;
  w->er.alloc(w->cap, c.stream);
  w->ec.alloc(w->cap, c.stream);
  sync(c.stream);
  return w.release();
}

void workspace_destroy(Workspace* w) { delete w; }

namespace {
void check_rc(const Workspace& w, uint64_t row, uint64_t col) {
  if (row >= w.base.csr.rows || col >= w.base.csr.cols)
    fail(RK_OUT_OF_RANGE, "entry (" + std::to_string(row) + ", " + std::to_string(col) + ") outside the matrix");
}
}  // namespace

bool workspace_has_entry(Workspace& w, uint64_t row, uint64_t col) {
  check_rc(w, row, col);
  cudaStream_t s = w.c->stream;
  DBuf<int32_t> f(1, s);
  ws_has_entry<<<1, 32, 0, s>>>(w.base.csr.ptr.get(), w.base.csr.idx.get(), w.er.get(), w.ec.get(), w.n_edges,
                                (uint32_t)row, (uint32_t)col, f.get());
  RK_LAUNCH_CHECK();
  int32_t h = 0;
  RK_CUDA_CHECK(cudaMemcpyAsync(&h, f.get(), sizeof h, cudaMemcpyDeviceToHost, s));
  sync(s);
  return h != 0;
}

void workspace_lonely(Workspace& w, uint64_t d, uint64_t r_lo, uint64_t r_hi, std::vector<uint64_t>& out) {
  if (d >= w.p.blocks) fail(RK_OUT_OF_RANGE, "block index " + std::to_string(d) + " out of range");
  cudaStream_t s = w.c->stream;
  out.clear();
  if (r_lo >= w.base.csr.rows && r_hi == r_lo + 1) fail(RK_OUT_OF_RANGE, "row " + std::to_string(r_lo));
  r_hi = std::min<uint64_t>(r_hi, w.base.csr.rows);
  if (r_hi <= r_lo) return;
  DBuf<uint8_t> flags(r_hi - r_lo, s);
  ws_lonely_flags<<<(unsigned)ceil_div(r_hi - r_lo, kWT), kWT, 0, s>>>(
      w.base.csr.ptr.get(), w.base.csr.idx.get(), w.er.get(), w.ec.get(), w.n_edges, (uint32_t)w.base.csr.rows,
      (uint32_t)w.p.begin(d), (uint32_t)w.p.end(d), (uint32_t)r_lo, (uint32_t)r_hi, flags.get());
  RK_LAUNCH_CHECK();
  std::vector<uint8_t> h;
  to_host(h, flags.get(), r_hi - r_lo, s);
  sync(s);
  for (uint64_t i = 0; i < h.size(); ++i)
    if (h[i]) out.push_back(r_lo + i);
}

void workspace_neighbor_columns(Workspace& w, uint64_t d, uint64_t row, std::vector<uint64_t>& out) {
  if (d >= w.p.blocks) fail(RK_OUT_OF_RANGE, "block index " + std::to_string(d) + " out of range");
  if (row >= w.base.csr.rows) fail(RK_OUT_OF_RANGE, "row " + std::to_string(row));
  cudaStream_t s = w.c->stream;
  const uint32_t rows = (uint32_t)w.base.csr.rows, b = (uint32_t)w.p.begin(d), e = (uint32_t)w.p.end(d);
  const uint32_t rw = (uint32_t)ceil_div(rows, 32), cw = (uint32_t)ceil_div(e - b, 32);
  DBuf<uint32_t> bits((uint64_t)rw + cw, s);
  bits.zero();
  uint32_t* cand = bits.get();
  uint32_t* colbits = bits.get() + rw;
  ws_candidates<<<64, kWT, 0, s>>>(w.base.csr.ptr.get(), w.base.csr.idx.get(), w.base.csc.ptr.get(),
                                   w.base.csc.idx.get(), w.er.get(), w.ec.get(), w.n_edges, (uint32_t)row, b, e, cand);
  RK_LAUNCH_CHECK();
  ws_block_columns<<<(unsigned)ceil_div(rows, kWT), kWT, 0, s>>>(w.base.csr.ptr.get(), w.base.csr.idx.get(),
                                                                  w.er.get(), w.ec.get(), w.n_edges, rows, cand, b, e,
                                                                  colbits);
  RK_LAUNCH_CHECK();
  DBuf<uint64_t> cols((uint64_t)(e - b) + 1, s);
  ws_compact_bits<<<1, 1024, 0, s>>>(colbits, cw, b, cols.get(), cols.get() + (e - b));
  RK_LAUNCH_CHECK();
  uint64_t n = 0;
  RK_CUDA_CHECK(cudaMemcpyAsync(&n, cols.get() + (e - b), sizeof n, cudaMemcpyDeviceToHost, s));
  sync(s);
  to_host(out, cols.get(), n, s);
  sync(s);
}

void workspace_insert(Workspace& w, uint64_t row, uint64_t col) {
  if (workspace_has_entry(w, row, col)) return;  // idempotent (repair.cpp:85-93)
  cudaStream_t s = w.c->stream;
  if (w.n_edges == w.cap) {
    const uint64_t nc = w.cap * 2;
    DBuf<uint32_t> r2(nc, s), c2(nc, s);
    RK_CUDA_CHECK(cudaMemcpyAsync(r2.get(), w.er.get(), w.n_edges * 4, cudaMemcpyDeviceToDevice, s));
    RK_CUDA_CHECK(cudaMemcpyAsync(c2.get(), w.ec.get(), w.n_edges * 4, cudaMemcpyDeviceToDevice, s));
    w.er = std::move(r2);
    w.ec = std::move(c2);
    w.cap = nc;
  }
  const uint32_t r = (uint32_t)row, c = (uint32_t)col;
  RK_CUDA_CHECK(cudaMemcpyAsync(w.er.get() + w.n_edges, &r, 4, cudaMemcpyHostToDevice, s));
  RK_CUDA_CHECK(cudaMemcpyAsync(w.ec.get() + w.n_edges, &c, 4, cudaMemcpyHostToDevice, s));
  sync(s);  // r, c are host stack values
  ++w.n_edges;
}

void workspace_to_matrix(Workspace& w, rk_sparse& out) {
  cudaStream_t s = w.c->stream;
  DevEdges e;
  e.n = w.n_edges;
  const uint64_t n = w.n_edges ? w.n_edges : 1;
  e.row.alloc(n, s);
  e.col.alloc(n, s);
  e.block.alloc(n, s);
  e.mech.alloc(n, s);
  if (w.n_edges) {
    RK_CUDA_CHECK(cudaMemcpyAsync(e.row.get(), w.er.get(), w.n_edges * 4, cudaMemcpyDeviceToDevice, s));
    RK_CUDA_CHECK(cudaMemcpyAsync(e.col.get(), w.ec.get(), w.n_edges * 4, cudaMemcpyDeviceToDevice, s));
  }
  DevMatrix m;
  apply_edges(w.base, e, m, s);
  csr_to_entries_host(m.csr, out, s);
}

}  // namespace rk
