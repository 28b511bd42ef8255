// rk_ingest.cu -- device sparse formats.
//
//  * upload_entries: the reference's SparseMatrix entry array (sorted (row, col),
//    proj/src/sparse_matrix.cpp:9-34) -> device CSR, validating the same
//    invariants the reference constructor enforces (range, explicit zero,
//    duplicate) plus sortedness (the reference sorts; the C ABI requires sorted input).
//  * csr_to_csc: column-major twin, rows ascending inside each column.
//  * apply_edges: the repaired matrix = input + repair edges with value 1.0
//    (RepairWorkspace::to_matrix, proj/src/repair.cpp:147-160), in both formats.
#include <cub/device/device_radix_sort.cuh>

#include "rk_internal.cuh"

namespace rk {
namespace {

constexpr int kT = 256;

inline unsigned blocks_for(uint64_t n, int t = kT) {
  uint64_t b = ceil_div(n, (uint64_t)t);
  if (b == 0) b = 1;
  if (b > (1u << 30)) b = (1u << 30);
  return (unsigned)b;
}

// status: [0] = first bad index (UINT64_MAX = none), [1] = error kind
__global__ void entries_to_csr(const rk_entry* e, uint64_t nnz, uint64_t rows, uint64_t cols,
                               uint64_t* row_ptr, uint32_t* idx, double* val,
                               unsigned long long* status) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const rk_entry x = e[i];
    int kind = 0;
    if (x.row >= rows || x.col >= cols) kind = 1;
    else if (x.value == 0.0) kind = 2;
    else if (i > 0) {
      const rk_entry y = e[i - 1];
      if (y.row > x.row || (y.row == x.row && y.col > x.col)) kind = 4;
      else if (y.row == x.row && y.col == x.col) kind = 3;
    }
    if (kind) {
      unsigned long long old = atomicMin(&status[0], (unsigned long long)i);
      (void)old;
      continue;
    }
    idx[i] = (uint32_t)x.col;
    val[i] = x.value;
    const uint64_t prev = i == 0 ? 0 : e[i - 1].row + 1;
    if (i == 0 || e[i - 1].row != x.row)
      for (uint64_t r = (i == 0 ? 0 : prev); r <= x.row; ++r) row_ptr[r] = i;
    if (i + 1 == nnz)
      for (uint64_t r = x.row + 1; r <= rows; ++r) row_ptr[r] = nnz;
  }
}

// first index i > 0 with e[i-1] > e[i] in (row, col) order (UINT64_MAX: sorted)
__global__ void find_unsorted(const rk_entry* e, uint64_t nnz, unsigned long long* first) {
  for (uint64_t i = 1 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const rk_entry x = e[i], y = e[i - 1];
    if (y.row > x.row || (y.row == x.row && y.col > x.col)) atomicMin(first, (unsigned long long)i);
  }
}

// sort key (row, col) in one u64; indices >= 2^32 only occur in out-of-range
// entries (dimensions are < 2^32), clamped -- they fail validation either way
__global__ void make_keys(const rk_entry* e, uint64_t nnz, uint64_t* key, uint64_t* idx) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = e[i].row < 0xffffffffull ? e[i].row : 0xffffffffull;
    const uint64_t c = e[i].col < 0xffffffffull ? e[i].col : 0xffffffffull;
    key[i] = (r << 32) | c;
    idx[i] = i;
  }
}

__global__ void gather_entries(const rk_entry* e, const uint64_t* idx, uint64_t nnz, rk_entry* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = e[idx[i]];
}

__global__ void empty_row_ptr(uint64_t* row_ptr, uint64_t rows) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r <= rows;
       r += (uint64_t)gridDim.x * blockDim.x)
    row_ptr[r] = 0;
}

__global__ void count_cols(const uint32_t* idx, uint64_t nnz, uint32_t* cnt) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[idx[i]], 1u);
}

// scatter rows into their columns (arbitrary order inside a column)
__global__ void scatter_csc(const uint64_t* row_ptr, const uint32_t* idx, const double* val,
                            uint64_t rows, const uint64_t* col_ptr, uint32_t* cursor,
                            uint32_t* out_row, double* out_val) {
  const int lane = threadIdx.x & 31;
  for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < rows;
       r += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
    for (uint64_t i = row_ptr[r] + lane; i < row_ptr[r + 1]; i += 32) {
      const uint32_t c = idx[i];
      const uint64_t pos = col_ptr[c] + atomicAdd(&cursor[c], 1u);
      out_row[pos] = (uint32_t)r;
      out_val[pos] = val[i];
    }
  }
}

// insertion sort of each segment by key (segments are short: a column of a
// sparse matrix); deterministic regardless of the scatter order
__global__ void sort_segments(const uint64_t* ptr, uint64_t nseg, uint32_t* key, double* val) {
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < nseg;
       s += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t lo = ptr[s], hi = ptr[s + 1];
    for (uint64_t i = lo + 1; i < hi; ++i) {
      const uint32_t k = key[i];
      const double v = val ? val[i] : 0.0;
      uint64_t j = i;
      while (j > lo && key[j - 1] > k) {
        key[j] = key[j - 1];
        if (val) val[j] = val[j - 1];
        --j;
      }
      key[j] = k;
      if (val) val[j] = v;
    }
  }
}

__global__ void count_edges(const uint32_t* e_key, uint64_t n, uint32_t* cnt) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[e_key[i]], 1u);
}

__global__ void scatter_edges(const uint32_t* e_key, const uint32_t* e_other, uint64_t n,
                              const uint64_t* eptr, uint32_t* cursor, uint32_t* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t k = e_key[i];
    out[eptr[k] + atomicAdd(&cursor[k], 1u)] = e_other[i];
  }
}

__global__ void add_counts(const uint64_t* old_ptr, const uint64_t* eptr, uint64_t nseg, uint64_t* cnt) {
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < nseg;
       s += (uint64_t)gridDim.x * blockDim.x)
    cnt[s] = (old_ptr[s + 1] - old_ptr[s]) + (eptr[s + 1] - eptr[s]);
}

// merged segment = old entries (sorted) + edge keys (sorted, value 1.0):
// one thread per entry (old entries, then edges): the entry's
// segment by binary search over the segment pointers, its rank among the other
// list's keys of that segment by binary search. Flat parallelism for both shapes
// -- 256 long CSR rows (a warp per row left most of the GPU idle: 47 us) and
// 262k one-entry CSC columns (a warp per column left most lanes idle)
__device__ __forceinline__ uint64_t segment_of(const uint64_t* ptr, uint64_t nseg, uint64_t i) {
  uint64_t lo = 0, hi = nseg;  // last s with ptr[s] <= i
  while (lo < hi) {
    const uint64_t mid = (lo + hi + 1) >> 1;
    if (ptr[mid] <= i) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void merge_flat(const uint64_t* __restrict__ old_ptr, const uint32_t* __restrict__ old_key,
                           const double* __restrict__ old_val, uint64_t old_n, const uint64_t* __restrict__ eptr,
                           const uint32_t* __restrict__ ekey, uint64_t e_n, uint64_t nseg,
                           const uint64_t* __restrict__ new_ptr, uint32_t* __restrict__ new_key,
                           double* __restrict__ new_val) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < old_n + e_n;
       t += (uint64_t)gridDim.x * blockDim.x) {
    if (t < old_n) {
      const uint64_t i = t, sg = segment_of(old_ptr, nseg, i);
      const uint32_t k = old_key[i];
      uint64_t lo = eptr[sg], hi = eptr[sg + 1];
      const uint64_t e0 = lo;
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (ekey[mid] < k) lo = mid + 1; else hi = mid;
      }
      const uint64_t pos = new_ptr[sg] + (i - old_ptr[sg]) + (lo - e0);
      new_key[pos] = k;
      new_val[pos] = old_val[i];
    } else {
      const uint64_t j = t - old_n, sg = segment_of(eptr, nseg, j);
      const uint32_t k = ekey[j];
      uint64_t lo = old_ptr[sg], hi = old_ptr[sg + 1];
      const uint64_t o0 = lo;
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (old_key[mid] < k) lo = mid + 1; else hi = mid;
      }
      const uint64_t pos = new_ptr[sg] + (lo - o0) + (j - eptr[sg]);
      new_key[pos] = k;
      new_val[pos] = 1.0;
    }
  }
}

__global__ void csr_to_entry_array(const uint64_t* row_ptr, const uint32_t* idx, const double* val,
                                   uint64_t rows, rk_entry* out) {
  const int lane = threadIdx.x & 31;
  for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < rows;
       r += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
    for (uint64_t i = row_ptr[r] + lane; i < row_ptr[r + 1]; i += 32) {
      rk_entry e;
      e.row = r;
      e.col = idx[i];
      e.value = val[i];
      out[i] = e;
    }
  }
}

// edges -> per-segment sorted key lists (segment = column or row)
void bucket_edges(const uint32_t* key, const uint32_t* other, uint64_t n, uint64_t nseg,
                  DBuf<uint64_t>& eptr, DBuf<uint32_t>& ekey, cudaStream_t s) {
  DBuf<uint32_t> cnt(nseg, s);
  cnt.zero();
  if (n) {
    count_edges<<<blocks_for(n), kT, 0, s>>>(key, n, cnt.get());
    RK_LAUNCH_CHECK();
  }
  eptr.alloc(nseg + 1, s);
  exclusive_scan_u32to64(cnt.get(), eptr.get(), nseg, s);
  ekey.alloc(n ? n : 1, s);
  if (n) {
    cnt.zero();
    scatter_edges<<<blocks_for(n), kT, 0, s>>>(key, other, n, eptr.get(), cnt.get(), ekey.get());
    RK_LAUNCH_CHECK();
    sort_segments<<<blocks_for(nseg), kT, 0, s>>>(eptr.get(), nseg, ekey.get(), nullptr);
    RK_LAUNCH_CHECK();
  }
}

template <class Out>
void merge_format(const DBuf<uint64_t>& old_ptr, const DBuf<uint32_t>& old_key, const DBuf<double>& old_val,
                  uint64_t nseg, uint64_t old_nnz, const uint32_t* key, const uint32_t* other, uint64_t n_edges,
                  Out& out, cudaStream_t s) {
  DBuf<uint64_t> eptr;
  DBuf<uint32_t> ekey;
  bucket_edges(key, other, n_edges, nseg, eptr, ekey, s);
  DBuf<uint64_t> cnt(nseg, s);
  add_counts<<<blocks_for(nseg), kT, 0, s>>>(old_ptr.get(), eptr.get(), nseg, cnt.get());
  RK_LAUNCH_CHECK();
  out.ptr.alloc(nseg + 1, s);
  exclusive_scan_u64(cnt.get(), out.ptr.get(), nseg, s);
  out.nnz = old_nnz + n_edges;
  out.idx.alloc(out.nnz ? out.nnz : 1, s);
  out.val.alloc(out.nnz ? out.nnz : 1, s);
  merge_flat<<<blocks_for(old_nnz + n_edges), kT, 0, s>>>(old_ptr.get(), old_key.get(), old_val.get(), old_nnz,
                                                          eptr.get(), ekey.get(), n_edges, nseg, out.ptr.get(),
                                                          out.idx.get(), out.val.get());
  RK_LAUNCH_CHECK();
}

}  // namespace

namespace {
__global__ void first_equal_adjacent(const uint64_t* key, uint64_t n, unsigned long long* first) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x + 1; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    if (key[i] == key[i - 1]) atomicMin(first, (unsigned long long)i);
}
}  // namespace

void sort_entries_device(const rk_entry* host_in, uint64_t n, rk_entry* host_sorted, int64_t* dup_a, int64_t* dup_b,
                         cudaStream_t s) {
  *dup_a = *dup_b = -1;
  if (n == 0) return;
  DBuf<rk_entry> staged(n, s), sorted(n, s);
  RK_CUDA_CHECK(cudaMemcpyAsync(staged.get(), host_in, n * sizeof(rk_entry), cudaMemcpyHostToDevice, s));
  DBuf<uint64_t> k_in(n, s), k_out(n, s), i_in(n, s), i_out(n, s);
  make_keys<<<blocks_for(n), kT, 0, s>>>(staged.get(), n, k_in.get(), i_in.get());
  RK_LAUNCH_CHECK();
  size_t tmp_bytes = 0;
  RK_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k_in.get(), k_out.get(), i_in.get(), i_out.get(),
                                                n, 0, 64, s));
  DBuf<unsigned char> tmp(tmp_bytes ? tmp_bytes : 1, s);
  RK_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp.get(), tmp_bytes, k_in.get(), k_out.get(), i_in.get(), i_out.get(),
                                                n, 0, 64, s));
  gather_entries<<<blocks_for(n), kT, 0, s>>>(staged.get(), i_out.get(), n, sorted.get());
  RK_LAUNCH_CHECK();
  DBuf<unsigned long long> first(1, s);
  RK_CUDA_CHECK(cudaMemsetAsync(first.get(), 0xff, sizeof(unsigned long long), s));
  first_equal_adjacent<<<blocks_for(n), kT, 0, s>>>(k_out.get(), n, first.get());
  RK_LAUNCH_CHECK();
  unsigned long long f = 0;
  RK_CUDA_CHECK(cudaMemcpyAsync(&f, first.get(), sizeof f, cudaMemcpyDeviceToHost, s));
  RK_CUDA_CHECK(cudaMemcpyAsync(host_sorted, sorted.get(), n * sizeof(rk_entry), cudaMemcpyDeviceToHost, s));
  sync(s);
  if (f != ~0ull) {
    uint64_t pair[2];
    RK_CUDA_CHECK(cudaMemcpyAsync(pair, i_out.get() + f - 1, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    sync(s);
    *dup_a = (int64_t)pair[0];
    *dup_b = (int64_t)pair[1];
  }
}

void upload_entries(const rk_sparse_view& a, DevMatrix& m, cudaStream_t s) {
  if (a.nnz && !a.entries) fail(RK_INVALID_ARGUMENT, "sparse view has entries == NULL");
  if (a.cols > 0xffffffffull || a.rows > 0xffffffffull)
    fail(RK_INVALID_ARGUMENT, "matrix dimensions above 2^32 are not supported");
  DevCsr& c = m.csr;
  c.rows = a.rows;
  c.cols = a.cols;
  c.nnz = a.nnz;
  c.ptr.alloc(a.rows + 1, s);
  c.idx.alloc(a.nnz ? a.nnz : 1, s);
  c.val.alloc(a.nnz ? a.nnz : 1, s);
  if (a.nnz == 0) {
    empty_row_ptr<<<blocks_for(a.rows + 1), kT, 0, s>>>(c.ptr.get(), a.rows);
    RK_LAUNCH_CHECK();
  } else {
    DBuf<rk_entry> staged(a.nnz, s);
    RK_CUDA_CHECK(cudaMemcpyAsync(staged.get(), a.entries, a.nnz * sizeof(rk_entry), cudaMemcpyHostToDevice, s));
    // any order is accepted, as by the reference constructor, which sorts by
    // (row, col) before validating (sparse_matrix.cpp:12-14): unsorted input is
    // sorted here with a stable device radix sort
    {
      DBuf<unsigned long long> first(1, s);
      RK_CUDA_CHECK(cudaMemsetAsync(first.get(), 0xff, sizeof(unsigned long long), s));
      find_unsorted<<<blocks_for(a.nnz), kT, 0, s>>>(staged.get(), a.nnz, first.get());
      RK_LAUNCH_CHECK();
      unsigned long long h_first = 0;
      RK_CUDA_CHECK(cudaMemcpyAsync(&h_first, first.get(), sizeof h_first, cudaMemcpyDeviceToHost, s));
      sync(s);
      if (h_first != ~0ull) {
        DBuf<uint64_t> k_in(a.nnz, s), k_out(a.nnz, s), i_in(a.nnz, s), i_out(a.nnz, s);
        make_keys<<<blocks_for(a.nnz), kT, 0, s>>>(staged.get(), a.nnz, k_in.get(), i_in.get());
        RK_LAUNCH_CHECK();
        size_t tmp_bytes = 0;
        RK_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k_in.get(), k_out.get(), i_in.get(),
                                                      i_out.get(), a.nnz, 0, 64, s));
        DBuf<unsigned char> tmp(tmp_bytes ? tmp_bytes : 1, s);
        RK_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp.get(), tmp_bytes, k_in.get(), k_out.get(), i_in.get(),
                                                      i_out.get(), a.nnz, 0, 64, s));
        DBuf<rk_entry> sorted(a.nnz, s);
        gather_entries<<<blocks_for(a.nnz), kT, 0, s>>>(staged.get(), i_out.get(), a.nnz, sorted.get());
        RK_LAUNCH_CHECK();
        staged = std::move(sorted);
      }
    }
    DBuf<unsigned long long> status(2, s);
    RK_CUDA_CHECK(cudaMemsetAsync(status.get(), 0xff, 2 * sizeof(unsigned long long), s));
    entries_to_csr<<<blocks_for(a.nnz), kT, 0, s>>>(staged.get(), a.nnz, a.rows, a.cols, c.ptr.get(),
                                                    c.idx.get(), c.val.get(), status.get());
    RK_LAUNCH_CHECK();
    unsigned long long bad = 0;
    RK_CUDA_CHECK(cudaMemcpyAsync(&bad, status.get(), sizeof bad, cudaMemcpyDeviceToHost, s));
    sync(s);
    if (bad != ~0ull) {
      rk_entry pair[2];  // (bad - 1, bad) of the (sorted) device array
      const uint64_t lo = bad ? bad - 1 : 0;
      RK_CUDA_CHECK(cudaMemcpyAsync(pair, staged.get() + lo, (bad ? 2 : 1) * sizeof(rk_entry),
                                    cudaMemcpyDeviceToHost, s));
      sync(s);
      const rk_entry& x = bad ? pair[1] : pair[0];
      std::string at = "(" + std::to_string(x.row) + ", " + std::to_string(x.col) + ")";
      if (x.row >= a.rows || x.col >= a.cols)
        fail(RK_INVALID_ARGUMENT, "sparse entry " + at + " outside " + std::to_string(a.rows) + "x" +
                                      std::to_string(a.cols));
      if (x.value == 0.0) fail(RK_INVALID_ARGUMENT, "sparse entry " + at + " stores zero");
      const rk_entry& y = pair[0];
      if (bad && y.row == x.row && y.col == x.col) fail(RK_INVALID_ARGUMENT, "duplicate sparse entry " + at);
      fail(RK_INVALID_ARGUMENT, "sparse entries must be sorted by (row, col); entry " +
                                    std::to_string(bad) + " " + at + " is out of order");
    }
  }
  csr_to_csc(c, m.csc, s);
}

void csr_to_csc(const DevCsr& a, DevCsc& out, cudaStream_t s) {
  out.rows = a.rows;
  out.cols = a.cols;
  out.nnz = a.nnz;
  DBuf<uint32_t> cnt(a.cols, s);
  cnt.zero();
  if (a.nnz) {
    count_cols<<<blocks_for(a.nnz), kT, 0, s>>>(a.idx.get(), a.nnz, cnt.get());
    RK_LAUNCH_CHECK();
  }
  out.ptr.alloc(a.cols + 1, s);
  exclusive_scan_u32to64(cnt.get(), out.ptr.get(), a.cols, s);
  out.idx.alloc(a.nnz ? a.nnz : 1, s);
  out.val.alloc(a.nnz ? a.nnz : 1, s);
  if (a.nnz) {
    cnt.zero();
    scatter_csc<<<blocks_for(a.rows * 32), kT, 0, s>>>(a.ptr.get(), a.idx.get(), a.val.get(), a.rows,
                                                       out.ptr.get(), cnt.get(), out.idx.get(), out.val.get());
    RK_LAUNCH_CHECK();
    sort_segments<<<blocks_for(a.cols), kT, 0, s>>>(out.ptr.get(), a.cols, out.idx.get(), out.val.get());
    RK_LAUNCH_CHECK();
  }
}

void apply_edges(const DevMatrix& a, const DevEdges& e, DevMatrix& out, cudaStream_t s) {
  out.csc.rows = out.csr.rows = a.csr.rows;
  out.csc.cols = out.csr.cols = a.csr.cols;
  // CSC: bucket edges by column, keys = rows
  merge_format(a.csc.ptr, a.csc.idx, a.csc.val, a.csc.cols, a.csc.nnz, e.col.get(), e.row.get(), e.n,
               out.csc, s);
  // CSR: bucket edges by row, keys = columns
  merge_format(a.csr.ptr, a.csr.idx, a.csr.val, a.csr.rows, a.csr.nnz, e.row.get(), e.col.get(), e.n,
               out.csr, s);
}

void csr_to_entries_host(const DevCsr& a, rk_sparse& out, cudaStream_t s) {
  out.rows = a.rows;
  out.cols = a.cols;
  out.nnz = a.nnz;
  out.entries = static_cast<rk_entry*>(host_alloc_bytes((a.nnz ? a.nnz : 1) * sizeof(rk_entry)));
  if (!a.nnz) return;
  DBuf<rk_entry> tmp(a.nnz, s);
  csr_to_entry_array<<<blocks_for(a.rows * 32), kT, 0, s>>>(a.ptr.get(), a.idx.get(), a.val.get(), a.rows,
                                                            tmp.get());
  RK_LAUNCH_CHECK();
  RK_CUDA_CHECK(cudaMemcpyAsync(out.entries, tmp.get(), a.nnz * sizeof(rk_entry), cudaMemcpyDeviceToHost, s));
  sync(s);
}

}  // namespace rk
