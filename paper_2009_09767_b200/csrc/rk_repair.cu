// rk_repair.cu -- rank check + checker repair on the device.
//
// Reference: proj/src/repair.cpp:42-216.
//  1. presence scan: one pass over the CSR marks (block, row) pairs that own an
//     entry; the complement, in (block, row) order, is exactly the reference's
//     sequence of lonely rows (blocks ascending, rows ascending, :171-179).
//  2. RandomChecker (:95-101): one thread per lonely row draws
//     KeyedRng(seed, d, row).below(width) -- independent rows, so the parallel
//     result is the sequential one bit for bit.
//  3. NeighborChecker / NeighborRandomChecker (:103-145, :184-209) are
//     order-dependent: every decision reads the workspace after all earlier
//     insertions. A single persistent CTA replays the lonely rows in reference
//     order; each step's candidate-row set and neighbor-column set are built
//     in parallel as bitmaps over the immutable CSR/CSC plus the overlay of
//     edges inserted so far, and the k-th set bit is picked with the same draw.
#include "rk_internal.cuh"

namespace rk {
namespace {

constexpr int kT = 256;

inline unsigned grid_for(uint64_t n, int t = kT) {
  uint64_t b = ceil_div(n, (uint64_t)t);
  if (b == 0) b = 1;
  if (b > (1u << 30)) b = 1u << 30;
  return (unsigned)b;
}

// presence[d * rows + r] = 1 when row r has an entry in block d:
// one thread per entry: the entry's row by binary search over
// row_ptr (cached), then the first entry of each (row, block) run writes. A warp
// per row left the GPU nearly idle (c2: 256 warps; c4: 525 dependent loads per
// lane)
__global__ void presence_flat_kernel(const uint64_t* __restrict__ row_ptr, const uint32_t* __restrict__ idx,
                                     uint64_t rows, uint64_t nnz, Partition p, uint32_t* __restrict__ presence) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t lo = 0, hi = rows - 1;  // last r with row_ptr[r] <= i
    while (lo < hi) {
      const uint64_t mid = (lo + hi + 1) >> 1;
      if (row_ptr[mid] <= i) lo = mid; else hi = mid - 1;
    }
    const uint64_t r = lo;
    const uint64_t d = p.block_of(idx[i]);
    if (i == row_ptr[r] || p.block_of(idx[i - 1]) != d) presence[d * rows + r] = 1u;
  }
}

// The same flags from the CSC: block d's entries are one contiguous slice of the
// column-ordered entries, so a CTA streams the slice's row indices (4 bytes per
// entry, coalesced, the only HBM traffic) and sets presence[d * rows + row] -- no
// search, same-value races only. grid = (slices of a block, blocks).
template <bool SMEM>
__global__ void __launch_bounds__(256) presence_csc_kernel(const uint64_t* __restrict__ col_ptr,
                                                           const uint32_t* __restrict__ row_idx, uint64_t rows,
                                                           uint64_t nnz, Partition p, uint32_t* __restrict__ presence) {
  extern __shared__ uint32_t sflag[];  // SMEM: the block's M flags, set in shared memory, written out once
  for (uint64_t d = blockIdx.y; d < p.blocks; d += gridDim.y) {
    const uint64_t e0 = col_ptr[p.begin(d)], e1 = col_ptr[p.end(d)];
    uint32_t* f = presence + d * rows;
    if (SMEM) {
      for (uint64_t t = threadIdx.x; t < rows; t += blockDim.x) sflag[t] = 0u;
      __syncthreads();
    }
    uint32_t* dst = SMEM ? sflag : f;
    // 16-byte loads from the slice's aligned start (entries outside [e0, e1) masked),
    // two per thread and step, both issued before the first flag store
    const uint64_t eb = e0 & ~(uint64_t)3;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 4;
    for (uint64_t e = eb + ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; e < e1; e += 2 * stride) {
      uint4 r[2];
      bool ok[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const uint64_t eu = e + u * stride;
        ok[u] = eu < e1;
        r[u] = make_uint4(0u, 0u, 0u, 0u);
        if (ok[u] && eu + 4 <= nnz) {
          r[u] = __ldcs(reinterpret_cast<const uint4*>(row_idx + eu));
        } else if (ok[u]) {
          r[u].x = eu < nnz ? row_idx[eu] : 0u;
          r[u].y = eu + 1 < nnz ? row_idx[eu + 1] : 0u;
          r[u].z = eu + 2 < nnz ? row_idx[eu + 2] : 0u;
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (!ok[u]) continue;
        const uint64_t eu = e + u * stride;
        if (eu >= e0 && eu < e1) dst[r[u].x] = 1u;
        if (eu + 1 >= e0 && eu + 1 < e1) dst[r[u].y] = 1u;
        if (eu + 2 >= e0 && eu + 2 < e1) dst[r[u].z] = 1u;
        if (eu + 3 >= e0 && eu + 3 < e1) dst[r[u].w] = 1u;
      }
    }
    if (SMEM) {
      __syncthreads();
      for (uint64_t t = threadIdx.x; t < rows; t += blockDim.x)
        if (sflag[t]) f[t] = 1u;
      __syncthreads();
    }
  }
}

__global__ void invert_flags(uint32_t* f, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    f[i] = f[i] ? 0u : 1u;
}

__global__ void compact_lonely(const uint32_t* flag, const uint64_t* pos, uint64_t rows, uint64_t n,
                               uint32_t* l_block, uint32_t* l_row) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (flag[i]) {
      const uint64_t k = pos[i];
      l_block[k] = (uint32_t)(i / rows);
      l_row[k] = (uint32_t)(i % rows);
    }
  }
}

__global__ void block_counts(const uint64_t* pos, uint64_t rows, uint64_t blocks, uint64_t* counts) {
  for (uint64_t d = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; d < blocks;
       d += (uint64_t)gridDim.x * blockDim.x)
    counts[d] = pos[(d + 1) * rows] - pos[d * rows];
}

// RandomChecker -- repair.cpp:95-101 (+ the driver branch :178-182)
__global__ void random_fill(const uint32_t* l_block, const uint32_t* l_row, uint64_t n, Partition p,
                            uint64_t seed, uint32_t* e_block, uint32_t* e_row, uint32_t* e_col,
                            int32_t* e_mech) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t d = l_block[i], row = l_row[i];
    KeyedRng g(seed, d, row);
    const uint64_t b = p.begin(d), w = p.end(d) - b;
    e_block[i] = (uint32_t)d;
    e_row[i] = (uint32_t)row;
    e_col[i] = (uint32_t)(b + g.below(w));
    e_mech[i] = 0;
  }
}

// ---------------------------------------------------------------------------
// ordered neighbor replay (single CTA)

constexpr int kReplayThreads = 1024;

struct ReplayArgs {
  const uint64_t* row_ptr; const uint32_t* col_idx;   // CSR of the input
  const uint64_t* col_ptr; const uint32_t* row_idx;   // CSC of the input
  uint64_t rows;
  Partition p;
  const uint32_t* l_block; const uint32_t* l_row; uint64_t n_lonely;
  uint64_t seed;
  int method;                        // 1 neighbor, 2 neighbor-random
  unsigned long long* cand;          // ceil(rows/64) words
  unsigned long long* nb;            // ceil(max width/64) words
  uint32_t* rowov; uint32_t rowov_cap;  // scratch: the lonely row's inserted columns
  uint32_t* e_block; uint32_t* e_row; uint32_t* e_col; int32_t* e_mech;  // capacity 2 * n_lonely
  unsigned long long* out_counts;    // [0] edges, [1] fallbacks, [2] overflow flag, [3] steps recomputed
  // speculation (null: off): every step's sets computed beforehand on the input alone
  const unsigned long long* spec_cand;  // n_lonely x cand_words
  const unsigned long long* spec_nb;    // n_lonely x nb_stride
  uint64_t nb_stride;
  const unsigned long long* spec_count;
  const uint32_t* spec_col;
  const uint64_t* spec_state;           // the step's KeyedRng state after its neighbor draw
};

// Speculation: step i's candidate rows and neighbor columns from the INPUT alone (no
// inserted edges), the neighbor draw included -- one CTA per lonely (block, row), all
// in parallel. The ordered replay then only checks whether the edges inserted before
// step i could have changed its sets (see neighbor_replay) and recomputes the few
// steps where they could.
__global__ void __launch_bounds__(256) speculate_kernel(ReplayArgs a, unsigned long long* cand_all,
                                                        unsigned long long* nb_all, unsigned long long* count_out,
                                                        uint32_t* col_out, uint64_t* state_out) {
  __shared__ unsigned long long s_red[8];
  __shared__ unsigned long long s_k;
  const uint64_t step = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t d = a.l_block[step], row = a.l_row[step];
  const uint64_t b = a.p.begin(d), e = a.p.end(d), width = e - b;
  const uint64_t cand_words = (a.rows + 63) / 64, nb_words = (width + 63) / 64;
  unsigned long long* cand = cand_all + step * cand_words;
  unsigned long long* nb = nb_all + step * a.nb_stride;
  for (uint64_t i = a.row_ptr[row] + tid; i < a.row_ptr[row + 1]; i += 256) {
    const uint64_t c = a.col_idx[i];
    if (c >= b && c < e) continue;
    for (uint64_t k = a.col_ptr[c]; k < a.col_ptr[c + 1]; ++k) {
      const uint32_t m = a.row_idx[k];
      atomicOr(&cand[m >> 6], 1ull << (m & 63));
    }
  }
  __syncthreads();
  for (uint64_t jj = tid; jj < width; jj += 256) {
    const uint64_t c = b + jj;
    for (uint64_t k = a.col_ptr[c], kend = a.col_ptr[c + 1]; k < kend; ++k) {
      const uint32_t m = a.row_idx[k];
      if ((cand[m >> 6] >> (m & 63)) & 1ull) {
        atomicOr(&nb[jj >> 6], 1ull << (jj & 63));
        break;
      }
    }
  }
  __syncthreads();
  unsigned long long mine = 0;
  for (uint64_t w = tid; w < nb_words; w += 256) mine += __popcll(nb[w]);
  for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if (lane == 0) s_red[warp] = mine;
  __syncthreads();
  if (tid == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < 8; ++w) t += s_red[w];
    KeyedRng g(a.seed, d, row);
    s_k = t ? g.below(t) : 0;  // no draw when the set is empty (repair.cpp:130)
    count_out[step] = t;
    state_out[step] = g.state;
    col_out[step] = 0xffffffffu;
    // the k-th set bit, ascending (a serial scan: one thread, nb_words words)
    if (t) {
      unsigned long long k = s_k;
      for (uint64_t w = 0; w < nb_words; ++w) {
        unsigned long long bits = nb[w];
        const unsigned long long pc = __popcll(bits);
        if (k < pc) {
          for (unsigned long long z = 0; z < k; ++z) bits &= bits - 1;
          col_out[step] = (uint32_t)(b + w * 64 + (__ffsll((long long)bits) - 1));
          break;
        }
        k -= pc;
      }
    }
  }
}

__device__ __forceinline__ bool csr_has(const uint64_t* row_ptr, const uint32_t* col_idx, uint64_t r,
                                        uint32_t c) {
  uint64_t lo = row_ptr[r], hi = row_ptr[r + 1];
  while (lo < hi) {
    uint64_t mid = (lo + hi) >> 1;
    if (col_idx[mid] < c) lo = mid + 1; else hi = mid;
  }
  return lo < row_ptr[r + 1] && col_idx[lo] == c;
}

__device__ __forceinline__ uint64_t csr_lower(const uint64_t* row_ptr, const uint32_t* col_idx, uint64_t r,
                                              uint64_t c) {
  uint64_t lo = row_ptr[r], hi = row_ptr[r + 1];
  while (lo < hi) {
    uint64_t mid = (lo + hi) >> 1;
    if (col_idx[mid] < c) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(kReplayThreads, 1) neighbor_replay(ReplayArgs a) {
  __shared__ unsigned long long s_red[kReplayThreads / 32];
  __shared__ unsigned long long s_count, s_k, s_col;
  __shared__ uint64_t s_state;
  __shared__ uint32_t s_n_edges, s_rowov_n, s_fallback;
  __shared__ int s_found;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t cand_words = (a.rows + 63) / 64;
  if (tid == 0) { s_n_edges = 0; s_fallback = 0; }
  __syncthreads();

  for (uint64_t step = 0; step < a.n_lonely; ++step) {
    const uint64_t d = a.l_block[step], row = a.l_row[step];
    const uint64_t b = a.p.begin(d), e = a.p.end(d), width = e - b;
    const uint64_t nb_words = (width + 63) / 64;
    const uint32_t n_edges = s_n_edges;
    for (uint64_t w = tid; w < cand_words; w += kReplayThreads) a.cand[w] = 0ull;
    for (uint64_t w = tid; w < nb_words; w += kReplayThreads) a.nb[w] = 0ull;
    if (tid == 0) s_rowov_n = 0;
    __syncthreads();
    // b0: the lonely row's inserted columns (all outside block d: the row is lonely in d)
    for (uint32_t j = tid; j < n_edges; j += kReplayThreads) {
      if (a.e_row[j] == row) {
        uint32_t k = atomicAdd(&s_rowov_n, 1u);
        if (k < a.rowov_cap) a.rowov[k] = a.e_col[j];
        else a.out_counts[2] = 1ull;
      }
    }
    __syncthreads();
    const uint32_t rowov_n = min(s_rowov_n, a.rowov_cap);
    // speculation check: step's sets from the input alone hold unless an earlier edge
    //   (1) put a column c on `row` (c in rowov) one of whose rows (input or inserted) is
    //       not already a candidate;
    //   (2) is (m, c) with c in [b, e), m a candidate, c not already a neighbor column;
    //   (3) is (m, c) with c outside [b, e) on one of `row`'s input columns, m not a candidate.
    // Otherwise the candidate and neighbor sets -- and so the draw -- are the speculated ones.
    bool spec_ok = false;  // uniform over the CTA
    if (a.spec_cand) {
      const unsigned long long* sc = a.spec_cand + step * cand_words;
      const unsigned long long* sn = a.spec_nb + step * a.nb_stride;
      auto in_cand = [&](uint32_t m) { return ((sc[m >> 6] >> (m & 63)) & 1ull) != 0ull; };
      bool changed = false;
      for (uint32_t q = tid; q < rowov_n && !changed; q += kReplayThreads) {
        const uint32_t c = a.rowov[q];
        for (uint64_t k = a.col_ptr[c]; k < a.col_ptr[c + 1] && !changed; ++k) changed = !in_cand(a.row_idx[k]);
      }
      for (uint32_t j = tid; j < n_edges && !changed; j += kReplayThreads) {
        const uint32_t m = a.e_row[j], c = a.e_col[j];
        if (c >= b && c < e) {
          const uint64_t jj = c - b;
          changed = in_cand(m) && !((sn[jj >> 6] >> (jj & 63)) & 1ull);
        } else {
          bool on_row = false;
          for (uint32_t q = 0; q < rowov_n && !on_row; ++q) on_row = a.rowov[q] == c;
          if (on_row || csr_has(a.row_ptr, a.col_idx, row, c)) changed = !in_cand(m);
        }
      }
      if (__syncthreads_or(changed ? 1 : 0) == 0) {
        if (tid == 0) {
          s_found = a.spec_count[step] > 0;
          s_col = a.spec_col[step];
          s_state = a.spec_state[step];
        }
        spec_ok = true;
      } else if (tid == 0) {
        atomicAdd(&a.out_counts[3], 1ull);
      }
    }
    if (!spec_ok) {
    // b1: rows sharing an input column with `row` outside [b, e) -- repair.cpp:111-117
    {
      const uint64_t lo = a.row_ptr[row], hi = a.row_ptr[row + 1];
      const uint64_t total = (hi - lo) + rowov_n;
      for (uint64_t i = tid; i < total; i += kReplayThreads) {
        const uint64_t c = i < hi - lo ? a.col_idx[lo + i] : a.rowov[i - (hi - lo)];
        if (c >= b && c < e) continue;
        for (uint64_t k = a.col_ptr[c]; k < a.col_ptr[c + 1]; ++k) {
          const uint32_t m = a.row_idx[k];
          atomicOr(&a.cand[m >> 6], 1ull << (m & 63));
        }
      }
    }
    // b2: rows that gained an inserted entry on one of `row`'s outside columns
    for (uint32_t j = tid; j < n_edges; j += kReplayThreads) {
      const uint32_t c = a.e_col[j];
      if (c >= b && c < e) continue;
      bool shares = csr_has(a.row_ptr, a.col_idx, row, c);
      for (uint32_t q = 0; q < rowov_n && !shares; ++q) shares = a.rowov[q] == c;
      if (shares) {
        const uint32_t m = a.e_row[j];
        atomicOr(&a.cand[m >> 6], 1ull << (m & 63));
      }
    }
    __syncthreads();
    // c: candidate rows' columns inside [b, e) -- repair.cpp:119-127. The same set
    // read from the block's side: a column of [b, e) is in it when one of its
    // (CSC) rows is a candidate. One pass over the block's columns instead of a
    // binary search in every candidate row (c5: ~2000 candidate rows of ~33k
    // entries each per lonely row -- 7 ms per step, 17 s for the replay)
    for (uint64_t jj = tid; jj < width; jj += kReplayThreads) {
      const uint64_t c = b + jj;
      for (uint64_t k = a.col_ptr[c], kend = a.col_ptr[c + 1]; k < kend; ++k) {
        const uint32_t m = a.row_idx[k];
        if ((a.cand[m >> 6] >> (m & 63)) & 1ull) {
          atomicOr(&a.nb[jj >> 6], 1ull << (jj & 63));
          break;
        }
      }
    }
    for (uint32_t j = tid; j < n_edges; j += kReplayThreads) {
      const uint32_t c = a.e_col[j];
      if (c < b || c >= e) continue;
      const uint32_t m = a.e_row[j];
      if ((a.cand[m >> 6] >> (m & 63)) & 1ull) {
        const uint64_t jj = c - b;
        atomicOr(&a.nb[jj >> 6], 1ull << (jj & 63));
      }
    }
    __syncthreads();
    // d: |neighbor_cols| and the k-th smallest column -- repair.cpp:129-133
    const uint64_t per = (nb_words + kReplayThreads - 1) / kReplayThreads;
    const uint64_t w0 = min((uint64_t)tid * per, nb_words), w1 = min(w0 + per, nb_words);
    unsigned long long mine = 0;
    for (uint64_t w = w0; w < w1; ++w) mine += __popcll(a.nb[w]);
    unsigned long long incl = mine;
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_red[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      unsigned long long t = s_red[lane];
      for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      s_red[lane] = t;
      if (lane == 31) {
        s_count = t;
        KeyedRng g(a.seed, d, row);
        s_found = t > 0;
        if (t > 0) s_k = g.below(t);  // no draw when the set is empty (repair.cpp:130)
        s_state = g.state;
      }
    }
    __syncthreads();
    const unsigned long long excl = (warp ? s_red[warp - 1] : 0ull) + incl - mine;
    if (s_found && s_k >= excl && s_k < excl + mine) {
      unsigned long long k = s_k - excl;
      for (uint64_t w = w0; w < w1; ++w) {
        unsigned long long bits = a.nb[w];
        const unsigned long long pc = __popcll(bits);
        if (k < pc) {
          for (unsigned long long z = 0; z < k; ++z) bits &= bits - 1;
          s_col = b + w * 64 + (__ffsll((long long)bits) - 1);
          break;
        }
        k -= pc;
      }
    }
    }  // !spec_ok
    __syncthreads();
    // e: record edges -- repair.cpp:184-209
    if (tid == 0) {
      KeyedRng g(0, 0, 0);
      g.state = s_state;
      uint32_t n = s_n_edges;
      uint32_t neighbor_col = 0xffffffffu;
      if (s_found) {
        neighbor_col = (uint32_t)s_col;
        a.e_block[n] = (uint32_t)d; a.e_row[n] = (uint32_t)row; a.e_col[n] = neighbor_col; a.e_mech[n] = 1;
        ++n;
      }
      if (a.method == 1) {
        if (!s_found) {
          a.e_block[n] = (uint32_t)d; a.e_row[n] = (uint32_t)row;
          a.e_col[n] = (uint32_t)(b + g.below(width)); a.e_mech[n] = 0;
          ++n;
          ++s_fallback;
        }
      } else {
        const uint32_t rc = (uint32_t)(b + g.below(width));
        if (rc != neighbor_col) {
          a.e_block[n] = (uint32_t)d; a.e_row[n] = (uint32_t)row; a.e_col[n] = rc; a.e_mech[n] = 0;
          ++n;
        }
      }
      s_n_edges = n;
    }
    __syncthreads();
  }
  if (tid == 0) {
    a.out_counts[0] = s_n_edges;
    a.out_counts[1] = s_fallback;
  }
}

__global__ void lonely_in_block(const uint64_t* row_ptr, const uint32_t* idx, uint64_t rows, uint64_t b,
                                uint64_t e, uint32_t* flag) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t lo = row_ptr[r], hi = row_ptr[r + 1];
    uint64_t p = lo;
    while (lo < hi) {
      uint64_t mid = (lo + hi) >> 1;
      if (idx[mid] < b) lo = mid + 1; else hi = mid;
    }
    p = lo;
    flag[r] = (p < row_ptr[r + 1] && idx[p] < e) ? 0u : 1u;
  }
}

__global__ void rng_eval(uint64_t n, uint64_t seed, const uint64_t* block, const uint64_t* row, uint64_t draws,
                         const uint64_t* bound, uint64_t* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    KeyedRng g(seed, block[i], row[i]);
    if (bound) {
      out[i] = g.below(bound[i]);
    } else {
      for (uint64_t k = 0; k < draws; ++k) out[i * draws + k] = g.next();
    }
  }
}

}  // namespace


// the rank check's presence flags (repair.cpp:42-50): from the CSC slices
// (RK_PRESENCE=csr: one thread per CSR entry with a row search)
static void presence_launch(const DevMatrix& a, const Partition& p, uint32_t* flag, cudaStream_t s) {
  if (tuning().presence_csr) {
    presence_flat_kernel<<<grid_for(a.csr.nnz), kT, 0, s>>>(a.csr.ptr.get(), a.csr.idx.get(), a.csr.rows, a.csr.nnz, p,
                                                             flag);
  } else {
    const uint64_t per_block = ceil_div(a.csc.nnz, p.blocks);
    const unsigned gx = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(64, ceil_div(per_block, 256 * 4 * 2)));
    const unsigned gy = (unsigned)std::min<uint64_t>(p.blocks, 65535);
    // flags through shared memory where a block has several entries per row on average (one global
    // store per present row instead of one per entry: the kernel was bound by the L2's scattered
    // 4-byte stores, c4 92 us for 68.7 MB) and the M flags fit
    const size_t fbytes = a.csr.rows * sizeof(uint32_t);
    if (fbytes <= 48 * 1024 && per_block >= 2 * a.csr.rows)
      presence_csc_kernel<true><<<dim3((unsigned)std::max<uint64_t>(1, std::min<uint64_t>(64, ceil_div(per_block, 8192))), gy), 256, fbytes, s>>>(a.csc.ptr.get(), a.csc.idx.get(), a.csr.rows,
                                                                   a.csc.nnz, p, flag);
    else
      presence_csc_kernel<false><<<dim3(gx, gy), 256, 0, s>>>(a.csc.ptr.get(), a.csc.idx.get(), a.csr.rows,
                                                               a.csc.nnz, p, flag);
  }
  RK_LAUNCH_CHECK();
}

void repair_device(const DevMatrix& a, const Partition& p, rk_method method, uint64_t seed, RepairOut& out,
                   cudaStream_t s) {
  const uint64_t rows = a.csr.rows, D = p.blocks;
  out.lonely_counts.assign(D, 0);
  out.fallback = 0;
  out.edges.n = 0;
  if (method == RK_NONE) {  // the input unchanged, zero lonely counts (repair.cpp:167-168)
    out.edges.block.alloc(1, s); out.edges.row.alloc(1, s); out.edges.col.alloc(1, s); out.edges.mech.alloc(1, s);
    return;
  }
  const uint64_t n_flags = D * rows;
  DBuf<uint32_t> flag(n_flags ? n_flags : 1, s);
  flag.zero();
  if (a.csr.nnz) {
    presence_launch(a, p, flag.get(), s);
  }
  invert_flags<<<grid_for(n_flags), kT, 0, s>>>(flag.get(), n_flags);
  RK_LAUNCH_CHECK();
  DBuf<uint64_t> pos(n_flags + 1, s);
  exclusive_scan_u32to64(flag.get(), pos.get(), n_flags, s);
  DBuf<uint64_t> counts(D, s);
  block_counts<<<grid_for(D), kT, 0, s>>>(pos.get(), rows, D, counts.get());
  RK_LAUNCH_CHECK();
  uint64_t n_lonely = 0;
  RK_CUDA_CHECK(cudaMemcpyAsync(&n_lonely, pos.get() + n_flags, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  to_host(out.lonely_counts, counts.get(), D, s);
  sync(s);
  DBuf<uint32_t> l_block(n_lonely ? n_lonely : 1, s), l_row(n_lonely ? n_lonely : 1, s);
  if (n_lonely) {
    compact_lonely<<<grid_for(n_flags), kT, 0, s>>>(flag.get(), pos.get(), rows, n_flags, l_block.get(),
                                                    l_row.get());
    RK_LAUNCH_CHECK();
  }
  flag.release();
  pos.release();
  const uint64_t cap = method == RK_RANDOM ? n_lonely : 2 * n_lonely;
  DevEdges& E = out.edges;
  E.block.alloc(cap ? cap : 1, s);
  E.row.alloc(cap ? cap : 1, s);
  E.col.alloc(cap ? cap : 1, s);
  E.mech.alloc(cap ? cap : 1, s);
  if (n_lonely == 0) return;
  if (method == RK_RANDOM) {
    random_fill<<<grid_for(n_lonely), kT, 0, s>>>(l_block.get(), l_row.get(), n_lonely, p, seed, E.block.get(),
                                                  E.row.get(), E.col.get(), E.mech.get());
    RK_LAUNCH_CHECK();
    E.n = n_lonely;
    return;
  }
  uint64_t max_w = p.end(D - 1) - p.begin(D - 1);
  if (p.width > max_w) max_w = p.width;
  DBuf<unsigned long long> cand((rows + 63) / 64 + 1, s), nbm((max_w + 63) / 64 + 1, s), counts3(4, s);
  const uint32_t rowov_cap = (uint32_t)std::min<uint64_t>(cap + 1, 1u << 24);
  DBuf<uint32_t> rowov(rowov_cap, s);
  counts3.zero();
  ReplayArgs ra;
  ra.row_ptr = a.csr.ptr.get(); ra.col_idx = a.csr.idx.get();
  ra.col_ptr = a.csc.ptr.get(); ra.row_idx = a.csc.idx.get();
  ra.rows = rows; ra.p = p;
  ra.l_block = l_block.get(); ra.l_row = l_row.get(); ra.n_lonely = n_lonely;
  ra.seed = seed; ra.method = method == RK_NEIGHBOR ? 1 : 2;
  ra.cand = cand.get(); ra.nb = nbm.get();
  ra.rowov = rowov.get(); ra.rowov_cap = rowov_cap;
  ra.e_block = E.block.get(); ra.e_row = E.row.get(); ra.e_col = E.col.get(); ra.e_mech = E.mech.get();
  ra.out_counts = counts3.get();
  ra.spec_cand = nullptr;
  // speculation: every step's sets on the input alone, in parallel (bitmaps of n_lonely x
  // (rows + width) bits; skipped when they would not fit a modest buffer)
  const uint64_t cand_words = (rows + 63) / 64, nb_words = (max_w + 63) / 64;
  const uint64_t spec_bytes = n_lonely * (cand_words + nb_words) * 8;
  DBuf<unsigned long long> spec_bits, spec_count;
  DBuf<uint32_t> spec_col;
  DBuf<uint64_t> spec_state;
  if (tuning().repair_speculate && spec_bytes <= (uint64_t(1) << 30)) {
    spec_bits.alloc(n_lonely * (cand_words + nb_words), s);
    spec_bits.zero();
    spec_count.alloc(n_lonely, s);
    spec_col.alloc(n_lonely, s);
    spec_state.alloc(n_lonely, s);
    ra.nb_stride = nb_words;
    unsigned long long* cand_all = spec_bits.get();
    unsigned long long* nb_all = spec_bits.get() + n_lonely * cand_words;
    speculate_kernel<<<(unsigned)n_lonely, 256, 0, s>>>(ra, cand_all, nb_all, spec_count.get(), spec_col.get(),
                                                         spec_state.get());
    RK_LAUNCH_CHECK();
    ra.spec_cand = cand_all;
    ra.spec_nb = nb_all;
    ra.spec_count = spec_count.get();
    ra.spec_col = spec_col.get();
    ra.spec_state = spec_state.get();
  }
  neighbor_replay<<<1, kReplayThreads, 0, s>>>(ra);
  RK_LAUNCH_CHECK();
  unsigned long long c3[4];
  RK_CUDA_CHECK(cudaMemcpyAsync(c3, counts3.get(), sizeof c3, cudaMemcpyDeviceToHost, s));
  sync(s);
  if (c3[2]) fail(RK_RUNTIME, "neighbor replay: inserted-column scratch overflow");
  E.n = c3[0];
  out.fallback = method == RK_NEIGHBOR ? c3[1] : 0;
  out.recomputed = ra.spec_cand ? c3[3] : n_lonely;
}

void lonely_rows_device(const DevMatrix& a, const Partition& p, uint64_t d, std::vector<uint64_t>& out,
                        cudaStream_t s) {
  const uint64_t rows = a.csr.rows;
  DBuf<uint32_t> flag(rows ? rows : 1, s);
  if (rows) {
    lonely_in_block<<<grid_for(rows), kT, 0, s>>>(a.csr.ptr.get(), a.csr.idx.get(), rows, p.begin(d), p.end(d),
                                                  flag.get());
    RK_LAUNCH_CHECK();
  }
  std::vector<uint32_t> h;
  to_host(h, flag.get(), rows, s);
  sync(s);
  out.clear();
  for (uint64_t r = 0; r < rows; ++r)
    if (h[r]) out.push_back(r);
}

void rng_eval_device(uint64_t n, uint64_t seed, const uint64_t* block, const uint64_t* row, uint64_t draws,
                     const uint64_t* bound, uint64_t* out, cudaStream_t s) {
  if (!n) return;
  rng_eval<<<grid_for(n), kT, 0, s>>>(n, seed, block, row, draws, bound, out);
  RK_LAUNCH_CHECK();
}

}  // namespace rk
