// rk_pipeline.cu -- host orchestration of the device kernels.
//
//  block_stage    run_block_task for a range of blocks (proj/src/pipeline.cpp:11-16):
//                 compaction -> batched QR (tall blocks) -> W = R^T -> batched
//                 Jacobi -> finalize into the record payloads U*Sigma
//                 (block_record.cpp:69-84).
//  merge_*        proxy_svd of the concatenated records (proj/src/proxy.cpp:40-46):
//                 P^T = [payload_0^T; payload_1^T; ...] is reduced by a TSQR tree
//                 (leaves = consecutive records, fixed pairwise tree) to R_P, and a
//                 Jacobi on W = R_P^T yields sigma and U of P directly -- V of P,
//                 which run_pipeline discards (proj/src/pipeline.cpp:112), is never
//                 formed.
//  dense_svd_dev  dense_svd (proj/src/svd.cpp:365-379) with V: QR -> Jacobi on R
//                 with accumulated rotations -> completion -> apply_q -> sign.
#include <algorithm>
#include <cstring>

#include <map>

#include "rk_pipeline.cuh"

namespace rk {

size_t jacobi_smem(uint32_t rows, uint32_t g, uint32_t cols_pad, bool with_v);

namespace {

unsigned grid_for(uint64_t n, unsigned cap = 65535 * 4) {
  uint64_t g = ceil_div(n, 256);
  if (g == 0) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

__global__ void nonfinite_blocks(const uint64_t* col_ptr, const double* val, uint64_t cols, Partition p,
                                 uint32_t* bad) {
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < cols;
       c += (uint64_t)gridDim.x * blockDim.x) {
    for (uint64_t k = col_ptr[c]; k < col_ptr[c + 1]; ++k)
      if (!isfinite(val[k])) { bad[p.block_of(c)] = 1u; break; }
  }
}

__global__ void count_nonfinite(const double* x, uint64_t n, unsigned* flag) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (!isfinite(x[i])) *flag = 1u;
}

// [ra; rb] (heights ha, hb; column-major with ld n) -> column-major (ha+hb) x n
__global__ void stack_r(const double* ra, uint32_t ha, const double* rb, uint32_t hb, uint32_t n, double* out) {
  const uint32_t h = ha + hb;
  const uint64_t total = (uint64_t)h * n;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = (uint32_t)(t % h), c = (uint32_t)(t / h);
    out[t] = i < ha ? ra[i + (uint64_t)c * n] : rb[(i - ha) + (uint64_t)c * n];
  }
}

// leaf = records [r0, r1) of P^T stacked: column-major h x n
// the leaf's stacked P^T rows: the first eff[rec] columns of each record (row-major
// n x kept[rec]); the columns past eff are exactly zero (see record_effective_cols)
__global__ void gather_leaf(const double* payload, const uint64_t* off, const uint32_t* kept, const uint32_t* eff,
                            uint32_t r0, uint32_t r1, uint32_t n, uint32_t h, double* out) {
  uint32_t base = 0;
  for (uint32_t rec = r0; rec < r1; ++rec) {
    const uint32_t k = kept[rec], e = eff[rec];
    const double* src = payload + off[rec];
    const uint64_t total = (uint64_t)e * n;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
         t += (uint64_t)gridDim.x * blockDim.x) {
      const uint32_t j = (uint32_t)(t % e), col = (uint32_t)(t / e);  // payload: row-major n x k
      out[(base + j) + (uint64_t)col * h] = src[(uint64_t)col * k + j];
    }
    base += e;
  }
}


// row-major rows x k (payload) -> column-major rows x k at dst (ld rows)
__global__ void rowmajor_to_colmajor(const double* src, uint32_t rows, uint32_t k, double* dst) {
  const uint64_t total = (uint64_t)rows * k;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = (uint32_t)(t % rows), c = (uint32_t)(t / rows);
    dst[t] = src[(uint64_t)i * k + c];
  }
}

// square column-major transpose (out = in^T), out has leading dimension n
__global__ void transpose_sq(const double* in, uint32_t n, double* out) {
  const uint64_t total = (uint64_t)n * n;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = (uint32_t)(t % n), c = (uint32_t)(t / n);
    out[t] = in[c + (uint64_t)i * n];
  }
}

__global__ void sign_kernel(double* u, uint32_t rows, uint32_t k, double* v, uint32_t vrows) {
  const int lane = threadIdx.x & 31;
  for (uint32_t j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < k; j += (gridDim.x * blockDim.x) >> 5) {
    double best = -1.0;
    uint32_t arg = 0;
    for (uint32_t i = lane; i < rows; i += 32) {
      const double mag = fabs(u[(uint64_t)i * k + j]);
      if (mag > best) { best = mag; arg = i; }
    }
    for (int o = 16; o; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const uint32_t oa = __shfl_xor_sync(0xffffffffu, arg, o);
      if (ob > best || (ob == best && oa < arg)) { best = ob; arg = oa; }
    }
    if (rows && u[(uint64_t)arg * k + j] < 0.0) {
      for (uint32_t i = lane; i < rows; i += 32) u[(uint64_t)i * k + j] = -u[(uint64_t)i * k + j];
      if (v)
        for (uint32_t i = lane; i < vrows; i += 32) v[(uint64_t)i * k + j] = -v[(uint64_t)i * k + j];
    }
  }
}

__global__ void identity_colmajor(double* v, uint32_t n, uint32_t ld, uint32_t ncols) {
  const uint64_t total = (uint64_t)ld * ncols;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = (uint32_t)(t % ld), c = (uint32_t)(t / ld);
    v[t] = (i == c && i < n) ? 1.0 : 0.0;
  }
}

// column-major (rows x cols, ld) -> row-major rows x cols
__global__ void colmajor_to_rowmajor(const double* src, uint64_t ld, uint32_t rows, uint32_t cols, double* dst) {
  const uint64_t total = (uint64_t)rows * cols;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = (uint32_t)(t / cols), c = (uint32_t)(t % cols);
    dst[t] = src[i + (uint64_t)c * ld];
  }
}

struct JacobiStats {
  uint64_t sweeps = 0, rotations = 0;
  bool failed = false;
  double residual = 0.0;
};

std::vector<JacobiStats> read_stats(const uint64_t* d_stats, size_t n, cudaStream_t s) {
  std::vector<uint64_t> h;
  to_host(h, d_stats, 8 * n, s);
  sync(s);
  std::vector<JacobiStats> out(n);
  for (size_t i = 0; i < n; ++i) {
    out[i].sweeps = h[8 * i];
    out[i].rotations = h[8 * i + 1];
    out[i].failed = h[8 * i + 2] != 0;
    std::memcpy(&out[i].residual, &h[8 * i + 3], 8);
  }
  return out;
}

std::string residual_text(double r) { return std::to_string(r); }

[[noreturn]] void throw_convergence(double residual) {
  fail(RK_CONVERGENCE, "one-sided Jacobi did not converge (residual " + residual_text(residual) + ")", residual);
}

void complete_and_sign(Ctx& c, double* u, uint32_t rows, uint32_t k, const uint8_t* d_def, double* v,
                       uint32_t vrows) {
  cudaStream_t s = c.stream;
  DBuf<int> fail_flag(1, s);
  fail_flag.zero();
  complete_columns_device(u, rows, k, d_def, fail_flag.get(), s);
  int h = 0;
  RK_CUDA_CHECK(cudaMemcpyAsync(&h, fail_flag.get(), sizeof h, cudaMemcpyDeviceToHost, s));
  sync(s);
  if (h) fail(RK_CONVERGENCE, "orthonormal completion has no independent direction (residual 0.000000)", 0.0);
  sign_rows(u, rows, k, v, vrows, s);
}

bool any_flag(const uint8_t* d, uint64_t n, cudaStream_t s) {
  std::vector<uint8_t> h;
  to_host(h, d, n, s);
  sync(s);
  for (uint8_t x : h)
    if (x) return true;
  return false;
}

}  // namespace

void sign_rows(double* u, uint32_t rows, uint32_t k, double* v, uint32_t vrows, cudaStream_t s) {
  if (!k) return;
  sign_kernel<<<grid_for((uint64_t)k * 32), 256, 0, s>>>(u, rows, k, v, vrows);
  RK_LAUNCH_CHECK();
}

void check_finite_or_throw(const double* x, uint64_t n, const char* what, cudaStream_t s) {
  if (!n) return;
  DBuf<unsigned> flag(1, s);
  flag.zero();
  count_nonfinite<<<grid_for(n), 256, 0, s>>>(x, n, flag.get());
  RK_LAUNCH_CHECK();
  unsigned h = 0;
  RK_CUDA_CHECK(cudaMemcpyAsync(&h, flag.get(), sizeof h, cudaMemcpyDeviceToHost, s));
  sync(s);
  if (h) fail(RK_INVALID_ARGUMENT, what);
}

// ---------------------------------------------------------------------------
// block stage

void block_stage(Ctx& c, const DevMatrix& a, const Partition& p, uint64_t d_lo, uint64_t d_hi, uint64_t keep,
                 BlockStageResult& out, BlockApiOut* api) {
  cudaStream_t s = c.stream;
  const uint32_t M = (uint32_t)a.csr.rows;
  const uint64_t nblk = d_hi - d_lo;
  out.offset.assign(nblk, 0);
  out.kept.assign(nblk, 0);
  out.eff.assign(nblk, 0);
  out.failures.assign(nblk, std::string());
  if (nblk == 0) return;

  // k per block (run_block_task, pipeline.cpp:12-13) and the densify cap (dense_matrix.cpp:62-75)
  std::vector<char> skip(nblk, 0);
  for (uint64_t i = 0; i < nblk; ++i) {
    const uint64_t d = d_lo + i;
    const uint64_t w = p.end(d) - p.begin(d);
    const uint64_t k_full = std::min<uint64_t>(M, w);
    const uint64_t k = keep == 0 ? k_full : std::min(keep, k_full);
    if (k == 0) {
      out.failures[i] = "block_svd: keep must be >= 1";
      skip[i] = 1;
    } else if ((uint64_t)M * w > (uint64_t(1) << 26)) {
      out.failures[i] = "dense_of: " + std::to_string(M) + "x" + std::to_string(w) + " exceeds the densification cap";
      skip[i] = 1;
    }
    out.kept[i] = skip[i] ? 0 : (uint32_t)k;
  }
  // non-finite values (svd.cpp:384-386)
  {
    DBuf<uint32_t> bad(p.blocks, s);
    bad.zero();
    if (a.csc.nnz) {
      nonfinite_blocks<<<grid_for(a.csc.cols), 256, 0, s>>>(a.csc.ptr.get(), a.csc.val.get(), a.csc.cols, p,
                                                            bad.get());
      RK_LAUNCH_CHECK();
    }
    std::vector<uint32_t> hb;
    to_host(hb, bad.get() + d_lo, nblk, s);
    sync(s);
    prof_mark(s, "blk nonfinite+sync");
    for (uint64_t i = 0; i < nblk; ++i)
      if (hb[i] && !skip[i]) {
        out.failures[i] = "block_svd: block has non-finite values";
        skip[i] = 1;
        out.kept[i] = 0;
      }
  }
  uint64_t total_payload = 0;
  for (uint64_t i = 0; i < nblk; ++i) {
    out.offset[i] = total_payload;
    total_payload += (uint64_t)M * out.kept[i];
  }
  out.payload.alloc(total_payload ? total_payload : 1, s);
  if (M == 0) return;

  const uint32_t cols_pad_full = jacobi_cols_pad(M, M, false, c.smem_optin);
  std::vector<char> done(nblk, 0);
  for (uint64_t i = 0; i < nblk; ++i) done[i] = skip[i];

  // the Jacobi width for a wide block of n < M real columns: planned for n rounded up
  // to 32 (few distinct widths, so few launches)
  std::map<std::pair<uint32_t, uint32_t>, uint32_t> pad_cache;
  auto narrow_pad = [&](uint32_t n, uint32_t rows) {
    const uint32_t r = std::min<uint32_t>(M, (n + 31) & ~31u);
    auto it = pad_cache.find({rows, r});
    if (it != pad_cache.end()) return it->second;
    const uint32_t pd = std::min<uint32_t>(cols_pad_full, jacobi_cols_pad(rows, r, false, c.smem_optin));
    pad_cache[{rows, r}] = pd;
    return pd;
  };

  // Wide blocks (compacted height n_d < M) on the reduced route: X = T^T (M x n_d)
  // = Q R by Householder QR, the Jacobi on R (n_d x n_d: columns of length n_d, not M),
  // then the slot = Q [R V; 0] = U Sigma (svd_tall's own QR -> Jacobi -> apply_q,
  // svd.cpp:316-332, applied to the tall X). Each slot has its Jacobi matrix (rows
  // padded to a multiple of 32 with zero rows) and its factored QR.
  struct Reduced {
    std::vector<double*> mats;
    std::vector<uint32_t> rows;
    std::vector<QrJob> qr;
  };

  // Jacobi + finalize of a set of W slots; records stats and writes payloads
  std::vector<double> sigma_host;  // sorted sigma of the Gram-route slots (read with the Jacobi stats)
  auto jacobi_finalize = [&](std::vector<double*>& slots, std::vector<uint32_t>& cols, std::vector<uint64_t>& blocks,
                             bool gram_ok, double* sigma_all /* nullable: slots x cols_pad */,
                             const std::vector<const uint32_t*>* row_perms = nullptr,
                             const Reduced* red = nullptr /* per slot; mats[q] == nullptr: not reduced */) {
    const size_t nb = slots.size();
    DBuf<double> alpha((uint64_t)nb * cols_pad_full, s);
    DBuf<uint64_t> stats(8 * nb, s);
    DBuf<uint32_t> order((uint64_t)nb * cols_pad_full, s);
    DBuf<double> fscratch((uint64_t)nb * cols_pad_full, s);
    stats.zero();
    // A wide block (n_d < M real columns: the compacted Householder route) runs its
    // tournament over a width planned for its own n_d, not over M: the columns past
    // n_d are zero and would only lengthen every sweep (c3: ~130 of 512). The width
    // is a function of the block's own data, so results do not depend on batching.
    // Jobs of one width share a launch; the finalize still sees cols_pad_full
    // columns (the slot's tail is zero: sigma 0, deficient).
    std::map<std::pair<uint32_t, uint32_t>, std::vector<JacobiJob>> by_pad;
    std::vector<uint32_t> jrows(nb, M);
    std::vector<ApplyQJob> aq;
    for (size_t q = 0; q < nb; ++q) {
      const bool reduced = red && red->mats[q];
      JacobiJob j{};
      j.w = reduced ? red->mats[q] : slots[q];
      j.v = nullptr;
      j.rows = reduced ? red->rows[q] : M;
      j.cols = std::max<uint32_t>(cols[q], 1);
      j.cols_pad = (j.cols >= M && !reduced) ? cols_pad_full : narrow_pad(j.cols, j.rows);
      j.alpha = alpha.get() + (uint64_t)q * cols_pad_full;
      j.stats = stats.get() + 8 * q;
      j.gram_ok = gram_ok ? 1u : 0u;
      j.rows_nz = reduced ? std::max<uint32_t>(cols[q], 1) : 0u;  // R is n_d x n_d
      jrows[q] = j.rows;
      by_pad[{j.rows, j.cols_pad}].push_back(j);
      if (reduced) aq.push_back({red->qr[q], red->mats[q], j.rows, cols[q], slots[q], qr_panel_nb(M)});
    }
    RK_CUDA_CHECK(cudaEventRecord(c.ev[9], s));
    {
      RK_NVTX("rk.blocks.jacobi");
      // launches sized so their matrices stay L2-resident (the kernel re-stages its
      // column groups every tournament step): c3's 512 reduced matrices are 168 MB
      const uint64_t cap = tuning().jacobi_chunk_mb << 20;
      {
        // one launch of the shared-memory kernel over every width class; the per-width
        // launches below then only certify
        std::vector<JacobiJob> every;
        for (auto& kv : by_pad)
          for (const JacobiJob& j : kv.second)
            if (jacobi_smem_fits(j, c.smem_optin)) every.push_back(j);
        if (!c.side) {
          RK_CUDA_CHECK(cudaStreamCreateWithFlags(&c.side, cudaStreamNonBlocking));
          for (auto& ev : c.side_ev) RK_CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        }
        const SideStream side{c.side, c.side_ev[0], c.side_ev[1]};
        if (!every.empty() && jacobi_smem_try(every, s, c.smem_optin, &side))
          for (auto& kv : by_pad)
            for (JacobiJob& j : kv.second)
              if (jacobi_smem_fits(j, c.smem_optin)) j.pre = 1;
      }
      for (auto& kv : by_pad) {
        std::vector<JacobiJob>& all = kv.second;
        const uint64_t per = (uint64_t)kv.first.first * kv.first.second * sizeof(double);
        const size_t n_chunk = cap ? std::max<size_t>(c.num_sms, cap / std::max<uint64_t>(per, 1)) : all.size();
        for (size_t i0 = 0; i0 < all.size(); i0 += n_chunk) {
          std::vector<JacobiJob> part(all.begin() + i0, all.begin() + std::min(all.size(), i0 + n_chunk));
          jacobi_batched(part, s, c.num_sms, c.smem_optin);
        }
      }
    }
    RK_CUDA_CHECK(cudaEventRecord(c.ev[10], s));
    apply_q_batched(aq, s);  // reduced slots: U Sigma = Q [R V; 0]
    prof_mark(s, "blk jacobi");
    std::vector<FinalJob> fj(nb);
    for (size_t q = 0; q < nb; ++q) {
      const uint64_t i = blocks[q];
      FinalJob& f = fj[q];
      std::memset(&f, 0, sizeof f);
      f.w = slots[q];
      f.rows = M;
      f.cols = cols_pad_full;
      f.k = out.kept[i];
      out.eff[i] = std::min<uint32_t>(out.kept[i], std::max<uint32_t>(cols[q], 1));  // columns past cols[q] are zero
      f.payload = out.payload.get() + out.offset[i];
      f.order = order.get() + (uint64_t)q * cols_pad_full;
      f.scratch = fscratch.get() + (uint64_t)q * cols_pad_full;
      f.sigma_all = sigma_all ? sigma_all + (uint64_t)q * cols_pad_full : nullptr;
      f.row_perm = row_perms ? (*row_perms)[q] : nullptr;
      if (api) {
        f.u = api->u.get() + out.offset[i];
        f.sigma = api->sigma.get() + i * (uint64_t)M;
        f.deficient = api->deficient.get() + i * (uint64_t)M;
      }
    }
    finalize_batched(fj, s);
    if (sigma_all) to_host(sigma_host, sigma_all, (uint64_t)nb * cols_pad_full, s);  // read with the stats
    std::vector<JacobiStats> js = read_stats(stats.get(), nb, s);  // synchronizes
    prof_mark(s, "blk finalize+stats");
    float ms_j = 0;
    cudaEventElapsedTime(&ms_j, c.ev[9], c.ev[10]);
    out.jacobi_ms += ms_j;
    for (size_t q = 0; q < nb; ++q) {
      out.sweeps_max = std::max(out.sweeps_max, js[q].sweeps);
      out.sweeps_sum += js[q].sweeps;
      out.rotations += js[q].rotations;
      const double cA = cols[q], Md = jrows[q];
      out.jacobi_flops += (double)js[q].sweeps * (cA * (cA - 1) / 2 * 2 * Md + 2 * Md * cA) +
                          (double)js[q].rotations * 6 * Md;
      if (js[q].failed) {
        out.failures[blocks[q]] = "one-sided Jacobi did not converge (residual " + residual_text(js[q].residual) + ")";
        out.conv_residual = js[q].residual;
      }
    }
    return js;
  };

  // 40 % of the free device memory; the estimate avoids cudaMemGetInfo (2-3 ms per
  // call on the B200 box) unless the whole stage may not fit in it
  const uint64_t need_all = nblk * (uint64_t)M * cols_pad_full * 8 * 2;
  const uint64_t budget = std::max<uint64_t>((uint64_t)(device_free_bytes(c, need_all * 3) * 0.4), 256ull << 20);
  prof_mark(s, "blk budget");

  // compacted row counts (multi-entry columns, merged single-entry rows) of every block:
  // the Householder route's plan, and a rank bound for route 1 (rank <= n_rows)
  DBuf<uint32_t> counts(2 * nblk, s);
  DBuf<double> single(nblk * (uint64_t)M, s);
  compaction_counts(a, p, d_lo, d_hi, counts.get(), single.get(), s);
  std::vector<uint32_t> hc;
  to_host(hc, counts.get(), 2 * nblk, s);
  sync(s);

  // ---- route 1: W = chol(A_d A_d^T), accepted when kappa <= kappa_max(M) ----
  if (gram_route_enabled() && M <= cholesky_max_rows()) {
    RK_NVTX("rk.blocks.gram_route");
    const double kmax = kappa_max(M);
    const uint64_t per_block = (uint64_t)M * cols_pad_full * 8 * 2;
    const uint64_t chunk = std::max<uint64_t>(1, budget / per_block);
    for (uint64_t i0 = 0; i0 < nblk; i0 += chunk) {
      const uint64_t i1 = std::min(nblk, i0 + chunk), nb = i1 - i0;
      // a block whose compacted height is below M is rank-deficient: its Gram is singular
      // and the Cholesky would only reject it (c3: every block, rank ~127 of 512)
      bool any = false;
      for (uint64_t i = i0; i < i1 && !any; ++i) any = !skip[i] && hc[2 * i] + hc[2 * i + 1] >= M;
      if (!any) continue;
      DBuf<double> W(nb * M * cols_pad_full, s);
      W.zero();
      RK_CUDA_CHECK(cudaEventRecord(c.ev[8], s));
      sparse_gram(a, p, d_lo + i0, nb, W.get(), (uint64_t)M * cols_pad_full, s);
      // rows by descending Gram diagonal (fewer Jacobi sweeps); U's rows are
      // un-permuted by the finalize (FinalJob::row_perm)
      DBuf<uint32_t> perm;
      const bool order = diag_order_enabled() && M <= 1280;
      if (order) {
        perm.alloc(nb * M, s);
        DBuf<double> Wp(nb * M * cols_pad_full, s);
        if (cols_pad_full != M) Wp.zero();
        diag_order(W.get(), (uint64_t)M * cols_pad_full, M, nb, perm.get(), Wp.get(), s);
        W = std::move(Wp);
      }
      std::vector<double*> ptrs(nb);
      for (uint64_t q = 0; q < nb; ++q) ptrs[q] = W.get() + q * M * cols_pad_full;
      DBuf<double*> dptrs(nb, s);
      DBuf<uint32_t> status(nb, s);
      DBuf<double> ratio(nb, s);
      to_device(dptrs.get(), ptrs.data(), nb, s);
      cholesky_batched(dptrs.get(), (uint32_t)nb, M, status.get(), ratio.get(), s);
      RK_CUDA_CHECK(cudaEventRecord(c.ev[11], s));
      std::vector<uint32_t> hst;
      std::vector<double> hrat;
      to_host(hst, status.get(), nb, s);
      to_host(hrat, ratio.get(), nb, s);
      sync(s);
      prof_mark(s, "blk gram+chol+sync");
      float ms_g = 0;
      cudaEventElapsedTime(&ms_g, c.ev[8], c.ev[11]);
      out.qr_ms += ms_g;
      out.qr_flops += (double)nb * M * (double)M * M / 3.0;
      std::vector<double*> slots;
      std::vector<uint32_t> cols;
      std::vector<uint64_t> blocks;
      std::vector<const uint32_t*> perms;
      for (uint64_t q = 0; q < nb; ++q) {
        const uint64_t i = i0 + q;
        if (skip[i] || hst[q] != 0 || !(hrat[q] <= kmax)) continue;
        slots.push_back(ptrs[q]);
        cols.push_back(M);
        blocks.push_back(i);
        perms.push_back(order ? perm.get() + q * M : nullptr);
      }
      if (slots.empty()) continue;
      DBuf<double> sig((uint64_t)slots.size() * cols_pad_full, s);
      jacobi_finalize(slots, cols, blocks, true, sig.get(), &perms);
      const std::vector<double>& hs = sigma_host;
      for (size_t q = 0; q < slots.size(); ++q) {
        const double smax = hs[q * cols_pad_full], smin = hs[q * cols_pad_full + M - 1];
        const uint64_t i = blocks[q];
        if (!out.failures[i].empty()) {  // redo on the Householder route
          out.failures[i].clear();
          continue;
        }
        if (smin > 0.0 && smax / smin <= kmax) done[i] = 1;
      }
    }
  }

  // ---- route 2: Householder (compaction -> TSQR -> W = R^T), as the reference ----
  std::vector<uint64_t> todo;
  for (uint64_t i = 0; i < nblk; ++i)
    if (!done[i]) todo.push_back(i);
  if (todo.empty()) return;
  const uint64_t aux_sz = 2 * (uint64_t)M + (ceil_div(M, 16) + 1) * 256;
  // TSQR leaf height of the tall blocks: at least 2M, so every leaf is tall (a wide
  // leaf makes the pairwise combines, ~4/3 M^3 each, dominate: c5 3x the flops)
  const uint32_t kLeafRows = std::max<uint32_t>(768, std::min<uint32_t>(2 * M, qr_max_rows()));
  // the reduced route pays when the padded R is clearly shorter than M (RK_WIDE_REDUCE=0: off)
  const bool reduce_on = tuning().wide_reduce;
  // R's rows padded with zero rows to a power of two (>= 32): the Jacobi kernel holds
  // Q x E (both powers of two) elements per column, so such a height takes its exact
  // (unpredicated) path at no extra cost per round (RK_WIDE_ROWS=32: multiples of 32)
  const bool rows_pow2 = tuning().wide_rows_pow2;
  auto red_rows = [&](uint32_t n) -> uint32_t {
    if (!rows_pow2) return (n + 31) & ~31u;
    uint32_t r = 32;
    while (r < n) r *= 2;
    return r;
  };
  auto reduce_wide = [&](uint32_t n) { return reduce_on && n >= 2 && red_rows(n) < M && red_rows(n) * 4 <= 3 * M; };

  RK_NVTX("rk.blocks.householder_route");
  size_t t0 = 0;
  while (t0 < todo.size()) {
    std::vector<BlockPlan> plans;
    uint64_t staging = 0, wdoubles = 0, planned = 0;
    size_t t1 = t0;
    for (; t1 < todo.size(); ++t1) {
      const uint64_t i1 = todo[t1];
      BlockPlan pl;
      pl.block = d_lo + i1;
      pl.n_multi = hc[2 * i1];
      pl.n_single = hc[2 * i1 + 1];
      pl.n_rows = pl.n_multi + pl.n_single;
      pl.tall = pl.n_rows > M;
      // staging + the TSQR forest (leaf R factors, then stacked pairs and their R
      // factors alive together: <= 3 M x M per leaf) + the Jacobi slot; a reduced
      // wide block stages X = T^T (M x n_d) and its R (rows_pad x n_pad)
      const uint64_t n_leaves = pl.tall ? ceil_div(pl.n_rows, kLeafRows) : 0;
      const bool red = !pl.tall && reduce_wide(pl.n_rows);
      const uint64_t rp = red_rows(pl.n_rows);
      const uint64_t need = (pl.tall ? (uint64_t)pl.n_rows * M + 3 * n_leaves * ((uint64_t)M * M + aux_sz) : 0) +
                            (red ? (uint64_t)pl.n_rows * M + rp * rp + aux_sz : 0) +
                            (uint64_t)M * cols_pad_full + aux_sz;
      if (!plans.empty() && (planned + need) * 8 > budget) break;
      planned += need;
      pl.offset = staging;
      staging += (pl.tall || red) ? (uint64_t)pl.n_rows * M : 0;
      wdoubles += (uint64_t)M * cols_pad_full + aux_sz;
      plans.push_back(pl);
    }
    const size_t nb = plans.size();
    // one padded width per M (not per chunk): the Jacobi group layout, and with it
    // the rotation order and rounding, depends only on the block's own data
    const uint32_t cols_pad = cols_pad_full;
    DBuf<double> st(staging ? staging : 1, s);
    DBuf<double> W((uint64_t)nb * M * cols_pad, s);
    if (staging) st.zero();
    W.zero();
    std::vector<BlockPlan> fill_tall, fill_wide;
    for (size_t q = 0; q < nb; ++q) {
      if (plans[q].tall || reduce_wide(plans[q].n_rows)) {
        fill_tall.push_back(plans[q]);  // staged (T for tall, X = T^T for reduced wide)
      } else {
        BlockPlan w = plans[q];
        w.offset = (uint64_t)q * M * cols_pad;  // W = T^T written straight into the Jacobi slot
        fill_wide.push_back(w);
      }
    }
    RK_CUDA_CHECK(cudaEventRecord(c.ev[8], s));
    compaction_fill(a, p, fill_tall, d_lo, single.get(), st.get(), s);
    compaction_fill(a, p, fill_wide, d_lo, single.get(), W.get(), s);
    // tall blocks: TSQR of T_d over row leaves of at most kLeafRows rows (factored in
    // place), pairwise tree, then W = R^T into the block's Jacobi slot
    {
      std::vector<std::vector<LeafRef>> trees;
      std::vector<size_t> tree_q;
      for (size_t q = 0; q < nb; ++q) {
        if (!plans[q].tall) continue;
        const uint32_t nr = plans[q].n_rows;
        const uint32_t L = (uint32_t)ceil_div(nr, kLeafRows);
        std::vector<LeafRef> leaves;
        for (uint32_t i = 0; i < L; ++i) {
          const uint64_t r0 = (uint64_t)nr * i / L, r1 = (uint64_t)nr * (i + 1) / L;
          leaves.push_back({st.get() + plans[q].offset + r0, nr, (uint32_t)(r1 - r0), 0u});
        }
        trees.push_back(std::move(leaves));
        tree_q.push_back(q);
        out.qr_flops += 2.0 * nr * (double)M * M - 2.0 / 3.0 * (double)M * M * M;
      }
      if (!trees.empty()) {
        std::vector<DBuf<double>> roots;
        tsqr_forest(c, M, trees, roots);
        for (size_t t = 0; t < trees.size(); ++t) {
          transpose_sq<<<grid_for((uint64_t)M * M), 256, 0, s>>>(roots[t].get(), M,
                                                                 W.get() + (uint64_t)tree_q[t] * M * cols_pad);
          RK_LAUNCH_CHECK();
        }
      }
    }
    // reduced wide blocks: QR of X = T^T in the staging buffer, R into its Jacobi matrix
    Reduced red;
    red.mats.assign(nb, nullptr);
    red.rows.assign(nb, 0);
    red.qr.assign(nb, QrJob{});
    DBuf<double> rmats, raux;
    {
      uint64_t rtot = 0, ntot = 0;
      for (size_t q = 0; q < nb; ++q)
        if (!plans[q].tall && reduce_wide(plans[q].n_rows)) {
          const uint64_t rp = red_rows(plans[q].n_rows);
          rtot += rp * narrow_pad(plans[q].n_rows, (uint32_t)rp);
          ++ntot;
        }
      if (ntot) {
        rmats.alloc(rtot, s);
        rmats.zero();
        raux.alloc(ntot * aux_sz, s);
        std::vector<QrJob> qj;
        std::vector<RJob> rj;
        uint64_t ro = 0, ao = 0;
        for (size_t q = 0; q < nb; ++q) {
          const uint32_t n = plans[q].n_rows;
          if (plans[q].tall || !reduce_wide(n)) continue;
          const uint32_t rp = red_rows(n);
          QrJob j;
          j.a = st.get() + plans[q].offset; j.lda = M; j.m = M; j.n = n;
          j.diag = raux.get() + ao; j.beta = j.diag + n; j.tmat = j.diag + 2 * (uint64_t)n;
          ao += aux_sz;
          qj.push_back(j);
          red.qr[q] = j;
          red.mats[q] = rmats.get() + ro;
          red.rows[q] = rp;
          ro += (uint64_t)rp * narrow_pad(n, rp);
          RJob r;
          r.a = j.a; r.lda = j.lda; r.diag = j.diag; r.m = M; r.n = n; r.w = red.mats[q]; r.ldw = rp;
          rj.push_back(r);
          out.qr_flops += 2.0 * M * (double)n * n - 2.0 / 3.0 * (double)n * n * n;
        }
        qr_batched(qj, s, c.num_sms);
        r_extract_batched(rj, /*transpose=*/false, s);
      }
    }
    RK_CUDA_CHECK(cudaEventRecord(c.ev[11], s));
    std::vector<double*> slots(nb);
    std::vector<uint32_t> cols(nb);
    std::vector<uint64_t> blocks(nb);
    for (size_t q = 0; q < nb; ++q) {
      slots[q] = W.get() + (uint64_t)q * M * cols_pad;
      cols[q] = std::min<uint32_t>(plans[q].n_rows, M);
      blocks[q] = plans[q].block - d_lo;
    }
    jacobi_finalize(slots, cols, blocks, false, nullptr, nullptr, &red);
    float ms_qr = 0;
    cudaEventElapsedTime(&ms_qr, c.ev[8], c.ev[11]);
    out.qr_ms += ms_qr;
    t0 = t1;
  }
}

// ---------------------------------------------------------------------------
// merge tree

std::vector<TreeLeaf> merge_leaves(const std::vector<uint32_t>& kept, uint32_t M) {
  std::vector<TreeLeaf> leaves;
  size_t r0 = 0;
  while (r0 < kept.size()) {
    size_t r1 = r0;
    uint32_t h = 0;
    while (r1 < kept.size() && h < M) h += kept[r1++];
    if (h > 0) leaves.push_back({(uint32_t)r0, (uint32_t)r1, h});
    r0 = r1;
  }
  return leaves;
}

namespace {

// QR every matrix of a level in place and extract the R factors (n x n column-major,
// rows >= min(h, n) zero); heights become min(h, n)
void qr_level(Ctx& c, std::vector<LeafRef>& mats, std::vector<DBuf<double>>& rs, uint32_t n) {
  cudaStream_t s = c.stream;
  const size_t cnt = mats.size();
  const uint64_t aux_sz = 2 * (uint64_t)n + (ceil_div(n, 16) + 1) * 256;
  DBuf<double> aux(cnt * aux_sz, s);
  std::vector<QrJob> qj;
  std::vector<RJob> rj;
  rs.clear();
  rs.reserve(cnt);
  for (size_t q = 0; q < cnt; ++q) {
    QrJob j;
    j.a = mats[q].a; j.lda = mats[q].lda; j.m = mats[q].m; j.n = n; j.split = mats[q].split;
    j.diag = aux.get() + q * aux_sz; j.beta = j.diag + n; j.tmat = j.diag + 2 * n;
    qj.push_back(j);
    rs.emplace_back((uint64_t)n * n, s);
    RJob r;
    r.a = j.a; r.lda = j.lda; r.diag = j.diag; r.m = j.m; r.n = n; r.w = rs.back().get(); r.ldw = n;
    rj.push_back(r);
  }
  qr_batched(qj, s, c.num_sms);
  r_extract_batched(rj, /*transpose=*/false, s);
  for (size_t q = 0; q < cnt; ++q) mats[q].m = std::min<uint32_t>(mats[q].m, n);
}

}  // namespace

// pairwise levels over the nodes of every tree, batched across trees: (0,1), (2,3), ...;
// an odd last node is carried up unchanged. Leaves each tree with one node.
void forest_reduce(Ctx& c, uint32_t n, std::vector<std::vector<DBuf<double>>>& nodes,
                   std::vector<std::vector<uint32_t>>& heights) {
  cudaStream_t s = c.stream;
  const size_t T = nodes.size();
  for (;;) {
    std::vector<LeafRef> stacked;
    std::vector<DBuf<double>> bufs;
    std::vector<std::pair<size_t, size_t>> where;  // (tree, pair index)
    for (size_t t = 0; t < T; ++t) {
      for (size_t q = 0; q + 1 < nodes[t].size(); q += 2) {
        const uint32_t h = heights[t][q] + heights[t][q + 1];
        bufs.emplace_back((uint64_t)h * n, s);
        stack_r<<<grid_for((uint64_t)h * n), 256, 0, s>>>(nodes[t][q].get(), heights[t][q], nodes[t][q + 1].get(),
                                                           heights[t][q + 1], n, bufs.back().get());
        RK_LAUNCH_CHECK();
        // a full n x n top triangle lets the combine skip the rows that stay zero
        stacked.push_back({bufs.back().get(), h, h, heights[t][q] == n ? n : 0u});
        where.push_back({t, q / 2});
      }
    }
    if (stacked.empty()) break;
    std::vector<DBuf<double>> out;
    qr_level(c, stacked, out, n);
    std::vector<std::vector<DBuf<double>>> next(T);
    std::vector<std::vector<uint32_t>> nh(T);
    size_t k = 0;
    for (size_t t = 0; t < T; ++t) {
      const size_t pairs = nodes[t].size() / 2;
      for (size_t q = 0; q < pairs; ++q, ++k) {
        next[t].push_back(std::move(out[k]));
        nh[t].push_back(stacked[k].m);
      }
      if (nodes[t].size() & 1) {
        next[t].push_back(std::move(nodes[t].back()));
        nh[t].push_back(heights[t].back());
      }
    }
    nodes = std::move(next);
    heights = std::move(nh);
  }
}

void tsqr_forest(Ctx& c, uint32_t n, std::vector<std::vector<LeafRef>>& leaves, std::vector<DBuf<double>>& roots) {
  cudaStream_t s = c.stream;
  const size_t T = leaves.size();
  // level 0: every leaf of every tree in one batch
  std::vector<LeafRef> flat;
  std::vector<size_t> owner;
  for (size_t t = 0; t < T; ++t)
    for (const LeafRef& L : leaves[t]) {
      flat.push_back(L);
      owner.push_back(t);
    }
  std::vector<DBuf<double>> rs;
  qr_level(c, flat, rs, n);
  std::vector<std::vector<DBuf<double>>> nodes(T);
  std::vector<std::vector<uint32_t>> heights(T);
  for (size_t q = 0; q < flat.size(); ++q) {
    nodes[owner[q]].push_back(std::move(rs[q]));
    heights[owner[q]].push_back(flat[q].m);
  }
  forest_reduce(c, n, nodes, heights);
  roots.clear();
  for (size_t t = 0; t < T; ++t) roots.push_back(std::move(nodes[t][0]));
}

void merge_subtree(Ctx& c, const double* payload, const std::vector<uint64_t>& offset,
                   const std::vector<uint32_t>& kept, uint32_t M, const std::vector<TreeLeaf>& leaves,
                   size_t leaf_lo, size_t leaf_hi, DBuf<double>& r_out, const std::vector<uint32_t>* eff_hint) {
  cudaStream_t s = c.stream;
  DBuf<uint64_t> doff(offset.size(), s);
  DBuf<uint32_t> dkept(kept.size(), s);
  to_device(doff.get(), offset.data(), offset.size(), s);
  to_device(dkept.get(), kept.data(), kept.size(), s);
  // the leaves keep the record grouping of `kept` (data-independent, so a shard's
  // subtree is a node of the whole tree), but stack only each record's nonzero columns
  const uint32_t rec_lo = leaves[leaf_lo].r0, rec_hi = leaves[leaf_hi - 1].r1;
  const std::vector<uint32_t> heff = record_eff_cols(payload, offset, kept, M, rec_lo, rec_hi, s, eff_hint);
  DBuf<uint32_t> deff(kept.size(), s);
  to_device(deff.get(), heff.data(), heff.size(), s);
  std::vector<DBuf<double>> bufs;
  std::vector<std::vector<LeafRef>> tree(1);
  for (size_t l = leaf_lo; l < leaf_hi; ++l) {
    const TreeLeaf& L = leaves[l];
    uint32_t h = 0;
    for (uint32_t r = L.r0; r < L.r1; ++r) h += heff[r];
    const uint32_t hb = std::max<uint32_t>(h, 1);  // an all-zero leaf: one zero row
    bufs.emplace_back((uint64_t)hb * M, s);
    if (h == 0) bufs.back().zero();
    else {
      gather_leaf<<<grid_for((uint64_t)h * M), 256, 0, s>>>(payload, doff.get(), dkept.get(), deff.get(), L.r0, L.r1,
                                                            M, h, bufs.back().get());
      RK_LAUNCH_CHECK();
    }
    tree[0].push_back({bufs.back().get(), hb, hb, 0u});
  }
  std::vector<DBuf<double>> roots;
  tsqr_forest(c, M, tree, roots);
  r_out = std::move(roots[0]);
  sync(s);  // host vectors (offset copies) are released
}

namespace {

// Jacobi on W (M x cp, ld M, `cols` real columns) and finalize into out (sigma, U);
// returns kappa = sigma_max / sigma_min over the `cols` columns
double merge_jacobi(Ctx& c, DBuf<double>& W, uint32_t M, uint32_t cols, uint32_t cp, MergeOut& out,
                    bool gram_ok = false, const uint32_t* row_perm = nullptr) {
  cudaStream_t s = c.stream;
  const uint32_t k = std::min(M, cols);
  out.k = k;
  out.sigma.alloc(k ? k : 1, s);
  out.u.alloc((uint64_t)M * (k ? k : 1), s);
  DBuf<double> alpha(cp, s);
  DBuf<uint64_t> stats(8, s);
  stats.zero();
  std::vector<JacobiJob> jj(1);
  jj[0].w = W.get(); jj[0].v = nullptr; jj[0].rows = M; jj[0].cols = cols; jj[0].cols_pad = cp;
  jj[0].alpha = alpha.get(); jj[0].stats = stats.get(); jj[0].gram_ok = gram_ok ? 1u : 0u;
  jacobi_batched(jj, s, c.num_sms, c.smem_optin, /*latency=*/true);
  prof_mark(s, "mrg jacobi");
  // finalize right behind the Jacobi (its result is discarded if the Jacobi
  // failed), then one readback of the statistics, the sorted sigma and the
  // deficiency flags: one host round trip instead of three
  DBuf<uint32_t> order(cp, s);
  DBuf<double> scratch(cp, s), sig_all(cp, s);
  DBuf<uint8_t> def(k ? k : 1, s);
  def.zero();
  FinalJob f;
  std::memset(&f, 0, sizeof f);
  f.w = W.get(); f.rows = M; f.cols = cp; f.k = k;
  f.u = out.u.get(); f.sigma = out.sigma.get(); f.sigma_all = sig_all.get();
  f.order = order.get(); f.scratch = scratch.get(); f.deficient = def.get();
  f.row_perm = row_perm;
  finalize_batched({f}, s);
  std::vector<uint64_t> hst;
  std::vector<double> hs;
  std::vector<uint8_t> hdef;
  to_host(hst, stats.get(), 8, s);
  to_host(hs, sig_all.get(), cols, s);
  to_host(hdef, def.get(), k, s);
  sync(s);
  prof_mark(s, "mrg finalize+sync");
  out.sweeps = hst[0];
  out.rotations = hst[1];
  if (hst[2] != 0) {
    if (gram_ok) return INFINITY;  // the caller falls back to the TSQR route
    double residual;
    std::memcpy(&residual, &hst[3], 8);
    throw_convergence(residual);
  }
  bool deficient = false;
  for (uint8_t x : hdef) deficient = deficient || x;
  if (deficient) complete_and_sign(c, out.u.get(), M, k, def.get(), nullptr, 0);
  const double smin = cols ? hs[cols - 1] : 0.0;
  return smin > 0.0 ? hs[0] / smin : INFINITY;
}

}  // namespace

void merge_finish(Ctx& c, std::vector<DBuf<double>>& roots, uint32_t M, MergeOut& out) {
  cudaStream_t s = c.stream;
  if (roots.size() > 1) {
    // the roots are the R factors of complete subtrees: continue the same pairwise tree
    std::vector<std::vector<DBuf<double>>> nodes(1);
    std::vector<std::vector<uint32_t>> heights(1, std::vector<uint32_t>(roots.size(), M));
    for (auto& r : roots) nodes[0].push_back(std::move(r));
    forest_reduce(c, M, nodes, heights);
    roots.clear();
    roots.push_back(std::move(nodes[0][0]));
  }
  const uint32_t cp = jacobi_cols_pad(M, M, false, c.smem_optin);
  DBuf<double> W((uint64_t)M * cp, s);
  W.zero();
  transpose_sq<<<grid_for((uint64_t)M * M), 256, 0, s>>>(roots[0].get(), M, W.get());
  RK_LAUNCH_CHECK();
  merge_jacobi(c, W, M, M, cp, out);
}

double jacobi_flops_of(uint64_t sweeps, uint64_t rotations, uint32_t rows, uint32_t cols) {
  const double c = cols, m = rows;
  return (double)sweeps * (c * (c - 1) / 2 * 2 * m + 2 * m * c) + (double)rotations * 6 * m;
}

bool gram_merge_eligible(uint32_t M) { return gram_route_enabled() && M <= cholesky_max_rows() && M % 8 == 0; }

// Gram route of the merge: W holds P P^T (M x cols_pad slot); R_P^T = chol(P P^T),
// accepted when kappa(P) <= kappa_max(M) (checked on the Cholesky diagonal, then on
// the computed sigma). Returns false -- out untouched -- when rejected.
bool gram_merge(Ctx& c, DBuf<double>& W, uint32_t M, MergeOut& out) {
  cudaStream_t s = c.stream;
  // the eigensolver route first (G itself, no Cholesky); it declines for clustered
  // spectra, M above its cluster-resident size, or kappa above the guard
  if (gram_merge_eig(c, W.get(), M, out)) return true;
  const uint32_t cp = jacobi_cols_pad(M, M, false, c.smem_optin);
  // rows by descending diagonal, as the blocks' Grams (fewer sweeps)
  DBuf<uint32_t> perm;
  if (diag_order_enabled()) {
    perm.alloc(M, s);
    DBuf<double> Wp((uint64_t)M * cp, s);
    if (cp != M) Wp.zero();
    diag_order(W.get(), (uint64_t)M * cp, M, 1, perm.get(), Wp.get(), s);
    W = std::move(Wp);
  }
  double* ptr = W.get();
  DBuf<double*> dptr(1, s);
  DBuf<uint32_t> status(1, s);
  DBuf<double> ratio(1, s);
  to_device(dptr.get(), &ptr, 1, s);
  cholesky_batched(dptr.get(), 1, M, status.get(), ratio.get(), s);
  uint32_t hst = 1;
  double hr = INFINITY;
  RK_CUDA_CHECK(cudaMemcpyAsync(&hst, status.get(), sizeof hst, cudaMemcpyDeviceToHost, s));
  RK_CUDA_CHECK(cudaMemcpyAsync(&hr, ratio.get(), sizeof hr, cudaMemcpyDeviceToHost, s));
  sync(s);
  prof_mark(s, "mrg chol+sync");
  const double kmax = kappa_max(M);
  if (hst == 0 && hr <= kmax) {
    MergeOut tmp;
    const double kappa = merge_jacobi(c, W, M, M, cp, tmp, true, perm.n ? perm.get() : nullptr);
    if (kappa <= kmax) {
      out = std::move(tmp);
      return true;
    }
  }
  return false;
}

void merge_records(Ctx& c, const double* payload, const std::vector<uint64_t>& offset,
                   const std::vector<uint32_t>& kept, uint32_t M, MergeOut& out, const std::vector<uint32_t>* eff_hint) {
  cudaStream_t s = c.stream;
  uint64_t total = 0;
  for (uint32_t k : kept) total += k;
  if (M == 0 || total == 0) {
    out.k = 0;
    out.sigma.alloc(1, s);
    out.u.alloc(1, s);
    return;
  }
  if (total > M) {
    // Gram route: R_P^T = chol(P P^T), accepted when kappa(P) <= kappa_max(M)
    if (gram_merge_eligible(M)) {
      const uint32_t cp = jacobi_cols_pad(M, M, false, c.smem_optin);
      DBuf<double> W((uint64_t)M * cp, s);
      W.zero();
      prof_mark(s, "mrg alloc");
      records_gram(payload, offset, kept, M, W.get(), s, eff_hint);
      prof_mark(s, "mrg syrk");
      if (gram_merge(c, W, M, out)) {
        const double Md = M;
        out.flops = Md * (Md + 1) * (double)total + Md * Md * Md / 3.0 + jacobi_flops_of(out.sweeps, out.rotations, M, M);
        return;
      }
    }
    std::vector<TreeLeaf> leaves = merge_leaves(kept, M);
    std::vector<DBuf<double>> roots(1);
    merge_subtree(c, payload, offset, kept, M, leaves, 0, leaves.size(), roots[0], eff_hint);
    merge_finish(c, roots, M, out);
    out.flops = 2.0 * (double)total * M * (double)M + jacobi_flops_of(out.sweeps, out.rotations, M, M);
    return;
  }
  // P^T is not taller than wide: Jacobi straight on P's columns (W = P)
  const uint32_t tc = (uint32_t)total;
  const uint32_t cp = jacobi_cols_pad(M, tc, false, c.smem_optin);
  DBuf<double> W((uint64_t)M * cp, s);
  W.zero();
  uint64_t col = 0;
  for (size_t r = 0; r < kept.size(); ++r) {
    if (!kept[r]) continue;
    rowmajor_to_colmajor<<<grid_for((uint64_t)M * kept[r]), 256, 0, s>>>(payload + offset[r], M, kept[r],
                                                                         W.get() + col * M);
    RK_LAUNCH_CHECK();
    col += kept[r];
  }
  merge_jacobi(c, W, M, tc, cp, out);
}

// ---------------------------------------------------------------------------
// dense_svd with V (svd.cpp:365-379 / svd_tall :316-332)

void dense_svd_dev(Ctx& c, const double* a, uint32_t rows, uint32_t cols, DenseSvdOut& out) {
  cudaStream_t s = c.stream;
  check_finite_or_throw(a, (uint64_t)rows * cols, "dense_svd: input has non-finite values", s);
  const uint32_t k = std::min(rows, cols);
  out.k = k;
  if (k == 0) {
    out.u.alloc(1, s); out.sigma.alloc(1, s); out.v.alloc(1, s);
    return;
  }
  const bool transposed = rows < cols;
  const uint32_t m = transposed ? cols : rows, n = k;  // B = transposed ? A^T : A, column-major m x n
  DBuf<double> B((uint64_t)m * n, s);
  // colmat_of (svd.cpp:39-49): column-major of A^T is A row-major as is
  if (transposed) {
    RK_CUDA_CHECK(cudaMemcpyAsync(B.get(), a, sizeof(double) * (uint64_t)m * n, cudaMemcpyDeviceToDevice, s));
  } else {
    rowmajor_to_colmajor<<<grid_for((uint64_t)m * n), 256, 0, s>>>(a, m, n, B.get());
    RK_LAUNCH_CHECK();
  }
  const bool with_qr = m > n;
  const uint64_t aux_sz = 2 * (uint64_t)n + (ceil_div(n, 16) + 1) * 256;
  DBuf<double> aux(aux_sz, s);
  QrJob qj;
  qj.a = B.get(); qj.lda = m; qj.m = m; qj.n = n; qj.diag = aux.get(); qj.beta = qj.diag + n; qj.tmat = qj.diag + 2 * n;
  const uint32_t cp = jacobi_cols_pad(n, n, true, c.smem_optin);
  DBuf<double> W((uint64_t)n * cp, s), Vr((uint64_t)cp * cp, s);
  W.zero();
  if (with_qr) {
    qr_batched({qj}, s, c.num_sms);
    RJob r;
    r.a = qj.a; r.lda = qj.lda; r.diag = qj.diag; r.m = m; r.n = n; r.w = W.get(); r.ldw = n;
    r_extract_batched({r}, /*transpose=*/false, s);
  } else {
    RK_CUDA_CHECK(cudaMemcpyAsync(W.get(), B.get(), sizeof(double) * (uint64_t)n * n, cudaMemcpyDeviceToDevice, s));
  }
  identity_colmajor<<<grid_for((uint64_t)cp * cp), 256, 0, s>>>(Vr.get(), n, cp, cp);
  RK_LAUNCH_CHECK();
  DBuf<double> alpha(cp, s);
  DBuf<uint64_t> stats(8, s);
  stats.zero();
  std::vector<JacobiJob> jj(1);
  jj[0].w = W.get(); jj[0].v = Vr.get(); jj[0].rows = n; jj[0].cols = n; jj[0].cols_pad = cp;
  jj[0].alpha = alpha.get(); jj[0].stats = stats.get();
  jacobi_batched(jj, s, c.num_sms, c.smem_optin);
  JacobiStats js = read_stats(stats.get(), 1, s)[0];
  if (js.failed) throw_convergence(js.residual);
  // sort, U_R = columns / sigma (+ completion), V_R permuted
  DBuf<double> ur((uint64_t)n * n, s), vr((uint64_t)n * n, s);  // row-major n x n
  DBuf<uint32_t> order(cp, s);
  DBuf<double> scratch(cp, s);
  DBuf<uint8_t> def(n, s);
  out.sigma.alloc(n, s);
  FinalJob f;
  std::memset(&f, 0, sizeof f);
  f.w = W.get(); f.rows = n; f.cols = n; f.k = n;
  f.u = ur.get(); f.sigma = out.sigma.get();
  f.order = order.get(); f.scratch = scratch.get(); f.deficient = def.get();
  f.v_in = Vr.get(); f.ldv = cp; f.v_out = vr.get();
  finalize_batched({f}, s);
  // the finalize sign flips are undone by the final sign convention below only
  // through U_A; completion must see the unflipped basis, which it does not
  // depend on (it only needs orthonormal placed columns)
  if (any_flag(def.get(), n, s)) {
    DBuf<int> fl(1, s);
    fl.zero();
    complete_columns_device(ur.get(), n, n, def.get(), fl.get(), s);
    int h = 0;
    RK_CUDA_CHECK(cudaMemcpyAsync(&h, fl.get(), sizeof h, cudaMemcpyDeviceToHost, s));
    sync(s);
    if (h) fail(RK_CONVERGENCE, "orthonormal completion has no independent direction (residual 0.000000)", 0.0);
  }
  // U_B (m x n row-major) = Q U_R when QR was used, else U_R
  DBuf<double> ub((uint64_t)m * n, s);
  if (with_qr) {
    DBuf<double> urc((uint64_t)n * n, s), ubc((uint64_t)m * n, s);
    rowmajor_to_colmajor<<<grid_for((uint64_t)n * n), 256, 0, s>>>(ur.get(), n, n, urc.get());
    RK_LAUNCH_CHECK();
    apply_q_device(qj, urc.get(), n, n, ubc.get(), s);
    colmajor_to_rowmajor<<<grid_for((uint64_t)m * n), 256, 0, s>>>(ubc.get(), m, m, n, ub.get());
    RK_LAUNCH_CHECK();
  } else {
    RK_CUDA_CHECK(cudaMemcpyAsync(ub.get(), ur.get(), sizeof(double) * (uint64_t)n * n, cudaMemcpyDeviceToDevice, s));
  }
  if (transposed) {  // U_A = V_B (n x n), V_A = U_B (m x n)
    out.u = std::move(vr);
    out.v = std::move(ub);
    sign_rows(out.u.get(), n, n, out.v.get(), m, s);
  } else {           // U_A = U_B (m x n), V_A = V_B
    out.u = std::move(ub);
    out.v = std::move(vr);
    sign_rows(out.u.get(), m, n, out.v.get(), n, s);
  }
  sync(s);
}

}  // namespace rk
