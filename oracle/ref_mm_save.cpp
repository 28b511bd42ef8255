// ref_mm_save.cpp -- TEST INFRASTRUCTURE ONLY. The reference's save_matrix_market
// (proj/src/matrix_market.cpp:121-132) as a standalone program: reads a COO dump
// (u64 rows, cols, nnz; u64 r[nnz]; u64 c[nnz]; f64 v[nnz]) and writes the .mtx.
// A separate process: in a Python process that has loaded numpy's bundled
// libraries, the reference's std::to_chars(double) path crashes inside ctypes.
#include <cstdint>
#include <cstdio>
#include <vector>

#include "ranky/matrix_market.hpp"

int main(int argc, char** argv) {
  if (argc != 3) return 2;
  FILE* f = std::fopen(argv[1], "rb");
  if (!f) return 3;
  uint64_t h[3];
  if (std::fread(h, 8, 3, f) != 3) return 4;
  std::vector<uint64_t> r(h[2]), c(h[2]);
  std::vector<double> v(h[2]);
  if (std::fread(r.data(), 8, h[2], f) != h[2] || std::fread(c.data(), 8, h[2], f) != h[2] ||
      std::fread(v.data(), 8, h[2], f) != h[2])
    return 5;
  std::fclose(f);
  std::vector<ranky::Entry> e(h[2]);
  for (uint64_t i = 0; i < h[2]; ++i) e[i] = {r[i], c[i], v[i]};
  ranky::save_matrix_market(ranky::SparseMatrix(h[0], h[1], std::move(e)), argv[2]);
  return 0;
}
