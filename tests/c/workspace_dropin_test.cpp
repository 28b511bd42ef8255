// RepairWorkspace through the B200 drop-in (paper_2009_09767_b200/dropin/ranky_dropin.cpp
// on rk_workspace_*), compiled against the reference's own headers and linked like
// oracle/_ref/ranky_acceptance_b200. The cases are those of the reference's
// proj/tests/repair_test.cpp: the brute-force neighbor oracle (:16-40) over 40
// instances (:127-146), isolated rows (:104-125), NeighborRandom (:148-175), plus a
// replay of the repair driver (proj/src/repair.cpp:162-216) through the single-row
// API that must equal ranky::repair's report and matrix. Exit status = failures.
#include <cstdio>
#include <set>
#include <vector>

#include "ranky/partition.hpp"
#include "ranky/repair.hpp"
#include "ranky/rng.hpp"
#include "ranky/synth.hpp"

using namespace ranky;

static int g_fail = 0;
#define CHECK(x)                                                         \
  do {                                                                   \
    if (!(x)) {                                                          \
      ++g_fail;                                                          \
      std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #x); \
    }                                                                    \
  } while (0)

static std::set<std::size_t> brute_force_neighbor_cols(const SparseMatrix& a, const BlockPartition& p,
                                                       std::size_t d, std::size_t row) {
  auto at = [&](std::size_t r, std::size_t c) {
    for (const Entry& e : a.entries())
      if (e.row == r && e.col == c) return e.value;
    return 0.0;
  };
  const ColumnRange& range = p.range(d);
  std::set<std::size_t> candidates;
  for (std::size_t n1 = 0; n1 < a.cols(); ++n1) {
    if (n1 >= range.begin && n1 < range.end) continue;
    if (at(row, n1) == 0.0) continue;
    for (std::size_t m1 = 0; m1 < a.rows(); ++m1)
      if (at(m1, n1) != 0.0) candidates.insert(m1);
  }
  std::set<std::size_t> cols;
  for (std::size_t m : candidates)
    for (std::size_t n2 = range.begin; n2 < range.end; ++n2)
      if (at(m, n2) != 0.0) cols.insert(n2);
  return cols;
}

int main() {
  {  // isolated row: no candidate, no change
    SparseMatrix a(3, 6, {{0, 0, 1.0}, {2, 4, 1.0}});
    BlockPartition p = partition_columns(6, 2);
    RepairWorkspace ws(a, p);
    KeyedRng rng(3, 0, 1);
    CHECK(!ws.apply_neighbor(0, 1, rng).has_value());
    CHECK(ws.to_matrix() == a);
  }
  {  // candidates without in-block columns
    SparseMatrix a(4, 8, {{0, 5, 1.0}, {1, 5, 1.0}, {1, 6, 1.0}, {2, 0, 1.0}, {3, 2, 1.0}});
    BlockPartition p = partition_columns(8, 2);
    CHECK(find_lonely_rows(a, p, 0) == (std::vector<std::size_t>{0, 1}));
    RepairWorkspace ws(a, p);
    CHECK(ws.lonely_rows(0) == (std::vector<std::size_t>{0, 1}));
    KeyedRng rng(3, 0, 0);
    CHECK(!ws.apply_neighbor(0, 0, rng).has_value());
    CHECK(ws.to_matrix() == a);
  }
  int checked = 0;
  for (std::uint64_t instance = 0; instance < 40; ++instance) {  // brute force
    SparseMatrix a = synth_bipartite(8, 16, 0.12, instance);
    BlockPartition p = partition_columns(16, 4);
    for (std::size_t d = 0; d < 4; ++d) {
      for (std::size_t row : find_lonely_rows(a, p, d)) {
        RepairWorkspace ws(a, p);
        KeyedRng rng(instance, d, row);
        auto col = ws.apply_neighbor(d, row, rng);
        auto expected = brute_force_neighbor_cols(a, p, d, row);
        if (expected.empty()) {
          CHECK(!col.has_value());
        } else {
          CHECK(col.has_value() && expected.count(*col) == 1);
          CHECK(col.has_value() && ws.has_entry(row, *col));
        }
        ++checked;
      }
    }
  }
  {  // NeighborRandom fills the row
    SparseMatrix a(3, 6, {{0, 0, 1.0}, {0, 2, 1.0}, {0, 5, 1.0}, {1, 5, 1.0}, {2, 1, 1.0}});
    BlockPartition p = partition_columns(6, 2);
    RepairWorkspace ws(a, p);
    KeyedRng rng(3, 0, 1);
    auto added = ws.apply_neighbor_random(0, 1, rng);
    CHECK(added.size() >= 1 && added.size() <= 2);
    for (std::size_t col : added) CHECK(col < 3 && ws.has_entry(1, col));
    CHECK(!ws.row_lonely_in_block(0, 1));
  }
  for (auto method : {RepairMethod::kRandom, RepairMethod::kNeighbor, RepairMethod::kNeighborRandom}) {
    for (std::uint64_t seed = 0; seed < 3; ++seed) {  // the driver replayed through the single-row API
      SparseMatrix a = synth_bipartite(16, 128, 0.05, seed);
      BlockPartition p = partition_columns(128, 8);
      RepairWorkspace ws(a, p);
      RepairReport rep;
      for (std::size_t d = 0; d < p.block_count(); ++d) {
        const auto rows = ws.lonely_rows(d);
        rep.lonely_counts.push_back(rows.size());
        for (std::size_t row : rows) {
          KeyedRng rng(17 + seed, d, row);
          if (method == RepairMethod::kRandom) {
            rep.added_edges.push_back({d, row, ws.apply_random(d, row, rng), RepairMethod::kRandom});
          } else if (method == RepairMethod::kNeighbor) {
            if (auto c = ws.apply_neighbor(d, row, rng)) {
              rep.added_edges.push_back({d, row, *c, RepairMethod::kNeighbor});
            } else {
              ++rep.fallback_count;
              rep.added_edges.push_back({d, row, ws.apply_random(d, row, rng), RepairMethod::kRandom});
            }
          } else {
            auto c = ws.apply_neighbor(d, row, rng);
            if (c) rep.added_edges.push_back({d, row, *c, RepairMethod::kNeighbor});
            const std::size_t r = ws.apply_random(d, row, rng);
            if (!c || r != *c) rep.added_edges.push_back({d, row, r, RepairMethod::kRandom});
          }
        }
      }
      auto [repaired, want] = repair(a, p, method, 17 + seed);
      CHECK(ws.to_matrix() == repaired);
      CHECK(rep.to_log() == want.to_log());
    }
  }
  std::printf("workspace drop-in: %d brute-force rows checked, %d failures\n", checked, g_fail);
  return g_fail;
}
