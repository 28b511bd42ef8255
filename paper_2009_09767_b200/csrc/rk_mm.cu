// rk_mm.cu -- Matrix Market coordinate files (proj/src/matrix_market.cpp:38-132,
// proj/include/ranky/matrix_market.hpp): load with the reference's validation and
// error messages (ranky::ParseError "... (line L)"), save byte-identically.
//
// Loading: the file is read whole; the entry lines are tokenised and parsed
// (std::from_chars, exact as the reference's) by host threads over line-aligned
// chunks, the first failing line decided in file order; the (row, col) sort that
// finds duplicates -- and yields the SparseMatrix order -- runs on the device
// (stable radix sort, sort_entries_device). Explicit zeros are then reported in
// file order, as the reference does after its duplicate scan.
#include <algorithm>
#include <charconv>
#include <cstdio>
#include <string>
#include <thread>
#include <vector>

#include "rk_internal.cuh"

namespace rk {
namespace {

constexpr const char* kBanner = "%%MatrixMarket matrix coordinate real general";

[[noreturn]] void parse_error(const std::string& what, uint64_t line) {
  fail(RK_PARSE, what + " (line " + std::to_string(line) + ")", (double)line);
}

bool is_ws(char ch) { return ch == ' ' || ch == '\t' || ch == '\n' || ch == '\v' || ch == '\f' || ch == '\r'; }

// split on whitespace (operator>> on std::string)
int tokens(const char* b, const char* e, const char** tb, const char** te, int cap) {
  int n = 0;
  while (b < e) {
    while (b < e && is_ws(*b)) ++b;
    if (b == e) break;
    const char* s = b;
    while (b < e && !is_ws(*b)) ++b;
    if (n < cap) {
      tb[n] = s;
      te[n] = b;
    }
    ++n;
  }
  return n;
}

bool parse_u(const char* b, const char* e, uint64_t& out) {
  auto r = std::from_chars(b, e, out);
  return r.ec == std::errc() && r.ptr == e;
}
bool parse_d(const char* b, const char* e, double& out) {
  auto r = std::from_chars(b, e, out);
  return r.ec == std::errc() && r.ptr == e;
}

struct Line {
  const char* b;
  const char* e;  // without the newline and a trailing '\r'
};

// getline over [p, end): the next line, advancing p
bool next_line(const char*& p, const char* end, Line& l) {
  if (p >= end) return false;
  const char* q = static_cast<const char*>(memchr(p, '\n', end - p));
  const char* le = q ? q : end;
  l.b = p;
  l.e = (le > p && le[-1] == '\r') ? le - 1 : le;
  p = q ? q + 1 : end;
  return true;
}

enum Status : int { kOk = 0, kEmpty = 1, kMalformed = 2, kOutside = 3 };

}  // namespace

void load_matrix_market(const std::string& path, rk_sparse& out, cudaStream_t s) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) fail(RK_RUNTIME, "cannot open " + path);
  std::string buf;
  std::fseek(f, 0, SEEK_END);
  const long sz = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  buf.resize(sz > 0 ? (size_t)sz : 0);
  const size_t got = sz > 0 ? std::fread(&buf[0], 1, (size_t)sz, f) : 0;
  std::fclose(f);
  buf.resize(got);
  const char* p = buf.data();
  const char* end = p + buf.size();
  Line l;
  uint64_t line_no = 0;
  if (!next_line(p, end, l)) parse_error("missing Matrix Market header", 1);
  ++line_no;
  if (std::string(l.b, l.e) != kBanner) parse_error("unsupported Matrix Market header '" + std::string(l.b, l.e) + "'",
                                                    line_no);
  uint64_t rows = 0, cols = 0, nnz = 0;
  for (;;) {
    if (!next_line(p, end, l)) parse_error("missing dimensions line", line_no + 1);
    ++line_no;
    if (l.e > l.b && l.b[0] == '%') continue;
    const char *tb[4], *te[4];
    const int n = tokens(l.b, l.e, tb, te, 4);
    if (n != 3 || !parse_u(tb[0], te[0], rows) || !parse_u(tb[1], te[1], cols) || !parse_u(tb[2], te[2], nnz))
      parse_error("malformed dimensions line '" + std::string(l.b, l.e) + "'", line_no);
    break;
  }
  // the rest: line-aligned chunks parsed by host threads
  const uint64_t first_line = line_no + 1;
  const char* body = p;
  const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  std::vector<const char*> cut(nt + 1);
  cut[0] = body;
  cut[nt] = end;
  for (unsigned t = 1; t < nt; ++t) {
    const char* c = body + (end - body) * (uint64_t)t / nt;
    if (c < cut[t - 1]) c = cut[t - 1];
    const char* q = c > body ? static_cast<const char*>(memchr(c - 1, '\n', end - (c - 1))) : nullptr;
    cut[t] = c == body ? body : (q ? q + 1 : end);
  }
  struct Chunk {
    std::vector<rk_entry> e;
    std::vector<uint32_t> e_line;  // line index within the chunk
    uint64_t lines = 0;
    int64_t bad_line = -1;  // first malformed / outside line index within the chunk
    int bad = kOk;
    uint64_t bad_entries_before = 0;  // entries parsed before the bad line
  };
  std::vector<Chunk> ch(nt);
  auto work = [&](unsigned t) {
    Chunk& c = ch[t];
    const char* q = cut[t];
    Line ln;
    while (next_line(q, cut[t + 1], ln)) {
      const uint64_t li = c.lines++;
      if (ln.e == ln.b) continue;
      if (c.bad) continue;  // keep counting lines
      const char *tb[4], *te[4];
      const int n = tokens(ln.b, ln.e, tb, te, 4);
      uint64_t r = 0, cc = 0;
      double v = 0.0;
      if (n != 3 || !parse_u(tb[0], te[0], r) || !parse_u(tb[1], te[1], cc) || !parse_d(tb[2], te[2], v)) {
        c.bad = kMalformed;
      } else if (r == 0 || cc == 0 || r > rows || cc > cols) {
        c.bad = kOutside;
      } else {
        c.e.push_back({r - 1, cc - 1, v});
        c.e_line.push_back((uint32_t)li);
        continue;
      }
      c.bad_line = (int64_t)li;
      c.bad_entries_before = c.e.size();
    }
  };
  {
    std::vector<std::thread> th;
    for (unsigned t = 1; t < nt; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
  }
  // file order: the nnz-th entry, then the first error before it, or trailing content
  std::vector<rk_entry> entries;
  std::vector<uint64_t> lines;
  entries.reserve(nnz);
  lines.reserve(nnz);
  uint64_t base = first_line;
  for (unsigned t = 0; t < nt; ++t) {
    const Chunk& c = ch[t];
    const uint64_t room = nnz - entries.size();
    const uint64_t usable = c.bad ? c.bad_entries_before : c.e.size();
    if (usable >= room) {  // the nnz-th entry is in this chunk
      for (uint64_t i = 0; i < room; ++i) {
        entries.push_back(c.e[i]);
        lines.push_back(base + c.e_line[i]);
      }
      // anything non-empty after it is trailing content
      const uint64_t last_li = room ? c.e_line[room - 1] : 0;
      int64_t trailing = -1;
      {
        const char* q = cut[t];
        Line ln;
        uint64_t li = 0;
        while (next_line(q, cut[t + 1], ln)) {
          if ((room == 0 || li > last_li) && ln.e != ln.b) {
            trailing = (int64_t)li;
            break;
          }
          ++li;
        }
        if (trailing >= 0) parse_error("unexpected content after " + std::to_string(nnz) + " entries",
                                       base + (uint64_t)trailing);
      }
      for (unsigned u = t + 1; u < nt; ++u) {
        const char* q = cut[u];
        Line ln;
        uint64_t li = 0;
        uint64_t b2 = base + c.lines;
        for (unsigned w = t + 1; w < u; ++w) b2 += ch[w].lines;
        while (next_line(q, cut[u + 1], ln)) {
          if (ln.e != ln.b) parse_error("unexpected content after " + std::to_string(nnz) + " entries", b2 + li);
          ++li;
        }
      }
      break;
    }
    if (c.bad) {
      const uint64_t ln = base + (uint64_t)c.bad_line;
      // the offending line's text, for the reference's message
      const char* q = cut[t];
      Line lx{};
      for (int64_t i = 0; i <= c.bad_line; ++i) next_line(q, cut[t + 1], lx);
      const std::string text(lx.b, lx.e);
      if (c.bad == kMalformed) parse_error("malformed entry '" + text + "'", ln);
      const char *tb[4], *te[4];
      tokens(lx.b, lx.e, tb, te, 4);
      parse_error("entry (" + std::string(tb[0], te[0]) + ", " + std::string(tb[1], te[1]) + ") outside " +
                      std::to_string(rows) + "x" + std::to_string(cols),
                  ln);
    }
    for (uint64_t i = 0; i < c.e.size(); ++i) {
      entries.push_back(c.e[i]);
      lines.push_back(base + c.e_line[i]);
    }
    base += c.lines;
  }
  if (entries.size() < nnz) {
    uint64_t last = first_line - 1;
    for (const Chunk& c : ch) last += c.lines;
    parse_error("expected " + std::to_string(nnz) + " entries, got " + std::to_string(entries.size()), last);
  }
  // duplicates: the device sort (matrix_market.cpp:104-119), then zeros in file order (:120-126)
  out.rows = rows;
  out.cols = cols;
  out.nnz = nnz;
  out.entries = static_cast<rk_entry*>(host_alloc_bytes((nnz ? nnz : 1) * sizeof(rk_entry)));
  int64_t da = -1, db = -1;
  sort_entries_device(entries.data(), nnz, out.entries, &da, &db, s);
  if (da >= 0) {
    const rk_entry& e = entries[da];
    parse_error("duplicate coordinate (" + std::to_string(e.row + 1) + ", " + std::to_string(e.col + 1) + ")",
                std::max(lines[da], lines[db]));
  }
  for (uint64_t i = 0; i < nnz; ++i)
    if (entries[i].value == 0.0)
      parse_error("explicit zero at (" + std::to_string(entries[i].row + 1) + ", " +
                      std::to_string(entries[i].col + 1) + ")",
                  lines[i]);
}

void save_matrix_market(const rk_sparse_view& a, const std::string& path) {
  // formatted by host threads into per-chunk buffers (std::to_chars shortest
  // round-trip form, matrix_market.cpp:31-35), written in order
  const uint64_t n = a.nnz;
  const unsigned nt = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(32, std::min<uint64_t>(
      std::thread::hardware_concurrency(), n / 65536 + 1)));
  std::vector<std::string> parts(nt);
  auto work = [&](unsigned t) {
    const uint64_t lo = n * t / nt, hi = n * (t + 1) / nt;
    std::string& o = parts[t];
    o.reserve((hi - lo) * 32);
    char tmp[96];
    for (uint64_t i = lo; i < hi; ++i) {
      const rk_entry& e = a.entries[i];
      char* q = std::to_chars(tmp, tmp + 32, e.row + 1).ptr;
      *q++ = ' ';
      q = std::to_chars(q, q + 32, e.col + 1).ptr;
      *q++ = ' ';
      q = std::to_chars(q, tmp + sizeof tmp, e.value).ptr;
      *q++ = '\n';
      o.append(tmp, q);
    }
  };
  {
    std::vector<std::thread> th;
    for (unsigned t = 1; t < nt; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
  }
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) fail(RK_RUNTIME, "cannot write " + path);
  const std::string head = std::string(kBanner) + "\n" + std::to_string(a.rows) + " " + std::to_string(a.cols) + " " +
                           std::to_string(a.nnz) + "\n";
  bool ok = std::fwrite(head.data(), 1, head.size(), f) == head.size();
  for (const std::string& part : parts) ok = ok && std::fwrite(part.data(), 1, part.size(), f) == part.size();
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) fail(RK_RUNTIME, "write failed for " + path);
}

}  // namespace rk
