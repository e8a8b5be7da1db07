// Matrix Market coordinate reader for the sparse ingest path.
//
// Replaces the reference's chunked pandas parser (formats.py:143-323:
// _parse_header, _parse_size_line, _parse_chunk, parse_matrix_market) and
// read_matrix_market_info (381-395) with a native, multi-threaded one whose
// triplets go straight to the device CSR builder (xb_rsvd_coo /
// xb_spmm_coo) or to the pool (pipeline.parse_matrix_market). The file is
// mmap'ed; the body is cut at line boundaries into one range per thread,
// each thread counts its lines (for 1-based line numbers), then parses its
// range with std::from_chars (correctly rounded, like the reference's
// round_trip converter).
//
// Same acceptance rules and messages as the reference: banner with five
// tokens, object "matrix", format "coordinate", field real | integer |
// pattern, symmetry general | symmetric; comment lines before the size line;
// a blank line there is an error; indices are numbers with an integral value
// in 1..rows / 1..cols; symmetric files may not hold entries above the
// diagonal, and their off-diagonal entries are mirrored. Output order
// matches the reference's: per chunk of `chunk_lines` body lines, the
// chunk's entries in file order followed by its mirrored entries (the order
// duplicate sums follow, core.py:287-303). Faults are reported in the
// reference's order too: chunk by chunk, the declared-count check first,
// then per chunk field-count faults before index / value / range /
// symmetry faults, each at its first line.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace xb {
namespace {

struct Mapped {
  const char* p = nullptr;
  size_t n = 0;
  int fd = -1;
  explicit Mapped(const char* path) {
    fd = ::open(path, O_RDONLY);
    XB_REQUIRE(fd >= 0, XB_EVALUE, std::string("cannot open ") + path);
    struct stat st;
    XB_REQUIRE(fstat(fd, &st) == 0, XB_EVALUE, std::string("cannot stat ") + path);
    n = (size_t)st.st_size;
    if (n) {
      void* m = mmap(nullptr, n, PROT_READ, MAP_PRIVATE, fd, 0);
      XB_REQUIRE(m != MAP_FAILED, XB_EVALUE, std::string("cannot map ") + path);
      p = static_cast<const char*>(m);
      madvise(m, n, MADV_SEQUENTIAL);
    }
  }
  ~Mapped() {
    if (p) munmap(const_cast<char*>(p), n);
    if (fd >= 0) ::close(fd);
  }
};

inline bool is_ws(char ch) { return ch == ' ' || ch == '\t' || ch == '\r' || ch == '\v' || ch == '\f'; }

// whitespace-split tokens of [b, e)
void split(const char* b, const char* e, std::vector<std::pair<const char*, const char*>>& out) {
  out.clear();
  while (b < e) {
    while (b < e && is_ws(*b)) ++b;
    if (b >= e) break;
    const char* s = b;
    while (b < e && !is_ws(*b)) ++b;
    out.emplace_back(s, b);
  }
}

std::string lower(const char* b, const char* e) {
  std::string s(b, e);
  for (auto& ch : s) ch = (char)std::tolower((unsigned char)ch);
  return s;
}

[[noreturn]] void fault(int64_t line, const std::string& msg) {
  throw ParseFaultError(line, msg);
}

// Python int(): optional sign, digits (underscores between digits allowed)
bool parse_int(const char* b, const char* e, int64_t* out) {
  std::string s;
  for (const char* q = b; q < e; ++q)
    if (*q != '_') s.push_back(*q);
  const char* sb = s.data();
  const char* se = sb + s.size();
  if (sb < se && *sb == '+') ++sb;
  if (sb == se) return false;
  auto r = std::from_chars(sb, se, *out);
  return r.ec == std::errc() && r.ptr == se;
}

// a float token (pandas round_trip: decimal / exponent / inf / nan forms)
bool parse_double(const char* b, const char* e, double* out) {
  if (b < e && *b == '+') ++b;
  if (b == e) return false;
  auto r = std::from_chars(b, e, *out);
  return r.ec == std::errc() && r.ptr == e;
}

struct Header {
  int field = 0;  // 0 real, 1 integer, 2 pattern
  bool symmetric = false;
  int64_t rows = 0, cols = 0, declared = 0;
  size_t body = 0;       // byte offset of the first body line
  int64_t body_line = 0;  // its 1-based line number
};

// [line begin, line end (excluding '\n'), next line begin)
inline const char* line_end(const char* b, const char* e) {
  const void* q = memchr(b, '\n', (size_t)(e - b));
  return q ? static_cast<const char*>(q) : e;
}

Header parse_head(const Mapped& f) {
  Header h;
  if (f.n == 0) fault(1, "empty file");
  const char* b = f.p;
  const char* e = f.p + f.n;
  const char* le = line_end(b, e);
  std::vector<std::pair<const char*, const char*>> t;
  split(b, le, t);
  if (t.empty() || std::string(t[0].first, t[0].second) != "%%MatrixMarket")
    fault(1, "not a Matrix Market file (missing %%MatrixMarket banner)");
  if (t.size() != 5) fault(1, "banner has " + std::to_string(t.size()) + " tokens, expected 5");
  const std::string obj = lower(t[1].first, t[1].second), fmt = lower(t[2].first, t[2].second),
                    field = lower(t[3].first, t[3].second), sym = lower(t[4].first, t[4].second);
  if (obj != "matrix") fault(1, "unsupported object '" + obj + "'");
  if (fmt != "coordinate") fault(1, "unsupported format '" + fmt + "', only coordinate is handled");
  if (field == "real") h.field = 0;
  else if (field == "integer") h.field = 1;
  else if (field == "pattern") h.field = 2;
  else fault(1, "unsupported field '" + field + "'");
  if (sym == "general") h.symmetric = false;
  else if (sym == "symmetric") h.symmetric = true;
  else fault(1, "unsupported symmetry '" + sym + "'");
  int64_t lineno = 1;
  b = le < e ? le + 1 : e;
  while (b < e) {
    le = line_end(b, e);
    ++lineno;
    const char* next = le < e ? le + 1 : e;
    if (*b == '%') {
      b = next;
      continue;
    }
    split(b, le, t);
    if (t.empty()) fault(lineno, "blank line before the size line");
    if (t.size() != 3) fault(lineno, "size line has " + std::to_string(t.size()) + " fields, expected 3");
    int64_t v[3];
    for (int i = 0; i < 3; ++i)
      if (!parse_int(t[i].first, t[i].second, &v[i]))
        fault(lineno, "size line is not three integers: '" + std::string(b, le) + "'");
    if (v[0] < 1 || v[1] < 1)
      fault(lineno, "matrix dimensions " + std::to_string(v[0]) + "x" + std::to_string(v[1]) +
                        " are not positive");
    if (v[2] < 0) fault(lineno, "negative entry count " + std::to_string(v[2]));
    h.rows = v[0];
    h.cols = v[1];
    h.declared = v[2];
    h.body = (size_t)(next - f.p);
    h.body_line = lineno + 1;
    return h;
  }
  fault(lineno, "file ends before the size line");
}

// Fault categories in the order the reference checks them within a chunk
// (formats.py:197-258): field count, row index, column index, value, row
// range, column range, symmetric upper entry.
constexpr int kCats = 7;

struct ChunkFaults {
  int64_t line[kCats];
  std::string msg[kCats];
  ChunkFaults() {
    for (auto& l : line) l = 0;
  }
};

struct Piece {
  const char* b;
  const char* e;
  int64_t first_line = 0, lines = 0;
  std::vector<int64_t> r, c;
  std::vector<double> v;
  // first fault per category for every chunk this piece touches
  std::vector<std::pair<int64_t, ChunkFaults>> faults;  // (chunk index, firsts)
};

// Validate + convert one range of whole lines.
void parse_piece(Piece& pc, const Header& h, int64_t chunk_lines) {
  const int want = h.field == 2 ? 2 : 3;
  std::vector<std::pair<const char*, const char*>> t;
  pc.r.reserve(pc.lines);
  pc.c.reserve(pc.lines);
  pc.v.reserve(pc.lines);
  int64_t line = pc.first_line;
  for (const char* b = pc.b; b < pc.e; ++line) {
    const char* le = line_end(b, pc.e);
    const char* next = le < pc.e ? le + 1 : pc.e;
    split(b, le, t);
    int cat = -1;
    std::string msg;
    double fi = 0, fj = 0, fv = 1.0;
    if ((int)t.size() != want) {
      cat = 0;
      msg = "expected " + std::to_string(want) + " fields, found " + std::to_string(t.size());
    } else if (!(parse_double(t[0].first, t[0].second, &fi) && std::isfinite(fi) &&
                 fi == std::floor(fi))) {
      cat = 1;
      msg = "malformed row index '" + std::string(t[0].first, t[0].second) + "'";
    } else if (!(parse_double(t[1].first, t[1].second, &fj) && std::isfinite(fj) &&
                 fj == std::floor(fj))) {
      cat = 2;
      msg = "malformed column index '" + std::string(t[1].first, t[1].second) + "'";
    } else if (want == 3 && (!parse_double(t[2].first, t[2].second, &fv) || std::isnan(fv))) {
      cat = 3;
      msg = "malformed value '" + std::string(t[2].first, t[2].second) + "'";
    } else {
      const int64_t r = (int64_t)fi - 1, c = (int64_t)fj - 1;
      if (r < 0 || r >= h.rows) {
        cat = 4;
        msg = "row index " + std::to_string(r + 1) + " outside 1.." + std::to_string(h.rows);
      } else if (c < 0 || c >= h.cols) {
        cat = 5;
        msg = "column index " + std::to_string(c + 1) + " outside 1.." + std::to_string(h.cols);
      } else if (h.symmetric && r < c) {
        cat = 6;
        msg = "entry above the diagonal in a symmetric matrix";
      } else {
        pc.r.push_back(r);
        pc.c.push_back(c);
        pc.v.push_back(fv);
      }
    }
    if (cat >= 0) {
      const int64_t chunk = (line - h.body_line) / chunk_lines;
      if (pc.faults.empty() || pc.faults.back().first != chunk) pc.faults.push_back({chunk, {}});
      ChunkFaults& f = pc.faults.back().second;
      if (!f.line[cat]) {
        f.line[cat] = line;
        f.msg[cat] = msg;
      }
    }
    b = next;
  }
}

}  // namespace

ParseFaultError::ParseFaultError(int64_t l, const std::string& m)
    : Error(XB_EPARSE, m), line(l) {}

}  // namespace xb

using namespace xb;

extern "C" {

int xb_mm_info(const char* path, int64_t* rows, int64_t* cols, int64_t* entries, int* field,
               int* symmetric, int64_t* err_line) {
  if (err_line) *err_line = 0;
  return guarded_api([&] {
    XB_REQUIRE(path, XB_EVALUE, "null path");
    try {
      Mapped f(path);
      const Header h = parse_head(f);
      if (rows) *rows = h.rows;
      if (cols) *cols = h.cols;
      if (entries) *entries = h.declared;
      if (field) *field = h.field;
      if (symmetric) *symmetric = h.symmetric ? 1 : 0;
    } catch (const ParseFaultError& e) {
      if (err_line) *err_line = e.line;
      throw;
    }
  });
}

int xb_mm_read(const char* path, int threads, int64_t chunk_lines, xb_coo* out, int64_t* err_line) {
  if (err_line) *err_line = 0;
  return guarded_api([&] {
    XB_REQUIRE(path && out, XB_EVALUE, "null argument");
    std::memset(out, 0, sizeof(*out));
    try {
      Mapped f(path);
      const Header h = parse_head(f);
      const char* b0 = f.p + h.body;
      const char* e0 = f.p + f.n;
      // split the body at line starts, one piece per thread
      int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
      nt = (int)std::max<int64_t>(1, std::min<int64_t>(nt, (int64_t)((e0 - b0) >> 16) + 1));
      std::vector<Piece> pcs(nt);
      const char* cur = b0;
      for (int i = 0; i < nt; ++i) {
        const char* want = b0 + (size_t)((e0 - b0) * (double)(i + 1) / nt);
        if (i == nt - 1 || want >= e0) {
          want = e0;
        } else {
          want = line_end(std::max(want, cur), e0);
          if (want < e0) ++want;
        }
        pcs[i].b = cur;
        pcs[i].e = want;
        cur = want;
      }
      auto count = [&](Piece& pc) {
        int64_t n = 0;
        for (const char* q = pc.b; q < pc.e;) {
          const char* le = line_end(q, pc.e);
          ++n;
          q = le < pc.e ? le + 1 : pc.e;
        }
        pc.lines = n;
      };
      {
        std::vector<std::thread> th;
        for (int i = 0; i < nt; ++i) th.emplace_back(count, std::ref(pcs[i]));
        for (auto& t : th) t.join();
      }
      int64_t total = 0;
      for (auto& pc : pcs) {
        pc.first_line = h.body_line + total;
        total += pc.lines;
      }
      const int64_t cl = chunk_lines > 0 ? chunk_lines : 500000;
      {
        std::vector<std::thread> th;
        for (int i = 0; i < nt; ++i)
          th.emplace_back(parse_piece, std::ref(pcs[i]), std::cref(h), cl);
        for (auto& t : th) t.join();
      }
      // the reference's order of rejection (formats.py:289-312): chunk by
      // chunk, the entry-count check before the chunk is parsed, then the
      // chunk's faults by category; after the last chunk, the short count
      const int64_t excess_chunk = total > h.declared ? h.declared / cl : -1;
      std::vector<std::pair<int64_t, ChunkFaults>> all;
      for (auto& pc : pcs)
        for (auto& f : pc.faults) {
          if (!all.empty() && all.back().first == f.first) {
            for (int k = 0; k < kCats; ++k)
              if (f.second.line[k] && (!all.back().second.line[k] ||
                                       f.second.line[k] < all.back().second.line[k])) {
                all.back().second.line[k] = f.second.line[k];
                all.back().second.msg[k] = f.second.msg[k];
              }
          } else {
            all.push_back(f);
          }
        }
      for (auto& f : all) {
        if (excess_chunk >= 0 && f.first >= excess_chunk) break;
        for (int k = 0; k < kCats; ++k)
          if (f.second.line[k]) fault(f.second.line[k], f.second.msg[k]);
      }
      if (excess_chunk >= 0)
        fault(h.body_line + h.declared,
              "more entries than the " + std::to_string(h.declared) + " declared on the size line");
      if (total < h.declared)
        fault(h.body_line - 1 + total,  // the last line read, as formats.py:308-312
              "size line declared " + std::to_string(h.declared) +
                  " entries but the file ends after " + std::to_string(total));
      // assemble in the reference's order: per chunk, entries then mirrors
      int64_t mirrors = 0;
      if (h.symmetric)
        for (auto& pc : pcs)
          for (size_t i = 0; i < pc.r.size(); ++i) mirrors += pc.r[i] > pc.c[i];
      const int64_t nnz = total + mirrors;
      out->rows = h.rows;
      out->cols = h.cols;
      out->nnz = nnz;
      out->field = h.field;
      out->symmetric = h.symmetric ? 1 : 0;
      out->r = static_cast<int64_t*>(std::malloc((size_t)std::max<int64_t>(nnz, 1) * 8));
      out->c = static_cast<int64_t*>(std::malloc((size_t)std::max<int64_t>(nnz, 1) * 8));
      out->v = static_cast<double*>(std::malloc((size_t)std::max<int64_t>(nnz, 1) * 8));
      if (!out->r || !out->c || !out->v) {
        xb_coo_free(out);
        throw std::bad_alloc();
      }
      // flat views over the pieces in file order
      std::vector<int64_t> base(nt + 1, 0);
      for (int i = 0; i < nt; ++i) base[i + 1] = base[i] + (int64_t)pcs[i].r.size();
      auto at = [&](int64_t g, int64_t* r, int64_t* c, double* v) {
        const int i = (int)(std::upper_bound(base.begin(), base.end(), g) - base.begin()) - 1;
        const int64_t j = g - base[i];
        *r = pcs[i].r[j];
        *c = pcs[i].c[j];
        *v = pcs[i].v[j];
      };
      int64_t o = 0;
      for (int64_t c0 = 0; c0 < total; c0 += cl) {
        const int64_t c1 = std::min(total, c0 + cl);
        for (int64_t g = c0; g < c1; ++g, ++o) at(g, out->r + o, out->c + o, out->v + o);
        if (h.symmetric)
          for (int64_t g = c0; g < c1; ++g) {
            int64_t r, c;
            double v;
            at(g, &r, &c, &v);
            if (r > c) {
              out->r[o] = c;
              out->c[o] = r;
              out->v[o] = v;
              ++o;
            }
          }
      }
    } catch (const ParseFaultError& e) {
      if (err_line) *err_line = e.line;
      throw;
    }
  });
}

void xb_coo_free(xb_coo* c) {
  if (!c) return;
  std::free(c->r);
  std::free(c->c);
  std::free(c->v);
  c->r = c->c = nullptr;
  c->v = nullptr;
  c->nnz = 0;
}

}  // extern "C"
