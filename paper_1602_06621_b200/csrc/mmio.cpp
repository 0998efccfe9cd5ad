// mmio.cpp -- matrix store ingest: Matrix Market reader / writer
// (src/matrix_market.cpp:63-233) and a binary CSR format, host side.
//
// The reader splits the text into per-thread chunks at line boundaries and
// parses them in parallel (strtoll / strtod, exactly the conversions the
// reference uses), then replays the reference's sequential acceptance rules
// in line order: the first offending data line wins, then end-of-file and
// trailing-data checks.  Sorting, duplicate detection and the CSR build run
// on the device (engine.cu, coo_to_csr); a duplicate is reported with the
// line of its later occurrence like the reference (:142-158).  The writer
// formats entries in parallel with the reference's "%.17g" and integer
// output, so its bytes equal the reference writer's.
#include "mmio.h"

#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace eqb {
namespace mm {
namespace {

[[noreturn]] void parse_fail(int64_t line, const std::string& msg) {
  throw std::runtime_error("matrix market: line " + std::to_string(line) + ": " + msg);
}

std::string lower(std::string s) {
  for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return s;
}

inline bool is_space(char c) {  // std::isspace in the "C" locale
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// one line as [b, e) with a trailing '\r' removed (LineReader::next, :30-38)
struct Line {
  const char* b;
  const char* e;
  std::string str() const { return std::string(b, e); }
  bool comment() const { return b != e && *b == '%'; }
};

int split_tokens(const Line& l, const char** tb, const char** te, int cap) {
  int n = 0;
  const char* p = l.b;
  while (p < l.e) {
    while (p < l.e && is_space(*p)) ++p;
    if (p >= l.e) break;
    const char* s = p;
    while (p < l.e && !is_space(*p)) ++p;
    if (n < cap) {
      tb[n] = s;
      te[n] = p;
    }
    ++n;
  }
  return n;
}

bool parse_index(const char* b, const char* e, long long& out) {  // :40-45
  if (b == e) return false;
  char buf[64];
  const size_t len = static_cast<size_t>(e - b);
  if (len >= sizeof buf) {
    std::string s(b, e);
    char* end = nullptr;
    out = std::strtoll(s.c_str(), &end, 10);
    return end == s.c_str() + s.size();
  }
  std::memcpy(buf, b, len);
  buf[len] = 0;
  char* end = nullptr;
  out = std::strtoll(buf, &end, 10);
  return end == buf + len;
}

bool parse_double(const char* b, const char* e, double& out) {  // :33-38
  if (b == e) return false;
  char buf[128];
  const size_t len = static_cast<size_t>(e - b);
  if (len >= sizeof buf) {
    std::string s(b, e);
    char* end = nullptr;
    out = std::strtod(s.c_str(), &end);
    return end == s.c_str() + s.size();
  }
  std::memcpy(buf, b, len);
  buf[len] = 0;
  char* end = nullptr;
  out = std::strtod(buf, &end);
  return end == buf + len;
}

// sequential line reader over [p, end)
struct Reader {
  const char* p;
  const char* end;
  int64_t line_no = 0;
  bool next(Line& l) {
    if (p >= end) return false;
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
    const char* le = nl ? nl : end;
    l.b = p;
    l.e = le;
    if (l.e > l.b && l.e[-1] == '\r') --l.e;
    p = nl ? nl + 1 : end;
    ++line_no;
    return true;
  }
};

int nthreads(size_t bytes) {
  const unsigned hc = std::max(1u, std::thread::hardware_concurrency());
  return static_cast<int>(std::max<size_t>(1, std::min<size_t>(hc, bytes / (1u << 20))));
}

// byte ranges at line starts covering [b, e)
std::vector<const char*> chunk_starts(const char* b, const char* e, int parts) {
  std::vector<const char*> s{b};
  const size_t len = static_cast<size_t>(e - b);
  for (int k = 1; k < parts; ++k) {
    const char* q = b + len * k / parts;
    if (q <= s.back()) continue;
    const char* nl = static_cast<const char*>(std::memchr(q, '\n', static_cast<size_t>(e - q)));
    if (!nl) break;
    if (nl + 1 > s.back() && nl + 1 < e) s.push_back(nl + 1);
  }
  s.push_back(e);
  return s;
}

enum : uint8_t { kOk = 0, kTokens = 1, kMalformed = 2, kRange = 3 };

struct CoordChunk {
  int64_t lines = 0;  // lines in the chunk
  std::vector<int64_t> row, col, line;  // line: chunk-relative (1-based)
  std::vector<double> val;
  std::vector<uint8_t> status;
  std::vector<std::string> raw;         // offending line text per failing entry
  std::vector<long long> bad_i, bad_j;  // parsed indices for range failures
  std::vector<int64_t> raw_at;          // entry index of raw / bad_i / bad_j
};

void parse_coord_chunk(const char* b, const char* e, long long m, long long n, CoordChunk& c) {
  Reader r{b, e};
  Line l;
  const char* tb[4];
  const char* te[4];
  while (r.next(l)) {
    if (l.comment()) continue;
    const int nt = split_tokens(l, tb, te, 4);
    if (nt == 0) continue;
    long long i = 0, j = 0;
    double v = 0.0;
    uint8_t st = kOk;
    if (nt != 3) {
      st = kTokens;
    } else if (!parse_index(tb[0], te[0], i) || !parse_index(tb[1], te[1], j) ||
               !parse_double(tb[2], te[2], v)) {
      st = kMalformed;
    } else if (i < 1 || i > m || j < 1 || j > n) {
      st = kRange;
    }
    if (st != kOk) {
      c.raw_at.push_back(static_cast<int64_t>(c.row.size()));
      c.raw.push_back(l.str());
      c.bad_i.push_back(i);
      c.bad_j.push_back(j);
    }
    c.row.push_back(i - 1);
    c.col.push_back(j - 1);
    c.val.push_back(v);
    c.line.push_back(r.line_no);
    c.status.push_back(st);
  }
  c.lines = r.line_no;
}

struct ArrayChunk {
  int64_t lines = 0;
  std::vector<int64_t> line_of_tok;  // chunk-relative line of every value token
  std::vector<double> val;
  std::vector<uint8_t> ok;
  std::vector<std::string> bad_tok;  // text of malformed tokens
  std::vector<int64_t> bad_at;
};

void parse_array_chunk(const char* b, const char* e, ArrayChunk& c) {
  Reader r{b, e};
  Line l;
  while (r.next(l)) {
    if (l.comment()) continue;
    const char* p = l.b;
    while (p < l.e) {
      while (p < l.e && is_space(*p)) ++p;
      if (p >= l.e) break;
      const char* s = p;
      while (p < l.e && !is_space(*p)) ++p;
      double v = 0.0;
      const bool good = parse_double(s, p, v);
      if (!good) {
        c.bad_at.push_back(static_cast<int64_t>(c.val.size()));
        c.bad_tok.push_back(std::string(s, p));
      }
      c.val.push_back(v);
      c.ok.push_back(good ? 1 : 0);
      c.line_of_tok.push_back(r.line_no);
    }
  }
  c.lines = r.line_no;
}

}  // namespace

void parse(const char* data, size_t len, Matrix& out) {
  Reader rd{data, data + len};
  Line line;
  if (!rd.next(line)) parse_fail(1, "empty input");
  const char* tb[8];
  const char* te[8];
  const int nh = split_tokens(line, tb, te, 8);
  std::vector<std::string> header;
  for (int k = 0; k < std::min(nh, 8); ++k) header.emplace_back(tb[k], te[k]);
  if (nh != 5 || lower(header[0]) != "%%matrixmarket")
    parse_fail(rd.line_no, "expected header '%%MatrixMarket matrix <format> real general'");
  if (lower(header[1]) != "matrix") parse_fail(rd.line_no, "unsupported object '" + header[1] + "'");
  const std::string format = lower(header[2]);
  if (format != "coordinate" && format != "array")
    parse_fail(rd.line_no, "unsupported format '" + header[2] + "'");
  if (lower(header[3]) != "real")
    parse_fail(rd.line_no, "unsupported field '" + header[3] + "' (only real is accepted)");
  if (lower(header[4]) != "general")
    parse_fail(rd.line_no, "unsupported symmetry '" + header[4] + "' (only general is accepted)");
  for (;;) {  // comments, then the size line (:90-96)
    if (!rd.next(line)) parse_fail(rd.line_no + 1, "missing size line");
    if (line.comment()) continue;
    if (split_tokens(line, tb, te, 8) == 0) continue;
    break;
  }
  const int ns = split_tokens(line, tb, te, 8);
  const int64_t body_line0 = rd.line_no;  // lines before the body
  const char* body = rd.p;
  const char* end = data + len;
  const int parts = nthreads(static_cast<size_t>(end - body));
  const std::vector<const char*> cs = chunk_starts(body, end, parts);
  const int nc = static_cast<int>(cs.size()) - 1;

  if (format == "coordinate") {
    if (ns != 3) parse_fail(rd.line_no, "coordinate size line needs 'rows cols nnz'");
    long long m = 0, n = 0, nnz = 0;
    if (!parse_index(tb[0], te[0], m) || !parse_index(tb[1], te[1], n) ||
        !parse_index(tb[2], te[2], nnz) || m <= 0 || n <= 0 || nnz < 0)
      parse_fail(rd.line_no, "invalid size line '" + line.str() + "'");
    std::vector<CoordChunk> ch(nc);
    {
      std::vector<std::thread> th;
      for (int k = 1; k < nc; ++k)
        th.emplace_back(parse_coord_chunk, cs[k], cs[k + 1], m, n, std::ref(ch[k]));
      if (nc > 0) parse_coord_chunk(cs[0], cs[1], m, n, ch[0]);
      for (auto& t : th) t.join();
    }
    // replay the sequential rules in line order (:102-131)
    out.dense = false;
    out.m = m;
    out.n = n;
    out.nnz = nnz;
    int64_t total_lines = body_line0, taken = 0;
    for (int k = 0; k < nc; ++k) total_lines += ch[k].lines;
    out.row.reserve(static_cast<size_t>(nnz));
    out.col.reserve(static_cast<size_t>(nnz));
    out.val.reserve(static_cast<size_t>(nnz));
    out.line.reserve(static_cast<size_t>(nnz));
    int64_t base = body_line0;
    for (int k = 0; k < nc; ++k) {
      const CoordChunk& c = ch[k];
      const int64_t cnt = static_cast<int64_t>(c.row.size());
      const int64_t use = std::min<int64_t>(cnt, nnz - taken);
      size_t bi = 0;
      for (int64_t q = 0; q < use; ++q) {
        if (c.status[q] != kOk) {
          while (c.raw_at[bi] != q) ++bi;
          const int64_t ln = base + c.line[q];
          if (c.status[q] == kTokens) parse_fail(ln, "entry line needs 'row col value'");
          if (c.status[q] == kMalformed) parse_fail(ln, "malformed entry '" + c.raw[bi] + "'");
          parse_fail(ln, "index (" + std::to_string(c.bad_i[bi]) + ", " +
                             std::to_string(c.bad_j[bi]) + ") out of range");
        }
      }
      out.row.insert(out.row.end(), c.row.begin(), c.row.begin() + use);
      out.col.insert(out.col.end(), c.col.begin(), c.col.begin() + use);
      out.val.insert(out.val.end(), c.val.begin(), c.val.begin() + use);
      for (int64_t q = 0; q < use; ++q) out.line.push_back(base + c.line[q]);
      taken += use;
      if (use < cnt)  // more data lines than declared
        parse_fail(base + c.line[use],
                   "trailing data after " + std::to_string(nnz) + " declared entries");
      base += c.lines;
    }
    if (taken < nnz)
      parse_fail(total_lines + 1, "unexpected end of file: expected " + std::to_string(nnz) +
                                      " entries, found " + std::to_string(taken));
    return;
  }

  // array format: column-major values, any number per line (:163-196)
  if (ns != 2) parse_fail(rd.line_no, "array size line needs 'rows cols'");
  long long m = 0, n = 0;
  if (!parse_index(tb[0], te[0], m) || !parse_index(tb[1], te[1], n) || m <= 0 || n <= 0)
    parse_fail(rd.line_no, "invalid size line '" + line.str() + "'");
  std::vector<ArrayChunk> ch(nc);
  {
    std::vector<std::thread> th;
    for (int k = 1; k < nc; ++k) th.emplace_back(parse_array_chunk, cs[k], cs[k + 1], std::ref(ch[k]));
    if (nc > 0) parse_array_chunk(cs[0], cs[1], ch[0]);
    for (auto& t : th) t.join();
  }
  const long long total = m * n;
  out.dense = true;
  out.m = m;
  out.n = n;
  out.nnz = total;
  out.dense_rowmajor.assign(static_cast<size_t>(total), 0.0);
  int64_t base = body_line0, count = 0, total_lines = body_line0;
  for (int k = 0; k < nc; ++k) total_lines += ch[k].lines;
  for (int k = 0; k < nc; ++k) {
    const ArrayChunk& c = ch[k];
    size_t bi = 0;
    const int64_t cnt = static_cast<int64_t>(c.val.size());
    for (int64_t q = 0; q < cnt; ++q) {
      const int64_t ln = base + c.line_of_tok[q];
      if (count >= total) {
        // the line that completed rows*cols has more tokens, or a later line
        const bool same_line = q > 0 && c.line_of_tok[q - 1] == c.line_of_tok[q];
        if (same_line) parse_fail(ln, "more values than rows*cols");
        parse_fail(ln, "trailing data after rows*cols values");
      }
      if (!c.ok[q]) {
        while (c.bad_at[bi] != q) ++bi;
        parse_fail(ln, "malformed value '" + c.bad_tok[bi] + "'");
      }
      out.dense_rowmajor[static_cast<size_t>((count % m) * n + count / m)] = c.val[q];
      ++count;
    }
    base += c.lines;
  }
  if (count < total)
    parse_fail(total_lines + 1, "unexpected end of file: expected " + std::to_string(total) +
                                    " values, found " + std::to_string(count));
}

void read_file(const std::string& path, std::string& buf) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw std::runtime_error("matrix market: cannot open '" + path + "'");
  std::fseek(f, 0, SEEK_END);
  const long sz = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  buf.resize(static_cast<size_t>(std::max(0L, sz)));
  const size_t got = sz > 0 ? std::fread(&buf[0], 1, buf.size(), f) : 0;
  std::fclose(f);
  if (got != buf.size()) throw std::runtime_error("matrix market: cannot open '" + path + "'");
}

// write_matrix_market (:209-233): entries in CSR order, 1-based, "%.17g"
void write_coordinate(const std::string& path, int64_t m, int64_t n, const int64_t* rp,
                      const int32_t* col, const double* val) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f)
    throw std::runtime_error("matrix market: cannot open '" + path + "' for writing");
  const int64_t nnz = rp[m];
  std::string head = "%%MatrixMarket matrix coordinate real general\n" + std::to_string(m) + " " +
                     std::to_string(n) + " " + std::to_string(nnz) + "\n";
  bool ok = std::fwrite(head.data(), 1, head.size(), f) == head.size();
  const int parts = std::max(1, std::min<int>(nthreads(static_cast<size_t>(nnz) * 32), 64));
  std::vector<std::string> out(parts);
  std::vector<std::thread> th;
  auto work = [&](int t) {
    const int64_t r0 = m * t / parts, r1 = m * (t + 1) / parts;
    std::string& s = out[t];
    s.reserve(static_cast<size_t>(rp[r1] - rp[r0]) * 36);
    char buf[96];
    for (int64_t i = r0; i < r1; ++i)
      for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
        const int w = std::snprintf(buf, sizeof buf, "%lld %lld %.17g\n",
                                    static_cast<long long>(i + 1),
                                    static_cast<long long>(col[k]) + 1, val[k]);
        s.append(buf, static_cast<size_t>(w));
      }
  };
  for (int t = 1; t < parts; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  for (const std::string& s : out) ok = ok && std::fwrite(s.data(), 1, s.size(), f) == s.size();
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) throw std::runtime_error("matrix market: write failed");
}

// dense: column-major values one per line
void write_array(const std::string& path, int64_t m, int64_t n, const double* rowmajor) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f)
    throw std::runtime_error("matrix market: cannot open '" + path + "' for writing");
  std::string head = "%%MatrixMarket matrix array real general\n" + std::to_string(m) + " " +
                     std::to_string(n) + "\n";
  bool ok = std::fwrite(head.data(), 1, head.size(), f) == head.size();
  const int parts = std::max(1, std::min<int>(nthreads(static_cast<size_t>(m * n) * 24), 64));
  std::vector<std::string> out(parts);
  std::vector<std::thread> th;
  auto work = [&](int t) {
    const int64_t j0 = n * t / parts, j1 = n * (t + 1) / parts;
    char buf[64];
    for (int64_t j = j0; j < j1; ++j)
      for (int64_t i = 0; i < m; ++i) {
        const int w = std::snprintf(buf, sizeof buf, "%.17g\n", rowmajor[i * n + j]);
        out[t].append(buf, static_cast<size_t>(w));
      }
  };
  for (int t = 1; t < parts; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  for (const std::string& s : out) ok = ok && std::fwrite(s.data(), 1, s.size(), f) == s.size();
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) throw std::runtime_error("matrix market: write failed");
}

// ---- binary CSR: "EQBCSR01", int64 m, n, nnz, int64 dense flag, then
// row_ptr (int64, m+1), col (int32, nnz), val (f64, nnz); dense: f64 m*n row-major
namespace {
constexpr char kMagic[8] = {'E', 'Q', 'B', 'C', 'S', 'R', '0', '1'};
}

void write_binary(const std::string& path, int64_t m, int64_t n, bool dense, const int64_t* rp,
                  const int32_t* col, const double* val, const double* rowmajor) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw std::runtime_error("binary csr: cannot open '" + path + "' for writing");
  const int64_t nnz = dense ? m * n : rp[m];
  const int64_t hdr[4] = {m, n, nnz, dense ? 1 : 0};
  bool ok = std::fwrite(kMagic, 1, 8, f) == 8 && std::fwrite(hdr, 8, 4, f) == 4;
  if (dense) {
    ok = ok && std::fwrite(rowmajor, 8, static_cast<size_t>(nnz), f) == static_cast<size_t>(nnz);
  } else {
    ok = ok && std::fwrite(rp, 8, static_cast<size_t>(m + 1), f) == static_cast<size_t>(m + 1);
    ok = ok && std::fwrite(col, 4, static_cast<size_t>(nnz), f) == static_cast<size_t>(nnz);
    ok = ok && std::fwrite(val, 8, static_cast<size_t>(nnz), f) == static_cast<size_t>(nnz);
  }
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) throw std::runtime_error("binary csr: write failed");
}

void read_binary_header(FILE* f, const std::string& path, int64_t hdr[4]) {
  char magic[8];
  if (std::fread(magic, 1, 8, f) != 8 || std::memcmp(magic, kMagic, 8) != 0 ||
      std::fread(hdr, 8, 4, f) != 4)
    throw std::runtime_error("binary csr: '" + path + "' is not an EQBCSR01 file");
  if (hdr[0] <= 0 || hdr[1] <= 0 || hdr[2] < 0 || (hdr[3] != 0 && hdr[3] != 1))
    throw std::runtime_error("binary csr: '" + path + "' has a corrupt header");
}

void read_exact(FILE* f, void* dst, size_t size, size_t count, const std::string& path) {
  // large reads in parallel would not help a single file descriptor; read in
  // 256 MB pieces so the destination (pinned by the caller) fills steadily
  char* p = static_cast<char*>(dst);
  size_t left = size * count;
  while (left > 0) {
    const size_t piece = std::min<size_t>(left, size_t(256) << 20);
    if (std::fread(p, 1, piece, f) != piece)
      throw std::runtime_error("binary csr: '" + path + "' is truncated");
    p += piece;
    left -= piece;
  }
}

}  // namespace mm
}  // namespace eqb
