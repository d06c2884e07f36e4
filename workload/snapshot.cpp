// Snapshot bundle I/O (see snapshot.hpp).
#include "snapshot.hpp"

#include <omp.h>

#include <algorithm>
#include <cctype>
#include <charconv>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <map>
#include <sstream>
#include <stdexcept>

namespace fpb {
namespace {

namespace fs = std::filesystem;

bool slurp(const std::string& path, std::string& out) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) return false;
  std::fseek(f, 0, SEEK_END);
  const long len = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  out.resize(len > 0 ? size_t(len) : 0);
  const size_t got = out.empty() ? 0 : std::fread(out.data(), 1, out.size(), f);
  std::fclose(f);
  out.resize(got);
  return true;
}

inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f'; }

// Whitespace-separated tokens of [b, e) split into chunks that never cut a token.
struct Chunks {
  std::vector<size_t> lo, hi;
  std::vector<long long> first;  // global index of each chunk's first token
  long long total = 0;
};

Chunks chunk_tokens(const std::string& s, size_t b, size_t e) {
  Chunks C;
  const size_t len = e - b;
  const int n = int(std::max<size_t>(1, std::min<size_t>(size_t(omp_get_max_threads()) * 8, len / (1u << 20))));
  std::vector<size_t> cut(static_cast<size_t>(n) + 1, e);
  cut[0] = b;
  for (int c = 1; c < n; ++c) {
    size_t p = b + len * size_t(c) / size_t(n);
    p = std::max(p, cut[c - 1]);
    while (p < e && !is_ws(s[p])) ++p;  // move to a token boundary
    cut[c] = p;
  }
  C.lo.assign(cut.begin(), cut.end() - 1);
  C.hi.assign(cut.begin() + 1, cut.end());
  std::vector<long long> cnt(static_cast<size_t>(n), 0);
#pragma omp parallel for schedule(dynamic, 1)
  for (int c = 0; c < n; ++c) {
    long long k = 0;
    bool in = false;
    for (size_t p = C.lo[c]; p < C.hi[c]; ++p) {
      const bool w = is_ws(s[p]);
      if (!w && !in) ++k;
      in = !w;
    }
    cnt[c] = k;
  }
  C.first.resize(static_cast<size_t>(n));
  for (int c = 0; c < n; ++c) C.first[c] = C.total, C.total += cnt[c];
  return C;
}

// Visit the tokens of chunk c in order: fn(global_index, begin, end) -> false stops the chunk.
template <class Fn>
void for_tokens(const std::string& s, const Chunks& C, int c, Fn fn) {
  long long g = C.first[c];
  size_t p = C.lo[c];
  const size_t e = C.hi[c];
  while (p < e) {
    while (p < e && is_ws(s[p])) ++p;
    if (p >= e) break;
    const size_t t0 = p;
    while (p < e && !is_ws(s[p])) ++p;
    if (!fn(g++, s.data() + t0, s.data() + p)) return;
  }
}

template <class T>
bool parse_num(const char* b, const char* e, T& out) {
  if (b < e && *b == '+') ++b;  // stream extraction accepts a leading '+'
  auto r = std::from_chars(b, e, out);
  return r.ec == std::errc() && r.ptr == e;
}

// from_triplets (csr.cpp): stable (row, col) order, duplicates summed from 0.0 in input order
Csr csr_from_entries(int rows, int cols, const std::vector<int>& ri, const std::vector<int>& cj,
                     const std::vector<double>& v) {
  const size_t m = v.size();
  Csr A(rows, cols);
  std::vector<int64_t> start(static_cast<size_t>(rows) + 1, 0);
  for (size_t k = 0; k < m; ++k) ++start[size_t(ri[k]) + 1];
  for (int r = 0; r < rows; ++r) start[size_t(r) + 1] += start[r];
  std::vector<int64_t> order(m);
  {
    std::vector<int64_t> next(start.begin(), start.end() - 1);
    for (size_t k = 0; k < m; ++k) order[size_t(next[ri[k]]++)] = int64_t(k);  // stable in file order
  }
  std::vector<int64_t> kept(static_cast<size_t>(rows), 0);
#pragma omp parallel for schedule(dynamic, 256)
  for (int r = 0; r < rows; ++r) {
    int64_t* o = order.data() + start[r];
    const int64_t len = start[r + 1] - start[r];
    std::stable_sort(o, o + len, [&](int64_t a, int64_t b) { return cj[a] < cj[b]; });
    int64_t distinct = 0;
    for (int64_t i = 0; i < len; ++i) distinct += (i == 0 || cj[o[i]] != cj[o[i - 1]]);
    kept[r] = distinct;
  }
  for (int r = 0; r < rows; ++r) A.rp[size_t(r) + 1] = A.rp[r] + kept[r];
  A.ci.resize(size_t(A.rp[rows]));
  A.v.resize(size_t(A.rp[rows]));
#pragma omp parallel for schedule(dynamic, 256)
  for (int r = 0; r < rows; ++r) {
    const int64_t* o = order.data() + start[r];
    const int64_t len = start[r + 1] - start[r];
    int64_t w = A.rp[r];
    for (int64_t i = 0; i < len;) {
      const int c = cj[o[i]];
      double sum = 0.0;
      for (; i < len && cj[o[i]] == c; ++i) sum += v[size_t(o[i])];
      A.ci[size_t(w)] = c;
      A.v[size_t(w)] = sum;
      ++w;
    }
  }
  return A;
}

// ------------------------------------------------------------------ JSON
struct JVal {
  enum Kind { null_, boolean, number, string, array, object } kind = null_;
  double num = 0.0;
  bool b = false;
  std::string str;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;
  const JVal* get(const std::string& k) const {
    for (const auto& [key, val] : obj)
      if (key == k) return &val;
    return nullptr;
  }
};

struct JParser {
  const std::string& s;
  size_t p = 0;
  [[noreturn]] void fail() { throw std::invalid_argument("import_snapshot: manifest.json is not valid JSON"); }
  void ws() {
    while (p < s.size() && is_ws(s[p])) ++p;
  }
  bool eat(char c) {
    ws();
    if (p < s.size() && s[p] == c) return ++p, true;
    return false;
  }
  std::string str() {
    if (!eat('"')) fail();
    std::string out;
    while (p < s.size() && s[p] != '"') {
      char c = s[p++];
      if (c == '\\') {
        if (p >= s.size()) fail();
        const char e = s[p++];
        switch (e) {
          case '"': case '\\': case '/': out.push_back(e); break;
          case 'b': out.push_back('\b'); break;
          case 'f': out.push_back('\f'); break;
          case 'n': out.push_back('\n'); break;
          case 'r': out.push_back('\r'); break;
          case 't': out.push_back('\t'); break;
          case 'u': {
            if (p + 4 > s.size()) fail();
            unsigned cp = 0;
            if (std::from_chars(s.data() + p, s.data() + p + 4, cp, 16).ptr != s.data() + p + 4) fail();
            p += 4;
            if (cp < 0x80) out.push_back(char(cp));
            else if (cp < 0x800) out.push_back(char(0xC0 | (cp >> 6))), out.push_back(char(0x80 | (cp & 0x3F)));
            else out.push_back(char(0xE0 | (cp >> 12))), out.push_back(char(0x80 | ((cp >> 6) & 0x3F))),
                 out.push_back(char(0x80 | (cp & 0x3F)));
            break;
          }
          default: fail();
        }
      } else {
        out.push_back(c);
      }
    }
    if (p >= s.size()) fail();
    ++p;
    return out;
  }
  JVal value() {
    ws();
    if (p >= s.size()) fail();
    JVal v;
    const char c = s[p];
    if (c == '{') {
      ++p;
      v.kind = JVal::object;
      if (eat('}')) return v;
      do {
        std::string k = str();
        if (!eat(':')) fail();
        v.obj.emplace_back(std::move(k), value());
      } while (eat(','));
      if (!eat('}')) fail();
    } else if (c == '[') {
      ++p;
      v.kind = JVal::array;
      if (eat(']')) return v;
      do v.arr.push_back(value());
      while (eat(','));
      if (!eat(']')) fail();
    } else if (c == '"') {
      v.kind = JVal::string;
      v.str = str();
    } else if (s.compare(p, 4, "true") == 0) {
      v.kind = JVal::boolean, v.b = true, p += 4;
    } else if (s.compare(p, 5, "false") == 0) {
      v.kind = JVal::boolean, p += 5;
    } else if (s.compare(p, 4, "null") == 0) {
      p += 4;
    } else {
      size_t q = p;
      while (q < s.size() && (std::isdigit(static_cast<unsigned char>(s[q])) || s[q] == '-' || s[q] == '+' ||
                              s[q] == '.' || s[q] == 'e' || s[q] == 'E'))
        ++q;
      v.kind = JVal::number;
      if (q == p || !parse_num(s.data() + p, s.data() + q, v.num)) fail();
      p = q;
    }
    return v;
  }
};

const JVal& need_key(const JVal& m, const char* k) {
  const JVal* v = m.get(k);
  if (!v) throw std::invalid_argument(std::string("import_snapshot: manifest has no \"") + k + "\"");
  return *v;
}
int need_int(const JVal& m, const char* k) {
  const JVal& v = need_key(m, k);
  if (v.kind != JVal::number || v.num != double(int(v.num)))
    throw std::invalid_argument(std::string("import_snapshot: manifest \"") + k + "\" is not an integer");
  return int(v.num);
}
const std::string& need_str(const JVal& m, const char* k) {
  const JVal& v = need_key(m, k);
  if (v.kind != JVal::string)
    throw std::invalid_argument(std::string("import_snapshot: manifest \"") + k + "\" is not a string");
  return v.str;
}

std::string json_escape(const std::string& s) {
  std::string o;
  for (char c : s) {
    if (c == '"' || c == '\\') o.push_back('\\'), o.push_back(c);
    else if (static_cast<unsigned char>(c) < 0x20) {
      char b[8];
      std::snprintf(b, sizeof b, "\\u%04x", unsigned(c));
      o += b;
    } else {
      o.push_back(c);
    }
  }
  return o;
}

std::string json_number(double x) {  // shortest round trip, integral values keep ".0" (nlohmann's dump)
  char b[64];
  auto r = std::to_chars(b, b + sizeof b, x);
  std::string s(b, r.ptr);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

}  // namespace

// ------------------------------------------------------------ Matrix Market
Csr read_matrix_market(const std::string& path) {
  std::string buf;
  if (!slurp(path, buf)) throw std::invalid_argument("cannot open matrix file: " + path);
  if (buf.empty()) throw std::invalid_argument("empty matrix file: " + path);
  size_t eol = buf.find('\n');
  if (eol == std::string::npos) eol = buf.size();
  {
    std::istringstream hs(buf.substr(0, eol));
    std::string banner, object, format, field, symmetry;
    hs >> banner >> object >> format >> field >> symmetry;
    if (banner != "%%MatrixMarket" || object != "matrix" || format != "coordinate")
      throw std::invalid_argument("unsupported MatrixMarket header in " + path);
    if (field != "real" || (symmetry != "general" && !symmetry.empty() && symmetry != "General"))
      throw std::invalid_argument("only real general coordinate matrices supported: " + path);
  }
  // first non-empty line that is not a comment is the size line
  size_t p = std::min(buf.size(), eol + 1);
  std::string size_line;
  while (p < buf.size()) {
    size_t e = buf.find('\n', p);
    if (e == std::string::npos) e = buf.size();
    if (e > p && buf[p] != '%') {
      size_line = buf.substr(p, e - p);
      p = std::min(buf.size(), e + 1);
      break;
    }
    p = e + 1;
  }
  std::istringstream ss(size_line);
  long rows = 0, cols = 0, entries = 0;
  if (!(ss >> rows >> cols >> entries) || rows < 0 || cols < 0 || entries < 0)
    throw std::invalid_argument("bad size line in " + path);
  const Chunks C = chunk_tokens(buf, std::min(p, buf.size()), buf.size());
  const long long need = 3LL * entries;
  std::vector<int> ri(static_cast<size_t>(entries)), cj(static_cast<size_t>(entries));
  std::vector<double> v(static_cast<size_t>(entries));
  // the first failing entry decides the error, as in the reference's sequential read: an
  // unparsable token stops the stream ("truncated"), else a parsed index outside the matrix
  // ("out of range"); key = 2 * entry + (0 truncated | 1 range), smallest key wins
  long long bad = (C.total < need) ? 2 * (C.total / 3) : (1LL << 62);
  const int n = int(C.lo.size());
#pragma omp parallel for schedule(dynamic, 1)
  for (int c = 0; c < n; ++c) {
    long long my = 1LL << 62;
    for_tokens(buf, C, c, [&](long long g, const char* b, const char* e) {
      if (g >= need) return false;
      const long long ent = g / 3;
      const int fld = int(g % 3);
      if (fld < 2) {
        long x = 0;
        if (!parse_num(b, e, x)) {
          my = std::min(my, 2 * ent);
        } else if (x < 1 || x > (fld == 0 ? rows : cols)) {
          my = std::min(my, 2 * ent + 1);
        } else {
          (fld == 0 ? ri : cj)[size_t(ent)] = int(x - 1);
        }
      } else if (!parse_num(b, e, v[size_t(ent)])) {
        my = std::min(my, 2 * ent);
      }
      return true;
    });
#pragma omp critical
    bad = std::min(bad, my);
  }
  if (bad < (1LL << 62)) {
    if (bad % 2 == 0) throw std::invalid_argument("truncated matrix data in " + path);
    throw std::invalid_argument("entry out of range in " + path);
  }
  std::string().swap(buf);
  return csr_from_entries(int(rows), int(cols), ri, cj, v);
}

void write_matrix_market(const std::string& path, const Csr& A) {
  std::FILE* f = std::fopen(path.c_str(), "w");
  if (!f) throw std::invalid_argument("cannot write matrix file: " + path);
  std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n");
  std::fprintf(f, "%d %d %lld\n", A.n_rows, A.n_cols, static_cast<long long>(A.nnz()));
  constexpr int kRows = 4096, kBatch = 256;  // format 256 chunks of rows in parallel, write them in order
  const int n_chunks = (A.n_rows + kRows - 1) / kRows;
  for (int c0 = 0; c0 < n_chunks; c0 += kBatch) {
    const int c1 = std::min(n_chunks, c0 + kBatch);
    std::vector<std::string> out(static_cast<size_t>(c1 - c0));
#pragma omp parallel for schedule(dynamic, 1)
    for (int c = c0; c < c1; ++c) {
      std::string& o = out[size_t(c - c0)];
      char line[96];
      const int r1 = std::min(A.n_rows, (c + 1) * kRows);
      for (int i = c * kRows; i < r1; ++i)
        for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k) {
          const int len = std::snprintf(line, sizeof line, "%d %d %.17g\n", i + 1, A.ci[k] + 1, A.v[k]);
          o.append(line, size_t(len));
        }
    }
    for (const auto& o : out) std::fwrite(o.data(), 1, o.size(), f);
  }
  if (std::fclose(f) != 0) throw std::invalid_argument("cannot write matrix file: " + path);
}

std::vector<double> read_vector_text(const std::string& path) {
  std::string buf;
  if (!slurp(path, buf)) throw std::invalid_argument("cannot open vector file: " + path);
  const Chunks C = chunk_tokens(buf, 0, buf.size());
  std::vector<double> v(static_cast<size_t>(C.total));
  int bad = 0;
  const int n = int(C.lo.size());
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad)
  for (int c = 0; c < n; ++c)
    for_tokens(buf, C, c, [&](long long g, const char* b, const char* e) {
      if (!parse_num(b, e, v[size_t(g)])) bad = 1;
      return true;
    });
  if (bad) throw std::invalid_argument("malformed vector file: " + path);
  return v;
}

void write_vector_text(const std::string& path, const std::vector<double>& v) {
  std::FILE* f = std::fopen(path.c_str(), "w");
  if (!f) throw std::invalid_argument("cannot write vector file: " + path);
  for (double x : v) std::fprintf(f, "%.17g\n", x);
  if (std::fclose(f) != 0) throw std::invalid_argument("cannot write vector file: " + path);
}

// ------------------------------------------------------------------ bundle
Workload import_snapshot(const std::string& dir) {
  auto path = [&](const std::string& name) { return (fs::path(dir) / name).string(); };
  std::string text;
  if (!slurp(path("manifest.json"), text))
    throw std::invalid_argument("import_snapshot: missing manifest.json in " + dir);
  JParser P{text};
  const JVal m = P.value();
  if (m.kind != JVal::object) P.fail();
  Workload W;
  HostSystem& J = W.J;
  J.n_u = need_int(m, "n_u");
  J.n_t = need_int(m, "n_t");
  J.n_p = need_int(m, "n_p");
  const JVal& dt = need_key(m, "dt");
  if (dt.kind != JVal::number) throw std::invalid_argument("import_snapshot: manifest \"dt\" is not a number");
  W.dt = dt.num;
  if (J.n_t != 3 * J.n_p) throw std::invalid_argument("import_snapshot: manifest violates n_t == 3*n_p");
  W.region = need_str(m, "region");
  if (int(W.region.size()) != J.n_p) throw std::invalid_argument("import_snapshot: region string length mismatch");
  for (char ch : W.region) {
    if (ch != 's' && ch != 'l' && ch != 'o') throw std::invalid_argument("import_snapshot: bad region label");
    (ch == 's' ? W.n_stick : ch == 'l' ? W.n_slip : W.n_open)++;
  }
  const JVal& blocks = need_key(m, "blocks");
  if (blocks.kind != JVal::object) throw std::invalid_argument("import_snapshot: manifest \"blocks\" is not an object");
  J.A = read_matrix_market(path(need_str(blocks, "A")));
  J.C1 = read_matrix_market(path(need_str(blocks, "C1")));
  J.Q1 = read_matrix_market(path(need_str(blocks, "Q1")));
  J.C2 = read_matrix_market(path(need_str(blocks, "C2")));
  J.H = read_matrix_market(path(need_str(blocks, "H")));
  J.Q2 = read_matrix_market(path(need_str(blocks, "Q2")));
  J.T = read_matrix_market(path(need_str(blocks, "T")));
  if (blocks.get("F_u")) J.F_u = read_matrix_market(path(need_str(blocks, "F_u")));
  J.check_shapes();
  if (m.get("coords")) {
    const std::vector<double> flat = read_vector_text(path(need_str(m, "coords")));
    if (int64_t(flat.size()) != J.n_u) throw std::invalid_argument("import_snapshot: coords length mismatch");
    for (size_t i = 0; i + 2 < flat.size(); i += 3) W.coords.push_back({flat[i], flat[i + 1], flat[i + 2]});
  }
  return W;
}

void export_snapshot(const std::string& dir, const HostSystem& J, const std::string& region, double dt,
                     const std::vector<std::array<double, 3>>& coords) {
  J.check_shapes();
  if (int(region.size()) != J.n_p) throw std::invalid_argument("export_snapshot: region labels size mismatch");
  for (char ch : region)
    if (ch != 's' && ch != 'l' && ch != 'o') throw std::invalid_argument("export_snapshot: bad region label");
  std::error_code ec;
  fs::create_directories(dir, ec);
  auto path = [&](const char* name) { return (fs::path(dir) / name).string(); };
  write_matrix_market(path("A.mtx"), J.A);
  write_matrix_market(path("C1.mtx"), J.C1);
  write_matrix_market(path("Q1.mtx"), J.Q1);
  write_matrix_market(path("C2.mtx"), J.C2);
  write_matrix_market(path("H.mtx"), J.H);
  write_matrix_market(path("Q2.mtx"), J.Q2);
  write_matrix_market(path("T.mtx"), J.T);
  write_matrix_market(path("F_u.mtx"), J.F_u.n_rows > 0 ? J.F_u : Csr(J.n_p, J.n_u));
  if (!coords.empty()) {
    std::vector<double> flat;
    flat.reserve(coords.size() * 3);
    for (const auto& c : coords) flat.insert(flat.end(), c.begin(), c.end());
    write_vector_text(path("coords.txt"), flat);
  }
  // keys in sorted order with two-space indentation, like the reference's nlohmann dump(2)
  std::FILE* f = std::fopen(path("manifest.json").c_str(), "w");
  if (!f) throw std::invalid_argument("cannot write manifest: " + path("manifest.json"));
  std::fprintf(f, "{\n  \"blocks\": {\n");
  const char* names[8] = {"A", "C1", "C2", "F_u", "H", "Q1", "Q2", "T"};
  for (int i = 0; i < 8; ++i) std::fprintf(f, "    \"%s\": \"%s.mtx\"%s\n", names[i], names[i], i < 7 ? "," : "");
  std::fprintf(f, "  },\n");
  if (!coords.empty()) std::fprintf(f, "  \"coords\": \"coords.txt\",\n");
  std::fprintf(f, "  \"dt\": %s,\n  \"n_p\": %d,\n  \"n_t\": %d,\n  \"n_u\": %d,\n  \"region\": \"%s\"\n}\n",
               json_number(dt).c_str(), J.n_p, J.n_t, J.n_u, json_escape(region).c_str());
  if (std::fclose(f) != 0) throw std::invalid_argument("cannot write manifest: " + path("manifest.json"));
}

}  // namespace fpb
