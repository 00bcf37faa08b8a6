// Native reader of the reference's graph file format
// (/root/reference/pkg/src/acedag/graphbuild.py:355-464).
//
// One pass over the bytes: a strict UTF-8 scan, the header fields, then one
// node per line with the reference's checks in the reference's order, so the
// first violation found here is the one the reference reports, at the same
// byte offset.  The node's tuple is kept as ascending label ids (graph.h), so
// the parent-union check is a merge of two sorted id lists and the duplicate
// check a TupleMap probe.  Messages that quote the offending text are
// composed by the Python shim from the line span (it has Python's repr); the
// C side keeps a plain description for other callers of the ABI.
//
// Restrictions (documented in DESIGN.md): numerals must be ASCII (Python's
// int() also takes other Unicode digits), and the first L nodes must be the
// order-1 seeds in one_particle_indices order -- the column layout every
// kernel relies on, and what build_graph always writes (graphbuild.py:127-130).
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "graph.h"

namespace acedag {
namespace {

// offset of the first byte of the first invalid sequence (what Python's
// strict decoder reports as UnicodeDecodeError.start), or -1
int64_t utf8_bad(const unsigned char* s, size_t n) {
  size_t i = 0;
  while (i < n) {
    const unsigned c = s[i];
    if (c < 0x80) {
      ++i;
      continue;
    }
    size_t need;
    unsigned lo = 0x80, hi = 0xBF;
    if (c >= 0xC2 && c <= 0xDF) need = 1;
    else if (c == 0xE0) need = 2, lo = 0xA0;
    else if (c >= 0xE1 && c <= 0xEC) need = 2;
    else if (c == 0xED) need = 2, hi = 0x9F;
    else if (c >= 0xEE && c <= 0xEF) need = 2;
    else if (c == 0xF0) need = 3, lo = 0x90;
    else if (c >= 0xF1 && c <= 0xF3) need = 3;
    else if (c == 0xF4) need = 3, hi = 0x8F;
    else return (int64_t)i;
    if (i + need >= n) return (int64_t)i;  // truncated sequence
    for (size_t k = 1; k <= need; ++k) {
      const unsigned d = s[i + k];
      const unsigned a = k == 1 ? lo : 0x80, b = k == 1 ? hi : 0xBF;
      if (d < a || d > b) return (int64_t)i;
    }
    i += need + 1;
  }
  return -1;
}

struct Span {
  const char* p = nullptr;
  size_t n = 0;
  bool eq(const char* lit) const { return n == std::strlen(lit) && std::memcmp(p, lit, n) == 0; }
};

bool is_ascii_digit(char c) { return c >= '0' && c <= '9'; }
// ASCII characters for which Python's str.isspace() holds
bool py_space(char c) { return c == ' ' || (c >= '\t' && c <= '\r') || (c >= '\x1c' && c <= '\x1f'); }

// Python int(text) for ASCII text: surrounding whitespace, one sign, digits
// with single underscores between them.  Saturates (the sign survives).
bool py_int(Span t, int64_t& v) {
  size_t b = 0, e = t.n;
  while (b < e && py_space(t.p[b])) ++b;
  while (e > b && py_space(t.p[e - 1])) --e;
  bool neg = false;
  if (b < e && (t.p[b] == '+' || t.p[b] == '-')) neg = t.p[b++] == '-';
  if (b == e) return false;
  uint64_t acc = 0;
  bool prev_digit = false, sat = false;
  for (size_t i = b; i < e; ++i) {
    const char c = t.p[i];
    if (c == '_') {
      if (!prev_digit || i + 1 == e) return false;
      prev_digit = false;
      continue;
    }
    if (!is_ascii_digit(c)) return false;
    prev_digit = true;
    if (!sat) {
      acc = acc * 10 + (uint64_t)(c - '0');
      if (acc > (uint64_t)INT64_MAX) sat = true;
    }
  }
  if (!prev_digit) return false;
  const int64_t m = sat ? INT64_MAX : (int64_t)acc;
  v = neg ? -m : m;
  return true;
}

// Python float(text) for the header's [0-9.]+ field
bool py_float_digits(Span t, double& v) {
  int dots = 0, digits = 0;
  for (size_t i = 0; i < t.n; ++i) {
    if (t.p[i] == '.') ++dots;
    else ++digits;
  }
  if (dots > 1 || digits == 0) return false;
  v = std::strtod(std::string(t.p, t.n).c_str(), nullptr);
  return true;
}

// splits s on sep into at most `cap` pieces (returns the true count)
size_t split(Span s, char sep, Span* out, size_t cap) {
  size_t k = 0, b = 0;
  for (size_t i = 0; i <= s.n; ++i) {
    if (i == s.n || s.p[i] == sep) {
      if (k < cap) out[k] = Span{s.p + b, i - b};
      ++k;
      b = i + 1;
    }
  }
  return k;
}

struct Header {
  Span version;
  int group = 0, p = 1, nu_max = 0, alg = 0;
  int64_t n = 1;
  Span degree;
};

// consumes `lit` at the cursor
bool take(Span line, size_t& at, const char* lit) {
  const size_t k = std::strlen(lit);
  if (at + k > line.n || std::memcmp(line.p + at, lit, k) != 0) return false;
  at += k;
  return true;
}
// the run of characters up to the next space (or the end)
Span field(Span line, size_t& at) {
  const size_t b = at;
  while (at < line.n && line.p[at] != ' ') ++at;
  return Span{line.p + b, at - b};
}
bool all_digits(Span s) {
  if (!s.n) return false;
  for (size_t i = 0; i < s.n; ++i)
    if (!is_ascii_digit(s.p[i])) return false;
  return true;
}

// the header pattern of graphbuild.py:363-366, field by field
bool parse_header(Span line, Header& h) {
  size_t at = 0;
  if (!take(line, at, "ACEDAG v")) return false;
  h.version = field(line, at);
  if (!all_digits(h.version) || !take(line, at, " group=")) return false;
  const Span g = field(line, at);
  static const char* groups[] = {"T", "SO2", "O3", "O3F"};
  h.group = -1;
  for (int i = 0; i < 4; ++i)
    if (g.eq(groups[i])) h.group = i;
  if (h.group < 0 || !take(line, at, " p=")) return false;
  const Span p = field(line, at);
  if (p.eq("1")) h.p = 1;
  else if (p.eq("2")) h.p = 2;
  else if (p.eq("inf")) h.p = 0;
  else return false;
  if (!take(line, at, " D=")) return false;
  h.degree = field(line, at);
  if (!h.degree.n) return false;
  for (size_t i = 0; i < h.degree.n; ++i)
    if (!is_ascii_digit(h.degree.p[i]) && h.degree.p[i] != '.') return false;
  if (!take(line, at, " numax=")) return false;
  const Span nm = field(line, at);
  int64_t v = 0;
  if (!all_digits(nm) || !py_int(nm, v)) return false;
  h.nu_max = v > (int64_t)1 << 30 ? 1 << 30 : (int)v;
  if (!take(line, at, " alg=")) return false;
  const Span a = field(line, at);
  if (a.eq("orig")) h.alg = 0;
  else if (a.eq("gen")) h.alg = 1;
  else return false;
  if (!take(line, at, " n=")) return false;
  const Span ns = field(line, at);
  if (!all_digits(ns) || !py_int(ns, h.n)) return false;
  return at == line.n;
}

// "ACEDAG v<digits>" followed by a word boundary: the version the reference
// names in its UnsupportedVersionError
bool version_prefix(Span line, Span& ver) {
  size_t at = 0;
  if (!take(line, at, "ACEDAG v")) return false;
  const size_t b = at;
  while (at < line.n && is_ascii_digit(line.p[at])) ++at;
  if (at == b) return false;
  if (at < line.n) {
    const unsigned char c = (unsigned char)line.p[at];
    const bool word = c >= 0x80 || std::isalnum(c) || c == '_';
    if (word) return false;
  }
  ver = Span{line.p + b, at - b};
  return true;
}

// parse_elements (indexsets.py:439-453) validity, then the label ids of the
// elements (-1 for a well-formed element outside this graph's label set)
struct Elements {
  int count = 0;
  int32_t id[kMaxOrder + 1];
};

bool parse_elements(const Graph& g, const std::unordered_map<uint64_t, int32_t>& lab, Span text, Elements& out,
                    bool& too_long) {
  const int k = g.group == kT ? 1 : (g.group == kSO2 ? 2 : (g.group == kO3 ? 3 : 4));
  too_long = false;
  const size_t ncomp = split(text, ',', nullptr, 0);
  std::vector<Span> tok(ncomp);
  split(text, ',', tok.data(), ncomp);
  std::vector<int64_t> c(ncomp);
  for (size_t i = 0; i < ncomp; ++i)
    if (!py_int(tok[i], c[i])) return false;
  if (ncomp == 0 || ncomp % k) return false;
  const size_t ne = ncomp / k;
  for (size_t e = 0; e < ne; ++e) {  // validate_element
    const int64_t* x = &c[e * k];
    if (g.group == kSO2 && x[0] < 0) return false;
    if (g.group == kO3 || g.group == kO3F) {
      if (x[0] < 0 || x[1] < 0) return false;
      const int64_t am = x[2] == INT64_MIN ? INT64_MAX : (x[2] < 0 ? -x[2] : x[2]);
      if (am > x[1]) return false;
      if (g.group == kO3F && x[3] < 0) return false;
    }
  }
  for (size_t e = 1; e < ne; ++e) {  // canonical order: Python tuple comparison
    const int64_t *a = &c[(e - 1) * k], *b = &c[e * k];
    for (int j = 0; j < k; ++j) {
      if (a[j] < b[j]) break;
      if (a[j] > b[j]) return false;
    }
  }
  if (ne > (size_t)kMaxOrder) {
    too_long = true;
    return true;
  }
  out.count = (int)ne;
  for (size_t e = 0; e < ne; ++e) {
    uint64_t key = 0;
    bool in_range = true;
    for (int j = 0; j < k; ++j) {
      const int64_t x = c[e * k + j];
      if (x < -32768 || x > 32767) in_range = false;
      key = key << 16 | (uint16_t)(int16_t)(in_range ? x : 0);
    }
    auto it = in_range ? lab.find(key) : lab.end();
    out.id[e] = it == lab.end() ? -1 : it->second;
  }
  return true;
}

uint64_t label_key(const Label& L) {
  uint64_t key = 0;
  for (int j = 0; j < L.ncomp; ++j) key = key << 16 | (uint16_t)(int16_t)L.comp[j];
  return key;
}

bool fail(GraphParseError& err, int kind, int64_t offset, const char* line, int64_t line_len, const char* base,
          const std::string& what) {
  err.kind = kind;
  err.offset = offset;
  err.line_start = line ? (int64_t)(line - base) : 0;
  err.line_len = line_len;
  err.message = what + " (at byte " + std::to_string(offset) + ")";
  return false;
}

}  // namespace

bool deserialize_graph(const char* data, size_t n, Graph& g, GraphParseError& err) {
  err = GraphParseError{};
  const int64_t bad = utf8_bad(reinterpret_cast<const unsigned char*>(data), n);
  if (bad >= 0) return fail(err, kGeNotUtf8, bad, nullptr, 0, data, "graph data is not valid UTF-8");
  const char* nl = static_cast<const char*>(std::memchr(data, '\n', n));
  const Span head{data, nl ? (size_t)(nl - data) : n};
  Header h;
  if (!parse_header(head, h)) {
    Span ver;
    if (version_prefix(head, ver) && !ver.eq("1"))
      return fail(err, kGeVersion, 0, data, (int64_t)head.n, data, "unsupported graph format version");
    return fail(err, kGeHeader, 0, data, (int64_t)head.n, data, "bad header line");
  }
  if (!h.version.eq("1")) return fail(err, kGeVersion, 0, data, (int64_t)head.n, data, "unsupported graph format version");
  double D = 0;
  if (!py_float_digits(h.degree, D)) return fail(err, kGeDegree, 0, data, (int64_t)head.n, data, "bad degree cap");
  try {
    init_graph(g, h.group, h.p, D, h.nu_max, h.alg, (int)(h.n > (1 << 30) ? (1 << 30) : h.n));
  } catch (const std::exception& e) {
    return fail(err, kGeLimit, 0, data, (int64_t)head.n, data, e.what());
  }
  std::unordered_map<uint64_t, int32_t> lab;
  lab.reserve(g.labels.size() * 2);
  for (size_t i = 0; i < g.labels.size(); ++i) lab.emplace(label_key(g.labels[i]), (int32_t)i);
  const int64_t L = g.n_seeds();
  g.ids.reserve((size_t)(n / 24) + 16);
  size_t pos = head.n + 1;  // offset of the next line (the reference adds 1 per split piece)
  if (!nl) pos = n + 1;
  Span parts[6];
  while (pos <= n) {
    const char* ls = data + pos;
    const char* le = static_cast<const char*>(std::memchr(ls, '\n', n - pos));
    const size_t len = le ? (size_t)(le - ls) : n - pos;
    const int64_t at = (int64_t)pos;
    pos += len + 1;
    if (!len) continue;
    const Span line{ls, len};
    auto bad_line = [&](int kind, const std::string& what) {
      return fail(err, kind, at, ls, (int64_t)len, data, what);
    };
    const size_t np = split(line, ' ', parts, 6);
    if (np != 4 && np != 5) return bad_line(kGeNodeLine, "bad node line");
    int64_t ident = 0, auxv = 0;
    if (!py_int(parts[0], ident) || !py_int(parts[1], auxv)) return bad_line(kGeNodeLine, "bad node line");
    const int64_t nodes = (int64_t)g.tuples.size();
    if (ident != nodes) return bad_line(kGeNotDense, "node ids must be dense and ascending");
    if (auxv != 0 && auxv != 1) return bad_line(kGeAuxFlag, "auxiliary flag must be 0 or 1");
    Elements el;
    bool too_long = false;
    if (!parse_elements(g, lab, parts[2], el, too_long)) return bad_line(kGeElements, "bad tuple field");
    Tuple t;
    int32_t pa = -1, pb = -1;
    if (parts[3].eq("-")) {
      if (np != 4) return bad_line(kGeParentField, "bad parent field");
      if (too_long || el.count != 1) return bad_line(kGeOrphan, "only order-1 nodes may lack parents");
    } else {
      if (np != 5) return bad_line(kGeParentField, "bad parent field");
      int64_t a = 0, b = 0;
      if (!py_int(parts[3], a) || !py_int(parts[4], b)) return bad_line(kGeParentIds, "bad parent ids");
      if (a < 0 || a >= ident || b < 0 || b >= ident) return bad_line(kGeParentOrder, "parent ids must precede node");
      if (too_long) return bad_line(kGeLimit, "node order above the native limit of 8");
      const Tuple &ta = g.tuples[a], &tb = g.tuples[b];
      // the union of the parents, as ascending label ids, against the node
      bool same = ta.len + tb.len == el.count;
      if (same) {
        int x = 0, y = 0;
        for (int i = 0; i < el.count; ++i) {
          const uint16_t nx = (y >= tb.len || (x < ta.len && ta.id[x] <= tb.id[y])) ? ta.id[x++] : tb.id[y++];
          if (el.id[i] != (int32_t)nx) {
            same = false;
            break;
          }
        }
      }
      if (!same) return bad_line(kGeUnion, "parents do not union to node");
      pa = (int32_t)a;
      pb = (int32_t)b;
    }
    if (el.count == 1 && auxv) return bad_line(kGeSeedAux, "order-1 nodes cannot be auxiliary");
    for (int i = 0; i < el.count; ++i) {
      if (el.id[i] < 0) return bad_line(kGeSeedLayout, "label outside the graph's one-particle set");
      t.id[t.len++] = (uint16_t)el.id[i];
    }
    if (t.len > 1 && (auxv != 0) == g.is_target(t)) return bad_line(kGeAuxMismatch, "auxiliary flag inconsistent on node");
    if (g.ids.get(t) >= 0) return bad_line(kGeDuplicate, "duplicate tuple at node");
    // the layout the kernels need: seeds first, in label order
    if ((ident < L) != (t.len == 1) || (t.len == 1 && t.id[0] != ident))
      return bad_line(kGeSeedLayout, "the first nodes must be the order-1 seeds in label order");
    g.add(t, pa, pb);
  }
  if (g.tuples.empty())
    return fail(err, kGeEmpty, (int64_t)n + 1, nullptr, 0, data, "graph has no nodes; order-1 seeds are mandatory");
  if ((int64_t)g.tuples.size() < L)
    return fail(err, kGeSeedLayout, (int64_t)n + 1, nullptr, 0, data, "graph lacks some order-1 seeds");
  return true;
}

}  // namespace acedag
