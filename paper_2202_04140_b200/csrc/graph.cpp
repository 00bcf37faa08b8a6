// Native DAG construction.  Follows the reference's insertion rules exactly
// so the serialized graph is byte-identical (checked against the golden
// SHA-256 values in tests/golden):
//   one_particle_indices  indexsets.py:170-191
//   target enumeration    indexsets.py:368-388 (set only; build re-sorts)
//   proper_splits         dependency.py:38-60
//   insert_original       graphbuild.py:150-167
//   insert_generalized    graphbuild.py:169-202
//   build_graph           graphbuild.py:243-268
//   serialize_graph       graphbuild.py:355-384
#include "graph.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

namespace acedag {

// ----------------------------------------------------------------- TupleMap
void TupleMap::reserve(size_t n) {
  size_t cap = 16;
  while (cap < 2 * n + 16) cap <<= 1;
  if (cap <= keys_.size()) return;
  std::vector<Tuple> ok;
  std::vector<int32_t> ov;
  ok.swap(keys_);
  ov.swap(vals_);
  keys_.assign(cap, Tuple());
  vals_.assign(cap, -1);
  mask_ = cap - 1;
  n_ = 0;
  for (size_t i = 0; i < ok.size(); ++i)
    if (ov[i] >= 0) put(ok[i], ov[i]);
}

void TupleMap::grow() { reserve(keys_.empty() ? 16 : keys_.size()); }

int32_t TupleMap::get(const Tuple& t) const {
  if (keys_.empty()) return -1;
  size_t i = t.hash() & mask_;
  while (true) {
    if (vals_[i] < 0) return -1;
    if (keys_[i] == t) return vals_[i];
    i = (i + 1) & mask_;
  }
}

void TupleMap::put(const Tuple& t, int32_t v) {
  if (2 * (n_ + 1) > keys_.size()) grow();
  size_t i = t.hash() & mask_;
  while (vals_[i] >= 0) {
    if (keys_[i] == t) {
      vals_[i] = v;
      return;
    }
    i = (i + 1) & mask_;
  }
  keys_[i] = t;
  vals_[i] = v;
  ++n_;
}

// --------------------------------------------------------------------- Spec
int Spec::int_cap() const { return (int)std::floor(max_degree); }

int64_t Spec::power_cap() const {
  if (p == 2) {
    long double d = max_degree;
    return (int64_t)std::floor(d * d);
  }
  return (int64_t)std::floor(max_degree);
}

int64_t Spec::power_key(const Tuple& t, const std::vector<Label>& labels) const {
  int64_t k = 0;
  for (int i = 0; i < t.len; ++i) {
    int64_t d = labels[t.id[i]].degree;
    if (p == 1) k += d;
    else if (p == 2) k += d * d;
    else k = std::max(k, d);
  }
  return k;
}

// ------------------------------------------------------------------- labels
static Label make_label(int ncomp, int a, int b = 0, int c = 0, int d = 0) {
  Label L;
  L.ncomp = ncomp;
  L.comp[0] = a; L.comp[1] = b; L.comp[2] = c; L.comp[3] = d;
  switch (ncomp) {  // indexsets.py:61-79
    case 1: L.degree = std::abs(a); L.m = a; L.l = 0; break;
    case 2: L.degree = a + std::abs(b); L.m = b; L.l = 0; break;
    case 3: L.degree = a + b; L.m = c; L.l = b; break;
    default: L.degree = a + b + d; L.m = c; L.l = b; break;
  }
  return L;
}

std::vector<Label> one_particle_indices(int group, int cap) {
  std::vector<Label> out;
  if (cap < 0) return out;
  if (group == kT) {
    for (int m = -cap; m <= cap; ++m) out.push_back(make_label(1, m));
  } else if (group == kSO2) {
    for (int n = 0; n <= cap; ++n)
      for (int m = -(cap - n); m <= cap - n; ++m) out.push_back(make_label(2, n, m));
  } else if (group == kO3) {
    for (int n = 0; n <= cap; ++n)
      for (int l = 0; l <= cap - n; ++l)
        for (int m = -l; m <= l; ++m) out.push_back(make_label(3, n, l, m));
  } else {
    for (int n = 0; n <= cap; ++n)
      for (int l = 0; l <= cap - n; ++l)
        for (int m = -l; m <= l; ++m)
          for (int f = 0; f <= cap - n - l; ++f) out.push_back(make_label(4, n, l, m, f));
  }
  return out;
}

// -------------------------------------------------------------------- Graph
static bool has_l(int group) { return group == kO3 || group == kO3F; }

bool Graph::satisfies_constraints(const Tuple& t) const {  // indexsets.py:157-163
  int ms = 0, ls = 0;
  for (int i = 0; i < t.len; ++i) {
    ms += labels[t.id[i]].m;
    ls += labels[t.id[i]].l;
  }
  if (ms != 0) return false;
  return !(has_l(group) && (ls & 1));
}

bool Graph::is_target(const Tuple& t) const {  // graphbuild.py:119-123
  if (nu_max > 0 && t.len > nu_max) return false;
  return satisfies_constraints(t) && spec.power_key(t, labels) <= spec.power_cap();
}

int32_t Graph::add(const Tuple& t, int32_t a, int32_t b) {  // graphbuild.py:132-137
  int32_t id = (int32_t)tuples.size();
  tuples.push_back(t);
  pa.push_back(a);
  pb.push_back(b);
  aux.push_back(t.len == 1 ? 0 : (is_target(t) ? 0 : 1));
  ids.put(t, id);
  return id;
}

void Graph::seed() {  // graphbuild.py:127-130
  for (size_t i = 0; i < labels.size(); ++i) {
    Tuple t;
    t.len = 1;
    t.id[0] = (uint16_t)i;
    add(t, -1, -1);
  }
}

// All unordered two-part splits, left <= right, sorted (dependency.py:38-60).
static int proper_splits(const Tuple& t, Tuple* left, Tuple* right) {
  int uid[kMaxOrder], cnt[kMaxOrder], ng = 0;
  for (int i = 0; i < t.len; ++i) {
    if (ng && uid[ng - 1] == t.id[i]) cnt[ng - 1]++;
    else { uid[ng] = t.id[i]; cnt[ng] = 1; ng++; }
  }
  int j[kMaxOrder] = {0};
  int n = 0;
  while (true) {
    Tuple l, r;
    for (int g = 0; g < ng; ++g) {
      for (int c = 0; c < j[g]; ++c) l.id[l.len++] = (uint16_t)uid[g];
      for (int c = j[g]; c < cnt[g]; ++c) r.id[r.len++] = (uint16_t)uid[g];
    }
    if (l.len && r.len && l <= r) { left[n] = l; right[n] = r; n++; }
    int g = 0;
    while (g < ng) {
      if (++j[g] <= cnt[g]) break;
      j[g] = 0;
      ++g;
    }
    if (g == ng) break;
  }
  // insertion sort by (left, right); n <= 128
  for (int a = 1; a < n; ++a) {
    Tuple kl = left[a], kr = right[a];
    int b = a - 1;
    while (b >= 0 && (kl < left[b] || (kl == left[b] && kr < right[b]))) {
      left[b + 1] = left[b];
      right[b + 1] = right[b];
      --b;
    }
    left[b + 1] = kl;
    right[b + 1] = kr;
  }
  return n;
}

static Tuple remove_one(const Tuple& t, uint16_t x) {
  Tuple r;
  bool done = false;
  for (int i = 0; i < t.len; ++i) {
    if (!done && t.id[i] == x) { done = true; continue; }
    r.id[r.len++] = t.id[i];
  }
  return r;
}

static std::string tuple_repr(const Graph& g, const Tuple& t) {
  std::string s = "(";
  for (int i = 0; i < t.len; ++i) {
    const Label& L = g.labels[t.id[i]];
    s += "(";
    for (int c = 0; c < L.ncomp; ++c) {
      s += std::to_string(L.comp[c]);
      if (L.ncomp == 1) s += ",";
      else if (c + 1 < L.ncomp) s += ", ";
    }
    s += ")";
    if (t.len == 1) s += ",";
    else if (i + 1 < t.len) s += ", ";
  }
  return s + ")";
}

std::string tuple_repr_public(const Graph& g, const Tuple& t) { return tuple_repr(g, t); }

int32_t Graph::insert_original(const Tuple& t) {  // graphbuild.py:150-167
  int32_t id = ids.get(t);
  if (id >= 0) return id;
  if (t.len == 1)
    throw std::invalid_argument("one-particle label outside the seeded range: " + tuple_repr(*this, t));
  Tuple L[128], R[128];
  int ns = proper_splits(t, L, R);
  for (int i = 0; i < ns; ++i) {
    int32_t a = ids.get(L[i]);
    if (a < 0) continue;
    int32_t b = ids.get(R[i]);
    if (b >= 0) return add(t, a, b);
  }
  // split off the max-degree label, ties towards the largest label
  uint16_t head = t.id[0];
  for (int i = 1; i < t.len; ++i) {
    const Label& c = labels[t.id[i]];
    const Label& h = labels[head];
    if (c.degree > h.degree || (c.degree == h.degree && t.id[i] > head)) head = t.id[i];
  }
  insert_original(remove_one(t, head));
  return insert_original(t);
}

int32_t Graph::insert_generalized(const Tuple& t, int nn) {  // graphbuild.py:169-187
  if (nn < 1) throw std::invalid_argument("n must be >= 1, got " + std::to_string(nn));
  int32_t id = ids.get(t);
  if (id >= 0) return id;
  if (t.len == 1)
    throw std::invalid_argument("one-particle label outside the seeded range: " + tuple_repr(*this, t));
  Tuple L[128], R[128];
  int ns = proper_splits(t, L, R);
  for (int i = 0; i < ns; ++i) {
    int32_t a = ids.get(L[i]);
    if (a < 0) continue;
    int32_t b = ids.get(R[i]);
    if (b >= 0) return add(t, a, b);
  }
  int size = std::min(nn, t.len - 1);
  // _max_block (graphbuild.py:189-202): max power_key, ties to the largest block
  Tuple best;
  int64_t best_key = -1;
  int pos[kMaxOrder];
  for (int i = 0; i < size; ++i) pos[i] = i;
  while (true) {
    Tuple blk;
    for (int i = 0; i < size; ++i) blk.id[blk.len++] = t.id[pos[i]];
    int64_t k = spec.power_key(blk, labels);
    if (k > best_key || (k == best_key && best < blk)) { best = blk; best_key = k; }
    int i = size - 1;
    while (i >= 0 && pos[i] == t.len - size + i) --i;
    if (i < 0) break;
    pos[i]++;
    for (int q = i + 1; q < size; ++q) pos[q] = pos[q - 1] + 1;
  }
  Tuple rest = t;
  for (int i = 0; i < best.len; ++i) rest = remove_one(rest, best.id[i]);
  insert_original(best);
  insert_generalized(rest, nn);
  return insert_generalized(t, nn);
}

std::vector<int32_t> Graph::target_ids() const {  // evaluator.py:214
  std::vector<int32_t> out;
  for (size_t i = 0; i < tuples.size(); ++i)
    if (!aux[i] && is_target(tuples[i])) out.push_back((int32_t)i);
  return out;
}

// Canonical invariant tuples of one order (the set of indexsets.py:368-388).
static void enumerate_order(const Graph& g, int order, std::vector<Tuple>& out) {
  const std::vector<Label>& lab = g.labels;
  const int L = (int)lab.size();
  const int p = g.spec.p;
  const int cap = g.spec.int_cap();
  const bool need_l = has_l(g.group);
  std::vector<int64_t> cost(L);
  for (int i = 0; i < L; ++i) {
    int64_t d = lab[i].degree;
    cost[i] = p == 1 ? d : (p == 2 ? d * d : 0);
  }
  Tuple cur;
  cur.len = (uint16_t)order;
  struct Rec {
    const Graph& g;
    const std::vector<Label>& lab;
    const std::vector<int64_t>& cost;
    std::vector<Tuple>& out;
    Tuple& cur;
    int L, p, cap, order;
    bool need_l;
    void run(int depth, int i0, int64_t rem, int msum, int lsum) {
      int slots = order - depth;
      if (slots == 0) {
        if (msum == 0 && (!need_l || (lsum & 1) == 0)) out.push_back(cur);
        return;
      }
      for (int i = i0; i < L; ++i) {
        int64_t c = cost[i];
        if (c > rem) continue;
        int nm = msum + lab[i].m;
        int64_t left = rem - c;
        if (p == 1) {
          if (std::abs(nm) > left) continue;
        } else if (std::abs(nm) > (int64_t)(slots - 1) * cap) {
          continue;
        }
        cur.id[depth] = (uint16_t)i;
        run(depth + 1, i, left, nm, lsum + lab[i].l);
      }
    }
  } rec{g, lab, cost, out, cur, L, p, cap, order, need_l};
  rec.run(0, 0, p == 0 ? 0 : g.spec.power_cap(), 0, 0);
}

void init_graph(Graph& g, int group, int p, double max_degree, int nu_max, int alg, int n) {
  if (group < 0 || group > 3) throw std::invalid_argument("unknown group");
  if (p != 0 && p != 1 && p != 2)
    throw std::invalid_argument("p must be 1, 2 or inf, got " + std::to_string(p));
  if (!(max_degree >= 0) || !std::isfinite(max_degree))
    throw std::invalid_argument("max_degree must be a finite non-negative number");
  if (alg != 0 && alg != 1) throw std::invalid_argument("alg must be one of ('orig', 'gen')");
  if (n < 1) throw std::invalid_argument("n must be >= 1, got " + std::to_string(n));
  g.group = group;
  g.spec.p = p;
  g.spec.max_degree = max_degree;
  g.nu_max = nu_max;
  g.alg = alg;
  g.n = n;
  g.labels = one_particle_indices(group, g.spec.int_cap());
  if (g.labels.size() >= 65535) throw std::invalid_argument("more than 65534 one-particle labels");
}

void build_graph(Graph& g, int group, int p, double max_degree, int nu_max, int alg, int n) {
  if (nu_max < 1) throw std::invalid_argument("nu_max must be >= 1, got " + std::to_string(nu_max));
  if (nu_max > kMaxOrder)
    throw std::invalid_argument("nu_max above the native limit of " + std::to_string(kMaxOrder));
  if (alg == 0) n = 1;
  init_graph(g, group, p, max_degree, nu_max, alg, n);
  g.seed();
  for (int order = 2; order <= nu_max; ++order) {
    std::vector<Tuple> targets;
    enumerate_order(g, order, targets);
    std::vector<int64_t> key(targets.size());
    for (size_t i = 0; i < targets.size(); ++i) key[i] = g.spec.power_key(targets[i], g.labels);
    std::vector<uint32_t> idx(targets.size());
    for (size_t i = 0; i < idx.size(); ++i) idx[i] = (uint32_t)i;
    std::sort(idx.begin(), idx.end(), [&](uint32_t a, uint32_t b) {
      if (key[a] != key[b]) return key[a] < key[b];
      return targets[a] < targets[b];
    });
    g.ids.reserve(g.tuples.size() + targets.size() + targets.size() / 8);
    for (uint32_t i : idx) {
      if (alg == 0) g.insert_original(targets[i]);
      else g.insert_generalized(targets[i], n);
    }
  }
}

void graph_from_parents(Graph& g, int group, int p, double max_degree, int nu_max, int alg,
                        int n, int64_t n_nodes, int64_t n_seeds, const int32_t* parents,
                        const uint8_t* auxf) {
  init_graph(g, group, p, max_degree, nu_max, alg, n);
  if (n_seeds != (int64_t)g.labels.size())
    throw std::invalid_argument("seed count does not match one_particle_indices for the spec");
  if (n_nodes < n_seeds) throw std::invalid_argument("fewer nodes than seeds");
  g.seed();
  g.ids.reserve((size_t)n_nodes);
  for (int64_t i = 0; i < n_nodes; ++i) {
    int32_t a = parents[2 * i], b = parents[2 * i + 1];
    if (i < n_seeds) {
      if (a != -1 || b != -1) throw std::invalid_argument("order-1 node " + std::to_string(i) + " has parents");
      continue;
    }
    if (a < 0 || b < 0 || a >= i || b >= i)
      throw std::invalid_argument("node " + std::to_string(i) + " has a non-topological parent");
    const Tuple &ta = g.tuples[a], &tb = g.tuples[b];
    if (ta.len + tb.len > kMaxOrder)
      throw std::invalid_argument("node order above the native limit");
    Tuple t;
    int x = 0, y = 0;
    while (x < ta.len || y < tb.len) {
      if (y >= tb.len || (x < ta.len && ta.id[x] <= tb.id[y])) t.id[t.len++] = ta.id[x++];
      else t.id[t.len++] = tb.id[y++];
    }
    if (g.ids.get(t) >= 0) throw std::invalid_argument("duplicate tuple at node " + std::to_string(i));
    int32_t id = g.add(t, a, b);
    if (auxf && auxf[i] != g.aux[id])
      throw std::invalid_argument("auxiliary flag inconsistent on node " + std::to_string(i));
  }
}

static std::string fmt_number(double x) {  // graphbuild.py:369-371
  if (x == std::floor(x) && std::fabs(x) < 9.2e18) return std::to_string((long long)x);
  char buf[64];
  for (int prec = 1; prec <= 17; ++prec) {
    snprintf(buf, sizeof buf, "%.*g", prec, x);
    if (strtod(buf, nullptr) == x) break;
  }
  return buf;
}

std::string Graph::serialize() const {  // graphbuild.py:374-384
  static const char* gname[] = {"T", "SO2", "O3", "O3F"};
  std::string s;
  s.reserve(tuples.size() * 48 + 128);
  s += "ACEDAG v1 group=";
  s += gname[group];
  s += " p=";
  s += spec.p == 0 ? "inf" : std::to_string(spec.p);
  s += " D=" + fmt_number(spec.max_degree);
  s += " numax=" + std::to_string(nu_max);
  s += alg == 0 ? " alg=orig" : " alg=gen";
  s += " n=" + std::to_string(n);
  s += "\n";
  char buf[32];
  for (size_t i = 0; i < tuples.size(); ++i) {
    int k = snprintf(buf, sizeof buf, "%zu %d ", i, (int)aux[i]);
    s.append(buf, k);
    const Tuple& t = tuples[i];
    for (int e = 0; e < t.len; ++e) {
      const Label& L = labels[t.id[e]];
      for (int c = 0; c < L.ncomp; ++c) {
        if (e || c) s += ',';
        k = snprintf(buf, sizeof buf, "%d", L.comp[c]);
        s.append(buf, k);
      }
    }
    if (pa[i] < 0) s += " -\n";
    else {
      k = snprintf(buf, sizeof buf, " %d %d\n", pa[i], pb[i]);
      s.append(buf, k);
    }
  }
  return s;
}

}  // namespace acedag
