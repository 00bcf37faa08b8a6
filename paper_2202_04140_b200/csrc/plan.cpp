// Plan compiler: DAG + coefficients -> K2 recursive program and K3 naive
// program (see plan.h for the re-parenting rationale).
#include "plan.h"

#include <algorithm>
#include <stdexcept>
#include <string>

namespace acedag {

std::string tuple_repr_public(const Graph& g, const Tuple& t);

std::string node_repr(const Graph& g, int64_t node) { return tuple_repr_public(g, g.tuples[node]); }

namespace {

struct PNode {
  Tuple t;
  int32_t parent = -1;  // plan index of the order-(o-1) parent (order >= 3)
  uint16_t sec = 0;     // secondary seed label (order >= 3); roots: sa/sb labels
  uint16_t sa = 0, sb = 0;
  int64_t coef = -1;    // row into the coefficient table
  int32_t graph_id = -1;
  std::vector<int32_t> kids;
};

Tuple drop_at(const Tuple& t, int pos) {
  Tuple r;
  for (int i = 0; i < t.len; ++i)
    if (i != pos) r.id[r.len++] = t.id[i];
  return r;
}

}  // namespace

void compile_plan(const Graph& g, const int64_t* node_ids, const double* c_re, const double* c_im,
                  int64_t n_coef, int n_out, int warps, PlanHost& P, uint32_t hot_rows) {
  const int64_t N = (int64_t)g.tuples.size();
  const int64_t L = g.n_seeds();
  if (n_out < 1) throw std::invalid_argument("n_out must be >= 1");
  P = PlanHost();
  P.n_out = n_out;
  P.complex_coef = c_im != nullptr;
  P.warps = warps;

  // ---- coefficient rows, validated like evaluate_model (evaluator.py:132-139)
  std::vector<int64_t> row_of(N, -1);
  std::vector<double> rows_re, rows_im;
  int64_t nrows = 0;
  for (int64_t i = 0; i < n_coef; ++i) {
    int64_t id = node_ids[i];
    if (id < 0 || id >= N) throw std::invalid_argument("coefficient node id out of range: " + std::to_string(id));
    if (g.aux[id] || !g.is_target(g.tuples[id]))
      throw std::domain_error("coefficient on non-target node: " + node_repr(g, id));
    int64_t r = row_of[id];
    if (r < 0) {
      r = row_of[id] = nrows++;
      rows_re.resize(nrows * n_out, 0.0);
      rows_im.resize(nrows * n_out, 0.0);
    }
    for (int o = 0; o < n_out; ++o) {
      rows_re[r * n_out + o] += c_re[i * n_out + o];
      if (c_im) rows_im[r * n_out + o] += c_im[i * n_out + o];
    }
  }

  // ---- plan forest: top-down parent choice per order
  std::vector<PNode> nodes;
  TupleMap pid;
  pid.reserve((size_t)nrows * 2 + 16);
  int max_order = 1;
  std::vector<std::vector<int32_t>> by_order(kMaxOrder + 1);
  std::vector<int32_t> singles;  // order-1 coefficient nodes
  for (int64_t id = 0; id < N; ++id) {
    if (row_of[id] < 0) continue;
    PNode n;
    n.t = g.tuples[id];
    n.coef = row_of[id];
    n.graph_id = (int32_t)id;
    int32_t k = (int32_t)nodes.size();
    nodes.push_back(n);
    pid.put(n.t, k);
    if (n.t.len == 1) singles.push_back(k);
    else by_order[n.t.len].push_back(k);
    max_order = std::max<int>(max_order, n.t.len);
  }
  for (int o = max_order; o >= 3; --o) {
    std::vector<int32_t>& lvl = by_order[o];
    // demand of each candidate parent among this level (for the greedy cover)
    TupleMap demand;
    demand.reserve(lvl.size() * 4 + 16);
    for (int32_t k : lvl) {
      const Tuple t = nodes[k].t;
      for (int j = 0; j < t.len; ++j) {
        if (j && t.id[j] == t.id[j - 1]) continue;
        Tuple c = drop_at(t, j);
        int32_t d = demand.get(c);
        demand.put(c, d < 0 ? 1 : d + 1);
      }
    }
    for (int32_t k : lvl) {
      const Tuple t = nodes[k].t;
      int pick = -1;
      // (1) an already planned (o-1)-subset
      for (int j = 0; j < t.len && pick < 0; ++j) {
        if (j && t.id[j] == t.id[j - 1]) continue;
        if (pid.get(drop_at(t, j)) >= 0) pick = j;
      }
      // (2) the reference's own (seed, node) split
      if (pick < 0 && nodes[k].graph_id >= 0) {
        int32_t a = g.pa[nodes[k].graph_id], b = g.pb[nodes[k].graph_id];
        int32_t seedp = g.tuples[a].len == 1 ? a : (g.tuples[b].len == 1 ? b : -1);
        if (seedp >= 0)
          for (int j = 0; j < t.len; ++j)
            if (t.id[j] == (uint16_t)seedp) { pick = j; break; }
      }
      // (3) the subset wanted by most nodes of this level
      if (pick < 0) {
        int32_t best = -1;
        for (int j = 0; j < t.len; ++j) {
          if (j && t.id[j] == t.id[j - 1]) continue;
          int32_t d = demand.get(drop_at(t, j));
          if (d > best) { best = d; pick = j; }
        }
      }
      Tuple par = drop_at(t, pick);
      int32_t pk = pid.get(par);
      if (pk < 0) {
        PNode n;
        n.t = par;
        int32_t gid = g.ids.get(par);
        n.graph_id = gid;
        pk = (int32_t)nodes.size();
        nodes.push_back(n);
        pid.put(par, pk);
        by_order[o - 1].push_back(pk);
        if (gid < 0) P.extra_nodes++;
      }
      nodes[k].parent = pk;
      nodes[k].sec = t.id[pick];
      nodes[pk].kids.push_back(k);
    }
  }
  for (int32_t k : by_order[2]) {
    nodes[k].sa = nodes[k].t.id[0];
    nodes[k].sb = nodes[k].t.id[1];
  }

  // ---- seed slots, hottest first (K2 keeps the head of the table in smem)
  std::vector<int64_t> use(L, 0);
  for (int32_t k : singles) use[nodes[k].t.id[0]]++;
  for (int32_t k : by_order[2]) { use[nodes[k].sa]++; use[nodes[k].sb]++; }
  for (int o = 3; o <= max_order; ++o)
    for (int32_t k : by_order[o]) use[nodes[k].sec]++;
  std::vector<int32_t> lab;
  for (int64_t i = 0; i < L; ++i)
    if (use[i]) lab.push_back((int32_t)i);
  std::stable_sort(lab.begin(), lab.end(), [&](int32_t a, int32_t b) { return use[a] > use[b]; });
  if (lab.size() >= kSingle) throw std::invalid_argument("more than 65534 seeds referenced");
  std::vector<uint16_t> slot(L, kSingle);
  for (size_t s = 0; s < lab.size(); ++s) {
    slot[lab[s]] = (uint16_t)s;
    P.slot_label.push_back((uint16_t)lab[s]);
  }

  // ---- DFS program; roots sorted by tuple, children by tuple
  auto by_tuple = [&](int32_t a, int32_t b) { return nodes[a].t < nodes[b].t; };
  std::vector<int32_t> roots = singles;
  roots.insert(roots.end(), by_order[2].begin(), by_order[2].end());
  std::sort(roots.begin(), roots.end(), by_tuple);
  // children by seed slot: the TMEM-resident seeds (slot < hot_rows) lead,
  // then the shared-memory rows, then the global-cache tail (distinct
  // children of one node have distinct seeds, so the order is total)
  auto hot = [&](int32_t k) { return slot[nodes[k].sec] < hot_rows; };
  for (auto& n : nodes)
    std::sort(n.kids.begin(), n.kids.end(),
              [&](int32_t a, int32_t b) { return slot[nodes[a].sec] < slot[nodes[b].sec]; });
  P.max_order = std::max(2, max_order);

  // Records (16 B): {c, byte offset of the seed row, #children, subtree size}.
  // A root is two records (its two seeds; an order-1 term pairs its seed with
  // the constant ONE row, slot U).  Every other record multiplies its seed
  // into the parent value held in registers.
  const uint32_t U = (uint32_t)lab.size();
  auto off_of = [&](uint32_t s) { return s * kRowBytes; };
  std::vector<int64_t> root_cost(roots.size(), 0);
  auto emit = [&](int32_t k, uint32_t off, uint32_t nch) {
    Op op;
    op.c = (k >= 0 && nodes[k].coef >= 0) ? rows_re[nodes[k].coef * n_out] : 0.0;
    op.off = off;
    if (nch > 0xFFFFu) throw std::invalid_argument("node with more than 65535 children");
    op.nch = (uint16_t)nch;
    op.skip = 0;
    P.ops.push_back(op);
    for (int o = 0; o < n_out; ++o) {
      const bool has = k >= 0 && nodes[k].coef >= 0;
      P.cre.push_back(has ? rows_re[nodes[k].coef * n_out + o] : 0.0);
      if (c_im) P.cim.push_back(has ? rows_im[nodes[k].coef * n_out + o] : 0.0);
    }
  };
  // preorder; `skip` = number of leading children with a TMEM-resident seed
  // (roots: second record's skip = hot flags of the two root seeds)
  auto nhot = [&](int32_t k) {
    uint16_t h = 0;
    for (int32_t q : nodes[k].kids) h += hot(q) ? 1 : 0;
    return h;
  };
  std::vector<int32_t> stack;
  std::vector<int64_t> op_root;
  for (size_t r = 0; r < roots.size(); ++r) {
    int32_t k = roots[r];
    op_root.push_back((int64_t)P.ops.size());
    if (nodes[k].t.len == 1) {
      const uint32_t s0 = slot[nodes[k].t.id[0]];
      emit(k, off_of(s0), 0);
      emit(-1, off_of(U), 0);
      P.ops.back().skip = (uint16_t)((s0 < hot_rows ? 1 : 0) | (U < hot_rows ? 2 : 0));
      root_cost[r] = 6;
      continue;
    }
    const uint32_t sa = slot[nodes[k].sa], sb = slot[nodes[k].sb];
    emit(k, off_of(sa), (uint32_t)nodes[k].kids.size());
    P.ops.back().skip = nhot(k);
    emit(-1, off_of(sb), 0);
    P.ops.back().skip = (uint16_t)((sa < hot_rows ? 1 : 0) | (sb < hot_rows ? 2 : 0));
    P.recursive_products++;
    int64_t cost = 8;
    stack.assign(nodes[k].kids.rbegin(), nodes[k].kids.rend());
    while (!stack.empty()) {
      const int32_t q = stack.back();
      stack.pop_back();
      emit(q, off_of(slot[nodes[q].sec]), (uint32_t)nodes[q].kids.size());
      P.ops.back().skip = nhot(q);
      P.recursive_products++;
      cost += nodes[q].kids.empty() ? 4 : 6;
      for (auto it = nodes[q].kids.rbegin(); it != nodes[q].kids.rend(); ++it) stack.push_back(*it);
    }
    root_cost[r] = cost;
  }
  // ---- work chunks at root boundaries, balanced by cost (grabbed dynamically
  // by the warps of a CTA; partial sums are combined in chunk order)
  int64_t total = 0;
  for (int64_t c : root_cost) total += c;
  const int chunks = warps;
  P.chunk.assign(chunks + 1, (int32_t)P.ops.size());
  P.chunk[0] = 0;
  int64_t acc = 0;
  int w = 1;
  for (size_t r = 0; r < roots.size() && w < chunks; ++r) {
    acc += root_cost[r];
    while (w < chunks && acc * chunks >= total * w) {
      P.chunk[w++] = (int32_t)(r + 1 < roots.size() ? op_root[r + 1] : P.ops.size());
    }
  }
  for (; w < chunks; ++w) P.chunk[w] = (int32_t)P.ops.size();

  // ---- naive program: coefficient nodes grouped by order, graph-id order
  std::vector<std::vector<int64_t>> nby(kMaxOrder + 1);
  int nmax = 1;
  for (int64_t id = 0; id < N; ++id)
    if (row_of[id] >= 0) {
      nby[g.tuples[id].len].push_back(id);
      nmax = std::max<int>(nmax, g.tuples[id].len);
    }
  P.naive_max_order = nmax;
  P.naive_seg.assign(kMaxOrder + 2, 0);
  int64_t rec = 0;
  for (int o = 1; o <= kMaxOrder; ++o) {
    P.naive_seg[o] = (int32_t)rec;
    for (int64_t id : nby[o]) {
      const Tuple& t = g.tuples[id];
      for (int i = 0; i < kMaxOrder; ++i) P.naive_slots.push_back(i < t.len ? slot[t.id[i]] : 0);
      for (int q = 0; q < n_out; ++q) {
        P.naive_cre.push_back(rows_re[row_of[id] * n_out + q]);
        if (c_im) P.naive_cim.push_back(rows_im[row_of[id] * n_out + q]);
      }
      P.naive_products += t.len - 1;
      rec++;
    }
  }
  P.naive_seg[kMaxOrder + 1] = (int32_t)rec;
  // order-1 seeds referenced by naive records that K2 does not need are
  // impossible: every coefficient node's seeds appear in some K2 record.
}

}  // namespace acedag
