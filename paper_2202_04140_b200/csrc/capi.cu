// C ABI of the B200 evaluator (include/acedag_b200.h): plan ownership,
// argument validation, kernel dispatch.  No host synchronisation on the hot
// calls (acedag_eval, acedag_eval_from_positions, acedag_pool*).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/acedag_b200.h"
#include "graph.h"
#include "kernels.cuh"
#include "horner.h"
#include "plan.h"
#include "pool.cuh"

#include <array>
#include <atomic>
namespace {
// kernels this library launched (bench.py's gpu_launches; acedag_launch_count)
std::atomic<int64_t> g_launches{0};
inline void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace

using namespace acedag;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(ACEDAG_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(call)                                   \
  do {                                             \
    cudaError_t e_ = (call);                       \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DevGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  ~DevBuf() { if (p) cudaFree(p); }
  cudaError_t upload(const std::vector<T>& v) {
    if (p) { cudaFree(p); p = nullptr; }
    n = v.size();
    if (!n) return cudaSuccess;
    cudaError_t e = cudaMalloc(&p, n * sizeof(T));
    if (e != cudaSuccess) return e;
    return cudaMemcpy(p, v.data(), n * sizeof(T), cudaMemcpyHostToDevice);
  }
  cudaError_t alloc(size_t count) {
    if (count <= n && p) return cudaSuccess;
    if (p) { cudaFree(p); p = nullptr; }
    n = count;
    return cudaMalloc(&p, n * sizeof(T));
  }
};

std::vector<int4> label_table(int group, int cap) {
  std::vector<Label> labs = one_particle_indices(group, cap);
  std::vector<int4> t(labs.size());
  for (size_t i = 0; i < labs.size(); ++i) {
    const Label& L = labs[i];
    if (group == kT) t[i] = make_int4(L.comp[0], 0, 0, 0);
    else if (group == kSO2) t[i] = make_int4(L.comp[0], L.comp[1], 0, 0);
    else t[i] = make_int4(L.comp[0], L.comp[1], L.comp[2], L.ncomp == 4 ? L.comp[3] : 0);
  }
  return t;
}

// per-device constant setup + label tables, created once
std::mutex g_mu;
std::map<int, bool> g_norms_ready;
std::map<std::tuple<int, int, int>, int4*> g_label_cache;

int ensure_norms(int dev) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_norms_ready[dev]) return 0;
  CK(cudaMemcpyToSymbol(dev::c_ylm_norm, kYlmNorm, sizeof(kYlmNorm)));
  double recip[ACEDAG_YLM_LMAX + 2];
  recip[0] = 0.0;
  for (int k = 1; k < ACEDAG_YLM_LMAX + 2; ++k) recip[k] = 1.0 / k;
  CK(cudaMemcpyToSymbol(dev::c_recip, recip, sizeof(recip)));
  // three-term recurrence of the NORMALISED functions Q_l^m = N_lm P_l^m:
  //   Q_l^m = A_lm cos(theta) Q_{l-1}^m - B_lm Q_{l-2}^m
  // A_lm = (2l-1)/(l-m) N_lm/N_{l-1,m}, B_lm = (l+m-1)/(l-m) N_lm/N_{l-2,m}
  {
    constexpr int n = (ACEDAG_YLM_LMAX + 1) * (ACEDAG_YLM_LMAX + 2) / 2;
    std::vector<double> ra(n, 0.0), rb(n, 0.0);
    auto idx = [](int l, int m) { return l * (l + 1) / 2 + m; };
    for (int l = 1; l <= ACEDAG_YLM_LMAX; ++l)
      for (int m = 0; m < l; ++m) {
        ra[idx(l, m)] = (2.0 * l - 1.0) / (l - m) * (kYlmNorm[idx(l, m)] / kYlmNorm[idx(l - 1, m)]);
        if (l - 2 >= m) rb[idx(l, m)] = (l + m - 1.0) / (l - m) * (kYlmNorm[idx(l, m)] / kYlmNorm[idx(l - 2, m)]);
      }
    CK(cudaMemcpyToSymbol(dev::c_ylm_a, ra.data(), n * sizeof(double)));
    CK(cudaMemcpyToSymbol(dev::c_ylm_b, rb.data(), n * sizeof(double)));
  }
  g_norms_ready[dev] = true;
  return 0;
}

int device_labels(int dev, int group, int cap, const int4** out) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_tuple(dev, group, cap);
  auto it = g_label_cache.find(key);
  if (it != g_label_cache.end()) { *out = it->second; return 0; }
  std::vector<int4> t = label_table(group, cap);
  int4* p = nullptr;
  CK(cudaMalloc(&p, std::max<size_t>(1, t.size()) * sizeof(int4)));
  if (!t.empty()) CK(cudaMemcpy(p, t.data(), t.size() * sizeof(int4), cudaMemcpyHostToDevice));
  g_label_cache[key] = p;
  *out = p;
  return 0;
}

// work chunks per program (ACEDAG_CHUNKS overrides): eight per warp of the
// 24-warp k2_horner (cfg2 K2: 128 chunks 1.778 ms, 192 1.753, 256 1.754, 384 1.773)
int plan_chunks() {
  static int c = [] {
    const char* e = getenv("ACEDAG_CHUNKS");
    int v = e ? atoi(e) : 192;
    return v < 1 ? 1 : (v > 8192 ? 8192 : v);
  }();
  return c;
}

// (n, l, m >= 0) triples of the O3 labels with cap, keeping those for which
// keep(label) or keep(label of -m) holds; int4 (n, l, m, label index)
template <class Keep>
std::vector<int4> triples(int cap, Keep keep) {
  std::vector<int4> tri;
  int lab = 0;
  for (int n = 0; n <= cap; ++n)
    for (int l = 0; l <= cap - n; ++l)
      for (int m = -l; m <= l; ++m, ++lab)
        if (m >= 0 && (keep(lab) || keep(lab - 2 * m))) tri.push_back(make_int4(n, l, m, lab));
  return tri;
}

int full_triples(int dev, int cap, const int4** out, int* n) {
  std::lock_guard<std::mutex> lk(g_mu);
  static std::map<std::pair<int, int>, std::pair<int4*, int>> cache;
  auto key = std::make_pair(dev, cap);
  auto it = cache.find(key);
  if (it == cache.end()) {
    std::vector<int4> tri = triples(cap, [](int) { return true; });
    int4* d = nullptr;
    CK(cudaMalloc(&d, std::max<size_t>(1, tri.size()) * sizeof(int4)));
    CK(cudaMemcpy(d, tri.data(), tri.size() * sizeof(int4), cudaMemcpyHostToDevice));
    it = cache.emplace(key, std::make_pair(d, (int)tri.size())).first;
  }
  *out = it->second.first;
  *n = it->second.second;
  return 0;
}

int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

}  // namespace

namespace {
int k2_mode();  // fp64 single-output kernel selection (dispatch, below)
}  // namespace

namespace {
// The same program with a smaller TMEM-resident set (k2_quad keeps the 32
// hottest slots): per node, the count of leading children whose slot is
// below `hot`, and a root's hot flags.  Needs slot-ordered children (plan).
std::vector<Op> reencode_hot(const PlanHost& H, uint32_t hot) {
  std::vector<Op> o = H.ops;
  std::function<size_t(size_t, uint32_t, uint32_t&)> walk = [&](size_t pos, uint32_t n, uint32_t& nh) -> size_t {
    nh = 0;
    for (uint32_t k = 0; k < n; ++k) {
      const size_t me = pos;
      nh += H.ops[me].off / kRowBytes < hot;
      uint32_t h2;
      pos = walk(me + 1, H.ops[me].nch, h2);
      o[me].skip = (uint16_t)h2;
    }
    return pos;
  };
  for (size_t ci = 0; ci + 1 < H.chunk.size(); ++ci) {
    size_t i = (size_t)H.chunk[ci];
    while (i < (size_t)H.chunk[ci + 1]) {
      const uint32_t sa = H.ops[i].off / kRowBytes, sb = H.ops[i + 1].off / kRowBytes;
      o[i + 1].skip = (uint16_t)((sa < hot ? 1 : 0) | (sb < hot ? 2 : 0));
      uint32_t nh;
      const size_t end = walk(i + 2, H.ops[i].nch, nh);
      o[i].skip = (uint16_t)nh;
      i = end;
    }
  }
  return o;
}
}  // namespace

struct acedag_graph {
  Graph g;
};

struct acedag_plan {
  std::shared_ptr<const Graph> g;
  int device = 0;
  int sms = 148;
  size_t smem_optin = 232448;
  DevBuf<int32_t> pa, pb;
  bool has_coef = false;
  PlanHost host;
  int U = 0;
  DevBuf<uint16_t> slot_label, slot_identity;
  DevBuf<int32_t> used_labels;
  // host-path compact layout: used labels ascending (coalesced gather) and
  // each slot's column in it
  DevBuf<int32_t> sorted_labels;
  DevBuf<uint16_t> slot_sorted;
  DevBuf<uint16_t> sorted_slot;  // inverse: sorted position -> slot
  DevBuf<int32_t> col_of;  // label -> seed slot or -1 (pool of used labels only)
  DevBuf<int4> tri;        // (n, l, m >= 0) triples the used labels need
  bool tri_pruned = false;  // every triple has l + m <= cap
  DevBuf<Op> ops;
  DevBuf<Op> opsQ;         // k2_quad: hot counts for its 32 TMEM slots
  // k2_horner encodings (encode_horner) for fp64 [0] and the fp32 mode [1]
  struct HornerProg {
    DevBuf<OpH> ops;
    DevBuf<int32_t> croots, chunk;
    bool ok = false;
    int us = 0;  // shared-memory rows
  } hp[2];
  DevBuf<int32_t> chunk;
  DevBuf<double> cre, cim;
  DevBuf<int32_t> nseg;
  DevBuf<uint16_t> nslots;
  DevBuf<double> ncre, ncim;
  // per-stream scratch (seed cold tails, chunk partials, pooled A): calls on
  // distinct streams may run concurrently
  struct Workspace {
    DevBuf<double> tail;  // split last-round partials
    DevBuf<double2> tiles;  // tile-major seed table (k_tile_seeds)
    DevBuf<double2> gcache;
    DevBuf<double2> ws_A;
    DevBuf<double> part;  // K2 partial sums
  };
  std::mutex ws_mu;
  std::map<void*, std::unique_ptr<Workspace>> wss;
  // acedag_eval_host pipeline: gather/copy stream, evaluation stream, double
  // buffered device chunks of seeds and results
  struct HostPipe {
    cudaStream_t sg = nullptr, sk = nullptr;
    cudaEvent_t start = nullptr, gdone[2] = {}, kdone[2] = {};
    DevBuf<unsigned char> buf[2], out[2];
    ~HostPipe() {
      if (sg) cudaStreamDestroy(sg);
      if (sk) cudaStreamDestroy(sk);
      for (cudaEvent_t e : {start, gdone[0], gdone[1], kdone[0], kdone[1]})
        if (e) cudaEventDestroy(e);
    }
    cudaError_t init() {
      if (sg) return cudaSuccess;
      cudaError_t e = cudaStreamCreateWithFlags(&sg, cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&sk, cudaStreamNonBlocking);
      for (cudaEvent_t* ev : {&start, &gdone[0], &gdone[1], &kdone[0], &kdone[1]})
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
      return e;
    }
  };
  std::mutex host_mu;
  HostPipe pipe;
  // acedag_plan_timing: CUDA events around each eval's phases
  // {start, after seed prep, after the main K2 kernel, end}
  struct Timing {
    bool on = false;
    std::mutex mu;
    std::vector<std::array<cudaEvent_t, 4>> ev;
    void clear() {
      for (auto& a : ev)
        for (cudaEvent_t e : a) cudaEventDestroy(e);
      ev.clear();
    }
    ~Timing() { clear(); }
  } timing;
  Workspace* ws(cudaStream_t s) {
    std::lock_guard<std::mutex> lk(ws_mu);
    auto& w = wss[(void*)s];
    if (!w) w.reset(new Workspace);
    return w.get();
  }
};

// hot-slot count the plan compiler orders children by (compile_plan); the
// programs of round 1 were compiled with 64, kept so results are unchanged
constexpr uint32_t kPlanHotRows = 64;

// ====================================================================== API
extern "C" {

int acedag_abi_version(void) { return ACEDAG_ABI_VERSION; }
const char* acedag_last_error(void) { return g_err.c_str(); }

int acedag_graph_build(int group, int p, double max_degree, int nu_max, int alg, int n,
                       acedag_graph** out) {
  if (!out) return fail(ACEDAG_EINVAL, "out is NULL");
  try {
    std::unique_ptr<acedag_graph> h(new acedag_graph);
    build_graph(h->g, group, p, max_degree, nu_max, alg, n);
    *out = h.release();
    return ACEDAG_OK;
  } catch (const std::bad_alloc&) {
    return fail(ACEDAG_ENOMEM, "out of host memory building the graph");
  } catch (const std::exception& e) {
    return fail(ACEDAG_EINVAL, e.what());
  }
}

int acedag_graph_from_parents(int group, int p, double max_degree, int nu_max, int alg, int n,
                              int64_t n_nodes, int64_t n_seeds, const int32_t* parents,
                              const uint8_t* aux, acedag_graph** out) {
  if (!out || !parents) return fail(ACEDAG_EINVAL, "NULL argument");
  try {
    std::unique_ptr<acedag_graph> h(new acedag_graph);
    graph_from_parents(h->g, group, p, max_degree, nu_max, alg, n, n_nodes, n_seeds, parents, aux);
    *out = h.release();
    return ACEDAG_OK;
  } catch (const std::bad_alloc&) {
    return fail(ACEDAG_ENOMEM, "out of host memory");
  } catch (const std::exception& e) {
    return fail(ACEDAG_EINVAL, e.what());
  }
}

void acedag_graph_destroy(acedag_graph* g) { delete g; }

int acedag_graph_info(const acedag_graph* h, int64_t* n_nodes, int64_t* n_seeds, int64_t* n_targets,
                      int64_t* n_aux, int32_t* max_order) {
  if (!h) return fail(ACEDAG_EINVAL, "graph is NULL");
  const Graph& g = h->g;
  int64_t aux = 0;
  int mo = 1;
  for (size_t i = 0; i < g.tuples.size(); ++i) {
    aux += g.aux[i];
    mo = std::max<int>(mo, g.tuples[i].len);
  }
  if (n_nodes) *n_nodes = (int64_t)g.tuples.size();
  if (n_seeds) *n_seeds = g.n_seeds();
  if (n_targets) *n_targets = (int64_t)g.target_ids().size();
  if (n_aux) *n_aux = aux;
  if (max_order) *max_order = mo;
  return ACEDAG_OK;
}

int acedag_graph_arrays(const acedag_graph* h, int32_t* parents, uint8_t* aux, int32_t* order,
                        int32_t* target_ids) {
  if (!h) return fail(ACEDAG_EINVAL, "graph is NULL");
  const Graph& g = h->g;
  for (size_t i = 0; i < g.tuples.size(); ++i) {
    if (parents) { parents[2 * i] = g.pa[i]; parents[2 * i + 1] = g.pb[i]; }
    if (aux) aux[i] = g.aux[i];
    if (order) order[i] = g.tuples[i].len;
  }
  if (target_ids) {
    std::vector<int32_t> t = g.target_ids();
    std::memcpy(target_ids, t.data(), t.size() * sizeof(int32_t));
  }
  return ACEDAG_OK;
}

int acedag_graph_node_seeds(const acedag_graph* h, int64_t node, int32_t* seeds_out, int32_t capacity) {
  if (!h || !seeds_out) return fail(ACEDAG_EINVAL, "NULL argument");
  const Graph& g = h->g;
  if (node < 0 || node >= (int64_t)g.tuples.size()) return fail(ACEDAG_EINVAL, "node id out of range");
  const Tuple& t = g.tuples[node];
  if (capacity < t.len) return fail(ACEDAG_EINVAL, "capacity below the node order");
  for (int i = 0; i < t.len; ++i) seeds_out[i] = t.id[i];
  return t.len;
}

int64_t acedag_graph_find(const acedag_graph* h, const int32_t* seeds, int32_t len) {
  if (!h || !seeds || len < 1 || len > kMaxOrder) return -1;
  Tuple t;
  for (int i = 0; i < len; ++i) {
    if (seeds[i] < 0 || seeds[i] >= h->g.n_seeds()) return -1;
    if (i && seeds[i] < seeds[i - 1]) return -1;
    t.id[t.len++] = (uint16_t)seeds[i];
  }
  return h->g.ids.get(t);
}

int acedag_graph_serialize(const acedag_graph* h, char* buf, int64_t* len) {
  if (!h || !len) return fail(ACEDAG_EINVAL, "NULL argument");
  try {
    std::string s = h->g.serialize();
    if (buf) {
      if (*len < (int64_t)s.size()) return fail(ACEDAG_EINVAL, "buffer too small");
      std::memcpy(buf, s.data(), s.size());
    }
    *len = (int64_t)s.size();
    return ACEDAG_OK;
  } catch (const std::bad_alloc&) {
    return fail(ACEDAG_ENOMEM, "out of host memory serializing");
  }
}

int acedag_graph_deserialize(const char* data, int64_t len, acedag_graph** out, int32_t* err_kind,
                             int64_t* err_offset, int64_t* err_line_start, int64_t* err_line_len) {
  if (err_kind) *err_kind = 0;
  if (!out || (len > 0 && !data) || len < 0) return fail(ACEDAG_EINVAL, "bad arguments");
  try {
    std::unique_ptr<acedag_graph> h(new acedag_graph);
    GraphParseError pe;
    if (!deserialize_graph(data ? data : "", (size_t)len, h->g, pe)) {
      if (err_kind) *err_kind = pe.kind;
      if (err_offset) *err_offset = pe.offset;
      if (err_line_start) *err_line_start = pe.line_start;
      if (err_line_len) *err_line_len = pe.line_len;
      return fail(ACEDAG_EFORMAT, pe.message);
    }
    *out = h.release();
    return ACEDAG_OK;
  } catch (const std::bad_alloc&) {
    return fail(ACEDAG_ENOMEM, "out of host memory reading the graph");
  }
}

int acedag_graph_spec(const acedag_graph* h, int32_t* group, int32_t* p, double* max_degree, int32_t* nu_max,
                      int32_t* alg, int32_t* n) {
  if (!h) return fail(ACEDAG_EINVAL, "graph is NULL");
  const Graph& g = h->g;
  if (group) *group = g.group;
  if (p) *p = g.spec.p;
  if (max_degree) *max_degree = g.spec.max_degree;
  if (nu_max) *nu_max = g.nu_max;
  if (alg) *alg = g.alg;
  if (n) *n = g.n;
  return ACEDAG_OK;
}

// ------------------------------------------------------------------ plans
int acedag_plan_create(const acedag_graph* h, int device, acedag_plan** out) {
  if (!h || !out) return fail(ACEDAG_EINVAL, "NULL argument");
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(ACEDAG_EINVAL, "device ordinal out of range");
  DevGuard dg(device);
  std::unique_ptr<acedag_plan> P(new (std::nothrow) acedag_plan);
  if (!P) return fail(ACEDAG_ENOMEM, "out of host memory");
  P->g = std::make_shared<const Graph>(h->g);
  P->device = device;
  int optin = 0;
  CK(cudaDeviceGetAttribute(&P->sms, cudaDevAttrMultiProcessorCount, device));
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  P->smem_optin = (size_t)optin;
  CK(P->pa.upload(P->g->pa));
  CK(P->pb.upload(P->g->pb));
  int rc = ensure_norms(device);
  if (rc) return rc;
  *out = P.release();
  return ACEDAG_OK;
}

void acedag_plan_destroy(acedag_plan* plan) {
  if (!plan) return;
  DevGuard dg(plan->device);
  delete plan;
}

int acedag_plan_set_coefficients(acedag_plan* P, const int64_t* node_ids, const double* c_re,
                                 const double* c_im, int64_t n_coef, int32_t n_out) {
  if (!P) return fail(ACEDAG_EINVAL, "plan is NULL");
  if (n_coef < 0 || n_out < 1 || (n_coef && (!node_ids || !c_re)))
    return fail(ACEDAG_EINVAL, "bad coefficient arguments");
  DevGuard dg(P->device);
  // compile into a local program: a rejected set (non-target id, order > 6)
  // leaves the plan evaluating its previous coefficients
  PlanHost H;
  try {
    compile_plan(*P->g, node_ids, c_re, c_im, n_coef, n_out, plan_chunks(), H, kPlanHotRows);
  } catch (const std::domain_error& e) {
    return fail(ACEDAG_ENOTTARGET, e.what());
  } catch (const std::bad_alloc&) {
    return fail(ACEDAG_ENOMEM, "out of host memory compiling the plan");
  } catch (const std::exception& e) {
    return fail(ACEDAG_EINVAL, e.what());
  }
  if (H.max_order > 6) return fail(ACEDAG_EUNSUPPORTED, "device programs support order <= 6");
  // from here on the device arrays change: the plan is unusable until every
  // upload has succeeded (a failed upload leaves it without coefficients)
  P->has_coef = false;
  P->host = std::move(H);
  const PlanHost& Hp = P->host;
  P->U = (int)Hp.slot_label.size();
  std::vector<uint16_t> ident(P->U);
  std::vector<int32_t> used(P->U);
  for (int i = 0; i < P->U; ++i) { ident[i] = (uint16_t)i; used[i] = Hp.slot_label[i]; }
  CK(P->slot_label.upload(Hp.slot_label));
  CK(P->slot_identity.upload(ident));
  CK(P->used_labels.upload(used));
  {
    std::vector<int32_t> sorted(used);
    std::sort(sorted.begin(), sorted.end());
    std::vector<uint16_t> pos(P->U);
    for (int i = 0; i < P->U; ++i)
      pos[i] = (uint16_t)(std::lower_bound(sorted.begin(), sorted.end(), used[i]) - sorted.begin());
    CK(P->sorted_labels.upload(sorted));
    CK(P->slot_sorted.upload(pos));
    std::vector<uint16_t> inv(P->U);
    for (int i = 0; i < P->U; ++i) inv[pos[i]] = (uint16_t)i;
    CK(P->sorted_slot.upload(inv));
  }
  {
    std::vector<int32_t> col((size_t)P->g->n_seeds(), -1);
    for (int i = 0; i < P->U; ++i) col[Hp.slot_label[i]] = i;
    CK(P->col_of.upload(col));
    if (P->g->group == kO3) {
      const int cap = P->g->spec.int_cap();
      std::vector<int4> tri = triples(cap, [&](int lab) { return col[lab] >= 0; });
      P->tri_pruned = true;
      for (const int4& q : tri) P->tri_pruned = P->tri_pruned && q.y + q.z <= cap;
      CK(P->tri.upload(tri));
    }
  }
  CK(P->ops.upload(Hp.ops));
  CK(P->chunk.upload(Hp.chunk));
  CK(P->opsQ.upload(reencode_hot(Hp, dev::kTmemRowsQ)));
  for (int f = 0; f < 2; ++f) {
    acedag_plan::HornerProg& hp = P->hp[f];
    hp.ok = false;
    // fp32: every order; fp64: order <= 4 unless ACEDAG_K2=horner (order 5-6 spill)
    if (f == 1 || Hp.max_order <= 4 || k2_mode() == 2) {
      const int hot = std::min(P->U, horner_hot_rows(f == 1));
      hp.us = std::min(P->U - hot, horner_us_max(P->smem_optin, f == 1, Hp.max_order));
      std::vector<OpH> oh;
      std::vector<int32_t> ch, cr;
      if (encode_horner(Hp, f == 1, (uint32_t)hot, (uint32_t)hp.us, oh, ch, cr)) {
        CK(hp.ops.upload(oh));
        CK(hp.chunk.upload(ch));
        CK(hp.croots.upload(cr));
        hp.ok = true;
      }
    }
  }
  {
    std::vector<double> padded(Hp.cre);
    // k2_mma prefetches two 4-record groups past the end of a chunk
    padded.resize(Hp.cre.size() + 16 * (size_t)Hp.n_out + 64, 0.0);
    CK(P->cre.upload(padded));
  }
  CK(P->cim.upload(Hp.cim));
  CK(P->nseg.upload(Hp.naive_seg));
  CK(P->nslots.upload(Hp.naive_slots));
  CK(P->ncre.upload(Hp.naive_cre));
  CK(P->ncim.upload(Hp.naive_cim));
  P->has_coef = true;
  return ACEDAG_OK;
}

int acedag_plan_program(const acedag_graph* h, const int64_t* node_ids, const double* c_re,
                        const double* c_im, int64_t n_coef, int32_t n_out, int32_t warps,
                        uint16_t* slot_label, int64_t* n_slots, void* ops, int64_t* n_ops,
                        int32_t* chunk, int64_t* stats) {
  if (!h || !n_slots || !n_ops || warps < 1 || n_out < 1 || (n_coef && (!node_ids || !c_re)))
    return fail(ACEDAG_EINVAL, "bad arguments");
  PlanHost H;
  try {
    compile_plan(h->g, node_ids, c_re, c_im, n_coef, n_out, warps, H);
  } catch (const std::domain_error& e) {
    return fail(ACEDAG_ENOTTARGET, e.what());
  } catch (const std::bad_alloc&) {
    return fail(ACEDAG_ENOMEM, "out of host memory compiling the plan");
  } catch (const std::exception& e) {
    return fail(ACEDAG_EINVAL, e.what());
  }
  if (slot_label) std::memcpy(slot_label, H.slot_label.data(), H.slot_label.size() * sizeof(uint16_t));
  if (ops) std::memcpy(ops, H.ops.data(), H.ops.size() * sizeof(Op));
  if (chunk) std::memcpy(chunk, H.chunk.data(), H.chunk.size() * sizeof(int32_t));
  if (stats) {
    stats[0] = H.recursive_products;
    stats[1] = H.extra_nodes;
    stats[2] = H.naive_products;
  }
  *n_slots = (int64_t)H.slot_label.size();
  *n_ops = (int64_t)H.ops.size();
  return ACEDAG_OK;
}

int acedag_plan_program_horner(const acedag_graph* h, const int64_t* node_ids, const double* c_re,
                               int64_t n_coef, int32_t warps, int32_t hot, int32_t us, void* ops, int64_t* n_ops,
                               int32_t* chunk, int32_t* croots) {
  if (!h || !n_ops || warps < 1 || hot < 0 || hot > (int)kHornerHot || us < 0 || (n_coef && (!node_ids || !c_re)))
    return fail(ACEDAG_EINVAL, "bad arguments");
  PlanHost H;
  std::vector<OpH> out;
  std::vector<int32_t> ch, cr;
  try {
    compile_plan(h->g, node_ids, c_re, nullptr, n_coef, 1, warps, H, (uint32_t)hot);
    if (!encode_horner(H, false, (uint32_t)hot, (uint32_t)us, out, ch, cr, true))
      return fail(ACEDAG_EUNSUPPORTED, "program does not fit the k2_horner record fields");
  } catch (const std::domain_error& e) {
    return fail(ACEDAG_ENOTTARGET, e.what());
  } catch (const std::bad_alloc&) {
    return fail(ACEDAG_ENOMEM, "out of host memory compiling the plan");
  } catch (const std::exception& e) {
    return fail(ACEDAG_EINVAL, e.what());
  }
  if (ops) std::memcpy(ops, out.data(), out.size() * sizeof(OpH));
  if (chunk) std::memcpy(chunk, ch.data(), ch.size() * sizeof(int32_t));
  if (croots) std::memcpy(croots, cr.data(), cr.size() * sizeof(int32_t));
  *n_ops = (int64_t)(out.size() / 4);
  return ACEDAG_OK;
}

int acedag_plan_info(const acedag_plan* P, int64_t* recursive_products, int64_t* extra_nodes,
                     int64_t* naive_products, int64_t* used_seeds) {
  if (!P) return fail(ACEDAG_EINVAL, "plan is NULL");
  if (!P->has_coef) return fail(ACEDAG_EINVAL, "plan has no coefficients");
  if (recursive_products) *recursive_products = P->host.recursive_products;
  if (extra_nodes) *extra_nodes = P->host.extra_nodes;
  if (naive_products) *naive_products = P->host.naive_products;
  if (used_seeds) *used_seeds = P->U;
  return ACEDAG_OK;
}

}  // extern "C"

// ------------------------------------------------------------ dispatch
namespace {

constexpr int kWarps = 32;  // general / naive kernels
constexpr int kNC = 8;

// SMs a concurrent kernel of the same call keeps (the host-path seed gather
// runs next to the persistent K2 grid); per thread so calls stay independent
thread_local int t_sm_reserve = 0;
// the eval_impl input is already k2_horner's tile-major table (positions path)
thread_local bool t_input_tiled = false;
// phase events of the eval being launched on this thread (acedag_plan_timing)
thread_local cudaEvent_t* t_tev = nullptr;
thread_local bool t_main_marked = false;
void mark_prep(cudaStream_t st) {
  if (t_tev) cudaEventRecord(t_tev[1], st);
}
void mark_main(cudaStream_t st) {
  if (t_tev) {
    cudaEventRecord(t_tev[2], st);
    t_main_marked = true;
  }
}
// CTAs of the host-path seed gather (ACEDAG_GATHER_CTAS overrides)
int gather_ctas() {
  static int v = [] {
    const char* e = getenv("ACEDAG_GATHER_CTAS");
    return e ? std::max(1, atoi(e)) : 4;
  }();
  return v;
}
bool host_trace() {
  static bool v = getenv("ACEDAG_HOST_TRACE") != nullptr;
  return v;
}

struct Launch {
  int grid, block, us, rows;
  size_t smem;
  bool hyb;
  acedag_plan::Workspace* ws;
};

// tile geometry of the general / naive / multi-output kernels: 32 sites per
// CTA, seed rows [Us][32] in smem (U used seeds plus the constant ONE row),
// the tail in the per-CTA global cache
int plan_launch(acedag_plan* P, int64_t S, size_t elem, size_t red_bytes, int warps, Launch& lc,
                int tile = 32) {
  const int64_t ntiles = (S + tile - 1) / tile;
  lc.block = warps * 32;
  lc.grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, P->sms - t_sm_reserve));
  lc.rows = P->U + 1;
  size_t avail = P->smem_optin > red_bytes ? P->smem_optin - red_bytes : 0;
  int us_max = (int)(avail / (tile * elem));
  lc.us = std::min(lc.rows, us_max);
  lc.hyb = lc.us < lc.rows;
  lc.smem = (size_t)lc.us * tile * elem + red_bytes;
  if (lc.hyb) {
    size_t need = (size_t)lc.grid * (lc.rows - lc.us) * tile;
    if (lc.ws->gcache.alloc(need) != cudaSuccess) return fail(ACEDAG_ENOMEM, "gcache allocation failed");
  }
  return 0;
}

template <typename K>
cudaError_t set_smem(K kernel, size_t smem) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

int nchunks(const acedag_plan* P) { return (int)P->host.chunk.size() - 1; }

// fp64 single-output kernel: ACEDAG_K2 = horner | quad forces one of the two
// for every order; default: k2_horner for order <= 4 (fp64 Horner spills at
// order 5-6), k2_quad above
int k2_mode() {
  static int m = [] {
    const char* e = getenv("ACEDAG_K2");
    if (e && std::string(e) == "quad") return 1;
    if (e && std::string(e) == "horner") return 2;
    return 0;
  }();
  return m;
}

// The last round of a persistent tile loop is short of tiles when ntiles is
// not a multiple of the grid; those tiles are split into `parts` program
// slices (up to the grid, at most ACEDAG_TAIL_PARTS, default 8) whose partial
// sums are added in slice order.  full = tiles run whole.
void tail_split(int64_t ntiles, int grid, int nchunk, int64_t& full, int& parts) {
  static int cap = [] {
    const char* e = getenv("ACEDAG_TAIL_PARTS");
    return e ? std::max(1, atoi(e)) : 8;
  }();
  const int64_t rem = ntiles % grid;
  full = ntiles;
  parts = 1;
  if (rem == 0) return;
  int p = (int)std::min<int64_t>(grid / rem, cap);
  p = std::min(p, std::max(1, nchunk / 8));
  if (p <= 1) return;
  full = ntiles - rem;
  parts = p;
}

// the tile-major seed copy (k_tile_seeds<TS>) for an eval_impl input, or
// false when the input layout is not one the plan knows
template <int TS, typename V = double2>
bool tile_seeds(acedag_plan* P, const V* A, int64_t S, int L, const uint16_t* slot_label,
                acedag_plan::Workspace* ws, cudaStream_t st, cudaError_t& e) {
  e = cudaSuccess;
  const int32_t* cols = nullptr;
  const uint16_t* slots = nullptr;
  if (slot_label == P->slot_label.p) {
    cols = P->sorted_labels.p;
    slots = P->sorted_slot.p;
  } else if (slot_label == P->slot_sorted.p) {
    slots = P->sorted_slot.p;
  } else if (slot_label != P->slot_identity.p) {
    return false;
  }
  const int64_t ntiles = (S + TS - 1) / TS;
  e = ws->tiles.alloc((size_t)ntiles * (P->U + 1) * TS);
  if (e != cudaSuccess) return true;
  constexpr size_t tsm = 32 * (TS + 1) * sizeof(V);
  // per call: the attribute is per device, and plans may live on several
  e = cudaFuncSetAttribute(dev::k_tile_seeds<TS, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm);
  if (e != cudaSuccess) return true;
  dev::k_tile_seeds<TS, V><<<(unsigned)ntiles, 512, tsm, st>>>(A, S, L, cols, slots, P->U,
                                                                   reinterpret_cast<V*>(ws->tiles.p)); note_launch();
  e = cudaGetLastError();
  return true;
}

// geometry of k2_quad: 128-site tiles, 32 hot rows in TMEM, 2 KB cold rows
// in shared memory, the tail read in place from the tile-major table
// warps per k2_quad CTA: since the walk is declared warp-uniform more warps
// at fewer registers win (cfg4, 4e4 sites: 16 x 128 registers 482 k sites/s,
// 20 x 96 531 k, 24 x 80 574 k, 28 x 72 568 k, 32 x 64 570 k)
#ifndef ACEDAG_QUAD_WARPS
#define ACEDAG_QUAD_WARPS 24
#endif
constexpr int kQuadWarps = ACEDAG_QUAD_WARPS;
int quad_launch(acedag_plan* P, int64_t S, Launch& lc) {
  const int64_t ntiles = (S + 127) / 128;
  lc.block = kQuadWarps * 32;
  lc.grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, P->sms - t_sm_reserve));
  lc.rows = P->U + 1;
  const int cold = std::max(0, lc.rows - (int)dev::kTmemRowsQ);
  // rings, TMEM slot + chunk counter (16 B), slot -> label table
  const size_t fixed = (size_t)kQuadWarps * dev::Ring3::kAlloc + 16 + (((size_t)lc.rows * 4 + 15) & ~(size_t)15);
  const int us_max = (int)((P->smem_optin - fixed) / 2048);
  lc.us = std::min(cold, us_max);
  lc.hyb = lc.us < cold;
  lc.smem = (size_t)lc.us * 2048 + fixed;
  return 0;
}

template <int NU, bool HYB>
cudaError_t launch_quad_k(acedag_plan* P, const double2* A, int64_t S, int L, const uint16_t* slot_label,
                          double* out, const Launch& lc, cudaStream_t st) {
  constexpr int W = kQuadWarps;
  constexpr int MAXU = NU <= 4 ? 2 : 1;
  cudaError_t e;
  if (!tile_seeds<128>(P, A, S, L, slot_label, lc.ws, st, e)) return cudaErrorInvalidValue;
  if (e != cudaSuccess) return e;
  A = lc.ws->tiles.p;
  mark_prep(st);
  auto k = dev::k2_quad<NU, W, MAXU, HYB, true>;
  e = set_smem(k, lc.smem);
  if (e != cudaSuccess) return e;
  e = lc.ws->part.alloc((size_t)lc.grid * nchunks(P) * 128);
  if (e != cudaSuccess) return e;
  const int64_t ntiles = (S + 127) / 128;
  int64_t full = ntiles;
  int parts = 1;
  tail_split(ntiles, lc.grid, nchunks(P), full, parts);
  if (parts > 1) {
    e = lc.ws->tail.alloc((size_t)(ntiles - full) * nchunks(P) * 128);
    if (e != cudaSuccess) return e;
  }
  k<<<lc.grid, lc.block, lc.smem, st>>>(A, S, L, slot_label, P->U, lc.us, P->opsQ.p, P->chunk.p, nchunks(P),
                                        out, nullptr, lc.ws->part.p, full, parts, lc.ws->tail.p); note_launch();
  mark_main(st);
  e = cudaGetLastError();
  if (e != cudaSuccess || parts == 1) return e;
  const int64_t rem = S - full * 128;
  dev::k_tail_reduce<<<(unsigned)((rem + 255) / 256), 256, 0, st>>>(lc.ws->tail.p, full * 128, S, 128, nchunks(P), out); note_launch();
  return cudaGetLastError();
}

template <int NU> struct QuadF64 {
  template <typename... A> static cudaError_t run(bool hyb, A... a) {
    return hyb ? launch_quad_k<NU, true>(a...) : launch_quad_k<NU, false>(a...);
  }
};

// k2_horner on the tile-major seed table (V: double2, or float2 for the fp32
// mode); false (nothing launched) when the input layout is not one
// tile_seeds knows
template <typename V>
bool run_horner(acedag_plan* P, const V* A, int64_t S, int L, const uint16_t* slot_label, double* out,
                Launch& lc, cudaStream_t st, cudaError_t& e) {
  constexpr bool f32 = sizeof(V) == 8;
  const acedag_plan::HornerProg& hp = P->hp[f32 ? 1 : 0];
  const void* table = A;  // already tile-major (the positions path's pool wrote it)
  if (!t_input_tiled) {
    if (!tile_seeds<128, V>(P, A, S, L, slot_label, lc.ws, st, e)) return false;
    if (e != cudaSuccess) return true;
    table = lc.ws->tiles.p;
  }
  mark_prep(st);
  const int64_t ntiles = (S + 127) / 128;
  // fewer tiles than SMs: the grid covers program slices of them too
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles * 8, P->sms - t_sm_reserve));
  const int nch = nchunks(P);
  e = lc.ws->part.alloc((size_t)grid * nch * 128 * 2);  // double-buffered per CTA
  if (e != cudaSuccess) return true;
  int64_t full = ntiles;
  int parts = 1;
  tail_split(ntiles, grid, nch, full, parts);
  if (parts > 1) {
    e = lc.ws->tail.alloc((size_t)(ntiles - full) * nch * 128);
    if (e != cudaSuccess) return true;
  }
  e = launch_horner(P->host.max_order, f32, table, S, P->U, hp.us, hp.ops.p, hp.chunk.p, hp.croots.p, nch,
                    out, lc.ws->part.p, full, parts, lc.ws->tail.p, grid, st);
  note_launch();
  mark_main(st);
  if (e != cudaSuccess || parts == 1) return true;
  const int64_t rem = S - full * 128;
  dev::k_tail_reduce<<<(unsigned)((rem + 255) / 256), 256, 0, st>>>(lc.ws->tail.p, full * 128, S, 128, nch, out);
  note_launch();
  e = cudaGetLastError();
  return true;
}

// k2_horner for fp64 order <= 4 and every fp32 order, at every batch size
// (so a site's value never depends on its batch); ACEDAG_K2 overrides fp64
bool use_horner(const acedag_plan* P, bool f32 = false) {
  const acedag_plan::HornerProg& hp = P->hp[f32 ? 1 : 0];
  if (!hp.ok) return false;
  if (f32) return true;
  return k2_mode() == 2 || (k2_mode() == 0 && P->host.max_order <= 4);
}

#ifndef ACEDAG_MMA_WARPS
#define ACEDAG_MMA_WARPS 16
#endif
constexpr int kMmaWarps = ACEDAG_MMA_WARPS;

template <int NU, bool HYB>
cudaError_t launch_mma(acedag_plan* P, const double2* A, int64_t S, int L, const uint16_t* slot_label,
                       double* out, const Launch& lc, cudaStream_t st) {
  auto k = dev::k2_mma<NU, kMmaWarps, HYB>;
  cudaError_t e = set_smem(k, lc.smem);
  if (e != cudaSuccess) return e;
  e = lc.ws->part.alloc((size_t)lc.grid * kMmaWarps * 32 * 32);
  if (e != cudaSuccess) return e;
  for (int o0 = 0; o0 < P->host.n_out; o0 += 32) {
    k<<<lc.grid, lc.block, lc.smem, st>>>(A, S, L, slot_label, P->U, lc.us, P->ops.p, P->chunk.p, nchunks(P),
                                          P->cre.p, P->host.n_out, o0, out, lc.ws->gcache.p, lc.ws->part.p); note_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <int NU, bool HYB>
cudaError_t launch_general(acedag_plan* P, const double2* A, int64_t S, int L,
                           const uint16_t* slot_label, int complex_out, void* out, const Launch& lc,
                           cudaStream_t st) {
  auto k = dev::k2_general<NU, kNC, HYB>;
  cudaError_t e = set_smem(k, lc.smem);
  if (e != cudaSuccess) return e;
  for (int o0 = 0; o0 < P->host.n_out; o0 += kNC) {
    k<<<lc.grid, lc.block, lc.smem, st>>>(A, S, L, slot_label, P->U, lc.us, P->ops.p, P->chunk.p,
                                          nchunks(P), P->cre.p,
                                          P->host.complex_coef ? P->cim.p : nullptr, P->host.n_out, o0,
                                          complex_out, out, lc.ws->gcache.p); note_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <int NU, bool GEN, bool HYB>
cudaError_t launch_naive(acedag_plan* P, const double2* A, int64_t S, int L,
                         const uint16_t* slot_label, int complex_out, void* out, const Launch& lc,
                         cudaStream_t st) {
  auto k = dev::k3_naive<NU, GEN, HYB>;
  cudaError_t e = set_smem(k, lc.smem);
  if (e != cudaSuccess) return e;
  for (int o0 = 0; o0 < P->host.n_out; ++o0) {
    k<<<lc.grid, lc.block, lc.smem, st>>>(A, S, L, slot_label, P->U, lc.us, P->nseg.p, P->nslots.p,
                                          P->ncre.p, P->host.complex_coef ? P->ncim.p : nullptr,
                                          P->host.n_out, o0, complex_out, out, lc.ws->gcache.p); note_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// runtime NU -> template
template <template <int> class F, typename... Args>
cudaError_t by_order(int nu, Args&&... a) {
  switch (nu) {
    case 2: return F<2>::run(a...);
    case 3: return F<3>::run(a...);
    case 4: return F<4>::run(a...);
    case 5: return F<5>::run(a...);
    case 6: return F<6>::run(a...);
  }
  return cudaErrorInvalidValue;
}

template <int NU> struct Mma {
  template <typename... A> static cudaError_t run(bool hyb, A... a) {
    return hyb ? launch_mma<NU, true>(a...) : launch_mma<NU, false>(a...);
  }
};
template <int NU> struct General {
  template <typename... A> static cudaError_t run(bool hyb, A... a) {
    return hyb ? launch_general<NU, true>(a...) : launch_general<NU, false>(a...);
  }
};
template <int NU> struct NaiveFast {
  template <typename... A> static cudaError_t run(bool hyb, A... a) {
    return hyb ? launch_naive<NU, false, true>(a...) : launch_naive<NU, false, false>(a...);
  }
};
template <int NU> struct NaiveGen {
  template <typename... A> static cudaError_t run(bool hyb, A... a) {
    return hyb ? launch_naive<NU, true, true>(a...) : launch_naive<NU, true, false>(a...);
  }
};

// which kernel eval_body launches (acedag_eval_kernel_name reports it)
enum class K2 { Horner, Quad, Mma, General, Naive, None };
K2 pick(const acedag_plan* P, int method, int prec, int out_kind) {
  const PlanHost& H = P->host;
  if (method == ACEDAG_METHOD_NAIVE) return prec == ACEDAG_PREC_F64 ? K2::Naive : K2::None;
  const bool fast = out_kind == ACEDAG_OUT_REAL && H.n_out == 1 && !H.complex_coef;
  if (prec == ACEDAG_PREC_F32) return fast && use_horner(P, true) ? K2::Horner : K2::None;
  if (fast) return use_horner(P) ? K2::Horner : K2::Quad;
  if (out_kind == ACEDAG_OUT_REAL && !H.complex_coef && H.n_out >= 8) return K2::Mma;
  return K2::General;
}

int eval_body(acedag_plan* P, int method, int prec, int out_kind, const void* A, int64_t S, int L,
              const uint16_t* slot_label, void* out, cudaStream_t st);

int eval_impl(acedag_plan* P, int method, int prec, int out_kind, const void* A, int64_t S, int L,
              const uint16_t* slot_label, void* out, cudaStream_t st) {
  if (!P->timing.on) return eval_body(P, method, prec, out_kind, A, S, L, slot_label, out, st);
  std::array<cudaEvent_t, 4> ev;
  for (auto& e : ev) cudaEventCreate(&e);
  cudaEventRecord(ev[0], st);
  cudaEventRecord(ev[1], st);  // no seed-prep phase unless the launcher marks one
  t_tev = ev.data();
  t_main_marked = false;
  const int rc = eval_body(P, method, prec, out_kind, A, S, L, slot_label, out, st);
  if (!t_main_marked) cudaEventRecord(ev[2], st);
  cudaEventRecord(ev[3], st);
  t_tev = nullptr;
  std::lock_guard<std::mutex> lk(P->timing.mu);
  P->timing.ev.push_back(ev);
  return rc;
}

int eval_body(acedag_plan* P, int method, int prec, int out_kind, const void* A, int64_t S, int L,
              const uint16_t* slot_label, void* out, cudaStream_t st) {
  const PlanHost& H = P->host;
  Launch lc;
  lc.ws = P->ws(st);
  cudaError_t e = cudaSuccess;
  switch (pick(P, method, prec, out_kind)) {
    case K2::None:
      if (method == ACEDAG_METHOD_NAIVE) return fail(ACEDAG_EUNSUPPORTED, "naive path is fp64 only");
      return fail(ACEDAG_EUNSUPPORTED,
                  "fp32 mode supports real coefficients and one real output on programs k2_horner can encode");
    case K2::Horner:
      if (prec == ACEDAG_PREC_F32) {
        if (!run_horner(P, (const float2*)A, S, L, slot_label, (double*)out, lc, st, e))
          return fail(ACEDAG_EINVAL, "unknown seed layout");
      } else if (!run_horner(P, (const double2*)A, S, L, slot_label, (double*)out, lc, st, e)) {
        return fail(ACEDAG_EINVAL, "unknown seed layout");
      }
      if (e != cudaSuccess) return cuda_fail(e, "k2_horner");
      return ACEDAG_OK;
    case K2::Quad: {
      int rc = quad_launch(P, S, lc);
      if (rc) return rc;
      e = by_order<QuadF64>(H.max_order, lc.hyb, P, (const double2*)A, S, L, slot_label, (double*)out, lc, st);
      break;
    }
    case K2::Mma: {
      // smem beyond the seed rows: 16 program rings + 16 x [8][36] staging
      int rc = plan_launch(P, S, sizeof(double2), kMmaWarps * 1024 + kMmaWarps * 8 * 36 * 8, kMmaWarps, lc);
      if (rc) return rc;
      e = by_order<Mma>(H.max_order, lc.hyb, P, (const double2*)A, S, L, slot_label, (double*)out, lc, st);
      break;
    }
    case K2::General: {
      int rc = plan_launch(P, S, sizeof(double2), 2 * kWarps * 32 * sizeof(double), kWarps, lc);
      if (rc) return rc;
      e = by_order<General>(H.max_order, lc.hyb, P, (const double2*)A, S, L, slot_label,
                            out_kind == ACEDAG_OUT_COMPLEX ? 1 : 0, out, lc, st);
      break;
    }
    case K2::Naive: {
      int rc = plan_launch(P, S, sizeof(double2), 2 * kWarps * 32 * sizeof(double), kWarps, lc);
      if (rc) return rc;
      const int nu = std::max(2, H.naive_max_order);
      const bool fast = out_kind == ACEDAG_OUT_REAL && H.n_out == 1 && !H.complex_coef;
      if (fast) e = by_order<NaiveFast>(nu, lc.hyb, P, (const double2*)A, S, L, slot_label, 0, out, lc, st);
      else
        e = by_order<NaiveGen>(nu, lc.hyb, P, (const double2*)A, S, L, slot_label,
                               out_kind == ACEDAG_OUT_COMPLEX ? 1 : 0, out, lc, st);
      break;
    }
  }
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  return ACEDAG_OK;
}

}  // namespace

extern "C" {

int acedag_eval(const acedag_plan* Pc, int method, int prec, int out_kind, const void* A, int64_t S,
                void* out, void* stream) {
  acedag_plan* P = const_cast<acedag_plan*>(Pc);
  if (!P || ((!out || !A) && S > 0)) return fail(ACEDAG_EINVAL, "NULL argument");
  if (!P->has_coef) return fail(ACEDAG_EINVAL, "plan has no coefficients (acedag_plan_set_coefficients)");
  if (method != ACEDAG_METHOD_RECURSIVE && method != ACEDAG_METHOD_NAIVE)
    return fail(ACEDAG_EINVAL, "unknown method");
  if (prec != ACEDAG_PREC_F64 && prec != ACEDAG_PREC_F32) return fail(ACEDAG_EINVAL, "unknown precision");
  if (out_kind != ACEDAG_OUT_REAL && out_kind != ACEDAG_OUT_COMPLEX)
    return fail(ACEDAG_EINVAL, "unknown output kind");
  if (S < 0) return fail(ACEDAG_EINVAL, "negative site count");
  if (S == 0) return ACEDAG_OK;
  DevGuard dg(P->device);
  return eval_impl(P, method, prec, out_kind, A, S, (int)P->g->n_seeds(), P->slot_label.p, out,
                   (cudaStream_t)stream);
}

int acedag_eval_host(const acedag_plan* Pc, int method, int prec, int out_kind, const void* A_host, int64_t S,
                     void* out_host, int64_t* h2d_bytes, void* stream) {
  acedag_plan* P = const_cast<acedag_plan*>(Pc);
  if (!P || ((!out_host || !A_host) && S > 0)) return fail(ACEDAG_EINVAL, "NULL argument");
  if (!P->has_coef) return fail(ACEDAG_EINVAL, "plan has no coefficients (acedag_plan_set_coefficients)");
  if (method != ACEDAG_METHOD_RECURSIVE && method != ACEDAG_METHOD_NAIVE)
    return fail(ACEDAG_EINVAL, "unknown method");
  if (prec != ACEDAG_PREC_F64 && prec != ACEDAG_PREC_F32) return fail(ACEDAG_EINVAL, "unknown precision");
  if (out_kind != ACEDAG_OUT_REAL && out_kind != ACEDAG_OUT_COMPLEX)
    return fail(ACEDAG_EINVAL, "unknown output kind");
  if (S < 0) return fail(ACEDAG_EINVAL, "negative site count");
  if (h2d_bytes) *h2d_bytes = 0;
  if (S == 0) return ACEDAG_OK;
  DevGuard dg(P->device);
  std::lock_guard<std::mutex> lk(P->host_mu);
  acedag_plan::HostPipe& H = P->pipe;
  cudaError_t e = H.init();
  if (e != cudaSuccess) return cuda_fail(e, "host pipeline streams");
  const size_t esz = prec == ACEDAG_PREC_F32 ? 8 : 16;
  const size_t ow = (size_t)P->host.n_out * (out_kind == ACEDAG_OUT_COMPLEX ? 16 : 8);
  const int L = (int)P->g->n_seeds(), U = P->U;
  // page-locked input is device-mapped (unified addressing): gather in place
  cudaPointerAttributes at;
  const bool mapped = cudaPointerGetAttributes(&at, A_host) == cudaSuccess && at.type == cudaMemoryTypeHost &&
                      at.devicePointer != nullptr;
  cudaGetLastError();
  const int width = mapped ? U : L;
  // two K2 rounds of 64-site tiles per chunk on the SMs the gather leaves free
  const int64_t chunk = std::min<int64_t>(S, (int64_t)2 * 64 * (P->sms - gather_ctas()));
  for (int b = 0; b < 2; ++b) {
    if (H.buf[b].alloc((size_t)chunk * width * esz) != cudaSuccess || H.out[b].alloc((size_t)chunk * ow) != cudaSuccess)
      return fail(ACEDAG_ENOMEM, "host pipeline buffers");
  }
  if ((e = cudaEventRecord(H.start, (cudaStream_t)stream)) != cudaSuccess ||
      (e = cudaStreamWaitEvent(H.sg, H.start, 0)) != cudaSuccess || (e = cudaStreamWaitEvent(H.sk, H.start, 0)) != cudaSuccess)
    return cuda_fail(e, "host pipeline ordering");
  const char* src = static_cast<const char*>(mapped ? at.devicePointer : A_host);
  char* dst = static_cast<char*>(out_host);
  int rc = ACEDAG_OK;
  t_sm_reserve = mapped ? gather_ctas() : 0;
  std::vector<cudaEvent_t> tr;  // ACEDAG_HOST_TRACE: per-chunk stage timings
  auto mark = [&](cudaStream_t s) {
    if (!host_trace()) return;
    cudaEvent_t ev;
    cudaEventCreate(&ev);
    cudaEventRecord(ev, s);
    tr.push_back(ev);
  };
  mark(H.sg);
  for (int64_t s0 = 0, i = 0; s0 < S && rc == ACEDAG_OK; s0 += chunk, ++i) {
    const int b = (int)(i & 1);
    const int64_t n = std::min(chunk, S - s0);
    if (i >= 2) cudaStreamWaitEvent(H.sg, H.kdone[b], 0);  // K2 of chunk i-2 is done with buf[b]
    mark(H.sg);
    if (mapped) {
      if (esz == 16)
        dev::k_gather_seeds<double2><<<gather_ctas(), 512, U * 4, H.sg>>>(
            reinterpret_cast<const double2*>(src) + s0 * L, n, L, P->sorted_labels.p, U,
            reinterpret_cast<double2*>(H.buf[b].p));
      else
        dev::k_gather_seeds<float2><<<gather_ctas(), 512, U * 4, H.sg>>>(
            reinterpret_cast<const float2*>(src) + s0 * L, n, L, P->sorted_labels.p, U,
            reinterpret_cast<float2*>(H.buf[b].p));
      note_launch();
      e = cudaGetLastError();
    } else {
      e = cudaMemcpyAsync(H.buf[b].p, src + (size_t)s0 * L * esz, (size_t)n * L * esz, cudaMemcpyHostToDevice, H.sg);
    }
    if (e != cudaSuccess) { rc = cuda_fail(e, "host pipeline input"); break; }
    mark(H.sg);
    cudaEventRecord(H.gdone[b], H.sg);
    cudaStreamWaitEvent(H.sk, H.gdone[b], 0);
    mark(H.sk);
    rc = eval_impl(P, method, prec, out_kind, H.buf[b].p, n, width, mapped ? P->slot_sorted.p : P->slot_label.p,
                   H.out[b].p, H.sk);
    if (rc) break;
    mark(H.sk);
    cudaEventRecord(H.kdone[b], H.sk);
    e = cudaMemcpyAsync(dst + (size_t)s0 * ow, H.out[b].p, (size_t)n * ow, cudaMemcpyDeviceToHost, H.sk);
    if (e != cudaSuccess) rc = cuda_fail(e, "host pipeline output");
  }
  t_sm_reserve = 0;
  mark(H.sk);
  cudaError_t e1 = cudaStreamSynchronize(H.sg), e2 = cudaStreamSynchronize(H.sk);
  if (!tr.empty()) {
    // [start, (gather begin, gather end, eval begin, eval end) per chunk..., end]
    for (size_t k = 1; k < tr.size(); ++k) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tr[0], tr[k]);
      fprintf(stderr, "%s%.3f", k == 1 ? "host trace ms:" : (k % 4 == 1 ? " |" : " "), ms);
    }
    fprintf(stderr, "\n");
    for (cudaEvent_t ev : tr) cudaEventDestroy(ev);
  }
  if (rc) return rc;
  if (e1 != cudaSuccess || e2 != cudaSuccess) return cuda_fail(e1 != cudaSuccess ? e1 : e2, "host pipeline");
  if (h2d_bytes) *h2d_bytes = S * (int64_t)width * (int64_t)esz;
  return ACEDAG_OK;
}

int64_t acedag_launch_count(void) { return g_launches.load(); }

int acedag_plan_timing(acedag_plan* P, int enable) {
  if (!P) return fail(ACEDAG_EINVAL, "plan is NULL");
  DevGuard dg(P->device);
  std::lock_guard<std::mutex> lk(P->timing.mu);
  P->timing.clear();
  P->timing.on = enable != 0;
  return ACEDAG_OK;
}

int acedag_plan_timing_read(acedag_plan* P, double* ms, int64_t* calls) {
  if (!P || !ms) return fail(ACEDAG_EINVAL, "NULL argument");
  DevGuard dg(P->device);
  std::lock_guard<std::mutex> lk(P->timing.mu);
  ms[0] = ms[1] = ms[2] = 0.0;
  for (auto& a : P->timing.ev) {
    cudaError_t e = cudaEventSynchronize(a[3]);
    if (e != cudaSuccess) return cuda_fail(e, "timing events");
    for (int k = 0; k < 3; ++k) {
      float t = 0.f;
      cudaEventElapsedTime(&t, a[k], a[k + 1]);
      ms[k] += t;
    }
  }
  if (calls) *calls = (int64_t)P->timing.ev.size();
  P->timing.clear();
  return ACEDAG_OK;
}

const char* acedag_eval_kernel_name(const acedag_plan* P, int method, int prec, int out_kind, int64_t S) {
  (void)S;  // the choice does not depend on the batch size
  if (!P || !P->has_coef) {
    fail(ACEDAG_EINVAL, "plan has no coefficients");
    return "";
  }
  switch (pick(P, method, prec, out_kind)) {
    case K2::Horner: return prec == ACEDAG_PREC_F32 ? "k2_horner (fp32)" : "k2_horner";
    case K2::Quad: return "k2_quad";
    case K2::Mma: return "k2_mma";
    case K2::General: return "k2_general";
    case K2::Naive: return "k3_naive";
    default: return "";
  }
}

int acedag_reduce_sites(const acedag_plan* P, const double* phi, int64_t S, double* out_total,
                        void* stream) {
  if (!P || !out_total || (S > 0 && !phi)) return fail(ACEDAG_EINVAL, "NULL argument");
  if (!P->has_coef) return fail(ACEDAG_EINVAL, "plan has no coefficients");
  DevGuard dg(P->device);
  dev::k_reduce_sites<<<P->host.n_out, 1024, 0, (cudaStream_t)stream>>>(phi, S, P->host.n_out, out_total); note_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "k_reduce_sites");
  return ACEDAG_OK;
}

int acedag_naive_products(const double* vals, const int32_t* lens, int64_t n, int32_t width,
                          double* out, void* stream) {
  if (n < 0 || width < 0 || !out || (n > 0 && width > 0 && !vals)) return fail(ACEDAG_EINVAL, "bad arguments");
  if (n == 0) return ACEDAG_OK;
  int grid = (int)std::min<int64_t>((n + 127) / 128, 148 * 16);
  dev::k_naive_products<<<grid, 128, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const double2*>(vals), lens, n, width, reinterpret_cast<double2*>(out)); note_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "k_naive_products");
  return ACEDAG_OK;
}

int acedag_eval_nodes(const acedag_plan* P, const double* A, int64_t S, double* node_vals, void* stream) {
  if (!P || ((!node_vals || !A) && S > 0)) return fail(ACEDAG_EINVAL, "NULL argument");
  if (S <= 0) return S < 0 ? fail(ACEDAG_EINVAL, "negative site count") : ACEDAG_OK;
  DevGuard dg(P->device);
  const int64_t N = (int64_t)P->g->tuples.size();
  const int L = (int)P->g->n_seeds();
  int grid = (int)std::min<int64_t>((S + 127) / 128, (int64_t)P->sms * 16);
  dev::k_eval_nodes<<<grid, 128, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const double2*>(A), S, L, N, P->pa.p, P->pb.p, reinterpret_cast<double2*>(node_vals)); note_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "k_eval_nodes");
  return ACEDAG_OK;
}

int acedag_check_coords(int group, const double* c, int64_t n) {
  static const int nc[4] = {1, 2, 3, 4};
  if (group < 0 || group > 3) return fail(ACEDAG_EINVAL, "unknown group");
  if (n > 0 && !c) return fail(ACEDAG_EINVAL, "NULL coordinates");
  for (int64_t i = 0; i < n; ++i) {
    const double* p = c + i * nc[group];
    char buf[96];
    if (group != kT && !(p[0] >= 0.0 && p[0] <= 1.0)) {
      snprintf(buf, sizeof buf, "%.17g", p[0]);
      return fail(ACEDAG_EDOMAIN, std::string("radius must lie in [0, 1], got ") + buf);
    }
    if (group == kO3F && !(p[3] >= -1.0 && p[3] <= 1.0)) {
      snprintf(buf, sizeof buf, "%.17g", p[3]);
      return fail(ACEDAG_EDOMAIN, std::string("feature value must lie in [-1, 1], got ") + buf);
    }
  }
  return ACEDAG_OK;
}

int acedag_pool(int group, int cap, const double* coords, const int32_t* counts, int64_t S, int32_t J,
                double* A_out, void* stream) {
  if (group < 0 || group > 3) return fail(ACEDAG_EINVAL, "unknown group");
  if (cap < 0 || S < 0 || J < 0 || !A_out || (S > 0 && J > 0 && !coords))
    return fail(ACEDAG_EINVAL, "bad pool arguments");
  if ((group == kO3 || group == kO3F) && cap > ACEDAG_YLM_LMAX)
    return fail(ACEDAG_EUNSUPPORTED, "degree cap above the compiled Y_lm table");
  const int dev = current_device();
  int rc = ensure_norms(dev);
  if (rc) return rc;
  const int4* labels = nullptr;
  rc = device_labels(dev, group, cap, &labels);
  if (rc) return rc;
  const int L = (int)one_particle_indices(group, cap).size();
  const int64_t total = S * (int64_t)L;
  if (total == 0) return ACEDAG_OK;
  int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 64);
  cudaStream_t st = (cudaStream_t)stream;
  double2* out = reinterpret_cast<double2*>(A_out);
  switch (group) {
    case 0: dev::pool_ref<0><<<grid, 256, 0, st>>>(coords, counts, S, J, labels, L, out); note_launch(); break;
    case 1: dev::pool_ref<1><<<grid, 256, 0, st>>>(coords, counts, S, J, labels, L, out); note_launch(); break;
    case 2: dev::pool_ref<2><<<grid, 256, 0, st>>>(coords, counts, S, J, labels, L, out); note_launch(); break;
    default: dev::pool_ref<3><<<grid, 256, 0, st>>>(coords, counts, S, J, labels, L, out); note_launch(); break;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "pool_ref");
  return ACEDAG_OK;
}

// col_of: label -> output column (or -1), NULL = every label at its index;
// tri/ntri: the triples to compute (NULL = all of this cap)
// prune: every triple has l + m <= cap (the plan's labels), so the Y_lm
// tables may skip the pairs above that line (pool_positions4 PRUNE)
// tile_rows > 0 (pool_positions5 only): write K2's tile-major table
static int pool_positions_impl(int cap, const double* xyz, const int32_t* counts, int64_t S, int J,
                               double r_in, double r_cut, const int32_t* col_of, const int4* tri,
                               int ntri, int64_t out_stride, double* A_out, cudaStream_t st, bool prune = false,
                               int tile_rows = 0) {
  if (cap < 0 || cap > ACEDAG_YLM_LMAX) return fail(ACEDAG_EUNSUPPORTED, "degree cap outside [0, 40]");
  if (!(r_cut > r_in) || !(r_in >= 0.0)) return fail(ACEDAG_EINVAL, "need 0 <= r_in < r_cut");
  const int dev = current_device();
  int rc = ensure_norms(dev);
  if (rc) return rc;
  const int4* labels = nullptr;
  rc = device_labels(dev, kO3, cap, &labels);
  if (rc) return rc;
  const int L = (int)one_particle_indices(kO3, cap).size();
  if (S == 0) return ACEDAG_OK;
  const size_t smem = dev::pool2_smem(cap, std::max(J, 1));
  int optin = 0;
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  if (smem > (size_t)optin) return fail(ACEDAG_EUNSUPPORTED, "too many neighbours per site for the pool tables");
  const int64_t stride = col_of ? out_stride : L;
  double2* out = reinterpret_cast<double2*>(A_out);
  int sms = 148;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int grid = (int)std::min<int64_t>(S, (int64_t)sms * 16);
  if (!tri) {  // every label: the cached full triple table of this cap
    int rc2 = full_triples(dev, cap, &tri, &ntri);
    if (rc2) return rc2;
  }
  // v4 (compile-time degree cap, warp per site) for caps 12 and 14 when the
  // triples fit its accumulators; ACEDAG_POOL=2 forces v2 (CTA per site)
  static const bool force_v2 = getenv("ACEDAG_POOL") && atoi(getenv("ACEDAG_POOL")) == 2;
  static const bool force_v4 = getenv("ACEDAG_POOL") && atoi(getenv("ACEDAG_POOL")) == 4;
  bool done = false;
  // v5 (accumulation on DMMA) for plan-driven pools with pruned tables
  if (!force_v2 && !force_v4 && prune && (cap == 12 || cap == 14)) {
    auto launch5 = [&](auto k, int W, size_t sm5) -> cudaError_t {
      cudaError_t e5 = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm5);
      if (e5 != cudaSuccess) return e5;
      const int g5 = (int)std::min<int64_t>((S + W - 1) / W, (int64_t)sms * 16);
      k<<<g5, W * 32, sm5, st>>>(xyz, counts, S, J, r_in, r_cut, col_of, stride, out, tile_rows);
      return cudaGetLastError();
    };
    cudaError_t e5 = cap == 12 ? launch5(dev::pool_positions5<12>, dev::Pool5Geom<12>::kW, dev::Pool5Geom<12>::kSmem)
                               : launch5(dev::pool_positions5<14>, dev::Pool5Geom<14>::kW, dev::Pool5Geom<14>::kSmem);
    note_launch();
    if (e5 != cudaSuccess) return cuda_fail(e5, "pool_positions5");
    done = true;
  }
  if (tile_rows > 0 && !done) return fail(ACEDAG_EINVAL, "tile-major pool output needs pool_positions5");
  if (!done && !force_v2 && (cap == 12 || cap == 14) && ntri <= 32 * 16) {
    auto launch4 = [&](auto k, int W, size_t wb) -> cudaError_t {
      const size_t sm4 = (size_t)W * wb;
      cudaError_t e4 = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm4);
      if (e4 != cudaSuccess) return e4;
      const int g4 = (int)std::min<int64_t>((S + W - 1) / W, (int64_t)sms * 64);
      k<<<g4, W * 32, sm4, st>>>(xyz, counts, S, J, r_in, r_cut, tri, ntri, col_of, stride, out);
      return cudaGetLastError();
    };
    cudaError_t e4;
#define ACEDAG_P4(C, PR)                                                                            \
  (ntri <= 256 ? launch4(dev::pool_positions4<C, 8, PR>, dev::Pool4Geom<C, PR>::kW,                \
                         dev::Pool4Geom<C, PR>::kWarpBytes)                                         \
               : launch4(dev::pool_positions4<C, 16, PR>, dev::Pool4Geom<C, PR>::kW,               \
                         dev::Pool4Geom<C, PR>::kWarpBytes))
    if (cap == 12) e4 = prune ? ACEDAG_P4(12, true) : ACEDAG_P4(12, false);
    else e4 = prune ? ACEDAG_P4(14, true) : ACEDAG_P4(14, false);
#undef ACEDAG_P4
    note_launch();
    if (e4 != cudaSuccess) return cuda_fail(e4, "pool_positions4");
    done = true;
  }
  if (!done) {
    CK(cudaFuncSetAttribute(dev::pool_positions2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dev::pool_positions2<<<grid, 256, smem, st>>>(xyz, counts, S, J, cap, r_in, r_cut, tri, ntri, col_of,
                                                  stride, out); note_launch();
  }
  (void)labels;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "pool_positions");
  return ACEDAG_OK;
}

int acedag_pool_positions(int cap, const double* xyz, const int32_t* counts, int64_t S, int32_t J,
                          double r_in, double r_cut, double* A_out, void* stream) {
  if (S < 0 || J < 0 || !A_out || (S > 0 && J > 0 && !xyz)) return fail(ACEDAG_EINVAL, "bad pool arguments");
  return pool_positions_impl(cap, xyz, counts, S, J, r_in, r_cut, nullptr, nullptr, 0, 0, A_out,
                             (cudaStream_t)stream);
}

int acedag_eval_from_positions(acedag_plan* P, const double* xyz, const int32_t* counts, int64_t S,
                               int32_t J, double r_in, double r_cut, int out_kind, void* out,
                               void* stream) {
  if (!P || !out || S < 0 || J < 0 || (S > 0 && J > 0 && !xyz)) return fail(ACEDAG_EINVAL, "bad arguments");
  if (!P->has_coef) return fail(ACEDAG_EINVAL, "plan has no coefficients");
  if (P->g->group != kO3) return fail(ACEDAG_EUNSUPPORTED, "positions input needs an O3 graph");
  if (S == 0) return ACEDAG_OK;
  DevGuard dg(P->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t chunk = 1 << 17;
  const int U = P->U;
  acedag_plan::Workspace* W = P->ws(st);
  if (W->ws_A.alloc((size_t)std::min<int64_t>(S, chunk) * U) != cudaSuccess)
    return fail(ACEDAG_ENOMEM, "workspace allocation failed");
  const int cap = P->g->spec.int_cap();
  const size_t osz = out_kind == ACEDAG_OUT_COMPLEX ? 16 : 8;
  // the pool writes k2_horner's tile-major table itself when that is the
  // kernel and the DMMA pool runs (no k_tile_seeds pass; ACEDAG_POOL_TILED=0
  // keeps the site-major workspace)
  static const bool pool_tiled = !(getenv("ACEDAG_POOL_TILED") && atoi(getenv("ACEDAG_POOL_TILED")) == 0);
  const bool tiled = pool_tiled && P->tri_pruned && (cap == 12 || cap == 14) && !getenv("ACEDAG_POOL") &&
                     pick(P, ACEDAG_METHOD_RECURSIVE, ACEDAG_PREC_F64, out_kind) == K2::Horner;
  if (tiled && W->ws_A.alloc((size_t)((std::min<int64_t>(S, chunk) + 127) / 128) * (U + 1) * 128) != cudaSuccess)
    return fail(ACEDAG_ENOMEM, "workspace allocation failed");
  for (int64_t s0 = 0; s0 < S; s0 += chunk) {
    const int64_t n = std::min(chunk, S - s0);
    int rc = pool_positions_impl(cap, xyz + s0 * J * 3, counts ? counts + s0 : nullptr, n, J, r_in, r_cut,
                                 P->col_of.p, P->tri.p, (int)P->tri.n, U, reinterpret_cast<double*>(W->ws_A.p), st,
                                 P->tri_pruned, tiled ? U + 1 : 0);
    if (rc) return rc;
    t_input_tiled = tiled;
    rc = eval_impl(P, ACEDAG_METHOD_RECURSIVE, ACEDAG_PREC_F64, out_kind, W->ws_A.p, n, U,
                   P->slot_identity.p, static_cast<char*>(out) + s0 * P->host.n_out * osz, st);
    t_input_tiled = false;
    if (rc) return rc;
  }
  return ACEDAG_OK;
}

}  // extern "C"
