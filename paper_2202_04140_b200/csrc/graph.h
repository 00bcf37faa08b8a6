// Host-side DAG representation shared by the builder, the plan compiler and
// the C ABI.  A tuple (multiset of one-particle labels) is stored as its
// ascending seed ids -- label ids are positions in one_particle_indices order
// (indexsets.py:170-191), which is lexicographic label order, so comparing id
// sequences is exactly Python's tuple comparison of label tuples.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace acedag {

constexpr int kMaxOrder = 8;  // tuple key packs 8 x 16-bit ids

struct Tuple {
  uint16_t len = 0;
  uint16_t id[kMaxOrder] = {0};
  bool operator==(const Tuple& o) const {
    if (len != o.len) return false;
    for (int i = 0; i < len; ++i)
      if (id[i] != o.id[i]) return false;
    return true;
  }
  // Python tuple ordering: lexicographic, a proper prefix sorts first.
  bool operator<(const Tuple& o) const {
    int n = len < o.len ? len : o.len;
    for (int i = 0; i < n; ++i)
      if (id[i] != o.id[i]) return id[i] < o.id[i];
    return len < o.len;
  }
  bool operator<=(const Tuple& o) const { return !(o < *this); }
  uint64_t hash() const {
    uint64_t h = 0x9E3779B97F4A7C15ull ^ len;
    for (int i = 0; i < len; ++i) {
      h ^= id[i] + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
      h *= 0xff51afd7ed558ccdull;
    }
    return h ^ (h >> 33);
  }
};

// Open-addressing map Tuple -> int32 id.
class TupleMap {
 public:
  void reserve(size_t n);
  int32_t get(const Tuple& t) const;  // -1 if absent
  void put(const Tuple& t, int32_t v);
  size_t size() const { return n_; }

 private:
  void grow();
  std::vector<Tuple> keys_;
  std::vector<int32_t> vals_;
  size_t n_ = 0, mask_ = 0;
};

struct Label {
  int comp[4];  // components in reference order, unused trailing zero
  int ncomp;
  int degree, m, l;
};

enum Group { kT = 0, kSO2 = 1, kO3 = 2, kO3F = 3 };

struct Spec {
  int p = 1;            // 1, 2, or 0 = inf
  double max_degree = 0;
  int int_cap() const;
  int64_t power_cap() const;
  int64_t power_key(const Tuple& t, const std::vector<Label>& labels) const;
};

std::vector<Label> one_particle_indices(int group, int cap);

struct Graph {
  int group = kO3;
  Spec spec;
  int nu_max = 0;  // 0 = uncapped
  int alg = 0;     // 0 orig, 1 gen
  int n = 1;
  std::vector<Label> labels;      // seeds, ids 0..L-1
  std::vector<Tuple> tuples;      // per node
  std::vector<int32_t> pa, pb;    // parents (-1 for seeds)
  std::vector<uint8_t> aux;
  TupleMap ids;

  int64_t n_seeds() const { return (int64_t)labels.size(); }
  bool satisfies_constraints(const Tuple& t) const;
  bool is_target(const Tuple& t) const;
  int32_t add(const Tuple& t, int32_t a, int32_t b);
  void seed();
  int32_t insert_original(const Tuple& t);
  int32_t insert_generalized(const Tuple& t, int n);
  std::vector<int32_t> target_ids() const;
  std::string serialize() const;
};

// Builds a graph; throws std::invalid_argument with reference messages.
void build_graph(Graph& g, int group, int p, double max_degree, int nu_max, int alg, int n);
// Empty graph (no nodes) with validated spec and its label table.
void init_graph(Graph& g, int group, int p, double max_degree, int nu_max, int alg, int n);
// Rebuild tuples from a parent relation; throws std::invalid_argument.
void graph_from_parents(Graph& g, int group, int p, double max_degree, int nu_max, int alg,
                        int n, int64_t n_nodes, int64_t n_seeds, const int32_t* parents,
                        const uint8_t* aux);

// Graph file reader (graphbuild.py:387-464 format).  On failure returns false
// and fills err: the kind of the first violation (GraphErr), the byte offset
// the reference reports for it and the offending line's byte span (the
// Python shim composes the reference's message from that line).
enum GraphErr {
  kGeOk = 0, kGeNotUtf8, kGeVersion, kGeHeader, kGeDegree, kGeNodeLine, kGeNotDense, kGeAuxFlag,
  kGeElements, kGeParentField, kGeOrphan, kGeParentIds, kGeParentOrder, kGeUnion, kGeSeedAux,
  kGeAuxMismatch, kGeDuplicate, kGeEmpty, kGeSeedLayout, kGeLimit
};
struct GraphParseError {
  int kind = kGeOk;
  int64_t offset = 0;      // byte offset reported with the error
  int64_t line_start = 0;  // span of the offending line (header: line 0)
  int64_t line_len = 0;
  std::string message;     // C-side description (ASCII; the shim rebuilds the reference's text)
};
bool deserialize_graph(const char* data, size_t n, Graph& g, GraphParseError& err);

}  // namespace acedag
