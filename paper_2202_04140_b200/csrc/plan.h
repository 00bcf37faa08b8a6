// Host-side compilation of a DAG + coefficients into device programs.
//
// Recursive program (kernel K2).  The reference evaluates every node as the
// product of its two stored parents in id order (evaluator.py:93-110), which
// on a GPU means keeping every intermediate of every site alive (226 KB/site
// at D=12, nu=4).  The plan instead evaluates the SAME set of product nodes
// as a forest in which every node of order o >= 3 is  seed x (a node of order
// o-1): the parent is kept in registers on a depth-first stack, the second
// factor is always a pooled seed read from shared memory.  Nodes whose
// reference parents are both non-seeds ("(2,2)" splits) are re-parented onto
// an (o-1)-subset that is already evaluated; only where none exists is a
// plan-only node added (counted in `extra_nodes`).  Node values therefore
// agree with evaluate_graph to rounding (re-association of a product of
// seeds); the bit-exact path is acedag_eval_nodes.
//
// Naive program (kernel K3): per coefficient node, its seed list, grouped by
// order (naive_eval, evaluator.py:113-121).
#pragma once
#include <cstdint>
#include <vector>

#include "graph.h"

namespace acedag {

// 16-byte program record, read warp-uniformly by K2.
struct alignas(16) Op {
  double c;       // first output's real coefficient (0 if the node carries none)
  uint32_t off;   // byte offset of the seed row in the [slot][32 sites] c128 table
  uint16_t nch;   // number of children that follow in DFS preorder
  uint16_t skip;  // leading children whose seed is TMEM-resident (k2_quad re-encoding);
                  // a root's second record: bit0/bit1 = its two seeds are
};
constexpr uint16_t kSingle = 0xFFFF;
constexpr uint32_t kRowBytes = 32 * 16;  // one slot row: 32 sites x complex128
constexpr uint32_t kTmemRows = 128;        // default hot-slot count of the host program view

struct PlanHost {
  int max_order = 2;                 // deepest order in the recursive program
  std::vector<uint16_t> slot_label;  // seed slot -> label id (seed node id)
  std::vector<Op> ops;               // DFS preorder, chunked per warp
  std::vector<double> cre, cim;      // [n_ops, n_out] coefficients per record
  int n_out = 1;
  bool complex_coef = false;
  int warps = 32;                    // number of work chunks
  std::vector<int32_t> chunk;        // [chunks+1] record offsets
  // naive program: per order o (1..max), records of o slots + coefficient row
  int naive_max_order = 1;
  std::vector<int32_t> naive_seg;    // [max+2] record offsets per order
  std::vector<uint16_t> naive_slots; // records * kMaxOrder (padded)
  std::vector<double> naive_cre, naive_cim;  // [records, n_out]
  // statistics
  int64_t recursive_products = 0, extra_nodes = 0, naive_products = 0;
};

// Throws std::invalid_argument (bad node id) or std::domain_error (non-target;
// message carries the tuple repr).
// hot_rows: seed slots below it are ordered first among a node's children;
// each node's children are ordered with those first and counted in `skip`
void compile_plan(const Graph& g, const int64_t* node_ids, const double* c_re,
                  const double* c_im, int64_t n_coef, int n_out, int warps, PlanHost& out,
                  uint32_t hot_rows = kTmemRows);

std::string node_repr(const Graph& g, int64_t node);

}  // namespace acedag
