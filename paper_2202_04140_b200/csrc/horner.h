// K2 Horner kernel (k2_horner): host-side encoding and launcher.
//
// The recursive program of plan.h evaluated bottom-up.  For a plan node u
// with value V_u (product of the seeds on its path) define
//     H_u = c_u + sum_{children q} s_q * H_q        (s_q: the child's seed)
// so that sum_{w in subtree(u)} c_w V_w = V_u * H_u and
//     phi = sum_roots Re(s_a * s_b * H_root).
// A leaf costs one complex FMA of a real coefficient (2 DFMA per site)
// instead of a product and a dot (3 DP instructions); an inner node one
// complex multiply-add (4 DFMA) instead of 5.  Node values are never formed;
// the node set and coefficients are exactly those of the plan, so the result
// equals evaluate_model's to rounding (evaluator.py:124-142).
#pragma once
#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#include "plan.h"

namespace acedag {

// 16-byte record, read warp-uniformly.  c: the coefficient (fp32 programs:
// a float in the low word).  z: the seed's class-scaled offset (TMEM row ->
// column row*16 (c128) or row*8 (c64) plus the lane-quadrant bits; shared /
// global row -> byte row*2048 (c128) or row*1024 (c64)).  w: nch | nhot << 15
// | nsm << 22 (children by class, in that order).  A root is two records; the second carries w = cls_a | cls_b << 2 |
// single << 4 (single: an order-1 coefficient, phi += c Re(s_a)).
// Order-4 programs (round 2): a root's order-3 children are sorted, inside
// each seed class, into S1 (one leaf, hot), S2 (two leaves, both hot) and the
// rest, and the root carries the run lengths instead of the class counts:
// r0.w = general runs (hot | shared << 10 | global << 20); second record:
// c bits = S1 | S2 << 16 of the hot (low word) and shared (high word)
// classes, w |= S1 << 8 | S2 << 20 of the global class.
struct alignas(16) OpH {
  double c;
  uint32_t z;
  uint32_t w;
};

constexpr uint32_t kHornerHot = 32;      // TMEM rows (4 sites x c128 = 16 columns each; c64: 64 rows)
inline int horner_hot_rows(bool f32) { return f32 ? 64 : (int)kHornerHot; }
inline int horner_row_bytes(bool f32) { return f32 ? 1024 : 2048; }
constexpr int kHornerWarps = 24;         // fp64, order <= 4 (16 above; fp32: horner_warps())
constexpr uint32_t kHornerRing = 2048;   // per-warp program ring: 3 blocks + mirror
// leaves per record group: a node of the last inner order with more is split
// into copies of the same seed (the first carrying its coefficient), so a
// node and its leaves always fit the 32-record ring window
constexpr uint32_t kMaxLeaves = 30;

// Re-encodes the plan's DFS program for k2_horner with `hot` TMEM rows and
// `us` shared-memory rows (slot order: hot, shared, global), chunked like the
// plan: chunk gets each chunk's first record, croots its number of roots.
// out holds four copies of the program (one per TMEM lane quadrant: hot
// records' z carries the quadrant's lane bits), chunk offsets index copy 0.
// Returns false when a count does not fit its field (another kernel is used).
// Programs deeper than order 4 are emitted once (the kernel adds the quadrant
// bits per fetch) unless four_copies asks for the four-copy view (host inspection).
bool encode_horner(const PlanHost& H, bool f32, uint32_t hot, uint32_t us, std::vector<OpH>& out,
                   std::vector<int32_t>& chunk, std::vector<int32_t>& croots, bool four_copies = false);

// shared-memory rows k2_horner can hold besides its rings
int horner_us_max(size_t smem_optin, bool f32, int nu);
size_t horner_smem(int us, bool f32, int nu);

// tiles: tile-major seed table [ntiles][U+1][128] c128 / c64 (k_tile_seeds<128>).
// part: [grid][2][nchunk][128]; tail: [(ntiles - full)][nchunk][128].
cudaError_t launch_horner(int nu, bool f32, const void* tiles, int64_t S, int U, int us, const OpH* ops,
                          const int32_t* chunk, const int32_t* croots, int nchunk, double* out, double* part,
                          int64_t full, int parts, double* tail, int grid, cudaStream_t st);

}  // namespace acedag
