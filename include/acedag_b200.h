/*
 * acedag_b200.h -- C ABI of the B200-native evaluator for the sparse symmetric
 * tensor contraction  phi_s = sum_k c_k prod_t A_{s,k_t}  (arXiv 2202.04140).
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `acedag` (/root/reference/pkg/src/acedag).  Every entry point names the
 * reference interface it replaces (file:line).  Signatures carry plain
 * pointers and sizes only; no torch or Python types cross this boundary.
 *
 * Conventions
 *   - Complex numbers are interleaved (re, im) float64 pairs ("c128") or
 *     float32 pairs ("c64").
 *   - A basis vector A is laid out [S, L] (site-major), labels in
 *     `one_particle_indices` order (indexsets.py:170-191): the seed node ids
 *     0..L-1 of every graph (graphbuild.py:127-130).
 *   - Device pointers are CUDA global-memory pointers on the plan's device;
 *     `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *     stream-ordered and never synchronise the host unless documented.
 *   - Every function returns 0 on success or a negative ACEDAG_E* code; the
 *     message is available from acedag_last_error() (thread-local).
 *   - A plan is immutable after acedag_plan_set_coefficients and may be used
 *     concurrently from several host threads on distinct streams.
 */
#ifndef ACEDAG_B200_H
#define ACEDAG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ACEDAG_ABI_VERSION 1

/* error codes (Python layer maps them onto the reference's exceptions) */
#define ACEDAG_OK 0
#define ACEDAG_EINVAL (-1)        /* bad argument -> ValueError            */
#define ACEDAG_EMISSING_SEED (-2) /* seed value missing -> KeyError         */
#define ACEDAG_ECUDA (-3)         /* CUDA runtime failure -> RuntimeError   */
#define ACEDAG_ENOMEM (-4)        /* allocation failure -> MemoryError      */
#define ACEDAG_ENOTTARGET (-5)    /* coefficient on non-target -> ValueError*/
#define ACEDAG_EDOMAIN (-6)       /* coordinate out of domain -> ValueError */
#define ACEDAG_EUNSUPPORTED (-7)  /* shape outside the compiled limits      */
#define ACEDAG_EFORMAT (-8)       /* malformed graph file -> GraphFormatError */

/* graph-file violation kinds (acedag_graph_deserialize), in the order the
 * reference checks them (graphbuild.py:387-464) */
#define ACEDAG_GE_NOT_UTF8 1
#define ACEDAG_GE_VERSION 2
#define ACEDAG_GE_HEADER 3
#define ACEDAG_GE_DEGREE 4
#define ACEDAG_GE_NODE_LINE 5
#define ACEDAG_GE_NOT_DENSE 6
#define ACEDAG_GE_AUX_FLAG 7
#define ACEDAG_GE_ELEMENTS 8
#define ACEDAG_GE_PARENT_FIELD 9
#define ACEDAG_GE_ORPHAN 10
#define ACEDAG_GE_PARENT_IDS 11
#define ACEDAG_GE_PARENT_ORDER 12
#define ACEDAG_GE_UNION 13
#define ACEDAG_GE_SEED_AUX 14
#define ACEDAG_GE_AUX_MISMATCH 15
#define ACEDAG_GE_DUPLICATE 16
#define ACEDAG_GE_EMPTY 17
#define ACEDAG_GE_SEED_LAYOUT 18 /* this build: seeds first, in label order */
#define ACEDAG_GE_LIMIT 19       /* this build: order <= 8, label count     */

/* symmetry groups (indexsets.py:37-52) */
#define ACEDAG_GROUP_T 0
#define ACEDAG_GROUP_SO2 1
#define ACEDAG_GROUP_O3 2
#define ACEDAG_GROUP_O3F 3

/* degree norm p (indexsets.py:109-146); 0 encodes p = inf */
#define ACEDAG_P_INF 0

/* evaluation methods for acedag_eval */
#define ACEDAG_METHOD_RECURSIVE 0 /* K2: DAG evaluation (evaluate_graph + c-dot) */
#define ACEDAG_METHOD_NAIVE 1     /* K3: naive product basis (naive_eval + c-dot) */

/* output kinds for acedag_eval */
#define ACEDAG_OUT_REAL 0    /* Re(phi)  : out is float64 [S, n_out]          */
#define ACEDAG_OUT_COMPLEX 1 /* phi      : out is c128    [S, n_out]          */

/* precision of the DAG arithmetic */
#define ACEDAG_PREC_F64 0 /* complex128 nodes                                 */
#define ACEDAG_PREC_F32 1 /* complex64 nodes, float64 accumulation of phi     */

typedef struct acedag_graph acedag_graph;
typedef struct acedag_plan acedag_plan;

int acedag_abi_version(void);
const char* acedag_last_error(void);

/* ------------------------------------------------------------------------
 * Host DAG (graphbuild.py:76-268).  Built natively (C++) with the exact
 * insertion rules of the reference, so serialize() is byte-identical to
 * `serialize_graph(build_graph(...))` (graphbuild.py:374-384).
 * ---------------------------------------------------------------------- */

/* replaces build_graph (graphbuild.py:243-268); alg 0 = "orig", 1 = "gen" */
int acedag_graph_build(int group, int p, double max_degree, int nu_max, int alg,
                       int n, acedag_graph** out);
/* wraps an externally built DAG (e.g. a reference EvalGraph flattened on the
 * host): parents[2*i], parents[2*i+1] are the parent ids of node i, or -1/-1
 * for the n_seeds order-1 nodes, which must be ids 0..n_seeds-1; aux[i] is
 * the auxiliary flag.  Tuples are rebuilt from the parent relation. */
int acedag_graph_from_parents(int group, int p, double max_degree, int nu_max,
                              int alg, int n, int64_t n_nodes, int64_t n_seeds,
                              const int32_t* parents, const uint8_t* aux,
                              acedag_graph** out);
void acedag_graph_destroy(acedag_graph* g);
/* sizes: nodes, seeds (labels L), targets, auxiliaries, max order */
int acedag_graph_info(const acedag_graph* g, int64_t* n_nodes, int64_t* n_seeds,
                      int64_t* n_targets, int64_t* n_aux, int32_t* max_order);
/* SoA export. parents [2*n_nodes] (seed rows -1), aux [n_nodes],
 * order [n_nodes], target_ids [n_targets] ascending (evaluator.py:214) */
int acedag_graph_arrays(const acedag_graph* g, int32_t* parents, uint8_t* aux,
                        int32_t* order, int32_t* target_ids);
/* tuple of node i as seed ids (length = order), ascending */
int acedag_graph_node_seeds(const acedag_graph* g, int64_t node, int32_t* seeds_out,
                            int32_t capacity);
/* node id of a tuple given as ascending seed ids, or -1 (graphbuild.py:116) */
int64_t acedag_graph_find(const acedag_graph* g, const int32_t* seeds, int32_t len);
/* serialize_graph (graphbuild.py:374-384).  Call with buf=NULL to get the
 * size in *len; then with a buffer of that size. */
int acedag_graph_serialize(const acedag_graph* g, char* buf, int64_t* len);
/* deserialize_graph (graphbuild.py:387-464): parses the versioned text
 * format natively.  On a malformed file returns ACEDAG_EFORMAT with the
 * violation kind in *err_kind (ACEDAG_GE_*), the byte offset the reference
 * reports in *err_offset and the offending line's byte span in
 * *err_line_start / *err_line_len (NULL pointers are allowed). */
int acedag_graph_deserialize(const char* data, int64_t len, acedag_graph** out,
                             int32_t* err_kind, int64_t* err_offset,
                             int64_t* err_line_start, int64_t* err_line_len);
/* the header fields of a graph (group, p (0 = inf), D, numax (0 = uncapped),
 * alg (0 orig, 1 gen), n) -- what EvalGraph carries (graphbuild.py:76-93) */
int acedag_graph_spec(const acedag_graph* g, int32_t* group, int32_t* p, double* max_degree,
                      int32_t* nu_max, int32_t* alg, int32_t* n);

/* ------------------------------------------------------------------------
 * Device plan: the DAG compiled into a per-warp evaluation program, resident
 * in HBM, plus coefficients.  Replaces the per-call Python object walk of
 * evaluate_graph / evaluate_model (evaluator.py:93-142).
 * ---------------------------------------------------------------------- */
int acedag_plan_create(const acedag_graph* g, int device, acedag_plan** out);
void acedag_plan_destroy(acedag_plan* plan);
/* Coefficients (evaluate_model's dict, evaluator.py:124-139): n_coef node ids
 * and values [n_coef, n_out] (c_im may be NULL for real coefficients).
 * ENOTTARGET if a node id is not a target (message names the id).  Builds
 * the device programs; synchronous. */
int acedag_plan_set_coefficients(acedag_plan* plan, const int64_t* node_ids,
                                 const double* c_re, const double* c_im,
                                 int64_t n_coef, int32_t n_out);
/* statistics of the compiled programs: products executed per site by the
 * recursive program, extra (plan-only) nodes, naive multiplications per
 * site, seeds referenced. */
int acedag_plan_info(const acedag_plan* plan, int64_t* recursive_products,
                     int64_t* extra_nodes, int64_t* naive_products,
                     int64_t* used_seeds);

/* Host-only view of the compiled recursive program (no device needed; used
 * by tests and tooling).  Two-call pattern: pass NULL buffers to get
 * *n_slots / *n_ops, then buffers of that size.  ops receives 16-byte records
 * {double c; uint32 seed-row byte offset (slot * 512); uint16 n_children;
 * uint16 hot children} in DFS preorder, a root as two records; chunk
 * receives warps+1 record offsets; stats = {recursive_products,
 * extra_nodes, naive_products}. */
int acedag_plan_program(const acedag_graph* g, const int64_t* node_ids,
                        const double* c_re, const double* c_im, int64_t n_coef,
                        int32_t n_out, int32_t warps, uint16_t* slot_label,
                        int64_t* n_slots, void* ops, int64_t* n_ops,
                        int32_t* chunk, int64_t* stats);

/* Host-only view of the k2_horner program (tests and tooling; replaces no
 * reference function -- it is the device form of evaluator.py:93-142's
 * work): the recursive program above re-encoded with `hot` TMEM rows and
 * `us` shared-memory rows (csrc/horner.h: 16-byte records {double c; uint32
 * z; uint32 w}, children ordered hot / shared / global with their counts in
 * w), real coefficients, one output.  *n_ops = records of one copy; ops
 * receives the four TMEM-lane-quadrant copies (4 * *n_ops records), chunk
 * warps+1 offsets into copy 0, croots the roots per chunk.  Two-call
 * pattern as acedag_plan_program. */
int acedag_plan_program_horner(const acedag_graph* g, const int64_t* node_ids,
                               const double* c_re, int64_t n_coef, int32_t warps,
                               int32_t hot, int32_t us, void* ops, int64_t* n_ops,
                               int32_t* chunk, int32_t* croots);

/* Kernels launched by this library since load (all plans and devices). */
int64_t acedag_launch_count(void);

/* Per-phase device timing of the evaluations on this plan (CUDA events on
 * the launching stream): enable (1) / disable (0); both clear the record.
 * _read synchronizes on the recorded events and returns the summed
 * milliseconds of {seed preparation (tile-major copy), main K2 kernel,
 * remainder (split-tail reduction)} and the number of evaluations, then
 * clears the record. */
int acedag_plan_timing(acedag_plan* plan, int enable);
int acedag_plan_timing_read(acedag_plan* plan, double* ms3, int64_t* calls);

/* Name of the kernel acedag_eval would launch for these arguments and S
 * sites (static string; "" and EINVAL on bad arguments).  For reporting. */
const char* acedag_eval_kernel_name(const acedag_plan* plan, int method, int prec,
                                    int out_kind, int64_t S);

/* phi for S sites: replaces evaluate_graph + sum(c * v) (evaluator.py:93-110,
 * 141-142) [method RECURSIVE] or sum(c * naive_eval) (evaluator.py:113-121)
 * [method NAIVE].  A: device c128 [S, L] (prec F64) or c64 (prec F32).
 * out: device float64 [S, n_out] (OUT_REAL) or c128 [S, n_out]. */
int acedag_eval(const acedag_plan* plan, int method, int prec, int out_kind,
                const void* A, int64_t S, void* out, void* stream);

/* acedag_eval on HOST buffers, end to end (evaluate_model's host-side call,
 * evaluator.py:124-142, for S sites at once).  A_host: c128 (F64) / c64 (F32)
 * [S, L]; out_host: as acedag_eval's out.  Page-locked A_host is read in
 * place over PCIe by a gather kernel that fetches only the seed columns the
 * plan uses, pipelined with the evaluation kernels; pageable A_host is copied
 * in row chunks.  Ordered after prior work on `stream`; synchronous (returns
 * with out_host written).  *h2d_bytes (may be NULL) receives the input bytes
 * moved host->device. */
int acedag_eval_host(const acedag_plan* plan, int method, int prec, int out_kind,
                     const void* A_host, int64_t S, void* out_host, int64_t* h2d_bytes,
                     void* stream);

/* Batched naive_eval (evaluator.py:113-121): out[r] = prod_t vals[r, t],
 * left to right from 1+0j with separate roundings (bit-identical).  vals:
 * device c128 [n_rows, width]; lens: device int32 [n_rows] (NULL = width). */
int acedag_naive_products(const double* vals, const int32_t* lens, int64_t n_rows,
                          int32_t width, double* out, void* stream);

/* Site total: out_total[o] += sum_s phi[s, o] for OUT_REAL (device float64
 * [n_out]); used by the sharded energy allreduce. */
int acedag_reduce_sites(const acedag_plan* plan, const double* phi, int64_t S,
                        double* out_total, void* stream);

/* Every node value, bit-identical to evaluate_graph (evaluator.py:93-110):
 * products with separate roundings (no FMA) in node-id order.
 * A: device c128 [S, L]; node_vals: device c128 [S, N]. */
int acedag_eval_nodes(const acedag_plan* plan, const double* A, int64_t S,
                      double* node_vals, void* stream);

/* ------------------------------------------------------------------------
 * Atomic basis (pool): replaces pool / one_particle (evaluator.py:61-90).
 * ---------------------------------------------------------------------- */

/* Reference convention: coords device float64 [S, J, ncoord(group)]
 * ((theta) | (r, theta) | (r, theta, phi) | (r, theta, phi, mu)), counts
 * device int32 [S] (NULL = all J).  A_out: device c128 [S, L] with
 * L = |one_particle_indices(group, cap)|.  Domain checks are the caller's
 * (acedag_check_coords). */
int acedag_pool(int group, int cap, const double* coords, const int32_t* counts,
                int64_t S, int32_t J, double* A_out, void* stream);
/* host-side domain check of reference coordinates (evaluator.py:46-58):
 * returns EDOMAIN with the message of the reference on the first bad row. */
int acedag_check_coords(int group, const double* coords_host, int64_t n_particles);

/* Positions convention (BASELINE cfg3/cfg5): xyz device float64 [S, J, 3]
 * Cartesian neighbour vectors, counts int32 [S] or NULL.  Each neighbour
 * contributes f_c(r) * T_n(2x-1) * Y_lm(r_hat) with x = (r - r_in)/(r_cut - r_in)
 * clamped to [0,1] and f_c(r) = (1 + cos(pi r / r_cut))/2 for r < r_cut. */
int acedag_pool_positions(int cap, const double* xyz, const int32_t* counts,
                          int64_t S, int32_t J, double r_in, double r_cut,
                          double* A_out, void* stream);

/* fused pool_positions + eval (RECURSIVE, F64, OUT_REAL or OUT_COMPLEX);
 * uses a plan-owned workspace for A (not re-entrant across streams). */
int acedag_eval_from_positions(acedag_plan* plan, const double* xyz,
                               const int32_t* counts, int64_t S, int32_t J,
                               double r_in, double r_cut, int out_kind,
                               void* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ACEDAG_B200_H */
