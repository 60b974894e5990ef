/*
 * hpeel_b200 C ABI: the drop-in boundary of the B200 H1 peeling core.
 *
 * Each entry point replaces one reference interface that a binding of the
 * H1 hot path calls (reference pybind module proj/bindings/module.cpp:97-230
 * over the C++ API in proj/include/hpeel/). Plain pointers and sizes only;
 * matrices are column-major FP64 (Eigen::MatrixXd layout,
 * proj/include/hpeel/rng.hpp:9) in the caller's point (input) order.
 *
 * Every function returning int returns HP_OK or an error code; the message is
 * in hp_last_error() (thread-local). Codes map to the reference's exception
 * types: std::invalid_argument, std::runtime_error, std::logic_error.
 */
#ifndef HPEEL_B200_H
#define HPEEL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HP_OK 0
#define HP_ERR_INVALID_ARGUMENT 1
#define HP_ERR_RUNTIME 2
#define HP_ERR_LOGIC 3

/* sample modes (proj/include/hpeel/coloring.hpp:21-26) */
#define HP_MODE_H1 0
#define HP_MODE_UNIF_STAGE1 1
#define HP_MODE_UNIF_STAGE2 2
#define HP_MODE_LEAF 3

/* black-box kinds: dense = DenseOperator (proj/include/hpeel/operators.hpp:56-69);
 * the kernel kinds are the on-the-fly BASELINE.json operators */
#define HP_OP_DENSE 0
#define HP_OP_LOG 1          /* log|x - y|, A_ii = 0 */
#define HP_OP_INVDIST_4PI 2  /* 1 / (4 pi |x - y|), A_ii = 0 */
#define HP_OP_EXP 3          /* exp(-|x - y| / param) */

/* formats / strategies (proj/include/hpeel/peeling.hpp:15-25) */
#define HP_FORMAT_H1 0
#define HP_FORMAT_UNIF_H1 1
#define HP_FORMAT_H1_PLUS_UNIF 2
#define HP_FORMAT_H2 3
#define HP_STRATEGY_GRAPH 0
#define HP_STRATEGY_FALLBACK_PATTERN 1

typedef struct hp_tree hp_tree;
typedef struct hp_plan hp_plan;
typedef struct hp_op hp_op;
typedef struct hp_rep hp_rep;

const char* hp_last_error(void);
int hp_device_count(int* count);
/* kernels launched by this library so far (bench.py gpu_launches) */
int64_t hp_launch_count(void);
int hp_device_synchronize(void);

/* ---- RNG: proj/include/hpeel/rng.hpp:37-50, proj/src/rng.cpp:31-59 ---- */
uint64_t hp_mix_seed(uint64_t seed, uint64_t tag);
/* rows x cols standard normal (gaussian_matrix), written column-major */
int hp_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out);
/* random_cloud (proj/src/operators.cpp:88-95): n x dim column-major */
int hp_random_cloud(int64_t n, int dim, uint64_t seed, double* out);

/* ---- Tree: PointCloud::from_raw + BoxTree::build + adjacency
 *      (proj/src/box_tree.cpp:55-70, :99-180, :214-300;
 *       binding build_tree proj/bindings/module.cpp:19-26) ---- */
int hp_tree_build(const double* raw, int64_t n, int dim, int leaf_capacity, hp_tree** out);
void hp_tree_free(hp_tree* tree);
/* info[0..7] = n, dim, depth, num_boxes, max_leaf_size, fully_populated,
 * leaf_capacity, sum of box point counts */
int hp_tree_info(const hp_tree* tree, int64_t* info);
/* per box: level, parent, coord (num_boxes x dim row-major), point lists in
 * CSR (pt_off has num_boxes + 1 entries); any output may be NULL */
int hp_tree_boxes(const hp_tree* tree, int* level, int* parent, int64_t* coord, int64_t* pt_off,
                  int* pts);
/* which: 0 neighbors, 1 interaction, 2 coarse_leaf_neighbors, 3 dense_partners,
 * 4 children (AdjacencyInfo, proj/include/hpeel/box_tree.hpp:91-104); CSR,
 * items may be NULL to query off[num_boxes] */
int hp_tree_lists(const hp_tree* tree, int which, int64_t* off, int* items);
int64_t hp_tree_cross_level_adjacencies(const hp_tree* tree);
/* admissible_pairs(level) (box_tree.cpp:302-313) or dense_pairs (level < 0,
 * :315-323); pairs may be NULL to query *count */
int hp_tree_pairs(const hp_tree* tree, int level, int64_t* count, int* pairs);
/* device layout: tree position -> input index, per-box [start, start+count) */
int hp_tree_layout(const hp_tree* tree, int* perm, int64_t* start, int64_t* count);

/* ---- Sampling plan: build_constraints / build_graph / plan_coloring /
 *      assemble_test_matrices / make_plan (proj/src/coloring.cpp:55-332,
 *      proj/src/peeling.cpp:98-154; binding level_coloring module.cpp:190-205).
 *      pairwise_graph: 0 inverted-index graph, 1 literal pairwise scan,
 *      2 implicit graph (no edge lists; the path compress() uses for
 *      single-payload sets), 3 the fallback-pattern strategy
 *      (fallback_pattern_matrices, proj/src/coloring.cpp:334-407: no sets,
 *      graph or coloring; matrices + hp_plan_block_map only) */
int hp_plan_build(const hp_tree* tree, int level, int mode, int width, uint64_t seed, int phase,
                  int pairwise_graph, hp_plan** out);
void hp_plan_free(hp_plan* plan);
/* info[0..7] = n_vertices, n_edges, n_colors, dsatur queue_ops, payload
 * entries, zero entries, owner entries, sum of color payload lists */
int hp_plan_info(const hp_plan* plan, int64_t* info);
int hp_plan_sets(const hp_plan* plan, int64_t* pay_off, int* pay_box, int* pay_tag,
                 int64_t* zero_off, int* zero, int64_t* own_off, int* owners);
int hp_plan_graph(const hp_plan* plan, int64_t* off, int* adj);
/* color per vertex (plan_coloring) and the pure DSatur coloring */
int hp_plan_coloring(const hp_plan* plan, int* color, int* dsatur_color, int* dsatur_colors);
/* per color: payload boxes (CSR) */
int hp_plan_matrices(const hp_plan* plan, int64_t* off, int* boxes);
/* fallback-pattern plans: block_to_matrix as (alpha, beta, matrix) triples
 * (beta = -1 for the uniform stage-1 boxes); triples may be NULL to count */
int hp_plan_block_map(const hp_plan* plan, int64_t* count, int* triples);
/* dense realization of one color (BlockTestMatrix::realize), n x width */
int hp_plan_realize(const hp_plan* plan, int color, double* out);
/* DSatur on an explicit graph (CSR) */
int hp_dsatur(int nv, const int64_t* off, const int* adj, int* color, int* num_colors,
              int64_t* queue_ops);

/* ---- Black boxes: LinearOperator (proj/include/hpeel/linear_operator.hpp:12-24) ---- */
int hp_op_dense(const double* a, int64_t n, int device, hp_op** out);
/* points: raw coordinates, n x dim column-major, input order */
int hp_op_kernel(int kind, const double* points, int64_t n, int dim, double param, int device,
                 hp_op** out);
/* Caller-supplied black box: the reference's virtual LinearOperator::apply /
 * apply_adjoint (proj/include/hpeel/linear_operator.hpp:19-20), called once
 * per color and side as residual_samples does (proj/src/peeling.cpp:165-177)
 * and once per color of the leaf probes (:490-524). fn computes
 * y = A x (adjoint = 0) or A^T x (adjoint = 1) for an n x w column-major x in
 * the caller's point order and returns 0 (nonzero = failure: compress fails
 * with HP_ERR_RUNTIME). device_pointers = 0: x and y are host arrays and
 * stream is NULL; 1: they are device pointers on `device` and the work must be
 * ordered on `stream` (a cudaStream_t). ctx is passed through. */
typedef int (*hp_apply_fn)(void* ctx, int adjoint, const double* x, int64_t w, double* y, void* stream);
int hp_op_callback(int64_t n, int symmetric, int device_pointers, hp_apply_fn fn, void* ctx, int device,
                   hp_op** out);
void hp_op_free(hp_op* op);
int hp_op_apply(const hp_op* op, int adjoint, const double* x, int64_t w, double* y);

/* ---- compress (proj/include/hpeel/peeling.hpp:66-68, binding compress_py
 *      module.cpp:65-93). format must be HP_FORMAT_H1; strategy
 *      HP_STRATEGY_GRAPH or HP_STRATEGY_FALLBACK_PATTERN (fully populated
 *      trees only, as in the reference); capture != 0 keeps the post-peel
 *      sample blocks for parity tests. ---- */
int hp_compress(const hp_op* op, const hp_tree* tree, int rank, int oversample, uint64_t seed,
                int format, int strategy, int capture, hp_rep** out);
void hp_rep_free(hp_rep* rep);

/* ---- multi-GPU (one process per GPU, owner-computes): NCCL
 *      communicator. Rank 0 calls hp_comm_unique_id and distributes the 128
 *      bytes. Each rank's representation holds the factors of the pairs that
 *      touch its boxes and the dense blocks of its leaves. ---- */
typedef struct hp_comm hp_comm;
int hp_comm_unique_id(unsigned char* id128);
int hp_comm_create(const unsigned char* id128, int rank, int world, int device, hp_comm** out);
void hp_comm_free(hp_comm* comm);
/* compress on this rank of `comm` (NULL: single GPU) */
int hp_compress_ex(const hp_op* op, const hp_tree* tree, int rank, int oversample, uint64_t seed,
                   int format, int strategy, int capture, hp_comm* comm, hp_rep** out);
/* compress on `world` ranks emulated by threads of this process on the
 * operator's device (the same sharded path, device copies instead of NCCL);
 * outs[g] = rank g's representation */
int hp_compress_group(const hp_op* op, const hp_tree* tree, int rank, int oversample, uint64_t seed,
                      int format, int strategy, int capture, int world, hp_rep** outs);
/* box ownership for `world` ranks: owner per box (-1 above the cut), the cut
 * level (levels below it are replicated) and the world + 1 tree-position
 * bounds of the ranks' point ranges; any output may be NULL */
int hp_shard_owners(const hp_tree* tree, int world, int* owner, int* cut, int64_t* point_bounds);
/* per-rank device memory plan in bytes: out[g * 4 + 0..3] = factors held,
 * dense blocks, largest level's samples + apply buffers, total estimate */
int hp_shard_memory_plan(const hp_tree* tree, int rank, int oversample, int world, double* out);
/* doubles shard `shard` sends to / receives from each of the `world` ranks
 * (send[world], recv[world]) in level `level`'s crossing-pair exchange
 * `phase` (1: V to the row owner, 2: U and B to the column owner) */
int hp_shard_exchange_counts(const hp_tree* tree, int rank, int world, int shard, int level, int phase,
                             int64_t* send, int64_t* recv);
/* hp_export_sizes for shard `shard` of `world` */
int hp_export_sizes_shard(const hp_tree* tree, int rank, int world, int shard, int64_t* factor_doubles,
                          int64_t* dense_doubles);
/* world and rank of a representation; *held = whether it holds block `pair`
 * of `level` (level < 0: dense block `pair`); outputs may be NULL */
int hp_rep_shard(const hp_rep* rep, int level, int64_t pair, int* world, int* shard, int* held);
/* the work partition every rank computes: world + 1 boundaries */
int hp_partition_ranges(const double* work, int64_t n, int world, int64_t* bounds);
/* totals[0..8] = forward_cols, adjoint_cols, max_sampling_colors,
 * wall_s_total, wall_s_net, net_flops, setup_ms, peak device bytes of this
 * compress, bytes this rank sent in sharded exchanges; *nphases = phase count */
int hp_rep_report(const hp_rep* rep, double* totals, int64_t* nphases);
/* per phase: ints[7] = is_leaf, level, colors, forward_cols, adjoint_cols, net_flops,
 * apply_path (K2: 0 FP64 DMMA, 1 int8 tensor cores) and
 * times[13] = wall_ms_total, wall_ms_net, apply_ms, peel_ms, qr_ms, bsolve_ms,
 * apply_flops, kernel_evals, host_wait_ms, start_ms (device time from the
 * first device work of compress to the phase start), peel_flops (K3),
 * qr_flops (K4, 2 m r^2 per U / V block), bsolve_flops (K5, the reference's
 * B-solve flop formulas) */
int hp_rep_phase(const hp_rep* rep, int64_t phase, int64_t* ints, double* times);
/* RunReport::to_csv (proj/src/peeling.cpp:478-488) */
int hp_rep_csv(const hp_rep* rep, char* buf, int64_t cap, int64_t* len);
int hp_rep_num_pairs(const hp_rep* rep, int level, int64_t* count);
/* block (alpha, beta) = pairs[pair] of `level`: ranks, then U (|I_a| x ku),
 * B (ku x kv), V (|I_b| x kv), rows in box.points order; outputs may be NULL */
int hp_rep_block(const hp_rep* rep, int level, int64_t pair, int* ku, int* kv, double* u,
                 double* b, double* v);
/* dense block of dense_pairs()[pair], |I_lam| x |I_mu| */
int hp_rep_dense_block(const hp_rep* rep, int64_t pair, double* d);
int hp_rep_apply(const hp_rep* rep, int adjoint, const double* x, int64_t w, double* y);
int hp_rep_storage(const hp_rep* rep, int64_t* total);
int hp_rep_sizes(const hp_rep* rep, int64_t* factor_doubles, int64_t* dense_doubles);
/* bulk device->host copy of all factors and dense blocks (internal layout) */
int hp_rep_export(const hp_rep* rep, double* host_factors, double* host_dense, int64_t* bytes);
/* sizes (doubles) of the host arrays hp_rep_export / hp_compress_export fill */
int hp_export_sizes(const hp_tree* tree, int rank, int64_t* factor_doubles, int64_t* dense_doubles);
/* pinned host memory (cudaHostAlloc) for the export arrays; hp_host_free releases it */
int hp_host_alloc(int64_t bytes, void** out);
void hp_host_free(void* p);
/* compress (as hp_compress_ex) with a streamed export: each level's factors
 * and then the dense leaf blocks are copied into host_factors / host_dense
 * (hp_rep_export layout) on a second stream as soon as they are final, so
 * with pinned arrays the device->host transfer overlaps the later levels.
 * Returns when the export is complete. Replaces compress() followed by a
 * host copy of the H1Rep (proj/include/hpeel/peeling.hpp:66-68). */
int hp_compress_export(const hp_op* op, const hp_tree* tree, int rank, int oversample, uint64_t seed,
                       int format, int strategy, hp_comm* comm, double* host_factors,
                       int64_t factor_doubles, double* host_dense, int64_t dense_doubles,
                       hp_rep** out);
/* .hrep files in the reference's format (save_rep / load_rep,
 * proj/include/hpeel/hmatrix.hpp:150-152, proj/src/serialize.cpp:156-250);
 * H1 only. hp_rep_load returns the representation and its embedded tree. */
int hp_rep_save(const hp_rep* rep, const char* path);
int hp_rep_load(const char* path, int device, hp_rep** out, hp_tree** tree_out);
/* save_dense_matrix / load_dense_matrix (hmatrix.hpp:155-156): "HPEELDM1"
 * files; load with out == NULL returns the shape only */
int hp_save_dense_matrix(const char* path, const double* a, int64_t rows, int64_t cols);
int hp_load_dense_matrix(const char* path, int64_t* rows, int64_t* cols, double* out, int64_t cap);
/* captured post-peel samples of pair `pair` at `level` (level < 0: leaf
 * probe block of dense pair `pair`): rows of the row box in box.points
 * order x (2r | leaf width) columns */
int hp_rep_captured(const hp_rep* rep, int level, int64_t pair, int64_t* rows, int64_t* cols,
                    double* out);
/* the same block of an H1 level before the peeling subtraction: the rows of
 * A Omega (resp. A^T Psi) the extraction reads */
int hp_rep_captured_raw(const hp_rep* rep, int level, int64_t pair, int64_t* rows, int64_t* cols,
                        double* out);
/* rel_error_power_method (proj/src/linalg.cpp:206-218; binding module.cpp:219-229) */
int hp_rel_error_power_method(const hp_rep* rep, const hp_op* op, int iters, uint64_t seed,
                              double* out);

#ifdef __cplusplus
}
#endif

#endif /* HPEEL_B200_H */
