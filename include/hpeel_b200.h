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
/* profiling only: 1 = K2 skips kernel evaluation, 2 = K2 skips DMMA, 0 = normal */
void hp_debug_set_k2_mode(int mode);
/* K2 arithmetic path: 0 = int8 tensor-core digit products (exact fixed-point
 * emulation of the FP64 contraction, k2_i8.cuh) wherever eligible (default),
 * 1 = FP64 DMMA for every apply (A/B tests) */
void hp_debug_set_k2_path(int path);
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
 *      single-payload sets) */
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
void hp_op_free(hp_op* op);
int hp_op_apply(const hp_op* op, int adjoint, const double* x, int64_t w, double* y);

/* ---- compress (proj/include/hpeel/peeling.hpp:66-68, binding compress_py
 *      module.cpp:65-93). format must be HP_FORMAT_H1 and strategy
 *      HP_STRATEGY_GRAPH (the hot path); capture != 0 keeps the post-peel
 *      sample blocks for parity tests. ---- */
int hp_compress(const hp_op* op, const hp_tree* tree, int rank, int oversample, uint64_t seed,
                int format, int strategy, int capture, hp_rep** out);
void hp_rep_free(hp_rep* rep);

/* ---- multi-GPU (one process per GPU): NCCL communicator.
 *      Rank 0 calls hp_comm_unique_id and distributes the 128 bytes. ---- */
typedef struct hp_comm hp_comm;
int hp_comm_unique_id(unsigned char* id128);
int hp_comm_create(const unsigned char* id128, int rank, int world, int device, hp_comm** out);
void hp_comm_free(hp_comm* comm);
/* compress with the black-box apply and leaf probes sharded over `comm`
 * (NULL: single GPU); emulate_shards > 1 splits the launches as that many
 * ranks would, in this process (tests) */
int hp_compress_ex(const hp_op* op, const hp_tree* tree, int rank, int oversample, uint64_t seed,
                   int format, int strategy, int capture, hp_comm* comm, int emulate_shards,
                   hp_rep** out);
/* the work partition every rank computes: world + 1 boundaries */
int hp_partition_ranges(const double* work, int64_t n, int world, int64_t* bounds);
/* totals[0..6] = forward_cols, adjoint_cols, max_sampling_colors,
 * wall_s_total, wall_s_net, net_flops, setup_ms; *nphases = phase count */
int hp_rep_report(const hp_rep* rep, double* totals, int64_t* nphases);
/* per phase: ints[7] = is_leaf, level, colors, forward_cols, adjoint_cols, net_flops,
 * apply_path (K2: 0 FP64 DMMA, 1 int8 tensor cores) and
 * times[12] = wall_ms_total, wall_ms_net, apply_ms, peel_ms, qr_ms, bsolve_ms,
 * apply_flops, kernel_evals, host_wait_ms, start_ms (device time from the
 * first device work of compress to the phase start), peel_flops (K3),
 * qr_flops (K4, 2 m r^2 per U / V block) */
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
/* rel_error_power_method (proj/src/linalg.cpp:206-218; binding module.cpp:219-229) */
int hp_rel_error_power_method(const hp_rep* rep, const hp_op* op, int iters, uint64_t seed,
                              double* out);

/* ---- K1 parity probe: payload rows of every level-`level` box for width r,
 *      both phases, on the device; out = n x 2r column-major in input order
 *      (columns [0, r) phase 0, [r, 2r) phase 1; rows not in a level box = 0). */
int hp_debug_payload(const hp_tree* tree, int level, int r, uint64_t seed, int device,
                     double* out);
/* K4 probe: the batched range finder on nb blocks stacked column-major (block
 * i is rows[i] x cols); q gets Q(:, :kmax) of each block stacked the same way
 * (zero columns beyond the kept rank), ranks the kept ranks, *ms the device
 * time of the QR stage. */
int hp_debug_qr(const double* blocks, const int* rows, int nb, int cols, int kmax, int device,
                double* q, int* ranks, double* ms);
/* device natural log used by the log-kernel black box, for accuracy tests */
int hp_debug_log(const double* x, int64_t n, int device, double* out);

#ifdef __cplusplus
}
#endif

#endif /* HPEEL_B200_H */
