// Launchers for the sm_100a kernels (K1..K7). Plain
// pointers and sizes; every pointer is device memory unless noted.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "device.cuh"

namespace hpeel {

// ---------------------------------------------------------------- K1 payload
/// Gaussian payload rows of the boxes at one level, fwd (phase 0) in columns
/// [0, r) and adjoint (phase 1) in [r, 2r) of the row-major N x gld buffer g;
/// columns [2r, gld) are zeroed. Rows of positions not covered stay untouched.
/// pos_box[pos] = box id at this level (or -1), local[pos] = rank of the point
/// in the box's input-ordered point list (proj/src/coloring.cpp:252-259).
void launch_payload_gaussian(double* g, int gld, int r, std::int64_t n, const int* pos_box,
                             const int* local, std::uint64_t seed, int level, cudaStream_t s);

// ---------------------------------------------------------------- K2 apply
/// Leaf identity-apply tile: up to 64 consecutive tree rows of a box against
/// the boxes of one color class.
struct SampleTask {
  std::int64_t row0;
  std::int64_t out;  // element offset of (tile row 0, col 0) in `out`
  int rows;
  int color;
  int ld;
  int pad;   // identity probes: columns written (|I_mu| of the compact dense block; 0 = w)
};
/// K2 row table entry: one output row of a sample block (element offset of
/// its column 0 and the block's column stride) and its tree position.
struct K2Row {
  std::int64_t out;
  int pos;
  int ld;
};
/// One K2 CTA: `rows` output rows all served by the payload of `color`.
/// ld > 0: one tile of a single box, row i = tree position pos + i written at
/// base + i with column stride ld. ld == 0: rows rowtab[base + i] (rows of
/// several small target boxes of the same color packed into one tile).
struct K2Task {
  std::int64_t base;
  int rows;
  int color;
  int ld;
  int pos;
};
int k2_mode();
/// K2 arithmetic path switch: true = int8 tensor-core digit products where
/// eligible (default), false = FP64 DMMA everywhere (hp_debug_set_k2_path).
bool k2_int8_enabled();
void set_k2_path(int path);
/// int8 K2 probe bits (path 2: skip the MMAs, path 3: skip the evaluation)
int k2_int8_debug();

__host__ __device__ inline K2Row k2_row(const K2Task& t, const K2Row* rowtab, int i) {
  if (t.ld > 0) return K2Row{t.base + i, t.pos + i, t.ld};
  return rowtab[t.base + i];
}
/// For each task row R = k2_row(task, rowtab, i):
/// out[R.out + (ocol0 + c) * R.ld] = sum_q K(R.pos, pc[q]) gc[q * gld + gcol0 + c]
/// over the payload rows q in [pay_off[color], pay_off[color+1]) of the task's
/// color, stored in color order: pc = tree positions, gc = payload rows,
/// xc = coordinates (dim x nnz). `trans` applies K^T (adjoint of a
/// non-symmetric dense operator).
/// `checked` = false promises that no tile row coincides with a payload row
/// (position or coordinates), so the evaluation skips those tests.
/// Rows per K2 CTA for an apply of `ncols` payload columns; K2Task.rows must
/// not exceed it.
int k2_tile_rows(int ncols);
void launch_sample_apply(const DevOp& op, bool trans, const K2Task* tasks, const K2Row* rowtab,
                         int ntasks, const std::int64_t* pay_off, const int* pc, const double* gc,
                         int gld, int gcol0, int ncols, const double* xc, std::int64_t nnz,
                         double* out, int ocol0, bool checked, cudaStream_t s);

/// Fused K2 variant (k_apply3.cu): every warp evaluates its own DMMA A
/// fragments; rows per CTA kFusedRows, sample width 2r <= 88. Selected by
/// k2 mode bit 2 (hp_debug_set_k2_mode) while it is being evaluated.
constexpr int kFusedRows = 128;
void launch_sample_apply_fused(const DevOp& op, bool trans, const K2Task* tasks,
                               const K2Row* rowtab, int ntasks, const std::int64_t* pay_off,
                               const int* pc, const double* gc, int gld, int gcol0, int ncols,
                               const double* xc, std::int64_t nnz, double* out, int ocol0,
                               cudaStream_t s);

/// flag |= 1 if two distinct points of one leaf (tree-order ranges
/// [leaf_start, +leaf_count)) have identical coordinates (x: dim x n SoA).
void launch_find_duplicates(const double* x, int dim, std::int64_t n, const std::int64_t* leaf_start,
                            const std::int64_t* leaf_count, int nleaves, int* flag, cudaStream_t s);

/// Leaf-phase identity probes (proj/src/coloring.cpp:271-277):
/// out[task.out + i + t * ld] = sum_{v in color} K(row0+i, start_v + t), t < |v|,
/// for t < w. Boxes of color c are pay_box[pay_off[c]..pay_off[c+1]) with
/// tree ranges (box_start, box_count).
void launch_identity_apply(const DevOp& op, const SampleTask* tasks, int ntasks,
                           const std::int64_t* pay_off, const int* pay_box,
                           const std::int64_t* box_start, const std::int64_t* box_count, int w,
                           double* out, cudaStream_t s);

// ---------------------------------------------------------------- K3 peel
/// Coefficient task: T = op(B) * sum_v F[rows of v]^T P_v (k x w), written at
/// t_out. F is a factor block (col-major, ld = frows) whose first row is tree
/// position f_row0; P_v are payload rows (gaussian rows of g at column gcol0,
/// or identity when gcol0 < 0). B is k x k col-major, transposed if btrans.
struct CoeffTask {
  std::int64_t f;      // factor offset
  std::int64_t b;      // B offset
  std::int64_t t_out;  // output offset (k x w col-major)
  std::int64_t f_row0; // tree position of factor row 0
  int frows;
  int seg_begin;       // payload segments [seg_begin, seg_end) in seg arrays
  int seg_end;
  int btrans;
};
/// segments: tree ranges (seg_start, seg_count) of the payload boxes.
void launch_peel_coeff(const CoeffTask* tasks, int ntasks, const double* factors,
                       const double* bmat, const std::int64_t* seg_start,
                       const std::int64_t* seg_count, const double* g, int gld, int gcol0, int k,
                       int w, double* tbuf, cudaStream_t s);

/// Apply task: out[out + i + (ocol0 + c) * ld] += alpha * sum_terms F_term[frow_off + i, :] T_term[:, c]
/// for i < rows (<= 64), c < w. Terms in CSR (term_off[task] .. term_off[task+1]).
/// One output tile: rows [out, out + rows) (column stride ld) accumulate the
/// term lists refs[ref_begin, ref_end).
struct PeelTask {
  std::int64_t out;
  int rows;
  int ld;
  int ref_begin;
  int ref_end;
  int cols;  // columns of this output block (<= w; compact dense blocks keep |I_mu|)
  int pad;
};
/// A shared term list [term_begin, term_end) read at row offset roff.
struct PeelRef {
  int term_begin;
  int term_end;
  std::int64_t roff;
};
struct PeelTerm {
  std::int64_t f;     // factor element offset of row 0 (plus the ref's roff)
  std::int64_t t;     // coefficient offset (k x w)
  int fld;            // factor leading dimension
  int pad;
};
void launch_peel_apply(const PeelTask* tasks, int ntasks, const PeelRef* refs, const PeelTerm* terms,
                       const double* factors, const double* tbuf, int k, int w, double* out,
                       int ocol0, double alpha, cudaStream_t s);

// ---------------------------------------------------------------- K4 QR
/// One block of a batched QR stage (col-major offsets into the stage buffers).
struct QrBlock {
  std::int64_t a;    // input block (ld lda); chunk stage overwrites it with reflectors
  std::int64_t out;  // chunk: R rows in the parent stacked matrix; top/backprop: Q output (ld ldo)
  std::int64_t tau;  // chunk/backprop: tau offset
  std::int64_t c;    // backprop: parent Q rows for this chunk (ld ldc)
  int rows;
  int lda;
  int ldo;
  int ldc;
  int rank_slot;     // top: index into ranks (or -1)
  int pad;
};
/// Rows of a block that the pivoted single-CTA QR (qr_top) holds in shared memory.
int qr_rows_max(int cols);
/// Rows per TSQR chunk (the back-propagation also stages kmax Q columns).
int qr_chunk_rows(int cols, int kmax);
/// Unpivoted Householder QR of each chunk in place (reflectors below the
/// diagonal), tau at tau + aux, R (min(rows,cols) x cols, upper) copied into
/// the parent stacked matrix at out (ld = ldo). max_rows bounds the blocks'
/// rows (sizes shared memory).
void launch_qr_chunk(const QrBlock* blocks, int nb, double* data, double* rout, double* tau,
                     int cols, int max_rows, cudaStream_t s);
/// Column-pivoted Householder QR of each top block, keep = first columns with
/// |R_jj| > tol * |R_00| capped at kmax (proj/src/linalg.cpp:53-78); writes
/// Q(:, :keep) to out (ld = ldo, kmax columns, zero beyond keep) and keep to
/// ranks[rank_slot].
void launch_qr_top(const QrBlock* blocks, int nb, double* data, double* outbuf, int* ranks,
                   int cols, int kmax, double tol, int max_rows, cudaStream_t s);
/// TSQR back-propagation: out(rows x kmax) = H_chunk [C; 0], C = r x kmax
/// block of the parent Q at c (ld = ldc).
void launch_qr_backprop(const QrBlock* blocks, int nb, const double* data, const double* tau,
                        const double* parent, double* outbuf, int cols, int kmax, int max_rows,
                        cudaStream_t s);

/// Register-resident QR (k_qr2.cu) for cols <= 96: columns padded to
/// qr_reg_cols(cols) (0 = unsupported), blocks of up to qr_reg_rows_max rows.
/// mode 0 = launch_qr_top contract, mode 1 = launch_qr_chunk contract.
int qr_reg_cols(int cols);
int qr_reg_rows_max(int cols);
/// rows per thread the register kernels use for a block of `rows` rows; a
/// block's arithmetic depends only on this, so batches are launched per class
int qr_reg_rpt(int cols, int rows);
void launch_qr_reg(int mode, const QrBlock* blocks, int nb, double* data, double* out, double* tau,
                   int* ranks, int cols, int kmax, double tol, int max_rows, cudaStream_t s);
/// launch_qr_backprop contract, kmax <= 96, rows <= qr_reg_rows_max(kmax).
void launch_qr_reg_backprop(const QrBlock* blocks, int nb, const double* data, const double* tau,
                            const double* parent, double* outbuf, int cols, int kmax, int max_rows,
                            cudaStream_t s);

/// Gram-based range finder (k_gqr.cu): staged pivoted Cholesky-QR on DMMA,
/// the same pivots / kept rank / span as launch_qr_top's pivoted Householder
/// QR (proj/src/linalg.cpp:53-78), blocks of any height. The input block is
/// destroyed (deflated in place).
struct GqrBlock {
  std::int64_t a;    // input block (col-major, ld lda)
  std::int64_t out;  // Q output (ld ldo, kmax columns, zero beyond the kept rank)
  int lda;
  int ldo;
  int rows;
  int rank_slot;     // index into ranks (or -1)
  int task0;         // first row task of this block
  int ntasks;
};
struct GqrTask {
  int block;
  int row0;
  int rows;
};
struct GqrState {    // per block, device-only
  int done, last, kq, j, keep, pad;
  double d00;
  unsigned long long amax;  // bit pattern of the block's largest |entry|
  unsigned char used[96];
};
constexpr int kGqrTaskRows = 256;
bool gqr_supported(int r, int kmax);
std::int64_t gqr_part_doubles(int r, int kmax);  // Gram workspace per row task
std::int64_t gqr_w_doubles(int r, int kmax);     // transform workspace per block
/// The power-of-two rescale of out-of-range blocks alone (launch_gqr runs it
/// itself): for the short blocks left to the Householder kernels, whose sums
/// of squares have the same [2^-300, 2^300] domain.
void launch_qr_rescale(const GqrBlock* blocks, int nb, const GqrTask* tasks, int nt, GqrState* state,
                       double* data, int r, cudaStream_t s);
/// ranks[rank_slot] = -1 for the blocks launch_qr_rescale found non-finite
/// (launch_gqr reports its own): qr_orthonormal's "non-finite matrix in qr".
void launch_qr_flag(const GqrBlock* blocks, int nb, const GqrState* state, int* ranks, cudaStream_t s);
void launch_gqr(const GqrBlock* blocks, int nb, const GqrTask* tasks, int nt, GqrState* state, double* data,
                double* q, double* part, double* wbuf, int* ranks, int r, int kmax, double tol,
                cudaStream_t s);

// ---------------------------------------------------------------- K5 B
/// Register-resident pivoted-QR B solve (k_bsolve2.cu, k <= 64, r <= 80):
/// bsolve_qr_kernel's contract; false when the widths are unsupported.
bool launch_bsolve_reg(int npairs, const double* gpu_, const double* middle, const double* vg, int r, int k,
                       const std::int64_t* boff, double* b, int* flags, cudaStream_t s);
/// out = X^T Y partial sums over row chunks: X (rows x nx, ld lx), Y (rows x ny,
/// ld ly). Tasks write nx x ny col-major partials; summed in task order by
/// launch_sum_partials.
struct GramTask {
  std::int64_t x;
  std::int64_t y;
  std::int64_t out;
  int rows;
  int lx;
  int ly;
  int x_rowmajor;  // X is row-major with row stride lx (payload buffer)
  int y_rowmajor;
  int pad;
};
void launch_gram(const GramTask* tasks, int ntasks, const double* xbase, const double* ybase,
                 int nx, int ny, double* out, cudaStream_t s);
/// dst[d + i] = sum_{p in [off[d], off[d+1])} src[p * len + i]
void launch_sum_partials(const std::int64_t* off, int ndst, const double* src, int len,
                         double* dst, cudaStream_t s);

/// Per pair: left = pinv(gpU) * middle, B = (pinv(VG^T) * left^T)^T with the
/// SVD cutoff tol * sigma_1 (proj/src/linalg.cpp:110-127, proj/src/peeling.cpp:252-269).
/// gpU r x k, middle r x r, VG k x r (all col-major, packed per pair at
/// stride), B k x k written at b + pair * k * k.
void launch_bsolve(int npairs, const double* gpu_, const double* middle, const double* vg,
                   int r, int k, double tol, const std::int64_t* boff, double* b, cudaStream_t s);

// ---------------------------------------------------------------- misc
/// dst[i * dsr + c * dsc] = src[map[i] * ssr + c * ssc] (map == nullptr: identity).
void launch_permute_rows(const double* src, std::int64_t ssr, std::int64_t ssc, const int* map,
                         std::int64_t rows, int w, double* dst, std::int64_t dsr, std::int64_t dsc,
                         cudaStream_t s);

/// y = K x or K^T x (tree order, x and y col-major n x w): full black-box
/// apply used by the power-method verifier (proj/src/linalg.cpp:179-196).
void launch_full_apply(const DevOp& op, bool trans, const double* x, int w, double* y,
                       cudaStream_t s);

/// Dense leaf blocks of H1Rep::apply (proj/src/hmatrix.cpp:59-73): for box b,
/// y[rows of b] += sum over tasks [off[b], off[b+1]) of D x[cols] (or D^T for
/// the adjoint, where the task's columns are the output rows). x, y row-major.
struct DenseTask {
  std::int64_t d;     // block offset, col-major rows x cols
  std::int64_t row0;  // tree position of the block rows (lambda)
  std::int64_t col0;  // tree position of the block cols (mu)
  int rows, cols;
};
void launch_dense_apply(const DenseTask* tasks, const int* box_off, int nboxes,
                        const double* dense, const double* x, int w, bool adjoint, double* y,
                        std::int64_t ldy, cudaStream_t s);

// ---------------------------------------------------------------- sharding / callback
/// dst[s.dst + i] = src[s.src + i] for i < s.len, one CTA per segment.
struct CopySeg {
  std::int64_t src;
  std::int64_t dst;
  std::int64_t len;
};
void launch_copy_segments(const double* src, const CopySeg* segs, int nseg, double* dst, cudaStream_t s);
/// dst[didx ? didx[e] : e] = src[sidx ? sidx[e] : e] for e < n.
void launch_move_i32(const int* src, const int* sidx, std::int64_t n, int* dst, const int* didx, cudaStream_t s);
/// One sample row read back from a black-box product Y (input order, column
/// stride ldy): out[out + (ocol0 + c) * ld] = Y[perm[pos] + c * ldy], c < min(w, cols).
struct GatherRow {
  std::int64_t out;
  int pos;
  int ld;
  int cols;
  int pad;
};
void launch_gather_sample_rows(const double* y, std::int64_t ldy, const int* perm, const GatherRow* rows,
                               std::int64_t nrows, int w, double* out, int ocol0, cudaStream_t s);
/// Dense test matrix of one color for a callback black box
/// (BlockTestMatrix::realize, proj/src/coloring.cpp:261-291), input order:
/// omega[perm[pos[q]] + c * ldo] = g[pos[q] * gld + gcol0 + c], c < w
/// (payload rows; the caller zero-fills the rest).
void launch_scatter_payload(const double* g, int gld, int gcol0, int w, const int* pos, std::int64_t cnt,
                            const int* perm, double* omega, std::int64_t ldo, cudaStream_t s);
/// Identity payloads [I | 0] of the leaf phase: omega[perm[start_b + t] + t * ldo] = 1, t < min(|b|, w).
void launch_scatter_identity(const int* boxes, int nbox, const std::int64_t* box_start,
                             const std::int64_t* box_count, const int* perm, int w, double* omega,
                             std::int64_t ldo, cudaStream_t s);

}  // namespace hpeel
