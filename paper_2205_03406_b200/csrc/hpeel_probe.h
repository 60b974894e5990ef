/*
 * Probe entry points of libhpeel_b200.so for tests and profiling tools. NOT
 * part of the drop-in boundary (include/hpeel_b200.h): the K2 switches make
 * compress() skip work and return invalid results.
 */
#ifndef HPEEL_PROBE_H
#define HPEEL_PROBE_H

#include <stdint.h>

#include "../../include/hpeel_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* K2 probe bits: 1 = skip kernel evaluation, 2 = skip DMMA (timing only, invalid
 * results); 4 = fused kernel, 8 = checked evaluation path, 16 = payload chunks
 * in reverse order (valid results: another FP64 summation order); 0 = normal */
void hp_debug_set_k2_mode(int mode);
/* K2 arithmetic path: 0 = int8 tensor-core digit products (exact fixed-point
 * emulation of the FP64 contraction, k2_i8.cuh) wherever eligible (default),
 * 1 = FP64 DMMA for every apply (A/B tests) */
void hp_debug_set_k2_path(int path);

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

#endif /* HPEEL_PROBE_H */
