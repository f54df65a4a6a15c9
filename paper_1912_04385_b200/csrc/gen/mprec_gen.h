/*
 * mprec_gen.h -- synthetic thermal Jacobian generator for the BASELINE.json
 * configurations.  Host-only test/bench input
 * infrastructure: it produces the block-sparse system that both the CPU
 * oracle and the GPU path consume, it is not part of the solve path.
 *
 * Every random number is a pure function of (seed, stream, index) (a
 * SplitMix64 counter hash), so the fill is embarrassingly parallel and
 * bit-identical for any thread count.
 *
 * Storage contract (identical to include/mprec_gpu.h):
 *   cells c = y*nx + x; 5-point pattern, block columns sorted ascending,
 *   diagonal block always present; blocks are nb x nb, COLUMN-MAJOR,
 *   intra-cell unknown order (s..., P, T): P = nb-2, T = nb-1
 *   (reference proj/include/mprec/field_layout.hpp:62-66).
 *
 * Builder decisions where BASELINE.json is ambiguous:
 *   1. seed-field noise eps ~ N(0, 0.1^2)  (N(0,0.01) read as variance);
 *   2. the flux block F is per cell and indexed by the upwind cell; both
 *      directions of a face share -T_f F_u;
 *   3. the reaction band is |x - y| <= 2;
 *   4. band edits are applied after the diagonal-block assembly.
 */
#ifndef MPREC_GEN_H
#define MPREC_GEN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mprec_gen_spec {
    int nx;
    int ny;
    int nb;             /* unknowns per cell, >= 2 */
    double kappa;       /* conduction multiplier on the (T,T) entry */
    double perm_sigma;  /* log-normal permeability sigma; 0 => k == 1 */
    int band;           /* 1 => reaction band |x-y| <= 2 */
    uint64_t seed;
} mprec_gen_spec;

/* Fill *out with BASELINE.json configuration `config_id` (1..5). Returns 0,
 * or -1 for an unknown id. */
int mprec_gen_config(int config_id, mprec_gen_spec* out);

/* Number of stored blocks of the nx x ny 5-point pattern. */
int64_t mprec_gen_nnzb(int nx, int ny);

/* Block pattern: row_ptr[nx*ny+1], col_idx[nnzb]. */
int mprec_gen_pattern(int nx, int ny, int* row_ptr, int* col_idx);

/* Block values (column-major nb x nb per stored block), x* and b = A x*.
 * Any of vals / xstar / b may be NULL to skip it (b needs vals and xstar).
 * nthreads <= 0 selects std::thread::hardware_concurrency(). */
int mprec_gen_fill(const mprec_gen_spec* spec, const int* row_ptr, const int* col_idx,
                   double* vals, double* xstar, double* b, int nthreads);

#ifdef __cplusplus
}
#endif

#endif
