/*
 * hpez_oracle.h -- CPU restatement of the HPEZ hot path (TEST INFRASTRUCTURE).
 *
 * This is the parity checker for the B200 kernels in paper_2311_12133_b200/.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load it.  The product path never links or calls it.
 *
 * Parity pin: tests/test_oracle_golden.py checks every function here against
 * golden vectors produced by the reference Python package itself
 * (tests/golden/make_golden.py, run with PYTHONPATH=/root/reference/pkg/src).
 *
 * Each function cites the reference file:line it restates.
 */
#ifndef HPEZ_ORACLE_H
#define HPEZ_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_RANK 5

enum { ORC_OK = 0, ORC_CORRUPT = 1, ORC_UNDERFLOW = 2, ORC_BADARG = 3 };
enum { ORC_ROUND_NONE = 0, ORC_ROUND_F32 = 1, ORC_ROUND_INT = 2 };

/* One level of the plan (plan.py:94-105 LevelSpec + LevelConfig). */
typedef struct {
    int32_t stride;
    int32_t kernel;        /* KERNEL_VARIANTS index, plan.py:25-31 */
    int32_t paradigm;      /* 0 = oned, 1 = multidim */
    int32_t n_order;       /* entries used in axis_order (oned only) */
    int32_t axis_order[ORC_MAX_RANK];
    double bound;
} orc_level;

/* interp.run_levels (interp.py:440-472).  direction 0 = compress, 1 =
 * decompress.  Compress: codes/outliers are outputs (capacity n_points),
 * *n_codes / *n_outl receive the counts.  Decompress: codes/outliers are
 * inputs with *n_codes / *n_outl available; on return they hold the number
 * consumed.  block_table is (n_levels, n_blocks) u8 or NULL.  Stats
 * (interp.py:89-118) are optional: err_sum/count per level, dense grids
 * (n_levels * N doubles, zero-initialised by the caller). */
int orc_run_levels(double *work, int rank, const int64_t *dims,
                   uint32_t frozen_mask, int direction, int64_t radius,
                   int rounding, int n_levels, const orc_level *levels,
                   const double *md_alpha, int block_size,
                   const uint8_t *block_table, int32_t *codes,
                   int64_t *n_codes, double *outliers, int64_t *n_outl,
                   double *stat_err_sum, int64_t *stat_count,
                   double *stat_dense);

/* lorenzo.lorenzo_pass (lorenzo.py:145-179). */
int orc_lorenzo(double *work, int rank, const int64_t *dims, double bound,
                int64_t radius, int order, int direction, int rounding,
                int32_t *codes, int64_t n_codes, double *outliers,
                int64_t *n_outl);

/* numpy pairwise float64 sum (used by PassStats and tune_blocks). */
double orc_pairwise_sum(const double *a, int64_t n);

/* huffman.code_lengths (huffman.py:19-48).  Returns ORC_BADARG if empty. */
int orc_code_lengths(const int64_t *freqs, int64_t n, uint8_t *lengths);
/* huffman.canonical_codes (huffman.py:51-88), code values only. */
int orc_canonical_codes(const uint8_t *lengths, int64_t n, uint64_t *values);
/* huffman._pack_bits (huffman.py:91-113); returns bytes written. */
int64_t orc_pack_bits(const int64_t *symbols, int64_t n,
                      const uint64_t *values, const uint8_t *lengths,
                      uint8_t *out);
/* huffman._unpack_symbols (huffman.py:116-141): returns bits used, -1
 * truncated, -2 invalid pattern. */
int64_t orc_unpack_symbols(const uint8_t *data, int64_t nbytes,
                           const uint8_t *lengths, int64_t n_lengths,
                           int64_t count, int64_t *out);

#ifdef __cplusplus
}
#endif
#endif
