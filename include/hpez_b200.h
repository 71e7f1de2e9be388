/*
 * hpez_b200.h -- C ABI of the B200-native HPEZ hot path (libhpez_b200.so).
 *
 * Plain pointers and sizes only; no torch types.  Device pointers are CUDA
 * global-memory pointers on the current device; `stream` is a cudaStream_t
 * passed as void*.  Every entry point returns an hpez_status.
 *
 * Each entry point names the reference interface it replaces (the reference
 * is the pure-Python package hpez 0.1.0, pkg/src/hpez/…).  The reference-side
 * binding a maintainer would add is shown in INTEGRATION.md.
 */
#ifndef HPEZ_B200_H
#define HPEZ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HPEZ_MAX_RANK 5 /* 4 grid axes + the tuner's stacked batch axis */

typedef enum {
    HPEZ_OK = 0,
    HPEZ_CORRUPT_STREAM = 1,    /* errors.CorruptStream (interp.py:80-83)   */
    HPEZ_OUTLIER_UNDERFLOW = 2, /* errors.OutlierUnderflow (quant.py:123)   */
    HPEZ_BAD_ARGUMENT = 3,      /* ValueError (interp.py:453-456, plan.py)  */
    HPEZ_CUDA_ERROR = 4,
    HPEZ_EMPTY_INPUT = 5,       /* errors.EmptyInput (huffman.py:27)        */
    HPEZ_INVALID_TABLE = 6,     /* errors.InvalidTable (huffman.py:69-74)   */
    HPEZ_TRUNCATED = 7          /* errors.TruncatedStream (huffman.py:171)  */
} hpez_status;

enum { HPEZ_COMPRESS = 0, HPEZ_DECOMPRESS = 1 };
/* quant.ROUND_NONE / ROUND_F32 / ROUND_INT (quant.py:27-29) */
enum { HPEZ_ROUND_NONE = 0, HPEZ_ROUND_F32 = 1, HPEZ_ROUND_INT = 2 };
/* storage of the working grid on the device */
enum { HPEZ_WORK_F32 = 0, HPEZ_WORK_F64 = 1 };
/* device code stream element type */
enum { HPEZ_CODES_U16 = 0, HPEZ_CODES_I32 = 1 };

/* One level of plan.LevelSpec (plan.py:94-98) with its LevelConfig
 * (plan.py:54-66).  kernel = index into plan.KERNEL_VARIANTS (plan.py:25-31);
 * paradigm 0 = PARADIGM_ONED, 1 = PARADIGM_MULTIDIM. */
typedef struct {
    int32_t stride;
    int32_t kernel;
    int32_t paradigm;
    int32_t n_order;
    int32_t axis_order[HPEZ_MAX_RANK];
    double bound;
} hpez_level;

/* Arguments of interp.run_levels (interp.py:440-445) minus the arrays. */
typedef struct {
    int32_t rank;
    int64_t dims[HPEZ_MAX_RANK];
    uint32_t frozen_mask;        /* bit a set: axis a in frozen_axes */
    int32_t direction;           /* HPEZ_COMPRESS / HPEZ_DECOMPRESS */
    int32_t rounding;            /* HPEZ_ROUND_* */
    int64_t radius;              /* 1 .. 2^30 */
    int32_t n_levels;
    const hpez_level *levels;    /* host, coarse to fine */
    const double *md_alpha;      /* host, `rank` weights, NULL = all ones */
    int32_t block_size;          /* 0 = no per-block table */
    const uint8_t *block_table;  /* host (n_levels, n_blocks) u8 or NULL */
    int32_t work_dtype;          /* HPEZ_WORK_F32 / HPEZ_WORK_F64 */
    int32_t code_dtype;          /* HPEZ_CODES_U16 (radius <= 32768) / I32 */
    int32_t with_stats;          /* PassStats (interp.py:89-118) wanted */
} hpez_sweep_desc;

typedef struct hpez_plan_s *hpez_plan;

/* Build the commit schedule of run_levels for one geometry/config
 * (interp.py:415-433 class enumeration, :322-411 commit split).  Host-side
 * only (no device allocation).  One run at a time per plan. */
int hpez_plan_create(const hpez_sweep_desc *desc, hpez_plan *out);
int hpez_plan_destroy(hpez_plan plan);
/* Device workspace of a plan (its commit / item tables and run scratch):
 * the caller allocates `bytes` of device memory and binds it once, before
 * the first run; runs then never allocate.  A plan run without a bound
 * workspace makes one allocation of this size itself at its first run. */
int hpez_plan_workspace_size(hpez_plan plan, int64_t *bytes);
int hpez_plan_bind_workspace(hpez_plan plan, void *workspace, int64_t bytes);
/* Number of codes the sweep produces / consumes (= points - anchors). */
int64_t hpez_plan_num_codes(hpez_plan plan);
int32_t hpez_plan_num_commits(hpez_plan plan);
int32_t hpez_plan_num_launches(hpez_plan plan);

/* Replaces interp.run_levels (interp.py:440-472).  `work` is updated in
 * place.  Compress: writes codes[0 .. num_codes) and up to `outl_cap`
 * outliers (f64, stream order).  Decompress: reads `codes_avail` codes and
 * `outl_cap` outliers; fewer codes than the plan needs -> CORRUPT_STREAM.
 * Stats (compress, with_stats plans): stat_err_sum/stat_count (device,
 * n_levels) are accumulated like PassStats.record (both may be null when
 * only the dense grids are wanted: tune_blocks); stat_dense (device,
 * n_levels * points doubles, zero-initialised) receives the dense error
 * grids.  Launches are asynchronous on `stream`; call hpez_sweep_finish. */
int hpez_sweep_run(hpez_plan plan, void *work, void *codes, int64_t codes_avail,
                   double *outliers, int64_t outl_cap, double *stat_err_sum,
                   int64_t *stat_count, double *stat_dense, void *stream);
/* Synchronise `stream`, report the outlier count (compress: produced, may
 * exceed outl_cap -> rerun with a larger buffer; decompress: consumed) and
 * the sweep status (OUTLIER_UNDERFLOW on an exhausted outlier stream). */
int hpez_sweep_finish(hpez_plan plan, void *stream, int64_t *n_outliers);
/* Compress out of place: the pipeline's `work = f64(grid)` copy
 * (pipeline.py:82) folded into the sweep.  Originals are read from `orig`
 * (never written); `work` receives the anchors and every reconstructed
 * point (escapes: their originals).  The plan must cover every non-anchor
 * point (the reference's level ladder) -> else BAD_ARGUMENT.  Decompress
 * plans ignore `orig`.  Otherwise as hpez_sweep_run. */
int hpez_sweep_run_from(hpez_plan plan, const void *orig, void *work, void *codes, int64_t codes_avail,
                        double *outliers, int64_t outl_cap, void *stream);
/* Tiled levels of the plan (tile.cu): out[0] = count, then per level
 * [first commit, grid, threads, smem bytes, TY, TX, ZC, intervals]. */
int hpez_plan_tile_info(hpez_plan plan, int64_t *out, int32_t cap);

/* Replaces lorenzo.lorenzo_pass (lorenzo.py:145-179) on a device grid.
 * Compress writes codes[N] and outliers; decompress reads them. */
int hpez_lorenzo(int32_t rank, const int64_t *dims, int32_t work_dtype, void *work,
                 double bound, int64_t radius, int32_t order, int32_t direction,
                 int32_t rounding, int32_t code_dtype, void *codes, int64_t n_codes,
                 double *outliers, int64_t outl_cap, int64_t *n_outliers, void *stream);

/* np.bincount(codes) of huffman.encode (huffman.py:151): counts[0..nbins). */
int hpez_histogram(const void *codes, int32_t code_dtype, int64_t n, uint32_t *counts,
                   int64_t nbins, void *stream);

/* huffman.code_lengths + canonical_codes (huffman.py:19-88), host side.
 * freqs/lengths/values are host arrays of n symbols. */
int hpez_huffman_table(const int64_t *freqs, int64_t n, uint8_t *lengths, uint64_t *values);

/* Bit count of the packed payload: sum(lengths[codes]) (huffman.py:154).
 * `lengths` is a device u8 table; result written to *nbits after a sync. */
int hpez_huffman_nbits(const void *codes, int32_t code_dtype, int64_t n,
                       const uint8_t *lengths_dev, int64_t *nbits, void *stream);

/* huffman._pack_bits (huffman.py:91-113): MSB-first canonical bit packing
 * of n codes into `out` (device, 4-byte aligned, ceil(nbits/32)*4 bytes).
 * max_len = longest code length in the table (1..64). */
int hpez_huffman_pack(const void *codes, int32_t code_dtype, int64_t n,
                      const uint8_t *lengths_dev, const uint64_t *values_dev,
                      int32_t max_len, uint8_t *out, int64_t nbits, void *stream);

/* huffman._unpack_symbols (huffman.py:116-141), host table-driven decoder.
 * Writes `count` symbols (int32) to out; returns TRUNCATED / INVALID_TABLE. */
int hpez_huffman_decode(const uint8_t *payload, int64_t nbytes, const uint8_t *lengths,
                        int64_t n_lengths, int64_t count, int32_t *out);

/* huffman._unpack_symbols (huffman.py:116-141) on the device: the same
 * `count` symbols and error statuses as hpez_huffman_decode, written to
 * out_dev as u16 (code_dtype HPEZ_CODES_U16, n_lengths <= 65536) or int32.
 * The payload comes from host memory (payload_host) or device memory
 * (payload_dev); exactly one is non-NULL.  Self-synchronising chunked
 * decode: speculative per-chunk decode, fix-up passes until every chunk
 * starts at its predecessor's exit, scanned offsets, write pass.  Blocks
 * the calling thread on `stream` for the pass count and the symbol total. */
int hpez_huffman_decode_device(const uint8_t *payload_host, const uint8_t *payload_dev, int64_t nbytes,
                               const uint8_t *lengths, int64_t n_lengths, int64_t count, void *out_dev,
                               int32_t code_dtype, void *stream);

/* tuner.tune_blocks scoring reduction (tuner.py:470-472): out[r] = numpy's
 * pairwise sum of rows[r, 0..rowlen) (= rows.sum(axis=1) bit for bit).  The
 * dense error grids come from bound-0 hpez_sweep_run trials with stats. */
int hpez_rows_pairwise_sum(const double *rows, int64_t nrows, int64_t rowlen, double *out,
                           void *stream);

/* Per-level code stream boundaries: out[0..n_levels] (n_levels + 1 entries),
 * level li owns codes [out[li], out[li+1]) -- PassStats.code_chunks. */
int hpez_plan_level_codes(hpez_plan plan, int64_t *out);

/* Plan diagnostics (12 int64): item counts, schedule flags and, when the
 * environment variable HPEZ_PROFILE is set at plan creation, the flow
 * kernel's clock64 phase counters (grab, wait, work, units).  out[6]: bit 0
 * fast coarse cluster path, bit 1 coarse levels in distributed shared
 * memory (coarse.cu). */
int hpez_plan_info(hpez_plan plan, int64_t *out);

/* Diagnostics: per commit, 6 values [kind (0 uniform, 1 mixed A, 2 mixed B),
 * level, lattice positions, items, members, fast id]; members are read from
 * the device tables, so the plan must have run once.  Returns the number of
 * commits written (at most cap / 6) or a negative status. */
int32_t hpez_plan_commit_stats(hpez_plan plan, int64_t *out, int32_t cap);

/* Diagnostics: out[0] = number of fine levels that run as row-fused launches
 * (csrc/row.cu: interp.run_level at strides 1, 2, 4, interp.py:415-433),
 * out[1] their first commit, out[2] launches, out[3] row-base entries,
 * out[4] same-level variant present, out[5] dynamic shared memory per CTA. */
int hpez_plan_row_info(hpez_plan plan, int64_t *out);

/* HPEZ_PROFILE plans only: out[0..24) per-level (first item start, last
 * item end) globaltimer stamps of the flow kernel, 12 levels x 2; out[24..72)
 * per-level accumulated (grab, wait, work) SM cycles and item count, 12 x 4. */
int hpez_plan_levels_timeline(hpez_plan plan, int64_t *out);

/* Select the CUDA device for subsequent calls from this host thread. */
int hpez_set_device(int32_t device);

/* Library build information (arch string) for provenance checks. */
const char *hpez_build_info(void);


/* ---- tuner sampling statistics and quality metrics ----
 * Reductions follow numpy's pairwise summation bit for bit; `scratch` is
 * device memory of hpez_reduce_scratch_bytes() bytes, `out` / `sums` are
 * device doubles.  Grids are f32 (is_f64 = 0) or f64 C-order arrays. */
int64_t hpez_reduce_scratch_bytes(void);
/* numpy a.sum() (pairwise) of a device f64 array. */
int hpez_pairwise_sum(const double *a, int64_t n, double *out, void *scratch, void *stream);
/* tuner.analyze_samples (tuner.py:86-124): for every axis a in lin_mask /
 * cub_mask, the pairwise sum of the squared linear / cubic residuals at the
 * strided interior sample (grid.py:198-219; box lo/size, n samples) into
 * sums[2a] / sums[2a+1] (divide by n for the reference's np.mean). */
int hpez_sample_stats(const void *grid, int32_t is_f64, int32_t rank, const int64_t *dims, const int64_t *lo,
                      const int64_t *size, int64_t n, uint32_t lin_mask, uint32_t cub_mask, double *sums,
                      void *scratch, void *stream);
/* metrics.psnr numerator (metrics.py:44-45): pairwise sum of (a - b)^2. */
int hpez_sq_diff_sum(const void *a, int32_t a_f64, const void *b, int32_t b_f64, int64_t n, double *out,
                     void *scratch, void *stream);
/* scipy.ndimage.uniform_filter1d(mode="reflect") of a C-order f64 array
 * along `axis` (metrics.py:78-82; window <= extent), out of place. */
int hpez_uniform_filter1d(const double *in, double *out, int32_t rank, const int64_t *dims, int32_t axis,
                          int32_t size, void *stream);
/* metrics.ssim operands: x, y, x*x, y*y, x*y as f64 arrays. */
int hpez_ssim_prep(const void *a, int32_t a_f64, const void *b, int32_t b_f64, int64_t n, double *x, double *y,
                   double *xx, double *yy, double *xy, void *stream);
/* metrics.ssim num/den at the centres lo + 2*i (cnt per axis), compact
 * row-major (metrics.py:83-93). */
int hpez_ssim_terms(const double *mu_x, const double *mu_y, const double *xx, const double *yy, const double *xy,
                    int32_t rank, const int64_t *dims, const int64_t *lo, const int64_t *cnt, double c1, double c2,
                    double *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif
