// row.h -- row-fused fine levels of the rank-3 sweep (row.cu), host
// interface used by the sweep planner (sweep.cu).
//
// The finest level (stride 1) of a multidim configuration holds 7/8 of a
// grid's points.  row.cu runs it as a handful of plain launches in which one
// warp owns one grid row (fixed z, y) at a time and computes BOTH classes of
// the row -- the x-even class, then the x-odd class that reads it -- from
// whole-row 16-byte loads of the neighbouring rows, keeping the row's fresh
// values in shared memory (f64) for the in-row stencil and writing complete
// sectors back (interp._LevelRunner.run_level, interp.py:415-433, with the
// uniform and the mixed per-block commits of interp.py:322-411).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace hpez {

// Classes of a rank-3 level in reference order (interp.py:417-418):
// 0 (z)  1 (y)  2 (x)  3 (z,y)  4 (z,x)  5 (y,x)  6 (z,y,x).
struct RowDesc {
    int32_t L[3];                // lattice extents of the level (coordinates / s)
    int32_t s;                   // level stride
    int32_t E0, E1;              // element strides of one lattice step along z and y
    int32_t has_table, const_tag;  // block table present / the level's tag (plan.encode_tag) when not
    int32_t bsh, bs0, bs1;       // log2(block size in lattice units), block-grid strides of z and y
    uint32_t oned_sel[7];        // per class: term index used by one-axis order p, 4 bits each
    int32_t any_same;            // some block of the level uses a same-level variant
    int32_t R;
    int32_t cny[2];              // class rows along y for y-even / y-odd rows
    int32_t commitA[7], commitB[7];  // plan commit of each class's first / second pass (-1: none)
    int64_t segA[7], segB[7];    // first entry of the class's rows in the row-base table
    int64_t n_entries;           // rows of all (class, pass) segments
    int64_t level_base;          // code index of the level's first code
    double bound, two_e, inv_two_e;
    double w[7][3];              // MD blend weights per class (interp._blend_weights)
};

struct RowRun {
    const float *orig;
    float *work;
    uint16_t *codes;
    const double *outl;
    int64_t outl_cap;
    uint32_t *esc_cnt;
    const int64_t *esc_off;
    int32_t *flags;
    const uint8_t *table;     // the level's block tags (device)
    const int64_t *rowbase;   // code offset (relative to the level) of every (class, pass, row)
    const CommitDev *commits;
    const int64_t *wbase;
};

struct RowSet {                  // rows z = z0 + i*zs (i < nz), y = y0 + j*ys (j < ny)
    int32_t rt, brow;            // row type (z odd) | (y odd) << 1; second same-level phase of the x-even class
    int32_t z0, zs, nz, y0, ys, ny;
};

struct RowLaunch {
    int32_t n, total;
    RowSet s[2];
};

struct RowPlan {
    RowDesc d;
    bool ok = false;
    int n_launch = 0;
    RowLaunch launch[4];
    int32_t first_commit = 0;    // plan commit index of the level's first commit
    // device (carved from the plan workspace)
    uint32_t *d_cnt = nullptr;
    int64_t *d_base = nullptr;
    int64_t *d_tmp = nullptr;
    int64_t *d_total = nullptr;
    size_t smem = 0;
    int threads = 0;
};

// Builds the row plan of one level (stride 1, 2 or 4) from its commits
// (reference order).  `tbl` is the level's host block table (or null, then
// `level_tag` is the level's own tag).  False when the level is not
// eligible: rank != 3, lattice x extent not a multiple of 4, a one-axis
// (oned) variant with a same-level split, blocks smaller than four lattice
// points or not a power of two.
bool row_plan_build(const GridDev &g, const CommitDev *cms, const uint32_t *vmask, int n, int first_commit,
                    const uint8_t *tbl, int64_t nblk, int level_tag, int64_t level_base, RowPlan *out);
// Row-base table: member counts per (class, pass, row) and their exclusive scan.
cudaError_t row_plan_setup(RowPlan &p, const uint8_t *d_table_level, cudaStream_t st);
cudaError_t row_plan_launch(const RowPlan &p, int dir, const RowRun &r, cudaStream_t st);

}  // namespace hpez
