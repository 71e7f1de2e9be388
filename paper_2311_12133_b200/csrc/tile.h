// tile.h -- shared-memory tiled level sweep (tile.cu), host interface used by
// the sweep planner (sweep.cu).
//
// One launch runs one whole level of a rank-3 uniform sweep
// (interp._LevelRunner.run_level, interp.py:415-433, with every class on the
// uniform path, interp.py:322-341).  The level's points form the stride-s
// sublattice; CTAs own (y, x) tiles x z-chunks of it, stream the chunk plane by
// plane through an f64 ring of planes in shared memory and recompute the
// halo points their owned points depend on, so no CTA ever waits on another.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace hpez {

constexpr int kTileMaxCommits = 16;
constexpr int kTileMaxTasks = 64;
constexpr int kTileMaxIntervals = 32;
constexpr int kTileEvenSlots = 8;  // ring slots (see slot_off in tile.cu)
constexpr int kTileOddSlots = 5;

struct TileCommit {
    int32_t v, split, phase, odd;  // class mask, split axis (-1), phase, axis 0 in v
    int32_t st[3], sh[3], cnt[3];  // lattice in sublattice units: j = st + (i << sh)
    int32_t box[4];                // compute-box extension beyond the owned tile: ylo, yhi, xlo, xhi
    int32_t item_base, p_item, pw; // stream bookkeeping (escape counts per (item, warp))
    int32_t fam, nax, kind;        // predictor: stencil family, 1 (1-D) .. 3 axes, layout (tk_axis)
    int32_t pad;
    int32_t axes[3];
    double w[3];                   // MD blend weights (nax >= 2)
    int64_t code_base;
};

struct TileDesc {
    int32_t L[3];                  // sublattice extents
    int32_t s;
    int32_t E0, E1;                // grid element strides of axes 0 and 1
    int32_t TY, TX, ZC;            // tile (owned) sizes
    int32_t tiles_y, tiles_x, chunks_z;
    int32_t HYe, HXe, HYo, HXo;    // ring halos (even / odd planes); HX even
    int32_t RYe, RXe, RYo, RXo;    // ring plane dims
    int32_t n_commits, n_iv;
    int32_t R;
    int64_t n_codes;               // whole code stream (bounds the aligned code-word loads)
    double bound, two_e, inv_two_e;
    int32_t iv_off[kTileMaxIntervals + 1];
    int8_t task_sel[kTileMaxTasks];   // 0: even plane 4m, 1: 4m+2, 2: odd 4m-3, 3: odd 4m-5
    int8_t task_c[kTileMaxTasks];
    int8_t lut[64];                   // ((z&3)<<4)|((y&3)<<2)|(x&3) -> commit, -1 = coarse
    TileCommit c[kTileMaxCommits];
};

struct TileRun {
    const void *orig;     // compress: originals (read-only)
    void *work;           // reconstruction (coarse points read, level points written)
    void *codes;
    const double *outl;   // decompress outliers
    int64_t outl_cap;
    uint32_t *esc_cnt;    // per (item, warp) escapes (compress: incremented)
    const int64_t *esc_off;  // per (item, warp) first outlier rank (decompress)
    int32_t *flags;
};

struct TilePlan {
    TileDesc d;
    int grid = 0;
    int threads = 0;
    size_t smem = 0;
};

// Builds the tiled plan of one level from its commit descriptors (reference
// order).  Returns false when the level is not eligible (rank != 3, frozen or
// mixed commits, > kTileMaxCommits commits, ring larger than shared memory).
bool tile_plan_build(const GridDev &g, const CommitDev *cms, int n, int64_t n_codes, TilePlan *out);

// Launches one level (f32 work, u16 codes).  dir = HPEZ_COMPRESS / HPEZ_DECOMPRESS.
cudaError_t tile_plan_launch(const TilePlan &p, int dir, const TileRun &r, cudaStream_t st);


// ---------------------------------------------------------------- coarse --
// Leading levels held in the distributed shared memory of one cluster
// (coarse.cu).  Lattices are in units of the stride-Sc sublattice.
constexpr int kCoarseMaxCommits = 96;
constexpr int kCoarseMaxGroups = 64;
constexpr int kCoarseMaxLevels = 6;
constexpr int kCoarseDsmemThreads = 1024;

struct CoarseCommit {
    int32_t st[3], sp[3], cnt[3];  // j = st + i * sp (sublattice units)
    int32_t sh[3];                 // log2(sp)
    int32_t s;                     // level stride (sublattice units)
    FastDiv fd_row, fd_x;          // division by cnt[1]*cnt[2] and by cnt[2]
    int32_t kind, fam;             // predictor layout (tk_axis) and family
    int32_t item_base, p_item, pw;
    double w[3];
    double bound, two_e, inv_two_e;
    int64_t code_base;
};

struct CoarseDesc {
    int32_t L[3];
    int32_t Sc, E0, E1, P;         // sublattice stride, grid strides, planes per CTA
    int32_t R;
    int32_t n_commits, n_groups, n_levels;
    int64_t n_codes;
    int32_t n_cc;                  // codes of the coarse levels = stream prefix [0, n_cc)
    int32_t grp_off[kCoarseMaxGroups + 1];
    int32_t lvl_s[kCoarseMaxLevels], lvl_sh[kCoarseMaxLevels];
    FastDiv fd_plane, fd_x, fd_P;   // division by L1*L2, by L2 and by P
    int8_t lut[kCoarseMaxLevels][64];
    CoarseCommit c[kCoarseMaxCommits];
};

struct CoarsePlan {
    CoarseDesc d;
    int ncta = 0;
    size_t smem = 0;
};

// group[i]: (level, DAG depth) group of commit i (non-decreasing runs define
// the cluster barriers).  False when not eligible (rank != 3, mixed
// commits, too many commits/groups, slab above shared memory).
bool coarse_dsmem_build(const GridDev &g, const CommitDev *cms, const int *group, int n, int64_t n_codes,
                        CoarsePlan *out);
cudaError_t coarse_dsmem_launch(const CoarsePlan &p, int dir, const TileRun &r, cudaStream_t st);

}  // namespace hpez
