// tile.cu -- one level of the rank-3 uniform sweep as a shared-memory tiled
// kernel (the drop-in for the levels of interp.run_levels, interp.py:440-472,
// whose classes all take the uniform path, interp.py:322-341).
//
// Geometry.  A level with stride s touches the stride-s sublattice; in its
// units every stencil offset is +-1, +-2 or +-3 and edge truncation is the
// same test as at stride 1 (c + k*s <= E-1  <=>  j + k <= L-1).  Classes with
// axis 0 in v have odd z (they read even planes at z+-1, +-3 and, for a
// same-level split along z, their own phase-0 points at z+-2); the others are
// in-plane problems of the even planes.
//
// Work split.  A CTA owns a TY x TX tile of (y, x) and a ZC-plane chunk of z.
// It streams z in macro-steps of 4 planes: step m computes the even planes
// 4m, 4m+2 and the odd planes 4m-7 (= 1 mod 4) and 4m-9 (= 3 mod 4), whose
// reads along z are then all complete (odd planes lag the even ones by the
// stencil reach).  Each commit is computed over its "need box": the owned
// tile grown by what its consumers read (host analysis), so halo points are
// recomputed locally and CTAs never wait on each other.  Planes live in an
// f64 ring in shared memory (8 even + 4 odd slots, x de-interleaved by parity
// so class lattices read consecutive words); the next step's planes are
// loaded into registers while the current one computes.
//
// Compress reads originals from a separate read-only buffer: a neighbour may
// already have written its reconstruction over a point this CTA still
// recomputes as halo.  Coarse points (earlier levels) are read from `work`,
// which no CTA writes during the level.  Decompress reads coarse values and
// codes only, so it is race-free in place.
#include <algorithm>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "stencil.cuh"
#include "tile.h"

namespace hpez {

__device__ __forceinline__ int floor_div4(int a) { return a >= 0 ? a >> 2 : -((3 - a) >> 2); }

__device__ __forceinline__ FastDiv dev_fastdiv(uint32_t d) {
    FastDiv f;
    f.d = d;
    if (d <= 1) {
        f.mul = 0;
        f.shr = 0;
        return f;
    }
    const uint32_t L = 32 - __clz(d - 1);
    f.mul = (uint32_t)(((1ull << (31 + L)) + d - 1) / d);
    f.shr = 31 + L - 32;
    return f;
}

// x position inside a ring row: de-interleaved by parity (even columns, then odd)
__device__ __forceinline__ int ring_x(int jx, int Xo, int half) {
    const int lx = jx - Xo;
    return (lx & 1) * half + (lx >> 1);
}

// element offset of x + u relative to x, for a target column of parity p
__device__ __forceinline__ int xdelta(int p, int u, int half) {
    return (((p + u) & 1) - p) * half + ((p + u) >> 1);
}

struct TileCtx {
    int Y0, X0, Z0, Y1, X1, Z1;
    int Yoe, Xoe, Yoo, Xoo;
    int pe, po;     // plane sizes (elements)
};

// Ring slots: even plane z -> (z/2) mod 8, odd plane z -> ((z-1)/2) mod 5.
// Step m reads even planes 4m-8 .. 4m+2 and odd planes 4m-7 .. 4m-3 while the
// next step's planes (4m+4, 4m+6; 4m-1, 4m+1) land in the remaining slots.
__device__ __forceinline__ int slot_off(const TileCtx &C, int z) {
    return (z & 1) ? kTileEvenSlots * C.pe + (((z >> 1) + 40) % kTileOddSlots) * C.po : ((z >> 1) & 7) * C.pe;
}

// Outlier rank of the zero code at stream position pos of commit cm:
// esc_off of its (item, warp) plus the zero codes before it in that range.
__device__ __noinline__ double tile_outlier(const TileCommit &cm, const TileRun &A, int64_t pos) {
    const int64_t item = pos / cm.p_item;
    const int64_t w = (pos - item * cm.p_item) / cm.pw;
    const int64_t e = (int64_t)(cm.item_base + item) * kItemWarps + w;
    const uint16_t *codes = (const uint16_t *)A.codes + cm.code_base;
    int64_t r = A.esc_off[e];
    for (int64_t q = item * cm.p_item + w * cm.pw; q < pos; q++) r += codes[q] == 0;
    if (r < A.outl_cap) return A.outl[r];
    atomicExch(A.flags, HPEZ_OUTLIER_UNDERFLOW);
    return 0.0;
}

__device__ __noinline__ void tile_escape(const TileCommit &cm, const TileRun &A, int64_t pos) {
    const int64_t item = pos / cm.p_item;
    const int64_t w = (pos - item * cm.p_item) / cm.pw;
    atomicAdd(A.esc_cnt + (int64_t)(cm.item_base + item) * kItemWarps + w, 1u);
}

// grid axis of blend term t for predictor layout KIND (0..2: 1-D along that
// axis; 3..5: MD over (0,1) (0,2) (1,2); 6: MD over (0,1,2))
template <int KIND> __device__ constexpr int tk_axis(int t) {
    return KIND < 3 ? KIND : KIND == 3 ? (t == 0 ? 0 : 1) : KIND == 4 ? (t == 0 ? 0 : 2) : KIND == 5 ? (t == 0 ? 1 : 2) : t;
}

// plane z of selector sel at macro-step m
__device__ __forceinline__ int sel_plane(int sel, int m) {
    return sel == 0 ? 4 * m : sel == 1 ? 4 * m + 2 : sel == 2 ? 4 * m - 3 : 4 * m - 5;
}
__device__ __forceinline__ bool plane_needed(const TileDesc &D, const TileCtx &C, int z) {
    if (z < 0 || z >= D.L[0]) return false;
    return (z & 1) ? (z >= C.Z0 + 1 && z <= C.Z1 + 1) : (z >= C.Z0 - 2 && z <= C.Z1 + 4);
}

constexpr int kUnit = 64;  // points per warp work unit (two per lane)

struct TaskGeo {  // per CTA and task (interval order): the need box on the commit lattice
    int32_t ci, sel;
    int32_t jy0, ny, jx0, nx;
    FastDiv fd;   // division by nx
    int32_t u0, nu;  // first unit within its interval, unit count
};

// Shared-memory layout after the rings (element counts, see tile_smem_bytes).
struct TileSmem {
    TaskGeo *tg;     // [kTileMaxTasks]
    int32_t *ivu;    // [kTileMaxIntervals] units per interval
    int32_t *slot;   // [16] ring offsets of planes 4m-8 .. 4m+7 of the current step
    int32_t *rowe, *rowo;  // [RYe], [RYo] row element offsets y*E1 (-1 outside the grid)
};

// One work unit: kUnit consecutive points (row-major over the need box) of
// task (commit cm, plane z).  Each lane computes two points: both points'
// stencils are loaded before either is used.
template <int DIR, int KIND, int FAM>
__device__ __forceinline__ void tile_unit(const TileDesc &D, const TileCtx &C, const TileRun &A, double *sm,
                                          const int32_t *slot, int zlo, const TaskGeo &g, const TileCommit &cm,
                                          int z, int t0) {
    constexpr int NAX = KIND < 3 ? 1 : KIND < 6 ? 2 : 3;
    constexpr int NF = Fam<FAM>::n;
    const int lane = threadIdx.x & 31;
    const int n = g.ny * g.nx;
    const bool zodd = z & 1;
    const int RXe = D.RXe, RXo = D.RXo, hXe = RXe >> 1, hXo = RXo >> 1;
    const int RX = zodd ? RXo : RXe;
    const int half = RX >> 1;
    const int Xo = zodd ? C.Xoo : C.Xoe;
    const int tb = slot[z - zlo];
    int zb[7];
#pragma unroll
    for (int d = 0; d < 7; d++) zb[d] = (KIND == 0 || KIND == 3 || KIND == 4 || KIND == 6) ? slot[z + d - 3 - zlo] : 0;
    const int px = (g.jx0 - Xo) & 1;  // parity of every target column of this commit
    int xd[NF];
#pragma unroll
    for (int i = 0; i < NF; i++) xd[i] = xdelta(px, Fam<FAM>::u(i), half);
    const int shy = cm.sh[1], shx = cm.sh[2];
    const int L0 = D.L[0], L1 = D.L[1], L2 = D.L[2];
    const bool owned_z = z >= C.Z0 && z < C.Z1;
    const int Yoe = C.Yoe, Xoe = C.Xoe, Yoo = C.Yoo, Xoo = C.Xoo;
    const int Y0 = C.Y0, Y1 = C.Y1, X0 = C.X0, X1 = C.X1;
    const int jy0 = g.jy0, jx0 = g.jx0, gnx = g.nx;
    const FastDiv fd = g.fd;
    int jy[2], jx[2], toff[2], offe[2], offo[2];
    bool valid[2];
    bool in_all = true;
    double x[2][NAX][6];
#pragma unroll
    for (int p = 0; p < 2; p++) {
        const int t = t0 + p * 32 + lane;
        valid[p] = t < n;
        const int tt = valid[p] ? t : 0;
        const int r = (int)fdiv((uint32_t)tt, fd);
        const int k = tt - r * gnx;
        jy[p] = jy0 + (r << shy);
        jx[p] = jx0 + (k << shx);
        offe[p] = (jy[p] - Yoe) * RXe + ring_x(jx[p], Xoe, hXe);
        offo[p] = (jy[p] - Yoo) * RXo + ring_x(jx[p], Xoo, hXo);
        toff[p] = tb + (zodd ? offo[p] : offe[p]);
        const int crd[3] = {z, jy[p], jx[p]};
        const int Lv[3] = {L0, L1, L2};
#pragma unroll
        for (int t3 = 0; t3 < NAX; t3++) {
            const int a = tk_axis<KIND>(t3);
            in_all &= Fam<FAM>::interior(crd[a], Lv[a], 1) || !valid[p];
#pragma unroll
            for (int i = 0; i < NF; i++) {
                const int u = Fam<FAM>::u(i);
                int o;
                if (a == 0) o = zb[u + 3] + ((u & 1) ? offe[p] : offo[p]);  // odd target: odd u -> even plane
                else if (a == 1) o = toff[p] + u * RX;
                else o = toff[p] + xd[i];
                x[p][t3][i] = sm[o];
            }
        }
    }
    double pred[2];
    const bool fast = __all_sync(0xffffffffu, in_all);
#pragma unroll
    for (int p = 0; p < 2; p++) {
        const int crd[3] = {z, jy[p], jx[p]};
        const int Lv[3] = {L0, L1, L2};
        double pt[NAX];
#pragma unroll
        for (int t3 = 0; t3 < NAX; t3++) {
            const int a = tk_axis<KIND>(t3);
            if (fast || Fam<FAM>::interior(crd[a], Lv[a], 1)) pt[t3] = Fam<FAM>::combine(x[p][t3]);
            else pt[t3] = edge_row<FAM>(x[p][t3], crd[a], Lv[a], 1);
        }
        if (NAX == 1) pred[p] = pt[0];
        else if (NAX == 2) pred[p] = DA(DM(cm.w[0], pt[0]), DM(cm.w[1], pt[NAX - 1]));
        else pred[p] = DA(DA(DM(cm.w[0], pt[0]), DM(cm.w[1], pt[1])), DM(cm.w[2], pt[NAX - 1]));
    }
    const int32_t R = D.R;
    const int zrow = ((z - cm.st[0]) >> cm.sh[0]) * cm.cnt[1];
    const int gz = z * D.E0;
#pragma unroll
    for (int p = 0; p < 2; p++) {
        if (!valid[p]) continue;
        const bool owned = owned_z && jy[p] >= Y0 && jy[p] < Y1 && jx[p] >= X0 && jx[p] < X1;
        const int pos = (zrow + ((jy[p] - cm.st[1]) >> shy)) * cm.cnt[2] + ((jx[p] - cm.st[2]) >> shx);
        const int gidx = D.s * (gz + jy[p] * D.E1 + jx[p]);
        if (DIR == HPEZ_COMPRESS) {
            double out;
            const int32_t code =
                quantize_point<HPEZ_ROUND_F32>(sm[toff[p]], pred[p], D.bound, D.two_e, D.inv_two_e, (double)R, R, &out);
            sm[toff[p]] = out;
            if (owned) {
                ((uint16_t *)A.codes)[cm.code_base + pos] = (uint16_t)code;
                ((float *)A.work)[gidx] = (float)out;
                if (code == 0) tile_escape(cm, A, pos);
            }
        } else {
            const int64_t code = (int64_t)__double_as_longlong(sm[toff[p]]);
            double val;
            if (code != 0) val = dequantize_point<HPEZ_ROUND_F32>(pred[p], code, D.two_e, (int64_t)R);
            else val = (double)(float)tile_outlier(cm, A, pos);
            sm[toff[p]] = val;
            if (owned) ((float *)A.work)[gidx] = (float)val;
        }
    }
}

template <int DIR>
__device__ __forceinline__ void tile_unit_dispatch(const TileDesc &D, const TileCtx &C, const TileRun &A, double *sm,
                                                   const int32_t *slot, int zlo, const TaskGeo &g, int z, int t0) {
    const TileCommit &cm = D.c[g.ci];
#define HPEZ_TK(K, F)                                                     \
    case K * 5 + F:                                                       \
        tile_unit<DIR, K, F>(D, C, A, sm, slot, zlo, g, cm, z, t0);       \
        return;
    switch (cm.kind * 5 + cm.fam) {
        HPEZ_TK(0, 0) HPEZ_TK(0, 1) HPEZ_TK(0, 2) HPEZ_TK(0, 3) HPEZ_TK(0, 4)
        HPEZ_TK(1, 0) HPEZ_TK(1, 1) HPEZ_TK(1, 2) HPEZ_TK(1, 3) HPEZ_TK(1, 4)
        HPEZ_TK(2, 0) HPEZ_TK(2, 1) HPEZ_TK(2, 2) HPEZ_TK(2, 3) HPEZ_TK(2, 4)
        HPEZ_TK(3, 0) HPEZ_TK(3, 1) HPEZ_TK(3, 2)
        HPEZ_TK(4, 0) HPEZ_TK(4, 1) HPEZ_TK(4, 2)
        HPEZ_TK(5, 0) HPEZ_TK(5, 1) HPEZ_TK(5, 2)
        HPEZ_TK(6, 0) HPEZ_TK(6, 1) HPEZ_TK(6, 2)
    default:
        break;
    }
#undef HPEZ_TK
}

__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Stream position of the non-coarse sublattice point (z, y, x).
__device__ __forceinline__ int64_t code_pos(const TileDesc &D, int z, int y, int x) {
    const TileCommit &cm = D.c[D.lut[((z & 3) << 4) | ((y & 3) << 2) | (x & 3)]];
    return cm.code_base + ((int64_t)((z - cm.st[0]) >> cm.sh[0]) * cm.cnt[1] + ((y - cm.st[1]) >> cm.sh[1])) * cm.cnt[2] +
           ((x - cm.st[2]) >> cm.sh[2]);
}

// Row r of the load set of step m: even planes 4m, 4m+2 (RYe rows each),
// then odd planes 4m-3, 4m-5 (RYo rows each).  Returns the plane (or -1).
__device__ __forceinline__ int load_row(const TileDesc &D, const TileCtx &C, int m, int r, int *rr, bool *even) {
    int sel;
    if (r < 2 * D.RYe) {
        sel = r >= D.RYe;
        *rr = r - sel * D.RYe;
    } else {
        r -= 2 * D.RYe;
        sel = 2 + (r >= D.RYo);
        *rr = r - (sel - 2) * D.RYo;
    }
    *even = sel < 2;
    const int z = sel_plane(sel, m);
    return plane_needed(D, C, z) ? z : -1;
}

// Asynchronous copies of step m's planes into their (dead) ring slots: one
// 32-bit word per point in the low half of its f64 slot -- compress: the
// original (targets) or reconstruction (coarse); decompress: the coarse value
// or the aligned code word holding the point's u16 code.
template <int DIR, int NT>
__device__ __forceinline__ void issue_loads(const TileDesc &D, const TileCtx &C, const TileRun &A, const TileSmem &S,
                                            int m, double *sm) {
    constexpr int NW = NT / 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nr = 2 * D.RYe + 2 * D.RYo;
    const float *orig = (const float *)A.orig;
    const float *work = (const float *)A.work;
    const uint16_t *codes = (const uint16_t *)A.codes;
    const int s = D.s, L2 = D.L[2];
    for (int r = warp; r < nr; r += NW) {
        int rr;
        bool even;
        const int z = load_row(D, C, m, r, &rr, &even);
        if (z < 0) continue;
        const int rowg = (even ? S.rowe : S.rowo)[rr];
        if (rowg < 0) continue;
        const int RX = even ? D.RXe : D.RXo, Xo = even ? C.Xoe : C.Xoo;
        const int half = RX >> 1;
        double *srow = sm + slot_off(C, z) + rr * RX;
        const int gbase = z * D.E0 + rowg;
        const int jy = (even ? C.Yoe : C.Yoo) + rr;
        for (int col = lane; col < RX; col += 32) {
            const int jx = Xo + col;
            if (jx < 0 || jx >= L2) continue;
            double *dst = srow + (col & 1) * half + (col >> 1);
            const int gi = s * (gbase + jx);
            const bool coarse = !((z | jy | jx) & 1);
            if (DIR == HPEZ_COMPRESS) {
                cp_async4(dst, coarse ? work + gi : orig + gi);
            } else if (coarse) {
                cp_async4(dst, work + gi);
            } else {
                const int64_t pos = code_pos(D, z, jy, jx);
                if (pos + 1 < D.n_codes || (pos & 1)) cp_async4(dst, codes + (pos & ~(int64_t)1));
                else *(uint32_t *)dst = codes[pos];  // last code, even index: no word past the end
            }
        }
    }
    cp_async_commit();
}

// Widen step m's planes in place: low word -> f64 value, or the code
// (decompress targets) as an integer payload.
template <int DIR, int NT>
__device__ __forceinline__ void widen_planes(const TileDesc &D, const TileCtx &C, int m, double *sm) {
    if (DIR == HPEZ_COMPRESS) {
#pragma unroll 1
        for (int sel = 0; sel < 4; sel++) {
            const int z = sel_plane(sel, m);
            if (!plane_needed(D, C, z)) continue;
            double *base = sm + slot_off(C, z);
            const int np = (z & 1) ? C.po : C.pe;
            for (int i = threadIdx.x; i < np; i += NT) base[i] = (double)__uint_as_float(*(const uint32_t *)(base + i));
        }
        return;
    }
    constexpr int NW = NT / 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nr = 2 * D.RYe + 2 * D.RYo;
    for (int r = warp; r < nr; r += NW) {
        int rr;
        bool even;
        const int z = load_row(D, C, m, r, &rr, &even);
        if (z < 0) continue;
        const int RX = even ? D.RXe : D.RXo, Xo = even ? C.Xoe : C.Xoo;
        const int jy = (even ? C.Yoe : C.Yoo) + rr;
        if (jy < 0 || jy >= D.L[1]) continue;
        const int half = RX >> 1;
        double *srow = sm + slot_off(C, z) + rr * RX;
        for (int col = lane; col < RX; col += 32) {
            const int lx = col < half ? 2 * col : 2 * (col - half) + 1;
            const int jx = Xo + lx;
            if (jx < 0 || jx >= D.L[2]) continue;
            double *slot = srow + col;
            const uint32_t wv = *(const uint32_t *)slot;
            if (!((z | jy | jx) & 1)) {
                *slot = (double)__uint_as_float(wv);
            } else {
                const int64_t pos = code_pos(D, z, jy, jx);
                *slot = __longlong_as_double((long long)((pos & 1) ? (wv >> 16) : (wv & 0xffffu)));
            }
        }
    }
}

template <int DIR, int NT>
__global__ void __launch_bounds__(NT, NT <= 256 ? 2 : 1) tile_level_kernel(const __grid_constant__ TileDesc D, const TileRun A) {
    constexpr int NW = NT / 32;
    extern __shared__ __align__(16) double tsm[];
    TileCtx C;
    int b = blockIdx.x;
    const int tx = b % D.tiles_x;
    b /= D.tiles_x;
    const int ty = b % D.tiles_y;
    const int tz = b / D.tiles_y;
    C.Y0 = ty * D.TY;
    C.X0 = tx * D.TX;
    C.Z0 = tz * D.ZC;
    C.Y1 = min(C.Y0 + D.TY, D.L[1]);
    C.X1 = min(C.X0 + D.TX, D.L[2]);
    C.Z1 = min(C.Z0 + D.ZC, D.L[0]);
    C.Yoe = C.Y0 - D.HYe;
    C.Xoe = C.X0 - D.HXe;
    C.Yoo = C.Y0 - D.HYo;
    C.Xoo = C.X0 - D.HXo;
    C.pe = D.RYe * D.RXe;
    C.po = D.RYo * D.RXo;
    TileSmem S;
    S.tg = (TaskGeo *)(tsm + kTileEvenSlots * C.pe + kTileOddSlots * C.po);
    S.ivu = (int32_t *)(S.tg + kTileMaxTasks);
    S.slot = S.ivu + kTileMaxIntervals;
    S.rowe = S.slot + 16;
    S.rowo = S.rowe + D.RYe;
    const int ntask = D.iv_off[D.n_iv];
    const int warp = threadIdx.x >> 5;
    for (int k = threadIdx.x; k < ntask; k += NT) {
        const int ci = D.task_c[k];
        const TileCommit &cm = D.c[ci];
        const int ylo = max(C.Y0 - cm.box[0], 0), yhi = min(C.Y1 - 1 + cm.box[1], D.L[1] - 1);
        const int xlo = max(C.X0 - cm.box[2], 0), xhi = min(C.X1 - 1 + cm.box[3], D.L[2] - 1);
        const int ky = 1 << cm.sh[1], kx = 1 << cm.sh[2];
        const int iy0 = ylo <= cm.st[1] ? 0 : (ylo - cm.st[1] + ky - 1) >> cm.sh[1];
        const int iy1 = yhi < cm.st[1] ? -1 : (yhi - cm.st[1]) >> cm.sh[1];
        const int ix0 = xlo <= cm.st[2] ? 0 : (xlo - cm.st[2] + kx - 1) >> cm.sh[2];
        const int ix1 = xhi < cm.st[2] ? -1 : (xhi - cm.st[2]) >> cm.sh[2];
        TaskGeo gg;
        gg.ci = ci;
        gg.sel = D.task_sel[k];
        gg.jy0 = cm.st[1] + (iy0 << cm.sh[1]);
        gg.ny = max(0, iy1 - iy0 + 1);
        gg.jx0 = cm.st[2] + (ix0 << cm.sh[2]);
        gg.nx = max(0, ix1 - ix0 + 1);
        gg.fd = dev_fastdiv((uint32_t)max(gg.nx, 1));
        gg.u0 = 0;
        gg.nu = (gg.ny * gg.nx + kUnit - 1) / kUnit;
        S.tg[k] = gg;
    }
    for (int r = threadIdx.x; r < D.RYe; r += NT) {
        const int y = C.Yoe + r;
        S.rowe[r] = y >= 0 && y < D.L[1] ? y * D.E1 : -1;
    }
    for (int r = threadIdx.x; r < D.RYo; r += NT) {
        const int y = C.Yoo + r;
        S.rowo[r] = y >= 0 && y < D.L[1] ? y * D.E1 : -1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int iv = 0; iv < D.n_iv; iv++) {
            int u = 0;
            for (int k = D.iv_off[iv]; k < D.iv_off[iv + 1]; k++) {
                S.tg[k].u0 = u;
                u += S.tg[k].nu;
            }
            S.ivu[iv] = u;
        }
    }
    const int m0 = floor_div4(C.Z0 - 2);
    const int m1 = floor_div4(min(C.Z1 + 1, D.L[0] - 1) + 5);
    if (threadIdx.x < 16) S.slot[threadIdx.x] = slot_off(C, 4 * m0 - 8 + (int)threadIdx.x);
    issue_loads<DIR, NT>(D, C, A, S, m0, tsm);
    cp_async_wait_all();
    __syncthreads();
    widen_planes<DIR, NT>(D, C, m0, tsm);
    __syncthreads();
    for (int m = m0; m <= m1; m++) {
        if (m < m1) issue_loads<DIR, NT>(D, C, A, S, m + 1, tsm);
        const int zlo = 4 * m - 8;
        for (int iv = 0; iv < D.n_iv; iv++) {
            const int nu = S.ivu[iv];
            const int k0 = D.iv_off[iv];
            for (int u = warp; u < nu; u += NW) {
                int k = k0;
                while (u >= S.tg[k].u0 + S.tg[k].nu) k++;
                const TaskGeo g = S.tg[k];
                const int z = sel_plane(g.sel, m);
                if (!plane_needed(D, C, z)) continue;
                tile_unit_dispatch<DIR>(D, C, A, tsm, S.slot, zlo, g, z, (u - g.u0) * kUnit);
            }
            __syncthreads();
        }
        if (m < m1) {
            cp_async_wait_all();
            __syncthreads();
            widen_planes<DIR, NT>(D, C, m + 1, tsm);
            if (threadIdx.x < 16) S.slot[threadIdx.x] = slot_off(C, 4 * (m + 1) - 8 + (int)threadIdx.x);
            __syncthreads();
        }
    }
}

// ------------------------------------------------------------------ host --
namespace {

struct Read {
    int axis;
    int reach;               // max |offset|
    std::vector<int> from;   // commits read
};

int fam_odd_reach(int fam) { return fam == FAM_LIN_I || fam == FAM_NAK_S ? 1 : 3; }

}  // namespace

bool tile_plan_build(const GridDev &g, const CommitDev *cms, int n, int64_t n_codes, TilePlan *out) {
    if (g.rank != 3 || n <= 0 || n > kTileMaxCommits) return false;
    TileDesc D{};
    const int s = cms[0].s;
    D.s = s;
    for (int a = 0; a < 3; a++) D.L[a] = (g.dims[a] - 1) / s + 1;
    D.E0 = g.estr[0];
    D.E1 = g.estr[1];
    D.R = (int32_t)g.radius;
    D.bound = cms[0].bound;
    D.two_e = cms[0].two_e;
    D.inv_two_e = cms[0].inv_two_e;
    D.n_commits = n;
    D.n_codes = n_codes;
    for (int i = 0; i < 64; i++) D.lut[i] = -1;
    for (int i = 0; i < n; i++) {
        const CommitDev &c = cms[i];
        if (c.kind != COMMIT_UNIFORM || c.s != s || c.bound != D.bound) return false;
        TileCommit &t = D.c[i];
        t.split = -1;
        t.v = 0;
        for (int a = 0; a < 3; a++) {
            if (c.start[a] % s || c.step[a] % s) return false;
            const int st = c.start[a] / s, sp = c.step[a] / s;
            if (sp != 2 && sp != 4) return false;  // frozen axis (step 1) not tiled
            t.st[a] = st;
            t.sh[a] = sp == 2 ? 1 : 2;
            t.cnt[a] = c.cnt[a];
            if (st & 1) t.v |= 1 << a;
            if (sp == 4) {
                t.split = a;
                t.phase = st == 3;
            }
        }
        t.odd = t.v & 1;
        t.item_base = c.item_base;
        t.p_item = c.p_item;
        t.pw = c.pw;
        t.code_base = c.code_base;
        t.fam = c.pred.fam;
        if (c.pred.md) {
            t.nax = c.pred.nax;
            for (int k = 0; k < t.nax; k++) {
                t.axes[k] = c.pred.axes[k];
                t.w[k] = c.pred.w[k];
            }
        } else {
            t.nax = 1;
            t.axes[0] = c.pred.axis;
        }
        if (t.nax == 1) t.kind = t.axes[0];
        else if (t.nax == 3) t.kind = 6;
        else t.kind = t.axes[0] == 0 ? (t.axes[1] == 1 ? 3 : 4) : 5;
        if (t.nax > 1 && t.fam > FAM_NAT_I) return false;
        // lattice residues mod 4 -> commit
        for (int r = 0; r < 64; r++) {
            const int rr[3] = {r >> 4, (r >> 2) & 3, r & 3};
            bool in = true;
            for (int a = 0; a < 3; a++) in &= ((rr[a] - t.st[a]) & ((1 << t.sh[a]) - 1)) == 0;
            if (in) {
                if (D.lut[r] >= 0) return false;
                D.lut[r] = (int8_t)i;
            }
        }
    }
    for (int r = 0; r < 64; r++) {
        const bool coarse = !((r >> 4) & 1) && !((r >> 2) & 1) && !(r & 1);
        if (coarse != (D.lut[r] < 0)) return false;  // every non-coarse residue owned by one commit
    }
    // reads of each commit
    std::vector<std::vector<Read>> reads(n);
    for (int i = 0; i < n; i++) {
        const TileCommit &t = D.c[i];
        for (int k = 0; k < t.nax; k++) {
            const int a = t.axes[k];
            Read rd{a, fam_odd_reach(t.fam), {}};
            const int w = t.v & ~(1 << a);
            for (int j = 0; j < i; j++)
                if (w && D.c[j].v == w) rd.from.push_back(j);
            reads[i].push_back(rd);
            if (t.fam == FAM_NAK_S || t.fam == FAM_NAT_S) {  // same-level: phase-0 points at +-2
                Read sl{a, 2, {}};
                for (int j = 0; j < i; j++)
                    if (D.c[j].v == t.v && D.c[j].phase == 0) sl.from.push_back(j);
                reads[i].push_back(sl);
            }
        }
    }
    // need boxes (owned tile grown by consumers' reads), reverse reference order
    std::vector<std::array<int, 4>> box(n, {0, 0, 0, 0});
    for (int i = n - 1; i >= 0; i--)
        for (const Read &rd : reads[i])
            for (int j : rd.from) {
                std::array<int, 4> b = box[i];
                if (rd.axis == 1) b[0] += rd.reach, b[1] += rd.reach;
                if (rd.axis == 2) b[2] += rd.reach, b[3] += rd.reach;
                for (int q = 0; q < 4; q++) box[j][q] = std::max(box[j][q], b[q]);
            }
    int hye = 0, hxe = 0, hyo = 0, hxo = 0;
    for (int i = 0; i < n; i++) {
        TileCommit &t = D.c[i];
        for (int q = 0; q < 4; q++) t.box[q] = box[i][q];
        int ry = 0, rx = 0;  // in-plane read reach
        for (const Read &rd : reads[i]) {
            if (rd.axis == 1) ry = std::max(ry, rd.reach);
            if (rd.axis == 2) rx = std::max(rx, rd.reach);
        }
        const int by = std::max(box[i][0], box[i][1]), bx = std::max(box[i][2], box[i][3]);
        if (t.odd) {
            hyo = std::max(hyo, by + ry);
            hxo = std::max(hxo, bx + rx);
            hye = std::max(hye, by);  // z reads land on even planes at the same (y, x)
            hxe = std::max(hxe, bx);
        } else {
            hye = std::max(hye, by + ry);
            hxe = std::max(hxe, bx + rx);
        }
    }
    D.HYe = hye;
    D.HYo = hyo;
    D.HXe = (hxe + 1) & ~1;
    D.HXo = (hxo + 1) & ~1;
    // schedule: tasks (plane selector, commit) in dependency intervals
    std::vector<int> tsel, tc, tt;
    std::vector<std::vector<int>> tidx(4, std::vector<int>(n, -1));
    for (int sel = 0; sel < 4; sel++)
        for (int i = 0; i < n; i++) {
            const TileCommit &t = D.c[i];
            if ((sel < 2) == (bool)t.odd) continue;
            if (sel >= 2 && t.split == 0 && t.phase != (sel == 3)) continue;
            int tm = 0;
            for (const Read &rd : reads[i])
                for (int j : rd.from) {
                    if (rd.axis != 0) {
                        if (tidx[sel][j] >= 0) tm = std::max(tm, tt[tidx[sel][j]] + 1);
                    } else if (rd.reach == 2) {  // z same-level: plane z+2 is the selector-2 plane
                        if (sel != 3 || tidx[2][j] < 0) return false;
                        tm = std::max(tm, tt[tidx[2][j]] + 1);
                    } else if (sel == 2 && rd.reach >= 3) {  // plane (4m-3)+3 = 4m: selector 0 of this step
                        if (tidx[0][j] < 0) return false;
                        tm = std::max(tm, tt[tidx[0][j]] + 1);
                    }
                }
            tidx[sel][i] = (int)tt.size();
            tsel.push_back(sel);
            tc.push_back(i);
            tt.push_back(tm);
        }
    const int niv = tt.empty() ? 0 : *std::max_element(tt.begin(), tt.end()) + 1;
    if (niv > kTileMaxIntervals || (int)tt.size() > kTileMaxTasks) return false;
    D.n_iv = niv;
    int k = 0;
    for (int iv = 0; iv < niv; iv++) {
        D.iv_off[iv] = k;
        for (size_t q = 0; q < tt.size(); q++)
            if (tt[q] == iv) {
                D.task_sel[k] = (int8_t)tsel[q];
                D.task_c[k] = (int8_t)tc[q];
                k++;
            }
    }
    D.iv_off[niv] = k;
    // tiling
    int TY = 16, TX = 32;
    if (const char *e = getenv("HPEZ_TILE_TY")) TY = std::max(4, atoi(e) & ~3);
    if (const char *e = getenv("HPEZ_TILE_TX")) TX = std::max(4, atoi(e) & ~3);
    TY = std::min(TY, (D.L[1] + 3) & ~3);
    TX = std::min(TX, (D.L[2] + 3) & ~3);
    D.TY = TY;
    D.TX = TX;
    D.RYe = TY + 2 * D.HYe;
    D.RXe = TX + 2 * D.HXe;
    D.RYo = TY + 2 * D.HYo;
    D.RXo = TX + 2 * D.HXo;
    D.tiles_y = (D.L[1] + TY - 1) / TY;
    D.tiles_x = (D.L[2] + TX - 1) / TX;
    int sms = 148;
    {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const size_t smem = (size_t)(kTileEvenSlots * D.RYe * D.RXe + kTileOddSlots * D.RYo * D.RXo) * sizeof(double) +
                        kTileMaxTasks * sizeof(TaskGeo) + (kTileMaxIntervals + 16 + D.RYe + D.RYo) * sizeof(int32_t);
    if (smem > 227 * 1024) return false;
    const int per_sm = std::max(1, (int)((228 * 1024) / (smem + 1024)));
    const int cols = D.tiles_y * D.tiles_x;
    int ZC = 64;
    if (const char *e = getenv("HPEZ_TILE_ZC")) ZC = std::max(4, atoi(e) & ~3);
    else {
        // enough CTAs for ~2 waves, chunks of at least 16 planes
        const int want = 2 * per_sm * sms;
        const int chunks = std::max(1, want / std::max(cols, 1));
        ZC = std::max(16, ((D.L[0] + chunks - 1) / chunks + 3) & ~3);
    }
    D.ZC = std::min(ZC, (D.L[0] + 3) & ~3);
    D.chunks_z = (D.L[0] + D.ZC - 1) / D.ZC;
    out->threads = 256;
    if (const char *e = getenv("HPEZ_TILE_NT")) out->threads = atoi(e) == 512 ? 512 : 256;
    out->d = D;
    out->grid = cols * D.chunks_z;
    out->smem = smem;
    return true;
}

template <int DIR>
static cudaError_t launch_dir(const TilePlan &p, const TileRun &r, cudaStream_t st) {
    if (p.threads == 256) {
        auto f = tile_level_kernel<DIR, 256>;
        cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
        if (e) return e;
        f<<<p.grid, 256, p.smem, st>>>(p.d, r);
    } else {
        auto f = tile_level_kernel<DIR, 512>;
        cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
        if (e) return e;
        f<<<p.grid, 512, p.smem, st>>>(p.d, r);
    }
    return cudaGetLastError();
}

cudaError_t tile_plan_launch(const TilePlan &p, int dir, const TileRun &r, cudaStream_t st) {
    if (p.grid <= 0) return cudaSuccess;
    return dir == HPEZ_COMPRESS ? launch_dir<HPEZ_COMPRESS>(p, r, st) : launch_dir<HPEZ_DECOMPRESS>(p, r, st);
}

}  // namespace hpez
