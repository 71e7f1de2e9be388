// row.cu -- the finest level of a rank-3 multidim sweep, one warp per grid row.
//
// Reference: interp._LevelRunner.run_level (interp.py:415-433) at stride 1,
// classes on the uniform path (interp.py:322-341) or the mixed per-block path
// (interp.py:350-411) with multidim variants (plan.KERNEL_VARIANTS 0..4,
// plan.py:25-31): classes of one axis predict 1-D along it (with the
// two-pass same-level split for variants 2 and 4), classes of two or three
// axes blend the inter-level rows of their axes (interp.py:300-311).
//
// Geometry.  A row (fixed z, y) holds two classes: its x-even points (class
// E = the odd axes among z, y; coarse points when z and y are even) and its
// x-odd points (class O = E + x).  Class E reads only OTHER rows (z +- 1, 3
// and/or y +- 1, 3; +- 2 for its second same-level pass); class O reads the
// same rows at odd x plus the row's own x-even values.  So a warp that owns
// the row loads each neighbouring row once with 16-byte loads, serves both
// classes from it, keeps the row's fresh values in a shared-memory row
// buffer (f64) for the in-row stencil, and writes the finished row back as
// complete 16-byte words.  Rows of one parity type depend only on rows of
// earlier types, so the level is 3-4 plain launches:
//   (z even, y even)  ->  (z odd, y even) + (z even, y odd)  ->  (z odd, y odd)
// with the middle one split in two when a same-level variant is present
// (first-pass rows z or y = 1 mod 4, then second-pass rows = 3 mod 4).
//
// Stream order.  Codes of a class are its first-pass members in row-major
// lattice order, then its second-pass members (interp.py:333-341, 374-411);
// a setup kernel counts the members of every (class, pass, row) and an
// exclusive scan turns the counts into the row's first code index.
// Escapes use the sweep plan's (item, warp) bookkeeping (sweep.cu).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "row.h"
#include "scan.cuh"
#include "stencil.cuh"

namespace hpez {

#ifndef HPEZ_ROW_OCC
#define HPEZ_ROW_OCC 3
#endif
constexpr int kRowWarps = 8;
constexpr int kRowThreads = kRowWarps * 32;

__host__ __device__ __forceinline__ int cnt_mod(int lo, int hi, int r, int m) {
    return (hi + m - 1 - r) / m - (lo + m - 1 - r) / m;  // j in [lo, hi) with j = r mod m
}
__host__ __device__ __forceinline__ bool variant_same(int k) { return k == 2 || k == 4; }
__host__ __device__ __forceinline__ int variant_fam(int k) { return (k + 1) >> 1; }  // 0 linear, 1 not-a-knot, 2 natural

__host__ __device__ constexpr int class_vmask(int c) {
    return c == 0 ? 1 : c == 1 ? 2 : c == 2 ? 4 : c == 3 ? 3 : c == 4 ? 5 : c == 5 ? 6 : 7;
}

// ------------------------------------------------------------ row bases --
// Members of (class c, pass b) in class row r: the mixed membership rule of
// interp.py:374-411, which for a constant tag is the uniform two-phase split
// of interp.py:333-341.
__global__ void __launch_bounds__(256) row_count_kernel(const __grid_constant__ RowDesc D,
                                                        const uint8_t *__restrict__ table, uint32_t *__restrict__ cnt) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= D.n_entries) return;
    int c = 0, b = 0;
    int64_t r = 0;
    for (int k = 0; k < 7; k++) {
        if (D.segA[k] >= 0 && i >= D.segA[k]) {
            c = k;
            b = 0;
            r = i - D.segA[k];
        }
        if (D.segB[k] >= 0 && i >= D.segB[k]) {
            c = k;
            b = 1;
            r = i - D.segB[k];
        }
    }
    const int vm = class_vmask(c);
    const int vz = vm & 1, vy = (vm >> 1) & 1, vx = (vm >> 2) & 1;
    const int cny = D.cny[vy];
    const int z = 2 * (int)(r / cny) + vz, y = 2 * (int)(r % cny) + vy;
    const int Lx = D.L[2];
    const bool single = vm == 1 || vm == 2 || vm == 4;
    const int nbx = D.has_table ? ((Lx - 1) >> D.bsh) + 1 : 1;
    uint32_t n = 0;
    for (int bx = 0; bx < nbx; bx++) {
        const int lo = D.has_table ? bx << D.bsh : 0;
        const int hi = D.has_table ? min(Lx, (bx + 1) << D.bsh) : Lx;
        const int k = D.has_table ? table[(z >> D.bsh) * D.bs0 + (y >> D.bsh) * D.bs1 + bx] : D.const_k;
        const int all = cnt_mod(lo, hi, vx, 2);
        int nA = all, nB = 0;
        if (single && variant_same(k)) {
            if (vm == 1) {
                nA = (z & 3) == 1 ? all : 0;
                nB = all - nA;
            } else if (vm == 2) {
                nA = (y & 3) == 1 ? all : 0;
                nB = all - nA;
            } else {
                nA = cnt_mod(lo, hi, 1, 4);
                nB = cnt_mod(lo, hi, 3, 4);
            }
        }
        n += b ? nB : nA;
    }
    cnt[i] = n;
}

// ----------------------------------------------------------- predictors --
__device__ __noinline__ double edge_inter(int fi, double m3, double m1, double p1, double p3, int c, int E) {
    const double x[6] = {m3, m1, p1, p3, 0.0, 0.0};
    return fi == 1 ? edge_row<FAM_NAK_I>(x, c, E, 1) : edge_row<FAM_NAT_I>(x, c, E, 1);
}

// Inter-level 1-D row of family fi at lattice coordinate c (extent E) over
// the values at c-3, c-1, c+1, c+3 (kernels.py:43-86; edge rows 106-150).
__device__ __forceinline__ double pred_inter(int fi, double m3, double m1, double p1, double p3, int c, int E) {
    if (fi == 0) return (c + 1 <= E - 1) ? DA(DM(0.5, m1), DM(0.5, p1)) : DM(1.0, m1);
    if (c >= 3 && c + 3 <= E - 1) {
        if (fi == 1) return DA(DA(DA(DM(-1.0 / 16, m3), DM(9.0 / 16, m1)), DM(9.0 / 16, p1)), DM(-1.0 / 16, p3));
        return DA(DA(DA(DM(-3.0 / 40, m3), DM(23.0 / 40, m1)), DM(23.0 / 40, p1)), DM(-3.0 / 40, p3));
    }
    return edge_inter(fi, m3, m1, p1, p3, c, E);
}

// Same-level 1-D row (second pass of a split class) over c-3 .. c+3.
__device__ __noinline__ double pred_same(int nat, double m3, double m2, double m1, double p1, double p2, double p3,
                                         int c, int E) {
    if (nat) {
        const double x[6] = {m3, m2, m1, p1, p2, p3};
        return Fam<FAM_NAT_S>::interior(c, E, 1) ? Fam<FAM_NAT_S>::combine(x) : edge_row<FAM_NAT_S>(x, c, E, 1);
    }
    const double x[6] = {m2, m1, p1, p2, 0.0, 0.0};
    return Fam<FAM_NAK_S>::interior(c, E, 1) ? Fam<FAM_NAK_S>::combine(x) : edge_row<FAM_NAK_S>(x, c, E, 1);
}

// ------------------------------------------------------------- escapes --
// (item, warp) unit of the sweep plan holding lattice point (z, y, x) of `commit`.
__device__ __noinline__ int64_t row_unit(const RowRun &A, int commit, int z, int y, int x) {
    const CommitDev &cm = A.commits[commit];
    const uint32_t j0 = (uint32_t)(z - cm.start[0]) / (uint32_t)cm.step[0];
    const uint32_t j1 = (uint32_t)(y - cm.start[1]) / (uint32_t)cm.step[1];
    const uint32_t j2 = (uint32_t)(x - cm.start[2]) / (uint32_t)cm.step[2];
    const uint32_t p = (j0 * (uint32_t)cm.cnt[1] + j1) * (uint32_t)cm.cnt[2] + j2;
    const uint32_t item = p / (uint32_t)cm.p_item;
    const uint32_t w = (p - item * (uint32_t)cm.p_item) / (uint32_t)cm.pw;
    return (int64_t)(cm.item_base + (int)item) * kItemWarps + w;
}

__device__ __noinline__ void row_escape(const RowRun &A, int commit, int z, int y, int x) {
    atomicAdd(A.esc_cnt + row_unit(A, commit, z, y, x), 1u);
}

// Outlier of the zero code at stream position ci: rank = the unit's first
// outlier rank plus the zero codes before ci in the unit (quant.py:115-129).
__device__ __noinline__ float row_outlier(const RowRun &A, int commit, int z, int y, int x, int64_t ci) {
    const int64_t e = row_unit(A, commit, z, y, x);
    int64_t r = A.esc_off[e];
    for (int64_t q = A.wbase[e]; q < ci; q++) r += A.codes[q] == 0;
    if (r < A.outl_cap) return (float)A.outl[r];
    atomicExch(A.flags, HPEZ_OUTLIER_UNDERFLOW);
    return 0.0f;
}

struct Q {  // level quantizer
    double bound, two_e, inv_two_e, Rd;
    int32_t R;
};

// One point: compress quantizes `orig` against pred (quant.py:80-105) and
// returns the code; decompress maps `code` back (quant.py:115-121).  *out is
// the value the decompressor sees.
template <int DIR>
__device__ __forceinline__ int32_t point(const Q &q, const RowRun &A, double pred, float orig, int32_t code, int commit,
                                         int z, int y, int x, int64_t ci, float *out) {
    if (DIR == HPEZ_COMPRESS) {
        double o;
        const int32_t c =
            quantize_point<HPEZ_ROUND_F32>((double)orig, pred, q.bound, q.two_e, q.inv_two_e, q.Rd, q.R, &o);
        *out = (float)o;
        if (c == 0) row_escape(A, commit, z, y, x);
        return c;
    }
    if (code != 0) *out = (float)dequantize_point<HPEZ_ROUND_F32>(pred, (int64_t)code, q.two_e, (int64_t)q.R);
    else *out = row_outlier(A, commit, z, y, x, ci);
    return code;
}

__device__ __forceinline__ void store_codes2(uint16_t *p, int32_t a, int32_t b) {
    if (((uintptr_t)p & 3) == 0) *reinterpret_cast<uint32_t *>(p) = (uint32_t)a | ((uint32_t)b << 16);
    else {
        p[0] = (uint16_t)a;
        p[1] = (uint16_t)b;
    }
}
__device__ __forceinline__ void load_codes2(const uint16_t *p, int32_t *a, int32_t *b) {
    if (((uintptr_t)p & 3) == 0) {
        const uint32_t v = *reinterpret_cast<const uint32_t *>(p);
        *a = (int32_t)(v & 0xffffu);
        *b = (int32_t)(v >> 16);
    } else {
        *a = p[0];
        *b = p[1];
    }
}

__device__ __forceinline__ float4 ld4(const float *p) { return *reinterpret_cast<const float4 *>(p); }
__device__ __forceinline__ void st4(float *p, float4 v) { *reinterpret_cast<float4 *>(p) = v; }

__device__ __forceinline__ int tag_of(const RowDesc &D, const RowRun &A, int z, int y, int x) {
    return D.has_table ? (int)A.table[(z >> D.bsh) * D.bs0 + (y >> D.bsh) * D.bs1 + (x >> D.bsh)] : D.const_k;
}

// ------------------------------------------------- rows (z even, y even) --
// Class (x) only: first pass at every x-odd point that is not a second-pass
// member, second pass (x = 3 mod 4 under a same-level variant) one chunk
// behind, reading the first-pass values at x +- 2 from the row buffer.
template <int DIR>
__device__ __noinline__ void process_row0_lag(const RowDesc &D, const RowRun &A, const Q &q, int z, int y, double *rb,
                                              int lane) {
    const int Lx = D.L[2], hx = Lx >> 1;
    const int rowidx = (z >> 1) * D.cny[0] + (y >> 1);
    const int rowoff = z * D.E0 + y * D.E1;
    const float *__restrict__ wrow = A.work + rowoff;
    const float *__restrict__ orow = A.orig + rowoff;
    const bool oop = DIR == HPEZ_COMPRESS && A.orig != A.work;
    int64_t baseA = D.level_base + A.rowbase[D.segA[2] + rowidx];
    int64_t baseB = D.segB[2] >= 0 ? D.level_base + A.rowbase[D.segB[2] + rowidx] : 0;
    const int cmA = D.commitA[2], cmB = D.commitB[2];
    const uint32_t lt = (1u << lane) - 1u;
    const int nch = (Lx + 127) >> 7;
    // carried second-pass state of the previous chunk
    bool p_act = false, p_same = false;
    int p_x0 = 0, p_nat = 0;
    float p_w0 = 0, p_w2 = 0, p_w4 = 0, p_w6 = 0, p_o3 = 0, p_r1 = 0, p_r3 = 0;
    int64_t p_ci = 0;
    for (int ch = 0; ch <= nch; ch++) {
        const int x0 = (ch << 7) + (lane << 2);
        const bool act = ch < nch && x0 < Lx;
        bool same = false;
        int nat = 0;
        float w0 = 0, w2 = 0, w4 = 0, w6 = 0, o3 = 0, r1 = 0, r3 = 0;
        int64_t ciB = 0;
        if (ch < nch) {
            float4 w = make_float4(0, 0, 0, 0), o = w, wp = w, wn = w;
            int k = 0;
            if (act) {
                w = ld4(wrow + x0);
                o = oop ? ld4(orow + x0) : w;
                k = tag_of(D, A, z, y, x0);
                if (x0 >= 4) wp = ld4(wrow + x0 - 4);  // coarse x0 - 2 (the neighbouring lane's line: L1 hit)
                if (x0 + 4 < Lx) wn = ld4(wrow + x0 + 4);
            }
            same = act && variant_same(k);
            nat = k == 4;
            const int fi = variant_fam(k);
            const uint32_t actm = __ballot_sync(0xffffffffu, act);
            const uint32_t nsm = __ballot_sync(0xffffffffu, act && !same);
            const uint32_t sm = __ballot_sync(0xffffffffu, same);
            const int64_t ciA = baseA + __popc(actm & lt) + __popc(nsm & lt);
            ciB = baseB + __popc(sm & lt);
            baseA += __popc(actm) + __popc(nsm);
            baseB += __popc(sm);
            w0 = w.x;
            w2 = w.z;
            w4 = wn.x;
            w6 = wn.z;
            o3 = o.w;
            if (act) {
                int32_t c1 = 0, c3 = 0;
                if (DIR == HPEZ_DECOMPRESS) {
                    c1 = A.codes[ciA];
                    if (!same) c3 = A.codes[ciA + 1];
                }
                const double d0 = (double)w.x, d2 = (double)w.z, d4 = (double)wn.x;
                const double pr1 = pred_inter(fi, fi ? (double)wp.z : 0.0, d0, d2, fi ? d4 : 0.0, x0 + 1, Lx);
                c1 = point<DIR>(q, A, pr1, o.y, c1, cmA, z, y, x0 + 1, ciA, &r1);
                if (DIR == HPEZ_COMPRESS) A.codes[ciA] = (uint16_t)c1;
                rb[x0 >> 1] = (double)r1;
                if (!same) {
                    const double pr3 = pred_inter(fi, fi ? d0 : 0.0, d2, d4, fi ? (double)wn.z : 0.0, x0 + 3, Lx);
                    c3 = point<DIR>(q, A, pr3, o.w, c3, cmA, z, y, x0 + 3, ciA + 1, &r3);
                    if (DIR == HPEZ_COMPRESS) A.codes[ciA + 1] = (uint16_t)c3;
                }
            }
        }
        __syncwarp();
        if (p_act) {
            if (p_same) {
                // second pass at x = p_x0 + 3: x +- 2 are first-pass values, x +- 1, 3 coarse
                const double a1 = rb[p_x0 >> 1];
                const double a5 = rb[min((p_x0 >> 1) + 2, hx - 1)];
                const double pr = pred_same(p_nat, (double)p_w0, a1, (double)p_w2, (double)p_w4, a5, (double)p_w6,
                                            p_x0 + 3, Lx);
                int32_t c3 = 0;
                if (DIR == HPEZ_DECOMPRESS) c3 = A.codes[p_ci];
                c3 = point<DIR>(q, A, pr, p_o3, c3, cmB, z, y, p_x0 + 3, p_ci, &p_r3);
                if (DIR == HPEZ_COMPRESS) A.codes[p_ci] = (uint16_t)c3;
            }
            st4(A.work + rowoff + p_x0, make_float4(p_w0, p_r1, p_w2, p_r3));
        }
        p_act = act;
        p_same = same;
        p_nat = nat;
        p_x0 = x0;
        p_w0 = w0;
        p_w2 = w2;
        p_w4 = w4;
        p_w6 = w6;
        p_o3 = o3;
        p_r1 = r1;
        p_r3 = r3;
        p_ci = ciB;
    }
}

// ------------------------------------- rows with z and/or y odd (RT 1..3) --
// Iteration `it` runs stage E of chunk it -- class E at x0, x0 + 2 from the
// .x/.z components of the neighbouring rows' 16-byte words, results into the
// row buffer -- and then stage O of chunk it - 1: class O at x0 + 1, x0 + 3
// from the .y/.w components of the same words (re-requested: they were
// fetched one iteration ago and hit L1) plus the row buffer's E values at
// x +- 1, 3, which by then include the first values of chunk it.  Chunks whose
// lanes all use the linear variant away from the grid faces take a
// straight-line path; the general path selects the row per lane.
struct CrossTaps {  // one cross axis of a row: coordinate, extent, clamped element offsets of -3, -1, +1, +3, -2, +2
    int c, L, off[4], off2[2];
    bool in1, in3;  // c + 1 <= L - 1; c - 3 >= 0 and c + 3 <= L - 1
};

// Inter-level row of family fi over float taps (kernels.py:43-86), edge rows
// through edge_inter (kernels.resolve_row, kernels.py:106-150).
__device__ __forceinline__ double pred_gen(int fi, float m3, float m1, float p1, float p3, bool in1, bool in3, int c,
                                           int E) {
    const double a = (double)m1, b = (double)p1;
    if (fi == 0) return in1 ? DA(DM(0.5, a), DM(0.5, b)) : DM(1.0, a);
    if (in3) {
        const double c0 = fi == 1 ? -1.0 / 16 : -3.0 / 40, c1 = fi == 1 ? 9.0 / 16 : 23.0 / 40;
        return DA(DA(DA(DM(c0, (double)m3), DM(c1, a)), DM(c1, b)), DM(c0, (double)p3));
    }
    return edge_inter(fi, (double)m3, a, b, (double)p3, c, E);
}
__device__ __forceinline__ double pred_gen_d(int fi, double m3, double a, double b, double p3, bool in1, bool in3,
                                             int c, int E) {
    if (fi == 0) return in1 ? DA(DM(0.5, a), DM(0.5, b)) : DM(1.0, a);
    if (in3) {
        const double c0 = fi == 1 ? -1.0 / 16 : -3.0 / 40, c1 = fi == 1 ? 9.0 / 16 : 23.0 / 40;
        return DA(DA(DA(DM(c0, m3), DM(c1, a)), DM(c1, b)), DM(c0, p3));
    }
    return edge_inter(fi, m3, a, b, p3, c, E);
}

// Rows whose blocks carry no same-level variant have a single pass: both
// x-odd points of a lane from its own 16-byte word and the next coarse value
// (shuffled from the next lane); only rows that cross a same-level block
// take the two-pass routine above.
template <int DIR>
__device__ __forceinline__ void process_row0(const RowDesc &D, const RowRun &A, const Q &q, int z, int y, double *rb,
                                             int lane) {
    const int Lx = D.L[2];
    if (D.any_same) {
        bool s = false;
        if (D.has_table) {
            const int nbx = ((Lx - 1) >> D.bsh) + 1;
            const uint8_t *t = A.table + (z >> D.bsh) * D.bs0 + (y >> D.bsh) * D.bs1;
            for (int b = lane; b < nbx; b += 32) s |= variant_same(t[b]);
        } else {
            s = true;
        }
        if (__any_sync(0xffffffffu, s)) {
            process_row0_lag<DIR>(D, A, q, z, y, rb, lane);
            return;
        }
    }
    const int rowidx = (z >> 1) * D.cny[0] + (y >> 1);
    const int rowoff = z * D.E0 + y * D.E1;
    const float *__restrict__ wrow = A.work + rowoff;
    const float *__restrict__ orow = A.orig + rowoff;
    const bool oop = DIR == HPEZ_COMPRESS && A.orig != A.work;
    const int64_t baseA = D.level_base + A.rowbase[D.segA[2] + rowidx];
    const int cmA = D.commitA[2];
    const int nch = (Lx + 127) >> 7;
    for (int it = 0; it < nch; it++) {
        const int x0 = (it << 7) + (lane << 2);
        const bool act = x0 < Lx;
        const int k = act ? tag_of(D, A, z, y, x0) : 0;
        const int fi = variant_fam(k);
        const bool lin = !__any_sync(0xffffffffu, fi != 0);
        float4 w = make_float4(0, 0, 0, 0), o = w;
        int32_t c1 = 0, c3 = 0;
        const int64_t ci = baseA + 2 * ((it << 5) + lane);
        if (act) {
            w = ld4(wrow + x0);
            if (oop) o = ld4(orow + x0);
            else o = w;
            if (DIR == HPEZ_DECOMPRESS) load_codes2(A.codes + ci, &c1, &c3);
        }
        const bool r4 = x0 + 4 <= Lx - 1;
        double pr1, pr3;
        if (lin) {
            float w4 = __shfl_down_sync(0xffffffffu, w.x, 1);
            if (lane == 31 && act && r4) w4 = wrow[x0 + 4];
            const double d0 = (double)w.x, d2 = (double)w.z;
            pr1 = DA(DM(0.5, d0), DM(0.5, d2));
            pr3 = r4 ? DA(DM(0.5, d2), DM(0.5, (double)w4)) : DM(1.0, d2);
        } else {
            float4 wp = make_float4(0, 0, 0, 0), wn = wp;
            if (act && x0 >= 4) wp = ld4(wrow + x0 - 4);
            if (act && r4) wn = ld4(wrow + x0 + 4);
            pr1 = pred_gen(fi, wp.z, w.x, w.z, wn.x, true, x0 >= 2 && r4, x0 + 1, Lx);
            pr3 = pred_gen(fi, w.x, w.z, wn.x, wn.z, r4, x0 + 6 <= Lx - 1, x0 + 3, Lx);
        }
        if (act) {
            float r1, r3;
            c1 = point<DIR>(q, A, pr1, o.y, c1, cmA, z, y, x0 + 1, ci, &r1);
            c3 = point<DIR>(q, A, pr3, o.w, c3, cmA, z, y, x0 + 3, ci + 1, &r3);
            if (DIR == HPEZ_COMPRESS) store_codes2(A.codes + ci, c1, c3);
            st4(A.work + rowoff + x0, make_float4(w.x, r1, w.z, r3));
        }
    }
}

template <int DIR, int RT, bool BROW>
__device__ __forceinline__ void process_rowN(const RowDesc &D, const RowRun &A, const Q &q, int z, int y, double *rb,
                                             int lane) {
    constexpr int VZ = RT & 1, VY = RT >> 1;
    constexpr int NC = VZ + VY;
    constexpr int CE = RT == 1 ? 0 : RT == 2 ? 1 : 3;
    constexpr int CO = RT == 1 ? 4 : RT == 2 ? 5 : 6;
    const int Lx = D.L[2], hx = Lx >> 1;
    const int rowidx = (z >> 1) * D.cny[VY] + (y >> 1);
    const int rowoff = z * D.E0 + y * D.E1;
    const float *__restrict__ orow = A.orig + rowoff;
    const float *__restrict__ wrow = A.work + rowoff;
    CrossTaps X[NC];
    bool lin_ok = true;  // every cross axis has its +1 neighbour (the linear row needs nothing else)
#pragma unroll
    for (int t = 0; t < NC; t++) {
        const bool isz = VZ && t == 0;
        X[t].c = isz ? z : y;
        X[t].L = isz ? D.L[0] : D.L[1];
        const int str = isz ? D.E0 : D.E1;
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int u = 2 * i - 3;
            X[t].off[i] = (X[t].c + u >= 0 && X[t].c + u <= X[t].L - 1) ? u * str : 0;
        }
        X[t].off2[0] = X[t].c - 2 >= 0 ? -2 * str : 0;
        X[t].off2[1] = X[t].c + 2 <= X[t].L - 1 ? 2 * str : 0;
        X[t].in1 = X[t].c + 1 <= X[t].L - 1;
        X[t].in3 = X[t].c >= 3 && X[t].c + 3 <= X[t].L - 1;
        lin_ok = lin_ok && X[t].in1;
    }
    int64_t baseEA = D.level_base + A.rowbase[D.segA[CE] + rowidx];
    int64_t baseEB = BROW ? D.level_base + A.rowbase[D.segB[CE] + rowidx] : 0;
    const int64_t baseO = D.level_base + A.rowbase[D.segA[CO] + rowidx];
    const int cmEA = D.commitA[CE], cmEB = D.commitB[CE], cmO = D.commitA[CO];
    const double we0 = D.w[CE][0], we1 = D.w[CE][1];
    const double wo0 = D.w[CO][0], wo1 = D.w[CO][1], wo2 = D.w[CO][2];
    const uint32_t lt = (1u << lane) - 1u;
    const int nch = (Lx + 127) >> 7;
    for (int it = 0; it <= nch; it++) {
        // ---------------------------------------------------- stage E --
        if (it < nch) {
            const int x0 = (it << 7) + (lane << 2);
            const bool act = x0 < Lx;
            const int k = act ? tag_of(D, A, z, y, x0) : 0;
            const int fi = variant_fam(k);
            const bool isB = BROW && act && variant_same(k);
            const bool lin = lin_ok && !__any_sync(0xffffffffu, fi != 0);
            int64_t ci;
            if (BROW) {
                const uint32_t am = __ballot_sync(0xffffffffu, act && !isB);
                const uint32_t bm = __ballot_sync(0xffffffffu, isB);
                ci = isB ? baseEB + 2 * __popc(bm & lt) : baseEA + 2 * __popc(am & lt);
                baseEA += 2 * __popc(am);
                baseEB += 2 * __popc(bm);
            } else {
                ci = baseEA + 2 * ((it << 5) + lane);
            }
            if (act) {
                float4 o = make_float4(0, 0, 0, 0);
                int32_t c0 = 0, c2 = 0;
                if (DIR == HPEZ_COMPRESS) o = ld4(orow + x0);
                else load_codes2(A.codes + ci, &c0, &c2);
                double pr0, pr2;
                if (lin) {
                    float4 a[NC][2];
#pragma unroll
                    for (int t = 0; t < NC; t++) {
                        a[t][0] = ld4(wrow + X[t].off[1] + x0);
                        a[t][1] = ld4(wrow + X[t].off[2] + x0);
                    }
                    double pa[NC], pb[NC];
#pragma unroll
                    for (int t = 0; t < NC; t++) {
                        pa[t] = DA(DM(0.5, (double)a[t][0].x), DM(0.5, (double)a[t][1].x));
                        pb[t] = DA(DM(0.5, (double)a[t][0].z), DM(0.5, (double)a[t][1].z));
                    }
                    pr0 = NC == 1 ? pa[0] : DA(DM(we0, pa[0]), DM(we1, pa[NC - 1]));
                    pr2 = NC == 1 ? pb[0] : DA(DM(we0, pb[0]), DM(we1, pb[NC - 1]));
                } else if (isB) {  // second same-level pass along the class axis (NC == 1)
                    float4 a[6];
#pragma unroll
                    for (int i = 0; i < 4; i++) a[i] = ld4(wrow + X[0].off[i] + x0);
                    a[4] = ld4(wrow + X[0].off2[0] + x0);
                    a[5] = ld4(wrow + X[0].off2[1] + x0);
                    const int nat = k == 4;
                    pr0 = pred_same(nat, (double)a[0].x, (double)a[4].x, (double)a[1].x, (double)a[2].x, (double)a[5].x,
                                    (double)a[3].x, X[0].c, X[0].L);
                    pr2 = pred_same(nat, (double)a[0].z, (double)a[4].z, (double)a[1].z, (double)a[2].z, (double)a[5].z,
                                    (double)a[3].z, X[0].c, X[0].L);
                } else {
                    double pa[NC], pb[NC];
#pragma unroll
                    for (int t = 0; t < NC; t++) {
                        float4 a[4];
                        a[0] = a[3] = make_float4(0, 0, 0, 0);
                        a[1] = ld4(wrow + X[t].off[1] + x0);
                        a[2] = ld4(wrow + X[t].off[2] + x0);
                        if (fi) {
                            a[0] = ld4(wrow + X[t].off[0] + x0);
                            a[3] = ld4(wrow + X[t].off[3] + x0);
                        }
                        pa[t] = pred_gen(fi, a[0].x, a[1].x, a[2].x, a[3].x, X[t].in1, X[t].in3, X[t].c, X[t].L);
                        pb[t] = pred_gen(fi, a[0].z, a[1].z, a[2].z, a[3].z, X[t].in1, X[t].in3, X[t].c, X[t].L);
                    }
                    pr0 = NC == 1 ? pa[0] : DA(DM(we0, pa[0]), DM(we1, pa[NC - 1]));
                    pr2 = NC == 1 ? pb[0] : DA(DM(we0, pb[0]), DM(we1, pb[NC - 1]));
                }
                const int cm = isB ? cmEB : cmEA;
                float e0, e2;
                c0 = point<DIR>(q, A, pr0, o.x, c0, cm, z, y, x0, ci, &e0);
                c2 = point<DIR>(q, A, pr2, o.z, c2, cm, z, y, x0 + 2, ci + 1, &e2);
                if (DIR == HPEZ_COMPRESS) store_codes2(A.codes + ci, c0, c2);
                *reinterpret_cast<double2 *>(rb + (x0 >> 1)) = make_double2((double)e0, (double)e2);
            }
        }
        __syncwarp();
        // ---------------------------------------------------- stage O --
        if (it > 0) {
            const int x0 = ((it - 1) << 7) + (lane << 2);
            const bool act = x0 < Lx;
            const int k = act ? tag_of(D, A, z, y, x0) : 0;
            const int fi = variant_fam(k);
            const bool lin = lin_ok && !__any_sync(0xffffffffu, fi != 0);
            if (act) {
                const int64_t ci = baseO + 2 * (((it - 1) << 5) + lane);
                const int h = x0 >> 1;
                float4 o = make_float4(0, 0, 0, 0);
                int32_t c1 = 0, c3 = 0;
                if (DIR == HPEZ_COMPRESS) o = ld4(orow + x0);
                else load_codes2(A.codes + ci, &c1, &c3);
                const double2 e02 = *reinterpret_cast<const double2 *>(rb + h);
                const bool r4 = x0 + 4 <= Lx - 1;
                double pr1, pr3;
                if (lin) {
                    float4 a[NC][2];
#pragma unroll
                    for (int t = 0; t < NC; t++) {
                        a[t][0] = ld4(wrow + X[t].off[1] + x0);
                        a[t][1] = ld4(wrow + X[t].off[2] + x0);
                    }
                    const double e4 = rb[min(h + 2, hx - 1)];
                    double pa[NC + 1], pb[NC + 1];
#pragma unroll
                    for (int t = 0; t < NC; t++) {
                        pa[t] = DA(DM(0.5, (double)a[t][0].y), DM(0.5, (double)a[t][1].y));
                        pb[t] = DA(DM(0.5, (double)a[t][0].w), DM(0.5, (double)a[t][1].w));
                    }
                    pa[NC] = DA(DM(0.5, e02.x), DM(0.5, e02.y));
                    pb[NC] = r4 ? DA(DM(0.5, e02.y), DM(0.5, e4)) : DM(1.0, e02.y);
                    if (NC == 1) {
                        pr1 = DA(DM(wo0, pa[0]), DM(wo1, pa[1]));
                        pr3 = DA(DM(wo0, pb[0]), DM(wo1, pb[1]));
                    } else {
                        pr1 = DA(DA(DM(wo0, pa[0]), DM(wo1, pa[1])), DM(wo2, pa[NC]));
                        pr3 = DA(DA(DM(wo0, pb[0]), DM(wo1, pb[1])), DM(wo2, pb[NC]));
                    }
                } else {
                    double pa[NC + 1], pb[NC + 1];
#pragma unroll
                    for (int t = 0; t < NC; t++) {
                        float4 a[4];
                        a[0] = a[3] = make_float4(0, 0, 0, 0);
                        a[1] = ld4(wrow + X[t].off[1] + x0);
                        a[2] = ld4(wrow + X[t].off[2] + x0);
                        if (fi) {
                            a[0] = ld4(wrow + X[t].off[0] + x0);
                            a[3] = ld4(wrow + X[t].off[3] + x0);
                        }
                        pa[t] = pred_gen(fi, a[0].y, a[1].y, a[2].y, a[3].y, X[t].in1, X[t].in3, X[t].c, X[t].L);
                        pb[t] = pred_gen(fi, a[0].w, a[1].w, a[2].w, a[3].w, X[t].in1, X[t].in3, X[t].c, X[t].L);
                    }
                    const double xm2 = rb[max(h - 1, 0)], x4v = rb[min(h + 2, hx - 1)], x6v = rb[min(h + 3, hx - 1)];
                    pa[NC] = pred_gen_d(fi, xm2, e02.x, e02.y, x4v, true, x0 >= 2 && r4, x0 + 1, Lx);
                    pb[NC] = pred_gen_d(fi, e02.x, e02.y, x4v, x6v, r4, x0 + 6 <= Lx - 1, x0 + 3, Lx);
                    if (NC == 1) {
                        pr1 = DA(DM(wo0, pa[0]), DM(wo1, pa[1]));
                        pr3 = DA(DM(wo0, pb[0]), DM(wo1, pb[1]));
                    } else {
                        pr1 = DA(DA(DM(wo0, pa[0]), DM(wo1, pa[1])), DM(wo2, pa[NC]));
                        pr3 = DA(DA(DM(wo0, pb[0]), DM(wo1, pb[1])), DM(wo2, pb[NC]));
                    }
                }
                float r1, r3;
                c1 = point<DIR>(q, A, pr1, o.y, c1, cmO, z, y, x0 + 1, ci, &r1);
                c3 = point<DIR>(q, A, pr3, o.w, c3, cmO, z, y, x0 + 3, ci + 1, &r3);
                if (DIR == HPEZ_COMPRESS) store_codes2(A.codes + ci, c1, c3);
                st4(A.work + rowoff + x0, make_float4((float)e02.x, r1, (float)e02.y, r3));
            }
        }
    }
}

template <int DIR>
__global__ void __launch_bounds__(kRowThreads, HPEZ_ROW_OCC) row_kernel(const __grid_constant__ RowDesc D,
                                                            const __grid_constant__ RowRun A,
                                                            const __grid_constant__ RowLaunch L) {
    extern __shared__ double s_rb[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *rb = s_rb + (size_t)warp * ((D.L[2] >> 1) + 4);
    Q q;
    q.bound = D.bound;
    q.two_e = D.two_e;
    q.inv_two_e = D.inv_two_e;
    q.R = D.R;
    q.Rd = (double)D.R;
    const int nw = (int)gridDim.x * kRowWarps;
    const int n0 = L.s[0].nz * L.s[0].ny;
    for (int r = (int)blockIdx.x * kRowWarps + warp; r < L.total; r += nw) {
        const RowSet &S = r < n0 ? L.s[0] : L.s[1];
        const int rr = r < n0 ? r : r - n0;
        const int iz = rr / S.ny, iy = rr - iz * S.ny;
        const int z = S.z0 + iz * S.zs, y = S.y0 + iy * S.ys;
        switch (S.rt * 2 + S.brow) {
        case 0: process_row0<DIR>(D, A, q, z, y, rb, lane); break;
        case 2: process_rowN<DIR, 1, false>(D, A, q, z, y, rb, lane); break;
        case 3: process_rowN<DIR, 1, true>(D, A, q, z, y, rb, lane); break;
        case 4: process_rowN<DIR, 2, false>(D, A, q, z, y, rb, lane); break;
        case 5: process_rowN<DIR, 2, true>(D, A, q, z, y, rb, lane); break;
        default: process_rowN<DIR, 3, false>(D, A, q, z, y, rb, lane); break;
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------ host --
static int cls_of_vmask(uint32_t vm) {
    for (int c = 0; c < 7; c++)
        if ((uint32_t)class_vmask(c) == vm) return c;
    return -1;
}

bool row_plan_build(const GridDev &g, const CommitDev *cms, const uint32_t *vmask, int n, int first_commit,
                    const uint8_t *tbl, int64_t nblk, int level_kernel, int level_paradigm, int64_t level_base,
                    RowPlan *out) {
    RowPlan P;
    RowDesc &D = P.d;
    memset(&D, 0, sizeof D);
    if (g.rank != 3 || n < 7 || cms[0].s != 1) return false;
    for (int a = 0; a < 3; a++) {
        D.L[a] = g.dims[a];
        if (g.dims[a] < 8) return false;
    }
    if (D.L[2] % 4 != 0 || g.estr[2] != 1) return false;
    if (g.npts >= (1ll << 31) || g.radius > 32768) return false;
    D.E0 = g.estr[0];
    D.E1 = g.estr[1];
    D.R = (int32_t)g.radius;
    D.has_table = tbl != nullptr;
    D.const_k = level_kernel;
    D.any_same = 0;
    if (tbl) {
        if (g.bs_log2 < 2) return false;
        D.bsh = g.bs_log2;
        D.bs0 = g.bstr[0];
        D.bs1 = g.bstr[1];
        for (int64_t b = 0; b < nblk; b++) {
            if (tbl[b] >= 5) return false;  // a one-axis (oned) variant somewhere in the level
            D.any_same |= variant_same(tbl[b]);
        }
    } else {
        if (level_paradigm != 1 || level_kernel < 0 || level_kernel >= 5) return false;
        D.any_same = variant_same(level_kernel);
    }
    D.cny[0] = (D.L[1] + 1) / 2;
    D.cny[1] = D.L[1] / 2;
    D.bound = cms[0].bound;
    D.two_e = cms[0].two_e;
    D.inv_two_e = cms[0].inv_two_e;
    D.level_base = level_base;
    for (int c = 0; c < 7; c++) {
        D.commitA[c] = D.commitB[c] = -1;
        D.segA[c] = D.segB[c] = -1;
    }
    // commits of the level -> (class, pass)
    for (int i = 0; i < n; i++) {
        const CommitDev &cm = cms[i];
        const int c = cls_of_vmask(vmask[i]);
        if (c < 0) return false;
        const bool single = c < 3;
        bool second = false;
        if (cm.kind == COMMIT_UNIFORM) {
            if (single) {
                if (cm.pred.md || cm.pred.axis != c) return false;
                second = cm.start[c] == 3;  // phase lattice 3, 7, ... of a split class (interp.py:333-341)
                if (second != (cm.pred.fam == FAM_NAK_S || cm.pred.fam == FAM_NAT_S)) return false;
            } else if (!cm.pred.md) {
                return false;
            }
        } else {
            second = cm.kind == COMMIT_MIXED_B;
            if (second && (!single || cm.phase != 0)) return false;
        }
        if (!single) {
            for (int t = 0; t < 3; t++) D.w[c][t] = cm.pred.w[t];
        }
        int32_t &slot = second ? D.commitB[c] : D.commitA[c];
        if (slot >= 0) return false;
        slot = first_commit + i;
    }
    for (int c = 0; c < 7; c++)
        if (D.commitA[c] < 0) return false;
    // (class, pass) row segments in stream order
    int64_t e = 0;
    for (int c = 0; c < 7; c++) {
        const int vm = class_vmask(c);
        const int64_t cnz = (vm & 1) ? D.L[0] / 2 : (D.L[0] + 1) / 2;
        const int64_t rows = cnz * D.cny[(vm >> 1) & 1];
        D.segA[c] = e;
        e += rows;
        if (c < 3 && D.any_same) {
            D.segB[c] = e;
            e += rows;
        }
    }
    D.n_entries = e;
    // a same-level member without a second-pass commit would have nowhere to go
    for (int c = 0; c < 3; c++)
        if (D.any_same && D.commitB[c] < 0) return false;
    // launches
    const int Lz = D.L[0], Ly = D.L[1];
    auto cnt = [](int a, int b, int c) { return a < b ? (b - 1 - a) / c + 1 : 0; };
    auto set = [&](int rt, int brow, int z0, int zs, int y0, int ys) {
        RowSet s{};
        s.rt = rt;
        s.brow = brow;
        s.z0 = z0;
        s.zs = zs;
        s.nz = cnt(z0, Lz, zs);
        s.y0 = y0;
        s.ys = ys;
        s.ny = cnt(y0, Ly, ys);
        return s;
    };
    auto add = [&](RowSet a, const RowSet *b) {
        RowLaunch &l = P.launch[P.n_launch++];
        l.n = b ? 2 : 1;
        l.s[0] = a;
        l.total = a.nz * a.ny;
        if (b) {
            l.s[1] = *b;
            l.total += b->nz * b->ny;
        }
    };
    P.n_launch = 0;
    add(set(0, 0, 0, 2, 0, 2), nullptr);
    if (!D.any_same) {
        const RowSet b = set(2, 0, 0, 2, 1, 2);
        add(set(1, 0, 1, 2, 0, 2), &b);
    } else {
        const RowSet b0 = set(2, 0, 0, 2, 1, 4), b1 = set(2, 1, 0, 2, 3, 4);
        add(set(1, 0, 1, 4, 0, 2), &b0);
        add(set(1, 1, 3, 4, 0, 2), &b1);
    }
    add(set(3, 0, 1, 2, 1, 2), nullptr);
    P.threads = kRowThreads;
    P.smem = (size_t)kRowWarps * ((D.L[2] >> 1) + 4) * sizeof(double);
    if (P.smem > 100 * 1024) return false;
    P.first_commit = first_commit;
    P.ok = true;
    *out = P;
    return true;
}

cudaError_t row_plan_setup(RowPlan &p, const uint8_t *d_table_level, cudaStream_t st) {
    if (!p.ok) return cudaSuccess;
    const int64_t n = p.d.n_entries;
    row_count_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(p.d, d_table_level, p.d_cnt);
    exclusive_scan(p.d_cnt, n, p.d_base, p.d_tmp, p.d_total, st);
    return cudaGetLastError();
}

cudaError_t row_plan_launch(const RowPlan &p, int dir, const RowRun &r, cudaStream_t st) {
    auto *f = dir == HPEZ_COMPRESS ? row_kernel<HPEZ_COMPRESS> : row_kernel<HPEZ_DECOMPRESS>;
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, p.threads, p.smem) != cudaSuccess || occ < 1) occ = 1;
    for (int i = 0; i < p.n_launch; i++) {
        const RowLaunch &l = p.launch[i];
        if (l.total <= 0) continue;
        const int grid = std::max(1, std::min((l.total + kRowWarps - 1) / kRowWarps, occ * sms));
        f<<<grid, p.threads, p.smem, st>>>(p.d, r, l);
    }
    return cudaGetLastError();
}

}  // namespace hpez
