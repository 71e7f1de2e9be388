// row.cu -- the fine levels of a rank-3 sweep, one warp per lattice row.
//
// Reference: interp._LevelRunner.run_level (interp.py:415-433) for a level of
// stride s, classes on the uniform path (interp.py:322-341) or the mixed
// per-block path (interp.py:350-411).  Supported variants (plan.encode_tag,
// plan.py:69-84): every multidim tag (classes of one axis predict 1-D along
// it, with the two-pass same-level split for variants 2 and 4; classes of two
// or three axes blend the inter-level rows of their axes, interp.py:300-311)
// and the one-axis (oned) tags without a same-level split (every class
// predicts along the axis its order visits last, interp.py:226-230).
//
// Geometry (lattice units: coordinate / s).  A row (fixed z, y) holds two
// classes: its x-even points (class E = the odd axes among z, y; coarse
// points when both are even) and its x-odd points (class O = E + x).  Class E
// reads only OTHER rows (z +- 1, 3 and/or y +- 1, 3; +- 2 for its second
// same-level pass); class O reads the same rows at odd x plus the row's own
// x-even values.  A warp owns the row: it reads the neighbouring rows with
// 16-byte loads, serves both classes from them, keeps the row's fresh values
// in a shared-memory row buffer (f64) for the in-row stencil and writes the
// finished row back as complete 16-byte words (stride 1).  Rows of one
// parity type depend only on rows of earlier types, so a level is 3-4 plain
// launches:
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

// CTAs per SM of the three instantiations (measured sweep, cfg4 / cfg5): rows with one of z, y odd 4
// (64 registers), (z even, y even) rows and (z odd, y odd) rows 3 (80 registers)
#ifndef HPEZ_ROW_OCC
#define HPEZ_ROW_OCC 4
#endif
#ifndef HPEZ_ROW_OCC0
#define HPEZ_ROW_OCC0 3
#endif
#ifndef HPEZ_ROW_OCC8
#define HPEZ_ROW_OCC8 3
#endif
#ifndef HPEZ_ROW_PF
#define HPEZ_ROW_PF 1
#endif
constexpr int kRowWarps = 8;
constexpr int kRowThreads = kRowWarps * 32;

__host__ __device__ __forceinline__ int cnt_mod(int lo, int hi, int r, int m) {
    return (hi + m - 1 - r) / m - (lo + m - 1 - r) / m;  // j in [lo, hi) with j = r mod m
}
// tag = p * 8 + k (plan.py:69-75): k the kernel variant, p = 0 multidim, 1..6 a one-axis order
__host__ __device__ __forceinline__ bool tag_same(int tag) { return tag == 2 || tag == 4; }
__host__ __device__ __forceinline__ int tag_fam(int tag) { return ((tag & 7) + 1) >> 1; }  // 0 linear, 1 not-a-knot, 2 natural

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
        const int tag = D.has_table ? table[(z >> D.bsh) * D.bs0 + (y >> D.bsh) * D.bs1 + bx] : D.const_tag;
        const int all = cnt_mod(lo, hi, vx, 2);
        int nA = all, nB = 0;
        if (single && tag_same(tag)) {
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
// the values at c-3, c-1, c+1, c+3 (kernels.py:43-86); in1 / in3: the +1
// neighbour / all four exist; edge rows through edge_inter
// (kernels.resolve_row, kernels.py:106-150).
__device__ __forceinline__ double pred_gen(int fi, double m3, double a, double b, double p3, bool in1, bool in3, int c,
                                           int E) {
    if (fi == 0) return in1 ? DA(DM(0.5, a), DM(0.5, b)) : DM(1.0, a);
    if (in3) {
        const double c0 = fi == 1 ? -1.0 / 16 : -3.0 / 40, c1 = fi == 1 ? 9.0 / 16 : 23.0 / 40;
        return DA(DA(DA(DM(c0, m3), DM(c1, a)), DM(c1, b)), DM(c0, p3));
    }
    return edge_inter(fi, m3, a, b, p3, c, E);
}

// Same-level 1-D row (second pass of a split class) over c-3 .. c+3.
__device__ __forceinline__ double pred_same(int nat, double m3, double m2, double m1, double p1, double p2, double p3,
                                         int c, int E) {
    if (nat) {
        const double x[6] = {m3, m2, m1, p1, p2, p3};
        return Fam<FAM_NAT_S>::interior(c, E, 1) ? Fam<FAM_NAT_S>::combine(x) : edge_row<FAM_NAT_S>(x, c, E, 1);
    }
    const double x[6] = {m2, m1, p1, p2, 0.0, 0.0};
    return Fam<FAM_NAK_S>::interior(c, E, 1) ? Fam<FAM_NAK_S>::combine(x) : edge_row<FAM_NAK_S>(x, c, E, 1);
}

// MD blend (interp.py:306-311) or, for a one-axis tag, the term of the axis
// its order visits last (sel = index of that axis among the class's axes).
template <int N>
__device__ __forceinline__ double combine_terms(const double (&p)[N], int sel, double w0, double w1, double w2) {
    if (N == 1) return p[0];
    double md;
    if (N == 2) md = DA(DM(w0, p[0]), DM(w1, p[N - 1]));
    else md = DA(DA(DM(w0, p[0]), DM(w1, p[1])), DM(w2, p[N - 1]));
    if (sel < 0) return md;
    return sel == 0 ? p[0] : (sel == 1 ? p[1] : p[N - 1]);
}

// ------------------------------------------------------------- escapes --
// (item, warp) unit of the sweep plan holding lattice point (z, y, x) of `commit`.
__device__ __noinline__ int64_t row_unit(const RowRun &A, int commit, int s, int z, int y, int x) {
    const CommitDev &cm = A.commits[commit];
    const uint32_t j0 = (uint32_t)(z * s - cm.start[0]) / (uint32_t)cm.step[0];
    const uint32_t j1 = (uint32_t)(y * s - cm.start[1]) / (uint32_t)cm.step[1];
    const uint32_t j2 = (uint32_t)(x * s - cm.start[2]) / (uint32_t)cm.step[2];
    const uint32_t p = (j0 * (uint32_t)cm.cnt[1] + j1) * (uint32_t)cm.cnt[2] + j2;
    const uint32_t item = p / (uint32_t)cm.p_item;
    const uint32_t w = (p - item * (uint32_t)cm.p_item) / (uint32_t)cm.pw;
    return (int64_t)(cm.item_base + (int)item) * kItemWarps + w;
}

__device__ __noinline__ void row_escape(const RowRun &A, int commit, int s, int z, int y, int x) {
    atomicAdd(A.esc_cnt + row_unit(A, commit, s, z, y, x), 1u);
}

// Outlier of the zero code at stream position ci: rank = the unit's first
// outlier rank plus the zero codes before ci in the unit (quant.py:115-129).
__device__ __noinline__ float row_outlier(const RowRun &A, int commit, int s, int z, int y, int x, int64_t ci) {
    const int64_t e = row_unit(A, commit, s, z, y, x);
    int64_t r = A.esc_off[e];
    for (int64_t q = A.wbase[e]; q < ci; q++) r += A.codes[q] == 0;
    if (r < A.outl_cap) return (float)A.outl[r];
    atomicExch(A.flags, HPEZ_OUTLIER_UNDERFLOW);
    return 0.0f;
}

struct Q {  // level quantizer
    double bound, two_e, inv_two_e, Rd;
    int32_t R, s;
};

// quant.quantize_block for one f32 point with a positive bound
// (quant.py:80-105), the reciprocal-multiply form of common.cuh's
// quantize_point: np.sign(x) * floor(|x| + 0.5) is copysign(floor, x) (a zero
// of either sign gives the same reconstruction and code), and a point out of
// the code range fails `fl < R` and escapes whatever its reconstruction.
__device__ __forceinline__ int32_t quant_f32(const Q &q, double pred, float origf, float *out) {
    const double orig = (double)origf;
    const double d = __dsub_rn(orig, pred);
    double x = __dmul_rn(d, q.inv_two_e);
    const double y = __dadd_rn(fabs(x), 0.5);
    double fl = floor(y);
    const double fr = __dsub_rn(y, fl);
    if (fr < 0x1p-20 || fr > 1.0 - 0x1p-20) {  // |x| + 0.5 >= 2^20 fails fl < R below on either path
        x = __ddiv_rn(d, q.two_e);
        fl = floor(__dadd_rn(fabs(x), 0.5));
    }
    const double k = copysign(fl, x);
    const float rf = __double2float_rn(__dadd_rn(pred, __dmul_rn(q.two_e, k)));
    const bool ok = fl < q.Rd && fabs(__dsub_rn((double)rf, orig)) <= q.bound;
    *out = ok ? rf : origf;
    return ok ? (int32_t)k + q.R : 0;
}

// Two points of one class: compress quantizes the originals against the
// predictions and returns the codes; decompress maps the codes back
// (quant.py:115-121).  *ra / *rb are the values the decompressor sees.
// Escapes (code 0) take the cold path.
template <int DIR>
__device__ __forceinline__ void point2(const Q &q, const RowRun &A, double pa, double pb, float oa, float ob, int32_t *ca,
                                       int32_t *cb, int commit, int z, int y, int xa, int xb, int64_t ci, float *ra,
                                       float *rb) {
    if (DIR == HPEZ_COMPRESS) {
        if (q.bound > 0.0) {
            *ca = quant_f32(q, pa, oa, ra);
            *cb = quant_f32(q, pb, ob, rb);
        } else {
            double o;
            *ca = quantize_point<HPEZ_ROUND_F32>((double)oa, pa, q.bound, q.two_e, q.inv_two_e, q.Rd, q.R, &o);
            *ra = (float)o;
            *cb = quantize_point<HPEZ_ROUND_F32>((double)ob, pb, q.bound, q.two_e, q.inv_two_e, q.Rd, q.R, &o);
            *rb = (float)o;
        }
        if (*ca == 0 || *cb == 0) {
            if (*ca == 0) row_escape(A, commit, q.s, z, y, xa);
            if (*cb == 0) row_escape(A, commit, q.s, z, y, xb);
        }
    } else {
        *ra = __double2float_rn(__dadd_rn(pa, __dmul_rn(q.two_e, (double)(*ca - q.R))));
        *rb = __double2float_rn(__dadd_rn(pb, __dmul_rn(q.two_e, (double)(*cb - q.R))));
        if (*ca == 0 || *cb == 0) {
            if (*ca == 0) *ra = row_outlier(A, commit, q.s, z, y, xa, ci);
            if (*cb == 0) *rb = row_outlier(A, commit, q.s, z, y, xb, ci + 1);
        }
    }
}

// One point (the second pass of the x class handles its points singly).
template <int DIR>
__device__ __forceinline__ void point1(const Q &q, const RowRun &A, double pa, float oa, int32_t *ca, int commit, int z,
                                       int y, int xa, int64_t ci, float *ra) {
    if (DIR == HPEZ_COMPRESS) {
        double o;
        *ca = quantize_point<HPEZ_ROUND_F32>((double)oa, pa, q.bound, q.two_e, q.inv_two_e, q.Rd, q.R, &o);
        *ra = (float)o;
        if (*ca == 0) row_escape(A, commit, q.s, z, y, xa);
    } else {
        if (*ca != 0) *ra = __double2float_rn(__dadd_rn(pa, __dmul_rn(q.two_e, (double)(*ca - q.R))));
        else *ra = row_outlier(A, commit, q.s, z, y, xa, ci);
    }
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

__device__ __forceinline__ void prefetch_l1(const void *p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }
__device__ __forceinline__ float4 ld4(const float *p) { return *reinterpret_cast<const float4 *>(p); }
__device__ __forceinline__ void st4(float *p, float4 v) { *reinterpret_cast<float4 *>(p) = v; }

// Four consecutive lattice points j0 .. j0 + 3 of a row (element stride S).
template <int S>
__device__ __forceinline__ float4 ldl(const float *row, int j) {
    const uint32_t j0 = (uint32_t)j;  // never negative: an unsigned index is one wide multiply-add
    if (S == 1) return ld4(row + j0);
    if (S == 2) {
        const float4 a = ld4(row + 2u * j0), b = ld4(row + 2u * j0 + 4u);
        return make_float4(a.x, a.z, b.x, b.z);
    }
    return make_float4(row[S * j0], row[S * (j0 + 1u)], row[S * (j0 + 2u)], row[S * (j0 + 3u)]);
}
// Stores the components selected by MASK (stride 1: the whole 16-byte word).
template <int S, int MASK>
__device__ __forceinline__ void stl(float *row, int j, float4 v) {
    const uint32_t j0 = (uint32_t)j;
    if (S == 1) {
        st4(row + j0, v);
        return;
    }
    if (MASK & 1) row[S * j0] = v.x;
    if (MASK & 2) row[S * (j0 + 1u)] = v.y;
    if (MASK & 4) row[S * (j0 + 2u)] = v.z;
    if (MASK & 8) row[S * (j0 + 3u)] = v.w;
}

// Block tags of one row: lane b holds the tag of x-block b (rows of at most 32
// blocks), so a chunk's tag is one shuffle.
struct RowTags {
    int reg;
    const uint8_t *row;
    int bsh, const_tag;
    bool table, in_reg;
};
__device__ __forceinline__ RowTags row_tags(const RowDesc &D, const RowRun &A, int z, int y, int lane) {
    RowTags T;
    T.table = D.has_table != 0;
    T.const_tag = D.const_tag;
    T.bsh = D.bsh;
    T.reg = 0;
    T.row = nullptr;
    T.in_reg = false;
    if (T.table) {
        const int nbx = ((D.L[2] - 1) >> D.bsh) + 1;
        T.row = A.table + (z >> D.bsh) * D.bs0 + (y >> D.bsh) * D.bs1;
        T.in_reg = nbx <= 32;
        if (T.in_reg && lane < nbx) T.reg = T.row[lane];
    }
    return T;
}
// called by the whole warp
__device__ __forceinline__ int tag_at(const RowTags &T, int x0, bool act) {
    if (!T.table) return act ? T.const_tag : 0;
    if (T.in_reg) {
        const int t = __shfl_sync(0xffffffffu, T.reg, (x0 >> T.bsh) & 31);
        return act ? t : 0;
    }
    return act ? (int)T.row[x0 >> T.bsh] : 0;
}

// ------------------------------------------------- rows (z even, y even) --
// Class (x) only.  Two-pass form: first pass at every x-odd point that is not
// a second-pass member, second pass (x = 3 mod 4 under a same-level variant)
// one chunk behind, reading the first-pass values at x +- 2 from the row buffer.
template <int DIR, int S>
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
    const RowTags T = row_tags(D, A, z, y, lane);
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
            const int tag = tag_at(T, x0, act);
            if (act) {
                w = ldl<S>(wrow, x0);
                o = oop ? ldl<S>(orow, x0) : w;
                if (x0 >= 4) wp = ldl<S>(wrow, x0 - 4);  // coarse x0 - 2 (the neighbouring lane's line: L1 hit)
                if (x0 + 4 < Lx) wn = ldl<S>(wrow, x0 + 4);
            }
            same = act && tag_same(tag);
            nat = tag == 4;
            const int fi = tag_fam(tag);
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
                const bool r4 = x0 + 4 <= Lx - 1;
                const double d0 = (double)w.x, d2 = (double)w.z, d4 = (double)wn.x;
                const double pr1 = pred_gen(fi, (double)wp.z, d0, d2, d4, true, x0 >= 2 && r4, x0 + 1, Lx);
                point1<DIR>(q, A, pr1, o.y, &c1, cmA, z, y, x0 + 1, ciA, &r1);
                if (DIR == HPEZ_COMPRESS) A.codes[ciA] = (uint16_t)c1;
                rb[x0 >> 1] = (double)r1;
                if (!same) {
                    const double pr3 = pred_gen(fi, d0, d2, d4, (double)wn.z, r4, x0 + 6 <= Lx - 1, x0 + 3, Lx);
                    point1<DIR>(q, A, pr3, o.w, &c3, cmA, z, y, x0 + 3, ciA + 1, &r3);
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
                point1<DIR>(q, A, pr, p_o3, &c3, cmB, z, y, p_x0 + 3, p_ci, &p_r3);
                if (DIR == HPEZ_COMPRESS) A.codes[p_ci] = (uint16_t)c3;
            }
            stl<S, 10>(A.work + rowoff, p_x0, make_float4(p_w0, p_r1, p_w2, p_r3));
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

// Rows whose blocks carry no same-level variant have a single pass: the four
// x-odd points of a lane from its own two 16-byte words and the next coarse
// value (shuffled from the next lane); only rows that cross a same-level
// block take the two-pass routine above.
template <int DIR, int S>
__device__ __forceinline__ void process_row0(const RowDesc &D, const RowRun &A, const Q &q, int z, int y, double *rb,
                                             int lane) {
    const int Lx = D.L[2];
    if (D.any_same) {
        bool s = false;
        if (D.has_table) {
            const int nbx = ((Lx - 1) >> D.bsh) + 1;
            const uint8_t *t = A.table + (z >> D.bsh) * D.bs0 + (y >> D.bsh) * D.bs1;
            for (int b = lane; b < nbx; b += 32) s |= tag_same(t[b]);
        } else {
            s = true;
        }
        if (__any_sync(0xffffffffu, s)) {
            process_row0_lag<DIR, S>(D, A, q, z, y, rb, lane);
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
    const RowTags T = row_tags(D, A, z, y, lane);
    // eight lattice points (two words, four x-odd points) per lane and iteration
    const int nch = (Lx + 255) >> 8;
    for (int it = 0; it < nch; it++) {
        const int x0 = (it << 8) + (lane << 3);
        const bool actA = x0 < Lx, actB = x0 + 4 < Lx;
        const int tagA = tag_at(T, x0, actA), tagB = tag_at(T, x0 + 4, actB);
        const int fA = tag_fam(tagA), fB = tag_fam(tagB);
        const bool lin = !__any_sync(0xffffffffu, (fA | fB) != 0);
        float4 wa = make_float4(0, 0, 0, 0), wb = wa, oa = wa, ob = wa;
        int32_t c1 = 0, c3 = 0, c5 = 0, c7 = 0;
        const int64_t ci = baseA + 4 * ((it << 5) + lane);
        if (actA) {
            wa = ldl<S>(wrow, x0);
            oa = oop ? ldl<S>(orow, x0) : wa;
            if (DIR == HPEZ_DECOMPRESS) load_codes2(A.codes + ci, &c1, &c3);
        }
        if (actB) {
            wb = ldl<S>(wrow, x0 + 4);
            ob = oop ? ldl<S>(orow, x0 + 4) : wb;
            if (DIR == HPEZ_DECOMPRESS) load_codes2(A.codes + ci + 2, &c5, &c7);
        }
        const bool r4 = x0 + 4 <= Lx - 1, r8 = x0 + 8 <= Lx - 1;
        double pr1, pr3, pr5, pr7;
        if (lin) {
            float w8 = __shfl_down_sync(0xffffffffu, wa.x, 1);
            if (lane == 31 && r8) w8 = wrow[S * (uint32_t)(x0 + 8)];
            const double d0 = (double)wa.x, d2 = (double)wa.z, d4 = (double)wb.x, d6 = (double)wb.z;
            pr1 = DA(DM(0.5, d0), DM(0.5, d2));
            pr3 = r4 ? DA(DM(0.5, d2), DM(0.5, d4)) : DM(1.0, d2);
            pr5 = DA(DM(0.5, d4), DM(0.5, d6));
            pr7 = r8 ? DA(DM(0.5, d6), DM(0.5, (double)w8)) : DM(1.0, d6);
        } else {
            float4 wp = make_float4(0, 0, 0, 0), wn = wp;
            if (actA && x0 >= 4) wp = ldl<S>(wrow, x0 - 4);
            if (r8) wn = ldl<S>(wrow, x0 + 8);
            const double d0 = (double)wa.x, d2 = (double)wa.z, d4 = (double)wb.x, d6 = (double)wb.z;
            const double d8 = (double)wn.x, d10 = (double)wn.z;
            pr1 = pred_gen(fA, (double)wp.z, d0, d2, d4, true, x0 >= 2 && r4, x0 + 1, Lx);
            pr3 = pred_gen(fA, d0, d2, d4, d6, r4, x0 + 6 <= Lx - 1, x0 + 3, Lx);
            pr5 = pred_gen(fB, d2, d4, d6, d8, true, r8, x0 + 5, Lx);
            pr7 = pred_gen(fB, d4, d6, d8, d10, r8, x0 + 10 <= Lx - 1, x0 + 7, Lx);
        }
        if (actA) {
            float r1, r3;
            point2<DIR>(q, A, pr1, pr3, oa.y, oa.w, &c1, &c3, cmA, z, y, x0 + 1, x0 + 3, ci, &r1, &r3);
            if (DIR == HPEZ_COMPRESS) store_codes2(A.codes + ci, c1, c3);
            stl<S, 10>(A.work + rowoff, x0, make_float4(wa.x, r1, wa.z, r3));
        }
        if (actB) {
            float r5, r7;
            point2<DIR>(q, A, pr5, pr7, ob.y, ob.w, &c5, &c7, cmA, z, y, x0 + 5, x0 + 7, ci + 2, &r5, &r7);
            if (DIR == HPEZ_COMPRESS) store_codes2(A.codes + ci + 2, c5, c7);
            stl<S, 10>(A.work + rowoff, x0 + 4, make_float4(wb.x, r5, wb.z, r7));
        }
    }
}

// ------------------------------------- rows with z and/or y odd (RT 1..3) --
// Iteration `it` runs stage E of chunk it -- class E at x0, x0 + 2 from the
// .x/.z components of the neighbouring rows' words, results into the row
// buffer -- and then stage O of chunk it - 1: class O at x0 + 1, x0 + 3 from
// the .y/.w components of the same words (re-requested: they were fetched
// one iteration ago and hit L1) plus the row buffer's E values at x +- 1, 3,
// which by then include the first values of chunk it.  Chunks whose blocks
// all carry tag 0 (multidim linear) away from the grid faces take a
// straight-line path with per-row tap pointers; the general path selects the
// row per lane.
struct CrossTaps {  // one cross axis of a row: coordinate, extent, clamped element offsets of -3, -1, +1, +3, -2, +2
    int c, L, off[4], off2[2];
    bool in1, in3;  // c + 1 <= L - 1; c - 3 >= 0 and c + 3 <= L - 1
};

// quant_f32 that also hands back the f64 image of the stored value (for the row buffer)
__device__ __forceinline__ int32_t quant_f32d(const Q &q, double pred, float origf, float *out, double *outd) {
    const double orig = (double)origf;
    const double d = __dsub_rn(orig, pred);
    double x = __dmul_rn(d, q.inv_two_e);
    const double y = __dadd_rn(fabs(x), 0.5);
    double fl = floor(y);
    const double fr = __dsub_rn(y, fl);
    if (fr < 0x1p-20 || fr > 1.0 - 0x1p-20) {  // |x| + 0.5 >= 2^20 fails fl < R below on either path
        x = __ddiv_rn(d, q.two_e);
        fl = floor(__dadd_rn(fabs(x), 0.5));
    }
    const double k = copysign(fl, x);
    const float rf = __double2float_rn(__dadd_rn(pred, __dmul_rn(q.two_e, k)));
    const double rd = (double)rf;
    const bool ok = fl < q.Rd && fabs(__dsub_rn(rd, orig)) <= q.bound;
    *out = ok ? rf : origf;
    *outd = ok ? rd : orig;
    return ok ? (int32_t)k + q.R : 0;
}

template <int DIR, int S, int RT, bool BROW>
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
    float *__restrict__ wout = A.work + rowoff;
    CrossTaps X[NC];
    const float *pm[NC], *pp[NC];  // rows at -1 / +1 of each cross axis
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
        pm[t] = wrow + X[t].off[1];
        pp[t] = wrow + X[t].off[2];
    }
    int64_t baseEA = D.level_base + A.rowbase[D.segA[CE] + rowidx];
    int64_t baseEB = BROW ? D.level_base + A.rowbase[D.segB[CE] + rowidx] : 0;
    uint16_t *__restrict__ cO = A.codes + (D.level_base + A.rowbase[D.segA[CO] + rowidx]);
    const int cmEA = D.commitA[CE], cmEB = D.commitB[CE], cmO = D.commitA[CO];
    const double we0 = D.w[CE][0], we1 = D.w[CE][1];
    const double wo0 = D.w[CO][0], wo1 = D.w[CO][1], wo2 = D.w[CO][2];
    // one-axis tags: the term each class uses per order p = tag >> 3, 4 bits each
    const uint32_t selE = D.oned_sel[CE], selO = D.oned_sel[CO];
    const uint32_t lt = (1u << lane) - 1u;
    const int nch = (Lx + 127) >> 7;
    const RowTags T = row_tags(D, A, z, y, lane);
    // chunks whose blocks all carry tag 0: bit b of nz set = block b has another tag
    uint32_t nz = 0xffffffffu;
    int bpc = 0;  // blocks per chunk (0: no per-chunk test, every chunk general unless nz == 0)
    if (lin_ok) {
        if (!T.table) {
            nz = T.const_tag == 0 ? 0u : 0xffffffffu;
        } else if (T.in_reg && T.bsh <= 7 && (Lx >> T.bsh) <= 32) {
            nz = __ballot_sync(0xffffffffu, T.reg != 0);
            bpc = 128 >> T.bsh;
        }
    }
    const uint32_t bmask = bpc >= 32 || bpc == 0 ? 0xffffffffu : ((1u << bpc) - 1u);
    auto is_plain = [&](int c) { return ((nz >> (bpc ? c * bpc : 0)) & bmask) == 0; };
    float p_e0 = 0.0f, p_e2 = 0.0f;  // stage E results of the previous chunk (for the finished word)
    for (int it = 0; it <= nch; it++) {
        float n_e0 = 0.0f, n_e2 = 0.0f;
        // ---------------------------------------------------- stage E --
        if (it < nch) {
            const int x0 = (it << 7) + (lane << 2);
            const bool act = x0 < Lx;
            if (HPEZ_ROW_PF && x0 + 128 < Lx) {
                // L1 prefetch of the next chunk's lines (originals and the +-1 rows)
                if (DIR == HPEZ_COMPRESS) prefetch_l1(orow + S * (x0 + 128));
#pragma unroll
                for (int t = 0; t < NC; t++) {
                    prefetch_l1(pm[t] + S * (x0 + 128));
                    prefetch_l1(pp[t] + S * (x0 + 128));
                }
            }
            if (is_plain(it)) {
                const int nact = min(32, (Lx - (it << 7)) >> 2);
                uint16_t *__restrict__ cp = A.codes + baseEA + 2 * lane;
                baseEA += 2 * nact;
                if (act) {
                    float ox = 0.0f, oz = 0.0f;
                    int32_t c0 = 0, c2 = 0;
                    if (DIR == HPEZ_COMPRESS) {
                        const float4 o = ldl<S>(orow, x0);
                        ox = o.x;
                        oz = o.z;
                    } else {
                        c0 = cp[0];
                        c2 = cp[1];
                    }
                    double pa[NC], pb[NC];
#pragma unroll
                    for (int t = 0; t < NC; t++) {
                        const float4 a = ldl<S>(pm[t], x0), b = ldl<S>(pp[t], x0);
                        pa[t] = DA(DM(0.5, (double)a.x), DM(0.5, (double)b.x));
                        pb[t] = DA(DM(0.5, (double)a.z), DM(0.5, (double)b.z));
                    }
                    const double pr0 = NC == 1 ? pa[0] : DA(DM(we0, pa[0]), DM(we1, pa[NC - 1]));
                    const double pr2 = NC == 1 ? pb[0] : DA(DM(we0, pb[0]), DM(we1, pb[NC - 1]));
                    double d0, d2;
                    if (DIR == HPEZ_COMPRESS && q.bound > 0.0) {
                        c0 = quant_f32d(q, pr0, ox, &n_e0, &d0);
                        c2 = quant_f32d(q, pr2, oz, &n_e2, &d2);
                        if (c0 == 0 || c2 == 0) {
                            if (c0 == 0) row_escape(A, cmEA, q.s, z, y, x0);
                            if (c2 == 0) row_escape(A, cmEA, q.s, z, y, x0 + 2);
                        }
                    } else {
                        point2<DIR>(q, A, pr0, pr2, ox, oz, &c0, &c2, cmEA, z, y, x0, x0 + 2, baseEA - 2 * nact + 2 * lane,
                                    &n_e0, &n_e2);
                        d0 = (double)n_e0;
                        d2 = (double)n_e2;
                    }
                    if (DIR == HPEZ_COMPRESS) {
                        cp[0] = (uint16_t)c0;
                        cp[1] = (uint16_t)c2;
                    }
                    *reinterpret_cast<double2 *>(rb + (x0 >> 1)) = make_double2(d0, d2);
                }
            } else {
                const int tag = tag_at(T, x0, act);
                const int fi = tag_fam(tag);
                const int p = tag >> 3;
                const int sel = p ? (int)((selE >> (4 * (p - 1))) & 15u) : -1;
                const bool isB = BROW && act && tag_same(tag);
                int64_t ci;
                const uint32_t am = __ballot_sync(0xffffffffu, act && !isB);
                if (BROW) {
                    const uint32_t bm = __ballot_sync(0xffffffffu, isB);
                    ci = isB ? baseEB + 2 * __popc(bm & lt) : baseEA + 2 * __popc(am & lt);
                    baseEB += 2 * __popc(bm);
                } else {
                    ci = baseEA + 2 * lane;
                }
                baseEA += 2 * __popc(am);
                if (act) {
                    float4 o = make_float4(0, 0, 0, 0);
                    int32_t c0 = 0, c2 = 0;
                    if (DIR == HPEZ_COMPRESS) o = ldl<S>(orow, x0);
                    else load_codes2(A.codes + ci, &c0, &c2);
                    double pr0, pr2;
                    if (isB) {  // second same-level pass along the class axis (NC == 1)
                        float4 a[6];
#pragma unroll
                        for (int i = 0; i < 4; i++) a[i] = ldl<S>(wrow + X[0].off[i], x0);
                        a[4] = ldl<S>(wrow + X[0].off2[0], x0);
                        a[5] = ldl<S>(wrow + X[0].off2[1], x0);
                        const int nat = tag == 4;
                        pr0 = pred_same(nat, (double)a[0].x, (double)a[4].x, (double)a[1].x, (double)a[2].x,
                                        (double)a[5].x, (double)a[3].x, X[0].c, X[0].L);
                        pr2 = pred_same(nat, (double)a[0].z, (double)a[4].z, (double)a[1].z, (double)a[2].z,
                                        (double)a[5].z, (double)a[3].z, X[0].c, X[0].L);
                    } else {
                        double pa[NC], pb[NC];
#pragma unroll
                        for (int t = 0; t < NC; t++) {
                            float4 a[4];
                            a[0] = a[3] = make_float4(0, 0, 0, 0);
                            a[1] = ldl<S>(pm[t], x0);
                            a[2] = ldl<S>(pp[t], x0);
                            if (fi) {
                                a[0] = ldl<S>(wrow + X[t].off[0], x0);
                                a[3] = ldl<S>(wrow + X[t].off[3], x0);
                            }
                            pa[t] = pred_gen(fi, (double)a[0].x, (double)a[1].x, (double)a[2].x, (double)a[3].x,
                                             X[t].in1, X[t].in3, X[t].c, X[t].L);
                            pb[t] = pred_gen(fi, (double)a[0].z, (double)a[1].z, (double)a[2].z, (double)a[3].z,
                                             X[t].in1, X[t].in3, X[t].c, X[t].L);
                        }
                        pr0 = combine_terms<NC>(pa, sel, we0, we1, 0.0);
                        pr2 = combine_terms<NC>(pb, sel, we0, we1, 0.0);
                    }
                    const int cm = isB ? cmEB : cmEA;
                    point2<DIR>(q, A, pr0, pr2, o.x, o.z, &c0, &c2, cm, z, y, x0, x0 + 2, ci, &n_e0, &n_e2);
                    if (DIR == HPEZ_COMPRESS) store_codes2(A.codes + ci, c0, c2);
                    *reinterpret_cast<double2 *>(rb + (x0 >> 1)) = make_double2((double)n_e0, (double)n_e2);
                }
            }
        }
        __syncwarp();
        // ---------------------------------------------------- stage O --
        if (it > 0) {
            const int x0 = ((it - 1) << 7) + (lane << 2);
            const bool act = x0 < Lx;
            const int h = x0 >> 1;
            const bool r4 = x0 + 4 <= Lx - 1;
            uint16_t *__restrict__ cp = cO + 2 * (((it - 1) << 5) + lane);
            if (is_plain(it - 1)) {
                if (act) {
                    float oy = 0.0f, ow = 0.0f;
                    int32_t c1 = 0, c3 = 0;
                    if (DIR == HPEZ_COMPRESS) {
                        const float4 o = ldl<S>(orow, x0);
                        oy = o.y;
                        ow = o.w;
                    } else {
                        c1 = cp[0];
                        c3 = cp[1];
                    }
                    const double2 e02 = *reinterpret_cast<const double2 *>(rb + h);
                    const double e4 = rb[min(h + 2, hx - 1)];
                    double pa[NC + 1], pb[NC + 1];
#pragma unroll
                    for (int t = 0; t < NC; t++) {
                        const float4 a = ldl<S>(pm[t], x0), b = ldl<S>(pp[t], x0);
                        pa[t] = DA(DM(0.5, (double)a.y), DM(0.5, (double)b.y));
                        pb[t] = DA(DM(0.5, (double)a.w), DM(0.5, (double)b.w));
                    }
                    pa[NC] = DA(DM(0.5, e02.x), DM(0.5, e02.y));
                    pb[NC] = r4 ? DA(DM(0.5, e02.y), DM(0.5, e4)) : DM(1.0, e02.y);
                    double pr1, pr3;
                    if (NC == 1) {
                        pr1 = DA(DM(wo0, pa[0]), DM(wo1, pa[1]));
                        pr3 = DA(DM(wo0, pb[0]), DM(wo1, pb[1]));
                    } else {
                        pr1 = DA(DA(DM(wo0, pa[0]), DM(wo1, pa[1])), DM(wo2, pa[NC]));
                        pr3 = DA(DA(DM(wo0, pb[0]), DM(wo1, pb[1])), DM(wo2, pb[NC]));
                    }
                    float r1, r3;
                    if (DIR == HPEZ_COMPRESS && q.bound > 0.0) {
                        c1 = quant_f32(q, pr1, oy, &r1);
                        c3 = quant_f32(q, pr3, ow, &r3);
                        if (c1 == 0 || c3 == 0) {
                            if (c1 == 0) row_escape(A, cmO, q.s, z, y, x0 + 1);
                            if (c3 == 0) row_escape(A, cmO, q.s, z, y, x0 + 3);
                        }
                    } else {
                        point2<DIR>(q, A, pr1, pr3, oy, ow, &c1, &c3, cmO, z, y, x0 + 1, x0 + 3, (int64_t)(cp - A.codes),
                                    &r1, &r3);
                    }
                    if (DIR == HPEZ_COMPRESS) {
                        cp[0] = (uint16_t)c1;
                        cp[1] = (uint16_t)c3;
                    }
                    stl<S, 15>(wout, x0, make_float4(p_e0, r1, p_e2, r3));
                }
            } else {
                const int tag = tag_at(T, x0, act);
                const int fi = tag_fam(tag);
                const int p = tag >> 3;
                const int sel = p ? (int)((selO >> (4 * (p - 1))) & 15u) : -1;
                if (act) {
                    const int64_t ci = (int64_t)(cp - A.codes);
                    float4 o = make_float4(0, 0, 0, 0);
                    int32_t c1 = 0, c3 = 0;
                    if (DIR == HPEZ_COMPRESS) o = ldl<S>(orow, x0);
                    else load_codes2(cp, &c1, &c3);
                    const double2 e02 = *reinterpret_cast<const double2 *>(rb + h);
                    double pa[NC + 1], pb[NC + 1];
#pragma unroll
                    for (int t = 0; t < NC; t++) {
                        float4 a[4];
                        a[0] = a[3] = make_float4(0, 0, 0, 0);
                        a[1] = ldl<S>(pm[t], x0);
                        a[2] = ldl<S>(pp[t], x0);
                        if (fi) {
                            a[0] = ldl<S>(wrow + X[t].off[0], x0);
                            a[3] = ldl<S>(wrow + X[t].off[3], x0);
                        }
                        pa[t] = pred_gen(fi, (double)a[0].y, (double)a[1].y, (double)a[2].y, (double)a[3].y, X[t].in1,
                                         X[t].in3, X[t].c, X[t].L);
                        pb[t] = pred_gen(fi, (double)a[0].w, (double)a[1].w, (double)a[2].w, (double)a[3].w, X[t].in1,
                                         X[t].in3, X[t].c, X[t].L);
                    }
                    const double xm2 = rb[max(h - 1, 0)], x4v = rb[min(h + 2, hx - 1)], x6v = rb[min(h + 3, hx - 1)];
                    pa[NC] = pred_gen(fi, xm2, e02.x, e02.y, x4v, true, x0 >= 2 && r4, x0 + 1, Lx);
                    pb[NC] = pred_gen(fi, e02.x, e02.y, x4v, x6v, r4, x0 + 6 <= Lx - 1, x0 + 3, Lx);
                    const double pr1 = combine_terms<NC + 1>(pa, sel, wo0, wo1, wo2);
                    const double pr3 = combine_terms<NC + 1>(pb, sel, wo0, wo1, wo2);
                    float r1, r3;
                    point2<DIR>(q, A, pr1, pr3, o.y, o.w, &c1, &c3, cmO, z, y, x0 + 1, x0 + 3, ci, &r1, &r3);
                    if (DIR == HPEZ_COMPRESS) store_codes2(cp, c1, c3);
                    stl<S, 15>(wout, x0, make_float4(p_e0, r1, p_e2, r3));
                }
            }
        }
        p_e0 = n_e0;
        p_e2 = n_e2;
    }
}

// RTM: the row types a launch holds (1: (z even, y even); 6 / 7: one of z, y odd, first-pass /
// second-pass rows; 8: both odd), so each instantiation carries -- and is register-allocated for -- only
// its own routines.
template <int DIR, int S, int RTM>
__global__ void __launch_bounds__(kRowThreads, RTM == 1 ? HPEZ_ROW_OCC0 : RTM == 8 ? HPEZ_ROW_OCC8 : HPEZ_ROW_OCC)
    row_kernel(const __grid_constant__ RowDesc D, const __grid_constant__ RowRun A, const __grid_constant__ RowLaunch L) {
    extern __shared__ double s_rb[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *rb = s_rb + (size_t)warp * ((D.L[2] >> 1) + 4);
    Q q;
    q.bound = D.bound;
    q.two_e = D.two_e;
    q.inv_two_e = D.inv_two_e;
    q.R = D.R;
    q.Rd = (double)D.R;
    q.s = D.s;
    const int nw = (int)gridDim.x * kRowWarps;
    const int n0 = L.s[0].nz * L.s[0].ny;
    for (int r = (int)blockIdx.x * kRowWarps + warp; r < L.total; r += nw) {
        const RowSet &S0 = r < n0 ? L.s[0] : L.s[1];
        const int rr = r < n0 ? r : r - n0;
        const int iz = rr / S0.ny, iy = rr - iz * S0.ny;
        const int z = S0.z0 + iz * S0.zs, y = S0.y0 + iy * S0.ys;
        const int kind = S0.rt * 2 + S0.brow;
        if (RTM == 1) {
            process_row0<DIR, S>(D, A, q, z, y, rb, lane);
        } else if (RTM == 6) {  // one of z, y odd, no second-pass lanes in these rows
            if (kind == 2) process_rowN<DIR, S, 1, false>(D, A, q, z, y, rb, lane);
            else process_rowN<DIR, S, 2, false>(D, A, q, z, y, rb, lane);
        } else if (RTM == 7) {  // one of z, y odd, second same-level pass rows
            if (kind == 3) process_rowN<DIR, S, 1, true>(D, A, q, z, y, rb, lane);
            else process_rowN<DIR, S, 2, true>(D, A, q, z, y, rb, lane);
        } else {
            process_rowN<DIR, S, 3, false>(D, A, q, z, y, rb, lane);
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

static bool tag_supported(int tag) {
    const int k = tag & 7, p = tag >> 3;
    if (k >= 5 || p > 6) return false;
    return p == 0 || k == 0 || k == 1 || k == 3;  // one-axis tags: no same-level split
}

bool row_plan_build(const GridDev &g, const CommitDev *cms, const uint32_t *vmask, int n, int first_commit,
                    const uint8_t *tbl, int64_t nblk, int level_tag, int64_t level_base, RowPlan *out) {
    RowPlan P;
    RowDesc &D = P.d;
    memset(&D, 0, sizeof D);
    if (g.rank != 3 || n < 7) return false;
    const int s = cms[0].s;
    if (s != 1 && s != 2 && s != 4) return false;
    D.s = s;
    for (int a = 0; a < 3; a++) {
        D.L[a] = (g.dims[a] - 1) / s + 1;
        if (D.L[a] < 8) return false;
    }
    if (D.L[2] % 4 != 0 || g.dims[2] % 4 != 0 || g.estr[2] != 1) return false;
    if (g.npts >= (1ll << 31) || g.radius > 32768) return false;
    D.E0 = g.estr[0] * s;
    D.E1 = g.estr[1] * s;
    D.R = (int32_t)g.radius;
    D.has_table = tbl != nullptr;
    D.const_tag = level_tag;
    D.any_same = 0;
    if (tbl) {
        int sl = 0;
        while ((1 << sl) < s) sl++;
        if (g.bs_log2 < 2 + sl) return false;  // a lane's four lattice points share one block
        D.bsh = g.bs_log2 - sl;
        D.bs0 = g.bstr[0];
        D.bs1 = g.bstr[1];
        for (int64_t b = 0; b < nblk; b++) {
            if (!tag_supported(tbl[b])) return false;
            D.any_same |= tag_same(tbl[b]);
        }
    } else {
        if (!tag_supported(level_tag)) return false;
        D.any_same = tag_same(level_tag);
        // a level that is same-level throughout runs every row on the two-stream routines, which
        // the flow kernel beats (cfg2: 0.58 / 0.52 ms against 0.51 / 0.44 ms); HPEZ_ROW=2 forces it
        const char *ev = getenv("HPEZ_ROW");
        if (D.any_same && !(ev && atoi(ev) == 2)) return false;
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
    // one-axis orders (plan.order_candidates, plan.py:37-51): the term index of the axis visited last
    static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    for (int c = 0; c < 7; c++) {
        const int vm = class_vmask(c);
        uint32_t packed = 0;
        for (int p = 0; p < 6; p++) {
            int best = -1, bpos = -1;
            for (int a = 0; a < 3; a++)
                if (vm >> a & 1)
                    for (int j = 0; j < 3; j++)
                        if (perms[p][j] == a && j > bpos) {
                            bpos = j;
                            best = a;
                        }
            int term = 0;
            for (int a = 0; a < best; a++)
                if (vm >> a & 1) term++;
            packed |= (uint32_t)term << (4 * p);
        }
        D.oned_sel[c] = packed;
    }
    // MD blend weights per class (interp._blend_weights, interp.py:233-238)
    bool have_w[7] = {true, true, true, false, false, false, false};
    // commits of the level -> (class, pass)
    for (int i = 0; i < n; i++) {
        const CommitDev &cm = cms[i];
        const int c = cls_of_vmask(vmask[i]);
        if (c < 0 || cm.s != s) return false;
        const bool single = c < 3;
        bool second = false;
        if (cm.kind == COMMIT_UNIFORM) {
            if (single) {
                if (cm.pred.md || cm.pred.axis != c) return false;
                second = cm.start[c] == 3 * s;  // phase lattice 3s, 7s, ... of a split class (interp.py:333-341)
                if (second != (cm.pred.fam == FAM_NAK_S || cm.pred.fam == FAM_NAT_S)) return false;
            } else if (cm.pred.md) {
                for (int t = 0; t < 3; t++) D.w[c][t] = cm.pred.w[t];
                have_w[c] = true;
            } else {
                have_w[c] = true;  // a one-axis class never blends
            }
        } else {
            second = cm.kind == COMMIT_MIXED_B;
            if (second && (!single || cm.phase != 0)) return false;
            if (!single) {
                for (int t = 0; t < 3; t++) D.w[c][t] = cm.pred.w[t];
                have_w[c] = true;
            }
        }
        int32_t &slot = second ? D.commitB[c] : D.commitA[c];
        if (slot >= 0) return false;
        slot = first_commit + i;
    }
    for (int c = 0; c < 7; c++)
        if (D.commitA[c] < 0 || !have_w[c]) return false;
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
        RowSet rs{};
        rs.rt = rt;
        rs.brow = brow;
        rs.z0 = z0;
        rs.zs = zs;
        rs.nz = cnt(z0, Lz, zs);
        rs.y0 = y0;
        rs.ys = ys;
        rs.ny = cnt(y0, Ly, ys);
        return rs;
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
    if (P.smem > 64 * 1024) return false;
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

typedef void (*row_fn)(const RowDesc, const RowRun, const RowLaunch);

template <int DIR, int S>
static row_fn pick_rtm(int rtm) {
    return rtm == 1 ? row_kernel<DIR, S, 1> : rtm == 6 ? row_kernel<DIR, S, 6> : rtm == 7 ? row_kernel<DIR, S, 7> : row_kernel<DIR, S, 8>;
}
template <int DIR>
static row_fn pick_row(int s, int rtm) {
    return s == 1 ? pick_rtm<DIR, 1>(rtm) : s == 2 ? pick_rtm<DIR, 2>(rtm) : pick_rtm<DIR, 4>(rtm);
}

cudaError_t row_plan_launch(const RowPlan &p, int dir, const RowRun &r, cudaStream_t st) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    for (int i = 0; i < p.n_launch; i++) {
        const RowLaunch &l = p.launch[i];
        if (l.total <= 0) continue;
        const int rt = l.s[0].rt;
        const int rtm = rt == 0 ? 1 : rt == 3 ? 8 : (l.s[0].brow ? 7 : 6);
        row_fn f = dir == HPEZ_COMPRESS ? pick_row<HPEZ_COMPRESS>(p.d.s, rtm) : pick_row<HPEZ_DECOMPRESS>(p.d.s, rtm);
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, p.threads, p.smem) != cudaSuccess || occ < 1) occ = 1;
        const int grid = std::max(1, std::min((l.total + kRowWarps - 1) / kRowWarps, occ * sms));
        f<<<grid, p.threads, p.smem, st>>>(p.d, r, l);
    }
    return cudaGetLastError();
}

}  // namespace hpez
