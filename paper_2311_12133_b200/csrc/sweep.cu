// sweep.cu -- B200 multi-level interpolation predict/quantize sweep and its
// inverse: the drop-in for interp.run_levels (interp.py:440-472).
//
// Host side: a plan restates the reference's commit schedule -- levels
// coarse to fine, parity classes combinations(active, m) in lexicographic
// order (interp.py:415-433), uniform commits with the optional same-level
// two-phase split (interp.py:322-341) and mixed per-block commits A / B_phase
// (interp.py:350-411).  Every commit's lattice is cut into work items
// (contiguous position ranges in row-major = stream order, 8 warps each).
//
// Device side (one sweep = a handful of launches):
//   * coarse kernel: one 1024-thread CTA runs the leading tiny commits back to
//     back with __syncthreads between commits (no launch or flag latency);
//   * flow kernel: a persistent grid pulls items in stream order from an
//     atomic counter, waits on per-item completion flags of the previous
//     commit's items within the stencil reach (+-3s along the outer axis),
//     predicts/quantizes its positions and publishes its flag.  Commits thus
//     pipeline plane by plane and the working set stays in the 126 MB L2;
//   * escapes are counted per (item, warp): compress compacts the outliers in
//     stream order afterwards (their originals are still in the grid),
//     decompress ranks them with a counting pre-pass over the code stream.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <set>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "pairwise.cuh"
#include "scan.cuh"
#include "stencil.cuh"
#include "tile.h"
#include "row.h"

#ifndef HPEZ_L1_PREFETCH
#define HPEZ_L1_PREFETCH 0  // measured slower on B200 (kept for experiments)
#endif
#ifndef HPEZ_FLOW_OCC
#define HPEZ_FLOW_OCC 4  // flow-kernel CTAs per SM the fast path is compiled for
#endif
#ifndef HPEZ_ILP2
#define HPEZ_ILP2 1  // fast path: two interior iterations per step
#endif

namespace hpez {

__constant__ RowEntry c_rows[kFamilies][64];
__constant__ FamDesc c_fam[kFamilies];

// ---------------------------------------------------------------- rows --
static const int kFamN[kFamilies] = {2, 4, 4, 4, 6};
static const int kFamU[kFamilies][6] = {{-1, 1}, {-3, -1, 1, 3}, {-3, -1, 1, 3},
                                        {-2, -1, 1, 2}, {-3, -2, -1, 1, 2, 3}};
// Full rows, exact rationals of kernels.py:43-74.
static const int kFamP[kFamilies][6] = {{1, 1}, {-1, 9, 9, -1}, {-3, 23, 23, -3},
                                        {-1, 4, 4, -1}, {3, -18, 46, 46, -18, 3}};
static const int kFamQ[kFamilies][6] = {{2, 2}, {16, 16, 16, 16}, {40, 40, 40, 40},
                                        {6, 6, 6, 6}, {62, 62, 62, 62, 62, 62}};

static RowEntry full_row(int fam) {
    RowEntry r{};
    r.n = kFamN[fam];
    for (int i = 0; i < r.n; i++) {
        r.off[i] = kFamU[fam][i];
        r.coef[i] = (double)kFamP[fam][i] / (double)kFamQ[fam][i];
    }
    return r;
}

// Edge-truncated rows (kernels.py:78-86).
static bool edge_row(const std::vector<int> &offs, RowEntry *r) {
    struct E { std::vector<int> off, p, q; };
    static const E tab[] = {
        {{-1, 1, 3}, {3, 3, -1}, {8, 4, 8}},  {{-3, -1, 1}, {-1, 3, 3}, {8, 4, 8}},
        {{-2, -1, 1}, {-1, 1, 1}, {3, 1, 3}}, {{-1, 1}, {1, 1}, {2, 2}},
        {{-3, -1}, {-1, 3}, {2, 2}},          {{-2, -1}, {-1, 2}, {1, 1}},
        {{-1}, {1}, {1}},
    };
    for (const E &e : tab) {
        if (e.off != offs) continue;
        *r = RowEntry{};
        r->n = (int)offs.size();
        for (int i = 0; i < r->n; i++) {
            r->off[i] = offs[i];
            r->coef[i] = (double)e.p[i] / (double)e.q[i];
        }
        return true;
    }
    return false;
}

// kernels.resolve_row (kernels.py:106-150) for one availability mask.
static RowEntry resolve(int fam, uint32_t mask) {
    const int n = kFamN[fam];
    if (mask == (1u << n) - 1u) return full_row(fam);
    std::set<int> keep;
    for (int i = 0; i < n; i++)
        if (mask >> i & 1) keep.insert(kFamU[fam][i]);
    auto sub = [&](std::initializer_list<int> c) {
        for (int v : c)
            if (!keep.count(v)) return false;
        return true;
    };
    std::vector<int> offs;
    if (fam == FAM_LIN_I) {
        offs = {-1};
    } else if (fam == FAM_NAK_I || fam == FAM_NAT_I) {
        if (sub({-1, 1, 3})) offs = {-1, 1, 3};
        else if (sub({-3, -1, 1})) offs = {-3, -1, 1};
        else if (sub({-1, 1})) offs = {-1, 1};
        else if (sub({-3, -1})) offs = {-3, -1};
        else offs = {-1};
    } else {
        if (sub({-2, -1, 1, 2})) offs = {-2, -1, 1, 2};
        else if (sub({-2, -1, 1})) offs = {-2, -1, 1};
        else if (sub({-2, -1})) offs = {-2, -1};
        else offs = {-1};
    }
    RowEntry r;
    if (!edge_row(offs, &r)) r = full_row(FAM_NAK_S);  // truncated 6-pt SL row
    return r;
}

static cudaError_t upload_rows() {
    static bool done = false;
    if (done) return cudaSuccess;
    static RowEntry rows[kFamilies][64];
    static FamDesc fam[kFamilies];
    for (int f = 0; f < kFamilies; f++) {
        fam[f] = FamDesc{};
        fam[f].n = kFamN[f];
        for (int i = 0; i < kFamN[f]; i++) fam[f].u[i] = kFamU[f][i];
        for (uint32_t m = 0; m < 64; m++) rows[f][m] = (m < (1u << kFamN[f])) ? resolve(f, m) : RowEntry{};
    }
    cudaError_t e = cudaMemcpyToSymbol(c_rows, rows, sizeof rows);
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_fam, fam, sizeof fam);
    if (e == cudaSuccess) done = true;
    return e;
}

// ---------------------------------------------------------- predictions --
// Grid reads go through L1: a unit starts only after a gpu-scope fence that
// invalidates this SM's L1 (MEMBAR.SC.GPU + CCTL.IVALL) and reads only points
// finalised by the commits it waited on.
template <typename T>
__device__ __forceinline__ double ldv(const T *__restrict__ w, int64_t i) {
    return (double)w[i];
}

// DM / DA: separately rounded f64 multiply / add (stencil.cuh)

// Generic row through the constant table (edges; any family).
template <typename T>
__device__ __noinline__ double pred_table(const T *__restrict__ w, int64_t idx, int c, int E, int s,
                                          int64_t sE, int fam) {
    const FamDesc &fd = c_fam[fam];
    uint32_t mask = 0;
    for (int i = 0; i < fd.n; i++) {
        const int p = c + fd.u[i] * s;
        mask |= (uint32_t)(p >= 0 && p < E) << i;
    }
    const RowEntry &r = c_rows[fam][mask];
    double acc = DM(r.coef[0], ldv(w, idx + r.off[0] * sE));
    for (int k = 1; k < r.n; k++) acc = DA(acc, DM(r.coef[k], ldv(w, idx + r.off[k] * sE)));
    return acc;
}

// 1-D prediction at grid index idx, coordinate c along an axis of extent E,
// stride s, element step sE = s * estr.  Interior points use the full row
// with literal coefficients; edge points fall back to the resolved table.
template <typename T>
__device__ __forceinline__ double pred_1d(const T *__restrict__ w, int64_t idx, int c, int E, int s,
                                          int64_t sE, int fam) {
    switch (fam) {
    case FAM_LIN_I:
        if (c + s <= E - 1) return DA(DM(0.5, ldv(w, idx - sE)), DM(0.5, ldv(w, idx + sE)));
        return DM(1.0, ldv(w, idx - sE));
    case FAM_NAK_I:
        if (c >= 3 * s && c + 3 * s <= E - 1) {
            const double a = ldv(w, idx - 3 * sE), b = ldv(w, idx - sE), d = ldv(w, idx + sE),
                         e = ldv(w, idx + 3 * sE);
            return DA(DA(DA(DM(-1.0 / 16, a), DM(9.0 / 16, b)), DM(9.0 / 16, d)), DM(-1.0 / 16, e));
        }
        break;
    case FAM_NAT_I:
        if (c >= 3 * s && c + 3 * s <= E - 1) {
            const double a = ldv(w, idx - 3 * sE), b = ldv(w, idx - sE), d = ldv(w, idx + sE),
                         e = ldv(w, idx + 3 * sE);
            return DA(DA(DA(DM(-3.0 / 40, a), DM(23.0 / 40, b)), DM(23.0 / 40, d)), DM(-3.0 / 40, e));
        }
        break;
    case FAM_NAK_S:
        if (c + 2 * s <= E - 1) {  // same-level targets sit at >= 3s
            const double a = ldv(w, idx - 2 * sE), b = ldv(w, idx - sE), d = ldv(w, idx + sE),
                         e = ldv(w, idx + 2 * sE);
            return DA(DA(DA(DM(-1.0 / 6, a), DM(4.0 / 6, b)), DM(4.0 / 6, d)), DM(-1.0 / 6, e));
        }
        break;
    default:  // FAM_NAT_S
        if (c + 3 * s <= E - 1) {
            const double a = ldv(w, idx - 3 * sE), b = ldv(w, idx - 2 * sE), d = ldv(w, idx - sE),
                         e = ldv(w, idx + sE), f = ldv(w, idx + 2 * sE), h = ldv(w, idx + 3 * sE);
            return DA(DA(DA(DA(DA(DM(3.0 / 62, a), DM(-18.0 / 62, b)), DM(46.0 / 62, d)),
                            DM(46.0 / 62, e)), DM(-18.0 / 62, f)), DM(3.0 / 62, h));
        }
        break;
    }
    return pred_table(w, idx, c, E, s, sE, fam);
}

// Register copy of a predictor (uniform per warp for uniform commits).
struct PredReg {
    int md, axis, fam, nax;
    int axes[kMaxRank];
    double w[kMaxRank];
};

__device__ __forceinline__ PredReg load_pred(const PredDev &p) {
    PredReg r;
    r.md = p.md;
    r.axis = p.axis;
    r.fam = p.fam;
    r.nax = p.nax;
#pragma unroll
    for (int i = 0; i < kMaxRank; i++) {
        r.axes[i] = p.axes[i];
        r.w[i] = p.w[i];
    }
    return r;
}

// arr[a] for a runtime-uniform a without local-memory indexing
__device__ __forceinline__ int pick(const int (&arr)[kMaxRank], int a) {
    int v = arr[0];
#pragma unroll
    for (int k = 1; k < kMaxRank; k++) v = a == k ? arr[k] : v;
    return v;
}

template <typename T>
__device__ __forceinline__ double predict(const T *__restrict__ w, int64_t idx, const int (&coord)[kMaxRank],
                                          const int (&dims)[kMaxRank], const int (&estr)[kMaxRank],
                                          const PredReg &p, int s) {
    if (!p.md) {
        const int a = p.axis;
        return pred_1d(w, idx, pick(coord, a), pick(dims, a), s, (int64_t)s * pick(estr, a), p.fam);
    }
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < kMaxRank; i++) {
        if (i < p.nax) {
            const int a = p.axes[i];
            const double t = DM(p.w[i], pred_1d(w, idx, pick(coord, a), pick(dims, a), s,
                                                (int64_t)s * pick(estr, a), p.fam));
            acc = i == 0 ? t : DA(acc, t);
        }
    }
    return acc;
}

// ------------------------------------------------------------ arguments --
struct SweepArgs {
    GridDev g;
    const CommitDev *commits;
    const int32_t *item_commit;
    const int32_t *flow_order;    // flow items in grab order
    const int32_t *dep_off;       // per item: first dependency interval
    const int2 *dep_rng;          // item-id intervals (inclusive)
    const int32_t *coarse_pairs;  // (commit, item) pairs of the coarse prefix
    const int32_t *coarse_groups; // [g0, g1) pair ranges, one per (level, depth)
    int32_t n_coarse_commits;     // commit descriptors [0, n) staged in the coarse kernel's smem
    int32_t n_groups;
    unsigned long long *prof;   // optional phase counters (HPEZ_PROFILE)
    int32_t dbg;                // HPEZ_DEBUG_NODEPS timing experiments only
    int32_t l2_prefetch;        // TMA bulk L2 prefetch of the next item (HPEZ_L2_PREFETCH=1)
    const int64_t *wbase;       // per (item, warp): code index of the first member
    const int32_t *wn;          // per (item, warp): member count
    uint32_t *esc_cnt;          // per (item, warp): escapes (compress, written)
    const int64_t *esc_off;     // per (item, warp): first outlier rank (decompress)
    uint32_t *done;             // per item completion flags
    int32_t *next;              // flow item counter
    int32_t *flags;             // status (outlier underflow)
    const TagInfo *tags;
    const uint8_t *slots;
    const uint8_t *table;
    void *work;
    const void *orig;           // compress: originals (== work when in place)
    void *codes;
    const double *outl;
    int64_t outl_cap;
    double *errbuf;
    double *dense;
    int32_t n_items;            // flow kernel: number of items
};

// Position -> lattice indices (row-major).
__device__ __forceinline__ void decode_pos(const CommitDev &cm, int rank, uint32_t p, int (&j)[kMaxRank]) {
#pragma unroll
    for (int a = kMaxRank - 1; a >= 0; a--) {
        if (a < rank) {
            const uint32_t q = a > 0 ? fdiv(p, cm.fd[a]) : 0u;
            j[a] = (int)(p - q * (uint32_t)cm.cnt[a]);
            p = q;
        }
    }
}

// Mixed-class membership and predictor of one position (interp.py:374-411).
__device__ __forceinline__ const PredDev *mixed_member(const SweepArgs &A, const CommitDev &cm,
                                                       const int (&coord)[kMaxRank], uint32_t jodd,
                                                       bool *member) {
    const GridDev &g = A.g;
    int64_t b = 0;
    if (g.bs_log2 >= 0)
        for (int a = 0; a < g.rank; a++) b += (int64_t)(coord[a] >> g.bs_log2) * g.bstr[a];
    else
        for (int a = 0; a < g.rank; a++) b += (int64_t)(coord[a] / g.block_size) * g.bstr[a];
    const int tag = A.table[(int64_t)cm.level * g.nblk + b];
    const TagInfo &ti = A.tags[cm.tag_off + A.slots[cm.slot_off + tag]];
    const int sp = ti.split;
    if (cm.kind == COMMIT_MIXED_A) {
        *member = sp < 0 || !((jodd >> sp) & 1u);
        return &ti.inter;
    }
    const int key = __popc(cm.axes_present & jodd & ~(1u << (sp < 0 ? 31 : sp)));
    *member = sp >= 0 && ((jodd >> sp) & 1u) && key == cm.phase;
    return &ti.same;
}

// One warp's share of one item: positions [p0, p0 + pw) of commit cm, in
// stream order, 32 at a time.  Commit geometry and the predictor live in
// registers; coordinates use static indexing only.
template <typename T, typename C, int DIR, int ROUND, bool STATS>
__device__ __forceinline__ void process_warp(const SweepArgs &A, const CommitDev &cmS, int item, int warp) {
    const int lane = threadIdx.x & 31;
    const int rank = A.g.rank;
    const uint32_t npos = cmS.npos;
    const uint32_t p0 = (uint32_t)(item - cmS.item_base) * (uint32_t)cmS.p_item + (uint32_t)warp * (uint32_t)cmS.pw;
    const uint32_t pend = min(p0 + (uint32_t)cmS.pw, npos);
    const int e = item * kItemWarps + warp;
    if (p0 >= pend) {
        if (DIR == HPEZ_COMPRESS && lane == 0) A.esc_cnt[e] = 0;
        return;
    }
    int st[kMaxRank], sp[kMaxRank], cn[kMaxRank], dims[kMaxRank], estr[kMaxRank];
#pragma unroll
    for (int a = 0; a < kMaxRank; a++) {
        st[a] = cmS.start[a];
        sp[a] = cmS.step[a];
        cn[a] = cmS.cnt[a];
        dims[a] = A.g.dims[a];
        estr[a] = A.g.estr[a];
    }
    const int s = cmS.s;
    const double bound = cmS.bound, two_e = cmS.two_e, inv_two_e = cmS.inv_two_e;
    const int64_t R = A.g.radius;
    const bool mixed = cmS.kind != COMMIT_UNIFORM;
    const PredReg upred = load_pred(cmS.pred);
    T *__restrict__ work = (T *)A.work;
    C *__restrict__ codes = (C *)A.codes;
    int64_t cbase = A.wbase[e];  // code index of this warp's first member
    const int64_t obase = DIR == HPEZ_DECOMPRESS ? A.esc_off[e] : 0;
    uint32_t nesc = 0;
    int j[kMaxRank];
    decode_pos(cmS, rank, p0 + lane, j);
    const bool inc = cn[rank - 1] >= 32;
    for (uint32_t pb = p0; pb < pend; pb += 32) {
        const uint32_t p = pb + lane;
        const bool valid = p < pend;
        int coord[kMaxRank];
        int64_t idx = 0;
        uint32_t jodd = 0;
#pragma unroll
        for (int a = 0; a < kMaxRank; a++) {
            coord[a] = st[a] + j[a] * sp[a];
            if (a < rank) {
                idx += coord[a] * estr[a];
                jodd |= (uint32_t)(j[a] & 1) << a;
            }
        }
        bool member = valid;
        PredReg pr = upred;
        if (mixed && valid) pr = load_pred(*mixed_member(A, cmS, coord, jodd, &member));
        const uint32_t mb = __ballot_sync(0xffffffffu, member);
        const int64_t ci = cbase + __popc(mb & ((1u << lane) - 1u));
        bool esc = false;
        if (member) {
            if (DIR == HPEZ_COMPRESS) {
                const double pred = predict(work, idx, coord, dims, estr, pr, s);
                const double orig = ldv((const T *)A.orig, idx);
                double out;
                const int64_t code = quantize_point<ROUND>(orig, pred, bound, two_e, inv_two_e, R, &out);
                __stcg(codes + ci, (C)code);
                esc = code == 0;
                if (!esc || A.orig != A.work) __stcg(work + idx, (T)out);
                if (STATS) {
                    const double err = fabs(__dsub_rn(orig, pred));
                    A.errbuf[ci] = err;
                    if (A.dense) A.dense[(int64_t)cmS.level * A.g.npts + idx] = err;
                }
            } else {
                const int64_t code = (int64_t)codes[ci];
                const double pred = predict(work, idx, coord, dims, estr, pr, s);  // loads overlap the code load
                if (code != 0) __stcg(work + idx, (T)dequantize_point<ROUND>(pred, code, two_e, R));
                else esc = true;
            }
        }
        const uint32_t eb = __ballot_sync(0xffffffffu, esc);
        if (DIR == HPEZ_DECOMPRESS && esc) {
            const int64_t o = obase + nesc + __popc(eb & ((1u << lane) - 1u));
            if (o < A.outl_cap) __stcg(work + idx, (T)A.outl[o]);
            else atomicExch(A.flags, HPEZ_OUTLIER_UNDERFLOW);
        }
        nesc += __popc(eb);
        cbase += __popc(mb);
        // advance the lattice indices by 32 positions
        if (inc) {
            const int x = rank - 1;
            int jx = pick(j, x) + 32;
            bool carry = jx >= pick(cn, x);
            if (carry) jx -= pick(cn, x);
#pragma unroll
            for (int a = kMaxRank - 1; a >= 0; a--) {
                if (a == x) j[a] = jx;
                else if (a < x && carry) {
                    j[a] += 1;
                    carry = j[a] >= cn[a];
                    if (carry) j[a] = 0;
                }
            }
        } else {
            decode_pos(cmS, rank, p + 32, j);
        }
    }
    if (DIR == HPEZ_COMPRESS && lane == 0) A.esc_cnt[e] = nesc;
}

// ------------------------------------------------- rank-3 fast paths --
// Uniform commits of 3-D grids (every benchmark configuration) run through
// one specialisation per (predictor layout, stencil family): KIND 0..2 = 1-D
// along axis 0/1/2, 3..5 = MD blend over axes (0,1) (0,2) (1,2), 6 = MD over
// (0,1,2).  Geometry is held in registers and lattice indices advance
// incrementally, so the per-point cost is the stencil, the quantizer and a
// few integer operations.
// grid axis of blend term t for a fast-path layout KIND
template <int KIND> __device__ constexpr int kind_axis(int t) {
    return KIND < 3 ? KIND : KIND == 3 ? (t == 0 ? 0 : 1) : KIND == 4 ? (t == 0 ? 0 : 2) : KIND == 5 ? (t == 0 ? 1 : 2) : t;
}

template <typename T, typename C, int DIR, int ROUND, int KIND, int FAM>
__device__ __forceinline__ void process_fast(const SweepArgs &A, const CommitDev &cm, int item, int warp) {
    const int lane = threadIdx.x & 31;
    const uint32_t p0 = (uint32_t)(item - cm.item_base) * (uint32_t)cm.p_item + (uint32_t)warp * (uint32_t)cm.pw;
    const uint32_t pend = min(p0 + (uint32_t)cm.pw, cm.npos);
    const int e = item * kItemWarps + warp;
    if (p0 >= pend) {
        if (DIR == HPEZ_COMPRESS && lane == 0) A.esc_cnt[e] = 0;
        return;
    }
    const int st0 = cm.start[0], st1 = cm.start[1], st2 = cm.start[2];
    const int sp0 = cm.step[0], sp1 = cm.step[1], sp2 = cm.step[2];
    const int cn1 = cm.cnt[1], cn2 = cm.cnt[2];
    const int D0 = A.g.dims[0], D1 = A.g.dims[1], D2 = A.g.dims[2];
    const int E0 = A.g.estr[0], E1 = A.g.estr[1];
    const int s = cm.s;
    const int sE0 = s * E0, sE1 = s * E1, sE2 = s;
    const double bound = cm.bound, two_e = cm.two_e, inv_two_e = cm.inv_two_e;
    const double w0 = cm.pred.w[0], w1 = cm.pred.w[1], w2 = cm.pred.w[2];
    const int64_t R = A.g.radius;
    const int32_t R32 = (int32_t)R;
    const double Rd = (double)R;
    T *__restrict__ work = (T *)A.work;
    const T *__restrict__ origp = (const T *)A.orig;
    const bool oop = A.orig != A.work;
    C *__restrict__ codes = (C *)A.codes;
    const int64_t cb = cm.code_base;
    C *__restrict__ cptr = codes + cb + p0 + lane;  // this lane's code slot, +32 per iteration
    const int64_t obase = DIR == HPEZ_DECOMPRESS ? A.esc_off[e] : 0;
    uint32_t nesc = 0;
    uint32_t p = p0 + lane;
    uint32_t r = fdiv(p, cm.fd[2]);
    int jx = (int)(p - r * (uint32_t)cn2);
    uint32_t q = fdiv(r, cm.fd[1]);
    int jy = (int)(r - q * (uint32_t)cn1);
    int jz = (int)q;
    constexpr int NAX = KIND < 3 ? 1 : KIND < 6 ? 2 : 3;
    const int Dv[3] = {D0, D1, D2};
    const int sEv[3] = {sE0, sE1, sE2};
    auto advance = [&](int &ax, int &ay, int &az) {
        ax += 32;
        while (ax >= cn2) {
            ax -= cn2;
            if (++ay >= cn1) {
                ay = 0;
                az++;
            }
        }
    };
    auto interior_at = [&](const int (&crd)[3]) {
        bool in = true;
#pragma unroll
        for (int t = 0; t < NAX; t++) in &= Fam<FAM>::interior(crd[kind_axis<KIND>(t)], Dv[kind_axis<KIND>(t)], s);
        return in;
    };
    auto blend = [&](const double (&pt)[NAX]) {
        if (NAX == 1) return pt[0];
        if (NAX == 2) return DA(DM(w0, pt[0]), DM(w1, pt[NAX - 1]));
        return DA(DA(DM(w0, pt[0]), DM(w1, pt[1])), DM(w2, pt[NAX - 1]));
    };
    uint32_t pb = p0;
#if HPEZ_ILP2
    // two full interior iterations per step: both iterations' stencil (and
    // original / code) loads are issued before either is consumed, halving
    // the exposed memory latency per point
    for (; pb + 64 <= pend; pb += 64) {
        int bx = jx, by = jy, bz = jz;
        advance(bx, by, bz);
        const int cA[3] = {st0 + jz * sp0, st1 + jy * sp1, st2 + jx * sp2};
        const int cB[3] = {st0 + bz * sp0, st1 + by * sp1, st2 + bx * sp2};
        if (!__all_sync(0xffffffffu, interior_at(cA) && interior_at(cB))) break;
        const int iA = cA[0] * E0 + cA[1] * E1 + cA[2], iB = cB[0] * E0 + cB[1] * E1 + cB[2];
        T vA[NAX][6], vB[NAX][6];
        T oA = T(0), oB = T(0);
        int64_t kA = 0, kB = 0;
        if (DIR == HPEZ_DECOMPRESS) {
            kA = (int64_t)cptr[0];
            kB = (int64_t)cptr[32];
        } else {
            oA = origp[iA];
            oB = origp[iB];
        }
#pragma unroll
        for (int t = 0; t < NAX; t++) {
            const int a = kind_axis<KIND>(t);
#pragma unroll
            for (int i = 0; i < Fam<FAM>::n; i++) {
                vA[t][i] = work[iA + Fam<FAM>::u(i) * sEv[a]];
                vB[t][i] = work[iB + Fam<FAM>::u(i) * sEv[a]];
            }
        }
        double ptA[NAX], ptB[NAX];
#pragma unroll
        for (int t = 0; t < NAX; t++) {
            ptA[t] = Fam<FAM>::combine(vA[t]);
            ptB[t] = Fam<FAM>::combine(vB[t]);
        }
        const double predA = blend(ptA), predB = blend(ptB);
        bool eA = false, eB = false;
        if (DIR == HPEZ_COMPRESS) {
            double out;
            int32_t c = quantize_point<ROUND>((double)oA, predA, bound, two_e, inv_two_e, Rd, R32, &out);
            cptr[0] = (C)c;
            eA = c == 0;
            if (!eA || oop) work[iA] = (T)out;
            c = quantize_point<ROUND>((double)oB, predB, bound, two_e, inv_two_e, Rd, R32, &out);
            cptr[32] = (C)c;
            eB = c == 0;
            if (!eB || oop) work[iB] = (T)out;
        } else {
            eA = kA == 0;
            eB = kB == 0;
            if (!eA) work[iA] = (T)dequantize_point<ROUND>(predA, kA, two_e, R);
            if (!eB) work[iB] = (T)dequantize_point<ROUND>(predB, kB, two_e, R);
        }
        const uint32_t ebA = __ballot_sync(0xffffffffu, eA);
        const uint32_t ebB = __ballot_sync(0xffffffffu, eB);
        if (DIR == HPEZ_DECOMPRESS && (ebA | ebB)) {
            const int64_t oa = obase + nesc + __popc(ebA & ((1u << lane) - 1u));
            const int64_t ob = obase + nesc + __popc(ebA) + __popc(ebB & ((1u << lane) - 1u));
            if (eA) {
                if (oa < A.outl_cap) __stcg(work + iA, (T)A.outl[oa]);
                else atomicExch(A.flags, HPEZ_OUTLIER_UNDERFLOW);
            }
            if (eB) {
                if (ob < A.outl_cap) __stcg(work + iB, (T)A.outl[ob]);
                else atomicExch(A.flags, HPEZ_OUTLIER_UNDERFLOW);
            }
        }
        nesc += __popc(ebA) + __popc(ebB);
        cptr += 64;
        jx = bx;
        jy = by;
        jz = bz;
        advance(jx, jy, jz);
    }
#endif
    for (; pb < pend; pb += 32) {
        const bool valid = pb + lane < pend;
        const int z = st0 + jz * sp0, y = st1 + jy * sp1, x = st2 + jx * sp2;
        const int idx = z * E0 + y * E1 + x;
        bool esc = false;
        const int crd[3] = {z, y, x};
        const bool in_all = interior_at(crd);
        // warp-uniform split: a warp with any edge lane loads every lane's
        // stencil with in-grid (clamped) addresses, so it still costs a single
        // memory round trip; only the row arithmetic differs per lane
        const bool warp_interior = __all_sync(0xffffffffu, in_all || !valid);
        if (valid) {
            double pred;
            double origv = 0.0;
            int64_t code = 0;
            // one memory round trip: every stencil value plus the original
            // (compress) or the code (decompress) is requested up front
            T v[NAX][6];
            T o = T(0);
            if (DIR == HPEZ_DECOMPRESS) code = (int64_t)*cptr;
            else o = origp[idx];
            double pt[NAX];
            if (warp_interior) {
#pragma unroll
                for (int t = 0; t < NAX; t++) {
                    const int a = kind_axis<KIND>(t);
#pragma unroll
                    for (int i = 0; i < Fam<FAM>::n; i++) v[t][i] = work[idx + Fam<FAM>::u(i) * sEv[a]];
                }
#pragma unroll
                for (int t = 0; t < NAX; t++) pt[t] = Fam<FAM>::combine(v[t]);
            } else {
#pragma unroll
                for (int t = 0; t < NAX; t++) {
                    const int a = kind_axis<KIND>(t);
#pragma unroll
                    for (int i = 0; i < Fam<FAM>::n; i++) {
                        const int u = Fam<FAM>::u(i);
                        const int cc = crd[a] + u * s;
                        const bool ok = u < 0 ? cc >= 0 : cc <= Dv[a] - 1;
                        v[t][i] = work[ok ? idx + u * sEv[a] : idx];
                    }
                }
#pragma unroll
                for (int t = 0; t < NAX; t++) {
                    const int a = kind_axis<KIND>(t);
                    double xv[6];
#pragma unroll
                    for (int i = 0; i < 6; i++) xv[i] = i < Fam<FAM>::n ? (double)v[t][i] : 0.0;
                    pt[t] = in_all ? Fam<FAM>::combine(v[t]) : edge_row<FAM>(xv, crd[a], Dv[a], s);
                }
            }
            pred = blend(pt);
            origv = (double)o;
            if (DIR == HPEZ_COMPRESS) {
                double out;
                const int32_t c = quantize_point<ROUND>(origv, pred, bound, two_e, inv_two_e, Rd, R32, &out);
                *cptr = (C)c;
                esc = c == 0;
                if (!esc || oop) work[idx] = (T)out;
            } else if (code != 0) {
                work[idx] = (T)dequantize_point<ROUND>(pred, code, two_e, R);
            } else {
                esc = true;
            }
        }
        const uint32_t eb = __ballot_sync(0xffffffffu, esc);
        if (DIR == HPEZ_DECOMPRESS && esc) {
            const int64_t o = obase + nesc + __popc(eb & ((1u << lane) - 1u));
            if (o < A.outl_cap) __stcg(work + idx, (T)A.outl[o]);
            else atomicExch(A.flags, HPEZ_OUTLIER_UNDERFLOW);
        }
        nesc += __popc(eb);
        cptr += 32;
        advance(jx, jy, jz);
        if (HPEZ_L1_PREFETCH && pb + 32 + lane < pend) {
            // L1 prefetch of the next iteration's stencil lines (clamped in-grid)
            const int nz = st0 + jz * sp0, ny = st1 + jy * sp1, nx = st2 + jx * sp2;
            const int nidx = nz * E0 + ny * E1 + nx;
            const int last = D0 * E0 - 1;
#pragma unroll
            for (int t = 0; t < NAX; t++) {
                const int a = kind_axis<KIND>(t);
#pragma unroll
                for (int i = 0; i < Fam<FAM>::n; i++) {
                    int q = nidx + Fam<FAM>::u(i) * sEv[a];
                    q = q < 0 ? 0 : (q > last ? last : q);
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(work + q));
                }
            }
            if (DIR == HPEZ_COMPRESS) asm volatile("prefetch.global.L1 [%0];" ::"l"(work + nidx));
            else asm volatile("prefetch.global.L1 [%0];" ::"l"(cptr));
        }
    }
    if (DIR == HPEZ_COMPRESS && lane == 0) A.esc_cnt[e] = nesc;
}

// fast_id = KIND * 5 + FAM (MD kinds use inter families 0..2 only)
template <typename T, typename C, int DIR, int ROUND>
__device__ __forceinline__ void process_dispatch(const SweepArgs &A, const CommitDev &cm, int item, int warp) {
#define HPEZ_FAST(K, F)                                                  \
    case K * 5 + F:                                                      \
        process_fast<T, C, DIR, ROUND, K, F>(A, cm, item, warp);         \
        return;
    switch (cm.fast_id) {
        HPEZ_FAST(0, 0) HPEZ_FAST(0, 1) HPEZ_FAST(0, 2) HPEZ_FAST(0, 3) HPEZ_FAST(0, 4)
        HPEZ_FAST(1, 0) HPEZ_FAST(1, 1) HPEZ_FAST(1, 2) HPEZ_FAST(1, 3) HPEZ_FAST(1, 4)
        HPEZ_FAST(2, 0) HPEZ_FAST(2, 1) HPEZ_FAST(2, 2) HPEZ_FAST(2, 3) HPEZ_FAST(2, 4)
        HPEZ_FAST(3, 0) HPEZ_FAST(3, 1) HPEZ_FAST(3, 2)
        HPEZ_FAST(4, 0) HPEZ_FAST(4, 1) HPEZ_FAST(4, 2)
        HPEZ_FAST(5, 0) HPEZ_FAST(5, 1) HPEZ_FAST(5, 2)
        HPEZ_FAST(6, 0) HPEZ_FAST(6, 1) HPEZ_FAST(6, 2)
    default:
        break;
    }
#undef HPEZ_FAST
}

// ------------------------------------------- mixed commits, fast path --
// One point's prediction for a rank-3 layout KIND and family FAM: every
// stencil value is loaded with an in-grid (clamped) address in one round
// trip; edge lanes take the truncated row (kernels.resolve_row).
struct Pt3 {  // one point of a rank-3 grid: coordinates, extents, element steps of stride s
    int crd[3], Dv[3], sEv[3];
};

template <typename T, int KIND, int FAM>
__device__ __forceinline__ double pred_point(const T *__restrict__ work, int idx, const Pt3 &P, int s, double w0,
                                             double w1, double w2) {
    constexpr int NAX = KIND < 3 ? 1 : KIND < 6 ? 2 : 3;
    const int(&crd)[3] = P.crd;
    const int(&Dv)[3] = P.Dv;
    const int(&sEv)[3] = P.sEv;
    T v[NAX][6];
#pragma unroll
    for (int t = 0; t < NAX; t++) {
        const int a = kind_axis<KIND>(t);
#pragma unroll
        for (int i = 0; i < Fam<FAM>::n; i++) {
            const int u = Fam<FAM>::u(i);
            const int cc = crd[a] + u * s;
            const bool ok = u < 0 ? cc >= 0 : cc <= Dv[a] - 1;
            v[t][i] = work[ok ? idx + u * sEv[a] : idx];
        }
    }
    double pt[NAX];
#pragma unroll
    for (int t = 0; t < NAX; t++) {
        const int a = kind_axis<KIND>(t);
        if (Fam<FAM>::interior(crd[a], Dv[a], s)) {
            pt[t] = Fam<FAM>::combine(v[t]);
        } else {
            double xv[6];
#pragma unroll
            for (int i = 0; i < 6; i++) xv[i] = i < Fam<FAM>::n ? (double)v[t][i] : 0.0;
            pt[t] = edge_row<FAM>(xv, crd[a], Dv[a], s);
        }
    }
    if (NAX == 1) return pt[0];
    if (NAX == 2) return DA(DM(w0, pt[0]), DM(w1, pt[NAX - 1]));
    return DA(DA(DM(w0, pt[0]), DM(w1, pt[1])), DM(w2, pt[NAX - 1]));
}

template <typename T>
__device__ __forceinline__ double mixed_pred(int fid, const T *__restrict__ work, int idx, const Pt3 &P, int s,
                                             double w0, double w1, double w2) {
#define HPEZ_MP(K, F) \
    case K * 5 + F:   \
        return pred_point<T, K, F>(work, idx, P, s, w0, w1, w2);
    switch (fid) {
        HPEZ_MP(0, 0) HPEZ_MP(0, 1) HPEZ_MP(0, 2) HPEZ_MP(0, 3) HPEZ_MP(0, 4)
        HPEZ_MP(1, 0) HPEZ_MP(1, 1) HPEZ_MP(1, 2) HPEZ_MP(1, 3) HPEZ_MP(1, 4)
        HPEZ_MP(2, 0) HPEZ_MP(2, 1) HPEZ_MP(2, 2) HPEZ_MP(2, 3) HPEZ_MP(2, 4)
        HPEZ_MP(3, 0) HPEZ_MP(3, 1) HPEZ_MP(3, 2)
        HPEZ_MP(4, 0) HPEZ_MP(4, 1) HPEZ_MP(4, 2)
        HPEZ_MP(5, 0) HPEZ_MP(5, 1) HPEZ_MP(5, 2)
        HPEZ_MP(6, 0) HPEZ_MP(6, 1) HPEZ_MP(6, 2)
    default:
        return 0.0;  // unreachable: the planner only emits the ids above
    }
#undef HPEZ_MP
}

// Mixed commit (interp.py:350-411) of a rank-3 grid: per point, the block
// tag (power-of-two block size: shifts) selects a precomputed descriptor
// held with the commit in shared memory -- membership rule (split axis)
// and specialised predictor -- so the dependent chain before the stencil
// loads is one table byte.  Lanes of one warp that disagree on the
// predictor take their switch cases one after the other.
template <typename T, typename C, int DIR, int ROUND>
__device__ __forceinline__ void process_mixed(const SweepArgs &A, const CommitDev &cm, int item, int warp) {
    const int lane = threadIdx.x & 31;
    const uint32_t p0 = (uint32_t)(item - cm.item_base) * (uint32_t)cm.p_item + (uint32_t)warp * (uint32_t)cm.pw;
    const uint32_t pend = min(p0 + (uint32_t)cm.pw, cm.npos);
    const int e = item * kItemWarps + warp;
    if (p0 >= pend) {
        if (DIR == HPEZ_COMPRESS && lane == 0) A.esc_cnt[e] = 0;
        return;
    }
    const int st0 = cm.start[0], st1 = cm.start[1], st2 = cm.start[2];
    const int sp0 = cm.step[0], sp1 = cm.step[1], sp2 = cm.step[2];
    const int cn1 = cm.cnt[1], cn2 = cm.cnt[2];
    const int E0 = A.g.estr[0], E1 = A.g.estr[1];
    const int s = cm.s;
    Pt3 P;
    P.Dv[0] = A.g.dims[0];
    P.Dv[1] = A.g.dims[1];
    P.Dv[2] = A.g.dims[2];
    P.sEv[0] = s * E0;
    P.sEv[1] = s * E1;
    P.sEv[2] = s;
    const double bound = cm.bound, two_e = cm.two_e, inv_two_e = cm.inv_two_e;
    const double w0 = cm.pred.w[0], w1 = cm.pred.w[1], w2 = cm.pred.w[2];
    const int64_t R = A.g.radius;
    const int32_t R32 = (int32_t)R;
    const double Rd = (double)R;
    const bool isA = cm.kind == COMMIT_MIXED_A;
    const uint32_t present = cm.axes_present;
    const int phase = cm.phase;
    const int bsh = A.g.bs_log2, bs0 = A.g.bstr[0], bs1 = A.g.bstr[1];
    const uint8_t *__restrict__ tl = A.table + (int64_t)cm.level * A.g.nblk;
    T *__restrict__ work = (T *)A.work;
    const T *__restrict__ origp = (const T *)A.orig;
    const bool oop = A.orig != A.work;
    C *__restrict__ codes = (C *)A.codes;
    int64_t cbase = A.wbase[e];
    if (A.wn[e] == 0) {  // no member in this warp's range (typical of B commits)
        if (DIR == HPEZ_COMPRESS && lane == 0) A.esc_cnt[e] = 0;
        return;
    }
    const int64_t obase = DIR == HPEZ_DECOMPRESS ? A.esc_off[e] : 0;
    uint32_t nesc = 0;
    uint32_t p = p0 + lane;
    uint32_t r = fdiv(p, cm.fd[2]);
    int jx = (int)(p - r * (uint32_t)cn2);
    uint32_t q = fdiv(r, cm.fd[1]);
    int jy = (int)(r - q * (uint32_t)cn1);
    int jz = (int)q;
    auto tag_at = [&](int x, int y, int z, bool ok) {
        return ok ? (int)__ldg(tl + (z >> bsh) * bs0 + (y >> bsh) * bs1 + (x >> bsh)) : 0;
    };
    // the next iteration's tag is loaded one iteration ahead
    int tag_next = tag_at(st2 + jx * sp2, st1 + jy * sp1, st0 + jz * sp0, p0 + lane < pend);
    for (uint32_t pb = p0; pb < pend; pb += 32) {
        const bool valid = pb + lane < pend;
        P.crd[0] = st0 + jz * sp0;
        P.crd[1] = st1 + jy * sp1;
        P.crd[2] = st2 + jx * sp2;
        const int idx = P.crd[0] * E0 + P.crd[1] * E1 + P.crd[2];
        const int tag = tag_next;
        const uint32_t jodd = (uint32_t)(jz & 1) | (uint32_t)(jy & 1) << 1 | (uint32_t)(jx & 1) << 2;
        jx += 32;
        while (jx >= cn2) {
            jx -= cn2;
            if (++jy >= cn1) {
                jy = 0;
                jz++;
            }
        }
        tag_next = tag_at(st2 + jx * sp2, st1 + jy * sp1, st0 + jz * sp0, pb + 32 + lane < pend);
        bool member = false;
        int fid = 0;
        if (valid) {
            const int desc = cm.tdesc[tag & 63];
            const int sp = (desc >> 6) - 1;
            if (isA) member = sp < 0 || !((jodd >> sp) & 1u);
            else member = sp >= 0 && ((jodd >> sp) & 1u) && __popc(present & jodd & ~(1u << sp)) == phase;
            fid = desc & 63;
        }
        const uint32_t mb = __ballot_sync(0xffffffffu, member);
        const int64_t ci = cbase + __popc(mb & ((1u << lane) - 1u));
        bool esc = false;
        if (member) {
            if (DIR == HPEZ_COMPRESS) {
                const T o = origp[idx];
                const double pred = mixed_pred<T>(fid, work, idx, P, s, w0, w1, w2);
                double out;
                const int32_t c = quantize_point<ROUND>((double)o, pred, bound, two_e, inv_two_e, Rd, R32, &out);
                codes[ci] = (C)c;
                esc = c == 0;
                if (!esc || oop) work[idx] = (T)out;
            } else {
                // the stencil loads do not wait for the code load (an escape's
                // prediction is simply discarded)
                const int64_t code = (int64_t)codes[ci];
                const double pred = mixed_pred<T>(fid, work, idx, P, s, w0, w1, w2);
                if (code != 0) work[idx] = (T)dequantize_point<ROUND>(pred, code, two_e, R);
                else esc = true;
            }
        }
        const uint32_t eb = __ballot_sync(0xffffffffu, esc);
        if (DIR == HPEZ_DECOMPRESS && esc) {
            const int64_t o = obase + nesc + __popc(eb & ((1u << lane) - 1u));
            if (o < A.outl_cap) __stcg(work + idx, (T)A.outl[o]);
            else atomicExch(A.flags, HPEZ_OUTLIER_UNDERFLOW);
        }
        nesc += __popc(eb);
        cbase += __popc(mb);
    }
    if (DIR == HPEZ_COMPRESS && lane == 0) A.esc_cnt[e] = nesc;
}

// Fast kernels: uniform commits through their specialisation, mixed
// commits through process_mixed.
template <typename T, typename C, int DIR, int ROUND>
__device__ __forceinline__ void process_any_fast(const SweepArgs &A, const CommitDev &cm, int item, int warp) {
    if (cm.fast_id >= 0) process_dispatch<T, C, DIR, ROUND>(A, cm, item, warp);
    else process_mixed<T, C, DIR, ROUND>(A, cm, item, warp);
}

// Leading small levels on one thread-block cluster (up to 16 CTAs x 1024
// threads, one per SM).  Every coarse commit descriptor sits in shared
// memory; the commits of one (level, DAG depth) group are independent, so
// their (item, warp) units are spread over all warps of the cluster, and
// groups are separated by a cluster barrier.  Its release/acquire form
// orders the grid writes at GPU scope and invalidates L1 on the wait side,
// so the plain L1-cached stencil loads of the next group see them.
constexpr int kCoarseThreads = 1024;

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <typename T, typename C, int DIR, int ROUND, bool STATS, bool FAST>
__global__ void __launch_bounds__(kCoarseThreads, 1) coarse_kernel(const __grid_constant__ SweepArgs A) {
    extern __shared__ __align__(16) unsigned char s_raw[];
    CommitDev *s_cm = reinterpret_cast<CommitDev *>(s_raw);
    const int n_words = A.n_coarse_commits * (int)(sizeof(CommitDev) / 4);
    for (int i = threadIdx.x; i < n_words; i += blockDim.x)
        ((uint32_t *)s_cm)[i] = ((const uint32_t *)A.commits)[i];
    __syncthreads();
    const int nwarps = (int)(gridDim.x * blockDim.x) >> 5;
    // units are dealt round-robin over the CTAs: coarse stencil loads are
    // uncoalesced (one line per lane), so the per-SM L1 request rate, not
    // latency, bounds a group when its warps crowd onto a few SMs
    const int gw = (int)((threadIdx.x >> 5) * gridDim.x + blockIdx.x);
    for (int g = 0; g < A.n_groups; g++) {
        const int t0 = A.coarse_groups[2 * g], t1 = A.coarse_groups[2 * g + 1];
        for (int u = gw; u < (t1 - t0) * kItemWarps; u += nwarps) {
            const int t = t0 + u / kItemWarps;
            const int c = A.coarse_pairs[2 * t], item = A.coarse_pairs[2 * t + 1];
            if (FAST) process_any_fast<T, C, DIR, ROUND>(A, s_cm[c], item, u % kItemWarps);
            else process_warp<T, C, DIR, ROUND, STATS>(A, s_cm[c], item, u % kItemWarps);
        }
        cluster_sync_all();
    }
}

// TMA bulk prefetch into L2 of everything an item reads that no earlier
// commit writes: its own originals (compress: one request per lattice row
// segment) or its code range (decompress).  Issued by one warp, one item
// ahead, so the DRAM latency overlaps the dependency wait and current work.
__device__ __forceinline__ void bulk_prefetch_l2(const void *p, uint64_t bytes) {
    uint64_t a = (uint64_t)p & ~(uint64_t)15;
    uint64_t e = ((uint64_t)p + bytes + 15) & ~(uint64_t)15;
    while (a < e) {
        const uint32_t n = (uint32_t)(e - a < (1ull << 20) ? e - a : (1ull << 20));
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(n) : "memory");
        a += n;
    }
}

template <typename T, typename C, int DIR>
__device__ __forceinline__ void prefetch_item(const SweepArgs &A, int item, int lane) {
    const CommitDev &cm = A.commits[A.item_commit[item]];
    const int rank = A.g.rank;
    const uint32_t P0 = (uint32_t)(item - cm.item_base) * (uint32_t)cm.p_item;
    const uint32_t P1 = min(P0 + (uint32_t)cm.p_item, cm.npos);
    if (DIR == HPEZ_DECOMPRESS) {
        if (lane == 0 && cm.kind == COMMIT_UNIFORM)
            bulk_prefetch_l2((const C *)A.codes + cm.code_base + P0, (uint64_t)(P1 - P0) * sizeof(C));
        return;
    }
    const int x = rank - 1;
    const uint32_t cx = (uint32_t)cm.cnt[x];
    const uint32_t r0 = P0 / cx, r1 = (P1 - 1) / cx;
    for (uint32_t r = r0 + lane; r <= r1; r += 32) {
        uint32_t q = r;
        int64_t base = 0;
        for (int a = x - 1; a >= 0; a--) {
            const uint32_t qq = a > 0 ? q / (uint32_t)cm.cnt[a] : 0u;
            const int ja = (int)(q - qq * (uint32_t)cm.cnt[a]);
            q = qq;
            base += (int64_t)(cm.start[a] + ja * cm.step[a]) * A.g.estr[a];
        }
        const uint32_t xa = r == r0 ? P0 - r * cx : 0u;
        const uint32_t xb = r == r1 ? P1 - 1 - r * cx : cx - 1;
        const int64_t lo = base + cm.start[x] + (int64_t)xa * cm.step[x];
        const int64_t hi = base + cm.start[x] + (int64_t)xb * cm.step[x];
        bulk_prefetch_l2((const T *)A.work + lo, (uint64_t)(hi - lo + 1) * sizeof(T));
    }
}

// Persistent dataflow kernel over the remaining items.
template <typename T, typename C, int DIR, int ROUND, bool STATS, bool FAST>
__global__ void __launch_bounds__(kItemThreads, FAST ? HPEZ_FLOW_OCC * 8 / kItemWarps : 3) flow_kernel(const __grid_constant__ SweepArgs A) {
    __shared__ CommitDev s_cm;
    __shared__ int s_item, s_next;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int cur = -1;
    bool first = true;
    unsigned long long t_grab = 0, t_wait = 0, t_work = 0, n_done = 0;
    // items are claimed two steps ahead: the atomic issued while item k runs
    // returns during its work and becomes item k + 2.  Two CTA barriers per
    // item: B (dependencies acquired, descriptor staged) and A (item written).
    int q_cur = 0, q_next = 0;
    if (threadIdx.x == 0) {
        s_item = atomicAdd(A.next, 1);
        s_next = q_cur = atomicAdd(A.next, 1);
        q_next = atomicAdd(A.next, 1);
    }
    __syncthreads();
    while (true) {
        const long long c0 = A.prof ? clock64() : 0;
        const int rel = s_item, nrel = s_next;
        if (rel >= A.n_items) break;
        const int item = A.flow_order[rel];
        const int c = A.item_commit[item];
        if (warp == 1 && A.l2_prefetch) {
            if (first) prefetch_item<T, C, DIR>(A, item, lane);
            if (nrel < A.n_items) prefetch_item<T, C, DIR>(A, A.flow_order[nrel], lane);
        }
        first = false;
        if (c != cur) {
            if (threadIdx.x < sizeof(CommitDev) / 4)
                ((uint32_t *)&s_cm)[threadIdx.x] = ((const uint32_t *)&A.commits[c])[threadIdx.x];
            cur = c;
        }
        const long long c1 = A.prof ? clock64() : 0;
        if (warp == 0 && !(A.dbg & 1)) {
            const int k0 = A.dep_off[item], k1 = A.dep_off[item + 1];
            // every dependency flag is polled with relaxed gpu-scope loads in one
            // pass (independent loads: one L2 round trip, not one per flag);
            // then a single acquire load invalidates this SM's L1 (CCTL.IVALL)
            // so the item's plain loads see the producers' writes, and bar.sync
            // below extends the ordering to the CTA
            while (true) {
                bool ok = true;
                for (int k = k0; k < k1; k++) {
                    const int2 d = A.dep_rng[k];
                    for (int q = d.x + lane; q <= d.y; q += 32) ok &= ld_relaxed(&A.done[q]) != 0;
                }
                if (__all_sync(0xffffffffu, ok)) break;
                __nanosleep(32);
            }
            if (lane == 0 && k1 > k0) (void)ld_acquire(&A.done[A.dep_rng[k0].x]);
        }
        __syncthreads();  // B
        const long long c2 = A.prof ? clock64() : 0;
        if (FAST) process_any_fast<T, C, DIR, ROUND>(A, s_cm, item, warp);
        else process_warp<T, C, DIR, ROUND, STATS>(A, s_cm, item, warp);
        if (threadIdx.x == 0) {  // nobody reads s_item / s_next again before barrier A
            s_item = q_cur;
            s_next = q_next;
            q_cur = q_next;
            if (q_next < A.n_items) q_next = atomicAdd(A.next, 1);
        }
        __syncthreads();  // A: CTA writes happen-before the gpu-scope release
        // released from the last warp: its fence overlaps warp 0's polling of
        // the next item's dependencies instead of delaying it
        if (threadIdx.x == kItemThreads - 32) st_release(&A.done[item], 1u);  // cumulative over the CTA's writes
        if (A.prof) {
            const long long c3 = clock64();
            t_grab += c1 - c0;
            t_wait += c2 - c1;
            t_work += c3 - c2;
            n_done++;
            if (threadIdx.x == 0) {  // per-level first start / last end (globaltimer ns)
                unsigned long long now;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                const int lv = s_cm.level < 12 ? s_cm.level : 11;
                atomicMin(A.prof + 8 + 2 * lv, now - (unsigned long long)((c3 - c2) / 1.9));
                atomicMax(A.prof + 9 + 2 * lv, now);
                atomicAdd(A.prof + 40 + 4 * lv, (unsigned long long)(c1 - c0));
                atomicAdd(A.prof + 41 + 4 * lv, (unsigned long long)(c2 - c1));
                atomicAdd(A.prof + 42 + 4 * lv, (unsigned long long)(c3 - c2));
                atomicAdd(A.prof + 43 + 4 * lv, 1ull);
            }
        }
    }
    if (A.prof && threadIdx.x == 0) {
        atomicAdd(A.prof + 0, t_grab);
        atomicAdd(A.prof + 1, t_wait);
        atomicAdd(A.prof + 2, t_work);
        atomicAdd(A.prof + 3, n_done);
    }
}

// Staged levels: every (level, DAG depth) group of the finest levels is one
// plain data-parallel launch.  The commits of a group never read each other
// (the depth is the longest path of the commit DAG), and every point they
// read belongs to an earlier group or level, so launch order is the whole
// synchronisation: no flags, no CTA barriers and no L1 invalidation.  Warps
// take (item, warp) units independently, in stream order.
constexpr int kStageMax = 24;
struct StageGroup {
    int32_t n;
    int32_t c[kStageMax];
    int32_t u_off[kStageMax + 1];  // unit prefix: n_items * kItemWarps per commit
};

template <typename T, typename C, int DIR, int ROUND, bool STATS, bool FAST>
__global__ void __launch_bounds__(kItemThreads, FAST ? HPEZ_FLOW_OCC * 8 / kItemWarps : 3)
    stage_kernel(const __grid_constant__ SweepArgs A, const __grid_constant__ StageGroup G) {
    __shared__ CommitDev s_cm[kStageMax];
    constexpr int W = sizeof(CommitDev) / 4;
    for (int i = threadIdx.x; i < G.n * W; i += blockDim.x)
        ((uint32_t *)s_cm)[i] = ((const uint32_t *)&A.commits[G.c[i / W]])[i % W];
    __syncthreads();
    const int nw = (int)(gridDim.x * blockDim.x) >> 5;
    const int total = G.u_off[G.n];
    int k = 0;
    for (int u = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); u < total; u += nw) {
        while (u >= G.u_off[k + 1]) k++;  // units ascend per warp
        const CommitDev &cm = s_cm[k];
        const int local = u - G.u_off[k];
        const int item = cm.item_base + local / kItemWarps, warp = local % kItemWarps;
        if (FAST) process_any_fast<T, C, DIR, ROUND>(A, cm, item, warp);
        else process_warp<T, C, DIR, ROUND, STATS>(A, cm, item, warp);
    }
}

// Zero codes of codes[b, b+n), walked by one warp in aligned 16-byte chunks
// (a few vector loads per lane instead of n/32 dependent scalar rounds).
// emit(i, r) is called for every zero code with its offset i in the range
// and its rank r among the range's zeros (ranks follow stream order).
// Returns the number of zero codes.  The chunks may touch the bytes of the
// enclosing aligned 16-byte blocks only.
template <typename C, typename F>
__device__ __forceinline__ uint32_t warp_zeros(const C *__restrict__ codes, int64_t b, int n, F &&emit) {
    constexpr int K = 16 / (int)sizeof(C);
    const int lane = threadIdx.x & 31;
    const int64_t mis = (int64_t)(((uintptr_t)codes & 15) / sizeof(C));
    const int64_t a0 = b - ((b + mis) % K);  // codes + a0 is 16-byte aligned
    const int nch = (int)((b + n - a0 + K - 1) / K);
    uint32_t total = 0;
    for (int c0 = 0; c0 < nch; c0 += 32) {
        const int ch = c0 + lane;
        uint32_t zm = 0;
        if (ch < nch) {
            const uint4 v = __ldg(reinterpret_cast<const uint4 *>(codes + a0) + ch);
            const C *cv = reinterpret_cast<const C *>(&v);
#pragma unroll
            for (int t = 0; t < K; t++) {
                const int64_t gi = a0 + (int64_t)ch * K + t;
                if (cv[t] == 0 && gi >= b && gi < b + n) zm |= 1u << t;
            }
        }
        const uint32_t cnt = __popc(zm);
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        uint32_t r = total + incl - cnt;
        while (zm) {
            const int t = __ffs(zm) - 1;
            zm &= zm - 1;
            emit((int)(a0 + (int64_t)ch * K + t - b), r++);
        }
        total += __shfl_sync(0xffffffffu, incl, 31);
    }
    return total;
}

// Decompress pre-pass: zero codes per (item, warp).
template <typename C>
__global__ void __launch_bounds__(256) count_zero_kernel(const C *__restrict__ codes, const int64_t *__restrict__ wbase,
                                                         const int32_t *__restrict__ wn, int64_t n_entries,
                                                         uint32_t *__restrict__ cnt) {
    const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (e >= n_entries) return;
    const int64_t b = wbase[e];
    const int n = wn[e];
    uint32_t z = 0;
    for (int i = lane; i < n; i += 32) z += codes[b + i] == 0;
    for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
    if (lane == 0) cnt[e] = z;
}


// Decompress pre-pass for u16 streams as a pure streaming read: CTA b owns
// entries [b*kZeroEpb, ...) whose code ranges are contiguous in the stream,
// reads them with aligned 16-byte loads, tests eight codes at once and only
// for a chunk holding a zero code searches the entry it belongs to.
constexpr int kZeroEpb = 32;
__global__ void __launch_bounds__(256) count_zero_stream_kernel(const uint16_t *__restrict__ codes,
                                                                const int64_t *__restrict__ wbase,
                                                                const int32_t *__restrict__ wn, int64_t n_entries,
                                                                uint32_t *__restrict__ cnt) {
    __shared__ int64_t s_base[kZeroEpb + 1];
    __shared__ uint32_t s_cnt[kZeroEpb];
    const int64_t e0 = (int64_t)blockIdx.x * kZeroEpb;
    const int ne = (int)min((int64_t)kZeroEpb, n_entries - e0);
    for (int i = threadIdx.x; i < ne; i += blockDim.x) {
        s_base[i] = wbase[e0 + i];
        s_cnt[i] = 0;
    }
    if (threadIdx.x == 0) s_base[ne] = wbase[e0 + ne - 1] + wn[e0 + ne - 1];
    __syncthreads();
    const int64_t c0 = s_base[0], c1 = s_base[ne];
    const int64_t mis = (int64_t)(((uintptr_t)codes & 15) / 2);
    const int64_t a0 = c0 - ((c0 + mis) % 8);  // codes + a0 is 16-byte aligned
    const int64_t nch = (c1 - a0 + 7) / 8;
    const uint4 *src = reinterpret_cast<const uint4 *>(codes + a0);
#pragma unroll 4
    for (int64_t ch = threadIdx.x; ch < nch; ch += blockDim.x) {
        const uint4 v = __ldg(src + ch);
        const uint64_t lo = ((uint64_t)v.y << 32) | v.x, hi = ((uint64_t)v.w << 32) | v.z;
        const uint64_t k1 = 0x0001000100010001ull, k8 = 0x8000800080008000ull;
        if (!(((lo - k1) & ~lo & k8) | ((hi - k1) & ~hi & k8))) continue;  // no zero halfword
        const uint16_t *cv = reinterpret_cast<const uint16_t *>(&v);
        for (int t = 0; t < 8; t++) {
            const int64_t q = a0 + ch * 8 + t;
            if (cv[t] != 0 || q < c0 || q >= c1) continue;
            int lo_e = 0, hi_e = ne - 1;  // largest e with s_base[e] <= q
            while (lo_e < hi_e) {
                const int mid = (lo_e + hi_e + 1) >> 1;
                if (s_base[mid] <= q) lo_e = mid;
                else hi_e = mid - 1;
            }
            atomicAdd(&s_cnt[lo_e], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < ne; i += blockDim.x) cnt[e0 + i] = s_cnt[i];
}

// Compress post-pass: outliers of every (item, warp) with escapes, in stream
// order, read back from the grid (escaped points keep their originals).  One
// warp screens 32 entries and replays only those that escaped.
template <typename T, typename C>
__global__ void __launch_bounds__(256) gather_outliers_kernel(const __grid_constant__ SweepArgs A, int64_t n_entries,
                                                              double *__restrict__ out, int64_t cap) {
    const int64_t e0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32;
    const int lane = threadIdx.x & 31;
    if (e0 >= n_entries) return;
    const bool has = e0 + lane < n_entries && A.esc_cnt[e0 + lane] != 0;
    uint32_t todo = __ballot_sync(0xffffffffu, has);
    const GridDev &g = A.g;
    const T *work = (const T *)A.orig;  // escaped points hold their originals in both buffers
    const C *codes = (const C *)A.codes;
    while (todo) {
        const int k = __ffs(todo) - 1;
        todo &= todo - 1;
        const int64_t e = e0 + k;
        const int item = (int)(e / kItemWarps), warp = (int)(e % kItemWarps);
        const CommitDev &cm = A.commits[A.item_commit[item]];
        const uint32_t p0 = (uint32_t)(item - cm.item_base) * (uint32_t)cm.p_item + (uint32_t)warp * (uint32_t)cm.pw;
        const uint32_t pend = min(p0 + (uint32_t)cm.pw, cm.npos);
        int64_t cbase = A.wbase[e];
        int64_t o = A.esc_off[e];
        if (cm.kind == COMMIT_UNIFORM) {
            warp_zeros(codes, cbase, (int)(pend - p0), [&](int i, uint32_t rk) {
                int j[kMaxRank];
                decode_pos(cm, g.rank, p0 + (uint32_t)i, j);
                int64_t idx = 0;
                for (int a = 0; a < g.rank; a++) idx += (int64_t)(cm.start[a] + j[a] * cm.step[a]) * g.estr[a];
                const int64_t r = o + rk;
                if (r < cap) out[r] = (double)work[idx];
            });
            continue;
        }
        for (uint32_t pb = p0; pb < pend; pb += 32) {
            const uint32_t p = pb + lane;
            const bool valid = p < pend;
            int j[kMaxRank], coord[kMaxRank];
            decode_pos(cm, g.rank, valid ? p : p0, j);
            int64_t idx = 0;
            uint32_t jodd = 0;
            for (int a = 0; a < g.rank; a++) {
                coord[a] = cm.start[a] + j[a] * cm.step[a];
                idx += (int64_t)coord[a] * g.estr[a];
                jodd |= (uint32_t)(j[a] & 1) << a;
            }
            bool member = valid;
            if (valid) mixed_member(A, cm, coord, jodd, &member);
            const uint32_t mb = __ballot_sync(0xffffffffu, member);
            const int64_t ci = cbase + __popc(mb & ((1u << lane) - 1u));
            const bool esc = member && codes[ci] == 0;
            const uint32_t eb = __ballot_sync(0xffffffffu, esc);
            if (esc) {
                const int64_t r = o + __popc(eb & ((1u << lane) - 1u));
                if (r < cap) out[r] = (double)work[idx];
            }
            o += __popc(eb);
            cbase += __popc(mb);
        }
    }
}

// Mixed setup: member counts per (item, warp) of mixed commits.
__global__ void __launch_bounds__(256) mixed_count_kernel(const __grid_constant__ SweepArgs A, int32_t *wn_out,
                                                          int32_t n_mixed_items, const int32_t *mixed_items) {
    const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= (int64_t)n_mixed_items * kItemWarps) return;
    const int item = mixed_items[t / kItemWarps], warp = (int)(t % kItemWarps);
    const CommitDev &cm = A.commits[A.item_commit[item]];
    const GridDev &g = A.g;
    const uint32_t p0 = (uint32_t)(item - cm.item_base) * (uint32_t)cm.p_item + (uint32_t)warp * (uint32_t)cm.pw;
    const uint32_t pend = min(p0 + (uint32_t)cm.pw, cm.npos);
    int n = 0;
    for (uint32_t pb = p0; pb < pend; pb += 32) {
        const uint32_t p = pb + lane;
        bool member = false;
        if (p < pend) {
            int j[kMaxRank], coord[kMaxRank];
            decode_pos(cm, g.rank, p, j);
            uint32_t jodd = 0;
            for (int a = 0; a < g.rank; a++) {
                coord[a] = cm.start[a] + j[a] * cm.step[a];
                jodd |= (uint32_t)(j[a] & 1) << a;
            }
            mixed_member(A, cm, coord, jodd, &member);
        }
        n += __popc(__ballot_sync(0xffffffffu, member));
    }
    if (lane == 0) wn_out[(int64_t)item * kItemWarps + warp] = n;
}

// ---------------------------------------------------- stats (tuning) --
// numpy pairwise sum of each commit's member errors (numpy order), one CTA
// of 256 threads per commit (pairwise.cuh).
__global__ void __launch_bounds__(256) commit_pairwise_kernel(const double *errbuf, const int64_t *commit_code_base,
                                                              const int64_t *commit_n, double *commit_sum) {
    __shared__ double s_val[256];
    __shared__ int8_t s_leaf[256];
    const int c = blockIdx.x;
    const int64_t base = commit_code_base[c], n = commit_n[c];
    if (n == 0) {
        if (threadIdx.x == 0) commit_sum[c] = 0.0;
        return;
    }
    const double r = np_pairwise_cta<8>(errbuf + base, n, s_val, s_leaf);
    if (threadIdx.x == 0) commit_sum[c] = r;
}

__global__ void stats_accumulate_kernel(int n_commits, const int32_t *commit_level, const double *commit_sum,
                                        const int64_t *commit_n, double *err_sum, int64_t *count) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int c = 0; c < n_commits; c++) {
        if (commit_n[c] == 0) continue;  // empty commits are never recorded
        err_sum[commit_level[c]] = __dadd_rn(err_sum[commit_level[c]], commit_sum[c]);
        count[commit_level[c]] += commit_n[c];
    }
}

// Per-commit code base and member count from the (item, warp) table: one
// CTA per commit, block-wide sum of its (item, warp) member counts.
__global__ void __launch_bounds__(256) commit_ranges_kernel(const CommitDev *commits, int nc, const int64_t *wbase,
                                                            const int32_t *wn, int64_t *cbase, int64_t *cn) {
    __shared__ int64_t s_w[8];
    const int c = blockIdx.x;
    if (c >= nc) return;
    const CommitDev &cm = commits[c];
    const int64_t e0 = (int64_t)cm.item_base * kItemWarps;
    const int64_t e1 = (int64_t)(cm.item_base + cm.n_items) * kItemWarps;
    int64_t n = 0;
    for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) n += wn[e];
    for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = n;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += s_w[w];
        cbase[c] = wbase[e0];
        cn[c] = t;
    }
}

// Out-of-place compress: copy the anchor lattice (multiples of A on every
// non-frozen axis, plan.py:142-161) from the originals into work.
__global__ void copy_anchors_kernel(GridDev g, uint32_t A, uint32_t frozen, int64_t na, const char *orig, char *work,
                                    int esz) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= na) return;
    int64_t idx = 0;
    for (int a = g.rank - 1; a >= 0; a--) {
        const int64_t n = (frozen >> a & 1) ? g.dims[a] : (g.dims[a] + A - 1) / A;
        const int64_t j = i % n;
        i /= n;
        idx += ((frozen >> a & 1) ? j : j * A) * g.estr[a];
    }
    if (esz == 4) ((float *)work)[idx] = ((const float *)orig)[idx];
    else ((double *)work)[idx] = ((const double *)orig)[idx];
}

// ----------------------------------------------------------- host plan --
struct Cfg {
    int spline = 0, same = 0, md = 0;
    std::vector<int> order;
};

static const int kVarSpline[5] = {0, 1, 1, 2, 2};
static const int kVarSame[5] = {0, 0, 1, 0, 1};
static int inter_fam(int spline) { return spline == 0 ? FAM_LIN_I : (spline == 1 ? FAM_NAK_I : FAM_NAT_I); }
static int same_fam(int spline) { return spline == 1 ? FAM_NAK_S : FAM_NAT_S; }

// CPython 3.12 builtin sum() over floats (Neumaier compensation), used by
// interp._blend_weights for `total = sum(w.values())`.
static double py_sum(const std::vector<double> &x) {
    if (x.empty()) return 0.0;
    volatile double f = 0.0 + x[0], c = 0.0;
    for (size_t i = 1; i < x.size(); i++) {
        volatile double t = f + x[i];
        if (std::fabs(f) >= std::fabs(x[i])) c += (f - t) + x[i];
        else c += (x[i] - t) + f;
        f = t;
    }
    double r = f;
    if (c != 0.0 && std::isfinite((double)c)) r += c;
    return r;
}

static int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

constexpr int64_t kStageMinPts = INT64_MAX;  // levels of at least this many points run as staged launches
constexpr uint32_t kCoarseMax = 20000;  // leading levels of at most this many points (cumulative) run on the coarse cluster (cfg2: levels 0-1; measured sweep, session 2)
constexpr int kCoarseCluster = 16;
static int kDiagScale = 16;  // diagonal order: item window width, in units of the dependency reach

struct Plan {
    hpez_sweep_desc d{};
    std::vector<hpez_level> levels;
    std::vector<double> md;
    std::vector<uint8_t> table;
    std::vector<int> active;
    GridDev g{};
    int64_t nblk_table = 0;

    std::vector<CommitDev> commits;
    std::vector<TagInfo> tags;
    std::vector<uint8_t> slots;
    bool has_mixed = false;
    int64_t num_codes = 0;
    std::vector<int64_t> level_codes;
    int32_t n_items = 0;
    int32_t c_coarse = 0;      // commits [0, c_coarse) run in the coarse kernel
    int32_t coarse_cluster = kCoarseCluster;  // CTAs in the coarse cluster
    bool coarse_fast = false, flow_fast = false, diag_order = false;
    int32_t first_flow_item = 0;
    std::vector<int32_t> item_commit;
    std::vector<int32_t> dep_off;     // per item: first entry in dep_rng
    std::vector<int2> dep_rng;        // item-id intervals an item waits on
    std::vector<int32_t> flow_order;  // flow items in grab order
    std::vector<int32_t> coarse_pairs;   // coarse (commit, item) pairs, depth-grouped
    std::vector<int32_t> coarse_groups;  // boundaries into coarse_pairs (pairs of ints)
    std::vector<uint32_t> c_vmask, c_reads;
    std::vector<int32_t> wn;   // member count per (item, warp); mixed filled on device
    std::vector<int32_t> mixed_items;
    int32_t c_tile = 0;             // commits [c_tile, n) run as tiled levels (tile.cu)
    int32_t c_stage = 0;            // commits [c_stage, c_tile) run as staged launches
    std::vector<StageGroup> stages; // one launch per (level, DAG depth) group
    bool stage_fast = false;
    std::vector<TilePlan> tiles;    // one per tiled level
    std::vector<RowPlan> rows;      // row-fused fine levels (row.cu), coarse to fine; commits [c_tile, n) when non-empty
    std::vector<int> row_level;     // level index of each row plan
    void *d_orig_scratch = nullptr; // originals copy for in-place compress with tiled levels
    std::vector<int> coarse_group;  // (level, depth) group of each coarse commit
    CoarsePlan cplan;               // coarse levels in distributed shared memory (coarse.cu)
    bool coarse_dsmem = false;
    cudaStream_t side = nullptr;    // decompress: the zero-count pre-pass runs beside the coarse kernel
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;

    // device
    CommitDev *d_commits = nullptr;
    int32_t *d_item_commit = nullptr;
    int32_t *d_flow_order = nullptr, *d_dep_off = nullptr, *d_coarse_pairs = nullptr, *d_coarse_groups = nullptr;
    int2 *d_dep_rng = nullptr;
    int64_t *d_wbase = nullptr;
    int32_t *d_wn = nullptr;
    uint32_t *d_esc_cnt = nullptr;
    int64_t *d_esc_off = nullptr;
    int64_t *d_scan_tmp = nullptr;
    int64_t *d_total = nullptr;   // [0] outlier total
    uint32_t *d_done = nullptr;
    int32_t *d_counters = nullptr;  // [0] next flow item, [1] flags
    TagInfo *d_tags = nullptr;
    uint8_t *d_slots = nullptr;
    uint8_t *d_table = nullptr;
    int32_t *d_mixed_items = nullptr;
    int64_t *d_cbase = nullptr, *d_cn = nullptr;
    int32_t *d_clevel = nullptr;
    double *d_errbuf = nullptr, *d_csum = nullptr;
    unsigned long long *d_prof = nullptr;
    std::vector<int32_t> clevel;    // level of each commit (stats accumulation)
    bool profile = false;           // HPEZ_PROFILE at plan creation
    bool setup_done = false;
    int64_t outl_cap_last = 0;
    int flow_grid = 0;

    void *ws = nullptr;             // device workspace (caller-bound or own_ws)
    size_t ws_bytes = 0;
    void *own_ws = nullptr;         // allocated by the plan only when no workspace was bound

    ~Plan() {
        if (own_ws) cudaFree(own_ws);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
        if (side) cudaStreamDestroy(side);
    }

    std::vector<std::vector<int>> order_candidates() const {  // plan.py:37-51
        std::vector<std::vector<int>> out;
        std::vector<int> ax = active;
        if (ax.size() <= 3) {
            do out.push_back(ax);
            while (std::next_permutation(ax.begin(), ax.end()));
            return out;
        }
        for (size_t a = 0; a < ax.size(); a++) {
            std::vector<int> o{ax[a]};
            for (size_t b = 0; b < ax.size(); b++)
                if (b != a) o.push_back(ax[b]);
            out.push_back(o);
        }
        return out;
    }

    bool decode_tag(int tag, Cfg *c) const {  // plan.decode_tag (plan.py:77-84)
        const int k = tag % 8, p = tag / 8;
        if (k >= 5) return false;
        c->spline = kVarSpline[k];
        c->same = kVarSame[k];
        if (p == 0) {
            c->md = 1;
            c->order.clear();
            return true;
        }
        auto oc = order_candidates();
        if (p - 1 >= (int)oc.size()) return false;
        c->md = 0;
        c->order = oc[p - 1];
        return true;
    }

    static int oned_axis(const Cfg &c, const std::vector<int> &v) {  // interp.py:226-230
        int best = v[0], bpos = -1;
        for (int a : v) {
            int pos = -1;
            for (size_t j = 0; j < c.order.size(); j++)
                if (c.order[j] == a) pos = (int)j;
            if (pos > bpos) {
                bpos = pos;
                best = a;
            }
        }
        return best;
    }

    static int split_axis(const Cfg &c, const std::vector<int> &v) {  // interp.py:313-320
        if (!c.same) return -1;
        if (!c.md) return oned_axis(c, v);
        return v.size() == 1 ? v[0] : -1;
    }

    PredDev make_pred(const Cfg &c, const std::vector<int> &v, bool same_pass) const {
        PredDev p{};
        if (!c.md || v.size() == 1) {  // interp.py:300-305
            p.md = 0;
            p.axis = !c.md ? oned_axis(c, v) : v[0];
            p.fam = same_pass ? same_fam(c.spline) : inter_fam(c.spline);
            return p;
        }
        p.md = 1;  // MD blend over sorted(v) (interp.py:306-311)
        p.fam = inter_fam(c.spline);
        p.nax = (int)v.size();
        std::vector<double> w;
        for (int a : v) w.push_back(md[a] > 0.0 ? md[a] : 0.0);
        const double tot = py_sum(w);
        for (size_t i = 0; i < v.size(); i++) {
            p.axes[i] = v[i];
            p.w[i] = tot <= 0.0 ? 1.0 / (double)v.size() : w[i] / tot;
        }
        return p;
    }

    CommitDev base_commit(int li, const int64_t *start, const int64_t *step, const int64_t *count) {
        CommitDev c{};
        c.level = li;
        c.s = levels[li].stride;
        c.bound = levels[li].bound;
        c.two_e = 2.0 * levels[li].bound;
        c.inv_two_e = c.two_e > 0.0 ? 1.0 / c.two_e : 0.0;
        int64_t npos = 1;
        for (int a = 0; a < d.rank; a++) {
            c.start[a] = (int32_t)start[a];
            c.step[a] = (int32_t)step[a];
            c.cnt[a] = (int32_t)count[a];
            c.fd[a] = make_fastdiv((uint32_t)count[a]);
            npos *= count[a];
        }
        for (int a = d.rank; a < kMaxRank; a++) {
            c.cnt[a] = 1;
            c.fd[a] = make_fastdiv(1);
        }
        c.npos = (uint32_t)npos;
        c.commit_id = (int)commits.size();
        return c;
    }

    static int64_t range_len(int64_t a, int64_t b, int64_t c) { return a < b ? (b - 1 - a) / c + 1 : 0; }

    void add_uniform(int li, const Cfg &c, const std::vector<int> &v, const int64_t *start,
                     const int64_t *step, const int64_t *count, int64_t *code_pos) {
        const int64_t s = levels[li].stride;
        const int split = split_axis(c, v);
        const int nph = split < 0 ? 1 : 2;
        for (int ph = 0; ph < nph; ph++) {
            int64_t st[kMaxRank], sp[kMaxRank], cn[kMaxRank];
            int64_t tot = 1;
            for (int a = 0; a < d.rank; a++) {
                st[a] = start[a];
                sp[a] = step[a];
                cn[a] = count[a];
            }
            if (split >= 0) {
                st[split] = ph == 0 ? s : 3 * s;
                sp[split] = 4 * s;
                cn[split] = range_len(st[split], d.dims[split], 4 * s);
            }
            for (int a = 0; a < d.rank; a++) tot *= cn[a];
            if (tot == 0) continue;
            CommitDev cm = base_commit(li, st, sp, cn);
            cm.kind = COMMIT_UNIFORM;
            cm.pred = make_pred(c, v, split >= 0 && ph == 1);
            cm.code_base = *code_pos;
            *code_pos += tot;
            commits.push_back(cm);
            uint32_t vm = 0;
            for (int a : v) vm |= 1u << a;
            c_vmask.push_back(vm);
            c_reads.push_back(cm.pred.md ? vm : (1u << cm.pred.axis));
        }
    }

    int build() {
        if (d.rank < 1 || d.rank > kMaxRank) return HPEZ_BAD_ARGUMENT;
        if (d.direction != HPEZ_COMPRESS && d.direction != HPEZ_DECOMPRESS) return HPEZ_BAD_ARGUMENT;
        if (d.radius < 1 || d.radius > (1ll << 30)) return HPEZ_BAD_ARGUMENT;
        if (d.code_dtype == HPEZ_CODES_U16 && d.radius > 32768) return HPEZ_BAD_ARGUMENT;
        g.rank = d.rank;
        g.radius = d.radius;
        int64_t n = 1;
        for (int a = d.rank - 1; a >= 0; a--) {
            if (d.dims[a] < 1) return HPEZ_BAD_ARGUMENT;
            g.dims[a] = (int32_t)d.dims[a];
            g.estr[a] = (int32_t)n;
            n *= d.dims[a];
            if (n >= (1ll << 31)) return HPEZ_BAD_ARGUMENT;  // per-field limit of this build
        }
        g.npts = n;
        for (int a = 0; a < d.rank; a++)
            if (!(d.frozen_mask >> a & 1)) active.push_back(a);
        md.assign(d.rank, 1.0);  // interp.py:457-458
        if (d.md_alpha)
            for (int a = 0; a < d.rank; a++) md[a] = d.md_alpha[a];
        const bool use_tbl = d.block_table && d.block_size > 0;
        g.block_size = use_tbl ? d.block_size : 1;
        if (use_tbl) {
            int64_t nb = 1;
            for (int a = d.rank - 1; a >= 0; a--) {
                g.bstr[a] = (int32_t)nb;
                nb *= (d.dims[a] + d.block_size - 1) / d.block_size;
            }
            nblk_table = nb;
            g.nblk = nb;
            g.bs_log2 = -1;
            for (int k = 0; k < 31; k++)
                if ((int64_t)1 << k == d.block_size) g.bs_log2 = k;
            table.assign(d.block_table, d.block_table + (size_t)nb * d.n_levels);
        }
        int64_t code_pos = 0;
        level_codes.assign(1, 0);
        for (int li = 0; li < d.n_levels; li++) {
            const hpez_level &lv = levels[li];
            if (lv.kernel < 0 || lv.kernel >= 5 || lv.stride < 1) return HPEZ_BAD_ARGUMENT;
            Cfg lc;
            lc.spline = kVarSpline[lv.kernel];
            lc.same = kVarSame[lv.kernel];
            lc.md = lv.paradigm == 1;
            lc.order.assign(lv.axis_order, lv.axis_order + lv.n_order);
            const int64_t s = lv.stride;
            const int na = (int)active.size();
            for (int m = 1; m <= na; m++) {
                std::vector<int> ci(m);
                for (int i = 0; i < m; i++) ci[i] = i;
                while (true) {
                    std::vector<int> v;
                    uint32_t vmask = 0;
                    for (int i = 0; i < m; i++) {
                        v.push_back(active[ci[i]]);
                        vmask |= 1u << active[ci[i]];
                    }
                    int64_t start[kMaxRank], step[kMaxRank], count[kMaxRank], tot = 1;
                    for (int a = 0; a < d.rank; a++) {  // interp._class_descriptor
                        if (d.frozen_mask >> a & 1) {
                            start[a] = 0;
                            step[a] = 1;
                        } else if (vmask >> a & 1) {
                            start[a] = s;
                            step[a] = 2 * s;
                        } else {
                            start[a] = 0;
                            step[a] = 2 * s;
                        }
                        count[a] = range_len(start[a], d.dims[a], step[a]);
                        tot *= count[a];
                    }
                    if (tot > 0) {
                        int st = use_tbl ? add_class_table(li, v, start, step, count, tot, &code_pos)
                                         : (add_uniform(li, lc, v, start, step, count, &code_pos), 0);
                        if (st) return st;
                    }
                    int i = m - 1;
                    while (i >= 0 && ci[i] == na - m + i) i--;
                    if (i < 0) break;
                    ci[i]++;
                    for (int k = i + 1; k < m; k++) ci[k] = ci[k - 1] + 1;
                }
            }
            level_codes.push_back(code_pos);
        }
        num_codes = code_pos;
        choose_tiles(false);
        build_items();
        choose_tiles(true);
        coarse_dsmem = false;
        const char *cd = getenv("HPEZ_COARSE_DSMEM");
        if (c_coarse > 0 && !(cd && atoi(cd) == 0) && d.rank == 3 && !d.with_stats && !d.frozen_mask &&
            d.work_dtype == HPEZ_WORK_F32 && d.rounding == HPEZ_ROUND_F32 && d.code_dtype == HPEZ_CODES_U16)
            coarse_dsmem = coarse_dsmem_build(g, commits.data(), coarse_group.data(), c_coarse, num_codes, &cplan);
        return HPEZ_OK;
    }

    int add_class_table(int li, const std::vector<int> &v, const int64_t *start, const int64_t *step,
                        const int64_t *count, int64_t tot, int64_t *code_pos) {
        // np.unique over the class lattice tags (interp.py:423-432): the set of
        // blocks hit per axis, then their product.
        std::vector<std::vector<int64_t>> hit(d.rank);
        for (int a = 0; a < d.rank; a++) {
            int64_t last = -1;
            for (int64_t j = 0; j < count[a]; j++) {
                int64_t b = (start[a] + j * step[a]) / d.block_size;
                if (b != last) hit[a].push_back(b);
                last = b;
            }
        }
        std::set<int> present;
        std::vector<size_t> it(d.rank, 0);
        const uint8_t *tl = table.data() + (size_t)li * nblk_table;
        while (true) {
            int64_t b = 0;
            for (int a = 0; a < d.rank; a++) b += hit[a][it[a]] * g.bstr[a];
            present.insert(tl[b]);
            int a = d.rank - 1;
            while (a >= 0 && ++it[a] == hit[a].size()) it[a--] = 0;
            if (a < 0) break;
        }
        if (present.size() == 1) {
            Cfg c;
            if (!decode_tag(*present.begin(), &c)) return HPEZ_BAD_ARGUMENT;
            add_uniform(li, c, v, start, step, count, code_pos);
            return 0;
        }
        has_mixed = true;
        const int tag_off = (int)tags.size();
        const int slot_off = (int)slots.size();
        slots.resize(slots.size() + 256, 0);
        uint32_t axes_present = 0;
        int slot = 0;
        for (int t : present) {
            Cfg c;
            if (!decode_tag(t, &c)) return HPEZ_BAD_ARGUMENT;
            TagInfo ti{};
            ti.split = split_axis(c, v);
            ti.inter = make_pred(c, v, false);
            if (ti.split >= 0) {
                axes_present |= 1u << ti.split;
                ti.same.md = 0;
                ti.same.axis = ti.split;
                ti.same.fam = same_fam(c.spline);
            }
            tags.push_back(ti);
            slots[slot_off + t] = (uint8_t)slot++;
        }
        const int nph = __builtin_popcount(axes_present);
        // mixed fast path: tag -> (split + 1) << 6 | specialisation of the
        // commit-A (inter-level) and commit-B (same-level) predictors
        bool mfast = true;
        uint8_t desc_a[64] = {}, desc_b[64] = {};
        for (int t : present) {
            const TagInfo &ti = tags[tag_off + slots[slot_off + t]];
            const int fa = fast_id_pred(ti.inter);
            const int fb = ti.split >= 0 ? fast_id_pred(ti.same) : 0;
            if (t >= 64 || fa < 0 || fb < 0) {
                mfast = false;
                continue;
            }
            desc_a[t] = (uint8_t)(((ti.split + 1) << 6) | fa);
            desc_b[t] = (uint8_t)(((ti.split + 1) << 6) | fb);
        }
        Cfg mdc;
        mdc.md = 1;
        mdc.spline = 0;
        mdc.same = 0;
        const PredDev mdw = make_pred(mdc, v, false);  // MD blend weights depend on the class only
        for (int ph = -1; ph < nph; ph++) {
            CommitDev cm = base_commit(li, start, step, count);
            cm.kind = ph < 0 ? COMMIT_MIXED_A : COMMIT_MIXED_B;
            cm.phase = ph < 0 ? 0 : ph;
            cm.axes_present = axes_present;
            cm.tag_off = tag_off;
            cm.slot_off = slot_off;
            cm.code_base = -1;
            cm.pred = mdw;
            memcpy(cm.tdesc, ph < 0 ? desc_a : desc_b, 64);
            cm.fast_id = mfast ? -2 : -1;
            commits.push_back(cm);
            uint32_t vm = 0;
            for (int a : v) vm |= 1u << a;
            c_vmask.push_back(vm);
            c_reads.push_back(vm);  // any tag may predict along any class axis
        }
        *code_pos += tot;
        return 0;
    }

    // Rank-3 specialisation id (KIND * 5 + FAM) of one predictor, or -1.
    int fast_id_pred(const PredDev &p) const {
        if (d.rank != 3) return -1;
        if (!p.md) return p.axis * 5 + p.fam;
        if (p.fam > FAM_NAT_I) return -1;
        if (p.nax == 3) return 6 * 5 + p.fam;
        if (p.nax != 2) return -1;
        const int a = p.axes[0], b = p.axes[1];
        const int kind = (a == 0 && b == 1) ? 3 : (a == 0 && b == 2) ? 4 : (a == 1 && b == 2) ? 5 : -1;
        return kind < 0 ? -1 : kind * 5 + p.fam;
    }

    // Uniform commits: their specialisation id or -1.  Mixed commits: -2
    // (process_mixed) when every tag has a specialisation, the grid is
    // rank 3 and the block size a power of two; else -1 (generic path).
    int fast_id_of(const CommitDev &cm) const {
        if (d.rank != 3 || d.with_stats) return -1;
        if (cm.kind != COMMIT_UNIFORM) return (cm.fast_id == -2 && g.bs_log2 >= 0) ? -2 : -1;
        return fast_id_pred(cm.pred);
    }

    // Item interval of commit `pv` covering the outer-axis window of item
    // `it` of commit `cm` (stencil reach +-3s, plus one plane of pv on each
    // side so that coverage stays transitive along dependency chains).
    int2 dep_interval(const CommitDev &cm, int it, const CommitDev &pv) const {
        const int64_t U = (int64_t)cm.npos / cm.cnt[0];
        const int64_t pa = (int64_t)it * cm.p_item;
        const int64_t pb = std::min<int64_t>(pa + cm.p_item, cm.npos) - 1;
        const int64_t zlo = cm.start[0] + (pa / U) * (int64_t)cm.step[0] - 3 * (int64_t)cm.s;
        const int64_t zhi = cm.start[0] + (pb / U) * (int64_t)cm.step[0] + 3 * (int64_t)cm.s;
        auto fl = [](int64_t a, int64_t b) { return a >= 0 ? a / b : -((-a + b - 1) / b); };
        int64_t ja = fl(zlo - pv.start[0], pv.step[0]);
        int64_t jb = -fl(-(zhi - pv.start[0]), pv.step[0]);
        ja = std::max<int64_t>(0, std::min<int64_t>(ja, pv.cnt[0] - 1));
        jb = std::max<int64_t>(0, std::min<int64_t>(jb, pv.cnt[0] - 1));
        const int64_t Up = (int64_t)pv.npos / pv.cnt[0];
        const int64_t qa = ja * Up, qb = std::min<int64_t>((jb + 1) * Up, pv.npos) - 1;
        return int2{pv.item_base + (int)(qa / pv.p_item), pv.item_base + (int)(qb / pv.p_item)};
    }

    // Work items, (item, warp) tables, the commit dependency DAG and the
    // dependency intervals.  A commit of class v at level l reads (a) points
    // of classes v \ {a} of level l for every axis a it predicts along,
    // (b) earlier phases of its own class (same-level stencils, mixed B
    // commits), (c) coarser points, all produced by ancestors of the sinks of
    // the previous level's DAG.  Items are grabbed in (level, depth, outer
    // coordinate) order, so independent commits run concurrently.
    void build_items() {
        const int sms = num_sms();
        if (const char *ev = getenv("HPEZ_DIAG_SCALE")) kDiagScale = std::max(1, atoi(ev));
        int pmax = 512 * kItemWarps;
        if (const char *ev = getenv("HPEZ_ITEM_MAX")) pmax = std::max(256, atoi(ev));
        int items_per_sm = 2;
        if (const char *ev = getenv("HPEZ_ITEMS_PER_SM")) items_per_sm = std::max(1, atoi(ev));
        uint32_t coarse_max = kCoarseMax;
        if (const char *ev = getenv("HPEZ_COARSE_MAX")) coarse_max = (uint32_t)atoi(ev);
        if (const char *ev = getenv("HPEZ_COARSE_CLUSTER")) coarse_cluster = std::max(1, std::min(16, atoi(ev)));
        const int nc = (int)commits.size();
        // coarse prefix: leading levels of at most coarse_max points (latency-bound)
        c_coarse = 0;
        {
            int c = 0;
            uint64_t pts = 0;
            while (c < c_tile) {
                int e = c;
                while (e < c_tile && commits[e].level == commits[c].level) pts += commits[e++].npos;
                if (pts > coarse_max || (size_t)e * sizeof(CommitDev) > 200 * 1024) break;
                c = e;
            }
            c_coarse = c;
        }
        int32_t item = 0;
        for (int ci = 0; ci < nc; ci++) {
            CommitDev &cm = commits[ci];
            int64_t p = (int64_t)cm.npos / (items_per_sm * sms);
            // coarse commits: one position per lane, so a warp unit is one round trip
            p = ci < c_coarse ? 256 : std::max<int64_t>(256, std::min<int64_t>(pmax, p));
            p = (p + 255) / 256 * 256;
            cm.p_item = (int32_t)p;
            cm.pw = (int32_t)(p / kItemWarps);
            cm.n_items = (int32_t)((cm.npos + p - 1) / p);
            cm.item_base = item;
            item += cm.n_items;
        }
        n_items = item;
        // staged levels: the trailing levels of at least stage_min points each
        // (HPEZ_STAGE_MIN; the flow kernel keeps the smaller ones)
        int64_t stage_min = kStageMinPts;
        if (const char *ev = getenv("HPEZ_STAGE_MIN")) stage_min = atoll(ev);
        c_stage = c_tile;
        while (c_stage > c_coarse) {
            int b = c_stage;
            const int lvl = commits[b - 1].level;
            int64_t pts = 0;
            while (b > 0 && commits[b - 1].level == lvl) pts += commits[--b].npos;
            if (pts < stage_min || b < c_coarse) break;
            c_stage = b;
        }
        // commit DAG
        std::vector<std::vector<int>> preds(nc);
        std::vector<int> depth(nc, 0);
        std::vector<int> prev_sinks;
        int lv_begin = 0;
        while (lv_begin < nc) {
            const int lvl = commits[lv_begin].level;
            int lv_end = lv_begin;
            while (lv_end < nc && commits[lv_end].level == lvl) lv_end++;
            std::vector<bool> has_succ(nc, false);
            for (int c = lv_begin; c < lv_end; c++) {
                for (int d : prev_sinks) preds[c].push_back(d);
                const uint32_t v = c_vmask[c], rd = c_reads[c];
                int dmax = 0;
                for (int d = lv_begin; d < c; d++) {
                    const uint32_t w = c_vmask[d];
                    bool dep = w == v;  // earlier phase of the same class
                    for (int a = 0; a < d_rank(); a++)
                        if ((rd >> a & 1) && (v >> a & 1) && w == (v & ~(1u << a))) dep = true;
                    if (dep) {
                        preds[c].push_back(d);
                        has_succ[d] = true;
                        dmax = std::max(dmax, depth[d] + 1);
                    }
                }
                depth[c] = dmax;
            }
            prev_sinks.clear();
            for (int c = lv_begin; c < lv_end; c++)
                if (!has_succ[c]) prev_sinks.push_back(c);
            lv_begin = lv_end;
        }
        // coarse schedule: (level, depth) groups of (commit, item) pairs
        coarse_pairs.clear();
        coarse_groups.clear();
        coarse_group.assign(c_coarse, 0);
        for (int c = 0; c < c_coarse;) {
            int e = c;
            while (e < c_coarse && commits[e].level == commits[c].level) e++;
            int maxd = 0;
            for (int k = c; k < e; k++) maxd = std::max(maxd, depth[k]);
            for (int dd = 0; dd <= maxd; dd++) {
                const int g0 = (int)coarse_pairs.size() / 2;
                for (int k = c; k < e; k++)
                    if (depth[k] == dd) coarse_group[k] = (int)coarse_groups.size() / 2;
                for (int k = c; k < e; k++)
                    if (depth[k] == dd)
                        for (int it = 0; it < commits[k].n_items; it++) {
                            coarse_pairs.push_back(k);
                            coarse_pairs.push_back(commits[k].item_base + it);
                        }
                const int g1 = (int)coarse_pairs.size() / 2;
                if (g1 > g0) {
                    coarse_groups.push_back(g0);
                    coarse_groups.push_back(g1);
                }
            }
            c = e;
        }
        // per-item tables and dependency intervals
        item_commit.assign(n_items, 0);
        wn.assign((size_t)n_items * kItemWarps, 0);
        dep_off.assign(n_items + 1, 0);
        dep_rng.clear();
        struct Key { int level, depth; int64_t z; int c, it; };
        std::vector<Key> keys;
        for (int ci = 0; ci < nc; ci++) {
            const CommitDev &cm = commits[ci];
            for (int it = 0; it < cm.n_items; it++) {
                const int gi = cm.item_base + it;
                item_commit[gi] = ci;
                for (int w = 0; w < kItemWarps; w++) {
                    const int64_t p0 = (int64_t)it * cm.p_item + (int64_t)w * cm.pw;
                    const int64_t p1 = std::min<int64_t>(p0 + cm.pw, cm.npos);
                    if (cm.kind == COMMIT_UNIFORM) wn[(size_t)gi * kItemWarps + w] = (int32_t)std::max<int64_t>(0, p1 - p0);
                }
                if (cm.kind != COMMIT_UNIFORM) mixed_items.push_back(gi);
                dep_off[gi] = (int32_t)dep_rng.size();
                if (ci >= c_coarse && ci < c_stage) {
                    for (int d : preds[ci])
                        if (d >= c_coarse) dep_rng.push_back(dep_interval(cm, it, commits[d]));
                    const int64_t U = (int64_t)cm.npos / cm.cnt[0];
                    const int64_t z = cm.start[0] + ((int64_t)it * cm.p_item / U) * (int64_t)cm.step[0];
                    keys.push_back(Key{cm.level, depth[ci], z, ci, it});
                }
            }
        }
        dep_off[n_items] = (int32_t)dep_rng.size();
        // Diagonal (wavefront) order within a level: key z + depth * W with W
        // wider than any dependency reach, so an item's dependencies are
        // always grabbed before it while the in-flight band of planes stays
        // small enough to live in L2.  Verified below; depth-major fallback.
        std::vector<int64_t> wlev(64, 0);
        for (const Key &k : keys) {
            const CommitDev &cm = commits[k.c];
            const int64_t U = (int64_t)cm.npos / cm.cnt[0];
            const int64_t pa = (int64_t)k.it * cm.p_item;
            const int64_t pb = std::min<int64_t>(pa + cm.p_item, cm.npos) - 1;
            const int64_t span = ((pb / U) - (pa / U)) * (int64_t)cm.step[0];
            wlev[k.level & 63] = std::max<int64_t>(wlev[k.level & 63], kDiagScale * (span + 7 * (int64_t)cm.s + 2 * cm.step[0] + 1));
        }
        auto order_by = [&](bool diag) {
            std::vector<Key> ks = keys;
            std::stable_sort(ks.begin(), ks.end(), [&](const Key &a, const Key &b) {
                if (a.level != b.level) return a.level < b.level;
                if (diag) {
                    const int64_t ka = a.z + a.depth * wlev[a.level & 63], kb = b.z + b.depth * wlev[b.level & 63];
                    if (ka != kb) return ka < kb;
                }
                if (a.depth != b.depth) return a.depth < b.depth;
                if (a.z != b.z) return a.z < b.z;
                if (a.c != b.c) return a.c < b.c;
                return a.it < b.it;
            });
            std::vector<int32_t> ord;
            for (const Key &k : ks) ord.push_back(commits[k.c].item_base + k.it);
            return ord;
        };
        auto valid = [&](const std::vector<int32_t> &ord) {
            std::vector<int32_t> pos(n_items, -1);
            for (size_t i = 0; i < ord.size(); i++) pos[ord[i]] = (int32_t)i;
            for (size_t i = 0; i < ord.size(); i++) {
                const int it = ord[i];
                for (int k = dep_off[it]; k < dep_off[it + 1]; k++)
                    for (int q = dep_rng[k].x; q <= dep_rng[k].y; q++)
                        if (pos[q] < 0 || pos[q] >= (int32_t)i) return false;
            }
            return true;
        };
        // stage groups: (level, depth) in order, commits of one group independent
        stages.clear();
        for (int c = c_stage; c < c_tile;) {
            int e = c;
            while (e < c_tile && commits[e].level == commits[c].level) e++;
            int maxd = 0;
            for (int k = c; k < e; k++) maxd = std::max(maxd, depth[k]);
            for (int dd = 0; dd <= maxd; dd++) {
                StageGroup G{};
                for (int k = c; k < e; k++) {
                    if (depth[k] != dd) continue;
                    if (G.n == kStageMax) {  // split an oversized group (still independent)
                        stages.push_back(G);
                        G = StageGroup{};
                    }
                    G.c[G.n] = k;
                    G.u_off[G.n + 1] = G.u_off[G.n] + commits[k].n_items * kItemWarps;
                    G.n++;
                }
                if (G.n) stages.push_back(G);
            }
            c = e;
        }
        flow_order = order_by(true);
        diag_order = valid(flow_order);
        if (!diag_order) flow_order = order_by(false);
        first_flow_item = 0;
        flow_grid = std::max(1, (int)flow_order.size());  // capped by occupancy at launch
        coarse_fast = flow_fast = stage_fast = true;
        for (int ci = 0; ci < c_tile; ci++) {
            CommitDev &cm = commits[ci];
            cm.fast_id = fast_id_of(cm);
            bool &f = ci < c_coarse ? coarse_fast : (ci < c_stage ? flow_fast : stage_fast);
            f = f && cm.fast_id != -1;
        }
        if (getenv("HPEZ_COARSE_GENERIC")) coarse_fast = false;
    }
    int d_rank() const { return d.rank; }

    // The finest levels as row-fused launches (row.cu): rank-3 f32 grids with
    // u16 codes, no stats, strides 1 / 2 / 4, multidim or split-free one-axis
    // variants, at least HPEZ_ROW_MIN points each (default 1M);
    // HPEZ_ROW=0 keeps them in the flow kernel, HPEZ_ROW_LEVELS caps how many.
    void choose_row() {
        const int nc = (int)commits.size();
        const char *ev = getenv("HPEZ_ROW");
        if (ev && atoi(ev) == 0) return;
        if (d.rank != 3 || d.with_stats || d.work_dtype != HPEZ_WORK_F32 || d.rounding != HPEZ_ROUND_F32 ||
            d.code_dtype != HPEZ_CODES_U16 || d.frozen_mask || d.direction > HPEZ_DECOMPRESS || nc == 0)
            return;
        int64_t min_pts = 1 << 20;
        if (const char *m = getenv("HPEZ_ROW_MIN")) min_pts = atoll(m);
        int max_levels = 3;
        if (const char *m = getenv("HPEZ_ROW_LEVELS")) max_levels = atoi(m);
        const bool use_tbl = !table.empty();
        const auto oc = order_candidates();
        int e = nc;
        while (e > 0 && (int)rows.size() < max_levels) {
            const int li = commits[e - 1].level;
            int b = e;
            int64_t pts = 0;
            while (b > 0 && commits[b - 1].level == li) pts += commits[--b].npos;
            if (pts < min_pts) break;
            // the level's own tag (plan.encode_tag, plan.py:69-75) when there is no table
            int tag = levels[li].kernel;
            if (levels[li].paradigm != 1) {
                int pi = -1;
                for (size_t k = 0; k < oc.size(); k++) {
                    bool same = (int)oc[k].size() == levels[li].n_order;
                    for (int j = 0; same && j < levels[li].n_order; j++) same = oc[k][j] == levels[li].axis_order[j];
                    if (same) pi = (int)k;
                }
                if (pi < 0) break;
                tag += 8 * (pi + 1);
            }
            RowPlan rp;
            if (!row_plan_build(g, &commits[b], &c_vmask[b], e - b, b,
                                use_tbl ? table.data() + (size_t)li * nblk_table : nullptr, nblk_table, tag,
                                level_codes[li], &rp))
                break;
            rows.insert(rows.begin(), rp);
            row_level.insert(row_level.begin(), li);
            c_tile = b;
            e = b;
        }
    }

    // Finest levels that run as shared-memory tiled launches (tile.cu):
    // rank-3 f32 grids with u16 codes, no stats, uniform commits, at least
    // HPEZ_TILE_MIN points (default 200k).  `final` builds the real plans
    // once build_items has assigned the (item, warp) stream bookkeeping.
    void choose_tiles(bool final) {
        const int nc = (int)commits.size();
        if (final) {
            tiles.clear();
            if (!rows.empty()) return;
            for (int c = c_tile; c < nc;) {
                int e = c;
                while (e < nc && commits[e].level == commits[c].level) e++;
                TilePlan tp;
                tile_plan_build(g, &commits[c], e - c, num_codes, &tp);
                tiles.push_back(tp);
                c = e;
            }
            return;
        }
        c_tile = nc;
        rows.clear();
        row_level.clear();
        choose_row();
        if (!rows.empty()) return;
        // opt-in (HPEZ_TILE=1): measured slower than the flow kernel on cfg2
        // so far (profiles/); kept parity-green for the tiling work ahead
        const char *ev = getenv("HPEZ_TILE");
        if (!ev || atoi(ev) == 0) return;
        if (d.rank != 3 || d.with_stats || d.work_dtype != HPEZ_WORK_F32 || d.rounding != HPEZ_ROUND_F32 ||
            d.code_dtype != HPEZ_CODES_U16 || d.frozen_mask)
            return;
        int64_t min_pts = 200000;
        if (const char *m = getenv("HPEZ_TILE_MIN")) min_pts = atoll(m);
        int c = nc;
        while (c > 0) {
            int b = c;
            const int lvl = commits[c - 1].level;
            int64_t pts = 0;
            while (b > 0 && commits[b - 1].level == lvl) pts += commits[--b].npos;
            if (pts < min_pts) break;
            TilePlan tp;
            if (!tile_plan_build(g, &commits[b], c - b, num_codes, &tp)) break;
            c = b;
        }
        c_tile = c;
    }
};

// Device workspace layout: every table and scratch array of a plan carved
// from one caller-provided block (hpez_plan_workspace_size / _bind), so a
// run never allocates.  Offsets are 256-byte aligned.
struct Carver {
    char *base;
    size_t off = 0;
    template <typename T>
    void take(T **p, size_t n) {
        off = (off + 255) & ~(size_t)255;
        *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
        off += std::max<size_t>(n, 1) * sizeof(T);
    }
};

static bool plan_stats(const Plan &p) { return p.d.with_stats && p.d.direction == HPEZ_COMPRESS; }

static size_t plan_layout(Plan &p, char *base) {
    Carver c{base};
    const size_t ni = (size_t)std::max(p.n_items, 1);
    const size_t ne = ni * kItemWarps;
    const size_t ntiles = (ne + kScanTile - 1) / kScanTile + 1;
    const size_t nc = std::max<size_t>(p.commits.size(), 1);
    c.take(&p.d_commits, p.commits.size());
    c.take(&p.d_item_commit, p.item_commit.size());
    c.take(&p.d_flow_order, p.flow_order.size());
    c.take(&p.d_dep_off, p.dep_off.size());
    c.take(&p.d_dep_rng, p.dep_rng.size());
    c.take(&p.d_coarse_pairs, p.coarse_pairs.size());
    c.take(&p.d_coarse_groups, p.coarse_groups.size());
    c.take(&p.d_wn, p.wn.size());
    c.take(&p.d_wbase, ne);
    c.take(&p.d_esc_cnt, ne);
    c.take(&p.d_esc_off, ne);
    c.take(&p.d_scan_tmp, ntiles);
    c.take(&p.d_total, 4);
    c.take(&p.d_done, ni);
    c.take(&p.d_counters, 4);
    c.take(&p.d_tags, p.tags.size());
    c.take(&p.d_slots, p.slots.size());
    c.take(&p.d_table, p.table.size());
    c.take(&p.d_mixed_items, p.mixed_items.size());
    c.take(&p.d_clevel, nc);
    c.take(&p.d_cbase, nc);
    c.take(&p.d_cn, nc);
    if (plan_stats(p)) {
        c.take(&p.d_csum, nc);
        c.take(&p.d_errbuf, (size_t)std::max<int64_t>(p.num_codes, 1));
    }
    if (p.profile) c.take(&p.d_prof, 96);
    for (RowPlan &rp : p.rows) {
        c.take(&rp.d_cnt, (size_t)rp.d.n_entries);
        c.take(&rp.d_base, (size_t)rp.d.n_entries);
        c.take(&rp.d_tmp, (size_t)scan_tmp_size(rp.d.n_entries));
        c.take(&rp.d_total, 4);
    }
    if (!p.tiles.empty() && p.d.direction == HPEZ_COMPRESS) {
        char *o;
        c.take(&o, (size_t)p.g.npts * (p.d.work_dtype == HPEZ_WORK_F32 ? 4 : 8));
        p.d_orig_scratch = o;
    }
    return c.off + 256;
}

template <typename T>
static cudaError_t up(T *d, const std::vector<T> &v, cudaStream_t st) {
    if (v.empty()) return cudaSuccess;
    return cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st);
}

static int cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return HPEZ_OK;
    fprintf(stderr, "hpez_b200: CUDA error %s\n", cudaGetErrorString(e));
    return HPEZ_CUDA_ERROR;
}

typedef void (*sweep_fn)(const SweepArgs);

typedef void (*stage_fn)(const SweepArgs, const StageGroup);

struct KernelSet {
    sweep_fn coarse, flow, coarse_fast, flow_fast;  // *_fast null when not instantiated
    stage_fn stage, stage_fast;
};

// Fast rank-3 paths are instantiated for the production element types:
// f32 grids (ROUND_F32, f32 storage) and f64 grids (ROUND_NONE), u16 codes.
template <typename T, typename C, int DIR, int ROUND>
static constexpr bool kFastTypes = (std::is_same<C, uint16_t>::value &&
                                    ((std::is_same<T, float>::value && ROUND == HPEZ_ROUND_F32) ||
                                     (std::is_same<T, double>::value && ROUND == HPEZ_ROUND_NONE)));

template <typename T, typename C, int DIR, int ROUND>
static KernelSet pick3(bool stats) {
    KernelSet k{};
    if (DIR == HPEZ_COMPRESS && stats) {
        k.coarse = coarse_kernel<T, C, DIR, ROUND, true, false>;
        k.flow = flow_kernel<T, C, DIR, ROUND, true, false>;
        k.stage = stage_kernel<T, C, DIR, ROUND, true, false>;
        return k;
    }
    k.coarse = coarse_kernel<T, C, DIR, ROUND, false, false>;
    k.flow = flow_kernel<T, C, DIR, ROUND, false, false>;
    k.stage = stage_kernel<T, C, DIR, ROUND, false, false>;
    if constexpr (kFastTypes<T, C, DIR, ROUND>) {
        k.coarse_fast = coarse_kernel<T, C, DIR, ROUND, false, true>;
        k.flow_fast = flow_kernel<T, C, DIR, ROUND, false, true>;
        k.stage_fast = stage_kernel<T, C, DIR, ROUND, false, true>;
    }
    return k;
}

template <typename T, typename C>
static KernelSet pick2(int dir, int round, bool stats) {
    if (dir == HPEZ_COMPRESS) {
        if (round == HPEZ_ROUND_F32) return pick3<T, C, HPEZ_COMPRESS, HPEZ_ROUND_F32>(stats);
        if (round == HPEZ_ROUND_INT) return pick3<T, C, HPEZ_COMPRESS, HPEZ_ROUND_INT>(stats);
        return pick3<T, C, HPEZ_COMPRESS, HPEZ_ROUND_NONE>(stats);
    }
    if (round == HPEZ_ROUND_F32) return pick3<T, C, HPEZ_DECOMPRESS, HPEZ_ROUND_F32>(false);
    if (round == HPEZ_ROUND_INT) return pick3<T, C, HPEZ_DECOMPRESS, HPEZ_ROUND_INT>(false);
    return pick3<T, C, HPEZ_DECOMPRESS, HPEZ_ROUND_NONE>(false);
}

static KernelSet pick(const hpez_sweep_desc &d) {
    const bool stats = d.with_stats != 0;
    if (d.work_dtype == HPEZ_WORK_F32) {
        if (d.code_dtype == HPEZ_CODES_U16) return pick2<float, uint16_t>(d.direction, d.rounding, stats);
        return pick2<float, int32_t>(d.direction, d.rounding, stats);
    }
    if (d.code_dtype == HPEZ_CODES_U16) return pick2<double, uint16_t>(d.direction, d.rounding, stats);
    return pick2<double, int32_t>(d.direction, d.rounding, stats);
}

static SweepArgs base_args(Plan &p) {
    SweepArgs A{};
    A.g = p.g;
    A.commits = p.d_commits;
    A.item_commit = p.d_item_commit;
    A.flow_order = p.d_flow_order;
    A.dep_off = p.d_dep_off;
    A.dep_rng = p.d_dep_rng;
    A.coarse_pairs = p.d_coarse_pairs;
    A.coarse_groups = p.d_coarse_groups;
    A.n_groups = (int32_t)(p.coarse_groups.size() / 2);
    A.prof = p.d_prof;
    A.dbg = getenv("HPEZ_DEBUG_NODEPS") ? 1 : 0;
    // TMA bulk L2 prefetch of the next item's code range: helps decompress, not compress (measured)
    A.l2_prefetch = getenv("HPEZ_L2_PREFETCH") ? atoi(getenv("HPEZ_L2_PREFETCH")) : p.d.direction == HPEZ_DECOMPRESS;
    A.wbase = p.d_wbase;
    A.wn = p.d_wn;
    A.esc_cnt = p.d_esc_cnt;
    A.esc_off = p.d_esc_off;
    A.done = p.d_done;
    A.next = p.d_counters;
    A.flags = p.d_counters + 1;
    A.tags = p.d_tags;
    A.slots = p.d_slots;
    A.table = p.d_table;
    return A;
}

static int plan_setup(Plan *p, cudaStream_t st) {
    cudaError_t e = cudaSuccess;
    if (!p->ws) {  // no caller workspace: one allocation, owned by the plan
        p->ws_bytes = plan_layout(*p, nullptr);
        e = cudaMalloc(&p->own_ws, p->ws_bytes);
        if (e) return cuda_status(e);
        p->ws = p->own_ws;
    }
    plan_layout(*p, (char *)(((uintptr_t)p->ws + 255) & ~(uintptr_t)255));
    e = up(p->d_commits, p->commits, st);
    if (!e) e = up(p->d_item_commit, p->item_commit, st);
    if (!e) e = up(p->d_flow_order, p->flow_order, st);
    if (!e) e = up(p->d_dep_off, p->dep_off, st);
    if (!e) e = up(p->d_dep_rng, p->dep_rng, st);
    if (!e) e = up(p->d_coarse_pairs, p->coarse_pairs, st);
    if (!e) e = up(p->d_coarse_groups, p->coarse_groups, st);
    if (!e) e = up(p->d_wn, p->wn, st);
    if (!e) e = up(p->d_tags, p->tags, st);
    if (!e) e = up(p->d_slots, p->slots, st);
    if (!e) e = up(p->d_table, p->table, st);
    if (!e) e = up(p->d_mixed_items, p->mixed_items, st);
    if (!e) e = up(p->d_clevel, p->clevel, st);
    if (!e && p->d_prof) {
        e = cudaMemsetAsync(p->d_prof, 0, 8 * sizeof(unsigned long long), st);
        if (!e) e = cudaMemsetAsync(p->d_prof + 8, 0xff, 24 * sizeof(unsigned long long), st);
        for (int l = 0; l < 12 && !e; l++) e = cudaMemsetAsync(p->d_prof + 9 + 2 * l, 0, sizeof(unsigned long long), st);
        if (!e) e = cudaMemsetAsync(p->d_prof + 32, 0, 64 * sizeof(unsigned long long), st);
    }
    if (e) return cuda_status(e);
    SweepArgs A = base_args(*p);
    if (!p->mixed_items.empty()) {
        const int64_t thr = (int64_t)p->mixed_items.size() * kItemWarps * 32;
        mixed_count_kernel<<<(unsigned)((thr + 255) / 256), 256, 0, st>>>(A, p->d_wn, (int32_t)p->mixed_items.size(),
                                                                         p->d_mixed_items);
    }
    // code index of every (item, warp)'s first member = exclusive scan of member counts
    if (p->n_items > 0)
        exclusive_scan(p->d_wn, (int64_t)p->n_items * kItemWarps, p->d_wbase, p->d_scan_tmp, p->d_total, st);
    if (!p->commits.empty())
        commit_ranges_kernel<<<(unsigned)p->commits.size(), 256, 0, st>>>(
            p->d_commits, (int)p->commits.size(), p->d_wbase, p->d_wn, p->d_cbase, p->d_cn);
    e = cudaGetLastError();
    for (size_t i = 0; i < p->rows.size() && !e; i++)
        e = row_plan_setup(p->rows[i], p->table.empty() ? nullptr : p->d_table + (size_t)p->row_level[i] * p->nblk_table, st);
    if (e) return cuda_status(e);
    p->setup_done = true;
    return HPEZ_OK;
}

}  // namespace hpez

using namespace hpez;

struct hpez_plan_s {
    Plan p;
};

extern "C" {

int hpez_plan_create(const hpez_sweep_desc *desc, hpez_plan *out) {
    if (!desc || !out) return HPEZ_BAD_ARGUMENT;
    if (desc->rank < 1 || desc->rank > kMaxRank || desc->n_levels < 0 || (desc->n_levels > 0 && !desc->levels))
        return HPEZ_BAD_ARGUMENT;
    std::unique_ptr<hpez_plan_s> h(new hpez_plan_s());
    Plan &p = h->p;
    p.d = *desc;
    p.levels.assign(desc->levels, desc->levels + desc->n_levels);
    int st = p.build();
    if (st) return st;
    p.d.levels = nullptr;
    p.d.md_alpha = nullptr;
    p.d.block_table = nullptr;
    cudaError_t e = upload_rows();
    if (e) return cuda_status(e);
    p.profile = getenv("HPEZ_PROFILE") != nullptr;
    p.clevel.assign(std::max<size_t>(p.commits.size(), 1), 0);
    for (size_t i = 0; i < p.commits.size(); i++) p.clevel[i] = p.commits[i].level;
    if (p.d.direction == HPEZ_DECOMPRESS && p.coarse_dsmem && !getenv("HPEZ_NO_FORK")) {
        // decompress: the zero-count pre-pass runs beside the coarse kernel
        e = cudaStreamCreateWithFlags(&p.side, cudaStreamNonBlocking);
        if (!e) e = cudaEventCreateWithFlags(&p.ev_fork, cudaEventDisableTiming);
        if (!e) e = cudaEventCreateWithFlags(&p.ev_join, cudaEventDisableTiming);
        if (e) return cuda_status(e);
    }
    p.ws_bytes = plan_layout(p, nullptr);
    *out = h.release();
    return HPEZ_OK;
}

int hpez_plan_workspace_size(hpez_plan plan, int64_t *bytes) {
    if (!plan || !bytes) return HPEZ_BAD_ARGUMENT;
    *bytes = (int64_t)plan->p.ws_bytes;
    return HPEZ_OK;
}

int hpez_plan_bind_workspace(hpez_plan plan, void *ws, int64_t bytes) {
    if (!plan || !ws || bytes < (int64_t)plan->p.ws_bytes) return HPEZ_BAD_ARGUMENT;
    Plan &p = plan->p;
    if (p.setup_done || p.own_ws) return HPEZ_BAD_ARGUMENT;  // bind once, before the first run
    p.ws = ws;
    return HPEZ_OK;
}

int hpez_plan_destroy(hpez_plan plan) {
    delete plan;
    return HPEZ_OK;
}

int64_t hpez_plan_num_codes(hpez_plan plan) { return plan ? plan->p.num_codes : -1; }
int32_t hpez_plan_num_commits(hpez_plan plan) { return plan ? (int32_t)plan->p.commits.size() : -1; }

int32_t hpez_plan_num_launches(hpez_plan plan) {
    if (!plan) return -1;
    const Plan &p = plan->p;
    int n = 0;
    if (!p.coarse_groups.empty() || p.coarse_dsmem) n++;
    if (!p.flow_order.empty()) n++;
    n += (int)p.stages.size();
    n += (int)p.tiles.size();
    for (const RowPlan &rp : p.rows) n += rp.n_launch;  // row-fused levels (row.cu)
    n += 1;  // escape scan (single-pass look-back kernel)
    n += 1;  // escape count pre-pass (decompress) or outlier gather (compress)
    if (p.d.with_stats && p.d.direction == HPEZ_COMPRESS) n += 2;
    return n;
}

// Diagnostics: [n_items, n_flow_items, coarse_commits, coarse_groups,
// diag_order, flow_fast, coarse_fast, dep_intervals] and, when the plan was
// built with HPEZ_PROFILE set, the flow kernel's accumulated clock64 phase
// counters [grab, wait, work, items] (out[8..11]).
int hpez_plan_levels_timeline(hpez_plan plan, int64_t *out) {  // 72 values, see the header
    if (!plan || !out || !plan->p.d_prof) return HPEZ_BAD_ARGUMENT;
    unsigned long long h[80];
    if (cudaMemcpy(h, plan->p.d_prof + 8, sizeof h, cudaMemcpyDeviceToHost) != cudaSuccess) return HPEZ_CUDA_ERROR;
    for (int i = 0; i < 24; i++) out[i] = (int64_t)h[i];
    for (int i = 0; i < 48; i++) out[24 + i] = (int64_t)h[32 + i];
    return HPEZ_OK;
}

int hpez_plan_info(hpez_plan plan, int64_t *out) {
    if (!plan || !out) return HPEZ_BAD_ARGUMENT;
    const Plan &p = plan->p;
    out[0] = p.n_items;
    out[1] = (int64_t)p.flow_order.size();
    out[2] = p.c_coarse;
    out[3] = (int64_t)p.coarse_groups.size() / 2;
    out[4] = p.diag_order;
    out[5] = p.flow_fast;
    out[6] = p.coarse_fast + 2 * p.coarse_dsmem;  // bit 1: coarse levels in distributed shared memory
    out[7] = (int64_t)p.dep_rng.size();
    for (int i = 8; i < 12; i++) out[i] = -1;
    if (p.d_prof) {
        unsigned long long h[4];
        if (cudaMemcpy(h, p.d_prof, sizeof h, cudaMemcpyDeviceToHost) == cudaSuccess)
            for (int i = 0; i < 4; i++) out[8 + i] = (int64_t)h[i];
    }
    return HPEZ_OK;
}

int32_t hpez_plan_commit_stats(hpez_plan plan, int64_t *out, int32_t cap) {
    if (!plan || !out || cap < 6) return -HPEZ_BAD_ARGUMENT;
    const Plan &p = plan->p;
    if (!p.setup_done) return -HPEZ_BAD_ARGUMENT;
    std::vector<int32_t> wn((size_t)std::max(p.n_items, 1) * kItemWarps);
    if (cudaMemcpy(wn.data(), p.d_wn, wn.size() * sizeof(int32_t), cudaMemcpyDeviceToHost) != cudaSuccess)
        return -HPEZ_CUDA_ERROR;
    int32_t k = 0;
    for (size_t c = 0; c < p.commits.size() && (k + 1) * 6 <= cap; c++, k++) {
        const CommitDev &cm = p.commits[c];
        int64_t m = 0;
        for (int64_t e = (int64_t)cm.item_base * kItemWarps; e < (int64_t)(cm.item_base + cm.n_items) * kItemWarps; e++)
            m += wn[e];
        const int64_t v[6] = {cm.kind, cm.level, cm.npos, cm.n_items, m, cm.fast_id};
        for (int i = 0; i < 6; i++) out[6 * k + i] = v[i];
    }
    return k;
}

int hpez_plan_level_codes(hpez_plan plan, int64_t *out) {
    if (!plan || !out) return HPEZ_BAD_ARGUMENT;
    for (size_t i = 0; i < plan->p.level_codes.size(); i++) out[i] = plan->p.level_codes[i];
    return HPEZ_OK;
}

int hpez_set_device(int32_t device) { return cuda_status(cudaSetDevice(device)); }

const char *hpez_build_info(void) { return "libhpez_b200 sm_100a f64 -fmad=false"; }

static int sweep_run(hpez_plan plan, const void *orig, void *work, void *codes, int64_t codes_avail, double *outliers,
                     int64_t outl_cap, double *stat_err_sum, int64_t *stat_count, double *stat_dense, void *stream) {
    if (!plan || !work) return HPEZ_BAD_ARGUMENT;
    Plan &p = plan->p;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t esz = p.d.work_dtype == HPEZ_WORK_F32 ? 4 : 8;
    if (p.d.direction != HPEZ_COMPRESS || !orig) orig = work;
    if (orig != work) {
        // anchors: the lattice no commit covers (plan.py:142-161)
        if (p.levels.empty() || p.d.with_stats) return HPEZ_BAD_ARGUMENT;
        const int64_t A = 2 * (int64_t)p.levels[0].stride;
        int64_t na = 1;
        for (int a = 0; a < p.d.rank; a++)
            na *= (p.d.frozen_mask >> a & 1) ? p.g.dims[a] : (p.g.dims[a] + A - 1) / A;
        if (na + p.num_codes != p.g.npts) return HPEZ_BAD_ARGUMENT;
        const int64_t thr = std::max<int64_t>(na, 1);
        copy_anchors_kernel<<<(unsigned)((thr + 255) / 256), 256, 0, st>>>(p.g, (uint32_t)A, p.d.frozen_mask, na,
                                                                           (const char *)orig, (char *)work, (int)esz);
    } else if (p.d.direction == HPEZ_COMPRESS && !p.tiles.empty()) {
        // tiled levels recompute halo points from originals that a neighbour
        // may already have overwritten in place: keep a copy
        if (!p.setup_done) {
            int s = plan_setup(&p, st);
            if (s) return s;
        }
        cudaError_t e = cudaMemcpyAsync(p.d_orig_scratch, work, (size_t)p.g.npts * esz, cudaMemcpyDeviceToDevice, st);
        if (e) return cuda_status(e);
        orig = p.d_orig_scratch;
    }
    if (p.d.direction == HPEZ_DECOMPRESS && codes_avail < p.num_codes) return HPEZ_CORRUPT_STREAM;
    if (p.num_codes > 0 && !codes) return HPEZ_BAD_ARGUMENT;
    const bool stats = p.d.with_stats && p.d.direction == HPEZ_COMPRESS;
    // stats: err_sum and count together, or neither (dense error grids only)
    if (stats && (!stat_err_sum) != (!stat_count)) return HPEZ_BAD_ARGUMENT;
    if (!p.setup_done) {
        int s = plan_setup(&p, st);
        if (s) return s;
    }
    const int64_t ne = (int64_t)p.n_items * kItemWarps;
    cudaError_t e = cudaMemsetAsync(p.d_counters, 0, 4 * sizeof(int32_t), st);
    if (!e) e = cudaMemsetAsync(p.d_total, 0, sizeof(int64_t), st);
    if (e) return cuda_status(e);
    if (p.n_items == 0) {  // no commits (e.g. a grid made of anchors only)
        p.outl_cap_last = outliers ? outl_cap : 0;
        return HPEZ_OK;
    }
    e = cudaMemsetAsync(p.d_done, 0, sizeof(uint32_t) * (size_t)p.n_items, st);
    if (e) return cuda_status(e);
    SweepArgs A = base_args(p);
    A.work = work;
    A.orig = orig;
    A.codes = codes;
    A.outl = outliers;
    A.outl_cap = outliers ? outl_cap : 0;
    A.errbuf = p.d_errbuf;
    A.dense = stat_dense;
    const KernelSet ks = pick(p.d);
    // decompress with the DSMEM coarse kernel: it ranks its own outliers (the
    // coarse levels are the stream prefix), so the zero-count pre-pass only
    // has to finish before the flow kernel and runs on a side stream
    const bool fork = p.d.direction == HPEZ_DECOMPRESS && p.coarse_dsmem && p.side;
    cudaStream_t pst = st;
    if (fork) {
        e = cudaEventRecord(p.ev_fork, st);
        if (!e) e = cudaStreamWaitEvent(p.side, p.ev_fork, 0);
        if (e) return cuda_status(e);
        pst = p.side;
    }
    if (p.d.direction == HPEZ_DECOMPRESS) {
        // outlier ranks: zero codes per (item, warp), then an exclusive scan
        const int64_t thr = ne * 32;
        if (p.d.code_dtype == HPEZ_CODES_U16)
            count_zero_stream_kernel<<<(unsigned)((ne + kZeroEpb - 1) / kZeroEpb), 256, 0, pst>>>(
                (const uint16_t *)codes, p.d_wbase, p.d_wn, ne, p.d_esc_cnt);
        else
            count_zero_kernel<<<(unsigned)((thr + 255) / 256), 256, 0, pst>>>((const int32_t *)codes, p.d_wbase, p.d_wn,
                                                                              ne, p.d_esc_cnt);
        exclusive_scan(p.d_esc_cnt, ne, p.d_esc_off, p.d_scan_tmp, p.d_total, pst);
    }
    if (fork) {
        e = cudaEventRecord(p.ev_join, p.side);
        if (e) return cuda_status(e);
    }
    if (p.coarse_dsmem) {
        if (p.d.direction == HPEZ_COMPRESS && p.c_coarse < (int)p.commits.size()) {
            const int64_t e1 = (int64_t)p.commits[p.c_coarse].item_base * kItemWarps;
            e = cudaMemsetAsync(p.d_esc_cnt, 0, (size_t)e1 * sizeof(uint32_t), st);
            if (e) return cuda_status(e);
        } else if (p.d.direction == HPEZ_COMPRESS) {
            e = cudaMemsetAsync(p.d_esc_cnt, 0, (size_t)ne * sizeof(uint32_t), st);
            if (e) return cuda_status(e);
        }
        TileRun cr{orig, work, codes, outliers, A.outl_cap, p.d_esc_cnt, p.d_esc_off, p.d_counters + 1};
        e = coarse_dsmem_launch(p.cplan, p.d.direction, cr, st);
        if (!e && fork) e = cudaStreamWaitEvent(st, p.ev_join, 0);
        if (e) return cuda_status(e);
    } else if (!p.coarse_groups.empty()) {
        sweep_fn f = (p.coarse_fast && ks.coarse_fast) ? ks.coarse_fast : ks.coarse;
        const size_t smem = (size_t)p.c_coarse * sizeof(CommitDev);
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(smem, 1));
        cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        A.n_coarse_commits = p.c_coarse;
        cudaError_t le = cudaErrorUnknown;
        for (int cl = p.coarse_cluster; cl >= 1 && le != cudaSuccess; cl /= 2) {
            cudaLaunchConfig_t lc{};
            lc.gridDim = dim3(cl);
            lc.blockDim = dim3(kCoarseThreads);
            lc.dynamicSmemBytes = smem;
            lc.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cl;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            lc.attrs = at;
            lc.numAttrs = 1;
            le = cudaLaunchKernelEx(&lc, f, A);
            if (le != cudaSuccess) cudaGetLastError();  // cluster too large here: halve it
        }
        if (le != cudaSuccess) return cuda_status(le);
    }
    if (!p.flow_order.empty()) {
        A.n_items = (int32_t)p.flow_order.size();
        sweep_fn f = (p.flow_fast && ks.flow_fast) ? ks.flow_fast : ks.flow;
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, kItemThreads, 0) != cudaSuccess || occ < 1) occ = 1;
        const int grid = std::min(p.flow_grid, occ * num_sms());
        f<<<grid, kItemThreads, 0, st>>>(A);
    }
    if (!p.stages.empty()) {
        stage_fn f = (p.stage_fast && ks.stage_fast) ? ks.stage_fast : ks.stage;
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, kItemThreads, 0) != cudaSuccess || occ < 1) occ = 1;
        for (const StageGroup &G : p.stages) {
            const int units = G.u_off[G.n];
            const int grid = std::max(1, std::min((units + kItemWarps - 1) / kItemWarps, occ * num_sms()));
            f<<<grid, kItemThreads, 0, st>>>(A, G);
        }
    }
    e = cudaGetLastError();
    if (e) return cuda_status(e);
    if (!p.tiles.empty()) {
        const int64_t e0 = (int64_t)p.commits[p.c_tile].item_base * kItemWarps;
        if (p.d.direction == HPEZ_COMPRESS) {
            e = cudaMemsetAsync(p.d_esc_cnt + e0, 0, (size_t)(ne - e0) * sizeof(uint32_t), st);
            if (e) return cuda_status(e);
        }
        TileRun tr{orig, work, codes, outliers, A.outl_cap, p.d_esc_cnt, p.d_esc_off, p.d_counters + 1};
        for (const TilePlan &tp : p.tiles) {
            e = tile_plan_launch(tp, p.d.direction, tr, st);
            if (e) return cuda_status(e);
        }
    }
    if (!p.rows.empty()) {
        const int64_t e0 = (int64_t)p.commits[p.c_tile].item_base * kItemWarps;
        if (p.d.direction == HPEZ_COMPRESS) {
            e = cudaMemsetAsync(p.d_esc_cnt + e0, 0, (size_t)(ne - e0) * sizeof(uint32_t), st);
            if (e) return cuda_status(e);
        }
        for (size_t i = 0; i < p.rows.size(); i++) {
            RowRun rr{};
            rr.orig = (const float *)orig;
            rr.work = (float *)work;
            rr.codes = (uint16_t *)codes;
            rr.outl = outliers;
            rr.outl_cap = A.outl_cap;
            rr.esc_cnt = p.d_esc_cnt;
            rr.esc_off = p.d_esc_off;
            rr.flags = p.d_counters + 1;
            rr.table = p.table.empty() ? nullptr : p.d_table + (size_t)p.row_level[i] * p.nblk_table;
            rr.rowbase = p.rows[i].d_base;
            rr.commits = p.d_commits;
            rr.wbase = p.d_wbase;
            e = row_plan_launch(p.rows[i], p.d.direction, rr, st);
            if (e) return cuda_status(e);
        }
    }
    if (p.d.direction == HPEZ_COMPRESS) {
        exclusive_scan(p.d_esc_cnt, ne, p.d_esc_off, p.d_scan_tmp, p.d_total, st);
        const int64_t thr = (ne + 31) / 32 * 32;
        auto *gk = p.d.work_dtype == HPEZ_WORK_F32
                       ? (p.d.code_dtype == HPEZ_CODES_U16 ? gather_outliers_kernel<float, uint16_t>
                                                           : gather_outliers_kernel<float, int32_t>)
                       : (p.d.code_dtype == HPEZ_CODES_U16 ? gather_outliers_kernel<double, uint16_t>
                                                           : gather_outliers_kernel<double, int32_t>);
        gk<<<(unsigned)((thr + 255) / 256), 256, 0, st>>>(A, ne, outliers, A.outl_cap);
    }
    if (stats && stat_err_sum && !p.commits.empty()) {
        commit_pairwise_kernel<<<(unsigned)p.commits.size(), 256, 0, st>>>(p.d_errbuf, p.d_cbase, p.d_cn, p.d_csum);
        stats_accumulate_kernel<<<1, 32, 0, st>>>((int)p.commits.size(), p.d_clevel, p.d_csum, p.d_cn, stat_err_sum,
                                                  stat_count);
    }
    e = cudaGetLastError();
    if (e) return cuda_status(e);
    p.outl_cap_last = A.outl_cap;
    return HPEZ_OK;
}

int hpez_sweep_run(hpez_plan plan, void *work, void *codes, int64_t codes_avail, double *outliers, int64_t outl_cap,
                   double *stat_err_sum, int64_t *stat_count, double *stat_dense, void *stream) {
    return sweep_run(plan, nullptr, work, codes, codes_avail, outliers, outl_cap, stat_err_sum, stat_count, stat_dense,
                     stream);
}

int hpez_sweep_run_from(hpez_plan plan, const void *orig, void *work, void *codes, int64_t codes_avail,
                        double *outliers, int64_t outl_cap, void *stream) {
    if (!orig) return HPEZ_BAD_ARGUMENT;
    return sweep_run(plan, orig, work, codes, codes_avail, outliers, outl_cap, nullptr, nullptr, nullptr, stream);
}

int hpez_plan_tile_info(hpez_plan plan, int64_t *out, int32_t cap) {
    if (!plan || !out || cap < 1) return HPEZ_BAD_ARGUMENT;
    const Plan &p = plan->p;
    out[0] = (int64_t)p.tiles.size();
    int k = 1, c = p.c_tile;
    for (const TilePlan &t : p.tiles) {
        const int64_t v[8] = {c, t.grid, t.threads, (int64_t)t.smem, t.d.TY, t.d.TX, t.d.ZC, t.d.n_iv};
        for (int i = 0; i < 8 && k < cap; i++) out[k++] = v[i];
        c += t.d.n_commits;
    }
    return HPEZ_OK;
}

int hpez_plan_row_info(hpez_plan plan, int64_t *out) {
    if (!plan || !out) return HPEZ_BAD_ARGUMENT;
    const Plan &p = plan->p;
    out[0] = (int64_t)p.rows.size();
    out[1] = p.rows.empty() ? -1 : p.c_tile;
    int nl = 0;
    int64_t ent = 0, same = 0;
    size_t smem = 0;
    for (const RowPlan &rp : p.rows) {
        nl += rp.n_launch;
        ent += rp.d.n_entries;
        same |= rp.d.any_same;
        smem = std::max(smem, rp.smem);
    }
    out[2] = nl;
    out[3] = ent;
    out[4] = same;
    out[5] = (int64_t)smem;
    return HPEZ_OK;
}

int hpez_sweep_finish(hpez_plan plan, void *stream, int64_t *n_outliers) {
    if (!plan) return HPEZ_BAD_ARGUMENT;
    Plan &p = plan->p;
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e) return cuda_status(e);
    int64_t n_out = 0;
    int32_t flags = 0;
    if (p.setup_done) {
        e = cudaMemcpy(&n_out, p.d_total, sizeof n_out, cudaMemcpyDeviceToHost);
        if (!e) e = cudaMemcpy(&flags, p.d_counters + 1, sizeof flags, cudaMemcpyDeviceToHost);
        if (e) return cuda_status(e);
    }
    if (n_outliers) *n_outliers = n_out;
    if (flags) return flags;
    if (p.d.direction == HPEZ_DECOMPRESS && n_out > p.outl_cap_last) return HPEZ_OUTLIER_UNDERFLOW;
    return HPEZ_OK;
}

}  // extern "C"
