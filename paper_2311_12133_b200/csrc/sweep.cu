// sweep.cu -- B200 multi-level interpolation predict/quantize sweep and its
// inverse: the drop-in for interp.run_levels (interp.py:440-472).
//
// Host side: a plan object restates the reference's commit schedule --
// levels coarse to fine, parity classes combinations(active, m) in
// lexicographic order (interp.py:415-433), uniform commits with the optional
// same-level two-phase split (interp.py:322-341) and mixed per-block commits
// A / B_phase (interp.py:350-411) -- and uploads it once.
//
// Device side: one launch per commit.  Each CTA owns a contiguous range of
// lattice positions in row-major order (the order codes and outliers are
// streamed in, interp.py:48-67), predicts every member from pre-commit state
// with the resolved 1-D rows or the MD blend, quantizes / dequantizes in
// f64 and writes the reconstruction in place.  Escapes are ranked with a
// block-wide ballot scan plus a decoupled look-back chained across every
// launch of the sweep, so outliers land in stream order without a second
// pass.  Mixed commits get their member offsets from a data-independent
// setup pass run once per plan.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <set>
#include <vector>

#include "common.cuh"

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
        for (uint32_t m = 0; m < 64; m++) {
            // a target always has its -1 neighbour (position >= stride)
            rows[f][m] = (m < (1u << kFamN[f])) ? resolve(f, m) : RowEntry{};
        }
    }
    cudaError_t e = cudaMemcpyToSymbol(c_rows, rows, sizeof rows);
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_fam, fam, sizeof fam);
    if (e == cudaSuccess) done = true;
    return e;
}

// ------------------------------------------------------ device kernels --
struct SweepPtrs {
    void *work;
    void *codes;
    double *outl;
    int64_t outl_cap;
    uint64_t *status;
    unsigned long long *ticket;
    int32_t *flags;
    const int64_t *blkoff;
    const TagInfo *tags;
    const uint8_t *slots;
    const uint8_t *table;
    double *errbuf;
    double *dense;
};

template <typename T>
__device__ __forceinline__ double predict_1d(const T *__restrict__ work, int64_t idx, int64_t c,
                                             int64_t E, int64_t s, int64_t sE, int fam) {
    const FamDesc &fd = c_fam[fam];
    uint32_t mask = 0;
#pragma unroll
    for (int i = 0; i < 6; i++) {
        if (i < fd.n) {
            int64_t p = c + (int64_t)fd.u[i] * s;
            mask |= (uint32_t)(p >= 0 && p < E) << i;
        }
    }
    const RowEntry &r = c_rows[fam][mask];
    double acc = __dmul_rn(r.coef[0], (double)work[idx + (int64_t)r.off[0] * sE]);
#pragma unroll
    for (int k = 1; k < 6; k++) {
        if (k < r.n)
            acc = __dadd_rn(acc, __dmul_rn(r.coef[k], (double)work[idx + (int64_t)r.off[k] * sE]));
    }
    return acc;
}

template <typename T>
__device__ __forceinline__ double predict(const GridDev &g, const T *__restrict__ work,
                                          int64_t idx, const int32_t (&coord)[kMaxRank],
                                          const PredDev &p, int64_t s) {
    if (!p.md)
        return predict_1d(work, idx, coord[p.axis], g.dims[p.axis], s, s * g.estr[p.axis], p.fam);
    double acc = 0.0;
    for (int i = 0; i < p.nax; i++) {
        const int a = p.axes[i];
        double t = __dmul_rn(p.w[i], predict_1d(work, idx, coord[a], g.dims[a], s, s * g.estr[a], p.fam));
        acc = i == 0 ? t : __dadd_rn(acc, t);
    }
    return acc;
}

template <typename C>
__device__ __forceinline__ int64_t load_code(const C *codes, int64_t i) {
    return (int64_t)codes[i];
}

template <typename T, typename C, int DIR, int ROUND, bool STATS, bool MIXED>
__global__ void __launch_bounds__(kThreads) commit_kernel(const __grid_constant__ GridDev g,
                                                          const __grid_constant__ CommitDev cm,
                                                          const __grid_constant__ SweepPtrs P) {
    __shared__ uint32_t s_rank[kItems * kWarps + 1];
    __shared__ unsigned long long s_ticket;
    __shared__ uint64_t s_excl;
    if (threadIdx.x == 0) s_ticket = atomicAdd(P.ticket, 1ull);
    __syncthreads();
    const uint64_t ticket = s_ticket;
    const uint32_t p0 = (uint32_t)(ticket - cm.blk_base) * (uint32_t)kBlockPos;
    T *__restrict__ work = (T *)P.work;
    C *__restrict__ codes = (C *)P.codes;
    const int64_t R = g.radius;

    int64_t idx[kItems];
    int32_t coord[kItems][kMaxRank];
    bool mem[kItems];
    const PredDev *pp[kItems];
    // pass 1: coordinates and membership
#pragma unroll
    for (int i = 0; i < kItems; i++) {
        const uint32_t pos = p0 + (uint32_t)(i * kThreads) + threadIdx.x;
        mem[i] = pos < cm.npos;
        uint32_t rem = mem[i] ? pos : 0u;
        int64_t id = 0;
        uint32_t jodd = 0;
#pragma unroll
        for (int a = kMaxRank - 1; a >= 0; a--) {
            if (a < g.rank) {
                uint32_t q = fdiv(rem, cm.cnt[a]);
                uint32_t j = rem - q * cm.cnt[a].d;
                rem = q;
                int64_t c = cm.start[a] + (int64_t)j * cm.step[a];
                coord[i][a] = (int32_t)c;
                id += c * g.estr[a];
                jodd |= (j & 1u) << a;
            }
        }
        idx[i] = id;
        pp[i] = &cm.pred;
        if (MIXED && mem[i]) {
            int64_t b = 0;
            for (int a = 0; a < g.rank; a++) b += (int64_t)(coord[i][a] / g.block_size) * g.bstr[a];
            const int tag = P.table[(int64_t)cm.level * g.nblk + b];
            const TagInfo &ti = P.tags[cm.tag_off + P.slots[cm.slot_off + tag]];
            const int sp = ti.split;
            if (cm.kind == COMMIT_MIXED_A) {
                mem[i] = sp < 0 || !((jodd >> sp) & 1u);
                pp[i] = &ti.inter;
            } else {
                int key = __popc(cm.axes_present & jodd & ~(1u << (sp < 0 ? 31 : sp)));
                mem[i] = sp >= 0 && ((jodd >> sp) & 1u) && key == cm.phase;
                pp[i] = &ti.same;
            }
        }
    }
    // pass 2: stream positions of the members
    int64_t ci[kItems];
    if (MIXED) {
        uint32_t r[kItems], tot;
        block_rank(mem, r, tot, s_rank);
        const int64_t base = P.blkoff[ticket];
#pragma unroll
        for (int i = 0; i < kItems; i++) ci[i] = base + r[i];
    } else {
#pragma unroll
        for (int i = 0; i < kItems; i++)
            ci[i] = cm.code_base + (int64_t)(p0 + (uint32_t)(i * kThreads) + threadIdx.x);
    }
    // pass 3: predict + quantize / dequantize
    bool esc[kItems];
    double val[kItems];
#pragma unroll
    for (int i = 0; i < kItems; i++) {
        esc[i] = false;
        val[i] = 0.0;
        if (!mem[i]) continue;
        if (DIR == HPEZ_COMPRESS) {
            const double pred = predict(g, work, idx[i], coord[i], *pp[i], cm.s);
            const double orig = (double)work[idx[i]];
            double out;
            const int64_t code = quantize_point<ROUND>(orig, pred, cm.bound, cm.two_e, R, &out);
            codes[ci[i]] = (C)code;
            esc[i] = code == 0;
            val[i] = orig;
            if (STATS) {
                const double err = fabs(__dsub_rn(orig, pred));
                P.errbuf[ci[i]] = err;
                if (P.dense) P.dense[(int64_t)cm.level * g.npts + idx[i]] = err;
            }
            if (!esc[i]) work[idx[i]] = (T)out;
        } else {
            const int64_t code = load_code(codes, ci[i]);
            if (code == 0) {
                esc[i] = true;
            } else {
                const double pred = predict(g, work, idx[i], coord[i], *pp[i], cm.s);
                work[idx[i]] = (T)dequantize_point<ROUND>(pred, code, cm.two_e, R);
            }
        }
    }
    // pass 4: escapes in stream order (outliers)
    uint32_t er[kItems], etot;
    block_rank(esc, er, etot, s_rank);
    if (threadIdx.x < 32) {
        uint64_t ex = lookback(P.status, ticket, etot);
        if (threadIdx.x == 0) s_excl = ex;
    }
    __syncthreads();
    const int64_t ex = (int64_t)s_excl;
#pragma unroll
    for (int i = 0; i < kItems; i++) {
        if (!esc[i]) continue;
        const int64_t o = ex + er[i];
        if (DIR == HPEZ_COMPRESS) {
            if (o < P.outl_cap) P.outl[o] = val[i];
        } else {
            if (o < P.outl_cap) work[idx[i]] = (T)P.outl[o];
            else atomicExch(P.flags, HPEZ_OUTLIER_UNDERFLOW);
        }
    }
}

// Data-independent member counts of mixed commits (one CTA per block).
__global__ void __launch_bounds__(kThreads) mixed_count_kernel(const GridDev g, const CommitDev cm,
                                                               const uint8_t *table,
                                                               const TagInfo *tags,
                                                               const uint8_t *slots,
                                                               int64_t *blkcnt) {
    __shared__ uint32_t s_rank[kItems * kWarps + 1];
    const uint32_t p0 = blockIdx.x * (uint32_t)kBlockPos;
    bool mem[kItems];
#pragma unroll
    for (int i = 0; i < kItems; i++) {
        const uint32_t pos = p0 + (uint32_t)(i * kThreads) + threadIdx.x;
        mem[i] = pos < cm.npos;
        if (!mem[i]) continue;
        uint32_t rem = pos, jodd = 0;
        int64_t b = 0;
        int32_t coord[kMaxRank];
        for (int a = g.rank - 1; a >= 0; a--) {
            uint32_t q = fdiv(rem, cm.cnt[a]);
            uint32_t j = rem - q * cm.cnt[a].d;
            rem = q;
            coord[a] = (int32_t)(cm.start[a] + (int64_t)j * cm.step[a]);
            jodd |= (j & 1u) << a;
        }
        for (int a = 0; a < g.rank; a++) b += (int64_t)(coord[a] / g.block_size) * g.bstr[a];
        const int tag = table[(int64_t)cm.level * g.nblk + b];
        const int sp = tags[cm.tag_off + slots[cm.slot_off + tag]].split;
        if (cm.kind == COMMIT_MIXED_A) {
            mem[i] = sp < 0 || !((jodd >> sp) & 1u);
        } else {
            int key = __popc(cm.axes_present & jodd & ~(1u << (sp < 0 ? 31 : sp)));
            mem[i] = sp >= 0 && ((jodd >> sp) & 1u) && key == cm.phase;
        }
    }
    uint32_t r[kItems], tot;
    block_rank(mem, r, tot, s_rank);
    if (threadIdx.x == 0) blkcnt[cm.blk_base + blockIdx.x] = tot;
}

// Exclusive scan of block counts over the commits of each mixed class, in
// commit order (A, B_0, B_1, ...).  One CTA per class.
struct ClassScan {
    int64_t class_base;
    int32_t c0, c1;  // commit index range
};

__global__ void __launch_bounds__(1024) mixed_scan_kernel(const ClassScan *cls,
                                                          const int64_t *commit_blk_base,
                                                          const int64_t *commit_nblk,
                                                          const int64_t *blkcnt, int64_t *blkoff,
                                                          int64_t *commit_code_base,
                                                          int64_t *commit_n) {
    __shared__ int64_t s_w[32];
    __shared__ int64_t s_carry;
    const ClassScan c = cls[blockIdx.x];
    if (threadIdx.x == 0) s_carry = c.class_base;
    __syncthreads();
    for (int k = c.c0; k < c.c1; k++) {
        const int64_t b0 = commit_blk_base[k], nb = commit_nblk[k];
        const int64_t start = s_carry;
        for (int64_t off = 0; off < nb; off += blockDim.x) {
            const int64_t i = off + threadIdx.x;
            int64_t v = i < nb ? blkcnt[b0 + i] : 0;
            // block inclusive scan
            int64_t x = v;
            const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
            for (int o = 1; o < 32; o <<= 1) {
                int64_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) s_w[warp] = x;
            __syncthreads();
            if (warp == 0) {
                int64_t w = lane < (int)(blockDim.x >> 5) ? s_w[lane] : 0;
                for (int o = 1; o < 32; o <<= 1) {
                    int64_t y = __shfl_up_sync(0xffffffffu, w, o);
                    if (lane >= o) w += y;
                }
                s_w[lane] = w;
            }
            __syncthreads();
            const int64_t wpre = warp ? s_w[warp - 1] : 0;
            const int64_t carry = s_carry;
            if (i < nb) blkoff[b0 + i] = carry + wpre + x - v;
            __syncthreads();
            if (threadIdx.x == blockDim.x - 1) s_carry = carry + wpre + x;
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            commit_code_base[k] = start;
            commit_n[k] = s_carry - start;
        }
        __syncthreads();
    }
}

// numpy pairwise sum (loops_utils.h pairwise_sum) of each commit's member
// errors, leaves in parallel, tree folded by one thread in recursion order.
__device__ double leaf_sum(const double *a, int64_t n) {
    if (n < 8) {
        double r = -0.0;
        for (int64_t i = 0; i < n; i++) r = __dadd_rn(r, a[i]);
        return r;
    }
    double r[8];
    for (int j = 0; j < 8; j++) r[j] = a[j];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
        for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], a[i + j]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; i++) res = __dadd_rn(res, a[i]);
    return res;
}

__global__ void commit_pairwise_kernel(const double *errbuf, const int64_t *commit_code_base,
                                       const int64_t *commit_n, double *commit_sum,
                                       double *leafbuf, const int64_t *leaf_off) {
    const int c = blockIdx.x;
    const int64_t base = commit_code_base[c], n = commit_n[c];
    double *leaves = leafbuf + leaf_off[c];
    // Leaves left to right (pairwise splits until n <= 128), then the fold in
    // the same recursion order.  Trial commits are small (<= ~35K members).
    if (n == 0) {
        if (threadIdx.x == 0) commit_sum[c] = 0.0;
        return;
    }
    int64_t leaf = 0;
    if (threadIdx.x == 0) {
        int64_t ls[64], ln[64];
        int top = 0;
        ls[0] = 0;
        ln[0] = n;
        top = 1;
        while (top) {
            top--;
            const int64_t s0 = ls[top], n0 = ln[top];
            if (n0 <= 128) {
                leaves[leaf++] = leaf_sum(errbuf + base + s0, n0);
                continue;
            }
            int64_t n2 = n0 / 2;
            n2 -= n2 % 8;
            ls[top] = s0 + n2;  // right child visited second
            ln[top] = n0 - n2;
            top++;
            ls[top] = s0;
            ln[top] = n2;
            top++;
        }
        // fold in the same recursion order
        double vs[64];
        int64_t fs[64], fn[64];
        int32_t state[64];
        int vt = 0;
        top = 0;
        fs[0] = 0;
        fn[0] = n;
        state[0] = 0;
        top = 1;
        int64_t li = 0;
        while (top) {
            const int t = top - 1;
            if (fn[t] <= 128) {
                vs[vt++] = leaves[li++];
                top--;
                continue;
            }
            int64_t n2 = fn[t] / 2;
            n2 -= n2 % 8;
            if (state[t] == 0) {
                state[t] = 1;
                fs[top] = fs[t];
                fn[top] = n2;
                state[top] = 0;
                top++;
            } else if (state[t] == 1) {
                state[t] = 2;
                fs[top] = fs[t] + n2;
                fn[top] = fn[t] - n2;
                state[top] = 0;
                top++;
            } else {
                const double b = vs[--vt], a = vs[--vt];
                vs[vt++] = __dadd_rn(a, b);
                top--;
            }
        }
        commit_sum[c] = vs[0];
    }
}

__global__ void stats_accumulate_kernel(int n_commits, const int32_t *commit_level,
                                        const double *commit_sum, const int64_t *commit_n,
                                        double *err_sum, int64_t *count) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int c = 0; c < n_commits; c++) {
        if (commit_n[c] == 0) continue;  // empty commits are never recorded
        err_sum[commit_level[c]] = __dadd_rn(err_sum[commit_level[c]], commit_sum[c]);
        count[commit_level[c]] += commit_n[c];
    }
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
    std::vector<ClassScan> classes;
    bool has_mixed = false;
    int64_t total_blocks = 0;
    int64_t num_codes = 0;
    int64_t leaf_total = 0;
    std::vector<int64_t> level_codes;

    // device
    uint64_t *d_status = nullptr;
    unsigned long long *d_counters = nullptr;  // [0] ticket, [1] flags
    int64_t *d_blkoff = nullptr;
    int64_t *d_blkcnt = nullptr;
    TagInfo *d_tags = nullptr;
    uint8_t *d_slots = nullptr;
    uint8_t *d_table = nullptr;
    ClassScan *d_classes = nullptr;
    int64_t *d_cblk = nullptr, *d_cnblk = nullptr, *d_cbase = nullptr, *d_cn = nullptr;
    int32_t *d_clevel = nullptr;
    double *d_errbuf = nullptr, *d_csum = nullptr, *d_leaves = nullptr;
    int64_t *d_leafoff = nullptr;
    bool setup_done = false;
    int64_t outl_cap_last = 0;
    int direction = 0;

    ~Plan() {
        void *ptrs[] = {d_status, d_counters, d_blkoff, d_blkcnt, d_tags, d_slots, d_table,
                        d_classes, d_cblk, d_cnblk, d_cbase, d_cn, d_clevel, d_errbuf,
                        d_csum, d_leaves, d_leafoff};
        for (void *p : ptrs)
            if (p) cudaFree(p);
    }

    // plan.order_candidates (plan.py:37-51)
    std::vector<std::vector<int>> order_candidates() const {
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
        int64_t npos = 1;
        for (int a = 0; a < d.rank; a++) {
            c.start[a] = start[a];
            c.step[a] = step[a];
            c.cnt[a] = make_fastdiv((uint32_t)count[a]);
            npos *= count[a];
        }
        for (int a = d.rank; a < kMaxRank; a++) c.cnt[a] = make_fastdiv(1);
        c.npos = (uint32_t)npos;
        c.nblocks = (uint32_t)((npos + kBlockPos - 1) / kBlockPos);
        c.blk_base = total_blocks;
        total_blocks += c.nblocks;
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
            g.dims[a] = d.dims[a];
            g.estr[a] = n;
            n *= d.dims[a];
        }
        g.npts = n;
        if (n >= (1ll << 31)) return HPEZ_BAD_ARGUMENT;  // per-field limit of this build
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
                g.bstr[a] = nb;
                nb *= (d.dims[a] + d.block_size - 1) / d.block_size;
            }
            nblk_table = nb;
            g.nblk = nb;
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
                        int st = use_tbl ? add_class_table(li, lc, v, start, step, count, tot, &code_pos)
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
        return HPEZ_OK;
    }

    int add_class_table(int li, const Cfg &, const std::vector<int> &v, const int64_t *start,
                        const int64_t *step, const int64_t *count, int64_t tot, int64_t *code_pos) {
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
        // mixed class
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
        ClassScan cs{};
        cs.class_base = *code_pos;
        cs.c0 = (int)commits.size();
        const int nph = __builtin_popcount(axes_present);
        for (int ph = -1; ph < nph; ph++) {
            CommitDev cm = base_commit(li, start, step, count);
            cm.kind = ph < 0 ? COMMIT_MIXED_A : COMMIT_MIXED_B;
            cm.phase = ph < 0 ? 0 : ph;
            cm.axes_present = axes_present;
            cm.tag_off = tag_off;
            cm.slot_off = slot_off;
            cm.code_base = -1;
            commits.push_back(cm);
        }
        cs.c1 = (int)commits.size();
        classes.push_back(cs);
        *code_pos += tot;
        return 0;
    }
};

template <typename T>
static cudaError_t dalloc(T **p, size_t n) {
    if (n == 0) n = 1;
    return cudaMalloc((void **)p, n * sizeof(T));
}

template <typename T>
static cudaError_t dupload(T **p, const std::vector<T> &v) {
    cudaError_t e = dalloc(p, v.size());
    if (e == cudaSuccess && !v.empty()) e = cudaMemcpy(*p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
    return e;
}

static int cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return HPEZ_OK;
    fprintf(stderr, "hpez_b200: CUDA error %s\n", cudaGetErrorString(e));
    return HPEZ_CUDA_ERROR;
}

typedef void (*commit_fn)(const GridDev, const CommitDev, const SweepPtrs);

template <typename T, typename C, int DIR, int ROUND>
static commit_fn pick3(bool stats, bool mixed) {
    if (DIR == HPEZ_COMPRESS && stats)
        return mixed ? commit_kernel<T, C, DIR, ROUND, true, true> : commit_kernel<T, C, DIR, ROUND, true, false>;
    return mixed ? commit_kernel<T, C, DIR, ROUND, false, true> : commit_kernel<T, C, DIR, ROUND, false, false>;
}

template <typename T, typename C>
static commit_fn pick2(int dir, int round, bool stats, bool mixed) {
    if (dir == HPEZ_COMPRESS) {
        if (round == HPEZ_ROUND_F32) return pick3<T, C, HPEZ_COMPRESS, HPEZ_ROUND_F32>(stats, mixed);
        if (round == HPEZ_ROUND_INT) return pick3<T, C, HPEZ_COMPRESS, HPEZ_ROUND_INT>(stats, mixed);
        return pick3<T, C, HPEZ_COMPRESS, HPEZ_ROUND_NONE>(stats, mixed);
    }
    if (round == HPEZ_ROUND_F32) return pick3<T, C, HPEZ_DECOMPRESS, HPEZ_ROUND_F32>(false, mixed);
    if (round == HPEZ_ROUND_INT) return pick3<T, C, HPEZ_DECOMPRESS, HPEZ_ROUND_INT>(false, mixed);
    return pick3<T, C, HPEZ_DECOMPRESS, HPEZ_ROUND_NONE>(false, mixed);
}

static commit_fn pick(const hpez_sweep_desc &d, bool mixed) {
    const bool stats = d.with_stats != 0;
    if (d.work_dtype == HPEZ_WORK_F32) {
        if (d.code_dtype == HPEZ_CODES_U16) return pick2<float, uint16_t>(d.direction, d.rounding, stats, mixed);
        return pick2<float, int32_t>(d.direction, d.rounding, stats, mixed);
    }
    if (d.code_dtype == HPEZ_CODES_U16) return pick2<double, uint16_t>(d.direction, d.rounding, stats, mixed);
    return pick2<double, int32_t>(d.direction, d.rounding, stats, mixed);
}

static int plan_setup(Plan *p, cudaStream_t st) {
    // device metadata, once per plan
    cudaError_t e = cudaSuccess;
    const size_t nb = (size_t)std::max<int64_t>(p->total_blocks, 1);
    e = dalloc(&p->d_status, nb);
    if (!e) e = dalloc(&p->d_counters, 4);
    if (!e) e = dalloc(&p->d_blkoff, nb);
    if (!e && p->has_mixed) e = dalloc(&p->d_blkcnt, nb);
    if (!e) e = dupload(&p->d_tags, p->tags);
    if (!e) e = dupload(&p->d_slots, p->slots);
    if (!e) e = dupload(&p->d_table, p->table);
    if (!e) e = dupload(&p->d_classes, p->classes);
    const size_t nc = p->commits.size();
    std::vector<int64_t> cblk(nc), cnblk(nc), cbase(nc), cn(nc);
    std::vector<int32_t> clevel(nc);
    for (size_t i = 0; i < nc; i++) {
        cblk[i] = p->commits[i].blk_base;
        cnblk[i] = p->commits[i].nblocks;
        cbase[i] = p->commits[i].code_base;
        cn[i] = p->commits[i].kind == COMMIT_UNIFORM ? (int64_t)p->commits[i].npos : 0;
        clevel[i] = p->commits[i].level;
    }
    if (!e) e = dupload(&p->d_cblk, cblk);
    if (!e) e = dupload(&p->d_cnblk, cnblk);
    if (!e) e = dupload(&p->d_cbase, cbase);
    if (!e) e = dupload(&p->d_cn, cn);
    if (!e) e = dupload(&p->d_clevel, clevel);
    if (e) return cuda_status(e);
    if (p->has_mixed) {
        for (const CommitDev &cm : p->commits) {
            if (cm.kind == COMMIT_UNIFORM) continue;
            mixed_count_kernel<<<cm.nblocks, kThreads, 0, st>>>(p->g, cm, p->d_table, p->d_tags,
                                                                p->d_slots, p->d_blkcnt);
        }
        mixed_scan_kernel<<<(unsigned)p->classes.size(), 1024, 0, st>>>(
            p->d_classes, p->d_cblk, p->d_cnblk, p->d_blkcnt, p->d_blkoff, p->d_cbase, p->d_cn);
        e = cudaGetLastError();
        if (e) return cuda_status(e);
    }
    if (p->d.with_stats && p->d.direction == HPEZ_COMPRESS) {
        // leaf offsets per commit (upper bound n/64 + 1 leaves each)
        std::vector<int64_t> loff(nc + 1, 0);
        int64_t tot = 0;
        for (size_t i = 0; i < nc; i++) {
            loff[i] = tot;
            tot += (int64_t)p->commits[i].npos / 64 + 2;
        }
        loff[nc] = tot;
        p->leaf_total = tot;
        e = dupload(&p->d_leafoff, loff);
        if (!e) e = dalloc(&p->d_leaves, (size_t)tot);
        if (!e) e = dalloc(&p->d_csum, nc);
        if (!e) e = dalloc(&p->d_errbuf, (size_t)std::max<int64_t>(p->num_codes, 1));
        if (e) return cuda_status(e);
    }
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
    if (desc->rank < 1 || desc->rank > kMaxRank || desc->n_levels < 0 ||
        (desc->n_levels > 0 && !desc->levels))
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
    *out = h.release();
    return HPEZ_OK;
}

int hpez_plan_destroy(hpez_plan plan) {
    delete plan;
    return HPEZ_OK;
}

int64_t hpez_plan_num_codes(hpez_plan plan) { return plan ? plan->p.num_codes : -1; }
int32_t hpez_plan_num_commits(hpez_plan plan) { return plan ? (int32_t)plan->p.commits.size() : -1; }
int32_t hpez_plan_num_launches(hpez_plan plan) { return plan ? (int32_t)plan->p.commits.size() : -1; }

int hpez_plan_level_codes(hpez_plan plan, int64_t *out) {
    if (!plan || !out) return HPEZ_BAD_ARGUMENT;
    for (size_t i = 0; i < plan->p.level_codes.size(); i++) out[i] = plan->p.level_codes[i];
    return HPEZ_OK;
}

int hpez_set_device(int32_t device) { return cuda_status(cudaSetDevice(device)); }

const char *hpez_build_info(void) { return "libhpez_b200 sm_100a f64 -fmad=false"; }

int hpez_sweep_run(hpez_plan plan, void *work, void *codes, int64_t codes_avail, double *outliers,
                   int64_t outl_cap, double *stat_err_sum, int64_t *stat_count, double *stat_dense,
                   void *stream) {
    if (!plan || !work) return HPEZ_BAD_ARGUMENT;
    Plan &p = plan->p;
    cudaStream_t st = (cudaStream_t)stream;
    if (p.d.direction == HPEZ_DECOMPRESS && codes_avail < p.num_codes) return HPEZ_CORRUPT_STREAM;
    if (p.num_codes > 0 && !codes) return HPEZ_BAD_ARGUMENT;
    if (p.d.with_stats && p.d.direction == HPEZ_COMPRESS && (!stat_err_sum || !stat_count))
        return HPEZ_BAD_ARGUMENT;
    if (!p.setup_done) {
        int s = plan_setup(&p, st);
        if (s) return s;
    }
    cudaError_t e = cudaMemsetAsync(p.d_status, 0, sizeof(uint64_t) * std::max<int64_t>(p.total_blocks, 1), st);
    if (!e) e = cudaMemsetAsync(p.d_counters, 0, 4 * sizeof(unsigned long long), st);
    if (e) return cuda_status(e);
    SweepPtrs P{};
    P.work = work;
    P.codes = codes;
    P.outl = outliers;
    P.outl_cap = outliers ? outl_cap : 0;
    P.status = p.d_status;
    P.ticket = p.d_counters;
    P.flags = (int32_t *)(p.d_counters + 1);
    P.blkoff = p.d_blkoff;
    P.tags = p.d_tags;
    P.slots = p.d_slots;
    P.table = p.d_table;
    P.errbuf = p.d_errbuf;
    P.dense = stat_dense;
    const commit_fn fu = pick(p.d, false), fm = pick(p.d, true);
    for (const CommitDev &cm : p.commits) {
        commit_fn f = cm.kind == COMMIT_UNIFORM ? fu : fm;
        f<<<cm.nblocks, kThreads, 0, st>>>(p.g, cm, P);
    }
    e = cudaGetLastError();
    if (e) return cuda_status(e);
    if (p.d.with_stats && p.d.direction == HPEZ_COMPRESS && !p.commits.empty()) {
        commit_pairwise_kernel<<<(unsigned)p.commits.size(), 32, 0, st>>>(
            p.d_errbuf, p.d_cbase, p.d_cn, p.d_csum, p.d_leaves, p.d_leafoff);
        stats_accumulate_kernel<<<1, 32, 0, st>>>((int)p.commits.size(), p.d_clevel, p.d_csum,
                                                  p.d_cn, stat_err_sum, stat_count);
        e = cudaGetLastError();
        if (e) return cuda_status(e);
    }
    p.outl_cap_last = P.outl_cap;
    return HPEZ_OK;
}

int hpez_sweep_finish(hpez_plan plan, void *stream, int64_t *n_outliers) {
    if (!plan) return HPEZ_BAD_ARGUMENT;
    Plan &p = plan->p;
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e) return cuda_status(e);
    int64_t n_out = 0;
    int32_t flags = 0;
    if (p.total_blocks > 0 && p.setup_done) {
        uint64_t last = 0;
        e = cudaMemcpy(&last, p.d_status + p.total_blocks - 1, sizeof last, cudaMemcpyDeviceToHost);
        if (!e) e = cudaMemcpy(&flags, p.d_counters + 1, sizeof flags, cudaMemcpyDeviceToHost);
        if (e) return cuda_status(e);
        n_out = (int64_t)(last & kValMask);
    }
    if (n_outliers) *n_outliers = n_out;
    if (flags) return flags;
    if (p.d.direction == HPEZ_DECOMPRESS && n_out > p.outl_cap_last) return HPEZ_OUTLIER_UNDERFLOW;
    return HPEZ_OK;
}

}  // extern "C"
