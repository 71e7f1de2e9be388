// coarse.cu -- the leading (small) levels of a rank-3 uniform sweep held
// entirely in the distributed shared memory of one thread-block cluster.
//
// The coarse levels (interp._LevelRunner.run_level, interp.py:415-433, for
// the first few strides) touch only the stride-Sc sublattice, Sc = stride
// of the last coarse level: 73,728 points on cfg2.  As f64 that is a few
// hundred KB, so the cluster keeps all of it on chip: CTA r owns the
// sublattice z-planes [r*P, (r+1)*P) in its shared memory.  The commits of
// one (level, DAG depth) group are independent; every CTA computes the
// group's points in its own planes (stencil reads along y and x are local,
// along z they go to the owning CTA over DSMEM) and groups are separated by
// cluster barriers -- no global-memory round trip between groups.  Codes
// and reconstructions stay in shared memory until the last group and are
// written to global memory once.
#include <algorithm>
#include <cstdlib>
#include <utility>
#include <vector>

#include "stencil.cuh"
#include "tile.h"

namespace hpez {

__device__ __forceinline__ uint32_t cl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// f64 at shared-memory address `la` (this CTA's layout) in CTA `rank`
__device__ __forceinline__ double ld_dsmem(uint32_t la, uint32_t rank) {
    uint32_t ra;
    double v;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rank));
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra) : "memory");
    return v;
}

template <int KIND> __device__ constexpr int ck_axis(int t) {
    return KIND < 3 ? KIND : KIND == 3 ? (t == 0 ? 0 : 1) : KIND == 4 ? (t == 0 ? 0 : 2) : KIND == 5 ? (t == 0 ? 1 : 2) : t;
}

// Outlier of the zero code at position pos of commit cm.  The coarse levels
// are the stream prefix [0, n_cc), so the rank is the number of zero codes
// before the point's stream index: a per-CTA prefix over 256-code chunks
// (zpre) plus a scan inside the chunk.  Independent of the decompress
// pre-pass, which therefore runs concurrently on a side stream.
constexpr int kCoarseZChunk = 256;
__device__ __noinline__ double coarse_outlier(const CoarseCommit &cm, const TileRun &A, int64_t pos,
                                              const uint32_t *zpre) {
    const int64_t q = cm.code_base + pos;
    const uint16_t *codes = (const uint16_t *)A.codes;
    const int64_t c = q / kCoarseZChunk;
    int64_t r = zpre[c];
    for (int64_t k = c * kCoarseZChunk; k < q; k++) r += codes[k] == 0;
    if (r < A.outl_cap) return A.outl[r];
    atomicExch(A.flags, HPEZ_OUTLIER_UNDERFLOW);
    return 0.0;
}

struct CoarseCtx {
    int z0, z1, P, L1, L2, L0;
    uint32_t sbase;  // shared address of this CTA's slab
};

// One point of commit cm at sublattice (z, y, x), slab index li.
template <int DIR, int KIND, int FAM>
__device__ __forceinline__ void coarse_point(const CoarseDesc &D, const CoarseCtx &X, const TileRun &A, double *slab,
                                             uint16_t *ccode, const CoarseCommit &cm, int z, int y, int x, int li,
                                             int64_t pos, const uint32_t *zpre) {
    constexpr int NAX = KIND < 3 ? 1 : KIND < 6 ? 2 : 3;
    constexpr int NF = Fam<FAM>::n;
    const int s = cm.s;
    const int crd[3] = {z, y, x};
    const int Lv[3] = {X.L0, X.L1, X.L2};
    double v[NAX][6];
    bool in_all = true;
#pragma unroll
    for (int t = 0; t < NAX; t++) {
        const int a = ck_axis<KIND>(t);
        in_all &= Fam<FAM>::interior(crd[a], Lv[a], s);
#pragma unroll
        for (int i = 0; i < NF; i++) {
            const int u = Fam<FAM>::u(i) * s;
            if (a == 0) {
                int zz = z + u;
                zz = zz < 0 ? 0 : (zz >= X.L0 ? X.L0 - 1 : zz);  // clamped rows are never used
                const uint32_t owner = fdiv((uint32_t)zz, D.fd_P);
                const uint32_t la = X.sbase + (uint32_t)((((zz - (int)owner * X.P) * X.L1 + y) * X.L2 + x) * 8);
                v[t][i] = ld_dsmem(la, owner);
            } else if (a == 1) {
                int yy = y + u;
                yy = yy < 0 ? 0 : (yy >= X.L1 ? X.L1 - 1 : yy);
                v[t][i] = slab[li + (yy - y) * X.L2];
            } else {
                int xx = x + u;
                xx = xx < 0 ? 0 : (xx >= X.L2 ? X.L2 - 1 : xx);
                v[t][i] = slab[li + (xx - x)];
            }
        }
    }
    double pt[NAX];
#pragma unroll
    for (int t = 0; t < NAX; t++) {
        const int a = ck_axis<KIND>(t);
        pt[t] = in_all || Fam<FAM>::interior(crd[a], Lv[a], s) ? Fam<FAM>::combine(v[t])
                                                                : edge_row<FAM>(v[t], crd[a], Lv[a], s);
    }
    double pred;
    if (NAX == 1) pred = pt[0];
    else if (NAX == 2) pred = DA(DM(cm.w[0], pt[0]), DM(cm.w[1], pt[NAX - 1]));
    else pred = DA(DA(DM(cm.w[0], pt[0]), DM(cm.w[1], pt[1])), DM(cm.w[2], pt[NAX - 1]));
    const int gidx = D.Sc * (z * D.E0 + y * D.E1 + x);
    const int32_t R = D.R;
    if (DIR == HPEZ_COMPRESS) {
        double out;
        const int32_t code = quantize_point<HPEZ_ROUND_F32>(slab[li], pred, cm.bound, cm.two_e, cm.inv_two_e,
                                                            (double)R, R, &out);
        slab[li] = out;
        ccode[li] = (uint16_t)code;  // written out after the last group
        if (code == 0) {
            const int64_t item = pos / cm.p_item;
            const int64_t w = (pos - item * cm.p_item) / cm.pw;
            atomicAdd(A.esc_cnt + (int64_t)(cm.item_base + item) * kItemWarps + w, 1u);
        }
    } else {
        const int64_t code = (int64_t)__double_as_longlong(slab[li]);
        const double val = code != 0 ? dequantize_point<HPEZ_ROUND_F32>(pred, code, cm.two_e, (int64_t)R)
                                     : (double)(float)coarse_outlier(cm, A, pos, zpre);
        slab[li] = val;
    }
    (void)gidx;
}

template <int DIR>
__device__ __forceinline__ void coarse_dispatch(const CoarseDesc &D, const CoarseCtx &X, const TileRun &A, double *slab,
                                                uint16_t *ccode, const CoarseCommit &cm, int z, int y, int x, int li,
                                                int64_t pos, const uint32_t *zpre) {
#define HPEZ_CK(K, F)                                                      \
    case K * 5 + F:                                                        \
        coarse_point<DIR, K, F>(D, X, A, slab, ccode, cm, z, y, x, li, pos, zpre); \
        return;
    switch (cm.kind * 5 + cm.fam) {
        HPEZ_CK(0, 0) HPEZ_CK(0, 1) HPEZ_CK(0, 2) HPEZ_CK(0, 3) HPEZ_CK(0, 4)
        HPEZ_CK(1, 0) HPEZ_CK(1, 1) HPEZ_CK(1, 2) HPEZ_CK(1, 3) HPEZ_CK(1, 4)
        HPEZ_CK(2, 0) HPEZ_CK(2, 1) HPEZ_CK(2, 2) HPEZ_CK(2, 3) HPEZ_CK(2, 4)
        HPEZ_CK(3, 0) HPEZ_CK(3, 1) HPEZ_CK(3, 2)
        HPEZ_CK(4, 0) HPEZ_CK(4, 1) HPEZ_CK(4, 2)
        HPEZ_CK(5, 0) HPEZ_CK(5, 1) HPEZ_CK(5, 2)
        HPEZ_CK(6, 0) HPEZ_CK(6, 1) HPEZ_CK(6, 2)
    default:
        break;
    }
#undef HPEZ_CK
}

// Commit index of the sublattice point (z, y, x), or -1 for an anchor.
__device__ __forceinline__ int coarse_commit_of(const CoarseDesc &D, int z, int y, int x) {
    for (int l = 0; l < D.n_levels; l++) {
        const int s = D.lvl_s[l], h = D.lvl_sh[l];
        if ((z | y | x) & (s - 1)) continue;  // not on this level's lattice
        const int r = (((z >> h) & 3) << 4) | (((y >> h) & 3) << 2) | ((x >> h) & 3);
        const int c = D.lut[l][r];
        if (c >= 0) return c;
    }
    return -1;
}

template <int DIR>
__global__ void __launch_bounds__(kCoarseDsmemThreads, 1) coarse_dsmem_kernel(const __grid_constant__ CoarseDesc D,
                                                                              const TileRun A) {
    extern __shared__ __align__(16) double slab[];
    CoarseCtx X;
    const int rank = (int)cl_rank();
    X.P = D.P;
    X.L0 = D.L[0];
    X.L1 = D.L[1];
    X.L2 = D.L[2];
    X.z0 = rank * D.P;
    X.z1 = min(X.z0 + D.P, X.L0);
    X.sbase = (uint32_t)__cvta_generic_to_shared(slab);
    const int plane = X.L1 * X.L2;
    const int nloc = max(0, X.z1 - X.z0) * plane;
    uint16_t *ccode = reinterpret_cast<uint16_t *>(slab + (size_t)D.P * plane);
    const float *orig = (const float *)A.orig;
    const float *work = (const float *)A.work;
    const uint16_t *codes = (const uint16_t *)A.codes;
    // load the slab: originals (compress) / anchors + codes (decompress)
    // per-CTA commit ranges: lattice planes in [z0, z1), point counts and
    // their prefix within the commit's group
    int32_t *c_iz0 = reinterpret_cast<int32_t *>((reinterpret_cast<uintptr_t>(ccode + (size_t)D.P * plane) + 15) &
                                                 ~(uintptr_t)15);
    int32_t *c_n = c_iz0 + kCoarseMaxCommits, *c_pre = c_n + kCoarseMaxCommits;
    uint32_t *c_zpre = reinterpret_cast<uint32_t *>(c_pre + kCoarseMaxCommits);  // decompress: zero-code prefix per chunk
    const int nzc = (D.n_cc + kCoarseZChunk - 1) / kCoarseZChunk;
    if (DIR == HPEZ_DECOMPRESS) {
        const int wq = threadIdx.x >> 5, ln = threadIdx.x & 31;
        for (int c = wq; c < nzc; c += (int)(blockDim.x >> 5)) {
            uint32_t z = 0;
            for (int k = c * kCoarseZChunk + ln; k < min((c + 1) * kCoarseZChunk, D.n_cc); k += 32)
                z += ((const uint16_t *)A.codes)[k] == 0;
            for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
            if (ln == 0) c_zpre[c + 1] = z;
        }
    }
    if ((int)threadIdx.x < D.n_commits) {
        const CoarseCommit &cm = D.c[threadIdx.x];
        const int iz0 = X.z0 <= cm.st[0] ? 0 : (X.z0 - cm.st[0] + cm.sp[0] - 1) >> cm.sh[0];
        const int iz1 = X.z1 - 1 < cm.st[0] ? -1 : min((X.z1 - 1 - cm.st[0]) >> cm.sh[0], cm.cnt[0] - 1);
        c_iz0[threadIdx.x] = iz0;
        c_n[threadIdx.x] = max(0, iz1 - iz0 + 1) * cm.cnt[1] * cm.cnt[2];
    }
    __syncthreads();
    if (DIR == HPEZ_DECOMPRESS && threadIdx.x == blockDim.x - 1) {  // exclusive prefix (runs beside the group prefix)
        c_zpre[0] = 0;
        for (int c = 1; c <= nzc; c++) c_zpre[c] += c_zpre[c - 1];
    }
    if (threadIdx.x < D.n_groups) {
        int acc = 0;
        for (int c = D.grp_off[threadIdx.x]; c < D.grp_off[threadIdx.x + 1]; c++) {
            c_pre[c] = acc;
            acc += c_n[c];
        }
    }
    for (int i = threadIdx.x; i < nloc; i += blockDim.x) {
        const int zl = (int)fdiv((uint32_t)i, D.fd_plane), r = i - zl * plane;
        const int y = (int)fdiv((uint32_t)r, D.fd_x), x = r - y * X.L2, z = X.z0 + zl;
        const int g = D.Sc * (z * D.E0 + y * D.E1 + x);
        if (DIR == HPEZ_COMPRESS) {
            slab[i] = (double)__ldg(orig + g);
        } else {
            const int c = coarse_commit_of(D, z, y, x);
            if (c < 0) {
                slab[i] = (double)__ldg(work + g);
            } else {
                const CoarseCommit &cm = D.c[c];
                const int64_t pos = ((int64_t)((z - cm.st[0]) >> cm.sh[0]) * cm.cnt[1] + ((y - cm.st[1]) >> cm.sh[1])) *
                                        cm.cnt[2] + ((x - cm.st[2]) >> cm.sh[2]);
                slab[i] = __longlong_as_double((long long)__ldg(codes + cm.code_base + pos));
            }
        }
    }
    cl_sync();
    for (int gi = 0; gi < D.n_groups; gi++) {
        // the group's points in this CTA's planes, flattened over its commits
        const int cg0 = D.grp_off[gi], cg1 = D.grp_off[gi + 1];
        const int total = c_pre[cg1 - 1] + c_n[cg1 - 1];
        for (int t = threadIdx.x; t < total; t += blockDim.x) {
            int c = cg0;
            while (t >= c_pre[c] + c_n[c]) c++;
            const CoarseCommit &cm = D.c[c];
            const int tt = t - c_pre[c];
            const int izr = (int)fdiv((uint32_t)tt, cm.fd_row), r = tt - izr * cm.fd_row.d;
            const int iz = c_iz0[c] + izr;
            const int iy = (int)fdiv((uint32_t)r, cm.fd_x), ix = r - iy * cm.cnt[2];
            const int z = cm.st[0] + (iz << cm.sh[0]), y = cm.st[1] + (iy << cm.sh[1]), x = cm.st[2] + (ix << cm.sh[2]);
            const int li = ((z - X.z0) * X.L1 + y) * X.L2 + x;
            const int64_t pos = ((int64_t)iz * cm.cnt[1] + iy) * cm.cnt[2] + ix;
            coarse_dispatch<DIR>(D, X, A, slab, ccode, cm, z, y, x, li, pos, c_zpre);
        }
        cl_sync();
    }
    // every point of the slab is final: write reconstructions (and codes)
    // out once, so no group barrier waits on outstanding global stores
    for (int i = threadIdx.x; i < nloc; i += blockDim.x) {
        const int zl = (int)fdiv((uint32_t)i, D.fd_plane), r = i - zl * plane;
        const int y = (int)fdiv((uint32_t)r, D.fd_x), x = r - y * X.L2, z = X.z0 + zl;
        const int c = coarse_commit_of(D, z, y, x);
        if (c < 0) continue;  // anchor
        const int g = D.Sc * (z * D.E0 + y * D.E1 + x);
        ((float *)A.work)[g] = (float)slab[i];
        if (DIR == HPEZ_COMPRESS) {
            const CoarseCommit &cm = D.c[c];
            const int64_t pos = ((int64_t)((z - cm.st[0]) >> cm.sh[0]) * cm.cnt[1] + ((y - cm.st[1]) >> cm.sh[1])) *
                                    cm.cnt[2] + ((x - cm.st[2]) >> cm.sh[2]);
            ((uint16_t *)A.codes)[cm.code_base + pos] = ccode[i];
        }
    }
}

bool coarse_dsmem_build(const GridDev &g, const CommitDev *cms, const int *group, int n, int64_t n_codes,
                        CoarsePlan *out) {
    if (g.rank != 3 || n <= 0 || n > kCoarseMaxCommits) return false;
    CoarseDesc D{};
    // sublattice of the last (finest) coarse level
    int Sc = cms[n - 1].s;
    for (int i = 0; i < n; i++) Sc = std::min(Sc, cms[i].s);
    D.Sc = Sc;
    for (int a = 0; a < 3; a++) D.L[a] = (g.dims[a] - 1) / Sc + 1;
    D.E0 = g.estr[0];
    D.E1 = g.estr[1];
    D.R = (int32_t)g.radius;
    D.n_codes = n_codes;
    D.n_commits = n;
    // groups must be contiguous and increasing in commit order
    std::vector<int> order(n);
    for (int i = 0; i < n; i++) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return group[a] < group[b]; });
    int ng = 0;
    for (int k = 0; k < n; k++) {
        const int i = order[k];
        if (k == 0 || group[i] != group[order[k - 1]]) {
            if (ng >= kCoarseMaxGroups) return false;
            D.grp_off[ng++] = k;
        }
        const CommitDev &c = cms[i];
        if (c.kind != COMMIT_UNIFORM || c.s % Sc) return false;
        CoarseCommit &t = D.c[k];
        for (int a = 0; a < 3; a++) {
            if (c.start[a] % Sc || c.step[a] % Sc || c.step[a] == 0) return false;
            t.st[a] = c.start[a] / Sc;
            t.sp[a] = c.step[a] / Sc;
            t.cnt[a] = c.cnt[a];
            if (t.sp[a] & (t.sp[a] - 1)) return false;
            t.sh[a] = __builtin_ctz((unsigned)t.sp[a]);
        }
        t.fd_row = make_fastdiv((uint32_t)(c.cnt[1] * c.cnt[2]));
        t.fd_x = make_fastdiv((uint32_t)c.cnt[2]);
        t.s = c.s / Sc;
        t.fam = c.pred.fam;
        int nax = 1, axes[3] = {c.pred.axis, 0, 0};
        if (c.pred.md) {
            nax = c.pred.nax;
            for (int q = 0; q < nax; q++) {
                axes[q] = c.pred.axes[q];
                t.w[q] = c.pred.w[q];
            }
        }
        if (nax > 1 && t.fam > FAM_NAT_I) return false;
        t.kind = nax == 1 ? axes[0] : nax == 3 ? 6 : (axes[0] == 0 ? (axes[1] == 1 ? 3 : 4) : 5);
        t.bound = c.bound;
        t.two_e = c.two_e;
        t.inv_two_e = c.inv_two_e;
        t.code_base = c.code_base;
        t.item_base = c.item_base;
        t.p_item = c.p_item;
        t.pw = c.pw;
    }
    D.n_groups = ng;
    D.grp_off[ng] = n;
    // per-level residue luts (decompress code preload)
    std::vector<int> lv_s;
    for (int k = 0; k < n; k++) {
        const int s = D.c[k].s;
        if (std::find(lv_s.begin(), lv_s.end(), s) == lv_s.end()) lv_s.push_back(s);
    }
    std::sort(lv_s.begin(), lv_s.end(), std::greater<int>());
    if ((int)lv_s.size() > kCoarseMaxLevels) return false;
    D.n_levels = (int)lv_s.size();
    for (int l = 0; l < D.n_levels; l++) {
        D.lvl_s[l] = lv_s[l];
        if (lv_s[l] & (lv_s[l] - 1)) return false;
        D.lvl_sh[l] = __builtin_ctz((unsigned)lv_s[l]);
        for (int r = 0; r < 64; r++) D.lut[l][r] = -1;
        for (int k = 0; k < n; k++) {
            const CoarseCommit &t = D.c[k];
            if (t.s != lv_s[l]) continue;
            for (int r = 0; r < 64; r++) {
                const int rr[3] = {r >> 4, (r >> 2) & 3, r & 3};
                bool in = true;
                for (int a = 0; a < 3; a++) {
                    const int st = t.st[a] / t.s, sp = t.sp[a] / t.s;  // lattice in level units
                    in &= ((rr[a] - st) % sp + sp) % sp == 0 && (sp == 2 || sp == 4);
                }
                if (in) {
                    if (D.lut[l][r] >= 0) return false;
                    D.lut[l][r] = (int8_t)k;
                }
            }
        }
    }
    // cluster: up to 16 CTAs, P planes each, slab within shared memory
    int ncta = 16;
    if (const char *e = getenv("HPEZ_COARSE_CLUSTER")) ncta = std::max(1, std::min(16, atoi(e)));
    ncta = std::min(ncta, D.L[0]);
    D.P = (D.L[0] + ncta - 1) / ncta;
    ncta = (D.L[0] + D.P - 1) / D.P;
    D.fd_plane = make_fastdiv((uint32_t)(D.L[1] * D.L[2]));
    D.fd_x = make_fastdiv((uint32_t)D.L[2]);
    D.fd_P = make_fastdiv((uint32_t)D.P);
    int64_t ncc = 0;
    for (int k = 0; k < n; k++) ncc = std::max<int64_t>(ncc, D.c[k].code_base + (int64_t)D.c[k].cnt[0] * D.c[k].cnt[1] * D.c[k].cnt[2]);
    for (int k = 0; k < n; k++) if (D.c[k].code_base < 0) return false;
    if (ncc >= (1ll << 30)) return false;
    // the in-kernel outlier ranking counts zero codes over [0, n_cc): the coarse commits' code
    // ranges must tile that stream prefix exactly, in order
    {
        std::vector<std::pair<int64_t, int64_t>> rng;  // (first code, codes) of every coarse commit
        for (int k = 0; k < n; k++)
            rng.push_back({D.c[k].code_base, (int64_t)D.c[k].cnt[0] * D.c[k].cnt[1] * D.c[k].cnt[2]});
        std::sort(rng.begin(), rng.end());
        int64_t pos = 0;
        for (const auto &r : rng) {
            if (r.first != pos) return false;
            pos += r.second;
        }
        if (pos != ncc) return false;
    }
    D.n_cc = (int32_t)ncc;
    const size_t smem = (size_t)D.P * D.L[1] * D.L[2] * (sizeof(double) + sizeof(uint16_t)) + 16 +
                        3 * kCoarseMaxCommits * sizeof(int32_t) +
                        (size_t)((ncc + kCoarseZChunk - 1) / kCoarseZChunk + 1) * sizeof(uint32_t);
    if (smem > 200 * 1024) return false;
    // the cluster must be schedulable here (non-portable sizes, MIG slices)
    {
        auto f = coarse_dsmem_kernel<HPEZ_COMPRESS>;
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(smem, 1));
        cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(ncta);
        lc.blockDim = dim3(kCoarseDsmemThreads);
        lc.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = ncta;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, f, &lc) != cudaSuccess || nclusters < 1) {
            cudaGetLastError();
            return false;
        }
    }
    out->d = D;
    out->ncta = ncta;
    out->smem = smem;
    return true;
}

template <int DIR>
static cudaError_t coarse_launch_dir(const CoarsePlan &p, const TileRun &r, cudaStream_t st) {
    auto f = coarse_dsmem_kernel<DIR>;
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(p.smem, 1));
    if (!e) e = cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e) return e;
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(p.ncta);
    lc.blockDim = dim3(kCoarseDsmemThreads);
    lc.dynamicSmemBytes = p.smem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = p.ncta;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    return cudaLaunchKernelEx(&lc, f, p.d, r);
}

cudaError_t coarse_dsmem_launch(const CoarsePlan &p, int dir, const TileRun &r, cudaStream_t st) {
    return dir == HPEZ_COMPRESS ? coarse_launch_dir<HPEZ_COMPRESS>(p, r, st) : coarse_launch_dir<HPEZ_DECOMPRESS>(p, r, st);
}

}  // namespace hpez
