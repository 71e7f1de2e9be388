// common.cuh -- shared device helpers for the B200 HPEZ kernels.
//
// Arithmetic contract: every floating-point step is a
// separately rounded IEEE f64 operation in the reference's order.  The library
// is compiled with -fmad=false and the hot spots use explicit __d*_rn
// intrinsics so no product/sum pair is ever contracted into an FMA.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "hpez_b200.h"

namespace hpez {

constexpr int kMaxRank = HPEZ_MAX_RANK;
constexpr int kThreads = 256;          // threads per commit CTA
constexpr int kItems = 4;              // lattice positions per thread
constexpr int kBlockPos = kThreads * kItems;
constexpr int kWarps = kThreads / 32;

// ------------------------------------------------------------ fast divmod --
// Division of u32 by a runtime constant (dividends < 2^31).
struct FastDiv {
    uint32_t d, mul, shr;
};

inline FastDiv make_fastdiv(uint32_t d) {
    FastDiv f;
    f.d = d;
    if (d <= 1) {
        f.mul = 0;
        f.shr = 0;
        return f;
    }
    uint32_t L = 0;  // ceil(log2 d)
    while ((1ull << L) < d) L++;
    const uint32_t p = 31 + L;
    f.mul = (uint32_t)(((1ull << p) + d - 1) / d);
    f.shr = p - 32;
    return f;
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv &f) {
    return f.d <= 1 ? n : (__umulhi(n, f.mul) >> f.shr);
}

// ------------------------------------------------------------- row table --
// Stencil families: nominal offsets of the 1-D rows (interp.py:37-45):
// 0 linear inter, 1 not-a-knot inter, 2 natural inter, 3 not-a-knot
// same-level, 4 natural same-level.  The resolved row for each in-bounds
// subset (kernels.resolve_row, kernels.py:106-150) lives in constant memory,
// indexed by the availability bitmask over the family's nominal offsets.
enum { FAM_LIN_I = 0, FAM_NAK_I = 1, FAM_NAT_I = 2, FAM_NAK_S = 3, FAM_NAT_S = 4 };
constexpr int kFamilies = 5;

struct RowEntry {
    int32_t n;
    int32_t off[6];
    double coef[6];
};

struct FamDesc {
    int32_t n;
    int32_t u[6];
};

// ------------------------------------------------------ geometry structs --
struct PredDev {            // one predictor of a member
    int32_t md;             // 0: 1-D along `axis`; 1: blend over `axes`
    int32_t axis;
    int32_t fam;
    int32_t nax;
    int32_t axes[kMaxRank];
    double w[kMaxRank];
};

struct TagInfo {            // per block tag of a mixed class (interp.py:350-411)
    PredDev inter;          // commit A prediction (tag_pred)
    PredDev same;           // commit B prediction (same-level along split)
    int32_t split;          // split axis or -1
    int32_t pad;
};

struct GridDev {
    int32_t rank;
    int32_t block_size;
    int64_t dims[kMaxRank];
    int64_t estr[kMaxRank];     // element strides
    int64_t bstr[kMaxRank];     // block-grid strides (row-major block index)
    int64_t npts;
    int64_t nblk;               // blocks per table level
    int64_t radius;
};

enum { COMMIT_UNIFORM = 0, COMMIT_MIXED_A = 1, COMMIT_MIXED_B = 2 };

struct CommitDev {
    int32_t kind;
    int32_t level;
    int32_t phase;
    uint32_t axes_present;      // mixed: split axes P
    int64_t start[kMaxRank];
    int64_t step[kMaxRank];
    FastDiv cnt[kMaxRank];
    uint32_t npos;
    uint32_t nblocks;
    int64_t s;
    double bound;
    double two_e;
    int64_t code_base;          // uniform commits: first code index
    int64_t blk_base;           // first ticket of this launch
    int32_t tag_off;            // mixed: TagInfo slot 0 of the class
    int32_t slot_off;           // mixed: 256-entry tag->slot map
    int32_t commit_id;
    int32_t pad;
    PredDev pred;               // uniform commits
};

// ------------------------------------------------------------- quantizer --
template <int ROUND>
__device__ __forceinline__ double round_native(double v) {
    // quant.round_native (quant.py:72-77)
    if (ROUND == HPEZ_ROUND_F32) return (double)__double2float_rn(v);
    if (ROUND == HPEZ_ROUND_INT) return rint(v);
    return v;
}

// quant.quantize_block for one point (quant.py:80-105).  Returns the code;
// *out is the decompressor-visible value (recon, or orig on escape).
template <int ROUND>
__device__ __forceinline__ int64_t quantize_point(double orig, double pred, double bound,
                                                  double two_e, int64_t R, double *out) {
    double recon;
    bool ok;
    int64_t code;
    if (bound > 0.0) {
        double x = __ddiv_rn(__dsub_rn(orig, pred), two_e);
        double fl = floor(__dadd_rn(fabs(x), 0.5));
        double k = x > 0.0 ? fl : (x < 0.0 ? -fl : 0.0);  // np.sign(x) * fl
        bool inr = fabs(k) < (double)R;
        if (!inr) k = 0.0;
        recon = round_native<ROUND>(__dadd_rn(pred, __dmul_rn(two_e, k)));
        ok = inr && (fabs(__dsub_rn(recon, orig)) <= bound);
        code = ok ? (int64_t)k + R : 0;
    } else {
        recon = round_native<ROUND>(pred);
        ok = recon == orig;
        code = ok ? R : 0;
    }
    *out = ok ? recon : orig;
    return code;
}

// quant.dequantize_block for a non-escape code (quant.py:115-121).
template <int ROUND>
__device__ __forceinline__ double dequantize_point(double pred, int64_t code, double two_e,
                                                   int64_t R) {
    double k = (double)(code - R);
    return round_native<ROUND>(__dadd_rn(pred, __dmul_rn(two_e, k)));
}

// ----------------------------------------------------- block-wide ranking --
// Exclusive ranks of flags ordered (item, thread) -- i.e. lattice position
// order p = base + i*kThreads + tid -- and the block total.  smem needs
// kItems*kWarps + 1 words.
__device__ __forceinline__ void block_rank(const bool (&f)[kItems], uint32_t (&rank)[kItems],
                                           uint32_t &total, uint32_t *smem) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < kItems; i++) {
        uint32_t m = __ballot_sync(0xffffffffu, f[i]);
        rank[i] = __popc(m & lt);
        if (lane == 0) smem[i * kWarps + warp] = __popc(m);
    }
    __syncthreads();
    static_assert(kItems * kWarps <= 32, "single-warp scan");
    if (warp == 0) {
        uint32_t v = lane < kItems * kWarps ? smem[lane] : 0u;
        uint32_t inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane < kItems * kWarps) smem[lane] = inc - v;
        if (lane == 31) smem[kItems * kWarps] = inc;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kItems; i++) rank[i] += smem[i * kWarps + warp];
    total = smem[kItems * kWarps];
    __syncthreads();
}

// ------------------------------------------------- decoupled look-back --
// Ticket-ordered prefix of per-block counts across every launch of a sweep.
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagInc = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t ld_volatile(const uint64_t *p) {
    return *(const volatile uint64_t *)p;
}
__device__ __forceinline__ void st_volatile(uint64_t *p, uint64_t v) {
    *(volatile uint64_t *)p = v;
}

// Called by all lanes of one warp.  Returns the exclusive prefix of block
// `ticket` and publishes its inclusive value.
__device__ __forceinline__ uint64_t lookback(uint64_t *status, uint64_t ticket, uint64_t agg) {
    const int lane = threadIdx.x & 31;
    if (ticket == 0) {
        if (lane == 0) st_volatile(&status[0], kFlagInc | agg);
        return 0;
    }
    if (lane == 0) st_volatile(&status[ticket], kFlagAgg | agg);
    uint64_t excl = 0;
    int64_t pos = (int64_t)ticket - 1;
    while (true) {
        int64_t q = pos - lane;
        uint64_t w = kFlagInc;
        if (q >= 0) {
            do {
                w = ld_volatile(&status[q]);
            } while ((w >> 62) == 0);
        }
        uint32_t inc = __ballot_sync(0xffffffffu, (w >> 62) == 2);
        uint64_t v = w & kValMask;
        if (inc) {
            int k = __ffs(inc) - 1;
            if (lane > k) v = 0;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (inc) break;
        pos -= 32;
    }
    __threadfence();
    if (lane == 0) st_volatile(&status[ticket], kFlagInc | (excl + agg));
    return excl;
}

}  // namespace hpez
