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

#ifndef HPEZ_ITEM_WARPS
#define HPEZ_ITEM_WARPS 8
#endif
constexpr int kMaxRank = HPEZ_MAX_RANK;
constexpr int kItemWarps = HPEZ_ITEM_WARPS;  // warps per work item
constexpr int kItemThreads = kItemWarps * 32;

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
    int32_t dims[kMaxRank];
    int32_t estr[kMaxRank];     // element strides
    int32_t bstr[kMaxRank];     // block-grid strides (row-major block index)
    int32_t bs_log2;            // log2(block_size) when it is a power of two, else -1
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
    int32_t start[kMaxRank];
    int32_t step[kMaxRank];
    int32_t cnt[kMaxRank];
    FastDiv fd[kMaxRank];
    uint32_t npos;
    int32_t s;
    double bound;
    double two_e;
    double inv_two_e;           // fl(1 / two_e), quantizer fast path
    int64_t code_base;          // uniform commits: code index of position 0
    int32_t item_base;          // first global item id
    int32_t n_items;
    int32_t p_item;             // positions per item (multiple of 256)
    int32_t pw;                 // positions per warp (p_item / 8)
    int32_t tag_off;            // mixed: TagInfo slot 0 of the class
    int32_t slot_off;           // mixed: 256-entry tag->slot map
    int32_t commit_id;
    int32_t fast_id;            // rank-3 uniform specialisation; -2 = mixed fast path; -1 = generic
    PredDev pred;               // uniform commits; mixed: the class's MD blend weights
    uint8_t tdesc[64];          // mixed fast path: tag -> (split axis + 1) << 6 | fast_id
};

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

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
// The quotient x = (orig - pred) / (2e) is formed as a product with the
// reciprocal.  Its error is a few ulps of |x| + 0.5 (< 2^-30 absolute when
// |x| + 0.5 < 2^20), so k = floor(|x| + 0.5) can only differ from the
// correctly rounded division when the fraction lies within 2^-20 of an
// integer, or when |x| + 0.5 >= 2^20 -- then the exact IEEE division decides.
template <int ROUND>
__device__ __forceinline__ int32_t quantize_point(double orig, double pred, double bound, double two_e,
                                                  double inv_two_e, double Rd, int32_t R, double *out) {
    double recon;
    bool ok;
    int32_t code;
    if (bound > 0.0) {
        const double d = __dsub_rn(orig, pred);
        double x = __dmul_rn(d, inv_two_e);
        const double y = __dadd_rn(fabs(x), 0.5);
        double fl = floor(y);
        const double fr = __dsub_rn(y, fl);
        if (fr < 0x1p-20 || fr > 1.0 - 0x1p-20 || y >= 0x1p20) {
            x = __ddiv_rn(d, two_e);
            fl = floor(__dadd_rn(fabs(x), 0.5));
        }
        double k = x > 0.0 ? fl : (x < 0.0 ? -fl : 0.0);  // np.sign(x) * fl
        const bool inr = fabs(k) < Rd;
        if (!inr) k = 0.0;
        recon = round_native<ROUND>(__dadd_rn(pred, __dmul_rn(two_e, k)));
        ok = inr && (fabs(__dsub_rn(recon, orig)) <= bound);
        code = ok ? (int32_t)k + R : 0;
    } else {
        recon = round_native<ROUND>(pred);
        ok = recon == orig;
        code = ok ? R : 0;
    }
    *out = ok ? recon : orig;
    return code;
}

// 64-bit-radius-free wrapper kept for the generic path
template <int ROUND>
__device__ __forceinline__ int64_t quantize_point(double orig, double pred, double bound, double two_e,
                                                  double inv_two_e, int64_t R, double *out) {
    return quantize_point<ROUND>(orig, pred, bound, two_e, inv_two_e, (double)R, (int32_t)R, out);
}

// quant.dequantize_block for a non-escape code (quant.py:115-121).
template <int ROUND>
__device__ __forceinline__ double dequantize_point(double pred, int64_t code, double two_e,
                                                   int64_t R) {
    const double k = (double)(code - R);
    return round_native<ROUND>(__dadd_rn(pred, __dmul_rn(two_e, k)));
}

// ------------------------------------------------------ memory ordering --
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t *p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

}  // namespace hpez
