// stencil.cuh -- compile-time 1-D interpolation rows shared by the sweep
// kernels (sweep.cu: item flow kernels; tile.cu: shared-memory level tiles).
// Literal coefficients of kernels.py:43-86 in the reference's left-to-right
// order; every product and sum is a separately rounded f64 operation.
#pragma once

#include "common.cuh"

namespace hpez {

#define DM(a, b) __dmul_rn((a), (b))
#define DA(a, b) __dadd_rn((a), (b))

// 1-D row of family FAM at coordinate c (extent E, stride s, element step sE)
// with every edge truncation of kernels.resolve_row (kernels.py:106-150)
// written out: inter-level cubic rows try (-1,1,3), (-3,-1,1), (-1,1),
// (-3,-1), (-1,); same-level rows (-2,-1,1,2), (-2,-1,1), (-2,-1); a
// truncated 6-point natural row falls back to the 4-point not-a-knot row.
// Edge rows of family FAM at coordinate c (extent E, stride s) over values
// x[] already loaded at the family's nominal offsets (Fam<FAM>::u order),
// with every truncation of kernels.resolve_row (kernels.py:106-150) written
// out: inter-level cubic rows try (-1,1,3), (-3,-1,1), (-1,1), (-3,-1),
// (-1,); same-level rows (-2,-1,1,2), (-2,-1,1), (-2,-1); a truncated
// 6-point natural row falls back to the 4-point not-a-knot row.  Offsets
// outside the grid were loaded from the target itself and are never used.
template <int FAM>
__device__ __forceinline__ double edge_row(const double (&x)[6], int c, int E, int s) {
    const bool r1 = c + s <= E - 1;
    if (FAM == FAM_LIN_I) return r1 ? DA(DM(0.5, x[0]), DM(0.5, x[1])) : DM(1.0, x[0]);
    if (FAM == FAM_NAK_I || FAM == FAM_NAT_I) {
        const double a = x[0], b = x[1], d = x[2], e = x[3];
        const bool l3 = c >= 3 * s, r3 = c + 3 * s <= E - 1;
        if (l3 && r3) {
            if (FAM == FAM_NAK_I)
                return DA(DA(DA(DM(-1.0 / 16, a), DM(9.0 / 16, b)), DM(9.0 / 16, d)), DM(-1.0 / 16, e));
            return DA(DA(DA(DM(-3.0 / 40, a), DM(23.0 / 40, b)), DM(23.0 / 40, d)), DM(-3.0 / 40, e));
        }
        if (r3) return DA(DA(DM(3.0 / 8, b), DM(3.0 / 4, d)), DM(-1.0 / 8, e));
        if (l3 && r1) return DA(DA(DM(-1.0 / 8, a), DM(3.0 / 4, b)), DM(3.0 / 8, d));
        if (r1) return DA(DM(0.5, b), DM(0.5, d));
        if (l3) return DA(DM(-0.5, a), DM(1.5, b));
        return DM(1.0, b);
    }
    // same-level families: targets sit at >= 3s, so only the right side truncates
    constexpr int o = FAM == FAM_NAT_S ? 1 : 0;
    const double b = x[o], d = x[o + 1], e = x[o + 2], f = x[o + 3];
    if (FAM == FAM_NAT_S && c + 3 * s <= E - 1)
        return DA(DA(DA(DA(DA(DM(3.0 / 62, x[0]), DM(-18.0 / 62, b)), DM(46.0 / 62, d)), DM(46.0 / 62, e)),
                     DM(-18.0 / 62, f)), DM(3.0 / 62, x[5]));
    if (c + 2 * s <= E - 1) return DA(DA(DA(DM(-1.0 / 6, b), DM(4.0 / 6, d)), DM(4.0 / 6, e)), DM(-1.0 / 6, f));
    if (r1) return DA(DA(DM(-1.0 / 3, b), DM(1.0, d)), DM(1.0 / 3, e));
    return DA(DM(-1.0, b), DM(2.0, d));
}

// Stencil families at compile time: nominal offsets, interior test and the
// full-row combination in the reference's left-to-right order.
template <int FAM> struct Fam;
template <> struct Fam<FAM_LIN_I> {
    static constexpr int n = 2;
    __device__ static constexpr int u(int i) { return i == 0 ? -1 : 1; }
    __device__ static bool interior(int c, int E, int s) { return c + s <= E - 1; }
    template <typename V> __device__ static double combine(const V (&v)[6]) {
        return DA(DM(0.5, (double)v[0]), DM(0.5, (double)v[1]));
    }
};
template <> struct Fam<FAM_NAK_I> {
    static constexpr int n = 4;
    __device__ static constexpr int u(int i) { return i == 0 ? -3 : i == 1 ? -1 : i == 2 ? 1 : 3; }
    __device__ static bool interior(int c, int E, int s) { return c >= 3 * s && c + 3 * s <= E - 1; }
    template <typename V> __device__ static double combine(const V (&v)[6]) {
        return DA(DA(DA(DM(-1.0 / 16, (double)v[0]), DM(9.0 / 16, (double)v[1])), DM(9.0 / 16, (double)v[2])),
                  DM(-1.0 / 16, (double)v[3]));
    }
};
template <> struct Fam<FAM_NAT_I> {
    static constexpr int n = 4;
    __device__ static constexpr int u(int i) { return i == 0 ? -3 : i == 1 ? -1 : i == 2 ? 1 : 3; }
    __device__ static bool interior(int c, int E, int s) { return c >= 3 * s && c + 3 * s <= E - 1; }
    template <typename V> __device__ static double combine(const V (&v)[6]) {
        return DA(DA(DA(DM(-3.0 / 40, (double)v[0]), DM(23.0 / 40, (double)v[1])), DM(23.0 / 40, (double)v[2])),
                  DM(-3.0 / 40, (double)v[3]));
    }
};
template <> struct Fam<FAM_NAK_S> {
    static constexpr int n = 4;
    __device__ static constexpr int u(int i) { return i == 0 ? -2 : i == 1 ? -1 : i == 2 ? 1 : 2; }
    __device__ static bool interior(int c, int E, int s) { return c + 2 * s <= E - 1; }
    template <typename V> __device__ static double combine(const V (&v)[6]) {
        return DA(DA(DA(DM(-1.0 / 6, (double)v[0]), DM(4.0 / 6, (double)v[1])), DM(4.0 / 6, (double)v[2])),
                  DM(-1.0 / 6, (double)v[3]));
    }
};
template <> struct Fam<FAM_NAT_S> {
    static constexpr int n = 6;
    __device__ static constexpr int u(int i) {
        return i == 0 ? -3 : i == 1 ? -2 : i == 2 ? -1 : i == 3 ? 1 : i == 4 ? 2 : 3;
    }
    __device__ static bool interior(int c, int E, int s) { return c + 3 * s <= E - 1; }
    template <typename V> __device__ static double combine(const V (&v)[6]) {
        return DA(DA(DA(DA(DA(DM(3.0 / 62, (double)v[0]), DM(-18.0 / 62, (double)v[1])), DM(46.0 / 62, (double)v[2])),
                        DM(46.0 / 62, (double)v[3])), DM(-18.0 / 62, (double)v[4])), DM(3.0 / 62, (double)v[5]));
    }
};

}  // namespace hpez
