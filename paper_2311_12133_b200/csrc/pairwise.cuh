// pairwise.cuh -- numpy's pairwise float64 sum (numpy/_core/src/umath/
// loops_utils.h.src, pairwise_sum) on the GPU, bit-identical: the same
// recursion tree (blocks of <= 128 summed with 8 accumulators, splits at
// n/2 rounded down to a multiple of 8), evaluated in parallel by one CTA.
// Used for the tuner's reductions that the reference performs with numpy
// (interp.py:274 err sums, tuner.py:470-472 block scores, tuner.py:111-115
// sample MSEs).
#pragma once

#include "common.cuh"

namespace hpez {

// Serial pairwise sum of a[0..n) (explicit stack; the reference's order).
__device__ __forceinline__ double np_pairwise_serial(const double *__restrict__ a, int64_t n) {
    int64_t ls[48], ln[48];
    double vs[48];
    int8_t state[48];
    int top = 1, vt = 0;
    ls[0] = 0;
    ln[0] = n;
    state[0] = 0;
    while (top) {
        const int t = top - 1;
        const int64_t n0 = ln[t];
        if (n0 <= 128) {
            const double *p = a + ls[t];
            double res;
            if (n0 < 8) {
                res = -0.0;
                for (int64_t i = 0; i < n0; i++) res = __dadd_rn(res, p[i]);
            } else {
                double r[8];
#pragma unroll
                for (int j = 0; j < 8; j++) r[j] = p[j];
                int64_t i;
                for (i = 8; i < n0 - (n0 % 8); i += 8) {
#pragma unroll
                    for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], p[i + j]);
                }
                res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                                __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
                for (; i < n0; i++) res = __dadd_rn(res, p[i]);
            }
            vs[vt++] = res;
            top--;
            continue;
        }
        int64_t n2 = n0 / 2;
        n2 -= n2 % 8;
        if (state[t] == 0) {
            state[t] = 1;
            ls[top] = ls[t];
            ln[top] = n2;
            state[top] = 0;
            top++;
        } else if (state[t] == 1) {
            state[t] = 2;
            ls[top] = ls[t] + n2;
            ln[top] = n0 - n2;
            state[top] = 0;
            top++;
        } else {
            const double b = vs[--vt], x = vs[--vt];
            vs[vt++] = __dadd_rn(x, b);
            top--;
        }
    }
    return vs[0];
}

// Parallel evaluation of the same tree by one CTA of 2^D threads (D <= 10):
// thread t follows the path given by the D bits of t (MSB first) and sums
// the subtree it reaches at depth D; a path that hits a leaf (n <= 128)
// earlier is owned by its leftmost thread.  The 2^D partial sums are then
// combined bottom-up, adding a node's children only where the tree has an
// internal node.  Call from every thread of the CTA; returns the sum in
// thread 0.  smem: 2^D doubles + 2^D bytes.
template <int D>
__device__ double np_pairwise_cta(const double *__restrict__ a, int64_t n, double *s_val, int8_t *s_leaf) {
    constexpr int NT = 1 << D;
    const int t = threadIdx.x;
    if (t < NT) {
        int64_t st = 0, len = n;
        int depth = 0;
        bool owner = true;
        for (; depth < D && len > 128; depth++) {
            int64_t n2 = len / 2;
            n2 -= n2 % 8;
            if ((t >> (D - 1 - depth)) & 1) {
                st += n2;
                len -= n2;
            } else {
                len = n2;
            }
        }
        // a leaf reached above depth D belongs to the thread whose remaining bits are 0
        if (depth < D && (t & ((1 << (D - depth)) - 1)) != 0) owner = false;
        s_leaf[t] = (int8_t)(len > 128 ? D + 1 : depth);  // depth at which the path became a leaf
        s_val[t] = owner ? np_pairwise_serial(a + st, len) : 0.0;
    }
    __syncthreads();
    for (int k = 1; k <= D; k++) {
        const int d = D - k;
        const int i = t;
        if (i < (NT >> k)) {
            const int t0 = i << k;
            if (s_leaf[t0] > d) s_val[t0] = __dadd_rn(s_val[t0], s_val[t0 + (1 << (k - 1))]);
        }
        __syncthreads();
    }
    return s_val[0];
}

}  // namespace hpez
