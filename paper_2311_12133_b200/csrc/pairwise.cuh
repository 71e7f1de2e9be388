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

// Element accessors: the summed sequence is a[i], or a function of i.
struct ArrayAt {
    const double *__restrict__ a;
    __device__ __forceinline__ double operator()(int64_t i) const { return a[i]; }
};

// Serial pairwise sum of f(base .. base+n) (explicit stack; the reference's order).
template <typename F>
__device__ __forceinline__ double np_pairwise_serial_f(const F &f, int64_t base, int64_t n) {
    int64_t ls[48], ln[48];
    double vs[48];
    int8_t state[48];
    int top = 1, vt = 0;
    ls[0] = base;
    ln[0] = n;
    state[0] = 0;
    while (top) {
        const int t = top - 1;
        const int64_t n0 = ln[t];
        if (n0 <= 128) {
            const int64_t p = ls[t];
            double res;
            if (n0 < 8) {
                res = -0.0;
                for (int64_t i = 0; i < n0; i++) res = __dadd_rn(res, f(p + i));
            } else {
                double r[8];
#pragma unroll
                for (int j = 0; j < 8; j++) r[j] = f(p + j);
                int64_t i;
                for (i = 8; i < n0 - (n0 % 8); i += 8) {
#pragma unroll
                    for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], f(p + i + j));
                }
                res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                                __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
                for (; i < n0; i++) res = __dadd_rn(res, f(p + i));
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

__device__ __forceinline__ double np_pairwise_serial(const double *__restrict__ a, int64_t n) {
    return np_pairwise_serial_f(ArrayAt{a}, 0, n);
}

// Path of thread t (D bits, MSB first) down the recursion tree of n
// elements: the subtree it sums (start, length), whether it owns it, and
// the depth at which the path became a leaf (D + 1: still internal at D).
template <int D>
__device__ __forceinline__ void np_pairwise_path(int t, int64_t n, int64_t *st, int64_t *len, bool *owner,
                                                 int *leaf_depth) {
    int64_t s0 = 0, l0 = n;
    int depth = 0;
    for (; depth < D && l0 > 128; depth++) {
        int64_t n2 = l0 / 2;
        n2 -= n2 % 8;
        if ((t >> (D - 1 - depth)) & 1) {
            s0 += n2;
            l0 -= n2;
        } else {
            l0 = n2;
        }
    }
    *owner = !(depth < D && (t & ((1 << (D - depth)) - 1)) != 0);
    *leaf_depth = l0 > 128 ? D + 1 : depth;
    *st = s0;
    *len = l0;
}

// Bottom-up combination of 2^D partial sums (s_val) with their leaf depths
// (s_leaf), by the threads of one CTA (any block size).  Result in s_val[0].
template <int D>
__device__ __forceinline__ void np_pairwise_combine(double *s_val, const int8_t *s_leaf) {
    constexpr int NT = 1 << D;
    for (int k = 1; k <= D; k++) {
        const int d = D - k;
        for (int i = threadIdx.x; i < (NT >> k); i += blockDim.x) {
            const int t0 = i << k;
            if (s_leaf[t0] > d) s_val[t0] = __dadd_rn(s_val[t0], s_val[t0 + (1 << (k - 1))]);
        }
        __syncthreads();
    }
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
        int64_t st, len;
        bool owner;
        int ld;
        np_pairwise_path<D>(t, n, &st, &len, &owner, &ld);
        s_leaf[t] = (int8_t)ld;
        s_val[t] = owner ? np_pairwise_serial(a + st, len) : 0.0;
    }
    __syncthreads();
    np_pairwise_combine<D>(s_val, s_leaf);
    return s_val[0];
}

// Grid-wide variant for long sequences: 2^D threads over several CTAs each
// sum one subtree of f(0 .. n) into partial[t] / leaf[t]; a second launch
// (np_pairwise_finish_kernel) combines them.
template <int D, typename F>
__global__ void __launch_bounds__(256) np_pairwise_partials_kernel(F f, int64_t n, double *partial, int8_t *leaf) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (1 << D)) return;
    int64_t st, len;
    bool owner;
    int ld;
    np_pairwise_path<D>(t, n, &st, &len, &owner, &ld);
    leaf[t] = (int8_t)ld;
    partial[t] = owner ? np_pairwise_serial_f(f, st, len) : 0.0;
}

template <int D>
__global__ void __launch_bounds__(1024) np_pairwise_finish_kernel(const double *partial, const int8_t *leaf,
                                                                  double *out) {
    extern __shared__ __align__(16) unsigned char smem[];
    double *s_val = reinterpret_cast<double *>(smem);
    int8_t *s_leaf = reinterpret_cast<int8_t *>(s_val + (1 << D));
    for (int i = threadIdx.x; i < (1 << D); i += blockDim.x) {
        s_val[i] = partial[i];
        s_leaf[i] = leaf[i];
    }
    __syncthreads();
    np_pairwise_combine<D>(s_val, s_leaf);
    if (threadIdx.x == 0) *out = s_val[0];
}

}  // namespace hpez
