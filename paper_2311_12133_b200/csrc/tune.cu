// tune.cu -- block-table scoring reductions for tuner.tune_blocks
// (tuner.py:461-474): per complete block, numpy's pairwise sum of the dense
// |orig - pred| grid rows (err_grids[li].reshape(n_full, -1).sum(axis=1)).
#include <cstdio>

#include "common.cuh"

namespace hpez {

// numpy pairwise_sum (loops_utils.h) over a[0..n), one thread, explicit stack.
__device__ double np_pairwise(const double *__restrict__ a, int64_t n) {
    int64_t ls[48], ln[48];
    double vs[48];
    int8_t state[48];
    int top = 0, vt = 0;
    ls[0] = 0;
    ln[0] = n;
    state[0] = 0;
    top = 1;
    while (top) {
        const int t = top - 1;
        const int64_t n0 = ln[t];
        if (n0 <= 128) {
            const double *p = a + ls[t];
            double res;
            if (n0 < 8) {
                res = -0.0;
                for (int64_t i = 0; i < n0; i++) res = __dadd_rn(res, __ldg(p + i));
            } else {
                double r[8];
#pragma unroll
                for (int j = 0; j < 8; j++) r[j] = __ldg(p + j);
                int64_t i;
                for (i = 8; i < n0 - (n0 % 8); i += 8) {
#pragma unroll
                    for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], __ldg(p + i + j));
                }
                res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                                __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
                for (; i < n0; i++) res = __dadd_rn(res, __ldg(p + i));
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

__global__ void rows_pairwise_kernel(const double *__restrict__ rows, int64_t nrows, int64_t len,
                                     double *__restrict__ out) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < nrows) out[r] = np_pairwise(rows + r * len, len);
}

}  // namespace hpez

using namespace hpez;

extern "C" int hpez_rows_pairwise_sum(const double *rows, int64_t nrows, int64_t rowlen, double *out,
                                      void *stream) {
    if (nrows < 0 || rowlen < 0 || (nrows > 0 && (!rows || !out))) return HPEZ_BAD_ARGUMENT;
    if (nrows == 0) return HPEZ_OK;
    rows_pairwise_kernel<<<(unsigned)((nrows + 127) / 128), 128, 0, (cudaStream_t)stream>>>(rows, nrows,
                                                                                           rowlen, out);
    cudaError_t e = cudaGetLastError();
    if (e) {
        fprintf(stderr, "hpez_b200: CUDA error %s\n", cudaGetErrorString(e));
        return HPEZ_CUDA_ERROR;
    }
    return HPEZ_OK;
}
