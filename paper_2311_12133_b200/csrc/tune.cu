// tune.cu -- block-table scoring reductions for tuner.tune_blocks
// (tuner.py:461-474): per complete block, numpy's pairwise sum of the dense
// |orig - pred| grid rows (err_grids[li].reshape(n_full, -1).sum(axis=1)).
#include <cstdio>

#include "common.cuh"
#include "pairwise.cuh"

namespace hpez {

__global__ void rows_pairwise_kernel(const double *__restrict__ rows, int64_t nrows, int64_t len,
                                     double *__restrict__ out) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < nrows) out[r] = np_pairwise_serial(rows + r * len, len);
}

// long rows: one CTA per row (pairwise.cuh)
__global__ void __launch_bounds__(256) rows_pairwise_cta_kernel(const double *__restrict__ rows, int64_t len,
                                                                double *__restrict__ out) {
    __shared__ double s_val[256];
    __shared__ int8_t s_leaf[256];
    const double r = np_pairwise_cta<8>(rows + (int64_t)blockIdx.x * len, len, s_val, s_leaf);
    if (threadIdx.x == 0) out[blockIdx.x] = r;
}

}  // namespace hpez

using namespace hpez;

extern "C" int hpez_rows_pairwise_sum(const double *rows, int64_t nrows, int64_t rowlen, double *out,
                                      void *stream) {
    if (nrows < 0 || rowlen < 0 || (nrows > 0 && (!rows || !out))) return HPEZ_BAD_ARGUMENT;
    if (nrows == 0) return HPEZ_OK;
    if (rowlen > 8192 && nrows < (1ll << 31))
        rows_pairwise_cta_kernel<<<(unsigned)nrows, 256, 0, (cudaStream_t)stream>>>(rows, rowlen, out);
    else
        rows_pairwise_kernel<<<(unsigned)((nrows + 127) / 128), 128, 0, (cudaStream_t)stream>>>(rows, nrows,
                                                                                               rowlen, out);
    cudaError_t e = cudaGetLastError();
    if (e) {
        fprintf(stderr, "hpez_b200: CUDA error %s\n", cudaGetErrorString(e));
        return HPEZ_CUDA_ERROR;
    }
    return HPEZ_OK;
}
