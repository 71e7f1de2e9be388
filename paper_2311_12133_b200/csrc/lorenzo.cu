// lorenzo.cu -- Lorenzo raster predictor with inline quantization on the GPU:
// the drop-in for lorenzo.lorenzo_pass (lorenzo.py:145-179).
//
// The reference is a sequential raster scan (numba, lorenzo.py:44-135): every
// point reads already-reconstructed backward neighbours.  All stencil offsets
// are >= 0 per axis and non-zero, so points on one hyperplane sum(coords) = d
// are independent: the scan becomes one launch per hyperplane, each thread
// evaluating its point with the reference's term order and quantizer.  Codes
// land at their raster index; outliers are compacted afterwards in raster
// order (compress) or scattered beforehand (decompress) with a chunked
// count / scan / rank pass, so the wavefront never needs an outlier cursor.
#include <algorithm>
#include <cstdio>
#include <vector>

#include "common.cuh"

namespace hpez {

constexpr int kLzMaxTerms = 80;  // 3^4 - 1
constexpr int kLzChunk = 4096;

struct LzStencil {
    int32_t n;
    int32_t pad;
    int8_t delta[kLzMaxTerms][4];
    int64_t flat[kLzMaxTerms];
    double coef[kLzMaxTerms];
};

__constant__ LzStencil c_lz;

struct LzGeom {
    int64_t dims[4];   // padded to rank 4 (leading 1s)
    int64_t estr[4];
    int64_t n;
    double bound, two_e;
    int64_t radius;
};

template <typename T, typename C, int DIR, int ROUND>
__global__ void __launch_bounds__(128) lorenzo_plane_kernel(const LzGeom g, int64_t d, T *__restrict__ work,
                                                            C *__restrict__ codes) {
    const int64_t w = blockIdx.z, z = blockIdx.y;
    const int64_t s = d - w - z;
    if (s < 0) return;
    const int64_t ylo = s - (g.dims[3] - 1) > 0 ? s - (g.dims[3] - 1) : 0;
    const int64_t yhi = s < g.dims[2] - 1 ? s : g.dims[2] - 1;
    const int64_t y = ylo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (y > yhi) return;
    const int64_t x = s - y;
    const int64_t c[4] = {w, z, y, x};
    const int64_t i = w * g.estr[0] + z * g.estr[1] + y * g.estr[2] + x;
    int64_t code = 0;
    if (DIR == HPEZ_DECOMPRESS) {
        code = (int64_t)codes[i];
        if (code == 0) return;  // outlier already scattered into work
    }
    double acc = 0.0;
    for (int t = 0; t < c_lz.n; t++) {
        bool ok = true;
#pragma unroll
        for (int a = 0; a < 4; a++) ok &= c[a] >= c_lz.delta[t][a];
        if (ok) acc = __dadd_rn(acc, __dmul_rn(c_lz.coef[t], (double)work[i - c_lz.flat[t]]));
    }
    const int64_t R = g.radius;
    if (DIR == HPEZ_COMPRESS) {
        // _scan_compress (lorenzo.py:60-88)
        const double orig = (double)work[i];
        if (g.bound > 0.0) {
            const double q = __ddiv_rn(__dsub_rn(orig, acc), g.two_e);
            double kq = floor(__dadd_rn(fabs(q), 0.5));
            if (q < 0.0) kq = -kq;
            if (-(double)R < kq && kq < (double)R) {
                const double recon = round_native<ROUND>(__dadd_rn(acc, __dmul_rn(g.two_e, kq)));
                if (fabs(__dsub_rn(recon, orig)) <= g.bound) {
                    code = (int64_t)kq + R;
                    work[i] = (T)recon;
                }
            }
        } else {
            const double recon = round_native<ROUND>(acc);
            if (recon == orig) {
                code = R;
                work[i] = (T)recon;
            }
        }
        codes[i] = (C)code;
    } else {
        // _scan_decompress (lorenzo.py:117-128)
        work[i] = (T)round_native<ROUND>(__dadd_rn(acc, __dmul_rn(g.two_e, (double)(code - R))));
    }
}

template <typename C>
__global__ void __launch_bounds__(256) zero_count_kernel(const C *__restrict__ codes, int64_t n,
                                                         uint64_t *__restrict__ cnt) {
    __shared__ uint32_t s[8];
    const int64_t base = (int64_t)blockIdx.x * kLzChunk;
    uint32_t k = 0;
    for (int j = threadIdx.x; j < kLzChunk; j += 256) {
        const int64_t i = base + j;
        k += i < n && codes[i] == 0;
    }
    for (int o = 16; o > 0; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = k;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < 8; w++) t += s[w];
        cnt[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(1024) lz_scan_kernel(uint64_t *v, int64_t n, uint64_t *total) {
    __shared__ uint64_t s_w[32];
    __shared__ uint64_t s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t off = 0; off < n; off += blockDim.x) {
        const int64_t i = off + threadIdx.x;
        const uint64_t x0 = i < n ? v[i] : 0;
        uint64_t x = x0;
        for (int o = 1; o < 32; o <<= 1) {
            uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_w[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint64_t w = lane < (int)(blockDim.x >> 5) ? s_w[lane] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            s_w[lane] = w;
        }
        __syncthreads();
        const uint64_t carry = s_carry;
        const uint64_t pre = (warp ? s_w[warp - 1] : 0) + x - x0;
        if (i < n) v[i] = carry + pre;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) s_carry = carry + pre + x0;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = s_carry;
}

// gather (compress: outl[r] = work[i]) or scatter (decompress: work[i] =
// outl[r]) for every zero code, r = raster-order rank.
template <typename T, typename C, bool GATHER>
__global__ void __launch_bounds__(256) zero_move_kernel(const C *__restrict__ codes, int64_t n,
                                                        const uint64_t *__restrict__ off, T *work,
                                                        double *outl, int64_t cap, int32_t *flag) {
    __shared__ uint32_t s_w[8];
    __shared__ uint32_t s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kLzChunk;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int j0 = 0; j0 < kLzChunk; j0 += 256) {
        const int64_t i = base + j0 + threadIdx.x;
        const bool z = i < n && codes[i] == 0;
        const uint32_t m = __ballot_sync(0xffffffffu, z);
        if (lane == 0) s_w[warp] = __popc(m);
        __syncthreads();
        uint32_t pre = s_carry;
        for (int w = 0; w < warp; w++) pre += s_w[w];
        pre += __popc(m & ((1u << lane) - 1u));
        if (z) {
            const int64_t r = (int64_t)off[blockIdx.x] + pre;
            if (GATHER) {
                if (r < cap) outl[r] = (double)work[i];
            } else {
                if (r < cap) work[i] = (T)outl[r];
                else atomicExch(flag, HPEZ_OUTLIER_UNDERFLOW);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t t = 0;
            for (int w = 0; w < 8; w++) t += s_w[w];
            s_carry += t;
        }
        __syncthreads();
    }
}

static int lz_cuda(cudaError_t e) {
    if (e == cudaSuccess) return HPEZ_OK;
    fprintf(stderr, "hpez_b200: CUDA error %s\n", cudaGetErrorString(e));
    return HPEZ_CUDA_ERROR;
}

template <typename T, typename C>
static int lorenzo_run(const LzGeom &g, int direction, int rounding, T *work, C *codes, double *outl,
                       int64_t outl_cap, int64_t *n_outl, cudaStream_t st) {
    const int64_t nchunks = (g.n + kLzChunk - 1) / kLzChunk;
    uint64_t *cnt = nullptr;
    int32_t *flag = nullptr;
    cudaError_t e = cudaMallocAsync((void **)&cnt, sizeof(uint64_t) * (size_t)(nchunks + 1), st);
    if (!e) e = cudaMallocAsync((void **)&flag, sizeof(int32_t), st);
    if (!e) e = cudaMemsetAsync(flag, 0, sizeof(int32_t), st);
    if (e) return lz_cuda(e);
    auto compact = [&](bool gather) {
        zero_count_kernel<C><<<(unsigned)nchunks, 256, 0, st>>>(codes, g.n, cnt);
        lz_scan_kernel<<<1, 1024, 0, st>>>(cnt, nchunks, cnt + nchunks);
        if (gather)
            zero_move_kernel<T, C, true><<<(unsigned)nchunks, 256, 0, st>>>(codes, g.n, cnt, work, outl,
                                                                           outl_cap, flag);
        else
            zero_move_kernel<T, C, false><<<(unsigned)nchunks, 256, 0, st>>>(codes, g.n, cnt, work, outl,
                                                                            outl_cap, flag);
    };
    if (direction == HPEZ_DECOMPRESS) compact(false);
    const int64_t planes = g.dims[0] + g.dims[1] + g.dims[2] + g.dims[3] - 3;
    const dim3 grid((unsigned)((g.dims[2] + 127) / 128), (unsigned)g.dims[1], (unsigned)g.dims[0]);
    typedef void (*fn_t)(const LzGeom, int64_t, T *, C *);
    fn_t f;
    if (direction == HPEZ_COMPRESS)
        f = rounding == HPEZ_ROUND_F32 ? lorenzo_plane_kernel<T, C, HPEZ_COMPRESS, HPEZ_ROUND_F32>
          : rounding == HPEZ_ROUND_INT ? lorenzo_plane_kernel<T, C, HPEZ_COMPRESS, HPEZ_ROUND_INT>
                                       : lorenzo_plane_kernel<T, C, HPEZ_COMPRESS, HPEZ_ROUND_NONE>;
    else
        f = rounding == HPEZ_ROUND_F32 ? lorenzo_plane_kernel<T, C, HPEZ_DECOMPRESS, HPEZ_ROUND_F32>
          : rounding == HPEZ_ROUND_INT ? lorenzo_plane_kernel<T, C, HPEZ_DECOMPRESS, HPEZ_ROUND_INT>
                                       : lorenzo_plane_kernel<T, C, HPEZ_DECOMPRESS, HPEZ_ROUND_NONE>;
    for (int64_t d = 0; d < planes; d++) f<<<grid, 128, 0, st>>>(g, d, work, codes);
    if (direction == HPEZ_COMPRESS) compact(true);
    e = cudaGetLastError();
    uint64_t total = 0;
    int32_t fl = 0;
    if (!e) e = cudaMemcpyAsync(&total, cnt + nchunks, sizeof total, cudaMemcpyDeviceToHost, st);
    if (!e) e = cudaMemcpyAsync(&fl, flag, sizeof fl, cudaMemcpyDeviceToHost, st);
    if (!e) e = cudaStreamSynchronize(st);
    cudaFreeAsync(cnt, st);
    cudaFreeAsync(flag, st);
    if (e) return lz_cuda(e);
    *n_outl = (int64_t)total;
    if (fl) return fl;
    if (direction == HPEZ_DECOMPRESS && (int64_t)total > outl_cap) return HPEZ_OUTLIER_UNDERFLOW;
    return HPEZ_OK;
}

}  // namespace hpez

using namespace hpez;

extern "C" int hpez_lorenzo(int32_t rank, const int64_t *dims, int32_t work_dtype, void *work, double bound,
                            int64_t radius, int32_t order, int32_t direction, int32_t rounding,
                            int32_t code_dtype, void *codes, int64_t n_codes, double *outliers,
                            int64_t outl_cap, int64_t *n_outliers, void *stream) {
    if (rank < 1 || rank > 4 || (order != 1 && order != 2) || !dims || !work || !n_outliers)
        return HPEZ_BAD_ARGUMENT;
    if (direction != HPEZ_COMPRESS && direction != HPEZ_DECOMPRESS) return HPEZ_BAD_ARGUMENT;
    if (radius < 1 || radius > (1ll << 30)) return HPEZ_BAD_ARGUMENT;
    if (code_dtype == HPEZ_CODES_U16 && radius > 32768) return HPEZ_BAD_ARGUMENT;
    LzGeom g{};
    int64_t n = 1;
    for (int a = 0; a < 4; a++) g.dims[a] = 1;
    for (int a = 0; a < rank; a++) {
        if (dims[a] < 1) return HPEZ_BAD_ARGUMENT;
        g.dims[4 - rank + a] = dims[a];
    }
    for (int a = 3; a >= 0; a--) {
        g.estr[a] = n;
        n *= g.dims[a];
    }
    g.n = n;
    if (direction == HPEZ_DECOMPRESS && n_codes != n) return HPEZ_CORRUPT_STREAM;  // lorenzo.py:171-173
    if (!codes) return HPEZ_BAD_ARGUMENT;
    g.bound = bound;
    g.two_e = 2.0 * bound;
    g.radius = radius;
    // build_stencil (lorenzo.py:24-41) over the padded rank-4 index space;
    // leading unit axes only contribute zero offsets, so the surviving terms
    // keep the rank-R itertools.product order.
    LzStencil sten{};
    const double w1[2] = {1.0, -1.0}, w2[3] = {1.0, -2.0, 1.0};
    const double *w = order == 1 ? w1 : w2;
    const int base = order + 1;
    int total = 1;
    for (int a = 0; a < rank; a++) total *= base;
    for (int t = 0; t < total; t++) {
        int o[4] = {0, 0, 0, 0}, rem = t, any = 0;
        for (int a = rank - 1; a >= 0; a--) {
            o[4 - rank + a] = rem % base;
            rem /= base;
        }
        for (int a = 0; a < 4; a++) any |= o[a];
        if (!any) continue;
        double c = -1.0;
        for (int a = 4 - rank; a < 4; a++) c *= w[o[a]];
        int64_t fl = 0;
        for (int a = 0; a < 4; a++) {
            sten.delta[sten.n][a] = (int8_t)o[a];
            fl += o[a] * g.estr[a];
        }
        sten.flat[sten.n] = fl;
        sten.coef[sten.n] = c;
        sten.n++;
    }
    cudaError_t e = cudaMemcpyToSymbolAsync(c_lz, &sten, sizeof sten, 0, cudaMemcpyHostToDevice,
                                            (cudaStream_t)stream);
    if (e) return lz_cuda(e);
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t cap = outliers ? outl_cap : 0;
    if (work_dtype == HPEZ_WORK_F32) {
        if (code_dtype == HPEZ_CODES_U16)
            return lorenzo_run(g, direction, rounding, (float *)work, (uint16_t *)codes, outliers, cap, n_outliers, st);
        return lorenzo_run(g, direction, rounding, (float *)work, (int32_t *)codes, outliers, cap, n_outliers, st);
    }
    if (code_dtype == HPEZ_CODES_U16)
        return lorenzo_run(g, direction, rounding, (double *)work, (uint16_t *)codes, outliers, cap, n_outliers, st);
    return lorenzo_run(g, direction, rounding, (double *)work, (int32_t *)codes, outliers, cap, n_outliers, st);
}
