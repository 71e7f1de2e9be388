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
#include <cstdlib>
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


// ---------------------------------------------------------- tile wavefront --
// Rank <= 3 grids: 8^3 tiles on tile diagonals tz + ty + tx = D.  A tile
// depends only on tiles of earlier diagonals (every stencil offset is
// backward and <= 2 < 8), so one warp runs a tile through its 22 internal
// hyperplanes lz + ly + lx = h (__syncwarp between them) and a grid barrier
// separates diagonals: 128 global steps on cfg2 instead of 1024 launches.
// Each warp stages its tile plus the 2-deep backward halo in shared memory.
constexpr int kLzT = 8;
constexpr int kLzH = 3 * (kLzT - 1) + 1;
__constant__ uint16_t c_lt_pts[kLzT * kLzT * kLzT];  // (lz << 6) | (ly << 3) | lx, sorted by h
__constant__ int16_t c_lt_off[kLzH + 1];

constexpr int kLzS = kLzT + 2;  // staged tile edge: 2-deep backward halo
constexpr int kLzTileThreads = 128;

// One point of a staged tile: neighbours from the warp's shared-memory copy
// sb (origin at tile - 2), reference term order, quantizer as in
// lorenzo_plane_kernel; the result goes to sb and to the grid.
template <typename T, typename C, int DIR, int ROUND>
__device__ __forceinline__ void lz_tile_point(const LzGeom &g, double *sb, int lz, int ly, int lx, int64_t z, int64_t y,
                                              int64_t x, T *__restrict__ work, C *__restrict__ codes, int64_t code) {
    const int64_t c[4] = {0, z, y, x};
    const int so = ((lz + 2) * kLzS + (ly + 2)) * kLzS + (lx + 2);
    const int64_t i = z * g.estr[1] + y * g.estr[2] + x;
    if (DIR == HPEZ_DECOMPRESS && code == 0) return;  // outlier already scattered (staged from work)
    if (DIR == HPEZ_COMPRESS) code = 0;                // escape unless the quantizer accepts
    double acc = 0.0;
    for (int t = 0; t < c_lz.n; t++) {
        bool ok = true;
#pragma unroll
        for (int a = 1; a < 4; a++) ok &= c[a] >= c_lz.delta[t][a];
        if (ok) {
            const int d = (c_lz.delta[t][1] * kLzS + c_lz.delta[t][2]) * kLzS + c_lz.delta[t][3];
            acc = __dadd_rn(acc, __dmul_rn(c_lz.coef[t], sb[so - d]));
        }
    }
    const int64_t R = g.radius;
    if (DIR == HPEZ_COMPRESS) {
        const double orig = sb[so];
        if (g.bound > 0.0) {
            const double q = __ddiv_rn(__dsub_rn(orig, acc), g.two_e);
            double kq = floor(__dadd_rn(fabs(q), 0.5));
            if (q < 0.0) kq = -kq;
            if (-(double)R < kq && kq < (double)R) {
                const double recon = round_native<ROUND>(__dadd_rn(acc, __dmul_rn(g.two_e, kq)));
                if (fabs(__dsub_rn(recon, orig)) <= g.bound) {
                    code = (int64_t)kq + R;
                    sb[so] = recon;
                    work[i] = (T)recon;
                }
            }
        } else {
            const double recon = round_native<ROUND>(acc);
            if (recon == orig) {
                code = R;
                sb[so] = recon;
                work[i] = (T)recon;
            }
        }
        codes[i] = (C)code;
    } else {
        const double v = round_native<ROUND>(__dadd_rn(acc, __dmul_rn(g.two_e, (double)(code - R))));
        sb[so] = v;
        work[i] = (T)v;
    }
}

template <typename T, typename C, int DIR, int ROUND>
__global__ void __launch_bounds__(kLzTileThreads) lorenzo_tile_kernel(const LzGeom g, T *__restrict__ work,
                                                                      C *__restrict__ codes, uint32_t *bar) {
    __shared__ double s_tile[kLzTileThreads / 32][kLzS * kLzS * kLzS];  // one staged tile per warp (8 KB each)
    __shared__ int32_t s_code[DIR == HPEZ_DECOMPRESS ? kLzTileThreads / 32 : 1][kLzT * kLzT * kLzT];
    const int64_t Z = g.dims[1], Y = g.dims[2], X = g.dims[3];
    const int ntz = (int)((Z + kLzT - 1) / kLzT), nty = (int)((Y + kLzT - 1) / kLzT), ntx = (int)((X + kLzT - 1) / kLzT);
    const int ndiag = ntz + nty + ntx - 2;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double *sb = s_tile[wib];
    const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
    uint32_t target = 0;
    for (int D = 0; D < ndiag; D++) {
        const int tz0 = max(0, D - (nty - 1) - (ntx - 1)), tz1 = min(ntz - 1, D);
        const int npair = (tz1 - tz0 + 1) * nty;
        for (int k = gw; k < npair; k += nwarps) {
            const int tz = tz0 + k / nty, ty = k % nty, tx = D - tz - ty;
            if (tx < 0 || tx >= ntx) continue;
            const int64_t z0 = (int64_t)tz * kLzT, y0 = (int64_t)ty * kLzT, x0 = (int64_t)tx * kLzT;
            // stage the tile and its backward halo (earlier diagonals: final)
            for (int q = lane; q < kLzS * kLzS * kLzS; q += 32) {
                const int sz = q / (kLzS * kLzS), sy = (q / kLzS) % kLzS, sx = q % kLzS;
                const int64_t z = z0 - 2 + sz, y = y0 - 2 + sy, x = x0 - 2 + sx;
                double v = 0.0;
                if (z >= 0 && y >= 0 && x >= 0 && z < Z && y < Y && x < X)
                    v = (double)__ldcg(work + z * g.estr[1] + y * g.estr[2] + x);
                sb[q] = v;
            }
            // decompress: the tile's codes, in h order
            int32_t *sc = s_code[DIR == HPEZ_DECOMPRESS ? wib : 0];
            if (DIR == HPEZ_DECOMPRESS)
                for (int q = lane; q < kLzT * kLzT * kLzT; q += 32) {
                    const int pk = c_lt_pts[q];
                    const int64_t z = z0 + (pk >> 6), y = y0 + ((pk >> 3) & 7), x = x0 + (pk & 7);
                    sc[q] = (z < Z && y < Y && x < X) ? (int32_t)__ldcg(codes + z * g.estr[1] + y * g.estr[2] + x) : 0;
                }
            __syncwarp();
            for (int h = 0; h < kLzH; h++) {
#pragma unroll 1
                for (int q = c_lt_off[h] + lane; q < c_lt_off[h + 1]; q += 32) {
                    const int pk = c_lt_pts[q];
                    const int lz = pk >> 6, ly = (pk >> 3) & 7, lx = pk & 7;
                    const int64_t z = z0 + lz, y = y0 + ly, x = x0 + lx;
                    if (z < Z && y < Y && x < X)
                        lz_tile_point<T, C, DIR, ROUND>(g, sb, lz, ly, lx, z, y, x, work, codes,
                                                        DIR == HPEZ_DECOMPRESS ? (int64_t)sc[q] : 0);
                }
                __syncwarp();
            }
        }
        // grid barrier between diagonals (all CTAs co-resident: cooperative launch)
        __syncthreads();
        target += gridDim.x;
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(bar, 1u);
            while (ld_acquire(bar) < target) __nanosleep(32);
        }
        __syncthreads();
    }
}

static bool lz_tile_table() {
    static bool done = false;
    if (done) return true;
    uint16_t pts[kLzT * kLzT * kLzT];
    int16_t off[kLzH + 1];
    int k = 0;
    for (int h = 0; h < kLzH; h++) {
        off[h] = (int16_t)k;
        for (int a = 0; a < kLzT; a++)
            for (int b = 0; b < kLzT; b++) {
                const int c = h - a - b;
                if (c >= 0 && c < kLzT) pts[k++] = (uint16_t)((a << 6) | (b << 3) | c);
            }
    }
    off[kLzH] = (int16_t)k;
    if (cudaMemcpyToSymbol(c_lt_pts, pts, sizeof pts) != cudaSuccess) return false;
    if (cudaMemcpyToSymbol(c_lt_off, off, sizeof off) != cudaSuccess) return false;
    done = true;
    return true;
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
    // opt-in (HPEZ_LORENZO_TILE=1): bit-exact, but measured slower than the
    // per-hyperplane launches on cfg2 so far (8.0 vs 7.2 ms, order 1)
    const char *lt = getenv("HPEZ_LORENZO_TILE");
    bool tiled = g.dims[0] == 1 && lt && atoi(lt) != 0 && lz_tile_table();
    if (tiled) {
        typedef void (*tf_t)(const LzGeom, T *, C *, uint32_t *);
        tf_t tf;
        if (direction == HPEZ_COMPRESS)
            tf = rounding == HPEZ_ROUND_F32 ? lorenzo_tile_kernel<T, C, HPEZ_COMPRESS, HPEZ_ROUND_F32>
               : rounding == HPEZ_ROUND_INT ? lorenzo_tile_kernel<T, C, HPEZ_COMPRESS, HPEZ_ROUND_INT>
                                            : lorenzo_tile_kernel<T, C, HPEZ_COMPRESS, HPEZ_ROUND_NONE>;
        else
            tf = rounding == HPEZ_ROUND_F32 ? lorenzo_tile_kernel<T, C, HPEZ_DECOMPRESS, HPEZ_ROUND_F32>
               : rounding == HPEZ_ROUND_INT ? lorenzo_tile_kernel<T, C, HPEZ_DECOMPRESS, HPEZ_ROUND_INT>
                                            : lorenzo_tile_kernel<T, C, HPEZ_DECOMPRESS, HPEZ_ROUND_NONE>;
        int occ = 0, dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tf, kLzTileThreads, 0) != cudaSuccess || occ < 1) occ = 1;
        const int64_t pairs = ((g.dims[1] + kLzT - 1) / kLzT) * ((g.dims[2] + kLzT - 1) / kLzT);
        const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)occ * sms, (pairs + 3) / 4));
        uint32_t *bar = nullptr;
        e = cudaMallocAsync((void **)&bar, sizeof(uint32_t), st);
        if (!e) e = cudaMemsetAsync(bar, 0, sizeof(uint32_t), st);
        if (e) return lz_cuda(e);
        LzGeom gg = g;
        void *args[] = {(void *)&gg, (void *)&work, (void *)&codes, (void *)&bar};
        e = cudaLaunchCooperativeKernel((const void *)tf, dim3(blocks), dim3(kLzTileThreads), args, 0, st);
        cudaFreeAsync(bar, st);
        if (e) {
            cudaGetLastError();
            tiled = false;  // cooperative launch unavailable: hyperplane launches
        }
    }
    if (!tiled)
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
