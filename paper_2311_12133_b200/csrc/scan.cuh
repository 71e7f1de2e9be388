// scan.cuh -- three-phase device exclusive scan (tile scan, single-CTA scan
// of tile sums, add-back) of 32/64-bit counts into int64 offsets; shared by
// the sweep (escape offsets) and the Huffman decoder (symbol offsets).
#pragma once
#include "common.cuh"

namespace hpez {

// ------------------------------------------------------- exclusive scan --
// Three-phase exclusive scan of n counts into i64 offsets.
constexpr int kScanBlock = 1024;
constexpr int kScanPer = 4;
constexpr int kScanTile = kScanBlock * kScanPer;

template <typename V>
static __global__ void __launch_bounds__(kScanBlock) scan_tiles_kernel(const V *__restrict__ in, int64_t n,
                                                                int64_t *__restrict__ out,
                                                                int64_t *__restrict__ tile_sum) {
    __shared__ int64_t s_w[32];
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanPer;
    int64_t v[kScanPer], t = 0;
    for (int k = 0; k < kScanPer; k++) {
        v[k] = base + k < n ? (int64_t)in[base + k] : 0;
        t += v[k];
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t x = t;
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int64_t w = s_w[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        s_w[lane] = w;
    }
    __syncthreads();
    int64_t run = (warp ? s_w[warp - 1] : 0) + x - t;
    for (int k = 0; k < kScanPer; k++) {
        if (base + k < n) out[base + k] = run;
        run += v[k];
    }
    if (threadIdx.x == kScanBlock - 1) tile_sum[blockIdx.x] = run;
}

static __global__ void __launch_bounds__(1024) scan_sums_kernel(int64_t *sums, int64_t n, int64_t *total) {
    __shared__ int64_t s_w[32];
    __shared__ int64_t s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t off = 0; off < n; off += blockDim.x) {
        const int64_t i = off + threadIdx.x;
        const int64_t x0 = i < n ? sums[i] : 0;
        int64_t x = x0;
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_w[warp] = x;
        __syncthreads();
        if (warp == 0) {
            int64_t w = s_w[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            s_w[lane] = w;
        }
        __syncthreads();
        const int64_t carry = s_carry;
        const int64_t pre = (warp ? s_w[warp - 1] : 0) + x - x0;
        if (i < n) sums[i] = carry + pre;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) s_carry = carry + pre + x0;
        __syncthreads();
    }
    if (threadIdx.x == 0 && total) *total = s_carry;
}

static __global__ void scan_add_kernel(int64_t *__restrict__ out, int64_t n, const int64_t *__restrict__ tile_off) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] += tile_off[i / kScanTile];
}

template <typename V>
static void exclusive_scan(const V *in, int64_t n, int64_t *out, int64_t *tmp, int64_t *total, cudaStream_t st) {
    if (n == 0) {
        cudaMemsetAsync(total, 0, sizeof(int64_t), st);
        return;
    }
    const int64_t tiles = (n + kScanTile - 1) / kScanTile;
    scan_tiles_kernel<V><<<(unsigned)tiles, kScanBlock, 0, st>>>(in, n, out, tmp);
    scan_sums_kernel<<<1, 1024, 0, st>>>(tmp, tiles, total);
    scan_add_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(out, n, tmp);
}


// scratch int64 entries exclusive_scan needs for n inputs
inline int64_t scan_tmp_size(int64_t n) { return (n + kScanTile - 1) / kScanTile + 1; }

}  // namespace hpez
