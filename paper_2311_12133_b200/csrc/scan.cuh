// scan.cuh -- device exclusive scan of 32/64-bit counts into int64 offsets
// (single-pass decoupled look-back); shared by the sweep (escape offsets)
// and the Huffman decoder (symbol offsets).
#pragma once
#include "common.cuh"

namespace hpez {

// ------------------------------------------------------- exclusive scan --
constexpr int kScanBlock = 1024;
constexpr int kScanPer = 4;
constexpr int kScanTile = kScanBlock * kScanPer;

// Decoupled look-back: every CTA claims the next tile
// from a counter, publishes its aggregate, walks back over its
// predecessors' published aggregates / inclusive prefixes and publishes its
// own inclusive prefix.  status[0, tiles) hold flag (2 bits) | value,
// status[tiles] is the tile counter; all zero on entry.
constexpr unsigned long long kScanFlagA = 1ull << 62, kScanFlagP = 2ull << 62, kScanVal = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long scan_ld_acquire(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void scan_st_release(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <typename V>
static __global__ void __launch_bounds__(kScanBlock) scan_single_kernel(const V *__restrict__ in, int64_t n,
                                                                        int64_t *__restrict__ out,
                                                                        unsigned long long *status, int64_t tiles,
                                                                        int64_t *total) {
    __shared__ int64_t s_w[32];
    __shared__ int64_t s_prefix;
    __shared__ int64_t s_tile;
    if (threadIdx.x == 0) s_tile = (int64_t)atomicAdd(status + tiles, 1ull);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t base = tile * kScanTile + (int64_t)threadIdx.x * kScanPer;
    int64_t v[kScanPer], t = 0;
#pragma unroll
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
    if (warp == 0) {
        // warp-wide look-back: lane j inspects tile (lb - 1 - j); the
        // closest predecessor with an inclusive prefix ends the walk
        const int64_t agg = s_w[31];
        if (tile > 0 && lane == 0) scan_st_release(status + tile, kScanFlagA | (unsigned long long)agg);
        int64_t excl = 0;
        for (int64_t lb = tile; lb > 0; lb -= 32) {
            const int64_t j = lb - 1 - lane;
            unsigned long long sv = 0;
            if (j >= 0)
                while (((sv = scan_ld_acquire(status + j)) >> 62) == 0) {
                }
            const uint32_t pm = __ballot_sync(0xffffffffu, j >= 0 && (sv & ~kScanVal) == kScanFlagP);
            const int stop = pm ? __ffs(pm) - 1 : 32;  // first lane (closest tile) holding a prefix
            int64_t pv = (j >= 0 && lane <= stop) ? (int64_t)(sv & kScanVal) : 0;
            for (int o = 16; o > 0; o >>= 1) pv += __shfl_xor_sync(0xffffffffu, pv, o);
            excl += pv;
            if (pm) break;
        }
        if (lane == 0) {
            scan_st_release(status + tile, kScanFlagP | (unsigned long long)(excl + agg));
            s_prefix = excl;
            if (tile == tiles - 1 && total) *total = excl + agg;
        }
    }
    __syncthreads();
    int64_t run = s_prefix + (warp ? s_w[warp - 1] : 0) + x - t;
#pragma unroll
    for (int k = 0; k < kScanPer; k++) {
        if (base + k < n) out[base + k] = run;
        run += v[k];
    }
}

// tmp: scan_tmp_size(n) int64 entries of scratch (look-back status + counter)
template <typename V>
static void exclusive_scan(const V *in, int64_t n, int64_t *out, int64_t *tmp, int64_t *total, cudaStream_t st) {
    if (n == 0) {
        cudaMemsetAsync(total, 0, sizeof(int64_t), st);
        return;
    }
    const int64_t tiles = (n + kScanTile - 1) / kScanTile;
    cudaMemsetAsync(tmp, 0, (size_t)(tiles + 1) * sizeof(int64_t), st);
    scan_single_kernel<V><<<(unsigned)tiles, kScanBlock, 0, st>>>(in, n, out, (unsigned long long *)tmp, tiles, total);
}


// scratch int64 entries exclusive_scan needs for n inputs
inline int64_t scan_tmp_size(int64_t n) { return (n + kScanTile - 1) / kScanTile + 1; }

}  // namespace hpez
