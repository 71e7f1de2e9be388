// huffman.cu -- quantization-code histogram and canonical Huffman coding:
// the drop-in for huffman.encode / decode (huffman.py:144-174) as used by
// container.pack_codes / unpack_codes (container.py:70-106).
//
// * histogram: warp-aggregated (match_any) increments into a shared-memory
//   window around the code centre, global atomics outside it.
// * table: heap Huffman lengths with the (freq, smallest symbol) tie-break and
//   canonical codes, on the host (<= 65,536 symbols).
// * pack: chunks of 4096 codes; per-chunk bit counts -> scan -> each CTA
//   assembles its chunk MSB-first in shared memory with atomicOr and stores
//   whole 32-bit words, OR-ing only the two boundary words globally.
// * decode: host table-driven canonical decoder (12-bit first-level LUT,
//   bit-serial continuation) with the reference's error semantics.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <queue>
#include <vector>

#include "common.cuh"

namespace hpez {

constexpr int kHistWindow = 8192;  // shared-memory bins around the centre (32 KB)
constexpr int kPackChunk = 4096;    // codes per pack CTA
constexpr int kPackThreads = 256;
constexpr int kPackPer = kPackChunk / kPackThreads;  // 16 codes per thread

template <typename C>
__global__ void __launch_bounds__(512) histogram_kernel(const C *__restrict__ codes, int64_t n,
                                                        uint32_t *__restrict__ counts, int64_t nbins,
                                                        int64_t lo) {
    __shared__ uint32_t win[kHistWindow];
    for (int i = threadIdx.x; i < kHistWindow; i += blockDim.x) win[i] = 0;
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
        const int64_t i = base + threadIdx.x;
        const bool valid = i < n;
        const uint32_t c = valid ? (uint32_t)codes[i] : 0xffffffffu;
        const uint32_t active = __ballot_sync(0xffffffffu, valid);
        if (!valid) continue;
        const uint32_t peers = __match_any_sync(active, c);
        const int leader = __ffs(peers) - 1;
        if ((int)(threadIdx.x & 31) == leader) {
            const uint32_t k = __popc(peers);
            const int64_t w = (int64_t)c - lo;
            if (w >= 0 && w < kHistWindow) atomicAdd(&win[w], k);
            else if ((int64_t)c < nbins) atomicAdd(&counts[c], k);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kHistWindow; i += blockDim.x) {
        const uint32_t v = win[i];
        if (v && lo + i < nbins) atomicAdd(&counts[lo + i], v);
    }
}

template <typename C>
__global__ void __launch_bounds__(kPackThreads) chunk_bits_kernel(const C *__restrict__ codes, int64_t n,
                                                                  const uint8_t *__restrict__ lengths,
                                                                  uint64_t *__restrict__ chunk_bits) {
    __shared__ uint64_t s[kPackThreads / 32];
    const int64_t base = (int64_t)blockIdx.x * kPackChunk;
    uint64_t b = 0;
    for (int k = 0; k < kPackPer; k++) {
        const int64_t i = base + k * kPackThreads + threadIdx.x;
        if (i < n) b += lengths[(uint32_t)codes[i]];
    }
    for (int o = 16; o > 0; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = b;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t t = 0;
        for (int w = 0; w < kPackThreads / 32; w++) t += s[w];
        chunk_bits[blockIdx.x] = t;
    }
}

// In-place exclusive scan of chunk bit counts (single CTA); total to *total.
__global__ void __launch_bounds__(1024) scan_u64_kernel(uint64_t *v, int64_t n, uint64_t *total) {
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
    if (threadIdx.x == 0 && total) *total = s_carry;
}

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// OR `len` (<= 64) MSB-first bits of `val` at bit offset `bit` into words[]
// (big-endian bit order within each u32).
__device__ __forceinline__ void put_bits_smem(uint32_t *words, uint64_t bit, uint64_t val, int len) {
    while (len > 0) {
        const uint32_t w = (uint32_t)(bit >> 5);
        const int used = (int)(bit & 31);
        const int take = min(32 - used, len);
        const uint32_t chunk = (uint32_t)((val >> (len - take)) & ((take == 32) ? 0xffffffffull : ((1ull << take) - 1)));
        atomicOr(&words[w], chunk << (32 - used - take));
        bit += take;
        len -= take;
    }
}

template <typename C>
__global__ void __launch_bounds__(kPackThreads) pack_kernel(const C *__restrict__ codes, int64_t n,
                                                            const uint8_t *__restrict__ lengths,
                                                            const uint64_t *__restrict__ values,
                                                            const uint64_t *__restrict__ chunk_off,
                                                            uint32_t *__restrict__ out_words,
                                                            int max_len) {
    extern __shared__ uint32_t sw[];
    __shared__ uint64_t s_w[kPackThreads / 32];
    const int64_t base = (int64_t)blockIdx.x * kPackChunk;
    const uint64_t bit0 = chunk_off[blockIdx.x];
    const uint32_t lead = (uint32_t)(bit0 & 31);  // bits before this chunk in its first word
    const int nwords = (int)(((uint64_t)kPackChunk * max_len + 63) / 32) + 1;
    for (int i = threadIdx.x; i < nwords; i += kPackThreads) sw[i] = 0;
    // each thread owns kPackPer consecutive codes
    const int64_t first = base + (int64_t)threadIdx.x * kPackPer;
    uint64_t mybits = 0;
    for (int k = 0; k < kPackPer; k++)
        if (first + k < n) mybits += lengths[(uint32_t)codes[first + k]];
    // block exclusive scan of mybits
    uint64_t x = mybits;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    uint64_t wpre = 0;
    for (int w = 0; w < warp; w++) wpre += s_w[w];
    uint64_t bit = lead + wpre + x - mybits;
    for (int k = 0; k < kPackPer; k++) {
        if (first + k >= n) break;
        const uint32_t c = (uint32_t)codes[first + k];
        const int L = lengths[c];
        put_bits_smem(sw, bit, values[c], L);
        bit += L;
    }
    __syncthreads();
    uint64_t total = 0;
    for (int w = 0; w < kPackThreads / 32; w++) total += s_w[w];
    const uint64_t end = lead + total;  // bit end within the local word frame
    const int used_words = (int)((end + 31) / 32);
    const uint64_t gw0 = bit0 >> 5;
    for (int i = threadIdx.x; i < used_words; i += kPackThreads) {
        const uint32_t v = bswap32(sw[i]);
        if (i == 0 || i == used_words - 1) atomicOr(&out_words[gw0 + i], v);
        else out_words[gw0 + i] = v;
    }
}

template <typename C>
__global__ void nbits_kernel(const C *__restrict__ codes, int64_t n, const uint8_t *__restrict__ lengths,
                             unsigned long long *total) {
    uint64_t b = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        b += lengths[(uint32_t)codes[i]];
    for (int o = 16; o > 0; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(total, (unsigned long long)b);
}

static int cuda_ok(cudaError_t e) {
    if (e == cudaSuccess) return HPEZ_OK;
    fprintf(stderr, "hpez_b200: CUDA error %s\n", cudaGetErrorString(e));
    return HPEZ_CUDA_ERROR;
}

static int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

// huffman.code_lengths (huffman.py:19-48) + canonical_codes (huffman.py:51-88)
static int build_table(const int64_t *freqs, int64_t n, uint8_t *lengths, uint64_t *values) {
    struct Node { int64_t f, minsym; int32_t id; };
    auto greater = [](const Node &a, const Node &b) {
        return a.f > b.f || (a.f == b.f && a.minsym > b.minsym);
    };
    std::priority_queue<Node, std::vector<Node>, decltype(greater)> pq(greater);
    std::vector<int32_t> parent;
    std::vector<int64_t> sym;
    memset(lengths, 0, (size_t)n);
    for (int64_t s = 0; s < n; s++) {
        if (freqs[s] < 0) return HPEZ_BAD_ARGUMENT;
        if (freqs[s]) {
            pq.push(Node{freqs[s], s, (int32_t)parent.size()});
            parent.push_back(-1);
            sym.push_back(s);
        }
    }
    if (parent.empty()) return HPEZ_EMPTY_INPUT;
    if (parent.size() == 1) {
        lengths[sym[0]] = 1;
    } else {
        while (pq.size() > 1) {
            Node a = pq.top(); pq.pop();
            Node b = pq.top(); pq.pop();
            int32_t id = (int32_t)parent.size();
            parent.push_back(-1);
            sym.push_back(-1);
            parent[a.id] = id;
            parent[b.id] = id;
            pq.push(Node{a.f + b.f, std::min(a.minsym, b.minsym), id});
        }
        std::vector<int32_t> depth(parent.size(), 0);
        for (int64_t i = (int64_t)parent.size() - 1; i >= 0; i--)
            depth[i] = parent[i] < 0 ? 0 : depth[parent[i]] + 1;
        for (size_t i = 0; i < parent.size(); i++)
            if (sym[i] >= 0) {
                if (depth[i] > 255) return HPEZ_INVALID_TABLE;
                lengths[sym[i]] = (uint8_t)depth[i];
            }
    }
    // canonical codes: (length, symbol) order, first_code recurrence
    int maxl = 0;
    std::vector<int64_t> cnt(257, 0);
    for (int64_t s = 0; s < n; s++)
        if (lengths[s]) {
            cnt[lengths[s]]++;
            maxl = std::max(maxl, (int)lengths[s]);
        }
    if (maxl > 64) return HPEZ_INVALID_TABLE;  // values are u64
    std::vector<uint64_t> next(maxl + 2, 0);
    uint64_t code = 0;
    for (int l = 1; l <= maxl; l++) {
        next[l] = code;
        code = (code + (uint64_t)cnt[l]) << 1;
    }
    for (int64_t s = 0; s < n; s++) values[s] = lengths[s] ? next[lengths[s]]++ : 0;
    return HPEZ_OK;
}

}  // namespace hpez

using namespace hpez;

extern "C" {

int hpez_histogram(const void *codes, int32_t code_dtype, int64_t n, uint32_t *counts, int64_t nbins,
                   void *stream) {
    if (n < 0 || nbins < 1 || (n > 0 && !codes) || !counts) return HPEZ_BAD_ARGUMENT;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(uint32_t) * (size_t)nbins, st);
    if (e) return cuda_ok(e);
    if (n == 0) return HPEZ_OK;
    const int64_t centre = nbins / 2;
    const int64_t lo = std::max<int64_t>(0, centre - kHistWindow / 2);
    const int blocks = (int)std::min<int64_t>((n + 511) / 512, (int64_t)num_sms() * 4);
    if (code_dtype == HPEZ_CODES_U16)
        histogram_kernel<<<blocks, 512, 0, st>>>((const uint16_t *)codes, n, counts, nbins, lo);
    else
        histogram_kernel<<<blocks, 512, 0, st>>>((const int32_t *)codes, n, counts, nbins, lo);
    return cuda_ok(cudaGetLastError());
}

int hpez_huffman_table(const int64_t *freqs, int64_t n, uint8_t *lengths, uint64_t *values) {
    if (!freqs || !lengths || !values || n < 0) return HPEZ_BAD_ARGUMENT;
    return build_table(freqs, n, lengths, values);
}

int hpez_huffman_nbits(const void *codes, int32_t code_dtype, int64_t n, const uint8_t *lengths_dev,
                       int64_t *nbits, void *stream) {
    if (!nbits || n < 0) return HPEZ_BAD_ARGUMENT;
    cudaStream_t st = (cudaStream_t)stream;
    unsigned long long *d = nullptr;
    cudaError_t e = cudaMallocAsync((void **)&d, sizeof *d, st);
    if (!e) e = cudaMemsetAsync(d, 0, sizeof *d, st);
    if (e) return cuda_ok(e);
    if (n > 0) {
        const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8);
        if (code_dtype == HPEZ_CODES_U16)
            nbits_kernel<<<blocks, 256, 0, st>>>((const uint16_t *)codes, n, lengths_dev, d);
        else
            nbits_kernel<<<blocks, 256, 0, st>>>((const int32_t *)codes, n, lengths_dev, d);
    }
    unsigned long long h = 0;
    e = cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, st);
    if (!e) e = cudaStreamSynchronize(st);
    cudaFreeAsync(d, st);
    if (e) return cuda_ok(e);
    *nbits = (int64_t)h;
    return HPEZ_OK;
}

int hpez_huffman_pack(const void *codes, int32_t code_dtype, int64_t n, const uint8_t *lengths_dev,
                      const uint64_t *values_dev, int32_t max_len, uint8_t *out, int64_t nbits,
                      void *stream) {
    if (n < 0 || nbits < 0 || max_len < 1 || max_len > 64 || (n > 0 && (!codes || !out)))
        return HPEZ_BAD_ARGUMENT;
    if (((uintptr_t)out & 3) != 0) return HPEZ_BAD_ARGUMENT;  // word-aligned output
    if (n == 0) return HPEZ_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nchunks = (n + kPackChunk - 1) / kPackChunk;
    uint64_t *off = nullptr;
    cudaError_t e = cudaMallocAsync((void **)&off, sizeof(uint64_t) * (size_t)(nchunks + 1), st);
    if (e) return cuda_ok(e);
    e = cudaMemsetAsync(out, 0, (size_t)((nbits + 31) / 32) * 4, st);
    if (e) return cuda_ok(e);
    const int maxl = max_len;
    if (code_dtype == HPEZ_CODES_U16)
        chunk_bits_kernel<<<(unsigned)nchunks, kPackThreads, 0, st>>>((const uint16_t *)codes, n, lengths_dev, off);
    else
        chunk_bits_kernel<<<(unsigned)nchunks, kPackThreads, 0, st>>>((const int32_t *)codes, n, lengths_dev, off);
    scan_u64_kernel<<<1, 1024, 0, st>>>(off, nchunks, off + nchunks);
    const size_t smem = (size_t)(((uint64_t)kPackChunk * maxl + 63) / 32 + 1) * 4;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(pack_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        cudaFuncSetAttribute(pack_kernel<int32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        attr = true;
    }
    if (code_dtype == HPEZ_CODES_U16)
        pack_kernel<<<(unsigned)nchunks, kPackThreads, smem, st>>>((const uint16_t *)codes, n, lengths_dev, values_dev,
                                                                   off, (uint32_t *)out, maxl);
    else
        pack_kernel<<<(unsigned)nchunks, kPackThreads, smem, st>>>((const int32_t *)codes, n, lengths_dev, values_dev,
                                                                   off, (uint32_t *)out, maxl);
    e = cudaGetLastError();
    cudaFreeAsync(off, st);
    return cuda_ok(e);
}

// huffman._unpack_symbols (huffman.py:116-141) with a 12-bit first-level LUT.
int hpez_huffman_decode(const uint8_t *payload, int64_t nbytes, const uint8_t *lengths, int64_t n_lengths,
                        int64_t count, int32_t *out) {
    if (count == 0) return HPEZ_OK;
    if (!lengths || !out || n_lengths <= 0) return HPEZ_BAD_ARGUMENT;
    // canonical tables + validity (huffman.canonical_codes, huffman.py:51-88)
    int maxl = 0;
    int64_t present = 0;
    std::vector<int64_t> cnt(258, 0);
    for (int64_t s = 0; s < n_lengths; s++)
        if (lengths[s]) {
            cnt[lengths[s]]++;
            present++;
            maxl = std::max(maxl, (int)lengths[s]);
        }
    if (present == 0 || maxl > 64) return HPEZ_INVALID_TABLE;
    if (present == 1) {
        if (maxl != 1) return HPEZ_INVALID_TABLE;
    } else {
        // Kraft equality sum cnt[l] * 2^(maxl-l) == 2^maxl (exact in 128-bit)
        unsigned __int128 k = 0;
        for (int l = 1; l <= maxl; l++) k += (unsigned __int128)cnt[l] << (maxl - l);
        if (k != ((unsigned __int128)1 << maxl)) return HPEZ_INVALID_TABLE;
    }
    std::vector<int64_t> first_code(maxl + 2, 0), first_rank(maxl + 2, 0);
    int64_t code = 0, rank = 0;
    for (int l = 1; l <= maxl; l++) {
        first_code[l] = code;
        first_rank[l] = rank;
        code = (code + cnt[l]) << 1;
        rank += cnt[l];
    }
    std::vector<int32_t> rank_sym((size_t)rank);
    {
        std::vector<int64_t> fill(first_rank.begin(), first_rank.end());
        for (int64_t s = 0; s < n_lengths; s++)
            if (lengths[s]) rank_sym[(size_t)fill[lengths[s]]++] = (int32_t)s;
    }
    constexpr int K = 12;
    struct Lut { int32_t sym; int8_t len; };
    std::vector<Lut> lut(1 << K, Lut{-1, 0});
    for (int l = 1; l <= std::min(maxl, K); l++)
        for (int64_t r = 0; r < cnt[l]; r++) {
            const int64_t c = first_code[l] + r;
            const int64_t lo = c << (K - l), hi = (c + 1) << (K - l);
            for (int64_t p = lo; p < hi; p++) lut[(size_t)p] = Lut{rank_sym[(size_t)(first_rank[l] + r)], (int8_t)l};
        }
    const int64_t nbits = nbytes * 8;
    int64_t bitpos = 0;
    auto peek = [&](int64_t pos, int k) -> uint32_t {  // k bits at pos, zero padded
        uint32_t v = 0;
        const int64_t byte = pos >> 3;
        uint64_t w = 0;
        for (int b = 0; b < 4; b++) w = (w << 8) | (byte + b < nbytes ? payload[byte + b] : 0);
        w <<= (pos & 7);
        v = (uint32_t)((w >> (32 - k)) & ((1u << k) - 1));
        return v;
    };
    for (int64_t i = 0; i < count; i++) {
        const Lut e = lut[peek(bitpos, K)];
        if (e.len > 0 && bitpos + e.len <= nbits) {
            out[i] = e.sym;
            bitpos += e.len;
            continue;
        }
        // bit-serial continuation, identical control flow to the reference
        int64_t c = 0;
        int len = 0;
        for (;;) {
            if (bitpos >= nbits) return HPEZ_TRUNCATED;
            const int bit = (payload[bitpos >> 3] >> (7 - (bitpos & 7))) & 1;
            bitpos++;
            c = (c << 1) | bit;
            len++;
            if (len > maxl) return HPEZ_INVALID_TABLE;
            if (cnt[len] > 0) {
                const int64_t off = c - first_code[len];
                if (off >= 0 && off < cnt[len]) {
                    out[i] = rank_sym[(size_t)(first_rank[len] + off)];
                    break;
                }
            }
        }
    }
    return HPEZ_OK;
}

}  // extern "C"
