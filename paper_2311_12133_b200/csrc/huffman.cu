// huffman.cu -- quantization-code histogram and canonical Huffman coding:
// the drop-in for huffman.encode / decode (huffman.py:144-174) as used by
// container.pack_codes / unpack_codes (container.py:70-106).
//
// * histogram: shared-memory window around the code centre (u16 streams:
//   16-byte loads, privatized window copies; i32: warp-aggregated match_any),
//   global atomics outside it.
// * table: heap Huffman lengths with the (freq, smallest symbol) tie-break and
//   canonical codes, on the host (<= 65,536 symbols).
// * pack: chunks of 4096 codes; per-chunk bit counts -> scan -> each CTA
//   assembles its chunk MSB-first in shared memory with atomicOr and stores
//   whole 32-bit words, OR-ing only the two boundary words globally.
// * decode: self-synchronising chunked device decoder (speculative chunk
//   decode, fix-up passes, scanned offsets, write pass) and a host
//   table-driven decoder, both with the reference's error semantics.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <queue>
#include <vector>

#include "common.cuh"
#include "scan.cuh"

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


// u16 streams: eight codes per 16-byte load; each group of warps owns a
// private copy of the shared-memory window (fewer same-address conflicts on
// the concentrated centre bins), merged into the global counts at the end.
constexpr int kHistCopies = 2;  // default window copies per CTA (HPEZ_HIST_COPIES)
__global__ void __launch_bounds__(512) histogram_u16_kernel(const uint16_t *__restrict__ codes, int64_t n,
                                                            uint32_t *__restrict__ counts, int64_t nbins,
                                                            int64_t lo, int copies) {
    extern __shared__ uint32_t hwin[];  // copies x kHistWindow
    for (int i = threadIdx.x; i < copies * kHistWindow; i += blockDim.x) hwin[i] = 0;
    __syncthreads();
    uint32_t *win = hwin + ((threadIdx.x >> 5) % copies) * kHistWindow;
    auto add = [&](uint32_t c) {
        const int64_t w = (int64_t)c - lo;
        if (w >= 0 && w < kHistWindow) atomicAdd(&win[w], 1u);
        else if ((int64_t)c < nbins) atomicAdd(&counts[c], 1u);
    };
    // head up to 16-byte alignment, vector body, tail
    const int64_t mis = (int64_t)(((uintptr_t)codes & 15) / 2);
    const int64_t head = mis ? std::min<int64_t>(n, 8 - mis) : 0;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    if (gtid < head) add(codes[gtid]);
    const int64_t nvec = (n - head) / 8;
    const uint4 *v = reinterpret_cast<const uint4 *>(codes + head);
#pragma unroll 2
    for (int64_t k = gtid; k < nvec; k += nthr) {
        const uint4 q = __ldg(v + k);
        const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int j = 0; j < 4; j++) {
            add(w4[j] & 0xffffu);
            add(w4[j] >> 16);
        }
    }
    for (int64_t i = head + nvec * 8 + gtid; i < n; i += nthr) add(codes[i]);
    __syncthreads();
    for (int i = threadIdx.x; i < kHistWindow; i += blockDim.x) {
        uint32_t t = 0;
        for (int c = 0; c < copies; c++) t += hwin[c * kHistWindow + i];
        if (t && lo + i < nbins) atomicAdd(&counts[lo + i], t);
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

// Canonical decode tables (huffman.canonical_codes, huffman.py:51-88) with
// the reference's validity rules, shared by the host and device decoders.
constexpr int kLutBits = 12;
struct Canon {
    int maxl = 0;
    int64_t present = 0;
    std::vector<int64_t> cnt, first_code, first_rank;
    std::vector<int32_t> rank_sym;
    std::vector<int32_t> lut_sym;  // 12-bit prefix -> symbol (codes <= 12 bits)
    std::vector<uint8_t> lut_len;  // 0 = prefix of a longer code
};

static int build_canon(const uint8_t *lengths, int64_t n_lengths, Canon &t) {
    t.cnt.assign(258, 0);
    for (int64_t s = 0; s < n_lengths; s++)
        if (lengths[s]) {
            t.cnt[lengths[s]]++;
            t.present++;
            t.maxl = std::max(t.maxl, (int)lengths[s]);
        }
    if (t.present == 0 || t.maxl > 64) return HPEZ_INVALID_TABLE;
    if (t.present == 1) {
        if (t.maxl != 1) return HPEZ_INVALID_TABLE;
    } else {
        // Kraft equality sum cnt[l] * 2^(maxl-l) == 2^maxl (exact in 128-bit)
        unsigned __int128 k = 0;
        for (int l = 1; l <= t.maxl; l++) k += (unsigned __int128)t.cnt[l] << (t.maxl - l);
        if (k != ((unsigned __int128)1 << t.maxl)) return HPEZ_INVALID_TABLE;
    }
    t.first_code.assign(t.maxl + 2, 0);
    t.first_rank.assign(t.maxl + 2, 0);
    int64_t code = 0, rank = 0;
    for (int l = 1; l <= t.maxl; l++) {
        t.first_code[l] = code;
        t.first_rank[l] = rank;
        code = (code + t.cnt[l]) << 1;
        rank += t.cnt[l];
    }
    t.rank_sym.resize((size_t)rank);
    std::vector<int64_t> fill(t.first_rank.begin(), t.first_rank.end());
    for (int64_t s = 0; s < n_lengths; s++)
        if (lengths[s]) t.rank_sym[(size_t)fill[lengths[s]]++] = (int32_t)s;
    t.lut_sym.assign(1 << kLutBits, -1);
    t.lut_len.assign(1 << kLutBits, 0);
    for (int l = 1; l <= std::min(t.maxl, kLutBits); l++)
        for (int64_t r = 0; r < t.cnt[l]; r++) {
            const int64_t c = t.first_code[l] + r;
            const int64_t lo = c << (kLutBits - l), hi = (c + 1) << (kLutBits - l);
            for (int64_t q = lo; q < hi; q++) {
                t.lut_sym[(size_t)q] = t.rank_sym[(size_t)(t.first_rank[l] + r)];
                t.lut_len[(size_t)q] = (uint8_t)l;
            }
        }
    return HPEZ_OK;
}

// ------------------------------------------------------ device decoder --
// Self-synchronising chunked decode of the single MSB-first stream (no
// format change).  The payload is cut into chunks of kDecChunk bits; chunk
// k owns the codewords that START in its bit range, so its true start is the
// first codeword boundary at or after its first bit, which is where its
// predecessor's decode exits.
//   1. spec: every chunk is decoded from its first bit (assumed boundary);
//      the first kDecMarks symbol starts of that path are recorded.
//   2. fix: each chunk restarts at its predecessor's exit and decodes only
//      until it lands on one of its recorded speculative starts (Huffman codes
//      resynchronise within a few codewords), then takes the speculative
//      count and exit from there.  Repeated until no chunk changes (one pass
//      in practice; pass i fixes chunk i at the latest).
//   3. exclusive scan of the per-chunk counts -> output offsets; total.
//   4. write: every chunk decodes from its true start into a shared-memory
//      stage laid out in output order, copied out coalesced.
// Complete (Kraft-equal) tables decode every bit string, so speculation
// never hits an invalid pattern.  Bits are read through a 4-word register
// window refilled one 32-bit word at a time.
constexpr int kDecChunk = 1024;   // bits per chunk (> 64, the longest code)
constexpr int kDecThreads = 256;  // spec / fix CTAs
constexpr int kDecWriteThreads = 128;
constexpr int kDecLut = 11;       // first-level table bits on the device
constexpr int kDecMarks = 16;     // speculative symbol starts kept per chunk
constexpr int kDecStage = 24576;  // staged output symbols per write CTA

struct DecDev {
    uint64_t limit[66];  // first_code[l] + cnt[l]: l-bit prefixes below it are codes
    uint64_t first_code[66];
    int64_t first_rank[66];
    int32_t maxl, pad;
    int32_t lut_sym[1 << kDecLut];
    uint8_t lut_len[1 << kDecLut];
};


struct BitReader {
    const uint32_t *__restrict__ w;
    int64_t wi;  // word index of a
    uint32_t a, b, c, d;
    __device__ __forceinline__ void init(const uint32_t *__restrict__ words, int64_t pos) {
        w = words;
        wi = pos >> 5;
        a = bswap32(w[wi]);
        b = bswap32(w[wi + 1]);
        c = bswap32(w[wi + 2]);
        d = bswap32(w[wi + 3]);
    }
    // 64 stream bits from `pos` (pos >> 5 == wi), MSB first
    __device__ __forceinline__ uint64_t peek(int64_t pos) const {
        const int sh = (int)(pos & 31);
        const uint64_t hi = ((uint64_t)a << 32) | b;
        return sh ? (hi << sh) | (uint64_t)(c >> (32 - sh)) : hi;
    }
    __device__ __forceinline__ void advance_to(int64_t pos) {
        while ((pos >> 5) > wi) {
            a = b;
            b = c;
            c = d;
            d = bswap32(w[wi + 4]);
            wi++;
        }
    }
};

// one codeword at the head of `win`: its length (0 = no code) and symbol
__device__ __forceinline__ int dec_symbol(const DecDev &T, const int32_t *__restrict__ rank_sym, uint64_t win,
                                          int32_t &sym) {
    const uint32_t p = (uint32_t)(win >> (64 - kDecLut));
    int len = T.lut_len[p];
    sym = T.lut_sym[p];
    if (len) return len;
    for (int l = kDecLut + 1; l <= T.maxl; l++) {
        const uint64_t cw = win >> (64 - l);
        if (cw < T.limit[l]) {
            sym = rank_sym[T.first_rank[l] + (int64_t)(cw - T.first_code[l])];
            return l;
        }
    }
    return 0;
}

__device__ __forceinline__ void load_tables(DecDev &S, const DecDev *__restrict__ G) {
    const uint32_t *src = (const uint32_t *)G;
    uint32_t *dst = (uint32_t *)&S;
    for (int i = threadIdx.x; i < (int)(sizeof(DecDev) / 4); i += blockDim.x) dst[i] = src[i];
    __syncthreads();
}

// pass 1: speculative decode of every chunk from its first bit
__global__ void __launch_bounds__(kDecThreads) dec_spec_kernel(const uint32_t *__restrict__ w, int64_t nbits,
                                                               int64_t nchunks, const DecDev *__restrict__ tab,
                                                               const int32_t *__restrict__ rank_sym,
                                                               uint16_t *__restrict__ marks,
                                                               int32_t *__restrict__ spec_cnt,
                                                               int64_t *__restrict__ spec_exit,
                                                               int64_t *__restrict__ start, int32_t *__restrict__ cnt,
                                                               int64_t *__restrict__ exit, uint32_t *flags) {
    __shared__ DecDev S;
    load_tables(S, tab);
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nchunks) return;
    const int64_t a = k * kDecChunk, end = min(a + kDecChunk, nbits);
    BitReader br;
    br.init(w, a);
    int64_t pos = a;
    int32_t n = 0;
    while (pos < end) {
        if (n < kDecMarks) marks[k * kDecMarks + n] = (uint16_t)(pos - a);
        int32_t sym;
        const int len = dec_symbol(S, rank_sym, br.peek(pos), sym);
        if (!len) {  // unreachable for complete tables
            atomicOr(flags, 1u);
            break;
        }
        if (pos + len > nbits) break;  // codeword cut off by the end of the payload
        n++;
        pos += len;
        br.advance_to(pos);
    }
    spec_cnt[k] = cnt[k] = n;
    spec_exit[k] = exit[k] = pos;
    start[k] = a;
}

// pass 2 (repeated while anything changes): restart at the predecessor's exit
__global__ void __launch_bounds__(kDecThreads) dec_fix_kernel(const uint32_t *__restrict__ w, int64_t nbits,
                                                              int64_t nchunks, const DecDev *__restrict__ tab,
                                                              const int32_t *__restrict__ rank_sym,
                                                              const uint16_t *__restrict__ marks,
                                                              const int32_t *__restrict__ spec_cnt,
                                                              const int64_t *__restrict__ spec_exit,
                                                              int64_t *__restrict__ start, int32_t *__restrict__ cnt,
                                                              const int64_t *__restrict__ exit_in,
                                                              int64_t *__restrict__ exit_out, uint32_t *flags,
                                                              uint32_t *changed) {
    __shared__ DecDev S;
    load_tables(S, tab);
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nchunks) return;
    const int64_t a = k ? exit_in[k - 1] : 0;
    if (a == start[k]) {
        exit_out[k] = exit_in[k];
        return;
    }
    *changed = 1u;
    start[k] = a;
    const int64_t base = k * kDecChunk, end = min(base + kDecChunk, nbits);
    if (a >= end) {
        cnt[k] = 0;
        exit_out[k] = a;
        return;
    }
    const int nsp = spec_cnt[k];
    const int nm = min(nsp, kDecMarks);
    BitReader br;
    br.init(w, a);
    int64_t pos = a;
    int32_t n = 0;
    int i = 0;
    while (pos < end) {
        while (i < nm && base + marks[k * kDecMarks + i] < pos) i++;
        if (i < nm && base + marks[k * kDecMarks + i] == pos) {  // joined the speculative path
            cnt[k] = n + (nsp - i);
            exit_out[k] = spec_exit[k];
            return;
        }
        int32_t sym;
        const int len = dec_symbol(S, rank_sym, br.peek(pos), sym);
        if (!len) {
            atomicOr(flags, 1u);
            break;
        }
        if (pos + len > nbits) break;
        n++;
        pos += len;
        br.advance_to(pos);
    }
    cnt[k] = n;
    exit_out[k] = pos;
}

// pass 4: decode from the true starts into an output-ordered stage
template <typename O>
__global__ void __launch_bounds__(kDecWriteThreads) dec_write_kernel(const uint32_t *__restrict__ w, int64_t nbits,
                                                                     int64_t nchunks, const DecDev *__restrict__ tab,
                                                                     const int32_t *__restrict__ rank_sym,
                                                                     const int64_t *__restrict__ start,
                                                                     const int32_t *__restrict__ cnt,
                                                                     const int64_t *__restrict__ off, int64_t count,
                                                                     O *__restrict__ out) {
    __shared__ DecDev S;
    extern __shared__ __align__(16) unsigned char s_stage_raw[];
    O *stage = reinterpret_cast<O *>(s_stage_raw);
    const int64_t k0 = (int64_t)blockIdx.x * kDecWriteThreads;
    const int64_t kl = min(k0 + kDecWriteThreads, nchunks) - 1;
    const int64_t b0 = off[k0];
    if (b0 >= count) return;  // uniform over the CTA
    load_tables(S, tab);
    const int64_t b1 = min(off[kl] + cnt[kl], count);
    const bool staged = b1 - b0 <= kDecStage;
    const int64_t k = k0 + threadIdx.x;
    if (k <= kl && off[k] < count) {
        const int64_t a = start[k], end = min((k + 1) * (int64_t)kDecChunk, nbits);
        int64_t o = off[k];
        const int64_t o1 = min(o + cnt[k], count);
        BitReader br;
        br.init(w, a);
        int64_t pos = a;
        while (o < o1) {
            int32_t sym;
            const int len = dec_symbol(S, rank_sym, br.peek(pos), sym);
            if (staged) stage[o - b0] = (O)sym;
            else out[o] = (O)sym;
            o++;
            pos += len;
            br.advance_to(pos);
        }
        (void)end;
    }
    if (!staged) return;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < b1 - b0; i += kDecWriteThreads) out[b0 + i] = stage[i];
}

// single-symbol tables (the only incomplete tree the reference accepts):
// every symbol is the bit 0; find the first 1 bit
__global__ void dec_first_one_kernel(const uint8_t *__restrict__ p, int64_t nbytes, unsigned long long *first) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nbytes || !p[i]) return;
    atomicMin(first, (unsigned long long)(i * 8 + (__clz((int)p[i]) - 24)));
}

template <typename O>
__global__ void dec_fill_kernel(O *__restrict__ out, int64_t n, O v) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = v;
}

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
    if (code_dtype == HPEZ_CODES_U16) {
        int copies = kHistCopies;
        if (const char *ev = getenv("HPEZ_HIST_COPIES")) copies = std::max(1, std::min(6, atoi(ev)));
        const size_t smem = sizeof(uint32_t) * copies * kHistWindow;
        e = cudaFuncSetAttribute(histogram_u16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e) return cuda_ok(e);
        const int per_sm = std::max(1, std::min(4, (int)(220 * 1024 / (smem + 1024))));
        const int vb = (int)std::min<int64_t>((n / 8 + 511) / 512 + 1, (int64_t)num_sms() * per_sm);
        histogram_u16_kernel<<<vb, 512, smem, st>>>((const uint16_t *)codes, n, counts, nbins, lo, copies);
    } else
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
    Canon t;
    if (int st = build_canon(lengths, n_lengths, t)) return st;
    const int maxl = t.maxl;
    const int64_t nbits = nbytes * 8;
    int64_t bitpos = 0;
    auto peek = [&](int64_t pos, int k) -> uint32_t {  // k bits at pos, zero padded
        const int64_t byte = pos >> 3;
        uint64_t w = 0;
        for (int b = 0; b < 4; b++) w = (w << 8) | (byte + b < nbytes ? payload[byte + b] : 0);
        w <<= (pos & 7);
        return (uint32_t)((w >> (32 - k)) & ((1u << k) - 1));
    };
    for (int64_t i = 0; i < count; i++) {
        const uint32_t q = peek(bitpos, kLutBits);
        const int len0 = t.lut_len[q];
        if (len0 > 0 && bitpos + len0 <= nbits) {
            out[i] = t.lut_sym[q];
            bitpos += len0;
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
            if (t.cnt[len] > 0) {
                const int64_t off = c - t.first_code[len];
                if (off >= 0 && off < t.cnt[len]) {
                    out[i] = t.rank_sym[(size_t)(t.first_rank[len] + off)];
                    break;
                }
            }
        }
    }
    return HPEZ_OK;
}

// Device decode of `count` symbols into out_dev (u16 or i32).  The payload
// is copied to the device from host memory (payload_host) or read from
// device memory (payload_dev, nbytes + 12 readable bytes, zero padded).
int hpez_huffman_decode_device(const uint8_t *payload_host, const uint8_t *payload_dev, int64_t nbytes,
                               const uint8_t *lengths, int64_t n_lengths, int64_t count, void *out_dev,
                               int32_t out_dtype, void *stream) {
    if (count == 0) return HPEZ_OK;
    if (!lengths || !out_dev || n_lengths <= 0 || (!payload_host && !payload_dev && nbytes > 0)) return HPEZ_BAD_ARGUMENT;
    if (out_dtype != HPEZ_CODES_U16 && out_dtype != HPEZ_CODES_I32) return HPEZ_BAD_ARGUMENT;
    if (out_dtype == HPEZ_CODES_U16 && n_lengths > 65536) return HPEZ_BAD_ARGUMENT;
    Canon t;
    if (int st = build_canon(lengths, n_lengths, t)) return st;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nbits = nbytes * 8;
    const int64_t nwords = (nbytes + 3) / 4 + 6;  // BitReader reads up to 5 words ahead
    uint32_t *w = nullptr;
    cudaError_t e = cudaMallocAsync((void **)&w, (size_t)nwords * 4, s);
    if (e) return cuda_ok(e);
    e = cudaMemsetAsync(w, 0, (size_t)nwords * 4, s);
    if (!e && nbytes)
        e = payload_dev ? cudaMemcpyAsync(w, payload_dev, (size_t)nbytes, cudaMemcpyDeviceToDevice, s)
                        : cudaMemcpyAsync(w, payload_host, (size_t)nbytes, cudaMemcpyHostToDevice, s);
    int status = HPEZ_OK;
    if (t.present == 1) {
        // one symbol, code "0": the reference fails at the first 1 bit
        // (InvalidTable, or TruncatedStream if it is the last payload bit)
        // or when the payload holds fewer than count bits
        unsigned long long *d_first = nullptr, h_first = ~0ull;
        if (!e) e = cudaMallocAsync((void **)&d_first, sizeof h_first, s);
        if (!e) e = cudaMemcpyAsync(d_first, &h_first, sizeof h_first, cudaMemcpyHostToDevice, s);
        if (!e && nbytes)
            dec_first_one_kernel<<<(unsigned)((nbytes + 255) / 256), 256, 0, s>>>((const uint8_t *)w, nbytes, d_first);
        if (!e) e = cudaMemcpyAsync(&h_first, d_first, sizeof h_first, cudaMemcpyDeviceToHost, s);
        if (!e) e = cudaStreamSynchronize(s);
        const int32_t sym = t.rank_sym[0];
        if (!e) {
            const int64_t j = (int64_t)h_first;
            if (h_first != ~0ull && j < std::min(count, nbits)) status = j + 1 >= nbits ? HPEZ_TRUNCATED : HPEZ_INVALID_TABLE;
            else if (nbits < count) status = HPEZ_TRUNCATED;
        }
        if (!e && status == HPEZ_OK) {
            const unsigned g = (unsigned)((count + 255) / 256);
            if (out_dtype == HPEZ_CODES_U16) dec_fill_kernel<<<g, 256, 0, s>>>((uint16_t *)out_dev, count, (uint16_t)sym);
            else dec_fill_kernel<<<g, 256, 0, s>>>((int32_t *)out_dev, count, sym);
            e = cudaGetLastError();
        }
        if (d_first) cudaFreeAsync(d_first, s);
        cudaFreeAsync(w, s);
        return e ? cuda_ok(e) : status;
    }
    // device tables: canonical limits + an 11-bit first-level table
    DecDev *h_tab = new DecDev();
    std::memset(h_tab, 0, sizeof(DecDev));
    h_tab->maxl = t.maxl;
    for (int l = 1; l <= t.maxl; l++) {
        h_tab->first_code[l] = (uint64_t)t.first_code[l];
        h_tab->limit[l] = (uint64_t)(t.first_code[l] + t.cnt[l]);
        h_tab->first_rank[l] = t.first_rank[l];
    }
    for (int l = 1; l <= std::min(t.maxl, kDecLut); l++)
        for (int64_t r = 0; r < t.cnt[l]; r++) {
            const int64_t c = t.first_code[l] + r;
            for (int64_t q = c << (kDecLut - l); q < (c + 1) << (kDecLut - l); q++) {
                h_tab->lut_sym[q] = t.rank_sym[(size_t)(t.first_rank[l] + r)];
                h_tab->lut_len[q] = (uint8_t)l;
            }
        }
    const int64_t nchunks = std::max<int64_t>(1, (nbits + kDecChunk - 1) / kDecChunk);
    DecDev *d_tab = nullptr;
    int32_t *d_rank = nullptr, *d_cnt = nullptr, *d_spec_cnt = nullptr;
    uint16_t *d_marks = nullptr;
    int64_t *d_start = nullptr, *d_exit = nullptr, *d_exit2 = nullptr, *d_spec_exit = nullptr, *d_off = nullptr,
            *d_tmp = nullptr;
    // d_res: [0] total symbols, [1] invalid-pattern flag, [2..] changed flag per fix pass
    constexpr int kFixPasses = 2;
    int64_t *d_res = nullptr;
    int64_t h_res[2 + kFixPasses] = {};
    if (!e) e = cudaMallocAsync((void **)&d_tab, sizeof(DecDev), s);
    if (!e) e = cudaMallocAsync((void **)&d_rank, t.rank_sym.size() * 4, s);
    if (!e) e = cudaMallocAsync((void **)&d_marks, (size_t)nchunks * kDecMarks * 2, s);
    if (!e) e = cudaMallocAsync((void **)&d_spec_cnt, (size_t)nchunks * 4, s);
    if (!e) e = cudaMallocAsync((void **)&d_cnt, (size_t)nchunks * 4, s);
    if (!e) e = cudaMallocAsync((void **)&d_spec_exit, (size_t)nchunks * 8, s);
    if (!e) e = cudaMallocAsync((void **)&d_start, (size_t)nchunks * 8, s);
    if (!e) e = cudaMallocAsync((void **)&d_exit, (size_t)nchunks * 8, s);
    if (!e) e = cudaMallocAsync((void **)&d_exit2, (size_t)nchunks * 8, s);
    if (!e) e = cudaMallocAsync((void **)&d_off, (size_t)nchunks * 8, s);
    if (!e) e = cudaMallocAsync((void **)&d_tmp, (size_t)scan_tmp_size(nchunks) * 8, s);
    if (!e) e = cudaMallocAsync((void **)&d_res, sizeof h_res, s);
    if (!e) e = cudaMemcpyAsync(d_tab, h_tab, sizeof(DecDev), cudaMemcpyHostToDevice, s);
    if (!e) e = cudaMemcpyAsync(d_rank, t.rank_sym.data(), t.rank_sym.size() * 4, cudaMemcpyHostToDevice, s);
    if (!e) e = cudaMemsetAsync(d_res, 0, sizeof h_res, s);
    uint32_t *d_invalid = (uint32_t *)(d_res + 1);
    const unsigned grid = (unsigned)((nchunks + kDecThreads - 1) / kDecThreads);
    auto fix = [&](uint32_t *changed) {
        dec_fix_kernel<<<grid, kDecThreads, 0, s>>>(w, nbits, nchunks, d_tab, d_rank, d_marks, d_spec_cnt,
                                                    d_spec_exit, d_start, d_cnt, d_exit, d_exit2, d_invalid,
                                                    changed);
        std::swap(d_exit, d_exit2);
    };
    if (!e) {
        dec_spec_kernel<<<grid, kDecThreads, 0, s>>>(w, nbits, nchunks, d_tab, d_rank, d_marks, d_spec_cnt,
                                                     d_spec_exit, d_start, d_cnt, d_exit, d_invalid);
        for (int i = 0; i < kFixPasses; i++) fix((uint32_t *)(d_res + 2 + i));
        exclusive_scan(d_cnt, nchunks, d_off, d_tmp, d_res, s);
        e = cudaGetLastError();
    }
    // one host round trip in the common case: the last fix pass changed nothing
    if (!e) e = cudaMemcpyAsync(h_res, d_res, sizeof h_res, cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaStreamSynchronize(s);
    for (int64_t it = kFixPasses; !e && h_res[1 + kFixPasses]; it++) {
        if (it > nchunks + 1) {  // cannot happen: pass i fixes chunk i at the latest
            e = cudaErrorUnknown;
            break;
        }
        e = cudaMemsetAsync(d_res + 1 + kFixPasses, 0, 8, s);
        fix((uint32_t *)(d_res + 1 + kFixPasses));
        exclusive_scan(d_cnt, nchunks, d_off, d_tmp, d_res, s);
        if (!e) e = cudaMemcpyAsync(h_res, d_res, sizeof h_res, cudaMemcpyDeviceToHost, s);
        if (!e) e = cudaStreamSynchronize(s);
    }
    if (!e && (uint32_t)h_res[1]) status = HPEZ_INVALID_TABLE;
    if (!e && status == HPEZ_OK && h_res[0] < count) status = HPEZ_TRUNCATED;
    if (!e && status == HPEZ_OK) {
        const unsigned wgrid = (unsigned)((nchunks + kDecWriteThreads - 1) / kDecWriteThreads);
        if (out_dtype == HPEZ_CODES_U16) {
            const size_t smem = kDecStage * sizeof(uint16_t);
            cudaFuncSetAttribute(dec_write_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            dec_write_kernel<uint16_t><<<wgrid, kDecWriteThreads, smem, s>>>(w, nbits, nchunks, d_tab, d_rank, d_start,
                                                                            d_cnt, d_off, count, (uint16_t *)out_dev);
        } else {
            const size_t smem = kDecStage * sizeof(int32_t);
            cudaFuncSetAttribute(dec_write_kernel<int32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            dec_write_kernel<int32_t><<<wgrid, kDecWriteThreads, smem, s>>>(w, nbits, nchunks, d_tab, d_rank, d_start,
                                                                           d_cnt, d_off, count, (int32_t *)out_dev);
        }
        e = cudaGetLastError();
    }
    for (void *q : {(void *)w, (void *)d_tab, (void *)d_rank, (void *)d_marks, (void *)d_spec_cnt, (void *)d_cnt,
                    (void *)d_spec_exit, (void *)d_start, (void *)d_exit, (void *)d_exit2, (void *)d_off,
                    (void *)d_tmp, (void *)d_res})
        if (q) cudaFreeAsync(q, s);
    delete h_tab;  // pageable H2D copies have consumed it by the synchronize above
    return e ? cuda_ok(e) : status;
}

}  // extern "C"
