// Hand-written sorting and scanning for the binning pipeline (sm_100a), replacing the CUB
// library kernels on the scoring path:
//   * stable LSD radix sort of (u32 key, u32 | u64 value) pairs, 8-bit digits, over several
//     independent segments in one launch per kernel (a sub-batch of views): the depth-rank
//     sort K2 (fp32 depth key, splat_render.cpp:40-45, runs fixed by k_tiefix) and the
//     stable row sort of the binning (K3, rows of at most 2^8 or 2^16 tile rows);
//   * exclusive scan of u32 / u64 counts into u64 offsets (row-pair offsets of the binning,
//     contributor-list offsets of retain_contributors).
// One pass = three kernels: per-tile digit histograms (digit-major), a per-segment exclusive
// scan of those counts, and a stable scatter. Inside a 2048-element tile each warp walks its
// 256 elements in order, 32 at a time; __match_any_sync groups the lanes of a digit, so an
// element's rank is (elements of its digit in earlier warps) + (earlier rounds of its warp)
// + (lower lanes of its round): the order of equal digits is the input order (stable).
#include "sgm_internal.h"

namespace sgm {

namespace {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kPerWarp = 256;                           // elements per warp per tile
constexpr int kSortTile = kSortWarps * kPerWarp;        // 2048
constexpr int kRounds = kPerWarp / 32;                  // 8
constexpr int kRadix = 256;

template <typename N>
__device__ __forceinline__ uint64_t seg_len(const N* n, int s) { return static_cast<uint64_t>(n[s]); }

// counts[(s * 256 + digit) * T + tile]; tiles past a segment's end count zero
template <typename N>
__global__ void __launch_bounds__(kSortThreads) k_sort_hist(const uint32_t* __restrict__ keys, size_t stride,
                                                           const N* __restrict__ n, int shift, int T,
                                                           uint32_t* __restrict__ counts) {
    __shared__ uint32_t h[kSortWarps][kRadix];
    const int s = blockIdx.y, t = blockIdx.x;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < kSortWarps * kRadix; i += kSortThreads) (&h[0][0])[i] = 0u;
    __syncthreads();
    const uint64_t len = seg_len(n, s);
    const uint64_t base = static_cast<uint64_t>(t) * kSortTile + static_cast<uint64_t>(w) * kPerWarp;
    const uint32_t* k = keys + static_cast<size_t>(s) * stride;
#pragma unroll 4
    for (int r = 0; r < kRounds; ++r) {
        const uint64_t i = base + r * 32 + lane;
        if (i < len) atomicAdd(&h[w][(k[i] >> shift) & 0xffu], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < kRadix; d += kSortThreads) {
        uint32_t c = 0;
#pragma unroll
        for (int q = 0; q < kSortWarps; ++q) c += h[q][d];
        counts[(static_cast<size_t>(s) * kRadix + d) * T + t] = c;
    }
}

// next_counts (not null): the next pass's per-tile digit histogram, accumulated here from each
// element's destination (its next-pass tile) and next digit, so no histogram kernel runs
// between the passes
template <typename V, typename N>
__global__ void __launch_bounds__(kSortThreads) k_sort_scatter(const uint32_t* __restrict__ kin, const V* __restrict__ vin,
                                                              uint32_t* __restrict__ kout, V* __restrict__ vout,
                                                              size_t stride, const N* __restrict__ n, int shift,
                                                              int T, const uint32_t* __restrict__ counts,
                                                              uint32_t* __restrict__ next_counts) {
    __shared__ uint32_t wc[kSortWarps][kRadix];  // per (warp, digit): count, then absolute base
    const int s = blockIdx.y, t = blockIdx.x;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t len = seg_len(n, s);
    const uint64_t tile0 = static_cast<uint64_t>(t) * kSortTile;
    if (tile0 >= len) return;
    for (int i = threadIdx.x; i < kSortWarps * kRadix; i += kSortThreads) (&wc[0][0])[i] = 0u;
    __syncthreads();
    const size_t so = static_cast<size_t>(s) * stride;
    const uint64_t base = tile0 + static_cast<uint64_t>(w) * kPerWarp;
    const unsigned lt = (1u << lane) - 1u;
    uint32_t key[kRounds];
    uint32_t rank[kRounds];  // digit << 16 | rank within the warp
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const uint64_t i = base + r * 32 + lane;
        const bool ok = i < len;
        key[r] = ok ? kin[so + i] : 0u;
        const int d = ok ? static_cast<int>((key[r] >> shift) & 0xffu) : kRadix + lane;  // unique when out of range
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        uint32_t before = 0;
        if (ok) before = wc[w][d];
        __syncwarp();
        if (ok && (peers & lt) == 0u) wc[w][d] = before + static_cast<uint32_t>(__popc(peers));
        __syncwarp();
        rank[r] = ok ? (static_cast<uint32_t>(d) << 16) | (before + static_cast<uint32_t>(__popc(peers & lt))) : 0xffffffffu;
    }
    __syncthreads();
    for (int d = threadIdx.x; d < kRadix; d += kSortThreads) {
        uint32_t run = counts[(static_cast<size_t>(s) * kRadix + d) * T + t];
#pragma unroll
        for (int q = 0; q < kSortWarps; ++q) {
            const uint32_t c = wc[q][d];
            wc[q][d] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        if (rank[r] == 0xffffffffu) continue;
        const uint64_t i = base + r * 32 + lane;
        const uint32_t d = rank[r] >> 16;
        const uint32_t pos = wc[w][d] + (rank[r] & 0xffffu);
        const size_t dst = so + pos;
        kout[dst] = key[r];
        vout[dst] = vin[so + i];
        if (next_counts)
            atomicAdd(&next_counts[(static_cast<size_t>(s) * kRadix + ((key[r] >> (shift + 8)) & 0xffu)) * T +
                                   pos / kSortTile], 1u);
    }
}

// ---- exclusive scan of counts into u64 offsets: block sums, a one-block scan of the block
// sums, then the scanned blocks ----
constexpr int kScanT = 1024;
constexpr int kScanItems = 4;
constexpr int kScanBlock = kScanT * kScanItems;
constexpr uint64_t kSmallScanU64 = 32 * 1024;  // one-launch scans up to this many counts

template <typename C>
__global__ void __launch_bounds__(kScanT) k_scan_sums(const C* __restrict__ in, uint64_t n,
                                                     unsigned long long* __restrict__ sums,
                                                     uint64_t seg_stride = 0) {
    __shared__ unsigned long long ws[kScanT / 32];
    in += blockIdx.y * seg_stride;
    sums += blockIdx.y * gridDim.x;
    const uint64_t b0 = static_cast<uint64_t>(blockIdx.x) * kScanBlock;
    unsigned long long v = 0;
#pragma unroll
    for (int q = 0; q < kScanItems; ++q) {
        const uint64_t i = b0 + static_cast<uint64_t>(q) * kScanT + threadIdx.x;
        if (i < n) v += static_cast<unsigned long long>(in[i]);
    }
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        unsigned long long u = ws[threadIdx.x];
        for (int o = 16; o > 0; o >>= 1) u += __shfl_down_sync(0xffffffffu, u, o);
        if (threadIdx.x == 0) sums[blockIdx.x] = u;
    }
}

// Block-wide exclusive scan of one value per thread (1024 threads); returns the thread's
// prefix and adds the block total to *carry (after every thread has read it).
template <typename T>
__device__ __forceinline__ T block_exclusive(T v, T* ws, T* carry) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    if (w == 0) {
        T u = ws[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T y = __shfl_up_sync(0xffffffffu, u, o);
            if (lane >= o) u += y;
        }
        ws[lane] = u;
    }
    __syncthreads();
    const T r = *carry + (w ? ws[w - 1] : T(0)) + x - v;
    __syncthreads();
    if (threadIdx.x == kScanT - 1) *carry += ws[kScanT / 32 - 1];
    __syncthreads();
    return r;
}

constexpr int kSmallItems = 8;  // consecutive counts per thread per round of the one-block scans

// per segment (block), exclusive scan in place of n u32 counts seg_stride apart, 8192 per
// round (small arrays: one launch); also zeroes `zero` (the next pass's counts)
__global__ void __launch_bounds__(kScanT) k_scan_small(uint32_t* __restrict__ a, uint64_t n, uint64_t seg_stride,
                                                      uint32_t* __restrict__ zero) {
    __shared__ uint32_t ws[kScanT / 32];
    __shared__ uint32_t carry;
    uint32_t* c = a + blockIdx.x * seg_stride;
    if (zero)
        for (uint64_t i = threadIdx.x; i < n; i += kScanT) zero[blockIdx.x * seg_stride + i] = 0u;
    if (threadIdx.x == 0) carry = 0u;
    __syncthreads();
    for (uint64_t b0 = 0; b0 < n; b0 += static_cast<uint64_t>(kScanT) * kSmallItems) {
        const uint64_t i0 = b0 + static_cast<uint64_t>(threadIdx.x) * kSmallItems;
        uint32_t v[kSmallItems];
        uint32_t sum = 0;
#pragma unroll
        for (int q = 0; q < kSmallItems; ++q) {
            v[q] = i0 + q < n ? c[i0 + q] : 0u;
            sum += v[q];
        }
        uint32_t run = block_exclusive<uint32_t>(sum, ws, &carry);
#pragma unroll
        for (int q = 0; q < kSmallItems; ++q)
            if (i0 + q < n) {
                c[i0 + q] = run;
                run += v[q];
            }
    }
}

// exclusive scan of the block sums in place (one block, any count)
__global__ void __launch_bounds__(kScanT) k_scan_top(unsigned long long* __restrict__ sums, uint32_t nb) {
    __shared__ unsigned long long part[kScanT];
    sums += static_cast<size_t>(blockIdx.x) * nb;  // one block per segment
    const int th = threadIdx.x;
    const uint32_t per = (nb + kScanT - 1) / kScanT;
    const uint32_t a = min(nb, th * per), b = min(nb, a + per);
    unsigned long long s = 0;
    for (uint32_t i = a; i < b; ++i) s += sums[i];
    part[th] = s;
    __syncthreads();
    for (int off = 1; off < kScanT; off <<= 1) {
        const unsigned long long v = th >= off ? part[th - off] : 0ull;
        __syncthreads();
        part[th] += v;
        __syncthreads();
    }
    unsigned long long run = part[th] - s;
    for (uint32_t i = a; i < b; ++i) {
        const unsigned long long v = sums[i];
        sums[i] = run;
        run += v;
    }
}

// out[i] = sums[block] + (exclusive prefix of in inside the block); element order is
// q-major across the block's threads: i = b0 + q * kScanT + thread
template <typename C, typename O>
__global__ void __launch_bounds__(kScanT) k_scan_apply(const C* in, uint64_t n,
                                                      const unsigned long long* __restrict__ sums,
                                                      O* out, uint64_t seg_stride = 0) {  // in == out allowed
    __shared__ unsigned long long ws[kScanT / 32];
    __shared__ unsigned long long carry;
    in += blockIdx.y * seg_stride;
    out += blockIdx.y * seg_stride;
    sums += blockIdx.y * gridDim.x;
    const uint64_t b0 = static_cast<uint64_t>(blockIdx.x) * kScanBlock;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = sums[blockIdx.x];
    __syncthreads();
    for (int q = 0; q < kScanItems; ++q) {
        const uint64_t i = b0 + static_cast<uint64_t>(q) * kScanT + threadIdx.x;
        const unsigned long long v = i < n ? static_cast<unsigned long long>(in[i]) : 0ull;
        unsigned long long x = v;  // inclusive warp scan
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) ws[w] = x;
        __syncthreads();
        if (w == 0) {
            unsigned long long u = ws[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, u, o);
                if (lane >= o) u += y;
            }
            ws[lane] = u;  // inclusive over warps
        }
        __syncthreads();
        const unsigned long long wprev = w ? ws[w - 1] : 0ull;
        if (i < n) out[i] = static_cast<O>(carry + wprev + x - v);
        __syncthreads();
        if (threadIdx.x == kScanT - 1) carry += ws[kScanT / 32 - 1];
        __syncthreads();
    }
}

}  // namespace

void exclusive_scan_u32_inplace(uint32_t* a, uint64_t n, int nseg, uint64_t seg_stride,
                                unsigned long long* scratch, cudaStream_t s);

size_t radix_sort_scratch_bytes(uint64_t max_len, int nseg) {
    const uint64_t T = (std::max<uint64_t>(max_len, 1) + kSortTile - 1) / kSortTile;
    const size_t counts = sizeof(uint32_t) * static_cast<size_t>(nseg) * kRadix * T;
    // two count buffers + the block sums of the counts' scan (16-byte aligned)
    const uint64_t nb = (static_cast<uint64_t>(kRadix) * T + kScanBlock - 1) / kScanBlock;
    return 2 * ((counts + 15) & ~size_t(15)) + 8 * (static_cast<size_t>(nseg) * nb + 2);
}

// counts of up to this many per segment are scanned by one block in one launch
constexpr uint64_t kSmallScan = 32 * 1024;

template <typename V, typename N>
bool radix_sort_pairs(uint32_t* keys, V* vals, uint32_t* keys_alt, V* vals_alt, size_t stride,
                      const N* d_n, uint64_t max_len, int nseg, int end_bit, uint32_t* scratch,
                      cudaStream_t s) {
    if (max_len == 0 || nseg == 0) return false;
    const int T = static_cast<int>((max_len + kSortTile - 1) / kSortTile);
    const dim3 grid(static_cast<unsigned>(T), static_cast<unsigned>(nseg));
    const uint64_t per = static_cast<uint64_t>(kRadix) * T;  // counts per segment
    const size_t cb = ((sizeof(uint32_t) * static_cast<size_t>(nseg) * per) + 15) & ~size_t(15);
    // two count buffers: this pass's (scanned) and the next pass's (built by the scatter)
    uint32_t* cnt[2] = {scratch, reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(scratch) + cb)};
    unsigned long long* sums = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(scratch) + 2 * cb);
    const bool small = per <= kSmallScan;
    // Small arrays (latency-bound, e.g. a single rendered view): the scatter also builds the next
    // pass's histogram (global atomics) and one block scans the counts, so a pass is two
    // launches. Large arrays: a histogram kernel per pass (the atomics would contend) and the
    // multi-block scan.
    bool alt = false;
    int c = 0;
    if (small) k_sort_hist<N><<<grid, kSortThreads, 0, s>>>(keys, stride, d_n, 0, T, cnt[0]);
    for (int shift = 0; shift < end_bit; shift += 8) {
        const uint32_t* ki = alt ? keys_alt : keys;
        const V* vi = alt ? vals_alt : vals;
        uint32_t* ko = alt ? keys : keys_alt;
        V* vo = alt ? vals : vals_alt;
        const bool more = shift + 8 < end_bit;
        if (small) {  // one block per segment; it also clears the next pass's counts
            k_scan_small<<<nseg, kScanT, 0, s>>>(cnt[c], per, per, more ? cnt[c ^ 1] : nullptr);
            k_sort_scatter<V, N><<<grid, kSortThreads, 0, s>>>(ki, vi, ko, vo, stride, d_n, shift, T, cnt[c],
                                                               more ? cnt[c ^ 1] : nullptr);
            c ^= 1;
        } else {
            k_sort_hist<N><<<grid, kSortThreads, 0, s>>>(ki, stride, d_n, shift, T, cnt[0]);
            exclusive_scan_u32_inplace(cnt[0], per, nseg, per, sums, s);
            k_sort_scatter<V, N><<<grid, kSortThreads, 0, s>>>(ki, vi, ko, vo, stride, d_n, shift, T, cnt[0],
                                                               nullptr);
        }
        alt = !alt;
    }
    return alt;
}

template bool radix_sort_pairs<uint32_t, uint32_t>(uint32_t*, uint32_t*, uint32_t*, uint32_t*, size_t,
                                                   const uint32_t*, uint64_t, int, int, uint32_t*,
                                                   cudaStream_t);
template bool radix_sort_pairs<unsigned long long, unsigned long long>(
    uint32_t*, unsigned long long*, uint32_t*, unsigned long long*, size_t, const unsigned long long*,
    uint64_t, int, int, uint32_t*, cudaStream_t);

int radix_sort_launches(int end_bit, uint64_t max_len) {
    const uint64_t T = (std::max<uint64_t>(max_len, 1) + kSortTile - 1) / kSortTile;
    const bool small = static_cast<uint64_t>(kRadix) * T <= kSmallScan;
    return small ? 1 + ((end_bit + 7) / 8) * 2 : ((end_bit + 7) / 8) * 5;
}

int exclusive_scan_launches(uint64_t n) { return n <= kSmallScanU64 ? 1 : 3; }

size_t exclusive_scan_scratch_bytes(uint64_t n) {
    return sizeof(unsigned long long) * ((std::max<uint64_t>(n, 1) + kScanBlock - 1) / kScanBlock + 1);
}

// one block, one launch: exclusive scan of n counts into u64 offsets (small n)
template <typename C>
__global__ void __launch_bounds__(kScanT) k_scan_small_u64(const C* __restrict__ in, uint64_t n,
                                                          unsigned long long* __restrict__ out) {
    __shared__ unsigned long long ws[kScanT / 32];
    __shared__ unsigned long long carry;
    if (threadIdx.x == 0) carry = 0ull;
    __syncthreads();
    for (uint64_t b0 = 0; b0 < n; b0 += static_cast<uint64_t>(kScanT) * kSmallItems) {
        const uint64_t i0 = b0 + static_cast<uint64_t>(threadIdx.x) * kSmallItems;
        unsigned long long v[kSmallItems];
        unsigned long long sum = 0;
#pragma unroll
        for (int q = 0; q < kSmallItems; ++q) {
            v[q] = i0 + q < n ? static_cast<unsigned long long>(in[i0 + q]) : 0ull;
            sum += v[q];
        }
        unsigned long long run = block_exclusive<unsigned long long>(sum, ws, &carry);
#pragma unroll
        for (int q = 0; q < kSmallItems; ++q)
            if (i0 + q < n) {
                out[i0 + q] = run;
                run += v[q];
            }
    }
}

template <typename C>
void exclusive_scan_u64(const C* in, uint64_t n, unsigned long long* out, unsigned long long* scratch,
                        cudaStream_t s) {
    if (n == 0) return;
    if (n <= kSmallScanU64) {
        k_scan_small_u64<C><<<1, kScanT, 0, s>>>(in, n, out);
        return;
    }
    const uint32_t nb = static_cast<uint32_t>((n + kScanBlock - 1) / kScanBlock);
    k_scan_sums<C><<<nb, kScanT, 0, s>>>(in, n, scratch);
    k_scan_top<<<1, kScanT, 0, s>>>(scratch, nb);
    k_scan_apply<C, unsigned long long><<<nb, kScanT, 0, s>>>(in, n, scratch, out);
}

// in-place exclusive scan of nseg arrays of n u32 counts each, seg_stride apart (the sort's
// digit-major tile counts per segment)
void exclusive_scan_u32_inplace(uint32_t* a, uint64_t n, int nseg, uint64_t seg_stride,
                                unsigned long long* scratch, cudaStream_t s) {
    if (n == 0 || nseg == 0) return;
    const uint32_t nb = static_cast<uint32_t>((n + kScanBlock - 1) / kScanBlock);
    const dim3 g(nb, static_cast<unsigned>(nseg));
    k_scan_sums<uint32_t><<<g, kScanT, 0, s>>>(a, n, scratch, seg_stride);
    k_scan_top<<<nseg, kScanT, 0, s>>>(scratch, nb);
    k_scan_apply<uint32_t, uint32_t><<<g, kScanT, 0, s>>>(a, n, scratch, a, seg_stride);
}

template void exclusive_scan_u64<uint32_t>(const uint32_t*, uint64_t, unsigned long long*,
                                           unsigned long long*, cudaStream_t);
template void exclusive_scan_u64<unsigned long long>(const unsigned long long*, uint64_t,
                                                     unsigned long long*, unsigned long long*,
                                                     cudaStream_t);

}  // namespace sgm
