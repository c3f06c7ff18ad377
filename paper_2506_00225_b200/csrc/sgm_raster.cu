// K4 / K5: the tile compositor (render) and the candidate scorer (score) for sm_100a.
//
// Reference: proj/src/splat_render.cpp:254-324 (compositor), :360-369
// (clipped_entropy), proj/src/explorer.cpp:195-203 (per-view n_missing and
// entropy sum). Built with --fmad=false; the only fused operations are the ones
// written explicitly (__fma_rn) below: the semantic scatter and the exp
// polynomial. Both stay within ~1 ulp of the reference's fp64 arithmetic.
//
// One CTA = 8 compute warps + 1 loader warp; it blends kItemsPerCta consecutive 8x8 pixel
// blocks (of one view, or crossing into the next). Per block, the loader forms batches of
// kNB Gaussians (depth order) two ahead and streams their rows through shared memory
// (double-buffered: cp.async.bulk copies completing on an mbarrier for score launches, 16-byte
// cp.async chunks for render launches); per batch the compute warps run
//   phase AB footprints and the exact transmittance chain, fused: thread (part, px) owns 4
//            contiguous entries of pixel px; segment products meet in shared memory
//            (render with retained contributor lists: footprints, then the sequential
//            per-pixel chain, so the lists come out in depth order);
//   phase C  the sparse semantic scatter. Warp g owns channel group g (C/8 channels) for
//            all 64 pixels, two pixels per lane, so no two warps touch the same
//            accumulator word. The accumulator is [C][32] double2 in shared memory (lane l
//            holds pixels 2l, 2l+1): one LDS.128 / 2 DFMA / STS.128 per (Gaussian, class)
//            entry covers the whole 8x8 block, and a warp's lanes hit 32 consecutive
//            16-byte words (no bank conflict). With k >= 24 classes per Gaussian the score
//            launch keeps groups 4-7 in tensor memory instead (kTm: tcgen05.ld/st, the same
//            two pixels per lane), off the shared-memory pipe.
// While the compute warps run a block's epilogue the loader stages the next block's first
// batch.
// Score epilogue: per (pixel, group) S1 = sum c, S2 = sum c ln c with
// c = clamp(p, 1e-3, 1) (a 128-entry table log, ~1 ulp); H = ln S1 - S2/S1
// (== -sum q ln q, q = c / S1); the tile's
// entropy and exact-zero-silhouette count go to a per-tile slot that a second
// kernel sums in a fixed order (deterministic, batching/sharding-invariant).
#include <algorithm>
#include <cstdlib>
#include <stdexcept>

#include "sgm_internal.h"
#include "sgm_device.cuh"

namespace sgm {

namespace {

constexpr int kCompute = 256;           // compute threads: warps 0-7
constexpr int kWarps = kCompute / 32;
constexpr int kThreads = kCompute + 32;  // + warp 8, the batch loader
constexpr int kNB = 16;            // Gaussians per staged batch
constexpr int kGroups = kWarps;    // channel groups: one warp each in phase C
// (view, block) items blended by one CTA in sequence. Measured on cfg1 (ms per 64 views):
// 1: 81.1, 2: 78.5, 4: 77.7, 8: 78.0, 16: 79.5; a persistent grid (one wave, items from an
// atomic counter) took 88.3, its CTAs holding the SMs the binning stream needs.
constexpr int kItemsPerCta = 4;

__host__ __device__ constexpr int align16(int b) { return (b + 15) & ~15; }

// barrier over the 8 compute warps only (the loader warp runs ahead between the per-batch
// block barriers)
__device__ __forceinline__ void compute_sync() { asm volatile("bar.sync 1, %0;\n" ::"n"(kCompute) : "memory"); }

struct Layout {  // byte offsets in dynamic shared memory
    int acc, w, segp, tpx, done, rm, stage0, stage_bytes, st_packed, st_bnd, st_idx, st_prob,
        st_color, total;
};

// accumulator row pitch in double2 units (render: +1 so the transposed write-out
// of the [channel][pixel] tile to the reference's [pixel][channel] layout is
// nearly conflict-free)
__host__ __device__ constexpr int acc_pitch(bool render) { return render ? 33 : 32; }

__host__ __device__ inline Layout make_layout(int C, int kpad, bool render, bool color = false, bool recs = false) {
    Layout L;
    L.acc = 0;
    L.w = align16(C * acc_pitch(render) * 16);
    L.segp = L.w + kNB * kTilePx * 8;          // [4][64] segment products (score phase B)
    L.tpx = L.segp + 4 * kTilePx * 8;          // [64] pixel transmittance
    L.done = L.tpx + kTilePx * 8;
    L.rm = L.done + kTilePx * 4;
    L.stage0 = L.rm + 2 * kNB * 8;
    L.st_packed = 0;
    L.st_bnd = kNB * static_cast<int>(sizeof(PackedSplat));      // [kNB] uint4 group bounds
    L.st_idx = L.st_bnd + kNB * 16;
    if (recs) {  // the 4-CTA score launch stages 16-byte records (DevMap::sem_rec)
        L.st_prob = L.st_idx;
        L.st_color = L.st_idx + kNB * kpad * 16;
    } else {
        L.st_prob = L.st_idx + kNB * kpad * 2;
        L.st_color = L.st_prob + kNB * kpad * 8;
    }
    L.stage_bytes = L.st_color + ((render || color) ? kNB * 32 : 0);
    L.total = L.stage0 + 2 * L.stage_bytes;
    // the score epilogue's per-(group, pixel) (S1, S2) exchange reuses the stages
    const int red = kGroups * kTilePx * 16;
    if (L.total < L.stage0 + red) L.total = L.stage0 + red;
    return L;
}

// index of pixel q's slot in a [row][pitch2] double2 array viewed as doubles: lane l
// holds the horizontally adjacent pixels 2l, 2l+1, so quarter-warp j (lanes 8j..8j+7)
// covers tile rows 2j, 2j+1 and its shared-memory wavefront is skipped when none of
// those 16 pixels receives weight from an entry
__device__ __forceinline__ int pair_slot(int row, int pitch2, int q) {
    return row * pitch2 * 2 + q;
}

// Tile-local pixel index q -> (column, row) in the 8x8 block: q / 16 selects a 4x4
// quadrant, so a quarter-warp (lanes 8j .. 8j+7, pixels 16j .. 16j+15) covers a compact
// 4x4 square: a Gaussian's disc leaves more quarter-warps without weight (and their
// shared-memory wavefronts skipped) than with row pairs. Horizontal pairs (2l, 2l+1) stay
// adjacent.
__device__ __forceinline__ int px_col(int q) { return ((q >> 4) & 1) * 4 + (q & 3); }
__device__ __forceinline__ int px_row(int q) { return (q >> 5) * 4 + ((q >> 2) & 3); }

// kRc (score mode): also accumulate each pixel's rendered colour and depth, written to
// vd.rc4[px][4] (the Fisher gain's pass-0 quantity, losses.cpp:285-288)
// kOcc: CTAs per SM the register budget is sized for; 4 when the shared-memory footprint
// allows it (small C, e.g. cfg3's 42 channels), else 3 (the 102-channel accumulator).
//
// Each CTA blends p.items_per_cta consecutive (view, block) items; the loader warp stages
// the next block's first batch while the compute warps run the current block's epilogue.
// (Not a persistent grid: CTAs still retire often enough for the prioritised binning
// stream's kernels to take their slots.)
// kItems: the depth-prefix binning launch (explicit item list, truncated-list flags and the
// incomplete-tile report); a separate instantiation, so the common launches carry none of it.
// kTm (3-CTA score launches): channel groups 4-7 accumulate in tensor memory (tcgen05.ld/st,
// one 32-lane quarter per warp) instead of shared memory, so their read-modify-writes leave
// the shared-memory pipe to the other groups, the staged weights and rows.
template <bool kRender, bool kDup, bool kAniso, bool kRc = false, int kOcc = 3, bool kItems = false,
          bool kRefDiv = false, bool kTm = false>
__global__ void __launch_bounds__(kThreads, kOcc) k_raster(RasterParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int C = p.map.C;
    const int kpad = p.map.kpad;
    const int Cg = p.groups.Cg;
    constexpr int apitch = acc_pitch(kRender);
    static_assert(!(kRc && kRender), "rc4 is a score-mode output");
    constexpr bool kRecs = !kRender && !kRc && kOcc == 4;  // (and kBulk)
    const Layout L = make_layout(C, kpad, kRender, kRc, kRecs);
    double2* acc2 = reinterpret_cast<double2*>(smem + L.acc);     // [C][apitch]
    double* acc = reinterpret_cast<double*>(smem + L.acc);
    double* W = reinterpret_cast<double*>(smem + L.w);             // [kNB][32] double2
    const double2* W2 = reinterpret_cast<const double2*>(smem + L.w);
    double* segp = reinterpret_cast<double*>(smem + L.segp);       // [4][64]
    double* sT = reinterpret_cast<double*>(smem + L.tpx);          // [64]
    int* sdone = reinterpret_cast<int*>(smem + L.done);            // [64]
    uint2* rm = reinterpret_cast<uint2*>(smem + L.rm);             // [2][kNB] (rank, map index)
    unsigned char* stg = smem + L.stage0;
    // epilogue exchanges reuse the weight buffer (the stages then hold the next block's
    // first batch): [kGroups][64] double2 (entropy) or [4][64][4] double (colour / depth)
    double2* red = reinterpret_cast<double2*>(smem + L.w);
    double* rcx = reinterpret_cast<double*>(smem + L.w);

    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const bool loader = warp == kWarps;
    const int px = t & (kTilePx - 1);  // this thread's pixel in phase A / B / epilogues
    const int g = warp;                // phase C / epilogue channel group
    const int c0 = g * Cg, c1 = min(C, c0 + Cg);
    const int tpv = p.tiles_per_view;
    const int total = p.n_items;

    __shared__ int scnt[2][3];  // block parity q: entries of batch b in scnt[q][b % 3]
    __shared__ uint32_t slive[2];  // batch b: entries with a nonzero weight at some pixel
    __shared__ int s_item;
    __shared__ uint8_t s_trunc[2];  // the block's bin list is a strict prefix (depth-prefix binning)
    __shared__ int s_exh;           // the block's list ran out with pixels still open
    __shared__ int s_view;          // (kItems) the block's view, for thread 0's epilogue
    __shared__ uint32_t s_tbase;    // (kTm) the CTA's tensor-memory columns
    __shared__ double red_d[2];                        // epilogue: the two pixel warps' entropy
    __shared__ unsigned long long red_u[2 + kWarps];   // their missing counts, then K per warp

    // ---- loader state (in shared memory, so the compute warps carry no registers for it):
    // the block it stages for, the current one and then the next ----
    struct LoaderState {
        const uint32_t* list;
        const PackedSplat* packed;
        const uint32_t* order;
        uint32_t L0, Ln, cursor;  // cursor: next bin entry to examine
        float bx0, bx1, by0, by1;
        int q;  // parity of the loader's block
    };
    __shared__ LoaderState ls;
    // batch b's records and rows into stage b & 1: per entry one bulk copy (TMA engine) per
    // record (PackedSplat 64 B, channel-group bounds 16 B, class row 2 kpad B, probability
    // row 8 kpad B, colour 32 B), completing on the stage's mbarrier (expected bytes armed
    // first). The loader alone waits on it, before the batch barrier that hands the stage
    // to the compute warps.
    __shared__ __align__(8) unsigned long long s_mbar[2];
    // (render launches keep 16-byte cp.async chunks: their larger register footprint spills
    // with the bulk-copy loader; the colour-writing score launch of the Fisher gain spills too,
    // but is faster with it: 423 -> 431 views/s)
    constexpr bool kBulk = !kRender;
    const int qi = kpad / 8, qp = kpad / 2;
    const int Q = 5 + qi + qp + ((kRender || kRc) ? 2 : 0);  // 16-byte chunks per Gaussian
    auto issue = [&](int b) {
        const int st = b & 1;
        unsigned char* sb = stg + st * L.stage_bytes;
        const int n = scnt[ls.q][b % 3];
        if constexpr (kBulk) {
            const uint32_t bar = smem_addr(&s_mbar[st]);
            if (lane == 0)
                mbar_expect_tx(bar, static_cast<unsigned>(n) * (64u + 16u + (kRecs ? 16u : 10u) * static_cast<unsigned>(kpad) +
                                                               (kRc ? 32u : 0u)));
            __syncwarp();
            if (lane < n) {
                const uint2 v = rm[st * kNB + lane];
                // the stage was last read (generic proxy) before the barrier this warp passed
                fence_proxy_async();
                bulk_g2s(sb + L.st_packed + lane * 64, ls.packed + v.x, 64u, bar);
                bulk_g2s(sb + L.st_bnd + lane * 16, p.map.gbounds + v.y, 16u, bar);
                if (kRc) bulk_g2s(sb + L.st_color + lane * 32, p.map.color4 + static_cast<size_t>(v.y) * 4, 32u, bar);
                if (kRecs) {
                    bulk_g2s(sb + L.st_idx + lane * kpad * 16, p.map.sem_rec + static_cast<size_t>(v.y) * kpad,
                             16u * kpad, bar);
                } else {
                    bulk_g2s(sb + L.st_idx + lane * kpad * 2, p.map.sem_idx + static_cast<size_t>(v.y) * kpad,
                             2u * kpad, bar);
                    bulk_g2s(sb + L.st_prob + lane * kpad * 8, p.map.sem_prob + static_cast<size_t>(v.y) * kpad,
                             8u * kpad, bar);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(bar);
        } else {
            const unsigned qmagic = static_cast<unsigned>((0x100000000ull + Q - 1) / Q);  // ceil(2^32 / Q)
            const uint2* slot = rm + st * kNB;
            for (int c = lane; c < n * Q; c += 32) {
                // c / Q by a multiply-high (exact: c < kNB * Q is far below 2^32 / Q^2)
                const int e = static_cast<int>(__umulhi(static_cast<unsigned>(c), qmagic));
                int q = c - e * Q;
                const uint2 v = slot[e];
                const unsigned char* src;
                unsigned char* dst;
                if (q < 4) {
                    src = reinterpret_cast<const unsigned char*>(ls.packed + v.x) + 16 * q;
                    dst = sb + L.st_packed + e * 64 + 16 * q;
                } else if (q == 4) {
                    src = reinterpret_cast<const unsigned char*>(p.map.gbounds + v.y);
                    dst = sb + L.st_bnd + e * 16;
                } else if ((q -= 5) < qi) {
                    src = reinterpret_cast<const unsigned char*>(p.map.sem_idx + static_cast<size_t>(v.y) * kpad) + 16 * q;
                    dst = sb + L.st_idx + e * kpad * 2 + 16 * q;
                } else if ((q -= qi) < qp) {
                    src = reinterpret_cast<const unsigned char*>(p.map.sem_prob + static_cast<size_t>(v.y) * kpad) + 16 * q;
                    dst = sb + L.st_prob + e * kpad * 8 + 16 * q;
                } else {
                    q -= qp;
                    src = reinterpret_cast<const unsigned char*>(p.map.color4 + static_cast<size_t>(v.y) * 4) + 16 * q;
                    dst = sb + L.st_color + e * 32 + 16 * q;
                }
                cp_async16(dst, src);
            }
            cp_async_commit();
        }
    };
    // Parity bits of the next mbarrier phase per stage. Compute threads: the phase of the next
    // batch they read from the stage (they wait on it after the batch barrier; the copies
    // were issued a whole batch earlier, so it is normally complete). Loader: the phase its
    // last copies into the stage complete (waited only for a batch the block never read).
    unsigned mphase = 0;
    auto wait_batch = [&](int b) {
        const int st = b & 1;
        mbar_wait(smem_addr(&s_mbar[st]), (mphase >> st) & 1u);
        mphase ^= 1u << st;
    };
    // Batches are formed by the loader warp two ahead (off the compute warps' path): the
    // next kNB entries of the bin (depth order) that can reach a pixel of this block. An
    // entry whose float probe circle (:276-278) misses the box of the block's pixel centres
    // by a relative margin above the probe's rounding cannot pass the prefilter at any
    // pixel, so skipping it changes nothing; about a fifth of the bin entries are such
    // corner entries of the square tile rectangle (:205-209). (The anisotropic mode has no
    // float probe: no skipping.)
    auto fill = [&](int b) {
        ViewDesc lv;
        lv.list = ls.list;
        lv.packed = ls.packed;
        lv.order = ls.order;
        uint32_t cursor = ls.cursor;
        const int filled = fill_batch<kNB>(lv, ls.L0, ls.Ln, cursor, rm + (b & 1) * kNB, !kAniso, ls.bx0,
                                           ls.bx1, ls.by0, ls.by1, lane);
        __syncwarp();
        if (lane == 0) {
            scnt[ls.q][b % 3] = filled;
            ls.cursor = cursor;
        }
        __syncwarp();
    };
    // claim the next block and stage its batch 0 (loader warp)
    int nclaimed = 0;
    auto claim = [&]() {
        const int it = nclaimed < p.items_per_cta ? blockIdx.x * p.items_per_cta + nclaimed : total;
        ++nclaimed;
        if (lane == 0) s_item = it;
        if (it >= total) return;
        int view, tile;
        if (kItems && p.item_list) {
            const uint2 vt = p.item_list[it];
            view = static_cast<int>(vt.x);
            tile = static_cast<int>(vt.y);
        } else {
            view = it / tpv;
            tile = it - view * tpv;
        }
        const ViewDesc* v = p.views + view;
        const int tbx = tile % p.raster_tiles_x, tby = tile / p.raster_tiles_x;
        const int bin = ((tby * kTile) / p.opt.ts) * p.opt.tiles_x + (tbx * kTile) / p.opt.ts;
        const uint2 rg = v->ranges[bin];
        if (lane == 0) {
            if (kItems)
                s_trunc[ls.q] = p.trunc ? p.trunc[static_cast<size_t>(view) * p.opt.tiles_x * p.opt.tiles_y + bin] : 0;
            ls.list = v->list;
            ls.packed = v->packed;
            ls.order = v->order;
            ls.L0 = rg.x;
            ls.Ln = rg.y - rg.x;
            ls.cursor = 0;
            ls.bx0 = static_cast<float>(tbx * kTile) + 0.5f;
            ls.bx1 = ls.bx0 + static_cast<float>(kTile - 1);
            ls.by0 = static_cast<float>(tby * kTile) + 0.5f;
            ls.by1 = ls.by0 + static_cast<float>(kTile - 1);
        }
        __syncwarp();
        fill(0);
        if (scnt[ls.q][0] > 0) issue(0);
    };

    if (t == 0) {
        mbar_init(smem_addr(&s_mbar[0]), 1);
        mbar_init(smem_addr(&s_mbar[1]), 1);
    }
    if constexpr (kTm) {
        if (warp == 0) tmem_alloc(&s_tbase);
        tmem_fence_before();
    }
    __syncthreads();
    if constexpr (kTm) tmem_fence_after();
    // (kTm) groups from p.tm_first on: this warp's lane quarter (warp % 4), channel c of the group
    // at columns 4 (c - c0), from column 0 for groups 4-7 and 64 for groups 0-3
    const bool tmg = kTm && g >= p.tm_first;
    const uint32_t tcol =
        kTm ? s_tbase + ((32u * static_cast<uint32_t>(warp & 3)) << 16) + (warp < 4 ? 64u : 0u) : 0u;
    if (loader) {
        if (lane == 0) ls.q = 0;
        __syncwarp();
        claim();
    }
    if (kItems && t == 0) s_exh = 0;
    __syncthreads();
    for (int q = 0;; q ^= 1) {  // q: parity of this block (the loader's lq matches it)
        const int item = s_item;
        if (item >= total) break;
        int view, tile;
        if (kItems && p.item_list) {
            const uint2 vt = p.item_list[item];
            view = static_cast<int>(vt.x);
            tile = static_cast<int>(vt.y);
        } else {
            view = item / tpv;
            tile = item - view * tpv;
        }
        const ViewDesc vd = p.views[view];
        if (kItems && t == 0) s_view = view;  // (not a register live across the block)
        const int bx = tile % p.raster_tiles_x, by = tile / p.raster_tiles_x;
        const int x = bx * kTile + px_col(px);
        const int y = by * kTile + px_row(px);
        const bool inside = x < p.cam.W && y < p.cam.H;
        const bool want_sem = !kRender || vd.sem != nullptr;
        if (!loader) {
            for (int i = t; i < C * apitch; i += kCompute) acc2[i] = make_double2(0.0, 0.0);
            if (tmg) {
                const uint32_t z[4] = {0u, 0u, 0u, 0u};
                for (int cc = 0; cc < c1 - c0; ++cc) tmem_st2(tcol + 4u * cc, z);
                tmem_wait_st();
            }
            if (t < kTilePx) {
                sdone[t] = inside ? 0 : 1;
                sT[t] = 1.0;
            }
            if (t < 2) slive[t] = 0u;
        }

        // render with retained contributor lists keeps the sequential per-pixel chain (the
        // lists are written in depth order); every other launch uses the fused segmented chain
        const bool seq = kRender && vd.contrib != nullptr;
        const double dpx = x + 0.5, dpy = y + 0.5;                                 // :261, :263
        const float fpx = static_cast<float>(dpx), fpy = static_cast<float>(dpy);  // :274
        // phase-B state (warps 0-1 own pixel t)
        double T = 1.0;
        double ac0 = 0.0, ac1 = 0.0, ac2 = 0.0, adep = 0.0;
        bool done = !inside;
        unsigned long long contrib = 0;
        uint32_t ncontrib_px = 0;  // retain_contributors: this pixel's list length so far
        const size_t pix_t = inside ? static_cast<size_t>(y) * p.cam.W + x : 0;
        const int e_first = t >> 6;  // phase A: this thread's entries e_first + 4i

        double rcs[4] = {0.0, 0.0, 0.0, 0.0};  // this (segment, pixel) thread's colour / depth
        int mine = loader ? 1 : 0;  // vote that this thread's pixel is done (the block stops when all are)
        for (int b = 0;; ++b) {
            if (!kBulk) cp_async_wait_all();  // (cp.async loader: batch b landed)
            // scnt for b+1 visible; W / bnd free; and the early termination of the whole
            // block (:312 for every pixel) decided on the previous batch's votes
            if (__syncthreads_and(mine)) {
                // batch b (if any) was issued but is never read: the loader waits for it before
                // the stage is used again
                if (kBulk && scnt[q][b % 3] > 0) {
                    if (loader)
                        wait_batch(b);
                    else
                        mphase ^= 1u << (b & 1);
                }
                break;
            }
            const int n = scnt[q][b % 3];
            if (n == 0) {  // the bin is exhausted with pixels still open
                if (kItems && t == 0) s_exh = 1;
                break;
            }
            if (loader) {  // batch b+1 in flight while the compute warps blend batch b
                if (kBulk) mphase ^= 1u << (b & 1);  // (batch b's phase: completed for the compute warps)
                if (b == 0) fill(1);
                if (scnt[q][(b + 1) % 3] > 0) issue(b + 1);
                fill(b + 2);  // rm slot b & 1 (batch b was issued last iteration), scnt[q][(b + 2) % 3]
                continue;
            }
            if (kBulk) wait_batch(b);  // batch b's bulk copies have landed
            if (t == 0) slive[(b + 1) & 1] = 0u;  // last read by phase C of batch b - 1
            const unsigned char* sb = stg + (b & 1) * L.stage_bytes;
            const PackedSplat* sp = reinterpret_cast<const PackedSplat*>(sb + L.st_packed);
            const uint16_t* sbnd = reinterpret_cast<const uint16_t*>(sb + L.st_bnd);  // [kNB][8]
            const uint16_t* si = reinterpret_cast<const uint16_t*>(sb + L.st_idx);
            const double* spr = reinterpret_cast<const double*>(sb + L.st_prob);
            const uint4* srec = reinterpret_cast<const uint4*>(sb + L.st_idx);  // (kRecs)
            const double* scol = reinterpret_cast<const double*>(sb + L.st_color);

            // footprint of entry e at this thread's pixel (:276-285); -1 = not a contributor
            auto footprint = [&](int e) -> double {
                double f = -1.0;
                if (kAniso) {
                    // f4 (no reference): f = alpha exp(-q / 2), q = d^T Sigma2D^-1 d, cut at
                    // q > trunc^2 -- the order of oracle/sgm_oracle.c composite()
                    const PackedSplatA& a = reinterpret_cast<const PackedSplatA&>(sp[e]);
                    const double dx = dpx - a.mx;
                    const double dy = dpy - a.my;
                    const double qf = (a.qa * (dx * dx) + (2.0 * a.qb) * (dx * dy)) + a.qc * (dy * dy);
                    if (!(qf > p.opt.cut_sq)) {
                        f = a.alpha * exp_footprint(-0.5 * qf);
                        if (f > kMaxFootprint) f = kMaxFootprint;
                    }
                } else {
                    const float4 pf = *reinterpret_cast<const float4*>(&sp[e].pmx);
                    const float fdx = fpx - pf.x;
                    const float fdy = fpy - pf.y;
                    if (!(fdx * fdx + fdy * fdy > pf.z)) {  // :276-278
                        const double dx = dpx - sp[e].mx;
                        const double dy = dpy - sp[e].my;
                        const double d2 = dx * dx + dy * dy;
                        if (!(d2 > sp[e].cutoff_d2)) {  // :283
                            if (kRefDiv) {
                                // render_reference (:90-92): exp(-d2 / (2 r^2)), f <= 0 skipped
                                f = sp[e].alpha * exp_footprint(-d2 / sp[e].inv_two_r2);
                                if (f > kMaxFootprint) f = kMaxFootprint;
                                if (!(f > 0.0)) f = -1.0;
                            } else {
                                f = sp[e].alpha * exp_footprint(-d2 * sp[e].inv_two_r2);  // :284
                                if (f > kMaxFootprint) f = kMaxFootprint;                 // :285
                            }
                        }
                    }
                }
                return f;
            };

            uint32_t nzbits = 0;  // entries this thread gave a nonzero weight
            if (seq) {
                // ---- phase A: footprints (independent of T) ----
                {
                    const bool pdone = sdone[px] != 0;
#pragma unroll
                    for (int i = 0; i < kNB / 4; ++i) {
                        const int e = e_first + 4 * i;
                        if (e >= n) break;
                        W[pair_slot(e, 32, px)] = pdone ? -1.0 : footprint(e);
                    }
                }
                compute_sync();
                // ---- phase B: transmittance chain (:286-312), sequential per pixel (warps
                // 0-1): colour/depth and the ordered contributor lists of retain_contributors ----
                if (t < kTilePx) {
                    for (int e = 0; e < n; ++e) {
                        const int s = pair_slot(e, 32, t);
                        const double f = W[s];
                        if (done || f < 0.0) {
                            W[s] = 0.0;
                            continue;
                        }
                        const double w = f * T;
                        W[s] = w;
                        if (vd.contrib) {  // retain_contributors (:310): depth ranks in order
                            if (vd.contrib_offset)
                                vd.contrib[vd.contrib_offset[pix_t] + ncontrib_px] = sp[e].aux;
                            ++ncontrib_px;
                        }
                        ac0 += scol[4 * e] * w;  // :289-291 (colour clamped at upload)
                        ac1 += scol[4 * e + 1] * w;
                        ac2 += scol[4 * e + 2] * w;
                        adep += sp[e].z * w;  // :293
                        ++contrib;
                        T = T * (1.0 - f);                        // :311
                        if (p.opt.early_exit && T < p.opt.eps)   // :312
                            done = true;
                        if (w != 0.0) nzbits |= 1u << e;
                    }
                    sdone[t] = done ? 1 : 0;
                }
            } else {
                // ---- footprints and transmittance fused. Thread (part, px) owns the
                // contiguous entries 4 part .. 4 part + 3 of pixel px (warp-uniform entries).
                // A segment starts at T_pixel * prod(earlier segments' (1 - f)) (fixed
                // association); since T only decreases, a segment starting below eps lies
                // after the early exit (:312). The pixel's T and done flag are read before the
                // barrier and written (by the exiting or the last segment) after it. ----
                const int part = t >> 6;
                const bool pdone = sdone[px] != 0;
                const double T0 = sT[px];
                double f[4];
                double prod = 1.0;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int e = 4 * part + i;
                    f[i] = (e < n && !pdone) ? footprint(e) : -1.0;
                    if (f[i] >= 0.0) prod = prod * (1.0 - f[i]);
                }
                segp[part * kTilePx + px] = prod;
                compute_sync();
                double Ts = T0;
#pragma unroll
                for (int k = 0; k < 3; ++k)
                    if (k < part) Ts = Ts * segp[k * kTilePx + px];
                bool exited = pdone || (p.opt.early_exit && Ts < p.opt.eps);
                double Tc = Ts;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int e = 4 * part + i;
                    if (e >= n) break;
                    const int s = pair_slot(e, 32, px);
                    if (exited || f[i] < 0.0) {
                        W[s] = 0.0;
                        continue;
                    }
                    const double wv = f[i] * Tc;
                    W[s] = wv;
                    if (wv != 0.0) nzbits |= 1u << e;
                    if (kRc || kRender) {  // this segment's share of the colour / depth (:289-293)
                        rcs[0] += scol[4 * e] * wv;
                        rcs[1] += scol[4 * e + 1] * wv;
                        rcs[2] += scol[4 * e + 2] * wv;
                        rcs[3] += sp[e].z * wv;
                    }
                    ++contrib;
                    Tc = Tc * (1.0 - f[i]);
                    if (p.opt.early_exit && Tc < p.opt.eps) exited = true;
                }
                // The pixel's T after the batch: the T of the segment where it exits (at most
                // one segment can: the later ones start below eps), else the last segment's. A
                // pixel done before the batch keeps its T. So the silhouette 1 - T is the
                // reference's.
                const bool start_exited = pdone || (p.opt.early_exit && Ts < p.opt.eps);
                if ((!start_exited && exited) || (part == 3 && !start_exited)) {
                    sT[px] = Tc;
                    sdone[px] = exited ? 1 : 0;
                }
            }
            {
                const uint32_t lv = __reduce_or_sync(0xffffffffu, nzbits);
                if (lane == 0 && lv) atomicOr(&slive[b & 1], lv);
            }
            compute_sync();

            // ---- phase C: sparse semantic scatter; warp g = channel group g, 64 px ----
            if (want_sem) {
                double2* accl = acc2 + lane;
                // the live entries (some pixel weighted) with classes in this warp's group, in
                // depth order (lane l tests entry l)
                const int glo = (lane < n && g > 0) ? sbnd[lane * 8 + g - 1] : 0;
                const int ghi = lane < n ? sbnd[lane * 8 + g] : 0;
                const uint32_t gb = static_cast<uint32_t>(glo) | (static_cast<uint32_t>(ghi) << 16);
                uint32_t todo = __ballot_sync(0xffffffffu, ghi > glo) & slive[b & 1];
                while (todo) {
                    const int e = __ffs(todo) - 1;
                    todo &= todo - 1u;
                    const double2 w = W2[e * 32 + lane];
                    const uint32_t be = __shfl_sync(0xffffffffu, gb, e);  // entry e's group bounds
                    const int lo = static_cast<int>(be & 0xffffu), hi = static_cast<int>(be >> 16);
                    const bool nz = (w.x != 0.0) | (w.y != 0.0);
                    const uint16_t* ei = si + e * kpad;
                    const double* ep = spr + e * kpad;
                    const uint4* er = srec + e * kpad;
                    // slot j's (class, probability): one broadcast LDS.128 of the record (kRecs)
                    auto cls = [&](int j, double& pj) -> int {
                        if constexpr (kRecs) {
                            const uint4 r = er[j];
                            pj = __hiloint2double(static_cast<int>(r.y), static_cast<int>(r.x));
                            return static_cast<int>(r.z);
                        } else {
                            pj = ep[j];
                            return ei[j];
                        }
                    };
                    // lanes without weight skip the read-modify-writes: predicated shared loads
                    // and stores (no branch, the warp stays converged), so their quarter-warps
                    // issue no wavefronts; the FMAs on the unloaded registers are discarded
                    const unsigned pz = nz ? 1u : 0u;
                    auto rmw = [&](int c, double pj) {
                        double2* a = accl + c * apitch;
                        const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(a));
                        double vx, vy;
                        asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q ld.shared.v2.f64 {%0, %1}, [%3]; }"
                                     : "=d"(vx), "=d"(vy) : "r"(pz), "r"(sa) : "memory");
                        vx = __fma_rn(pj, w.x, vx);  // :307
                        vy = __fma_rn(pj, w.y, vy);
                        asm volatile("{ .reg .pred q; setp.ne.u32 q, %0, 0; @q st.shared.v2.f64 [%1], {%2, %3}; }"
                                     :: "r"(pz), "r"(sa), "d"(vx), "d"(vy) : "memory");
                    };
                    if (tmg) {
                        // tensor memory: every lane takes part (.sync.aligned); a weightless
                        // lane adds p * 0 = +0 to a nonnegative sum, which leaves it unchanged.
                        // Each store completes before the next load (a later entry may hit the
                        // same class).
                        int j = lo;
                        if (!kDup) {
#pragma unroll 1
                            for (; j + 2 <= hi; j += 2) {
                                double p0, p1;
                                const int ca = cls(j, p0), cb = cls(j + 1, p1);
                                uint32_t ra[4], rb[4];
                                tmem_ld2(tcol + 4u * static_cast<uint32_t>(ca - c0), ra);
                                tmem_ld2(tcol + 4u * static_cast<uint32_t>(cb - c0), rb);
                                tmem_wait_ld();
                                double2 a = tmem_unpack(ra), bq = tmem_unpack(rb);
                                a.x = __fma_rn(p0, w.x, a.x);  // :307
                                a.y = __fma_rn(p0, w.y, a.y);
                                bq.x = __fma_rn(p1, w.x, bq.x);
                                bq.y = __fma_rn(p1, w.y, bq.y);
                                tmem_pack(a, ra);
                                tmem_pack(bq, rb);
                                tmem_st2(tcol + 4u * static_cast<uint32_t>(ca - c0), ra);
                                tmem_st2(tcol + 4u * static_cast<uint32_t>(cb - c0), rb);
                                tmem_wait_st();
                            }
                        }
#pragma unroll 1
                        for (; j < hi; ++j) {  // (repeated classes: one at a time, in order)
                            double pj;
                            const int c = cls(j, pj);
                            uint32_t r[4];
                            tmem_ld2(tcol + 4u * static_cast<uint32_t>(c - c0), r);
                            tmem_wait_ld();
                            double2 a = tmem_unpack(r);
                            a.x = __fma_rn(pj, w.x, a.x);
                            a.y = __fma_rn(pj, w.y, a.y);
                            tmem_pack(a, r);
                            tmem_st2(tcol + 4u * static_cast<uint32_t>(c - c0), r);
                            tmem_wait_st();
                        }
                    } else if (kDup) {
#pragma unroll 1
                        for (int j = lo; j < hi; ++j) {  // repeated classes: in order
                            double pj;
                            const int c = cls(j, pj);
                            rmw(c, pj);
                        }
                    } else {
                        int j = lo;
#pragma unroll 1
                        for (; j + 2 <= hi; j += 2) {  // two distinct classes: both loads first
                            double p0, p1;
                            const int c0 = cls(j, p0), c1 = cls(j + 1, p1);
                            const unsigned s0 = static_cast<unsigned>(__cvta_generic_to_shared(accl + c0 * apitch));
                            const unsigned s1 = static_cast<unsigned>(__cvta_generic_to_shared(accl + c1 * apitch));
                            double ax, ay, bx, by;
                            asm volatile("{ .reg .pred q; setp.ne.u32 q, %4, 0;\n"
                                         " @q ld.shared.v2.f64 {%0, %1}, [%5];\n"
                                         " @q ld.shared.v2.f64 {%2, %3}, [%6]; }"
                                         : "=d"(ax), "=d"(ay), "=d"(bx), "=d"(by)
                                         : "r"(pz), "r"(s0), "r"(s1) : "memory");
                            ax = __fma_rn(p0, w.x, ax);
                            ay = __fma_rn(p0, w.y, ay);
                            bx = __fma_rn(p1, w.x, bx);
                            by = __fma_rn(p1, w.y, by);
                            asm volatile("{ .reg .pred q; setp.ne.u32 q, %0, 0;\n"
                                         " @q st.shared.v2.f64 [%1], {%3, %4};\n"
                                         " @q st.shared.v2.f64 [%2], {%5, %6}; }"
                                         :: "r"(pz), "r"(s0), "r"(s1), "d"(ax), "d"(ay), "d"(bx), "d"(by)
                                         : "memory");
                        }
                        if (j < hi) {
                            double pj;
                            const int c = cls(j, pj);
                            rmw(c, pj);
                        }
                    }
                }
            }
            mine = seq ? ((t < kTilePx) ? (done ? 1 : 0) : 1) : sdone[px];
        }

        if (loader) {
            // every copy of this block has landed (read by the compute warps, or waited for
            // above) and the compute warps no longer read the stages: stage the next block's
            // batch 0
            if (lane == 0) ls.q ^= 1;
            __syncwarp();
            claim();
        } else {
            if (kRender) {
                if (!seq) {  // fused chain: the pixel's 4 segment sums in a fixed order, T from sT
                    const int part = t >> 6;
#pragma unroll
                    for (int ch = 0; ch < 4; ++ch) rcx[(part * kTilePx + px) * 4 + ch] = rcs[ch];
                    compute_sync();
                    if (t < kTilePx) {
                        double r4[4];
#pragma unroll
                        for (int ch = 0; ch < 4; ++ch)
                            r4[ch] = ((rcx[(0 * kTilePx + t) * 4 + ch] + rcx[(1 * kTilePx + t) * 4 + ch]) +
                                      rcx[(2 * kTilePx + t) * 4 + ch]) + rcx[(3 * kTilePx + t) * 4 + ch];
                        ac0 = r4[0];
                        ac1 = r4[1];
                        ac2 = r4[2];
                        adep = r4[3];
                        T = sT[t];
                    }
                }
                if (t < kTilePx && inside) {
                    const size_t pix = static_cast<size_t>(y) * p.cam.W + x;
                    if (vd.sil) vd.sil[pix] = 1.0 - T;  // :314
                    if (vd.color) {
                        vd.color[pix * 3] = ac0;
                        vd.color[pix * 3 + 1] = ac1;
                        vd.color[pix * 3 + 2] = ac2;
                    }
                    if (vd.depth) vd.depth[pix] = adep;
                    if (vd.contrib && !vd.contrib_offset) vd.contrib_count[pix] = ncontrib_px;
                }
                if (vd.sem) {  // warp per pixel, lanes over its C channels (coalesced rows)
                    for (int qq = warp; qq < kTilePx; qq += kWarps) {
                        const int qx = bx * kTile + px_col(qq);
                        const int qy = by * kTile + px_row(qq);
                        if (qx >= p.cam.W || qy >= p.cam.H) continue;
                        double* dst = vd.sem + (static_cast<size_t>(qy) * p.cam.W + qx) * C;
                        for (int c = lane; c < C; c += 32) dst[c] = acc[pair_slot(c, apitch, qq)];
                    }
                }
            } else {
                // clipped_entropy (:360-369) split by channel group: warp g, pixels 2 lane, 2 lane + 1
                double S1x = 0.0, S2x = 0.0, S1y = 0.0, S2y = 0.0;
                // a channel below the clamp at all 64 pixels (about a fifth of them) takes the
                // clamped constant's log once: the same operands, so the same sums
                const double lclamp = log_table(0.001);
#pragma unroll 2
                for (int c = c0; c < c1; ++c) {
                    double2 v;
                    if (tmg) {
                        uint32_t r[4];
                        tmem_ld2(tcol + 4u * static_cast<uint32_t>(c - c0), r);
                        tmem_wait_ld();
                        v = tmem_unpack(r);
                    } else {
                        v = acc2[c * apitch + lane];
                    }
                    const double ax = clamp_prob(v.x), ay = clamp_prob(v.y);
                    S1x += ax;
                    S1y += ay;
                    if (__all_sync(0xffffffffu, ax == 0.001 && ay == 0.001)) {
                        S2x = __fma_rn(0.001, lclamp, S2x);
                        S2y = __fma_rn(0.001, lclamp, S2y);
                    } else {
                        S2x = __fma_rn(ax, log_table(ax), S2x);
                        S2y = __fma_rn(ay, log_table(ay), S2y);
                    }
                }
                red[g * kTilePx + 2 * lane] = make_double2(S1x, S2x);
                red[g * kTilePx + 2 * lane + 1] = make_double2(S1y, S2y);
                compute_sync();
                if (t < kTilePx) {  // warps 0-1: pixel t
                    double S1 = 0.0, S2 = 0.0;
#pragma unroll
                    for (int k = 0; k < kGroups; ++k) {
                        S1 += red[k * kTilePx + t].x;
                        S2 += red[k * kTilePx + t].y;
                    }
                    double h = inside ? log(S1) - S2 / S1 : 0.0;
                    // fixed shuffle tree over the warp's 32 pixels: deterministic
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) h += __shfl_down_sync(0xffffffffu, h, o);
                    const unsigned m = __reduce_add_sync(0xffffffffu, (inside && 1.0 - sT[t] == 0.0) ? 1u : 0u);  // explorer.cpp:198
                    if (lane == 0) {
                        red_d[warp] = h;
                        red_u[warp] = m;
                    }
                }
            }
            // K (contributors) for the measurement counters: per-warp sums (integers, any order)
            {
                const unsigned cw = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(contrib));
                if (lane == 0) red_u[2 + warp] = cw;
            }
            compute_sync();
            if (t == 0) {
                if (!kRender) {
                    vd.ent_partial[tile] = red_d[0] + red_d[1];
                    vd.miss_partial[tile] = static_cast<uint32_t>(red_u[0] + red_u[1]);
                }
                // a truncated list ran out before every pixel exited: the tile is redone
                // from a longer depth prefix (its partials above are then overwritten)
                if (kItems) {
                    if (s_exh && s_trunc[q] && p.incomplete)
                        p.incomplete[static_cast<size_t>(s_view) * tpv + atomicAdd(p.n_incomplete + s_view, 1u)] =
                            static_cast<uint32_t>(tile);
                    s_exh = 0;
                }
                unsigned long long k = 0;
#pragma unroll
                for (int w = 0; w < kWarps; ++w) k += red_u[2 + w];
                if (vd.contributors && k) atomicAdd(vd.contributors, k);
            }
            if (kRc) {  // the pixel's colour / depth: its 4 segments summed in a fixed order
                const int part = t >> 6;
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) rcx[(part * kTilePx + px) * 4 + ch] = rcs[ch];
                compute_sync();
                if (t < kTilePx && inside) {
                    const size_t pix = static_cast<size_t>(y) * p.cam.W + x;
#pragma unroll
                    for (int ch = 0; ch < 4; ++ch)
                        vd.rc4[pix * 4 + ch] = ((rcx[(0 * kTilePx + t) * 4 + ch] + rcx[(1 * kTilePx + t) * 4 + ch]) +
                                                rcx[(2 * kTilePx + t) * 4 + ch]) + rcx[(3 * kTilePx + t) * 4 + ch];
                }
            }
        }
        // the epilogue is done with acc / W / red_u; the next block's item and batch 0 are staged
        __syncthreads();
    }
    if constexpr (kTm) {
        tmem_fence_before();
        __syncthreads();
        tmem_fence_after();
        if (warp == 0) tmem_dealloc(s_tbase);
    }
}

// The first channel group the 3-CTA score raster keeps in tensor memory (kGroups: none).
// Measured (B200): with k = 32 classes per Gaussian (cfg4: about four read-modify-writes per
// entry and group, the shared-memory pipe 88% busy) groups 4-7 in TMEM give 167 -> 185 views/s;
// with k = 16 (cfg1: two per entry and group, TMEM's wait per read-modify-write exposed) 908 ->
// 891, so TMEM is used from k = 24. SGM_TM_FIRST=g overrides (groups g..7; g < 4 needs C <= 128).
int raster_tm_first(const DevMap& m) {
    const int cg4 = (m.C + kGroups - 1) / kGroups * 4;  // columns per group
    int first = m.k >= 24 ? 4 : kGroups;
    if (const char* e = std::getenv("SGM_TM_FIRST")) first = std::atoi(e);
    if (first < 4 && cg4 > 64) first = 4;
    if (cg4 > 128) first = kGroups;
    return std::max(0, std::min(kGroups, first));
}

template <bool kRender, bool kDup, bool kAniso, bool kRc = false>
void launch_t(const RasterParams& p0, int n_views, cudaStream_t s) {
    RasterParams p = p0;
    p.n_items = p.item_list ? p.n_item_list : p.tiles_per_view * n_views;
    if (p.n_items == 0) return;
    const size_t smem = static_cast<size_t>(make_layout(p.map.C, p.map.kpad, kRender, kRc).total);
    // four CTAs per SM when four fit in shared memory (228 KB, 1 KB reserved per CTA)
    // (score mode only: the render and rc variants would spill at the 4-CTA register budget);
    // that variant stages the 16-byte semantic records
    const bool four = !kRender && !kRc && raster_score_records(p.map);
    const size_t smem4 = static_cast<size_t>(make_layout(p.map.C, p.map.kpad, false, false, true).total);
    // (render: usually one view per launch, so shorter CTAs balance the last wave better)
    p.items_per_cta = kRender ? 2 : kItemsPerCta;
    const int grid = (p.n_items + p.items_per_cta - 1) / p.items_per_cta;
    if constexpr (!kRender && !kRc) {
        p.tm_first = raster_tm_first(p.map);
        const bool tm = p.tm_first < kGroups;
        if (p.item_list || p.trunc) {
            if (tm) {
                cudaFuncSetAttribute(k_raster<kRender, kDup, kAniso, kRc, 3, true, false, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
                k_raster<kRender, kDup, kAniso, kRc, 3, true, false, true><<<grid, kThreads, smem, s>>>(p);
                return;
            }
            cudaFuncSetAttribute(k_raster<kRender, kDup, kAniso, kRc, 3, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            k_raster<kRender, kDup, kAniso, kRc, 3, true><<<grid, kThreads, smem, s>>>(p);
            return;
        }
        if (four) {
            if (p.map.n && !p.map.sem_rec) throw std::logic_error("score raster: DevMap::sem_rec not built (map_records)");
            cudaFuncSetAttribute(k_raster<kRender, kDup, kAniso, kRc, 4, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem4));
            k_raster<kRender, kDup, kAniso, kRc, 4, false><<<grid, kThreads, smem4, s>>>(p);
            return;
        }
    }
    if constexpr (kRender && !kAniso) {
        if (p.opt.ref_div) {  // render_reference's footprint form
            cudaFuncSetAttribute(k_raster<kRender, kDup, kAniso, kRc, 3, false, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            k_raster<kRender, kDup, kAniso, kRc, 3, false, true><<<grid, kThreads, smem, s>>>(p);
            return;
        }
    }
    if constexpr (!kRender && !kRc) {
        if (p.tm_first < kGroups) {
            cudaFuncSetAttribute(k_raster<kRender, kDup, kAniso, kRc, 3, false, false, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            k_raster<kRender, kDup, kAniso, kRc, 3, false, false, true><<<grid, kThreads, smem, s>>>(p);
            return;
        }
    }
    cudaFuncSetAttribute(k_raster<kRender, kDup, kAniso, kRc, 3, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k_raster<kRender, kDup, kAniso, kRc, 3, false><<<grid, kThreads, smem, s>>>(p);
}

}  // namespace

GroupParams choose_groups(int C, int k) {
    (void)k;
    GroupParams gp;
    gp.P = kGroups;
    gp.Cg = (C + kGroups - 1) / kGroups;
    return gp;
}

bool raster_score_records(const DevMap& m) {
    return make_layout(m.C, m.kpad, false, false, true).total + 2048 <= 228 * 1024 / 4;
}

size_t raster_smem_bytes(const DevMap& m, const GroupParams& gp, bool render) {
    (void)gp;
    return static_cast<size_t>(make_layout(m.C, m.kpad, render).total);
}

template <bool kRender>
void launch_mode(const RasterParams& p, int n_views, cudaStream_t s) {
    if (p.map.aniso) {
        if (p.map.dup_idx)
            launch_t<kRender, true, true>(p, n_views, s);
        else
            launch_t<kRender, false, true>(p, n_views, s);
    } else if (p.map.dup_idx) {
        launch_t<kRender, true, false>(p, n_views, s);
    } else {
        launch_t<kRender, false, false>(p, n_views, s);
    }
}

void launch_raster_score(const RasterParams& p, int n_views, cudaStream_t s) {
    if (p.want_rc && !p.map.aniso) {  // Fisher gain: colour / depth planes for its pass 1
        if (p.map.dup_idx)
            launch_t<false, true, false, true>(p, n_views, s);
        else
            launch_t<false, false, false, true>(p, n_views, s);
        return;
    }
    launch_mode<false>(p, n_views, s);
}

void launch_raster_render(const RasterParams& p, int n_views, cudaStream_t s) {
    launch_mode<true>(p, n_views, s);
}

}  // namespace sgm
