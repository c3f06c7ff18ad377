// The host pipeline that drives the sm_100a kernels for batches of views.
//
// Pipeline for a batch of views (all on the ctx stream):
//   1. K1 k_preprocess over (Gaussian, view): compact visible (z, index), count V, P and
//      the row pairs R (tile rows spanned)
//   2. one D2H of the per-view V/P/R counts (the only host sync before the results)
//   3. per view (binning stream): CUB radix sort on fp32(z) -> k_tiefix -> k_pack ->
//      k_bin_hist + k_bin_scan (tile ranges) -> k_emit_rows + CUB stable row sort ->
//      k_row_segs / k_seg_count / k_seg_scan / k_seg_pass (ordered scatter into the tile lists)
//   4. raster launches of 8 views each over (8x8 block, view), overlapping the binning of
//      the next 8 views
//   5. k_reduce_scores (score) / planes already written (render)
// Views whose pair lists do not fit the scratch budget together are split into
// sub-batches; results do not depend on the split (per-view work is independent).
#include <cstdlib>

#include "sgm_ctx.h"

namespace sgm {


CamParams to_cam(const sgm_camera* c) {
    if (!c) fail(SGM_ERR_INVALID, "camera is null");
    if (c->width <= 0 || c->height <= 0) fail(SGM_ERR_INVALID, "camera: resolution must be positive");
    return CamParams{c->width, c->height, c->fx, c->fy, c->cx, c->cy};
}

OptParams to_opt(const sgm_options* o, const CamParams& cam) {
    sgm_options d{1, 1e-4, 0.01, 3.0, 8};
    const sgm_options& s = o ? *o : d;
    if (s.tile_size <= 0 || s.tile_size % kTile != 0)
        fail(SGM_ERR_UNSUPPORTED, "tile_size %d: this build bins at multiples of %d", s.tile_size,
             kTile);
    OptParams p;
    p.early_exit = s.early_exit ? 1 : 0;
    p.eps = s.transmittance_eps;
    p.z_near = s.z_near;
    p.trunc = s.truncation_sigmas;
    p.cut_sq = s.truncation_sigmas * s.truncation_sigmas;
    p.ts = s.tile_size;
    p.tiles_x = (cam.W + s.tile_size - 1) / s.tile_size;
    p.tiles_y = (cam.H + s.tile_size - 1) / s.tile_size;
    return p;
}

PoseParams to_pose(const sgm_pose& p) {
    PoseParams q;
    for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) q.Rcw[3 * i + k] = p.R[3 * k + i];  // R_cw = R^T
    for (int i = 0; i < 3; ++i) q.t[i] = p.t[i];
    return q;
}

unsigned tile_bits(uint64_t tiles) {
    unsigned b = 1;
    while ((1ull << b) < tiles) ++b;
    return b;
}


// K2 (after the sub-batch's depth sort) + K3 pack of one view: runs of equal fp32 depth keys
// fixed by the full key, PackedSplat / bounds / tile rectangles per depth rank.
static void pack_view(sgm_ctx* ctx, cudaStream_t s, const sgm_map* map, const CamParams& cam,
                      const OptParams& o, const PoseParams* d_pose, const uint32_t* keys,
                      uint32_t* vals, uint32_t V, PackedSplat* packed, uint4* bounds) {
    if (V == 0) return;
    launch_tiefix(map->dev, d_pose, cam, o, keys, vals, V, s);
    launch_pack(map->dev, d_pose, cam, o, map->groups, vals, V, packed,
                ctx->counts.as<unsigned long long>(), ctx->rects.as<int4>(), bounds, s);
    ctx->stats.kernel_launches += (V >= 2 ? 1 : 0) + 1;
}

// K3 counts over the ranks < Ve (a depth prefix when Ve < V): tile ranges from the
// rectangles' 2D difference array (bins outside `mask` empty; total pairs to d_total), and
// the row-pair offsets roff[0..Ve] (roff[Ve] = the prefix's row pairs).
// kRankChunks > 0 with a cap: pass 1 of depth-prefix binning, where only ranks that can reach
// a bin's first `cap` entries get row pairs (k_bin_hist_prefix).
constexpr int kRankChunks = 64;
static void bin_counts(sgm_ctx* ctx, cudaStream_t s, const OptParams& o, uint32_t Ve, uint2* ranges,
                       int bin_tiles, const uint8_t* mask, unsigned long long* d_total,
                       uint32_t cap = 0xffffffffu, uint8_t* trunc = nullptr, bool prefix_rows = false) {
    CK(cudaMemsetAsync(ranges, 0, sizeof(uint2) * bin_tiles, s));
    if (Ve == 0) {
        if (d_total) CK(cudaMemsetAsync(d_total, 0, 8, s));
        CK(cudaMemsetAsync(ctx->offsets.p, 0, 8, s));
        return;
    }
    const int X = o.tiles_x + 1, Y = o.tiles_y + 1;
    int* diff = ctx->bdiff.as<int>();
    CK(cudaMemsetAsync(diff, 0, sizeof(int) * X * Y, s));
    unsigned long long* rows = ctx->counts.as<unsigned long long>();
    unsigned long long* roff = ctx->offsets.as<unsigned long long>();
    if (prefix_rows) {
        const size_t cells = static_cast<size_t>(X) * Y * kRankChunks;
        CK(cudaMemsetAsync(ctx->cdiff.p, 0, sizeof(int) * cells, s));
        CK(cudaMemsetAsync(ctx->csat.p, 0, sizeof(int) * cells, s));
        launch_bin_hist_prefix(ctx->rects.as<int4>(), Ve, o.tiles_x, o.tiles_y, cap, kRankChunks,
                               ctx->cdiff.as<int>(), ctx->csat.as<int>(), diff, rows, s);
        ctx->stats.kernel_launches += 5;  // (+ the k_bin_hist counted below)
    } else {
        launch_bin_hist(ctx->rects.as<int4>(), Ve, o.tiles_x, diff, rows, s);
    }
    launch_bin_scan(diff, o.tiles_x, o.tiles_y, ranges, s, mask, d_total, cap, trunc);
    CK(cudaMemsetAsync(rows + Ve, 0, sizeof(unsigned long long), s));
    exclusive_scan_u64<unsigned long long>(rows, Ve + 1, roff, ctx->scan_tmp.as<unsigned long long>(), s);
    ctx->stats.kernel_launches += 2 + exclusive_scan_launches(Ve + 1);
}

// K3 lists (row-bucketed, no sort of the P pairs) over the ranks < Ve: the (row, rank) pairs
// (R of them, d_R on the device) in rank order, stably sorted by row; then per row segment a
// warp scatters its ranks into the tile lists in rank order (sgm_kernels.cu). Bins outside
// `mask` get no entries.
static const unsigned long long* bin_lists(sgm_ctx* ctx, cudaStream_t s, const OptParams& o,
                                           uint32_t Ve, uint64_t R, const unsigned long long* d_R,
                                           uint32_t* list, const uint2* ranges, const uint8_t* mask,
                                           bool part = false, uint64_t P = 0) {
    if (R == 0) return nullptr;
    const unsigned long long* roff = ctx->offsets.as<unsigned long long>();
    uint32_t* rk = ctx->tkeys.as<uint32_t>();
    unsigned long long* rv = ctx->rvals.as<unsigned long long>();
    launch_emit_rows(roff, ctx->rects.as<int4>(), Ve, R, rk, rv, s);
    // each tile row's (row, rank) pairs in rank order: a stable sort on the row key
    const int rbits = static_cast<int>(tile_bits(static_cast<uint64_t>(o.tiles_y)));
    const bool ralt = radix_sort_pairs<unsigned long long, unsigned long long>(
        rk, rv, ctx->tkeys_alt.as<uint32_t>(), ctx->tvals_alt.as<unsigned long long>(), 0, d_R, R, 1,
        rbits, ctx->sort_tmp.as<uint32_t>(), s);
    const uint32_t* qk = ralt ? ctx->tkeys_alt.as<uint32_t>() : rk;
    const unsigned long long* qv = ralt ? ctx->tvals_alt.as<unsigned long long>() : rv;
    ctx->stats.kernel_launches += radix_sort_launches(rbits, R);
    uint2* rranges = ctx->rranges.as<uint2>();
    CK(cudaMemsetAsync(rranges, 0, sizeof(uint2) * o.tiles_y, s));
    launch_ranges(qk, R, rranges, s);
    const uint64_t G = row_scatter_segments(R, o.tiles_y);  // buffers sized by the caller
    launch_row_scatter(qv, rranges, ranges, o.tiles_x, o.tiles_y, R,
                       ctx->segs.as<uint4>(), reinterpret_cast<uint32_t*>(ctx->segs.as<char>() + sizeof(uint4) * G),
                       ctx->segcnt.as<uint32_t>(), list, s, mask, part,
                       /*cols: rows of wide entries (cfg4), walked column by column*/ P >= 16 * R);
    ctx->stats.kernel_launches += 7;
    return qv;
}

// Bins one view (step 3): pack, then the full bins (every rank).
static void bin_view(sgm_ctx* ctx, cudaStream_t s, const sgm_map* map, const CamParams& cam,
                     const OptParams& o, const PoseParams* d_pose, uint32_t* keys, uint32_t* vals,
                     uint32_t V, uint64_t P, uint64_t R, const unsigned long long* d_R,
                     PackedSplat* packed, uint4* bounds, uint32_t* list, uint2* ranges, int bin_tiles) {
    pack_view(ctx, s, map, cam, o, d_pose, keys, vals, V, packed, bounds);
    if (V == 0 || P == 0) {
        CK(cudaMemsetAsync(ranges, 0, sizeof(uint2) * bin_tiles, s));
        return;
    }
    bin_counts(ctx, s, o, V, ranges, bin_tiles, nullptr, nullptr);
    bin_lists(ctx, s, o, V, R, d_R, list, ranges, nullptr, false, P);
}

// Reserves the row-pair scratch of the binning for up to R row pairs.
static void reserve_rows(sgm_ctx* ctx, const OptParams& o, uint64_t R, size_t NS, int kSub) {
    const uint64_t r = std::max<uint64_t>(R, 1);
    CK(ctx->tkeys.reserve(4 * r));
    CK(ctx->tkeys_alt.reserve(4 * r));
    CK(ctx->tvals_alt.reserve(8 * r));
    CK(ctx->rvals.reserve(8 * r));
    CK(ctx->sort_tmp.reserve(std::max(radix_sort_scratch_bytes(r, 1), radix_sort_scratch_bytes(NS, kSub))));
    CK(ctx->scan_tmp.reserve(exclusive_scan_scratch_bytes(NS + 1)));
    // row-scatter segments (reserved before the launches: a reallocation synchronises)
    const uint64_t G = row_scatter_segments(r, o.tiles_y);
    CK(ctx->segs.reserve(sizeof(uint4) * G + 16));
    CK(ctx->segcnt.reserve(sizeof(uint32_t) * G * o.tiles_x));
}

// Depth-prefix binning of "dense" views (cfg4: bins averaging hundreds of thousands of
// entries). The raster's early exit (:312) consumes a short prefix of every bin, so each bin
// first gets only its first `cap` entries (a prefix of its full list, same rank order),
// flagged when that drops entries (pass 1, pipelined like any view). A block that exhausts a
// flagged list with pixels still open is reported incomplete; after the group's rasters, the
// full lists of those tiles' bins are built (pass 2) and those tiles redone. A block that
// completes inside its prefix stops where it would have stopped on the full list, so every
// tile's result is the full-list result.
constexpr uint64_t kDenseAvg = 65536;  // entries per bin on average: a dense view
constexpr uint64_t kForceAvg = 4096;   // (SGM_PREFIX_BINNING=1: dense from this average)
constexpr uint32_t kPrefixCap = 8192;  // entries per bin of pass 1 (cfg4: 120 vs 106 views/s
                                       // with full lists; 256: 85, 2048: 110, 32768: 111)

// pass 1 of a dense view on stream s (no host sync: the list region holds cap entries per bin)
static void bin_dense_view(sgm_ctx* ctx, cudaStream_t s, const sgm_map* map, const CamParams& cam,
                           const OptParams& o, const PoseParams* d_pose, uint32_t* keys, const ViewDesc& d,
                           uint32_t V, uint64_t P, uint64_t R, const unsigned long long* d_R, int bin_tiles,
                           uint32_t cap, uint8_t* trunc) {
    pack_view(ctx, s, map, cam, o, d_pose, keys, const_cast<uint32_t*>(d.order), V,
              const_cast<PackedSplat*>(d.packed), const_cast<uint4*>(d.bounds));
    uint2* ranges = const_cast<uint2*>(d.ranges);
    if (V == 0 || P == 0) {
        CK(cudaMemsetAsync(ranges, 0, sizeof(uint2) * bin_tiles, s));
        CK(cudaMemsetAsync(trunc, 0, bin_tiles, s));
        return;
    }
    bin_counts(ctx, s, o, V, ranges, bin_tiles, nullptr, nullptr, cap, trunc, true);
    // the row pairs of the ranks that can reach a prefix: their count (a host round trip on the
    // binning stream; the raster of the previous sub-batch runs meanwhile)
    const unsigned long long* d_R1 = ctx->offsets.as<unsigned long long>() + V;
    unsigned long long R1 = 0;
    CK(cudaMemcpyAsync(&R1, d_R1, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    (void)R;
    if (R1) bin_lists(ctx, s, o, V, R1, d_R1, const_cast<uint32_t*>(d.list), ranges, nullptr, true, P);
}

// pass 2 of a dense view whose raster reported `ninc` incomplete tiles (in `inc`): the view is
// binned again from its depth order (the binning scratch has served later views since), with
// full lists for the bins of those tiles only, and those tiles are rastered again (their
// per-tile partials overwritten). Synchronous on s; runs before the group's score reduction.
static void redo_dense_view(sgm_ctx* ctx, cudaStream_t s, const sgm_map* map, const CamParams& cam,
                            const OptParams& o, const PoseParams* d_pose, uint32_t* keys, ViewDesc d,
                            ViewDesc* d_desc, uint32_t V, uint64_t P, uint64_t R,
                            const unsigned long long* d_R, int bin_tiles, int rtx, const uint32_t* inc,
                            uint32_t ninc, RasterParams rp) {
    CK(ctx->franges.reserve(sizeof(uint2) * bin_tiles));
    CK(ctx->bmask.reserve(bin_tiles + 16));
    CK(ctx->redo.reserve(sizeof(uint2) * ninc + 16));
    CK(ctx->dense_tot.reserve(64));
    unsigned long long* d_tot = ctx->dense_tot.as<unsigned long long>();
    uint8_t* mask = ctx->bmask.as<uint8_t>();
    uint2* full = ctx->franges.as<uint2>();
    CK(cudaMemsetAsync(mask, 0, bin_tiles, s));
    launch_redo_items(inc, ninc, 0, rtx, o.ts / kTile, o.tiles_x, ctx->redo.as<uint2>(), mask, s);
    pack_view(ctx, s, map, cam, o, d_pose, keys, const_cast<uint32_t*>(d.order), V,
              const_cast<PackedSplat*>(d.packed), const_cast<uint4*>(d.bounds));
    bin_counts(ctx, s, o, V, full, bin_tiles, mask, d_tot, 0xffffffffu, nullptr);
    unsigned long long P2 = 0;
    CK(cudaMemcpyAsync(&P2, d_tot, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (P2 >= (1ull << 32)) fail(SGM_ERR_UNSUPPORTED, "view has %llu tile pairs (>= 2^32)", P2);
    CK(ctx->list2.reserve(4 * std::max<unsigned long long>(P2, 1)));
    bin_lists(ctx, s, o, V, R, d_R, ctx->list2.as<uint32_t>(), full, mask, true, P);
    d.list = ctx->list2.as<uint32_t>();
    d.ranges = full;
    CK(cudaMemcpyAsync(d_desc, &d, sizeof(ViewDesc), cudaMemcpyHostToDevice, s));
    rp.views = d_desc;
    rp.trunc = nullptr;
    rp.incomplete = nullptr;
    rp.n_incomplete = nullptr;
    rp.item_list = ctx->redo.as<uint2>();
    rp.n_item_list = static_cast<int>(ninc);
    launch_raster_score(rp, 1, s);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));  // (d lives on this stack frame)
    ctx->stats.kernel_launches += 3;
    ctx->stats.raster_launches += 1;
}

// Runs n views. Score mode writes n_missing/entropy_sum (host); render mode (n == 1)
// writes planes to device targets. Binning of sub-batch i+1 (on ctx->bin_stream)
// overlaps the raster of sub-batch i (on ctx->stream).
void run_views(sgm_ctx* ctx, const sgm_map* map, const CamParams& cam, const OptParams& o,
               uint64_t n, const PoseParams* poses, Mode mode, const RenderTargets& rt,
               double* h_missing, double* h_entropy, Fisher fk, double* h_fisher, double* d_H) {
    cudaStream_t s = ctx->stream;
    cudaStream_t sb = ctx->bin_stream;
    const uint64_t N = map->dev.n;
    const int bin_tiles = o.tiles_x * o.tiles_y;
    const int rtx = (cam.W + kTile - 1) / kTile;
    const int rty = (cam.H + kTile - 1) / kTile;
    const int rtiles = rtx * rty;
    ctx->last_valid = false;
    // (the render layout bounds every raster variant: wider accumulator rows, colour stage)
    need_smem(ctx->device, raster_smem_bytes(map->dev, map->groups, true), map->dev.C, "raster");

    // batch size bounded by a scratch budget for the per-view N-sized arrays
    const size_t per_view = std::max<uint64_t>(N, 1) * (4 + 4 + sizeof(PackedSplat) + 16) +
                            static_cast<size_t>(bin_tiles) * sizeof(uint2) +
                            static_cast<size_t>(rtiles) * 12 + 256;
    const size_t budget = size_t(12) << 30;
    uint64_t B = std::max<uint64_t>(1, std::min<uint64_t>(n, std::max<size_t>(1, budget / per_view)));
    B = std::min<uint64_t>(B, 64);
    if (mode == Mode::Render) B = 1;

    const size_t NS = std::max<uint64_t>(N, 1);
    CK(ctx->poses.reserve(sizeof(PoseParams) * B));
    CK(ctx->vcount.reserve(4 * B));
    CK(ctx->pcount.reserve(16 * B));  // pairs P | row pairs R per view
    CK(ctx->bdiff.reserve(sizeof(int) * (o.tiles_x + 1) * (o.tiles_y + 1)));
    CK(ctx->rranges.reserve(sizeof(uint2) * o.tiles_y));
    CK(ctx->keys.reserve(4 * NS * B));
    CK(ctx->vals.reserve(4 * NS * B));
    CK(ctx->keys_alt.reserve(4 * NS * std::min<uint64_t>(B, 8)));  // a sub-batch of depth sorts
    CK(ctx->rects.reserve(sizeof(int4) * NS));
    CK(ctx->vals_alt.reserve(4 * NS * std::min<uint64_t>(B, 8)));
    CK(ctx->packed.reserve(sizeof(PackedSplat) * NS * B));
    CK(ctx->bounds.reserve(sizeof(uint4) * NS * B));
    CK(ctx->counts.reserve(8 * (NS + 1)));
    CK(ctx->offsets.reserve(8 * (NS + 1)));
    CK(ctx->ranges.reserve(sizeof(uint2) * bin_tiles * B));
    CK(ctx->ent_part.reserve(8ull * rtiles * B));
    CK(ctx->miss_part.reserve(4ull * rtiles * B));
    CK(ctx->views.reserve(sizeof(ViewDesc) * B));
    CK(ctx->out.reserve(24 * B));
    if (fk == Fisher::Gain) {
        CK(ctx->fis_part.reserve(8ull * rtiles * B));
        // rendered colour / depth per view for the gain's Jacobian pass (written by the
        // score raster, so k_fisher skips its own pass 0)
        CK(ctx->rcbuf.reserve(32ull * cam.W * cam.H * B));
    }
    CK(ctx->contributors.reserve(8));
    CK(ctx->h_counts.reserve(32 * B + 16));  // V (u32) | P | R | contributors
    CK(ctx->h_views.reserve(sizeof(ViewDesc) * B));
    CK(ctx->h_poses.reserve(sizeof(PoseParams) * B));
    CK(ctx->h_out.reserve(24 * B));

    const int kSub = 8;  // views per raster launch (binning of the next 8 overlaps)
    bool rows_ready = false;  // map_ready done (before the first raster launch)
    for (uint64_t b0 = 0; b0 < n; b0 += B) {
        const int nb = static_cast<int>(std::min<uint64_t>(B, n - b0));
        if (ctx->profiling) CK(cudaEventRecord(ctx->ev[0], s));
        std::memcpy(ctx->h_poses.p, poses + b0, sizeof(PoseParams) * nb);
        CK(cudaMemcpyAsync(ctx->poses.p, ctx->h_poses.p, sizeof(PoseParams) * nb,
                           cudaMemcpyHostToDevice, s));
        CK(cudaMemsetAsync(ctx->vcount.p, 0, 4 * nb, s));
        CK(cudaMemsetAsync(ctx->pcount.p, 0, 16 * nb, s));
        CK(cudaMemsetAsync(ctx->contributors.p, 0, 8, s));
        launch_preprocess(map->dev, ctx->poses.as<PoseParams>(), cam, o, nb, ctx->keys.as<uint32_t>(),
                          ctx->vals.as<uint32_t>(), NS, ctx->vcount.as<uint32_t>(),
                          ctx->pcount.as<unsigned long long>(),
                          ctx->pcount.as<unsigned long long>() + nb, s);
        ctx->stats.kernel_launches += (N > 0) ? 1 : 0;
        uint32_t* hv = ctx->h_counts.as<uint32_t>();
        unsigned long long* hp = reinterpret_cast<unsigned long long*>(ctx->h_counts.as<char>() + 8 * B);
        CK(cudaMemcpyAsync(hv, ctx->vcount.p, 4 * nb, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(hp, ctx->pcount.p, 16 * nb, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        std::vector<uint32_t> V(hv, hv + nb);
        std::vector<uint64_t> P(hp, hp + nb);
        std::vector<uint64_t> R(hp + nb, hp + 2 * nb);  // (row, rank) pairs of the binning

        // Depth-prefix binning (bin_dense_view) serves the plain score mode's dense views: bins
        // averaging more than kDenseAvg entries (cfg4), or lists past 2^31 entries.
        // SGM_PREFIX_BINNING=1 lowers the threshold to kForceAvg, =0 turns it off;
        // SGM_PREFIX_CAP sets the pass-1 entries per bin.
        const char* pb = std::getenv("SGM_PREFIX_BINNING");
        const int prefix_mode = pb ? (pb[0] == '0' ? 0 : 2) : 1;
        const char* pc = std::getenv("SGM_PREFIX_CAP");
        const uint32_t cap = pc ? std::max(1u, static_cast<uint32_t>(std::atoi(pc))) : kPrefixCap;
        const uint64_t dense_pairs = uint64_t(2) << 30;
        auto dense = [&](int v) {
            if (prefix_mode == 0 || mode != Mode::Score || fk != Fisher::None) return false;
            const uint64_t avg = prefix_mode == 2 ? kForceAvg : kDenseAvg;
            return P[v] > avg * static_cast<uint64_t>(bin_tiles) || P[v] > dense_pairs;
        };
        // list entries a view needs: its pairs, or cap per bin for a dense view
        auto list_len = [&](int v) {
            return dense(v) ? std::min<uint64_t>(P[v], static_cast<uint64_t>(cap) * bin_tiles) : P[v];
        };
        // groups of views whose lists fit ctx->list_budget together (a fifth of the device), so
        // the binning of each sub-batch overlaps the raster of the previous one
        const uint64_t pair_budget = ctx->list_budget;
        int v0 = 0;
        while (v0 < nb) {
            int v1 = v0;
            uint64_t sumP = 0;
            while (v1 < nb && (v1 == v0 || sumP + list_len(v1) <= pair_budget)) sumP += list_len(v1++);
            int ndense = 0;
            for (int v = v0; v < v1; ++v) {
                ndense += dense(v) ? 1 : 0;
                if (!dense(v) && P[v] >= (1ull << 32))  // (a dense view's lists hold prefixes)
                    fail(SGM_ERR_UNSUPPORTED, "view has %llu tile pairs (>= 2^32)",
                         static_cast<unsigned long long>(P[v]));
            }
            uint64_t maxR = 1;
            for (int v = v0; v < v1; ++v) maxR = std::max<uint64_t>(maxR, R[v]);
            CK(ctx->tvals.reserve(4 * std::max<uint64_t>(sumP, 1)));
            reserve_rows(ctx, o, maxR, NS, kSub);
            const int ng = v1 - v0;
            if (ndense) {  // per view of the group: truncation flags, incomplete tiles, their count
                CK(ctx->trunc8.reserve(static_cast<size_t>(bin_tiles) * ng + 16));
                CK(ctx->incomplete.reserve(4 * static_cast<size_t>(rtiles) * ng + 16));
                CK(ctx->dense_tot.reserve(16 + 4 * static_cast<size_t>(ng) + 16));
                const size_t cells = static_cast<size_t>(o.tiles_x + 1) * (o.tiles_y + 1) * kRankChunks;
                CK(ctx->cdiff.reserve(sizeof(int) * cells));
                CK(ctx->csat.reserve(sizeof(int) * cells));
            }
            uint32_t* d_ninc = ndense ? reinterpret_cast<uint32_t*>(ctx->dense_tot.as<char>() + 16) : nullptr;
            // descriptors for the whole group (list offsets known from the counts)
            ViewDesc* hvd = ctx->h_views.as<ViewDesc>();
            uint64_t list_off = 0;
            for (int v = v0; v < v1; ++v) {
                ViewDesc d{};
                d.order = ctx->vals.as<uint32_t>() + NS * v;
                d.pose = ctx->poses.as<PoseParams>() + v;
                d.fis_partial = fk == Fisher::Gain ? ctx->fis_part.as<double>() + static_cast<size_t>(rtiles) * v
                                                   : nullptr;
                d.ranges = ctx->ranges.as<uint2>() + static_cast<size_t>(bin_tiles) * v;
                d.list = ctx->tvals.as<uint32_t>() + list_off;
                d.packed = ctx->packed.as<PackedSplat>() + NS * v;
                d.bounds = ctx->bounds.as<uint4>() + NS * v;
                d.ent_partial = ctx->ent_part.as<double>() + static_cast<size_t>(rtiles) * v;
                d.miss_partial = ctx->miss_part.as<uint32_t>() + static_cast<size_t>(rtiles) * v;
                d.color = rt.color;
                d.depth = rt.depth;
                d.sil = rt.sil;
                d.sem = rt.sem;
                d.contributors = ctx->contributors.as<unsigned long long>();
                d.contrib = rt.contrib;
                d.contrib_count = rt.contrib_count;
                d.contrib_offset = rt.contrib_offset;
                d.rc4 = fk == Fisher::Gain
                            ? ctx->rcbuf.as<double>() + 4ull * cam.W * cam.H * static_cast<size_t>(v)
                            : nullptr;
                hvd[v - v0] = d;
                list_off += list_len(v);
                ctx->stats.visible += V[v];
                ctx->stats.pairs += P[v];  // (the reference's pairs, also for a dense view)
            }
            const int ngroup = v1 - v0;
            CK(cudaMemcpyAsync(ctx->views.p, hvd, sizeof(ViewDesc) * ngroup, cudaMemcpyHostToDevice, s));
            if (ndense) CK(cudaMemsetAsync(d_ninc, 0, 4 * static_cast<size_t>(ngroup), s));
            // the binning stream starts after everything already queued on s
            CK(cudaEventRecord(ctx->ev_ready, s));
            CK(cudaStreamWaitEvent(sb, ctx->ev_ready, 0));
            RasterParams rp{};
            rp.map = map->dev;
            rp.cam = cam;
            rp.opt = o;
            rp.tiles_per_view = rtiles;
            rp.raster_tiles_x = rtx;
            rp.channels = rt.channels;
            rp.groups = map->groups;
            rp.want_rc = fk == Fisher::Gain ? 1 : 0;
            // sub-batches of 1, 2, 4, then kSub views: the first raster starts after one view's
            // binning instead of kSub views' (the pipeline fill), and each sub-batch's binning
            // still hides under the previous one's raster (about 1/3 of its time per view). A
            // sub-batch holds dense views only, or none (its raster reports incomplete tiles).
            int sub = 0;
            for (int s0 = v0, s1 = v0, len = 1; s0 < v1; s0 = s1, ++sub) {
                while (s1 < v1 && s1 - s0 < len && dense(s1) == dense(s0)) ++s1;
                len = std::min(kSub, 2 * len);
                {  // K2 for the sub-batch: one segmented radix sort of its views' depth keys
                    uint32_t maxV = 0;
                    for (int v = s0; v < s1; ++v) maxV = std::max(maxV, V[v]);
                    const bool alt = radix_sort_pairs<uint32_t, uint32_t>(
                        ctx->keys.as<uint32_t>() + NS * s0, ctx->vals.as<uint32_t>() + NS * s0,
                        ctx->keys_alt.as<uint32_t>(), ctx->vals_alt.as<uint32_t>(), NS,
                        ctx->vcount.as<uint32_t>() + s0, maxV, s1 - s0, 32, ctx->sort_tmp.as<uint32_t>(), sb);
                    if (alt) fail(SGM_ERR_CUDA, "depth sort: odd pass count");  // 4 passes: in place
                    ctx->stats.kernel_launches += maxV ? radix_sort_launches(32, maxV) : 0;
                }
                const bool dsub = dense(s0);
                for (int v = s0; v < s1; ++v) {
                    const ViewDesc& d = hvd[v - v0];
                    if (dsub) {
                        bin_dense_view(ctx, sb, map, cam, o, ctx->poses.as<PoseParams>() + v,
                                       ctx->keys.as<uint32_t>() + NS * v, d, V[v], P[v], R[v],
                                       ctx->pcount.as<unsigned long long>() + nb + v, bin_tiles, cap,
                                       ctx->trunc8.as<uint8_t>() + static_cast<size_t>(bin_tiles) * (v - v0));
                        continue;
                    }
                    bin_view(ctx, sb, map, cam, o, ctx->poses.as<PoseParams>() + v,
                             ctx->keys.as<uint32_t>() + NS * v, const_cast<uint32_t*>(d.order), V[v],
                             P[v], R[v], ctx->pcount.as<unsigned long long>() + nb + v,
                             const_cast<PackedSplat*>(d.packed), const_cast<uint4*>(d.bounds),
                             const_cast<uint32_t*>(d.list), const_cast<uint2*>(d.ranges), bin_tiles);
                }
                const int slot = sub & 1;
                CK(cudaEventRecord(ctx->ev_binned[slot], sb));
                // the raster reads the semantic rows: the map's upload (phase B) has to be done;
                // the binning just queued runs meanwhile
                if (!rows_ready) {
                    map_ready(ctx, map);
                    if (mode == Mode::Score && raster_score_records(map->dev)) map_records(ctx, map);
                    rows_ready = true;
                    rp.map = map->dev;  // (dup_idx known now)
                }
                CK(cudaStreamWaitEvent(s, ctx->ev_binned[slot], 0));
                rp.views = ctx->views.as<ViewDesc>() + (s0 - v0);
                rp.trunc = dsub ? ctx->trunc8.as<uint8_t>() + static_cast<size_t>(bin_tiles) * (s0 - v0) : nullptr;
                rp.incomplete = dsub ? ctx->incomplete.as<uint32_t>() + static_cast<size_t>(rtiles) * (s0 - v0) : nullptr;
                rp.n_incomplete = dsub ? d_ninc + (s0 - v0) : nullptr;
                const int pr = sub % 16;  // profiling event pair
                if (ctx->profiling) CK(cudaEventRecord(ctx->ev_r[2 * pr], s));
                FisherParams fp{};
                fp.H = d_H;
                fp.invp = map->fisher_invp.as<double>();
                if (fk == Fisher::Prior) {
                    launch_fisher_prior(rp, fp, s1 - s0, s);
                } else {
                    if (mode == Mode::Score)
                        launch_raster_score(rp, s1 - s0, s);
                    else
                        launch_raster_render(rp, s1 - s0, s);
                    if (fk == Fisher::Gain) {
                        launch_fisher_gain(rp, fp, s1 - s0, s);
                        ctx->stats.kernel_launches += 1;
                    }
                }
                CK(cudaGetLastError());
                if (ctx->profiling) CK(cudaEventRecord(ctx->ev_r[2 * pr + 1], s));
                ctx->stats.kernel_launches += 1;
                ctx->stats.raster_launches += 1;
            }
            if (ndense) {  // pass 2 of the dense views with incomplete tiles
                std::vector<uint32_t> hn(ngroup);
                CK(cudaMemcpyAsync(hn.data(), d_ninc, 4 * static_cast<size_t>(ngroup), cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                rp.trunc = nullptr;
                rp.incomplete = nullptr;
                rp.n_incomplete = nullptr;
                for (int v = v0; v < v1; ++v) {
                    if (!dense(v) || hn[v - v0] == 0) continue;
                    redo_dense_view(ctx, s, map, cam, o, ctx->poses.as<PoseParams>() + v,
                                    ctx->keys.as<uint32_t>() + NS * v, hvd[v - v0],
                                    ctx->views.as<ViewDesc>() + (v - v0), V[v], P[v], R[v],
                                    ctx->pcount.as<unsigned long long>() + nb + v, bin_tiles, rtx,
                                    ctx->incomplete.as<uint32_t>() + static_cast<size_t>(rtiles) * (v - v0),
                                    hn[v - v0], rp);
                }
            }
            if (mode == Mode::Score && fk != Fisher::Prior) {
                double* dfis = fk == Fisher::Gain ? ctx->out.as<double>() + 2 * ngroup : nullptr;
                launch_reduce_scores(ctx->views.as<ViewDesc>(), ngroup, rtiles, ctx->out.as<double>(),
                                     ctx->out.as<double>() + ngroup, dfis, s);
                ctx->stats.kernel_launches += 1;
                double* ho = ctx->h_out.as<double>();
                CK(cudaMemcpyAsync(ho, ctx->out.p, 24 * ngroup, cudaMemcpyDeviceToHost, s));
                unsigned long long* kc = hp + 2 * B;
                CK(cudaMemcpyAsync(kc, ctx->contributors.p, 8, cudaMemcpyDeviceToHost, s));
                CK(cudaMemsetAsync(ctx->contributors.p, 0, 8, s));
                CK(cudaStreamSynchronize(s));
                for (int v = 0; v < ngroup; ++v) {
                    h_missing[b0 + v0 + v] = ho[v];
                    h_entropy[b0 + v0 + v] = ho[ngroup + v];
                    if (h_fisher) h_fisher[b0 + v0 + v] = ho[2 * ngroup + v];
                }
                ctx->stats.contributors += *kc;
            } else {
                unsigned long long* kc = hp + 2 * B;
                CK(cudaMemcpyAsync(kc, ctx->contributors.p, 8, cudaMemcpyDeviceToHost, s));
                CK(cudaMemsetAsync(ctx->contributors.p, 0, 8, s));
                CK(cudaStreamSynchronize(s));
                ctx->stats.contributors += *kc;
            }
            if (ctx->profiling) {
                const int nsub = std::min(16, sub);
                for (int q = 0; q < nsub; ++q) {
                    float ms = 0;
                    CK(cudaEventElapsedTime(&ms, ctx->ev_r[2 * q], ctx->ev_r[2 * q + 1]));
                    ctx->stats.raster_ms += ms;
                }
            }
            v0 = v1;
        }
        if (ctx->profiling) {
            CK(cudaEventRecord(ctx->ev[3], s));
            CK(cudaEventSynchronize(ctx->ev[3]));
            float total = 0;
            CK(cudaEventElapsedTime(&total, ctx->ev[0], ctx->ev[3]));
            ctx->stats.binning_ms += total;  // whole-batch span; raster share in raster_ms
        }
        ctx->stats.views += nb;
        if (mode == Mode::Render) {
            ctx->last_valid = true;
            ctx->last_V = V[0];
            ctx->last_P = P[0];
            ctx->last_bin_tiles = bin_tiles;
            ctx->last_map = map;
            ctx->last_cam = cam;
            ctx->last_opt = o;
            ctx->last_pose = poses[0];
        }
    }
}

void map_ready(sgm_ctx* ctx, const sgm_map* cmap) {
    sgm_map* map = const_cast<sgm_map*>(cmap);  // the staging state is not the snapshot
    if (map->rows_pending) {
        map->rows_thread.join();
        map->rows_pending = false;
        if (ctx->rows_owner == map) ctx->rows_owner = nullptr;
        map->dev.dup_idx = map->rows_dup;
    }
    if (map->rows_code != SGM_OK) fail(map->rows_code, "map upload: %s", map->rows_msg.c_str());
    if (map->ev_rows) CK(cudaStreamWaitEvent(ctx->stream, map->ev_rows, 0));
    if (!map->dev.gbounds && map->dev.n) map_group_bounds(ctx, map, ctx->stream);
}

void map_records(sgm_ctx* ctx, const sgm_map* cmap) {
    sgm_map* map = const_cast<sgm_map*>(cmap);  // a derived array, like the group bounds
    if (map->rec_valid || map->dev.n == 0) return;
    CK(map->rec.reserve(16 * map->dev.n * static_cast<size_t>(map->dev.kpad)));
    map->dev.sem_rec = map->rec.as<uint4>();
    launch_sem_records(map->dev, map->rec.as<uint4>(), ctx->stream);
    ctx->stats.kernel_launches += 1;
    map->rec_valid = true;
}

void map_group_bounds(sgm_ctx* ctx, sgm_map* map, cudaStream_t s) {
    const size_t ns = std::max<uint64_t>(map->dev.n, 1);
    CK(map->gbnd.reserve(16 * ns));
    map->dev.gbounds = map->gbnd.as<uint4>();
    launch_group_bounds(map->dev, map->groups, map->gbnd.as<uint4>(), s);
    ctx->stats.kernel_launches += map->dev.n ? 1 : 0;
}

int guard(sgm_ctx* ctx, const std::function<void()>& fn) {
    try {
        fn();
        if (ctx) ctx->err.clear();
        return SGM_OK;
    } catch (const SgmError& e) {
        if (ctx) ctx->err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        if (ctx) ctx->err = "host allocation failed";
        return SGM_ERR_OOM;
    } catch (const std::exception& e) {
        if (ctx) ctx->err = e.what();
        return SGM_ERR_INVALID;
    }
}

void need_ctx(sgm_ctx* ctx) {
    if (!ctx) fail(SGM_ERR_INVALID, "ctx is null");
    CK(cudaSetDevice(ctx->device));
}

void do_render(sgm_ctx* ctx, const sgm_map* map, const sgm_camera* camera, const sgm_pose* pose,
               uint32_t channels, const sgm_options* opt, double* d_color, double* d_depth,
               double* d_sil, double* d_sem, uint64_t* n_proj, bool reference_form) {
    need_ctx(ctx);
    if (!map) fail(SGM_ERR_INVALID, "map is null");
    if (!pose) fail(SGM_ERR_INVALID, "pose is null");
    const CamParams cam = to_cam(camera);
    OptParams o = to_opt(opt, cam);
    o.ref_div = reference_form ? 1 : 0;
    const PoseParams p = to_pose(*pose);
    RenderTargets rt;
    rt.channels = channels;
    rt.color = (channels & SGM_COLOR) ? d_color : nullptr;
    rt.depth = (channels & SGM_DEPTH) ? d_depth : nullptr;
    rt.sem = (channels & SGM_SEMANTICS) ? d_sem : nullptr;
    rt.sil = d_sil;
    ctx->last_has_contrib = false;
    if (channels & SGM_RETAIN_CONTRIBUTORS) {
        // pass 1: per-pixel contributor counts (splat_render.cpp:215-216, 310)
        const size_t px = static_cast<size_t>(cam.W) * cam.H;
        CK(ctx->ccount.reserve(4 * (px + 1)));
        CK(ctx->coffset.reserve(8 * (px + 1)));
        CK(ctx->contrib.reserve(4));
        CK(cudaMemsetAsync(ctx->ccount.p, 0, 4 * (px + 1), ctx->stream));
        rt.contrib = ctx->contrib.as<uint32_t>();
        rt.contrib_count = ctx->ccount.as<uint32_t>();
        run_views(ctx, map, cam, o, 1, &p, Mode::Render, rt, nullptr, nullptr);
        // offsets = exclusive scan (flatten_contributors, :125-137)
        CK(ctx->scan_tmp.reserve(exclusive_scan_scratch_bytes(px + 1)));
        exclusive_scan_u64<uint32_t>(ctx->ccount.as<uint32_t>(), px + 1,
                                     ctx->coffset.as<unsigned long long>(),
                                     ctx->scan_tmp.as<unsigned long long>(), ctx->stream);
        ctx->stats.kernel_launches += exclusive_scan_launches(px + 1);
        unsigned long long total = 0;
        CK(cudaMemcpyAsync(&total, ctx->coffset.as<unsigned long long>() + px, 8,
                           cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        if (total >= (1ull << 32)) fail(SGM_ERR_UNSUPPORTED, "more than 2^32 contributors");
        CK(ctx->contrib.reserve(4 * std::max<unsigned long long>(total, 1)));
        // pass 2: write the depth-ordered contributor ranks
        rt.contrib = ctx->contrib.as<uint32_t>();
        rt.contrib_offset = ctx->coffset.as<unsigned long long>();
        run_views(ctx, map, cam, o, 1, &p, Mode::Render, rt, nullptr, nullptr);
        ctx->last_ncontrib = total;
        ctx->last_has_contrib = true;
        ctx->last_px = static_cast<int>(px);
    } else {
        run_views(ctx, map, cam, o, 1, &p, Mode::Render, rt, nullptr, nullptr);
    }
    if (n_proj) *n_proj = ctx->last_V;
}



// The mapping step on device-resident frame planes: render(all(true)) with contributor
// counts, mapping_loss + semantic_loss, backward, projection->world chain, KL clip and the
// finiteness check (losses.cpp:40-362). Gradients stay in ctx->bw_grad:
//   center 3NS | log_radius NS | opacity_logit NS | color 3NS | sem k*NS | proj 5NS
// (NS = max(N, 1)); report = LossReport fields. Throws like the reference on a non-finite
// gradient.
void backward_core(sgm_ctx* ctx, const sgm_map* map, const CamParams& cam, const OptParams& o,
                   const PoseParams& p, const float* f_rgb, const float* f_depth,
                   const float* f_sem, const double weights[7], int include_mapping,
                   int include_semantic, double report[7]) {
    cudaStream_t s = ctx->stream;
    const size_t px = static_cast<size_t>(cam.W) * cam.H;
    const int C = map->dev.C, k = map->dev.k;
    const uint64_t N = map->dev.n;
    const size_t NS = std::max<uint64_t>(N, 1);
    // device planes: rendered (sil, color, depth, sem) + frame (rgb, depth, sem)
    const size_t rend_b = 8 * px * (5 + C);
    CK(ctx->planes.reserve(rend_b));
    CK(ctx->ccount.reserve(4 * (px + 1)));
    CK(ctx->contrib.reserve(4));
    CK(ctx->bw_flags.reserve(px + 16));
    const size_t nlb = backward_loss_blocks(cam.W, cam.H);
    CK(ctx->bw_part.reserve(64 * nlb + 64 + 64));
    CK(ctx->bw_grad.reserve(8 * (NS * (8 + k) + 5 * NS) + 64));
    double* d_sil = ctx->planes.as<double>();
    double* d_color = d_sil + px;
    double* d_depth = d_color + 3 * px;
    double* d_sem = d_depth + px;
    CK(cudaMemsetAsync(ctx->ccount.p, 0, 4 * (px + 1), s));
    // 1. forward render + contributor counts (the reference's render(..., all(true)))
    RenderTargets rt;
    rt.channels = SGM_COLOR | SGM_DEPTH | SGM_SEMANTICS;
    rt.color = d_color;
    rt.depth = d_depth;
    rt.sil = d_sil;
    rt.sem = d_sem;
    rt.contrib = ctx->contrib.as<uint32_t>();
    rt.contrib_count = ctx->ccount.as<uint32_t>();
    run_views(ctx, map, cam, o, 1, &p, Mode::Render, rt, nullptr, nullptr);
    const uint32_t V = ctx->last_V;
    // 2. loss masks, reports and mask counts
    double* g = ctx->bw_grad.as<double>();
    BackwardParams b{};
    b.W = cam.W;
    b.H = cam.H;
    b.C = C;
    b.color = d_color;
    b.depth = d_depth;
    b.sil = d_sil;
    b.sem = d_sem;
    b.ccount = ctx->ccount.as<uint32_t>();
    b.rgb = f_rgb;
    b.fdepth = f_depth;
    b.fsem = f_sem;
    b.flags = ctx->bw_flags.as<uint8_t>();
    b.tau = std::log(weights[2]);
    b.lambda_hd = weights[0];
    b.lambda_cos = weights[1];
    b.use_hd = weights[3] != 0.0;
    b.use_cos = weights[4] != 0.0;
    b.use_kl = weights[5] != 0.0;
    b.include_mapping = include_mapping != 0;
    b.include_semantic = include_semantic != 0;
    double* totals = ctx->bw_part.as<double>() + 8 * nlb;
    b.totals = totals;
    b.gcenter = g;
    b.glogr = g + 3 * NS;
    b.glogit = g + 4 * NS;
    b.gcolor = g + 5 * NS;
    b.gsem = g + 8 * NS;
    b.gproj = g + (8 + k) * NS;
    b.sem_perm = map->dev.sem_perm;
    CK(cudaMemsetAsync(g, 0, 8 * (NS * (8 + k) + 5 * NS), s));
    launch_loss_pixels(b, ctx->bw_part.as<double>(), totals, s);
    // 3. backward over the block lists of the render above (same binning)
    RasterParams rp{};
    rp.map = map->dev;
    rp.cam = cam;
    rp.opt = o;
    rp.views = ctx->views.as<ViewDesc>();
    rp.tiles_per_view = ((cam.W + kTile - 1) / kTile) * ((cam.H + kTile - 1) / kTile);
    rp.raster_tiles_x = (cam.W + kTile - 1) / kTile;
    rp.channels = rt.channels;
    rp.groups = map->groups;
    need_smem(ctx->device, backward_smem_bytes(map->dev.C, map->dev.kpad), map->dev.C, "backward");
    launch_backward(rp, b, s);
    // 4. projection -> world, KL clipping, finiteness
    launch_chain(map->dev, ctx->poses.as<PoseParams>(), cam, o, ctx->vals.as<uint32_t>(), V,
                 b.gproj, b, s);
    if (b.use_kl && b.include_semantic && weights[6] > 0.0)
        launch_kl_clip(b.gsem, N, k, weights[6], s);
    unsigned long long* bad = reinterpret_cast<unsigned long long*>(totals + 8);
    CK(cudaMemsetAsync(bad, 0xff, 5 * 8, s));
    const double* arrs[5] = {b.gcenter, b.glogr, b.glogit, b.gcolor, b.gsem};
    const uint64_t lens[5] = {3 * N, N, N, 3 * N, static_cast<uint64_t>(k) * N};
    for (int a = 0; a < 5; ++a) launch_finite(arrs[a], lens[a], bad + a, s);
    ctx->stats.kernel_launches += 4 + 5;
    CK(cudaGetLastError());
    double h_tot[8];
    unsigned long long h_bad[5];
    CK(cudaMemcpyAsync(h_tot, totals, 64, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(h_bad, bad, 40, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    static const char* names[5] = {"center", "log_radius", "opacity_logit", "color", "sem"};
    static const uint64_t stride[5] = {3, 1, 1, 3, 0};
    for (int a = 0; a < 5; ++a)
        if (h_bad[a] != ~0ull)  // losses.cpp:349-360
            fail(SGM_ERR_INVALID, "backward: non-finite gradient for gaussian %llu parameter %s",
                 static_cast<unsigned long long>(h_bad[a] / (a == 4 ? k : stride[a])), names[a]);
    report[0] = h_tot[3] > 0 ? h_tot[0] / h_tot[3] : 0.0;  // photometric (:57)
    report[1] = h_tot[4] > 0 ? h_tot[1] / h_tot[4] : 0.0;  // depth (:58)
    report[2] = h_tot[5] > 0 ? h_tot[2] / h_tot[5] : 0.0;  // semantic (:158)
    report[3] = h_tot[3];
    report[4] = h_tot[4];
    report[5] = h_tot[5];
    report[6] = h_tot[6];
}



// Device -> pageable host copies of large planes (a full render is px (5 + C) doubles:
// 698 MB at cfg1). A plain cudaMemcpy to pageable memory is staged by the driver at about
// 15 GB/s and pays the fresh pages' faults serially; here the planes go through a ring of
// pinned buffers in kChunk pieces (DMA at full PCIe rate) while a pool of host threads
// copies the finished pieces out in parallel.
void copy_out(sgm_ctx* ctx, const std::vector<CopyOut>& segs) {
    constexpr size_t kChunk = size_t(16) << 20;
    constexpr int kSlots = 4;
    cudaStream_t s = ctx->stream;
    size_t total = 0;
    for (const auto& g : segs) total += g.bytes;
    if (total <= 2 * kChunk) {  // small: direct copies
        for (const auto& g : segs)
            CK(cudaMemcpyAsync(g.dst, g.src, g.bytes, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        return;
    }
    struct Piece {
        char* dst;
        const char* src;
        size_t bytes;
    };
    std::vector<Piece> pieces;
    for (const auto& g : segs)
        for (size_t o = 0; o < g.bytes; o += kChunk)
            pieces.push_back({static_cast<char*>(g.dst) + o, static_cast<const char*>(g.src) + o,
                              std::min(kChunk, g.bytes - o)});
    CK(ctx->h_ring.reserve(kSlots * kChunk));
    for (int k = 0; k < kSlots; ++k)
        if (!ctx->ev_ring[k]) CK(cudaEventCreateWithFlags(&ctx->ev_ring[k], cudaEventDisableTiming));
    const unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const size_t np = pieces.size();
    std::unique_ptr<std::atomic<unsigned>[]> copied(new std::atomic<unsigned>[np]);
    for (size_t j = 0; j < np; ++j) copied[j].store(0);
    std::atomic<size_t> issued{0};  // pieces whose D2H + event are enqueued
    std::atomic<int> err{0};
    auto worker = [&](unsigned w) {
        // this thread's runtime calls must target the ctx's device (not device 0)
        if (cudaSetDevice(ctx->device) != cudaSuccess) {
            err.store(1);
            return;
        }
        for (size_t j = 0; j < np; ++j) {
            while (issued.load(std::memory_order_acquire) <= j && !err.load()) std::this_thread::yield();
            if (err.load()) return;
            const int slot = static_cast<int>(j % kSlots);
            if (cudaEventSynchronize(ctx->ev_ring[slot]) != cudaSuccess) err.store(1);
            const Piece& pc = pieces[j];
            const size_t a = pc.bytes * w / nth, b = pc.bytes * (w + 1) / nth;
            std::memcpy(pc.dst + a, ctx->h_ring.as<char>() + slot * kChunk + a, b - a);
            copied[j].fetch_add(1, std::memory_order_release);
        }
    };
    std::vector<std::thread> pool;
    for (unsigned w = 0; w < nth; ++w) pool.emplace_back(worker, w);
    cudaError_t e = cudaSuccess;
    for (size_t j = 0; j < np && e == cudaSuccess; ++j) {
        const int slot = static_cast<int>(j % kSlots);
        if (j >= kSlots)  // the slot's previous piece must be copied out first
            while (copied[j - kSlots].load(std::memory_order_acquire) < nth && !err.load())
                std::this_thread::yield();
        e = cudaMemcpyAsync(ctx->h_ring.as<char>() + slot * kChunk, pieces[j].src, pieces[j].bytes,
                            cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_ring[slot], s);
        issued.store(j + 1, std::memory_order_release);
    }
    if (e != cudaSuccess) err.store(1);
    for (auto& th : pool) th.join();
    CK(e);
    if (err.load()) fail(SGM_ERR_CUDA, "device-to-host copy failed");
    CK(cudaStreamSynchronize(s));
}


}  // namespace sgm
