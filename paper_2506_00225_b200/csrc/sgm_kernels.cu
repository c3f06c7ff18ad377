// B200 (sm_100a) kernels of the candidate-view render + scoring path.
//
// Compiled with --fmad=false: every fp64/fp32 expression below is evaluated
// with one rounding per operation, in the reference's C++ evaluation order, so
// projections and tile rectangles are bit-identical to the reference build
// (which has no FMA: proj/CMakeLists.txt:3,8-10, default -march=x86-64).
//
//   K1 k_preprocess      project_splats transform/cull + tile count   splat_render.cpp:15-39, 205-209
//   K2 CUB radix sort on the fp32-rounded depth (monotone) + k_tiefix: runs of
//      equal fp32 keys re-sorted by the full fp64 (z, mx, my, alpha) key  splat_render.cpp:40-45
//   K3 k_pack, then row-bucketed binning without sorting the (tile, rank) pairs:
//      k_bin_hist + k_bin_scan (tile ranges from a 2D difference array), k_emit_rows + CUB
//      stable row sort (each tile row's ranks in rank order), k_row_segs / k_seg_pass /
//      k_seg_scan (ordered, coalesced scatter into the tile lists)   splat_render.cpp:189-213
//   K4/K5 raster: see sgm_raster.cu
//   k_reduce_scores     deterministic per-view n_missing / entropy_sum   explorer.cpp:195-203
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdio>

#include "sgm_internal.h"

namespace sgm {

namespace {

// static_cast<int>(double) as the reference binary executes it (x86-64
// cvttsd2si): out-of-range and NaN give INT_MIN. CUDA's cvt saturates instead.
__device__ __forceinline__ int to_int_x86(double v) {
    return (v > -2147483649.0 && v < 2147483648.0) ? static_cast<int>(v) : INT_MIN;
}

// Projection of one Gaussian: centre, depth, the binning reach per axis and, in
// the anisotropic mode, the conic.
struct Proj {
    double mx, my, z, rad;  // rad: rad_px (isotropic) / sqrt(largest eigenvalue) (anisotropic)
    double rx, ry;          // truncated reach along x / y (isotropic: trunc * rad_px, :34, :205)
    double qa, qb, qc;      // anisotropic only: inverse 2D covariance
};

// EWA projection (no reference): Sigma2D = J R_cw Sigma R_cw^T J^T with J
// the pinhole Jacobian at pc. Same operation order as oracle/sgm_oracle.c ewa_project
// (no contraction), so projections and bins are bit-identical to the oracle.
__device__ __forceinline__ bool ewa(const DevMap& m, uint64_t i, const PoseParams& P,
                                    const CamParams& cam, const OptParams& o, double pcx,
                                    double pcy, double pcz, Proj& q) {
    // Jacobian at the view direction clamped to 1.3x the half field of view (as 3D
    // Gaussian splatting does), so off-frustum centres near z_near stay bounded
    const double limx = 1.3 * ((0.5 * cam.W) / cam.fx);
    const double limy = 1.3 * ((0.5 * cam.H) / cam.fy);
    const double rxz = pcx / pcz, ryz = pcy / pcz;
    const double txz = rxz < -limx ? -limx : (limx < rxz ? limx : rxz);  // std::clamp order
    const double tyz = ryz < -limy ? -limy : (limy < ryz ? limy : ryz);
    const double tx = txz * pcz, ty = tyz * pcz;
    const double zz = pcz * pcz;
    const double j00 = cam.fx / pcz, j02 = -(cam.fx * tx) / zz;
    const double j11 = cam.fy / pcz, j12 = -(cam.fy * ty) / zz;
    const double* R = P.Rcw;  // row-major R_cw
    const double a0 = j00 * R[0] + j02 * R[6], a1 = j00 * R[1] + j02 * R[7], a2 = j00 * R[2] + j02 * R[8];
    const double b0 = j11 * R[3] + j12 * R[6], b1 = j11 * R[4] + j12 * R[7], b2 = j11 * R[5] + j12 * R[8];
    const uint64_t n = m.n;
    const double sxx = m.cov[i], sxy = m.cov[n + i], sxz = m.cov[2 * n + i];
    const double syy = m.cov[3 * n + i], syz = m.cov[4 * n + i], szz = m.cov[5 * n + i];
    const double ta0 = (sxx * a0 + sxy * a1) + sxz * a2;
    const double ta1 = (sxy * a0 + syy * a1) + syz * a2;
    const double ta2 = (sxz * a0 + syz * a1) + szz * a2;
    const double tb0 = (sxx * b0 + sxy * b1) + sxz * b2;
    const double tb1 = (sxy * b0 + syy * b1) + syz * b2;
    const double tb2 = (sxz * b0 + syz * b1) + szz * b2;
    const double va = (a0 * ta0 + a1 * ta1) + a2 * ta2;
    const double vb = (b0 * ta0 + b1 * ta1) + b2 * ta2;
    const double vc = (b0 * tb0 + b1 * tb1) + b2 * tb2;
    const double det = va * vc - vb * vb;
    if (!(det > 0.0)) return false;
    q.rx = o.trunc * sqrt(va);
    q.ry = o.trunc * sqrt(vc);
    if (q.mx + q.rx < 0 || q.mx - q.rx > cam.W || q.my + q.ry < 0 || q.my - q.ry > cam.H)
        return false;
    q.qa = vc / det;
    q.qb = -vb / det;
    q.qc = va / det;
    const double hm = 0.5 * (va + vc), hd = 0.5 * (va - vc);
    q.rad = sqrt(hm + sqrt(hd * hd + vb * vb));
    return true;
}

// project_splats for one Gaussian (splat_render.cpp:24-37). Returns visibility.
__device__ __forceinline__ bool project(const DevMap& m, uint64_t i, const PoseParams& P,
                                        const CamParams& cam, const OptParams& o, Proj& q) {
    const double d0 = m.cx[i] - P.t[0];
    const double d1 = m.cy[i] - P.t[1];
    const double d2 = m.cz[i] - P.t[2];
    // Eigen lazy coefficient product: row = x0 + (x1 + x2)  (:25)
    const double pcz = P.Rcw[6] * d0 + (P.Rcw[7] * d1 + P.Rcw[8] * d2);
    if (pcz <= o.z_near) return false;  // :26
    const double pcx = P.Rcw[0] * d0 + (P.Rcw[1] * d1 + P.Rcw[2] * d2);
    const double pcy = P.Rcw[3] * d0 + (P.Rcw[4] * d1 + P.Rcw[5] * d2);
    q.z = pcz;
    q.mx = cam.fx * pcx / pcz + cam.cx;  // :29
    q.my = cam.fy * pcy / pcz + cam.cy;  // :30
    if (m.aniso) return ewa(m, i, P, cam, o, pcx, pcy, pcz, q);
    q.rad = m.rad[i] * cam.fy / pcz;     // :31 (exp done on host)
    const double reach = o.trunc * q.rad;  // :34
    q.rx = q.ry = reach;
    if (q.mx + reach < 0 || q.mx - reach > cam.W || q.my + reach < 0 || q.my - reach > cam.H)
        return false;  // :35-37
    return true;
}

struct Rect {
    int tx0, tx1, ty0, ty1;
};

__device__ __forceinline__ Rect tile_rect(const Proj& q, const OptParams& o) {
    // reach = trunc * rad_px (:205), per axis in the anisotropic mode
    Rect r;
    r.tx0 = max(0, to_int_x86((q.mx - q.rx) / o.ts));               // :206
    r.tx1 = min(o.tiles_x - 1, to_int_x86((q.mx + q.rx) / o.ts));   // :207
    r.ty0 = max(0, to_int_x86((q.my - q.ry) / o.ts));               // :208
    r.ty1 = min(o.tiles_y - 1, to_int_x86((q.my + q.ry) / o.ts));   // :209
    return r;
}

__device__ __forceinline__ unsigned long long rect_count(const Rect& r) {
    if (r.tx1 < r.tx0 || r.ty1 < r.ty0) return 0ull;
    return static_cast<unsigned long long>(r.tx1 - r.tx0 + 1) *
           static_cast<unsigned long long>(r.ty1 - r.ty0 + 1);
}

// ---------------------------------------------------------------- K1
// grid (ceil(N/256), views). Compacts visible Gaussians per view (order is
// arbitrary; the full-key sort below canonicalises it) and counts pairs.
// Order-preserving map of a float to uint32 (negative values reversed).
__device__ __forceinline__ uint32_t sortable(float f) {
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__global__ void __launch_bounds__(256) k_preprocess(DevMap m, const PoseParams* __restrict__ poses,
                                                    CamParams cam, OptParams o, uint32_t* keys,
                                                    uint32_t* vals, size_t stride,
                                                    uint32_t* vcount,
                                                    unsigned long long* pcount,
                                                    unsigned long long* rcount) {
    const int v = blockIdx.y;
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const PoseParams& P = poses[v];
    Proj q;
    const bool vis = i < m.n && project(m, i, P, cam, o, q);
    const Rect rc0 = vis ? tile_rect(q, o) : Rect{0, -1, 0, -1};
    unsigned long long cnt = vis ? rect_count(rc0) : 0ull;
    unsigned long long rows = cnt ? static_cast<unsigned long long>(rc0.ty1 - rc0.ty0 + 1) : 0ull;

    // block-aggregated compaction: one atomic per block and view (per-warp atomics on the
    // view's counter serialise in L2 and dominated this kernel)
    const unsigned mask = __ballot_sync(0xffffffffu, vis);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        cnt += __shfl_down_sync(0xffffffffu, cnt, off);
        rows += __shfl_down_sync(0xffffffffu, rows, off);
    }
    __shared__ uint32_t wvis[8];
    __shared__ unsigned long long wcnt[8], wrows[8];
    __shared__ uint32_t bbase;
    if (lane == 0) {
        wvis[warp] = static_cast<uint32_t>(__popc(mask));
        wcnt[warp] = cnt;
        wrows[warp] = rows;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tot = 0;
        unsigned long long tc = 0, tr = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
            const uint32_t c = wvis[w];
            wvis[w] = tot;  // exclusive offset of warp w
            tot += c;
            tc += wcnt[w];
            tr += wrows[w];
        }
        bbase = tot ? atomicAdd(&vcount[v], tot) : 0u;
        if (tc) {
            atomicAdd(&pcount[v], tc);
            atomicAdd(&rcount[v], tr);
        }
    }
    __syncthreads();
    if (vis) {
        const uint32_t pos = bbase + wvis[warp] + __popc(mask & ((1u << lane) - 1u));
        keys[v * stride + pos] = sortable(static_cast<float>(q.z));  // monotone in z
        vals[v * stride + pos] = static_cast<uint32_t>(i);
    }
}

// ---------------------------------------------------------------- K2 tie fix-up
// The radix sort orders by fp32(z), which is monotone in z, so the exact order
// (z, mx, my, alpha) of splat_render.cpp:40-45 only has to be restored inside
// runs of equal fp32 keys (map index breaks exact 4-key ties, which std::sort
// leaves unspecified). One thread per run: insertion sort for short runs,
// heapsort for long ones (degenerate maps, e.g. a fronto-parallel plane).
struct FullKey {
    double z, mx, my, al;
    uint32_t i;
};

__device__ __forceinline__ FullKey full_key(const DevMap& m, uint32_t i, const PoseParams& P,
                                            const CamParams& cam, const OptParams& o) {
    FullKey k;
    Proj q;
    project(m, i, P, cam, o, q);
    k.mx = q.mx;
    k.my = q.my;
    k.z = q.z;
    k.al = m.alpha[i];
    k.i = i;
    return k;
}

__device__ __forceinline__ bool key_less(const FullKey& a, const FullKey& b) {
    if (a.z != b.z) return a.z < b.z;
    if (a.mx != b.mx) return a.mx < b.mx;
    if (a.my != b.my) return a.my < b.my;
    if (a.al != b.al) return a.al < b.al;
    return a.i < b.i;
}

__global__ void k_tiefix(DevMap m, const PoseParams* __restrict__ pose, CamParams cam, OptParams o,
                         const uint32_t* __restrict__ key, uint32_t* idx, uint32_t V) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r + 1 >= V) return;
    if (key[r] != key[r + 1]) return;
    if (r > 0 && key[r - 1] == key[r]) return;  // not the head of the run
    uint32_t e = r + 1;
    while (e < V && key[e] == key[r]) ++e;
    const PoseParams P = *pose;
    const uint32_t n = e - r;
    uint32_t* a = idx + r;
    if (n <= 32) {
        for (uint32_t q = 1; q < n; ++q) {
            const uint32_t iq = a[q];
            const FullKey kq = full_key(m, iq, P, cam, o);
            uint32_t b = q;
            while (b > 0) {
                const FullKey kb = full_key(m, a[b - 1], P, cam, o);
                if (!key_less(kq, kb)) break;
                a[b] = a[b - 1];
                --b;
            }
            a[b] = iq;
        }
        return;
    }
    // heapsort (max-heap) on a[0, n)
    auto sift = [&](uint32_t root, uint32_t end) {
        while (true) {
            uint32_t child = 2 * root + 1;
            if (child >= end) break;
            FullKey kc = full_key(m, a[child], P, cam, o);
            if (child + 1 < end) {
                const FullKey k2 = full_key(m, a[child + 1], P, cam, o);
                if (key_less(kc, k2)) {
                    ++child;
                    kc = k2;
                }
            }
            if (!key_less(full_key(m, a[root], P, cam, o), kc)) break;
            const uint32_t tmp = a[root];
            a[root] = a[child];
            a[child] = tmp;
            root = child;
        }
    };
    for (uint32_t s0 = n / 2; s0-- > 0;) sift(s0, n);
    for (uint32_t end = n - 1; end > 0; --end) {
        const uint32_t tmp = a[0];
        a[0] = a[end];
        a[end] = tmp;
        sift(0, end);
    }
}

// ---------------------------------------------------------------- K3
// PackedSplat + Probe per depth rank (splat_render.cpp:191-204) and tile counts.
__global__ void k_pack(DevMap m, const PoseParams* __restrict__ pose, CamParams cam, OptParams o,
                       GroupParams gp, const uint32_t* __restrict__ idx, uint32_t V,
                       PackedSplat* packed, unsigned long long* counts, int4* rects,
                       uint4* bounds) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= V) return;
    const uint32_t i = idx[r];
    Proj q;
    project(m, i, *pose, cam, o, q);
    const uint32_t aux = r;  // depth rank (contributor id)
    if (m.aniso) {
        PackedSplatA pa;
        pa.mx = q.mx;
        pa.my = q.my;
        pa.qa = q.qa;
        pa.qb = q.qb;
        pa.alpha = m.alpha[i];
        pa.z = q.z;
        pa.qc = q.qc;
        pa.pad = 0;
        pa.aux = aux;
        reinterpret_cast<PackedSplatA*>(packed)[r] = pa;
    } else {
        const double rad = q.rad;
        PackedSplat ps;
        ps.mx = q.mx;
        ps.my = q.my;
        // :194; render_reference keeps the divisor 2 r^2 itself (:91)
        ps.inv_two_r2 = o.ref_div ? 2.0 * rad * rad : 1.0 / (2.0 * rad * rad);
        ps.cutoff_d2 = o.cut_sq * rad * rad;      // :195
        ps.alpha = m.alpha[i];
        ps.z = q.z;
        ps.pmx = static_cast<float>(q.mx);  // :201
        ps.pmy = static_cast<float>(q.my);  // :202
        ps.pcut = static_cast<float>(ps.cutoff_d2 * (1.0 + 1e-5)) + 1e-6f;  // :203
        ps.aux = aux;
        packed[r] = ps;
    }
    const Rect rc = tile_rect(q, o);
    counts[r] = rect_count(rc);
    rects[r] = make_int4(rc.tx0, rc.ty0, rc.tx1 - rc.tx0 + 1, rc.ty1 - rc.ty0 + 1);
    (void)gp;
    (void)bounds;  // the channel-group bounds are per map (k_group_bounds), not per view
}

// Raster channel groups of each Gaussian's class-sorted row: b[g] = #entries with class <
// (g + 1) * Cg for g = 0..6, b[7] = k (u16 each). Per map, once (not per view): the binning
// then needs no semantic rows, so their upload can overlap it.
__global__ void k_group_bounds(DevMap m, GroupParams gp, uint4* __restrict__ out) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m.n) return;
    const uint16_t* row = m.sem_idx + i * m.kpad;
    uint32_t b[8];
    int j = 0;
    for (int g = 0; g < 7; ++g) {
        const int lim = (g + 1) * gp.Cg;
        while (j < m.k && row[j] < lim) ++j;
        b[g] = static_cast<uint32_t>(j);
    }
    b[7] = static_cast<uint32_t>(m.k);
    out[i] = make_uint4(b[0] | (b[1] << 16), b[2] | (b[3] << 16), b[4] | (b[5] << 16), b[6] | (b[7] << 16));
}

// Emits (tile row, rank | column range) pairs in rank order at the scanned per-rank row
// counts: one per tile row a rectangle spans; a stable sort on the row key then yields
// every row's ranks in rank order (the input of the per-row scatter below).
// Load-balanced: each thread emits kPerThread consecutive pairs. The first pair's rank
// comes from a binary search over the scanned counts; then the thread walks forward
// (pairs of one rank are contiguous).
constexpr int kPerThread = 8;
__global__ void k_emit_rows(const unsigned long long* __restrict__ offsets, const int4* __restrict__ rects,
                            uint32_t V, unsigned long long R, uint32_t* row_keys,
                            unsigned long long* row_vals) {
    const unsigned long long i0 =
        (static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x) * kPerThread;
    if (i0 >= R) return;
    // largest r with offsets[r] <= i0
    uint32_t lo = 0, hi = V;  // offsets[V] == R > i0
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) / 2;
        if (offsets[mid] <= i0) lo = mid; else hi = mid;
    }
    uint32_t r = lo;
    unsigned long long beg = offsets[r], end = offsets[r + 1];
    int4 rc = rects[r];
    const unsigned long long i1 = min(R, i0 + kPerThread);
    for (unsigned long long i = i0; i < i1; ++i) {
        if (i >= end) {
            ++r;
            beg = end;
            end = offsets[r + 1];
            if (i >= end) {  // ranks without pairs (depth-prefix binning skips most): search
                uint32_t a = r, b = V;
                while (b - a > 1) {
                    const uint32_t mid = (a + b) / 2;
                    if (offsets[mid] <= i) a = mid; else b = mid;
                }
                r = a;
                beg = offsets[r];
                end = offsets[r + 1];
            }
            rc = rects[r];
        }
        const uint32_t j = static_cast<uint32_t>(i - beg);
        row_keys[i] = static_cast<uint32_t>(rc.y) + j;
        row_vals[i] = (static_cast<unsigned long long>(r) << 32) |
                      (static_cast<unsigned long long>(rc.x) << 16) |
                      static_cast<unsigned long long>(rc.x + rc.z - 1);
    }
}

// ---------------------------------------------------------------- row-bucketed binning
// The bins of :210-212 are, per tile, the ranks whose rectangle covers the tile, in rank
// order. Built without sorting the (tile, rank) pairs:
//   k_bin_hist   per rank: 2D difference-array corners of its rectangle (tile counts) and
//                its row count (number of tile rows spanned);
//   k_bin_scan   one CTA: 2D prefix of the difference array -> per-tile counts -> exclusive
//                scan in bin order -> ranges[bin] = (begin, end);
//   rows         (row, rank) pairs emitted in rank order and stably sorted by row (small:
//                one pair per spanned row, not per tile) -> each row's ranks in rank order;
//   row scatter  each row's ranks cut into segments of kSeg; per (segment, 32 columns) one
//                warp appends the covering ranks to the columns' lists in rank order
//                (k_row_segs, k_seg_count, k_seg_scan, k_seg_pass below).
__global__ void k_bin_hist(const int4* __restrict__ rects, uint32_t V, int tiles_x,
                           int* __restrict__ diff, unsigned long long* __restrict__ rows) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= V) return;
    const int4 rc = rects[r];
    const bool any = rc.z > 0 && rc.w > 0;
    rows[r] = any ? static_cast<unsigned long long>(rc.w) : 0ull;
    if (!any) return;
    const int X = tiles_x + 1;
    const int x0 = rc.x, x1 = rc.x + rc.z, y0 = rc.y, y1 = rc.y + rc.w;  // half-open
    atomicAdd(&diff[y0 * X + x0], 1);
    atomicAdd(&diff[y0 * X + x1], -1);
    atomicAdd(&diff[y1 * X + x0], -1);
    atomicAdd(&diff[y1 * X + x1], 1);
}

// Depth-prefix binning, pass 1: which ranks can reach a bin's first `cap` entries. The
// ranks are cut into kRankChunks chunks; per chunk, the bins' entry counts (2D difference
// arrays, one per chunk); a bin is open in chunk c while fewer than cap entries precede the
// chunk; a rank of chunk c whose rectangle covers no open bin is in no bin's prefix, so it
// emits no row pairs (k_bin_hist_prefix). Its entries still count, so the truncation flags
// and capped counts are the full lists'.
__global__ void k_chunk_hist(const int4* __restrict__ rects, uint32_t V, int nc, int tiles_x, int tiles_y,
                             int* __restrict__ diffc) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= V) return;
    const int4 rc = rects[r];
    if (rc.z <= 0 || rc.w <= 0) return;
    const int X = tiles_x + 1, Y = tiles_y + 1;
    int* d = diffc + static_cast<size_t>(static_cast<uint64_t>(r) * nc / V) * X * Y;
    const int x0 = rc.x, x1 = rc.x + rc.z, y0 = rc.y, y1 = rc.y + rc.w;
    atomicAdd(&d[y0 * X + x0], 1);
    atomicAdd(&d[y0 * X + x1], -1);
    atomicAdd(&d[y1 * X + x0], -1);
    atomicAdd(&d[y1 * X + x1], 1);
}

// In place, one CTA per chunk: inclusive 2D prefix sums of a W x H int array (pitch W):
// rows (a warp per row, 32 columns at a time) then columns (a thread per column).
__global__ void __launch_bounds__(1024) k_prefix2d(int* __restrict__ a, int W, int H) {
    int* d = a + static_cast<size_t>(blockIdx.x) * W * H;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    for (int y = warp; y < H; y += 32) {
        int carry = 0;
        for (int x0 = 0; x0 < W; x0 += 32) {
            const int x = x0 + lane;
            int v = x < W ? d[y * W + x] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += u;
            }
            v += carry;
            if (x < W) d[y * W + x] = v;
            carry = __shfl_sync(0xffffffffu, v, 31);
        }
    }
    __syncthreads();
    for (int x = t; x < W; x += blockDim.x) {
        int acc = 0;
        for (int y = 0; y < H; ++y) {
            acc += d[y * W + x];
            d[y * W + x] = acc;
        }
    }
}

// per bin: open flags per chunk into the summed-area arrays (one-cell zero border:
// sat[c][(y + 1) * (X) + x + 1] with X = tiles_x + 1)
__global__ void k_chunk_open(const int* __restrict__ cnt, int nc, int tiles_x, int tiles_y, uint32_t cap,
                             int* __restrict__ sat) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= tiles_x * tiles_y) return;
    const int y = i / tiles_x, x = i - y * tiles_x;
    const int X = tiles_x + 1, Y = tiles_y + 1;
    uint32_t cum = 0;
    for (int c = 0; c < nc; ++c) {
        sat[static_cast<size_t>(c) * X * Y + (y + 1) * X + x + 1] = cum < cap ? 1 : 0;
        cum += static_cast<uint32_t>(cnt[static_cast<size_t>(c) * X * Y + y * X + x]);
    }
}

// k_bin_hist for pass 1: every rank counts in its bins; only ranks covering an open bin of
// their chunk get row pairs
// the whole view's difference array: the sum of the chunks' (before their prefix sums)
__global__ void k_chunk_sum(const int* __restrict__ diffc, int nc, int cells, int* __restrict__ diff) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cells) return;
    int v = 0;
    for (int c = 0; c < nc; ++c) v += diffc[static_cast<size_t>(c) * cells + i];
    diff[i] = v;
}

// k_bin_hist for pass 1: only ranks covering an open bin of their chunk get row pairs (the
// view's bin counts come from the chunks' difference arrays, k_chunk_sum)
__global__ void k_bin_hist_prefix(const int4* __restrict__ rects, uint32_t V, int nc, int tiles_x,
                                  int tiles_y, const int* __restrict__ sat, unsigned long long* __restrict__ rows) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= V) return;
    const int4 rc = rects[r];
    rows[r] = 0ull;
    if (rc.z <= 0 || rc.w <= 0) return;
    const int X = tiles_x + 1, Y = tiles_y + 1;
    const int x0 = rc.x, x1 = rc.x + rc.z, y0 = rc.y, y1 = rc.y + rc.w;  // half-open
    const int* S = sat + static_cast<size_t>(static_cast<uint64_t>(r) * nc / V) * X * Y;
    const int open = S[y1 * X + x1] - S[y0 * X + x1] - S[y1 * X + x0] + S[y0 * X + x0];
    if (open > 0) rows[r] = static_cast<unsigned long long>(rc.w);
}

constexpr int kScanThreads = 1024;
// One CTA: the 2D difference array becomes per-tile counts (prefix along x: a warp per row,
// 32 columns at a time with shuffle scans; then along y: a thread per column, coalesced across
// the columns), then an exclusive scan over the bins in row-major order (1024 bins per round,
// warp scans + a carry) gives ranges[bin] = (begin, end).
__global__ void __launch_bounds__(kScanThreads) k_bin_scan(int* __restrict__ diff, int tiles_x,
                                                           int tiles_y, uint2* __restrict__ ranges,
                                                           const uint8_t* __restrict__ mask,
                                                           unsigned long long* __restrict__ total,
                                                           uint32_t cap, uint8_t* __restrict__ trunc) {
    const int X = tiles_x + 1;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    for (int y = warp; y < tiles_y; y += kScanThreads / 32) {
        int carry = 0;
        for (int x0 = 0; x0 < tiles_x; x0 += 32) {
            const int x = x0 + lane;
            int v = x < tiles_x ? diff[y * X + x] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += u;
            }
            v += carry;
            if (x < tiles_x) diff[y * X + x] = v;
            carry = __shfl_sync(0xffffffffu, v, 31);
        }
    }
    __syncthreads();
    for (int x = t; x < tiles_x; x += kScanThreads) {
        int acc = 0;
        for (int y = 0; y < tiles_y; ++y) {
            acc += diff[y * X + x];
            diff[y * X + x] = acc;
        }
    }
    __syncthreads();
    __shared__ uint32_t wsum[kScanThreads / 32];
    __shared__ uint32_t base;
    if (t == 0) base = 0u;
    const int T = tiles_x * tiles_y;
    for (int b0 = 0; b0 < T; b0 += kScanThreads) {
        const int b = b0 + t;
        uint32_t c = b < T ? static_cast<uint32_t>(diff[(b / tiles_x) * X + b % tiles_x]) : 0u;
        if (mask && b < T && !mask[b]) c = 0u;  // bins outside the mask get empty lists
        if (trunc && b < T) trunc[b] = c > cap ? 1 : 0;
        if (c > cap) c = cap;  // depth-prefix binning: the first `cap` entries of the bin
        uint32_t v = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
        }
        if (lane == 31) wsum[warp] = v;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t u = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += u;
            }
            wsum[lane] = w;  // inclusive over the warps
        }
        __syncthreads();
        const uint32_t begin = base + (warp ? wsum[warp - 1] : 0u) + v - c;
        if (b < T) ranges[b] = make_uint2(begin, begin + c);
        __syncthreads();
        if (t == kScanThreads - 1) base += wsum[kScanThreads / 32 - 1];
        __syncthreads();
    }
    if (total && t == 0) *total = base;
}

// the redo pass of depth-prefix binning: (view, tile) items and the bin mask of the tiles
// the raster reported incomplete
__global__ void k_redo_items(const uint32_t* __restrict__ incomplete, uint32_t n, uint32_t view,
                             int raster_tiles_x, int per_bin, int tiles_x, uint2* __restrict__ items,
                             uint8_t* __restrict__ mask) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t t = incomplete[i];
    items[i] = make_uint2(view, t);
    const int tx = static_cast<int>(t % raster_tiles_x), ty = static_cast<int>(t / raster_tiles_x);
    mask[(ty / per_bin) * tiles_x + tx / per_bin] = 1;
}

// Each tile row's list (ranks in rank order) is cut into segments of kSeg entries; a
// segment x 32-column block is one warp's work unit. The column cursors live in the
// registers of the lanes (lane l <-> column cb + l). Lanes load 32 consecutive entries of
// a chunk; a ballot keeps the entries whose column span meets the block. A sparse chunk
// (under two covering entries per column of the block: cfg1 / cfg3) is walked entry by entry
// in rank order, the entry broadcast and every lane whose column it covers appending its
// rank to that column's list; a dense chunk (cfg4) is walked column by column, a ballot
// giving the covering entries consecutive slots of the column's list (coalesced stores).
//   k_seg_count counts per (segment, column), k_seg_scan turns them into per-segment
//   bases, k_seg_pass writes. Segments of a row are independent, so dense rows spread over
//   the GPU.
constexpr int kSeg = 1024;

__global__ void __launch_bounds__(1024) k_row_segs(const uint2* __restrict__ row_ranges, int tiles_y,
                                                   uint4* __restrict__ segs, uint32_t* __restrict__ nseg_out) {
    // segment g = (row, begin, end, -): each row's list cut into kSeg pieces, rows in order.
    // Thread t owns a contiguous block of rows; a block scan places its segments.
    __shared__ uint32_t part[1024];
    const int t = threadIdx.x;
    const int per = (tiles_y + 1023) / 1024;
    const int y0 = min(tiles_y, t * per), y1 = min(tiles_y, y0 + per);
    uint32_t mine = 0;
    for (int y = y0; y < y1; ++y) {
        const uint2 rr = row_ranges[y];
        mine += (rr.y - rr.x + kSeg - 1) / kSeg;
    }
    part[t] = mine;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        const uint32_t v = t >= off ? part[t - off] : 0u;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    uint32_t g = part[t] - mine;
    for (int y = y0; y < y1; ++y) {
        const uint2 rr = row_ranges[y];
        for (uint32_t b = rr.x; b < rr.y; b += kSeg) segs[g++] = make_uint4(y, b, min(rr.y, b + kSeg), 0u);
    }
    if (t == 1023) *nseg_out = part[1023];
}

// kPart: depth-prefix binning (lists holding only a bin's first entries, or only the bins in
// `mask`): positions are relative to the bin and writes stop at the bin's list length. The
// plain instantiation writes every entry at absolute cursors.
template <bool kPart>
__global__ void __launch_bounds__(256) k_seg_pass(const unsigned long long* __restrict__ row_list,
                                                  const uint4* __restrict__ segs,
                                                  const uint32_t* __restrict__ nseg, int tiles_x,
                                                  const uint32_t* __restrict__ cnt, uint32_t* __restrict__ list,
                                                  const uint8_t* __restrict__ mask,
                                                  const uint2* __restrict__ tile_ranges) {
    const uint32_t g = blockIdx.x;
    if (g >= *nseg) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cb = (blockIdx.y * (blockDim.x >> 5) + warp) * 32;
    if (cb >= tiles_x) return;
    const uint4 sg = segs[g];
    const int col = cb + lane;
    bool has = col < tiles_x;
    uint32_t cur = 0, len = 0, base = 0;
    if (kPart) {
        has = has && (!mask || mask[static_cast<size_t>(sg.x) * tiles_x + col]);
        const uint2 tr = has ? tile_ranges[static_cast<size_t>(sg.x) * tiles_x + col] : make_uint2(0u, 0u);
        base = tr.x;
        len = tr.y - tr.x;
        cur = has ? cnt[static_cast<size_t>(g) * tiles_x + col] : 0u;  // position in the bin
        has = has && cur < len;
        // every column of this block already holds its list: nothing to do
        if (!__any_sync(0xffffffffu, has)) return;
    } else {
        cur = has ? cnt[static_cast<size_t>(g) * tiles_x + col] : 0u;  // absolute cursor
    }
    const int last = min(tiles_x, cb + 32) - 1;
    for (uint32_t b0 = sg.y; b0 < sg.z; b0 += 32) {
        // (kPart) the columns whose list still takes entries; none left: this warp is done
        const uint32_t open = kPart ? __ballot_sync(0xffffffffu, has && cur < len) : 0xffffffffu;
        if (kPart && !open) break;
        const bool valid = b0 + lane < sg.z;
        const unsigned long long e = valid ? row_list[b0 + lane] : 0ull;
        const int x0 = static_cast<int>((e >> 16) & 0xffffu);
        const int x1 = static_cast<int>(e & 0xffffu);
        const bool rel = valid && x0 <= last && x1 >= cb;
        uint32_t m = __ballot_sync(0xffffffffu, rel);
        if (!m) continue;
        // (entry, column) pairs of the chunk in this block: sparse below two per column
        const int span = rel ? min(x1, last) - max(x0, cb) + 1 : 0;
        if (__reduce_add_sync(0xffffffffu, static_cast<unsigned>(span)) < 64u) {
            while (m) {  // sparse: the chunk's entries that reach this block, in rank order
                const int j = __ffs(m) - 1;
                m &= m - 1u;
                const unsigned long long ej = __shfl_sync(0xffffffffu, e, j);
                const int jx0 = static_cast<int>((ej >> 16) & 0xffffu), jx1 = static_cast<int>(ej & 0xffffu);
                if (has && jx0 <= col && col <= jx1) {
                    if (kPart) {
                        if (cur < len) list[base + cur] = static_cast<uint32_t>(ej >> 32);
                        ++cur;
                    } else {
                        list[cur++] = static_cast<uint32_t>(ej >> 32);
                    }
                }
            }
        } else {
            // dense: per column, a ballot gives the covering entries consecutive slots of that
            // column's list (coalesced stores)
            const int lo = max(cb, __reduce_min_sync(0xffffffffu, rel ? x0 : INT_MAX));
            const int hi = min(last, __reduce_max_sync(0xffffffffu, rel ? x1 : INT_MIN));
            // the chunk's columns (kPart: the open ones only), ascending
            uint32_t cols = (0xffffffffu >> (31 - (hi - cb))) & (0xffffffffu << (lo - cb)) & open;
            while (cols) {
                const int owner = __ffs(cols) - 1;
                cols &= cols - 1u;
                const int c = cb + owner;
                const bool cov = rel && x0 <= c && c <= x1;
                const uint32_t bal = __ballot_sync(0xffffffffu, cov);
                const uint32_t at = __shfl_sync(0xffffffffu, cur, owner);
                const uint32_t pos = at + __popc(bal & ((1u << lane) - 1u));
                if (kPart) {
                    const uint32_t clen = __shfl_sync(0xffffffffu, len, owner);
                    const uint32_t cbase = __shfl_sync(0xffffffffu, base, owner);
                    if (cov && pos < clen) list[cbase + pos] = static_cast<uint32_t>(e >> 32);
                } else if (cov) {
                    list[pos] = static_cast<uint32_t>(e >> 32);
                }
                if (lane == owner) cur += __popc(bal);
            }
        }
    }
}

// Dense rows (cfg4: entries spanning tens of columns): one CTA per segment, the segment's
// column spans in registers (32 entries per lane) and ranks in shared memory; each warp walks
// whole columns, so a column's share of the segment (hundreds of entries) is written by one
// warp front to back: full sectors, instead of the block walk's few-entry pieces per chunk.
// kPart: depth-prefix binning (positions relative to the bin, writes stop at the bin's list
// length, bins outside `mask` skipped); a column whose list is full stops walking.
template <bool kPart>
__global__ void __launch_bounds__(256) k_seg_pass_cols(const unsigned long long* __restrict__ row_list,
                                                       const uint4* __restrict__ segs,
                                                       const uint32_t* __restrict__ nseg, int tiles_x,
                                                       const uint32_t* __restrict__ cnt,
                                                       uint32_t* __restrict__ list,
                                                       const uint8_t* __restrict__ mask,
                                                       const uint2* __restrict__ tile_ranges) {
    __shared__ uint32_t srank[kSeg];
    const uint32_t g = blockIdx.x;
    if (g >= *nseg) return;
    const uint4 sg = segs[g];
    const int n = static_cast<int>(sg.z - sg.y);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int kPer = kSeg / 32;
    if constexpr (kPart) {  // segments past every column's prefix (most of a dense row): nothing to load
        bool need = false;
        for (int col = threadIdx.x; col < tiles_x; col += blockDim.x) {
            const size_t bin = static_cast<size_t>(sg.x) * tiles_x + col;
            if (mask && !mask[bin]) continue;
            const uint2 tr = tile_ranges[bin];
            need = need || cnt[static_cast<size_t>(g) * tiles_x + col] < tr.y - tr.x;
        }
        if (!__syncthreads_or(need)) return;
    }
    // entry 32 k + lane of the segment: (first column << 16) | (last - first); past the end of
    // the segment an empty span (0xffff << 16 | 0: no column reaches it)
    uint32_t xw[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const int i = 32 * k + lane;
        const unsigned long long e = i < n ? row_list[sg.y + i] : 0ull;
        if (warp == 0 && i < n) srank[i] = static_cast<uint32_t>(e >> 32);
        const uint32_t a = static_cast<uint32_t>((e >> 16) & 0xffffu), b = static_cast<uint32_t>(e & 0xffffu);
        xw[k] = i < n ? (a << 16) | (b - a) : 0xffff0000u;
    }
    __syncthreads();
    const uint32_t lt = (1u << lane) - 1u;
    for (int col = warp; col < tiles_x; col += blockDim.x >> 5) {
        uint32_t cur = cnt[static_cast<size_t>(g) * tiles_x + col];
        if constexpr (kPart) {
            const size_t bin = static_cast<size_t>(sg.x) * tiles_x + col;
            if (mask && !mask[bin]) continue;
            const uint2 tr = tile_ranges[bin];
            const uint32_t len = tr.y - tr.x;
            uint32_t* out = list + tr.x;
            for (int k = 0; k < kPer && cur < len; ++k) {
                const bool cov = static_cast<uint32_t>(col) - (xw[k] >> 16) <= (xw[k] & 0xffffu);
                const uint32_t bal = __ballot_sync(0xffffffffu, cov);
                const uint32_t pos = cur + __popc(bal & lt);
                if (cov && pos < len) out[pos] = srank[32 * k + lane];
                cur += __popc(bal);
            }
        } else {
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                const bool cov = static_cast<uint32_t>(col) - (xw[k] >> 16) <= (xw[k] & 0xffffu);
                const uint32_t bal = __ballot_sync(0xffffffffu, cov);
                if (cov) list[cur + __popc(bal & lt)] = srank[32 * k + lane];
                cur += __popc(bal);
            }
        }
    }
}

// Pass 0 without ballots: a segment's per-column counts from a shared-memory difference
// array (+1 at x0, -1 at x1 + 1 per entry), prefix-summed over the columns.
__global__ void __launch_bounds__(256) k_seg_count(const unsigned long long* __restrict__ row_list,
                                                   const uint4* __restrict__ segs,
                                                   const uint32_t* __restrict__ nseg, int tiles_x,
                                                   uint32_t* __restrict__ cnt) {
    extern __shared__ int sdiff[];  // [tiles_x + 1]
    const uint32_t g = blockIdx.x;
    if (g >= *nseg) return;
    const uint4 sg = segs[g];
    for (int c = threadIdx.x; c <= tiles_x; c += blockDim.x) sdiff[c] = 0;
    __syncthreads();
    for (uint32_t i = sg.y + threadIdx.x; i < sg.z; i += blockDim.x) {
        const unsigned long long e = row_list[i];
        atomicAdd(&sdiff[(e >> 16) & 0xffffu], 1);
        atomicAdd(&sdiff[(e & 0xffffu) + 1], -1);
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // one warp: running prefix over the columns, 32 at a time
        int carry = 0;
        for (int c0 = 0; c0 < tiles_x; c0 += 32) {
            const int c = c0 + threadIdx.x;
            int v = c < tiles_x ? sdiff[c] : 0;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, v, off);
                if (static_cast<int>(threadIdx.x) >= off) v += u;
            }
            v += carry;
            if (c < tiles_x) cnt[static_cast<size_t>(g) * tiles_x + c] = static_cast<uint32_t>(v);
            carry = __shfl_sync(0xffffffffu, v, 31);
        }
    }
}

// per (row, column): exclusive scan of the segment counts over the row's segments: each
// segment's first list cursor (or position in the bin). One CTA per (row, 32 columns): the
// row's segments split over 8 warps (lane = column), warp sums combined in shared memory.
__global__ void __launch_bounds__(256) k_seg_scan(const uint4* __restrict__ segs,
                                                  const uint32_t* __restrict__ nseg,
                                                  const uint2* __restrict__ tile_ranges, int tiles_x,
                                                  int tiles_y, uint32_t* __restrict__ cnt) {
    const int y = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int x = blockIdx.y * 32 + lane;
    __shared__ uint32_t s_rng[2];
    __shared__ uint32_t wsum[8][32];
    if (threadIdx.x < 2) {  // the row's segments [first, end): contiguous, found by binary search
        const uint32_t G = *nseg;
        const int key = y + static_cast<int>(threadIdx.x);
        uint32_t lo = 0, hi = G;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) / 2;
            if (static_cast<int>(segs[mid].x) < key) lo = mid + 1; else hi = mid;
        }
        s_rng[threadIdx.x] = lo;
    }
    __syncthreads();
    const uint32_t g0 = s_rng[0], ng = s_rng[1] - s_rng[0];
    const uint32_t per = (ng + 7) / 8;
    const uint32_t a = g0 + min(ng, warp * per), b = g0 + min(ng, (warp + 1) * per);
    const bool on = x < tiles_x;
    uint32_t sum = 0;
    if (on)
        for (uint32_t g = a; g < b; ++g) sum += cnt[static_cast<size_t>(g) * tiles_x + x];
    wsum[warp][lane] = sum;
    __syncthreads();
    if (!on) return;
    // absolute list cursors, or (tile_ranges null: depth-prefix binning) positions in the bin
    uint32_t run = tile_ranges ? tile_ranges[static_cast<size_t>(y) * tiles_x + x].x : 0u;
    for (int w = 0; w < warp; ++w) run += wsum[w][lane];
    for (uint32_t g = a; g < b; ++g) {
        const size_t k = static_cast<size_t>(g) * tiles_x + x;
        const uint32_t c = cnt[k];
        cnt[k] = run;
        run += c;
    }
}

__global__ void k_ranges(const uint32_t* __restrict__ keys, uint64_t P, uint2* ranges) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= P) return;
    const uint32_t t = keys[i];
    if (i == 0 || keys[i - 1] != t) ranges[t].x = static_cast<uint32_t>(i);
    if (i + 1 == P || keys[i + 1] != t) ranges[t].y = static_cast<uint32_t>(i + 1);
}

// Per view: n_missing and entropy_sum from the per-tile partials, summed in a
// fixed order that depends only on the tile count (sharding-invariant).
__global__ void __launch_bounds__(256) k_reduce_scores(const ViewDesc* __restrict__ views, int tiles,
                                                       double* out_missing, double* out_entropy,
                                                       double* out_fisher) {
    __shared__ double sd[256];
    __shared__ double sf[256];
    __shared__ unsigned long long su[256];
    const ViewDesc vd = views[blockIdx.x];
    const int t = threadIdx.x;
    const int per = (tiles + 255) / 256;
    double h = 0.0, fi = 0.0;
    unsigned long long m = 0;
    for (int i = t * per; i < min(tiles, (t + 1) * per); ++i) {
        h += vd.ent_partial[i];
        m += vd.miss_partial[i];
        if (out_fisher) fi += vd.fis_partial[i];
    }
    sd[t] = h;
    su[t] = m;
    sf[t] = fi;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (t < s) {
            sd[t] += sd[t + s];
            su[t] += su[t + s];
            sf[t] += sf[t + s];
        }
        __syncthreads();
    }
    if (t == 0) {
        out_missing[blockIdx.x] = static_cast<double>(su[0]);
        out_entropy[blockIdx.x] = sd[0];
        if (out_fisher) out_fisher[blockIdx.x] = sf[0];
    }
}

__global__ void k_debug_projections(DevMap m, const PoseParams* __restrict__ pose, CamParams cam,
                                    OptParams o, const uint32_t* __restrict__ idx, uint32_t V,
                                    double* out6) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= V) return;
    const uint32_t i = idx[r];
    Proj q;
    project(m, i, *pose, cam, o, q);
    out6[6 * r] = q.mx;
    out6[6 * r + 1] = q.my;
    out6[6 * r + 2] = q.rad;
    out6[6 * r + 3] = q.z;
    out6[6 * r + 4] = m.alpha[i];
    out6[6 * r + 5] = static_cast<double>(i);
}

__global__ void k_bins_to_ids(const uint32_t* __restrict__ list, uint64_t P,
                              const PackedSplat* __restrict__ packed, int aniso, float cut,
                              uint32_t* ids, float* probe3) {
    const uint64_t b = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= P) return;
    const uint32_t r = list[b];
    if (ids) ids[b] = r;
    if (probe3 && aniso) {  // anisotropic: centre and the Mahalanobis cut
        const PackedSplat ps = packed[r];
        probe3[3 * b] = static_cast<float>(ps.mx);
        probe3[3 * b + 1] = static_cast<float>(ps.my);
        probe3[3 * b + 2] = cut;
    } else if (probe3) {
        const PackedSplat ps = packed[r];
        probe3[3 * b] = ps.pmx;
        probe3[3 * b + 1] = ps.pmy;
        probe3[3 * b + 2] = ps.pcut;
    }
}

// Class-sorts each Gaussian's sparse row (stable insertion sort: a Gaussian
// listing a class twice keeps their order) and pads it to kpad with
// (0xffff, 0.0). Per-class addition order in the compositor is unchanged.
__global__ void k_sort_rows(const uint16_t* __restrict__ idx, const double* __restrict__ prob,
                            uint64_t n, int k, int kpad, uint16_t* out_idx, double* out_prob,
                            uint16_t* out_perm) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint16_t* oi = out_idx + i * kpad;
    double* op = out_prob + i * kpad;
    uint16_t* om = out_perm + i * kpad;
    for (int j = 0; j < k; ++j) {
        const uint16_t c = idx[i * k + j];
        const double pv = prob[i * k + j];
        int q = j;
        while (q > 0 && oi[q - 1] > c) {
            oi[q] = oi[q - 1];
            op[q] = op[q - 1];
            om[q] = om[q - 1];
            --q;
        }
        oi[q] = c;
        op[q] = pv;
        om[q] = static_cast<uint16_t>(j);
    }
    for (int j = k; j < kpad; ++j) {
        oi[j] = 0xffff;
        op[j] = 0.0;
        om[j] = 0;
    }
}

// The same for k <= 32, coalesced: a group of G lanes (G = the power of two >= k) per row,
// lane j holding entry j; its slot is its stable rank (entries of smaller class, or of the
// same class and earlier position), found by broadcasting the row's classes.
__global__ void k_sort_rows_group(const uint16_t* __restrict__ idx, const double* __restrict__ prob,
                                  uint64_t n, int k, int kpad, int G, uint16_t* __restrict__ out_idx,
                                  double* __restrict__ out_prob, uint16_t* __restrict__ out_perm) {
    const uint64_t gt = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t row = gt / static_cast<unsigned>(G);
    const int j = static_cast<int>(gt % static_cast<unsigned>(G));
    const bool live = row < n;
    const bool mine = live && j < k;
    int c = 0x10000;  // above every class id
    double pv = 0.0;
    if (mine) {
        c = idx[row * k + j];
        pv = prob[row * k + j];
    }
    int rank = 0;
    for (int m = 0; m < k; ++m) {
        const int cm = __shfl_sync(0xffffffffu, c, m, G);
        rank += (cm < c || (cm == c && m < j)) ? 1 : 0;
    }
    if (mine) {
        out_idx[row * kpad + rank] = static_cast<uint16_t>(c);
        out_prob[row * kpad + rank] = pv;
        out_perm[row * kpad + rank] = static_cast<uint16_t>(j);
    }
    if (live)
        for (int q = k + j; q < kpad; q += G) {
            out_idx[row * kpad + q] = 0xffff;
            out_prob[row * kpad + q] = 0.0;
            out_perm[row * kpad + q] = 0;
        }
}

inline unsigned blocks_for(uint64_t n, unsigned threads) {
    return static_cast<unsigned>((n + threads - 1) / threads);
}

}  // namespace

// ---------------------------------------------------------------- launchers
void launch_preprocess(const DevMap& m, const PoseParams* d_poses, const CamParams& cam,
                       const OptParams& o, int n_views, uint32_t* keys, uint32_t* vals,
                       size_t stride, uint32_t* vcount, unsigned long long* pcount,
                       unsigned long long* rcount, cudaStream_t s) {
    if (m.n == 0 || n_views == 0) return;
    dim3 grid(blocks_for(m.n, 256), n_views);
    k_preprocess<<<grid, 256, 0, s>>>(m, d_poses, cam, o, keys, vals, stride, vcount, pcount,
                                      rcount);
}

void launch_tiefix(const DevMap& m, const PoseParams* d_pose, const CamParams& cam,
                   const OptParams& o, const uint32_t* key, uint32_t* idx, uint32_t V,
                   cudaStream_t s) {
    if (V < 2) return;
    k_tiefix<<<blocks_for(V, 256), 256, 0, s>>>(m, d_pose, cam, o, key, idx, V);
}

void launch_pack(const DevMap& m, const PoseParams* d_pose, const CamParams& cam,
                 const OptParams& o, const GroupParams& gp, const uint32_t* idx, uint32_t V,
                 PackedSplat* packed, unsigned long long* counts, int4* rects, uint4* bounds,
                 cudaStream_t s) {
    if (V == 0) return;
    k_pack<<<blocks_for(V, 256), 256, 0, s>>>(m, d_pose, cam, o, gp, idx, V, packed, counts, rects,
                                              bounds);
}

void launch_emit_rows(const unsigned long long* offsets, const int4* rects, uint32_t V,
                      unsigned long long R, uint32_t* row_keys, unsigned long long* row_vals,
                      cudaStream_t s) {
    if (V == 0 || R == 0) return;
    const unsigned long long threads = (R + kPerThread - 1) / kPerThread;
    k_emit_rows<<<blocks_for(threads, 256), 256, 0, s>>>(offsets, rects, V, R, row_keys, row_vals);
}

void launch_bin_hist_prefix(const int4* rects, uint32_t V, int tiles_x, int tiles_y, uint32_t cap, int nc,
                            int* diffc, int* sat, int* diff, unsigned long long* rows, cudaStream_t s) {
    if (V == 0) return;
    const int X = tiles_x + 1, Y = tiles_y + 1;  // (diffc and sat zeroed by the caller)
    k_chunk_hist<<<blocks_for(V, 256), 256, 0, s>>>(rects, V, nc, tiles_x, tiles_y, diffc);
    k_chunk_sum<<<blocks_for(static_cast<uint64_t>(X) * Y, 256), 256, 0, s>>>(diffc, nc, X * Y, diff);
    k_prefix2d<<<nc, 1024, 0, s>>>(diffc, X, Y);
    k_chunk_open<<<blocks_for(static_cast<uint64_t>(tiles_x) * tiles_y, 256), 256, 0, s>>>(diffc, nc, tiles_x,
                                                                                           tiles_y, cap, sat);
    k_prefix2d<<<nc, 1024, 0, s>>>(sat, X, Y);
    k_bin_hist_prefix<<<blocks_for(V, 256), 256, 0, s>>>(rects, V, nc, tiles_x, tiles_y, sat, rows);
}

void launch_bin_hist(const int4* rects, uint32_t V, int tiles_x, int* diff,
                     unsigned long long* rows, cudaStream_t s) {
    if (V == 0) return;
    k_bin_hist<<<blocks_for(V, 256), 256, 0, s>>>(rects, V, tiles_x, diff, rows);
}

void launch_bin_scan(int* diff, int tiles_x, int tiles_y, uint2* ranges, cudaStream_t s,
                     const uint8_t* mask, unsigned long long* total, uint32_t cap, uint8_t* trunc) {
    k_bin_scan<<<1, kScanThreads, 0, s>>>(diff, tiles_x, tiles_y, ranges, mask, total, cap, trunc);
}

void launch_redo_items(const uint32_t* incomplete, uint32_t n, uint32_t view, int raster_tiles_x,
                       int per_bin, int tiles_x, uint2* items, uint8_t* mask, cudaStream_t s) {
    if (n == 0) return;
    k_redo_items<<<blocks_for(n, 256), 256, 0, s>>>(incomplete, n, view, raster_tiles_x, per_bin,
                                                    tiles_x, items, mask);
}

void launch_row_scatter(const unsigned long long* row_list, const uint2* row_ranges,
                        const uint2* tile_ranges, int tiles_x, int tiles_y, uint64_t R, uint4* segs,
                        uint32_t* nseg, uint32_t* cnt, uint32_t* list, cudaStream_t s,
                        const uint8_t* mask, bool part, bool cols) {
    if (R == 0) return;
    const uint64_t gmax = R / kSeg + static_cast<uint64_t>(tiles_y) + 1;
    k_row_segs<<<1, 1024, 0, s>>>(row_ranges, tiles_y, segs, nseg);
    const int blocks = (tiles_x + 31) / 32;  // 32-column blocks, one warp each
    const int warps = std::min(8, blocks);
    const dim3 grid(static_cast<unsigned>(gmax), static_cast<unsigned>((blocks + warps - 1) / warps));
    k_seg_count<<<static_cast<unsigned>(gmax), 256, sizeof(int) * (tiles_x + 1), s>>>(
        row_list, segs, nseg, tiles_x, cnt);
    k_seg_scan<<<dim3(static_cast<unsigned>(tiles_y), static_cast<unsigned>((tiles_x + 31) / 32)), 256, 0, s>>>(
        segs, nseg, part ? nullptr : tile_ranges, tiles_x, tiles_y, cnt);
    if (part)  // (the block walk: faster than k_seg_pass_cols on the short prefixes)
        k_seg_pass<true><<<grid, 32 * warps, 0, s>>>(row_list, segs, nseg, tiles_x, cnt, list, mask, tile_ranges);
    else if (cols)
        k_seg_pass_cols<false><<<static_cast<unsigned>(gmax), 256, 0, s>>>(row_list, segs, nseg, tiles_x, cnt,
                                                                           list, nullptr, nullptr);
    else
        k_seg_pass<false><<<grid, 32 * warps, 0, s>>>(row_list, segs, nseg, tiles_x, cnt, list, nullptr, nullptr);
}

// k_seg_pass alone over the segments of a previous launch_row_scatter (the redo pass of
// depth-prefix binning: the same row list and per-segment positions, other ranges / mask)
void launch_seg_pass(const unsigned long long* row_list, const uint2* tile_ranges, int tiles_x,
                     uint64_t G, const uint4* segs, const uint32_t* nseg, const uint32_t* cnt,
                     uint32_t* list, const uint8_t* mask, cudaStream_t s, bool cols) {
    if (G == 0) return;
    if (cols) {
        k_seg_pass_cols<true><<<static_cast<unsigned>(G), 256, 0, s>>>(row_list, segs, nseg, tiles_x, cnt, list,
                                                                       mask, tile_ranges);
        return;
    }
    const int blocks = (tiles_x + 31) / 32;
    const int warps = std::min(8, blocks);
    const dim3 grid(static_cast<unsigned>(G), static_cast<unsigned>((blocks + warps - 1) / warps));
    k_seg_pass<true><<<grid, 32 * warps, 0, s>>>(row_list, segs, nseg, tiles_x, cnt, list, mask, tile_ranges);
}

uint64_t row_scatter_segments(uint64_t R, int tiles_y) {
    return R / kSeg + static_cast<uint64_t>(tiles_y) + 1;
}

void launch_ranges(const uint32_t* sorted_tiles, uint64_t P, uint2* ranges, cudaStream_t s) {
    if (P == 0) return;
    k_ranges<<<blocks_for(P, 256), 256, 0, s>>>(sorted_tiles, P, ranges);
}

void launch_reduce_scores(const ViewDesc* views, int n_views, int tiles, double* out_missing,
                          double* out_entropy, double* out_fisher, cudaStream_t s) {
    if (n_views == 0) return;
    k_reduce_scores<<<n_views, 256, 0, s>>>(views, tiles, out_missing, out_entropy, out_fisher);
}

void launch_debug_projections(const DevMap& m, const PoseParams* d_pose, const CamParams& cam,
                              const OptParams& o, const uint32_t* idx, uint32_t V,
                              double* out6, cudaStream_t s) {
    if (V == 0) return;
    k_debug_projections<<<blocks_for(V, 256), 256, 0, s>>>(m, d_pose, cam, o, idx, V, out6);
}

void launch_sort_rows(const uint16_t* idx, const double* prob, uint64_t n, int k, int kpad,
                      uint16_t* out_idx, double* out_prob, uint16_t* out_perm, cudaStream_t s) {
    if (n == 0) return;
    if (k <= 32) {
        int G = 1;
        while (G < k) G <<= 1;
        k_sort_rows_group<<<blocks_for(n * G, 256), 256, 0, s>>>(idx, prob, n, k, kpad, G, out_idx,
                                                                 out_prob, out_perm);
        return;
    }
    k_sort_rows<<<blocks_for(n, 256), 256, 0, s>>>(idx, prob, n, k, kpad, out_idx, out_prob,
                                                   out_perm);
}

// DevMap::sem_rec from the class-sorted rows: one thread per (Gaussian, slot), coalesced
__global__ void k_sem_records(const uint16_t* __restrict__ idx, const double* __restrict__ prob,
                              uint64_t slots, uint4* __restrict__ out) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= slots) return;
    const double pv = prob[i];
    out[i] = make_uint4(static_cast<unsigned>(__double2loint(pv)), static_cast<unsigned>(__double2hiint(pv)),
                        idx[i], 0u);
}

void launch_sem_records(const DevMap& m, uint4* out, cudaStream_t s) {
    const uint64_t slots = m.n * static_cast<uint64_t>(m.kpad);
    if (slots == 0) return;
    k_sem_records<<<blocks_for(slots, 256), 256, 0, s>>>(m.sem_idx, m.sem_prob, slots, out);
}

void launch_group_bounds(const DevMap& m, const GroupParams& gp, uint4* out, cudaStream_t s) {
    if (m.n == 0) return;
    k_group_bounds<<<blocks_for(m.n, 256), 256, 0, s>>>(m, gp, out);
}

void launch_bins_to_ids(const uint32_t* list, uint64_t P, const PackedSplat* packed, int aniso,
                        double cut_sq, uint32_t* ids, float* probe3, cudaStream_t s) {
    if (P == 0) return;
    k_bins_to_ids<<<blocks_for(P, 256), 256, 0, s>>>(list, P, packed, aniso,
                                                     static_cast<float>(cut_sq), ids, probe3);
}

}  // namespace sgm
