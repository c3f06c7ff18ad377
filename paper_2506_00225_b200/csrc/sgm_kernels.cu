// B200 (sm_100a) kernels of the candidate-view render + scoring path.
//
// Compiled with --fmad=false: every fp64/fp32 expression below is evaluated
// with one rounding per operation, in the reference's C++ evaluation order, so
// projections and tile rectangles are bit-identical to the reference build
// (which has no FMA: proj/CMakeLists.txt:3,8-10, default -march=x86-64).
//
//   K1 k_preprocess      project_splats transform/cull + tile count   splat_render.cpp:15-39, 205-209
//   K2 (CUB radix sort on fp64 z) + k_tiefix (z, mx, my, alpha) order  splat_render.cpp:40-45
//   K3 k_pack / k_emit / (CUB stable tile sort) / k_ranges             splat_render.cpp:189-213
//   K4/K5 k_raster<render|score>   tile compositor + clipped entropy    splat_render.cpp:254-324, 360-369
//   k_reduce_scores     deterministic per-view n_missing / entropy_sum   explorer.cpp:195-203
#include <cfloat>
#include <climits>
#include <cstdio>

#include "sgm_internal.h"

namespace sgm {

namespace {

constexpr int kBatch = 32;  // Gaussians staged in shared memory per raster step

// static_cast<int>(double) as the reference binary executes it (x86-64
// cvttsd2si): out-of-range and NaN give INT_MIN. CUDA's cvt saturates instead.
__device__ __forceinline__ int to_int_x86(double v) {
    return (v > -2147483649.0 && v < 2147483648.0) ? static_cast<int>(v) : INT_MIN;
}

// project_splats for one Gaussian (splat_render.cpp:24-37). Returns visibility.
__device__ __forceinline__ bool project(const DevMap& m, uint64_t i, const PoseParams& P,
                                        const CamParams& cam, const OptParams& o, double& mx,
                                        double& my, double& rad_px, double& z) {
    const double d0 = m.cx[i] - P.t[0];
    const double d1 = m.cy[i] - P.t[1];
    const double d2 = m.cz[i] - P.t[2];
    // Eigen lazy coefficient product: row = x0 + (x1 + x2)  (:25)
    const double pcz = P.Rcw[6] * d0 + (P.Rcw[7] * d1 + P.Rcw[8] * d2);
    if (pcz <= o.z_near) return false;  // :26
    const double pcx = P.Rcw[0] * d0 + (P.Rcw[1] * d1 + P.Rcw[2] * d2);
    const double pcy = P.Rcw[3] * d0 + (P.Rcw[4] * d1 + P.Rcw[5] * d2);
    z = pcz;
    mx = cam.fx * pcx / pcz + cam.cx;       // :29
    my = cam.fy * pcy / pcz + cam.cy;       // :30
    rad_px = m.rad[i] * cam.fy / pcz;       // :31 (exp done on host)
    const double reach = o.trunc * rad_px;  // :34
    if (mx + reach < 0 || mx - reach > cam.W || my + reach < 0 || my - reach > cam.H)
        return false;  // :35-37
    return true;
}

struct Rect {
    int tx0, tx1, ty0, ty1;
};

__device__ __forceinline__ Rect tile_rect(double mx, double my, double rad_px,
                                          const OptParams& o) {
    const double reach = o.trunc * rad_px;  // :205
    Rect r;
    r.tx0 = max(0, to_int_x86((mx - reach) / o.ts));               // :206
    r.tx1 = min(o.tiles_x - 1, to_int_x86((mx + reach) / o.ts));   // :207
    r.ty0 = max(0, to_int_x86((my - reach) / o.ts));               // :208
    r.ty1 = min(o.tiles_y - 1, to_int_x86((my + reach) / o.ts));   // :209
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
__global__ void __launch_bounds__(256) k_preprocess(DevMap m, const PoseParams* __restrict__ poses,
                                                    CamParams cam, OptParams o, double* keys,
                                                    uint32_t* vals, size_t stride,
                                                    uint32_t* vcount,
                                                    unsigned long long* pcount) {
    const int v = blockIdx.y;
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const PoseParams& P = poses[v];
    double mx = 0, my = 0, rad = 0, z = 0;
    const bool vis = i < m.n && project(m, i, P, cam, o, mx, my, rad, z);
    unsigned long long cnt = vis ? rect_count(tile_rect(mx, my, rad, o)) : 0ull;

    const unsigned mask = __ballot_sync(0xffffffffu, vis);
    const int lane = threadIdx.x & 31;
    uint32_t base = 0;
    if (mask) {
        const int leader = __ffs(mask) - 1;
        if (lane == leader) base = atomicAdd(&vcount[v], static_cast<uint32_t>(__popc(mask)));
        base = __shfl_sync(0xffffffffu, base, leader);
    }
    if (vis) {
        const uint32_t pos = base + __popc(mask & ((1u << lane) - 1u));
        keys[v * stride + pos] = z;
        vals[v * stride + pos] = static_cast<uint32_t>(i);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, off);
    if (lane == 0 && cnt) atomicAdd(&pcount[v], cnt);
}

// ---------------------------------------------------------------- K2 tie fix-up
// After the radix sort on z, runs of equal z are re-ordered by (mx, my, alpha)
// and finally map index (splat_render.cpp:40-45; index breaks exact 4-key ties,
// which std::sort leaves unspecified).
__device__ __forceinline__ bool proj_less(double amx, double amy, double aal, uint32_t ai,
                                          double bmx, double bmy, double bal, uint32_t bi) {
    if (amx != bmx) return amx < bmx;
    if (amy != bmy) return amy < bmy;
    if (aal != bal) return aal < bal;
    return ai < bi;
}

__global__ void k_tiefix(DevMap m, const PoseParams* __restrict__ pose, CamParams cam, OptParams o,
                         const double* __restrict__ z, uint32_t* idx, uint32_t V) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r + 1 >= V) return;
    if (!(z[r] == z[r + 1])) return;
    if (r > 0 && z[r - 1] == z[r]) return;  // not the head of the run
    uint32_t e = r + 1;
    while (e < V && z[e] == z[r]) ++e;
    // insertion sort idx[r, e) (runs are a handful of entries)
    for (uint32_t a = r + 1; a < e; ++a) {
        const uint32_t ia = idx[a];
        double amx, amy, arad, az;
        project(m, ia, *pose, cam, o, amx, amy, arad, az);
        const double aal = m.alpha[ia];
        uint32_t b = a;
        while (b > r) {
            const uint32_t ib = idx[b - 1];
            double bmx, bmy, brad, bz;
            project(m, ib, *pose, cam, o, bmx, bmy, brad, bz);
            if (!proj_less(amx, amy, aal, ia, bmx, bmy, m.alpha[ib], ib)) break;
            idx[b] = ib;
            --b;
        }
        idx[b] = ia;
    }
}

// ---------------------------------------------------------------- K3
// PackedSplat + Probe per depth rank (splat_render.cpp:191-204) and tile counts.
__global__ void k_pack(DevMap m, const PoseParams* __restrict__ pose, CamParams cam, OptParams o,
                       const uint32_t* __restrict__ idx, uint32_t V, PackedSplat* packed,
                       unsigned long long* counts) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= V) return;
    const uint32_t i = idx[r];
    double mx, my, rad, z;
    project(m, i, *pose, cam, o, mx, my, rad, z);
    PackedSplat ps;
    ps.mx = mx;
    ps.my = my;
    ps.inv_two_r2 = 1.0 / (2.0 * rad * rad);  // :194
    ps.cutoff_d2 = o.cut_sq * rad * rad;      // :195
    ps.alpha = m.alpha[i];
    ps.z = z;
    ps.pmx = static_cast<float>(mx);  // :201
    ps.pmy = static_cast<float>(my);  // :202
    ps.pcut = static_cast<float>(ps.cutoff_d2 * (1.0 + 1e-5)) + 1e-6f;  // :203
    ps.map_index = i;
    packed[r] = ps;
    counts[r] = rect_count(tile_rect(mx, my, rad, o));
}

// Emits (bin, rank) pairs in rank order at the scanned offsets; a stable sort on
// the bin key then yields every bin in depth order (:210-212). rad_px is not kept
// in PackedSplat (64 B); the rectangle is re-derived by re-projecting, which is
// bit-identical to the count pass.
__global__ void k_emit2(DevMap m, const PoseParams* __restrict__ pose, CamParams cam, OptParams o,
                        const PackedSplat* __restrict__ packed,
                        const unsigned long long* __restrict__ offsets, uint32_t V,
                        uint32_t* tile_keys, uint32_t* tile_vals) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= V) return;
    unsigned long long at = offsets[r];
    if (at == offsets[r + 1]) return;
    double mx, my, rad, z;
    project(m, packed[r].map_index, *pose, cam, o, mx, my, rad, z);
    const Rect rc = tile_rect(mx, my, rad, o);
    for (int ty = rc.ty0; ty <= rc.ty1; ++ty)
        for (int tx = rc.tx0; tx <= rc.tx1; ++tx) {
            tile_keys[at] = static_cast<uint32_t>(ty * o.tiles_x + tx);
            tile_vals[at] = r;
            ++at;
        }
}

__global__ void k_ranges(const uint32_t* __restrict__ keys, uint64_t P, uint2* ranges) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= P) return;
    const uint32_t t = keys[i];
    if (i == 0 || keys[i - 1] != t) ranges[t].x = static_cast<uint32_t>(i);
    if (i + 1 == P || keys[i + 1] != t) ranges[t].y = static_cast<uint32_t>(i + 1);
}

__device__ __forceinline__ double clamp_prob(double v) {
    // std::clamp(v, 0.001, 1.0) (splat_render.cpp:362)
    return v < 0.001 ? 0.001 : (1.0 < v ? 1.0 : v);
}

// ---------------------------------------------------------------- K4 / K5
// One CTA = one 8x8 pixel block of one view; one thread = one pixel. The
// per-pixel semantic accumulator lives in shared memory as [channel][pixel]
// (pitch 64, or 65 when the epilogue transposes it to the reference's
// channel-fastest layout), so the warp-uniform Gaussian's k scatters hit 32
// consecutive doubles: conflict-free.
template <bool kRender, bool kDup>
__global__ void __launch_bounds__(kTilePx) k_raster(RasterParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int C = p.map.C;
    const int k = p.map.k;
    constexpr int pitch = kRender ? kTilePx + 1 : kTilePx;
    double* acc = reinterpret_cast<double*>(smem);
    double* s_mx = acc + C * pitch;
    double* s_my = s_mx + kBatch;
    double* s_inv = s_my + kBatch;
    double* s_cut = s_inv + kBatch;
    double* s_alpha = s_cut + kBatch;
    double* s_z = s_alpha + kBatch;
    double* s_prob = s_z + kBatch;                 // kBatch * k
    double* s_col = s_prob + kBatch * k;           // kBatch * 4 (render)
    float* s_pmx = reinterpret_cast<float*>(s_col + (kRender ? kBatch * 4 : 0));
    float* s_pmy = s_pmx + kBatch;
    float* s_pcut = s_pmy + kBatch;
    uint32_t* s_map = reinterpret_cast<uint32_t*>(s_pcut + kBatch);
    uint16_t* s_idx = reinterpret_cast<uint16_t*>(s_map + kBatch);  // kBatch * k
    __shared__ double red_d[kTilePx];
    __shared__ unsigned long long red_u[kTilePx];

    const ViewDesc vd = p.views[blockIdx.y];
    const int tile = blockIdx.x;
    const int bx = tile % p.raster_tiles_x, by = tile / p.raster_tiles_x;
    const int t = threadIdx.x;
    const int x = bx * kTile + (t & (kTile - 1));
    const int y = by * kTile + (t / kTile);
    const bool inside = x < p.cam.W && y < p.cam.H;
    const int bin = ((by * kTile) / p.opt.ts) * p.opt.tiles_x + (bx * kTile) / p.opt.ts;
    const uint2 rg = vd.ranges[bin];

    for (int c = 0; c < C; ++c) acc[c * pitch + t] = 0.0;

    const double px = x + 0.5, py = y + 0.5;  // :261, :263
    const float pxf = static_cast<float>(px), pyf = static_cast<float>(py);  // :274
    double T = 1.0;
    double ac0 = 0.0, ac1 = 0.0, ac2 = 0.0, adep = 0.0;
    bool done = !inside;
    unsigned long long contrib = 0;

    for (uint32_t base = rg.x; base < rg.y; base += kBatch) {
        const int n = min(static_cast<uint32_t>(kBatch), rg.y - base);
        __syncthreads();  // previous batch fully consumed
        if (t < n) {
            const uint32_t r = vd.list[base + t];
            const PackedSplat ps = vd.packed[r];
            s_mx[t] = ps.mx;
            s_my[t] = ps.my;
            s_inv[t] = ps.inv_two_r2;
            s_cut[t] = ps.cutoff_d2;
            s_alpha[t] = ps.alpha;
            s_z[t] = ps.z;
            s_pmx[t] = ps.pmx;
            s_pmy[t] = ps.pmy;
            s_pcut[t] = ps.pcut;
            s_map[t] = ps.map_index;
            if (kRender) {
                const double4 cc = reinterpret_cast<const double4*>(p.map.color4)[ps.map_index];
                s_col[4 * t] = cc.x;
                s_col[4 * t + 1] = cc.y;
                s_col[4 * t + 2] = cc.z;
            }
        }
        __syncthreads();
        for (int l = t; l < n * k; l += kTilePx) {
            const int e = l / k;
            const int j = l - e * k;
            const size_t src = static_cast<size_t>(s_map[e]) * k + j;
            s_idx[l] = p.map.sem_idx[src];
            s_prob[l] = p.map.sem_prob[src];
        }
        __syncthreads();
        if (!done) {
            for (int e = 0; e < n; ++e) {
                const float fdx = pxf - s_pmx[e];
                const float fdy = pyf - s_pmy[e];
                if (fdx * fdx + fdy * fdy > s_pcut[e]) continue;  // :276-278
                const double dx = px - s_mx[e];
                const double dy = py - s_my[e];
                const double d2 = dx * dx + dy * dy;
                if (d2 > s_cut[e]) continue;  // :283
                double f = s_alpha[e] * exp(-d2 * s_inv[e]);  // :284
                if (f > kMaxFootprint) f = kMaxFootprint;     // :285
                const double w = f * T;
                if (kRender) {
                    ac0 += s_col[4 * e] * w;  // :289-291 (colour pre-clamped)
                    ac1 += s_col[4 * e + 1] * w;
                    ac2 += s_col[4 * e + 2] * w;
                    adep += s_z[e] * w;  // :293
                }
                if (!kRender || (p.channels & 4u)) {
                    const uint16_t* ei = s_idx + e * k;
                    const double* ep = s_prob + e * k;
                    if (kDup) {
                        for (int j = 0; j < k; ++j) {  // sequential: repeated classes
                            double* a = &acc[ei[j] * pitch + t];
                            *a = *a + ep[j] * w;  // :307
                        }
                    } else {
                        int j = 0;
                        for (; j + 8 <= k; j += 8) {
                            int ad[8];
                            double pv[8], av[8];
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                ad[q] = ei[j + q] * pitch + t;
                                pv[q] = ep[j + q];
                            }
#pragma unroll
                            for (int q = 0; q < 8; ++q) av[q] = acc[ad[q]];
#pragma unroll
                            for (int q = 0; q < 8; ++q) acc[ad[q]] = av[q] + pv[q] * w;
                        }
                        for (; j < k; ++j) {
                            double* a = &acc[ei[j] * pitch + t];
                            *a = *a + ep[j] * w;
                        }
                    }
                }
                ++contrib;
                T = T * (1.0 - f);                                  // :311
                if (p.opt.early_exit && T < p.opt.eps) {           // :312
                    done = true;
                    break;
                }
            }
        }
        if (__syncthreads_and(done)) break;
    }

    if (kRender) {
        if (inside) {
            const size_t pix = static_cast<size_t>(y) * p.cam.W + x;
            if (vd.sil) vd.sil[pix] = 1.0 - T;  // :314
            if (vd.color) {
                vd.color[pix * 3] = ac0;
                vd.color[pix * 3 + 1] = ac1;
                vd.color[pix * 3 + 2] = ac2;
            }
            if (vd.depth) vd.depth[pix] = adep;
        }
        if (vd.sem) {
            __syncthreads();
            for (int l = t; l < kTilePx * C; l += kTilePx) {
                const int q = l / C;
                const int c = l - q * C;
                const int qx = bx * kTile + (q & (kTile - 1));
                const int qy = by * kTile + q / kTile;
                if (qx < p.cam.W && qy < p.cam.H)
                    vd.sem[(static_cast<size_t>(qy) * p.cam.W + qx) * C + c] = acc[c * pitch + q];
            }
        }
    } else {
        // clipped_entropy of this pixel (:360-369), reference summation order.
        double h = 0.0;
        unsigned long long miss = 0;
        if (inside) {
            double total = 0.0;
            for (int c = 0; c < C; ++c) total += clamp_prob(acc[c * pitch + t]);
            for (int c = 0; c < C; ++c) {
                const double q = clamp_prob(acc[c * pitch + t]) / total;
                h -= q * log(q);
            }
            miss = (1.0 - T == 0.0) ? 1ull : 0ull;  // explorer.cpp:198
        }
        red_d[t] = h;
        red_u[t] = miss;
        __syncthreads();
        for (int s = kTilePx / 2; s > 0; s >>= 1) {  // fixed tree: deterministic
            if (t < s) {
                red_d[t] += red_d[t + s];
                red_u[t] += red_u[t + s];
            }
            __syncthreads();
        }
        if (t == 0) {
            vd.ent_partial[tile] = red_d[0];
            vd.miss_partial[tile] = static_cast<uint32_t>(red_u[0]);
        }
    }
    // K (contributors) for the measurement counters
    red_u[t] = contrib;
    __syncthreads();
    for (int s = kTilePx / 2; s > 0; s >>= 1) {
        if (t < s) red_u[t] += red_u[t + s];
        __syncthreads();
    }
    if (t == 0 && vd.contributors && red_u[0]) atomicAdd(vd.contributors, red_u[0]);
}

// Per view: n_missing and entropy_sum from the per-tile partials, summed in a
// fixed order that depends only on the tile count (sharding-invariant).
__global__ void __launch_bounds__(256) k_reduce_scores(const ViewDesc* __restrict__ views, int tiles,
                                                       double* out_missing, double* out_entropy) {
    __shared__ double sd[256];
    __shared__ unsigned long long su[256];
    const ViewDesc vd = views[blockIdx.x];
    const int t = threadIdx.x;
    const int per = (tiles + 255) / 256;
    double h = 0.0;
    unsigned long long m = 0;
    for (int i = t * per; i < min(tiles, (t + 1) * per); ++i) {
        h += vd.ent_partial[i];
        m += vd.miss_partial[i];
    }
    sd[t] = h;
    su[t] = m;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (t < s) {
            sd[t] += sd[t + s];
            su[t] += su[t + s];
        }
        __syncthreads();
    }
    if (t == 0) {
        out_missing[blockIdx.x] = static_cast<double>(su[0]);
        out_entropy[blockIdx.x] = sd[0];
    }
}

__global__ void k_debug_projections(DevMap m, const PoseParams* __restrict__ pose, CamParams cam,
                                    OptParams o, const uint32_t* __restrict__ idx, uint32_t V,
                                    double* out6) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= V) return;
    const uint32_t i = idx[r];
    double mx, my, rad, z;
    project(m, i, *pose, cam, o, mx, my, rad, z);
    out6[6 * r] = mx;
    out6[6 * r + 1] = my;
    out6[6 * r + 2] = rad;
    out6[6 * r + 3] = z;
    out6[6 * r + 4] = m.alpha[i];
    out6[6 * r + 5] = static_cast<double>(i);
}

__global__ void k_bins_to_ids(const uint32_t* __restrict__ list, uint64_t P,
                              const PackedSplat* __restrict__ packed, uint32_t* ids,
                              float* probe3) {
    const uint64_t b = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= P) return;
    const uint32_t r = list[b];
    if (ids) ids[b] = r;
    if (probe3) {
        const PackedSplat ps = packed[r];
        probe3[3 * b] = ps.pmx;
        probe3[3 * b + 1] = ps.pmy;
        probe3[3 * b + 2] = ps.pcut;
    }
}

inline unsigned blocks_for(uint64_t n, unsigned threads) {
    return static_cast<unsigned>((n + threads - 1) / threads);
}

}  // namespace

// ---------------------------------------------------------------- launchers
void launch_preprocess(const DevMap& m, const PoseParams* d_poses, const CamParams& cam,
                       const OptParams& o, int n_views, double* keys, uint32_t* vals,
                       size_t stride, uint32_t* vcount, unsigned long long* pcount,
                       cudaStream_t s) {
    if (m.n == 0 || n_views == 0) return;
    dim3 grid(blocks_for(m.n, 256), n_views);
    k_preprocess<<<grid, 256, 0, s>>>(m, d_poses, cam, o, keys, vals, stride, vcount, pcount);
}

void launch_tiefix(const DevMap& m, const PoseParams* d_pose, const CamParams& cam,
                   const OptParams& o, const double* z, uint32_t* idx, uint32_t V,
                   cudaStream_t s) {
    if (V < 2) return;
    k_tiefix<<<blocks_for(V, 256), 256, 0, s>>>(m, d_pose, cam, o, z, idx, V);
}

void launch_pack(const DevMap& m, const PoseParams* d_pose, const CamParams& cam,
                 const OptParams& o, const uint32_t* idx, uint32_t V, PackedSplat* packed,
                 unsigned long long* counts, cudaStream_t s) {
    if (V == 0) return;
    k_pack<<<blocks_for(V, 256), 256, 0, s>>>(m, d_pose, cam, o, idx, V, packed, counts);
}

void launch_emit_pairs(const DevMap& m, const PoseParams* d_pose, const CamParams& cam,
                       const OptParams& o, const PackedSplat* packed,
                       const unsigned long long* offsets, uint32_t V, uint32_t* tile_keys,
                       uint32_t* tile_vals, cudaStream_t s) {
    if (V == 0) return;
    k_emit2<<<blocks_for(V, 128), 128, 0, s>>>(m, d_pose, cam, o, packed, offsets, V, tile_keys,
                                               tile_vals);
}

void launch_ranges(const uint32_t* sorted_tiles, uint64_t P, uint2* ranges, cudaStream_t s) {
    if (P == 0) return;
    k_ranges<<<blocks_for(P, 256), 256, 0, s>>>(sorted_tiles, P, ranges);
}

size_t raster_smem_bytes(int C, int k, bool render) {
    const int pitch = render ? kTilePx + 1 : kTilePx;
    size_t b = static_cast<size_t>(C) * pitch * sizeof(double);
    b += static_cast<size_t>(kBatch) * 6 * sizeof(double);
    b += static_cast<size_t>(kBatch) * k * sizeof(double);
    if (render) b += static_cast<size_t>(kBatch) * 4 * sizeof(double);
    b += static_cast<size_t>(kBatch) * 3 * sizeof(float);
    b += static_cast<size_t>(kBatch) * sizeof(uint32_t);
    b += static_cast<size_t>(kBatch) * k * sizeof(uint16_t);
    return (b + 15) & ~static_cast<size_t>(15);
}

int raster_batch_entries() { return kBatch; }

template <bool kRender, bool kDup>
static void launch_raster_t(const RasterParams& p, int n_views, cudaStream_t s) {
    const size_t smem = raster_smem_bytes(p.map.C, p.map.k, kRender);
    static size_t configured = 0;
    if (smem > configured) {
        cudaFuncSetAttribute(k_raster<kRender, kDup>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        configured = smem;
    }
    dim3 grid(p.tiles_per_view, n_views);
    k_raster<kRender, kDup><<<grid, kTilePx, smem, s>>>(p);
}

void launch_raster_score(const RasterParams& p, int n_views, cudaStream_t s) {
    if (p.map.dup_idx)
        launch_raster_t<false, true>(p, n_views, s);
    else
        launch_raster_t<false, false>(p, n_views, s);
}

void launch_raster_render(const RasterParams& p, int n_views, cudaStream_t s) {
    if (p.map.dup_idx)
        launch_raster_t<true, true>(p, n_views, s);
    else
        launch_raster_t<true, false>(p, n_views, s);
}

void launch_reduce_scores(const ViewDesc* views, int n_views, int tiles, double* out_missing,
                          double* out_entropy, cudaStream_t s) {
    if (n_views == 0) return;
    k_reduce_scores<<<n_views, 256, 0, s>>>(views, tiles, out_missing, out_entropy);
}

void launch_debug_projections(const DevMap& m, const PoseParams* d_pose, const CamParams& cam,
                              const OptParams& o, const uint32_t* idx, uint32_t V,
                              double* out6, cudaStream_t s) {
    if (V == 0) return;
    k_debug_projections<<<blocks_for(V, 256), 256, 0, s>>>(m, d_pose, cam, o, idx, V, out6);
}

void launch_bins_to_ids(const uint32_t* list, uint64_t P, const PackedSplat* packed,
                        uint32_t* ids, float* probe3, cudaStream_t s) {
    if (P == 0) return;
    k_bins_to_ids<<<blocks_for(P, 256), 256, 0, s>>>(list, P, packed, ids, probe3);
}

}  // namespace sgm
