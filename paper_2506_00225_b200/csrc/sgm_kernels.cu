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
//   K3 k_pack / k_emit_lb (load-balanced over pairs) / CUB stable tile sort / k_ranges
//                                                                       splat_render.cpp:189-213
//   K4/K5 raster: see sgm_raster.cu
//   k_reduce_scores     deterministic per-view n_missing / entropy_sum   explorer.cpp:195-203
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
                                                    unsigned long long* pcount) {
    const int v = blockIdx.y;
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const PoseParams& P = poses[v];
    Proj q;
    const bool vis = i < m.n && project(m, i, P, cam, o, q);
    unsigned long long cnt = vis ? rect_count(tile_rect(q, o)) : 0ull;

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
        keys[v * stride + pos] = sortable(static_cast<float>(q.z));  // monotone in z
        vals[v * stride + pos] = static_cast<uint32_t>(i);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, off);
    if (lane == 0 && cnt) atomicAdd(&pcount[v], cnt);
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
        ps.inv_two_r2 = 1.0 / (2.0 * rad * rad);  // :194
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
    if (bounds) {
        // raster channel groups of the class-sorted row: b[g] = #entries with class <
        // (g + 1) * Cg for g = 0..6, b[7] = k (u16 each)
        const uint16_t* row = m.sem_idx + static_cast<size_t>(i) * m.kpad;
        uint32_t b[8];
        int j = 0;
        for (int g = 0; g < 7; ++g) {
            const int lim = (g + 1) * gp.Cg;
            while (j < m.k && row[j] < lim) ++j;
            b[g] = static_cast<uint32_t>(j);
        }
        b[7] = static_cast<uint32_t>(m.k);
        bounds[r] = make_uint4(b[0] | (b[1] << 16), b[2] | (b[3] << 16), b[4] | (b[5] << 16),
                               b[6] | (b[7] << 16));
    }
}

// Emits (bin, rank) pairs in rank order at the scanned offsets; a stable sort on
// the bin key then yields every bin in depth order (:210-212). rad_px is not kept
// in PackedSplat (64 B); the rectangle is re-derived by re-projecting, which is
// bit-identical to the count pass.
// Load-balanced: each thread emits kPerThread consecutive pairs. The first
// pair's rank comes from a binary search over the scanned counts; then the
// thread walks forward (pairs of one rank are contiguous).
constexpr int kPerThread = 8;
__global__ void k_emit_lb(const unsigned long long* __restrict__ offsets, const int4* __restrict__ rects,
                          uint32_t V, unsigned long long P, int tiles_x, uint32_t* tile_keys,
                          uint32_t* tile_vals) {
    const unsigned long long i0 =
        (static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x) * kPerThread;
    if (i0 >= P) return;
    // largest r with offsets[r] <= i0
    uint32_t lo = 0, hi = V;  // offsets[V] == P > i0
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) / 2;
        if (offsets[mid] <= i0) lo = mid; else hi = mid;
    }
    uint32_t r = lo;
    unsigned long long beg = offsets[r], end = offsets[r + 1];
    int4 rc = rects[r];
    const unsigned long long i1 = min(P, i0 + kPerThread);
    for (unsigned long long i = i0; i < i1; ++i) {
        while (i >= end) {
            ++r;
            beg = end;
            end = offsets[r + 1];
            rc = rects[r];
        }
        const uint32_t j = static_cast<uint32_t>(i - beg);
        const uint32_t dy = j / static_cast<uint32_t>(rc.z);
        const uint32_t dx = j - dy * static_cast<uint32_t>(rc.z);
        tile_keys[i] = static_cast<uint32_t>((rc.y + static_cast<int>(dy)) * tiles_x + rc.x + static_cast<int>(dx));
        tile_vals[i] = r;
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

inline unsigned blocks_for(uint64_t n, unsigned threads) {
    return static_cast<unsigned>((n + threads - 1) / threads);
}

}  // namespace

// ---------------------------------------------------------------- launchers
void launch_preprocess(const DevMap& m, const PoseParams* d_poses, const CamParams& cam,
                       const OptParams& o, int n_views, uint32_t* keys, uint32_t* vals,
                       size_t stride, uint32_t* vcount, unsigned long long* pcount,
                       cudaStream_t s) {
    if (m.n == 0 || n_views == 0) return;
    dim3 grid(blocks_for(m.n, 256), n_views);
    k_preprocess<<<grid, 256, 0, s>>>(m, d_poses, cam, o, keys, vals, stride, vcount, pcount);
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

void launch_emit_pairs(const unsigned long long* offsets, const int4* rects, uint32_t V,
                       unsigned long long P, const OptParams& o, uint32_t* tile_keys,
                       uint32_t* tile_vals, cudaStream_t s) {
    if (V == 0 || P == 0) return;
    const unsigned long long threads = (P + kPerThread - 1) / kPerThread;
    k_emit_lb<<<blocks_for(threads, 256), 256, 0, s>>>(offsets, rects, V, P, o.tiles_x, tile_keys,
                                                       tile_vals);
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
    k_sort_rows<<<blocks_for(n, 256), 256, 0, s>>>(idx, prob, n, k, kpad, out_idx, out_prob,
                                                   out_perm);
}

void launch_bins_to_ids(const uint32_t* list, uint64_t P, const PackedSplat* packed, int aniso,
                        double cut_sq, uint32_t* ids, float* probe3, cudaStream_t s) {
    if (P == 0) return;
    k_bins_to_ids<<<blocks_for(P, 256), 256, 0, s>>>(list, P, packed, aniso,
                                                     static_cast<float>(cut_sq), ids, probe3);
}

}  // namespace sgm
