// the mapping caller of render -- mapping_loss / semantic_loss and the analytic
// backward pass of proj/src/losses.cpp:40-362 on sm_100a.
//
// Pipeline for one posed frame (sgm_backward, sgm_capi.cu):
//   1. the raster kernel renders colour, depth, silhouette and semantics into device planes
//      and counts each pixel's contributors (covered <=> non-empty list, :188);
//   2. k_loss_pixels: per pixel the loss masks (S > 0.99, depth > 0, raw entropy < ln k,
//      covered), the loss terms of mapping_loss (:40-59) and semantic_loss (:139-160), and
//      fixed-order per-block partial sums (deterministic reports);
//   3. k_backward (one 256-thread CTA per 8x8 block): dL/dC per pixel (:226-236), dq of the
//      semantic pixel loss (:69-133) in shared memory, then one pass over the block's depth-
//      ordered list: phase A footprints (clamp recorded), phase B the transmittance chain with
//      dL/df_j = sum_c dL/dC_c (v_c T_j - S_c/(1-f_j)) + dL/dD (z T_j - S_d/(1-f_j)), the suffix
//      S = R - P_j from the inclusive prefix (no reverse sweep, :272-308), phase C per
//      (Gaussian, pixel) the projection-space terms (:297-304), colour (:291-294) and sparse
//      semantic terms (:262-269), reduced over the block and accumulated with fp64 RED;
//   4. k_chain: projection -> world per depth rank (:312-335); k_kl_clip (:337-347);
//      k_finite: the non-finite check (:349-360).
#include "sgm_device.cuh"
#include "sgm_internal.h"

namespace sgm {

namespace {

constexpr int kBThreads = 256;
constexpr int kBNB = 16;
constexpr double kSilhouetteMask = 0.99;  // losses.cpp:9
constexpr double kGradEps = 1e-8;         // :10
constexpr double kResidualDeadband = 1e-6;  // :13
constexpr double kHellingerGradFloor = 1e-3;  // :15

__device__ __forceinline__ double sign_of(double x) {  // :17-21
    if (x > kResidualDeadband) return 1.0;
    if (x < -kResidualDeadband) return -1.0;
    return 0.0;
}

// raw_entropy (splat_render.cpp:371-376) of one frame pixel (float probs, fp64 log)
__device__ __forceinline__ double raw_entropy(const float* p, int C) {
    double h = 0.0;
    for (int m = 0; m < C; ++m)
        if (p[m] > 0.0f) h -= static_cast<double>(p[m]) * log(static_cast<double>(p[m]));
    return h;
}

// ---------------------------------------------------------------- loss pixels
// One thread per pixel. Writes per-pixel flags and per-block partial sums:
//   part[block][0..7] = {photo, depth, semantic, n_photo, n_depth, n_sem_q (covered by q),
//                        n_uncovered, n_sem_bwd (covered by contributors)}
__global__ void __launch_bounds__(256) k_loss_pixels(BackwardParams b, double* part) {
    const int px = blockIdx.x * blockDim.x + threadIdx.x;
    const int npx = b.W * b.H;
    double v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (px < npx) {
        const double S = b.sil[px];
        uint8_t flags = 0;
        if (S > kSilhouetteMask) {  // mapping_loss :46-56
            v[3] = 1.0;
            for (int c = 0; c < 3; ++c) v[0] += fabs(b.color[3 * px + c] - static_cast<double>(b.rgb[3 * px + c]));
            const float gt = b.fdepth[px];
            if (gt > 0.0f) {
                v[4] = 1.0;
                v[1] = fabs(b.depth[px] - static_cast<double>(gt));
            }
            flags |= 1;
        }
        const int C = b.C;
        const float* p = b.fsem + static_cast<size_t>(px) * C;
        if (raw_entropy(p, C) < b.tau) {  // semantic_loss :147
            const double* q = b.sem + static_cast<size_t>(px) * C;
            bool any = false;
            for (int m = 0; m < C; ++m)
                if (q[m] != 0.0) any = true;
            if (any) {  // semantic_pixel value (:83-133), no gradient here
                double val = 0.0;
                if (b.use_kl) {
                    double kl = 0.0;
                    for (int m = 0; m < C; ++m) {
                        const double pm = p[m];
                        if (pm <= 0.0) continue;
                        kl += pm * log(pm / fmax(q[m], kGradEps));
                    }
                    val += b.lambda_hd * kl;
                } else if (b.use_hd) {
                    double bc = 0.0;
                    for (int m = 0; m < C; ++m) bc += sqrt(fmax(static_cast<double>(p[m]) * q[m], 0.0));
                    val += b.lambda_hd * sqrt(fmax(1.0 - bc, 0.0));
                }
                if (b.use_cos) {
                    double dot = 0.0, np2 = 0.0, nq2 = 0.0;
                    for (int m = 0; m < C; ++m) {
                        const double pm = p[m];
                        dot += pm * q[m];
                        np2 += pm * pm;
                        nq2 += q[m] * q[m];
                    }
                    val += b.lambda_cos * (1.0 - dot / (sqrt(np2) * sqrt(nq2) + kGradEps));
                }
                v[2] = val;
                v[5] = 1.0;
            } else {
                v[6] = 1.0;
            }
            if (b.ccount[px] > 0) {  // backward's mask (:188-193)
                v[7] = 1.0;
                flags |= 2;
            }
        }
        b.flags[px] = flags;
    }
    __shared__ double red[8][256];
    for (int q = 0; q < 8; ++q) red[q][threadIdx.x] = v[q];
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s)
            for (int q = 0; q < 8; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x < 8) part[blockIdx.x * 8 + threadIdx.x] = red[threadIdx.x][0];
}

// fixed-order sum of the per-block partials -> totals[8]
__global__ void k_loss_totals(const double* part, int nblocks, double* totals) {
    const int q = threadIdx.x;
    if (q >= 8) return;
    double s = 0.0;
    for (int i = 0; i < nblocks; ++i) s += part[i * 8 + q];
    totals[q] = s;
}

// ---------------------------------------------------------------- backward
struct BLayout {
    int dq, f, w, dldf, pxd, gacc, emap, rm, done, stage0, stage_bytes, st_idx, st_prob,
        st_color, total;
};

__host__ __device__ inline BLayout bw_layout(int C, int kpad) {
    BLayout L;
    L.dq = 0;                                   // [C][65] dL/dq (semantic)
    L.f = (C * 65 * 8 + 15) & ~15;              // [kBNB][64] footprint code
    L.w = L.f + kBNB * kTilePx * 8;             // [kBNB][64] w
    L.dldf = L.w + kBNB * kTilePx * 8;          // [kBNB][64] dL/df
    L.pxd = L.dldf + kBNB * kTilePx * 8;        // [64][8] per pixel: dLdC(3), dLdD, R(3), D
    L.gacc = L.pxd + kTilePx * 8 * 8;           // [kBNB][2][8] warp sums
    L.emap = L.gacc + kBNB * 2 * 8 * 8;         // [2][kBNB] map index
    L.rm = L.emap + 2 * kBNB * 4;               // [2][kBNB] (rank, map index)
    L.done = L.rm + 2 * kBNB * 8;               // [64]
    L.stage0 = L.done + kTilePx * 4;
    L.st_idx = kBNB * static_cast<int>(sizeof(PackedSplat));
    L.st_prob = L.st_idx + kBNB * kpad * 2;
    L.st_color = L.st_prob + kBNB * kpad * 8;
    L.stage_bytes = L.st_color + kBNB * 32;
    L.total = L.stage0 + 2 * L.stage_bytes;
    return L;
}

constexpr double kNotContrib = -1.0;
constexpr double kClamped = -2.0;

__global__ void __launch_bounds__(kBThreads, 2) k_backward(RasterParams p, BackwardParams b) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int C = p.map.C, k = p.map.k, kpad = p.map.kpad;
    const BLayout L = bw_layout(C, kpad);
    double* dq = reinterpret_cast<double*>(smem + L.dq);
    double* F = reinterpret_cast<double*>(smem + L.f);
    double* Wv = reinterpret_cast<double*>(smem + L.w);
    double* DL = reinterpret_cast<double*>(smem + L.dldf);
    double* pxd = reinterpret_cast<double*>(smem + L.pxd);
    double* gacc = reinterpret_cast<double*>(smem + L.gacc);
    uint32_t* emap = reinterpret_cast<uint32_t*>(smem + L.emap);
    uint2* rm = reinterpret_cast<uint2*>(smem + L.rm);
    int* sdone = reinterpret_cast<int*>(smem + L.done);
    unsigned char* stg = smem + L.stage0;

    const ViewDesc vd = p.views[0];
    const int tile = blockIdx.x;
    const int bx = tile % p.raster_tiles_x, by = tile / p.raster_tiles_x;
    const int t = threadIdx.x;
    const int lane = t & 31;
    const int px = t & (kTilePx - 1);
    const int x = bx * kTile + (px & (kTile - 1));
    const int y = by * kTile + px / kTile;
    const bool inside = x < p.cam.W && y < p.cam.H;
    const size_t pix = inside ? static_cast<size_t>(y) * p.cam.W + x : 0;
    const int bin = ((by * kTile) / p.opt.ts) * p.opt.tiles_x + (bx * kTile) / p.opt.ts;
    const uint2 rg = vd.ranges[bin];
    const uint32_t L0 = rg.x;
    const uint32_t Ln = rg.y - rg.x;
    const double dpx = x + 0.5, dpy = y + 0.5;
    const float fpx = static_cast<float>(dpx), fpy = static_cast<float>(dpy);
    const int e_first = t >> 6;
    const double n_photo = b.totals[3], n_depth = b.totals[4], n_sem = b.totals[7];

    // ---- per-pixel seeds: dL/dC, dL/dD (:226-236) and the rendered R ----
    if (t < kTilePx) {
        double* d = pxd + t * 8;
        for (int q = 0; q < 8; ++q) d[q] = 0.0;
        sdone[t] = 1;
        if (inside) {
            const uint8_t fl = b.flags[pix];
            const bool map_masked = b.include_mapping && (fl & 1);
            if (map_masked) {
                for (int c = 0; c < 3; ++c)
                    d[c] = 0.5 * sign_of(b.color[3 * pix + c] - static_cast<double>(b.rgb[3 * pix + c])) / n_photo;
                if (b.fdepth[pix] > 0.0f)
                    d[3] = sign_of(b.depth[pix] - static_cast<double>(b.fdepth[pix])) / n_depth;
            }
            for (int c = 0; c < 3; ++c) d[4 + c] = b.color[3 * pix + c];
            d[7] = b.depth[pix];
            const bool sem_px = b.include_semantic && (fl & 2);
            if (b.ccount[pix] > 0 && (map_masked || sem_px)) sdone[t] = 0;  // :216-221
        }
    }
    // ---- dq of the semantic pixel loss (:69-133), 4 threads per pixel ----
    {
        const int q4 = t & 3, pq = t >> 2;  // 64 pixels x 4 channel quarters
        const int qx = bx * kTile + (pq & (kTile - 1)), qy = by * kTile + pq / kTile;
        const bool qin = qx < p.cam.W && qy < p.cam.H;
        const size_t qpix = qin ? static_cast<size_t>(qy) * p.cam.W + qx : 0;
        const bool sem_px = qin && b.include_semantic && (b.flags[qpix] & 2);
        const float* pp = b.fsem + qpix * C;
        const double* qq = b.sem + qpix * C;
        double bc = 0.0, dot = 0.0, np2 = 0.0, nq2 = 0.0;
        if (sem_px)
            for (int m = q4; m < C; m += 4) {
                const double pm = pp[m], qm = qq[m];
                bc += sqrt(fmax(pm * qm, 0.0));
                dot += pm * qm;
                np2 += pm * pm;
                nq2 += qm * qm;
            }
#pragma unroll
        for (int o = 1; o < 4; o <<= 1) {
            bc += __shfl_xor_sync(0xffffffffu, bc, o);
            dot += __shfl_xor_sync(0xffffffffu, dot, o);
            np2 += __shfl_xor_sync(0xffffffffu, np2, o);
            nq2 += __shfl_xor_sync(0xffffffffu, nq2, o);
        }
        const double hd = sqrt(fmax(1.0 - bc, 0.0));
        const double dhd_dbc = -1.0 / (2.0 * hd + kGradEps);
        const double np = sqrt(np2), nq = sqrt(nq2);
        const double denom = np * nq + kGradEps;
        const double inv_n = 1.0 / n_sem;
        for (int m = q4; m < C; m += 4) {
            double g = 0.0;
            if (sem_px) {
                const double pm = pp[m], qm = qq[m];
                if (b.use_kl) {
                    if (pm > 0.0 && qm > kGradEps) g += b.lambda_hd * (-pm / fmax(qm, kGradEps));
                } else if (b.use_hd && hd > kHellingerGradFloor) {
                    if (pm > 0.0 && qm > 0.0) g += b.lambda_hd * dhd_dbc * (pm / (2.0 * sqrt(pm * qm) + kGradEps));
                }
                if (b.use_cos && nq > 0.0)
                    g += -b.lambda_cos * (pm / denom - dot * (np * qm / nq) / (denom * denom));
                g *= inv_n;
            }
            dq[m * 65 + pq] = g;
        }
    }
    __syncthreads();

    constexpr int Qc = 4 + 2;  // PackedSplat + colour (16-byte chunks); rows copied separately
    const int qi = kpad / 8, qp = kpad / 2;
    const int Q = Qc + qi + qp;
    __shared__ int scnt[3];  // entries of batch bb in scnt[bb % 3]
    auto issue = [&](int bb) {
        unsigned char* sb = stg + (bb & 1) * L.stage_bytes;
        const int n = scnt[bb % 3];
        const uint2* slot = rm + (bb & 1) * kBNB;
        for (int c = t; c < n * Q; c += kBThreads) {
            const int e = c / Q;
            int q = c - e * Q;
            const uint2 v = slot[e];
            const unsigned char* src;
            unsigned char* dst;
            if (q < 4) {
                src = reinterpret_cast<const unsigned char*>(vd.packed + v.x) + 16 * q;
                dst = sb + e * 64 + 16 * q;
                if (q == 0) emap[(bb & 1) * kBNB + e] = v.y;
            } else if (q < 6) {
                src = reinterpret_cast<const unsigned char*>(p.map.color4 + static_cast<size_t>(v.y) * 4) + 16 * (q - 4);
                dst = sb + L.st_color + e * 32 + 16 * (q - 4);
            } else if ((q -= 6) < qi) {
                src = reinterpret_cast<const unsigned char*>(p.map.sem_idx + static_cast<size_t>(v.y) * kpad) + 16 * q;
                dst = sb + L.st_idx + e * kpad * 2 + 16 * q;
            } else {
                q -= qi;
                src = reinterpret_cast<const unsigned char*>(p.map.sem_prob + static_cast<size_t>(v.y) * kpad) + 16 * q;
                dst = sb + L.st_prob + e * kpad * 8 + 16 * q;
            }
            const unsigned sdst = static_cast<unsigned>(__cvta_generic_to_shared(dst));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sdst), "l"(src) : "memory");
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    // batches skip bin entries that cannot reach a pixel of the block (fill_batch)
    const float bx0 = static_cast<float>(bx * kTile) + 0.5f, bx1 = bx0 + static_cast<float>(kTile - 1);
    const float by0 = static_cast<float>(by * kTile) + 0.5f, by1 = by0 + static_cast<float>(kTile - 1);
    uint32_t cursor = 0;
    auto fill = [&](int bb) {
        if ((t >> 5) != 0) return;
        const int filled = fill_batch<kBNB>(vd, L0, Ln, cursor, rm + (bb & 1) * kBNB, true, bx0, bx1,
                                            by0, by1, lane);
        if (lane == 0) scnt[bb % 3] = filled;
    };

    fill(0);
    fill(1);
    __syncthreads();
    if (scnt[0] > 0) issue(0);
    double T = 1.0, Pc[4] = {0.0, 0.0, 0.0, 0.0};
    bool done = t < kTilePx ? sdone[t] != 0 : true;
    for (int bb = 0;; ++bb) {
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncthreads();
        const int n = scnt[bb % 3];
        if (n == 0) break;  // the bin is exhausted
        if (scnt[(bb + 1) % 3] > 0) issue(bb + 1);
        fill(bb + 2);
        const unsigned char* sb = stg + (bb & 1) * L.stage_bytes;
        const PackedSplat* sp = reinterpret_cast<const PackedSplat*>(sb);
        const double* scol = reinterpret_cast<const double*>(sb + L.st_color);
        const uint16_t* si = reinterpret_cast<const uint16_t*>(sb + L.st_idx);
        const uint32_t* em = emap + (bb & 1) * kBNB;

        // phase A: footprints (:242-257), clamp recorded
        {
            const bool pdone = sdone[px] != 0;
#pragma unroll
            for (int i = 0; i < kBNB / 4; ++i) {
                const int e = e_first + 4 * i;
                if (e >= n) break;
                double f = kNotContrib;
                if (!pdone) {
                    const float4 pf = *reinterpret_cast<const float4*>(&sp[e].pmx);
                    const float fdx = fpx - pf.x, fdy = fpy - pf.y;
                    if (!(fdx * fdx + fdy * fdy > pf.z)) {
                        const double dx = dpx - sp[e].mx, dy = dpy - sp[e].my;
                        const double d2 = dx * dx + dy * dy;
                        if (!(d2 > sp[e].cutoff_d2)) {
                            f = sp[e].alpha * exp_footprint(-d2 * sp[e].inv_two_r2);
                            if (f > kMaxFootprint) f = kClamped;
                        }
                    }
                }
                F[e * kTilePx + px] = f;
            }
        }
        __syncthreads();
        // phase B: transmittance chain; dL/df with S = R - P (:272-308)
        if (t < kTilePx) {
            const double* d = pxd + t * 8;
            for (int e = 0; e < n; ++e) {
                const int s = e * kTilePx + t;
                const double code = F[s];
                if (done || code == kNotContrib) {
                    F[s] = kNotContrib;
                    Wv[s] = 0.0;
                    DL[s] = 0.0;
                    continue;
                }
                const double f = code == kClamped ? kMaxFootprint : code;
                const double w = f * T;
                const double i1f = 1.0 / (1.0 - f);
                double dldf = 0.0;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    Pc[c] += scol[4 * e + c] * w;
                    dldf += d[c] * (scol[4 * e + c] * T - (d[4 + c] - Pc[c]) * i1f);
                }
                Pc[3] += sp[e].z * w;
                dldf += d[3] * (sp[e].z * T - (d[7] - Pc[3]) * i1f);
                Wv[s] = w;
                DL[s] = dldf;
                T = T * (1.0 - f);
                if (p.opt.early_exit && T < p.opt.eps) done = true;
            }
            sdone[t] = done ? 1 : 0;
        }
        __syncthreads();
        // phase C: per (Gaussian, pixel) terms, reduced over the block's pixels
#pragma unroll 1
        for (int i = 0; i < kBNB / 4; ++i) {
            const int e = e_first + 4 * i;
            if (e >= n) break;  // warp-uniform
            double G[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // alpha, mx, my, rad, z, color rgb
            const int s = e * kTilePx + px;
            const double code = F[s];
            const bool contrib = code != kNotContrib;
            if (contrib) {
                const bool clamped = code == kClamped;
                const double f = clamped ? kMaxFootprint : code;
                const double w = Wv[s], dldf = DL[s];
                const PackedSplat& g = sp[e];
                const double* d = pxd + px * 8;
                const double r2 = 0.5 / g.inv_two_r2;
                const double r = sqrt(r2);
                if (!clamped && r > 0.0) {  // :297-304
                    const double dx = dpx - g.mx, dy = dpy - g.my;
                    G[0] = dldf * f / g.alpha;
                    G[1] = dldf * f * dx / r2;
                    G[2] = dldf * f * dy / r2;
                    G[3] = dldf * f * (dx * dx + dy * dy) / (r2 * r);
                }
                G[4] = d[3] * w;  // g_z (:296)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const double cc = scol[4 * e + c];
                    if (cc > 0.0 && cc < 1.0) G[5 + c] = d[c] * w;  // :291-294
                }
            }
            if (!__any_sync(0xffffffffu, contrib)) {
                if (lane < 8) gacc[(e * 2 + (px >> 5)) * 8 + lane] = 0.0;
                continue;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                double v = G[q];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
                if (lane == 0) gacc[(e * 2 + (px >> 5)) * 8 + q] = v;
            }
        }
        __syncthreads();
        if (t < n * 8) {
            const int e = t >> 3, q = t & 7;
            const double v = gacc[(e * 2) * 8 + q] + gacc[(e * 2 + 1) * 8 + q];
            if (v != 0.0) {
                const uint32_t rank = sp[e].aux;
                if (q < 5)
                    atomicAdd(&b.gproj[static_cast<size_t>(rank) * 5 + q], v);
                else
                    atomicAdd(&b.gcolor[static_cast<size_t>(em[e]) * 3 + (q - 5)], v);
            }
        }
        // sparse semantic terms: g.sem[i][j] += sum_px dq[idx_j][px] w (:262-269)
        if (b.include_semantic) {
            for (int u = t; u < n * k; u += kBThreads) {
                const int e = u / k, j = u - e * k;
                const int c = si[e * kpad + j];
                double sum = 0.0;
                for (int q = 0; q < kTilePx; ++q) sum += dq[c * 65 + q] * Wv[e * kTilePx + q];
                if (sum != 0.0) {
                    const uint32_t m = em[e];
                    const uint16_t orig = b.sem_perm[static_cast<size_t>(m) * kpad + j];
                    atomicAdd(&b.gsem[static_cast<size_t>(m) * k + orig], sum);
                }
            }
        }
        const int mine = (t < kTilePx) ? (done ? 1 : 0) : 1;
        if (__syncthreads_and(mine)) break;
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// ---------------------------------------------------------------- projection -> world
__global__ void k_chain(DevMap m, const PoseParams* __restrict__ pose, CamParams cam, OptParams o,
                        const uint32_t* __restrict__ order, uint32_t V,
                        const double* __restrict__ gproj, BackwardParams b) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= V) return;
    const double* g = gproj + static_cast<size_t>(r) * 5;
    if (g[0] == 0 && g[1] == 0 && g[2] == 0 && g[3] == 0 && g[4] == 0) return;  // :315-316
    const uint32_t i = order[r];
    const PoseParams P = *pose;
    // re-project (bit-identical to the render): mx, my, rad_px, z
    const double d0 = m.cx[i] - P.t[0], d1 = m.cy[i] - P.t[1], d2 = m.cz[i] - P.t[2];
    const double z = P.Rcw[6] * d0 + (P.Rcw[7] * d1 + P.Rcw[8] * d2);
    const double pcx = P.Rcw[0] * d0 + (P.Rcw[1] * d1 + P.Rcw[2] * d2);
    const double pcy = P.Rcw[3] * d0 + (P.Rcw[4] * d1 + P.Rcw[5] * d2);
    const double mx = cam.fx * pcx / z + cam.cx;
    const double my = cam.fy * pcy / z + cam.cy;
    const double rad = m.rad[i] * cam.fy / z;
    const double al = m.alpha[i];
    (void)o;
    const double dX = g[1] * cam.fx / z;  // :323-326
    const double dY = g[2] * cam.fy / z;
    const double dZ = g[4] - g[1] * (mx - cam.cx) / z - g[2] * (my - cam.cy) / z - g[3] * rad / z;
    for (int a = 0; a < 3; ++a) {  // dworld = pose.R * dcam, R = Rcw^T (:327-331)
        const double dw = P.Rcw[a] * dX + (P.Rcw[3 + a] * dY + P.Rcw[6 + a] * dZ);
        b.gcenter[static_cast<size_t>(i) * 3 + a] += dw;
    }
    b.glogr[i] += g[3] * rad;              // :333
    b.glogit[i] += g[0] * al * (1.0 - al);  // :334
}

__global__ void k_kl_clip(double* gsem, uint64_t n, int k, double clip) {  // :337-347
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double n2 = 0.0;
    for (int j = 0; j < k; ++j) n2 += gsem[i * k + j] * gsem[i * k + j];
    const double nrm = sqrt(n2);
    if (nrm > clip) {
        const double s = clip / nrm;
        for (int j = 0; j < k; ++j) gsem[i * k + j] *= s;
    }
}

// first non-finite entry per parameter array (:349-360): bad[a] = min index * stride-free
__global__ void k_finite(const double* v, uint64_t len, unsigned long long* bad) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < len && !isfinite(v[i])) atomicMin(bad, static_cast<unsigned long long>(i));
}

inline unsigned nblk(uint64_t n, unsigned th) { return static_cast<unsigned>((n + th - 1) / th); }

}  // namespace

size_t backward_loss_blocks(int W, int H) { return nblk(static_cast<uint64_t>(W) * H, 256); }

void launch_loss_pixels(const BackwardParams& b, double* part, double* totals, cudaStream_t s) {
    const unsigned nb = nblk(static_cast<uint64_t>(b.W) * b.H, 256);
    k_loss_pixels<<<nb, 256, 0, s>>>(b, part);
    k_loss_totals<<<1, 32, 0, s>>>(part, static_cast<int>(nb), totals);
}

size_t backward_smem_bytes(int C, int kpad) { return static_cast<size_t>(bw_layout(C, kpad).total); }

void launch_backward(const RasterParams& p, const BackwardParams& b, cudaStream_t s) {
    const size_t smem = static_cast<size_t>(bw_layout(p.map.C, p.map.kpad).total);
    // (per launch: the attribute is per device, and contexts on several devices may share
    // the process)
    cudaFuncSetAttribute(k_backward, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k_backward<<<static_cast<unsigned>(p.tiles_per_view), kBThreads, smem, s>>>(p, b);
}

void launch_chain(const DevMap& m, const PoseParams* d_pose, const CamParams& cam, const OptParams& o,
                  const uint32_t* order, uint32_t V, const double* gproj, const BackwardParams& b,
                  cudaStream_t s) {
    if (V == 0) return;
    k_chain<<<nblk(V, 256), 256, 0, s>>>(m, d_pose, cam, o, order, V, gproj, b);
}

void launch_kl_clip(double* gsem, uint64_t n, int k, double clip, cudaStream_t s) {
    if (n == 0) return;
    k_kl_clip<<<nblk(n, 256), 256, 0, s>>>(gsem, n, k, clip);
}

void launch_finite(const double* v, uint64_t len, unsigned long long* bad, cudaStream_t s) {
    if (len == 0) return;
    k_finite<<<nblk(len, 256), 256, 0, s>>>(v, len, bad);
}

}  // namespace sgm
