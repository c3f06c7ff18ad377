// K6 / K7: diagonal Fisher information of the rendered colour and depth with respect to
// the Gaussian parameters, accumulated through the blend (new feature, no
// reference counterpart; parity pinned by finite differences of the oracle renderer).
//
// Parameters per Gaussian: theta = (mu_x, mu_y, mu_z, log_radius, opacity_logit, c_r, c_g,
// c_b); channels: R, G, B, depth. The per-pixel Jacobian is the analytic chain of
// proj/src/losses.cpp:242-335 with a unit seed per channel, chained to world space per
// pixel before squaring:  H[i][theta] += sum_px sum_ch (dR_ch(px)/dtheta_i)^2.
//
// One CTA (8 compute warps + 1 loader warp, as in the raster) = one 8x8 block of one view;
// two passes over the block's depth-ordered list (same cp.async staging as the raster):
//   pass 0  footprints and the segmented transmittance chain -> rendered R_ch per pixel
//           (skipped in gain mode when the score raster wrote R: vd.rc4)
//   pass 1  the chain again; then per (entry, pixel) dR_ch/df_j = v_ch T_j - S_ch / (1 - f_j)
//           with the suffix S = R - P_j (P_j the inclusive prefix, so no reverse sweep is
//           needed), the 8 squared Jacobians in registers, reduced over the warp's 32 pixels
//           (a butterfly), then
//             prior mode: one fp64 RED per (Gaussian, parameter, tile) into H
//             gain mode : sum_theta H_tile[theta] / (H_prior[theta] + lambda) accumulated per
//                         (entry slot, parameter) thread, folded per tile in a fixed order
//                         (deterministic per-view gain).
#include "sgm_device.cuh"
#include "sgm_internal.h"

namespace sgm {

namespace {

constexpr int kFCompute = 256;            // compute threads: warps 0-7
constexpr int kFThreads = kFCompute + 32;  // + warp 8, the batch loader
constexpr int kFNB = 16;

// barrier over the 8 compute warps only (the loader warp runs ahead between the per-batch
// block barriers)
__device__ __forceinline__ void fisher_sync() { asm volatile("bar.sync 1, %0;\n" ::"n"(kFCompute) : "memory"); }

struct FLayout {
    int red, gacc, emap, rm, done, pose, segp, sseg, st, sp, src, stage0, stage_bytes,
        st_color, total;
};

__host__ __device__ inline FLayout fisher_layout() {
    FLayout L;
    L.red = 0;                                // [kFNB][2][8] per-half J^2 sums
    L.gacc = L.red + kFNB * 2 * 8 * 8;        // [kFNB][8] gain terms
    L.emap = L.gacc + kFNB * 8 * 8;           // [2][kFNB] map index
    L.rm = L.emap + 2 * kFNB * 4;             // [2][kFNB] (rank, map index)
    L.done = L.rm + 2 * kFNB * 8;             // [64]
    L.pose = L.done + kTilePx * 4;            // Rcw (9 doubles) + pad
    L.segp = L.pose + 16 * 8;                 // [4][64] segment products of (1 - f)
    L.sseg = L.segp + 4 * kTilePx * 8;        // [4][4][64] segment colour / depth sums (part, channel, pixel)
    L.st = L.sseg + 4 * kTilePx * 4 * 8;      // [64] pixel transmittance at the batch start
    L.sp = L.st + kTilePx * 8;                // [2][4][64] prefix P at the batch start
    L.src = L.sp + 2 * kTilePx * 4 * 8;       // [4][64] rendered R (pass 0 result)
    L.stage0 = L.src + kTilePx * 4 * 8;
    L.st_color = kFNB * static_cast<int>(sizeof(PackedSplat));
    L.stage_bytes = L.st_color + kFNB * 32;
    L.total = L.stage0 + 2 * L.stage_bytes;
    return L;
}

// footprint codes in the f array
constexpr double kNotContrib = -1.0;
constexpr double kClamped = -2.0;

template <bool kGain>
__global__ void __launch_bounds__(kFThreads, 3) k_fisher(RasterParams p, FisherParams fp) {
    extern __shared__ __align__(16) unsigned char smem[];
    const FLayout L = fisher_layout();
    double* red = reinterpret_cast<double*>(smem + L.red);
    double* gacc = reinterpret_cast<double*>(smem + L.gacc);
    uint32_t* emap = reinterpret_cast<uint32_t*>(smem + L.emap);
    uint2* rm = reinterpret_cast<uint2*>(smem + L.rm);
    int* sdone = reinterpret_cast<int*>(smem + L.done);
    double* sR = reinterpret_cast<double*>(smem + L.pose);  // camera-from-world rotation
    double* segp = reinterpret_cast<double*>(smem + L.segp);
    double* sseg = reinterpret_cast<double*>(smem + L.sseg);
    double* sT = reinterpret_cast<double*>(smem + L.st);
    double* sPb = reinterpret_cast<double*>(smem + L.sp);
    double* sRc = reinterpret_cast<double*>(smem + L.src);
    unsigned char* stg = smem + L.stage0;

    const ViewDesc vd = p.views[blockIdx.y];
    const int tile = blockIdx.x;
    const int bx = tile % p.raster_tiles_x, by = tile / p.raster_tiles_x;
    const int t = threadIdx.x;
    const int lane = t & 31;
    const int px = t & (kTilePx - 1);
    const int x = bx * kTile + (px & (kTile - 1));
    const int y = by * kTile + px / kTile;
    const bool inside = x < p.cam.W && y < p.cam.H;
    const int bin = ((by * kTile) / p.opt.ts) * p.opt.tiles_x + (bx * kTile) / p.opt.ts;
    const uint2 rg = vd.ranges[bin];
    const uint32_t L0 = rg.x;
    const uint32_t Ln = rg.y - rg.x;
    const double dpx = x + 0.5, dpy = y + 0.5;
    const float fpx = static_cast<float>(dpx), fpy = static_cast<float>(dpy);

    constexpr int Q = 4 + 2;  // 16-byte chunks per Gaussian: PackedSplat + colour
    __shared__ int scnt[3];  // entries of batch b in scnt[b % 3]
    const bool loader = (t >> 5) == kFCompute / 32;
    auto issue = [&](int b) {  // loader warp
        unsigned char* sb = stg + (b & 1) * L.stage_bytes;
        const int n = scnt[b % 3];
        const uint2* slot = rm + (b & 1) * kFNB;
        for (int c = lane; c < n * Q; c += 32) {
            const int e = c / Q;
            const int q = c - e * Q;
            const uint2 v = slot[e];
            const unsigned char* src;
            unsigned char* dst;
            if (q < 4) {
                src = reinterpret_cast<const unsigned char*>(vd.packed + v.x) + 16 * q;
                dst = sb + e * 64 + 16 * q;
                if (q == 0) emap[(b & 1) * kFNB + e] = v.y;
            } else {
                src = reinterpret_cast<const unsigned char*>(p.map.color4 + static_cast<size_t>(v.y) * 4) + 16 * (q - 4);
                dst = sb + L.st_color + e * 32 + 16 * (q - 4);
            }
            const unsigned sdst = static_cast<unsigned>(__cvta_generic_to_shared(dst));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sdst), "l"(src) : "memory");
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    // batches (formed by the loader warp two ahead) skip bin entries that cannot reach a
    // pixel of the block (fill_batch)
    const float bx0 = static_cast<float>(bx * kTile) + 0.5f, bx1 = bx0 + static_cast<float>(kTile - 1);
    const float by0 = static_cast<float>(by * kTile) + 0.5f, by1 = by0 + static_cast<float>(kTile - 1);
    uint32_t cursor = 0;
    auto fill = [&](int b) {
        const int filled = fill_batch<kFNB>(vd, L0, Ln, cursor, rm + (b & 1) * kFNB, true, bx0, bx1,
                                            by0, by1, lane);
        if (lane == 0) scnt[b % 3] = filled;
    };

    if (t < 9) sR[t] = vd.pose->Rcw[t];
    double Rc[4] = {0.0, 0.0, 0.0, 0.0};  // pass 0 result (threads t < 64)
    // gain mode after a score raster that wrote the rendered colour / depth planes (rc4):
    // pass 0 is skipped (the planes are the same sums, in a fixed segment order)
    const bool haveR = kGain && vd.rc4 != nullptr;
    if (t < kTilePx)
        for (int ch = 0; ch < 4; ++ch) sRc[ch * kTilePx + t] = 0.0;
    if (haveR && t < kTilePx && inside) {
        const size_t pix = static_cast<size_t>(y) * p.cam.W + x;
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) sRc[ch * kTilePx + t] = vd.rc4[pix * 4 + ch];
    }
    const int part = t >> 6;  // phase AB: this thread's segment (entries 4 part .. 4 part + 3)
    double gthr = 0.0;  // gain mode: this thread's (entry slot, parameter) share, batch order

    for (int pass = haveR ? 1 : 0; pass < 2; ++pass) {
        if (t < kTilePx) {
            sdone[t] = inside ? 0 : 1;
            sT[t] = 1.0;
            for (int ch = 0; ch < 4; ++ch) sPb[ch * kTilePx + t] = 0.0;
        }
        if (loader) {  // batch 0 of this pass; batch 1 is formed in iteration 0
            cursor = 0;
            fill(0);
            __syncwarp();
            if (scnt[0] > 0) issue(0);
        }
        __syncthreads();
        if (pass == 1)
            for (int ch = 0; ch < 4; ++ch) Rc[ch] = sRc[ch * kTilePx + px];  // R of this thread's pixel
        int mine = loader ? 1 : 0;  // vote that this thread's pixel is done
        for (int b = 0;; ++b) {
            asm volatile("cp.async.wait_all;\n" ::: "memory");
            // batch b landed; and the block's early termination (every pixel done, :312)
            if (__syncthreads_and(mine)) break;
            const int n = scnt[b % 3];
            if (n == 0) break;  // the bin is exhausted
            if (loader) {
                if (b == 0) {
                    fill(1);
                    __syncwarp();
                }
                if (scnt[(b + 1) % 3] > 0) issue(b + 1);
                fill(b + 2);
                continue;
            }
            const unsigned char* sb = stg + (b & 1) * L.stage_bytes;
            const PackedSplat* sp = reinterpret_cast<const PackedSplat*>(sb);
            const double* scol = reinterpret_cast<const double*>(sb + L.st_color);
            const uint32_t* em = emap + (b & 1) * kFNB;
            // pass 1: the per-Gaussian constants of the Jacobian chain, once per entry (the
            // gain buffer is free during the batches; read in phase C after two barriers)
            double* sEnt = gacc;  // [kFNB][8]
            if (pass == 1 && t < n) {
                const PackedSplat& g = sp[t];
                const double r = sqrt(0.5 / g.inv_two_r2);
                const double inv_r2 = 2.0 * g.inv_two_r2;
                sEnt[t * 8 + 0] = r;
                sEnt[t * 8 + 1] = 1.0 / g.z;
                sEnt[t * 8 + 2] = g.alpha > 0.0 ? 1.0 / g.alpha : 0.0;
                sEnt[t * 8 + 3] = inv_r2;
                sEnt[t * 8 + 4] = inv_r2 / r;
                sEnt[t * 8 + 5] = g.alpha * (1.0 - g.alpha);
                sEnt[t * 8 + 6] = g.mx - p.cam.cx;
                sEnt[t * 8 + 7] = g.my - p.cam.cy;
            }

            // phase AB: thread (part, px) owns the contiguous entries 4 part .. 4 part + 3 of
            // pixel px (warp-uniform entries). Footprints (splat_render.cpp:276-285, clamp
            // recorded) and the segment product of (1 - f); after a barrier each segment starts
            // at T_px * prod(earlier segments) (fixed association) and runs the exact chain
            // (w = f T, T *= 1 - f, exit after accumulating, :312), summing its colour / depth.
            // Pass 1 then forms dR/df_j = v T_j - (R - P_j) / (1 - f_j) (losses.cpp:285-288)
            // with P_j = P at the batch start + earlier segments' sums + the local prefix.
            const bool pdone = sdone[px] != 0;
            const double T0 = sT[px];
            double fcode[4];
            double prod = 1.0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int e = 4 * part + i;
                double f = kNotContrib;
                if (e < n && !pdone) {
                    const float4 pf = *reinterpret_cast<const float4*>(&sp[e].pmx);
                    const float fdx = fpx - pf.x;
                    const float fdy = fpy - pf.y;
                    if (!(fdx * fdx + fdy * fdy > pf.z)) {
                        const double dx = dpx - sp[e].mx;
                        const double dy = dpy - sp[e].my;
                        const double d2 = dx * dx + dy * dy;
                        if (!(d2 > sp[e].cutoff_d2)) {
                            f = sp[e].alpha * exp_footprint(-d2 * sp[e].inv_two_r2);
                            if (f > kMaxFootprint) f = kClamped;
                        }
                    }
                }
                fcode[i] = f;
                if (f != kNotContrib) prod = prod * (1.0 - (f == kClamped ? kMaxFootprint : f));
            }
            segp[part * kTilePx + px] = prod;
            fisher_sync();
            double Ts = T0;
#pragma unroll
            for (int q = 0; q < 3; ++q)
                if (q < part) Ts = Ts * segp[q * kTilePx + px];
            bool exited = pdone || (p.opt.early_exit && Ts < p.opt.eps);
            double Tc = Ts;
            double Sg[4] = {0.0, 0.0, 0.0, 0.0};
            double Tj[4], wj[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int e = 4 * part + i;
                Tj[i] = 0.0;
                wj[i] = 0.0;
                if (e >= n) continue;
                const int s = e * kTilePx + px;
                if (exited || fcode[i] == kNotContrib) {
                    fcode[i] = kNotContrib;
                    continue;
                }
                const double f = fcode[i] == kClamped ? kMaxFootprint : fcode[i];
                const double w = f * Tc;
                Tj[i] = Tc;
                wj[i] = w;
                const double v[4] = {scol[4 * e], scol[4 * e + 1], scol[4 * e + 2], sp[e].z};
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) Sg[ch] += v[ch] * w;
                Tc = Tc * (1.0 - f);
                if (p.opt.early_exit && Tc < p.opt.eps) exited = true;
            }
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) sseg[(part * 4 + ch) * kTilePx + px] = Sg[ch];
            if (part == 3) {  // the pixel's T and done flag for the next batch
                sT[px] = Tc;
                sdone[px] = (pdone || (p.opt.early_exit && Tc < p.opt.eps)) ? 1 : 0;
            }
            fisher_sync();
            {
                const double* Pb = sPb + (b & 1) * kTilePx * 4;
                double* Pn = sPb + ((b + 1) & 1) * kTilePx * 4;
                if (pass == 0) {
                    if (part == 0)  // R accumulates batch by batch, segments in a fixed order
                        for (int ch = 0; ch < 4; ++ch)
                            sRc[ch * kTilePx + px] += ((sseg[(0 * 4 + ch) * kTilePx + px] + sseg[(1 * 4 + ch) * kTilePx + px]) +
                                                 sseg[(2 * 4 + ch) * kTilePx + px]) + sseg[(3 * 4 + ch) * kTilePx + px];
                } else {
                    double P[4];
#pragma unroll
                    for (int ch = 0; ch < 4; ++ch) {
                        P[ch] = Pb[ch * kTilePx + px];
#pragma unroll
                        for (int q = 0; q < 3; ++q)
                            if (q < part) P[ch] += sseg[(q * 4 + ch) * kTilePx + px];
                    }
                    // per entry: dR_ch/df (losses.cpp:285-288), then the squared Jacobians of the
                    // 8 parameters at this pixel, reduced over the warp's 32 pixels (the warp's
                    // entries are uniform: entry e of half-tile px >> 5)
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int e = 4 * part + i;
                        if (e >= n) break;  // warp-uniform
                        const bool contrib = fcode[i] != kNotContrib;
                        double J[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                        if (contrib) {
                            const bool clamped = fcode[i] == kClamped;
                            const double f = clamped ? kMaxFootprint : fcode[i];
                            const double w = wj[i];
                            const double i1f = 1.0 / (1.0 - f);
                            const double v[4] = {scol[4 * e], scol[4 * e + 1], scol[4 * e + 2], sp[e].z};
                            double dR[4];
#pragma unroll
                            for (int ch = 0; ch < 4; ++ch) {
                                P[ch] += v[ch] * w;
                                dR[ch] = v[ch] * Tj[i] - (Rc[ch] - P[ch]) * i1f;
                            }
                            const PackedSplat& g = sp[e];
                            // d f / d(param) (losses.cpp:297-304); zero when clamped or alpha == 0
                            const bool chain = !clamped && g.alpha > 0.0;
                            const double* ek = sEnt + e * 8;  // r, 1/z, 1/alpha, 1/r^2, 1/r^3, ...
                            const double r = ek[0];
                            const double iz = ek[1];
                            const double dx = dpx - g.mx, dy = dpy - g.my;
                            const double d2 = dx * dx + dy * dy;
                            const double fa = chain ? f * ek[2] : 0.0;
                            const double fmx = chain ? f * dx * ek[3] : 0.0;
                            const double fmy = chain ? f * dy * ek[3] : 0.0;
                            const double fr = chain ? f * d2 * ek[4] : 0.0;
                            // d_cam(ch) = dR_ch/df * u + [ch == depth] * w * e_z with
                            // u = (fmx fx/z, fmy fy/z, -(fmx (mx-cx) + fmy (my-cy) + fr r) / z)
                            // (losses.cpp:323-326), so with v = R u (world, R = Rcw^T):
                            //   sum_ch J_a^2 = S_rgb v_a^2 + (dR_D/df v_a + w R_{a,z})^2
                            const double ux = fmx * p.cam.fx * iz;
                            const double uy = fmy * p.cam.fy * iz;
                            const double uz = -(fmx * ek[6] + fmy * ek[7] + fr * r) * iz;
                            const double Srgb = dR[0] * dR[0] + dR[1] * dR[1] + dR[2] * dR[2];
                            const double Sall = Srgb + dR[3] * dR[3];
#pragma unroll
                            for (int a = 0; a < 3; ++a) {
                                const double va = sR[a] * ux + sR[3 + a] * uy + sR[6 + a] * uz;
                                const double dep = dR[3] * va + w * sR[6 + a];
                                J[a] = Srgb * va * va + dep * dep;
                            }
                            const double jl = fr * r;     // d/d log_r (:333)
                            const double jo = fa * ek[5];  // d/d logit (:334)
                            J[3] = Sall * jl * jl;
                            J[4] = Sall * jo * jo;
#pragma unroll
                            for (int ch = 0; ch < 3; ++ch) {
                                const double c = v[ch];
                                if (c > 0.0 && c < 1.0) J[5 + ch] = w * w;  // losses.cpp:291-294
                            }
                        }
                        double* rslot = red + (e * 2 + (px >> 5)) * 8;
                        if (!__any_sync(0xffffffffu, contrib)) {
                            if (lane < 8) rslot[lane] = 0.0;
                            continue;
                        }
                        // butterfly reduce-scatter of the 8 sums over the warp's 32 pixels (9
                        // double shuffles instead of 8 trees of 5; fixed pattern, deterministic):
                        // halve the parameter set at xor 16, 8, 4, then add across xor 2, 1; lane
                        // l ends with parameter (l >> 2) & 7
                        const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
                        double K4[4], K2[2];
#pragma unroll
                        for (int k4 = 0; k4 < 4; ++k4) {
                            const double send = h16 ? J[k4] : J[k4 + 4];
                            const double keep = h16 ? J[k4 + 4] : J[k4];
                            K4[k4] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
                        }
#pragma unroll
                        for (int k2 = 0; k2 < 2; ++k2) {
                            const double send = h8 ? K4[k2] : K4[k2 + 2];
                            const double keep = h8 ? K4[k2 + 2] : K4[k2];
                            K2[k2] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
                        }
                        double sv = (h4 ? K2[1] : K2[0]) + __shfl_xor_sync(0xffffffffu, h4 ? K2[0] : K2[1], 4);
                        sv += __shfl_xor_sync(0xffffffffu, sv, 2);
                        sv += __shfl_xor_sync(0xffffffffu, sv, 1);
                        if ((lane & 3) == 0) rslot[(lane >> 2) & 7] = sv;
                    }
                    if (part == 0)  // P at the next batch's start (the other buffer)
                        for (int ch = 0; ch < 4; ++ch)
                            Pn[ch * kTilePx + px] = Pb[ch * kTilePx + px] +
                                              (((sseg[(0 * 4 + ch) * kTilePx + px] + sseg[(1 * 4 + ch) * kTilePx + px]) +
                                                sseg[(2 * 4 + ch) * kTilePx + px]) + sseg[(3 * 4 + ch) * kTilePx + px]);
                }
            }

            // pass 1: the squared-Jacobian sums of the batch's entries -> H (prior) or the
            // gain (red is rewritten by the next batch, two barriers later)
            if (pass == 1) {
                fisher_sync();
                if (t < n * 8) {
                    const int e = t >> 3, q = t & 7;
                    const double sum = red[(e * 2) * 8 + q] + red[(e * 2 + 1) * 8 + q];
                    const size_t slot = static_cast<size_t>(em[e]) * 8 + q;
                    if (kGain)
                        gthr += sum * fp.invp[slot];
                    else if (sum != 0.0)
                        atomicAdd(&fp.H[slot], sum);
                }
            }
            mine = sdone[px];
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncthreads();
    }
    if (kGain) {  // the tile's gain: threads 0..127 in a fixed order (deterministic)
        double v = gthr;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (lane == 0 && t < kFNB * 8) gacc[t >> 5] = v;
        __syncthreads();
        if (t == 0) vd.fis_partial[tile] = ((gacc[0] + gacc[1]) + gacc[2]) + gacc[3];
    }
}

template <bool kGain>
void launch_fisher_t(const RasterParams& p, const FisherParams& fp, int n_views, cudaStream_t s) {
    auto kern = k_fisher<kGain>;
    const size_t smem = static_cast<size_t>(fisher_layout().total);
    // (per launch: the attribute is per device, and contexts on several devices may share
    // the process)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    dim3 grid(static_cast<unsigned>(p.tiles_per_view), static_cast<unsigned>(n_views), 1);
    kern<<<grid, kFThreads, smem, s>>>(p, fp);
}

__global__ void k_fisher_invp(const double* __restrict__ H, double lambda, size_t n, double* invp) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) invp[i] = 1.0 / (H[i] + lambda);
}

}  // namespace

void launch_fisher_prior(const RasterParams& p, const FisherParams& fp, int n_views, cudaStream_t s) {
    launch_fisher_t<false>(p, fp, n_views, s);
}

void launch_fisher_gain(const RasterParams& p, const FisherParams& fp, int n_views, cudaStream_t s) {
    launch_fisher_t<true>(p, fp, n_views, s);
}

void launch_fisher_invp(const double* H, double lambda, size_t n, double* invp, cudaStream_t s) {
    if (n == 0) return;
    k_fisher_invp<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(H, lambda, n, invp);
}

}  // namespace sgm
