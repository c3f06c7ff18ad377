// Device helpers shared by the raster (sgm_raster.cu) and Fisher (sgm_fisher.cu) kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "sgm_internal.h"

namespace sgm {
namespace {

// exp(x) for the footprint argument x = -d2 / (2 r^2) in [-cut^2/2, 0]:
// Cody-Waite reduction by ln 2 and a degree-13 Taylor polynomial (|r| <= ln2/2,
// truncation < 2.5e-16 relative). Coefficients live in the constant bank so the
// DFMAs take them as operands (no 64-bit immediate moves).
static __constant__ double c_exp[16] = {
    1.4426950408889634,      // log2(e)
    0.6931467056274414,      // ln2 hi (low 32 mantissa bits zero: k * hi is exact)
    4.7493250390941725e-07,  // ln2 lo
    1.6059043836821613e-10,  // 1/13!
    2.08767569878681e-09,    // 1/12!
    2.505210838544172e-08,   // 1/11!
    2.755731922398589e-07,   // 1/10!
    2.7557319223985893e-06,  // 1/9!
    2.48015873015873e-05,    // 1/8!
    0.0001984126984126984,   // 1/7!
    0.001388888888888889,    // 1/6!
    0.008333333333333333,    // 1/5!
    0.041666666666666664,    // 1/4!
    0.16666666666666666,     // 1/3!
    0.5,                     // 1/2!
    1.0};

__device__ __forceinline__ double exp_footprint(double x) {
    if (x < -700.0) return 0.0;  // (outside the footprint range; keeps the scaling valid)
    const double shifter = 6755399441055744.0;  // 1.5 * 2^52: round-to-int in the low word
    const double t = __fma_rn(x, c_exp[0], shifter);
    const double kf = t - shifter;
    const int k = __double2loint(t);
    double r = __fma_rn(-kf, c_exp[1], x);
    r = __fma_rn(-kf, c_exp[2], r);
    double p = c_exp[3];
#pragma unroll
    for (int i = 4; i < 15; ++i) p = __fma_rn(p, r, c_exp[i]);
    p = __fma_rn(p, r, 1.0);
    p = __fma_rn(p, r, 1.0);
    // scale by 2^k (k >= -1011 here, so the result stays normal)
    return __hiloint2double(__double2hiint(p) + k * (1 << 20), __double2loint(p));
}

// log(x) for normal x > 0 (the epilogue's clamped probabilities, [1e-3, 1]):
// x = m 2^e, m in [1,2); c = RN(1 / centre of m's 1/128 interval); r = m c - 1
// (|r| <= 2^-8, exact-ish via FMA); log x = e ln2 - log c + log1p(r) with a
// degree-7 series. ~1e-16 absolute error; ~16 instructions.
static __device__ const double2 g_logtab[128] = {
#include "sgm_logtab.inc"
};
static __constant__ double c_log[10] = {0.14285714285714285,  -0.16666666666666666, 0.2, -0.25,
                                 0.3333333333333333,   -0.5,                 1.0,
                                 0.6931467056274414,   4.7493250390941725e-07, 0.0};

__device__ __forceinline__ double log_table(double x) {
    const int hi = __double2hiint(x);
    const int lo = __double2loint(x);
    const double e = static_cast<double>((hi >> 20) - 1023);
    const int i = (hi >> 13) & 0x7f;
    const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, lo);
    const double2 tc = __ldg(&g_logtab[i]);
    const double r = __fma_rn(m, tc.x, -1.0);
    double q = c_log[0];
#pragma unroll
    for (int j = 1; j < 7; ++j) q = __fma_rn(q, r, c_log[j]);
    const double l1p = q * r;
    return __fma_rn(e, c_log[7], tc.y + __fma_rn(e, c_log[8], l1p));
}

__device__ __forceinline__ double clamp_prob(double v) {
    // std::clamp(v, 0.001, 1.0) (splat_render.cpp:362)
    return v < 0.001 ? 0.001 : (1.0 < v ? 1.0 : v);
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc) : "memory");
}
// Forms one batch of up to kB bin entries (depth order) for an 8x8 pixel block: called by
// all 32 lanes of one warp; `cursor` (the next bin entry to examine, same in every lane)
// advances past the consumed entries; slot[i] = (depth rank, map index). With `skip`, an
// entry whose float probe circle (splat_render.cpp:276-278) misses the box of the block's
// pixel centres [bx0, bx1] x [by0, by1] by a relative margin above the probe's fp32
// rounding is passed over: it cannot pass the prefilter at any pixel, so the composite is
// unchanged. Returns the number of entries placed.
template <int kB>
__device__ __forceinline__ int fill_batch(const ViewDesc& vd, uint32_t L0, uint32_t Ln,
                                          uint32_t& cursor, uint2* slot, bool skip, float bx0,
                                          float bx1, float by0, float by1, int lane) {
    int filled = 0;
    while (filled < kB && cursor < Ln) {
        const uint32_t q = cursor + lane;
        bool keep = false;
        uint32_t r = 0;
        if (q < Ln) {
            r = vd.list[L0 + q];
            keep = true;
            if (skip) {
                const float4 pf = *reinterpret_cast<const float4*>(&vd.packed[r].pmx);
                const double ex = fmax(fmax(static_cast<double>(bx0) - pf.x, 0.0), static_cast<double>(pf.x) - bx1);
                const double ey = fmax(fmax(static_cast<double>(by0) - pf.y, 0.0), static_cast<double>(pf.y) - by1);
                keep = !((ex * ex + ey * ey) * (1.0 - 1e-6) > static_cast<double>(pf.z));
            }
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        const int need = kB - filled;
        const int avail = __popc(bal);
        const int rank = __popc(bal & ((1u << lane) - 1u));
        // entries consumed: through the need-th kept one, else the whole window
        const uint32_t lastk = __ballot_sync(0xffffffffu, keep && rank == need - 1);
        const uint32_t used = avail > need ? static_cast<uint32_t>(__ffs(lastk)) : min(32u, Ln - cursor);
        if (keep && rank < need) slot[filled + rank] = make_uint2(r, vd.order[r]);
        filled += min(avail, need);
        cursor += used;
    }
    return filled;
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

// ---- bulk copies (TMA engine, cp.async.bulk) completing on an mbarrier ----
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, unsigned bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, unsigned parity) {
    asm volatile(
        "{ .reg .pred P1;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        " @!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(bar), "r"(parity) : "memory");
}
// generic-proxy accesses of this thread ordered before its later async-proxy (bulk copy) ones
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
// global -> shared bulk copy of `bytes` (a multiple of 16, both addresses 16-byte aligned)
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, unsigned bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(smem_addr(smem_dst)), "l"(gsrc), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

}  // namespace

// ---- tensor memory (tcgen05): an fp64 accumulator slice per warp. Addresses are
// (lane << 16) | column; a warp reaches only the 32 lanes of its quarter (warp % 4). ----
constexpr uint32_t kTmemCols = 128;  // columns allocated per CTA (3 CTAs per SM: 384 of 512)
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {  // one warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n" ::"r"(smem_addr(dst_smem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t base) {  // the allocating warp
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;\n" ::"r"(base));
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
// two fp64 per lane (4 columns from addr): lane l's pixels 2l, 2l+1
__device__ __forceinline__ void tmem_ld2(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr) : "memory");
}
__device__ __forceinline__ void tmem_st2(uint32_t addr, const uint32_t (&r)[4]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};\n"
                 ::"r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]) : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ double2 tmem_unpack(const uint32_t (&r)[4]) {
    return make_double2(__hiloint2double(static_cast<int>(r[1]), static_cast<int>(r[0])),
                        __hiloint2double(static_cast<int>(r[3]), static_cast<int>(r[2])));
}
__device__ __forceinline__ void tmem_pack(double2 v, uint32_t (&r)[4]) {
    r[0] = static_cast<uint32_t>(__double2loint(v.x));
    r[1] = static_cast<uint32_t>(__double2hiint(v.x));
    r[2] = static_cast<uint32_t>(__double2loint(v.y));
    r[3] = static_cast<uint32_t>(__double2hiint(v.y));
}

}  // namespace sgm
