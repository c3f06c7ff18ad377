// Evaluation metrics on device-resident render planes:
// semantic_metrics (proj/src/evaluator.cpp:93-238) and photometric_metrics (:274-297)
// without copying the px*(5+C) fp64 planes of each view to the host.
//
// Per view (k_eval_view, 32-pixel tiles staged in shared memory with coalesced loads):
//   gt label = Frame::label_at (first max over the float simplex, frame.hpp:41-47);
//   pixels labelled "unknown" are skipped (:111); pred = argmax_channel (first max);
//   top-1 / top-3 (strictly-higher count with index tie-break, :120-123) counters and the
//   C x C confusion matrix (warp-aggregated 64-bit atomics); the per-class AP score
//   float(q[c] / s) (0 when s <= 1e-9, :163-164) of every pixel, class-major, written as
//   32 consecutive floats per class row.
// At report time each class is stable-radix-sorted by descending score (ties keep the
// (view, pixel) order of the reference's std::stable_sort, :168-169). Unknown-labelled
// pixels get the largest key, so they sort after every valid score and leave the ranks of
// the valid ones as in the reference's compacted list; AP is the sum over positives of
// (recall - prev_recall) * precision (:170-180).
// k_eval_photo: per-pixel squared colour error and valid-depth |error|, reduced in a
// fixed order (deterministic).
#include "sgm_internal.h"

namespace sgm {

namespace {

constexpr int kEvalThreads = 256;
constexpr int kTileP = 32;  // pixels per k_eval_view block

__global__ void __launch_bounds__(kEvalThreads) k_eval_view(
    const double* __restrict__ sem, const double* __restrict__ sil, const float* __restrict__ fsem,
    int px, int C, unsigned long long* __restrict__ confusion,
    unsigned long long* __restrict__ counters, uint16_t* __restrict__ label,
    float* __restrict__ scores) {
    extern __shared__ __align__(16) unsigned char esm[];
    double* q_s = reinterpret_cast<double*>(esm);            // [32][C]
    float* f_s = reinterpret_cast<float*>(q_s + kTileP * C);  // [32][C]
    __shared__ double s_sil[kTileP];
    const int base = blockIdx.x * kTileP;
    const int np = min(kTileP, px - base);
    const size_t off = static_cast<size_t>(base) * C;
    for (int i = threadIdx.x; i < np * C; i += blockDim.x) {
        q_s[i] = sem[off + i];
        f_s[i] = fsem[off + i];
    }
    if (threadIdx.x < np) s_sil[threadIdx.x] = sil[base + threadIdx.x];
    __syncthreads();
    if (threadIdx.x < 32) {
        const int p = threadIdx.x;
        bool ok = false;
        int gt = 0, pred = 0, higher = 0;
        if (p < np) {
            const float* f = f_s + p * C;
            for (int m = 1; m < C; ++m)  // Frame::label_at (frame.hpp:41-47)
                if (f[m] > f[gt]) gt = m;
            ok = gt != C - 1;  // unknown_class()
            if (ok) {
                const double* q = q_s + p * C;
                for (int m = 1; m < C; ++m)  // argmax_channel (evaluator.cpp:18-23)
                    if (q[m] > q[pred]) pred = m;
                const double qg = q[gt];
                for (int m = 0; m < C; ++m)  // :120-123
                    if (q[m] > qg || (q[m] == qg && m < gt)) ++higher;
            }
            label[base + p] = ok ? static_cast<uint16_t>(gt) : static_cast<uint16_t>(0xffff);
        }
        // confusion: warp-aggregated over equal (gt, pred) cells
        const unsigned act = __ballot_sync(0xffffffffu, ok);
        if (ok) {
            const int cell = gt * C + pred;
            const unsigned same = __match_any_sync(act, cell);
            if (p == __ffs(same) - 1)
                atomicAdd(&confusion[cell], static_cast<unsigned long long>(__popc(same)));
        }
        unsigned top1 = ok && pred == gt, top3 = ok && higher < 3, tot = ok;
        for (int o = 16; o; o >>= 1) {
            top1 += __shfl_xor_sync(0xffffffffu, top1, o);
            top3 += __shfl_xor_sync(0xffffffffu, top3, o);
            tot += __shfl_xor_sync(0xffffffffu, tot, o);
        }
        if (p == 0 && tot) {
            atomicAdd(&counters[0], static_cast<unsigned long long>(top1));
            atomicAdd(&counters[1], static_cast<unsigned long long>(top3));
            atomicAdd(&counters[2], static_cast<unsigned long long>(tot));
        }
    }
    // AP scores float(q[c] / s) (0 when s <= 1e-9), evaluator.cpp:163-164
    const int p = threadIdx.x & 31;
    if (p < np) {
        const double sv = s_sil[p];
        const double* q = q_s + p * C;
        for (int c = threadIdx.x >> 5; c < C - 1; c += kEvalThreads / 32)
            scores[static_cast<size_t>(c) * px + base + p] =
                sv > 1e-9 ? static_cast<float>(q[c] / sv) : 0.0f;
    }
}

// Per-block partial sums of (sum (colour - rgb)^2, sum |depth - gt| over gt > 0, count).
__global__ void __launch_bounds__(kEvalThreads) k_eval_photo(
    const double* __restrict__ color, const double* __restrict__ depth,
    const float* __restrict__ rgb, const float* __restrict__ gdepth, int px,
    double* __restrict__ part) {
    __shared__ double s_mse[kEvalThreads], s_dep[kEvalThreads], s_cnt[kEvalThreads];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double mse = 0.0, dep = 0.0, cnt = 0.0;
    if (i < px) {
        for (int c = 0; c < 3; ++c) {
            const double d = color[3 * static_cast<size_t>(i) + c] - rgb[3 * static_cast<size_t>(i) + c];
            mse += d * d;  // mapper.cpp:101-103
        }
        const float g = gdepth[i];
        if (!(g <= 0)) {  // evaluator.cpp:286
            dep = fabs(depth[i] - g);
            cnt = 1.0;
        }
    }
    s_mse[threadIdx.x] = mse;
    s_dep[threadIdx.x] = dep;
    s_cnt[threadIdx.x] = cnt;
    __syncthreads();
    for (int s = kEvalThreads / 2; s > 0; s >>= 1) {  // fixed tree
        if (threadIdx.x < s) {
            s_mse[threadIdx.x] += s_mse[threadIdx.x + s];
            s_dep[threadIdx.x] += s_dep[threadIdx.x + s];
            s_cnt[threadIdx.x] += s_cnt[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[3 * blockIdx.x] = s_mse[0];
        part[3 * blockIdx.x + 1] = s_dep[0];
        part[3 * blockIdx.x + 2] = s_cnt[0];
    }
}

__global__ void k_eval_photo_sum(const double* __restrict__ part, int nb, double* __restrict__ out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double a = 0.0, b = 0.0, c = 0.0;  // fixed order over blocks
    for (int i = 0; i < nb; ++i) {
        a += part[3 * i];
        b += part[3 * i + 1];
        c += part[3 * i + 2];
    }
    out[0] = a;
    out[1] = b;
    out[2] = c;
}

// Descending-order radix key of a non-negative float score; unknown pixels last.
__global__ void k_eval_keys(const float* __restrict__ s, const uint16_t* __restrict__ label,
                            uint32_t T, int c, uint32_t* __restrict__ keys,
                            uint32_t* __restrict__ pos) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= T) return;
    uint32_t u = __float_as_uint(s[j]);
    u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);  // ascending-sortable
    keys[j] = label[j] == 0xffff ? 0xffffffffu : ~u;  // descending
    pos[j] = label[j] == c;
}

// AP terms at sorted positions i holding a positive: (tp/P - (tp-1)/P) * (tp/(i+1)).
__global__ void k_eval_ap_terms(const uint32_t* __restrict__ pos, const uint32_t* __restrict__ tp,
                                uint32_t T, double P, double* __restrict__ terms) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= T) return;
    if (!pos[i]) {
        terms[i] = 0.0;
        return;
    }
    const double t = static_cast<double>(tp[i]);
    const double recall = t / P;
    const double prev = (t - 1.0) / P;
    terms[i] = (recall - prev) * (t / (static_cast<double>(i) + 1.0));
}

inline unsigned nb(uint64_t n, unsigned t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

size_t eval_view_smem(int C) { return static_cast<size_t>(kTileP) * C * 12; }

void launch_eval_view(const double* sem, const double* sil, const float* fsem, int px, int C,
                      unsigned long long* confusion, unsigned long long* counters, uint16_t* label,
                      float* scores, cudaStream_t s) {
    const size_t smem = eval_view_smem(C);
    // (per launch: the attribute is per device, and contexts on several devices may share
    // the process)
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_eval_view, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    if (px > 0)
        k_eval_view<<<nb(px, kTileP), kEvalThreads, smem, s>>>(sem, sil, fsem, px, C, confusion,
                                                               counters, label, scores);
}

int eval_photo_blocks(int px) { return static_cast<int>(nb(px, kEvalThreads)); }

void launch_eval_photo(const double* color, const double* depth, const float* rgb,
                       const float* gdepth, int px, double* part, double* out, cudaStream_t s) {
    const int b = eval_photo_blocks(px);
    if (px > 0) k_eval_photo<<<b, kEvalThreads, 0, s>>>(color, depth, rgb, gdepth, px, part);
    k_eval_photo_sum<<<1, 32, 0, s>>>(part, px > 0 ? b : 0, out);
}

void launch_eval_keys(const float* scores, const uint16_t* label, uint32_t T, int c, uint32_t* keys,
                      uint32_t* pos, cudaStream_t s) {
    if (T > 0) k_eval_keys<<<nb(T, 256), 256, 0, s>>>(scores, label, T, c, keys, pos);
}

void launch_eval_ap_terms(const uint32_t* pos, const uint32_t* tp, uint32_t T, double P,
                          double* terms, cudaStream_t s) {
    if (T > 0) k_eval_ap_terms<<<nb(T, 256), 256, 0, s>>>(pos, tp, T, P, terms);
}

}  // namespace sgm
