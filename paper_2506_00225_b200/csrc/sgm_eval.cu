// Evaluation metrics on device-resident render planes:
// semantic_metrics (proj/src/evaluator.cpp:93-238) and photometric_metrics (:274-297)
// without copying the px*(5+C) fp64 planes of each view to the host.
//
// Per view (k_eval_pixels, one thread per pixel):
//   gt label = Frame::label_at (first max over the float simplex, frame.hpp:41-47);
//   pixels labelled "unknown" are skipped (:111); pred = argmax_channel (first max);
//   top-1 / top-3 (strictly-higher count with index tie-break, :120-123) counters and the
//   C x C confusion matrix (a shared-memory histogram flushed with 64-bit atomics).
// The valid pixels are compacted in pixel order; k_eval_scores writes the per-class AP
// score float(q[c] / s) (0 when s <= 1e-9, :163-164) for every valid pixel, class-major.
// At report time each class is stable-radix-sorted by descending score (ties keep the
// (view, pixel) order of the reference's std::stable_sort, :168-169) and AP is the
// sum over positives of (recall - prev_recall) * precision (:170-180).
// k_eval_photo: per-pixel squared colour error and valid-depth |error|, reduced in a
// fixed order (deterministic).
#include "sgm_internal.h"

namespace sgm {

namespace {

constexpr int kEvalThreads = 256;

__global__ void __launch_bounds__(kEvalThreads) k_eval_pixels(
    const double* __restrict__ sem, const float* __restrict__ fsem, int px, int C,
    unsigned long long* __restrict__ confusion, unsigned long long* __restrict__ counters,
    uint8_t* __restrict__ valid, uint16_t* __restrict__ label, int use_smem) {
    extern __shared__ unsigned int hist[];  // [C][C], or none: global atomics (large C)
    const bool local = use_smem != 0;
    if (local)
        for (int i = threadIdx.x; i < C * C; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    unsigned top1 = 0, top3 = 0, total = 0;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < px) {
        const float* f = fsem + static_cast<size_t>(i) * C;
        int gt = 0;
        for (int m = 1; m < C; ++m)
            if (f[m] > f[gt]) gt = m;
        const bool ok = gt != C - 1;  // unknown_class() == num_classes
        valid[i] = ok;
        label[i] = static_cast<uint16_t>(gt);
        if (ok) {
            const double* q = sem + static_cast<size_t>(i) * C;
            int pred = 0;
            for (int m = 1; m < C; ++m)
                if (q[m] > q[pred]) pred = m;
            if (local) atomicAdd(&hist[gt * C + pred], 1u);
            else atomicAdd(&confusion[gt * C + pred], 1ull);
            ++total;
            top1 += pred == gt;
            const double qg = q[gt];
            int higher = 0;
            for (int m = 0; m < C; ++m)
                if (q[m] > qg || (q[m] == qg && m < gt)) ++higher;
            top3 += higher < 3;
        }
    }
    for (int o = 16; o; o >>= 1) {
        top1 += __shfl_xor_sync(0xffffffffu, top1, o);
        top3 += __shfl_xor_sync(0xffffffffu, top3, o);
        total += __shfl_xor_sync(0xffffffffu, total, o);
    }
    if ((threadIdx.x & 31) == 0 && total) {
        atomicAdd(&counters[0], static_cast<unsigned long long>(top1));
        atomicAdd(&counters[1], static_cast<unsigned long long>(top3));
        atomicAdd(&counters[2], static_cast<unsigned long long>(total));
    }
    __syncthreads();
    if (local)
        for (int j = threadIdx.x; j < C * C; j += blockDim.x)
            if (hist[j]) atomicAdd(&confusion[j], static_cast<unsigned long long>(hist[j]));
}

// scores[c * T + j] for the view's valid pixels j (pixel index idx[j]); M = C - 1 classes
__global__ void k_eval_scores(const double* __restrict__ sem, const double* __restrict__ sil,
                              const uint32_t* __restrict__ idx, const uint16_t* __restrict__ label,
                              uint32_t T, int C, float* __restrict__ scores,
                              uint16_t* __restrict__ lab_out) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= T) return;
    const uint32_t i = idx[j];
    lab_out[j] = label[i];
    const double s = sil[i];
    const double* q = sem + static_cast<size_t>(i) * C;
    for (int c = 0; c < C - 1; ++c)
        scores[static_cast<size_t>(c) * T + j] = s > 1e-9 ? static_cast<float>(q[c] / s) : 0.0f;
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

// Descending-order radix key of a non-negative float score (ties keep input order).
__global__ void k_eval_keys(const float* __restrict__ s, const uint16_t* __restrict__ label,
                            uint32_t T, int c, uint32_t* __restrict__ keys,
                            uint32_t* __restrict__ pos) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= T) return;
    uint32_t u = __float_as_uint(s[j]);
    u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);  // ascending-sortable
    keys[j] = ~u;                                      // descending
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

size_t eval_pixels_smem(int C) { return 4ull * C * C; }

void launch_eval_pixels(const double* sem, const float* fsem, int px, int C,
                        unsigned long long* confusion, unsigned long long* counters, uint8_t* valid,
                        uint16_t* label, cudaStream_t s) {
    size_t smem = eval_pixels_smem(C);
    const int use_smem = smem <= 200 * 1024 ? 1 : 0;
    if (!use_smem) smem = 0;
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        cudaFuncSetAttribute(k_eval_pixels, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        configured = smem;
    }
    if (px > 0)
        k_eval_pixels<<<nb(px, kEvalThreads), kEvalThreads, smem, s>>>(
            sem, fsem, px, C, confusion, counters, valid, label, use_smem);
}

void launch_eval_scores(const double* sem, const double* sil, const uint32_t* idx,
                        const uint16_t* label, uint32_t T, int C, float* scores, uint16_t* lab_out,
                        cudaStream_t s) {
    if (T > 0) k_eval_scores<<<nb(T, 256), 256, 0, s>>>(sem, sil, idx, label, T, C, scores, lab_out);
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
