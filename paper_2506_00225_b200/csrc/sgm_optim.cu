// On-device map optimisation: the Adam step of AdamState::step
// (proj/src/mapper.cpp:10-51) with apply_semantic_step (proj/src/gaussian_map.cpp:51-63),
// opacity pruning (gaussian_map.cpp:97-124, AdamState::compact mapper.cpp:53-69), and the
// re-derivation of the render snapshot (DevMap) from the master parameters.
//
// Master parameters and both Adam moments share the gradient layout of backward_core
// (NS = max(N, 1)):  center 3NS | log_radius NS | opacity_logit NS | color 3NS | sem k*NS.
// Arithmetic follows the reference expression by expression (--fmad=false), so one step
// from identical gradients gives identical parameters. The activations of the snapshot
// (exp, sigmoid) use CUDA's exp (<= 1 ulp from glibc's), see DESIGN.md.
#include "sgm_internal.h"

namespace sgm {

namespace {

struct AdamSeg {
    double lr[5];  // center, radius, opacity, color (sem handled by k_adam_sem)
};

// update(), mapper.cpp:16-25, over center | log_radius | opacity_logit | color.
__global__ void k_adam(double* __restrict__ P, const double* __restrict__ G, double* __restrict__ M,
                       double* __restrict__ Vv, uint64_t n, uint64_t ns, AdamSeg seg, double b1,
                       double b2, double eps, double bc1, double bc2) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= 8 * ns) return;
    int s;
    uint64_t local;
    if (i < 3 * ns) {
        s = 0;
        local = i;
        if (local >= 3 * n) return;
    } else if (i < 4 * ns) {
        s = 1;
        local = i - 3 * ns;
        if (local >= n) return;
    } else if (i < 5 * ns) {
        s = 2;
        local = i - 4 * ns;
        if (local >= n) return;
    } else {
        s = 3;
        local = i - 5 * ns;
        if (local >= 3 * n) return;
    }
    const double g = G[i];
    const double m = b1 * M[i] + (1 - b1) * g;
    const double v = b2 * Vv[i] + (1 - b2) * g * g;
    M[i] = m;
    Vv[i] = v;
    const double mh = m / bc1;
    const double vh = v / bc2;
    P[i] -= seg.lr[s] * mh / (sqrt(vh) + eps);
}

// Semantic rows, mapper.cpp:32-50 + apply_semantic_step. One thread per Gaussian.
__global__ void k_adam_sem(double* __restrict__ probs, const double* __restrict__ G,
                           double* __restrict__ M, double* __restrict__ Vv, uint64_t n, int k,
                           double lr, double b1, double b2, double eps_sem, double bc1, double bc2) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint64_t base = i * k;
    double gbar = 0.0;
    for (int j = 0; j < k; ++j) gbar += G[base + j];
    gbar /= k;
    double total = 0.0;
    for (int j = 0; j < k; ++j) {
        const uint64_t idx = base + j;
        const double gj = G[idx] - gbar;
        const double m = b1 * M[idx] + (1 - b1) * gj;
        const double v = b2 * Vv[idx] + (1 - b2) * gj * gj;
        M[idx] = m;
        Vv[idx] = v;
        const double mh = m / bc1;
        const double vh = v / bc2;
        const double delta = -lr * mh / (sqrt(vh) + eps_sem);
        const double x = probs[idx] + delta;
        const double p = 0.0 < x ? x : 0.0;  // std::max(0.0, x)
        probs[idx] = p;
        total += p;
    }
    if (total <= 0.0) {
        for (int j = 0; j < k; ++j) probs[base + j] = 1.0 / k;
    } else {
        for (int j = 0; j < k; ++j) probs[base + j] /= total;
    }
}

// Render snapshot from master parameters: SoA geometry with the activations, clamped
// colour, class-sorted probabilities through the upload permutation.
__global__ void k_derive(const double* __restrict__ P, uint64_t n, uint64_t ns, int k, int kpad,
                         const uint16_t* __restrict__ perm, double* __restrict__ geo,
                         double* __restrict__ color4, double* __restrict__ sprob) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    geo[i] = P[3 * i];
    geo[ns + i] = P[3 * i + 1];
    geo[2 * ns + i] = P[3 * i + 2];
    geo[3 * ns + i] = exp(P[3 * ns + i]);                     // radius()
    geo[4 * ns + i] = 1.0 / (1.0 + exp(-P[4 * ns + i]));      // sigmoid, geometry.hpp:84
    for (int c = 0; c < 3; ++c) {
        const double v = P[5 * ns + 3 * i + c];
        color4[4 * i + c] = v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);  // std::clamp(v, 0, 1)
    }
    color4[4 * i + 3] = 0.0;
    const double* pr = P + 8 * ns + i * k;
    for (int q = 0; q < k; ++q) sprob[i * kpad + q] = pr[perm[i * kpad + q]];
}

__global__ void k_keep_flags(const double* __restrict__ logit, uint64_t n, double thr,
                             uint8_t* __restrict__ keep) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i < n) keep[i] = (1.0 / (1.0 + exp(-logit[i]))) >= thr;  // gaussian_map.cpp:102
}

// Gathers the kept rows of one [stride]-wide segment: dst[j*stride + s] = src[kept[j]*stride + s].
template <typename T>
__global__ void k_gather(const T* __restrict__ src, T* __restrict__ dst,
                         const uint32_t* __restrict__ kept, uint64_t m, int stride) {
    const uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (e >= m * stride) return;
    const uint64_t j = e / stride;
    const int s = static_cast<int>(e - j * stride);
    dst[e] = src[static_cast<uint64_t>(kept[j]) * stride + s];
}

inline unsigned nblk(uint64_t n) { return static_cast<unsigned>((n + 255) / 256); }

}  // namespace

void launch_adam(double* P, const double* G, double* M, double* V, uint64_t n, int k,
                 const AdamHyper& h, double bc1, double bc2, cudaStream_t s) {
    if (n == 0) return;
    const uint64_t ns = n;
    AdamSeg seg{{h.lr_center, h.lr_radius, h.lr_opacity, h.lr_color, 0.0}};
    k_adam<<<nblk(8 * ns), 256, 0, s>>>(P, G, M, V, n, ns, seg, h.beta1, h.beta2, h.eps, bc1, bc2);
    k_adam_sem<<<static_cast<unsigned>((n + 127) / 128), 128, 0, s>>>(
        P + 8 * ns, G + 8 * ns, M + 8 * ns, V + 8 * ns, n, k, h.lr_sem, h.beta1, h.beta2, h.eps_sem,
        bc1, bc2);
}

void launch_derive(const double* P, uint64_t n, int k, int kpad, const uint16_t* perm, double* geo,
                   double* color4, double* sprob, cudaStream_t s) {
    if (n == 0) return;
    k_derive<<<nblk(n), 256, 0, s>>>(P, n, n, k, kpad, perm, geo, color4, sprob);
}

void launch_keep_flags(const double* logit, uint64_t n, double thr, uint8_t* keep, cudaStream_t s) {
    if (n) k_keep_flags<<<nblk(n), 256, 0, s>>>(logit, n, thr, keep);
}

void launch_gather_f64(const double* src, double* dst, const uint32_t* kept, uint64_t m, int stride,
                       cudaStream_t s) {
    if (m && stride) k_gather<double><<<nblk(m * stride), 256, 0, s>>>(src, dst, kept, m, stride);
}

void launch_gather_u16(const uint16_t* src, uint16_t* dst, const uint32_t* kept, uint64_t m,
                       int stride, cudaStream_t s) {
    if (m && stride) k_gather<uint16_t><<<nblk(m * stride), 256, 0, s>>>(src, dst, kept, m, stride);
}

}  // namespace sgm
