// Host-side pieces of the C ABI that stay on the CPU by design:
// combine_scores and its softmaxes, look_at/camera_pose, clipped_entropy.
// These are O(#views) fp64 scalar code; they are restated here (not linked from
// the reference) with the reference's exact evaluation order so results are
// bit-identical. Built with -ffp-contract=off.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <vector>

#include "../../include/sgm.h"

namespace {

// stable_softmax, proj/src/explorer.cpp:209-222.
std::vector<double> stable_softmax(const std::vector<double>& v) {
    std::vector<double> out(v.size(), 0.0);
    double mx = -std::numeric_limits<double>::infinity();
    for (double x : v)
        if (std::isfinite(x)) mx = std::max(mx, x);
    if (!std::isfinite(mx)) return out;
    double sum = 0.0;
    for (size_t i = 0; i < v.size(); ++i) {
        out[i] = std::isfinite(v[i]) ? std::exp(v[i] - mx) : 0.0;
        sum += out[i];
    }
    for (auto& x : out) x /= sum;
    return out;
}

// Eigen 3.3+ redux order for 3-vectors: x0 + (x1 + x2).
inline double sqnorm3(const double v[3]) { return v[0] * v[0] + (v[1] * v[1] + v[2] * v[2]); }

inline void normalize3(double v[3]) {
    const double z = sqnorm3(v);
    if (z > 0.0) {
        const double s = std::sqrt(z);
        v[0] /= s;
        v[1] /= s;
        v[2] /= s;
    }
}

inline void cross3(const double a[3], const double b[3], double o[3]) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}

}  // namespace

extern "C" {

// clipped_entropy, proj/src/splat_render.cpp:360-369.
double sgm_clipped_entropy(const double* probs, uint64_t n) {
    auto clampd = [](double v) { return v < 0.001 ? 0.001 : (1.0 < v ? 1.0 : v); };
    double total = 0.0;
    for (uint64_t i = 0; i < n; ++i) total += clampd(probs[i]);
    double h = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        const double q = clampd(probs[i]) / total;
        h -= q * std::log(q);
    }
    return h;
}

// combine_scores, proj/src/explorer.cpp:225-248.
int sgm_combine_scores(uint64_t n, const double* n_missing, const double* entropy_sum,
                       const double* positions3, const double current[3], double* i_geo,
                       double* i_sem, double* i_total) {
    if (n == 0) return 0;
    if (!n_missing || !entropy_sum || !positions3 || !current || !i_geo || !i_sem || !i_total)
        return -1;
    std::vector<double> log_missing(n), entropy(n), dist(n);
    for (uint64_t i = 0; i < n; ++i) {
        log_missing[i] = n_missing[i] > 0.0 ? std::log(n_missing[i])
                                            : -std::numeric_limits<double>::infinity();
        entropy[i] = entropy_sum[i];
        const double d[3] = {positions3[3 * i] - current[0], positions3[3 * i + 1] - current[1],
                             positions3[3 * i + 2] - current[2]};
        dist[i] = std::sqrt(sqnorm3(d));  // (position - current).norm()
    }
    const std::vector<double> geo = stable_softmax(log_missing);
    const std::vector<double> sem = stable_softmax(entropy);
    const std::vector<double> dist_soft = stable_softmax(dist);
    int any = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const double dist_factor = n == 1 ? 1.0 : 1.0 - dist_soft[i];
        i_geo[i] = geo[i];
        i_sem[i] = sem[i];
        i_total[i] = dist_factor * geo[i] * sem[i];
        if (i_total[i] > 0.0) any = 1;
    }
    return any;
}

// The combined scalar gain of the Fisher extension (no reference counterpart):
//   gain_v   = fisher_gain_v + w_sem * entropy_sum_v
//   i_gain_v = softmax(ln gain_v)                      (as Eq. 6 treats the missing count)
//   i_total  = (n == 1 ? 1 : 1 - softmax(dist)_v) * i_gain_v          (Eq. 8's motion cost)
// with the reference's stable_softmax and distance (explorer.cpp:209-248). gain_v <= 0 (or
// not finite) takes no share. Returns 1 if some i_total > 0, 0 if none (or n == 0), -1 on
// invalid arguments.
int sgm_combine_scores_fisher(uint64_t n, const double* fisher_gain, const double* entropy_sum,
                              const double* positions3, const double current[3], double w_sem,
                              double* gain, double* i_total) {
    if (n == 0) return 0;
    if (!fisher_gain || !entropy_sum || !positions3 || !current || !gain || !i_total) return -1;
    if (!std::isfinite(w_sem) || w_sem < 0.0) return -1;
    std::vector<double> log_gain(n), dist(n);
    for (uint64_t i = 0; i < n; ++i) {
        gain[i] = fisher_gain[i] + w_sem * entropy_sum[i];
        log_gain[i] = gain[i] > 0.0 ? std::log(gain[i]) : -std::numeric_limits<double>::infinity();
        const double d[3] = {positions3[3 * i] - current[0], positions3[3 * i + 1] - current[1],
                             positions3[3 * i + 2] - current[2]};
        dist[i] = std::sqrt(sqnorm3(d));
    }
    const std::vector<double> share = stable_softmax(log_gain);
    const std::vector<double> dist_soft = stable_softmax(dist);
    int any = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const double dist_factor = n == 1 ? 1.0 : 1.0 - dist_soft[i];
        i_total[i] = dist_factor * share[i];
        if (i_total[i] > 0.0) any = 1;
    }
    return any;
}

// look_at, proj/include/splatmap/geometry.hpp:44-56 (up = +Y).
void sgm_look_at(const double position[3], const double target[3], sgm_pose* out) {
    static const double up[3] = {0.0, 1.0, 0.0};
    static const double ux[3] = {1.0, 0.0, 0.0};
    double z[3] = {target[0] - position[0], target[1] - position[1], target[2] - position[2]};
    normalize3(z);
    double x[3], y[3];
    cross3(z, up, x);
    if (std::sqrt(sqnorm3(x)) < 1e-9) cross3(z, ux, x);
    normalize3(x);
    cross3(z, x, y);
    for (int i = 0; i < 3; ++i) {
        out->R[3 * i + 0] = x[i];
        out->R[3 * i + 1] = y[i];
        out->R[3 * i + 2] = z[i];
        out->t[i] = position[i];
    }
}

// CandidatePose::camera_pose(), proj/include/splatmap/explorer.hpp:105.
void sgm_candidate_pose(const double position[3], const double direction[3], sgm_pose* out) {
    const double target[3] = {position[0] + direction[0], position[1] + direction[1],
                              position[2] + direction[2]};
    sgm_look_at(position, target, out);
}

// fibonacci_directions, proj/src/explorer.cpp:142-155 (libm sin/cos/sqrt, as the reference).
void sgm_fibonacci_directions(int32_t count, double max_elevation_deg, double* out3) {
    if (count <= 0 || !out3) return;
    const double golden_angle = M_PI * (3.0 - std::sqrt(5.0));
    const double s_max = std::sin(max_elevation_deg * M_PI / 180.0);  // deg_to_rad, geometry.hpp:86
    for (int j = 0; j < count; ++j) {
        const double s = count == 1 ? 0.0 : s_max * (1.0 - (2.0 * j + 1.0) / count);
        const double r = std::sqrt(std::max(0.0, 1.0 - s * s));
        const double az = golden_angle * j;
        out3[3 * j + 0] = r * std::cos(az);
        out3[3 * j + 1] = s;
        out3[3 * j + 2] = r * std::sin(az);
    }
}

}  // extern "C"
