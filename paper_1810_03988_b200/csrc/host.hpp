// host.hpp — host-only setup helpers of the hot path (no per-pixel work).
//
// These are the pieces SURVEY §8(b) keeps on the host because they are
// per-engine or per-frame setup, not stages: overlap regions, the BRIEF
// pattern, Gaussian taps and Harris window weights, LSH bit positions and the
// probe set, Homography algebra, the canvas, and the PROSAC termination table.
// They use the same libstdc++ <random> and glibc libm as the reference, so the
// constants handed to the kernels are bit-identical to the reference's.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <random>
#include <vector>

#include "common.cuh"

namespace lpb {
namespace host {

// partition_regions (fraction path), lorb.hpp:100-138
inline std::vector<lp_region> partition_regions(int ncams, const int* w, const int* h,
                                                double f, int ph) {
    if (f <= 0.0) throw Status(LP_NO_OVERLAP, "overlap fraction must be > 0");
    if (f > 1.0) throw Status(LP_OVERLAP_EXCEEDS_IMAGE, "overlap fraction must be <= 1");
    std::vector<lp_region> out;
    for (int i = 0; i + 1 < ncams; ++i) {
        lp_region left{static_cast<int>(std::lround(w[i] * (1.0 - f))), 0, w[i], h[i], i};
        lp_region right{0, 0, static_cast<int>(std::lround(w[i + 1] * f)), h[i + 1], i + 1};
        for (lp_region* r : {&left, &right}) {
            r->x0 += ph;
            r->y0 += ph;
            r->x1 -= ph;
            r->y1 -= ph;
            if (r->x0 >= r->x1 || r->y0 >= r->y1)
                throw Status(LP_REGION_TOO_SMALL, "overlap strip smaller than 2*patch_half");
        }
        out.push_back(left);
        out.push_back(right);
    }
    return out;
}

// brief_pattern, lorb.hpp:303-330: Box-Muller per coordinate, rejected into
// [-ph, ph], drawn px, py, qx, qy per pair from mt19937_64(seed).
inline std::vector<lp_pair> brief_pattern(int n_d, int ph, std::uint64_t seed) {
    if (n_d < 1) throw Status(LP_BAD_PARAMS, "brief_pattern: n_d must be >= 1");
    std::mt19937_64 rng(seed);
    const double sigma = ph / 2.5;
    auto coord = [&]() {
        for (;;) {
            double u1 = (static_cast<double>(rng()) + 1.0) / (static_cast<double>(rng.max()) + 2.0);
            double u2 = static_cast<double>(rng()) / (static_cast<double>(rng.max()) + 1.0);
            double g = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2) * sigma;
            int v = static_cast<int>(std::lround(g));
            if (v >= -ph && v <= ph) return v;
        }
    };
    std::vector<lp_pair> pat(n_d);
    for (auto& p : pat) {
        p.px = coord();
        p.py = coord();
        p.qx = coord();
        p.qy = coord();
    }
    return pat;
}

// gaussian_kernel, imgops.hpp:35-47 (float taps; float overloads of exp/ceil)
inline std::vector<float> gaussian_kernel(float sigma) {
    if (!(sigma > 0.0f)) throw Status(LP_INVALID_SIGMA, "gaussian kernel: sigma must be > 0");
    const int radius = static_cast<int>(std::ceil(3.0f * sigma));
    std::vector<float> k(2 * radius + 1);
    float sum = 0.0f;
    for (int i = -radius; i <= radius; ++i) {
        float v = std::exp(-(static_cast<float>(i) * i) / (2.0f * sigma * sigma));
        k[i + radius] = v;
        sum += v;
    }
    for (float& v : k) v /= sum;
    return k;
}

// harris_response window weights, lorb.hpp:213-227 (FP64, normalised)
inline std::vector<double> harris_weights(float sigma, int* radius_out) {
    const int radius = static_cast<int>(std::ceil(3.0f * sigma));
    const double s2 = 2.0 * static_cast<double>(sigma) * sigma;
    std::vector<double> w((2 * radius + 1) * (2 * radius + 1));
    double sum = 0.0;
    for (int v = -radius; v <= radius; ++v)
        for (int u = -radius; u <= radius; ++u) {
            double g = std::exp(-(u * u + v * v) / s2);
            w[(v + radius) * (2 * radius + 1) + (u + radius)] = g;
            sum += g;
        }
    for (double& x : w) x /= sum;
    *radius_out = radius;
    return w;
}

// LshIndex bit sampling, matchlsh.hpp:44-59
inline std::vector<int> lsh_bit_positions(int n_d, int tables, int bits, std::uint64_t seed) {
    if (tables < 1) throw Status(LP_BAD_PARAMS, "build_index: L must be >= 1");
    if (bits < 1 || (n_d > 0 && bits > 2 * n_d))
        throw Status(LP_BAD_PARAMS, "build_index: k must be in [1, 2*n_d]");
    std::mt19937_64 rng(seed);
    std::vector<int> out;
    const int domain = n_d > 0 ? 2 * n_d : bits;
    for (int t = 0; t < tables; ++t) {
        std::vector<int> positions(domain);
        std::iota(positions.begin(), positions.end(), 0);
        for (int i = 0; i < bits; ++i) {
            std::uniform_int_distribution<int> pick(i, domain - 1);
            std::swap(positions[i], positions[pick(rng)]);
        }
        out.insert(out.end(), positions.begin(), positions.begin() + bits);
    }
    return out;
}

// probe_sequence, matchlsh.hpp:104-128
inline std::vector<std::uint64_t> probe_sequence(int k, int t) {
    if (t < 1) throw Status(LP_BAD_PARAMS, "probe_sequence: t_probes must be >= 1");
    if (k < 1 || k >= 63) throw Status(LP_BAD_PARAMS, "probe_sequence: k must be in [1,62]");
    if (static_cast<std::uint64_t>(t) > (std::uint64_t{1} << k))
        throw Status(LP_TOO_MANY_PROBES, "probe_sequence: t_probes exceeds 2^k");
    std::vector<std::uint64_t> masks{0};
    for (int card = 1; static_cast<int>(masks.size()) < t && card <= k; ++card) {
        std::vector<int> idx(card);
        std::iota(idx.begin(), idx.end(), 0);
        for (;;) {
            std::uint64_t m = 0;
            for (int i : idx) m |= std::uint64_t{1} << i;
            masks.push_back(m);
            if (static_cast<int>(masks.size()) >= t) break;
            int i = card - 1;
            while (i >= 0 && idx[i] == k - card + i) --i;
            if (i < 0) break;
            ++idx[i];
            for (int j = i + 1; j < card; ++j) idx[j] = idx[j - 1] + 1;
        }
    }
    return masks;
}

// The probe set as a membership predicate for the device matcher: every mask
// of popcount <= full_card is present, plus an explicit list of the masks of
// popcount full_card+1 that the sequence reached.
struct ProbeSet {
    int full_card = -1;
    std::vector<std::uint64_t> partial;
};
inline ProbeSet probe_set(int k, int t) {
    auto masks = probe_sequence(k, t);
    ProbeSet ps;
    std::vector<std::uint64_t> count_by_card(k + 2, 0);
    for (auto m : masks) count_by_card[__builtin_popcountll(m)]++;
    // binomial(k, c) masks of cardinality c exist
    auto binom = [](int n, int r) {
        double v = 1;
        for (int i = 1; i <= r; ++i) v = v * (n - r + i) / i;
        return static_cast<std::uint64_t>(v + 0.5);
    };
    int c = 0;
    while (c <= k && count_by_card[c] == binom(k, c)) ++c;
    ps.full_card = c - 1;
    for (auto m : masks)
        if (__builtin_popcountll(m) > ps.full_card) ps.partial.push_back(m);
    return ps;
}

// Homography algebra, homography.hpp:25-62
inline double h_det(const double* h) {
    return h[0] * (h[4] * h[8] - h[5] * h[7]) - h[1] * (h[3] * h[8] - h[5] * h[6]) +
           h[2] * (h[3] * h[7] - h[4] * h[6]);
}
inline void h_apply(const double* h, double x, double y, double* ox, double* oy) {
    double w = h[6] * x + h[7] * y + h[8];
    *ox = (h[0] * x + h[1] * y + h[2]) / w;
    *oy = (h[3] * x + h[4] * y + h[5]) / w;
}
inline void h_inverse(const double* h, double* out) {
    double d = h_det(h);
    if (std::abs(d) < 1e-12) throw Status(LP_SINGULAR_HOMOGRAPHY, "homography not invertible");
    double inv[9] = {(h[4] * h[8] - h[5] * h[7]) / d, (h[2] * h[7] - h[1] * h[8]) / d,
                     (h[1] * h[5] - h[2] * h[4]) / d, (h[5] * h[6] - h[3] * h[8]) / d,
                     (h[0] * h[8] - h[2] * h[6]) / d, (h[2] * h[3] - h[0] * h[5]) / d,
                     (h[3] * h[7] - h[4] * h[6]) / d, (h[1] * h[6] - h[0] * h[7]) / d,
                     (h[0] * h[4] - h[1] * h[3]) / d};
    std::memcpy(out, inv, sizeof inv);
    if (std::abs(out[8]) > 1e-12)
        for (int i = 0; i < 9; ++i) out[i] /= inv[8];
}
inline void h_compose(const double* a, const double* b, double* out) {
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            double s = 0;
            for (int k = 0; k < 3; ++k) s += a[r * 3 + k] * b[k * 3 + c];
            out[r * 3 + c] = s;
        }
    if (std::abs(out[8]) > 1e-12) {
        const double d8 = out[8];
        for (int i = 0; i < 8; ++i) out[i] /= d8;
        out[8] /= out[8];
    }
}

// compute_canvas, compose.hpp:32-68 (offsets returned separately)
inline lp_canvas compute_canvas(int n, const int* w, const int* h, const lp_homography* hs) {
    if (n < 1) throw Status(LP_BAD_PARAMS, "compute_canvas: dims/homographies size mismatch");
    double minx = std::numeric_limits<double>::max(), miny = minx;
    double maxx = std::numeric_limits<double>::lowest(), maxy = maxx;
    for (int i = 0; i < n; ++i) {
        if (std::abs(h_det(hs[i].h)) < 1e-9)
            throw Status(LP_SINGULAR_HOMOGRAPHY, "compute_canvas: singular homography");
        const double cs[4][2] = {{0, 0}, {static_cast<double>(w[i]), 0},
                                 {0, static_cast<double>(h[i])},
                                 {static_cast<double>(w[i]), static_cast<double>(h[i])}};
        for (auto& c : cs) {
            double x, y;
            h_apply(hs[i].h, c[0], c[1], &x, &y);
            minx = std::min(minx, x);
            miny = std::min(miny, y);
            maxx = std::max(maxx, x);
            maxy = std::max(maxy, y);
        }
    }
    lp_canvas cv;
    cv.origin_x = static_cast<int>(std::floor(minx));
    cv.origin_y = static_cast<int>(std::floor(miny));
    cv.width = static_cast<int>(std::ceil(maxx)) - cv.origin_x;
    cv.height = static_cast<int>(std::ceil(maxy)) - cv.origin_y;
    return cv;
}

// PROSAC termination test, homography.hpp:255-261, tabulated with glibc
// pow/log for every (n_total, inlier_count): tab[n*(nmax+1)+c] = the first
// iteration t at which the reference would stop with c inliers out of n
// (max_iter + 1 = never). Depends only on confidence and max_iter.
inline std::vector<int> prosac_exit_table(int nmax, int max_iter, double confidence) {
    std::vector<int> tab(static_cast<size_t>(nmax + 1) * (nmax + 1), max_iter + 1);
    const double rhs = std::log(1.0 - confidence);
    for (int n = 4; n <= nmax; ++n)
        for (int c = 4; c <= n; ++c) {
            double w = static_cast<double>(c) / n;
            double p_fail = 1.0 - std::pow(w, 4);
            int t_exit = max_iter + 1;
            if (p_fail < 1e-12) {
                t_exit = 1;
            } else {
                const double l = std::log(p_fail);
                // (double)t * l is non-increasing in t; find the first t with t*l <= rhs
                double guess = std::ceil(rhs / l);
                long long t0 = guess < 1 ? 1 : (guess > max_iter + 2 ? max_iter + 2 : static_cast<long long>(guess));
                while (t0 > 1 && static_cast<double>(t0 - 1) * l <= rhs) --t0;
                while (t0 <= max_iter && !(static_cast<double>(t0) * l <= rhs)) ++t0;
                t_exit = t0 <= max_iter ? static_cast<int>(t0) : max_iter + 1;
            }
            tab[static_cast<size_t>(n) * (nmax + 1) + c] = t_exit;
        }
    return tab;
}

}  // namespace host
}  // namespace lpb
