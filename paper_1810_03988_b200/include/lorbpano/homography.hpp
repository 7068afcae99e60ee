// Drop-in for proj/include/lorbpano/homography.hpp. The DLT and PROSAC run on
// the B200 (lp_dlt_homography, lp_prosac_homography: exact libstdc++ sampler,
// FP64 Jacobi SVD, warp-parallel scoring); the 3x3 algebra stays host code.
// No Eigen dependency.
#ifndef LORBPANO_HOMOGRAPHY_HPP
#define LORBPANO_HOMOGRAPHY_HPP

#include <array>
#include <cmath>
#include <cstdint>
#include <utility>
#include <vector>

#include "lorbpano/b200_runtime.hpp"
#include "lorbpano/error.hpp"

namespace lorbpano {

/// 3x3 projective transform normalised to h33 = 1 (homography.hpp:16-63).
struct Homography {
    std::array<double, 9> h = {1, 0, 0, 0, 1, 0, 0, 0, 1};

    static Homography identity() { return Homography{}; }
    static Homography translation(double tx, double ty) { return Homography{{1, 0, tx, 0, 1, ty, 0, 0, 1}}; }

    double det() const {
        return h[0] * (h[4] * h[8] - h[5] * h[7]) - h[1] * (h[3] * h[8] - h[5] * h[6]) +
               h[2] * (h[3] * h[7] - h[4] * h[6]);
    }

    std::pair<double, double> apply(double x, double y) const {
        const double w = h[6] * x + h[7] * y + h[8];
        return {(h[0] * x + h[1] * y + h[2]) / w, (h[3] * x + h[4] * y + h[5]) / w};
    }

    Homography inverse() const {
        const double d = det();
        if (std::abs(d) < 1e-12) throw SingularHomography("homography not invertible");
        const std::array<double, 9> adj = {h[4] * h[8] - h[5] * h[7], h[2] * h[7] - h[1] * h[8],
                                           h[1] * h[5] - h[2] * h[4], h[5] * h[6] - h[3] * h[8],
                                           h[0] * h[8] - h[2] * h[6], h[2] * h[3] - h[0] * h[5],
                                           h[3] * h[7] - h[4] * h[6], h[1] * h[6] - h[0] * h[7],
                                           h[0] * h[4] - h[1] * h[3]};
        Homography out;
        for (int i = 0; i < 9; ++i) out.h[i] = adj[i] / d;
        const double s = out.h[8];
        if (std::abs(s) > 1e-12)
            for (double& v : out.h) v /= s;
        return out;
    }

    /// this ∘ other (other first)
    Homography compose(const Homography& o) const {
        Homography out;
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
                double acc = 0;
                for (int k = 0; k < 3; ++k) acc += h[r * 3 + k] * o.h[k * 3 + c];
                out.h[r * 3 + c] = acc;
            }
        if (std::abs(out.h[8]) > 1e-12) {
            const double s = out.h[8];
            for (int i = 0; i < 8; ++i) out.h[i] /= s;
            out.h[8] /= out.h[8];
        }
        return out;
    }
};

struct Correspondence {
    double sx = 0, sy = 0;
    double dx = 0, dy = 0;
    float quality = 0.0f;
};
static_assert(sizeof(Correspondence) == sizeof(lp_corr), "Correspondence layout");
static_assert(sizeof(Homography) == sizeof(lp_homography), "Homography layout");

namespace detail {

struct Normalizer {
    double cx = 0, cy = 0, scale = 1;
    std::pair<double, double> apply(double x, double y) const { return {(x - cx) * scale, (y - cy) * scale}; }
};

/// homography.hpp:81-97
inline Normalizer hartley_normalizer(const std::vector<Correspondence>& pairs, bool src) {
    Normalizer n;
    for (const auto& p : pairs) {
        n.cx += src ? p.sx : p.dx;
        n.cy += src ? p.sy : p.dy;
    }
    n.cx /= pairs.size();
    n.cy /= pairs.size();
    double md = 0;
    for (const auto& p : pairs) {
        const double x = (src ? p.sx : p.dx) - n.cx, y = (src ? p.sy : p.dy) - n.cy;
        md += std::sqrt(x * x + y * y);
    }
    md /= pairs.size();
    n.scale = md > 1e-12 ? std::sqrt(2.0) / md : 1.0;
    return n;
}

/// homography.hpp:99-108
inline bool three_collinear(const std::vector<Correspondence>& p) {
    for (std::size_t i = 0; i < p.size(); ++i)
        for (std::size_t j = i + 1; j < p.size(); ++j)
            for (std::size_t k = j + 1; k < p.size(); ++k)
                if (std::abs((p[j].sx - p[i].sx) * (p[k].sy - p[i].sy) - (p[j].sy - p[i].sy) * (p[k].sx - p[i].sx)) <
                    1e-9)
                    return true;
    return false;
}

}  // namespace detail

/// homography.hpp:112-144 on the GPU
inline Homography dlt_homography(const std::vector<Correspondence>& pairs) {
    if (pairs.size() < 4) throw InsufficientMatches("dlt: need at least 4 pairs");
    Homography out;
    b200::check(lp_dlt_homography(b200::ctx(), reinterpret_cast<const lp_corr*>(pairs.data()),
                                  static_cast<int>(pairs.size()), reinterpret_cast<lp_homography*>(&out)));
    return out;
}

/// homography.hpp:146-152
inline double symmetric_transfer_error(const Homography& h, const Homography& h_inv, const Correspondence& c) {
    const auto [fx, fy] = h.apply(c.sx, c.sy);
    const auto [bx, by] = h_inv.apply(c.dx, c.dy);
    return std::hypot(fx - c.dx, fy - c.dy) + std::hypot(bx - c.sx, by - c.sy);
}

enum class SamplingMode { Prosac, Uniform };

struct ProsacConfig {
    double threshold_px = 3.0;
    int max_iter = 1000;
    double confidence = 0.99;
    std::uint64_t seed = 0;
    SamplingMode sampling = SamplingMode::Prosac;
    double t_total = 200000.0;
};

struct ProsacResult {
    Homography model;
    std::vector<bool> inlier_mask;
    int inlier_count = 0;
    int iterations = 0;
};

struct ProsacTrace {
    std::vector<int> pool_sizes;
    std::vector<std::array<int, 4>> samples;
};

/// homography.hpp:178-286 on the GPU (sampler replayed bit-exactly on device)
inline ProsacResult prosac_homography(const std::vector<Correspondence>& matches, const ProsacConfig& cfg,
                                      ProsacTrace* trace = nullptr) {
    const int n = static_cast<int>(matches.size());
    if (n < 4) throw InsufficientMatches("prosac: need at least 4 matches");
    lp_prosac_config c{cfg.threshold_px, cfg.max_iter, cfg.sampling == SamplingMode::Uniform ? 1 : 0,
                       cfg.confidence, cfg.seed, cfg.t_total};
    ProsacResult r;
    std::vector<std::uint8_t> mask(n);
    std::vector<int> pools, samples;
    if (trace) {
        pools.resize(std::max(cfg.max_iter, 1));
        samples.resize(4 * pools.size());
    }
    lp_homography model;
    const lp_status st = lp_prosac_homography(b200::ctx(), reinterpret_cast<const lp_corr*>(matches.data()), n, &c,
                                              &model, mask.data(), &r.inlier_count, &r.iterations,
                                              trace ? pools.data() : nullptr, trace ? samples.data() : nullptr);
    if (trace)
        for (int t = 0; t < r.iterations; ++t) {
            trace->pool_sizes.push_back(pools[t]);
            trace->samples.push_back({samples[4 * t], samples[4 * t + 1], samples[4 * t + 2], samples[4 * t + 3]});
        }
    b200::check(st);
    for (int i = 0; i < 9; ++i) r.model.h[i] = model.h[i];
    r.inlier_mask.assign(mask.begin(), mask.end());
    return r;
}

}  // namespace lorbpano

#endif
