// Drop-in for proj/include/lorbpano/lorb.hpp: L-ORB extraction with the same
// PODs, signatures and exceptions; FAST, Harris, NMS, top-N, BRIEF and the
// fused extract_features run on the B200 through the C-ABI. Overlap regions
// and the BRIEF pattern are host setup.
#ifndef LORBPANO_LORB_HPP
#define LORBPANO_LORB_HPP

#include <algorithm>
#include <array>
#include <cassert>
#include <cmath>
#include <cstdint>
#include <random>
#include <utility>
#include <vector>

#include "lorbpano/b200_runtime.hpp"
#include "lorbpano/image.hpp"
#include "lorbpano/imgops.hpp"

namespace lorbpano {

struct Keypoint {
    int x = 0;
    int y = 0;
    float response = 0.0f;
    int region_id = 0;
};

/// Half-open rectangle [x0,x1) x [y0,y1) on one camera (lorb.hpp:24-32).
struct DetectionRegion {
    int x0 = 0, y0 = 0, x1 = 0, y1 = 0;
    int camera_id = 0;

    int width() const { return x1 - x0; }
    int height() const { return y1 - y0; }
    bool contains(int x, int y) const { return x >= x0 && x < x1 && y >= y0 && y < y1; }
};

struct BriefPattern {
    struct Pair {
        int px, py, qx, qy;
    };
    std::vector<Pair> pairs;
    int patch_half = 15;
    std::uint64_t seed = 0;
};

/// Ternary code in two bitplanes (lorb.hpp:43-69): trit +1 <-> gt bit, -1 <-> lt bit.
struct Descriptor {
    static constexpr int kMaxWords = 8;

    int n_d = 0;
    std::array<std::uint64_t, kMaxWords> gt{};
    std::array<std::uint64_t, kMaxWords> lt{};

    static int words(int n_d) { return (n_d + 63) / 64; }

    explicit Descriptor(int nd = 0) : n_d(nd) { assert(nd <= kMaxWords * 64); }

    void set_trit(int i, int value) {
        const std::uint64_t bit = std::uint64_t{1} << (i % 64);
        if (value > 0) gt[i / 64] |= bit;
        else if (value < 0) lt[i / 64] |= bit;
    }
    int trit(int i) const {
        const std::uint64_t bit = std::uint64_t{1} << (i % 64);
        return (gt[i / 64] & bit) ? 1 : ((lt[i / 64] & bit) ? -1 : 0);
    }
};

struct ExtractionConfig {
    std::uint8_t fast_threshold = 20;
    int fast_arc = 9;
    float harris_alpha = 0.04f;
    float harris_threshold = 0.0f;
    float harris_sigma = 1.0f;
    int top_n = 500;
    int n_d = 256;
    float brief_blur_sigma = 2.0f;
    int patch_half = 15;

    void validate() const {  // lorb.hpp:82-89
        if (fast_arc < 9 || fast_arc > 16) throw BadParams("fast_arc must be in [9,16]");
        if (top_n < 4) throw BadParams("top_n must be >= 4");
        if (n_d < 64 || n_d > 512) throw BadParams("n_d must be in [64,512]");
        if (!(harris_sigma > 0.0f)) throw InvalidSigma("harris_sigma must be > 0");
        if (!(brief_blur_sigma > 0.0f)) throw InvalidSigma("brief_blur_sigma must be > 0");
        if (patch_half < 1) throw BadParams("patch_half must be >= 1");
    }
};

struct CameraLayout {
    double overlap_fraction = 0.25;
    std::vector<DetectionRegion> explicit_regions;
};

static_assert(sizeof(Keypoint) == sizeof(lp_keypoint), "Keypoint layout");
static_assert(sizeof(DetectionRegion) == sizeof(lp_region), "DetectionRegion layout");
static_assert(sizeof(BriefPattern::Pair) == sizeof(lp_pair), "BriefPattern::Pair layout");

namespace b200 {
inline lp_region region(const DetectionRegion& r) { return lp_region{r.x0, r.y0, r.x1, r.y1, r.camera_id}; }
inline lp_extraction_config config(const ExtractionConfig& c) {
    return lp_extraction_config{c.fast_threshold, c.fast_arc, c.harris_alpha, c.harris_threshold,
                                c.harris_sigma, c.top_n, c.n_d, c.brief_blur_sigma, c.patch_half};
}
inline void pack(const Descriptor& d, std::uint64_t* out) {
    const int W = Descriptor::words(d.n_d);
    for (int i = 0; i < W; ++i) {
        out[i] = d.gt[i];
        out[W + i] = d.lt[i];
    }
}
inline Descriptor unpack(const std::uint64_t* in, int n_d) {
    Descriptor d(n_d);
    const int W = Descriptor::words(n_d);
    for (int i = 0; i < W; ++i) {
        d.gt[i] = in[i];
        d.lt[i] = in[W + i];
    }
    return d;
}
}  // namespace b200

/// lorb.hpp:100-138 (host setup: strip arithmetic)
inline std::vector<DetectionRegion> partition_regions(const CameraLayout& layout,
                                                      const std::vector<std::pair<int, int>>& dims,
                                                      int patch_half) {
    auto inset = [&](DetectionRegion r, const char* what) {
        r.x0 += patch_half;
        r.y0 += patch_half;
        r.x1 -= patch_half;
        r.y1 -= patch_half;
        if (r.x0 >= r.x1 || r.y0 >= r.y1) throw RegionTooSmall(what);
        return r;
    };
    std::vector<DetectionRegion> out;
    if (!layout.explicit_regions.empty()) {
        for (const auto& r : layout.explicit_regions)
            out.push_back(inset(r, "explicit region smaller than 2*patch_half"));
        return out;
    }
    const double f = layout.overlap_fraction;
    if (f <= 0.0) throw NoOverlap("overlap fraction must be > 0");
    if (f > 1.0) throw OverlapExceedsImage("overlap fraction must be <= 1");
    for (std::size_t i = 0; i + 1 < dims.size(); ++i) {
        const auto [wl, hl] = dims[i];
        const auto [wr, hr] = dims[i + 1];
        const auto l = inset({static_cast<int>(std::lround(wl * (1.0 - f))), 0, wl, hl, static_cast<int>(i)},
                             "overlap strip smaller than 2*patch_half");
        const auto r = inset({0, 0, static_cast<int>(std::lround(wr * f)), hr, static_cast<int>(i + 1)},
                             "overlap strip smaller than 2*patch_half");
        out.push_back(l);
        out.push_back(r);
    }
    return out;
}

/// Radius-3 Bresenham ring, clockwise from (0,-3) (lorb.hpp:140-159).
inline const std::array<std::pair<int, int>, 16>& fast_ring() {
    static const std::array<std::pair<int, int>, 16> ring = {
        {{0, -3}, {1, -3}, {2, -2}, {3, -1}, {3, 0}, {3, 1}, {2, 2}, {1, 3},
         {0, 3}, {-1, 3}, {-2, 2}, {-3, 1}, {-3, 0}, {-3, -1}, {-2, -2}, {-1, -3}}};
    return ring;
}

/// lorb.hpp:192-205 on the GPU (raster order)
inline std::vector<std::pair<int, int>> fast_corners(const ImageU8& img, const DetectionRegion& region,
                                                     std::uint8_t threshold, int arc) {
    const long long cap = std::max(1LL, static_cast<long long>(std::max(region.width(), 0)) *
                                            std::max(region.height(), 0));
    std::vector<std::pair<int, int>> out(static_cast<std::size_t>(std::min<long long>(cap, 1LL << 28)));
    int n = 0;
    b200::check(lp_fast_corners(b200::ctx(), img.data.data(), img.width, img.height, img.channels,
                                b200::region(region), threshold, arc, &out[0].first,
                                static_cast<int>(out.size()), &n));
    out.resize(n);
    return out;
}

/// lorb.hpp:209-250 on the GPU (FP64 window sums, float result)
inline std::vector<float> harris_response(const ImageU8& img, const std::vector<std::pair<int, int>>& points,
                                          float alpha, float sigma) {
    if (img.channels != 1) throw UnsupportedFormat("harris_response: grayscale input required");
    std::vector<float> out(points.size());
    if (points.empty()) return out;
    b200::check(lp_harris_response(b200::ctx(), img.data.data(), img.width, img.height, img.channels,
                                   &points[0].first, static_cast<int>(points.size()), alpha, sigma,
                                   out.data()));
    return out;
}

/// lorb.hpp:254-288 on the GPU (survivors keep input order)
inline std::vector<Keypoint> nms(const std::vector<Keypoint>& candidates, int radius = 1) {
    std::vector<Keypoint> out(candidates.size());
    int n = 0;
    if (candidates.empty()) return {};
    b200::check(lp_nms(b200::ctx(), reinterpret_cast<const lp_keypoint*>(candidates.data()),
                       static_cast<int>(candidates.size()), radius, reinterpret_cast<lp_keypoint*>(out.data()),
                       &n));
    out.resize(n);
    return out;
}

/// lorb.hpp:291-299 on the GPU: (response desc, y asc, x asc), at most n
inline std::vector<Keypoint> select_top_n(std::vector<Keypoint> points, int n) {
    if (n < 1) throw BadParams("select_top_n: n must be >= 1");
    std::vector<Keypoint> out(std::min<std::size_t>(points.size(), static_cast<std::size_t>(n)));
    int k = 0;
    if (points.empty()) return out;
    b200::check(lp_select_top_n(b200::ctx(), reinterpret_cast<const lp_keypoint*>(points.data()),
                                static_cast<int>(points.size()), n, reinterpret_cast<lp_keypoint*>(out.data()),
                                &k));
    out.resize(k);
    return out;
}

/// lorb.hpp:301-330 (host setup; libstdc++ mt19937_64 + glibc, like the reference)
inline BriefPattern brief_pattern(int n_d, int patch_half, std::uint64_t seed) {
    if (n_d < 1) throw BadParams("brief_pattern: n_d must be >= 1");
    BriefPattern pat;
    pat.patch_half = patch_half;
    pat.seed = seed;
    std::mt19937_64 gen(seed);
    const double sd = patch_half / 2.5;
    const double lo_den = static_cast<double>(gen.max()) + 2.0, hi_den = static_cast<double>(gen.max()) + 1.0;
    auto draw = [&] {
        for (;;) {
            const double u1 = (static_cast<double>(gen()) + 1.0) / lo_den;
            const double u2 = static_cast<double>(gen()) / hi_den;
            const int v = static_cast<int>(std::lround(std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2) * sd));
            if (v >= -patch_half && v <= patch_half) return v;
        }
    };
    pat.pairs.resize(n_d);
    for (auto& p : pat.pairs) {
        p.px = draw();
        p.py = draw();
        p.qx = draw();
        p.qy = draw();
    }
    return pat;
}

/// lorb.hpp:333-350 on the GPU
inline Descriptor brief_descriptor(const ImageF32& smoothed, const Keypoint& kp, const BriefPattern& pat) {
    const int n_d = static_cast<int>(pat.pairs.size());
    std::vector<std::uint64_t> d(2 * Descriptor::words(n_d));
    b200::check(lp_brief_descriptors(b200::ctx(), smoothed.data.data(), smoothed.width, smoothed.height,
                                     reinterpret_cast<const lp_keypoint*>(&kp), 1,
                                     reinterpret_cast<const lp_pair*>(pat.pairs.data()), n_d, pat.patch_half,
                                     d.data()));
    return b200::unpack(d.data(), n_d);
}

struct Feature {
    Keypoint keypoint;
    Descriptor descriptor;
};

namespace detail {

/// Region crop blurred on the GPU (lorb.hpp:357-382): values equal a
/// full-image blur wherever BRIEF samples them.
struct SmoothedCrop {
    ImageF32 img;
    int off_x = 0, off_y = 0;

    float at_global(int x, int y) const { return img.at(x - off_x, y - off_y); }
};

inline SmoothedCrop smoothed_crop(const ImageU8& img, const DetectionRegion& region, int patch_half, float sigma) {
    const int margin = patch_half + static_cast<int>(std::ceil(3.0f * sigma));
    const int cx0 = std::max(0, region.x0 - margin), cy0 = std::max(0, region.y0 - margin);
    const int cx1 = std::min(img.width, region.x1 + margin), cy1 = std::min(img.height, region.y1 + margin);
    ImageF32 crop(cx1 - cx0, cy1 - cy0, 1);
    for (int y = cy0; y < cy1; ++y)
        for (int x = cx0; x < cx1; ++x) crop.at(x - cx0, y - cy0) = img.at(x, y);
    return SmoothedCrop{gaussian_blur(crop, sigma), cx0, cy0};
}

}  // namespace detail

/// lorb.hpp:386-413 on the GPU: all regions in one launch sequence
inline std::vector<Feature> extract_features(const ImageU8& img, const std::vector<DetectionRegion>& regions,
                                             const ExtractionConfig& cfg, const BriefPattern& pat) {
    cfg.validate();
    if (regions.empty()) return {};
    std::vector<lp_region> rs;
    for (const auto& r : regions) rs.push_back(b200::region(r));
    const int cap = static_cast<int>(regions.size()) * cfg.top_n;
    const int W2 = 2 * Descriptor::words(cfg.n_d);
    std::vector<lp_keypoint> kps(cap);
    std::vector<std::uint64_t> desc(static_cast<std::size_t>(cap) * W2);
    int n = 0;
    const lp_extraction_config c = b200::config(cfg);
    b200::check(lp_extract_features(b200::ctx(), img.data.data(), img.width, img.height, img.channels, rs.data(),
                                    static_cast<int>(rs.size()), &c,
                                    reinterpret_cast<const lp_pair*>(pat.pairs.data()), kps.data(), desc.data(),
                                    cap, &n));
    std::vector<Feature> out;
    out.reserve(n);
    for (int i = 0; i < n; ++i)
        out.push_back(Feature{Keypoint{kps[i].x, kps[i].y, kps[i].response, kps[i].region_id},
                              b200::unpack(desc.data() + static_cast<std::size_t>(i) * W2, cfg.n_d)});
    return out;
}

}  // namespace lorbpano

#endif
