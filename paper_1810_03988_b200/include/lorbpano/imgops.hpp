// Drop-in for proj/include/lorbpano/imgops.hpp: same API; the per-pixel
// operators (gaussian_blur, downsample, upsample, gaussian_pyramid) run on
// the B200 through the C-ABI. to_grayscale and gradients (test utilities, off
// the stitching path) stay host code.
#ifndef LORBPANO_IMGOPS_HPP
#define LORBPANO_IMGOPS_HPP

#include <cmath>
#include <vector>

#include "lorbpano/b200_runtime.hpp"
#include "lorbpano/image.hpp"

namespace lorbpano {

/// Central-difference gradients (imgops.hpp:11-15).
struct GradientPair {
    ImageF32 ix;
    ImageF32 iy;
};

/// Level 0 is full resolution; dims halve with floor (imgops.hpp:17-20).
struct Pyramid {
    std::vector<ImageF32> levels;
};

/// imgops.hpp:22-33 (host; rgb -> luma with the reference's float weights)
inline ImageU8 to_grayscale(const ImageU8& img) {
    if (img.channels == 1) return img;
    if (img.channels != 3) throw UnsupportedFormat("to_grayscale: channels must be 1 or 3");
    ImageU8 g(img.width, img.height, 1, ColorSpace::Gray);
    const std::size_t n = static_cast<std::size_t>(img.width) * img.height;
    for (std::size_t i = 0; i < n; ++i) {
        const std::uint8_t* p = &img.data[3 * i];
        g.data[i] = to_u8(0.299f * p[0] + 0.587f * p[1] + 0.114f * p[2]);
    }
    return g;
}

/// imgops.hpp:35-47 (host constant: float taps normalised by their float sum)
inline std::vector<float> gaussian_kernel(float sigma) {
    if (!(sigma > 0.0f)) throw InvalidSigma("gaussian kernel: sigma must be > 0");
    const int r = static_cast<int>(std::ceil(3.0f * sigma));
    std::vector<float> taps(2 * r + 1);
    float total = 0.0f;
    for (int i = -r; i <= r; ++i) {
        taps[i + r] = std::exp(-(static_cast<float>(i) * i) / (2.0f * sigma * sigma));
        total += taps[i + r];
    }
    for (float& t : taps) t /= total;
    return taps;
}

/// imgops.hpp:50-72 on the GPU (separable, clamp-to-edge, exact FP32 order)
inline ImageF32 gaussian_blur(const ImageF32& img, float sigma) {
    ImageF32 out(img.width, img.height, img.channels, img.color_space);
    b200::check(lp_gaussian_blur(b200::ctx(), img.data.data(), img.width, img.height, img.channels,
                                 sigma, out.data.data()));
    return out;
}

inline ImageF32 gaussian_blur(const ImageU8& img, float sigma) { return gaussian_blur(to_f32(img), sigma); }

/// imgops.hpp:78-103 (host test utility)
template <typename T>
inline GradientPair gradients(const Raster<T>& img) {
    if (img.channels != 1) throw UnsupportedFormat("gradients: grayscale input required");
    if (img.width < 3 || img.height < 3) throw ImageTooSmall("gradients: need at least 3x3");
    const int W = img.width, H = img.height;
    GradientPair g{ImageF32(W, H, 1), ImageF32(W, H, 1)};
    auto v = [&](int x, int y) { return static_cast<float>(img.at(x, y)); };
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            g.ix.at(x, y) = x == 0 ? v(1, y) - v(0, y)
                          : x == W - 1 ? v(x, y) - v(x - 1, y)
                                       : (v(x + 1, y) - v(x - 1, y)) / 2.0f;
            g.iy.at(x, y) = y == 0 ? v(x, 1) - v(x, 0)
                          : y == H - 1 ? v(x, y) - v(x, y - 1)
                                       : (v(x, y + 1) - v(x, y - 1)) / 2.0f;
        }
    return g;
}

/// imgops.hpp:106-116 on the GPU
inline ImageF32 downsample(const ImageF32& img) {
    if (img.width < 2 || img.height < 2) throw ImageTooSmall("downsample: need at least 2x2");
    ImageF32 out(img.width / 2, img.height / 2, img.channels, img.color_space);
    b200::check(lp_downsample(b200::ctx(), img.data.data(), img.width, img.height, img.channels,
                              out.data.data()));
    return out;
}

/// imgops.hpp:119-140 on the GPU (align-corners bilinear)
inline ImageF32 upsample(const ImageF32& img, int target_w, int target_h) {
    if (std::abs(target_w - 2 * img.width) > 1 || std::abs(target_h - 2 * img.height) > 1)
        throw BadTargetDims("upsample: target dims must be ~2x source");
    ImageF32 out(target_w, target_h, img.channels, img.color_space);
    b200::check(lp_upsample(b200::ctx(), img.data.data(), img.width, img.height, img.channels,
                            target_w, target_h, out.data.data()));
    return out;
}

namespace b200 {
// packed level-0-first buffer <-> Pyramid
inline std::size_t pyramid_floats(int w, int h, int ch, int levels) {
    std::size_t n = 0;
    for (int k = 0; k < levels; ++k, w /= 2, h /= 2) n += static_cast<std::size_t>(w) * h * ch;
    return n;
}
inline Pyramid unpack_pyramid(const std::vector<float>& flat, int w, int h, int ch, ColorSpace cs, int levels) {
    Pyramid p;
    std::size_t off = 0;
    for (int k = 0; k < levels; ++k, w /= 2, h /= 2) {
        ImageF32 lv(w, h, ch, cs);
        std::copy(flat.begin() + off, flat.begin() + off + lv.data.size(), lv.data.begin());
        off += lv.data.size();
        p.levels.push_back(std::move(lv));
    }
    return p;
}
}  // namespace b200

/// imgops.hpp:142-153 on the GPU
inline Pyramid gaussian_pyramid(const ImageF32& img, int levels) {
    if (levels < 1) throw TooManyLevels("pyramid: levels must be >= 1");
    std::vector<float> flat(b200::pyramid_floats(img.width, img.height, img.channels, levels));
    b200::check(lp_gaussian_pyramid(b200::ctx(), img.data.data(), img.width, img.height, img.channels,
                                    levels, flat.data()));
    return b200::unpack_pyramid(flat, img.width, img.height, img.channels, img.color_space, levels);
}

}  // namespace lorbpano

#endif
