// Drop-in for proj/include/lorbpano/compose.hpp: warp, linear seam masks,
// Laplacian build/collapse and the multi-band blend on the B200 through the
// C-ABI; the canvas geometry is host setup.
#ifndef LORBPANO_COMPOSE_HPP
#define LORBPANO_COMPOSE_HPP

#include <algorithm>
#include <cmath>
#include <limits>
#include <utility>
#include <vector>

#include "lorbpano/homography.hpp"
#include "lorbpano/image.hpp"
#include "lorbpano/imgops.hpp"

namespace lorbpano {

/// Canvas pixel (x,y) <-> reference-frame point (x+origin_x, y+origin_y) (compose.hpp:16-24).
struct Canvas {
    int width = 0;
    int height = 0;
    int origin_x = 0;
    int origin_y = 0;
    std::vector<std::pair<int, int>> offsets;
};

using BlendMask = ImageF32;

/// compose.hpp:30-68 (host geometry)
inline Canvas compute_canvas(const std::vector<std::pair<int, int>>& dims, const std::vector<Homography>& homs) {
    if (dims.empty() || dims.size() != homs.size()) throw BadParams("compute_canvas: dims/homographies size mismatch");
    double lo_x = std::numeric_limits<double>::max(), lo_y = lo_x;
    double hi_x = std::numeric_limits<double>::lowest(), hi_y = hi_x;
    Canvas cv;
    for (std::size_t i = 0; i < dims.size(); ++i) {
        if (std::abs(homs[i].det()) < 1e-9) throw SingularHomography("compute_canvas: singular homography");
        const double w = dims[i].first, h = dims[i].second;
        double cam_x = std::numeric_limits<double>::max(), cam_y = cam_x;
        for (const auto& [px, py] : {std::pair<double, double>{0, 0}, {w, 0}, {0, h}, {w, h}}) {
            const auto [x, y] = homs[i].apply(px, py);
            lo_x = std::min(lo_x, x);
            lo_y = std::min(lo_y, y);
            hi_x = std::max(hi_x, x);
            hi_y = std::max(hi_y, y);
            cam_x = std::min(cam_x, x);
            cam_y = std::min(cam_y, y);
        }
        cv.offsets.emplace_back(static_cast<int>(std::floor(cam_x)), static_cast<int>(std::floor(cam_y)));
    }
    cv.origin_x = static_cast<int>(std::floor(lo_x));
    cv.origin_y = static_cast<int>(std::floor(lo_y));
    cv.width = static_cast<int>(std::ceil(hi_x)) - cv.origin_x;
    cv.height = static_cast<int>(std::ceil(hi_y)) - cv.origin_y;
    for (auto& o : cv.offsets) {
        o.first -= cv.origin_x;
        o.second -= cv.origin_y;
    }
    return cv;
}

/// compose.hpp:70-95 on the GPU (FP64 inverse map, bilinear, coverage)
inline std::pair<ImageF32, ImageF32> warp_image(const ImageF32& img, const Homography& h, const Canvas& canvas) {
    ImageF32 out(canvas.width, canvas.height, img.channels, img.color_space);
    ImageF32 cov(canvas.width, canvas.height, 1);
    const lp_canvas cv{canvas.width, canvas.height, canvas.origin_x, canvas.origin_y};
    b200::check(lp_warp_image(b200::ctx(), img.data.data(), img.width, img.height, img.channels,
                              reinterpret_cast<const lp_homography*>(&h), &cv, out.data.data(), cov.data.data()));
    return {std::move(out), std::move(cov)};
}

/// compose.hpp:97-131 on the GPU
inline std::vector<BlendMask> linear_seam_mask(const std::vector<ImageF32>& coverages) {
    if (coverages.empty()) throw BadParams("linear_seam_mask: no coverage masks");
    const int w = coverages[0].width, h = coverages[0].height;
    for (const auto& c : coverages)
        if (c.width != w || c.height != h) throw MaskMismatch("linear_seam_mask: coverage dims differ");
    const std::size_t np = static_cast<std::size_t>(w) * h;
    std::vector<float> in(np * coverages.size()), out(in.size());
    for (std::size_t i = 0; i < coverages.size(); ++i) {
        if (coverages[i].channels != 1) throw MaskMismatch("linear_seam_mask: coverage must be single-channel");
        std::copy(coverages[i].data.begin(), coverages[i].data.end(), in.begin() + i * np);
    }
    b200::check(lp_linear_seam_mask(b200::ctx(), in.data(), static_cast<int>(coverages.size()), w, h, out.data()));
    std::vector<BlendMask> masks;
    for (std::size_t i = 0; i < coverages.size(); ++i) {
        BlendMask m(w, h, 1);
        std::copy(out.begin() + i * np, out.begin() + (i + 1) * np, m.data.begin());
        masks.push_back(std::move(m));
    }
    return masks;
}

/// compose.hpp:133-147 on the GPU
inline Pyramid build_laplacian(const ImageF32& img, int levels) {
    if (levels < 1) throw TooManyLevels("build_laplacian: levels must be >= 1");
    std::vector<float> flat(b200::pyramid_floats(img.width, img.height, img.channels, levels));
    b200::check(lp_build_laplacian(b200::ctx(), img.data.data(), img.width, img.height, img.channels, levels,
                                   flat.data()));
    return b200::unpack_pyramid(flat, img.width, img.height, img.channels, img.color_space, levels);
}

/// compose.hpp:149-158 on the GPU
inline ImageF32 collapse_laplacian(const Pyramid& p) {
    if (p.levels.empty()) throw TooManyLevels("collapse_laplacian: empty pyramid");
    const ImageF32& l0 = p.levels[0];
    const int L = static_cast<int>(p.levels.size());
    std::vector<float> flat;
    flat.reserve(b200::pyramid_floats(l0.width, l0.height, l0.channels, L));
    int w = l0.width, h = l0.height;
    for (int k = 0; k < L; ++k, w /= 2, h /= 2) {
        const ImageF32& lv = p.levels[k];
        // the reference upsamples each coarser level to the finer level's dims;
        // packed levels must follow the floor-halving chain
        if (lv.width != w || lv.height != h || lv.channels != l0.channels)
            throw BadTargetDims("collapse_laplacian: level dims must halve with floor");
        flat.insert(flat.end(), lv.data.begin(), lv.data.end());
    }
    ImageF32 out(l0.width, l0.height, l0.channels, l0.color_space);
    b200::check(lp_collapse_laplacian(b200::ctx(), flat.data(), l0.width, l0.height, l0.channels, L,
                                      out.data.data()));
    return out;
}

/// compose.hpp:160-215 on the GPU (windowed multi-band blend, exact order)
inline ImageU8 multiband_blend(const std::vector<ImageF32>& images, const std::vector<BlendMask>& masks, int levels) {
    if (images.empty() || images.size() != masks.size())
        throw MaskMismatch("multiband_blend: image/mask count mismatch");
    const int w = images[0].width, h = images[0].height, ch = images[0].channels;
    for (std::size_t i = 0; i < images.size(); ++i)
        if (images[i].width != w || images[i].height != h || images[i].channels != ch || masks[i].width != w ||
            masks[i].height != h)
            throw MaskMismatch("multiband_blend: raster dims differ");
    const std::size_t np = static_cast<std::size_t>(w) * h;
    std::vector<float> im(np * ch * images.size()), mk(np * images.size());
    for (std::size_t i = 0; i < images.size(); ++i) {
        std::copy(images[i].data.begin(), images[i].data.end(), im.begin() + i * np * ch);
        std::copy(masks[i].data.begin(), masks[i].data.begin() + np, mk.begin() + i * np);
    }
    ImageU8 out(w, h, ch, images[0].color_space);
    b200::check(lp_multiband_blend(b200::ctx(), im.data(), mk.data(), static_cast<int>(images.size()), w, h, ch,
                                   levels, out.data.data()));
    return out;
}

}  // namespace lorbpano

#endif
