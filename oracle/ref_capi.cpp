// oracle/ref_capi.cpp — TEST INFRASTRUCTURE ONLY (never shipped, never on the
// product path). Compiles the UNMODIFIED reference headers in place
// (/root/reference/proj/include/lorbpano/*.hpp, via -I) against the oracle
// shims (shim/png.h, shim/Eigen/Dense) and exposes them through ref_* entry
// points whose signatures mirror include/lorbpano_b200.h (minus the context),
// so tests can run the reference itself, the C restatement (lorb_oracle.c) and
// the CUDA path on identical inputs. Built by oracle/Makefile into
// oracle/_ref/liblorbref.so with the reference's Release flags
// (-O3 -DNDEBUG, no -march; -ffp-contract=off pins FP32 bits).
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "lorbpano/cli.hpp"
#include "lorbpano/compose.hpp"
#include "lorbpano/homography.hpp"
#include "lorbpano/lorb.hpp"
#include "lorbpano/matchlsh.hpp"
#include "lorbpano/pipeline.hpp"
#include "lorbpano/synth.hpp"
#include "lorbpano_b200.h"

using namespace lorbpano;

namespace {

thread_local std::string g_err;

int code_of(const std::exception& e) {
#define LP_MAP(T, C) \
    if (dynamic_cast<const T*>(&e)) return C;
    LP_MAP(FileNotFound, LP_FILE_NOT_FOUND)
    LP_MAP(UnsupportedFormat, LP_UNSUPPORTED_FORMAT)
    LP_MAP(CorruptData, LP_CORRUPT_DATA)
    LP_MAP(InvalidSigma, LP_INVALID_SIGMA)
    LP_MAP(ImageTooSmall, LP_IMAGE_TOO_SMALL)
    LP_MAP(BadTargetDims, LP_BAD_TARGET_DIMS)
    LP_MAP(NoOverlap, LP_NO_OVERLAP)
    LP_MAP(OverlapExceedsImage, LP_OVERLAP_EXCEEDS_IMAGE)
    LP_MAP(RegionTooSmall, LP_REGION_TOO_SMALL)
    LP_MAP(WindowOutOfBounds, LP_WINDOW_OUT_OF_BOUNDS)
    LP_MAP(PatchOutOfBounds, LP_PATCH_OUT_OF_BOUNDS)
    LP_MAP(LengthMismatch, LP_LENGTH_MISMATCH)
    LP_MAP(BadParams, LP_BAD_PARAMS)
    LP_MAP(TooManyProbes, LP_TOO_MANY_PROBES)
    LP_MAP(ParamMismatch, LP_PARAM_MISMATCH)
    LP_MAP(EmptyInput, LP_EMPTY_INPUT)
    LP_MAP(DegenerateConfiguration, LP_DEGENERATE_CONFIGURATION)
    LP_MAP(NumericalFailure, LP_NUMERICAL_FAILURE)
    LP_MAP(InsufficientMatches, LP_INSUFFICIENT_MATCHES)
    LP_MAP(NoModelFound, LP_NO_MODEL_FOUND)
    LP_MAP(SingularHomography, LP_SINGULAR_HOMOGRAPHY)
    LP_MAP(MaskMismatch, LP_MASK_MISMATCH)
    LP_MAP(TooManyLevels, LP_TOO_MANY_LEVELS)
    LP_MAP(CapacityOverflow, LP_CAPACITY_OVERFLOW)
    LP_MAP(NoValidHomographyYet, LP_NO_VALID_HOMOGRAPHY_YET)
    LP_MAP(ParseError, LP_PARSE_ERROR)
    LP_MAP(ValidationError, LP_VALIDATION_ERROR)
    LP_MAP(MissingFrames, LP_MISSING_FRAMES)
#undef LP_MAP
    return LP_INTERNAL;
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return LP_OK;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

ImageU8 u8_image(const std::uint8_t* p, int w, int h, int ch) {
    ImageU8 img(w, h, ch, ch == 1 ? ColorSpace::Gray : ColorSpace::RGB);
    std::memcpy(img.data.data(), p, img.data.size());
    return img;
}
ImageF32 f32_image(const float* p, int w, int h, int ch) {
    ImageF32 img(w, h, ch, ch == 1 ? ColorSpace::Gray : ColorSpace::RGB);
    std::memcpy(img.data.data(), p, img.data.size() * sizeof(float));
    return img;
}
ExtractionConfig ext_cfg(const lp_extraction_config* c) {
    ExtractionConfig e;
    e.fast_threshold = static_cast<std::uint8_t>(c->fast_threshold);
    e.fast_arc = c->fast_arc;
    e.harris_alpha = c->harris_alpha;
    e.harris_threshold = c->harris_threshold;
    e.harris_sigma = c->harris_sigma;
    e.top_n = c->top_n;
    e.n_d = c->n_d;
    e.brief_blur_sigma = c->brief_blur_sigma;
    e.patch_half = c->patch_half;
    return e;
}
MatchConfig match_cfg(const lp_match_config* c) {
    MatchConfig m;
    m.tables = c->tables;
    m.bits = c->bits;
    m.t_probes = c->t_probes;
    m.max_distance = c->max_distance;
    m.ratio = c->ratio;
    m.seed = c->seed;
    return m;
}
ProsacConfig prosac_cfg(const lp_prosac_config* c) {
    ProsacConfig p;
    p.threshold_px = c->threshold_px;
    p.max_iter = c->max_iter;
    p.confidence = c->confidence;
    p.seed = c->seed;
    p.sampling = c->sampling ? SamplingMode::Uniform : SamplingMode::Prosac;
    p.t_total = c->t_total;
    return p;
}
StitchParams stitch_params(const lp_params* p) {
    StitchParams s;
    s.extraction = ext_cfg(&p->extraction);
    s.matching = match_cfg(&p->matching);
    s.prosac = prosac_cfg(&p->prosac);
    s.blend_levels = p->blend_levels;
    s.seed = p->seed;
    return s;
}
int words(int n_d) { return (n_d + 63) / 64; }
void pack_desc(const Descriptor& d, std::uint64_t* out) {
    const int W = words(d.n_d);
    for (int i = 0; i < W; ++i) {
        out[i] = d.gt[i];
        out[W + i] = d.lt[i];
    }
}
Descriptor unpack_desc(const std::uint64_t* in, int n_d) {
    Descriptor d(n_d);
    const int W = words(n_d);
    for (int i = 0; i < W; ++i) {
        d.gt[i] = in[i];
        d.lt[i] = in[W + i];
    }
    return d;
}
lp_keypoint to_lp(const Keypoint& k) { return lp_keypoint{k.x, k.y, k.response, k.region_id}; }
Keypoint from_lp(const lp_keypoint& k) { return Keypoint{k.x, k.y, k.response, k.region_id}; }
std::vector<Correspondence> corrs(const lp_corr* c, int n) {
    std::vector<Correspondence> v(n);
    for (int i = 0; i < n; ++i) v[i] = Correspondence{c[i].sx, c[i].sy, c[i].dx, c[i].dy, c[i].quality};
    return v;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void ref_params_default(lp_params* p) {
    StitchParams s;
    PipelineConfig pc;
    std::memset(p, 0, sizeof *p);
    p->extraction = lp_extraction_config{s.extraction.fast_threshold, s.extraction.fast_arc,
                                         s.extraction.harris_alpha, s.extraction.harris_threshold,
                                         s.extraction.harris_sigma, s.extraction.top_n,
                                         s.extraction.n_d, s.extraction.brief_blur_sigma,
                                         s.extraction.patch_half};
    p->matching.tables = s.matching.tables;
    p->matching.bits = s.matching.bits;
    p->matching.t_probes = s.matching.t_probes;
    p->matching.max_distance = s.matching.max_distance;
    p->matching.ratio = s.matching.ratio;
    p->matching.seed = s.matching.seed;
    p->prosac.threshold_px = s.prosac.threshold_px;
    p->prosac.max_iter = s.prosac.max_iter;
    p->prosac.sampling = 0;
    p->prosac.confidence = s.prosac.confidence;
    p->prosac.seed = s.prosac.seed;
    p->prosac.t_total = s.prosac.t_total;
    p->blend_levels = s.blend_levels;
    p->homography_refresh = pc.homography_refresh;
    p->seed = s.seed;
    p->overlap_fraction = CameraLayout{}.overlap_fraction;
}

// ---- synth (synth.hpp) ----
int ref_synth_texture(int w, int h, std::uint64_t seed, float smooth_sigma, std::uint8_t* out) {
    return guard([&] {
        auto t = synth::texture(w, h, seed, smooth_sigma);
        std::memcpy(out, t.data.data(), t.data.size());
    });
}
int ref_synth_planted_pair(int w, int h, double overlap, std::uint64_t seed, std::uint8_t* left,
                           std::uint8_t* right, double* true_h) {
    return guard([&] {
        auto p = synth::planted_pair(w, h, overlap, seed);
        std::memcpy(left, p.left.data.data(), p.left.data.size());
        std::memcpy(right, p.right.data.data(), p.right.data.size());
        for (int i = 0; i < 9; ++i) true_h[i] = p.true_h.h[i];
    });
}
int ref_synth_sequence_frame(int w, int h, double overlap, std::uint64_t seed, std::uint64_t frame,
                             std::uint8_t* left, std::uint8_t* right) {
    return guard([&] {
        auto p = synth::planted_pair(w, h, overlap, seed);
        auto cams = synth::sequence_frame(p, frame);
        std::memcpy(left, cams[0].data.data(), cams[0].data.size());
        std::memcpy(right, cams[1].data.data(), cams[1].data.size());
    });
}
int ref_synth_rotate(const std::uint8_t* img, int w, int h, double degrees, std::uint8_t* out) {
    return guard([&] {
        auto r = synth::rotate(u8_image(img, w, h, 1), degrees);
        std::memcpy(out, r.data.data(), r.data.size());
    });
}

// ---- lorb.hpp ----
int ref_partition_regions(const int* dims, int ncams, double overlap, int patch_half,
                          lp_region* out, int cap, int* count) {
    return guard([&] {
        std::vector<std::pair<int, int>> d;
        for (int i = 0; i < ncams; ++i) d.emplace_back(dims[2 * i], dims[2 * i + 1]);
        CameraLayout lay;
        lay.overlap_fraction = overlap;
        auto r = partition_regions(lay, d, patch_half);
        *count = static_cast<int>(r.size());
        for (int i = 0; i < *count && i < cap; ++i)
            out[i] = lp_region{r[i].x0, r[i].y0, r[i].x1, r[i].y1, r[i].camera_id};
    });
}
int ref_brief_pattern(int n_d, int patch_half, std::uint64_t seed, lp_pair* out) {
    return guard([&] {
        auto p = brief_pattern(n_d, patch_half, seed);
        for (int i = 0; i < n_d; ++i)
            out[i] = lp_pair{p.pairs[i].px, p.pairs[i].py, p.pairs[i].qx, p.pairs[i].qy};
    });
}
int ref_fast_corners(const std::uint8_t* img, int w, int h, int ch, lp_region r, int thr, int arc,
                     int* xy, int cap, int* count) {
    return guard([&] {
        auto c = fast_corners(u8_image(img, w, h, ch), DetectionRegion{r.x0, r.y0, r.x1, r.y1, r.camera_id},
                              static_cast<std::uint8_t>(thr), arc);
        *count = static_cast<int>(c.size());
        for (int i = 0; i < *count && i < cap; ++i) {
            xy[2 * i] = c[i].first;
            xy[2 * i + 1] = c[i].second;
        }
    });
}
int ref_harris_response(const std::uint8_t* img, int w, int h, int ch, const int* xy, int n,
                        float alpha, float sigma, float* out) {
    return guard([&] {
        std::vector<std::pair<int, int>> pts(n);
        for (int i = 0; i < n; ++i) pts[i] = {xy[2 * i], xy[2 * i + 1]};
        auto r = harris_response(u8_image(img, w, h, ch), pts, alpha, sigma);
        std::memcpy(out, r.data(), r.size() * sizeof(float));
    });
}
int ref_nms(const lp_keypoint* in, int n, int radius, lp_keypoint* out, int* count) {
    return guard([&] {
        std::vector<Keypoint> v(n);
        for (int i = 0; i < n; ++i) v[i] = from_lp(in[i]);
        auto r = nms(v, radius);
        *count = static_cast<int>(r.size());
        for (int i = 0; i < *count; ++i) out[i] = to_lp(r[i]);
    });
}
int ref_select_top_n(const lp_keypoint* in, int n, int top_n, lp_keypoint* out, int* count) {
    return guard([&] {
        std::vector<Keypoint> v(n);
        for (int i = 0; i < n; ++i) v[i] = from_lp(in[i]);
        auto r = select_top_n(v, top_n);
        *count = static_cast<int>(r.size());
        for (int i = 0; i < *count; ++i) out[i] = to_lp(r[i]);
    });
}
int ref_gaussian_kernel(float sigma, float* out, int* n) {
    return guard([&] {
        auto k = gaussian_kernel(sigma);
        *n = static_cast<int>(k.size());
        std::memcpy(out, k.data(), k.size() * sizeof(float));
    });
}
int ref_gaussian_blur(const float* in, int w, int h, int ch, float sigma, float* out) {
    return guard([&] {
        auto r = gaussian_blur(f32_image(in, w, h, ch), sigma);
        std::memcpy(out, r.data.data(), r.data.size() * sizeof(float));
    });
}
int ref_brief_descriptors(const float* sm, int w, int h, const lp_keypoint* kps, int n,
                          const lp_pair* pairs, int n_d, int patch_half, std::uint64_t* out) {
    return guard([&] {
        BriefPattern pat;
        pat.patch_half = patch_half;
        for (int i = 0; i < n_d; ++i)
            pat.pairs.push_back(BriefPattern::Pair{pairs[i].px, pairs[i].py, pairs[i].qx, pairs[i].qy});
        auto img = f32_image(sm, w, h, 1);
        for (int i = 0; i < n; ++i) pack_desc(brief_descriptor(img, from_lp(kps[i]), pat), out + static_cast<std::size_t>(i) * 2 * words(n_d));
    });
}
int ref_extract_features(const std::uint8_t* img, int w, int h, int ch, const lp_region* regions,
                         int nreg, const lp_extraction_config* cfg, const lp_pair* pairs,
                         lp_keypoint* kp_out, std::uint64_t* desc_out, int cap, int* count) {
    return guard([&] {
        std::vector<DetectionRegion> rs;
        for (int i = 0; i < nreg; ++i)
            rs.push_back(DetectionRegion{regions[i].x0, regions[i].y0, regions[i].x1, regions[i].y1,
                                         regions[i].camera_id});
        BriefPattern pat;
        pat.patch_half = cfg->patch_half;
        for (int i = 0; i < cfg->n_d; ++i)
            pat.pairs.push_back(BriefPattern::Pair{pairs[i].px, pairs[i].py, pairs[i].qx, pairs[i].qy});
        auto f = extract_features(u8_image(img, w, h, ch), rs, ext_cfg(cfg), pat);
        *count = static_cast<int>(f.size());
        for (int i = 0; i < *count && i < cap; ++i) {
            kp_out[i] = to_lp(f[i].keypoint);
            pack_desc(f[i].descriptor, desc_out + static_cast<std::size_t>(i) * 2 * words(cfg->n_d));
        }
    });
}

// ---- matchlsh.hpp ----
int ref_descriptor_distances(const std::uint64_t* a, const std::uint64_t* b, int n, int n_d, int* out) {
    return guard([&] {
        const int W2 = 2 * words(n_d);
        for (int i = 0; i < n; ++i)
            out[i] = descriptor_distance(unpack_desc(a + static_cast<std::size_t>(i) * W2, n_d),
                                         unpack_desc(b + static_cast<std::size_t>(i) * W2, n_d));
    });
}
int ref_lsh_bit_positions(int n_d, int tables, int bits, std::uint64_t seed, int* out) {
    return guard([&] {
        std::vector<Descriptor> one{Descriptor(n_d)};
        LshIndex idx(one, tables, bits, seed);
        for (int t = 0; t < tables; ++t)
            for (int i = 0; i < bits; ++i) out[t * bits + i] = idx.tables()[t].bit_positions[i];
    });
}
int ref_probe_sequence(int k, int t, std::uint64_t* out) {
    return guard([&] {
        auto p = probe_sequence(k, t);
        std::memcpy(out, p.data(), p.size() * sizeof(std::uint64_t));
    });
}
int ref_match_features(const std::uint64_t* a, int na, const std::uint64_t* b, int nb, int n_d,
                       const lp_match_config* cfg, lp_match* out, int cap, int* count) {
    return guard([&] {
        std::vector<Descriptor> sa, sb;
        const int W2 = 2 * words(n_d);
        for (int i = 0; i < na; ++i) sa.push_back(unpack_desc(a + static_cast<std::size_t>(i) * W2, n_d));
        for (int i = 0; i < nb; ++i) sb.push_back(unpack_desc(b + static_cast<std::size_t>(i) * W2, n_d));
        auto m = match_features(sa, sb, match_cfg(cfg));
        *count = static_cast<int>(m.size());
        for (int i = 0; i < *count && i < cap; ++i)
            out[i] = lp_match{m[i].query_id, m[i].train_id, m[i].distance, m[i].quality};
    });
}

int ref_lsh_query(const std::uint64_t* train, int nt, const std::uint64_t* queries, int nq, int n_d,
                  const lp_match_config* cfg, int query_id0, long long* offsets, lp_match* out, long long cap,
                  long long* total) {
    return guard([&] {
        *total = 0;
        if (nq <= 0) return;
        const int W2 = 2 * words(n_d);
        std::vector<Descriptor> st;
        for (int i = 0; i < nt; ++i) st.push_back(unpack_desc(train + static_cast<std::size_t>(i) * W2, n_d));
        const MatchConfig mc = match_cfg(cfg);
        LshIndex index = build_index(st, mc.tables, mc.bits, mc.seed);
        long long n = 0;
        offsets[0] = 0;
        for (int q = 0; q < nq; ++q) {
            auto hits = query(index, unpack_desc(queries + static_cast<std::size_t>(q) * W2, n_d), mc.t_probes,
                              mc.max_distance, query_id0 + q);
            for (const auto& m : hits) {
                if (n < cap) out[n] = lp_match{m.query_id, m.train_id, m.distance, m.quality};
                ++n;
            }
            offsets[q + 1] = n;
        }
        *total = n;
    });
}

// ---- homography.hpp ----
int ref_dlt_homography(const lp_corr* c, int n, lp_homography* out) {
    return guard([&] {
        auto h = dlt_homography(corrs(c, n));
        for (int i = 0; i < 9; ++i) out->h[i] = h.h[i];
    });
}
int ref_symmetric_transfer_errors(const lp_homography* h, const lp_homography* hi, const lp_corr* c, int n,
                                  double* out) {
    return guard([&] {
        Homography a, b;
        for (int i = 0; i < 9; ++i) {
            a.h[i] = h->h[i];
            b.h[i] = hi->h[i];
        }
        auto v = corrs(c, n);
        for (int i = 0; i < n; ++i) out[i] = symmetric_transfer_error(a, b, v[i]);
    });
}
int ref_prosac_homography(const lp_corr* c, int n, const lp_prosac_config* cfg, lp_homography* model,
                          std::uint8_t* mask, int* inlier_count, int* iterations, int* trace_pool,
                          int* trace_samples) {
    ProsacTrace tr;
    int* iters_out = iterations;
    int st = guard([&] {
        auto r = prosac_homography(corrs(c, n), prosac_cfg(cfg), &tr);
        for (int i = 0; i < 9; ++i) model->h[i] = r.model.h[i];
        for (int i = 0; i < n; ++i) mask[i] = r.inlier_mask[i] ? 1 : 0;
        *inlier_count = r.inlier_count;
        *iters_out = r.iterations;
    });
    if (st != LP_OK) *iterations = static_cast<int>(tr.pool_sizes.size());
    for (std::size_t t = 0; t < tr.pool_sizes.size(); ++t) {
        if (trace_pool) trace_pool[t] = tr.pool_sizes[t];
        if (trace_samples)
            for (int j = 0; j < 4; ++j) trace_samples[4 * t + j] = tr.samples[t][j];
    }
    return st;
}

// ---- compose.hpp / imgops.hpp ----
int ref_compute_canvas(const int* dims, const lp_homography* hs, int n, lp_canvas* out, int* offsets) {
    return guard([&] {
        std::vector<std::pair<int, int>> d;
        std::vector<Homography> H(n);
        for (int i = 0; i < n; ++i) {
            d.emplace_back(dims[2 * i], dims[2 * i + 1]);
            for (int j = 0; j < 9; ++j) H[i].h[j] = hs[i].h[j];
        }
        auto c = compute_canvas(d, H);
        *out = lp_canvas{c.width, c.height, c.origin_x, c.origin_y};
        if (offsets)
            for (int i = 0; i < n; ++i) {
                offsets[2 * i] = c.offsets[i].first;
                offsets[2 * i + 1] = c.offsets[i].second;
            }
    });
}
int ref_warp_image(const float* img, int w, int h, int ch, const lp_homography* hom,
                   const lp_canvas* cv, float* out, float* cov) {
    return guard([&] {
        Homography H;
        for (int j = 0; j < 9; ++j) H.h[j] = hom->h[j];
        Canvas c;
        c.width = cv->width;
        c.height = cv->height;
        c.origin_x = cv->origin_x;
        c.origin_y = cv->origin_y;
        auto [o, v] = warp_image(f32_image(img, w, h, ch), H, c);
        std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
        std::memcpy(cov, v.data.data(), v.data.size() * sizeof(float));
    });
}
int ref_linear_seam_mask(const float* covs, int n, int w, int h, float* masks) {
    return guard([&] {
        std::vector<ImageF32> c;
        for (int i = 0; i < n; ++i) c.push_back(f32_image(covs + static_cast<std::size_t>(i) * w * h, w, h, 1));
        auto m = linear_seam_mask(c);
        for (int i = 0; i < n; ++i)
            std::memcpy(masks + static_cast<std::size_t>(i) * w * h, m[i].data.data(), sizeof(float) * w * h);
    });
}
int ref_downsample(const float* in, int w, int h, int ch, float* out) {
    return guard([&] {
        auto r = downsample(f32_image(in, w, h, ch));
        std::memcpy(out, r.data.data(), r.data.size() * sizeof(float));
    });
}
int ref_upsample(const float* in, int w, int h, int ch, int tw, int th, float* out) {
    return guard([&] {
        auto r = upsample(f32_image(in, w, h, ch), tw, th);
        std::memcpy(out, r.data.data(), r.data.size() * sizeof(float));
    });
}
static void pack_pyr(const Pyramid& p, float* out) {
    for (const auto& l : p.levels) {
        std::memcpy(out, l.data.data(), l.data.size() * sizeof(float));
        out += l.data.size();
    }
}
int ref_gaussian_pyramid(const float* in, int w, int h, int ch, int levels, float* out) {
    return guard([&] { pack_pyr(gaussian_pyramid(f32_image(in, w, h, ch), levels), out); });
}
int ref_build_laplacian(const float* in, int w, int h, int ch, int levels, float* out) {
    return guard([&] { pack_pyr(build_laplacian(f32_image(in, w, h, ch), levels), out); });
}
int ref_collapse_laplacian(const float* packed, int w, int h, int ch, int levels, float* out) {
    return guard([&] {
        Pyramid p;
        int lw = w, lh = h;
        for (int k = 0; k < levels; ++k) {
            p.levels.push_back(f32_image(packed, lw, lh, ch));
            packed += static_cast<std::size_t>(lw) * lh * ch;
            lw /= 2;
            lh /= 2;
        }
        auto r = collapse_laplacian(p);
        std::memcpy(out, r.data.data(), r.data.size() * sizeof(float));
    });
}
int ref_multiband_blend(const float* images, const float* masks, int n, int w, int h, int ch,
                        int levels, std::uint8_t* out) {
    return guard([&] {
        std::vector<ImageF32> im, mk;
        for (int i = 0; i < n; ++i) {
            im.push_back(f32_image(images + static_cast<std::size_t>(i) * w * h * ch, w, h, ch));
            mk.push_back(f32_image(masks + static_cast<std::size_t>(i) * w * h, w, h, 1));
        }
        auto r = multiband_blend(im, mk, levels);
        std::memcpy(out, r.data.data(), r.data.size());
    });
}

// ---- pipeline.hpp: one frame through the serial stage bodies ----
static RigLayout rig_layout(int ncams, double overlap) {
    RigLayout layout;
    layout.cameras.resize(ncams);
    layout.overlap.overlap_fraction = overlap;
    return layout;
}

int ref_stitch_frame(int ncams, int w, int h, const lp_params* params,
                     const std::uint8_t* const* images, std::uint64_t frame_index, lp_frame_out* out) {
    return guard([&] {
        PipelineConfig pc;
        pc.mode = PipelineMode::Serial;
        pc.homography_refresh = params->homography_refresh;
        StitchEngine eng(rig_layout(ncams, params->overlap_fraction), stitch_params(params), pc);
        FramePacket pkt;
        pkt.frame_index = frame_index;
        for (int c = 0; c < ncams; ++c) pkt.images.push_back(u8_image(images[c], w, h, 1));
        pkt.keypoints.resize(ncams);
        pkt.descriptors.resize(ncams);
        pkt.pair_matches.resize(ncams - 1);
        eng.stage_rectify_crop(pkt);
        eng.stage_detect(pkt);
        eng.stage_describe(pkt);
        eng.stage_match_estimate(pkt);
        eng.stage_warp_blend(pkt);
        const int n_d = params->extraction.n_d;
        const int W2 = 2 * words(n_d);
        for (int c = 0; c < ncams; ++c) {
            if (out->kp_counts) out->kp_counts[c] = static_cast<int>(pkt.keypoints[c].size());
            for (std::size_t i = 0; i < pkt.keypoints[c].size() && static_cast<int>(i) < out->cap_kp; ++i) {
                if (out->keypoints) out->keypoints[static_cast<std::size_t>(c) * out->cap_kp + i] = to_lp(pkt.keypoints[c][i]);
                if (out->descriptors)
                    pack_desc(pkt.descriptors[c][i],
                              out->descriptors + (static_cast<std::size_t>(c) * out->cap_kp + i) * W2);
            }
            if (out->homographies)
                for (int j = 0; j < 9; ++j) out->homographies[c].h[j] = pkt.homographies[c].h[j];
        }
        for (int p = 0; p + 1 < ncams; ++p) {
            if (out->match_counts) out->match_counts[p] = static_cast<int>(pkt.pair_matches[p].size());
            for (std::size_t i = 0; i < pkt.pair_matches[p].size() && static_cast<int>(i) < out->cap_matches; ++i)
                if (out->matches) {
                    const Match& m = pkt.pair_matches[p][i];
                    out->matches[static_cast<std::size_t>(p) * out->cap_matches + i] =
                        lp_match{m.query_id, m.train_id, m.distance, m.quality};
                }
        }
        std::vector<std::pair<int, int>> dims(ncams, {w, h});
        Canvas cv = compute_canvas(dims, pkt.homographies);
        out->canvas = lp_canvas{cv.width, cv.height, cv.origin_x, cv.origin_y};
        out->estimated = 1;
        if (out->panorama) {
            if (pkt.composite.data.size() > out->pano_cap) throw CapacityOverflow("panorama capacity");
            std::memcpy(out->panorama, pkt.composite.data.data(), pkt.composite.data.size());
        }
    });
}

// ---- RigLayout with rectification / crops (pipeline.hpp:240-247, 391-417) ----
static RigLayout rig_layout_cams(int ncams, double overlap, const lp_camera* cams) {
    RigLayout layout = rig_layout(ncams, overlap);
    for (int c = 0; c < ncams; ++c) {
        for (int j = 0; j < 9; ++j) layout.cameras[c].pre_transform.h[j] = cams[c].pre_transform.h[j];
        if (cams[c].has_crop) {
            const lp_region& r = cams[c].crop;
            layout.cameras[c].crop = DetectionRegion{r.x0, r.y0, r.x1, r.y1, c};
        }
    }
    return layout;
}

// StitchEngine::stage_rectify_crop alone; outputs[c] >= w*h bytes
int ref_rectify_crop(int ncams, int w, int h, const lp_camera* cams, const std::uint8_t* const* images,
                     std::uint8_t* const* outputs, int* out_w, int* out_h) {
    return guard([&] {
        lp_params p;
        ref_params_default(&p);
        StitchEngine eng(rig_layout_cams(ncams, p.overlap_fraction, cams), stitch_params(&p), PipelineConfig{});
        FramePacket pkt;
        for (int c = 0; c < ncams; ++c) pkt.images.push_back(u8_image(images[c], w, h, 1));
        eng.stage_rectify_crop(pkt);
        for (int c = 0; c < ncams; ++c) {
            out_w[c] = pkt.images[c].width;
            out_h[c] = pkt.images[c].height;
            std::memcpy(outputs[c], pkt.images[c].data.data(), pkt.images[c].data.size());
        }
    });
}

// one frame through the serial stage bodies over a RigLayout
int ref_stitch_frame_layout(int ncams, int w, int h, const lp_camera* cams, const lp_params* params,
                            const std::uint8_t* const* images, std::uint64_t frame_index, lp_frame_out* out) {
    return guard([&] {
        PipelineConfig pc;
        pc.mode = PipelineMode::Serial;
        pc.homography_refresh = params->homography_refresh;
        StitchEngine eng(rig_layout_cams(ncams, params->overlap_fraction, cams), stitch_params(params), pc);
        FramePacket pkt;
        pkt.frame_index = frame_index;
        for (int c = 0; c < ncams; ++c) pkt.images.push_back(u8_image(images[c], w, h, 1));
        pkt.keypoints.resize(ncams);
        pkt.descriptors.resize(ncams);
        pkt.pair_matches.resize(ncams - 1);
        eng.stage_rectify_crop(pkt);
        eng.stage_detect(pkt);
        eng.stage_describe(pkt);
        eng.stage_match_estimate(pkt);
        eng.stage_warp_blend(pkt);
        const int W2 = 2 * words(params->extraction.n_d);
        std::vector<std::pair<int, int>> dims;
        for (int c = 0; c < ncams; ++c) {
            dims.emplace_back(pkt.images[c].width, pkt.images[c].height);
            if (out->kp_counts) out->kp_counts[c] = static_cast<int>(pkt.keypoints[c].size());
            for (std::size_t i = 0; i < pkt.keypoints[c].size() && static_cast<int>(i) < out->cap_kp; ++i) {
                if (out->keypoints) out->keypoints[static_cast<std::size_t>(c) * out->cap_kp + i] = to_lp(pkt.keypoints[c][i]);
                if (out->descriptors)
                    pack_desc(pkt.descriptors[c][i],
                              out->descriptors + (static_cast<std::size_t>(c) * out->cap_kp + i) * W2);
            }
            if (out->homographies)
                for (int j = 0; j < 9; ++j) out->homographies[c].h[j] = pkt.homographies[c].h[j];
        }
        for (int p = 0; p + 1 < ncams; ++p) {
            if (out->match_counts) out->match_counts[p] = static_cast<int>(pkt.pair_matches[p].size());
            for (std::size_t i = 0; i < pkt.pair_matches[p].size() && static_cast<int>(i) < out->cap_matches; ++i)
                if (out->matches) {
                    const Match& m = pkt.pair_matches[p][i];
                    out->matches[static_cast<std::size_t>(p) * out->cap_matches + i] =
                        lp_match{m.query_id, m.train_id, m.distance, m.quality};
                }
        }
        Canvas cv = compute_canvas(dims, pkt.homographies);
        out->canvas = lp_canvas{cv.width, cv.height, cv.origin_x, cv.origin_y};
        out->estimated = 1;
        if (out->panorama) {
            if (pkt.composite.data.size() > out->pano_cap) throw CapacityOverflow("panorama capacity");
            std::memcpy(out->panorama, pkt.composite.data.data(), pkt.composite.data.size());
        }
    });
}

// CPU baseline: runs StitchEngine::run over `nframes` copies of the given
// frame (pipeline.hpp:369-387). mode 0 = serial, 1 = pipelined. Reports the
// reference's own Metrics (frames_out / wall_seconds, per-stage means in ms,
// stage order of pipeline.hpp:26-34).
int ref_run_engine_out(int ncams, int w, int h, const lp_params* params,
                       const std::uint8_t* const* images, int nframes, int mode, int frames_in_flight,
                       int workers_per_stage, double* fps, double* stage_ms_mean,
                       std::uint8_t* pano, std::size_t pano_cap, lp_canvas* canvas);

int ref_run_engine(int ncams, int w, int h, const lp_params* params,
                   const std::uint8_t* const* images, int nframes, int mode, int frames_in_flight,
                   int workers_per_stage, double* fps, double* stage_ms_mean) {
    return ref_run_engine_out(ncams, w, h, params, images, nframes, mode, frames_in_flight,
                              workers_per_stage, fps, stage_ms_mean, nullptr, 0, nullptr);
}

// As ref_run_engine, and the last frame's composite leaves through the sink
// (pipeline.hpp:369-387 FrameSink) into `pano` (canvas dims into `canvas`):
// bench.py compares it with the GPU rig's panorama of the same frame.
int ref_run_engine_out(int ncams, int w, int h, const lp_params* params,
                       const std::uint8_t* const* images, int nframes, int mode, int frames_in_flight,
                       int workers_per_stage, double* fps, double* stage_ms_mean,
                       std::uint8_t* pano, std::size_t pano_cap, lp_canvas* canvas) {
    return guard([&] {
        PipelineConfig pc;
        pc.mode = mode ? PipelineMode::Pipelined : PipelineMode::Serial;
        pc.frames_in_flight = frames_in_flight;
        pc.workers_per_stage = workers_per_stage;
        pc.homography_refresh = params->homography_refresh;
        StitchEngine eng(rig_layout(ncams, params->overlap_fraction), stitch_params(params), pc);
        std::vector<ImageU8> cams;
        for (int c = 0; c < ncams; ++c) cams.push_back(u8_image(images[c], w, h, 1));
        int produced = 0;
        FrameSource src = [&]() -> std::optional<std::vector<ImageU8>> {
            if (produced >= nframes) return std::nullopt;
            ++produced;
            return cams;
        };
        std::string sink_err;
        FrameSink sink = [&](const FramePacket& pk) {
            if (!pano) return;
            if (pk.composite.data.size() > pano_cap) {
                sink_err = "panorama capacity";
                return;
            }
            std::memcpy(pano, pk.composite.data.data(), pk.composite.data.size());
            if (canvas) *canvas = lp_canvas{pk.composite.width, pk.composite.height, 0, 0};
        };
        Metrics m = eng.run(src, sink);
        if (!sink_err.empty()) throw CapacityOverflow(sink_err);
        if (!m.drops.empty()) throw NumericalFailure("reference dropped a frame: " + m.drops[0].reason);
        *fps = m.frames_per_second;
        for (int s = 0; s < kNumStages; ++s) stage_ms_mean[s] = m.stage_summary(static_cast<Stage>(s)).mean / 1e6;
    });
}

// The reference's StitchEngine (Serial) over a sequence of frames
// (images[f * ncams + c]): frame f's composite into panos + f * pano_stride
// with its dims in dims[2f], dims[2f+1], or dropped[f] = 1 when the engine
// dropped it (pipeline.hpp run_stage -> Metrics::drops). Sequence parity
// tests compare the device rig against it frame by frame (HomographyCache
// fallbacks and drops included).
static void run_sequence(const RigLayout& layout, int ncams, int w, int h, const lp_params* params,
                         const std::uint8_t* const* images, int nframes, std::uint8_t* panos, std::size_t pano_stride,
                         int* dims, int* dropped) {
    {
        PipelineConfig pc;
        pc.mode = PipelineMode::Serial;
        pc.homography_refresh = params->homography_refresh;
        StitchEngine eng(layout, stitch_params(params), pc);
        int produced = 0;
        FrameSource src = [&]() -> std::optional<std::vector<ImageU8>> {
            if (produced >= nframes) return std::nullopt;
            std::vector<ImageU8> cams;
            for (int c = 0; c < ncams; ++c)
                cams.push_back(u8_image(images[static_cast<std::size_t>(produced) * ncams + c], w, h, 1));
            ++produced;
            return cams;
        };
        std::string sink_err;
        FrameSink sink = [&](const FramePacket& pk) {
            const std::uint64_t f = pk.frame_index;
            if (pk.composite.data.size() > pano_stride) {
                sink_err = "panorama capacity";
                return;
            }
            std::memcpy(panos + f * pano_stride, pk.composite.data.data(), pk.composite.data.size());
            dims[2 * f] = pk.composite.width;
            dims[2 * f + 1] = pk.composite.height;
        };
        for (int f = 0; f < nframes; ++f) dropped[f] = 0;
        Metrics m = eng.run(src, sink);
        if (!sink_err.empty()) throw CapacityOverflow(sink_err);
        for (const DroppedFrame& d : m.drops)
            if (d.frame_index < static_cast<std::uint64_t>(nframes)) dropped[d.frame_index] = 1;
    }
}
int ref_run_sequence(int ncams, int w, int h, const lp_params* params, const std::uint8_t* const* images,
                     int nframes, std::uint8_t* panos, std::size_t pano_stride, int* dims, int* dropped) {
    return guard([&] {
        run_sequence(rig_layout(ncams, params->overlap_fraction), ncams, w, h, params, images, nframes, panos,
                     pano_stride, dims, dropped);
    });
}
// the same over a RigLayout (pre-transforms and crops, pipeline.hpp:240-247)
int ref_run_sequence_layout(int ncams, int w, int h, const lp_camera* cams, const lp_params* params,
                            const std::uint8_t* const* images, int nframes, std::uint8_t* panos,
                            std::size_t pano_stride, int* dims, int* dropped) {
    return guard([&] {
        run_sequence(rig_layout_cams(ncams, params->overlap_fraction, cams), ncams, w, h, params, images, nframes,
                     panos, pano_stride, dims, dropped);
    });
}

// nthreads independent serial engines, each running `frames_per_thread`
// frames (SURVEY §8(d) mode iii). Returns aggregate frames/s.
int ref_run_engines_parallel(int ncams, int w, int h, const lp_params* params,
                             const std::uint8_t* const* images, int frames_per_thread, int nthreads,
                             double* agg_fps) {
    std::vector<int> st(nthreads, 0);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> ths;
    for (int t = 0; t < nthreads; ++t)
        ths.emplace_back([&, t] {
            double fps = 0, ms[kNumStages];
            st[t] = ref_run_engine(ncams, w, h, params, images, frames_per_thread, 0, 1, 1, &fps, ms);
        });
    for (auto& th : ths) th.join();
    double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *agg_fps = static_cast<double>(frames_per_thread) * nthreads / secs;
    for (int s : st)
        if (s) return s;
    return LP_OK;
}

}  // extern "C"
