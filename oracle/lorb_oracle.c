/* lorb_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A plain-C restatement of the reference's per-frame stitching hot path
 * (arXiv 1810.03988 reference `lorbpano`, /root/reference/proj/include/lorbpano).
 * Every function cites the reference file:line it follows. It is compiled with
 * the reference's FP discipline (-O3, no -march, -ffp-contract=off) so float and
 * double results are bit-identical to the reference built the same way.
 *
 * Third-party arithmetic restated here:
 *  - libstdc++ (GCC 13.3) std::mt19937_64 and std::uniform_int_distribution<int>
 *    (Lemire's nearly-divisionless downscaling for 64-bit generators), used by
 *    lorb.hpp:309, matchlsh.hpp:47-56, homography.hpp:188,214;
 *  - Eigen3 JacobiSVD (homography.hpp:127-128, version unpinned, absent here),
 *    restated exactly as the oracle shim does (oracle/shim/Eigen/Dense):
 *    Householder QR with a canonical blocked dot product, then a one-sided
 *    Jacobi SVD of the 9x9 factor; V column 8 = smallest singular value.
 *  - glibc libm exp/expf/log/cos/sqrt/pow/hypot/lround/roundf (same library).
 * Parity of this file with the reference itself is pinned by
 * tests/test_oracle_golden.py against fixtures made by tests/golden/make_golden.py.
 */
#define _GNU_SOURCE
#include "lorb_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}
const char* orc_last_error(void) { return g_err; }

#define TRY(x)                \
    do {                      \
        int st_ = (x);        \
        if (st_ != LP_OK) { rc = st_; goto done; } \
    } while (0)

static void* xcalloc(size_t n, size_t sz) {
    void* p = calloc(n ? n : 1, sz ? sz : 1);
    if (!p) { fprintf(stderr, "orc: out of memory\n"); abort(); }
    return p;
}

static int imin(int a, int b) { return a < b ? a : b; }
static int imax(int a, int b) { return a > b ? a : b; }

/* ------------------------------------------------------------------------ */
/* libstdc++ std::mt19937_64 (n=312, m=156, r=31, a=0xB5026F5AA96619E9, ...)   */
typedef struct { uint64_t mt[312]; int idx; } mt64;

static void mt64_seed(mt64* r, uint64_t s) {
    r->mt[0] = s;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = 312;
}
static uint64_t mt64_next(mt64* r) {
    if (r->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
        }
        r->idx = 0;
    }
    uint64_t y = r->mt[r->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}
/* std::uniform_int_distribution<int>(a, b)(mt19937_64): 128-bit Lemire. */
static int uid_int(mt64* r, int a, int b) {
    const uint64_t range = (uint64_t)(int64_t)b - (uint64_t)(int64_t)a + 1ULL;
    unsigned __int128 p = (unsigned __int128)mt64_next(r) * range;
    uint64_t low = (uint64_t)p;
    if (low < range) {
        const uint64_t thr = (0ULL - range) % range;
        while (low < thr) {
            p = (unsigned __int128)mt64_next(r) * range;
            low = (uint64_t)p;
        }
    }
    return (int)((uint64_t)(p >> 64) + (uint64_t)(int64_t)a);
}

/* ------------------------------------------------------------------------ */
void orc_params_default(lp_params* p) {
    memset(p, 0, sizeof *p);
    /* ExtractionConfig lorb.hpp:71-80 */
    p->extraction.fast_threshold = 20;
    p->extraction.fast_arc = 9;
    p->extraction.harris_alpha = 0.04f;
    p->extraction.harris_threshold = 0.0f;
    p->extraction.harris_sigma = 1.0f;
    p->extraction.top_n = 500;
    p->extraction.n_d = 256;
    p->extraction.brief_blur_sigma = 2.0f;
    p->extraction.patch_half = 15;
    /* MatchConfig matchlsh.hpp:161-167 */
    p->matching.tables = 4;
    p->matching.bits = 16;
    p->matching.t_probes = 16;
    p->matching.max_distance = 64;
    p->matching.ratio = 0.8f;
    p->matching.seed = 0;
    /* ProsacConfig homography.hpp:156-162 */
    p->prosac.threshold_px = 3.0;
    p->prosac.max_iter = 1000;
    p->prosac.sampling = 0;
    p->prosac.confidence = 0.99;
    p->prosac.seed = 0;
    p->prosac.t_total = 200000.0;
    /* StitchParams pipeline.hpp:249-255, PipelineConfig 199-204, CameraLayout lorb.hpp:94 */
    p->blend_levels = 4;
    p->homography_refresh = 1;
    p->seed = 0;
    p->overlap_fraction = 0.25;
}

/* partition_regions, lorb.hpp:100-138 (fraction path) */
int orc_partition_regions(const int* dims, int ncams, double f, int ph, lp_region* out, int cap,
                          int* count) {
    if (f <= 0.0) return fail(LP_NO_OVERLAP, "overlap fraction must be > 0");
    if (f > 1.0) return fail(LP_OVERLAP_EXCEEDS_IMAGE, "overlap fraction must be <= 1");
    int n = 0;
    for (int i = 0; i + 1 < ncams; ++i) {
        const int wl = dims[2 * i], hl = dims[2 * i + 1];
        const int wr = dims[2 * i + 2], hr = dims[2 * i + 3];
        lp_region rr[2] = {{(int)lround(wl * (1.0 - f)), 0, wl, hl, i},
                           {0, 0, (int)lround(wr * f), hr, i + 1}};
        for (int k = 0; k < 2; ++k) {
            rr[k].x0 += ph;
            rr[k].y0 += ph;
            rr[k].x1 -= ph;
            rr[k].y1 -= ph;
            if (rr[k].x0 >= rr[k].x1 || rr[k].y0 >= rr[k].y1)
                return fail(LP_REGION_TOO_SMALL, "overlap strip smaller than 2*patch_half");
        }
        for (int k = 0; k < 2; ++k) {
            if (n < cap) out[n] = rr[k];
            ++n;
        }
    }
    *count = n;
    return LP_OK;
}

/* brief_pattern, lorb.hpp:303-330 (Box-Muller, one coordinate at a time) */
static int brief_coord(mt64* rng, double sigma, int ph) {
    for (;;) {
        double u1 = ((double)mt64_next(rng) + 1.0) / ((double)UINT64_MAX + 2.0);
        double u2 = (double)mt64_next(rng) / ((double)UINT64_MAX + 1.0);
        double g = sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2) * sigma;
        int v = (int)lround(g);
        if (v >= -ph && v <= ph) return v;
    }
}
int orc_brief_pattern(int n_d, int ph, uint64_t seed, lp_pair* out) {
    if (n_d < 1) return fail(LP_BAD_PARAMS, "brief_pattern: n_d must be >= 1");
    mt64 rng;
    mt64_seed(&rng, seed);
    const double sigma = ph / 2.5;
    for (int i = 0; i < n_d; ++i) {
        out[i].px = brief_coord(&rng, sigma, ph);
        out[i].py = brief_coord(&rng, sigma, ph);
        out[i].qx = brief_coord(&rng, sigma, ph);
        out[i].qy = brief_coord(&rng, sigma, ph);
    }
    return LP_OK;
}

/* gaussian_kernel, imgops.hpp:35-47 (float taps, float normalisation) */
int orc_gaussian_kernel(float sigma, float* k, int* n) {
    if (!(sigma > 0.0f)) return fail(LP_INVALID_SIGMA, "gaussian kernel: sigma must be > 0");
    const int radius = (int)ceilf(3.0f * sigma);
    float sum = 0.0f;
    for (int i = -radius; i <= radius; ++i) {
        float v = expf(-((float)i * (float)i) / (2.0f * sigma * sigma));
        k[i + radius] = v;
        sum += v;
    }
    for (int i = 0; i < 2 * radius + 1; ++i) k[i] /= sum;
    *n = 2 * radius + 1;
    return LP_OK;
}

/* ------------------------------------------------------------------------ */
/* FAST-9: fast_ring lorb.hpp:141-159, longest_arc 164-176, segment test 178-188 */
static const int RING[16][2] = {{0, -3}, {1, -3}, {2, -2}, {3, -1}, {3, 0}, {3, 1},
                                {2, 2},  {1, 3},  {0, 3},  {-1, 3}, {-2, 2}, {-3, 1},
                                {-3, 0}, {-3, -1}, {-2, -2}, {-1, -3}};

static int longest_arc(unsigned mask) {
    if (mask == 0xFFFFu) return 16;
    int best = 0, run = 0;
    for (int i = 0; i < 32; ++i) {
        if (mask & (1u << (i % 16))) {
            ++run;
            if (run > best) best = run;
        } else {
            run = 0;
        }
    }
    return best < 16 ? best : 16;
}

static int segment_test(const uint8_t* img, int w, int x, int y, int t, int arc) {
    const int c = img[(size_t)y * w + x];
    unsigned br = 0, dk = 0;
    for (int i = 0; i < 16; ++i) {
        int v = img[(size_t)(y + RING[i][1]) * w + x + RING[i][0]];
        if (v > c + t) br |= 1u << i;
        if (v < c - t) dk |= 1u << i;
    }
    return longest_arc(br) >= arc || longest_arc(dk) >= arc;
}

/* fast_corners, lorb.hpp:192-205: raster order over region ∩ [3,w-3)x[3,h-3) */
int orc_fast_corners(const uint8_t* img, int w, int h, int ch, lp_region r, int thr, int arc,
                     int* xy, int cap, int* count) {
    if (ch != 1) return fail(LP_UNSUPPORTED_FORMAT, "fast_corners: grayscale input required");
    const int x0 = imax(r.x0, 3), x1 = imin(r.x1, w - 3);
    const int y0 = imax(r.y0, 3), y1 = imin(r.y1, h - 3);
    if (x0 >= x1 || y0 >= y1) return fail(LP_REGION_TOO_SMALL, "fast_corners: region too small");
    const int t = (uint8_t)thr;
    int n = 0;
    for (int y = y0; y < y1; ++y)
        for (int x = x0; x < x1; ++x)
            if (segment_test(img, w, x, y, t, arc)) {
                if (n < cap) {
                    xy[2 * n] = x;
                    xy[2 * n + 1] = y;
                }
                ++n;
            }
    *count = n;
    return LP_OK;
}

/* harris_response, lorb.hpp:209-250: FP64 normalised Gaussian window,
 * central differences, v-outer/u-inner accumulation, cast to float. */
int orc_harris_response(const uint8_t* img, int w, int h, int ch, const int* xy, int n,
                        float alpha, float sigma, float* out) {
    if (ch != 1) return fail(LP_UNSUPPORTED_FORMAT, "harris_response: grayscale input required");
    const int radius = (int)ceilf(3.0f * sigma);
    const double s2 = 2.0 * (double)sigma * sigma;
    const int K = 2 * radius + 1;
    double* wt = xcalloc((size_t)K * K, sizeof(double));
    double sum = 0.0;
    for (int v = -radius; v <= radius; ++v)
        for (int u = -radius; u <= radius; ++u) {
            double g = exp(-(u * u + v * v) / s2);
            wt[(v + radius) * K + (u + radius)] = g;
            sum += g;
        }
    for (int i = 0; i < K * K; ++i) wt[i] /= sum;
    for (int p = 0; p < n; ++p) {
        const int px = xy[2 * p], py = xy[2 * p + 1];
        if (px - radius - 1 < 0 || px + radius + 1 >= w || py - radius - 1 < 0 ||
            py + radius + 1 >= h) {
            free(wt);
            return fail(LP_WINDOW_OUT_OF_BOUNDS, "harris_response: window does not fit");
        }
        double a = 0.0, b = 0.0, c = 0.0;
        for (int v = -radius; v <= radius; ++v)
            for (int u = -radius; u <= radius; ++u) {
                const int x = px + u, y = py + v;
                double ix = ((double)img[(size_t)y * w + x + 1] - img[(size_t)y * w + x - 1]) / 2.0;
                double iy = ((double)img[(size_t)(y + 1) * w + x] - img[(size_t)(y - 1) * w + x]) / 2.0;
                double t = wt[(v + radius) * K + (u + radius)];
                a += t * ix * ix;
                b += t * iy * iy;
                c += t * ix * iy;
            }
        out[p] = (float)((a * b - c * c) - alpha * (a + b) * (a + b));
    }
    free(wt);
    return LP_OK;
}

/* nms, lorb.hpp:254-288: dense index grid over the candidate bbox; ties to
 * the smaller (y,x); output keeps input order. */
int orc_nms(const lp_keypoint* c, int n, int radius, lp_keypoint* out, int* count) {
    *count = 0;
    if (n == 0) return LP_OK;
    int minx = c[0].x, maxx = c[0].x, miny = c[0].y, maxy = c[0].y;
    for (int i = 0; i < n; ++i) {
        minx = imin(minx, c[i].x);
        maxx = imax(maxx, c[i].x);
        miny = imin(miny, c[i].y);
        maxy = imax(maxy, c[i].y);
    }
    const int w = maxx - minx + 1, h = maxy - miny + 1;
    int* grid = xcalloc((size_t)w * h, sizeof(int));
    for (size_t i = 0; i < (size_t)w * h; ++i) grid[i] = -1;
    for (int i = 0; i < n; ++i) grid[(size_t)(c[i].y - miny) * w + (c[i].x - minx)] = i;
    int k = 0;
    for (int i = 0; i < n; ++i) {
        int wins = 1;
        for (int dy = -radius; dy <= radius && wins; ++dy)
            for (int dx = -radius; dx <= radius && wins; ++dx) {
                if (dx == 0 && dy == 0) continue;
                int gx = c[i].x - minx + dx, gy = c[i].y - miny + dy;
                if (gx < 0 || gx >= w || gy < 0 || gy >= h) continue;
                int j = grid[(size_t)gy * w + gx];
                if (j < 0) continue;
                const lp_keypoint* o = &c[j];
                if (o->response > c[i].response ||
                    (o->response == c[i].response &&
                     (o->y < c[i].y || (o->y == c[i].y && o->x < c[i].x))))
                    wins = 0;
            }
        if (wins) out[k++] = c[i];
    }
    free(grid);
    *count = k;
    return LP_OK;
}

/* select_top_n, lorb.hpp:291-299: total order (response desc, y asc, x asc) */
static int kp_cmp(const void* pa, const void* pb) {
    const lp_keypoint* a = pa;
    const lp_keypoint* b = pb;
    if (a->response != b->response) return a->response > b->response ? -1 : 1;
    if (a->y != b->y) return a->y < b->y ? -1 : 1;
    if (a->x != b->x) return a->x < b->x ? -1 : 1;
    return 0;
}
int orc_select_top_n(const lp_keypoint* in, int n, int top_n, lp_keypoint* out, int* count) {
    if (top_n < 1) return fail(LP_BAD_PARAMS, "select_top_n: n must be >= 1");
    lp_keypoint* tmp = xcalloc((size_t)n, sizeof *tmp);
    memcpy(tmp, in, sizeof *tmp * (size_t)n);
    qsort(tmp, (size_t)n, sizeof *tmp, kp_cmp);
    const int k = n < top_n ? n : top_n;
    memcpy(out, tmp, sizeof *tmp * (size_t)k);
    free(tmp);
    *count = k;
    return LP_OK;
}

/* gaussian_blur, imgops.hpp:50-72: horizontal then vertical, clamp-to-edge,
 * acc = 0.0f; acc += k[i] * v in tap order i = -r..r. */
int orc_gaussian_blur(const float* in, int w, int h, int ch, float sigma, float* out) {
    float k[256];
    int nk;
    int st = orc_gaussian_kernel(sigma, k, &nk);
    if (st) return st;
    const int r = nk / 2;
    float* tmp = xcalloc((size_t)w * h * ch, sizeof(float));
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x)
            for (int c = 0; c < ch; ++c) {
                float acc = 0.0f;
                for (int i = -r; i <= r; ++i) {
                    int xx = x + i < 0 ? 0 : (x + i >= w ? w - 1 : x + i);
                    acc += k[i + r] * in[((size_t)y * w + xx) * ch + c];
                }
                tmp[((size_t)y * w + x) * ch + c] = acc;
            }
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x)
            for (int c = 0; c < ch; ++c) {
                float acc = 0.0f;
                for (int i = -r; i <= r; ++i) {
                    int yy = y + i < 0 ? 0 : (y + i >= h ? h - 1 : y + i);
                    acc += k[i + r] * tmp[((size_t)yy * w + x) * ch + c];
                }
                out[((size_t)y * w + x) * ch + c] = acc;
            }
    free(tmp);
    return LP_OK;
}

/* brief_descriptor, lorb.hpp:333-350 + Descriptor::set_trit 56-62 */
static int brief_one(const float* sm, int w, int h, lp_keypoint kp, const lp_pair* pairs,
                     int n_d, int ph, uint64_t* d) {
    if (kp.x - ph < 0 || kp.x + ph >= w || kp.y - ph < 0 || kp.y + ph >= h)
        return fail(LP_PATCH_OUT_OF_BOUNDS, "brief_descriptor: patch does not fit");
    const int W = (n_d + 63) / 64;
    memset(d, 0, sizeof(uint64_t) * 2 * (size_t)W);
    for (int i = 0; i < n_d; ++i) {
        float ip = sm[(size_t)(kp.y + pairs[i].py) * w + kp.x + pairs[i].px];
        float iq = sm[(size_t)(kp.y + pairs[i].qy) * w + kp.x + pairs[i].qx];
        uint64_t bit = 1ULL << (i % 64);
        if (ip > iq)
            d[i / 64] |= bit;
        else if (ip < iq)
            d[W + i / 64] |= bit;
    }
    return LP_OK;
}
int orc_brief_descriptors(const float* sm, int w, int h, const lp_keypoint* kps, int n,
                          const lp_pair* pairs, int n_d, int ph, uint64_t* out) {
    const int W2 = 2 * ((n_d + 63) / 64);
    for (int i = 0; i < n; ++i) {
        int st = brief_one(sm, w, h, kps[i], pairs, n_d, ph, out + (size_t)i * W2);
        if (st) return st;
    }
    return LP_OK;
}

/* ExtractionConfig::validate, lorb.hpp:82-89 */
static int validate_ext(const lp_extraction_config* c) {
    if (c->fast_arc < 9 || c->fast_arc > 16) return fail(LP_BAD_PARAMS, "fast_arc must be in [9,16]");
    if (c->top_n < 4) return fail(LP_BAD_PARAMS, "top_n must be >= 4");
    if (c->n_d < 64 || c->n_d > 512) return fail(LP_BAD_PARAMS, "n_d must be in [64,512]");
    if (!(c->harris_sigma > 0.0f)) return fail(LP_INVALID_SIGMA, "harris_sigma must be > 0");
    if (!(c->brief_blur_sigma > 0.0f)) return fail(LP_INVALID_SIGMA, "brief_blur_sigma must be > 0");
    if (c->patch_half < 1) return fail(LP_BAD_PARAMS, "patch_half must be >= 1");
    return LP_OK;
}

/* detect one region: FAST -> Harris -> threshold -> NMS -> top-N
 * (lorb.hpp:396-404; identical in stage_detect pipeline.hpp:426-437). */
static int detect_region(const uint8_t* img, int w, int h, lp_region r, int ri,
                         const lp_extraction_config* cfg, lp_keypoint* out, int* count) {
    int rc = LP_OK;
    *count = 0;
    const int cap = w * h;
    int* xy = xcalloc((size_t)cap * 2, sizeof(int));
    float* resp = NULL;
    lp_keypoint *cand = NULL, *kept = NULL;
    int nc = 0;
    TRY(orc_fast_corners(img, w, h, 1, r, cfg->fast_threshold, cfg->fast_arc, xy, cap, &nc));
    if (nc == 0) goto done;
    resp = xcalloc((size_t)nc, sizeof(float));
    TRY(orc_harris_response(img, w, h, 1, xy, nc, cfg->harris_alpha, cfg->harris_sigma, resp));
    cand = xcalloc((size_t)nc, sizeof *cand);
    int m = 0;
    for (int i = 0; i < nc; ++i)
        if (resp[i] >= cfg->harris_threshold) {
            lp_keypoint k = {xy[2 * i], xy[2 * i + 1], resp[i], ri};
            cand[m++] = k;
        }
    kept = xcalloc((size_t)(m ? m : 1), sizeof *kept);
    int nk = 0;
    TRY(orc_nms(cand, m, 1, kept, &nk));
    TRY(orc_select_top_n(kept, nk, cfg->top_n, out, count));
done:
    free(xy);
    free(resp);
    free(cand);
    free(kept);
    return rc;
}

/* detail::smoothed_crop, lorb.hpp:369-382: region +- (patch_half + ceil(3 sigma)),
 * clipped to the image, u8 -> f32, gaussian_blur. */
typedef struct { float* img; int w, h, ox, oy; } crop_t;
static int smoothed_crop(const uint8_t* img, int w, int h, lp_region r, int ph, float sigma,
                         crop_t* c) {
    const int margin = ph + (int)ceilf(3.0f * sigma);
    const int x0 = imax(0, r.x0 - margin), y0 = imax(0, r.y0 - margin);
    const int x1 = imin(w, r.x1 + margin), y1 = imin(h, r.y1 + margin);
    c->w = x1 - x0;
    c->h = y1 - y0;
    c->ox = x0;
    c->oy = y0;
    float* raw = xcalloc((size_t)c->w * c->h, sizeof(float));
    for (int y = y0; y < y1; ++y)
        for (int x = x0; x < x1; ++x) raw[(size_t)(y - y0) * c->w + (x - x0)] = img[(size_t)y * w + x];
    c->img = xcalloc((size_t)c->w * c->h, sizeof(float));
    int st = orc_gaussian_blur(raw, c->w, c->h, 1, sigma, c->img);
    free(raw);
    return st;
}

/* extract_features, lorb.hpp:388-413 */
int orc_extract_features(const uint8_t* img, int w, int h, int ch, const lp_region* regions,
                         int nreg, const lp_extraction_config* cfg, const lp_pair* pairs,
                         lp_keypoint* kp_out, uint64_t* desc_out, int cap, int* count) {
    int st = validate_ext(cfg);
    if (st) return st;
    if (ch != 1) return fail(LP_UNSUPPORTED_FORMAT, "fast_corners: grayscale input required");
    const int W2 = 2 * ((cfg->n_d + 63) / 64);
    lp_keypoint* sel = xcalloc((size_t)cfg->top_n, sizeof *sel);
    uint64_t* d = xcalloc((size_t)W2, sizeof(uint64_t));
    int n = 0;
    for (int ri = 0; ri < nreg; ++ri) {
        int ns = 0;
        st = detect_region(img, w, h, regions[ri], ri, cfg, sel, &ns);
        if (st) break;
        if (ns == 0) continue;
        crop_t c;
        st = smoothed_crop(img, w, h, regions[ri], cfg->patch_half, cfg->brief_blur_sigma, &c);
        if (st) break;
        for (int i = 0; i < ns && !st; ++i) {
            lp_keypoint local = {sel[i].x - c.ox, sel[i].y - c.oy, sel[i].response, sel[i].region_id};
            st = brief_one(c.img, c.w, c.h, local, pairs, cfg->n_d, cfg->patch_half, d);
            if (!st && n < cap) {
                kp_out[n] = sel[i];
                memcpy(desc_out + (size_t)n * W2, d, sizeof(uint64_t) * W2);
            }
            if (!st) ++n;
        }
        free(c.img);
        if (st) break;
    }
    free(sel);
    free(d);
    *count = n;
    return st;
}

/* ------------------------------------------------------------------------ */
/* descriptor_distance, matchlsh.hpp:25-33 */
static int dist_packed(const uint64_t* a, const uint64_t* b, int W) {
    int d = 0;
    for (int i = 0; i < W; ++i) {
        d += __builtin_popcountll(a[i] ^ b[i]);
        d += __builtin_popcountll(a[W + i] ^ b[W + i]);
    }
    return d;
}
int orc_descriptor_distances(const uint64_t* a, const uint64_t* b, int n, int n_d, int* out) {
    const int W = (n_d + 63) / 64;
    for (int i = 0; i < n; ++i) out[i] = dist_packed(a + (size_t)i * 2 * W, b + (size_t)i * 2 * W, W);
    return LP_OK;
}

/* LshIndex bit sampling, matchlsh.hpp:47-59: per table a partial Fisher-Yates
 * over [0, 2 n_d) driven by uniform_int_distribution<int>(i, domain-1). */
int orc_lsh_bit_positions(int n_d, int tables, int bits, uint64_t seed, int* out) {
    if (tables < 1) return fail(LP_BAD_PARAMS, "build_index: L must be >= 1");
    if (bits < 1 || (n_d > 0 && bits > 2 * n_d)) return fail(LP_BAD_PARAMS, "build_index: k must be in [1, 2*n_d]");
    mt64 rng;
    mt64_seed(&rng, seed);
    const int domain = n_d > 0 ? 2 * n_d : bits;
    int* pos = xcalloc((size_t)domain, sizeof(int));
    for (int t = 0; t < tables; ++t) {
        for (int i = 0; i < domain; ++i) pos[i] = i;
        for (int i = 0; i < bits; ++i) {
            int j = uid_int(&rng, i, domain - 1);
            int tmp = pos[i];
            pos[i] = pos[j];
            pos[j] = tmp;
        }
        for (int i = 0; i < bits; ++i) out[t * bits + i] = pos[i];
    }
    free(pos);
    return LP_OK;
}

/* probe_sequence, matchlsh.hpp:104-128 */
int orc_probe_sequence(int k, int t, uint64_t* out) {
    if (t < 1) return fail(LP_BAD_PARAMS, "probe_sequence: t_probes must be >= 1");
    if (k < 1 || k >= 63) return fail(LP_BAD_PARAMS, "probe_sequence: k must be in [1,62]");
    if ((uint64_t)t > (1ULL << k)) return fail(LP_TOO_MANY_PROBES, "probe_sequence: t_probes exceeds 2^k");
    int n = 0;
    out[n++] = 0;
    int idx[64];
    for (int card = 1; n < t && card <= k; ++card) {
        for (int i = 0; i < card; ++i) idx[i] = i;
        for (;;) {
            uint64_t m = 0;
            for (int i = 0; i < card; ++i) m |= 1ULL << idx[i];
            out[n++] = m;
            if (n >= t) break;
            int i = card - 1;
            while (i >= 0 && idx[i] == k - card + i) --i;
            if (i < 0) break;
            ++idx[i];
            for (int j = i + 1; j < card; ++j) idx[j] = idx[j - 1] + 1;
        }
    }
    return LP_OK;
}

/* LshIndex::hash_key, matchlsh.hpp:77-86 */
static uint64_t hash_key(const uint64_t* d, int n_d, int W, const int* pos, int bits) {
    uint64_t key = 0;
    for (int i = 0; i < bits; ++i) {
        int p = pos[i];
        const uint64_t* plane = p < n_d ? d : d + W;
        int bit = p < n_d ? p : p - n_d;
        if ((plane[bit / 64] >> (bit % 64)) & 1ULL) key |= 1ULL << i;
    }
    return key;
}

typedef struct { uint64_t key; int id; } kid_t;
static int kid_cmp(const void* pa, const void* pb) {
    const kid_t* a = pa;
    const kid_t* b = pb;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    return a->id < b->id ? -1 : (a->id > b->id);
}
static int hit_cmp(const void* pa, const void* pb) { /* (distance, train_id), matchlsh.hpp:155-157 */
    const lp_match* a = pa;
    const lp_match* b = pb;
    if (a->distance != b->distance) return a->distance < b->distance ? -1 : 1;
    return a->train_id < b->train_id ? -1 : (a->train_id > b->train_id);
}
static int out_cmp(const void* pa, const void* pb) { /* quality desc, query_id asc, 188-191 */
    const lp_match* a = pa;
    const lp_match* b = pb;
    if (a->quality != b->quality) return a->quality > b->quality ? -1 : 1;
    return a->query_id < b->query_id ? -1 : (a->query_id > b->query_id);
}

/* match_features, matchlsh.hpp:173-193, with LshIndex (41-63) and query
 * (132-159): buckets are the (key, id)-sorted train list of each table. */
int orc_match_features(const uint64_t* a, int na, const uint64_t* b, int nb, int n_d,
                       const lp_match_config* cfg, lp_match* out, int cap, int* count) {
    if (na == 0 || nb == 0) return fail(LP_EMPTY_INPUT, "match_features: empty set");
    const int L = cfg->tables, k = cfg->bits, W = (n_d + 63) / 64;
    int* pos = xcalloc((size_t)(L > 0 ? L : 1) * (k > 0 ? k : 1), sizeof(int));
    int st = orc_lsh_bit_positions(n_d, L, k, cfg->seed, pos);
    if (st) { free(pos); return st; }
    uint64_t* probes = xcalloc((size_t)(cfg->t_probes > 0 ? cfg->t_probes : 1), sizeof(uint64_t));
    st = orc_probe_sequence(k, cfg->t_probes, probes);
    if (st) { free(pos); free(probes); return st; }
    const int T = cfg->t_probes;
    kid_t* tab = xcalloc((size_t)L * nb, sizeof(kid_t));
    for (int t = 0; t < L; ++t) {
        for (int j = 0; j < nb; ++j) {
            tab[(size_t)t * nb + j].key = hash_key(b + (size_t)j * 2 * W, n_d, W, pos + t * k, k);
            tab[(size_t)t * nb + j].id = j;
        }
        qsort(tab + (size_t)t * nb, (size_t)nb, sizeof(kid_t), kid_cmp);
    }
    uint8_t* seen = xcalloc((size_t)nb, 1);
    lp_match* hits = xcalloc((size_t)nb, sizeof(lp_match));
    lp_match* res = xcalloc((size_t)na, sizeof(lp_match));
    int nres = 0;
    for (int q = 0; q < na; ++q) {
        const uint64_t* qd = a + (size_t)q * 2 * W;
        memset(seen, 0, (size_t)nb);
        int nh = 0;
        for (int t = 0; t < L; ++t) {
            const uint64_t key = hash_key(qd, n_d, W, pos + t * k, k);
            const kid_t* tb = tab + (size_t)t * nb;
            for (int p = 0; p < T; ++p) {
                const uint64_t want = key ^ probes[p];
                int lo = 0, hi = nb; /* first index with key >= want */
                while (lo < hi) {
                    int mid = (lo + hi) / 2;
                    if (tb[mid].key < want) lo = mid + 1; else hi = mid;
                }
                for (int i = lo; i < nb && tb[i].key == want; ++i) {
                    const int id = tb[i].id;
                    if (seen[id]) continue;
                    seen[id] = 1;
                    int d = dist_packed(qd, b + (size_t)id * 2 * W, W);
                    if (d <= cfg->max_distance) {
                        lp_match m = {q, id, d, 1.0f - (float)d / (2.0f * n_d)};
                        hits[nh++] = m;
                    }
                }
            }
        }
        if (nh == 0) continue;
        qsort(hits, (size_t)nh, sizeof(lp_match), hit_cmp);
        if (nh >= 2 && !(hits[0].distance < cfg->ratio * (float)hits[1].distance)) continue;
        res[nres++] = hits[0];
    }
    qsort(res, (size_t)nres, sizeof(lp_match), out_cmp);
    for (int i = 0; i < nres && i < cap; ++i) out[i] = res[i];
    *count = nres;
    free(pos);
    free(probes);
    free(tab);
    free(seen);
    free(hits);
    free(res);
    return LP_OK;
}

/* query, matchlsh.hpp:132-159, for nq queries against build_index(train):
 * per query every probed candidate within max_distance, sorted by
 * (distance, train_id); offsets[q] .. offsets[q + 1] index `out`. */
int orc_lsh_query(const uint64_t* train, int nt, const uint64_t* queries, int nq, int n_d,
                  const lp_match_config* cfg, int query_id0, long long* offsets, lp_match* out, long long cap,
                  long long* total) {
    *total = 0;
    if (nq <= 0) return LP_OK;
    for (int q = 0; q <= nq; ++q) offsets[q] = 0;
    if (nt == 0) return LP_OK;
    const int L = cfg->tables, k = cfg->bits, W = (n_d + 63) / 64;
    int* pos = xcalloc((size_t)(L > 0 ? L : 1) * (k > 0 ? k : 1), sizeof(int));
    int st = orc_lsh_bit_positions(n_d, L, k, cfg->seed, pos);
    if (st) { free(pos); return st; }
    uint64_t* probes = xcalloc((size_t)(cfg->t_probes > 0 ? cfg->t_probes : 1), sizeof(uint64_t));
    st = orc_probe_sequence(k, cfg->t_probes, probes);
    if (st) { free(pos); free(probes); return st; }
    const int T = cfg->t_probes;
    kid_t* tab = xcalloc((size_t)L * nt, sizeof(kid_t));
    for (int t = 0; t < L; ++t) {
        for (int j = 0; j < nt; ++j) {
            tab[(size_t)t * nt + j].key = hash_key(train + (size_t)j * 2 * W, n_d, W, pos + t * k, k);
            tab[(size_t)t * nt + j].id = j;
        }
        qsort(tab + (size_t)t * nt, (size_t)nt, sizeof(kid_t), kid_cmp);
    }
    uint8_t* seen = xcalloc((size_t)nt, 1);
    lp_match* hits = xcalloc((size_t)nt, sizeof(lp_match));
    long long n = 0;
    for (int q = 0; q < nq; ++q) {
        const uint64_t* qd = queries + (size_t)q * 2 * W;
        memset(seen, 0, (size_t)nt);
        int nh = 0;
        for (int t = 0; t < L; ++t) {
            const uint64_t key = hash_key(qd, n_d, W, pos + t * k, k);
            const kid_t* tb = tab + (size_t)t * nt;
            for (int p = 0; p < T; ++p) {
                const uint64_t want = key ^ probes[p];
                int lo = 0, hi = nt;
                while (lo < hi) {
                    int mid = (lo + hi) / 2;
                    if (tb[mid].key < want) lo = mid + 1; else hi = mid;
                }
                for (int i = lo; i < nt && tb[i].key == want; ++i) {
                    const int id = tb[i].id;
                    if (seen[id]) continue;
                    seen[id] = 1;
                    int d = dist_packed(qd, train + (size_t)id * 2 * W, W);
                    if (d <= cfg->max_distance) {
                        lp_match m = {query_id0 + q, id, d, 1.0f - (float)d / (2.0f * n_d)};
                        hits[nh++] = m;
                    }
                }
            }
        }
        qsort(hits, (size_t)nh, sizeof(lp_match), hit_cmp);
        for (int i = 0; i < nh; ++i, ++n)
            if (n < cap) out[n] = hits[i];
        offsets[q + 1] = n;
    }
    *total = n;
    free(pos);
    free(probes);
    free(tab);
    free(seen);
    free(hits);
    return LP_OK;
}

/* ------------------------------------------------------------------------ */
/* Homography helpers, homography.hpp:25-62 */
static double h_det(const double* h) {
    return h[0] * (h[4] * h[8] - h[5] * h[7]) - h[1] * (h[3] * h[8] - h[5] * h[6]) +
           h[2] * (h[3] * h[7] - h[4] * h[6]);
}
static void h_apply(const double* h, double x, double y, double* ox, double* oy) {
    double w = h[6] * x + h[7] * y + h[8];
    *ox = (h[0] * x + h[1] * y + h[2]) / w;
    *oy = (h[3] * x + h[4] * y + h[5]) / w;
}
static int h_inverse(const double* h, double* out) {
    double d = h_det(h);
    if (fabs(d) < 1e-12) return fail(LP_SINGULAR_HOMOGRAPHY, "homography not invertible");
    double inv[9] = {(h[4] * h[8] - h[5] * h[7]) / d, (h[2] * h[7] - h[1] * h[8]) / d,
                     (h[1] * h[5] - h[2] * h[4]) / d, (h[5] * h[6] - h[3] * h[8]) / d,
                     (h[0] * h[8] - h[2] * h[6]) / d, (h[2] * h[3] - h[0] * h[5]) / d,
                     (h[3] * h[7] - h[4] * h[6]) / d, (h[1] * h[6] - h[0] * h[7]) / d,
                     (h[0] * h[4] - h[1] * h[3]) / d};
    memcpy(out, inv, sizeof inv);
    if (fabs(out[8]) > 1e-12)
        for (int i = 0; i < 9; ++i) out[i] /= inv[8];
    return LP_OK;
}
static void h_compose(const double* a, const double* b, double* out) { /* a ∘ b */
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            double s = 0;
            for (int k = 0; k < 3; ++k) s += a[r * 3 + k] * b[k * 3 + c];
            out[r * 3 + c] = s;
        }
    if (fabs(out[8]) > 1e-12) {
        const double d8 = out[8];
        for (int i = 0; i < 8; ++i) out[i] /= d8;
        out[8] /= out[8];
    }
}

/* Eigen JacobiSVD restatement — identical to oracle/shim/Eigen/Dense. */
static double dot_blocked(const double* a, int sa, const double* b, int sb, int r0, int r1) {
    double p[256];
    for (int l = 0; l < 256; ++l) p[l] = 0.0;
    for (int i = r0; i < r1; ++i) p[i & 255] += a[(size_t)i * sa] * b[(size_t)i * sb];
    for (int s = 128; s >= 1; s >>= 1)
        for (int l = 0; l < s; ++l) p[l] += p[l + s];
    return p[0];
}
/* column dot product of the 9x9 Jacobi factor, fixed pairwise-tree order
 * (shim: oracle/shim/Eigen/Dense dot9) */
static double dot9(const double* r, int c0, int c1) {
    double p[9];
    for (int i = 0; i < 9; ++i) p[i] = r[i * 9 + c0] * r[i * 9 + c1];
    return (((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]))) + p[8];
}

/* a: m x 9 row-major (modified). Writes V column of the smallest singular value. */
static void svd_null_vector(double* a, int m, double* hv) {
    enum { N = 9 };
    double r[N * N];
    memset(r, 0, sizeof r);
    if (m > N) {
        /* Householder step j, sums below the diagonal in the canonical
         * blocked order, diagonal terms separately (shim) */
        for (int j = 0; j < N; ++j) {
            const double S = dot_blocked(a + j, N, a + j, N, j + 1, m);
            const double alpha = a[(size_t)j * N + j];
            const double normx = sqrt(alpha * alpha + S);
            if (normx == 0.0) continue;
            const double beta = alpha >= 0.0 ? -normx : normx;
            const double v0 = alpha - beta;
            const double vn2 = v0 * v0 + S;
            for (int k = j + 1; k < N; ++k) {
                const double f = 2.0 * (v0 * a[(size_t)j * N + k] + dot_blocked(a + j, N, a + k, N, j + 1, m)) / vn2;
                a[(size_t)j * N + k] = a[(size_t)j * N + k] - f * v0;
                for (int i = j + 1; i < m; ++i) a[(size_t)i * N + k] = a[(size_t)i * N + k] - f * a[(size_t)i * N + j];
            }
            a[(size_t)j * N + j] = beta;
            for (int i = j + 1; i < m; ++i) a[(size_t)i * N + j] = 0.0;
        }
        for (int i = 0; i < N; ++i)
            for (int k = 0; k < N; ++k) r[i * N + k] = k < i ? 0.0 : a[(size_t)i * N + k];
    } else {
        for (int i = 0; i < m; ++i)
            for (int k = 0; k < N; ++k) r[i * N + k] = a[(size_t)i * N + k];
    }
    double V[N * N];
    memset(V, 0, sizeof V);
    for (int i = 0; i < N; ++i) V[i * N + i] = 1.0;
    const double eps2 = 1e-30;
    for (int sweep = 0; sweep < 60; ++sweep) {
        int rotated = 0;
        /* round-robin ordering (shim: oracle/shim/Eigen/Dense) */
        for (int rnd = 0; rnd < 9; ++rnd)
            for (int kk = 1; kk <= 4; ++kk) {
                int p = (rnd + kk) % 9, q = (rnd - kk + 9) % 9;
                if (p > q) {
                    const int tmp = p;
                    p = q;
                    q = tmp;
                }
                const double al = dot9(r, p, p), be = dot9(r, q, q), ga = dot9(r, p, q);
                if (ga == 0.0 || ga * ga <= eps2 * (al * be) || fabs(ga) <= 2.220446049250313e-16 * fmax(al, be))
                    continue;
                rotated = 1;
                /* tan = sgn(d) 2g / (|d| + hypot(d, 2g)), d = be - al (shim) */
                const double d = be - al, g2 = 2.0 * ga;
                const double u = fabs(d) + sqrt(d * d + g2 * g2);
                const double w = sqrt(u * u + g2 * g2);
                const double c = u / w;
                const double s = (d >= 0.0 ? g2 : -g2) / w;
                for (int i = 0; i < N; ++i) {
                    const double up = r[i * N + p], uq = r[i * N + q];
                    r[i * N + p] = c * up - s * uq;
                    r[i * N + q] = s * up + c * uq;
                }
                for (int i = 0; i < N; ++i) {
                    const double vp = V[i * N + p], vq = V[i * N + q];
                    V[i * N + p] = c * vp - s * vq;
                    V[i * N + q] = s * vp + c * vq;
                }
            }
        if (!rotated) break;
    }
    double sv[N];
    for (int j = 0; j < N; ++j) sv[j] = sqrt(dot9(r, j, j));
    /* stable descending order; take the last column */
    int order[N];
    for (int i = 0; i < N; ++i) order[i] = i;
    for (int i = 1; i < N; ++i) { /* insertion sort = stable */
        int x = order[i], j = i - 1;
        while (j >= 0 && sv[x] > sv[order[j]]) {
            order[j + 1] = order[j];
            --j;
        }
        order[j + 1] = x;
    }
    for (int i = 0; i < N; ++i) hv[i] = V[i * N + order[N - 1]];
}

/* shim Matrix3d ops (oracle/shim/Eigen/Dense) used at homography.hpp:130-137 */
static void m3_mul(const double* a, const double* b, double* o) {
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += a[r * 3 + k] * b[k * 3 + c];
            o[r * 3 + c] = s;
        }
}
static void m3_inverse(const double* m, double* inv) {
#define M(r, c) m[(r) * 3 + (c)]
    double cof[9];
    cof[0] = M(1, 1) * M(2, 2) - M(1, 2) * M(2, 1);
    cof[1] = M(1, 2) * M(2, 0) - M(1, 0) * M(2, 2);
    cof[2] = M(1, 0) * M(2, 1) - M(1, 1) * M(2, 0);
    cof[3] = M(0, 2) * M(2, 1) - M(0, 1) * M(2, 2);
    cof[4] = M(0, 0) * M(2, 2) - M(0, 2) * M(2, 0);
    cof[5] = M(0, 1) * M(2, 0) - M(0, 0) * M(2, 1);
    cof[6] = M(0, 1) * M(1, 2) - M(0, 2) * M(1, 1);
    cof[7] = M(0, 2) * M(1, 0) - M(0, 0) * M(1, 2);
    cof[8] = M(0, 0) * M(1, 1) - M(0, 1) * M(1, 0);
    const double det = M(0, 0) * cof[0] + M(0, 1) * cof[1] + M(0, 2) * cof[2];
#undef M
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) inv[r * 3 + c] = cof[c * 3 + r] / det;
}

/* hartley_normalizer, homography.hpp:81-97 (sequential sums) */
typedef struct { double cx, cy, scale; } norm_t;
static norm_t hartley(const lp_corr* p, int n, int src) {
    norm_t q = {0, 0, 1};
    for (int i = 0; i < n; ++i) {
        q.cx += src ? p[i].sx : p[i].dx;
        q.cy += src ? p[i].sy : p[i].dy;
    }
    q.cx /= (double)n;
    q.cy /= (double)n;
    double md = 0;
    for (int i = 0; i < n; ++i) {
        double x = (src ? p[i].sx : p[i].dx) - q.cx, y = (src ? p[i].sy : p[i].dy) - q.cy;
        md += sqrt(x * x + y * y);
    }
    md /= (double)n;
    q.scale = md > 1e-12 ? sqrt(2.0) / md : 1.0;
    return q;
}
/* three_collinear, homography.hpp:99-108 */
static int three_collinear(const lp_corr* p, int n) {
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j)
            for (int k = j + 1; k < n; ++k) {
                double cross = (p[j].sx - p[i].sx) * (p[k].sy - p[i].sy) -
                               (p[j].sy - p[i].sy) * (p[k].sx - p[i].sx);
                if (fabs(cross) < 1e-9) return 1;
            }
    return 0;
}

/* dlt_homography, homography.hpp:114-144 */
int orc_dlt_homography(const lp_corr* p, int n, lp_homography* out) {
    if (n < 4) return fail(LP_INSUFFICIENT_MATCHES, "dlt: need at least 4 pairs");
    if (n == 4 && three_collinear(p, n))
        return fail(LP_DEGENERATE_CONFIGURATION, "dlt: 3 collinear source points");
    const norm_t ns = hartley(p, n, 1), nd = hartley(p, n, 0);
    double* a = xcalloc((size_t)2 * n * 9, sizeof(double));
    for (int i = 0; i < n; ++i) {
        const double x = (p[i].sx - ns.cx) * ns.scale, y = (p[i].sy - ns.cy) * ns.scale;
        const double u = (p[i].dx - nd.cx) * nd.scale, v = (p[i].dy - nd.cy) * nd.scale;
        double* r0 = a + (size_t)(2 * i) * 9;
        double* r1 = r0 + 9;
        r0[0] = -x; r0[1] = -y; r0[2] = -1; r0[3] = 0; r0[4] = 0; r0[5] = 0;
        r0[6] = u * x; r0[7] = u * y; r0[8] = u;
        r1[0] = 0; r1[1] = 0; r1[2] = 0; r1[3] = -x; r1[4] = -y; r1[5] = -1;
        r1[6] = v * x; r1[7] = v * y; r1[8] = v;
    }
    double hv[9];
    svd_null_vector(a, 2 * n, hv);
    free(a);
    const double ts[9] = {ns.scale, 0, -ns.scale * ns.cx, 0, ns.scale, -ns.scale * ns.cy, 0, 0, 1};
    const double td[9] = {nd.scale, 0, -nd.scale * nd.cx, 0, nd.scale, -nd.scale * nd.cy, 0, 0, 1};
    double tdi[9], t1[9], hm[9];
    m3_inverse(td, tdi);
    m3_mul(tdi, hv, t1);
    m3_mul(t1, ts, hm);
    if (fabs(hm[8]) < 1e-12) return fail(LP_NUMERICAL_FAILURE, "dlt: h33 vanished");
    const double s = hm[8];
    for (int i = 0; i < 9; ++i) hm[i] /= s;
    if (fabs(h_det(hm)) < 1e-9) return fail(LP_DEGENERATE_CONFIGURATION, "dlt: singular homography");
    memcpy(out->h, hm, sizeof hm);
    return LP_OK;
}

/* symmetric_transfer_error, homography.hpp:147-152 */
static double ste(const double* h, const double* hi, const lp_corr* c) {
    double fx, fy, bx, by;
    h_apply(h, c->sx, c->sy, &fx, &fy);
    h_apply(hi, c->dx, c->dy, &bx, &by);
    return hypot(fx - c->dx, fy - c->dy) + hypot(bx - c->sx, by - c->sy);
}

int orc_symmetric_transfer_errors(const lp_homography* h, const lp_homography* hi, const lp_corr* c, int n,
                                  double* out) {
    for (int i = 0; i < n; ++i) out[i] = ste(h->h, hi->h, c + i);
    return LP_OK;
}

/* prosac_homography, homography.hpp:182-286 */
int orc_prosac_homography(const lp_corr* m, int n, const lp_prosac_config* cfg,
                          lp_homography* model, uint8_t* mask_out, int* inlier_count,
                          int* iterations, int* trace_pool, int* trace_samples) {
    enum { KS = 4 };
    *iterations = 0;
    if (n < KS) return fail(LP_INSUFFICIENT_MATCHES, "prosac: need at least 4 matches");
    mt64 rng;
    mt64_seed(&rng, cfg->seed);
    double t_n = cfg->t_total;
    for (int i = 0; i < KS; ++i) t_n *= (double)(KS - i) / (n - i);
    double t_n_prime = 1.0;
    int pool = cfg->sampling == 0 ? KS : n;
    double best_h[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    int best_count = 0;
    double best_err = 0.0;
    uint8_t* best_mask = xcalloc((size_t)n, 1);
    uint8_t* mask = xcalloc((size_t)n, 1);
    int sample[KS] = {0, 0, 0, 0};
    for (int t = 1; t <= cfg->max_iter; ++t) {
        while (cfg->sampling == 0 && pool < n && (double)t > t_n_prime) {
            double t_next = t_n * (double)(pool + 1) / (pool + 1 - KS);
            t_n_prime += ceil(t_next - t_n);
            t_n = t_next;
            ++pool;
        }
        for (int i = 0; i < KS; ++i)
            for (;;) {
                int v = uid_int(&rng, 0, pool - 1);
                int dup = 0;
                for (int j = 0; j < i; ++j) dup |= sample[j] == v;
                if (!dup) {
                    sample[i] = v;
                    break;
                }
            }
        if (trace_pool) trace_pool[t - 1] = pool;
        if (trace_samples)
            for (int j = 0; j < KS; ++j) trace_samples[4 * (t - 1) + j] = sample[j];
        *iterations = t;
        lp_corr mini[KS] = {m[sample[0]], m[sample[1]], m[sample[2]], m[sample[3]]};
        lp_homography h;
        double hi[9];
        if (orc_dlt_homography(mini, KS, &h) != LP_OK) continue;
        if (h_inverse(h.h, hi) != LP_OK) continue;
        int count = 0;
        double err = 0.0;
        for (int i = 0; i < n; ++i) {
            double e = ste(h.h, hi, &m[i]);
            mask[i] = e <= cfg->threshold_px;
            if (mask[i]) {
                ++count;
                err += e;
            }
        }
        if (count > best_count || (count == best_count && count > 0 && err < best_err)) {
            memcpy(best_h, h.h, sizeof best_h);
            best_count = count;
            memcpy(best_mask, mask, (size_t)n);
            best_err = err;
        }
        if (best_count >= KS) {
            double w = (double)best_count / n;
            double p_fail = 1.0 - pow(w, KS);
            if (p_fail < 1e-12 || (double)t * log(p_fail) <= log(1.0 - cfg->confidence)) break;
        }
    }
    int rc = LP_OK;
    if (best_count < KS) {
        rc = fail(LP_NO_MODEL_FOUND, "prosac: no hypothesis with >= 4 inliers");
        goto done;
    }
    {
        lp_corr* in = xcalloc((size_t)best_count, sizeof(lp_corr));
        int k = 0;
        for (int i = 0; i < n; ++i)
            if (best_mask[i]) in[k++] = m[i];
        lp_homography refit;
        double ri[9];
        if (orc_dlt_homography(in, k, &refit) == LP_OK && h_inverse(refit.h, ri) == LP_OK) {
            memcpy(best_h, refit.h, sizeof best_h);
            best_count = 0;
            for (int i = 0; i < n; ++i) {
                best_mask[i] = ste(refit.h, ri, &m[i]) <= cfg->threshold_px;
                if (best_mask[i]) ++best_count;
            }
        }
        free(in);
    }
    if (best_count < KS) {
        rc = fail(LP_NO_MODEL_FOUND, "prosac: refit lost the consensus");
        goto done;
    }
    memcpy(model->h, best_h, sizeof best_h);
    memcpy(mask_out, best_mask, (size_t)n);
    *inlier_count = best_count;
done:
    free(best_mask);
    free(mask);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* compute_canvas, compose.hpp:32-68 */
int orc_compute_canvas(const int* dims, const lp_homography* hs, int n, lp_canvas* out,
                       int* offsets) {
    if (n < 1) return fail(LP_BAD_PARAMS, "compute_canvas: dims/homographies size mismatch");
    double minx = 1.7976931348623157e308, miny = minx, maxx = -1.7976931348623157e308, maxy = maxx;
    for (int i = 0; i < n; ++i) {
        if (fabs(h_det(hs[i].h)) < 1e-9) return fail(LP_SINGULAR_HOMOGRAPHY, "compute_canvas: singular homography");
        const double w = dims[2 * i], h = dims[2 * i + 1];
        const double cs[4][2] = {{0, 0}, {w, 0}, {0, h}, {w, h}};
        double cminx = 1.7976931348623157e308, cminy = cminx;
        for (int k = 0; k < 4; ++k) {
            double x, y;
            h_apply(hs[i].h, cs[k][0], cs[k][1], &x, &y);
            minx = (x < minx) ? x : minx; /* std::min */
            miny = (y < miny) ? y : miny;
            maxx = (maxx < x) ? x : maxx;
            maxy = (maxy < y) ? y : maxy;
            cminx = (x < cminx) ? x : cminx;
            cminy = (y < cminy) ? y : cminy;
        }
        if (offsets) {
            offsets[2 * i] = (int)floor(cminx);
            offsets[2 * i + 1] = (int)floor(cminy);
        }
    }
    out->origin_x = (int)floor(minx);
    out->origin_y = (int)floor(miny);
    out->width = (int)ceil(maxx) - out->origin_x;
    out->height = (int)ceil(maxy) - out->origin_y;
    if (offsets)
        for (int i = 0; i < n; ++i) {
            offsets[2 * i] -= out->origin_x;
            offsets[2 * i + 1] -= out->origin_y;
        }
    return LP_OK;
}

/* warp_image, compose.hpp:72-95: FP64 inverse map + bilinear with clamped taps */
int orc_warp_image(const float* img, int w, int h, int ch, const lp_homography* hom,
                   const lp_canvas* cv, float* out, float* cov) {
    if (fabs(h_det(hom->h)) < 1e-9) return fail(LP_SINGULAR_HOMOGRAPHY, "warp_image: singular homography");
    double hi[9];
    int st = h_inverse(hom->h, hi);
    if (st) return st;
    const int W = cv->width, H = cv->height;
    memset(out, 0, sizeof(float) * (size_t)W * H * ch);
    memset(cov, 0, sizeof(float) * (size_t)W * H);
#define AT(X, Y, C) img[((size_t)((Y) < 0 ? 0 : ((Y) >= h ? h - 1 : (Y))) * w + \
                         ((X) < 0 ? 0 : ((X) >= w ? w - 1 : (X)))) * ch + (C)]
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            double sx, sy;
            h_apply(hi, x + cv->origin_x, y + cv->origin_y, &sx, &sy);
            if (sx < 0.0 || sx > w - 1 || sy < 0.0 || sy > h - 1) continue;
            const int x0 = (int)sx, y0 = (int)sy;
            const double ax = sx - x0, ay = sy - y0;
            for (int c = 0; c < ch; ++c) {
                double v00 = AT(x0, y0, c), v10 = AT(x0 + 1, y0, c);
                double v01 = AT(x0, y0 + 1, c), v11 = AT(x0 + 1, y0 + 1, c);
                out[((size_t)y * W + x) * ch + c] =
                    (float)((1 - ay) * ((1 - ax) * v00 + ax * v10) + ay * ((1 - ax) * v01 + ax * v11));
            }
            cov[(size_t)y * W + x] = 1.0f;
        }
#undef AT
    return LP_OK;
}

/* linear_seam_mask, compose.hpp:101-131 */
int orc_linear_seam_mask(const float* covs, int n, int w, int h, float* masks) {
    if (n < 1) return fail(LP_BAD_PARAMS, "linear_seam_mask: no coverage masks");
    for (int c = 0; c < n; ++c) {
        const float* cov = covs + (size_t)c * w * h;
        float* dist = masks + (size_t)c * w * h;
        for (int y = 0; y < h; ++y) {
            float d = 0.0f;
            for (int x = 0; x < w; ++x) {
                d = cov[(size_t)y * w + x] > 0.0f ? d + 1.0f : 0.0f;
                dist[(size_t)y * w + x] = d;
            }
            d = 0.0f;
            for (int x = w - 1; x >= 0; --x) {
                d = cov[(size_t)y * w + x] > 0.0f ? d + 1.0f : 0.0f;
                float cur = dist[(size_t)y * w + x];
                dist[(size_t)y * w + x] = d < cur ? d : cur; /* std::min(cur, d) */
            }
        }
    }
    for (size_t i = 0; i < (size_t)w * h; ++i) {
        float sum = 0.0f;
        for (int c = 0; c < n; ++c) sum += masks[(size_t)c * w * h + i];
        if (sum > 0.0f)
            for (int c = 0; c < n; ++c) masks[(size_t)c * w * h + i] /= sum;
    }
    return LP_OK;
}

/* downsample, imgops.hpp:106-116 */
int orc_downsample(const float* in, int w, int h, int ch, float* out) {
    if (w < 2 || h < 2) return fail(LP_IMAGE_TOO_SMALL, "downsample: need at least 2x2");
    float* bl = xcalloc((size_t)w * h * ch, sizeof(float));
    int st = orc_gaussian_blur(in, w, h, ch, 1.0f, bl);
    const int ow = w / 2, oh = h / 2;
    for (int y = 0; y < oh; ++y)
        for (int x = 0; x < ow; ++x)
            for (int c = 0; c < ch; ++c)
                out[((size_t)y * ow + x) * ch + c] = bl[((size_t)(2 * y) * w + 2 * x) * ch + c];
    free(bl);
    return st;
}

/* upsample, imgops.hpp:119-140: bilinear, align-corners float scale */
int orc_upsample(const float* in, int w, int h, int ch, int tw, int th, float* out) {
    if (abs(tw - 2 * w) > 1 || abs(th - 2 * h) > 1)
        return fail(LP_BAD_TARGET_DIMS, "upsample: target dims must be ~2x source");
    const float sx = tw > 1 ? (float)(w - 1) / (float)(tw - 1) : 0.0f;
    const float sy = th > 1 ? (float)(h - 1) / (float)(th - 1) : 0.0f;
#define AT(X, Y, C) in[((size_t)((Y) < 0 ? 0 : ((Y) >= h ? h - 1 : (Y))) * w + \
                        ((X) < 0 ? 0 : ((X) >= w ? w - 1 : (X)))) * ch + (C)]
    for (int y = 0; y < th; ++y)
        for (int x = 0; x < tw; ++x) {
            float fx = (float)x * sx, fy = (float)y * sy;
            int x0 = (int)fx, y0 = (int)fy;
            float ax = fx - (float)x0, ay = fy - (float)y0;
            for (int c = 0; c < ch; ++c) {
                float v00 = AT(x0, y0, c), v10 = AT(x0 + 1, y0, c);
                float v01 = AT(x0, y0 + 1, c), v11 = AT(x0 + 1, y0 + 1, c);
                out[((size_t)y * tw + x) * ch + c] =
                    (1 - ay) * ((1 - ax) * v00 + ax * v10) + ay * ((1 - ax) * v01 + ax * v11);
            }
        }
#undef AT
    return LP_OK;
}

static size_t pyr_total(int w, int h, int ch, int levels) {
    size_t s = 0;
    for (int k = 0; k < levels; ++k) {
        s += (size_t)w * h * ch;
        w /= 2;
        h /= 2;
    }
    return s;
}

/* gaussian_pyramid, imgops.hpp:142-153 (packed, level 0 first) */
int orc_gaussian_pyramid(const float* in, int w, int h, int ch, int levels, float* out) {
    if (levels < 1) return fail(LP_TOO_MANY_LEVELS, "pyramid: levels must be >= 1");
    memcpy(out, in, sizeof(float) * (size_t)w * h * ch);
    float* prev = out;
    for (int i = 1; i < levels; ++i) {
        if (w < 2 || h < 2) return fail(LP_TOO_MANY_LEVELS, "pyramid: image too small for requested levels");
        float* next = prev + (size_t)w * h * ch;
        int st = orc_downsample(prev, w, h, ch, next);
        if (st) return st;
        prev = next;
        w /= 2;
        h /= 2;
    }
    return LP_OK;
}

/* build_laplacian, compose.hpp:134-147 */
int orc_build_laplacian(const float* in, int w, int h, int ch, int levels, float* out) {
    if (levels < 1) return fail(LP_TOO_MANY_LEVELS, "build_laplacian: levels must be >= 1");
    int st = orc_gaussian_pyramid(in, w, h, ch, levels, out);
    if (st) return st;
    float* lv = out;
    int lw = w, lh = h;
    for (int k = 0; k + 1 < levels; ++k) {
        float* nx = lv + (size_t)lw * lh * ch;
        float* up = xcalloc((size_t)lw * lh * ch, sizeof(float));
        st = orc_upsample(nx, lw / 2, lh / 2, ch, lw, lh, up);
        for (size_t i = 0; i < (size_t)lw * lh * ch; ++i) lv[i] -= up[i];
        free(up);
        if (st) return st;
        lv = nx;
        lw /= 2;
        lh /= 2;
    }
    return LP_OK;
}

/* collapse_laplacian, compose.hpp:149-158 */
int orc_collapse_laplacian(const float* packed, int w, int h, int ch, int levels, float* out) {
    if (levels < 1) return fail(LP_TOO_MANY_LEVELS, "collapse_laplacian: empty pyramid");
    const float* lv[32];
    int dw[32], dh[32];
    const float* p = packed;
    int lw = w, lh = h;
    for (int k = 0; k < levels; ++k) {
        lv[k] = p;
        dw[k] = lw;
        dh[k] = lh;
        p += (size_t)lw * lh * ch;
        lw /= 2;
        lh /= 2;
    }
    float* acc = xcalloc((size_t)dw[levels - 1] * dh[levels - 1] * ch, sizeof(float));
    memcpy(acc, lv[levels - 1], sizeof(float) * (size_t)dw[levels - 1] * dh[levels - 1] * ch);
    for (int k = levels - 2; k >= 0; --k) {
        float* up = xcalloc((size_t)dw[k] * dh[k] * ch, sizeof(float));
        int st = orc_upsample(acc, dw[k + 1], dh[k + 1], ch, dw[k], dh[k], up);
        free(acc);
        if (st) { free(up); return st; }
        for (size_t i = 0; i < (size_t)dw[k] * dh[k] * ch; ++i) up[i] = lv[k][i] + up[i];
        acc = up;
    }
    memcpy(out, acc, sizeof(float) * (size_t)w * h * ch);
    free(acc);
    return LP_OK;
}

static uint8_t to_u8(float v) { /* image.hpp:66-71 */
    float r = roundf(v);
    if (r < 0.0f) r = 0.0f;
    if (r > 255.0f) r = 255.0f;
    return (uint8_t)r;
}

/* multiband_blend, compose.hpp:162-215 */
int orc_multiband_blend(const float* images, const float* masks, int n, int w, int h, int ch,
                        int levels, uint8_t* out) {
    if (n < 1) return fail(LP_MASK_MISMATCH, "multiband_blend: image/mask count mismatch");
    if (levels < 1) return fail(LP_TOO_MANY_LEVELS, "build_laplacian: levels must be >= 1");
    const size_t tot = pyr_total(w, h, ch, levels), totm = pyr_total(w, h, 1, levels);
    float* lap = xcalloc(tot, sizeof(float));
    float* mp = xcalloc(totm, sizeof(float));
    float* acc = xcalloc(tot, sizeof(float));
    float* wsum = xcalloc(totm, sizeof(float));
    int st = LP_OK;
    for (int c = 0; c < n && !st; ++c) {
        st = orc_build_laplacian(images + (size_t)c * w * h * ch, w, h, ch, levels, lap);
        if (!st) st = orc_gaussian_pyramid(masks + (size_t)c * w * h, w, h, 1, levels, mp);
        if (st) break;
        size_t off = 0, offm = 0;
        int lw = w, lh = h;
        for (int k = 0; k < levels; ++k) {
            for (size_t i = 0; i < (size_t)lw * lh; ++i) {
                float wgt = mp[offm + i];
                wsum[offm + i] += wgt;
                for (int cc = 0; cc < ch; ++cc) acc[off + i * ch + cc] += wgt * lap[off + i * ch + cc];
            }
            off += (size_t)lw * lh * ch;
            offm += (size_t)lw * lh;
            lw /= 2;
            lh /= 2;
        }
    }
    if (!st) {
        size_t off = 0, offm = 0;
        int lw = w, lh = h;
        for (int k = 0; k < levels; ++k) {
            for (size_t i = 0; i < (size_t)lw * lh; ++i) {
                float s = wsum[offm + i];
                if (s > 1e-6f && fabsf(s - 1.0f) > 1e-6f)
                    for (int cc = 0; cc < ch; ++cc) acc[off + i * ch + cc] /= s;
            }
            off += (size_t)lw * lh * ch;
            offm += (size_t)lw * lh;
            lw /= 2;
            lh /= 2;
        }
        float* col = xcalloc((size_t)w * h * ch, sizeof(float));
        st = orc_collapse_laplacian(acc, w, h, ch, levels, col);
        for (size_t i = 0; i < (size_t)w * h && !st; ++i) {
            float covered = 0.0f;
            for (int c = 0; c < n; ++c) covered += masks[(size_t)c * w * h + i];
            for (int cc = 0; cc < ch; ++cc) out[i * ch + cc] = covered > 0.0f ? to_u8(col[i * ch + cc]) : 0;
        }
        free(col);
    }
    free(lap);
    free(mp);
    free(acc);
    free(wsum);
    return st;
}

/* ------------------------------------------------------------------------ */
/* One frame through StitchEngine's serial stage bodies (pipeline.hpp:391-521)
 * with identity pre-transforms and no crop, as the BASELINE configs use. */
int orc_stitch_frame(int ncams, int w, int h, const lp_params* P, const uint8_t* const* images,
                     uint64_t frame_index, lp_frame_out* out) {
    int rc = LP_OK;
    const lp_extraction_config* ec = &P->extraction;
    int vst = validate_ext(ec);
    if (vst) return vst;
    if (ncams < 1) return fail(LP_BAD_PARAMS, "stitch engine: no cameras");
    if (P->homography_refresh < 1) return fail(LP_BAD_PARAMS, "homography cache: K must be >= 1");
    const int n_d = ec->n_d, W2 = 2 * ((n_d + 63) / 64), top = ec->top_n;
    /* StitchEngine ctor: brief_pattern(n_d, patch_half, params.seed), pipeline.hpp:345 */
    lp_pair* pat = xcalloc((size_t)n_d, sizeof(lp_pair));
    int* dims = xcalloc((size_t)2 * ncams, sizeof(int));
    lp_region* regions = xcalloc((size_t)2 * ncams + 2, sizeof(lp_region));
    lp_keypoint** kps = xcalloc((size_t)ncams, sizeof(void*));
    uint64_t** descs = xcalloc((size_t)ncams, sizeof(void*));
    int* nkp = xcalloc((size_t)ncams, sizeof(int));
    lp_homography* chain = xcalloc((size_t)ncams, sizeof(lp_homography));
    float *warped = NULL, *cov = NULL, *masks = NULL;
    lp_match* matches = NULL;
    lp_corr* corr = NULL;
    uint8_t* pano = NULL;
    TRY(orc_brief_pattern(n_d, ec->patch_half, P->seed, pat));
    for (int c = 0; c < ncams; ++c) {
        dims[2 * c] = w;
        dims[2 * c + 1] = h;
    }
    /* stage_rectify_crop, pipeline.hpp:391-417 */
    int nreg = 0;
    TRY(orc_partition_regions(dims, ncams, P->overlap_fraction, ec->patch_half, regions,
                              2 * ncams + 2, &nreg));
    /* stage_detect, pipeline.hpp:419-442 */
    for (int c = 0; c < ncams; ++c) {
        kps[c] = xcalloc((size_t)2 * top, sizeof(lp_keypoint));
        descs[c] = xcalloc((size_t)2 * top * W2, sizeof(uint64_t));
        for (int ri = 0; ri < nreg; ++ri) {
            if (regions[ri].camera_id != c) continue;
            int ns = 0;
            TRY(detect_region(images[c], w, h, regions[ri], ri, ec, kps[c] + nkp[c], &ns));
            nkp[c] += ns;
        }
    }
    /* stage_describe, pipeline.hpp:444-469 */
    for (int c = 0; c < ncams; ++c)
        for (int ri = 0; ri < nreg; ++ri) {
            if (regions[ri].camera_id != c) continue;
            int any = 0;
            for (int i = 0; i < nkp[c]; ++i) any |= kps[c][i].region_id == ri;
            if (!any) continue;
            crop_t cr;
            TRY(smoothed_crop(images[c], w, h, regions[ri], ec->patch_half, ec->brief_blur_sigma, &cr));
            for (int i = 0; i < nkp[c] && rc == LP_OK; ++i) {
                if (kps[c][i].region_id != ri) continue;
                lp_keypoint local = {kps[c][i].x - cr.ox, kps[c][i].y - cr.oy, kps[c][i].response, ri};
                rc = brief_one(cr.img, cr.w, cr.h, local, pat, n_d, ec->patch_half, descs[c] + (size_t)i * W2);
            }
            free(cr.img);
            if (rc) goto done;
        }
    /* stage_match_estimate, pipeline.hpp:471-497, through a fresh
     * HomographyCache (259-286): the estimator always runs; if it throws the
     * cache is empty and NoValidHomographyYet is raised. */
    matches = xcalloc((size_t)2 * top + 1, sizeof(lp_match));
    corr = xcalloc((size_t)2 * top + 1, sizeof(lp_corr));
    memset(chain, 0, sizeof(lp_homography) * ncams);
    chain[0].h[0] = chain[0].h[4] = chain[0].h[8] = 1.0;
    for (int i = 0; i + 1 < ncams; ++i) {
        int nm = 0;
        int st = orc_match_features(descs[i + 1], nkp[i + 1], descs[i], nkp[i], n_d, &P->matching,
                                    matches, 2 * top + 1, &nm);
        if (st == LP_OK) {
            if (out->match_counts) out->match_counts[i] = nm;
            for (int k = 0; k < nm && out->matches && k < out->cap_matches; ++k)
                out->matches[(size_t)i * out->cap_matches + k] = matches[k];
            for (int k = 0; k < nm; ++k) {
                const lp_keypoint* s = &kps[i + 1][matches[k].query_id];
                const lp_keypoint* d = &kps[i][matches[k].train_id];
                lp_corr cc = {(double)s->x, (double)s->y, (double)d->x, (double)d->y, matches[k].quality, 0};
                corr[k] = cc;
            }
            lp_prosac_config pc = P->prosac;
            pc.seed = P->seed ^ (frame_index * 0x9e3779b97f4a7c15ULL + (uint64_t)i);
            lp_homography hm;
            uint8_t* msk = xcalloc((size_t)nm + 1, 1);
            int cnt = 0, its = 0;
            st = orc_prosac_homography(corr, nm, &pc, &hm, msk, &cnt, &its, NULL, NULL);
            free(msk);
            if (st == LP_OK) h_compose(chain[i].h, hm.h, chain[i + 1].h);
        }
        if (st != LP_OK) {
            rc = fail(LP_NO_VALID_HOMOGRAPHY_YET, "no homography cached yet");
            goto done;
        }
    }
    /* stage_warp_blend, pipeline.hpp:499-521 */
    {
        lp_canvas cv;
        TRY(orc_compute_canvas(dims, chain, ncams, &cv, NULL));
        const size_t np = (size_t)cv.width * cv.height;
        warped = xcalloc(np * ncams, sizeof(float));
        cov = xcalloc(np * ncams, sizeof(float));
        masks = xcalloc(np * ncams, sizeof(float));
        float* f32 = xcalloc((size_t)w * h, sizeof(float));
        for (int c = 0; c < ncams && rc == LP_OK; ++c) {
            for (size_t i = 0; i < (size_t)w * h; ++i) f32[i] = images[c][i];
            rc = orc_warp_image(f32, w, h, 1, &chain[c], &cv, warped + np * c, cov + np * c);
        }
        free(f32);
        if (rc) goto done;
        TRY(orc_linear_seam_mask(cov, ncams, cv.width, cv.height, masks));
        int levels = P->blend_levels;
        while (levels > 1 && (cv.width < (1 << (levels - 1)) || cv.height < (1 << (levels - 1)))) --levels;
        pano = xcalloc(np, 1);
        TRY(orc_multiband_blend(warped, masks, ncams, cv.width, cv.height, 1, levels, pano));
        out->canvas = cv;
        if (out->panorama) {
            if (np > out->pano_cap) {
                rc = fail(LP_CAPACITY_OVERFLOW, "panorama capacity");
                goto done;
            }
            memcpy(out->panorama, pano, np);
        }
    }
    for (int c = 0; c < ncams; ++c) {
        if (out->kp_counts) out->kp_counts[c] = nkp[c];
        for (int i = 0; i < nkp[c] && i < out->cap_kp; ++i) {
            if (out->keypoints) out->keypoints[(size_t)c * out->cap_kp + i] = kps[c][i];
            if (out->descriptors)
                memcpy(out->descriptors + ((size_t)c * out->cap_kp + i) * W2, descs[c] + (size_t)i * W2,
                       sizeof(uint64_t) * W2);
        }
        if (out->homographies) out->homographies[c] = chain[c];
    }
    out->estimated = 1;
done:
    for (int c = 0; c < ncams; ++c) {
        free(kps[c]);
        free(descs[c]);
    }
    free(pat);
    free(dims);
    free(regions);
    free(kps);
    free(descs);
    free(nkp);
    free(chain);
    free(warped);
    free(cov);
    free(masks);
    free(matches);
    free(corr);
    free(pano);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Synthetic inputs, synth.hpp:18-115 (the BASELINE configs' generators).    */
static uint8_t to_u8_c(float v) { return to_u8(v); }

int orc_synth_texture(int w, int h, uint64_t seed, float smooth_sigma, uint8_t* out) {
    mt64 rng;
    mt64_seed(&rng, seed);
    const size_t n = (size_t)w * h;
    float* noise = xcalloc(n, sizeof(float));
    float* bl = xcalloc(n, sizeof(float));
    for (size_t i = 0; i < n; ++i) noise[i] = (float)(mt64_next(&rng) % 256);
    int st = orc_gaussian_blur(noise, w, h, 1, smooth_sigma, bl);
    if (st) { free(noise); free(bl); return st; }
    float lo = bl[0], hi = bl[0];
    for (size_t i = 0; i < n; ++i) {
        lo = bl[i] < lo ? bl[i] : lo; /* std::min(lo, v) */
        hi = hi < bl[i] ? bl[i] : hi; /* std::max(hi, v) */
    }
    const float scale = hi > lo ? 255.0f / (hi - lo) : 0.0f;
    for (size_t i = 0; i < n; ++i) out[i] = to_u8_c((bl[i] - lo) * scale);
    free(noise);
    free(bl);
    return LP_OK;
}

int orc_synth_planted_pair(int w, int h, double overlap, uint64_t seed, uint8_t* left,
                           uint8_t* right, double* true_h) {
    const int shift = (int)lround(w * (1.0 - overlap));
    const int ww = w + shift;
    uint8_t* wide = xcalloc((size_t)ww * h, 1);
    int st = orc_synth_texture(ww, h, seed, 1.5f, wide);
    if (st) { free(wide); return st; }
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            left[(size_t)y * w + x] = wide[(size_t)y * ww + x];
            right[(size_t)y * w + x] = wide[(size_t)y * ww + x + shift];
        }
    const double t[9] = {1, 0, (double)shift, 0, 1, 0, 0, 0, 1};
    memcpy(true_h, t, sizeof t);
    free(wide);
    return LP_OK;
}

int orc_synth_sequence_frame(int w, int h, double overlap, uint64_t seed, uint64_t frame,
                             uint8_t* left, uint8_t* right) {
    double th[9];
    int st = orc_synth_planted_pair(w, h, overlap, seed, left, right, th);
    if (st) return st;
    const int size = imax(4, h / 16);
    const int px = (int)((frame * 7) % (uint64_t)(w - size));
    const int py = (int)((frame * 3) % (uint64_t)(h - size));
    for (int y = py; y < py + size; ++y)
        for (int x = px; x < px + size; ++x) left[(size_t)y * w + x] = 255;
    const double shift = th[2];
    for (int y = py; y < py + size; ++y)
        for (int x = px; x < px + size; ++x) {
            int rx = x - (int)shift;
            if (rx >= 0 && rx < w) right[(size_t)y * w + rx] = 255;
        }
    return LP_OK;
}

/* rotate, synth.hpp:37-60 */
int orc_synth_rotate(const uint8_t* img, int w, int h, double degrees, uint8_t* out) {
    const double rad = degrees * M_PI / 180.0;
    const double c = cos(rad), s = sin(rad);
    const double cx = (w - 1) / 2.0, cy = (h - 1) / 2.0;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            double dx = x - cx, dy = y - cy;
            double sx = c * dx + s * dy + cx;
            double sy = -s * dx + c * dy + cy;
            int x0 = (int)floor(sx), y0 = (int)floor(sy);
            double ax = sx - x0, ay = sy - y0;
#define CL(X, Y) img[(size_t)((Y) < 0 ? 0 : ((Y) >= h ? h - 1 : (Y))) * w + ((X) < 0 ? 0 : ((X) >= w ? w - 1 : (X)))]
            double v00 = CL(x0, y0), v10 = CL(x0 + 1, y0), v01 = CL(x0, y0 + 1), v11 = CL(x0 + 1, y0 + 1);
#undef CL
            out[(size_t)y * w + x] =
                to_u8_c((float)((1 - ay) * ((1 - ax) * v00 + ax * v10) + ay * ((1 - ax) * v01 + ax * v11)));
        }
    return LP_OK;
}

/* StitchEngine::stage_rectify_crop, pipeline.hpp:391-417: per camera
 * warp_image(to_f32(img), pre_transform, own canvas) + to_u8_image when the
 * pre-transform is not exactly the identity (compose.hpp:72-95,
 * image.hpp:80-85), then the crop (BadParams when outside the image). */
int orc_rectify_crop(int ncams, int w, int h, const lp_camera* cams, const uint8_t* const* images,
                     uint8_t* const* outputs, int* out_w, int* out_h) {
    static const double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    const size_t np = (size_t)w * h;
    float* f32 = (float*)malloc(sizeof(float) * np);
    float* warped = (float*)malloc(sizeof(float) * np);
    float* cov = (float*)malloc(sizeof(float) * np);
    uint8_t* tmp = (uint8_t*)malloc(np);
    int st = LP_OK;
    for (int c = 0; c < ncams && st == LP_OK; ++c) {
        int identity = 1;
        for (int j = 0; j < 9; ++j)
            if (!(cams[c].pre_transform.h[j] == I[j])) identity = 0;
        if (identity) {
            memcpy(tmp, images[c], np);
        } else {
            const lp_canvas self = {w, h, 0, 0};
            for (size_t i = 0; i < np; ++i) f32[i] = (float)images[c][i];
            st = orc_warp_image(f32, w, h, 1, &cams[c].pre_transform, &self, warped, cov);
            if (st) break;
            for (size_t i = 0; i < np; ++i) tmp[i] = to_u8(warped[i]);
        }
        int x0 = 0, y0 = 0, cw = w, ch = h;
        if (cams[c].has_crop) {
            const lp_region r = cams[c].crop;
            if (r.x0 < 0 || r.y0 < 0 || r.x1 > w || r.y1 > h || r.x1 - r.x0 < 1 || r.y1 - r.y0 < 1) {
                st = fail(LP_BAD_PARAMS, "rectify_crop: crop outside image");
                break;
            }
            x0 = r.x0;
            y0 = r.y0;
            cw = r.x1 - r.x0;
            ch = r.y1 - r.y0;
        }
        for (int y = 0; y < ch; ++y) memcpy(outputs[c] + (size_t)y * cw, tmp + (size_t)(y + y0) * w + x0, cw);
        out_w[c] = cw;
        out_h[c] = ch;
    }
    free(f32);
    free(warped);
    free(cov);
    free(tmp);
    return st;
}
