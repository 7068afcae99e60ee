/* lorbpano_b200.h — C-ABI of the B200-native stitching hot path.
 *
 * This is the drop-in boundary under the reference's C++ API
 * (/root/reference/proj/include/lorbpano/ headers). Every entry point names the
 * reference function it replaces (file:line, relative to proj/include/lorbpano/).
 * The C++ drop-in headers (paper_1810_03988_b200/include/lorbpano/) forward to
 * these functions and re-throw lp_status codes as the matching lorbpano::Error
 * subclass, so the reference's callers (StitchEngine stage bodies, CLI, tests)
 * keep their exception behaviour.
 *
 * Conventions
 *  - plain pointers + sizes, no C++ or torch types;
 *  - every pixel/feature pointer may be HOST or DEVICE memory (detected with
 *    cudaPointerGetAttributes); host buffers are staged through the context's
 *    device arena;
 *  - outputs go to caller buffers with an explicit capacity and a count out-param;
 *  - errors are returned as lp_status, never thrown across the ABI;
 *    lp_last_error() gives the message (thread-local);
 *  - images are row-major, interleaved channels (Raster<T>, image.hpp:22-60);
 *  - descriptors are packed as 2*W uint64 words per descriptor, W = ceil(n_d/64):
 *    gt[0..W) then lt[0..W) (Descriptor, lorb.hpp:45-69, without the n_d field).
 */
#ifndef LORBPANO_B200_H
#define LORBPANO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 0 = ok; 1..28 mirror the error.hpp:19-56 declaration order. */
typedef enum lp_status {
    LP_OK = 0,
    LP_FILE_NOT_FOUND = 1,
    LP_UNSUPPORTED_FORMAT = 2,
    LP_CORRUPT_DATA = 3,
    LP_INVALID_SIGMA = 4,
    LP_IMAGE_TOO_SMALL = 5,
    LP_BAD_TARGET_DIMS = 6,
    LP_NO_OVERLAP = 7,
    LP_OVERLAP_EXCEEDS_IMAGE = 8,
    LP_REGION_TOO_SMALL = 9,
    LP_WINDOW_OUT_OF_BOUNDS = 10,
    LP_PATCH_OUT_OF_BOUNDS = 11,
    LP_LENGTH_MISMATCH = 12,
    LP_BAD_PARAMS = 13,
    LP_TOO_MANY_PROBES = 14,
    LP_PARAM_MISMATCH = 15,
    LP_EMPTY_INPUT = 16,
    LP_DEGENERATE_CONFIGURATION = 17,
    LP_NUMERICAL_FAILURE = 18,
    LP_INSUFFICIENT_MATCHES = 19,
    LP_NO_MODEL_FOUND = 20,
    LP_SINGULAR_HOMOGRAPHY = 21,
    LP_MASK_MISMATCH = 22,
    LP_TOO_MANY_LEVELS = 23,
    LP_CAPACITY_OVERFLOW = 24,
    LP_NO_VALID_HOMOGRAPHY_YET = 25,
    LP_PARSE_ERROR = 26,
    LP_VALIDATION_ERROR = 27,
    LP_MISSING_FRAMES = 28,
    LP_CUDA_ERROR = 100,
    LP_NO_DEVICE = 101,
    LP_INTERNAL = 102
} lp_status;

/* ---- POD mirrors (layouts identical to the reference structs on x86-64) ---- */

/* DetectionRegion, lorb.hpp:25-32 (20 B) */
typedef struct lp_region { int x0, y0, x1, y1, camera_id; } lp_region;
/* Keypoint, lorb.hpp:17-22 (16 B) */
typedef struct lp_keypoint { int x, y; float response; int region_id; } lp_keypoint;
/* BriefPattern::Pair, lorb.hpp:35-37 (16 B) */
typedef struct lp_pair { int px, py, qx, qy; } lp_pair;
/* Match, matchlsh.hpp:16-21 (16 B) */
typedef struct lp_match { int query_id, train_id, distance; float quality; } lp_match;
/* Correspondence, homography.hpp:66-70 (40 B incl. tail padding) */
typedef struct lp_corr { double sx, sy, dx, dy; float quality; int pad_; } lp_corr;
/* Homography, homography.hpp:17-63 (72 B) */
typedef struct lp_homography { double h[9]; } lp_homography;
/* Canvas, compose.hpp:18-24 (offsets omitted: not used by warp/blend) */
typedef struct lp_canvas { int width, height, origin_x, origin_y; } lp_canvas;

/* ExtractionConfig, lorb.hpp:71-90 */
typedef struct lp_extraction_config {
    int fast_threshold; /* uint8 range */
    int fast_arc;
    float harris_alpha;
    float harris_threshold;
    float harris_sigma;
    int top_n;
    int n_d;
    float brief_blur_sigma;
    int patch_half;
} lp_extraction_config;

/* MatchConfig, matchlsh.hpp:161-168 */
typedef struct lp_match_config {
    int tables, bits, t_probes, max_distance;
    float ratio;
    int pad_;
    uint64_t seed;
} lp_match_config;

/* ProsacConfig, homography.hpp:156-163 (sampling: 0 = Prosac, 1 = Uniform) */
typedef struct lp_prosac_config {
    double threshold_px;
    int max_iter;
    int sampling;
    double confidence;
    uint64_t seed;
    double t_total;
} lp_prosac_config;

/* StitchParams (pipeline.hpp:249-255) + CameraLayout.overlap_fraction
 * (lorb.hpp:93-96) + PipelineConfig.homography_refresh (pipeline.hpp:199-204). */
typedef struct lp_params {
    lp_extraction_config extraction;
    lp_match_config matching;
    lp_prosac_config prosac;
    int blend_levels;
    int homography_refresh;
    uint64_t seed;
    double overlap_fraction;
} lp_params;

/* Fills the reference defaults (lorb.hpp:71-80, matchlsh.hpp:161-167,
 * homography.hpp:156-162, pipeline.hpp:199-204,249-255, README overlap 0.25). */
void lp_params_default(lp_params* p);

/* ---- context ---- */
typedef struct lp_ctx lp_ctx;
lp_status lp_ctx_create(int device, lp_ctx** out);
void lp_ctx_destroy(lp_ctx* ctx);
/* cudaStream_t the context enqueues on (NULL = its own stream). */
lp_status lp_ctx_set_stream(lp_ctx* ctx, void* cuda_stream);
const char* lp_last_error(void);
/* number of kernels this process launched through the library so far */
uint64_t lp_kernel_launches(void);

/* Page-locked host memory (cudaHostAlloc) for frames in flight: inputs and
 * outputs there move by DMA asynchronously; pageable ones make the copy
 * synchronous with the host. NULL on failure. */
void* lp_host_alloc(size_t bytes);
/* synth::texture (synth.hpp:17-34): the reference's seeded test/bench input
 * (mt19937_64 noise, gaussian_blur, contrast stretch), w x h u8 into out.
 * Host only, byte-identical to the reference's. */
lp_status lp_synth_texture(int w, int h, uint64_t seed, float sigma, uint8_t* out);
/* The same, write-combined (cudaHostAllocWriteCombined): for frames the host
 * writes once and only the device reads (not snooped during the copy in;
 * slow for host reads). Freed with lp_host_free. */
void* lp_host_alloc_wc(size_t bytes);
void lp_host_free(void* p);

/* ---- L-ORB primitives (lorb.hpp) ---- */

/* fast_corners, lorb.hpp:192-205: (x,y) pairs in raster order. */
lp_status lp_fast_corners(lp_ctx* ctx, const uint8_t* img, int w, int h, int channels,
                          lp_region region, int threshold, int arc, int* xy_out, int cap,
                          int* count);
/* harris_response, lorb.hpp:209-250 (FP64 accumulation, float result). */
lp_status lp_harris_response(lp_ctx* ctx, const uint8_t* img, int w, int h, int channels,
                             const int* xy, int n, float alpha, float sigma, float* out);
/* nms, lorb.hpp:254-288: survivors in input order. */
lp_status lp_nms(lp_ctx* ctx, const lp_keypoint* in, int n, int radius, lp_keypoint* out,
                 int* count);
/* select_top_n, lorb.hpp:291-299: (response desc, y asc, x asc), at most top_n. */
lp_status lp_select_top_n(lp_ctx* ctx, const lp_keypoint* in, int n, int top_n,
                          lp_keypoint* out, int* count);
/* gaussian_blur, imgops.hpp:50-72 (separable, clamp-to-edge, FP32, no FMA). */
lp_status lp_gaussian_blur(lp_ctx* ctx, const float* in, int w, int h, int channels,
                           float sigma, float* out);
/* brief_descriptor, lorb.hpp:333-350, batched over keypoints. */
lp_status lp_brief_descriptors(lp_ctx* ctx, const float* smoothed, int w, int h,
                               const lp_keypoint* kps, int n, const lp_pair* pairs, int n_d,
                               int patch_half, uint64_t* desc_out);
/* extract_features, lorb.hpp:388-413: all regions of one image in one pass. */
lp_status lp_extract_features(lp_ctx* ctx, const uint8_t* img, int w, int h, int channels,
                              const lp_region* regions, int n_regions,
                              const lp_extraction_config* cfg, const lp_pair* pairs,
                              lp_keypoint* kp_out, uint64_t* desc_out, int cap, int* count);

/* ---- matching (matchlsh.hpp) ---- */

/* query (matchlsh.hpp:132-159) of nq descriptors against the LSH index of
 * the nt train descriptors (build_index with cfg's tables / bits / seed, the
 * cfg.t_probes probe set, cfg.max_distance): for query q every hit within
 * max_distance, sorted by (distance, train id), in out[offsets[q] ..
 * offsets[q + 1]) with query_id = query_id0 + q. offsets has nq + 1 entries;
 * *total is the hit count (out holds min(total, cap)). */
lp_status lp_lsh_query(lp_ctx* ctx, const uint64_t* train, int nt, const uint64_t* queries, int nq, int n_d,
                       const lp_match_config* cfg, int query_id0, long long* offsets, lp_match* out, long long cap,
                       long long* total);
/* descriptor_distance, matchlsh.hpp:25-33, elementwise over n pairs. */
lp_status lp_descriptor_distances(lp_ctx* ctx, const uint64_t* a, const uint64_t* b, int n,
                                  int n_d, int* out);
/* match_features, matchlsh.hpp:173-193 (index on set_b, queries set_a). */
lp_status lp_match_features(lp_ctx* ctx, const uint64_t* set_a, int na, const uint64_t* set_b,
                            int nb, int n_d, const lp_match_config* cfg, lp_match* out, int cap,
                            int* count);

/* ---- homography (homography.hpp) ---- */

/* dlt_homography, homography.hpp:114-144 */
lp_status lp_dlt_homography(lp_ctx* ctx, const lp_corr* pairs, int n, lp_homography* out);
/* symmetric_transfer_error (homography.hpp:147-152) of each of n pairs:
 * |H(s) - d| + |H^-1(d) - s| with glibc's hypot, bit-identical to the
 * reference's std::hypot. */
lp_status lp_symmetric_transfer_errors(lp_ctx* ctx, const lp_homography* h, const lp_homography* h_inv,
                                       const lp_corr* pairs, int n, double* out);
/* prosac_homography, homography.hpp:182-286. trace_* optional (NULL), sized
 * max_iter and 4*max_iter; *iterations gives the filled length. */
lp_status lp_prosac_homography(lp_ctx* ctx, const lp_corr* matches, int n,
                               const lp_prosac_config* cfg, lp_homography* model,
                               uint8_t* inlier_mask, int* inlier_count, int* iterations,
                               int* trace_pool, int* trace_samples);

/* ---- compositor (compose.hpp, imgops.hpp) ---- */

/* warp_image, compose.hpp:72-95 */
lp_status lp_warp_image(lp_ctx* ctx, const float* img, int w, int h, int channels,
                        const lp_homography* hom, const lp_canvas* canvas, float* out,
                        float* coverage);
/* linear_seam_mask, compose.hpp:101-131: n packed w*h coverages -> n masks */
lp_status lp_linear_seam_mask(lp_ctx* ctx, const float* coverages, int n, int w, int h,
                              float* masks);
/* downsample / upsample, imgops.hpp:106-140 */
lp_status lp_downsample(lp_ctx* ctx, const float* in, int w, int h, int channels, float* out);
lp_status lp_upsample(lp_ctx* ctx, const float* in, int w, int h, int channels, int tw, int th,
                      float* out);
/* gaussian_pyramid (imgops.hpp:142-153), build_laplacian (compose.hpp:134-147):
 * levels packed level-0 first; dims halve with floor. */
lp_status lp_gaussian_pyramid(lp_ctx* ctx, const float* in, int w, int h, int channels,
                              int levels, float* out_packed);
lp_status lp_build_laplacian(lp_ctx* ctx, const float* in, int w, int h, int channels,
                             int levels, float* out_packed);
/* collapse_laplacian, compose.hpp:149-158 */
lp_status lp_collapse_laplacian(lp_ctx* ctx, const float* packed, int w, int h, int channels,
                                int levels, float* out);
/* multiband_blend, compose.hpp:162-215: n packed images and masks */
lp_status lp_multiband_blend(lp_ctx* ctx, const float* images, const float* masks, int n,
                             int w, int h, int channels, int levels, uint8_t* out);

/* ---- per-frame stitching engine (pipeline.hpp:419-521) ---- */

typedef struct lp_rig lp_rig;

/* Host-visible per-frame results (all pointers optional). Capacities are per
 * camera (keypoints/descriptors: cap_kp) and per pair (matches: cap_matches). */
typedef struct lp_frame_out {
    uint8_t* panorama;        /* host or device, >= pano_cap bytes */
    size_t pano_cap;
    lp_canvas canvas;         /* out */
    lp_homography* homographies; /* ncams, out (into camera-0 frame) */
    int* kp_counts;           /* ncams */
    lp_keypoint* keypoints;   /* ncams * cap_kp */
    uint64_t* descriptors;    /* ncams * cap_kp * 2W */
    int cap_kp;
    int* match_counts;        /* ncams-1 */
    lp_match* matches;        /* (ncams-1) * cap_matches */
    int cap_matches;
    int estimated;            /* out: 1 if this frame ran the estimator */
    float stage_ms[4];        /* out: detect, describe, match_estimate, warp_blend (device time) */
} lp_frame_out;

/* RigLayout::Camera (pipeline.hpp:240-247): a rectifying pre-transform
 * (identity = none) and an optional crop (DetectionRegion, camera_id unused). */
typedef struct lp_camera {
    lp_homography pre_transform;
    int has_crop;
    lp_region crop;
} lp_camera;

/* StitchEngine::stage_rectify_crop (pipeline.hpp:391-417) for one frame: per
 * camera, warp_image(to_f32(img), pre_transform, own w x h canvas) +
 * to_u8_image when pre_transform is not exactly the identity, then the crop.
 * Errors: SingularHomography (|det| < 1e-9), BadParams (crop outside image).
 * images / outputs host or device; outputs[c] receives out_w[c] x out_h[c]
 * bytes (at most w * h). */
lp_status lp_rectify_crop(lp_ctx* ctx, int ncams, int w, int h, const lp_camera* cams,
                          const uint8_t* const* images, uint8_t* const* outputs, int* out_w, int* out_h);

/* brief_pattern (lorb.hpp:303-330): the n_d test pairs the engine draws from
 * mt19937_64(seed) (StitchEngine ctor, pipeline.hpp:345). Host only. */
lp_status lp_brief_pattern(int n_d, int patch_half, uint64_t seed, lp_pair* out);

/* ---- frame ingest / egress formats ---- */
/* load_pnm (image.hpp:88-126, binary P5/P6, maxval 255): with out == NULL or
 * cap too small only the header is read into w/h/channels (returns
 * CapacityOverflow when out is non-NULL and too small). Errors as the
 * reference: FileNotFound, UnsupportedFormat, CorruptData. Host only. */
lp_status lp_load_pnm(const char* path, uint8_t* out, size_t cap, int* w, int* h, int* channels);
/* save_pnm (image.hpp:194-204): P5 for 1 channel, P6 for 3. Host only. */
lp_status lp_save_pnm(const char* path, const uint8_t* data, int w, int h, int channels);
/* The CLI sink's gray -> RGB triplication (cli.hpp:138-145) on the device:
 * rgb[3i + c] = gray[i]; gray / rgb host or device. */
lp_status lp_gray_to_rgb(lp_ctx* ctx, const uint8_t* gray, size_t n, uint8_t* rgb);

/* StitchEngine(RigLayout{ncams identity cameras, overlap}, StitchParams, K),
 * pipeline.hpp:343-350; all cameras w x h grayscale. */
lp_status lp_rig_create(lp_ctx* ctx, int ncams, int w, int h, const lp_params* params,
                        lp_rig** out);
/* The same engine over a RigLayout (pipeline.hpp:240-247): every w x h raw
 * frame passes stage_rectify_crop on the device before detection. The
 * rectified cameras must share one size (the device rig's frame geometry);
 * lp_rig_panorama_capacity and the stages use that size. */
lp_status lp_rig_create_layout(lp_ctx* ctx, int ncams, int w, int h, const lp_camera* cams,
                               const lp_params* params, lp_rig** out);
void lp_rig_destroy(lp_rig* rig);
/* A frame whose panorama did not fit the caller's buffer (pano_cap) is still
 * stitched: lp_rig_wait / lp_rig_wait_frame deliver everything else (the
 * canvas included) and return LP_CAPACITY_OVERFLOW; the panorama stays in
 * the frame's slot until the slot's next frame, and this copies it into dst
 * (host or device, cap bytes; the reference's BufferPool grows for such
 * canvases, pipeline.hpp:68-109). */
lp_status lp_rig_copy_panorama(lp_rig* rig, uint64_t ticket, uint8_t* dst, size_t cap);
/* A new StitchEngine's state on an existing rig (pipeline.hpp:343-350 with
 * the same layout and parameters): waits for the frames in flight, then
 * forgets the cached homographies (HomographyCache empty again) and every
 * per-frame record; device arenas, graphs and staging are kept. */
lp_status lp_rig_reset(lp_rig* rig);
/* One frame through detect -> describe -> match_estimate (HomographyCache,
 * pipeline.hpp:259-286) -> warp_blend. images[c] host or device. */
lp_status lp_rig_stitch(lp_rig* rig, const uint8_t* const* images, uint64_t frame_index,
                        lp_frame_out* out);
/* Compulsory bytes (inputs once + outputs once, in the kernel's data types)
 * one launch of `kernel_key` ("k_warp/0", "k_blend_level/3", ... as the
 * profiler names them) moves for the rig's last frame; < 0 if unknown. */
double lp_rig_algorithmic_bytes(lp_rig* rig, const char* kernel_key);
/* Algorithmic work of one launch of `kernel_key` by pipe, for the roofline:
 * out6[0] compulsory bytes, [1] FP64 add/mul/compare ops, [2] FP64
 * divisions + square roots, [3] FP32 ops, [4] 32-bit POPC ops, [5] SMs the
 * launch can occupy (0 = all). Launch-varying counts (Harris candidates) are
 * averaged over `launches` launches since lp_rig_work_reset. Profiling only. */
lp_status lp_rig_algorithmic_work(lp_rig* rig, const char* kernel_key, long long launches, double* out6);
lp_status lp_rig_work_reset(lp_rig* rig);

/* Failure injection (tests of the per-frame failure path): the frame
 * submitted with `frame_index` raises device status `code` on its slot, as a
 * kernel of that frame would; lp_rig_wait on its ticket returns `code`, the
 * rig's other frames are unaffected (pipeline.hpp run_stage: a failed stage
 * drops its frame into Metrics::drops and the engine carries on). */
lp_status lp_rig_inject_fault(lp_rig* rig, uint64_t frame_index, int code);

/* ---- diagnostics: per-kernel device time (CUDA events around each launch) ---- */
void lp_profile_enable(int on);
void lp_profile_reset(void);
/* fills up to cap entries: names (name_stride bytes each) "kernel/occurrence",
 * summed ms, launch count; returns the number of distinct keys */
int lp_profile_read(char* names, int name_stride, double* total_ms, long long* launches, int cap);

/* Frames in flight (the pipelined mode of StitchEngine::run_pipelined,
 * pipeline.hpp:660-711, as CUDA streams): enqueue ingest copy -> stages ->
 * panorama egress for one frame and return immediately with a ticket; up to
 * 3 frames overlap (copies in both directions run beside the stages).
 * `panorama` (host or device, may be NULL) must stay valid until
 * lp_rig_wait(ticket) returns; host buffers should be pinned for overlap. */
lp_status lp_rig_submit(lp_rig* rig, const uint8_t* const* images, uint64_t frame_index,
                        uint8_t* panorama, size_t pano_cap, uint64_t* ticket);
lp_status lp_rig_wait(lp_rig* rig, uint64_t ticket, lp_canvas* canvas);
/* Frames in flight WITH their per-frame results (StitchEngine's FramePacket,
 * pipeline.hpp:50-65): out->panorama receives the panorama as in
 * lp_rig_submit; the keypoints / descriptors / matches requested in `out`
 * are staged per frame slot and, with the canvas, the estimate flag, the
 * homographies and the device stage times, land in `out` at
 * lp_rig_wait_frame. `out` must stay valid until then; collect a ticket
 * before submitting 3 more frames (the slot is reused). */
lp_status lp_rig_submit_frame(lp_rig* rig, const uint8_t* const* images, uint64_t frame_index, lp_frame_out* out,
                              uint64_t* ticket);
lp_status lp_rig_wait_frame(lp_rig* rig, uint64_t ticket, lp_frame_out* out);

/* Egress format of lp_rig_submit / lp_rig_stitch panoramas: 1 = the PPM sink's
 * 3-channel RGB (gray triplicated on the device before the copy out,
 * cli.hpp:138-145; 3 x canvas bytes), 0 = gray (default). */
lp_status lp_rig_set_egress(lp_rig* rig, int channels_rgb);
/* Upper bound on panorama bytes for this rig's current homographies. */
size_t lp_rig_panorama_capacity(lp_rig* rig);
/* The stream the rig's work is enqueued on (cudaStream_t). */
void* lp_rig_stream(lp_rig* rig);
/* Frame scheduler: 2 (default) runs each frame's extraction, matching and
 * estimate on one of three rotating feature streams, concurrently with the
 * compositor stream; 1 runs every stage in order on the rig stream. */
lp_status lp_rig_set_streams(lp_rig* rig, int nstreams);
/* Compositor launch chain replayed as a CUDA graph per frame slot (default
 * 1); 0 launches every kernel individually. */
lp_status lp_rig_set_graphs(lp_rig* rig, int on);

#ifdef __cplusplus
}
#endif

#endif
