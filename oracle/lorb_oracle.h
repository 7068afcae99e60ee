/* lorb_oracle.h — TEST INFRASTRUCTURE ONLY: the plain-C restatement oracle.
 * Entry points are the C-ABI of include/lorbpano_b200.h with an orc_ prefix
 * and no context argument; see lorb_oracle.c for the per-function citations.
 * Pinned against the reference itself (oracle/_ref) by tests/golden. */
#ifndef LORB_ORACLE_H
#define LORB_ORACLE_H
#include "lorbpano_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);
void orc_params_default(lp_params* p);
int orc_partition_regions(const int* dims, int ncams, double overlap, int patch_half,
                          lp_region* out, int cap, int* count);
int orc_brief_pattern(int n_d, int patch_half, uint64_t seed, lp_pair* out);
int orc_gaussian_kernel(float sigma, float* out, int* n);
int orc_fast_corners(const uint8_t* img, int w, int h, int ch, lp_region r, int thr, int arc,
                     int* xy, int cap, int* count);
int orc_harris_response(const uint8_t* img, int w, int h, int ch, const int* xy, int n,
                        float alpha, float sigma, float* out);
int orc_nms(const lp_keypoint* in, int n, int radius, lp_keypoint* out, int* count);
int orc_select_top_n(const lp_keypoint* in, int n, int top_n, lp_keypoint* out, int* count);
int orc_gaussian_blur(const float* in, int w, int h, int ch, float sigma, float* out);
int orc_brief_descriptors(const float* sm, int w, int h, const lp_keypoint* kps, int n,
                          const lp_pair* pairs, int n_d, int patch_half, uint64_t* out);
int orc_extract_features(const uint8_t* img, int w, int h, int ch, const lp_region* regions,
                         int nreg, const lp_extraction_config* cfg, const lp_pair* pairs,
                         lp_keypoint* kp_out, uint64_t* desc_out, int cap, int* count);
int orc_descriptor_distances(const uint64_t* a, const uint64_t* b, int n, int n_d, int* out);
int orc_lsh_bit_positions(int n_d, int tables, int bits, uint64_t seed, int* out);
int orc_probe_sequence(int k, int t, uint64_t* out);
int orc_match_features(const uint64_t* a, int na, const uint64_t* b, int nb, int n_d,
                       const lp_match_config* cfg, lp_match* out, int cap, int* count);
int orc_lsh_query(const uint64_t* train, int nt, const uint64_t* queries, int nq, int n_d,
                  const lp_match_config* cfg, int query_id0, long long* offsets, lp_match* out, long long cap,
                  long long* total);
int orc_dlt_homography(const lp_corr* c, int n, lp_homography* out);
int orc_symmetric_transfer_errors(const lp_homography* h, const lp_homography* hi, const lp_corr* c, int n,
                                  double* out);
int orc_prosac_homography(const lp_corr* c, int n, const lp_prosac_config* cfg,
                          lp_homography* model, uint8_t* mask, int* inlier_count, int* iterations,
                          int* trace_pool, int* trace_samples);
int orc_compute_canvas(const int* dims, const lp_homography* hs, int n, lp_canvas* out,
                       int* offsets);
int orc_warp_image(const float* img, int w, int h, int ch, const lp_homography* hom,
                   const lp_canvas* cv, float* out, float* cov);
int orc_linear_seam_mask(const float* covs, int n, int w, int h, float* masks);
int orc_downsample(const float* in, int w, int h, int ch, float* out);
int orc_upsample(const float* in, int w, int h, int ch, int tw, int th, float* out);
int orc_gaussian_pyramid(const float* in, int w, int h, int ch, int levels, float* out);
int orc_build_laplacian(const float* in, int w, int h, int ch, int levels, float* out);
int orc_collapse_laplacian(const float* packed, int w, int h, int ch, int levels, float* out);
int orc_multiband_blend(const float* images, const float* masks, int n, int w, int h, int ch,
                        int levels, uint8_t* out);
int orc_synth_texture(int w, int h, uint64_t seed, float smooth_sigma, uint8_t* out);
int orc_synth_planted_pair(int w, int h, double overlap, uint64_t seed, uint8_t* left,
                           uint8_t* right, double* true_h);
int orc_synth_sequence_frame(int w, int h, double overlap, uint64_t seed, uint64_t frame,
                             uint8_t* left, uint8_t* right);
int orc_synth_rotate(const uint8_t* img, int w, int h, double degrees, uint8_t* out);
int orc_rectify_crop(int ncams, int w, int h, const lp_camera* cams, const uint8_t* const* images,
                     uint8_t* const* outputs, int* out_w, int* out_h);
int orc_stitch_frame(int ncams, int w, int h, const lp_params* params,
                     const uint8_t* const* images, uint64_t frame_index, lp_frame_out* out);

#ifdef __cplusplus
}
#endif
#endif
