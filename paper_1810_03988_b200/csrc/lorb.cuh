// lorb.cuh — L-ORB extraction on the device (lorb.hpp:141-413).
#pragma once
#include "common.cuh"

namespace lpb {

// One detection region as the device sees it: scan area = region ∩
// [3,w-3) x [3,h-3) (lorb.hpp:196-198), plus its tile range in the flat grid.
struct DevRegion {
    int img;                 // index into the image table
    int x0, y0, x1, y1;      // scan area (non-empty)
    int rx0, ry0, rx1, ry1;  // the DetectionRegion itself (for the BRIEF crop)
    int tiles_x, ntiles;     // detect tiles (kDetTileX x kDetTileY) over the scan area
    int out_slot;            // which output group (camera) the keypoints belong to
};

constexpr int kDetTileX = 96;    // output tile of the detect kernel (columns; 96 measured faster than 64)
constexpr int kDetTileY = 32;    // (rows)
constexpr int kMaxHarrisR = 12;  // harris_sigma <= 4 (radius ceil(3 sigma)); the generic tile's static smem
constexpr int kMaxBlurR = 24;    // brief_blur_sigma <= 8
constexpr int kTopnSortCap = 8192;  // k_topn_radix's shared sort; larger top_n: global radix sort per region
constexpr int kDescribeFastBlurR = 6;  // k_describe6's blur radius (sigma = 2)
constexpr int kTopnRankCap = 2048;   // k_topn fast path: rank placement of <= 2048 keys
constexpr int kTopnHistBins = 4096;  // first radix digit: top 12 key bits

// Everything the fused extractor needs, all device pointers.
struct ExtractArgs {
    const DevRegion* regions;
    int nregions;
    int max_tiles;           // largest per-region tile count (grid.x; grid.y = region)
    const DevImage* images;
    const double* harris_w;  // (2R+1)^2
    double hw[49];           // the same weights in the parameter bank when R <= 3
    int harris_r;
    float alpha, threshold;
    int fast_t, fast_arc;
    int top_n;
    uint64_t* surv;          // nregions * surv_cap survivor keys
    unsigned* surv_count;    // nregions
    unsigned* hist;          // nregions * kTopnHistBins (top-12-bit key histogram)
    int surv_cap;
    lp_keypoint* kp_region;  // nregions * top_n
    int* count_region;       // nregions
    const float* blur_taps;  // 2*RB+1
    float btaps[2 * kMaxBlurR + 1];  // the same taps in the parameter bank
    int blur_r;
    const lp_pair* pairs;
    int n_d, patch_half;
    int nslots;              // output groups (cameras)
    lp_keypoint* kp_out;     // nslots * cap_slot
    uint64_t* desc_out;      // nslots * cap_slot * 2W
    int cap_slot;
    int* slot_count;         // nslots
    int* status;             // device status word
    // optional (k_describe6): the LSH keys of every descriptor (hash_key,
    // matchlsh.hpp:70-80) in the matcher's layout, nslots * cap_slot * tables
    uint64_t* lsh_keys;
    const int* lsh_bitpos;   // tables * bits
    int lsh_tables, lsh_bits;
    // optional (k_detect9): running count of FAST candidates whose FP64 Harris
    // response was evaluated (each tile's own pixels), for the roofline
    unsigned long long* work_cand;
};

// stage_detect + stage_describe for every region of every image in 4 launches
// (detect tiles -> per-region top-N -> describe). Counts stay on the device.
void extract_launch(const ExtractArgs& a, cudaStream_t s);

// ---- stage-isolated primitives (C-ABI lp_fast_corners ... lp_brief_descriptors) ----
void fast_flags_launch(const uint8_t* img, int w, int h, int x0, int y0, int x1, int y1, int t,
                       int arc, uint8_t* flags, cudaStream_t s);
void harris_points_launch(const uint8_t* img, int w, int h, const int* xy, int n,
                          const double* wts, int r, float alpha, float* out, int* status,
                          cudaStream_t s);
void nms_generic_launch(const lp_keypoint* in, int n, int radius, int minx, int miny, int gw,
                        int gh, int* grid, uint8_t* keep, cudaStream_t s);
void blur_launch(const float* in, float* tmp, float* out, int w, int h, int ch, const float* taps,
                 int r, cudaStream_t s);
void brief_generic_launch(const float* sm, int w, int h, const lp_keypoint* kps, int n,
                          const lp_pair* pairs, int n_d, int ph, uint64_t* out, int* status,
                          cudaStream_t s);

}  // namespace lpb
