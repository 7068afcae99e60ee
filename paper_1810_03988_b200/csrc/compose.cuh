// compose.cuh — warp + seam + multi-band blend on the device (compose.hpp:32-215).
#pragma once
#include "common.cuh"

namespace lpb {

// A camera's window at one pyramid level: everything of that camera outside
// it is exactly zero in the reference's full-canvas arrays.
struct Win {
    int x0, y0, w, h;
};

struct ComposeArgs {
    int ncams, levels;
    int W[kMaxLevels], H[kMaxLevels];     // canvas dims per level
    int origin_x, origin_y;
    const Win* win;                       // ncams * levels (device)
    float* const* G;                      // ncams * levels image pyramid buffers (device ptrs)
    float* const* M;                      // ncams * levels mask pyramid buffers
    uint8_t* const* cov;                  // ncams coverage (level-0 window)
    float* const* R;                      // levels collapse buffers (R[0] unused)
    const float* down_taps;               // 7 taps of gaussian_kernel(1.0f)
    // warp source: u8 grayscale cameras
    const DevImage* src;                  // ncams (device)
    const double* hinv;                   // ncams * 9 (device)
    uint8_t* out;                         // W[0] x H[0]
};

// Full per-frame compositor: warp, seam masks, pyramids, band blend + collapse.
void compose_launch(const ComposeArgs& a, const Win* host_win, cudaStream_t s);
// Pyramid + blend + collapse only (masks and level-0 images already in G/M).
void blend_launch(const ComposeArgs& a, const Win* host_win, cudaStream_t s);

// ---- stage-isolated primitives ----
void warp_generic_launch(const float* img, int w, int h, int ch, const double* hinv, int cw, int chh,
                         int ox, int oy, float* out, float* cov, cudaStream_t s);
void seam_generic_launch(const float* covs, int n, int w, int h, float* masks, cudaStream_t s);
void downsample_launch(const float* in, int w, int h, int ch, const float* taps, float* tmp,
                       float* out, cudaStream_t s);
void upsample_launch(const float* in, int w, int h, int ch, int tw, int th, float* out,
                     cudaStream_t s);
void sub_launch(float* a, const float* b, size_t n, cudaStream_t s);  // a -= b
void add_launch(float* a, const float* b, size_t n, cudaStream_t s);  // a = a + b

}  // namespace lpb
