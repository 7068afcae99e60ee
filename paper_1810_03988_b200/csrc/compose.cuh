// compose.cuh — warp + seam + multi-band blend on the device (compose.hpp:32-215).
#pragma once
#include <cuda.h>  // CUtensorMap

#include "common.cuh"

namespace lpb {

// A camera's window at one pyramid level: everything of that camera outside
// it is exactly zero in the reference's full-canvas arrays.
struct Win {
    int x0, y0, w, h;
    int p;  // row pitch in elements (w rounded up to a multiple of 4: float4 rows)
};

constexpr int kMaxCompCams = 32;   // cameras per rig on the fused compositor path
constexpr int kMaxCompLevels = 12; // blend levels (canvas >= 2^11 px per side for 12)
constexpr int kRunSlots = 4;       // coverage runs stored inline per window row
constexpr int kBlendAlignX = 64;   // level-0 window x alignment (blend tile width at level 0)

// k_pyr_down output tile (level k+1) and its staged level-k box
constexpr int PD2_TX = 64, PD2_TY = 16;
constexpr int PD2_BW = 2 * PD2_TX + 8, PD2_BH = 2 * PD2_TY + 6;  // box 136 x 38 (134 used; rows of 16 B)

// Tensor maps of one k_pyr_down2 launch (level k -> k+1): every camera's
// level-k image and mask window as a 2-D f32 tensor (window-local
// coordinates, pitch w.p), box PD2_BW x PD2_BH. Passed by value as a
// __grid_constant__ parameter; ok == 0 -> the cp.async staging path.
struct PyrTma {
    CUtensorMap g[kMaxCompCams], m[kMaxCompCams];
    int ok;
};

// Tensor maps of one k_blend_lean launch at level k (< levels - 1): every
// camera's level-(k+1) image window and the level-(k+1) collapse result R,
// box lean_cx(TXK) x lean_cy(TXK); ok == 0 -> cp.async staging.
struct BlendTma {
    CUtensorMap g[kMaxCompCams], r;
    int ok;
};
// staged coarse tile of k_blend_lean<TXK>: rows, columns (16-byte rows)
__host__ __device__ constexpr int lean_cy(int txk) { return 4096 / txk / 2 + 3; }
__host__ __device__ constexpr int lean_cx(int txk) { return (txk / 2 + 3 + 3 + 3) / 4 * 4; }

// Encode a 2-D f32 tensor map (w x h elements, row pitch `pitch` elements,
// box bw x bh, zero fill out of bounds). False if the driver refuses.
bool tma_encode_f32_2d(CUtensorMap* m, const float* base, int w, int h, int pitch, int bw, int bh);

// Passed by value (constant bank): all per-camera geometry and pointers.
struct ComposeArgs {
    int ncams, levels;
    int W[kMaxCompLevels], H[kMaxCompLevels];  // canvas dims per level
    int origin_x, origin_y;
    int analytic_masks;   // 1: level-0 masks from coverage runs; 0: from M[c][0] buffers
    Win win[kMaxCompCams][kMaxCompLevels];
    float* G[kMaxCompCams][kMaxCompLevels];    // image pyramid windows
    float* M[kMaxCompCams][kMaxCompLevels];    // mask pyramid windows (M[c][0] only if !analytic)
    uint32_t* cov[kMaxCompCams];               // level-0 coverage bits, cov_words per window row
    int cov_words[kMaxCompCams];
    int2* run_rows[kMaxCompCams];              // per window row: (offset into runs, count)
    int run_base[kMaxCompCams];                // inline slots: row r of camera c owns
                                               // runs[run_base[c] + kRunSlots*r ...]
    int2* runs;                                // coverage runs [start, end) window-local
    int runs_cap;                              // inline slots + overflow area
    int runs_overflow_base;
    int* runs_used;                            // overflow allocations (rows with > kRunSlots runs)
    float* R[kMaxCompLevels];                  // collapse buffers, levels >= 1
    int Rp[kMaxCompLevels];                    // their row pitch (W[k] rounded up to 4)
    float down_taps[7];                        // gaussian_kernel(1.0f)
    DevImage src[kMaxCompCams];                // u8 grayscale cameras
    double hinv[kMaxCompCams][9];
    uint8_t* out;                              // W[0] x H[0]
    int* status;
    // host pointer (never read on the device): PyrTma per source level k,
    // owned by the ComposeBuffers that built this geometry, or null
    const PyrTma* pyr_tma;
    const BlendTma* blend_tma;  // host pointer: BlendTma per level k < levels - 1, or null
};

// stage_rectify_crop (pipeline.hpp:391-417) of one camera: dst (w x h, the
// crop's size) from src (in_w x in_h)
struct RectCam {
    const uint8_t* src;
    uint8_t* dst;
    double hinv[9];  // inverse of pre_transform (Homography::inverse)
    int identity;    // pre_transform exactly the identity: crop copy only
    int x0, y0, w, h;  // crop (the whole image when there is none)
};
void rectify_launch(const RectCam* cams, int ncams, int in_w, int in_h, int max_w, int max_h, cudaStream_t s);

// Full per-frame compositor: warp, coverage runs, pyramids, band blend + collapse.
void compose_launch(const ComposeArgs& a, cudaStream_t s);
const void* warp_kernel_fn();  // k_warp, for patching its node in a captured chain
// Pyramid + blend + collapse only (level-0 images and masks already in G/M).
void blend_launch(const ComposeArgs& a, cudaStream_t s);

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
