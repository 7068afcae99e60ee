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
constexpr int kMaskTileX = 128, kMaskTileY = 16;  // k_mask0's tile (and the mask-tile flags' grain)
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
// k_blend_lean's tile: kLeanPx pixels for kLeanThreads threads (16 per thread)
#ifndef LPB_LEAN_PX
#define LPB_LEAN_PX 2048
#endif
constexpr int kLeanPx = LPB_LEAN_PX, kLeanThreads = LPB_LEAN_PX / 16;
__host__ __device__ constexpr int lean_cy(int txk) { return kLeanPx / txk / 2 + 3; }
__host__ __device__ constexpr int lean_cx(int txk) { return (txk / 2 + 3 + 3 + 3) / 4 * 4; }

// Encode a 2-D f32 tensor map (w x h elements, row pitch `pitch` elements,
// box bw x bh, zero fill out of bounds). False if the driver refuses.
bool tma_encode_f32_2d(CUtensorMap* m, const float* base, int w, int h, int pitch, int bw, int bh);

// ---- compositor geometry of one homography set (host and device) ----
// canvas (compute_canvas, compose.hpp:32-68), blend levels
// (pipeline.hpp:511-514, gaussian_pyramid's size check), each camera's
// level-0 window = projected-corner bbox + (4 * 2^L + 8) px, y aligned to
// 2^(L-1), x to max(2^(L-1), 64), and the inverse maps
// (Homography::inverse, homography.hpp:36-48). One function for the host
// (prepare_compositor) and the device (k_geom), so both derive the same
// integers from the same doubles.
struct RigGeom {
    int cw, ch, ox, oy;  // canvas width, height, origin
    int levels;
    Win win0[kMaxCompCams];
};

__host__ __device__ inline double geom_det(const double* h) {
    return h[0] * (h[4] * h[8] - h[5] * h[7]) - h[1] * (h[3] * h[8] - h[5] * h[6]) + h[2] * (h[3] * h[7] - h[4] * h[6]);
}

// per camera: projected-corner bbox (compute_canvas's loop body,
// compose.hpp:44-55) and whether a corner lies behind the camera
struct CamBox {
    double mnx, mny, mxx, mxy;
    int behind;
};
__host__ __device__ inline CamBox geom_cam_box(const double* m, int w, int h) {
    CamBox b{1.7976931348623157e308, 1.7976931348623157e308, -1.7976931348623157e308, -1.7976931348623157e308, 0};
    const double cs[4][2] = {{0, 0}, {static_cast<double>(w), 0}, {0, static_cast<double>(h)},
                             {static_cast<double>(w), static_cast<double>(h)}};
    for (int q = 0; q < 4; ++q) {
        const double wd = m[6] * cs[q][0] + m[7] * cs[q][1] + m[8];
        if (wd <= 0) b.behind = 1;
        const double x = (m[0] * cs[q][0] + m[1] * cs[q][1] + m[2]) / wd;
        const double y = (m[3] * cs[q][0] + m[4] * cs[q][1] + m[5]) / wd;
        b.mnx = fmin(b.mnx, x);
        b.mny = fmin(b.mny, y);
        b.mxx = fmax(b.mxx, x);
        b.mxy = fmax(b.mxy, y);
    }
    return b;
}
// Homography::inverse (homography.hpp:36-48), det != 0
__host__ __device__ inline void geom_cam_inverse(const double* m, double* out) {
    const double d = geom_det(m);
    const double inv[9] = {(m[4] * m[8] - m[5] * m[7]) / d, (m[2] * m[7] - m[1] * m[8]) / d,
                           (m[1] * m[5] - m[2] * m[4]) / d, (m[5] * m[6] - m[3] * m[8]) / d,
                           (m[0] * m[8] - m[2] * m[6]) / d, (m[2] * m[3] - m[0] * m[5]) / d,
                           (m[3] * m[7] - m[4] * m[6]) / d, (m[1] * m[6] - m[0] * m[7]) / d,
                           (m[0] * m[4] - m[1] * m[3]) / d};
    const double i8 = inv[8];
    for (int j = 0; j < 9; ++j) out[j] = fabs(i8) > 1e-12 ? inv[j] / i8 : inv[j];
}
// canvas from the union of the boxes, then the blend levels; 0 or an lp_status
__host__ __device__ inline int geom_canvas(const CamBox* bx, int ncams, int blend_levels, RigGeom* g) {
    double minx = 1.7976931348623157e308, miny = minx, maxx = -minx, maxy = -minx;
    for (int c = 0; c < ncams; ++c) {
        minx = fmin(minx, bx[c].mnx);
        miny = fmin(miny, bx[c].mny);
        maxx = fmax(maxx, bx[c].mxx);
        maxy = fmax(maxy, bx[c].mxy);
    }
    g->ox = static_cast<int>(floor(minx));
    g->oy = static_cast<int>(floor(miny));
    g->cw = static_cast<int>(ceil(maxx)) - g->ox;
    g->ch = static_cast<int>(ceil(maxy)) - g->oy;
    int levels = blend_levels;
    while (levels > 1 && (g->cw < (1 << (levels - 1)) || g->ch < (1 << (levels - 1)))) --levels;
    if (levels < 1 || levels > kMaxCompLevels) return LP_TOO_MANY_LEVELS;
    int ww = g->cw, hh = g->ch;
    for (int i = 1; i < levels; ++i) {
        if (ww < 2 || hh < 2) return LP_TOO_MANY_LEVELS;
        ww /= 2;
        hh /= 2;
    }
    g->levels = levels;
    return 0;
}
// one camera's level-0 window on the canvas
__host__ __device__ inline Win geom_cam_window(const CamBox& b, const RigGeom& g) {
    const int align = 1 << (g.levels - 1);
    const int align_x = align > kBlendAlignX ? align : kBlendAlignX;
    const int margin = 4 * (1 << g.levels) + 8;
    if (b.behind) return Win{0, 0, (g.cw + align_x - 1) / align_x * align_x, g.ch, 0};
    long long x0 = static_cast<long long>(floor(b.mnx)) - g.ox - margin;
    long long y0 = static_cast<long long>(floor(b.mny)) - g.oy - margin;
    long long x1 = static_cast<long long>(ceil(b.mxx)) - g.ox + margin;
    long long y1 = static_cast<long long>(ceil(b.mxy)) - g.oy + margin;
    x0 = x0 > 0 ? (x0 / align_x) * align_x : 0;
    y0 = y0 > 0 ? (y0 / align) * align : 0;
    const long long xcap = (g.cw + align_x - 1) / align_x * align_x;
    const long long xr = (x1 + align_x - 1) / align_x * align_x;
    x1 = xr < xcap ? xr : xcap;
    y1 = y1 < g.ch ? y1 : g.ch;
    return Win{static_cast<int>(x0), static_cast<int>(y0), static_cast<int>(x1 - x0 > 0 ? x1 - x0 : 0),
               static_cast<int>(y1 - y0 > 0 ? y1 - y0 : 0), 0};
}

// 0 on success, else the lp_status the reference would throw (host order:
// a singular camera first, then the levels check)
__host__ __device__ inline int rig_geometry(int ncams, int w, int h, int blend_levels, const lp_homography* H,
                                            RigGeom* g, double* hinv) {
    CamBox bx[kMaxCompCams];
    for (int c = 0; c < ncams; ++c) {
        if (fabs(geom_det(H[c].h)) < 1e-9) return LP_SINGULAR_HOMOGRAPHY;
        bx[c] = geom_cam_box(H[c].h, w, h);
    }
    const int st = geom_canvas(bx, ncams, blend_levels, g);
    if (st) return st;
    for (int c = 0; c < ncams; ++c) {
        geom_cam_inverse(H[c].h, hinv + 9 * c);
        g->win0[c] = geom_cam_window(bx[c], *g);
    }
    for (int c = ncams; c < kMaxCompCams; ++c) g->win0[c] = Win{0, 0, 0, 0, 0};
    return 0;
}


// Can arenas built for `ref` compose a frame of geometry `g`? The same canvas
// and levels, and every camera's window inside ref's: a larger window only
// computes more of the reference's zero canvas around the camera (DESIGN.md
// §3, windows), and ref's windows keep the alignment the blend tiles need.
// Small homography jitter between re-registrations then keeps the arenas.
__host__ __device__ inline bool fits_geometry(const RigGeom& g, const RigGeom& ref, int ncams) {
    if (g.cw != ref.cw || g.ch != ref.ch || g.ox != ref.ox || g.oy != ref.oy || g.levels != ref.levels) return false;
    for (int c = 0; c < ncams; ++c) {
        const Win& a = g.win0[c];
        const Win& b = ref.win0[c];
        if (a.w == 0 || a.h == 0) continue;
        if (b.w == 0 || b.h == 0 || a.x0 < b.x0 || a.y0 < b.y0 || a.x0 + a.w > b.x0 + b.w || a.y0 + a.h > b.y0 + b.h)
            return false;
    }
    return true;
}

// ---- inverse maps in __constant__ memory: k_warp reads camera c's map as
// constant-bank operands from c_hinv[hinv_base + c]; the rig updates them by
// stream-ordered copies (from the host after a host-side estimate, or from
// the device after k_geom), so no launch parameters change per frame
constexpr int kConstHinvSlots = 896;  // cameras of all live rigs (64 KB constant bank)
int hinv_slots_alloc(int n);           // first of n consecutive slots (throws CapacityOverflow)
void hinv_slots_free(int base, int n);
void hinv_upload(int base, const double* src, int n, bool src_on_device, cudaStream_t s);

// ---- k_geom: the estimator's verdict on the device (HomographyCache,
// pipeline.hpp:259-286) for a re-registering frame that does not synchronise
// the host: the new chain if the estimate succeeded, else the cached one;
// its inverse maps; whether its geometry equals the one the compositor
// arenas were built for. The record lands in host-mapped memory.
struct GeomOutcome {
    unsigned long long ticket;
    int done, estimated, same, status;
    int which;  // arenas the verdict fits: 0 the submit-time ones, 1 the alternate, -1 neither
    lp_homography H[kMaxCompCams];
};
struct GeomArgs {
    int ncams, w, h, blend_levels;
    const lp_homography* chain;
    const int* chain_status;
    lp_homography* cached;  // device copy of the cache, updated on success
    const RigGeom* ref;     // geometry of the compositor arenas
    double* hinv;           // 9 * ncams, written only when the geometry could be derived
    GeomOutcome* out;       // host-mapped
    unsigned long long ticket;
    int* skip;              // the slot's compositor skip word: 1 when this verdict does not fit the arenas
    // an alternate kept geometry whose compositor is enqueued too (nullptr:
    // none): its skip word is cleared only when the verdict fits it and not `ref`
    const RigGeom* ref2;
    int* skip2;
};
void geom_launch(const GeomArgs& a, cudaStream_t s);

// Passed by value (constant bank): all per-camera geometry and pointers.
struct MaskState {
    int valid;  // this frame's maps equal `key`: every mask buffer is current
    int have;   // `key` holds the maps of the last compose that made the masks
    unsigned next_runs, next_mask0;  // k_runs / k_mask0 work counters (reset by k_warp)
    unsigned runs_done;              // k_runs_mask0: run items finished (reset by k_warp)
    double key[kMaxCompCams][9];
};

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
    // level-0 mask tiles (k_mask0's 128 x 16 tiles of the camera window):
    // 0 every pixel +0, 1 every pixel exactly 1, 2 mixed (null without runs)
    uint8_t* mtile[kMaxCompCams];
    int mtile_w[kMaxCompCams];                 // tiles per window row
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
    // the same frames as 2-D textures: k_warp takes a pixel's four bilinear
    // taps with one tex2Dgather (clamp-to-edge = the reference's x1 / y1
    // clamp) instead of four byte loads; 0 -> byte loads
    cudaTextureObject_t tex[kMaxCompCams];
    int use_tex;
    int blend_unit;                            // k_blend_lean's single-camera unit-weight tiles
    // seam masks (coverage runs, M pyramid, tile flags) depend only on the
    // inverse maps and the windows: k_warp's first CTA compares this frame's
    // maps with the ones the arenas' masks were made from and sets `valid`;
    // k_runs / k_mask0 / the mask half of k_pyr_down then skip. Null: always
    // recompute (caller-provided masks, LPB_MASK_REUSE=0)
    struct MaskState* mask_state;
    // the slot's skip word (null: never): set by k_geom when the frame's
    // device verdict does not fit the arenas it is composed on (the host
    // recomposes it, repair), so the compositor's kernels exit at once;
    // cleared after the frame by k_status_take
    const int* skip;
    int hinv_base;                             // camera c's inverse map: c_hinv[hinv_base + c]
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
