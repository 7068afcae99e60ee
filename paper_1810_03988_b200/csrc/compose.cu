// compose.cu — warp + linear seam + multi-band (Laplacian pyramid) blend, sm_100a.
//
// The reference materialises, per camera, full-canvas float rasters for the
// warp, coverage, seam mask, Laplacian pyramid and mask pyramid
// (compose.hpp:72-215). Here every camera only owns a window of the canvas:
// its coverage bounding box dilated by the pyramid support (>= 4*2^L+8 px at
// level 0) and aligned to 2^(L-1). Outside its window a camera's warped
// image, mask, Gaussian levels and Laplacian bands are exactly zero in the
// reference, and a zero-weight term adds +-0 to a +0-seeded accumulator, so
// skipping it leaves every accumulator bit-identical.
//
// Kernels per frame (L levels):
//   k_warp        FP64 inverse map + bilinear (compose.hpp:72-95) -> G0, cov
//   k_seam_rows   per row, warp-ballot run lengths -> min(forward, backward)
//                 distance (compose.hpp:108-120)
//   k_seam_norm   per pixel camera-ordered sum and division (123-129)
//   k_pyr_down    (L-1)x: shared-memory tile, 7-tap σ=1 blur evaluated only
//                 at the kept even samples (imgops.hpp:106-116), image and
//                 mask pyramids in one pass
//   k_blend_level Lx, top to bottom: the band of every camera
//                 (G_k - upsample(G_k+1), compose.hpp:134-147) weighted by
//                 its mask level and accumulated in camera order (182-192),
//                 renormalised (196-202), and collapsed with the upsampled
//                 coarser result (149-158); level 0 writes the u8 panorama
//                 with to_u8 where any camera covers (206-213).
// Accumulation orders are the reference's; FP ops are round-to-nearest, no FMA.
#include "compose.cuh"

namespace lpb {

__device__ __forceinline__ bool in_win(const Win& w, int x, int y) {
    return x >= w.x0 && x < w.x0 + w.w && y >= w.y0 && y < w.y0 + w.h;
}
// value of a windowed buffer at canvas-level coordinates (zero outside)
__device__ __forceinline__ float win_at(const float* buf, const Win& w, int x, int y) {
    return in_win(w, x, y) ? buf[static_cast<size_t>(y - w.y0) * w.w + (x - w.x0)] : 0.0f;
}

// ---------------------------------------------------------------------------
__global__ void k_warp(ComposeArgs a) {
    const int c = blockIdx.z;
    const Win w = a.win[c * a.levels];
    const int lx = blockIdx.x * blockDim.x + threadIdx.x, ly = blockIdx.y * blockDim.y + threadIdx.y;
    if (lx >= w.w || ly >= w.h) return;
    const int x = w.x0 + lx, y = w.y0 + ly;
    const double* hi = a.hinv + c * 9;
    const DevImage im = a.src[c];
    const double X = static_cast<double>(x + a.origin_x), Y = static_cast<double>(y + a.origin_y);
    const double wd = hi[6] * X + hi[7] * Y + hi[8];
    const double sx = (hi[0] * X + hi[1] * Y + hi[2]) / wd;
    const double sy = (hi[3] * X + hi[4] * Y + hi[5]) / wd;
    float v = 0.0f;
    uint8_t cv = 0;
    if (!(sx < 0.0 || sx > im.w - 1 || sy < 0.0 || sy > im.h - 1)) {
        const int x0 = static_cast<int>(sx), y0 = static_cast<int>(sy);
        const double ax = sx - x0, ay = sy - y0;
        const int x1 = min(x0 + 1, im.w - 1), y1 = min(y0 + 1, im.h - 1);
        const uint8_t* r0 = im.p + static_cast<size_t>(y0) * im.w;
        const uint8_t* r1 = im.p + static_cast<size_t>(y1) * im.w;
        const double v00 = __ldg(r0 + x0), v10 = __ldg(r0 + x1);
        const double v01 = __ldg(r1 + x0), v11 = __ldg(r1 + x1);
        v = __double2float_rn((1 - ay) * ((1 - ax) * v00 + ax * v10) + ay * ((1 - ax) * v01 + ax * v11));
        cv = 1;
    }
    a.G[c * a.levels][static_cast<size_t>(ly) * w.w + lx] = v;
    a.cov[c][static_cast<size_t>(ly) * w.w + lx] = cv;
}

// one warp per (camera, window row): forward / backward run lengths by ballot
template <typename CovT>
__device__ void seam_row(const CovT* cov, float* dist, int w) {
    const int lane = threadIdx.x & 31;
    int carry = -1;  // last uncovered x (window-local); the outside counts as uncovered
    for (int base = 0; base < w; base += 32) {
        const int x = base + lane;
        const bool covered = x < w && cov[x] > CovT(0);
        const unsigned z = __ballot_sync(0xffffffffu, !covered);
        const unsigned upto = z & (lane == 31 ? 0xffffffffu : ((2u << lane) - 1u));
        const int lz = upto ? base + 31 - __clz(upto) : carry;
        if (x < w) dist[x] = static_cast<float>(x - lz);
        if (z) carry = base + 31 - __clz(z);
    }
    int carry_r = w;  // next uncovered x
    for (int base = ((w - 1) / 32) * 32; base >= 0; base -= 32) {
        const int x = base + lane;
        const bool covered = x < w && cov[x] > CovT(0);
        const unsigned z = __ballot_sync(0xffffffffu, !covered);
        const unsigned from = z & ~((1u << lane) - 1u);
        const int nz = from ? base + __ffs(from) - 1 : carry_r;
        if (x < w) {
            const float b = static_cast<float>(nz - x);
            const float f = dist[x];
            dist[x] = b < f ? b : f;  // std::min(fwd, bwd)
        }
        if (z) carry_r = base + __ffs(z) - 1;
    }
}

__global__ void k_seam_rows(ComposeArgs a) {
    const int c = blockIdx.y;
    const Win w = a.win[c * a.levels];
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (row >= w.h) return;
    seam_row<uint8_t>(a.cov[c] + static_cast<size_t>(row) * w.w, a.M[c * a.levels] + static_cast<size_t>(row) * w.w,
                      w.w);
}

__global__ void k_seam_norm(ComposeArgs a) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= a.W[0] || y >= a.H[0]) return;
    float sum = 0.0f;
    for (int c = 0; c < a.ncams; ++c) {
        const Win w = a.win[c * a.levels];
        if (in_win(w, x, y)) sum = fadd(sum, a.M[c * a.levels][static_cast<size_t>(y - w.y0) * w.w + (x - w.x0)]);
    }
    if (!(sum > 0.0f)) return;
    for (int c = 0; c < a.ncams; ++c) {
        const Win w = a.win[c * a.levels];
        if (in_win(w, x, y)) {
            float* p = a.M[c * a.levels] + static_cast<size_t>(y - w.y0) * w.w + (x - w.x0);
            *p = __fdiv_rn(*p, sum);
        }
    }
}

// ---------------------------------------------------------------------------
// level k -> k+1 for both image and mask pyramids of one camera
constexpr int PD_TX = 32, PD_TY = 8;
constexpr int PD_IN_W = 2 * PD_TX + 6, PD_IN_H = 2 * PD_TY + 6;

__global__ void __launch_bounds__(PD_TX * PD_TY) k_pyr_down(ComposeArgs a, int k) {
    __shared__ float sG[PD_IN_H][PD_IN_W + 1];
    __shared__ float sM[PD_IN_H][PD_IN_W + 1];
    __shared__ float tG[PD_IN_H][PD_TX + 1];
    __shared__ float tM[PD_IN_H][PD_TX + 1];
    const int c = blockIdx.z;
    const Win wi = a.win[c * a.levels + k], wo = a.win[c * a.levels + k + 1];
    const int X0 = wo.x0 + blockIdx.x * PD_TX, Y0 = wo.y0 + blockIdx.y * PD_TY;
    if (X0 >= wo.x0 + wo.w || Y0 >= wo.y0 + wo.h) return;
    const float* Gi = a.G[c * a.levels + k];
    const float* Mi = a.M[c * a.levels + k];
    const int Wk = a.W[k], Hk = a.H[k];
    const int xb = 2 * X0 - 3, yb = 2 * Y0 - 3;
    const int tid = threadIdx.y * PD_TX + threadIdx.x;
    for (int i = tid; i < PD_IN_H * PD_IN_W; i += PD_TX * PD_TY) {
        const int r = i / PD_IN_W, cc = i - r * PD_IN_W;
        const int gx = min(max(xb + cc, 0), Wk - 1), gy = min(max(yb + r, 0), Hk - 1);
        sG[r][cc] = win_at(Gi, wi, gx, gy);
        sM[r][cc] = win_at(Mi, wi, gx, gy);
    }
    __syncthreads();
    float kt[7];
#pragma unroll
    for (int q = 0; q < 7; ++q) kt[q] = a.down_taps[q];
    // horizontal blur at the even columns 2X (tmp rows cover 2Y-3 .. 2Y+3)
    for (int i = tid; i < PD_IN_H * PD_TX; i += PD_TX * PD_TY) {
        const int r = i / PD_TX, xo = i - r * PD_TX;
        float g = 0.0f, m = 0.0f;
#pragma unroll
        for (int q = 0; q < 7; ++q) {
            g = fadd(g, fmul(kt[q], sG[r][2 * xo + q]));
            m = fadd(m, fmul(kt[q], sM[r][2 * xo + q]));
        }
        tG[r][xo] = g;
        tM[r][xo] = m;
    }
    __syncthreads();
    const int xo = threadIdx.x, yo = threadIdx.y;
    const int X = X0 + xo, Y = Y0 + yo;
    if (X >= wo.x0 + wo.w || Y >= wo.y0 + wo.h) return;
    float g = 0.0f, m = 0.0f;
#pragma unroll
    for (int q = 0; q < 7; ++q) {
        g = fadd(g, fmul(kt[q], tG[2 * yo + q][xo]));
        m = fadd(m, fmul(kt[q], tM[2 * yo + q][xo]));
    }
    const size_t o = static_cast<size_t>(Y - wo.y0) * wo.w + (X - wo.x0);
    a.G[c * a.levels + k + 1][o] = g;
    a.M[c * a.levels + k + 1][o] = m;
}

// upsample (imgops.hpp:119-140) of a level-(k+1) raster read through `fetch`
struct UpGeom {
    float sx, sy;
    int w, h;  // source (coarse) dims
};
__device__ __forceinline__ UpGeom up_geom(int w, int h, int tw, int th) {
    UpGeom g;
    g.sx = tw > 1 ? __fdiv_rn(static_cast<float>(w - 1), static_cast<float>(tw - 1)) : 0.0f;
    g.sy = th > 1 ? __fdiv_rn(static_cast<float>(h - 1), static_cast<float>(th - 1)) : 0.0f;
    g.w = w;
    g.h = h;
    return g;
}
template <typename F>
__device__ __forceinline__ float up_sample(const UpGeom& g, int x, int y, F fetch) {
    const float fx = fmul(static_cast<float>(x), g.sx), fy = fmul(static_cast<float>(y), g.sy);
    const int x0 = static_cast<int>(fx), y0 = static_cast<int>(fy);
    const float ax = fsub(fx, static_cast<float>(x0)), ay = fsub(fy, static_cast<float>(y0));
    const int xa = min(max(x0, 0), g.w - 1), xb = min(max(x0 + 1, 0), g.w - 1);
    const int ya = min(max(y0, 0), g.h - 1), yb = min(max(y0 + 1, 0), g.h - 1);
    const float v00 = fetch(xa, ya), v10 = fetch(xb, ya), v01 = fetch(xa, yb), v11 = fetch(xb, yb);
    const float oax = fsub(1.0f, ax), oay = fsub(1.0f, ay);
    return fadd(fmul(oay, fadd(fmul(oax, v00), fmul(ax, v10))),
                fmul(ay, fadd(fmul(oax, v01), fmul(ax, v11))));
}

__device__ __forceinline__ uint8_t to_u8(float v) {  // image.hpp:66-71
    float r = roundf(v);
    if (r < 0.0f) r = 0.0f;
    if (r > 255.0f) r = 255.0f;
    return static_cast<uint8_t>(r);
}

__global__ void k_blend_level(ComposeArgs a, int k) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= a.W[k] || y >= a.H[k]) return;
    const bool top = k == a.levels - 1;
    const UpGeom ug = top ? UpGeom{0, 0, 1, 1} : up_geom(a.W[k + 1], a.H[k + 1], a.W[k], a.H[k]);
    float acc = 0.0f, ws = 0.0f;
    for (int c = 0; c < a.ncams; ++c) {
        const Win w = a.win[c * a.levels + k];
        if (!in_win(w, x, y)) continue;
        const size_t o = static_cast<size_t>(y - w.y0) * w.w + (x - w.x0);
        const float wt = a.M[c * a.levels + k][o];
        float band = a.G[c * a.levels + k][o];
        if (!top) {
            const Win wn = a.win[c * a.levels + k + 1];
            const float* Gn = a.G[c * a.levels + k + 1];
            band = fsub(band, up_sample(ug, x, y, [&](int xx, int yy) { return win_at(Gn, wn, xx, yy); }));
        }
        ws = fadd(ws, wt);
        acc = fadd(acc, fmul(wt, band));
    }
    if (ws > 1e-6f && fabsf(fsub(ws, 1.0f)) > 1e-6f) acc = __fdiv_rn(acc, ws);
    if (!top) {
        const float* Rn = a.R[k + 1];
        const int wn = a.W[k + 1];
        acc = fadd(acc, up_sample(ug, x, y, [&](int xx, int yy) { return Rn[static_cast<size_t>(yy) * wn + xx]; }));
    }
    if (k > 0)
        a.R[k][static_cast<size_t>(y) * a.W[k] + x] = acc;
    else
        a.out[static_cast<size_t>(y) * a.W[0] + x] = ws > 0.0f ? to_u8(acc) : 0;
}

void blend_launch(const ComposeArgs& a, const Win* hw, cudaStream_t s) {
    for (int k = 0; k + 1 < a.levels; ++k) {
        int mw = 0, mh = 0;
        for (int c = 0; c < a.ncams; ++c) {
            mw = std::max(mw, hw[c * a.levels + k + 1].w);
            mh = std::max(mh, hw[c * a.levels + k + 1].h);
        }
        if (mw == 0 || mh == 0) continue;
        dim3 grid(cdiv(mw, PD_TX), cdiv(mh, PD_TY), a.ncams);
        LPB_LAUNCH(k_pyr_down, grid, dim3(PD_TX, PD_TY), 0, s, a, k);
    }
    for (int k = a.levels - 1; k >= 0; --k) {
        dim3 grid(cdiv(a.W[k], 32), cdiv(a.H[k], 8));
        LPB_LAUNCH(k_blend_level, grid, dim3(32, 8), 0, s, a, k);
    }
}

void compose_launch(const ComposeArgs& a, const Win* hw, cudaStream_t s) {
    int mw = 0, mh = 0;
    for (int c = 0; c < a.ncams; ++c) {
        mw = std::max(mw, hw[c * a.levels].w);
        mh = std::max(mh, hw[c * a.levels].h);
    }
    dim3 g0(cdiv(mw, 32), cdiv(mh, 8), a.ncams);
    LPB_LAUNCH(k_warp, g0, dim3(32, 8), 0, s, a);
    dim3 g1(cdiv(mh, 8), a.ncams);
    LPB_LAUNCH(k_seam_rows, g1, 256, 0, s, a);
    dim3 g2(cdiv(a.W[0], 32), cdiv(a.H[0], 8));
    LPB_LAUNCH(k_seam_norm, g2, dim3(32, 8), 0, s, a);
    blend_launch(a, hw, s);
}

// ---------------------------------------------------------------------------
// stage-isolated primitives (full-canvas, channels)
__global__ void k_warp_generic(const float* img, int w, int h, int ch, const double* hi, int cw,
                               int chh, int ox, int oy, float* out, float* cov) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= cw || y >= chh) return;
    const double X = static_cast<double>(x + ox), Y = static_cast<double>(y + oy);
    const double wd = hi[6] * X + hi[7] * Y + hi[8];
    const double sx = (hi[0] * X + hi[1] * Y + hi[2]) / wd;
    const double sy = (hi[3] * X + hi[4] * Y + hi[5]) / wd;
    const size_t o = static_cast<size_t>(y) * cw + x;
    if (sx < 0.0 || sx > w - 1 || sy < 0.0 || sy > h - 1) {
        for (int c = 0; c < ch; ++c) out[o * ch + c] = 0.0f;
        cov[o] = 0.0f;
        return;
    }
    const int x0 = static_cast<int>(sx), y0 = static_cast<int>(sy);
    const double ax = sx - x0, ay = sy - y0;
    const int x1 = min(x0 + 1, w - 1), y1 = min(y0 + 1, h - 1);
    for (int c = 0; c < ch; ++c) {
        const double v00 = img[(static_cast<size_t>(y0) * w + x0) * ch + c];
        const double v10 = img[(static_cast<size_t>(y0) * w + x1) * ch + c];
        const double v01 = img[(static_cast<size_t>(y1) * w + x0) * ch + c];
        const double v11 = img[(static_cast<size_t>(y1) * w + x1) * ch + c];
        out[o * ch + c] =
            __double2float_rn((1 - ay) * ((1 - ax) * v00 + ax * v10) + ay * ((1 - ax) * v01 + ax * v11));
    }
    cov[o] = 1.0f;
}
void warp_generic_launch(const float* img, int w, int h, int ch, const double* hinv, int cw, int chh,
                         int ox, int oy, float* out, float* cov, cudaStream_t s) {
    dim3 g(cdiv(cw, 32), cdiv(chh, 8));
    LPB_LAUNCH(k_warp_generic, g, dim3(32, 8), 0, s, img, w, h, ch, hinv, cw, chh, ox, oy, out, cov);
}

__global__ void k_seam_generic_rows(const float* covs, int n, int w, int h, float* masks) {
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int c = blockIdx.y;
    if (row >= h) return;
    const size_t o = (static_cast<size_t>(c) * h + row) * w;
    seam_row<float>(covs + o, masks + o, w);
}
__global__ void k_seam_generic_norm(int n, int w, int h, float* masks) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t np = static_cast<size_t>(w) * h;
    if (i >= np) return;
    float sum = 0.0f;
    for (int c = 0; c < n; ++c) sum = fadd(sum, masks[c * np + i]);
    if (sum > 0.0f)
        for (int c = 0; c < n; ++c) masks[c * np + i] = __fdiv_rn(masks[c * np + i], sum);
}
void seam_generic_launch(const float* covs, int n, int w, int h, float* masks, cudaStream_t s) {
    LPB_LAUNCH(k_seam_generic_rows, dim3(cdiv(h, 8), n), 256, 0, s, covs, n, w, h, masks);
    LPB_LAUNCH(k_seam_generic_norm, cdiv(static_cast<long long>(w) * h, 256), 256, 0, s, n, w, h, masks);
}

__global__ void k_down_h(const float* in, int w, int h, int ch, const float* taps, float* tmp) {
    // horizontal σ=1 blur at even columns only: tmp is (w/2) x h x ch
    const int ow = w / 2;
    const long long n = static_cast<long long>(ow) * h * ch;
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int c = static_cast<int>(i % ch);
    const long long p = i / ch;
    const int xo = static_cast<int>(p % ow), y = static_cast<int>(p / ow);
    float acc = 0.0f;
    for (int q = -3; q <= 3; ++q) {
        const int xx = min(max(2 * xo + q, 0), w - 1);
        acc = fadd(acc, fmul(taps[q + 3], in[(static_cast<size_t>(y) * w + xx) * ch + c]));
    }
    tmp[i] = acc;
}
__global__ void k_down_v(const float* tmp, int w, int h, int ch, const float* taps, float* out) {
    const int ow = w / 2, oh = h / 2;
    const long long n = static_cast<long long>(ow) * oh * ch;
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int c = static_cast<int>(i % ch);
    const long long p = i / ch;
    const int xo = static_cast<int>(p % ow), yo = static_cast<int>(p / ow);
    float acc = 0.0f;
    for (int q = -3; q <= 3; ++q) {
        const int yy = min(max(2 * yo + q, 0), h - 1);
        acc = fadd(acc, fmul(taps[q + 3], tmp[(static_cast<size_t>(yy) * ow + xo) * ch + c]));
    }
    out[i] = acc;
}
void downsample_launch(const float* in, int w, int h, int ch, const float* taps, float* tmp,
                       float* out, cudaStream_t s) {
    const long long n1 = static_cast<long long>(w / 2) * h * ch;
    const long long n2 = static_cast<long long>(w / 2) * (h / 2) * ch;
    if (n1 > 0) LPB_LAUNCH(k_down_h, cdiv(n1, 256), 256, 0, s, in, w, h, ch, taps, tmp);
    if (n2 > 0) LPB_LAUNCH(k_down_v, cdiv(n2, 256), 256, 0, s, tmp, w, h, ch, taps, out);
}

__global__ void k_upsample(const float* in, int w, int h, int ch, int tw, int th, float* out) {
    const long long n = static_cast<long long>(tw) * th * ch;
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int c = static_cast<int>(i % ch);
    const long long p = i / ch;
    const int x = static_cast<int>(p % tw), y = static_cast<int>(p / tw);
    const UpGeom g = up_geom(w, h, tw, th);
    out[i] = up_sample(g, x, y, [&](int xx, int yy) { return in[(static_cast<size_t>(yy) * w + xx) * ch + c]; });
}
void upsample_launch(const float* in, int w, int h, int ch, int tw, int th, float* out,
                     cudaStream_t s) {
    const long long n = static_cast<long long>(tw) * th * ch;
    if (n > 0) LPB_LAUNCH(k_upsample, cdiv(n, 256), 256, 0, s, in, w, h, ch, tw, th, out);
}

__global__ void k_sub(float* a, const float* b, size_t n) {
    size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) a[i] = fsub(a[i], b[i]);
}
__global__ void k_add(float* a, const float* b, size_t n) {
    size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) a[i] = fadd(a[i], b[i]);
}
void sub_launch(float* a, const float* b, size_t n, cudaStream_t s) {
    if (n) LPB_LAUNCH(k_sub, cdiv(static_cast<long long>(n), 256), 256, 0, s, a, b, n);
}
void add_launch(float* a, const float* b, size_t n, cudaStream_t s) {
    if (n) LPB_LAUNCH(k_add, cdiv(static_cast<long long>(n), 256), 256, 0, s, a, b, n);
}

}  // namespace lpb
