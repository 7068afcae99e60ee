// lorb.cu — L-ORB extraction kernels for sm_100a.
//
// Fused path (stage_detect + stage_describe, pipeline.hpp:419-469):
//   k_detect   one CTA per 32x32 output tile of a region: the u8 tile plus a
//              halo is staged once in shared memory;
//              FAST-9 (lorb.hpp:141-205) runs on the tile + 1-px ring, FAST
//              corners are compacted into a shared list, FP64 Harris
//              (lorb.hpp:209-250) runs densely over that list from shared
//              integer gradients, the 3x3 NMS (lorb.hpp:254-288) runs on the
//              response map, and survivors are appended to a per-region key
//              list with warp-aggregated atomics (ballot + popc).
//   k_topn     one CTA per region: MSB radix select over the 64-bit key
//              (response desc, y asc, x asc) = select_top_n's total order
//              (lorb.hpp:291-299), then a shared-memory bitonic sort.
//   k_describe one warp per keypoint: the 43x43 patch (BRIEF pattern half
//              15 + blur radius 6) is blurred in shared memory with the exact
//              separable σ=2 order of gaussian_blur (imgops.hpp:50-72), then
//              256 ternary tests are packed into gt/lt planes with ballots
//              (lorb.hpp:333-350). Values equal the reference's region-crop
//              blur at every sampled point (test_lorb.cpp:301-343).
// All FP ops are explicit round-to-nearest (no FMA), matching the reference.

#include "lorb.cuh"
#include "prims.cuh"

namespace lpb {

// ---------------------------------------------------------------------------
// FAST segment test on a 16-bit ring mask: a circular run of >= arc set bits
// exists iff AND of the arc rotations is non-zero (== longest_arc >= arc).
__device__ __forceinline__ bool has_arc(unsigned m, int arc) {
    unsigned m32 = m | (m << 16);
    unsigned r = m32;
    for (int s = 1; s < arc; ++s) r &= (m32 >> s);
    return (r & 0xFFFFu) != 0u;
}

__constant__ int c_ring_dx[16] = {0, 1, 2, 3, 3, 3, 2, 1, 0, -1, -2, -3, -3, -3, -2, -1};
__constant__ int c_ring_dy[16] = {-3, -3, -2, -1, 0, 1, 2, 3, 3, 3, 2, 1, 0, -1, -2, -3};

// ---------------------------------------------------------------------------
// k_detect<RT, ARCT>: generic instance (any Harris radius <= kMaxHarrisR, any
// arc), one CTA per kDetTileX x kDetTileY output tile, grid (tiles, regions)
constexpr int TX = kDetTileX, TY = kDetTileY;
constexpr int NX = TX + 2, NY = TY + 2;                 // response grid: tile + 1-px ring
constexpr int HALO_MAX = kMaxHarrisR + 2;              // harris R + gradient 1 + NMS 1
constexpr int IMG_MAX_X = TX + 2 * HALO_MAX, IMG_MAX_Y = TY + 2 * HALO_MAX;
constexpr int GRAD_MAX_X = TX + 2 + 2 * kMaxHarrisR, GRAD_MAX_Y = TY + 2 + 2 * kMaxHarrisR;
constexpr int GEN_DYN_SMEM = 2 * GRAD_MAX_X * GRAD_MAX_Y * static_cast<int>(sizeof(short));

// survivors of the 3x3 NMS -> per-region key list (ballot-aggregated
// atomics) and the first radix digit histogram of k_topn
__device__ __forceinline__ void emit_survivor(const ExtractArgs& a, int ri, bool keep, uint64_t key) {
    const int lane = threadIdx.x & 31;
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (!m) return;
    const int leader = __ffs(m) - 1;
    unsigned pos = 0;
    if (lane == leader) pos = atomicAdd(&a.surv_count[ri], static_cast<unsigned>(__popc(m)));
    pos = __shfl_sync(0xffffffffu, pos, leader);
    if (keep) {
        const unsigned slot = pos + __popc(m & ((1u << lane) - 1u));
        if (slot < static_cast<unsigned>(a.surv_cap))
            a.surv[static_cast<size_t>(ri) * a.surv_cap + slot] = key;
        else
            dev_fail(a.status, LP_CAPACITY_OVERFLOW);
        // first radix digit of k_topn: top 12 key bits (sign, exponent, 3 mantissa bits)
        atomicAdd(&a.hist[static_cast<size_t>(ri) * kTopnHistBins + (key >> 52)], 1u);
    }
}

// 3x3 NMS of one candidate on the response grid (lorb.hpp:254-288): NaN marks
// "not a thresholded candidate"; exact ties go to the smaller (y, x)
__device__ __forceinline__ bool nms_wins(const float* resp, int i, float r) {
    bool keep = true;
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
        for (int dx = -1; dx <= 1; ++dx) {
            if (dx == 0 && dy == 0) continue;
            const float o = resp[i + dy * NX + dx];
            if (o > r || (o == r && (dy < 0 || (dy == 0 && dx < 0)))) keep = false;
        }
    return keep;
}

template <int RT, int ARCT>
__global__ void __launch_bounds__(256) k_detect(ExtractArgs a) {
    // integer central differences; the Harris loop forms the reference's exact
    // double (double(I(x+1)) - I(x-1)) / 2.0 (lorb.hpp:239-240) per tap
    __shared__ uint8_t s_img[IMG_MAX_X * IMG_MAX_Y];
    // the two gradient planes (GEN_DYN_SMEM bytes) in dynamic shared memory:
    // with them the static footprint would pass the 48 KB static limit
    extern __shared__ __align__(16) short s_gdyn[];
    short* s_gx = s_gdyn;
    short* s_gy = s_gdyn + GRAD_MAX_X * GRAD_MAX_Y;
    __shared__ float s_resp[NX * NY];
    __shared__ short s_cand[NX * NY];
    __shared__ double s_w[(2 * kMaxHarrisR + 1) * (2 * kMaxHarrisR + 1)];
    __shared__ int s_ncand;

    const int ri = blockIdx.y;
    const DevRegion rg = a.regions[ri];
    const int t = blockIdx.x;
    if (t >= rg.ntiles) return;
    const DevImage im = a.images[rg.img];
    const int ox = rg.x0 + (t % rg.tiles_x) * TX;
    const int oy = rg.y0 + (t / rg.tiles_x) * TY;
    const int R = RT > 0 ? RT : a.harris_r;
    const int arc = ARCT > 0 ? ARCT : a.fast_arc;
    const int halo = (R + 1 > 3 ? R + 1 : 3) + 1;
    const int iw = TX + 2 * halo, ih = TY + 2 * halo;
    const int gw = TX + 2 + 2 * R, gh = TY + 2 + 2 * R;
    const int tid = threadIdx.x;

    const int K = 2 * R + 1;
    for (int i = tid; i < K * K; i += blockDim.x) s_w[i] = a.harris_w[i];
    if (tid == 0) s_ncand = 0;

    // stage the u8 tile + halo (clamped coordinates; clamped texels are never
    // consumed by a valid test).
    const int gx0 = ox - halo, gy0 = oy - halo;
    for (int i = tid; i < iw * ih; i += blockDim.x) {
        int ly = i / iw, lx = i - ly * iw;
        int gx = min(max(gx0 + lx, 0), im.w - 1);
        int gy = min(max(gy0 + ly, 0), im.h - 1);
        s_img[ly * iw + lx] = __ldg(im.p + static_cast<size_t>(gy) * im.w + gx);
    }
    for (int i = tid; i < NX * NY; i += blockDim.x) s_resp[i] = __int_as_float(0x7fc00000);
    __syncthreads();

    // integer central differences over the Harris window area
    const int goff = halo - 1 - R;  // gradient (0,0) sits at image-local (goff, goff)
    for (int i = tid; i < gw * gh; i += blockDim.x) {
        int ly = i / gw, lx = i - ly * gw;
        int ix = lx + goff, iy = ly + goff;
        s_gx[i] = static_cast<short>(int(s_img[iy * iw + ix + 1]) - int(s_img[iy * iw + ix - 1]));
        s_gy[i] = static_cast<short>(int(s_img[(iy + 1) * iw + ix]) - int(s_img[(iy - 1) * iw + ix]));
    }

    // FAST on the tile + 1-px ring, restricted to the scan area
    for (int i = tid; i < NX * NY; i += blockDim.x) {
        int ly = i / NX, lx = i - ly * NX;
        int px = ox - 1 + lx, py = oy - 1 + ly;
        if (px < rg.x0 || px >= rg.x1 || py < rg.y0 || py >= rg.y1) continue;
        int cx = px - gx0, cy = py - gy0;
        int c = s_img[cy * iw + cx];
        unsigned br = 0, dk = 0;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            int v = s_img[(cy + c_ring_dy[k]) * iw + cx + c_ring_dx[k]];
            br |= (v > c + a.fast_t) ? (1u << k) : 0u;
            dk |= (v < c - a.fast_t) ? (1u << k) : 0u;
        }
        if (has_arc(br, arc) || has_arc(dk, arc)) {
            if (px - R - 1 < 0 || px + R + 1 >= im.w || py - R - 1 < 0 || py + R + 1 >= im.h) {
                dev_fail(a.status, LP_WINDOW_OUT_OF_BOUNDS);
                continue;
            }
            int slot = atomicAdd(&s_ncand, 1);
            s_cand[slot] = static_cast<short>(i);
        }
    }
    __syncthreads();

    // FP64 Harris over the compacted candidates (lorb.hpp:235-247)
    const int nc = s_ncand;
    const double alpha = static_cast<double>(a.alpha);
    for (int j = tid; j < nc; j += blockDim.x) {
        int i = s_cand[j];
        int ly = i / NX, lx = i - ly * NX;
        // gradient-local centre of this pixel
        int gcx = lx + R, gcy = ly + R;
        double sa = 0.0, sb = 0.0, sc = 0.0;
        for (int v = -R; v <= R; ++v) {
            const short* rx = s_gx + (gcy + v) * gw + gcx;
            const short* ry = s_gy + (gcy + v) * gw + gcx;
            const double* wr = s_w + (v + R) * K + R;
            for (int u = -R; u <= R; ++u) {
                const double ix = static_cast<double>(rx[u]) / 2.0;
                const double iy = static_cast<double>(ry[u]) / 2.0;
                const double wt = wr[u];
                sa = dadd(sa, dmul(dmul(wt, ix), ix));
                sb = dadd(sb, dmul(dmul(wt, iy), iy));
                sc = dadd(sc, dmul(dmul(wt, ix), iy));
            }
        }
        double s = dadd(sa, sb);
        double r = dsub(dsub(dmul(sa, sb), dmul(sc, sc)), dmul(dmul(alpha, s), s));
        float rf = __double2float_rn(r);
        if (rf >= a.threshold) s_resp[i] = rf;
    }
    __syncthreads();

    // 3x3 NMS among thresholded candidates; survivors -> per-region key list
    for (int base = 0; base < TX * TY; base += blockDim.x) {
        const int i = base + tid;
        bool keep = false;
        uint64_t key = 0;
        if (i < TX * TY) {
            const int ly = i / TX + 1, lx = i % TX + 1;
            const float r = s_resp[ly * NX + lx];
            if (r == r) {
                keep = nms_wins(s_resp, ly * NX + lx, r);
                key = kp_key(r, ox + lx - 1, oy + ly - 1);
            }
        }
        emit_survivor(a, ri, keep, key);
    }
}

// ---------------------------------------------------------------------------
// k_detect9: the default configuration (Harris radius 3, FAST arc 9).
//  * the tile is staged as 32-bit words aligned to global 4-pixel groups;
//  * FAST tests four pixels per thread in SIMD-within-a-register form: per
//    ring position one byte-permute builds the four ring values, bytewise
//    unsigned compares against saturated c+t / c-t leave one flag per byte
//    (msb), and the arc-9 test is AND-of-3 (x2) + OR over the 16 rotations;
//  * Harris folds the reference's /2.0 of both gradients into one exact *0.25
//    per sum (binary scaling commutes with every rounding on the way), reads
//    packed (gx, gy) shorts and takes the 49 window weights from the
//    parameter bank, fully unrolled in the reference's v-then-u order;
//  * NMS runs over the candidate list only.
namespace d9 {
constexpr int FW = (NX + 6) / 4;   // FAST words per row: 4 px each, global-aligned
constexpr int SWW = FW + 2;        // staged words per row (one each side for the ring)
constexpr int SB = 4 * SWW;        // staged row pitch in bytes
constexpr int SH = TY + 10;        // staged rows oy-5 .. oy+TY+4
constexpr int GX = TX + 8, GY = TY + 8;  // gradient grid: ox-4 .. ox+TX+3, oy-4 .. oy+TY+3
constexpr int NTASK = NY * FW;
__device__ constexpr int ring_dx(int k) {
    constexpr int t[16] = {0, 1, 2, 3, 3, 3, 2, 1, 0, -1, -2, -3, -3, -3, -2, -1};
    return t[k];
}
__device__ constexpr int ring_dy(int k) {
    constexpr int t[16] = {-3, -3, -2, -1, 0, 1, 2, 3, 3, 3, 2, 1, 0, -1, -2, -3};
    return t[k];
}

// msb of byte b = (x_b > y_b), unsigned; other bits are don't-care
__device__ __forceinline__ uint32_t gt_u8(uint32_t x, uint32_t y) {
    const uint32_t t = (x | 0x80808080u) - ((y & 0x7f7f7f7fu) + 0x01010101u);
    return (x & ~y) | (~(x ^ y) & t);
}
__device__ __forceinline__ uint32_t arc9(const uint32_t (&f)[16]) {
    uint32_t t3[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) t3[k] = f[k] & f[(k + 1) & 15] & f[(k + 2) & 15];
    uint32_t any = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) any |= t3[k] & t3[(k + 3) & 15] & t3[(k + 6) & 15];
    return any;
}
}  // namespace d9

__global__ void __launch_bounds__(256, 4) k_detect9(const __grid_constant__ ExtractArgs a) {
    using namespace d9;
    __shared__ uint32_t s_img[SH * SWW];
    __shared__ __align__(16) int s_grad[GY * GX];  // (gx & 0xffff) | gy << 16
    __shared__ float s_resp[NX * NY];
    __shared__ short s_cand[NX * NY];
    __shared__ int s_ncand, s_ninner;

    const int ri = blockIdx.y;
    const DevRegion rg = a.regions[ri];
    const int t = blockIdx.x;
    if (t >= rg.ntiles) return;
    const DevImage im = a.images[rg.img];
    const int ox = rg.x0 + (t % rg.tiles_x) * TX;
    const int oy = rg.y0 + (t / rg.tiles_x) * TY;
    const int fx0 = (ox - 1) & ~3;  // first FAST word (ox >= 3)
    const int gx0 = fx0 - 4, gy0 = oy - 5;
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid == 0) s_ncand = s_ninner = 0;

    // ---- stage: SH rows x SWW words
    const bool inside = gx0 >= 0 && gy0 >= 0 && gx0 + SB <= im.w && gy0 + SH <= im.h && (im.w & 3) == 0 &&
                        (reinterpret_cast<uintptr_t>(im.p) & 3) == 0;
    if (inside) {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(im.p + static_cast<size_t>(gy0) * im.w + gx0);
        const int pitch = im.w >> 2;
        // register-free global->shared copies: every word of the tile in
        // flight at once instead of a load->store latency per iteration
        for (int i = tid; i < SH * SWW; i += 256) {
            const int r = i / SWW, q = i - r * SWW;
            cp_async4(&s_img[i], src + static_cast<size_t>(r) * pitch + q, true);
        }
        cp_async_wait_all();
    } else {  // clamped bytes; clamped texels never reach a valid test
        for (int i = tid; i < SH * SWW; i += 256) {
            const int r = i / SWW, q = i - r * SWW;
            const uint8_t* row = im.p + static_cast<size_t>(min(max(gy0 + r, 0), im.h - 1)) * im.w;
            uint32_t v = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b)
                v |= static_cast<uint32_t>(__ldg(row + min(max(gx0 + 4 * q + b, 0), im.w - 1))) << (8 * b);
            s_img[i] = v;
        }
    }
    for (int i = tid; i < NX * NY; i += 256) s_resp[i] = __int_as_float(0x7fc00000);
    __syncthreads();

    // ---- gradients (integer central differences) over the Harris support,
    // four columns per task in 16-bit lanes: gradient column gc sits at staged
    // byte gc + xo (xo in 1..4, the same for the whole tile), so every row
    // segment is one funnel shift of two staged words; (0x8000 + a - b) per
    // lane cannot borrow across lanes, and its top bit flipped is (a - b)
    // modulo 2^16: the (gx & 0xffff) | gy << 16 words come out by byte permutes
    {
        const int xo = ox - fx0;
        const int sU = 8 * (xo & 3), kU = xo >> 2;                  // bytes gc+xo .. +3 (rows above / below)
        const int sL = 8 * ((xo - 1) & 3), kL = (xo - 1) >> 2;      // bytes gc+xo-1 .. +2 (centre row)
        const int sR = 8 * ((xo + 1) & 3), kR = (xo + 1) >> 2;      // bytes gc+xo+1 .. +4 (centre row)
        constexpr int GW = GX / 4;                                  // four-column groups per row
        for (int i = tid; i < GY * GW; i += 256) {
            const int gr = i / GW, g4 = i - gr * GW;
            const uint32_t* row = s_img + (gr + 1) * SWW + g4;
            const uint32_t up = __funnelshift_r(row[kU - SWW], row[kU + 1 - SWW], sU);
            const uint32_t dn = __funnelshift_r(row[kU + SWW], row[kU + 1 + SWW], sU);
            const uint32_t lf = __funnelshift_r(row[kL], row[kL + 1], sL);
            const uint32_t rt = __funnelshift_r(row[kR], row[kR + 1], sR);
            uint4 out;
            {
                const uint32_t dx = (__byte_perm(rt, 0, 0x4140) + 0x80008000u - __byte_perm(lf, 0, 0x4140)) ^ 0x80008000u;
                const uint32_t dy = (__byte_perm(dn, 0, 0x4140) + 0x80008000u - __byte_perm(up, 0, 0x4140)) ^ 0x80008000u;
                out.x = __byte_perm(dx, dy, 0x5410);
                out.y = __byte_perm(dx, dy, 0x7632);
            }
            {
                const uint32_t dx = (__byte_perm(rt, 0, 0x4342) + 0x80008000u - __byte_perm(lf, 0, 0x4342)) ^ 0x80008000u;
                const uint32_t dy = (__byte_perm(dn, 0, 0x4342) + 0x80008000u - __byte_perm(up, 0, 0x4342)) ^ 0x80008000u;
                out.z = __byte_perm(dx, dy, 0x5410);
                out.w = __byte_perm(dx, dy, 0x7632);
            }
            *reinterpret_cast<uint4*>(&s_grad[gr * GX + 4 * g4]) = out;
        }
    }

    // ---- FAST-9, four pixels per task (row r of the response grid, word j)
    {
        const uint32_t T4 = static_cast<uint32_t>(a.fast_t) * 0x01010101u;
        const int cx_lo = max(rg.x0, ox - 1), cx_hi = min(rg.x1, ox + TX + 1);
#pragma unroll 1
        for (int t0 = 0; t0 < NTASK; t0 += 256) {
            if (t0 + (tid & ~31) >= NTASK) break;  // the tail round: warps without a task leave
            const int task = t0 + tid;
            const bool valid = task < NTASK;
            const int tk = valid ? task : 0;
            const int r = tk / FW, j = tk - r * FW;
            const uint32_t* w0 = s_img + (r + 1) * SWW + j;  // row y-3, word j-1 of the centre
            uint32_t wv[7][3];
#pragma unroll
            for (int dy = 0; dy < 7; ++dy)
#pragma unroll
                for (int q = 0; q < 3; ++q) wv[dy][q] = w0[dy * SWW + q];
            const uint32_t C = wv[3][1];
            const uint32_t Hc = __vaddus4(C, T4), Lc = __vsubus4(C, T4);
            // brighter flag in bit 7, darker flag in bit 6 of every byte: one
            // AND/OR arc network tests both runs at once
            uint32_t fc[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const int dx = ring_dx(k), dy = ring_dy(k) + 3;
                uint32_t v;
                if (dx == 0)
                    v = wv[dy][1];
                else if (dx > 0)
                    v = __byte_perm(wv[dy][1], wv[dy][2], dx | (dx + 1) << 4 | (dx + 2) << 8 | (dx + 3) << 12);
                else
                    v = __byte_perm(wv[dy][0], wv[dy][1], (4 + dx) | (5 + dx) << 4 | (6 + dx) << 8 | (7 + dx) << 12);
                fc[k] = (gt_u8(v, Hc) & 0x80808080u) | ((gt_u8(Lc, v) >> 1) & 0x40404040u);
            }
            uint32_t F = arc9(fc) & 0xC0C0C0C0u;
            F = (F | (F << 1)) & 0x80808080u;
            // scan area (lorb.hpp:196-198) and the tile + ring
            const int y = oy - 1 + r, x4 = fx0 + 4 * j;
            if (!valid || y < rg.y0 || y >= rg.y1) F = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if (x4 + b < cx_lo || x4 + b >= cx_hi) F &= ~(0x80u << (8 * b));
            // harris_response's window test (lorb.hpp:232-234)
            if (F && (x4 - 4 < 0 || x4 + 3 + 4 >= im.w || y - 4 < 0 || y + 4 >= im.h)) {
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int x = x4 + b;
                    if ((F >> (8 * b + 7)) & 1u && (x - 4 < 0 || x + 4 >= im.w || y - 4 < 0 || y + 4 >= im.h)) {
                        dev_fail(a.status, LP_WINDOW_OUT_OF_BOUNDS);
                        F &= ~(0x80u << (8 * b));
                    }
                }
            }
            // warp prefix of the corner counts, one shared atomic per warp
            const int n = __popc(F);
            int incl = n;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += v;
            }
            int base = 0;
            if (lane == 31) base = atomicAdd(&s_ncand, incl);
            base = __shfl_sync(0xffffffffu, base, 31) + incl - n;
            const int gi = r * NX + (x4 - (ox - 1));
            while (F) {
                const int b = (__ffs(F) - 8) >> 3;
                F &= F - 1;
                s_cand[base++] = static_cast<short>(gi + b);
            }
        }
    }
    __syncthreads();

    // ---- FP64 Harris over the candidates (lorb.hpp:235-247), exact x4 scaled
    const int nc = s_ncand;
    const double alpha = static_cast<double>(a.alpha);
    int ninner = 0;  // the tile's own candidates (the ring belongs to its neighbours)
    for (int jj = tid; jj < nc; jj += 256) {
        const int i = s_cand[jj];
        const int ly = i / NX, lx = i - ly * NX;
        ninner += lx >= 1 && lx <= TX && ly >= 1 && ly <= TY;
        const int* g0 = s_grad + ly * GX + lx;  // tap (u, v) = (-3, -3)
        double sa = 0.0, sb = 0.0, sc = 0.0;
#pragma unroll
        for (int v = 0; v < 7; ++v)
#pragma unroll
            for (int u = 0; u < 7; ++u) {
                const int g = g0[v * GX + u];
                const double ix = static_cast<double>(static_cast<short>(g & 0xffff));
                const double iy = static_cast<double>(g >> 16);
                const double wt = a.hw[v * 7 + u];
                const double wx = dmul(wt, ix), wy = dmul(wt, iy);
                sa = dadd(sa, dmul(wx, ix));
                sb = dadd(sb, dmul(wy, iy));
                sc = dadd(sc, dmul(wx, iy));
            }
        sa = dmul(sa, 0.25);
        sb = dmul(sb, 0.25);
        sc = dmul(sc, 0.25);
        const double s = dadd(sa, sb);
        const double r = dsub(dsub(dmul(sa, sb), dmul(sc, sc)), dmul(dmul(alpha, s), s));
        const float rf = __double2float_rn(r);
        if (rf >= a.threshold) s_resp[i] = rf;
    }
    if (a.work_cand) {  // Harris evaluations, for the roofline (lp_rig_algorithmic_work)
        ninner = __reduce_add_sync(0xffffffffu, ninner);
        if (lane == 0 && ninner) atomicAdd(&s_ninner, ninner);
    }
    __syncthreads();
    if (a.work_cand && tid == 0 && s_ninner) atomicAdd(a.work_cand, static_cast<unsigned long long>(s_ninner));

    // ---- 3x3 NMS over the tile's candidates; survivors -> key list
    for (int b0 = 0; b0 < nc; b0 += 256) {
        if (b0 + (tid & ~31) >= nc) break;  // warps past the last candidate
        const int jj = b0 + tid;
        bool keep = false;
        uint64_t key = 0;
        if (jj < nc) {
            const int i = s_cand[jj];
            const int ly = i / NX, lx = i - ly * NX;
            const float r = s_resp[i];
            if (lx >= 1 && lx <= TX && ly >= 1 && ly <= TY && r == r) {
                keep = nms_wins(s_resp, i, r);
                key = kp_key(r, ox + lx - 1, oy + ly - 1);
            }
        }
        emit_survivor(a, ri, keep, key);
    }
}

// ---------------------------------------------------------------------------
__global__ void k_iota_int(int* p, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = i;
}

// k_topn: exact per-region select_top_n via MSB radix select + bitonic sort
__device__ void bitonic_desc(uint64_t* v, int n_pow2) {
    for (int k = 2; k <= n_pow2; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n_pow2; i += blockDim.x) {
                int p = i ^ j;
                if (p > i) {
                    uint64_t x = v[i], y = v[p];
                    bool desc = (i & k) == 0;
                    if (desc ? (x < y) : (x > y)) {
                        v[i] = y;
                        v[p] = x;
                    }
                }
            }
            __syncthreads();
        }
}

// Fast path (top_n <= kTopnRankCap): the first radix digit (12 bits) comes
// from the histogram k_detect built, refinement digits are 8 bits, and the
// <= kTopnRankCap gathered keys are placed by rank (count of larger keys; keys
// are unique), which needs no barriers and no sorting network.
__global__ void __launch_bounds__(1024) k_topn(ExtractArgs a) {
    __shared__ uint64_t s_keys[kTopnRankCap];
    __shared__ unsigned s_hist[kTopnHistBins];
    __shared__ unsigned s_wsum[32];
    __shared__ uint64_t s_prefix;
    __shared__ int s_pbits, s_k, s_bucket, s_m;
    const int ri = blockIdx.x;
    const int n = min(static_cast<int>(a.surv_count[ri]), a.surv_cap);
    const uint64_t* keys = a.surv + static_cast<size_t>(ri) * a.surv_cap;
    const int top_n = a.top_n;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int m;
    if (n <= top_n) {
        m = n;
        for (int i = tid; i < n; i += blockDim.x) s_keys[i] = keys[i];
    } else {
        for (int i = tid; i < kTopnHistBins; i += blockDim.x)
            s_hist[i] = a.hist[static_cast<size_t>(ri) * kTopnHistBins + i];
        __syncthreads();
        // descending-bin suffix scan: thread t owns bins 4095-4t .. 4092-4t
        unsigned v[4], local = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            v[j] = s_hist[kTopnHistBins - 1 - (4 * tid + j)];
            local += v[j];
        }
        unsigned incl = local;
        for (int off = 1; off < 32; off <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += t;
        }
        if (lane == 31) s_wsum[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            unsigned ws = s_wsum[lane], wi = ws;
            for (int off = 1; off < 32; off <<= 1) {
                const unsigned t = __shfl_up_sync(0xffffffffu, wi, off);
                if (lane >= off) wi += t;
            }
            s_wsum[lane] = wi - ws;  // exclusive
        }
        __syncthreads();
        const unsigned excl = s_wsum[warp] + incl - local;
        if (excl < static_cast<unsigned>(top_n) && static_cast<unsigned>(top_n) <= excl + local) {
            unsigned cum = excl;
            for (int j = 0; j < 4; ++j) {
                if (cum + v[j] >= static_cast<unsigned>(top_n)) {
                    s_prefix = static_cast<uint64_t>(kTopnHistBins - 1 - (4 * tid + j));
                    s_k = top_n - static_cast<int>(cum);
                    s_bucket = static_cast<int>(v[j]);
                    s_pbits = 12;
                    break;
                }
                cum += v[j];
            }
        }
        __syncthreads();
        // 8-bit refinement digits until the candidate set fits
        while ((top_n - s_k) + s_bucket > kTopnRankCap && s_pbits < 64) {
            const uint64_t prefix = s_prefix;
            const int pbits = s_pbits;
            const int dbits = pbits + 8 <= 64 ? 8 : 64 - pbits;
            for (int i = tid; i < 256; i += blockDim.x) s_hist[i] = 0;
            __syncthreads();
            for (int i0 = tid; i0 < n; i0 += 8 * 1024) {  // 8 keys in flight per thread
                uint64_t kk[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) kk[u] = i0 + 1024 * u < n ? __ldg(keys + i0 + 1024 * u) : 0ull;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (i0 + 1024 * u < n && (kk[u] >> (64 - pbits)) == prefix)
                        atomicAdd(&s_hist[(kk[u] >> (64 - pbits - dbits)) & ((1u << dbits) - 1u)], 1u);
            }
            __syncthreads();
            if (tid == 0) {
                unsigned cum = 0;
                int sel = 0;
                for (int d = (1 << dbits) - 1; d >= 0; --d) {
                    if (cum + s_hist[d] >= static_cast<unsigned>(s_k)) {
                        sel = d;
                        break;
                    }
                    cum += s_hist[d];
                }
                s_k -= static_cast<int>(cum);
                s_bucket = static_cast<int>(s_hist[sel]);
                s_prefix = (prefix << dbits) | static_cast<uint64_t>(sel);
                s_pbits = pbits + dbits;
            }
            __syncthreads();
        }
        if (tid == 0) s_m = 0;
        __syncthreads();
        const uint64_t prefix = s_prefix;
        const int sh = 64 - s_pbits;
        for (int i0 = tid; i0 < n; i0 += 8 * 1024) {  // 8 keys in flight per thread
            uint64_t kk[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) kk[u] = i0 + 1024 * u < n ? __ldg(keys + i0 + 1024 * u) : 0ull;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (i0 + 1024 * u < n && (sh == 64 ? 0 : (kk[u] >> sh)) >= prefix) {
                    const int slot = atomicAdd(&s_m, 1);
                    if (slot < kTopnRankCap) s_keys[slot] = kk[u];
                }
        }
        __syncthreads();
        m = min(s_m, kTopnRankCap);
    }
    __syncthreads();
    const int out_n = min(m, top_n);
    for (int i = tid; i < m; i += blockDim.x) {
        const uint64_t key = s_keys[i];
        int r = 0;
        for (int j = 0; j < m; ++j) r += s_keys[j] > key;
        if (r < out_n) {
            float resp;
            int x, y;
            kp_unkey(key, &resp, &x, &y);
            a.kp_region[static_cast<size_t>(ri) * top_n + r] = lp_keypoint{x, y, resp, ri};
        }
    }
    if (tid == 0) a.count_region[ri] = out_n;
}

// General path (any top_n <= kTopnSortCap): MSB radix select + bitonic sort.
__global__ void __launch_bounds__(1024) k_topn_radix(ExtractArgs a) {
    extern __shared__ uint64_t s_keys[];  // kTopnSortCap
    __shared__ unsigned s_hist[256];
    __shared__ uint64_t s_prefix;
    __shared__ int s_pbits, s_k, s_bucket, s_m;
    const int ri = blockIdx.x;
    const int n = min(static_cast<int>(a.surv_count[ri]), a.surv_cap);
    const uint64_t* keys = a.surv + static_cast<size_t>(ri) * a.surv_cap;
    const int top_n = a.top_n;
    const int tid = threadIdx.x;
    int m;
    if (n <= top_n) {
        m = n;
        for (int i = tid; i < n; i += blockDim.x) s_keys[i] = keys[i];
    } else {
        if (tid == 0) {
            s_prefix = 0;
            s_pbits = 0;
            s_k = top_n;
        }
        __syncthreads();
        for (;;) {
            for (int i = tid; i < 256; i += blockDim.x) s_hist[i] = 0;
            __syncthreads();
            const uint64_t prefix = s_prefix;
            const int pbits = s_pbits;
            for (int i = tid; i < n; i += blockDim.x) {
                uint64_t k = keys[i];
                if (pbits == 0 || (k >> (64 - pbits)) == prefix)
                    atomicAdd(&s_hist[(k >> (56 - pbits)) & 255u], 1u);
            }
            __syncthreads();
            if (tid == 0) {
                unsigned cum = 0;
                int sel = 0;
                for (int d = 255; d >= 0; --d) {
                    if (cum + s_hist[d] >= static_cast<unsigned>(s_k)) {
                        sel = d;
                        break;
                    }
                    cum += s_hist[d];
                }
                s_k -= static_cast<int>(cum);
                s_bucket = static_cast<int>(s_hist[sel]);
                s_prefix = (prefix << 8) | static_cast<uint64_t>(sel);
                s_pbits = pbits + 8;
            }
            __syncthreads();
            const int above = top_n - s_k;
            if (above + s_bucket <= kTopnSortCap || s_pbits == 64) break;
        }
        if (tid == 0) s_m = 0;
        __syncthreads();
        const uint64_t prefix = s_prefix;
        const int sh = 64 - s_pbits;
        for (int i = tid; i < n; i += blockDim.x) {
            uint64_t k = keys[i];
            uint64_t top = sh == 64 ? 0 : (k >> sh);
            if (top >= prefix) {
                int slot = atomicAdd(&s_m, 1);
                if (slot < kTopnSortCap) s_keys[slot] = k;
            }
        }
        __syncthreads();
        m = min(s_m, kTopnSortCap);
    }
    int p2 = 1;
    while (p2 < m) p2 <<= 1;
    for (int i = m + tid; i < p2; i += blockDim.x) s_keys[i] = 0;
    __syncthreads();
    bitonic_desc(s_keys, p2);
    const int out_n = min(m, top_n);
    for (int i = tid; i < out_n; i += blockDim.x) {
        float r;
        int x, y;
        kp_unkey(s_keys[i], &r, &x, &y);
        a.kp_region[static_cast<size_t>(ri) * top_n + i] = lp_keypoint{x, y, r, ri};
    }
    if (tid == 0) a.count_region[ri] = out_n;
}

// ---------------------------------------------------------------------------
// k_describe: one warp per keypoint
__global__ void __launch_bounds__(256) k_describe(ExtractArgs a, int warp_bytes) {
    extern __shared__ __align__(16) unsigned char s_dyn[];
    lp_pair* s_pairs = reinterpret_cast<lp_pair*>(s_dyn);
    float* s_taps = reinterpret_cast<float*>(s_pairs + a.n_d);
    const int warps = blockDim.x / 32;
    unsigned char* s_warp_base = s_dyn + ((a.n_d * sizeof(lp_pair) + (2 * kMaxBlurR + 1) * 4 + 15) & ~15);
    for (int i = threadIdx.x; i < a.n_d; i += blockDim.x) s_pairs[i] = a.pairs[i];
    for (int i = threadIdx.x; i < 2 * a.blur_r + 1; i += blockDim.x) s_taps[i] = a.blur_taps[i];
    if (blockIdx.x == 0 && threadIdx.x < a.nslots) {
        int tot = 0;
        for (int r = 0; r < a.nregions; ++r)
            if (a.regions[r].out_slot == static_cast<int>(threadIdx.x)) tot += a.count_region[r];
        a.slot_count[threadIdx.x] = tot;
    }
    __syncthreads();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gslot = blockIdx.x * warps + warp;
    const int ri = gslot / a.top_n, i = gslot - ri * a.top_n;
    if (ri >= a.nregions || i >= a.count_region[ri]) return;
    const DevRegion rg = a.regions[ri];
    const DevImage im = a.images[rg.img];
    const lp_keypoint kp = a.kp_region[static_cast<size_t>(ri) * a.top_n + i];
    int off = 0;
    for (int r = 0; r < ri; ++r)
        if (a.regions[r].out_slot == rg.out_slot) off += a.count_region[r];
    const int idx = off + i;
    const int P = a.patch_half, RB = a.blur_r;
    const int pw = 2 * P + 1, iw = pw + 2 * RB;

    // smoothed_crop bounds (lorb.hpp:371-375) for the PatchOutOfBounds test (336-338)
    const int margin = P + RB;
    const int cx0 = max(0, rg.rx0 - margin), cy0 = max(0, rg.ry0 - margin);
    const int cx1 = min(im.w, rg.rx1 + margin), cy1 = min(im.h, rg.ry1 + margin);
    if (kp.x - P < cx0 || kp.x + P >= cx1 || kp.y - P < cy0 || kp.y + P >= cy1) {
        if (lane == 0) dev_fail(a.status, LP_PATCH_OUT_OF_BOUNDS);
        return;
    }

    unsigned char* sw = s_warp_base + static_cast<size_t>(warp) * warp_bytes;
    uint8_t* s_in = sw;                                                   // iw x iw
    float* s_tmp = reinterpret_cast<float*>(sw + ((iw * iw + 15) & ~15));  // iw rows x pw cols
    float* s_S = s_tmp + iw * pw;                                         // pw x pw
    const int bx = kp.x - P - RB, by = kp.y - P - RB;
    for (int j = lane; j < iw * iw; j += 32) {
        int ly = j / iw, lx = j - ly * iw;
        int gx = min(max(bx + lx, 0), im.w - 1), gy = min(max(by + ly, 0), im.h - 1);
        s_in[j] = __ldg(im.p + static_cast<size_t>(gy) * im.w + gx);
    }
    __syncwarp();
    // horizontal pass: every staged row, the pw patch columns
    for (int j = lane; j < iw * pw; j += 32) {
        int ly = j / pw, lx = j - ly * pw;
        const uint8_t* row = s_in + ly * iw + lx;
        float acc = 0.0f;
        for (int q = 0; q <= 2 * RB; ++q) acc = fadd(acc, fmul(s_taps[q], static_cast<float>(row[q])));
        s_tmp[j] = acc;
    }
    __syncwarp();
    // vertical pass
    for (int j = lane; j < pw * pw; j += 32) {
        int ly = j / pw, lx = j - ly * pw;
        float acc = 0.0f;
        for (int q = 0; q <= 2 * RB; ++q) acc = fadd(acc, fmul(s_taps[q], s_tmp[(ly + q) * pw + lx]));
        s_S[j] = acc;
    }
    __syncwarp();
    // ternary tests -> gt / lt bitplanes
    const int W = (a.n_d + 63) / 64;
    uint64_t* d = a.desc_out + (static_cast<size_t>(rg.out_slot) * a.cap_slot + idx) * 2 * W;
    for (int w = 0; w < W; ++w) {
        unsigned g[2], l[2];
        for (int h = 0; h < 2; ++h) {
            int pi = w * 64 + h * 32 + lane;
            bool gt = false, lt = false;
            if (pi < a.n_d) {
                lp_pair pr = s_pairs[pi];
                float ip = s_S[(P + pr.py) * pw + P + pr.px];
                float iq = s_S[(P + pr.qy) * pw + P + pr.qx];
                gt = ip > iq;
                lt = ip < iq;
            }
            g[h] = __ballot_sync(0xffffffffu, gt);
            l[h] = __ballot_sync(0xffffffffu, lt);
        }
        if (lane == 0) {
            d[w] = static_cast<uint64_t>(g[0]) | (static_cast<uint64_t>(g[1]) << 32);
            d[W + w] = static_cast<uint64_t>(l[0]) | (static_cast<uint64_t>(l[1]) << 32);
        }
    }
    if (lane == 0) a.kp_out[static_cast<size_t>(rg.out_slot) * a.cap_slot + idx] = kp;
}

// ---------------------------------------------------------------------------
// k_describe6: the default blur radius (sigma = 2 -> 13 taps), one warp per
// keypoint. The 43x43 u8 patch is staged with 8 loads in flight per lane, the
// horizontal pass is unrolled with the taps in the parameter bank, and the
// vertical pass is evaluated only at the pattern's sample points, straight
// into the tests: S(p) is the same 13-tap sum in the same order as the full
// crop blur (imgops.hpp:50-72), so the descriptor is bit-identical while 512
// instead of 961 vertical sums are formed and no 31x31 plane is stored
// (7 KB of shared memory per warp instead of 11 KB).
constexpr int D6_RB = kDescribeFastBlurR;
__global__ void __launch_bounds__(256) k_describe6(const __grid_constant__ ExtractArgs a, int warp_bytes) {
    extern __shared__ __align__(16) unsigned char s_dyn[];
    lp_pair* s_pairs = reinterpret_cast<lp_pair*>(s_dyn);
    const int warps = blockDim.x / 32;
    unsigned char* s_warp_base = s_dyn + ((a.n_d * sizeof(lp_pair) + 15) & ~15);
    for (int i = threadIdx.x; i < a.n_d; i += blockDim.x) s_pairs[i] = a.pairs[i];
    if (blockIdx.x == 0 && threadIdx.x < a.nslots) {
        int tot = 0;
        for (int r = 0; r < a.nregions; ++r)
            if (a.regions[r].out_slot == static_cast<int>(threadIdx.x)) tot += a.count_region[r];
        a.slot_count[threadIdx.x] = tot;
    }
    __syncthreads();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gslot = blockIdx.x * warps + warp;
    const int ri = gslot / a.top_n, i = gslot - ri * a.top_n;
    if (ri >= a.nregions || i >= a.count_region[ri]) return;
    const DevRegion rg = a.regions[ri];
    const DevImage im = a.images[rg.img];
    const lp_keypoint kp = a.kp_region[static_cast<size_t>(ri) * a.top_n + i];
    int off = 0;
    for (int r = 0; r < ri; ++r)
        if (a.regions[r].out_slot == rg.out_slot) off += a.count_region[r];
    const int idx = off + i;
    const int P = a.patch_half;
    const int pw = 2 * P + 1, iw = pw + 2 * D6_RB;

    // smoothed_crop bounds (lorb.hpp:371-375) for the PatchOutOfBounds test (336-338)
    const int margin = P + D6_RB;
    const int cx0 = max(0, rg.rx0 - margin), cy0 = max(0, rg.ry0 - margin);
    const int cx1 = min(im.w, rg.rx1 + margin), cy1 = min(im.h, rg.ry1 + margin);
    if (kp.x - P < cx0 || kp.x + P >= cx1 || kp.y - P < cy0 || kp.y + P >= cy1) {
        if (lane == 0) dev_fail(a.status, LP_PATCH_OUT_OF_BOUNDS);
        return;
    }
    const int rowb = (iw + 6) / 4 * 4;  // staged row pitch: the words covering a row at any alignment
    uint8_t* s_in = s_warp_base + static_cast<size_t>(warp) * warp_bytes;            // iw x rowb u8
    float* s_tmp = reinterpret_cast<float*>(s_in + ((iw * rowb + 15) & ~15));        // iw x pw
    const int bx = kp.x - P - D6_RB, by = kp.y - P - D6_RB;
    // interior patches: the aligned words covering each row by cp.async, all
    // in flight at once; patches at the image border: clamped byte loads
    const int ax = bx & ~3, nw = (bx - ax + iw + 3) / 4;
    const bool words = ax >= 0 && by >= 0 && ax + 4 * nw <= im.w && by + iw <= im.h && (im.w & 3) == 0 &&
                       (reinterpret_cast<uintptr_t>(im.p) & 3) == 0;
    const int spitch = words ? rowb : iw, soff = words ? bx - ax : 0;
    if (words) {
        uint32_t* s_w = reinterpret_cast<uint32_t*>(s_in);
        for (int j = lane; j < iw * nw; j += 32) {
            const int ly = j / nw, q = j - ly * nw;
            cp_async4(s_w + ly * (rowb / 4) + q, im.p + static_cast<size_t>(by + ly) * im.w + ax + 4 * q, true);
        }
        cp_async_wait_all();
    }
    // stage the u8 patch; 8 loads in flight per lane
    for (int j0 = lane; !words && j0 < iw * iw; j0 += 32 * 8) {
        uint8_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = j0 + 32 * u;
            v[u] = 0;
            if (j < iw * iw) {
                const int ly = j / iw, lx = j - ly * iw;
                const int gx = min(max(bx + lx, 0), im.w - 1), gy = min(max(by + ly, 0), im.h - 1);
                v[u] = __ldg(im.p + static_cast<size_t>(gy) * im.w + gx);
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (j0 + 32 * u < iw * iw) s_in[j0 + 32 * u] = v[u];
    }
    __syncwarp();
    // horizontal pass: every staged row, the pw patch columns, two adjacent
    // columns per lane (14 staged pixels converted once for both sums)
    const int pw2 = (pw + 1) / 2;
    for (int j = lane; j < iw * pw2; j += 32) {
        const int ly = j / pw2, lx = 2 * (j - ly * pw2);
        const uint8_t* row = s_in + ly * spitch + soff + lx;
        float v[2 * D6_RB + 2];
#pragma unroll
        for (int q = 0; q < 2 * D6_RB + 2; ++q) v[q] = lx + q < iw ? static_cast<float>(row[q]) : 0.0f;
        float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
        for (int q = 0; q <= 2 * D6_RB; ++q) {
            a0 = fadd(a0, fmul(a.btaps[q], v[q]));
            a1 = fadd(a1, fmul(a.btaps[q], v[q + 1]));
        }
        s_tmp[ly * pw + lx] = a0;
        if (lx + 1 < pw) s_tmp[ly * pw + lx + 1] = a1;
    }
    __syncwarp();
    // vertical pass at the sample points + ternary tests -> gt / lt bitplanes
    auto S = [&](int x, int y) {  // patch coordinates in [-P, P]
        const float* col = s_tmp + (P + y) * pw + (P + x);
        float acc = 0.0f;
#pragma unroll
        for (int q = 0; q <= 2 * D6_RB; ++q) acc = fadd(acc, fmul(a.btaps[q], col[q * pw]));
        return acc;
    };
    const int W = (a.n_d + 63) / 64;
    uint64_t* d = a.desc_out + (static_cast<size_t>(rg.out_slot) * a.cap_slot + idx) * 2 * W;
    for (int w = 0; w < W; ++w) {
        unsigned g[2], l[2];
        for (int h = 0; h < 2; ++h) {
            const int pi = w * 64 + h * 32 + lane;
            bool gt = false, lt = false;
            if (pi < a.n_d) {
                const lp_pair pr = s_pairs[pi];
                const float ip = S(pr.px, pr.py), iq = S(pr.qx, pr.qy);
                gt = ip > iq;
                lt = ip < iq;
            }
            g[h] = __ballot_sync(0xffffffffu, gt);
            l[h] = __ballot_sync(0xffffffffu, lt);
        }
        const uint64_t gw = static_cast<uint64_t>(g[0]) | (static_cast<uint64_t>(g[1]) << 32);
        const uint64_t lw = static_cast<uint64_t>(l[0]) | (static_cast<uint64_t>(l[1]) << 32);
        if (lane == 0) {
            d[w] = gw;
            d[W + w] = lw;
        }
        if (a.lsh_keys && lane == 0) {  // the words again for the key bits (the u8 patch is done with)
            reinterpret_cast<uint64_t*>(s_in)[w] = gw;
            reinterpret_cast<uint64_t*>(s_in)[W + w] = lw;
        }
    }
    if (a.lsh_keys) {
        // lane b builds bit b of every table's key; a ballot assembles it
        // (the same bits k_lsh_keys extracts, matchlsh.hpp:70-80)
        __syncwarp();
        const uint64_t* dw = reinterpret_cast<const uint64_t*>(s_in);
        uint64_t* out = a.lsh_keys + (static_cast<size_t>(rg.out_slot) * a.cap_slot + idx) * a.lsh_tables;
        for (int t = 0; t < a.lsh_tables; ++t) {
            uint64_t key = 0;
            for (int b0 = 0; b0 < a.lsh_bits; b0 += 32) {
                const int b = b0 + lane;
                unsigned v = 0;
                if (b < a.lsh_bits) {
                    const int p = __ldg(a.lsh_bitpos + t * a.lsh_bits + b);
                    const int q = p < a.n_d ? p : p - a.n_d;
                    v = static_cast<unsigned>((dw[(p < a.n_d ? 0 : W) + (q >> 6)] >> (q & 63)) & 1ull);
                }
                key |= static_cast<uint64_t>(__ballot_sync(0xffffffffu, v)) << b0;
            }
            if (lane == 0) out[t] = key;
        }
    }
    if (lane == 0) a.kp_out[static_cast<size_t>(rg.out_slot) * a.cap_slot + idx] = kp;
}

// top_n > kTopnSortCap: per region, the survivor keys (descending = the
// reference's (response desc, y asc, x asc) order, lorb.hpp:291-299) sorted
// by the global radix sort (prims.cuh) as two chained stable 32-bit passes
// over the inverted key (low word, then high word); slots past the survivor
// count carry ~0 and, being later in input order, stay behind every survivor
__global__ void k_topn_words(ExtractArgs a, int ri, int half, const int* idx, uint32_t* words) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.surv_cap) return;
    const int n = min(static_cast<int>(a.surv_count[ri]), a.surv_cap);
    const int j = idx ? idx[i] : i;
    const uint64_t k = j < n ? ~a.surv[static_cast<size_t>(ri) * a.surv_cap + j] : ~0ull;
    words[i] = half ? static_cast<uint32_t>(k >> 32) : static_cast<uint32_t>(k);
}
__global__ void k_topn_emit(ExtractArgs a, int ri, const int* idx) {
    const int n = min(static_cast<int>(a.surv_count[ri]), a.surv_cap);
    const int out_n = min(n, a.top_n);
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) a.count_region[ri] = out_n;
    if (i >= out_n) return;
    float r;
    int x, y;
    kp_unkey(a.surv[static_cast<size_t>(ri) * a.surv_cap + idx[i]], &r, &x, &y);
    a.kp_region[static_cast<size_t>(ri) * a.top_n + i] = lp_keypoint{x, y, r, ri};
}
static void topn_global(const ExtractArgs& a, cudaStream_t s) {
    const int n = a.surv_cap;
    DBuf ka(sizeof(uint32_t) * n, s), kb(sizeof(uint32_t) * n, s), ia(sizeof(int) * n, s), ib(sizeof(int) * n, s),
        hist(sizeof(unsigned) * 256 * cdiv(n, kPrimTile), s);
    for (int ri = 0; ri < a.nregions; ++ri) {
        LPB_LAUNCH(k_iota_int, cdiv(n, 256), 256, 0, s, ia.as<int>(), n);
        LPB_LAUNCH(k_topn_words, cdiv(n, 256), 256, 0, s, a, ri, 0, static_cast<const int*>(nullptr), ka.as<uint32_t>());
        radix_sort_pairs(ka.as<uint32_t>(), ia.as<int>(), kb.as<uint32_t>(), ib.as<int>(), n, 32, hist.as<unsigned>(), s);
        LPB_LAUNCH(k_topn_words, cdiv(n, 256), 256, 0, s, a, ri, 1, ia.as<int>(), ka.as<uint32_t>());
        radix_sort_pairs(ka.as<uint32_t>(), ia.as<int>(), kb.as<uint32_t>(), ib.as<int>(), n, 32, hist.as<unsigned>(), s);
        LPB_LAUNCH(k_topn_emit, cdiv(a.top_n, 256), 256, 0, s, a, ri, ia.as<int>());
    }
}

void extract_launch(const ExtractArgs& a, cudaStream_t s) {
    if (a.nregions == 0) return;
    LPB_CUDA(cudaMemsetAsync(a.surv_count, 0, sizeof(unsigned) * a.nregions, s));
    LPB_CUDA(cudaMemsetAsync(a.hist, 0, sizeof(unsigned) * kTopnHistBins * a.nregions, s));
    if (a.max_tiles > 0) {
        // the local name keeps the profiler key "k_detect/0" for either instance
        const bool d9 = a.harris_r == 3 && a.fast_arc == 9;
        auto* k_detect = d9 ? &lpb::k_detect9 : &lpb::k_detect<0, 0>;
        if (!d9) ensure_dyn_smem(reinterpret_cast<const void*>(k_detect), GEN_DYN_SMEM);
        LPB_LAUNCH(k_detect, dim3(a.max_tiles, a.nregions), 256, d9 ? 0 : GEN_DYN_SMEM, s, a);
    }
    if (a.top_n <= kTopnRankCap) {
        LPB_LAUNCH(k_topn, a.nregions, 1024, 0, s, a);
    } else if (a.top_n > kTopnSortCap) {
        topn_global(a, s);
    } else {
        const int topn_smem = kTopnSortCap * sizeof(uint64_t);
        ensure_dyn_smem(reinterpret_cast<const void*>(k_topn_radix), topn_smem);
        LPB_LAUNCH(k_topn_radix, a.nregions, 1024, topn_smem, s, a);
    }
    const int P = a.patch_half, RB = a.blur_r;
    const int pw = 2 * P + 1, iw = pw + 2 * RB;
    if (RB == D6_RB) {
        const int rowb6 = (iw + 6) / 4 * 4;  // k_describe6's staged row pitch
        const int warp_bytes6 = (((iw * rowb6 + 15) & ~15) + iw * pw * 4 + 15) & ~15;
        const int head6 = (a.n_d * static_cast<int>(sizeof(lp_pair)) + 15) & ~15;
        int warps6 = 8;
        while (warps6 > 1 && head6 + warps6 * warp_bytes6 > 200 * 1024) warps6 >>= 1;
        const int smem6 = head6 + warps6 * warp_bytes6;
        // one profiler key for both implementations (k_describe/0)
        auto* k_describe = &k_describe6;
        ensure_dyn_smem(reinterpret_cast<const void*>(k_describe), smem6);
        LPB_LAUNCH(k_describe, cdiv(a.nregions * a.top_n, warps6), warps6 * 32, smem6, s, a, warp_bytes6);
        return;
    }
    const int warp_bytes = (((iw * iw + 15) & ~15) + (iw * pw + pw * pw) * 4 + 15) & ~15;
    const int head = (a.n_d * static_cast<int>(sizeof(lp_pair)) + (2 * kMaxBlurR + 1) * 4 + 15) & ~15;
    int warps = 8;
    while (warps > 1 && head + warps * warp_bytes > 200 * 1024) warps >>= 1;
    const int smem = head + warps * warp_bytes;
    if (smem > 227 * 1024) throw Status(LP_BAD_PARAMS, "describe: patch too large for shared memory");
    ensure_dyn_smem(reinterpret_cast<const void*>(k_describe), smem);
    const int total = a.nregions * a.top_n;
    LPB_LAUNCH(k_describe, cdiv(total, warps), warps * 32, smem, s, a, warp_bytes);
}

// ---------------------------------------------------------------------------
// Stage-isolated primitives
__global__ void k_fast_flags(const uint8_t* img, int w, int h, int x0, int y0, int x1, int y1,
                             int t, int arc, uint8_t* flags) {
    const int sw = x1 - x0;
    const long long n = static_cast<long long>(sw) * (y1 - y0);
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        int x = x0 + static_cast<int>(i % sw), y = y0 + static_cast<int>(i / sw);
        int c = img[static_cast<size_t>(y) * w + x];
        unsigned br = 0, dk = 0;
        for (int k = 0; k < 16; ++k) {
            int v = img[static_cast<size_t>(y + c_ring_dy[k]) * w + x + c_ring_dx[k]];
            br |= (v > c + t) ? (1u << k) : 0u;
            dk |= (v < c - t) ? (1u << k) : 0u;
        }
        flags[i] = (has_arc(br, arc) || has_arc(dk, arc)) ? 1 : 0;
    }
}
void fast_flags_launch(const uint8_t* img, int w, int h, int x0, int y0, int x1, int y1, int t,
                       int arc, uint8_t* flags, cudaStream_t s) {
    long long n = static_cast<long long>(x1 - x0) * (y1 - y0);
    LPB_LAUNCH(k_fast_flags, std::min<long long>(cdiv(n, 256), 148 * 16), 256, 0, s, img, w, h,
               x0, y0, x1, y1, t, arc, flags);
}

__global__ void k_harris_points(const uint8_t* img, int w, int h, const int* xy, int n,
                                const double* wts, int R, float alpha, float* out, int* status) {
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int px = xy[2 * p], py = xy[2 * p + 1];
    if (px - R - 1 < 0 || px + R + 1 >= w || py - R - 1 < 0 || py + R + 1 >= h) {
        dev_fail(status, LP_WINDOW_OUT_OF_BOUNDS);
        return;
    }
    const int K = 2 * R + 1;
    double sa = 0.0, sb = 0.0, sc = 0.0;
    for (int v = -R; v <= R; ++v)
        for (int u = -R; u <= R; ++u) {
            const int x = px + u, y = py + v;
            const size_t o = static_cast<size_t>(y) * w + x;
            double ix = (static_cast<double>(img[o + 1]) - img[o - 1]) / 2.0;
            double iy = (static_cast<double>(img[o + w]) - img[o - w]) / 2.0;
            double wt = wts[(v + R) * K + (u + R)];
            sa = dadd(sa, dmul(dmul(wt, ix), ix));
            sb = dadd(sb, dmul(dmul(wt, iy), iy));
            sc = dadd(sc, dmul(dmul(wt, ix), iy));
        }
    double s = dadd(sa, sb);
    out[p] = __double2float_rn(dsub(dsub(dmul(sa, sb), dmul(sc, sc)),
                                    dmul(dmul(static_cast<double>(alpha), s), s)));
}
void harris_points_launch(const uint8_t* img, int w, int h, const int* xy, int n,
                          const double* wts, int r, float alpha, float* out, int* status,
                          cudaStream_t s) {
    if (n == 0) return;
    LPB_LAUNCH(k_harris_points, cdiv(n, 128), 128, 0, s, img, w, h, xy, n, wts, r, alpha, out,
               status);
}

// generic nms (lorb.hpp:254-288): dense grid over the bbox, last index wins
__global__ void k_nms_scatter(const lp_keypoint* in, int n, int minx, int miny, int gw, int* grid) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    atomicMax(&grid[static_cast<size_t>(in[i].y - miny) * gw + (in[i].x - minx)], i);
}
__global__ void k_nms_check(const lp_keypoint* in, int n, int radius, int minx, int miny, int gw,
                            int gh, const int* grid, uint8_t* keep) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const lp_keypoint k = in[i];
    bool wins = true;
    for (int dy = -radius; dy <= radius && wins; ++dy)
        for (int dx = -radius; dx <= radius && wins; ++dx) {
            if (dx == 0 && dy == 0) continue;
            int gx = k.x - minx + dx, gy = k.y - miny + dy;
            if (gx < 0 || gx >= gw || gy < 0 || gy >= gh) continue;
            int j = grid[static_cast<size_t>(gy) * gw + gx];
            if (j < 0) continue;
            const lp_keypoint o = in[j];
            if (o.response > k.response ||
                (o.response == k.response && (o.y < k.y || (o.y == k.y && o.x < k.x))))
                wins = false;
        }
    keep[i] = wins ? 1 : 0;
}
void nms_generic_launch(const lp_keypoint* in, int n, int radius, int minx, int miny, int gw,
                        int gh, int* grid, uint8_t* keep, cudaStream_t s) {
    LPB_CUDA(cudaMemsetAsync(grid, 0xff, sizeof(int) * static_cast<size_t>(gw) * gh, s));
    LPB_LAUNCH(k_nms_scatter, cdiv(n, 256), 256, 0, s, in, n, minx, miny, gw, grid);
    LPB_LAUNCH(k_nms_check, cdiv(n, 256), 256, 0, s, in, n, radius, minx, miny, gw, gh, grid, keep);
}

// generic separable blur (imgops.hpp:50-72), global-memory form
__global__ void k_blur_h(const float* in, float* out, int w, int h, int ch, const float* taps, int r) {
    long long n = static_cast<long long>(w) * h * ch;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        int c = static_cast<int>(i % ch);
        long long p = i / ch;
        int x = static_cast<int>(p % w), y = static_cast<int>(p / w);
        float acc = 0.0f;
        for (int q = -r; q <= r; ++q) {
            int xx = min(max(x + q, 0), w - 1);
            acc = fadd(acc, fmul(taps[q + r], in[(static_cast<size_t>(y) * w + xx) * ch + c]));
        }
        out[i] = acc;
    }
}
__global__ void k_blur_v(const float* in, float* out, int w, int h, int ch, const float* taps, int r) {
    long long n = static_cast<long long>(w) * h * ch;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        int c = static_cast<int>(i % ch);
        long long p = i / ch;
        int x = static_cast<int>(p % w), y = static_cast<int>(p / w);
        float acc = 0.0f;
        for (int q = -r; q <= r; ++q) {
            int yy = min(max(y + q, 0), h - 1);
            acc = fadd(acc, fmul(taps[q + r], in[(static_cast<size_t>(yy) * w + x) * ch + c]));
        }
        out[i] = acc;
    }
}
void blur_launch(const float* in, float* tmp, float* out, int w, int h, int ch, const float* taps,
                 int r, cudaStream_t s) {
    long long n = static_cast<long long>(w) * h * ch;
    int g = static_cast<int>(std::min<long long>(cdiv(n, 256), 148 * 32));
    LPB_LAUNCH(k_blur_h, g, 256, 0, s, in, tmp, w, h, ch, taps, r);
    LPB_LAUNCH(k_blur_v, g, 256, 0, s, tmp, out, w, h, ch, taps, r);
}

// brief_descriptor on a pre-smoothed image (lorb.hpp:333-350): warp per keypoint
__global__ void k_brief_generic(const float* sm, int w, int h, const lp_keypoint* kps, int n,
                                const lp_pair* pairs, int n_d, int ph, uint64_t* out, int* status) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= n) return;
    const lp_keypoint kp = kps[warp];
    if (kp.x - ph < 0 || kp.x + ph >= w || kp.y - ph < 0 || kp.y + ph >= h) {
        if (lane == 0) dev_fail(status, LP_PATCH_OUT_OF_BOUNDS);
        return;
    }
    const int W = (n_d + 63) / 64;
    uint64_t* d = out + static_cast<size_t>(warp) * 2 * W;
    for (int wd = 0; wd < W; ++wd) {
        unsigned g[2], l[2];
        for (int hh = 0; hh < 2; ++hh) {
            int pi = wd * 64 + hh * 32 + lane;
            bool gt = false, lt = false;
            if (pi < n_d) {
                lp_pair p = pairs[pi];
                float ip = sm[static_cast<size_t>(kp.y + p.py) * w + kp.x + p.px];
                float iq = sm[static_cast<size_t>(kp.y + p.qy) * w + kp.x + p.qx];
                gt = ip > iq;
                lt = ip < iq;
            }
            g[hh] = __ballot_sync(0xffffffffu, gt);
            l[hh] = __ballot_sync(0xffffffffu, lt);
        }
        if (lane == 0) {
            d[wd] = static_cast<uint64_t>(g[0]) | (static_cast<uint64_t>(g[1]) << 32);
            d[W + wd] = static_cast<uint64_t>(l[0]) | (static_cast<uint64_t>(l[1]) << 32);
        }
    }
}
void brief_generic_launch(const float* sm, int w, int h, const lp_keypoint* kps, int n,
                          const lp_pair* pairs, int n_d, int ph, uint64_t* out, int* status,
                          cudaStream_t s) {
    if (n == 0) return;
    LPB_LAUNCH(k_brief_generic, cdiv(n, 4), 128, 0, s, sm, w, h, kps, n, pairs, n_d, ph, out, status);
}

}  // namespace lpb
