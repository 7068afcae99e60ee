// homography.cu — FP64 DLT and PROSAC on the device (homography.hpp:114-286).
//
// One CTA (256 threads) per camera pair runs the whole estimator:
//  * sampling: libstdc++ mt19937_64 + uniform_int_distribution<int> (Lemire,
//    128-bit product via __umul64hi) and the Chum-Matas growth schedule are
//    replayed bit-exactly by one thread (homography.hpp:188-222);
//  * hypotheses: chunks of 8 iterations, one warp each: the 4-point DLT
//    (Hartley normalisation, 8x9 system, one-sided Jacobi SVD; homography.hpp:
//    81-144) with lane i owning row i of the 9x9 factor in registers and the
//    column dot products reduced by shuffles in the fixed tree order the
//    oracle's Eigen restatement uses; then warp-parallel symmetric transfer
//    errors (147-152) with the inlier error sum accumulated in index order;
//  * the sequential best-model / early-exit scan (248-261) on one thread, the
//    termination test read from a host-built glibc table (exact);
//  * the refit on all inliers (266-282): block-parallel inlier compaction,
//    Householder QR with the canonical 256-lane blocked dot product, then the
//    warp Jacobi SVD of the 9x9 factor.
// Compiled with --fmad=false: every FP64 expression rounds like the x86 oracle.
#include <cooperative_groups.h>

#include "homography.cuh"
#include <math_constants.h>

namespace lpb {

// ---- libstdc++ std::mt19937_64 / uniform_int_distribution<int> ----
struct Mt64 {
    uint64_t mt[312];
    int idx;
};
__device__ void mt_seed(Mt64& r, uint64_t s) {
    r.mt[0] = s;
    for (int i = 1; i < 312; ++i)
        r.mt[i] = 6364136223846793005ull * (r.mt[i - 1] ^ (r.mt[i - 1] >> 62)) + static_cast<uint64_t>(i);
    r.idx = 312;
}
__device__ uint64_t mt_next(Mt64& r) {
    if (r.idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (r.mt[i] & 0xFFFFFFFF80000000ull) | (r.mt[(i + 1) % 312] & 0x7FFFFFFFull);
            uint64_t xa = x >> 1;
            if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
            r.mt[i] = r.mt[(i + 156) % 312] ^ xa;
        }
        r.idx = 0;
    }
    uint64_t y = r.mt[r.idx++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
}
// the first twist of a freshly seeded state by one warp: the serial loop's
// data flow is three parallel phases (i < 156 reads only old words; 156 <= i
// < 311 reads old words and the new words i-156; i = 311 reads new words 0
// and 155), so the resulting state is the serial one exactly
__device__ void mt_twist_warp(Mt64& r) {
    const int lane = threadIdx.x & 31;
    auto step = [&](int i) {
        const uint64_t x = (r.mt[i] & 0xFFFFFFFF80000000ull) | (r.mt[(i + 1) % 312] & 0x7FFFFFFFull);
        uint64_t xa = x >> 1;
        if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
        return r.mt[(i + 156) % 312] ^ xa;
    };
    uint64_t v[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int i = lane + 32 * k;
        if (i < 156) v[k] = step(i);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int i = lane + 32 * k;
        if (i < 156) r.mt[i] = v[k];
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int i = 156 + lane + 32 * k;
        if (i < 311) v[k] = step(i);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int i = 156 + lane + 32 * k;
        if (i < 311) r.mt[i] = v[k];
    }
    __syncwarp();
    if (lane == 0) {
        r.mt[311] = step(311);
        r.idx = 0;
    }
    __syncwarp();
}
// the same draw with the state index in a register (the sampler's draws
// then form a short dependency chain: one shared load + tempering each)
__device__ __forceinline__ uint64_t mt_next_reg(Mt64& r, int& idx) {
    if (idx >= 312) {
        r.idx = idx;
        const uint64_t y = mt_next(r);  // twists, then consumes word 0
        idx = r.idx;
        return y;
    }
    uint64_t y = r.mt[idx++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
}
__device__ __forceinline__ int uid_int_reg(Mt64& r, int& idx, int a, int b) {
    const uint64_t range = static_cast<uint64_t>(static_cast<int64_t>(b)) -
                           static_cast<uint64_t>(static_cast<int64_t>(a)) + 1ull;
    uint64_t x = mt_next_reg(r, idx);
    uint64_t low = x * range, high = __umul64hi(x, range);
    if (low < range) {
        const uint64_t thr = (0ull - range) % range;
        while (low < thr) {
            x = mt_next_reg(r, idx);
            low = x * range;
            high = __umul64hi(x, range);
        }
    }
    return static_cast<int>(high + static_cast<uint64_t>(static_cast<int64_t>(a)));
}
__device__ int uid_int(Mt64& r, int a, int b) {
    const uint64_t range = static_cast<uint64_t>(static_cast<int64_t>(b)) -
                           static_cast<uint64_t>(static_cast<int64_t>(a)) + 1ull;
    uint64_t x = mt_next(r);
    uint64_t low = x * range, high = __umul64hi(x, range);
    if (low < range) {
        const uint64_t thr = (0ull - range) % range;
        while (low < thr) {
            x = mt_next(r);
            low = x * range;
            high = __umul64hi(x, range);
        }
    }
    return static_cast<int>(high + static_cast<uint64_t>(static_cast<int64_t>(a)));
}

// ---- Homography algebra (homography.hpp:25-62) ----
__device__ __forceinline__ double h_det(const double* h) {
    return h[0] * (h[4] * h[8] - h[5] * h[7]) - h[1] * (h[3] * h[8] - h[5] * h[6]) +
           h[2] * (h[3] * h[7] - h[4] * h[6]);
}
__device__ __forceinline__ void h_apply(const double* h, double x, double y, double& ox, double& oy) {
    double w = h[6] * x + h[7] * y + h[8];
    ox = (h[0] * x + h[1] * y + h[2]) / w;
    oy = (h[3] * x + h[4] * y + h[5]) / w;
}
__device__ bool h_inverse(const double* h, double* out) {
    double d = h_det(h);
    if (fabs(d) < 1e-12) return false;
    double inv[9] = {(h[4] * h[8] - h[5] * h[7]) / d, (h[2] * h[7] - h[1] * h[8]) / d,
                     (h[1] * h[5] - h[2] * h[4]) / d, (h[5] * h[6] - h[3] * h[8]) / d,
                     (h[0] * h[8] - h[2] * h[6]) / d, (h[2] * h[3] - h[0] * h[5]) / d,
                     (h[3] * h[7] - h[4] * h[6]) / d, (h[1] * h[6] - h[0] * h[7]) / d,
                     (h[0] * h[4] - h[1] * h[3]) / d};
    for (int i = 0; i < 9; ++i) out[i] = inv[i];
    if (fabs(out[8]) > 1e-12)
        for (int i = 0; i < 9; ++i) out[i] /= inv[8];
    return true;
}
// std::hypot as glibc >= 2.35 computes it on x86-64 (the reference's libm;
// no FMA in that build): order the magnitudes, the EPS / LARGE / TINY
// shortcuts with 2^-600 scaling, then h = sqrt(ax^2 + ay^2) corrected by one
// exact-residual Newton step (Borges, "An improved algorithm for hypot(a, b)",
// the non-FMA variant). CUDA's hypot is not that function and can differ in
// the last ulp, which could move an error across the inlier threshold or
// flip an equal-count error-sum tie (homography.hpp:206-221); this one is
// bit-identical to the host's (tests/test_gpu_parity.py: ste bit parity, and
// oracle/hypot_check.c against libm on 5e7 inputs). --fmad=false keeps every
// product and sum below separately rounded, as in the x86 build.
__device__ __forceinline__ double glibc_hypot_kernel(double ax, double ay) {
    double h = sqrt(ax * ax + ay * ay);
    double t1, t2;
    if (h <= 2.0 * ay) {
        const double delta = h - ay;
        t1 = ax * (2.0 * delta - ax);
        t2 = (delta - 2.0 * (ax - ay)) * delta;
    } else {
        const double delta = h - ax;
        t1 = 2.0 * delta * (ax - 2.0 * ay);
        t2 = (4.0 * delta - ay) * ay + delta * delta;
    }
    h -= (t1 + t2) / (2.0 * h);
    return h;
}
__device__ double glibc_hypot(double x, double y) {
    if (!isfinite(x) || !isfinite(y)) {
        if (isinf(x) || isinf(y)) return CUDART_INF;
        return x + y;  // NaN
    }
    x = fabs(x);
    y = fabs(y);
    const double ax = x < y ? y : x, ay = x < y ? x : y;
    constexpr double kScale = 0x1p-600, kLarge = 0x1p+511, kTiny = 0x1p-511, kEps = 0x1p-54;
    if (ax > kLarge) {
        if (ay <= ax * kEps) return ax + ay;
        return glibc_hypot_kernel(ax * kScale, ay * kScale) / kScale;
    }
    if (ay < kTiny) {
        if (ax >= ay / kEps) return ax + ay;
        return glibc_hypot_kernel(ax / kScale, ay / kScale) * kScale;
    }
    if (ay <= ax * kEps) return ax + ay;
    return glibc_hypot_kernel(ax, ay);
}
__device__ __forceinline__ double ste(const double* h, const double* hi, const lp_corr& c) {
    double fx, fy, bx, by;
    h_apply(h, c.sx, c.sy, fx, fy);
    h_apply(hi, c.dx, c.dy, bx, by);
    return glibc_hypot(fx - c.dx, fy - c.dy) + glibc_hypot(bx - c.sx, by - c.sy);
}

struct Norm {
    double cx, cy, scale;
};

// ---- warp-parallel one-sided Jacobi SVD of a 9x9 factor ----
constexpr unsigned kFull = 0xffffffffu;


// dot9's fixed pairwise order (oracle/shim/Eigen/Dense) over one lane's
// column: (((p0+p1)+(p2+p3))+((p4+p5)+(p6+p7)))+p8
__device__ __forceinline__ double col_dot9(const double (&a)[9], const double (&b)[9]) {
    double p[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) p[i] = a[i] * b[i];
    return (((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]))) + p[8];
}

// Lane j (< 9) holds column j of the 9x9 factor in col (col[i] = R(i, j));
// lanes >= 9 hold zeros. On return every lane holds the whole null vector hv
// (V column of the smallest singular value, stable descending order as
// Eigen::JacobiSVD sorts).
//
// Round-robin ordering shared with the oracles: round r rotates the four
// disjoint column pairs {(r+k) mod 9, (r-k) mod 9}, k = 1..4, i.e. lane j's
// partner is (2r - j) mod 9 (lane r mod 9 rests). Both lanes of a pair fetch
// each other's R and V columns (18 shuffles for all four pairs), form alpha,
// beta, gamma locally in dot9's order, compute the same rotation and update
// their own column: the products, sums and rotation formulas of the oracle,
// so the result is bit-identical to it.
__device__ void warp_jacobi_null(double (&col)[9], double (&hv)[9]) {
    const int lane = threadIdx.x & 31;
    double V[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) V[i] = lane == i ? 1.0 : 0.0;
    const double eps2 = 1e-30;
    for (int sweep = 0; sweep < 60; ++sweep) {
        bool rotated = false;
#pragma unroll 1
        for (int rnd = 0; rnd < 9; ++rnd) {
            int partner = lane;
            if (lane < 9) {
                partner = 2 * rnd - lane;
                partner += partner < 0 ? 9 : 0;
                partner += partner < 0 ? 9 : 0;
                partner -= partner >= 9 ? 9 : 0;
            }
            double oc[9], ov[9];
            // each lane's own squared norm is its partner's other one (the
            // same products in the same order): one shuffle instead of a dot
            const double own = col_dot9(col, col);
            const double other = __shfl_sync(kFull, own, partner);
#pragma unroll
            for (int i = 0; i < 9; ++i) oc[i] = __shfl_sync(kFull, col[i], partner);
#pragma unroll
            for (int i = 0; i < 9; ++i) ov[i] = __shfl_sync(kFull, V[i], partner);
            if (partner == lane) continue;
            const bool low = lane < partner;  // this lane holds column p (p < q)
            const double ga = col_dot9(col, oc);
            const double al = low ? own : other, be = low ? other : own;
            if (ga == 0.0 || ga * ga <= eps2 * (al * be) || fabs(ga) <= 2.220446049250313e-16 * fmax(al, be))
                continue;
            rotated = true;
            // the rotation that zeroes gamma: tan = sgn(d) 2g / (|d| + hypot(d, 2g)),
            // d = beta - alpha, as c = u / w and s = sgn(d) 2g / w with
            // u = |d| + hypot(d, 2g), w = hypot(u, 2g): two square roots and
            // two independent divisions on the dependency chain
            const double d = be - al, g2 = 2.0 * ga;
            const double u = fabs(d) + sqrt(d * d + g2 * g2);
            const double w = sqrt(u * u + g2 * g2);
            const double c = u / w;
            const double sn = (d >= 0.0 ? g2 : -g2) / w;
            // column p: c*up - s*uq; column q: s*up + c*uq. Both as
            // c*own + s'*other with s' = -s on p (negation and commuted
            // addition are exact), so the pair runs without divergence
            const double so = low ? -sn : sn;
#pragma unroll
            for (int i = 0; i < 9; ++i) {
                col[i] = c * col[i] + so * oc[i];
                V[i] = c * V[i] + so * ov[i];
            }
        }
        if (!__any_sync(kFull, rotated)) break;
    }
    const double myv = sqrt(col_dot9(col, col));
    double sv[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) sv[j] = __shfl_sync(kFull, myv, j);
    int order[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) order[i] = i;
    for (int i = 1; i < 9; ++i) {  // stable descending (insertion sort)
        const int x = order[i];
        int j = i - 1;
        while (j >= 0 && sv[x] > sv[order[j]]) {
            order[j + 1] = order[j];
            --j;
        }
        order[j + 1] = x;
    }
    const int jmin = order[8];
#pragma unroll
    for (int i = 0; i < 9; ++i) hv[i] = __shfl_sync(kFull, V[i], jmin);
}

// denormalise H = Td^-1 * Hn * Ts, scale h33, degeneracy checks
// (homography.hpp:129-143 with the shim's Matrix3d arithmetic)
__device__ int dlt_denormalize(const double* hv, Norm ns, Norm nd, double* H) {
    const double ts[9] = {ns.scale, 0, -ns.scale * ns.cx, 0, ns.scale, -ns.scale * ns.cy, 0, 0, 1};
    const double td[9] = {nd.scale, 0, -nd.scale * nd.cx, 0, nd.scale, -nd.scale * nd.cy, 0, 0, 1};
    double cof[9];
    cof[0] = td[4] * td[8] - td[5] * td[7];
    cof[1] = td[5] * td[6] - td[3] * td[8];
    cof[2] = td[3] * td[7] - td[4] * td[6];
    cof[3] = td[2] * td[7] - td[1] * td[8];
    cof[4] = td[0] * td[8] - td[2] * td[6];
    cof[5] = td[1] * td[6] - td[0] * td[7];
    cof[6] = td[1] * td[5] - td[2] * td[4];
    cof[7] = td[2] * td[3] - td[0] * td[5];
    cof[8] = td[0] * td[4] - td[1] * td[3];
    const double det = td[0] * cof[0] + td[1] * cof[1] + td[2] * cof[2];
    double tdi[9];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) tdi[r * 3 + c] = cof[c * 3 + r] / det;
    double t1[9], hm[9];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += tdi[r * 3 + k] * hv[k * 3 + c];
            t1[r * 3 + c] = s;
        }
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += t1[r * 3 + k] * ts[k * 3 + c];
            hm[r * 3 + c] = s;
        }
    if (fabs(hm[8]) < 1e-12) return LP_NUMERICAL_FAILURE;
    const double s8 = hm[8];
    for (int i = 0; i < 9; ++i) hm[i] /= s8;
    if (fabs(h_det(hm)) < 1e-9) return LP_DEGENERATE_CONFIGURATION;
    for (int i = 0; i < 9; ++i) H[i] = hm[i];
    return LP_OK;
}

// 4-point DLT by one warp (homography.hpp:114-144 with n == 4); every lane
// returns the same status and H
__device__ int dlt_minimal_warp(const lp_corr* p, double* H) {
    const int lane = threadIdx.x & 31;
    for (int i = 0; i < 4; ++i)
        for (int j = i + 1; j < 4; ++j)
            for (int k = j + 1; k < 4; ++k) {
                const double cross = (p[j].sx - p[i].sx) * (p[k].sy - p[i].sy) -
                                     (p[j].sy - p[i].sy) * (p[k].sx - p[i].sx);
                if (fabs(cross) < 1e-9) return LP_DEGENERATE_CONFIGURATION;
            }
    Norm ns{0, 0, 1}, nd{0, 0, 1};
    for (int i = 0; i < 4; ++i) {
        ns.cx += p[i].sx;
        ns.cy += p[i].sy;
        nd.cx += p[i].dx;
        nd.cy += p[i].dy;
    }
    ns.cx /= 4.0;
    ns.cy /= 4.0;
    nd.cx /= 4.0;
    nd.cy /= 4.0;
    double ms = 0, md = 0;
    for (int i = 0; i < 4; ++i) {
        double x = p[i].sx - ns.cx, y = p[i].sy - ns.cy;
        ms += sqrt(x * x + y * y);
        x = p[i].dx - nd.cx;
        y = p[i].dy - nd.cy;
        md += sqrt(x * x + y * y);
    }
    ms /= 4.0;
    md /= 4.0;
    ns.scale = ms > 1e-12 ? sqrt(2.0) / ms : 1.0;
    nd.scale = md > 1e-12 ? sqrt(2.0) / md : 1.0;
    // column `lane` of the 8x9 system (zero-padded to 9x9): rows 2k, 2k+1 of
    // point k are [-x,-y,-1,0,0,0,ux,uy,u] and [0,0,0,-x,-y,-1,vx,vy,v]
    double cl[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) cl[i] = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const lp_corr c = p[k];
        const double x = (c.sx - ns.cx) * ns.scale, y = (c.sy - ns.cy) * ns.scale;
        const double u = (c.dx - nd.cx) * nd.scale, v = (c.dy - nd.cy) * nd.scale;
        double e0 = 0.0, e1 = 0.0;
        switch (lane) {
            case 0: e0 = -x; break;
            case 1: e0 = -y; break;
            case 2: e0 = -1; break;
            case 3: e1 = -x; break;
            case 4: e1 = -y; break;
            case 5: e1 = -1; break;
            case 6: e0 = u * x; e1 = v * x; break;
            case 7: e0 = u * y; e1 = v * y; break;
            case 8: e0 = u; e1 = v; break;
            default: break;
        }
        cl[2 * k] = e0;
        cl[2 * k + 1] = e1;
    }
    double hv[9];
    warp_jacobi_null(cl, hv);
    return dlt_denormalize(hv, ns, nd, H);
}

// ---- block-wide pieces (blockDim.x == 256) ----
// phase timestamps of pair 0 (A/B builds only: scripts/variant.sh with
// -DLPB_PROSAC_TRACE; scripts/probes/prosac_trace.py prints them)
#ifdef LPB_PROSAC_TRACE
__device__ unsigned long long g_pt_t[64];
__device__ const char* g_pt_tag[64];
__device__ int g_pt_n;
#define PTRACE(tag)                                                                          \
    do {                                                                                     \
        if (threadIdx.x == 0 && blockIdx.x == 0 && g_pt_n < 64) {                            \
            unsigned long long t_;                                                           \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                           \
            g_pt_t[g_pt_n] = t_;                                                             \
            g_pt_tag[g_pt_n++] = tag;                                                        \
        }                                                                                    \
    } while (0)
#define PTRACE_FLUSH()                                                                       \
    do {                                                                                     \
        if (threadIdx.x == 0 && blockIdx.x == 0) {                                          \
            for (int i_ = 0; i_ < g_pt_n; ++i_) printf("PT %s %llu\n", g_pt_tag[i_], g_pt_t[i_]); \
            g_pt_n = 0;                                                                      \
        }                                                                                    \
    } while (0)
#else
#define PTRACE(tag) \
    do {            \
    } while (0)
#define PTRACE_FLUSH() \
    do {               \
    } while (0)
#endif

struct RefitShared {
    double red[9][256];
    double r[81];
    double H[9];
    double f[8], beta, v0;  // one Householder step's scalars
    int skip;
    Norm ns, nd;
    int status;
};

// dlt_homography over p[idx[0..m)] (p[0..m) when idx is null), block-wide.
// Scratch (shared or global): A 2m x 9, vbuf 2m, terms 2m. Returns the status
// on every thread; H valid on every thread.
__device__ int dlt_block(const lp_corr* p, const int* idx, int m, double* A, double* vbuf, double* terms,
                         double* H, RefitShared& sh) {
    const int tid = threadIdx.x;
    auto P = [&](int i) -> const lp_corr& { return idx ? p[idx[i]] : p[i]; };
    if (tid == 0) {
        sh.status = LP_OK;
        if (m < 4) sh.status = LP_INSUFFICIENT_MATCHES;
        if (m == 4) {
            lp_corr q[4];
            for (int i = 0; i < 4; ++i) q[i] = P(i);
            for (int i = 0; i < 4 && sh.status == LP_OK; ++i)
                for (int j = i + 1; j < 4; ++j)
                    for (int k = j + 1; k < 4; ++k) {
                        const double cross = (q[j].sx - q[i].sx) * (q[k].sy - q[i].sy) -
                                             (q[j].sy - q[i].sy) * (q[k].sx - q[i].sx);
                        if (fabs(cross) < 1e-9) sh.status = LP_DEGENERATE_CONFIGURATION;
                    }
        }
        // hartley_normalizer centroids: sequential sums (homography.hpp:83-88)
        Norm ns{0, 0, 1}, nd{0, 0, 1};
#pragma unroll 8
        for (int i = 0; i < m; ++i) {  // loads run ahead; the adds stay in order
            const lp_corr c = P(i);
            ns.cx += c.sx;
            ns.cy += c.sy;
            nd.cx += c.dx;
            nd.cy += c.dy;
        }
        ns.cx /= static_cast<double>(m);
        ns.cy /= static_cast<double>(m);
        nd.cx /= static_cast<double>(m);
        nd.cy /= static_cast<double>(m);
        sh.ns = ns;
        sh.nd = nd;
    }
    __syncthreads();
    PTRACE("centroid");
    if (sh.status != LP_OK) return sh.status;
    {
        const Norm ns = sh.ns, nd = sh.nd;
        for (int i = tid; i < m; i += blockDim.x) {  // distance terms, in parallel
            const lp_corr c = P(i);
            double x = c.sx - ns.cx, y = c.sy - ns.cy;
            terms[i] = sqrt(x * x + y * y);
            x = c.dx - nd.cx;
            y = c.dy - nd.cy;
            terms[m + i] = sqrt(x * x + y * y);
        }
    }
    __syncthreads();
    if (tid == 0) {  // mean distances: sequential sums (homography.hpp:89-95)
        double ms = 0, md = 0;
#pragma unroll 8
        for (int i = 0; i < m; ++i) {  // two independent chains, one loop
            ms += terms[i];
            md += terms[m + i];
        }
        ms /= static_cast<double>(m);
        md /= static_cast<double>(m);
        sh.ns.scale = ms > 1e-12 ? sqrt(2.0) / ms : 1.0;
        sh.nd.scale = md > 1e-12 ? sqrt(2.0) / md : 1.0;
    }
    __syncthreads();
    PTRACE("scale");
    const Norm ns = sh.ns, nd = sh.nd;
    const int rows = 2 * m;
    for (int i = tid; i < m; i += blockDim.x) {
        const lp_corr c = P(i);
        const double x = (c.sx - ns.cx) * ns.scale, y = (c.sy - ns.cy) * ns.scale;
        const double u = (c.dx - nd.cx) * nd.scale, v = (c.dy - nd.cy) * nd.scale;
        double* r0 = A + static_cast<size_t>(2 * i) * 9;
        double* r1 = r0 + 9;
        r0[0] = -x; r0[1] = -y; r0[2] = -1; r0[3] = 0; r0[4] = 0; r0[5] = 0;
        r0[6] = u * x; r0[7] = u * y; r0[8] = u;
        r1[0] = 0; r1[1] = 0; r1[2] = 0; r1[3] = -x; r1[4] = -y; r1[5] = -1;
        r1[6] = v * x; r1[7] = v * y; r1[8] = v;
    }
    __syncthreads();
    if (rows > 9) {
        // Householder QR (oracle/shim/Eigen/Dense JacobiSVD preconditioner).
        // Step j needs S = sum_{i>j} a_ij^2 and D_k = sum_{i>j} a_ij a_ik in
        // the canonical blocked order (lane = row & 255, rows ascending, then
        // the pairwise tree): thread t owns rows i = t mod 256 throughout, so
        // the pass that applies step j also accumulates step j+1's partial
        // sums from the rows it just wrote; one block reduction per column.
        double pp[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) pp[k] = 0.0;
        auto acc = [&](const double* row, int jj) {
            const double x = row[jj];
            pp[0] = pp[0] + x * x;
#pragma unroll
            for (int t = 0; t < 8; ++t)
                if (jj + 1 + t < 9) pp[1 + t] = pp[1 + t] + x * row[jj + 1 + t];
        };
        for (int i = tid; i < rows; i += 256)
            if (i > 0) acc(A + static_cast<size_t>(i) * 9, 0);
        for (int j = 0; j < 9; ++j) {
#pragma unroll
            for (int k = 0; k < 9; ++k) sh.red[k][tid] = pp[k];
            __syncthreads();
            if (tid < 32) {
                double red[9];
#pragma unroll
                for (int k = 0; k < 9; ++k) {
                    const double a0 = sh.red[k][tid] + sh.red[k][tid + 128];
                    const double a1 = sh.red[k][tid + 32] + sh.red[k][tid + 160];
                    const double a2 = sh.red[k][tid + 64] + sh.red[k][tid + 192];
                    const double a3 = sh.red[k][tid + 96] + sh.red[k][tid + 224];
                    double x = (a0 + a2) + (a1 + a3);
                    for (int o = 16; o >= 1; o >>= 1) x = x + __shfl_down_sync(kFull, x, o);
                    red[k] = x;
                }
                if (tid == 0) {
                    const double* rj = A + static_cast<size_t>(j) * 9;
                    const double alpha = rj[j];
                    const double normx = sqrt(alpha * alpha + red[0]);
                    sh.skip = normx == 0.0;
                    const double beta = alpha >= 0.0 ? -normx : normx;
                    const double v0 = alpha - beta;
                    const double vn2 = v0 * v0 + red[0];
                    for (int t = 0; t < 8; ++t)
                        sh.f[t] = j + 1 + t < 9 ? 2.0 * (v0 * rj[j + 1 + t] + red[1 + t]) / vn2 : 0.0;
                    sh.beta = beta;
                    sh.v0 = v0;
                }
            }
            __syncthreads();
            const bool skip = sh.skip;
            double f[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) f[t] = sh.f[t];
            const double beta = sh.beta, v0 = sh.v0;
#pragma unroll
            for (int k = 0; k < 9; ++k) pp[k] = 0.0;
            for (int i = j + ((tid - j) & 255); i < rows; i += 256) {
                double* row = A + static_cast<size_t>(i) * 9;
                if (!skip) {
                    const double vi = i == j ? v0 : row[j];
#pragma unroll
                    for (int t = 0; t < 8; ++t)
                        if (j + 1 + t < 9) row[j + 1 + t] = row[j + 1 + t] - f[t] * vi;
                    row[j] = i == j ? beta : 0.0;
                }
                if (j < 8 && i > j + 1) acc(row, j + 1);
            }
        }
        __syncthreads();
        for (int i = tid; i < 81; i += blockDim.x) {
            const int r = i / 9, c = i % 9;
            sh.r[i] = c < r ? 0.0 : A[static_cast<size_t>(r) * 9 + c];
        }
    } else {
        for (int i = tid; i < 81; i += blockDim.x) {
            const int r = i / 9;
            sh.r[i] = r < rows ? A[i] : 0.0;
        }
    }
    __syncthreads();
    PTRACE("qr");
    if (tid < 32) {
        double cl[9], hv[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) cl[i] = tid < 9 ? sh.r[i * 9 + tid] : 0.0;
        warp_jacobi_null(cl, hv);
        if (tid == 0) {
            double Hh[9];
            sh.status = dlt_denormalize(hv, ns, nd, Hh);
            for (int i = 0; i < 9; ++i) sh.H[i] = Hh[i];
        }
    }
    __syncthreads();
    PTRACE("svd");
    const int st = sh.status;
    for (int i = 0; i < 9; ++i) H[i] = sh.H[i];
    __syncthreads();
    return st;
}

// order-preserving compaction of {i < n : flag(i)} into idx (block-wide);
// returns the count on every thread
template <typename F>
__device__ int block_compact(int n, int* idx, F flag) {
    __shared__ int s_w[8];  // survivors per warp of the current 256
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int base = 0;
    for (int b0 = 0; b0 < n; b0 += 256) {
        const int i = b0 + threadIdx.x;
        const bool f = i < n && flag(i);
        const unsigned m = __ballot_sync(0xffffffffu, f);
        if (lane == 0) s_w[warp] = __popc(m);
        __syncthreads();
        int pos = base, total = 0;
        for (int w = 0; w < 8; ++w) {
            pos += w < warp ? s_w[w] : 0;
            total += s_w[w];
        }
        if (f) idx[pos + __popc(m & ((1u << lane) - 1u))] = i;
        base += total;
        __syncthreads();
    }
    return base;
}

constexpr int kChunk = kProsacClusterCtas;  // hypotheses per round = warps per CTA (or CTAs per cluster)
__device__ __forceinline__ double* s_dyn_refit() {
    extern __shared__ __align__(16) double s_dyn[];
    return s_dyn;
}

struct ProsacShared {
    Mt64 rng;
    int samples[kChunk][4];
    int pools[kChunk];
    double h[kChunk][9];
    double hi[kChunk][9];
    int valid[kChunk];
    int cnt[kChunk];
    double err[kChunk];
    double e[kChunk][32];
    uint8_t in[kChunk][32];
    double best_h[9], best_hi[9];
    int best_count, iterations, done, final_count;
    // cluster mode: hypothesis h of a round is scored by cluster rank h,
    // which writes its verdict here in rank 0's shared memory (DSMEM)
    struct Verdict {
        int valid, cnt;
        double err;
        double h[9], hi[9];
    } rres[kChunk];
    int c_ok, c_cnt;
    double c_err;
    double H[9], Hi[9];
    int refit_ok;
    RefitShared refit;
};

// Launched either as one CTA per pair (8 hypotheses per round, one warp
// each) or as a cluster of kChunk CTAs per pair: every rank runs the same
// deterministic sampler, rank h takes hypothesis h of the round (its 4-point
// DLT on warp 0 without FP64 contention from the others, the scoring by the
// whole CTA), verdicts meet in rank 0's shared memory, rank 0 decides and
// refits. Same hypotheses, same order of decisions, same sums: same result.
__device__ __forceinline__ void prosac_body(const ProsacArgs& a) {
    __shared__ ProsacShared S;
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int nr = static_cast<int>(cl.num_blocks());
    const bool clustered = nr == kChunk;
    const int rank = clustered ? static_cast<int>(cl.block_rank()) : 0;
    const int pair = clustered ? static_cast<int>(blockIdx.x) / kChunk : static_cast<int>(blockIdx.x);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (a.pair_status[pair] != LP_OK) return;
    PTRACE("start");
    const int n = a.counts[pair];
    const lp_corr* m = a.corr + static_cast<size_t>(pair) * a.cap;
    if (n < 4) {
        if (tid == 0 && rank == 0) {
            a.pair_status[pair] = LP_INSUFFICIENT_MATCHES;
            a.iterations[pair] = 0;
        }
        return;
    }
    // sampler state lives in thread 0's registers across rounds
    double t_n = 0, t_n_prime = 1.0;
    int pool = 0;
    double best_err = 0.0;
    if (tid == 0) {
        const uint64_t seed = a.per_pair_seed
                                  ? (a.seed ^ (a.frame * 0x9e3779b97f4a7c15ull + static_cast<uint64_t>(pair)))
                                  : a.seed;
        mt_seed(S.rng, seed);
        PTRACE("seeded");
        t_n = a.t_total;
        for (int i = 0; i < 4; ++i) t_n *= static_cast<double>(4 - i) / (n - i);
        pool = a.uniform ? n : 4;
        S.best_count = 0;
        S.iterations = 0;
        S.done = 0;
        for (int i = 0; i < 9; ++i) S.best_h[i] = (i % 4 == 0) ? 1.0 : 0.0;
    }
    __syncthreads();
    if (warp == 0) mt_twist_warp(S.rng);  // the first draw's twist, in parallel
    __syncthreads();
    PTRACE("twisted");
    const int* exit_row = a.exit_tab + (a.nmax > 0 ? static_cast<size_t>(n) * (a.nmax + 1) : 0);
    // cluster mode needs every error of a hypothesis in shared memory
    const bool cmode = clustered && n <= 27 * a.smem_rows;
    if (clustered && !cmode && rank != 0) return;  // rank 0 alone, one warp per hypothesis
    for (int t0 = 1; t0 <= a.max_iter; t0 += kChunk) {
        const int chunk = min(kChunk, a.max_iter - t0 + 1);
        if (tid == 0) {
            for (int h = 0; h < chunk; ++h) {
                const int t = t0 + h;
                while (!a.uniform && pool < n && static_cast<double>(t) > t_n_prime) {
                    double t_next = t_n * static_cast<double>(pool + 1) / (pool + 1 - 4);
                    t_n_prime += ceil(t_next - t_n);
                    t_n = t_next;
                    ++pool;
                }
                // homography.hpp:212-222: four distinct indices by rejection
                int idx = S.rng.idx, smp[4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    for (;;) {
                        const int v = uid_int_reg(S.rng, idx, 0, pool - 1);
                        bool dup = false;
#pragma unroll
                        for (int j = 0; j < i; ++j) dup |= smp[j] == v;
                        if (!dup) {
                            smp[i] = v;
                            break;
                        }
                    }
                S.rng.idx = idx;
#pragma unroll
                for (int i = 0; i < 4; ++i) S.samples[h][i] = smp[i];
                S.pools[h] = pool;
            }
        }
        __syncthreads();
        PTRACE("sampled");
        if (cmode) {
            if (rank < chunk) {
                double H[9], Hi[9];
                if (warp == 0) {
                    lp_corr q[4];
                    for (int i = 0; i < 4; ++i) q[i] = m[S.samples[rank][i]];
                    const bool ok = dlt_minimal_warp(q, H) == LP_OK && h_inverse(H, Hi);
                    if (lane == 0) {
                        S.c_ok = ok;
                        for (int i = 0; i < 9; ++i) {
                            S.h[0][i] = H[i];
                            S.hi[0][i] = Hi[i];
                        }
                    }
                }
                __syncthreads();
                const bool ok = S.c_ok;
                for (int i = 0; i < 9; ++i) {
                    H[i] = S.h[0][i];
                    Hi[i] = S.hi[0][i];
                }
                if (ok) {
                    // errors of all correspondences in parallel (-1: outlier),
                    // then the count and the in-order error sum
                    // (homography.hpp:240-247) by thread 0
                    double* se = s_dyn_refit();
                    for (int i = tid; i < n; i += 256) {
                        const double e = ste(H, Hi, m[i]);
                        se[i] = e <= a.threshold ? e : -1.0;
                    }
                    __syncthreads();
                    if (tid == 0) {
                        int count = 0;
                        double err = 0.0;
                        for (int i = 0; i < n; ++i) {
                            const double v = se[i];
                            if (v >= 0.0) {
                                ++count;
                                err += v;
                            }
                        }
                        S.c_cnt = count;
                        S.c_err = err;
                    }
                    __syncthreads();
                }
                if (tid == 0) {
                    ProsacShared::Verdict* v = cl.map_shared_rank(&S.rres[rank], 0);
                    v->valid = ok;
                    v->cnt = ok ? S.c_cnt : 0;
                    v->err = ok ? S.c_err : 0.0;
                    for (int i = 0; i < 9; ++i) {
                        v->h[i] = H[i];
                        v->hi[i] = Hi[i];
                    }
                }
            }
            cl.sync();
            if (rank == 0 && tid == 0) {
                for (int h = 0; h < chunk; ++h) {
                    S.valid[h] = S.rres[h].valid;
                    S.cnt[h] = S.rres[h].cnt;
                    S.err[h] = S.rres[h].err;
                    for (int i = 0; i < 9; ++i) {
                        S.h[h][i] = S.rres[h].h[i];
                        S.hi[h][i] = S.rres[h].hi[i];
                    }
                }
            }
        } else if (warp < chunk) {
            lp_corr q[4];
            for (int i = 0; i < 4; ++i) q[i] = m[S.samples[warp][i]];
            double H[9], Hi[9];
            const bool ok = dlt_minimal_warp(q, H) == LP_OK && h_inverse(H, Hi);
            PTRACE("minimal");
            if (ok) {
                int count = 0;
                double err = 0.0;
                for (int base = 0; base < n; base += 32) {
                    const int i = base + lane;
                    if (i < n) {
                        const double e = ste(H, Hi, m[i]);
                        S.e[warp][lane] = e;
                        S.in[warp][lane] = e <= a.threshold;
                    }
                    __syncwarp();
                    if (lane == 0) {  // homography.hpp:240-247 order
                        const int lim = min(32, n - base);
                        for (int k = 0; k < lim; ++k)
                            if (S.in[warp][k]) {
                                ++count;
                                err += S.e[warp][k];
                            }
                    }
                    __syncwarp();
                }
                if (lane == 0) {
                    S.cnt[warp] = count;
                    S.err[warp] = err;
                    for (int i = 0; i < 9; ++i) {
                        S.h[warp][i] = H[i];
                        S.hi[warp][i] = Hi[i];
                    }
                }
            }
            if (lane == 0) S.valid[warp] = ok;
        }
        __syncthreads();
        PTRACE("scored");
        if (tid == 0 && rank == 0) {
            for (int h = 0; h < chunk; ++h) {
                const int t = t0 + h;
                if (a.trace_pool) a.trace_pool[static_cast<size_t>(pair) * a.max_iter + t - 1] = S.pools[h];
                if (a.trace_samples)
                    for (int j = 0; j < 4; ++j)
                        a.trace_samples[(static_cast<size_t>(pair) * a.max_iter + t - 1) * 4 + j] = S.samples[h][j];
                S.iterations = t;
                if (!S.valid[h]) continue;
                const int count = S.cnt[h];
                const double err = S.err[h];
                if (count > S.best_count || (count == S.best_count && count > 0 && err < best_err)) {
                    for (int i = 0; i < 9; ++i) {
                        S.best_h[i] = S.h[h][i];
                        S.best_hi[i] = S.hi[h][i];
                    }
                    S.best_count = count;
                    best_err = err;
                }
                if (S.best_count >= 4 && t >= exit_row[S.best_count]) {
                    S.done = 1;
                    break;
                }
            }
        }
        __syncthreads();
        if (cmode) {
            cl.sync();  // rank 0's decision is complete
            if (tid == 0) S.c_ok = *cl.map_shared_rank(&S.done, 0);
            __syncthreads();
            if (S.c_ok) break;
        } else if (S.done) {
            break;
        }
    }
    if (cmode) {
        // every rank has read rank 0's verdict; only rank 0 goes on (no rank
        // reads another's shared memory after this point)
        cl.sync();
        if (rank != 0) return;
    }
    if (S.best_count < 4) {
        if (tid == 0) {
            a.pair_status[pair] = LP_NO_MODEL_FOUND;
            a.iterations[pair] = S.iterations;
        }
        return;
    }
    // refit on all inliers of the best hypothesis (homography.hpp:266-282)
    double* A = a.scratch + static_cast<size_t>(pair) * prosac_scratch_doubles(a.cap);
    double* vbuf = A + static_cast<size_t>(2 * a.cap) * 9;
    double* terms = vbuf + 2 * a.cap;
    int* idx = reinterpret_cast<int*>(terms + 2 * a.cap);
    uint8_t* mask = a.mask ? a.mask + static_cast<size_t>(pair) * a.cap : nullptr;
    double bh[9], bhi[9];
    for (int i = 0; i < 9; ++i) {
        bh[i] = S.best_h[i];
        bhi[i] = S.best_hi[i];
    }
    const int n_in = block_compact(n, idx, [&](int i) { return ste(bh, bhi, m[i]) <= a.threshold; });
    double Hr[9], Hri[9];
    int st;
    PTRACE("compacted");
    if (n_in <= a.smem_rows) {
        // the inliers and the whole refit system in shared memory: the
        // sequential Hartley sums and the blocked QR passes read on-chip
        double* s_refit = s_dyn_refit();
        double* sA = s_refit;                                        // 2 n_in x 9
        double* sv = sA + static_cast<size_t>(2 * a.smem_rows) * 9;  // 2 n_in
        double* st_terms = sv + 2 * a.smem_rows;                     // 2 n_in
        lp_corr* sc = reinterpret_cast<lp_corr*>(st_terms + 2 * a.smem_rows);
        for (int i = tid; i < n_in; i += blockDim.x) sc[i] = m[idx[i]];
        __syncthreads();
        PTRACE("staged");
        st = dlt_block(sc, nullptr, n_in, sA, sv, st_terms, Hr, S.refit);
    } else {
        st = dlt_block(m, idx, n_in, A, vbuf, terms, Hr, S.refit);
    }
    if (tid == 0) {
        S.refit_ok = st == LP_OK && h_inverse(Hr, Hri);
        for (int i = 0; i < 9; ++i) {
            S.H[i] = S.refit_ok ? Hr[i] : bh[i];
            S.Hi[i] = S.refit_ok ? Hri[i] : bhi[i];
        }
        S.final_count = 0;
    }
    __syncthreads();
    double fh[9], fhi[9];
    for (int i = 0; i < 9; ++i) {
        fh[i] = S.H[i];
        fhi[i] = S.Hi[i];
    }
    int local = 0;
    for (int i = tid; i < n; i += blockDim.x) {
        const bool in = ste(fh, fhi, m[i]) <= a.threshold;
        if (mask) mask[i] = in;
        local += in;
    }
    for (int off = 16; off > 0; off >>= 1) local += __shfl_xor_sync(kFull, local, off);
    if (lane == 0) atomicAdd(&S.final_count, local);
    __syncthreads();
    PTRACE("end");
    PTRACE_FLUSH();
    if (tid == 0) {
        const int cnt = S.final_count;
        for (int i = 0; i < 9; ++i) a.model[pair].h[i] = fh[i];
        a.inlier_count[pair] = cnt;
        a.iterations[pair] = S.iterations;
        a.pair_status[pair] = cnt < 4 ? LP_NO_MODEL_FOUND : LP_OK;
    }
}

__global__ void __launch_bounds__(256, 1) k_prosac(ProsacArgs a);

void prosac_launch(const ProsacArgs& a0, cudaStream_t s) {
    ProsacArgs a = a0;
    // refit rows kept on chip: 2 rows x 9 + 2 + 2 doubles and one lp_corr per inlier
    a.smem_rows = std::min(a.cap, kRefitSmemRows);
    const int smem = a.smem_rows * static_cast<int>(2 * 9 * 8 + 2 * 8 + 2 * 8 + sizeof(lp_corr));
    ensure_dyn_smem(reinterpret_cast<const void*>(&k_prosac), smem);
    // a cluster of kChunk CTAs per pair (LPB_PROSAC_CLUSTER=0: one CTA)
    static const bool use_cluster = [] {
        const char* e = std::getenv("LPB_PROSAC_CLUSTER");
        return !(e && std::strcmp(e, "0") == 0);
    }();
    if (!use_cluster) {
        LPB_LAUNCH(k_prosac, a.npairs, 256, smem, s, a);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.npairs * kChunk);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kChunk;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const int pt = prof_begin("k_prosac", s);
    const cudaError_t e = cudaLaunchKernelEx(&cfg, k_prosac, a);
    if (e != cudaSuccess) {
        // no room for an 8-CTA cluster (a partitioned or busy device): the
        // one-CTA launch computes the same result
        cudaGetLastError();
        k_prosac<<<a.npairs, 256, smem, s>>>(a);
        LPB_CUDA(cudaGetLastError());
    }
    prof_end(pt, s);
    note_launch();
}

// HomographyCache chain (pipeline.hpp:474-494): chain[0] = I, chain[i+1] =
// chain[i] * H_pair(i), renormalised by h33; first failing pair's status wins
__device__ void chain_compose(const lp_homography* ph, const int* pst, int npairs, lp_homography* chain,
                              int* chain_status) {
    int st = LP_OK;
    for (int i = 0; i < npairs; ++i)
        if (pst[i] != LP_OK && st == LP_OK) st = pst[i];
    *chain_status = st;
    if (st != LP_OK) return;
    double c[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    for (int i = 0; i < 9; ++i) chain[0].h[i] = c[i];
    for (int p = 0; p < npairs; ++p) {
        const double* b = ph[p].h;
        double o[9];
        for (int r = 0; r < 3; ++r)
            for (int cc = 0; cc < 3; ++cc) {
                double s = 0;
                for (int k = 0; k < 3; ++k) s += c[r * 3 + k] * b[k * 3 + cc];
                o[r * 3 + cc] = s;
            }
        if (fabs(o[8]) > 1e-12) {
            const double d8 = o[8];
            for (int i = 0; i < 8; ++i) o[i] /= d8;
            o[8] /= o[8];
        }
        for (int i = 0; i < 9; ++i) {
            c[i] = o[i];
            chain[p + 1].h[i] = o[i];
        }
    }
}

__global__ void k_chain(const lp_homography* ph, const int* pst, int npairs, lp_homography* chain,
                        int* chain_status) {
    if (threadIdx.x == 0) chain_compose(ph, pst, npairs, chain, chain_status);
}

__global__ void __launch_bounds__(256, 1) k_prosac(ProsacArgs a) {
    prosac_body(a);
    if (!a.chain_counter || threadIdx.x != 0) return;
    namespace cg = cooperative_groups;
    const cg::cluster_group cl = cg::this_cluster();
    if (cl.num_blocks() > 1 && cl.block_rank() != 0) return;
    // every pair's verdict is final: the last one composes the chain
    __threadfence();
    if (atomicAdd(a.chain_counter, 1u) == static_cast<unsigned>(a.npairs - 1)) {
        __threadfence();
        chain_compose(a.model, a.pair_status, a.npairs, a.chain, a.chain_status);
        *a.chain_counter = 0u;
    }
}

void chain_launch(const lp_homography* pair_h, const int* pair_status, int npairs,
                  lp_homography* chain, int* chain_status, cudaStream_t s) {
    LPB_LAUNCH(k_chain, 1, 32, 0, s, pair_h, pair_status, npairs, chain, chain_status);
}

__global__ void __launch_bounds__(256) k_dlt(const lp_corr* c, int n, double* scratch,
                                             lp_homography* out, int* status) {
    __shared__ RefitShared sh;
    double* A = scratch;
    double* vbuf = A + static_cast<size_t>(2 * n) * 9;
    double* terms = vbuf + 2 * n;
    int* idx = reinterpret_cast<int*>(terms + 2 * n);
    for (int i = threadIdx.x; i < n; i += blockDim.x) idx[i] = i;
    __syncthreads();
    double H[9];
    const int st = dlt_block(c, idx, n, A, vbuf, terms, H, sh);
    if (threadIdx.x == 0) {
        *status = st;
        if (st == LP_OK)
            for (int i = 0; i < 9; ++i) out->h[i] = H[i];
    }
}

void dlt_launch(const lp_corr* c, int n, double* scratch, lp_homography* out, int* status,
                cudaStream_t s) {
    LPB_LAUNCH(k_dlt, 1, 256, 0, s, c, n, scratch, out, status);
}

// symmetric_transfer_error (homography.hpp:147-152) of n correspondences
__global__ void k_ste(lp_homography h, lp_homography hi, const lp_corr* c, int n, double* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = ste(h.h, hi.h, c[i]);
}
void ste_launch(const lp_homography& h, const lp_homography& hi, const lp_corr* c, int n, double* out,
                cudaStream_t s) {
    if (n > 0) LPB_LAUNCH(k_ste, cdiv(n, 256), 256, 0, s, h, hi, c, n, out);
}

}  // namespace lpb
