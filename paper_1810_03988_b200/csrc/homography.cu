// homography.cu — FP64 DLT and PROSAC on the device (homography.hpp:114-286).
//
// One CTA (256 threads) per camera pair runs the whole estimator:
//  * sampling: libstdc++ mt19937_64 + uniform_int_distribution<int> (Lemire,
//    128-bit product via __umul64hi) and the Chum-Matas growth schedule are
//    replayed bit-exactly by one thread (homography.hpp:188-222);
//  * hypotheses: chunks of 8 iterations, one warp each: the 4-point DLT
//    (Hartley normalisation, 8x9 system, one-sided Jacobi SVD of the padded
//    9x9, denormalisation, h33 scaling; homography.hpp:81-144) on lane 0, then
//    warp-parallel symmetric-transfer-error scoring (147-152) with the inlier
//    error sum accumulated in the reference's index order;
//  * the sequential best-model / early-exit scan (248-261) on one thread, with
//    the termination test read from a host-built glibc table (exact);
//  * the final refit on all inliers: block-parallel Householder QR with the
//    canonical 256-lane blocked dot product shared with the oracle's Eigen
//    restatement, then the 9x9 Jacobi SVD (266-282).
// Compiled with --fmad=false: every FP64 expression rounds like the x86 oracle.
#include "homography.cuh"

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
__device__ __forceinline__ double ste(const double* h, const double* hi, const lp_corr& c) {
    double fx, fy, bx, by;
    h_apply(h, c.sx, c.sy, fx, fy);
    h_apply(hi, c.dx, c.dy, bx, by);
    return hypot(fx - c.dx, fy - c.dy) + hypot(bx - c.sx, by - c.sy);
}

struct Norm {
    double cx, cy, scale;
};

// one-sided Jacobi SVD of the 9x9 factor r (row-major), V column of the
// smallest singular value -> hv. Mirrors oracle/shim/Eigen/Dense exactly.
__device__ void jacobi_null_vector(double* r, double* hv) {
    constexpr int N = 9;
    double V[N * N];
    for (int i = 0; i < N * N; ++i) V[i] = 0.0;
    for (int i = 0; i < N; ++i) V[i * N + i] = 1.0;
    const double eps = 1e-15;
    for (int sweep = 0; sweep < 60; ++sweep) {
        bool rotated = false;
        for (int p = 0; p < N - 1; ++p)
            for (int q = p + 1; q < N; ++q) {
                double al = 0, be = 0, ga = 0;
                for (int i = 0; i < N; ++i) {
                    al += r[i * N + p] * r[i * N + p];
                    be += r[i * N + q] * r[i * N + q];
                    ga += r[i * N + p] * r[i * N + q];
                }
                if (ga == 0.0 || fabs(ga) <= eps * sqrt(al * be)) continue;
                rotated = true;
                const double zeta = (be - al) / (2.0 * ga);
                const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + t * t);
                const double s = c * t;
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
    for (int j = 0; j < N; ++j) {
        double s = 0;
        for (int i = 0; i < N; ++i) s += r[i * N + j] * r[i * N + j];
        sv[j] = sqrt(s);
    }
    int order[N];
    for (int i = 0; i < N; ++i) order[i] = i;
    for (int i = 1; i < N; ++i) {
        int x = order[i], j = i - 1;
        while (j >= 0 && sv[x] > sv[order[j]]) {
            order[j + 1] = order[j];
            --j;
        }
        order[j + 1] = x;
    }
    for (int i = 0; i < N; ++i) hv[i] = V[i * N + order[N - 1]];
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

// 4-point DLT by one thread (homography.hpp:114-144 with n == 4)
__device__ int dlt_minimal(const lp_corr* p, double* H) {
    for (int i = 0; i < 4; ++i)
        for (int j = i + 1; j < 4; ++j)
            for (int k = j + 1; k < 4; ++k) {
                double cross = (p[j].sx - p[i].sx) * (p[k].sy - p[i].sy) -
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
    double r[81];
    for (int i = 0; i < 81; ++i) r[i] = 0.0;
    for (int i = 0; i < 4; ++i) {
        const double x = (p[i].sx - ns.cx) * ns.scale, y = (p[i].sy - ns.cy) * ns.scale;
        const double u = (p[i].dx - nd.cx) * nd.scale, v = (p[i].dy - nd.cy) * nd.scale;
        double* r0 = r + (2 * i) * 9;
        double* r1 = r0 + 9;
        r0[0] = -x; r0[1] = -y; r0[2] = -1; r0[6] = u * x; r0[7] = u * y; r0[8] = u;
        r1[3] = -x; r1[4] = -y; r1[5] = -1; r1[6] = v * x; r1[7] = v * y; r1[8] = v;
    }
    double hv[9];
    jacobi_null_vector(r, hv);
    return dlt_denormalize(hv, ns, nd, H);
}

// ---- block-wide pieces (blockDim.x == 256) ----
// canonical blocked dot products (oracle/shim/Eigen/Dense dot_blocked): lane
// l = row & 255 accumulates rows in increasing order, then a pairwise tree.
template <int K>
__device__ void block_dots(const double* v, int sv, const double* const* cols, int sc, int r0,
                           int r1, double (*s_red)[256], double* out) {
    const int l = threadIdx.x;
    double p[K];
#pragma unroll
    for (int k = 0; k < K; ++k) p[k] = 0.0;
    const int i0 = r0 + ((l - (r0 & 255)) & 255);
    for (int i = i0; i < r1; i += 256) {
        const double vi = v[static_cast<size_t>(i) * sv];
#pragma unroll
        for (int k = 0; k < K; ++k)
            if (cols[k]) p[k] = p[k] + vi * cols[k][static_cast<size_t>(i) * sc];
    }
#pragma unroll
    for (int k = 0; k < K; ++k) s_red[k][l] = p[k];
    __syncthreads();
    for (int s = 128; s >= 1; s >>= 1) {
        if (l < s)
#pragma unroll
            for (int k = 0; k < K; ++k) s_red[k][l] = s_red[k][l] + s_red[k][l + s];
        __syncthreads();
    }
#pragma unroll
    for (int k = 0; k < K; ++k) out[k] = s_red[k][0];
    __syncthreads();
}

struct RefitShared {
    double red[8][256];
    double r[81];
    double f[8];
    double scal[4];
    Norm ns, nd;
    int status;
};

// dlt_homography over idx[0..m) of p (block-wide). A: 2m x 9 scratch, v: 2m scratch.
__device__ int dlt_block(const lp_corr* p, const int* idx, int m, double* A, double* vbuf,
                         double* H, RefitShared& sh) {
    const int tid = threadIdx.x;
    if (tid == 0) {
        sh.status = LP_OK;
        if (m < 4) sh.status = LP_INSUFFICIENT_MATCHES;
        if (m == 4) {
            lp_corr q[4];
            for (int i = 0; i < 4; ++i) q[i] = p[idx[i]];
            for (int i = 0; i < 4 && sh.status == LP_OK; ++i)
                for (int j = i + 1; j < 4; ++j)
                    for (int k = j + 1; k < 4; ++k) {
                        double cross = (q[j].sx - q[i].sx) * (q[k].sy - q[i].sy) -
                                       (q[j].sy - q[i].sy) * (q[k].sx - q[i].sx);
                        if (fabs(cross) < 1e-9) sh.status = LP_DEGENERATE_CONFIGURATION;
                    }
        }
        // hartley_normalizer, sequential sums (homography.hpp:81-97)
        Norm ns{0, 0, 1}, nd{0, 0, 1};
        for (int i = 0; i < m; ++i) {
            ns.cx += p[idx[i]].sx;
            ns.cy += p[idx[i]].sy;
        }
        for (int i = 0; i < m; ++i) {
            nd.cx += p[idx[i]].dx;
            nd.cy += p[idx[i]].dy;
        }
        ns.cx /= static_cast<double>(m);
        ns.cy /= static_cast<double>(m);
        nd.cx /= static_cast<double>(m);
        nd.cy /= static_cast<double>(m);
        double ms = 0, md = 0;
        for (int i = 0; i < m; ++i) {
            double x = p[idx[i]].sx - ns.cx, y = p[idx[i]].sy - ns.cy;
            ms += sqrt(x * x + y * y);
        }
        for (int i = 0; i < m; ++i) {
            double x = p[idx[i]].dx - nd.cx, y = p[idx[i]].dy - nd.cy;
            md += sqrt(x * x + y * y);
        }
        ms /= static_cast<double>(m);
        md /= static_cast<double>(m);
        ns.scale = ms > 1e-12 ? sqrt(2.0) / ms : 1.0;
        nd.scale = md > 1e-12 ? sqrt(2.0) / md : 1.0;
        sh.ns = ns;
        sh.nd = nd;
    }
    __syncthreads();
    if (sh.status != LP_OK) return sh.status;
    const Norm ns = sh.ns, nd = sh.nd;
    const int rows = 2 * m;
    for (int i = tid; i < m; i += blockDim.x) {
        const lp_corr c = p[idx[i]];
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
        // Householder QR (oracle/shim/Eigen/Dense JacobiSVD preconditioner)
        for (int j = 0; j < 9; ++j) {
            const double* cj[1] = {A + j};
            double nrm2;
            block_dots<1>(A + j, 9, cj, 9, j, rows, sh.red, &nrm2);
            const double normx = sqrt(nrm2);
            if (normx == 0.0) continue;
            const double alpha = A[static_cast<size_t>(j) * 9 + j];
            const double beta = alpha >= 0.0 ? -normx : normx;
            for (int i = tid; i < rows; i += blockDim.x)
                vbuf[i] = i < j ? 0.0 : (i == j ? alpha - beta : A[static_cast<size_t>(i) * 9 + j]);
            __syncthreads();
            const double* cv[1] = {vbuf};
            double vn2;
            block_dots<1>(vbuf, 1, cv, 1, j, rows, sh.red, &vn2);
            const double* ck[8];
            for (int k = 0; k < 8; ++k) ck[k] = (j + 1 + k < 9) ? A + j + 1 + k : nullptr;
            double dk[8];
            block_dots<8>(vbuf, 1, ck, 9, j, rows, sh.red, dk);
            double f[8];
            for (int k = 0; k < 8; ++k) f[k] = 2.0 * dk[k] / vn2;
            for (int i = j + tid; i < rows; i += blockDim.x) {
                const double vi = vbuf[i];
                double* row = A + static_cast<size_t>(i) * 9;
                for (int k = j + 1; k < 9; ++k) row[k] = row[k] - f[k - j - 1] * vi;
                row[j] = i == j ? beta : 0.0;
            }
            __syncthreads();
        }
        for (int i = tid; i < 81; i += blockDim.x) {
            int r = i / 9, c = i % 9;
            sh.r[i] = c < r ? 0.0 : A[static_cast<size_t>(r) * 9 + c];
        }
    } else {
        for (int i = tid; i < 81; i += blockDim.x) {
            int r = i / 9;
            sh.r[i] = r < rows ? A[i] : 0.0;
        }
    }
    __syncthreads();
    if (tid == 0) {
        double r[81], hv[9];
        for (int i = 0; i < 81; ++i) r[i] = sh.r[i];
        jacobi_null_vector(r, hv);
        double Hh[9];
        sh.status = dlt_denormalize(hv, ns, nd, Hh);
        if (sh.status == LP_OK)
            for (int i = 0; i < 9; ++i) H[i] = Hh[i];
    }
    __syncthreads();
    return sh.status;
}

constexpr int kChunk = 8;  // hypotheses per round = warps per CTA

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
    int best_count, iterations, done, n_in, final_count;
    double H[9];
    RefitShared refit;
};

__global__ void __launch_bounds__(256) k_prosac(ProsacArgs a) {
    __shared__ ProsacShared S;
    const int pair = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (a.pair_status[pair] != LP_OK) return;
    const int n = a.counts[pair];
    const lp_corr* m = a.corr + static_cast<size_t>(pair) * a.cap;
    if (n < 4) {
        if (tid == 0) {
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
        t_n = a.t_total;
        for (int i = 0; i < 4; ++i) t_n *= static_cast<double>(4 - i) / (n - i);
        pool = a.uniform ? n : 4;
        S.best_count = 0;
        S.iterations = 0;
        S.done = 0;
        for (int i = 0; i < 9; ++i) S.best_h[i] = (i % 4 == 0) ? 1.0 : 0.0;
    }
    const int* exit_row = a.exit_tab + (a.nmax > 0 ? static_cast<size_t>(n) * (a.nmax + 1) : 0);
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
                for (int i = 0; i < 4; ++i)
                    for (;;) {
                        int v = uid_int(S.rng, 0, pool - 1);
                        bool dup = false;
                        for (int j = 0; j < i; ++j) dup |= S.samples[h][j] == v;
                        if (!dup) {
                            S.samples[h][i] = v;
                            break;
                        }
                    }
                S.pools[h] = pool;
            }
        }
        __syncthreads();
        if (warp < chunk) {
            if (lane == 0) {
                lp_corr q[4];
                for (int i = 0; i < 4; ++i) q[i] = m[S.samples[warp][i]];
                double H[9], Hi[9];
                int ok = dlt_minimal(q, H) == LP_OK && h_inverse(H, Hi);
                S.valid[warp] = ok;
                if (ok)
                    for (int i = 0; i < 9; ++i) {
                        S.h[warp][i] = H[i];
                        S.hi[warp][i] = Hi[i];
                    }
            }
            __syncwarp();
            if (S.valid[warp]) {
                double hh[9], hhi[9];
                for (int i = 0; i < 9; ++i) {
                    hh[i] = S.h[warp][i];
                    hhi[i] = S.hi[warp][i];
                }
                int count = 0;
                double err = 0.0;
                for (int base = 0; base < n; base += 32) {
                    const int i = base + lane;
                    if (i < n) {
                        const double e = ste(hh, hhi, m[i]);
                        S.e[warp][lane] = e;
                        S.in[warp][lane] = e <= a.threshold;
                    }
                    __syncwarp();
                    if (lane == 0) {
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
                }
            }
        }
        __syncthreads();
        if (tid == 0) {
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
        if (S.done) break;
    }
    if (S.best_count < 4) {
        if (tid == 0) {
            a.pair_status[pair] = LP_NO_MODEL_FOUND;
            a.iterations[pair] = S.iterations;
        }
        return;
    }
    // refit on all inliers of the best hypothesis (homography.hpp:266-282)
    double* A = a.scratch + static_cast<size_t>(pair) * (2 * a.cap * 9 + 2 * a.cap + a.cap);
    double* vbuf = A + static_cast<size_t>(2 * a.cap) * 9;
    int* idx = reinterpret_cast<int*>(vbuf + 2 * a.cap);
    uint8_t* mask = a.mask ? a.mask + static_cast<size_t>(pair) * a.cap : nullptr;
    if (tid == 0) {
        int k = 0;
        for (int i = 0; i < n; ++i)
            if (ste(S.best_h, S.best_hi, m[i]) <= a.threshold) idx[k++] = i;
        S.n_in = k;
    }
    __syncthreads();
    double Hr[9];
    int st = dlt_block(m, idx, S.n_in, A, vbuf, Hr, S.refit);
    if (tid == 0) {
        double Hri[9];
        const double* use_h = S.best_h;
        const double* use_hi = S.best_hi;
        if (st == LP_OK && h_inverse(Hr, Hri)) {
            for (int i = 0; i < 9; ++i) {
                S.H[i] = Hr[i];
                S.best_hi[i] = Hri[i];
            }
            use_h = S.H;
        } else {
            for (int i = 0; i < 9; ++i) S.H[i] = S.best_h[i];
            use_h = S.H;
        }
        int cnt = 0;
        for (int i = 0; i < n; ++i) {
            bool in = ste(use_h, use_hi, m[i]) <= a.threshold;
            if (mask) mask[i] = in;
            cnt += in;
        }
        S.final_count = cnt;
        for (int i = 0; i < 9; ++i) a.model[pair].h[i] = S.H[i];
        a.inlier_count[pair] = cnt;
        a.iterations[pair] = S.iterations;
        a.pair_status[pair] = cnt < 4 ? LP_NO_MODEL_FOUND : LP_OK;
    }
}

void prosac_launch(const ProsacArgs& a, cudaStream_t s) {
    if (a.npairs <= 0) return;
    LPB_LAUNCH(k_prosac, a.npairs, 256, 0, s, a);
}

__global__ void k_chain(const lp_homography* ph, const int* pst, int npairs, lp_homography* chain,
                        int* chain_status) {
    if (threadIdx.x != 0) return;
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

void chain_launch(const lp_homography* pair_h, const int* pair_status, int npairs,
                  lp_homography* chain, int* chain_status, cudaStream_t s) {
    LPB_LAUNCH(k_chain, 1, 32, 0, s, pair_h, pair_status, npairs, chain, chain_status);
}

__global__ void __launch_bounds__(256) k_dlt(const lp_corr* c, int n, double* scratch,
                                             lp_homography* out, int* status) {
    __shared__ RefitShared sh;
    double* A = scratch;
    double* vbuf = A + static_cast<size_t>(2 * n) * 9;
    int* idx = reinterpret_cast<int*>(vbuf + 2 * n);
    for (int i = threadIdx.x; i < n; i += blockDim.x) idx[i] = i;
    __syncthreads();
    double H[9];
    int st = dlt_block(c, idx, n, A, vbuf, H, sh);
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

}  // namespace lpb
