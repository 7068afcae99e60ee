// homography.cuh — device DLT + PROSAC (homography.hpp:114-286), batched over pairs.
#pragma once
#include "common.cuh"

namespace lpb {

struct ProsacArgs {
    int npairs;
    const lp_corr* corr;        // npairs * cap, quality-sorted (match order)
    const int* counts;          // npairs (n_total per pair)
    int cap;
    double threshold;
    int max_iter;
    int uniform;                // SamplingMode::Uniform
    double t_total;
    uint64_t seed;              // per-pair seed = seed ^ (frame * golden + pair) when per_pair_seed
    uint64_t frame;
    int per_pair_seed;
    const int* exit_tab;        // (nmax+1)^2 termination table, host-built with glibc
    int nmax;
    double* scratch;            // npairs * 2*cap*9 doubles (refit system)
    lp_homography* model;       // npairs
    uint8_t* mask;              // npairs * cap (optional)
    int* inlier_count;          // npairs
    int* iterations;            // npairs
    int* trace_pool;            // npairs * max_iter (optional)
    int* trace_samples;         // npairs * max_iter * 4 (optional)
    int* pair_status;           // npairs: in = upstream status (0 ok), out = PROSAC status
    int smem_rows;              // set by prosac_launch: refits with <= this many inliers run in shared memory
    // optional: the last pair to finish composes the camera chain
    // (pipeline.hpp:474-494) in the same launch; counter zero on entry
    lp_homography* chain;       // npairs + 1
    int* chain_status;
    unsigned* chain_counter;
};

constexpr int kProsacClusterCtas = 8;  // k_prosac: CTAs per pair (one thread-block cluster)
constexpr int kRefitSmemRows = 800;  // 800 x 232 B = 186 KB of dynamic shared memory

// scratch doubles per pair: refit system A (2cap x 9), Householder vector
// (2cap), Hartley distance terms (2cap), inlier index list (cap ints)
__host__ __device__ inline size_t prosac_scratch_doubles(int cap) { return static_cast<size_t>(cap) * 24; }

void prosac_launch(const ProsacArgs& a, cudaStream_t s);

// chain[0] = I, chain[i+1] = chain[i] ∘ H_i (pipeline.hpp:474-493); any pair
// failure sets *chain_status (the estimator throws).
void chain_launch(const lp_homography* pair_h, const int* pair_status, int npairs,
                  lp_homography* chain, int* chain_status, cudaStream_t s);

// dlt_homography on one correspondence set (C-ABI lp_dlt_homography)
// symmetric_transfer_error of each correspondence (glibc hypot, bit-exact)
void ste_launch(const lp_homography& h, const lp_homography& hi, const lp_corr* c, int n, double* out,
                cudaStream_t s);
void dlt_launch(const lp_corr* c, int n, double* scratch, lp_homography* out, int* status,
                cudaStream_t s);

}  // namespace lpb
