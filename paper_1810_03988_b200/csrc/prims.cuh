// prims.cuh — order-preserving compaction and a stable LSD radix sort, the
// building blocks of the stage-isolated primitives (lp_fast_corners, lp_nms,
// lp_select_top_n; lorb.hpp:192-299). Tiles of 2048 elements walked in eight
// rounds of 256 consecutive elements, so every ranking is in input order:
// compaction ranks by warp ballots, the sort ranks equal digits by
// __match_any_sync. Offsets come from one exclusive scan of per-tile counts
// (compaction) or of the digit-major [256][tiles] histogram (sort).
#pragma once
#include "common.cuh"

namespace lpb {

constexpr int kPrimTile = 2048;  // elements per tile: 8 rounds x 256 threads

// ---- exclusive scan of n ints in place by one CTA (carry across chunks);
// *total (optional) gets the sum
static __global__ void __launch_bounds__(1024) k_scan_exclusive(unsigned* a, int n, int* total) {
    __shared__ unsigned s_warp[32];
    __shared__ unsigned s_carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (int base = 0; base < n; base += 1024) {
        const int i = base + tid;
        const unsigned v = i < n ? a[i] : 0u;
        unsigned x = v;  // inclusive warp scan
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_warp[warp] = x;
        __syncthreads();
        if (warp == 0) {
            unsigned w = s_warp[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            s_warp[lane] = w;  // inclusive over warps
        }
        __syncthreads();
        const unsigned carry = s_carry;
        const unsigned excl = carry + (warp ? s_warp[warp - 1] : 0u) + x - v;
        if (i < n) a[i] = excl;
        __syncthreads();
        if (tid == 1023) s_carry = carry + s_warp[31];
        __syncthreads();
    }
    if (total && tid == 0) *total = static_cast<int>(s_carry);
}

// ---- compaction: counts per tile, then scatter by ballot ranks
static __global__ void __launch_bounds__(256) k_flag_count(const uint8_t* flags, int n, unsigned* tile_count) {
    const int base = blockIdx.x * kPrimTile;
    int c = 0;
#pragma unroll
    for (int r = 0; r < kPrimTile / 256; ++r) {
        const int i = base + r * 256 + threadIdx.x;
        c += __syncthreads_count(i < n && flags[i]);
    }
    if (threadIdx.x == 0) tile_count[blockIdx.x] = static_cast<unsigned>(c);
}

// write(i, j): flagged element i is the j-th survivor
template <class W>
static __global__ void __launch_bounds__(256) k_flag_scatter(const uint8_t* flags, int n, const unsigned* tile_off, W write) {
    __shared__ unsigned s_w[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int base = blockIdx.x * kPrimTile;
    unsigned running = tile_off[blockIdx.x];
    for (int r = 0; r < kPrimTile / 256; ++r) {
        const int i = base + r * 256 + tid;
        const bool f = i < n && flags[i];
        const unsigned m = __ballot_sync(0xffffffffu, f);
        if (lane == 0) s_w[warp] = __popc(m);
        __syncthreads();
        unsigned before = running;
        for (int w = 0; w < warp; ++w) before += s_w[w];
        if (f) write(i, static_cast<int>(before + __popc(m & ((1u << lane) - 1u))));
        unsigned all = 0;
        for (int w = 0; w < 8; ++w) all += s_w[w];
        running += all;
        __syncthreads();
    }
}

// ---- stable LSD radix sort pass (8-bit digit at `shift`) of 32-bit keys
// with int payloads
static __global__ void __launch_bounds__(256) k_radix_hist(const uint32_t* keys, int n, int shift, unsigned* hist,
                                                     int ntiles) {
    __shared__ unsigned s_h[256];
    s_h[threadIdx.x] = 0;
    __syncthreads();
    const int base = blockIdx.x * kPrimTile;
    for (int r = 0; r < kPrimTile / 256; ++r) {
        const int i = base + r * 256 + threadIdx.x;
        if (i < n) atomicAdd(&s_h[(keys[i] >> shift) & 255u], 1u);
    }
    __syncthreads();
    hist[threadIdx.x * ntiles + blockIdx.x] = s_h[threadIdx.x];  // digit-major: one scan orders digits, then tiles
}

static __global__ void __launch_bounds__(256) k_radix_scatter(const uint32_t* kin, const int* vin, int n, int shift,
                                                        const unsigned* off, int ntiles, uint32_t* kout, int* vout) {
    __shared__ unsigned s_wc[8][256];  // this round: elements per (warp, digit)
    __shared__ unsigned s_run[256];    // this tile so far: elements per digit
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int base = blockIdx.x * kPrimTile;
    s_run[tid] = off[tid * ntiles + blockIdx.x];
    for (int r = 0; r < kPrimTile / 256; ++r) {
#pragma unroll
        for (int w = 0; w < 8; ++w) s_wc[w][tid] = 0;
        __syncthreads();
        const int i = base + r * 256 + tid;
        const bool live = i < n;
        const uint32_t k = live ? kin[i] : 0u;
        const unsigned d = live ? (k >> shift) & 255u : 256u;  // 256: no digit
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const unsigned rank = __popc(peers & ((1u << lane) - 1u));
        if (live && rank == 0) s_wc[warp][d] = __popc(peers);
        __syncthreads();
        // thread t: digit t's per-warp exclusive prefix, then the running count
        {
            unsigned acc = s_run[tid];
            for (int w = 0; w < 8; ++w) {
                const unsigned c = s_wc[w][tid];
                s_wc[w][tid] = acc;
                acc += c;
            }
            s_run[tid] = acc;
        }
        __syncthreads();
        if (live) {
            const unsigned pos = s_wc[warp][d] + rank;
            kout[pos] = k;
            vout[pos] = vin[i];
        }
        __syncthreads();
    }
}

// Stable ascending sort of (keys, vals) by the low `bits` bits of the keys
// (multiple of 8). Ping-pongs between the (a) and (b) buffers; the result is
// left in (a). `hist` holds 256 * tiles unsigned.
inline void radix_sort_pairs(uint32_t* ka, int* va, uint32_t* kb, int* vb, int n, int bits, unsigned* hist,
                             cudaStream_t s) {
    if (n <= 1) return;
    const int tiles = cdiv(n, kPrimTile);
    for (int shift = 0; shift < bits; shift += 8) {
        LPB_LAUNCH(k_radix_hist, tiles, 256, 0, s, ka, n, shift, hist, tiles);
        LPB_LAUNCH(k_scan_exclusive, 1, 1024, 0, s, hist, 256 * tiles, static_cast<int*>(nullptr));
        LPB_LAUNCH(k_radix_scatter, tiles, 256, 0, s, ka, va, n, shift, hist, tiles, kb, vb);
        std::swap(ka, kb);
        std::swap(va, vb);
    }
    if ((bits / 8) & 1) {  // odd pass count: the result sits in (b)
        LPB_CUDA(cudaMemcpyAsync(kb, ka, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, s));
        LPB_CUDA(cudaMemcpyAsync(vb, va, sizeof(int) * n, cudaMemcpyDeviceToDevice, s));
    }
}

}  // namespace lpb
