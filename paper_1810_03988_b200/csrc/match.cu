// match.cu — multi-probe LSH matching with Hamming ratio test (matchlsh.hpp).
//
// The reference builds L bucket tables over the train set and, per query,
// probes T buckets per table (matchlsh.hpp:132-159). On the device the same
// candidate set is produced by the equivalent pairwise predicate (SURVEY §8(a)
// H16, verified): train j is a candidate of query q iff for some table t,
// key_t(q) XOR key_t(j) is one of the probe masks. Candidates are deduplicated
// by construction, distances are __popc over the gt/lt planes
// (matchlsh.hpp:25-33), and each warp keeps the lexicographic top-2
// (distance, train_id) of one query, which is all the ratio test
// (matchlsh.hpp:183-186) needs. A per-pair CTA then orders accepted matches by
// (quality desc, query_id asc) = (distance asc, query_id asc) by rank
// placement and emits the Correspondence list for PROSAC (pipeline.hpp:480-488).
#include "match.cuh"
#include "prims.cuh"

#include <algorithm>
#include <vector>

namespace lpb {

// one warp per descriptor: lane b extracts bit b of a table's key (hash_key,
// matchlsh.hpp:70-80) and a ballot assembles the key; all tables' loads are
// issued before the ballots
__global__ void k_lsh_keys(MatchArgs a) {
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int slot = gw / a.cap, i = gw - slot * a.cap;
    if (slot >= a.nslots || i >= a.counts[slot]) return;  // warp-uniform
    const int W = (a.n_d + 63) / 64;
    const uint64_t* d = a.desc + (static_cast<size_t>(slot) * a.cap + i) * 2 * W;
    uint64_t* out = a.keys + (static_cast<size_t>(slot) * a.cap + i) * a.tables;
    for (int t0 = 0; t0 < a.tables; t0 += 4) {
        unsigned bits[4][2];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int t = t0 + u, b = 32 * h + lane;
                unsigned v = 0;
                if (t < a.tables && b < a.bits) {
                    const int p = __ldg(a.bitpos + t * a.bits + b);
                    const int q = p < a.n_d ? p : p - a.n_d;  // bit within its plane
                    v = static_cast<unsigned>((__ldg(d + (p < a.n_d ? 0 : W) + (q >> 6)) >> (q & 63)) & 1ull);
                }
                bits[u][h] = v;
            }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint64_t lo = __ballot_sync(0xffffffffu, bits[u][0]);
            const uint64_t hi = __ballot_sync(0xffffffffu, bits[u][1]);
            if (lane == 0 && t0 + u < a.tables) out[t0 + u] = lo | (hi << 32);
        }
    }
}

__device__ __forceinline__ bool in_probe_set(uint64_t x, const MatchArgs& a) {
    const int p = __popcll(x);
    if (p <= a.full_card) return true;
    if (p != a.full_card + 1) return false;
    for (int i = 0; i < a.npartial; ++i)
        if (a.partial[i] == x) return true;
    return false;
}

// lexicographic (distance, id) insert into a top-2
__device__ __forceinline__ void top2_insert(int d, int j, int& d0, int& j0, int& d1, int& j1) {
    if (d < d0 || (d == d0 && j < j0)) {
        d1 = d0;
        j1 = j0;
        d0 = d;
        j0 = j;
    } else if (d < d1 || (d == d1 && j < j1)) {
        d1 = d;
        j1 = j;
    }
}

constexpr int kMaxW = 8;  // n_d <= 512
constexpr int kFinalizeSmemMax = 64 << 10;  // k_match_finalize's key array (16K accepted matches)

// one warp per query (large problems: enough warps, and a small register
// footprint keeps 6 CTAs per SM resident)
__global__ void __launch_bounds__(256) k_match_query_warp(MatchArgs a, int /*split*/) {
    const int pair = blockIdx.y;
    const int qs = a.qslot0 + pair, ts = a.tslot0 + pair;
    const int nq = a.counts[qs], nt = a.counts[ts];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int W = (a.n_d + 63) / 64;
    const uint64_t* tkeys = a.keys + static_cast<size_t>(ts) * a.cap * a.tables;
    const uint64_t* tdesc = a.desc + static_cast<size_t>(ts) * a.cap * 2 * W;
    const int q_base = blockIdx.x * (blockDim.x >> 5) + warp;
    for (int qq = 0; qq < 1; ++qq) {
        const int q = q_base + qq;
        if (q >= nq) return;
        uint64_t qk[8];
        for (int t = 0; t < a.tables && t < 8; ++t)
            qk[t] = a.keys[(static_cast<size_t>(qs) * a.cap + q) * a.tables + t];
        uint64_t qd[2 * kMaxW];
        const uint64_t* qdp = a.desc + (static_cast<size_t>(qs) * a.cap + q) * 2 * W;
        for (int w = 0; w < 2 * W; ++w) qd[w] = qdp[w];
        const int BIG = 0x7fffffff;
        int d0 = BIG, j0 = BIG, d1 = BIG, j1 = BIG;
        for (int j = lane; j < nt; j += 32) {
            bool cand = false;
            for (int t = 0; t < a.tables; ++t) {
                const uint64_t tk = tkeys[static_cast<size_t>(j) * a.tables + t];
                const uint64_t qkt = t < 8 ? qk[t] : a.keys[(static_cast<size_t>(qs) * a.cap + q) * a.tables + t];
                if (in_probe_set(qkt ^ tk, a)) {
                    cand = true;
                    break;
                }
            }
            if (!cand) continue;
            const uint64_t* td = tdesc + static_cast<size_t>(j) * 2 * W;
            int d = 0;
            for (int w = 0; w < 2 * W; ++w) d += __popcll(qd[w] ^ td[w]);
            if (d <= a.max_distance) top2_insert(d, j, d0, j0, d1, j1);
        }
        // warp merge of the per-lane top-2 lists
        for (int off = 16; off > 0; off >>= 1) {
            int od0 = __shfl_xor_sync(0xffffffffu, d0, off), oj0 = __shfl_xor_sync(0xffffffffu, j0, off);
            int od1 = __shfl_xor_sync(0xffffffffu, d1, off), oj1 = __shfl_xor_sync(0xffffffffu, j1, off);
            top2_insert(od0, oj0, d0, j0, d1, j1);
            top2_insert(od1, oj1, d0, j0, d1, j1);
        }
        if (lane == 0) {
            int4 r;
            r.x = j0 == BIG ? -1 : j0;
            r.y = d0;
            r.z = j1 == BIG ? -1 : d1;  // second-best distance, or -1 when < 2 hits
            r.w = 0;
            a.qres[static_cast<size_t>(pair) * a.cap + q] = r;
        }
    }
}

// `split` warps per query (2, 4 or 8; 8 / split queries per CTA), each
// scanning every split-th block of 32 train descriptors: small problems put
// more warps in flight and fewer serial load round trips on each; their
// lexicographic top-2 lists merge in shared memory (the top-2 of
// (distance, id) does not depend on the visiting order)
__global__ void __launch_bounds__(256, 4) k_match_query_split(MatchArgs a, int split) {
    __shared__ int4 s_top[8];
    const int pair = blockIdx.y;
    const int qs = a.qslot0 + pair, ts = a.tslot0 + pair;
    const int nq = a.counts[qs], nt = a.counts[ts];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int part = warp % split;
    const int W = (a.n_d + 63) / 64;
    const uint64_t* tkeys = a.keys + static_cast<size_t>(ts) * a.cap * a.tables;
    const uint64_t* tdesc = a.desc + static_cast<size_t>(ts) * a.cap * 2 * W;
    const int q = blockIdx.x * (8 / split) + warp / split;
    const int BIG = 0x7fffffff;
    int d0 = BIG, j0 = BIG, d1 = BIG, j1 = BIG;
    if (q < nq) {
        // the query's keys stay in registers (a guarded full unroll: a runtime
        // trip count would put them on the stack); its descriptor is read
        // (L1) only for the few candidates
        uint64_t qk[8];
#pragma unroll
        for (int t = 0; t < 8; ++t)
            qk[t] = t < a.tables ? a.keys[(static_cast<size_t>(qs) * a.cap + q) * a.tables + t] : 0ull;
        const uint64_t* qdp = a.desc + (static_cast<size_t>(qs) * a.cap + q) * 2 * W;
        for (int j = 32 * part + lane; j < nt; j += 32 * split) {
            bool cand = false;
            if (a.tables <= 8) {
                uint64_t tk[8];  // all of train j's keys in flight, then the tests
#pragma unroll
                for (int t = 0; t < 8; ++t)
                    tk[t] = t < a.tables ? __ldg(tkeys + static_cast<size_t>(j) * a.tables + t) : 0ull;
#pragma unroll
                for (int t = 0; t < 8; ++t) cand = cand || (t < a.tables && in_probe_set(qk[t] ^ tk[t], a));
            } else {
                for (int t = 0; t < a.tables; ++t) {
                    const uint64_t tk = tkeys[static_cast<size_t>(j) * a.tables + t];
                    const uint64_t qkt = a.keys[(static_cast<size_t>(qs) * a.cap + q) * a.tables + t];
                    if (in_probe_set(qkt ^ tk, a)) {
                        cand = true;
                        break;
                    }
                }
            }
            if (!cand) continue;
            const uint64_t* td = tdesc + static_cast<size_t>(j) * 2 * W;
            int d = 0;
            for (int w = 0; w < 2 * W; ++w) d += __popcll(__ldg(qdp + w) ^ td[w]);
            if (d <= a.max_distance) top2_insert(d, j, d0, j0, d1, j1);
        }
        // warp merge of the per-lane top-2 lists
        for (int off = 16; off > 0; off >>= 1) {
            int od0 = __shfl_xor_sync(0xffffffffu, d0, off), oj0 = __shfl_xor_sync(0xffffffffu, j0, off);
            int od1 = __shfl_xor_sync(0xffffffffu, d1, off), oj1 = __shfl_xor_sync(0xffffffffu, j1, off);
            top2_insert(od0, oj0, d0, j0, d1, j1);
            top2_insert(od1, oj1, d0, j0, d1, j1);
        }
        if (lane == 0) s_top[warp] = make_int4(d0, j0, d1, j1);
    }
    __syncthreads();
    if (q < nq && part == 0 && lane == 0) {
        for (int k = 1; k < split; ++k) {
            const int4 o = s_top[warp + k];
            top2_insert(o.x, o.y, d0, j0, d1, j1);
            top2_insert(o.z, o.w, d0, j0, d1, j1);
        }
        int4 r;
        r.x = j0 == BIG ? -1 : j0;
        r.y = d0;
        r.z = j1 == BIG ? -1 : d1;  // second-best distance, or -1 when < 2 hits
        r.w = 0;
        a.qres[static_cast<size_t>(pair) * a.cap + q] = r;
    }
}

// per pair: ratio test, (distance, query) order, matches + correspondences
__global__ void __launch_bounds__(1024) k_match_finalize(MatchArgs a) {
    extern __shared__ uint32_t s_k[];
    __shared__ int s_n;
    const int pair = blockIdx.x;
    const int qs = a.qslot0 + pair, ts = a.tslot0 + pair;
    const int nq = a.counts[qs], nt = a.counts[ts];
    if (threadIdx.x == 0) {
        s_n = 0;
        if (nq == 0 || nt == 0) dev_fail(a.pair_status + pair, LP_EMPTY_INPUT);
    }
    __syncthreads();
    if (nq == 0 || nt == 0) {
        if (threadIdx.x == 0) a.match_counts[pair] = 0;
        return;
    }
    for (int q = threadIdx.x; q < nq; q += blockDim.x) {
        const int4 r = a.qres[static_cast<size_t>(pair) * a.cap + q];
        if (r.x < 0) continue;
        if (r.z >= 0 && !(static_cast<float>(r.y) < fmul(a.ratio, static_cast<float>(r.z)))) continue;
        const int slot = atomicAdd(&s_n, 1);
        s_k[slot] = (static_cast<uint32_t>(r.y) << 21) | static_cast<uint32_t>(q);
    }
    __syncthreads();
    const int n = s_n;
    // (distance, query) keys are unique: each accepted match goes straight to
    // its rank in ascending order (matchlsh.hpp:188-191), no sorting network
    const float denom = fmul(2.0f, static_cast<float>(a.n_d));
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t key = s_k[i];
        int r = 0;
        for (int j = 0; j < n; ++j) r += s_k[j] < key;
        const int q = static_cast<int>(key & 0x1FFFFFu);
        const int d = static_cast<int>(key >> 21);
        const int4 qr = a.qres[static_cast<size_t>(pair) * a.cap + q];
        lp_match m;
        m.query_id = q;
        m.train_id = qr.x;
        m.distance = d;
        m.quality = fsub(1.0f, __fdiv_rn(static_cast<float>(d), denom));
        a.matches[static_cast<size_t>(pair) * a.cap + r] = m;
        const lp_keypoint sk = a.kps[static_cast<size_t>(qs) * a.cap + q];
        const lp_keypoint tk = a.kps[static_cast<size_t>(ts) * a.cap + qr.x];
        lp_corr c;
        c.sx = static_cast<double>(sk.x);
        c.sy = static_cast<double>(sk.y);
        c.dx = static_cast<double>(tk.x);
        c.dy = static_cast<double>(tk.y);
        c.quality = m.quality;
        c.pad_ = 0;
        a.corr[static_cast<size_t>(pair) * a.cap + r] = c;
    }
    if (threadIdx.x == 0) a.match_counts[pair] = n;
}

// Large pairs (more accepted matches than k_match_finalize's shared-memory
// rank placement holds): every query writes its (distance, query) key, or
// ~0 if rejected, at its own index; a stable radix sort of the cap keys
// (prims.cuh) orders them, and the emitter writes rank i from sorted key i.
__global__ void k_match_keys(MatchArgs a, int pair, uint32_t* keys) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= a.cap) return;
    const int qs = a.qslot0 + pair, nq = a.counts[qs], nt = a.counts[a.tslot0 + pair];
    uint32_t k = ~0u;
    if (q < nq && nt > 0) {
        const int4 r = a.qres[static_cast<size_t>(pair) * a.cap + q];
        if (r.x >= 0 && !(r.z >= 0 && !(static_cast<float>(r.y) < fmul(a.ratio, static_cast<float>(r.z)))))
            k = (static_cast<uint32_t>(r.y) << 21) | static_cast<uint32_t>(q);
    }
    keys[q] = k;
}
__global__ void k_match_emit(MatchArgs a, int pair, const uint32_t* keys) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.cap) return;
    const int qs = a.qslot0 + pair, ts = a.tslot0 + pair;
    if (i == 0 && (a.counts[qs] == 0 || a.counts[ts] == 0)) {
        dev_fail(a.pair_status + pair, LP_EMPTY_INPUT);
        a.match_counts[pair] = 0;
    }
    const uint32_t key = keys[i];
    if (key == ~0u) return;
    if (i + 1 == a.cap || keys[i + 1] == ~0u) a.match_counts[pair] = i + 1;
    const int q = static_cast<int>(key & 0x1FFFFFu), d = static_cast<int>(key >> 21);
    const int4 qr = a.qres[static_cast<size_t>(pair) * a.cap + q];
    lp_match m;
    m.query_id = q;
    m.train_id = qr.x;
    m.distance = d;
    m.quality = fsub(1.0f, __fdiv_rn(static_cast<float>(d), fmul(2.0f, static_cast<float>(a.n_d))));
    a.matches[static_cast<size_t>(pair) * a.cap + i] = m;
    const lp_keypoint sk = a.kps[static_cast<size_t>(qs) * a.cap + q];
    const lp_keypoint tk = a.kps[static_cast<size_t>(ts) * a.cap + qr.x];
    lp_corr c;
    c.sx = static_cast<double>(sk.x);
    c.sy = static_cast<double>(sk.y);
    c.dx = static_cast<double>(tk.x);
    c.dy = static_cast<double>(tk.y);
    c.quality = m.quality;
    c.pad_ = 0;
    a.corr[static_cast<size_t>(pair) * a.cap + i] = c;
}
__global__ void k_zero_int(int* p) { *p = 0; }

// ---- query(): every candidate within max_distance, one warp per query.
// Pass 1 counts each query's hits, pass 2 writes (query, distance, id) as a
// 64-bit key (query << 43 | distance << 32 | id) into the query's segment;
// one stable radix sort of the keys orders every segment by (distance, id).
template <bool EMIT>
__global__ void __launch_bounds__(256) k_lsh_query(MatchArgs a, int nq, unsigned* count, const unsigned* offset,
                                                   uint32_t* key_lo, uint32_t* key_hi) {
    const int q = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (q >= nq) return;
    const int qs = a.qslot0, ts = a.tslot0;
    const int nt = a.counts[ts];
    const int W = (a.n_d + 63) / 64;
    const uint64_t* tkeys = a.keys + static_cast<size_t>(ts) * a.cap * a.tables;
    const uint64_t* qkeys = a.keys + (static_cast<size_t>(qs) * a.cap + q) * a.tables;
    const uint64_t* qd = a.desc + (static_cast<size_t>(qs) * a.cap + q) * 2 * W;
    const uint64_t* tdesc = a.desc + static_cast<size_t>(ts) * a.cap * 2 * W;
    unsigned pos = EMIT ? offset[q] : 0u, n = 0;
    for (int j0 = 0; j0 < nt; j0 += 32) {
        const int j = j0 + lane;
        bool hit = false;
        int d = 0;
        if (j < nt) {
            bool cand = false;
            for (int t = 0; t < a.tables && !cand; ++t)
                cand = in_probe_set(qkeys[t] ^ tkeys[static_cast<size_t>(j) * a.tables + t], a);
            if (cand) {
                const uint64_t* td = tdesc + static_cast<size_t>(j) * 2 * W;
                for (int w = 0; w < 2 * W; ++w) d += __popcll(qd[w] ^ td[w]);
                hit = d <= a.max_distance;
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (EMIT && hit) {
            const unsigned slot = pos + n + __popc(m & ((1u << lane) - 1u));
            key_lo[slot] = static_cast<uint32_t>(j);
            key_hi[slot] = (static_cast<uint32_t>(q) << 11) | static_cast<uint32_t>(d);
        }
        n += __popc(m);
    }
    if (!EMIT && lane == 0) count[q] = n;
}
__global__ void k_lsh_query_out(MatchArgs a, long long total, long long cap, int query_id0, const uint32_t* key_lo,
                                const uint32_t* key_hi, const int* order, lp_match* out) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= total || i >= cap) return;
    const int s = order[i];
    lp_match m;
    m.query_id = query_id0 + static_cast<int>(key_hi[s] >> 11);
    m.train_id = static_cast<int>(key_lo[s]);
    m.distance = static_cast<int>(key_hi[s] & 0x7FFu);
    m.quality = fsub(1.0f, __fdiv_rn(static_cast<float>(m.distance), fmul(2.0f, static_cast<float>(a.n_d))));
    out[i] = m;
}
__global__ void k_gather_u32(const uint32_t* src, const int* idx, long long n, uint32_t* dst) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[idx[i]];
}
__global__ void k_iota_q(int* p, long long n) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) p[i] = static_cast<int>(i);
}

long long lsh_query_launch(const MatchArgs& a, int nq, int query_id0, long long* offsets, lp_match* out,
                           long long cap, cudaStream_t s) {
    if (nq <= 0) return 0;
    if (a.n_d > 64 * kMaxW) throw Status(LP_BAD_PARAMS, "query: n_d too large");
    if (nq >= (1 << 21)) throw Status(LP_BAD_PARAMS, "query: too many queries in one call");
    if (!a.keys_ready)
        LPB_LAUNCH(k_lsh_keys, cdiv(static_cast<long long>(a.nslots) * a.cap * 32, 256), 256, 0, s, a);
    DBuf cnt(sizeof(unsigned) * (nq + 1), s), tot(sizeof(int), s);
    LPB_LAUNCH(k_lsh_query<false>, cdiv(nq, 8), 256, 0, s, a, nq, cnt.as<unsigned>(),
               static_cast<const unsigned*>(nullptr), static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr));
    LPB_LAUNCH(k_scan_exclusive, 1, 1024, 0, s, cnt.as<unsigned>(), nq + 1, tot.as<int>());
    std::vector<unsigned> off(nq + 1);
    LPB_CUDA(cudaMemcpyAsync(off.data(), cnt.p, sizeof(unsigned) * (nq + 1), cudaMemcpyDeviceToHost, s));
    LPB_CUDA(cudaStreamSynchronize(s));
    const long long total = off[nq];
    for (int q = 0; q <= nq; ++q) offsets[q] = off[q];
    if (total == 0) return 0;
    if (total >= (1LL << 31)) throw Status(LP_CAPACITY_OVERFLOW, "query: too many hits");
    const int n = static_cast<int>(total);
    DBuf lo(sizeof(uint32_t) * n, s), hi(sizeof(uint32_t) * n, s), ka(sizeof(uint32_t) * n, s),
        kb(sizeof(uint32_t) * n, s), ia(sizeof(int) * n, s), ib(sizeof(int) * n, s),
        hist(sizeof(unsigned) * 256 * cdiv(n, kPrimTile), s);
    LPB_LAUNCH(k_lsh_query<true>, cdiv(nq, 8), 256, 0, s, a, nq, static_cast<unsigned*>(nullptr), cnt.as<unsigned>(),
               lo.as<uint32_t>(), hi.as<uint32_t>());
    // (query, distance) major, train id minor: stable by id, then by the high word
    LPB_LAUNCH(k_iota_q, cdiv(n, 256), 256, 0, s, ia.as<int>(), static_cast<long long>(n));
    LPB_CUDA(cudaMemcpyAsync(ka.p, lo.p, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, s));
    radix_sort_pairs(ka.as<uint32_t>(), ia.as<int>(), kb.as<uint32_t>(), ib.as<int>(), n, 32, hist.as<unsigned>(), s);
    LPB_LAUNCH(k_gather_u32, cdiv(n, 256), 256, 0, s, hi.as<uint32_t>(), ia.as<int>(), static_cast<long long>(n),
               ka.as<uint32_t>());
    radix_sort_pairs(ka.as<uint32_t>(), ia.as<int>(), kb.as<uint32_t>(), ib.as<int>(), n, 32, hist.as<unsigned>(), s);
    LPB_LAUNCH(k_lsh_query_out, cdiv(std::min<long long>(n, cap), 256), 256, 0, s, a, total, cap, query_id0,
               lo.as<uint32_t>(), hi.as<uint32_t>(), ia.as<int>(), out);
    return total;
}

void match_launch(const MatchArgs& a, cudaStream_t s) {
    if (a.npairs <= 0) return;
    if (a.n_d > 64 * kMaxW) throw Status(LP_BAD_PARAMS, "match: n_d too large");
    if (a.cap >= (1 << 21)) throw Status(LP_BAD_PARAMS, "match: too many descriptors");
    if (a.bits > 64) throw Status(LP_BAD_PARAMS, "match: more than 64 key bits");
    if (!a.keys_ready)
        LPB_LAUNCH(k_lsh_keys, cdiv(static_cast<long long>(a.nslots) * a.cap * 32, 256), 256, 0, s, a);
    // about 32 warps per SM in total: split the scans of small problems,
    // keep one warp per query on large ones (setup per warp is the cost there)
    const long long queries = static_cast<long long>(a.npairs) * a.cap;
    int split = 1;
    while (split < 8 && queries * split * 2 <= 148LL * 32) split <<= 1;
    dim3 grid(cdiv(a.cap, 8 / split), a.npairs);
    // one profiler key (k_match_query/0) for either kernel
    auto* k_match_query = split > 1 ? &k_match_query_split : &k_match_query_warp;
    LPB_LAUNCH(k_match_query, grid, 256, 0, s, a, split);
    int p2 = 1;
    while (p2 < a.cap) p2 <<= 1;
    const int smem = p2 * 4;
    if (smem <= kFinalizeSmemMax) {  // O(n^2 / 1024) rank placement in shared memory
        ensure_dyn_smem(reinterpret_cast<const void*>(k_match_finalize), smem);
        LPB_LAUNCH(k_match_finalize, a.npairs, 1024, smem, s, a);
        return;
    }
    const int tiles = cdiv(a.cap, kPrimTile);
    DBuf ka(sizeof(uint32_t) * a.cap, s), kb(sizeof(uint32_t) * a.cap, s), va(sizeof(int) * a.cap, s),
        vb(sizeof(int) * a.cap, s), hist(sizeof(unsigned) * 256 * tiles, s);
    for (int p = 0; p < a.npairs; ++p) {
        LPB_LAUNCH(k_match_keys, cdiv(a.cap, 256), 256, 0, s, a, p, ka.as<uint32_t>());
        radix_sort_pairs(ka.as<uint32_t>(), va.as<int>(), kb.as<uint32_t>(), vb.as<int>(), a.cap, 32,
                         hist.as<unsigned>(), s);
        LPB_LAUNCH(k_zero_int, 1, 1, 0, s, a.match_counts + p);
        LPB_LAUNCH(k_match_emit, cdiv(a.cap, 256), 256, 0, s, a, p, ka.as<uint32_t>());
    }
}

}  // namespace lpb
