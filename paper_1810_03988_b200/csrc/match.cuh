// match.cuh — device LSH matcher (matchlsh.hpp:173-193), batched over camera pairs.
#pragma once
#include "common.cuh"

namespace lpb {

struct MatchArgs {
    int npairs;
    int qslot0, tslot0;         // pair p queries slot qslot0+p against train slot tslot0+p
    int nslots;                 // descriptor slots that need LSH keys
    const uint64_t* desc;       // nslots * cap * 2W
    const lp_keypoint* kps;     // nslots * cap
    const int* counts;          // nslots
    int cap, n_d;
    const int* bitpos;          // tables * bits
    int tables, bits;
    int full_card;              // probe set: all masks with popcount <= full_card ...
    const uint64_t* partial;    // ... plus these
    int npartial;
    int max_distance;
    float ratio;
    uint64_t* keys;             // nslots * cap * tables (scratch)
    int4* qres;                 // npairs * cap (scratch)
    lp_match* matches;          // npairs * cap
    lp_corr* corr;              // npairs * cap
    int* match_counts;          // npairs
    int* pair_status;           // npairs
    int keys_ready;             // the extractor already wrote `keys` (k_describe6)
};

void match_launch(const MatchArgs& a, cudaStream_t s);

// query (matchlsh.hpp:132-159) for nq query descriptors (slot qslot0) against
// the index of slot tslot0: every train descriptor reached by a probed bucket
// of some table, within max_distance, sorted by (distance, id). Output:
// offsets[q] .. offsets[q + 1] index `out` (query_id = query_id0 + q).
// Returns the total hit count (host sync); out holds min(total, cap) hits.
long long lsh_query_launch(const MatchArgs& a, int nq, int query_id0, long long* offsets, lp_match* out,
                           long long cap, cudaStream_t s);

}  // namespace lpb
