"""query (matchlsh.hpp:132-159): every probed candidate within max_distance,
sorted by (distance, id), for a batch of queries against build_index(train).
The device entry (lp_lsh_query: one warp per query, the pairwise probe
predicate, a radix sort of (query, distance, id) keys) against the
reference's own LshIndex + query and the C restatement."""
import numpy as np
import pytest


def descriptors(n, seed, n_d=256):
    rng = np.random.default_rng(seed)
    W = n_d // 64
    gt = rng.integers(0, 2**63, size=(n, W), dtype=np.uint64)
    lt = rng.integers(0, 2**63, size=(n, W), dtype=np.uint64) & ~gt
    return np.concatenate([gt, lt], axis=1)


def noisy(d, seed, flips=6):
    rng = np.random.default_rng(seed)
    out = d.copy()
    W = d.shape[1] // 2
    for i in range(len(out)):
        for b in rng.integers(0, 64 * W, size=flips):
            out[i, b // 64] ^= np.uint64(1) << np.uint64(b % 64)
    out[:, W:] &= ~out[:, :W]
    return out


CONFIGS = [(4, 16, 16, 64), (6, 12, 40, 80), (1, 20, 1, 512), (8, 10, 3, 30)]


@pytest.mark.parametrize("tables,bits,t_probes,maxd", CONFIGS)
def test_query_orc_matches_reference(orc, ref, tables, bits, t_probes, maxd):
    train = descriptors(400, 3)
    q = np.concatenate([noisy(train[::7], 4), descriptors(20, 5)])
    cfg = orc.default_params().matching
    cfg.tables, cfg.bits, cfg.t_probes, cfg.max_distance, cfg.seed = tables, bits, t_probes, maxd, 42
    a = orc.lsh_query(train, q, 256, cfg, 7)
    b = ref.lsh_query(train, q, 256, cfg, 7)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.gpu
@pytest.mark.parametrize("tables,bits,t_probes,maxd", CONFIGS)
def test_query_device_matches_reference(lp, ref, tables, bits, t_probes, maxd):
    train = descriptors(3000, 13)
    q = np.concatenate([noisy(train[::5], 14), noisy(train[::11], 15, 20), descriptors(200, 16)])
    cfg = ref.default_params().matching
    cfg.tables, cfg.bits, cfg.t_probes, cfg.max_distance, cfg.seed = tables, bits, t_probes, maxd, 42
    a = lp.lsh_query(train, q, 256, cfg, 0)
    b = ref.lsh_query(train, q, 256, cfg, 0)
    assert a[1].shape[0] > 0
    assert np.array_equal(a[0], b[0])
    assert np.array_equal(a[1], b[1])


@pytest.mark.gpu
def test_query_device_edge_cases(lp, ref):
    cfg = ref.default_params().matching
    train = descriptors(50, 21)
    # an empty index: no hits, offsets all zero
    off, hits = lp.lsh_query(train[:0], train[:3], 256, cfg)
    assert hits.shape[0] == 0 and not off.any()
    # n_d = 512 and a query set larger than the train set
    t512 = descriptors(64, 22, 512)
    q512 = noisy(np.concatenate([t512, t512, t512]), 23)
    a = lp.lsh_query(t512, q512, 512, cfg, 100)
    b = ref.lsh_query(t512, q512, 512, cfg, 100)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
