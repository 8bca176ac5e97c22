"""Device-built synthetic index (config D fixture, prag_gpu_index_synthetic):
GPU search == exact host restatement (tests/_synth_ref.py) on sampled
queries. The 1B-entry run is gated by PRAG_CONFIG_D=1 (72 GB of HBM, minutes)."""
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import _synth_ref as R  # noqa: E402

pytestmark = pytest.mark.gpu


def _model(nlist, d, m, seed):
    rng = np.random.default_rng(seed)
    cents = rng.standard_normal((nlist, d)).astype(np.float32)
    words = (rng.standard_normal((m, 256, d // m)) * 0.3).astype(np.float32)
    return cents, words


def _check(ix, cents, words, seed, queries, nprobe, k):
    import paper_2403_05676_b200 as pg
    sizes = ix.list_sizes()
    r = ix.search_batch(queries, k, nprobe)
    for i, q in enumerate(queries):
        ids, dist, sc = R.search(q, cents, words, sizes, seed, nprobe, k)
        c = int(r.count[i])
        assert c == len(ids) and int(r.scanned[i]) == sc
        assert (r.ids[i, :c] == ids).all(), (i, r.ids[i, :c], ids)
        assert (r.dist[i, :c].view(np.uint32) == dist.view(np.uint32)).all()


@pytest.mark.parametrize("m", [32, 64])
def test_synthetic_index_matches_host_restatement(m):
    import paper_2403_05676_b200 as pg
    cents, words = _model(256, 384, m, 5)
    seed = 99 + m
    ix = pg.GpuIndex.synthetic(cents, words, 300_000, seed=seed, sigma=1.0)
    assert ix.ntotal == 300_000 and int(ix.list_sizes().sum()) == 300_000
    rng = np.random.default_rng(1)
    q = (cents[rng.integers(0, 256, 6)] + rng.standard_normal((6, 384)).astype(np.float32) * 0.5).astype(np.float32)
    for nprobe, k in [(1, 10), (16, 10), (5, 32)]:
        _check(ix, cents, words, seed, q, nprobe, k)
    # k > 32 takes the generic path, which gathers from the lane-skewed tiles
    # (the only code copy in HBM)
    _check(ix, cents, words, seed, q, 4, 33)
    ix.set_scan_path(1)
    _check(ix, cents, words, seed, q, 16, 10)
    ix.set_scan_path(0)


@pytest.mark.skipif(os.environ.get("PRAG_CONFIG_D") != "1", reason="set PRAG_CONFIG_D=1 (1B entries, 72 GB HBM)")
def test_config_d_1b_sampled_parity():
    import paper_2403_05676_b200 as pg
    cents, words = _model(16384, 384, 64, 11)
    seed = 2024
    ix = pg.GpuIndex.synthetic(cents, words, 1_000_000_000, seed=seed, sigma=1.0)
    rng = np.random.default_rng(2)
    q = (cents[rng.integers(0, 16384, 2)] + rng.standard_normal((2, 384)).astype(np.float32) * 0.5).astype(np.float32)
    sizes = ix.list_sizes()
    print(f"\nconfig D: ntotal={ix.ntotal} nlist={ix.nlist} m={ix.nsq} device_bytes={ix.desc.device_bytes} "
          f"list p50={int(np.median(sizes))} max={int(sizes.max())}")
    for nprobe, k in [(16, 10), (64, 32)]:
        _check(ix, cents, words, seed, q, nprobe, k)
        r = ix.search_batch(q, k, nprobe)
        for i in range(q.shape[0]):
            print(f"  nprobe={nprobe} k={k} q{i}: scanned_vectors={int(r.scanned[i])} "
                  f"ids[:5]={r.ids[i, :5].tolist()} == host restatement (ids, distance bits, scanned)")


@pytest.mark.parametrize("m", [32, 64])
def test_synthetic_store_roundtrip_through_oracle(tmp_path, m):
    """prag_gpu_index_store rebuilds the plain codes from the lane-skewed
    tiles (the only copy in HBM; m = 64 tail bytes are stored + 1): the
    written PRAGIX01 searched by the CPU oracle equals the GPU search and the
    restatement."""
    import _oracle as O
    import paper_2403_05676_b200 as pg
    cents, words = _model(128, 384, m, 8)
    seed = 700 + m
    ix = pg.GpuIndex.synthetic(cents, words, 60_000, seed=seed, sigma=1.0)
    p = str(tmp_path / f"synth{m}.pragix")
    ix.store(p)
    oi = O.OracleIndex(p)
    rng = np.random.default_rng(4)
    q = (cents[rng.integers(0, 128, 5)] + rng.standard_normal((5, 384)).astype(np.float32) * 0.5).astype(np.float32)
    for nprobe, k in [(1, 10), (8, 40), (128, 5)]:
        r = ix.search_batch(q, k, nprobe)
        o_ids, o_dist, o_cnt, o_sc = oi.search(q, nprobe, k)
        assert (r.count == o_cnt).all() and (r.scanned == o_sc).all()
        for i in range(q.shape[0]):
            c = int(o_cnt[i])
            assert (r.ids[i, :c] == o_ids[i, :c]).all()
            assert (r.dist[i, :c].view(np.uint32) == o_dist[i, :c].view(np.uint32)).all()
    _check(ix, cents, words, seed, q, 8, 40)
