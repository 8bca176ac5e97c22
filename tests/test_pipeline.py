"""Config-E harness: the perf-model host logic (CPU) and the GPU pipelined
loop (retrieval on a side stream overlapped with the synthetic decode)."""
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from paper_2403_05676_b200 import pipeline as PL  # noqa: E402


def _model(pts):
    return PL.InferencePerfModel([PL.InferenceBucket(p, 8, s) for p, s in pts])


def test_predict_chunk_budget_kats():
    """perfmodel.hpp:162-183: interpolation, clamping below, extrapolation."""
    m = _model([(100, 1.0), (200, 2.0), (400, 3.0)])
    assert PL.predict_chunk_budget(m, 150) == (1.5, False)
    assert PL.predict_chunk_budget(m, 50) == (1.0, True)
    assert PL.predict_chunk_budget(m, 100) == (1.0, False)
    assert PL.predict_chunk_budget(m, 300) == (2.5, False)
    assert PL.predict_chunk_budget(m, 400) == (3.0, False)
    s, ex = PL.predict_chunk_budget(m, 600)
    assert ex and abs(s - 4.0) < 1e-12
    assert PL.predict_chunk_budget(_model([(100, 2.0)]), 100) == (2.0, False)
    with pytest.raises(ValueError):
        PL.predict_chunk_budget(_model([]), 1)


def test_calibrate_inference_median_and_warning():
    calls = []

    def gen(p):
        calls.append(p)
        return {64: 1.0, 128: 0.5}[p]
    m = PL.calibrate_inference(gen, [128, 64, 64], 16, repeats=3, warmups=2)
    assert [b.position for b in m.buckets] == [64, 128]
    assert len(calls) == 10 and m.monotonicity_warning


@pytest.mark.gpu
def test_piperag_loop_matches_blocking_and_overlaps():
    import torch
    import paper_2403_05676_b200 as pg
    import _oracle as O
    from conftest import load_golden
    path, z, _ = load_golden("d384_m32")
    ix = pg.GpuIndex.load(path, 0)
    q = torch.from_numpy(z["queries"]).cuda()
    dec = PL.SyntheticDecoder(params=64_000_000, max_positions=512)
    eng = PL.PipelineEngine(dec, ix, q, k=2)
    tr_b = eng.run("retro", 256, 32, nprobe=8)
    tr_p = eng.run("piperag", 256, 32, nprobe=8)
    assert tr_b.retrieval_count == tr_p.retrieval_count == 8
    # same queries, same nprobe -> identical retrieval results, and the oracle's
    oi = O.OracleIndex(path)
    for j, (rb, rp) in enumerate(zip(tr_b.results, tr_p.results)):
        assert torch.equal(rb.ids, rp.ids) and torch.equal(rb.dist, rp.dist)
        qi = j % z["queries"].shape[0]
        oids, _, ocnt, _ = oi.search(z["queries"][qi:qi + 1], 8, 2)
        assert (rb.ids.cpu().numpy().view(np.uint64)[0, :ocnt[0]] == oids[0, :ocnt[0]]).all()
    # pipelining hides retrieval behind decode: never slower than blocking
    assert tr_p.total_latency_s <= tr_b.total_latency_s * 1.05
    assert tr_p.stall_time_s <= tr_p.total_latency_s
    kinds = {e.kind for e in tr_p.events}
    assert {"ret_start", "ret_end", "gen_chunk_start", "gen_chunk_end"} <= kinds
