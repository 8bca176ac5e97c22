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
    """Fixed query rows (no token sequence): both modes retrieve the same
    queries, so their results are identical and equal to the oracle's."""
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
    oi = O.OracleIndex(path)
    for j, (rb, rp) in enumerate(zip(tr_b.results, tr_p.results)):
        assert torch.equal(rb.ids, rp.ids) and torch.equal(rb.dist, rp.dist)
        qi = j % z["queries"].shape[0]
        oids, _, ocnt, _ = oi.search(z["queries"][qi:qi + 1], 8, 2)
        assert (rb.ids.cpu().numpy().view(np.uint64)[0, :ocnt[0]] == oids[0, :ocnt[0]]).all()
    assert tr_p.stall_time_s <= tr_p.total_latency_s
    kinds = {e.kind for e in tr_p.events}
    assert {"ret_start", "ret_end", "gen_chunk_start", "gen_chunk_end"} <= kinds


def test_make_query_window_semantics():
    """pipeline.hpp:122-144: the window of m tokens ending s before chunk j;
    chunk 1 is never stale; positions before 0 are the pad token 0."""
    import torch
    eng = PL.PipelineEngine.__new__(PL.PipelineEngine)
    eng.tokens = torch.arange(1, 201, dtype=torch.int32)
    w = eng.query_window(1, 8, 4, 4)          # prompt chunk C_1 = positions [0, 8)
    assert w.tolist() == [[1, 2, 3, 4, 5, 6, 7, 8]]
    w = eng.query_window(3, 8, 4, 0)          # retro: ends just before chunk 3 (starts at 16)
    assert w.tolist() == [list(range(9, 17))]
    w = eng.query_window(3, 8, 4, 4)          # piperag: one interval stale
    assert w.tolist() == [list(range(5, 13))]
    w = eng.query_window(2, 8, 4, 10)         # begins 6 before position 0: padded
    assert w.tolist() == [[0, 0, 0, 0, 0, 0, 1, 2]]
    try:
        eng.query_window(60, 8, 4, 0)
    except ValueError:
        pass
    else:
        raise AssertionError("window past the generated tokens must fail")


@pytest.mark.gpu
def test_piperag_query_windows_embedded_on_gpu_and_overlap_wins():
    """The loop as the reference runs it: each retrieval embeds its query
    window (stale by one interval in piperag, pipeline.hpp:70-76) on the GPU
    and searches it; every result equals the oracle on that embedded query.
    PipeRAG's overlap (side stream, optionally with the decode pinned to
    S - R SMs) must not be slower than RETRO's blocking retrieval."""
    import torch
    import paper_2403_05676_b200 as pg
    import _oracle as O
    from conftest import load_golden
    path, z, _ = load_golden("d384_m32")
    ix = pg.GpuIndex.load(path, 0)
    dec = PL.SyntheticDecoder(params=128_000_000, max_positions=1024)
    gen = torch.Generator().manual_seed(3)
    tokens = torch.randint(1, 257, (64 + 512,), generator=gen, dtype=torch.int32).cuda()
    emb = pg.GpuChunkEmbedder(384, seed=11, vocab=257)
    oi = O.OracleIndex(path)
    totals = {}
    for mode, rs in (("retro", None), ("piperag", None), ("piperag", 8)):
        eng = PL.PipelineEngine(dec, ix, None, k=2, embedder=emb, tokens=tokens, retrieval_sms=rs)
        eng.run(mode, 512, 32, nprobe=16)  # warm
        best = min((eng.run(mode, 512, 32, nprobe=16) for _ in range(3)), key=lambda t: t.total_latency_s)
        totals[(mode, rs)] = best.total_latency_s
        assert best.retrieval_count == 16
        for j, (r, qv) in enumerate(zip(best.results, best.queries), start=1):
            # the window this retrieval used, embedded by the reference recipe
            want_q = emb.embed(eng.query_window(j, 64, 32, 32 if mode == "piperag" else 0).cpu().numpy())
            assert (qv.cpu().numpy().view(np.uint32) == want_q.view(np.uint32)).all()
            oids, odist, ocnt, _ = oi.search(want_q, 16, 2)
            c = int(ocnt[0])
            assert (r.ids.cpu().numpy().view(np.uint64)[0, :c] == oids[0, :c]).all()
            assert (r.dist.cpu().numpy()[0, :c].view(np.uint32) == odist[0, :c].view(np.uint32)).all()
    best_piperag = min(totals[("piperag", None)], totals[("piperag", 8)])
    assert best_piperag <= totals[("retro", None)] * 1.002, totals
