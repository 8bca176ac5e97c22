"""Captured searches (prag_gpu_plan_*): a CUDA-graph replay over fixed
buffers returns exactly what prag_gpu_search returns, and new queries written
into the captured buffer are searched by the next launch."""
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
pytestmark = pytest.mark.gpu


def test_plan_replay_equals_search(tmp_path):
    import torch
    import paper_2403_05676_b200 as pg
    from paper_2403_05676_b200 import fixtures as F
    os.environ.setdefault("PRAG_FIXTURE_DIR", str(tmp_path))
    p, q, _ = F.ensure_fixture(300_000, 384, 256, 32, seed=21, nq=64, log=lambda *a: None)
    ix = pg.GpuIndex.load(p, 0)
    s = torch.cuda.Stream()
    for nq, nprobe, k, path in [(64, 16, 10, 0), (1, 8, 2, 0), (16, 64, 32, 0), (8, 4, 50, 1)]:
        ix.set_scan_path(path)
        qd = torch.from_numpy(q[:nq].copy()).cuda()
        out = pg.BatchResult(torch.empty((nq, k), dtype=torch.int64, device="cuda"),
                             torch.empty((nq, k), dtype=torch.float32, device="cuda"),
                             torch.empty((nq,), dtype=torch.int32, device="cuda"),
                             torch.empty((nq,), dtype=torch.int64, device="cuda"))
        plan = ix.plan(qd, k, nprobe, out, stream=s)
        for rot in (0, 5, 17):  # new queries in the captured buffer
            qd.copy_(torch.from_numpy(np.roll(q, rot, axis=0)[:nq].copy()))
            plan.launch(stream=s)
            s.synchronize()
            ref = ix.search_batch(np.roll(q, rot, axis=0)[:nq], k, nprobe)
            got_ids = out.ids.cpu().numpy().view(np.uint64)
            got_dist = out.dist.cpu().numpy()
            got_cnt = out.count.cpu().numpy()
            assert (got_cnt == ref.count).all()
            for i in range(nq):
                c = int(ref.count[i])
                assert (got_ids[i, :c] == ref.ids[i, :c]).all(), (nq, nprobe, k, rot, i)
                assert (got_dist[i, :c].view(np.uint32) == ref.dist[i, :c].view(np.uint32)).all()
        plan.close()
    ix.set_scan_path(0)


def test_unaligned_device_queries(tmp_path):
    """Device query buffers need only 4-byte alignment (a row view of a
    larger tensor at any float offset): same results as host queries."""
    import torch
    import paper_2403_05676_b200 as pg
    from paper_2403_05676_b200 import fixtures as F
    os.environ.setdefault("PRAG_FIXTURE_DIR", str(tmp_path))
    p, q, _ = F.ensure_fixture(300_000, 384, 256, 32, seed=21, nq=64, log=lambda *a: None)
    ix = pg.GpuIndex.load(p, 0)
    nq, k, nprobe = 24, 10, 16
    ref = ix.search_batch(q[:nq], k, nprobe)
    for off in (1, 2, 3):
        buf = torch.zeros(nq * q.shape[1] + off, dtype=torch.float32, device="cuda")
        qd = buf[off:].view(nq, q.shape[1])
        qd.copy_(torch.from_numpy(q[:nq].copy()))
        assert qd.data_ptr() % 16 != 0
        r = ix.search_batch(qd, k, nprobe)
        torch.cuda.synchronize()
        assert (r.count.cpu().numpy() == ref.count).all()
        assert (r.ids.cpu().numpy().view(np.uint64) == ref.ids).all(), off
        assert (r.dist.cpu().numpy().view(np.uint32) == ref.dist.view(np.uint32)).all(), off
