"""Config A (BASELINE.json configs[0], the reference's own CPU-runnable case)
end to end on one B200, exactly as SURVEY.md 8(d) defines it:
  data    x[i][j] = SplitMix64(1).next_gaussian(), 1M x 384 (test_annindex.cpp:12-19)
  index   prag::train_index, nlist 1024, nsq 32, seed 7, sample cap 32768 --
          built here by prag_gpu_train_index (bit-exact with the reference's,
          tests/test_gpu_train.py), list percentiles printed beside the
          reference's (p50 7, p90 4,195, max 8,294, avg 977,
          77.7k scanned per query at nprobe 16)
  queries 64 rows via SplitMix64(13).next_below(N) + 0.05 N(0,1) (annindex_main.cpp:66-74)
  search  nq 64, nprobe 16, k 10: GPU vs the C oracle (bit-exact check), GPU
          device time and host->host time, and the reference prag::search
          (oracle/_ref/ref_tool bench) on the same PRAGIX01 file.
  python tools/config_a.py [--out gpurun_out/config_a.json]
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    import _oracle as O
    import paper_2403_05676_b200 as pg

    t0 = time.time()
    v = O.random_vectors(a.n, 384, 1)
    gen_s = time.time() - t0
    q = O.noisy_queries(v, 64, 13, 0.05)
    xd = torch.from_numpy(v).cuda()
    pg.train_index(xd[:20000], pg.TrainParams(nlist=16, n_subquantizers=32, kmeans_iterations=1))  # warm-up
    torch.cuda.synchronize()
    t0 = time.time()
    t = pg.train_index(xd, pg.TrainParams(nlist=1024, n_subquantizers=32))
    train_s = time.time() - t0
    del xd
    sizes = np.diff(t.list_off.astype(np.int64))
    res = {"workload": "config A: 1M x 384 SplitMix64(1) gaussians, reference train_index(nlist 1024, nsq 32, seed 7) "
                       "built on the GPU, 64 queries, nprobe 16, k 10",
           "gen_vectors_s_host": round(gen_s, 1), "gpu_train_s": round(train_s, 3),
           "reference_train_s_survey": 1006,
           "lists": {"p50": int(np.median(sizes)), "p90": int(np.percentile(sizes, 90)), "max": int(sizes.max()),
                     "avg": round(float(sizes.mean()), 1),
                     "survey_reference": {"p50": 7, "p90": 4195, "max": 8294, "avg": 977}}}
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "a.pragix")
        t.write_pragix(path)
        res["pragix_bytes"] = os.path.getsize(path)
        ix = pg.GpuIndex.load(path)
        # parity against the oracle (and the reference search when present)
        r = ix.search_batch(q, 10, 16)
        oi, od, oc, osc = O.OracleIndex(path).search(q, 16, 10)
        res["bit_exact_vs_oracle"] = bool((r.ids == oi).all() and (r.dist.view(np.uint32) == od.view(np.uint32)).all()
                                          and (r.count == oc).all() and (r.scanned == osc).all())
        res["scanned_per_query_avg"] = float(np.mean(r.scanned))
        # device time (code array 32 MB: L2-resident, the reference's own reuse pattern)
        s = torch.cuda.Stream()
        qd = torch.from_numpy(q).cuda()
        for _ in range(5):
            ix.search_batch(qd, 10, 16, stream=s)
        torch.cuda.synchronize()
        dev = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            ix.search_batch(qd, 10, 16, stream=s)
            e1.record(s)
            e1.synchronize()
            dev.append(e0.elapsed_time(e1))
        host = []
        for _ in range(a.reps):
            t1 = time.perf_counter()
            ix.search_batch(q, 10, 16)
            host.append((time.perf_counter() - t1) * 1e3)
        res["gpu"] = {"device_p50_ms": round(statistics.median(dev), 4),
                      "device_qps": round(64 / (statistics.median(dev) / 1e3), 1),
                      "host_to_host_p50_ms": round(statistics.median(host), 4),
                      "host_to_host_qps": round(64 / (statistics.median(host) / 1e3), 1)}
        ref = os.path.join(REPO, "oracle", "_ref", "ref_tool")
        if os.path.exists(ref):
            qp = os.path.join(tmp, "q.f32")
            q.tofile(qp)
            threads = os.cpu_count() or 1
            out = subprocess.run([ref, "bench", path, qp, "64", "16", "10", str(threads), "3", "1", "60"],
                                 capture_output=True, text=True, timeout=900).stdout
            try:
                res["reference_cpu"] = {**json.loads(out.strip().splitlines()[-1]), "threads": threads}
            except Exception:
                res["reference_cpu"] = {"raw": out[-400:]}
    print(json.dumps(res, indent=1))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
