#!/usr/bin/env python
"""IVF-PQ search benchmark (BASELINE.json configs[1] at N=1).

Workload (one "step" = one batch search): synthetic 10M x 384 fp32 DB,
IVF nlist=4096, PQ m=32 x 8-bit (PRAGIX01 fixture built by
paper_2403_05676_b200/fixtures.py), nq=64 queries (DB row + 0.05 N(0,1)),
nprobe=16, k=10. The nprobe sweep 1..128 x nq {1,16,64} is reported beside
the headline in "sweep", with the GPU-recalibrated performance model.

  value : queries/s, queries and outputs resident in HBM, CUDA events on the
          search stream around each step, L2 flushed (256 MiB memset) between
          steps, ALL ranks' queries / max-over-ranks time.
  e2e   : same metric through the C ABI with pinned HOST buffers (H2D of the
          queries and D2H of ids/dist/count/scanned inside the timed region).
  --impl reference : the unmodified reference prag::search (oracle/_ref,
          compiled from /root/reference) on this box's host cores, same
          index file and queries.

N>1 (torchrun): the 10M index fits one GPU, so each rank holds a replica
and searches its own 64-query batches (queries are independent units: no
data-path collective, "scaling": "weak"; value = all ranks' queries over the
max-over-ranks time). PRAG_BENCH_MODE=shard-lists instead shards the
inverted lists by LPT over ranks (load_shard), NCCL all_gather of per-shard
top-k and the exact merge kernel on rank 0 -- same DB and queries for every
N ("scaling": "strong"), the layout for indexes beyond one GPU (configs C/D).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CFG = dict(n=10_000_000, d=384, nlist=4096, nsq=32, seed=1, nq=64, nprobe=16, k=10)
SWEEP_NPROBE = [1, 2, 4, 8, 16, 32, 64, 128]
SWEEP_NQ = [1, 16, 64]
METRIC = "ivfpq_search_queries_per_s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                clk, cmax, util = float(parts[0]), float(parts[1]), float(parts[2])
            except ValueError:
                continue
            mx = max(mx, cmax)
            if util > 0:
                sm.append(clk)
                for nm, v in zip(names, parts[3:7]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples_under_load": len(sm),
                "window": "nvidia-smi -lms 20 over a 1 s pre-roll of back-to-back steps + the timed region"}


def reference_arm(args, path, queries, cfg):
    """Unmodified reference prag::search on all host cores (oracle/_ref/ref_tool)."""
    tool = os.path.join(REPO, "oracle", "_ref", "ref_tool")
    if not os.path.exists(tool):
        return {"impl": "reference", "unavailable": "oracle/_ref/ref_tool not built (needs /root/reference at build)"}
    qp = path + f".bench_q{cfg['nq']}.f32"
    queries[:cfg["nq"]].astype(np.float32).tofile(qp)
    threads = os.cpu_count() or 1
    out = subprocess.run([tool, "bench", path, qp, str(cfg["nq"]), str(cfg["nprobe"]), str(cfg["k"]), str(threads),
                          str(args.steps), str(args.warmup), str(args.ref_seconds)], capture_output=True, text=True,
                         check=True)
    r = json.loads(out.stdout.strip().splitlines()[-1])
    # the reference's own protocol is one thread running queries in sequence
    # (perfmodel_main.cpp:57-63): one bounded batch on a single core beside it
    one = subprocess.run([tool, "bench", path, qp, str(cfg["nq"]), str(cfg["nprobe"]), str(cfg["k"]), "1", "1", "0",
                          "1"], capture_output=True, text=True)
    if one.returncode == 0:
        try:
            r["single_thread_qps"] = json.loads(one.stdout.strip().splitlines()[-1])["qps"]
        except Exception:
            pass
    return r, threads


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--small", action="store_true", help="1M-vector variant for quick checks")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=20.0)
    args = ap.parse_args()
    assert args.warmup >= 3, "W >= 3 warm-up steps"

    cfg = dict(CFG)
    if args.small:
        cfg.update(n=1_000_000, nlist=1024)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    import torch
    import torch.distributed as dist
    from paper_2403_05676_b200 import fixtures as F

    # PRAG_BENCH_BACKEND=gloo runs the N>1 path functionally on fewer GPUs
    # than ranks (ranks share devices round-robin); numbers from such a run
    # are not bench values
    backend = os.environ.get("PRAG_BENCH_BACKEND", "nccl" if args.impl == "ours" else "gloo")
    if torch.cuda.is_available() and backend == "gloo":
        local = local % torch.cuda.device_count()
    if world > 1:
        dist.init_process_group(backend, device_id=torch.device("cuda", local) if backend == "nccl" else None)
    torch.cuda.set_device(local)

    # fixture: rank 0 builds (or reuses the cache), the others wait
    if rank == 0:
        path, queries, meta = F.ensure_fixture(cfg["n"], cfg["d"], cfg["nlist"], cfg["nsq"], cfg["seed"], nq=64,
                                               log=log)
    if world > 1:
        dist.barrier()
    if rank != 0:
        path, queries, meta = F.ensure_fixture(cfg["n"], cfg["d"], cfg["nlist"], cfg["nsq"], cfg["seed"], nq=64,
                                               log=log)
    # N > 1: the index fits one GPU (config B), so by default every rank holds
    # a replica and serves its own query batches -- queries are independent
    # units, no data-path collective, weak scaling. PRAG_BENCH_MODE=shard-lists
    # instead splits the inverted lists across ranks (the mode
    # for indexes larger than one GPU) with one NCCL exchange per batch.
    mode = os.environ.get("PRAG_BENCH_MODE", "replicas") if world > 1 else "single"
    if mode not in ("single", "replicas", "shard-lists"):
        raise SystemExit(f"PRAG_BENCH_MODE must be replicas or shard-lists, not {mode}")
    workload = (f"ivfpq search: {cfg['n'] // 1_000_000}M x {cfg['d']} fp32 DB, nlist={cfg['nlist']}, "
                f"PQ m={cfg['nsq']}x8b, nq={cfg['nq']}, nprobe={cfg['nprobe']}, k={cfg['k']}")
    config = {"workload": workload, "n": cfg["n"], "d": cfg["d"], "nlist": cfg["nlist"], "m": cfg["nsq"],
              "nq": cfg["nq"], "nprobe": cfg["nprobe"], "k": cfg["k"], "lists": meta,
              "l2": "flushed between timed steps (256 MiB memset)",
              "parallelism": {"single": "single GPU", "replicas": f"query-parallel replicas x{world}",
                              "shard-lists": f"list-sharded x{world}"}[mode]}

    if args.impl == "reference":
        if rank != 0:
            dist.barrier() if world > 1 else None
            return
        res = reference_arm(args, path, queries, cfg)
        if isinstance(res, dict):
            print(json.dumps(res))
            return
        r, threads = res
        qps = r["qps"]
        line = {"impl": "reference", "metric": METRIC, "value": qps, "unit": "queries/s", "n_gpus": world,
                "steps": r["reps"], "warmup": args.warmup, "ms_per_step": r["p50_s"] * 1e3,
                "higher_is_better": True, "scaling": "weak" if mode == "replicas" else "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": config,
                "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": threads, "kind": "reference",
                                 "single_thread_value": r.get("single_thread_qps"),
                                 "sample": f"{r['reps']} timed batches of {cfg['nq']} queries (p50), "
                                           f"prag::search on {threads} std::threads, index via load_index",
                                 "cpu": cpu_model()},
                "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        if world > 1:
            dist.barrier()
        return

    import paper_2403_05676_b200 as pg

    dev = torch.device("cuda", local)
    if mode == "shard-lists":
        ix = pg.GpuIndex.load_shard(path, rank, world, local)
    else:
        ix = pg.GpuIndex.load(path, local)
    if mode == "replicas":  # each rank its own batch (same cost: a rotation of the fixture queries)
        queries = np.ascontiguousarray(np.roll(queries, 8 * rank, axis=0))
    stream = torch.cuda.Stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    nq, k, nprobe = cfg["nq"], cfg["k"], cfg["nprobe"]
    qdev = torch.from_numpy(queries[:nq]).to(dev)
    from paper_2403_05676_b200 import distributed as PD

    # a serving loop reuses its device buffers: each (query buffer, nprobe, k)
    # gets result buffers and a captured search (prag_gpu_plan: one CUDA-graph
    # launch for the five kernels) on first use
    plans = {}

    def step_dev(qd, nprobe_, k_):
        key = (qd.data_ptr(), qd.shape[0], nprobe_, k_)
        if key not in plans:
            nq_ = qd.shape[0]
            out = pg.BatchResult(torch.empty((nq_, k_), dtype=torch.int64, device=dev),
                                 torch.empty((nq_, k_), dtype=torch.float32, device=dev),
                                 torch.empty((nq_,), dtype=torch.int32, device=dev),
                                 torch.empty((nq_,), dtype=torch.int64, device=dev))
            plans[key] = ix.plan(qd, k_, nprobe_, out, stream=stream)
        with torch.cuda.stream(stream):
            r = plans[key].launch(stream=stream)
            if mode == "shard-lists":  # one packed NCCL all-gather of the per-shard top-k, exact merge on rank 0
                r = PD.gather_merge(r, k_)
        return r

    def timed(fn, steps, warmup):
        ts = []
        for i in range(warmup + steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize(dev)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            if i >= warmup:
                ts.append(e0.elapsed_time(e1))
        t = torch.tensor(ts, dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.cpu().tolist()

    # ---------------- headline: device-resident
    with ClockSampler(local) as clk:
        # pre-roll: back-to-back steps for ~1 s so the clock sampler sees this
        # load (the timed region itself is only tens of ms)
        # (every rank must run the same number of steps: each one contains a
        # collective, so with N > 1 the ranks agree on when to stop)
        t_end = time.time() + 1.0
        while True:
            step_dev(qdev, nprobe, k)
            torch.cuda.synchronize(dev)
            stop = time.time() >= t_end
            if world > 1:
                flag = torch.tensor([1 if stop else 0], dtype=torch.int32,
                                    device=dev if backend == "nccl" else "cpu")
                dist.all_reduce(flag, op=dist.ReduceOp.MAX)
                stop = bool(flag.item())
            if stop:
                break
        t_dev = timed(lambda: step_dev(qdev, nprobe, k), args.steps, args.warmup)
        # e2e: pinned host queries -> host results through the public API: the
        # query batch is copied into a captured plan's device buffer, the plan
        # runs, and the four result arrays (one contiguous device block) come
        # back in one copy
        qhost = torch.from_numpy(queries[:nq].copy()).pin_memory()
        h_out = pg.BatchResult(torch.empty((nq, k), dtype=torch.int64).pin_memory(),
                               torch.empty((nq, k), dtype=torch.float32).pin_memory(),
                               torch.empty((nq,), dtype=torch.int32).pin_memory(),
                               torch.empty((nq,), dtype=torch.int64).pin_memory())
        o_dist = nq * k * 8
        o_cnt = o_dist + ((nq * k * 4 + 7) & ~7)
        o_sc = o_cnt + ((nq * 4 + 7) & ~7)
        blk_bytes = o_sc + nq * 8

        def views(blk):
            return pg.BatchResult(blk[:o_dist].view(torch.int64).view(nq, k),
                                  blk[o_dist:o_dist + nq * k * 4].view(torch.float32).view(nq, k),
                                  blk[o_cnt:o_cnt + nq * 4].view(torch.int32), blk[o_sc:].view(torch.int64))
        d_blk = torch.empty(blk_bytes, dtype=torch.uint8, device=dev)
        h_blk = torch.empty(blk_bytes, dtype=torch.uint8).pin_memory()
        h_out = views(h_blk)
        q_buf = torch.empty((nq, cfg["d"]), dtype=torch.float32, device=dev)
        e2e_plan = ix.plan(q_buf, k, nprobe, views(d_blk), stream=stream) if mode != "shard-lists" else None

        def step_e2e():
            if mode != "shard-lists":
                with torch.cuda.stream(stream):
                    q_buf.copy_(qhost, non_blocking=True)
                    e2e_plan.launch(stream=stream)
                    h_blk.copy_(d_blk, non_blocking=True)
                stream.synchronize()
            else:
                qd = qhost.to(dev, non_blocking=True)
                r = step_dev(qd, nprobe, k)
                if rank == 0:
                    for a, b in zip((r.ids, r.dist, r.count, r.scanned), (h_out.ids, h_out.dist, h_out.count,
                                                                          h_out.scanned)):
                        b.copy_(a, non_blocking=True)
                stream.synchronize()

        t_e2e = []
        for i in range(args.warmup + args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            torch.cuda.synchronize(dev)
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            step_e2e()
            dt = (time.perf_counter() - t0) * 1e3
            if i >= args.warmup:
                t_e2e.append(dt)
        if world > 1:
            tt = torch.tensor(t_e2e, dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_e2e = tt.cpu().tolist()
    clocks = clk.summary()

    total_q = nq * world if mode == "replicas" else nq  # replicas: each rank its own batch
    ms_per_step = sum(t_dev) / len(t_dev)
    value = total_q * len(t_dev) / (sum(t_dev) / 1e3)
    e2e_ms = sum(t_e2e) / len(t_e2e)
    e2e_val = total_q * len(t_e2e) / (sum(t_e2e) / 1e3)

    # ---------------- roofline of the dominant kernel (fused LUT+scan+select)
    ix.set_profiling(True)
    tm_acc = {"scan_ms": 0.0, "total_ms": 0.0, "scanned_bytes": 0, "coarse_ms": 0.0, "select_ms": 0.0,
              "plan_ms": 0.0, "final_ms": 0.0, "work_items": 0, "coarse_window": 0}
    prof_steps = max(5, min(args.steps, 20))
    for i in range(prof_steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        torch.cuda.synchronize(dev)
        ix.search_batch(qdev, k, nprobe, stream=stream)
        torch.cuda.synchronize(dev)
        t = ix.last_timings()
        for key in tm_acc:
            tm_acc[key] += t[key]
    ix.set_profiling(False)
    hbm, peak_src = peaks()
    scan_ms = tm_acc["scan_ms"] / prof_steps
    bytes_launch = tm_acc["scanned_bytes"] / prof_steps
    achieved = bytes_launch / (scan_ms / 1e3) / 1e9 if scan_ms > 0 else 0.0
    traffic = None
    tp = os.path.join(REPO, "profiles", "ncu_scan_traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            if tj.get("workload") == workload:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            pass
    # K1 (tcgen05 3xTF32 GEMM pre-filter): flops actually issued to the tensor
    # pipe (3 MMAs per product) over K1's CUDA-event time, against the TF32
    # dense peak (half the measured bf16 figure: kind::tf32 runs at 1/2 rate)
    k1_ms = tm_acc["coarse_ms"] / prof_steps
    k1_flops = 3 * 2 * nq * cfg["nlist"] * cfg["d"]
    bf16 = None
    try:
        bf16 = float(json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["bf16_tflops"])
    except Exception:
        bf16 = 2250.0
    roofline_coarse = {"bound": "tensor", "kernel": "coarse_tc_kernel (tcgen05 kind::tf32, 3xTF32)",
                       "achieved": round(k1_flops / (k1_ms / 1e3) / 1e12, 2) if k1_ms > 0 else None,
                       "peak": round(bf16 / 2, 1), "unit": "TFLOP/s",
                       "peak_source": "MEASURED_PEAKS.json bf16_tflops / 2 (TF32 rate)",
                       "kernel_ms": round(k1_ms, 4), "flops_per_launch": k1_flops,
                       "window_lists_per_query": round(tm_acc["coarse_window"] / prof_steps / nq, 2),
                       "note": "latency-bound at this GEMM size (nq x nlist x d = 64 x 4096 x 384)"}
    if roofline_coarse["achieved"] is not None:
        roofline_coarse["frac"] = round(roofline_coarse["achieved"] / roofline_coarse["peak"], 4)
    roofline = {"bound": "hbm", "kernel": "scan_skew_kernel (ADC list scan + warp top-k)", "achieved": round(achieved, 1),
                "peak": hbm, "unit": "GB/s", "frac": round(achieved / hbm, 4), "traffic": traffic,
                "peak_source": peak_src, "alg_bytes_per_launch": int(bytes_launch),
                "kernel_ms": round(scan_ms, 4), "kernel_share_of_step": round(scan_ms / (tm_acc["total_ms"] /
                                                                                        prof_steps), 3),
                "phase_ms": {p: round(tm_acc[p] / prof_steps, 4) for p in
                             ("coarse_ms", "select_ms", "plan_ms", "scan_ms", "final_ms", "total_ms")}}

    # ---------------- sweep (rank-synchronous), perf model on the GPU curve
    sweep = []
    if not args.no_sweep:
        for nq_s in SWEEP_NQ:
            qd = torch.from_numpy(queries[:nq_s]).to(dev)
            for np_s in SWEEP_NPROBE:
                ts = timed(lambda: step_dev(qd, np_s, k), max(5, args.steps // 5), 3)
                p50 = statistics.median(ts)
                sweep.append({"nq": nq_s, "nprobe": np_s, "p50_ms": round(p50, 4), "qps": round(nq_s / (p50 / 1e3),
                                                                                              1)})
    perf_models = {}
    if world == 1 and not args.no_sweep:
        for nq_s in (1, 64):
            m, lat = pg.calibrate_gpu(ix, queries[:nq_s], k, SWEEP_NPROBE, repeats=5, warmups=2)
            perf_models[str(nq_s)] = {"slope_s": m.slope_s, "intercept_s": m.intercept_s,
                                      "fit_residual_s": m.fit_residual_s, "clamped": m.clamped,
                                      "select_nprobe_10ms": pg.select_nprobe(m, 10e-3, ix.nlist),
                                      "select_nprobe_1ms": pg.select_nprobe(m, 1e-3, ix.nlist)}

    # ---------------- CPU baseline (rank 0, N=1): the reference on host cores
    cpu_baseline = None
    if rank == 0 and world == 1:
        try:
            res = reference_arm(argparse.Namespace(steps=5, warmup=1, ref_seconds=args.ref_seconds), path, queries,
                                cfg)
            if isinstance(res, tuple):
                r, threads = res
                cpu_baseline = {"value": r["qps"], "unit": "queries/s", "cores": threads, "kind": "reference",
                                "single_thread_value": r.get("single_thread_qps"),
                                "sample": f"{r['reps']} batches x {cfg['nq']} queries, nprobe={nprobe}, k={k} "
                                          f"(p50 {r['p50_s'] * 1e3:.1f} ms/batch), prag::search on {threads} "
                                          f"threads, same PRAGIX01 file", "cpu": cpu_model()}
            else:
                cpu_baseline = res
        except Exception as e:  # report, never fake
            cpu_baseline = {"unavailable": str(e)[:200]}

    if rank == 0:
        h2d = nq * cfg["d"] * 4
        d2h = nq * k * 12 + nq * 4 + nq * 8
        line = {"metric": METRIC, "value": round(value, 1), "unit": "queries/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
                "p50_batch_ms": round(statistics.median(t_dev), 4), "higher_is_better": True,
                "scaling": "weak" if mode == "replicas" else "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": config,
                "e2e": {"value": round(e2e_val, 1), "unit": "queries/s", "ms_per_step": round(e2e_ms, 4),
                        "p50_batch_ms": round(statistics.median(t_e2e), 4), "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h},
                # our kernels per timed step: K1, K1b, K2 (+planner), K3, K4; list sharding adds the merge
                "gpu_launches": 5 * args.steps + (args.steps if mode == "shard-lists" else 0),
                "roofline": roofline, "roofline_coarse": roofline_coarse, "cpu_baseline": cpu_baseline, "clocks": clocks, "sweep": sweep,
                "perf_model": perf_models}
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
