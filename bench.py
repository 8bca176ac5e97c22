#!/usr/bin/env python
"""IVF-PQ search benchmark (BASELINE.json configs[1] at N=1, configs[2] at N>1).

One "step" = one batch search.

N=1 (default): config B -- synthetic 10M x 384 fp32 DB, IVF nlist=4096, PQ
m=32 x 8-bit (PRAGIX01 fixture built by paper_2403_05676_b200/fixtures.py),
nq=64 queries (DB row + 0.05 N(0,1)), nprobe=16, k=10. The nprobe sweep
1..128 x nq {1,16,64} is reported beside the headline in "sweep", with the
GPU-recalibrated performance model.

N>1 (torchrun, one rank per GPU): config C -- 100M x 384, nlist 16384, PQ
m=64 (6.4 GB of codes) built in HBM by prag_gpu_index_synthetic and SHARDED
BY INVERTED LIST across the ranks (LPT on list bytes); every step is one
collective search through the C ABI: K1-K4 on each rank's lists, one
ncclAllGather of the per-shard top-k issued by libprag_gpu on the search
stream (inside the captured plan), the exact merge kernel. Same DB and
queries for every N: "scaling": "strong". PRAG_BENCH_CONFIG=C runs the same
workload unsharded at N=1 (the scaling denominator); PRAG_BENCH_MODE=replicas
runs config B as query-parallel replicas instead (weak scaling, no
collective).

  value : queries/s, queries and outputs resident in HBM, CUDA events on the
          search stream around each step, L2 flushed (256 MiB memset) between
          steps, all queries of the step / max-over-ranks time.
  e2e   : the same metric through the drop-in call, prag_gpu_search with
          pinned HOST query and result buffers (H2D of the queries and D2H of
          ids/dist/count/scanned inside the call, every step). e2e.variants
          adds pageable host buffers and the captured-plan path.
  parity: the last timed step's output compared bit for bit (ids, distance
          bits, counts, scanned_vectors) with the reference's own
          prag::search (oracle/_ref/ref_tool on the same PRAGIX01 file and
          queries) for config B, and with the exact host restatement of the
          synthetic index (tests/_synth_ref.py, pinned to the reference by
          tests/test_ref_synth.py) on sampled queries for config C. A
          mismatch fails the run (exit 1) after the line is printed.
  --impl reference : the unmodified reference prag::search (oracle/_ref,
          compiled from /root/reference) on this box's host cores, same index
          and queries, same metric.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CFG_B = dict(name="B", n=10_000_000, d=384, nlist=4096, nsq=32, seed=1, nq=64, nprobe=16, k=10)
CFG_C = dict(name="C", n=100_000_000, d=384, nlist=16384, nsq=64, seed=2024, model_seed=11, sigma=1.0, nq=64,
             nprobe=16, k=10)
SWEEP_NPROBE = [1, 2, 4, 8, 16, 32, 64, 128]
SWEEP_NQ = [1, 16, 64]
METRIC = "ivfpq_search_queries_per_s"
TOOL = os.path.join(REPO, "oracle", "_ref", "ref_tool")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), float(j.get("bf16_tflops", 2250.0)), "measured (MEASURED_PEAKS.json)"
    return 6650.0, 2250.0, "fallback (B200_PROFILING.md)"


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
                "window": "nvidia-smi -lms 20 over a 1 s pre-roll of back-to-back steps + the timed regions"}


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ----------------------------------------------------------------- workloads
def synth_model(cfg):
    """Centroids, codebook and queries of the config-C synthetic index (the
    recipe of tools/config_d.py: N(0,1) centroids, 0.3 N(0,1) codewords,
    queries = a centroid + 0.5 N(0,1))."""
    rng = np.random.default_rng(cfg["model_seed"])
    cents = rng.standard_normal((cfg["nlist"], cfg["d"])).astype(np.float32)
    words = (rng.standard_normal((cfg["nsq"], 256, cfg["d"] // cfg["nsq"])) * 0.3).astype(np.float32)
    q = (cents[rng.integers(0, cfg["nlist"], 64)] +
         rng.standard_normal((64, cfg["d"])).astype(np.float32) * 0.5).astype(np.float32)
    return cents, words, q


def workload_name(cfg, world, mode):
    if cfg["name"] == "B":
        w = (f"config B: ivfpq search, {cfg['n'] // 1_000_000}M x {cfg['d']} fp32 DB, nlist={cfg['nlist']}, "
             f"PQ m={cfg['nsq']}x8b, nq={cfg['nq']}, nprobe={cfg['nprobe']}, k={cfg['k']}")
    else:
        w = (f"config C: ivfpq search, {cfg['n'] // 1_000_000}M x {cfg['d']} DB (synthetic codes in HBM), "
             f"nlist={cfg['nlist']}, PQ m={cfg['nsq']}x8b, nq={cfg['nq']}, nprobe={cfg['nprobe']}, k={cfg['k']}")
    if mode == "shard-lists":
        w += f", lists sharded over {world} GPUs"
    elif mode == "replicas":
        w += f", {world} query-parallel replicas"
    return w


# ----------------------------------------------------------------- reference
def reference_bench(cfg, path, queries, threads, steps, warmup, seconds, out_bin=None, tmp=None):
    """The unmodified reference prag::search on `threads` host threads
    (oracle/_ref/ref_tool); config C runs on the same synthetic index rebuilt
    as the reference's IvfIndex (ref_tool synth-bench)."""
    if not os.path.exists(TOOL):
        return None, "oracle/_ref/ref_tool not built (needs /root/reference at build)"
    tmp = tmp or tempfile.mkdtemp(prefix="prag_bench_")
    qp = os.path.join(tmp, f"q{cfg['nq']}.f32")
    queries[:cfg["nq"]].astype(np.float32).tofile(qp)
    if cfg["name"] == "B":
        cmd = [TOOL, "bench", path, qp, str(cfg["nq"]), str(cfg["nprobe"]), str(cfg["k"]), str(threads), str(steps),
               str(warmup), str(seconds)] + ([out_bin] if out_bin else [])
    else:
        cp, wp, sp = path
        cmd = [TOOL, "synth-bench", cp, wp, sp, str(cfg["nlist"]), str(cfg["d"]), str(cfg["nsq"]), str(cfg["seed"]), qp,
               str(cfg["nq"]), str(cfg["nprobe"]), str(cfg["k"]), str(threads), str(steps), str(warmup), str(seconds)]
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        return None, f"ref_tool failed: {out.stderr.strip()[-200:]}"
    return json.loads(out.stdout.strip().splitlines()[-1]), None


def write_synth_inputs(cfg, cents, words, sizes, tmp):
    cp, wp, sp = (os.path.join(tmp, x) for x in ("cents.f32", "words.f32", "sizes.u64"))
    cents.tofile(cp)
    words.tofile(wp)
    np.ascontiguousarray(sizes, dtype=np.uint64).tofile(sp)
    return cp, wp, sp


def read_ref_results(path, nq, k):
    ids = np.zeros((nq, k), np.uint64)
    dist = np.zeros((nq, k), np.float32)
    cnt = np.zeros(nq, np.uint32)
    sc = np.zeros(nq, np.uint64)
    with open(path, "rb") as f:
        for i in range(nq):
            c, _sl, s = np.frombuffer(f.read(16), dtype=np.dtype([("c", "<u4"), ("l", "<u4"), ("s", "<u8")]))[0]
            rec = np.frombuffer(f.read(12 * k), dtype=[("id", "<u8"), ("d", "<f4")])
            cnt[i], sc[i] = c, s
            ids[i, :c] = rec["id"][:c]
            dist[i, :c] = rec["d"][:c]
    return ids, dist, cnt, sc


def compare(name, got, want, rows=None):
    """Bit-exact comparison of (ids, dist, count, scanned) on the given rows."""
    gi, gd, gc, gs = (np.asarray(x) for x in got)
    wi, wd, wc, ws = want
    rows = range(len(wc)) if rows is None else rows
    bad = []
    for j, i in enumerate(rows):
        c = int(wc[j])
        ok = int(gc[i]) == c and int(gs[i]) == int(ws[j])
        ok = ok and (gi[i, :c].astype(np.uint64) == wi[j, :c]).all()
        ok = ok and (gd[i, :c].view(np.uint32) == wd[j, :c].view(np.uint32)).all()
        if not ok:
            bad.append(int(i))
    return {"checked_queries": len(list(rows)), "mismatched_queries": bad, "ok": not bad, "against": name}


def fields(r):
    return r.ids, r.dist, r.count, r.scanned


def to_np(r):
    def cv(t):
        t = t.detach().cpu() if hasattr(t, "detach") else t
        a = t.numpy() if hasattr(t, "numpy") else np.asarray(t)
        return a.view(np.uint64) if a.dtype == np.int64 else a.view(np.uint32) if a.dtype == np.int32 else a
    return cv(r.ids), cv(r.dist), cv(r.count), cv(r.scanned)


# ----------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--small", action="store_true", help="1M-vector config B / 10M config C for quick checks")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=20.0)
    args = ap.parse_args()
    assert args.warmup >= 3, "W >= 3 warm-up steps"

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    mode = os.environ.get("PRAG_BENCH_MODE", "shard-lists" if world > 1 else "single")
    if mode not in ("single", "replicas", "shard-lists"):
        raise SystemExit(f"PRAG_BENCH_MODE must be single, replicas or shard-lists, not {mode}")
    if world == 1 and mode == "replicas":
        mode = "single"
    cname = os.environ.get("PRAG_BENCH_CONFIG", "C" if mode == "shard-lists" else "B")
    cfg = dict(CFG_C if cname == "C" else CFG_B)
    if args.small:
        cfg.update(n=1_000_000, nlist=1024) if cname == "B" else cfg.update(n=10_000_000, nlist=4096)

    import torch
    import torch.distributed as dist

    # PRAG_BENCH_BACKEND=gloo runs the N>1 path functionally on fewer GPUs
    # than ranks (ranks share devices round-robin; the exchange then goes
    # through torch.distributed instead of libprag_gpu's NCCL communicator);
    # numbers from such a run are not bench values
    backend = os.environ.get("PRAG_BENCH_BACKEND", "nccl" if args.impl == "ours" else "gloo")
    if torch.cuda.is_available() and backend == "gloo":
        local = local % torch.cuda.device_count()
    if world > 1:
        dist.init_process_group(backend, device_id=torch.device("cuda", local) if backend == "nccl" else None)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    workload = workload_name(cfg, world, mode)
    scaling = "weak" if mode == "replicas" else "strong"
    parallelism = {"single": "single GPU", "replicas": f"query-parallel replicas x{world}",
                   "shard-lists": f"inverted lists sharded over {world} GPUs (LPT on bytes, lists >= 4x the mean "
                                  f"striped over all ranks), NCCL all-gather "
                                  f"of per-shard top-k + exact merge"}[mode]

    import paper_2403_05676_b200 as pg
    from paper_2403_05676_b200 import distributed as PD

    # ------------------------------------------------------------ workload
    tmp = tempfile.mkdtemp(prefix="prag_bench_")
    meta = {}
    if cfg["name"] == "B":
        from paper_2403_05676_b200 import fixtures as F
        if rank == 0:
            path, queries, meta = F.ensure_fixture(cfg["n"], cfg["d"], cfg["nlist"], cfg["nsq"], cfg["seed"], nq=64,
                                                   log=log)
        if world > 1:
            dist.barrier()
        if rank != 0:
            path, queries, meta = F.ensure_fixture(cfg["n"], cfg["d"], cfg["nlist"], cfg["nsq"], cfg["seed"], nq=64,
                                                   log=log)
        cents = words = sizes = None
    else:
        cents, words, queries = synth_model(cfg)
        path = None
    config = {"workload": workload, "n": cfg["n"], "d": cfg["d"], "nlist": cfg["nlist"], "m": cfg["nsq"],
              "nq": cfg["nq"], "nprobe": cfg["nprobe"], "k": cfg["k"],
              "l2": "flushed between timed steps (256 MiB memset)", "parallelism": parallelism}

    # ------------------------------------------------------------ reference arm
    if args.impl == "reference":
        if rank != 0:
            if world > 1:
                dist.barrier()
            return
        threads = os.cpu_count() or 1
        if cfg["name"] == "C":
            # list sizes of the synthetic index (the GPU builder's, so both
            # sides hold the same lists; the build is not timed)
            ixs = pg.GpuIndex.synthetic(cents, words, cfg["n"], seed=cfg["seed"], sigma=cfg["sigma"], device=local)
            sizes = ixs.list_sizes()
            ixs.close()
            src = write_synth_inputs(cfg, cents, words, sizes, tmp)
        else:
            src = path
        r, err = reference_bench(cfg, src, queries, threads, args.steps, args.warmup, args.ref_seconds, tmp=tmp)
        if r is None:
            print(json.dumps({"impl": "reference", "unavailable": err}))
        else:
            qps = r["qps"]
            print(json.dumps({
                "impl": "reference", "metric": METRIC, "value": qps, "unit": "queries/s", "n_gpus": world,
                "steps": r["reps"], "warmup": args.warmup, "ms_per_step": r["p50_s"] * 1e3, "higher_is_better": True,
                "scaling": scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": config,
                "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": threads, "kind": "reference",
                                 "sample": f"{r['reps']} timed batches of {cfg['nq']} queries (p50; bounded to "
                                           f"~{args.ref_seconds:.0f} s), prag::search on {threads} std::threads",
                                 "index_build_or_load_s": r.get("load_s"), "cpu": cpu_model()},
                "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        if world > 1:
            dist.barrier()
        return

    # ------------------------------------------------------------ our index
    sharded = mode == "shard-lists" and world > 1
    use_comm = sharded and backend == "nccl"
    t0 = time.time()
    if cfg["name"] == "B":
        if sharded:
            ix = pg.GpuIndex.load_shard(path, rank, world, local)
        else:
            ix = pg.GpuIndex.load(path, local)
    else:
        if sharded:
            ix = pg.GpuIndex.synthetic_shard(cents, words, cfg["n"], rank, world, seed=cfg["seed"],
                                             sigma=cfg["sigma"], device=local)
        else:
            ix = pg.GpuIndex.synthetic(cents, words, cfg["n"], seed=cfg["seed"], sigma=cfg["sigma"], device=local)
    comm = None
    if use_comm:  # searches on this shard become collective (NCCL inside libprag_gpu)
        comm = PD.make_comm(local)
        ix.attach_comm(comm)
    build_s = time.time() - t0
    sizes = ix.list_sizes().astype(np.int64)
    if sharded:  # every list lives on exactly one shard: the global sizes are the sum
        st = torch.from_numpy(sizes).to(dev if backend == "nccl" else "cpu")
        dist.all_reduce(st)
        sizes = st.cpu().numpy().astype(np.int64)
    if cfg["name"] == "C":
        meta = {"list_p50": int(np.median(sizes)), "list_p90": int(np.percentile(sizes, 90)),
                "list_max": int(sizes.max()), "list_avg": float(sizes.mean()), "build_s": round(build_s, 2),
                "codes_GB_total": round(float(sizes.sum()) * cfg["nsq"] / 1e9, 2),
                "data": "synthetic codes and list sizes (prag_gpu_index_synthetic, log-normal sigma 1.0)"}
    config["lists"] = meta

    if mode == "replicas":  # each rank its own batch (same cost: a rotation of the fixture queries)
        queries = np.ascontiguousarray(np.roll(queries, 8 * rank, axis=0))
    stream = torch.cuda.Stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    nq, k, nprobe, d = cfg["nq"], cfg["k"], cfg["nprobe"], cfg["d"]
    qdev = torch.from_numpy(queries[:nq]).to(dev)
    gather_torch = sharded and not use_comm  # gloo functional runs

    # a serving loop reuses its device buffers: each (query buffer, nprobe, k)
    # gets result buffers and a captured search (prag_gpu_plan: one CUDA-graph
    # launch for the kernel chain, with the NCCL exchange when sharded) on
    # first use
    plans = {}

    def dev_out(nq_, k_):
        return pg.BatchResult(torch.empty((nq_, k_), dtype=torch.int64, device=dev),
                              torch.empty((nq_, k_), dtype=torch.float32, device=dev),
                              torch.empty((nq_,), dtype=torch.int32, device=dev),
                              torch.empty((nq_,), dtype=torch.int64, device=dev))

    def step_dev(qd, nprobe_, k_):
        key = (qd.data_ptr(), qd.shape[0], nprobe_, k_)
        if key not in plans:
            plans[key] = ix.plan(qd, k_, nprobe_, dev_out(qd.shape[0], k_), stream=stream)
        with torch.cuda.stream(stream):
            r = plans[key].launch(stream=stream)
            if gather_torch:
                r = PD.gather_merge(r, k_)
        return r

    def sync_all():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()

    def max_over_ranks(ts):
        t = torch.tensor(ts, dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.cpu().tolist()

    def timed(fn, steps, warmup):
        ts = []
        for i in range(warmup + steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            sync_all()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            if i >= warmup:
                ts.append(e0.elapsed_time(e1))
        return max_over_ranks(ts)

    # e2e through the drop-in call: prag_gpu_search with HOST buffers
    def host_bufs(pinned):
        def mk(shape, dt):
            t = torch.empty(shape, dtype=dt)
            return t.pin_memory() if pinned else t
        qh = mk((nq, d), torch.float32)
        qh.copy_(torch.from_numpy(queries[:nq]))
        out = pg.BatchResult(mk((nq, k), torch.int64).numpy().view(np.uint64), mk((nq, k), torch.float32).numpy(),
                             mk((nq,), torch.int32).numpy().view(np.uint32), mk((nq,), torch.int64).numpy().view(np.uint64))
        return qh.numpy(), out

    def timed_host(fn, steps, warmup):
        ts = []
        for i in range(warmup + steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            sync_all()
            t0_ = time.perf_counter()
            fn()
            dt = (time.perf_counter() - t0_) * 1e3
            if i >= warmup:
                ts.append(dt)
        return max_over_ranks(ts)

    # ------------------------------------------------------------ timed regions
    q_pin, out_pin = host_bufs(True)
    q_page, out_page = host_bufs(False)
    with ClockSampler(local) as clk:
        # pre-roll: back-to-back steps for ~1 s so the clock sampler sees this
        # load; every rank runs the same number of steps (each step may
        # contain a collective), so the ranks agree on when to stop
        t_end = time.time() + 1.0
        while True:
            step_dev(qdev, nprobe, k)
            torch.cuda.synchronize(dev)
            stop = time.time() >= t_end
            if world > 1:
                flag = torch.tensor([1 if stop else 0], dtype=torch.int32, device=dev if backend == "nccl" else "cpu")
                dist.all_reduce(flag, op=dist.ReduceOp.MAX)
                stop = bool(flag.item())
            if stop:
                break
        t_dev = timed(lambda: step_dev(qdev, nprobe, k), args.steps, args.warmup)
        last_dev = step_dev(qdev, nprobe, k)
        torch.cuda.synchronize(dev)
        last_dev = to_np(last_dev) if last_dev is not None else None
        if gather_torch:
            t_e2e = t_page = None
        else:
            t_e2e = timed_host(lambda: ix.search_batch(q_pin, k, nprobe, stream=stream, out=out_pin), args.steps,
                               args.warmup)
            t_page = timed_host(lambda: ix.search_batch(q_page, k, nprobe, stream=stream, out=out_page), args.steps,
                                args.warmup)
        # the captured plan fed from pinned host memory (H2D into the plan's
        # query buffer, graph launch, one D2H of the four result arrays)
        q_buf = torch.empty((nq, d), dtype=torch.float32, device=dev)
        qhost_t = torch.from_numpy(q_pin)
        plan_out = dev_out(nq, k)
        host_plan_out = [torch.empty_like(x, device="cpu").pin_memory() for x in fields(plan_out)]
        e2e_plan = None if gather_torch else ix.plan(q_buf, k, nprobe, plan_out, stream=stream)

        def step_plan_host():
            with torch.cuda.stream(stream):
                q_buf.copy_(qhost_t, non_blocking=True)
                e2e_plan.launch(stream=stream)
                for a_, b_ in zip(fields(plan_out), host_plan_out):
                    b_.copy_(a_, non_blocking=True)
            stream.synchronize()
        t_plan = None if gather_torch else timed_host(step_plan_host, args.steps, args.warmup)
    clocks = clk.summary()

    total_q = nq * world if mode == "replicas" else nq
    ms_per_step = sum(t_dev) / len(t_dev)
    value = total_q * len(t_dev) / (sum(t_dev) / 1e3)

    def rate(ts):
        return None if not ts else total_q * len(ts) / (sum(ts) / 1e3)

    # ------------------------------------------------------------ parity
    parity = {"ok": None}
    if rank == 0 or mode == "replicas":
        if cfg["name"] == "B" and rank == 0 and os.path.exists(TOOL):
            qp = os.path.join(tmp, "parity_q.f32")
            queries[:nq].astype(np.float32).tofile(qp)
            ob = os.path.join(tmp, "parity_ref.bin")
            rr = subprocess.run([TOOL, "search", path, qp, str(nq), str(nprobe), str(k), ob], capture_output=True,
                                text=True)
            if rr.returncode == 0 and last_dev is not None:
                want = read_ref_results(ob, nq, k)
                parity = compare("reference prag::search (oracle/_ref/ref_tool search, same PRAGIX01 file)",
                                 last_dev, want)
                if not gather_torch:
                    parity["e2e_host_output"] = compare("reference", fields(out_pin), want)["ok"]
                    parity["ok"] = parity["ok"] and parity["e2e_host_output"]
            else:
                parity = {"ok": None, "error": (rr.stderr or "")[-200:]}
        elif cfg["name"] == "C" and rank == 0:
            sys.path.insert(0, os.path.join(REPO, "tests"))
            import _synth_ref as R  # test infrastructure, used here only as the checker
            rows = [0, 1, 2, 3]
            want = [R.search(queries[i], cents, words, sizes, cfg["seed"], nprobe, k) for i in rows]
            wi = np.zeros((len(rows), k), np.uint64)
            wd = np.zeros((len(rows), k), np.float32)
            wc = np.zeros(len(rows), np.uint32)
            ws = np.zeros(len(rows), np.uint64)
            for j, (ii, dd, sc) in enumerate(want):
                wc[j], ws[j] = len(ii), sc
                wi[j, :len(ii)] = ii
                wd[j, :len(ii)] = dd
            parity = compare("exact host restatement of prag::search on the synthetic index (tests/_synth_ref.py; "
                             "== the reference prag::search, tests/test_ref_synth.py)", last_dev, (wi, wd, wc, ws),
                             rows)
            if not gather_torch:
                parity["e2e_host_output"] = compare("restatement", fields(out_pin), (wi, wd, wc, ws), rows)["ok"]
                parity["ok"] = parity["ok"] and parity["e2e_host_output"]

    # ------------------------------------------------------------ roofline (K3) + K1
    hbm, bf16, peak_src = peaks()
    ix_local = ix
    if use_comm:
        ix.attach_comm(None)  # per-shard timings: profile the local K1-K4 chain
    ix_local.set_profiling(True)
    acc = {"scan_ms": 0.0, "total_ms": 0.0, "scanned_bytes": 0, "coarse_ms": 0.0, "select_ms": 0.0, "plan_ms": 0.0,
           "final_ms": 0.0, "work_items": 0, "coarse_window": 0}
    prof_steps = max(5, min(args.steps, 20))
    for _ in range(prof_steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        torch.cuda.synchronize(dev)
        ix_local.search_batch(qdev, k, nprobe, stream=stream)
        torch.cuda.synchronize(dev)
        t = ix_local.last_timings()
        for key in acc:
            acc[key] += t[key]
    ix_local.set_profiling(False)
    if use_comm:
        ix.attach_comm(comm)
    scan_ms = acc["scan_ms"] / prof_steps
    bytes_launch = acc["scanned_bytes"] / prof_steps
    achieved = bytes_launch / (scan_ms / 1e3) / 1e9 if scan_ms > 0 else 0.0
    # unique probed-list bytes of this rank's lists
    lists, _ = ix_local.probe(queries[:nq], nprobe)
    local_sizes = ix_local.list_sizes().astype(np.int64)
    uniq_bytes = int(local_sizes[np.unique(lists)].sum()) * cfg["nsq"]
    traffic, traffic_note = None, "no ncu capture for this workload and kernel build"
    tp = os.path.join(REPO, "profiles", "ncu_scan_traffic.json")
    k3_sha = hashlib.sha1(open(os.path.join(REPO, "paper_2403_05676_b200", "csrc", "scan_skew.cu"), "rb").read()
                          ).hexdigest()
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            if tj.get("workload") != workload:
                traffic_note = "ncu capture is for another workload"
            elif tj.get("k3_source_sha1") != k3_sha:
                traffic_note = "ncu capture is of another K3 build (scan_skew.cu sha1 differs): not used"
            else:
                traffic = tj.get("dram_bytes_per_launch")
                traffic_note = f"ncu --set full capture {tj.get('source')} (same scan_skew.cu sha1), per launch"
        except Exception:
            pass
    k1_ms = acc["coarse_ms"] / prof_steps
    k1_flops = 3 * 2 * nq * cfg["nlist"] * d
    roofline_coarse = {"bound": "tensor", "kernel": "coarse_tc_kernel (tcgen05 kind::tf32, 3xTF32)",
                       "achieved": round(k1_flops / (k1_ms / 1e3) / 1e12, 2) if k1_ms > 0 else None,
                       "peak": round(bf16 / 2, 1), "unit": "TFLOP/s",
                       "peak_source": "MEASURED_PEAKS.json bf16_tflops / 2 (TF32 rate)",
                       "kernel_ms": round(k1_ms, 4), "flops_per_launch": k1_flops,
                       "window_lists_per_query": round(acc["coarse_window"] / prof_steps / nq, 2),
                       "note": f"latency-bound at this GEMM size (nq x nlist x d = {nq} x {cfg['nlist']} x {d})"}
    if roofline_coarse["achieved"] is not None:
        roofline_coarse["frac"] = round(roofline_coarse["achieved"] / roofline_coarse["peak"], 4)
    roofline = {"bound": "hbm", "kernel": f"scan_skew_kernel<{cfg['nsq']}> (ADC list scan + warp top-k)",
                "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s", "frac": round(achieved / hbm, 4),
                "traffic": traffic, "traffic_source": traffic_note, "peak_source": peak_src,
                "alg_bytes_per_launch": int(bytes_launch), "unique_probed_bytes": uniq_bytes,
                "unique_frac": round(uniq_bytes / (scan_ms / 1e3) / 1e9 / hbm, 4) if scan_ms > 0 else None,
                "alg_bytes_definition": "sum over the batch of scanned_vectors x m (SURVEY.md 8d B_alg)",
                "kernel_ms": round(scan_ms, 4),
                "kernel_share_of_step": round(scan_ms / (acc["total_ms"] / prof_steps), 3),
                "phase_ms": {p: round(acc[p] / prof_steps, 4) for p in
                             ("coarse_ms", "select_ms", "plan_ms", "scan_ms", "final_ms", "total_ms")},
                "scope": "rank 0's shard (per-shard K1-K4 chain, no exchange)" if sharded else "whole index"}

    # ------------------------------------------------------------ sweep + perf model
    sweep = []
    if not args.no_sweep:
        for nq_s in SWEEP_NQ:
            qd = torch.from_numpy(queries[:nq_s]).to(dev)
            for np_s in SWEEP_NPROBE:
                ts = timed(lambda: step_dev(qd, np_s, k), max(5, args.steps // 5), 3)
                p50 = statistics.median(ts)
                r_ = step_dev(qd, np_s, k)
                torch.cuda.synchronize(dev)
                balg = int(np.asarray(to_np(r_)[3]).astype(np.int64).sum()) * cfg["nsq"] if r_ is not None else None
                lst, _ = ix_local.probe(queries[:nq_s], np_s)
                ub = int(sizes_for_probe(local_sizes, lst)) * cfg["nsq"]
                row = {"nq": nq_s, "nprobe": np_s, "p50_ms": round(p50, 4), "qps": round(nq_s / (p50 / 1e3), 1),
                       "B_alg_MB": round(balg / 1e6, 2) if balg is not None else None,
                       "unique_MB_local": round(ub / 1e6, 2)}
                if balg is not None:
                    row["B_alg_over_search_frac"] = round(balg / (p50 / 1e3) / 1e9 / (hbm * world), 4)
                sweep.append(row)
    perf_models = {}
    if world == 1 and not args.no_sweep:
        for nq_s in (1, 64):
            m, lat = pg.calibrate_gpu(ix, queries[:nq_s], k, SWEEP_NPROBE, repeats=5, warmups=2)
            perf_models[str(nq_s)] = {"slope_s": m.slope_s, "intercept_s": m.intercept_s,
                                      "fit_residual_s": m.fit_residual_s, "clamped": m.clamped,
                                      "select_nprobe_10ms": pg.select_nprobe(m, 10e-3, ix.nlist),
                                      "select_nprobe_1ms": pg.select_nprobe(m, 1e-3, ix.nlist)}

    # ------------------------------------------------------------ CPU baseline (rank 0, N=1)
    cpu_baseline = None
    if rank == 0 and world == 1:
        threads = os.cpu_count() or 1
        src = path if cfg["name"] == "B" else write_synth_inputs(cfg, cents, words, sizes, tmp)
        r, err = reference_bench(cfg, src, queries, threads, 5, 1, args.ref_seconds, tmp=tmp)
        if r is None:
            cpu_baseline = {"unavailable": err}
        else:
            cpu_baseline = {"value": r["qps"], "unit": "queries/s", "cores": threads, "kind": "reference",
                            "sample": f"{r['reps']} batches x {nq} queries, nprobe={nprobe}, k={k} (p50 "
                                      f"{r['p50_s'] * 1e3:.1f} ms/batch), prag::search on {threads} threads, same "
                                      f"index", "cpu": cpu_model()}
            if cfg["name"] == "B":
                # the reference's own protocol: one thread, queries in sequence (perfmodel_main.cpp:57-63)
                r1, _ = reference_bench(cfg, src, queries, 1, 1, 0, 1.0, tmp=tmp)
                if r1:
                    cpu_baseline["single_thread_value"] = r1["qps"]

    if rank == 0:
        h2d = nq * d * 4
        d2h = nq * k * 12 + nq * 4 + nq * 8
        # our kernels per step: K1, K1b, K2 (+planner CTA), K3, K4; sharded adds the merge kernel
        per_step = 5 + (1 if sharded else 0)
        line = {"metric": METRIC, "value": round(value, 1), "unit": "queries/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
                "p50_batch_ms": round(statistics.median(t_dev), 4), "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (config B: SplitMix-style N(0,1) DB and queries, GPU-trained index; config C: "
                        "synthetic codes built in HBM)", "config": config,
                "e2e": None if t_e2e is None else {
                    "value": round(rate(t_e2e), 1), "unit": "queries/s", "ms_per_step": round(sum(t_e2e) / len(t_e2e), 4),
                    "p50_batch_ms": round(statistics.median(t_e2e), 4), "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "path": "prag_gpu_search (C ABI) with pinned host query/result buffers, host wall clock per call",
                    "variants": {
                        "pageable_host_buffers": round(rate(t_page), 1) if t_page else None,
                        "captured_plan_pinned": round(rate(t_plan), 1) if t_plan else None}},
                "parity": parity,
                "gpu_launches": per_step * args.steps, "roofline": roofline, "roofline_coarse": roofline_coarse,
                "cpu_baseline": cpu_baseline, "clocks": clocks, "sweep": sweep, "perf_model": perf_models}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        if use_comm:
            ix.attach_comm(None)
            comm.close()
        dist.destroy_process_group()
    if rank == 0 and parity.get("ok") is False:
        log("PARITY FAILURE: the timed output differs from the reference")
        sys.exit(1)


def sizes_for_probe(sizes, lists):
    return sizes[np.unique(np.asarray(lists))].sum()


if __name__ == "__main__":
    main()
