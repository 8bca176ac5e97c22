"""PipeRAG's pipelined generation loop on one B200 (BASELINE.json configs[4]).

The reference overlaps retrieval with generation using a std::thread worker
and a mutex/condition-variable mailbox (pipeline.hpp:471-554, mailbox
:316-351). Here both sides are GPU work on one device:

  * decode     -- the main stream runs the synthetic RETRO-style decode
                  (prag_gpu_synthetic_decode: the model's fp32 weights plus
                  the KV cache of earlier positions streamed per token),
                  standing in for SyntheticGenerator (generator.hpp:220-252);
  * retrieval  -- a high-priority side stream runs the query embedding
                  (prag_gpu_embed, ChunkEmbedder::embed bit-identical) and
                  the IVF-PQ search of the next chunk (prag_gpu_search,
                  device pointers, async);
  * mailbox    -- a CUDA event per chunk: ready(j) = cudaEventQuery,
                  take(j) = cudaStreamWaitEvent on the main stream; the stall
                  is the device time the main stream spends blocked on it;
  * SMs        -- with `retrieval_sms` = R, the piperag decode runs on the
                  other S - R SMs (prag_gpu_synthetic_decode_sms: one CTA per
                  SM) and the search sizes its persistent grids to R SMs
                  (prag_gpu_set_sm_budget), so the side stream has SMs of its
                  own instead of waiting for decode kernels to drain.

Modes and their schedule follow PipelineEngine::run_impl (pipeline.hpp
:414-452): "retro" retrieves (blocking) before every chunk, "piperag" launches
chunk j+1's retrieval before generating chunk j. The query of chunk j is the
window of m tokens ending `staleness` tokens before chunk j starts
(make_query_window, pipeline.hpp:122-144; staleness = interval for piperag
and 0 for retro, pipeline.hpp:70-76), embedded on the GPU; without a token
sequence the engine falls back to fixed query rows.
With the auto nprobe policy, nprobe = select_nprobe(retrieval model,
predict_chunk_budget(inference model, position)) (pipeline.hpp:414-420,
perfmodel.hpp:148-183). All timestamps are CUDA events on the device clock.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from ._lib import check, lib
from .ivfpq import BatchResult, GpuIndex, RetrievalPerfModel, select_nprobe

try:
    import torch
except Exception:  # pragma: no cover
    torch = None


# ------------------------------------------------ inference perf model
@dataclass
class InferenceBucket:
    """perfmodel.hpp:28-32."""
    position: int
    m: int
    seconds: float


@dataclass
class InferencePerfModel:
    """perfmodel.hpp:34-37."""
    buckets: List[InferenceBucket] = field(default_factory=list)
    monotonicity_warning: bool = False


def calibrate_inference(generate: Callable[[int], float], positions: Sequence[int], m_prime: int,
                        repeats: int = 3, warmups: int = 2) -> InferencePerfModel:
    """perfmodel.hpp:121-143: per-position median chunk latency."""
    if not positions:
        raise ValueError("calibrate_inference: positions must be non-empty")
    model = InferencePerfModel()
    for p in sorted(set(int(x) for x in positions)):
        for _ in range(warmups):
            generate(p)
        runs = sorted(generate(p) for _ in range(repeats))
        n = len(runs)
        med = runs[n // 2] if n % 2 else 0.5 * (runs[n // 2 - 1] + runs[n // 2])
        model.buckets.append(InferenceBucket(p, m_prime, med))
    for a, b in zip(model.buckets, model.buckets[1:]):
        if b.seconds < 0.8 * a.seconds:
            model.monotonicity_warning = True
    return model


def predict_chunk_budget(model: InferencePerfModel, position: int):
    """perfmodel.hpp:162-183 -> (seconds, extrapolated)."""
    b = model.buckets
    if not b:
        raise ValueError("predict_chunk_budget: model not calibrated")
    if len(b) == 1:
        return b[0].seconds, position != b[0].position
    if position <= b[0].position:
        return b[0].seconds, position < b[0].position
    if position >= b[-1].position:
        if position == b[-1].position:
            return b[-1].seconds, False
        p0, p1 = b[-2], b[-1]
        slope = (p1.seconds - p0.seconds) / float(p1.position - p0.position)
        return p1.seconds + slope * float(position - p1.position), True
    for i in range(1, len(b)):
        if position <= b[i].position:
            t = float(position - b[i - 1].position) / float(b[i].position - b[i - 1].position)
            return b[i - 1].seconds + t * (b[i].seconds - b[i - 1].seconds), False
    return b[-1].seconds, False


# ------------------------------------------------------------- decoder
class SyntheticDecoder:
    """Memory-bound decode stand-in: `params` fp32 weights streamed per token
    plus `kv_bytes_per_token` of KV cache per earlier position."""

    def __init__(self, params: int = 582_000_000, cols: int = 4096, kv_bytes_per_token: int = 2 * 24 * 1024 * 4,
                 max_positions: int = 4096, device: int = 0, stream=None, sms: Optional[int] = None):
        assert torch is not None
        self.dev = torch.device("cuda", device)
        self.cols = cols
        self.rows = params // cols
        self.w = torch.randn(self.rows * cols, device=self.dev, dtype=torch.float32)
        self.x = torch.randn(cols, device=self.dev, dtype=torch.float32)
        self.y = torch.empty(self.rows + 1, device=self.dev, dtype=torch.float32)
        self.kv_per_tok = kv_bytes_per_token // 16 * 4  # floats, multiple of 4
        self.kv = torch.randn(self.kv_per_tok * max_positions, device=self.dev, dtype=torch.float32)
        self.max_positions = max_positions
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.dev)
        self.sms = sms  # None: every SM (grid of 4 CTAs per SM); else one CTA on each of `sms` SMs

    def bytes_per_token(self, position: int) -> int:
        return self.rows * self.cols * 4 + min(position, self.max_positions) * self.kv_per_tok * 4

    def step(self, position: int, stream=None) -> None:
        s = stream if stream is not None else self.stream
        kvf = min(position, self.max_positions) * self.kv_per_tok
        args = (C.c_void_p(self.w.data_ptr()), self.rows, self.cols, C.c_void_p(self.x.data_ptr()),
                C.c_void_p(self.y.data_ptr()), C.c_void_p(self.kv.data_ptr()), kvf)
        if self.sms:
            check(lib().prag_gpu_synthetic_decode_sms(*args, int(self.sms), C.c_void_p(s.cuda_stream)))
        else:
            check(lib().prag_gpu_synthetic_decode(*args, C.c_void_p(s.cuda_stream)))

    def generate_chunk(self, position: int, m_prime: int, stream=None) -> None:
        for o in range(m_prime):
            self.step(position + o, stream)

    def time_chunk(self, position: int, m_prime: int) -> float:
        """Seconds for one m'-token chunk at `position` (CUDA events)."""
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(self.stream)
        self.generate_chunk(position, m_prime)
        e1.record(self.stream)
        e1.synchronize()
        return e0.elapsed_time(e1) / 1e3


# ------------------------------------------------------------ pipeline
@dataclass
class TraceEvent:
    kind: str
    chunk_index: int
    t: float


@dataclass
class GenerationTrace:
    """pipeline.hpp:277-303 (device-clock timestamps)."""
    mode: str
    events: List[TraceEvent] = field(default_factory=list)
    total_latency_s: float = 0.0
    stall_time_s: float = 0.0
    retrieval_count: int = 0
    stall_count: int = 0
    nprobe_used: List[int] = field(default_factory=list)
    results: List[BatchResult] = field(default_factory=list)
    queries: List[object] = field(default_factory=list)  # the embedded query of each retrieval

    def durations(self, start_kind: str):
        end = {"gen_chunk_start": "gen_chunk_end", "ret_start": "ret_end"}.get(start_kind, "stall_end")
        starts, out = {}, {}
        for e in self.events:
            if e.kind == start_kind:
                starts[e.chunk_index] = e.t
            if e.kind == end:
                out[e.chunk_index] = e.t - starts[e.chunk_index]
        return out


class PipelineEngine:
    """Runs one generation of `total_tokens` with retrieval every `interval`
    tokens (m'), for mode in {"retro", "piperag"}."""

    STALL_EPS_S = 2e-6  # a wait shorter than this is an already-delivered context

    def __init__(self, decoder: SyntheticDecoder, index: GpuIndex, queries=None, k: int = 2,
                 retrieval_model: Optional[RetrievalPerfModel] = None,
                 inference_model: Optional[InferencePerfModel] = None, safety_margin: float = 0.10,
                 embedder=None, tokens=None, retrieval_sms: Optional[int] = None):
        self.dec = decoder
        self.ix = index
        self.q = queries  # fallback: CUDA tensor [n_queries, d]; chunk j uses row (j-1) % n
        # the token sequence (CUDA int32 [>= m + total_tokens]: prompt chunk,
        # then the generated tokens) and the GPU ChunkEmbedder for query windows
        self.embedder = embedder
        self.tokens = tokens
        self.retrieval_sms = retrieval_sms
        self.k = k
        self.rmodel = retrieval_model
        self.imodel = inference_model
        self.margin = safety_margin
        dev = decoder.dev
        lo, hi = torch.cuda.Stream.priority_range()
        self.side = torch.cuda.Stream(dev, priority=hi)  # retrieval: highest priority
        self.main = decoder.stream

    def _nprobe(self, j: int, m: int, mp: int, fixed: Optional[int]) -> int:
        if fixed is not None:
            return min(int(fixed), self.ix.nlist)
        budget, _ = predict_chunk_budget(self.imodel, m + (j - 1) * mp)
        return select_nprobe(self.rmodel, budget, self.ix.nlist, self.margin)

    def query_window(self, j: int, m: int, mp: int, s: int):
        """make_query_window (pipeline.hpp:122-144) over the token sequence:
        the m tokens ending s before chunk j starts (j == 1: non-stale),
        pad token 0 before position 0; a [1, m] view or padded copy."""
        s_eff = 0 if j == 1 else s
        begin = m + (j - 1) * mp - s_eff - m
        if begin + m > self.tokens.shape[0]:
            raise ValueError("make_query_window: window extends past generated tokens")
        if begin >= 0:
            return self.tokens[begin:begin + m].view(1, m)
        w = torch.zeros((1, m), dtype=self.tokens.dtype, device=self.tokens.device)
        w[0, -begin:] = self.tokens[:begin + m]
        return w

    def run(self, mode: str, total_tokens: int, interval: int, query_window: int = 64,
            nprobe: Optional[int] = 16) -> GenerationTrace:
        if mode not in ("retro", "piperag"):
            raise ValueError("mode must be retro or piperag")
        if self.tokens is None and self.q is None:
            raise ValueError("PipelineEngine needs a token sequence (+ embedder) or fixed query rows")
        if nprobe is None and (self.rmodel is None or self.imodel is None):
            raise ValueError("auto nprobe needs retrieval and inference perf models")
        mp, m = interval, query_window
        n_chunks = total_tokens // mp
        tr = GenerationTrace(mode)
        ev = []  # (kind, chunk, event)

        def rec(kind, j, stream):
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            ev.append((kind, j, e))
            return e

        staleness = mp if mode == "piperag" else 0  # pipeline.hpp:70-76

        def retrieve(j, stream):
            npb = self._nprobe(j, m, mp, nprobe)
            rec("ret_start", j, stream)
            if self.tokens is not None:
                qv = self.embedder.embed(self.query_window(j, m, mp, staleness), stream=stream)
            else:
                qi = (j - 1) % self.q.shape[0]
                qv = self.q[qi:qi + 1]
            r = self.ix.search_batch(qv, self.k, npb, stream=stream)
            done = rec("ret_end", j, stream)
            tr.nprobe_used.append(npb)
            tr.retrieval_count += 1
            tr.results.append(r)
            tr.queries.append(qv)
            return done

        # SM partition for the overlapped mode: decode on S - R SMs, search on R
        part = mode == "piperag" and self.retrieval_sms
        saved = self.dec.sms
        if part:
            total = torch.cuda.get_device_properties(self.dec.dev).multi_processor_count
            self.dec.sms = max(1, total - int(self.retrieval_sms))
            self.ix.set_sm_budget(int(self.retrieval_sms))

        t0 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(self.dec.dev)
        t0.record(self.main)
        stalls = []
        if mode == "retro":
            for j in range(1, n_chunks + 1):
                retrieve(j, self.main)
                rec("gen_chunk_start", j, self.main)
                self.dec.generate_chunk(m + (j - 1) * mp, mp, self.main)
                rec("gen_chunk_end", j, self.main)
        else:
            self.side.wait_stream(self.main)
            pending = {1: retrieve(1, self.side)}
            for j in range(1, n_chunks + 1):
                done = pending.pop(j)
                # mailbox.take(j) as a device-side wait; the stall is the time
                # the main stream spends blocked on it (0 when the context was
                # delivered before decode reached chunk j: mailbox.ready(j))
                s0 = rec("stall_start", j, self.main)
                self.main.wait_event(done)
                s1 = rec("stall_end", j, self.main)
                stalls.append((j, s0, s1))
                if j + 1 <= n_chunks:
                    # chunk j+1's retrieval is launched before chunk j is generated
                    launch = torch.cuda.Event()
                    launch.record(self.main)
                    self.side.wait_event(launch)
                    pending[j + 1] = retrieve(j + 1, self.side)
                rec("gen_chunk_start", j, self.main)
                self.dec.generate_chunk(m + (j - 1) * mp, mp, self.main)
                rec("gen_chunk_end", j, self.main)
        t1 = rec("end", 0, self.main)
        self.main.wait_stream(self.side)
        torch.cuda.synchronize(self.dec.dev)
        if part:
            self.dec.sms = saved
            self.ix.set_sm_budget(0)
        stalled = set()
        for j, s0, s1 in stalls:
            dt = s0.elapsed_time(s1) / 1e3
            if dt > self.STALL_EPS_S:
                tr.stall_time_s += dt
                tr.stall_count += 1
                stalled.add(j)
        tr.events = sorted((TraceEvent(k, j, t0.elapsed_time(e) / 1e3) for k, j, e in ev
                            if k != "end" and (not k.startswith("stall") or j in stalled)), key=lambda x: x.t)
        tr.total_latency_s = t0.elapsed_time(t1) / 1e3
        return tr
