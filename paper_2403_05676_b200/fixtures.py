"""Synthetic IVF-PQ fixtures (index build is OFF the search hot path).

The reference trains its index with scalar k-means (annindex.hpp:64-241);
SURVEY.md 3(D) measures that at 1,006 s for 1M x 384 and extrapolates ~1.6 h
for 10M, so the bench/test fixtures at B scale are built here instead, with
the same recipe shape -- k-means on a training sample (Lloyd iterations),
nearest-centroid assignment of every vector, residual PQ codebooks by k-means
per subspace, nearest-codeword encoding -- using torch matmuls (cuBLAS) on the
GPU when present. The result is written as PRAGIX01 (annindex.hpp:335-359) so
the CPU oracle, the reference (oracle/_ref) and the GPU path all read the same
bytes. Data follow the reference recipes: x ~ N(0, I) rows
(test_annindex.cpp:12-19) and queries = a DB row + 0.05 N(0, 1)
(annindex_main.cpp:66-74).
"""
from __future__ import annotations

import hashlib
import json
import os
import struct
import time

import numpy as np
import torch


def write_pragix(path, centroids, codewords, list_off, ids, codes) -> None:
    """PRAGIX01 writer from flat SoA arrays (list-major)."""
    centroids = np.ascontiguousarray(centroids, dtype=np.float32)
    codewords = np.ascontiguousarray(codewords, dtype=np.float32)
    nlist, d = centroids.shape
    nsq = codewords.shape[0]
    tmp = path + ".tmp"
    with open(tmp, "wb") as f:
        f.write(b"PRAGIX01")
        f.write(struct.pack("<IIII", 1, nlist, d, nsq))
        f.write(centroids.tobytes())
        f.write(codewords.tobytes())
        rec = np.dtype([("id", "<u8"), ("code", "u1", (nsq,))])
        for l in range(nlist):
            b, e = int(list_off[l]), int(list_off[l + 1])
            f.write(struct.pack("<Q", e - b))
            if e > b:
                r = np.empty(e - b, dtype=rec)
                r["id"] = ids[b:e]
                r["code"] = codes[b:e]
                f.write(r.tobytes())
    os.replace(tmp, path)


def read_pragix(path):
    """PRAGIX01 reader (annindex.hpp:361-411) into flat list-major arrays:
    (centroids [nlist][d], codewords [nsq][256][d/nsq], list_off [nlist+1],
    ids [n], codes [n][nsq])."""
    buf = open(path, "rb").read()
    if buf[:8] != b"PRAGIX01":
        raise ValueError("bad magic")
    _ver, nlist, d, nsq = struct.unpack_from("<IIII", buf, 8)
    at = 24
    cents = np.frombuffer(buf, np.float32, nlist * d, at).reshape(nlist, d)
    at += 4 * nlist * d
    sub = d // nsq
    words = np.frombuffer(buf, np.float32, nsq * 256 * sub, at).reshape(nsq, 256, sub)
    at += 4 * nsq * 256 * sub
    rec = np.dtype([("id", "<u8"), ("code", "u1", (nsq,))])
    off = [0]
    ids, codes = [], []
    for _ in range(nlist):
        (ln,) = struct.unpack_from("<Q", buf, at)
        at += 8
        r = np.frombuffer(buf, rec, ln, at)
        at += ln * rec.itemsize
        ids.append(r["id"])
        codes.append(r["code"])
        off.append(off[-1] + ln)
    return (cents.copy(), words.copy(), np.array(off, dtype=np.uint64),
            np.concatenate(ids).astype(np.uint64) if ids else np.zeros(0, np.uint64),
            np.concatenate(codes).reshape(-1, nsq) if codes else np.zeros((0, nsq), np.uint8))


def _chunk_rows(seed: int, chunk: int, rows: int, d: int, device) -> torch.Tensor:
    g = torch.Generator(device=device)
    g.manual_seed((seed * 1000003 + chunk) & 0x7FFFFFFFFFFFFFFF)
    return torch.randn(rows, d, generator=g, device=device, dtype=torch.float32)


def _kmeans(x: torch.Tensor, k: int, iters: int, gen: torch.Generator) -> torch.Tensor:
    """Lloyd iterations from a random-row init; empty clusters re-seeded from
    the farthest points (annindex.hpp:117-126 spirit)."""
    n = x.shape[0]
    perm = torch.randperm(n, generator=gen, device="cpu")[:k].to(x.device)
    c = x[perm].clone()
    for _ in range(iters):
        d2 = (x * x).sum(1, keepdim=True) - 2.0 * x @ c.T + (c * c).sum(1)[None, :]
        best, a = d2.min(1)
        cnt = torch.bincount(a, minlength=k)
        s = torch.zeros_like(c).index_add_(0, a, x)
        nz = cnt > 0
        c[nz] = s[nz] / cnt[nz, None].to(x.dtype)
        if (~nz).any():
            far = best.topk(int((~nz).sum())).indices
            c[~nz] = x[far]
    return c


def _kmeans_batched(x: torch.Tensor, k: int, iters: int, gen: torch.Generator) -> torch.Tensor:
    """k-means for every subspace at once: x [m, n, s] -> codewords [m, k, s]."""
    m, n, s = x.shape
    perm = torch.randperm(n, generator=gen, device="cpu")[:k].to(x.device)
    c = x[:, perm, :].clone()
    for _ in range(iters):
        d2 = (x * x).sum(2, keepdim=True) - 2.0 * torch.bmm(x, c.transpose(1, 2)) + (c * c).sum(2)[:, None, :]
        best, a = d2.min(2)  # [m, n]
        for j in range(m):
            cnt = torch.bincount(a[j], minlength=k)
            sm = torch.zeros(k, s, device=x.device).index_add_(0, a[j], x[j])
            nz = cnt > 0
            c[j, nz] = sm[nz] / cnt[nz, None].to(x.dtype)
            if (~nz).any():
                far = best[j].topk(int((~nz).sum())).indices
                c[j, ~nz] = x[j, far]
    return c


def build_ivfpq(n: int, d: int, nlist: int, nsq: int, seed: int = 1, device=None, train_sample: int = 131072,
                iters: int = 10, nq: int = 64, chunk: int = 1 << 20, log=print):
    """Returns (centroids, codewords, list_off, ids, codes, queries) as numpy."""
    if device is None:
        device = "cuda" if torch.cuda.is_available() else "cpu"
    dev = torch.device(device)
    sub = d // nsq
    gen = torch.Generator(device="cpu")
    gen.manual_seed(seed)
    t0 = time.time()
    nchunks = (n + chunk - 1) // chunk
    # training sample: the first rows of the first chunks (data are i.i.d.)
    S = min(n, max(train_sample, 16 * nlist))
    parts, got, ci = [], 0, 0
    while got < S:
        rows = min(chunk, n - ci * chunk)
        x = _chunk_rows(seed, ci, rows, d, dev)
        parts.append(x[: S - got])
        got += parts[-1].shape[0]
        ci += 1
    xs = torch.cat(parts)
    cents = _kmeans(xs, nlist, iters, gen)
    c2 = (cents * cents).sum(1)
    # residual codebooks from the sample
    a = ((xs * xs).sum(1, keepdim=True) - 2.0 * xs @ cents.T + c2[None, :]).argmin(1)
    res = (xs - cents[a]).reshape(S, nsq, sub).transpose(0, 1).contiguous()
    words = _kmeans_batched(res, min(256, S), iters, gen)
    if words.shape[1] < 256:
        words = torch.cat([words, torch.zeros(nsq, 256 - words.shape[1], sub, device=dev)], 1)
    w2 = (words * words).sum(2)  # [nsq, 256]
    log(f"[fixtures] trained nlist={nlist} nsq={nsq} on {S} rows in {time.time() - t0:.1f}s ({device})")
    assign = np.empty(n, dtype=np.int64)
    codes = np.empty((n, nsq), dtype=np.uint8)
    qrng = np.random.default_rng(seed + 13)
    qrows = np.sort(qrng.choice(n, size=min(nq, n), replace=False)) if nq else np.zeros(0, np.int64)
    queries = np.zeros((len(qrows), d), dtype=np.float32)
    blk = max(1024, min(chunk, (1 << 31) // max(nlist, 256 * nsq)))  # bound the distance matrices
    for ci in range(nchunks):
        r0 = ci * chunk
        rows = min(chunk, n - r0)
        xc = _chunk_rows(seed, ci, rows, d, dev)
        for b0 in range(0, rows, blk):
            x = xc[b0:b0 + blk]
            br = x.shape[0]
            aa = ((x * x).sum(1, keepdim=True) - 2.0 * x @ cents.T + c2[None, :]).argmin(1)
            r = (x - cents[aa]).reshape(br, nsq, sub).transpose(0, 1)  # [nsq, rows, sub]
            dd = w2[:, None, :] - 2.0 * torch.bmm(r, words.transpose(1, 2))
            cc = dd.argmin(2).T.contiguous()  # [rows, nsq]
            assign[r0 + b0:r0 + b0 + br] = aa.cpu().numpy()
            codes[r0 + b0:r0 + b0 + br] = cc.to(torch.uint8).cpu().numpy()
        x = xc
        sel = qrows[(qrows >= r0) & (qrows < r0 + rows)]
        if len(sel):
            idx = np.searchsorted(qrows, sel)
            queries[idx] = x[torch.as_tensor(sel - r0, device=dev)].cpu().numpy()
    noise = np.random.default_rng(seed + 14).standard_normal(queries.shape).astype(np.float32)
    queries = (queries + np.float32(0.05) * noise).astype(np.float32)
    order = np.argsort(assign, kind="stable")  # ids ascending within each list, as train_index
    sizes = np.bincount(assign, minlength=nlist).astype(np.uint64)
    list_off = np.zeros(nlist + 1, dtype=np.uint64)
    np.cumsum(sizes, out=list_off[1:])
    ids = order.astype(np.uint64)
    codes = codes[order]
    log(f"[fixtures] encoded {n} vectors in {time.time() - t0:.1f}s; list sizes p50={int(np.median(sizes))} "
        f"p90={int(np.percentile(sizes, 90))} max={int(sizes.max())} avg={n / nlist:.0f}")
    return (cents.cpu().numpy(), words.cpu().numpy(), list_off, ids, codes, queries)


def fixture_dir() -> str:
    p = os.environ.get("PRAG_FIXTURE_DIR", "/tmp/prag_fixtures")
    os.makedirs(p, exist_ok=True)
    return p


def ensure_fixture(n: int, d: int, nlist: int, nsq: int, seed: int = 1, nq: int = 64, log=print):
    """Builds (or reuses) a PRAGIX01 fixture; returns (index_path, queries [nq, d], meta)."""
    key = f"ivfpq_n{n}_d{d}_l{nlist}_m{nsq}_s{seed}_q{nq}"
    base = os.path.join(fixture_dir(), key)
    meta_p = base + ".json"
    if os.path.exists(meta_p) and os.path.exists(base + ".pragix") and os.path.exists(base + ".q.f32"):
        with open(meta_p) as f:
            meta = json.load(f)
        q = np.fromfile(base + ".q.f32", dtype=np.float32).reshape(-1, d)
        return base + ".pragix", q, meta
    t0 = time.time()
    cents, words, list_off, ids, codes, queries = build_ivfpq(n, d, nlist, nsq, seed=seed, nq=nq, log=log)
    write_pragix(base + ".pragix", cents, words, list_off, ids, codes)
    queries.tofile(base + ".q.f32")
    sizes = np.diff(list_off.astype(np.int64))
    meta = {"n": n, "d": d, "nlist": nlist, "nsq": nsq, "seed": seed, "nq": nq,
            "list_p50": int(np.median(sizes)), "list_p90": int(np.percentile(sizes, 90)),
            "list_max": int(sizes.max()), "list_avg": n / nlist, "build_s": round(time.time() - t0, 2),
            "sha1_head": hashlib.sha1(open(base + ".pragix", "rb").read(1 << 20)).hexdigest()}
    with open(meta_p, "w") as f:
        json.dump(meta, f)
    log(f"[fixtures] wrote {base}.pragix in {time.time() - t0:.1f}s")
    return base + ".pragix", queries, meta
