"""TEST INFRASTRUCTURE: exact host restatement of prag::search
(annindex.hpp:277-313) for the device-built synthetic index
(prag_gpu_index_synthetic), whose codes are defined by a formula instead of a
file. Every float op is a separate IEEE fp32 numpy ufunc (no FMA), in the
reference's order: sequential folds over d (coarse), sub_dim (LUT) and the
subquantizers (ADC), then (distance, id) ordering."""
import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def fin64(z):
    z = z.astype(np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


def codes_for(seed, g, m):
    """[len(g), m] u8 code bytes of global entries g (include/prag_gpu.h)."""
    g = np.asarray(g, dtype=np.uint64)
    out = np.empty((len(g), m), dtype=np.uint8)
    with np.errstate(over="ignore"):
        for i in range(m // 8):
            w = fin64(np.uint64(seed) + np.uint64(8) * g + np.uint64(i) + GOLDEN)
            for b in range(8):
                out[:, 8 * i + b] = ((w >> np.uint64(8 * b)) & np.uint64(0xFF)).astype(np.uint8)
    return out


def fold_sq(a, b):
    """Sequential fp32 squared-L2 over the last axis (common.hpp:73-80)."""
    acc = np.zeros(np.broadcast_shapes(a.shape[:-1], b.shape[:-1]), dtype=np.float32)
    for j in range(a.shape[-1]):
        d = (a[..., j] - b[..., j]).astype(np.float32)
        acc = (acc + (d * d).astype(np.float32)).astype(np.float32)
    return acc


def search(q, cents, words, list_sizes, seed, nprobe, k):
    """(ids, dist, scanned) for one query."""
    q = np.asarray(q, np.float32)
    nlist, d = cents.shape
    m, _, sub = words.shape
    cd = fold_sq(q[None, :], cents)
    order = np.lexsort((np.arange(nlist), cd))[:nprobe]
    off = np.zeros(nlist + 1, dtype=np.uint64)
    np.cumsum(np.asarray(list_sizes, dtype=np.uint64), out=off[1:])
    all_d, all_id = [], []
    scanned = 0
    for l in order:
        n = int(off[l + 1] - off[l])
        scanned += n
        if n == 0:
            continue
        r = (q - cents[l]).astype(np.float32)
        table = fold_sq(r.reshape(m, 1, sub), words)  # [m][256]
        g = off[l] + np.arange(n, dtype=np.uint64)
        c = codes_for(seed, g, m)
        acc = np.zeros(n, dtype=np.float32)
        for s in range(m):
            acc = (acc + table[s, c[:, s]]).astype(np.float32)
        all_d.append(acc)
        all_id.append(g)
    if not all_d:
        return np.zeros(0, np.uint64), np.zeros(0, np.float32), scanned
    dd = np.concatenate(all_d)
    ii = np.concatenate(all_id)
    sel = np.lexsort((ii, dd))[:k]
    return ii[sel], dd[sel], scanned
