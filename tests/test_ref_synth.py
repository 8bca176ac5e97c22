"""The reference-arm driver for the device-built synthetic index (configs C/D):
oracle/_ref/ref_tool synth-search rebuilds it as the reference's own
IvfIndex/PqCodebook and runs the unmodified prag::search; it must equal the
exact host restatement tests/_synth_ref.py (the formula the GPU builds from)."""
import os
import struct
import subprocess

import numpy as np
import pytest

import _synth_ref as R

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(REPO, "oracle", "_ref", "ref_tool")


def _read_results(path, nq, k):
    out = []
    with open(path, "rb") as f:
        for _ in range(nq):
            cnt, _sl, sc = struct.unpack("<IIQ", f.read(16))
            rec = np.frombuffer(f.read(12 * k), dtype=[("id", "<u8"), ("d", "<f4")])
            out.append((rec["id"][:cnt].copy(), rec["d"][:cnt].copy(), sc))
    return out


@pytest.mark.skipif(not os.path.exists(TOOL), reason="oracle/_ref/ref_tool not built (needs /root/reference)")
@pytest.mark.parametrize("m", [32, 64])
def test_ref_tool_synth_search_equals_restatement(tmp_path, m):
    rng = np.random.default_rng(3 + m)
    nlist, d, seed = 24, 128, 77 + m
    cents = rng.standard_normal((nlist, d)).astype(np.float32)
    words = (rng.standard_normal((m, 256, d // m)) * 0.3).astype(np.float32)
    sizes = rng.integers(0, 400, nlist).astype(np.uint64)
    sizes[3] = 0
    q = (cents[rng.integers(0, nlist, 5)] + rng.standard_normal((5, d)).astype(np.float32) * 0.5).astype(np.float32)
    for name, arr in (("c", cents), ("w", words), ("s", sizes), ("q", q)):
        arr.tofile(tmp_path / f"{name}.bin")
    for nprobe, k in ((1, 10), (6, 7), (24, 32)):
        outp = tmp_path / "out.bin"
        subprocess.run([TOOL, "synth-search", str(tmp_path / "c.bin"), str(tmp_path / "w.bin"), str(tmp_path / "s.bin"),
                        str(nlist), str(d), str(m), str(seed), str(tmp_path / "q.bin"), "5", str(nprobe), str(k),
                        str(outp)], check=True)
        got = _read_results(outp, 5, k)
        for i in range(5):
            ids, dist, sc = R.search(q[i], cents, words, sizes, seed, nprobe, k)
            gi, gd, gs = got[i]
            assert gs == sc
            np.testing.assert_array_equal(gi, ids)
            np.testing.assert_array_equal(gd.view(np.uint32), dist.view(np.uint32))
