"""CPU-side checks of the C ABI library (no GPU needed): it loads, exports
every symbol include/prag_gpu.h declares, refuses to compute without a device
(no CPU fallback), and its host-only logic (shard planning, performance
model) matches the reference behaviour (test_perfmodel.cpp KATs)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2403_05676_b200 as pg
from paper_2403_05676_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(REPO, "include", "prag_gpu.h")).read()
    return sorted(set(re.findall(r"\b(prag_gpu_[a-z_]+)\s*\(", src)) - {"prag_gpu_measure_fn"})


def test_library_exports_every_header_symbol():
    L = C.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(L, s), s
    bound = {n for n, _, _ in _lib.SYMBOLS}
    assert set(syms) <= bound


def test_no_cpu_fallback_without_device(tmp_path):
    if pg.device_count() > 0:
        pytest.skip("GPU present")
    p = os.path.join(REPO, "tests", "golden", "four_points.pragix")
    with pytest.raises(pg.NoDeviceError):
        pg.GpuIndex.load(p)
    with pytest.raises(pg.NoDeviceError):
        pg.merge_topk(np.zeros((1, 1, 1), np.uint64), np.zeros((1, 1, 1), np.float32),
                      np.zeros((1, 1), np.uint32), None, 1)


def _plan_restated(sizes, world):
    """Stripe rule + LPT, restated (index_io.cpp plan_shards_lpt)."""
    sizes = [int(x) for x in sizes]
    total, nl = sum(sizes), len(sizes)
    owner = np.zeros(nl, np.uint32)
    load = [0] * world
    rest = []
    for l, n in enumerate(sizes):
        if world > 1 and n >= world * 1024 and n * nl >= 4 * total:
            owner[l] = world
            for r in range(world):
                load[r] += n * (r + 1) // world - n * r // world
        else:
            rest.append(l)
    for l in sorted(rest, key=lambda l: (-sizes[l], l)):
        r = min(range(world), key=lambda i: (load[i], i))
        owner[l] = r
        load[r] += sizes[l]
    return owner, load


def test_plan_shards_lpt():
    rng = np.random.default_rng(0)
    flat = rng.integers(0, 5000, size=1000).astype(np.uint64)  # nothing to stripe
    skew = np.minimum(rng.lognormal(7.0, 1.5, size=1000), 2e6).astype(np.uint64)
    for sizes in (flat, skew):
        for world in (1, 2, 4, 8):
            owner = pg.plan_shards(sizes, world)
            ref, load = _plan_restated(sizes, world)
            np.testing.assert_array_equal(owner, ref)
            whole = owner < world
            if sizes is flat:
                assert whole.all()
            elif world > 1:
                assert (~whole).any()  # the skewed sizes have lists to stripe
            # balance bound: max load <= mean + largest whole list
            biggest = int(sizes[whole].max()) if whole.any() else 0
            assert max(load) <= sizes.sum() / world + biggest
            # ranges: every entry of every list on exactly one rank
            cover = np.zeros(len(sizes), np.uint64)
            prev_end = np.zeros(len(sizes), np.uint64)
            for r in range(world):
                b, e = pg.plan_shard_ranges(sizes, world, r)
                assert (b <= e).all() and (e <= sizes).all()
                held = e > b
                assert (held[whole] == (owner[whole] == r)).all()
                st = ~whole
                assert (b[st] == prev_end[st]).all()  # stripes are consecutive, in rank order
                prev_end[st] = e[st]
                cover += e - b
                assert int((e - b).sum()) == load[r]
            np.testing.assert_array_equal(cover, sizes)
    with pytest.raises(pg.ConfigError):
        pg.plan_shards(flat, 0)
    with pytest.raises(pg.ConfigError):
        pg.plan_shard_ranges(flat, 2, 2)


def test_select_nprobe_kats():
    """test_perfmodel.cpp:54-68."""
    m = pg.RetrievalPerfModel(0.5e-3, 2e-3, 0.0, False)
    assert pg.select_nprobe(m, 10e-3, 1024, 0.0) == 16
    assert pg.select_nprobe(m, 10e-3, 1024) == 14
    assert pg.select_nprobe(m, 10e-3, 8, 0.0) == 8
    assert pg.select_nprobe(m, 1e-3, 1024) == 1
    assert pg.select_nprobe(m, 0.0, 1024) == 1
    assert pg.select_nprobe(pg.RetrievalPerfModel(0.0, 2e-3), 10e-3, 64) == 64


def test_select_nprobe_monotone():
    """test_perfmodel.cpp:70-79."""
    m = pg.RetrievalPerfModel(0.3e-3, 1e-3)
    prev = 0
    for b in np.arange(0.0, 50e-3 + 1e-12, 0.5e-3):
        n = pg.select_nprobe(m, float(b), 128)
        assert n >= max(prev, 1) and n <= 128
        prev = n


def test_calibrate_exact_line():
    """test_perfmodel.cpp:11-19."""
    m = pg.calibrate_retrieval(lambda n: 2e-3 + 0.5e-3 * n, [1, 2, 4, 8, 16, 32])
    assert m.slope_s == pytest.approx(0.5e-3, rel=0.01)
    assert m.intercept_s == pytest.approx(2e-3, rel=0.01)
    assert m.fit_residual_s < 1e-9 and not m.clamped
    assert m.predict(10) == pytest.approx(7e-3)


def test_calibrate_median_robust():
    """test_perfmodel.cpp:21-32."""
    calls = [0]

    def timer(n):
        calls[0] += 1
        t = 1e-3 * n
        if calls[0] % 5 == 0:
            t += 50e-3
        return t
    m = pg.calibrate_retrieval(timer, [1, 2, 4, 8], 5)
    assert m.slope_s == pytest.approx(1e-3, rel=0.05)


def test_calibrate_clamp_and_validation():
    """test_perfmodel.cpp:34-52."""
    m = pg.calibrate_retrieval(lambda n: 5e-3, [1, 4, 16])
    assert abs(m.slope_s) < 1e-12 and m.intercept_s == pytest.approx(5e-3) and not m.clamped
    m = pg.calibrate_retrieval(lambda n: 10e-3 - 0.1e-3 * n, [1, 4, 16])
    assert m.slope_s == 0.0 and m.clamped
    with pytest.raises(pg.ConfigError):
        pg.calibrate_retrieval(lambda n: 1e-3, [4])
    with pytest.raises(pg.ConfigError):
        pg.calibrate_retrieval(lambda n: 1e-3, [4, 4, 4])
    with pytest.raises(pg.ConfigError):
        pg.calibrate_retrieval(lambda n: 1e-3, [1, 2], 2)


def test_perf_model_json_roundtrip(tmp_path):
    """perfmodel.hpp:190-223 schema (clamped not serialised)."""
    m = pg.RetrievalPerfModel(1.25e-4, 3e-5, 1e-6, True)
    p = str(tmp_path / "perf.json")
    pg.store_perf_model(m, p)
    back = pg.load_perf_model(p)
    assert (back.slope_s, back.intercept_s, back.fit_residual_s) == (m.slope_s, m.intercept_s, m.fit_residual_s)
    assert back.clamped is False
    with pytest.raises(pg.FormatError):
        pg.load_perf_model(str(tmp_path / "missing.json"))


def test_no_fma_contraction_in_sass():
    """Exactness guard: the reference folds are
    separately rounded mul/add; no kernel may contract them into FFMA. The
    only fused op allowed is the scan's explicit FFMA2 with 0/1 masks
    (x*1 + acc == acc + x exactly). coarse_tc_kernel is exempt: it computes
    the approximate GEMM-form pre-filter and its error bound; the exact
    distances that decide the probe order come from select_window_kernel.
    decode_part_kernel is the config-E generator stand-in, not retrieval.
    embed_kernel's only fused ops are inside the correctly rounded IEEE
    double division / square root sequences (__ddiv_rn, __dsqrt_rn)."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([exe, "-sass", _lib.LIB_PATH], capture_output=True, text=True, check=True).stdout
    func = None
    ffma2_funcs = set()
    for line in sass.splitlines():
        if "Function :" in line:
            func = line.split("Function :")[1].strip()
        toks = line.split()
        if any(t == "FFMA" or t.startswith("FFMA.") for t in toks) and not any(
                x in (func or "") for x in ("coarse_tc_kernel", "decode_part_kernel", "embed_kernel",
                                            "centroid_kernel")):
            raise AssertionError(f"FFMA in {func}: {line.strip()}")
        if any(t.startswith("FFMA2") for t in toks):
            ffma2_funcs.add(func)
    # FFMA2 only as the 0/1-masked fold step of the skewed scan (K3 and the
    # batch-1 kernel, which share it: skew_common.cuh)
    assert ffma2_funcs and all("scan_skew_kernel" in f or "search1_kernel" in f for f in ffma2_funcs), ffma2_funcs


def test_headers_compile_standalone(tmp_path):
    """The boundary headers stand alone: prag_gpu.h as C99 (any FFI's view),
    prag_gpu.hpp as C++17 without the reference tree, and a program linking
    libprag_gpu.so runs (no GPU needed for prag_gpu_device_count)."""
    import shutil
    import subprocess
    inc = os.path.join(REPO, "include")
    if not shutil.which("gcc") or not shutil.which("g++"):
        pytest.skip("no host compiler")
    c = tmp_path / "t.c"
    c.write_text('#include "prag_gpu.h"\nint f(void) { prag_gpu_train_params p = {0}; (void)p;'
                 ' return prag_gpu_version(); }\n')
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I" + inc, "-c", str(c), "-o", str(tmp_path / "t.o")],
                   check=True)
    cpp = tmp_path / "t.cpp"
    cpp.write_text('#include "prag_gpu.hpp"\nint main() { prag::gpu::SearchParams p; p.nprobe = 4; (void)p;'
                   ' return prag_gpu_device_count() >= 0 ? 0 : 1; }\n')
    libdir = os.path.dirname(_lib.LIB_PATH)
    exe = tmp_path / "t"
    subprocess.run(["g++", "-std=c++17", "-Wall", "-Wextra", "-Werror", "-DPRAG_GPU_NO_REFERENCE", "-I" + inc,
                    str(cpp), "-L" + libdir, "-lprag_gpu", "-Wl,-rpath," + libdir, "-o", str(exe)], check=True)
    assert subprocess.run([str(exe)]).returncode == 0
