"""The retrieval service on the GPU:
prag::gpu::GpuRetrievalService (include/prag_gpu_service.hpp) against the
reference prag::RetrievalService (service.hpp:243-362) over loopback TCP with
the reference RetrievalClient: identical responses sequentially and under
concurrent clients (batched on the GPU), identical error frames. Built from
tests/cpp/service_dropin.cpp by oracle/Makefile (needs /root/reference at
build time; the prebuilt binary travels to the box)."""
import os
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(REPO, "oracle", "_ref", "service_dropin")

pytestmark = pytest.mark.gpu


def test_gpu_retrieval_service_is_a_drop_in():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/service_dropin not built (needs /root/reference at build time)")
    r = subprocess.run([BIN, "60", "8", "40"], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASS" in r.stdout
