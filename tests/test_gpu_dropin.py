"""The C++ drop-in boundary on the GPU: prag::gpu::GpuRetriever (include/
prag_gpu.hpp) swapped in for the reference prag::LocalRetriever
(pipeline.hpp:213-249) on the same objects must give identical
RetrievalOutcomes. The binary is built from tests/cpp/retriever_dropin.cpp
against the unmodified reference headers by oracle/Makefile (it needs
/root/reference at build time, so the prebuilt copy travels to the box)."""
import os
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(REPO, "oracle", "_ref", "retriever_dropin")

pytestmark = pytest.mark.gpu


def test_gpu_retriever_is_a_drop_in_for_local_retriever():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/retriever_dropin not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASS" in r.stdout
