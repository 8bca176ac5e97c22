"""The fast path's pool selection under large pools: many small work items
per CTA (PRAG_GPU_ITEMS_PER_CTA, read once when the library loads, hence a
subprocess) give each query up to hundreds of item lists, so the selection
runs its threshold pass with many survivors, the register radix select and
the multi-pass fallback. Must equal the oracle bit for bit."""
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("items_per_cta", [1, 48])
def test_pool_selection_paths_match_oracle(items_per_cta, tmp_path):
    env = dict(os.environ, PRAG_GPU_ITEMS_PER_CTA=str(items_per_cta))
    r = subprocess.run([sys.executable, os.path.join(HERE, "_pool_paths_check.py"), str(tmp_path)], env=env,
                       capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
