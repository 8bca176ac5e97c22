"""Device query embedding against the reference's own
prag::ChunkEmbedder::embed (tokendb.hpp:95-112), run through oracle/_ref/
ref_tool: bit-identical fp32 outputs."""
import os
import subprocess
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import _oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu


def _ref_embed(tmp_path, tokens, d, seed):
    tp = str(tmp_path / "tok.u32")
    op = str(tmp_path / "emb.f32")
    np.ascontiguousarray(tokens, dtype=np.uint32).tofile(tp)
    O.ref_run("embed", tp, tokens.shape[0], tokens.shape[1], d, seed, op)
    return np.fromfile(op, dtype=np.float32).reshape(tokens.shape[0], d)


@pytest.mark.parametrize("d,seed", [(384, 7), (64, 123456789), (2, 1)])
def test_gpu_embed_bit_identical_to_reference(tmp_path, d, seed):
    if not O.ref_available():
        pytest.skip("oracle/_ref/ref_tool not built")
    import paper_2403_05676_b200 as pg
    rng = np.random.default_rng(d + seed)
    m = 64
    tok = rng.integers(0, 257, (40, m)).astype(np.uint32)
    tok[0] = 0                      # all PAD -> e_0
    tok[1, :60] = 0                 # mostly PAD
    tok[2] = 7                      # one token repeated
    tok[3, ::2] = 0
    emb = pg.GpuChunkEmbedder(d, seed, vocab=257)
    got = emb.embed(tok)
    ref = _ref_embed(tmp_path, tok, d, seed)
    assert (got.view(np.uint32) == ref.view(np.uint32)).all()
    assert got[0, 0] == 1.0 and (got[0, 1:] == 0).all()


def test_gpu_embed_device_pointers_and_vocab_check(tmp_path):
    import torch
    import paper_2403_05676_b200 as pg
    emb = pg.GpuChunkEmbedder(384, 7, vocab=257)
    tok = np.random.default_rng(1).integers(0, 257, (8, 32)).astype(np.uint32)
    host = emb.embed(tok)
    dev = emb.embed(torch.from_numpy(tok.view(np.int32)).cuda())
    torch.cuda.synchronize()
    assert (dev.cpu().numpy().view(np.uint32) == host.view(np.uint32)).all()
    with pytest.raises(pg.ConfigError):
        pg.GpuChunkEmbedder(1, 7)


def test_gpu_embed_ids_beyond_vocab(tmp_path):
    """ChunkEmbedder::embed computes any id's vector on demand
    (tokendb.hpp:63-80): host token ids past the resident table embed
    bit-identically to the reference, mixed with in-table ids in one batch."""
    if not O.ref_available():
        pytest.skip("oracle/_ref/ref_tool not built")
    import paper_2403_05676_b200 as pg
    emb = pg.GpuChunkEmbedder(384, 7, vocab=257)
    tok = np.random.default_rng(2).integers(0, 257, (6, 32)).astype(np.uint32)
    tok[1, 5] = 300
    tok[2, :4] = [70000, 70000, 1 << 20, 258]  # (the reference's cache resize overflows at 2^32-1)
    tok[4, 31] = 300
    got = emb.embed(tok)
    ref = _ref_embed(tmp_path, tok, 384, 7)
    assert (got.view(np.uint32) == ref.view(np.uint32)).all()
    again = emb.embed(tok[:1])  # a later in-table call is unaffected
    assert (again.view(np.uint32) == ref[:1].view(np.uint32)).all()
