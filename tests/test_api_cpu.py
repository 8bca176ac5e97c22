"""Host-side API mirrors that need no GPU: recall_at_k (annindex.hpp:317-327),
TrainParams defaults (annindex.hpp:152-160), SearchParams defaults
(annindex.hpp:35-39)."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import paper_2403_05676_b200 as pg  # noqa: E402


def _res(ids):
    return pg.SearchResult([pg.ScoredId(i, float(n)) for n, i in enumerate(ids)], len(ids), 1)


def test_recall_at_k_matches_reference_definition():
    assert pg.recall_at_k(_res([1, 2]), _res([])) == 1.0          # empty exact set
    assert pg.recall_at_k(_res([]), _res([3, 4])) == 0.0
    assert pg.recall_at_k(_res([4, 9, 3]), _res([3, 4])) == 1.0
    assert pg.recall_at_k(_res([4, 7]), _res([3, 4])) == 0.5
    # each exact neighbour counts once even if the approx list repeats it
    assert pg.recall_at_k(_res([4, 4]), _res([4, 5])) == 0.5


def test_param_defaults_follow_the_reference():
    t = pg.TrainParams()
    assert (t.nlist, t.n_subquantizers, t.seed, t.kmeans_iterations, t.train_sample_cap) == (64, 0, 7, 25, 32768)
    p = pg.SearchParams()
    assert (p.nprobe, p.k, p.exact_rerank) == (1, 2, False)
