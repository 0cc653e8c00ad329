"""bench.py's roofline accounting against SURVEY.md §8d's per-unit figure:
one C4 node with E = 10 ring entries is 9,360 algorithmic bytes
(4·[d + E·(K·d + d_e) + K·d] + E·16) plus 16 B of ring meta per row."""

import importlib.util
import os

from paper_2603_21090_b200.config import Dims

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_recompute_bytes_matches_survey_per_node_figure():
    b = _bench()
    g = Dims(d_s=100, d_e=0, d_t=100, d_m=100, d_k=50, heads=2, layers=2)
    assert b.recompute_bytes(g, 1, 10) == 9360 + 16
    # linear in rows and entries; the time-basis flag does not change the count
    assert b.recompute_bytes(g, 3, 25, time_basis=True) == 3 * 1216 + 25 * 816


def test_recompute_flops_folded_formulation():
    b = _bench()
    g = Dims(d_s=100, d_e=0, d_t=100, d_m=100, d_k=50, heads=2, layers=2)
    # per node and layer: q (200x100), q~ (2 x 50x200), c (2 x 200x50), out (100x100) MACs
    per_node_l = 2 * (200 * 100 + 100 * 200 + 2 * 200 * 50 + 100 * 100)
    per_entry_l = 2 * (2 * 2 * 200)
    assert b.recompute_flops(g, 1, 10) == 2 * (per_node_l + 10 * per_entry_l)
