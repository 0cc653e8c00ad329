"""DySAT at 1M nodes: a few batches and full recomputes (for ncu launch lists)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_21090_b200.dysat import DySATConfig, DySATEngine, init_dysat_params  # noqa: E402
from paper_2603_21090_b200.streamio import generate_stream  # noqa: E402

n, m = 1_000_000, 30_000
st = generate_stream(5, n, m, attachment="preferential", d_e=0)
cfg = DySATConfig(n=n, d_in=64, d=128, heads_s=16, heads_t=16, window=8, fanout=20,
                  snapshot_len=1e9, max_snapshots=16, batch_size=600)
eng = DySATEngine(cfg, init_dysat_params(0, cfg))
for lo in range(0, 6000, 600):
    eng.process_batch_arrays(st.src[lo:lo + 600], st.dst[lo:lo + 600], st.t[lo:lo + 600])
eng.full_recompute()
torch.cuda.synchronize()
print("ok", eng.snapshot)
