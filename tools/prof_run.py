"""Workload driver for ncu: the bench.py C4 engine, prefix ingestion, then
N batches through the graph path. Never report numbers from this under
ncu; it exists so the profiler sees the same kernels bench.py times.

    python tools/prof_run.py [--prefix 120000] [--batches 20] [--recompute affected]
"""

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2603_21090_b200.config import Dims, RunConfig  # noqa: E402
from paper_2603_21090_b200.engine import IncrementalEngine  # noqa: E402
from paper_2603_21090_b200.params import init_params  # noqa: E402
from paper_2603_21090_b200.streamio import generate_stream  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prefix", type=int, default=120_000)
    ap.add_argument("--batches", type=int, default=20)
    ap.add_argument("--batch", type=int, default=600)
    ap.add_argument("--nodes", type=int, default=2_600_000)
    ap.add_argument("--recompute", default="affected")
    ap.add_argument("--rebuild", default="adaptive")
    ap.add_argument("--graph", action="store_true",
                    help="keep CUDA-graph replay (ncu cannot profile kernels of a graph "
                         "with conditional nodes; the default runs the same kernels eagerly)")
    a = ap.parse_args()
    dims = Dims(d_s=100, d_e=0, d_t=100, d_m=100, d_k=50, heads=2, layers=2)
    cfg = RunConfig(dims=dims, batch_size=a.batch, fanout=10, nodes=a.nodes, aggregator="last",
                    rebuild=a.rebuild)
    B = a.batch
    st = generate_stream(2, a.nodes, a.prefix + a.batches * B, attachment="preferential", d_e=0)
    eng = IncrementalEngine(cfg, init_params(0, dims), recompute=a.recompute)
    if not a.graph:
        eng.set_profiling(True)
    for lo in range(0, a.prefix + a.batches * B, B):
        eng.process_batch_arrays(st.src[lo:lo + B], st.dst[lo:lo + B], st.t[lo:lo + B])
    torch.cuda.synchronize()
    r = eng._rep
    print(f"done: last batch |A|={r.affected} |D|={r.direct} E_A={r.entries_affected}")


if __name__ == "__main__":
    main()
