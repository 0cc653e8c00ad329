"""Workload driver for ncu: the bench.py C4 engine fast-forwarded through the
stream (graph replay: ncu cannot see kernels of a graph with conditional
nodes, so the fast-forward is not profiled), then N batches run eagerly
(profiling mode: the same kernels, one launch each) for ncu to capture.
Never report numbers from this under ncu.

    python tools/prof_run.py [--edges 30000000] [--batches 20] [--recompute affected]
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2603_21090_b200.config import Dims, RunConfig  # noqa: E402
from paper_2603_21090_b200.engine import IncrementalEngine  # noqa: E402
from paper_2603_21090_b200.feeder import DeviceStream  # noqa: E402
from paper_2603_21090_b200.params import init_params  # noqa: E402
from paper_2603_21090_b200.streamio import generate_stream  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--edges", type=int, default=30_000_000, help="fast-forward length")
    ap.add_argument("--batches", type=int, default=20)
    ap.add_argument("--batch", type=int, default=600)
    ap.add_argument("--nodes", type=int, default=2_600_000)
    ap.add_argument("--recompute", default="affected")
    ap.add_argument("--rebuild", default="adaptive")
    a = ap.parse_args()
    dims = Dims(d_s=100, d_e=0, d_t=100, d_m=100, d_k=50, heads=2, layers=2)
    cfg = RunConfig(dims=dims, batch_size=a.batch, fanout=10, nodes=a.nodes, aggregator="last",
                    rebuild=a.rebuild)
    B = a.batch
    n = a.edges + a.batches * B
    st = generate_stream(2, a.nodes, n, attachment="preferential", d_e=0)
    eng = IncrementalEngine(cfg, init_params(0, dims), recompute=a.recompute)
    eng.reserve(nodes=a.nodes, edges=n + B, batch=B, batches=n // B + 8)
    DeviceStream(eng, st, B, 0, a.edges).run()
    torch.cuda.synchronize()
    eng.set_profiling(True)
    torch.cuda.profiler.start()  # ncu --profile-from-start off captures from here
    for lo in range(a.edges, n, B):
        eng.process_batch_arrays(st.src[lo:lo + B], st.dst[lo:lo + B], st.t[lo:lo + B])
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    r = eng._rep
    print(f"done: last batch |A|={r.affected} |D|={r.direct} E_A={r.entries_affected}")


if __name__ == "__main__":
    main()
