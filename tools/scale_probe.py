"""Probe: batch time and |A| as the C4 stream grows to 30M edges (B200).

    python tools/scale_probe.py [--edges 30000000] [--batch 600] [--every 2000]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_21090_b200.config import Dims, RunConfig  # noqa: E402
from paper_2603_21090_b200.engine import IncrementalEngine  # noqa: E402
from paper_2603_21090_b200.params import init_params  # noqa: E402
from paper_2603_21090_b200.streamio import generate_stream  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--edges", type=int, default=30_000_000)
    ap.add_argument("--batch", type=int, default=600)
    ap.add_argument("--every", type=int, default=2000)
    ap.add_argument("--nodes", type=int, default=2_600_000)
    ap.add_argument("--recompute", default="affected")
    a = ap.parse_args()
    B = a.batch
    t0 = time.time()
    st = generate_stream(2, a.nodes, a.edges, attachment="preferential", d_e=0)
    print(f"generated {a.edges} edges in {time.time() - t0:.1f}s", flush=True)
    dims = Dims(d_s=100, d_e=0, d_t=100, d_m=100, d_k=50, heads=2, layers=2)
    cfg = RunConfig(dims=dims, batch_size=B, fanout=10, nodes=a.nodes, aggregator="last",
                    rebuild="adaptive")
    eng = IncrementalEngine(cfg, init_params(0, dims), recompute=a.recompute)
    nb = a.edges // B
    eng.reserve(nodes=a.nodes, edges=a.edges + B, batch=B, batches=nb + 8)
    dev = eng.device
    src = torch.tensor(st.src.astype(np.int32), device=dev)
    dst = torch.tensor(st.dst.astype(np.int32), device=dev)
    ts = torch.tensor(st.t, device=dev)
    stream = torch.cuda.current_stream(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    t_wall = time.time()
    ev0.record(stream)
    lo_chunk = 0
    for b in range(nb):
        lo, hi = b * B, (b + 1) * B
        last = (b + 1) % a.every == 0 or b == nb - 1
        eng.process_batch_device(src[lo:hi], dst[lo:hi], ts[lo:hi],
                                 max_id=int(max(st.src[lo:hi].max(), st.dst[lo:hi].max())),
                                 t_first=float(st.t[lo]), t_last=float(st.t[hi - 1]),
                                 report=last)
        if last:
            ev1.record(stream)
            torch.cuda.synchronize()
            ms = ev0.elapsed_time(ev1) / (b + 1 - lo_chunk)
            r = eng._rep
            print(f"m={hi:>9} batch_ms={ms:.3f} |A|={r.affected} |D|={r.direct} "
                  f"E_A={r.entries_affected} rebuild={r.rebuild_kind}/{r.rebuild_nodes} "
                  f"cum={r.cum_count} drift={r.global_drift:.3f}", flush=True)
            lo_chunk = b + 1
            ev0.record(stream)
    print(f"wall {time.time() - t_wall:.1f}s", flush=True)


if __name__ == "__main__":
    main()
