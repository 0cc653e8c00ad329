#!/usr/bin/env python
"""Headline benchmark: streamed edges/s and p50/p99 batch latency of the
StreamTGN exact-mode incremental path (2-layer TGN, 2.6M nodes), B200.

Workload (BASELINE.json metric; SURVEY.md §8d config C4 at B=600):
  dims d_s=d_m=d_t=100, d_k=50, H=2, K=2, d_e=0, L=10, aggregator last,
  drift-aware rebuild (adaptive, gamma=0.9, delta_max=0.5, alpha=0.1),
  init_params(0), synthetic preferential power-law stream
  generate_stream(seed=2, n=2.6M, m=30M) (the reference's generator, same
  edges, replayed natively). The engine fast-forwards through the stream
  (device-resident batches, one graph replay each) and times the LAST
  batches of the 30M-edge stream: W warm-up, K timed, then the e2e leg and
  the per-stage profile. On the way it also times 100 batches right after
  the first 120K edges: the window the CPU reference is timed on
  ("window"); at the end it sweeps the batch size over 100..10K ("sweep").

One JSON line (rank 0). `value` = device-timed throughput with inputs
already in HBM (CUDA events on the engine stream, max over ranks);
`e2e` = the same metric through the public host-buffer API
(process_batch_arrays: H2D of the batch + D2H of the scores per step).
Inputs are larger than L2 (26 GB of resident state; a batch at the end of
the stream touches ~1 GB of rings), so no explicit flush.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "streamed edges/sec and p50/p99 batch latency (2-layer TGN, 2.6M nodes)"
UNIT = "edges/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=600)
    ap.add_argument("--nodes", type=int, default=2_600_000)
    ap.add_argument("--edges", type=int, default=30_000_000,
                    help="stream length; the timed batches are the last ones of it")
    ap.add_argument("--prefix", type=int, default=120_000,
                    help="CPU-reference window: edges fast-forwarded before its timed batches")
    ap.add_argument("--window-steps", type=int, default=100)
    ap.add_argument("--sweep", default="100,300,1000,3000,10000")
    ap.add_argument("--sweep-steps", type=int, default=30)
    ap.add_argument("--no-rebuild-leg", action="store_true")
    ap.add_argument("--no-direct-leg", action="store_true")
    ap.add_argument("--seed", type=int, default=2)
    ap.add_argument("--rebuild", default="adaptive")
    ap.add_argument("--recompute", default="affected", choices=["affected", "direct"])
    ap.add_argument("--cpu-batches", type=int, default=6)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-batches", type=int, default=20)
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--config-legs", default="C1,C2,C3,C5",
                    help="other BASELINE.json configs to run after the C4 legs ('' = none)")
    ap.add_argument("--c3-edges", type=int, default=30_000_000)
    ap.add_argument("--latency-steps", type=int, default=1000,
                    help="device-timed batches of the end-of-stream latency leg (p50/p99)")
    return ap.parse_args()


def workload(args):
    from paper_2603_21090_b200.config import Dims, RunConfig
    from paper_2603_21090_b200.params import init_params
    dims = Dims(d_s=100, d_e=0, d_t=100, d_x=0, d_m=100, d_k=50, heads=2, layers=2)
    cfg = RunConfig(dims=dims, batch_size=args.batch, fanout=10, nodes=args.nodes,
                    aggregator="last", rebuild=args.rebuild, gamma=0.9, delta_max=0.5,
                    alpha=0.1, seed=0)
    return dims, cfg, init_params(0, dims)


def config_json(args, n_gpus):
    """The workload (identical in both arms); where in the stream each arm's timed
    batches sit is reported beside it under "timed_batches"."""
    return {"workload": "C4: TGN 2-layer exact-mode incremental inference, synthetic "
                        "preferential power-law stream, drift-aware rebuild",
            "nodes": args.nodes, "batch_edges": args.batch, "fanout_L": 10, "layers_K": 2,
            "d_memory": 100, "d_time": 100, "heads": 2, "d_k": 50, "d_edge": 0,
            "edges": args.edges,
            "stream": f"generate_stream(seed={args.seed}, n={args.nodes}, m={args.edges}, "
                      f"preferential, d_e=0)",
            "rebuild": args.rebuild, "recompute": args.recompute,
            "parallelism": f"replicas{n_gpus}" if n_gpus > 1 else "single",
            "l2": "inputs larger than L2 (26 GB resident state), no flush"}


def make_stream(args, n_edges, rank):
    """The C4 stream. Every rank replays the same stream (replicas of one serving
    engine, weak scaling): the sharded full-rebuild leg all-gathers rows across
    ranks and needs identical replicas (`rank` is kept for the call sites)."""
    from paper_2603_21090_b200.streamio import generate_stream
    return generate_stream(args.seed, args.nodes, n_edges, attachment="preferential",
                           d_e=0)


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.tmp = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=self.tmp, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.tmp.flush()
        rows = []
        with open(self.tmp.name) as fh:
            for line in fh:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.tmp.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({nm for r in rows for nm, v in zip(names, r[5:9]) if v == "Active"})
        busy = [x for x in sm if x > 0.5 * mx] or sm
        return {"sm_mhz": float(np.median(busy)), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


# ---------------------------------------------------------------------------
REF_PKG = os.path.join(ROOT, "baseline", "_ref")


def stock_reference():
    """The unmodified reference package installed in baseline/_ref (pip --target of
    /root/reference/pkg), or None when it is not installed there."""
    if not os.path.isdir(os.path.join(REF_PKG, "streamtgn")):
        return None
    os.environ.setdefault("STREAMTGN_NUMBA", "1")
    if REF_PKG not in sys.path:
        sys.path.insert(0, REF_PKG)
    import streamtgn
    from streamtgn import engine, kernels, params, streamio
    from streamtgn import config as rconfig
    assert os.path.dirname(streamtgn.__file__).startswith(REF_PKG), streamtgn.__file__
    return {"engine": engine, "kernels": kernels, "params": params, "streamio": streamio,
            "config": rconfig}


def _zero_pipeline(qbase, offsets, payload, feat, dt, omega, phi0, wq, wk, wv, wo):
    """Shape-correct zero outputs of pipeline_many: the fast-forward to the timed
    stream position skips the attention arithmetic (topology, caches, memory and
    drift still advance through the stock code); the timed batches run the stock
    kernel."""
    N, d, E = qbase.shape[0], qbase.shape[1], payload.shape[0]
    K, H, _, d_k = wq.shape
    return (np.zeros((N, K, d)), np.zeros((E, K, H)), np.zeros((E, K, H, d_k)),
            np.full((N, K, H), -np.inf), np.zeros((N, K, H)), np.zeros((N, K, H, d_k)))


def cpu_reference(args, B_count, warmup=1):
    """Time the reference CPU path on the host: the stock reference from
    baseline/_ref (IncrementalEngine.process_batch, numba backend) when it is
    installed, else the oracle port (oracle/, bitwise-pinned to the reference).
    Both fast-forward the first `args.prefix` edges of the same stream, run
    `warmup` untimed full batches, then time B_count full batches.
    Returns (edges/s, per-batch seconds, sample description, kind)."""
    B = args.batch
    m = args.prefix + (warmup + B_count) * B
    ref = stock_reference()
    if ref is not None:
        rc = ref["config"]
        dims = rc.Dims(d_s=100, d_e=0, d_t=100, d_x=0, d_m=100, d_k=50, heads=2, layers=2)
        cfg = rc.RunConfig(dims=dims, batch_size=B, fanout=10, nodes=args.nodes,
                           aggregator="last", rebuild=args.rebuild, gamma=0.9, delta_max=0.5,
                           alpha=0.1, seed=0)
        params = ref["params"].init_params(0, dims)
        edges = ref["streamio"].generate_stream(args.seed, args.nodes, m,
                                                attachment="preferential", d_e=0)
        eng = ref["engine"].IncrementalEngine(cfg, params)
        kern = ref["kernels"]
        stock = kern.pipeline_many
        kern.pipeline_many = _zero_pipeline
        try:
            for lo in range(0, args.prefix, B):
                eng.process_batch(edges[lo:lo + B])
        finally:
            kern.pipeline_many = stock
        step = lambda lo: eng.process_batch(edges[lo:lo + B])  # noqa: E731
        what = ("stock reference streamtgn.engine.IncrementalEngine.process_batch from "
                "baseline/_ref (float64, numba backend, 1 thread)")
        kind = "reference"
    else:
        from oracle.stgn_oracle import Oracle
        dims, cfg, params = workload(args)
        st = make_stream(args, m, 0)
        orc = Oracle(cfg, params)
        for lo in range(0, args.prefix, B):
            orc.process_batch(st.src[lo:lo + B], st.dst[lo:lo + B], st.t[lo:lo + B],
                              st.feat[lo:lo + B], compute=False)
        step = lambda lo: orc.process_batch(st.src[lo:lo + B], st.dst[lo:lo + B],  # noqa: E731
                                            st.t[lo:lo + B], st.feat[lo:lo + B])
        what = "oracle port (float64 numpy+numba, 1 thread; baseline/_ref not installed)"
        kind = "port"
    for k in range(warmup):  # untimed full batches (numba compile, caches)
        step(args.prefix + k * B)
    times = []
    for k in range(warmup, warmup + B_count):
        t0 = time.perf_counter()
        step(args.prefix + k * B)
        times.append(time.perf_counter() - t0)
    times = np.array(times)
    k0 = args.prefix // B + warmup
    sample = (f"{what} on batches {k0}..{k0 + B_count - 1} of the same stream ({B_count} x {B} "
              f"edges) after a fast-forward through the first {args.prefix} edges (attention "
              f"arithmetic skipped there, state advanced by the same code) and {warmup} untimed "
              f"batches. Bounded sample: the CPU path takes ~1.5 s per batch here and would need "
              f"~96 GB for the 30M-edge payload store; at the end of the stream its per-batch "
              f"work (|A|) is ~25x larger, so this sample overstates the CPU's throughput there")
    return B_count * B / float(times.sum()), times, sample, kind


def timed_position(args, pos0=None):
    if pos0 is None:
        return (f"bounded CPU sample: batches right after the first {args.prefix} edges of the "
                f"stream (the GPU arm reports this same position as its 'window' leg)")
    return (f"the last batches of the {args.edges}-edge stream, after {pos0} edges are ingested "
            f"(the 'window' leg times the position right after the first {args.prefix} edges)")


def run_reference(args, world, rank):
    if rank != 0:
        return
    # one step = one 600-edge batch of the reference on the host (~1-2 s each); capped so the
    # whole run (fast-forward ~1 min + warm-up + steps) stays within a few minutes
    steps = max(1, min(args.steps, 30))
    warm = max(1, min(args.warmup, 5))
    value, times, sample, kind = cpu_reference(args, steps, warmup=warm)
    ms = float(times.mean() * 1e3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
        "warmup": warm, "ms_per_step": ms, "p50_ms": float(np.percentile(times, 50) * 1e3),
        "p99_ms": float(np.percentile(times, 99) * 1e3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_json(args, world), "impl": "reference",
        "timed_batches": timed_position(args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": kind,
                         "sample": sample, "host_nproc": os.cpu_count()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# BASELINE.json configs other than the headline C4; CPU figures are the
# reference's own process_batch measured in this container
CONFIGS = {
    "C1": dict(desc="TGN 1-layer, Wikipedia-shaped stream", nodes=9_227, edges=157_474, d_e=172,
               layers=1, batch=200, seed=0, memoryless=False,
               cpu_ref={"p50_ms": 796.0, "p99_ms": 1348.0, "edges_per_s": 267,
                        "window": "first 20K edges", "full_stream_edges_per_s": 78}),
    "C2": dict(desc="TGN 2-layer, Reddit-shaped stream", nodes=10_985, edges=672_447, d_e=172,
               layers=2, batch=600, seed=1, memoryless=False,
               cpu_ref={"p50_ms": 5462.0, "p99_ms": 10464.0, "edges_per_s": 115,
                        "window": "first 30K edges"}),
    "C3": dict(desc="TGAT 2-layer (memoryless: GRU tensors zeroed), power-law 2.6M nodes",
               nodes=2_600_000, edges=None, d_e=0, layers=2, batch=600, seed=2, memoryless=True,
               cpu_ref=None),
}


def config_legs(args, torch, dev):
    """Each config on its own engine: the whole stream fed from HBM, one CUDA event per
    batch (C1, C2: every batch of the stream is timed; C3: the last 1,000 batches of a
    --c3-edges stream after a device fast-forward). Mean/max |A| of C1/C2 come from an
    untimed replay on a second engine that reports every batch."""
    from paper_2603_21090_b200.config import Dims, RunConfig
    from paper_2603_21090_b200.engine import IncrementalEngine
    from paper_2603_21090_b200.feeder import DeviceStream
    from paper_2603_21090_b200.params import init_params, memoryless
    from paper_2603_21090_b200.streamio import generate_stream
    out = {}
    for name in [c for c in args.config_legs.split(",") if c and c != "C5"]:
        c = CONFIGS[name]
        m = c["edges"] or args.c3_edges
        dims = Dims(d_s=100, d_e=c["d_e"], d_t=100, d_x=0, d_m=100, d_k=50, heads=2,
                    layers=c["layers"])
        cfg = RunConfig(dims=dims, batch_size=c["batch"], fanout=10, nodes=c["nodes"],
                        aggregator="last", rebuild="adaptive", gamma=0.9, delta_max=0.5,
                        alpha=0.1)
        params = init_params(0, dims)
        if c["memoryless"]:
            memoryless(params)
        t0 = time.perf_counter()
        st = generate_stream(c["seed"], c["nodes"], m, attachment="preferential", d_e=c["d_e"])
        t_gen = time.perf_counter() - t0
        B = c["batch"]

        def fresh():
            e = IncrementalEngine(cfg, params)
            e.reserve(nodes=c["nodes"], edges=m + B, batch=B, batches=m // B + 8)
            return e
        eng = fresh()
        stream = torch.cuda.current_stream(dev)
        nb = -(-m // B)
        if c["edges"] is None:   # C3: fast-forward, then the last 1,000 batches
            k_t = max(0, nb - 1000)
            feed = DeviceStream(eng, st, B)
            feed.run(0, k_t, report_last=True)
            a_start = int(eng._rep.affected)
        else:
            k_t = 0
            feed = DeviceStream(eng, st, B)
        # warm-up: C1/C2 time the whole stream from an empty graph, so the CUDA graph is
        # captured on a throwaway engine first (same dims, same max batch)
        if k_t == 0:
            w_eng = fresh()
            DeviceStream(w_eng, st, B, 0, 3 * B).run(0, 3, report_last=True)
            w_eng.sync()
            del w_eng
        ms, per = _timed_batches(torch, stream, feed, k_t, nb - k_t)
        eng.sync()
        n_t = m - k_t * B
        leg = {"workload": c["desc"], "nodes": c["nodes"], "edges": m, "d_edge": c["d_e"],
               "layers_K": c["layers"], "batch_edges": B, "timed_batches": nb - k_t,
               "timed_edges": n_t, "value": n_t / (ms / 1e3), "unit": UNIT,
               "p50_ms": float(np.percentile(per, 50)), "p99_ms": float(np.percentile(per, 99)),
               "generate_s": t_gen, "recompute_kernel": "bf16x3" if eng.info()["bf16x3"] else
               ("split-tf32" if eng.info()["tensor_cores"] else "ffma"),
               "memory_kernel": "bf16x3" if eng.info()["memory_bf16x3"] else "ffma",
               "cpu_reference": c["cpu_ref"]}
        if c["edges"] is not None:
            rep = fresh()
            rf = DeviceStream(rep, st, B)
            aff = []
            for k in range(nb):
                rf.batch(k, report=True)
                aff.append(int(rep._rep.affected))
            aff = np.array(aff)
            leg["affected_mean"] = float(aff.mean())
            leg["affected_max"] = int(aff.max())
            leg["affected_frac_mean"] = float(aff.mean() / c["nodes"])
            del rep, rf
        else:
            leg["affected_at_window_start"] = a_start
            leg["affected_frac_at_window_start"] = a_start / c["nodes"]
            leg["timed_position"] = f"edges {k_t * B}..{m} (the end of the stream)"
        out[name] = leg
        del feed, eng, st
        torch.cuda.empty_cache()
    return out


def dysat_leg(torch, dev, n=1_000_000, m=3_000_000, B=600, snapshots=10):
    """configs[4]: DySAT incremental inference on a 1M-node synthetic snapshot stream vs full
    recompute (paper_2603_21090_b200/dysat.py; the reference has no DySAT code, so there is no
    reference number and parity is pinned only to oracle/dysat_oracle.py). The whole stream is
    fed from HBM in B-edge batches split at snapshot boundaries, one CUDA event per batch; a
    batch that crosses a boundary includes the O(|V|) roll (every node recomputed)."""
    from paper_2603_21090_b200.dysat import DySATConfig, DySATEngine, init_dysat_params
    from paper_2603_21090_b200.streamio import generate_stream
    st = generate_stream(5, n, m, attachment="preferential", d_e=0)
    span = float(st.t[-1]) + 1.0
    cfg = DySATConfig(n=n, d_in=64, d=128, heads_s=16, heads_t=16, window=8, fanout=20,
                      snapshot_len=span / snapshots, max_snapshots=snapshots + 2, batch_size=B)
    eng = DySATEngine(cfg, init_dysat_params(0, cfg))
    src = torch.from_numpy(st.src.astype(np.int32)).to(dev)
    dst = torch.from_numpy(st.dst.astype(np.int32)).to(dev)
    snap = np.floor(st.t / cfg.snapshot_len).astype(np.int64)
    segs = []   # (lo, hi, snapshot) batches of at most B edges inside one snapshot
    lo = 0
    while lo < m:
        hi = min(lo + B, m)
        k = int(snap[lo])
        hi = lo + int(np.searchsorted(snap[lo:hi], k, side="right"))
        segs.append((lo, hi, k))
        lo = hi
    stream = torch.cuda.current_stream(dev)
    for lo, hi, k in segs[:3]:   # warm-up (snapshot 0 batches; re-run below from a fresh engine)
        eng.process_batch_device(src[lo:hi], dst[lo:hi], float(st.t[hi - 1]), k)
    torch.cuda.synchronize()
    del eng
    eng = DySATEngine(cfg, init_dysat_params(0, cfg))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(segs) + 1)]
    rolls = []
    torch.cuda.synchronize()
    ev[0].record(stream)
    for q, (lo, hi, k) in enumerate(segs):
        if k > eng.snapshot:
            rolls.append(q)
        eng.process_batch_device(src[lo:hi], dst[lo:hi], float(st.t[hi - 1]), k)
        ev[q + 1].record(stream)
    torch.cuda.synchronize()
    per = np.array([ev[q].elapsed_time(ev[q + 1]) for q in range(len(segs))])
    total = float(ev[0].elapsed_time(ev[-1]))
    plain = np.delete(per, rolls)
    full = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.full_recompute()
        e1.record(stream)
        torch.cuda.synchronize()
        full.append(e0.elapsed_time(e1))
    full_ms = float(np.median(full))
    p50 = float(np.percentile(plain, 50))
    # HBM bytes of one full recompute (dysat.cuh header): per node, L list ids + the gathered
    # P rows of its list (the snapshot's lists are empty after the last roll: self only),
    # 2 (W-1) history rows read, 2 history rows + 1 embedding row written, + its own P row
    d4 = 4 * eng.ld
    fb = n * (d4 + 2 * (cfg.window - 1) * d4 + 3 * d4 + 4 * cfg.fanout)
    return {"workload": "DySAT (1 structural layer, 16 heads; 1 temporal layer, 16 heads, window "
                        "8; d = 128, node features 64, L = 20) on a synthetic preferential "
                        f"stream, {n:,} nodes, {m:,} edges, {snapshots} snapshots, B = {B}",
            "value": m / (total / 1e3), "unit": UNIT, "batches": len(segs),
            "p50_ms": p50, "p99_ms": float(np.percentile(plain, 99)),
            "roll_ms_mean": float(np.mean(per[rolls])) if rolls else None, "rolls": len(rolls),
            "full_recompute_ms": full_ms, "full_recompute_hbm_gbs": fb / (full_ms / 1e3) / 1e9,
            "speedup_vs_full_recompute": full_ms / p50,
            "affected_per_batch": "the batch endpoints (one structural layer on static features)",
            "parity": "oracle/dysat_oracle.py (tests/test_gpu_dysat.py); unpinned vs the "
                      "reference, which ships no DySAT code",
            "cpu_reference": None}


def operator_leg(torch, dev, N=10_000, E_per=10, reps=20):
    """The operator-level drop-in (kernels.pipeline_many, S/kernels/__init__.py:42-44) at the
    C4 widths (K = 2, d = 100, d_e = 0, H = 2, d_k = 50): node-pipelines/s through the C ABI
    with device-resident inputs (CUDA events around `reps` calls) and through the numpy API
    (host arrays in and out, host clock). BASELINE.md §2 measured the reference's numba kernel
    at 1,735 node-pipelines/s (K = 2, d_e = 0, L = 10)."""
    import ctypes as C
    from paper_2603_21090_b200 import _lib, kernels
    from paper_2603_21090_b200.config import Dims
    from paper_2603_21090_b200.params import init_params
    dims = Dims(d_s=100, d_e=0, d_t=100, d_x=0, d_m=100, d_k=50, heads=2, layers=2)
    p = init_params(0, dims)
    rng = np.random.default_rng(0)
    E = N * E_per
    qbase = rng.standard_normal((N, 100))
    offsets = np.arange(0, E + 1, E_per, dtype=np.int64)
    payload = rng.standard_normal((E, 2, 100))
    feat = np.zeros((E, 0))
    dt = rng.uniform(0, 1e4, E)
    phi0 = np.empty(100)
    phi0[0::2], phi0[1::2] = 1.0, 0.0
    phi0 *= np.sqrt(1.0 / 100)
    kernels.pipeline_many(qbase[:8], offsets[:9], payload[:80], feat[:80], dt[:80], p.omega, phi0,
                          p.w_q, p.w_k, p.w_v, p.w_o)  # warm-up
    t0 = time.perf_counter()
    for _ in range(3):
        kernels.pipeline_many(qbase, offsets, payload, feat, dt, p.omega, phi0, p.w_q, p.w_k,
                              p.w_v, p.w_o)
    host_s = (time.perf_counter() - t0) / 3
    f32 = lambda a: torch.tensor(np.ascontiguousarray(a, dtype=np.float32), device=dev)  # noqa: E731
    t = dict(q=f32(qbase), off=torch.tensor(offsets, device=dev), pay=f32(payload),
             feat=f32(np.zeros((E, 1))), dt=torch.tensor(dt, device=dev),
             om=torch.tensor(p.omega, device=dev), phi0=f32(phi0), wq=f32(p.w_q), wk=f32(p.w_k),
             wv=f32(p.w_v), wo=f32(p.w_o))
    outs = [torch.zeros(sh, dtype=torch.float32, device=dev) for sh in
            ((N, 2, 100), (E, 2, 2), (E, 2, 2, 50), (N, 2, 2), (N, 2, 2), (N, 2, 2, 50))]
    ds = _lib.dims_struct(dims)
    L = _lib.lib()
    stream = torch.cuda.current_stream(dev)
    ptr = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731

    def call():
        _lib.check(L.stgn_pipeline_many(
            C.byref(ds), N, E, ptr(t["q"]), ptr(t["off"]), ptr(t["pay"]), ptr(t["feat"]),
            ptr(t["dt"]), ptr(t["om"]), ptr(t["phi0"]), ptr(t["wq"]), ptr(t["wk"]), ptr(t["wv"]),
            ptr(t["wo"]), *[ptr(o) for o in outs], C.c_void_p(stream.cuda_stream)), "pipeline_many")
    call()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    ev[0].record(stream)
    for _ in range(reps):
        call()
    ev[1].record(stream)
    torch.cuda.synchronize()
    dev_ms = ev[0].elapsed_time(ev[1]) / reps
    return {"nodes": N, "entries_per_node": E_per, "widths": "K=2, d=100, d_e=0, H=2, d_k=50",
            "device_ms_per_call": dev_ms, "node_pipelines_per_s": N / (dev_ms / 1e3),
            "numpy_api_ms_per_call": host_s * 1e3, "numpy_api_node_pipelines_per_s": N / host_s,
            "cpu_reference_node_pipelines_per_s": 1735,
            "note": "stgn_pipeline_many returns every per-entry intermediate of the reference "
                    "operator (scores, values, maxlog, zsum, qvecs): FFMA kernel with per-entry "
                    "K/V projections"}


def _timed_batches(torch, stream, feed, k0, K):
    """Feed batches k0..k0+K-1 of a DeviceStream, one CUDA event after each;
    returns (total ms, per-batch ms)."""
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
    torch.cuda.synchronize()
    ev[0].record(stream)
    for k in range(K):
        feed.batch(k0 + k)
        ev[k + 1].record(stream)
    torch.cuda.synchronize()
    per = np.array([ev[k].elapsed_time(ev[k + 1]) for k in range(K)])
    return float(ev[0].elapsed_time(ev[K])), per


def _e2e_leg(torch, eng, st, pos, n, B):
    """n batches from host arrays through StreamingEngine.submit/drain; returns
    (edges/s, wall seconds) by the host clock around all steps."""
    from paper_2603_21090_b200.streaming import StreamingEngine
    se = StreamingEngine(eng, depth=3, max_batch=B)
    host = [(np.ascontiguousarray(st.src[pos + k * B: pos + (k + 1) * B]),
             np.ascontiguousarray(st.dst[pos + k * B: pos + (k + 1) * B]),
             np.ascontiguousarray(st.t[pos + k * B: pos + (k + 1) * B])) for k in range(n)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for s_, d_, t_ in host:
        se.submit(s_, d_, t_)
    got = se.drain()
    wall = time.perf_counter() - t0
    assert len(got) == n
    return n * B / wall, wall


def _max_over_ranks(torch, dist, world, dev, x):
    if world == 1:
        return x
    tt = torch.tensor([x], device=dev, dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    return float(tt.item())


def run_ours(args, world, rank, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2603_21090_b200.engine import IncrementalEngine
    from paper_2603_21090_b200.feeder import DeviceStream
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dims, cfg, params = workload(args)
    B, W, K = args.batch, args.warmup, args.steps
    KE = args.e2e_steps if args.e2e_steps is not None else K
    P = args.profile_batches
    sweep = [int(x) for x in args.sweep.split(",") if x] if args.sweep else []
    SW = args.sweep_steps
    LAT = args.latency_steps
    tail = (W + K + LAT + KE + min(KE, 50) + P) * B
    total = max(args.edges, tail + B)
    n_sweep = sum((3 + SW) * b for b in sweep) + 2 * (3 + min(K, 100)) * B + 50 * B  # + direct, delta, sync legs
    t_gen = time.perf_counter()
    st = make_stream(args, total + n_sweep, rank)
    t_gen = time.perf_counter() - t_gen
    eng = IncrementalEngine(cfg, params, recompute=args.recompute)
    eng.reserve(nodes=args.nodes, edges=total + n_sweep + B, batch=B,
                batches=(total + n_sweep) // min([B] + sweep) + 8)
    stream = eng._torch.cuda.current_stream(dev)
    pos0 = total - tail            # the timed batches are the last ones of the stream
    t_ff = time.perf_counter()
    feed = DeviceStream(eng, st, B, 0, pos0)
    # 0) fast-forward; on the way, time the window the CPU reference is measured on
    win = None
    wk0 = args.prefix // B
    if args.prefix and wk0 + args.window_steps <= feed.n_batches:
        feed.run(0, wk0, report_last=False)
        w_ms, w_per = _timed_batches(torch, stream, feed, wk0, args.window_steps)
        win = {"value": args.window_steps * B / (w_ms / 1e3), "unit": UNIT,
               "p50_ms": float(np.percentile(w_per, 50)), "p99_ms": float(np.percentile(w_per, 99)),
               "stream_position": f"edges {wk0 * B}..{(wk0 + args.window_steps) * B}",
               "steps": args.window_steps, "affected_last": None}
        # the same window end to end through the public streaming API (pinned host batches,
        # uploads and score read-backs inside the timed region), on the next window_steps batches
        k_e = wk0 + args.window_steps
        n_e = min(args.window_steps, feed.n_batches - k_e)
        eng.sync()
        e_val, e_wall = _e2e_leg(torch, eng, st, k_e * B, n_e, B)
        win["e2e"] = {"value": e_val, "unit": UNIT, "steps": n_e, "wall_s": e_wall,
                      "h2d_bytes_per_step": B * 16, "d2h_bytes_per_step": B * 8,
                      "stream_position": f"edges {k_e * B}..{(k_e + n_e) * B}"}
        feed.run(k_e + n_e, None, report_last=True)
        win["affected_last"] = int(eng._rep.affected)
    else:
        feed.run(0, None, report_last=True)
    eng.sync()
    t_ff = time.perf_counter() - t_ff
    del feed
    # 1) device-resident inputs for warm-up + timed batches
    feed = DeviceStream(eng, st, B, pos0, pos0 + (W + K) * B)
    feed.run(0, W, report_last=True)
    rep_nA = int(eng._rep.affected)
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)  # let the sampler attach before the timed region
    total_ms, per = _timed_batches(torch, stream, feed, W, K)
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    total_ms = _max_over_ranks(torch, dist, world, dev, total_ms)
    value = world * K * B / (total_ms / 1e3)
    pos = pos0 + (W + K) * B
    del feed
    # 1b) latency distribution: LAT device-timed batches (CUDA event per batch) right
    # after the timed ones, at the end-of-stream state (p50/p99 over >= 1,000)
    lat = None
    if LAT:
        lf = DeviceStream(eng, st, B, pos, pos + LAT * B)
        l_ms, l_per = _timed_batches(torch, stream, lf, 0, LAT)
        lat = {"steps": LAT, "value": LAT * B / (l_ms / 1e3), "unit": UNIT,
               "p50_ms": float(np.percentile(l_per, 50)), "p90_ms": float(np.percentile(l_per, 90)),
               "p99_ms": float(np.percentile(l_per, 99)), "p999_ms": float(np.percentile(l_per, 99.9)),
               "max_ms": float(l_per.max()),
               "frac_batches_under_1ms": float(np.mean(l_per < 1.0)),
               "stream_position": f"edges {pos}..{pos + LAT * B} (end of the stream)"}
        pos += LAT * B
        del lf

    # 2) e2e: the public streaming API (StreamingEngine): every step copies its
    # batch from pinned host memory to the GPU and reads its scores back to
    # pinned host memory; uploads/read-backs overlap the neighbouring batches'
    # graphs (relaxed-order batched streaming); timed until the last score is
    # on the host
    from paper_2603_21090_b200.streaming import StreamingEngine
    se = StreamingEngine(eng, depth=3, max_batch=B)
    host = [(np.ascontiguousarray(st.src[pos + k * B: pos + (k + 1) * B]),
             np.ascontiguousarray(st.dst[pos + k * B: pos + (k + 1) * B]),
             np.ascontiguousarray(st.t[pos + k * B: pos + (k + 1) * B])) for k in range(KE)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_wall = time.perf_counter()
    for s_, d_, t_ in host:
        se.submit(s_, d_, t_)
    got = se.drain()
    t_wall = time.perf_counter() - t_wall
    assert len(got) == KE
    e2e_ms = _max_over_ranks(torch, dist, world, dev, t_wall * 1e3)
    e2e_value = world * KE * B / (e2e_ms / 1e3)
    pos += KE * B
    # the synchronous host-buffer call (process_batch_arrays): per-call latency
    sync_lat = []
    for k in range(min(KE, 50)):
        sl = slice(pos + k * B, pos + (k + 1) * B)
        t1 = time.perf_counter()
        eng.process_batch_arrays(st.src[sl], st.dst[sl], st.t[sl])
        sync_lat.append(time.perf_counter() - t1)
    pos += min(KE, 50) * B
    e2e_lat = np.array(sync_lat)

    # 3) per-stage device times (events, no graph) for the roofline
    info0 = eng.info()
    eng.set_profiling(True)
    stage_acc, attn_bytes, attn_flops, attn_ms, nA_list, eA_list = {}, [], [], [], [], []
    g = dims
    for k in range(P):
        sl = slice(pos + k * B, pos + (k + 1) * B)
        eng.process_batch_arrays(st.src[sl], st.dst[sl], st.t[sl])
        times, launches = eng.stage_times()
        for nm, v in times.items():
            stage_acc.setdefault(nm, []).append(v)
        r = eng._rep
        # one launch recomputes A (pre-batch memory) and V_direct (post-batch memory)
        nA = int(r.affected) + (int(r.direct) if args.recompute == "affected" else 0)
        EA = int(r.entries_affected) + int(r.entries_direct)
        attn_bytes.append(recompute_bytes(g, nA, EA, time_basis=bool(info0.get("bf16x3"))))
        attn_flops.append(recompute_flops(g, nA, EA))
        attn_ms.append(times["recompute"])
        nA_list.append(nA)
        eA_list.append(EA)
    eng.set_profiling(False)
    pos += P * B
    stage_ms = {nm: float(np.mean(v)) for nm, v in stage_acc.items()}
    a_ms = float(np.mean(attn_ms))
    achieved_gbs = float(np.mean(attn_bytes)) / (a_ms / 1e3) / 1e9
    peaks = {}
    pk_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk_path):
        with open(pk_path) as fh:
            peaks = json.load(fh)
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else \
        "fallback (B200_PROFILING.md)"
    info = eng.info()
    traffic = None  # DRAM bytes per launch of the same kernel from the committed ncu capture
    tr_path = os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")
    if os.path.exists(tr_path) and info.get("bf16x3"):
        with open(tr_path) as fh:
            traffic = json.load(fh).get("traffic_bytes_per_launch")

    # 3b) full rebuild (C4's O(|V|) path: rebuild_nodes(None)), node-id range per rank
    rb = None
    if not args.no_rebuild_leg:
        from paper_2603_21090_b200.dist import shard_range
        n_all = eng.node_count
        lo, hi = shard_range(n_all, world, rank)
        ents = int(eng._tab.ring_cnt[lo:hi].to(torch.int64).sum().item())
        r_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        r_ev[0].record(stream)
        if world == 1:
            eng.rebuild_nodes(None)
        else:  # each rank recomputes its node-id range, one NCCL all-gather of the rows
            eng.distributed_full_rebuild()
        r_ev[1].record(stream)
        torch.cuda.synchronize()
        r_ms = _max_over_ranks(torch, dist, world, dev, float(r_ev[0].elapsed_time(r_ev[1])))
        by = recompute_bytes(g, hi - lo, ents, time_basis=bool(info0.get("bf16x3")))
        rb = {"nodes": n_all, "nodes_per_rank": hi - lo, "ms": r_ms,
              "nodes_per_s": n_all / (r_ms / 1e3), "entries_rank0": ents,
              "algorithmic_bytes_rank0": by,
              "achieved_gbs_rank0": by / (r_ms / 1e3) / 1e9,
              "frac_hbm": by / (r_ms / 1e3) / 1e9 / hbm_peak,
              "sharding": (f"node-id ranges over {world} ranks + NCCL all-gather of the final "
                           f"rows (distributed_full_rebuild)") if world > 1 else "single GPU"}

    # 3c) the value-identical V_direct-only recompute on the same state ("measure
    # and report both"); the headline above is the literal recompute over A
    direct = None
    if args.recompute == "affected" and not args.no_direct_leg:
        eng.set_recompute("direct")
        KD = min(K, 100)
        df = DeviceStream(eng, st, B, pos, pos + (3 + KD) * B)
        df.run(0, 3, report_last=True)
        d_ms, d_per = _timed_batches(torch, stream, df, 3, KD)
        d_ms = _max_over_ranks(torch, dist, world, dev, d_ms)
        direct = {"value": world * KD * B / (d_ms / 1e3), "unit": UNIT, "steps": KD,
                  "p50_ms": float(np.percentile(d_per, 50)), "p99_ms": float(np.percentile(d_per, 99)),
                  "note": "recompute over V_direct only; A is still computed exactly and its "
                          "embeddings are bit-identical (payloads frozen at insertion)"}
        pos += (3 + KD) * B
        del df
        eng.set_recompute("affected")

    # 3d) the reference's delta mode on the same state (S/engine.py:276-331; K = 2 has no
    # attention states, so every non-skipped node of A is an attn_miss and is recomputed)
    delta = None
    if args.recompute == "affected" and not args.no_direct_leg:
        eng.set_recompute("delta")
        KD = min(K, 100)
        df = DeviceStream(eng, st, B, pos, pos + (3 + KD) * B)
        df.run(0, 3, report_last=True)
        d_ms, d_per = _timed_batches(torch, stream, df, 3, KD)
        d_ms = _max_over_ranks(torch, dist, world, dev, d_ms)
        r = eng._rep
        delta = {"value": world * KD * B / (d_ms / 1e3), "unit": UNIT, "steps": KD,
                 "p50_ms": float(np.percentile(d_per, 50)),
                 "p99_ms": float(np.percentile(d_per, 99)),
                 "sample_batch": {"affected": int(r.affected), "embed_skip": int(r.embed_skip),
                                "attn_hit": int(r.attn_hit), "attn_miss": int(r.attn_miss)},
                 "note": "cfg.mode = delta: A \\ V_direct nodes with an empty change record "
                         "keep their cached row; the rest are recomputed"}
        pos += (3 + KD) * B
        del df
        eng.set_recompute("affected")

    # 4) batch-size sweep (C4: 100..10K edges/batch) at the end-of-stream state
    sweep_out = []
    for b in sweep:
        sf = DeviceStream(eng, st, b, pos, pos + (3 + SW) * b)
        sf.run(0, 3, report_last=True)
        s_ms, s_per = _timed_batches(torch, stream, sf, 3, SW)
        s_ms = _max_over_ranks(torch, dist, world, dev, s_ms)
        sweep_out.append({"batch_edges": b, "value": world * SW * b / (s_ms / 1e3),
                          "p50_ms": float(np.percentile(s_per, 50)),
                          "p99_ms": float(np.percentile(s_per, 99)),
                          "affected_last": int(eng._rep.affected)})
        pos += (3 + SW) * b
        del sf

    # 5) the other configs of BASELINE.json (C1, C2 full streams; C3 TGAT at the C4 scale)
    cfg_legs = config_legs(args, torch, dev) if (args.config_legs and rank == 0) else None
    op_leg = operator_leg(torch, dev) if (args.config_legs and rank == 0) else None
    dy_leg = (dysat_leg(torch, dev) if (rank == 0 and "C5" in args.config_legs.split(","))
              else None)

    line = None
    if rank == 0:
        h2d = B * (4 + 4 + 8)
        d2h = B * 8
        kname = ("attn4_kernel (tcgen05 bf16x3, 128-row tiles)" if info.get("bf16x3") else
                 "attn3_kernel (tcgen05 split-TF32)" if info.get("tensor_cores") else
                 "attn2_kernel (FFMA)")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": total_ms / K,
            "p50_ms": float(np.percentile(per, 50)), "p99_ms": float(np.percentile(per, 99)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (reference generator, native replay; random-init weights)",
            "config": config_json(args, world),
            "timed_batches": timed_position(args, pos0),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "api": "StreamingEngine.submit/drain "
                    "(pinned host batches, pipelined uploads and score read-backs), host "
                    "wall clock around all steps", "wall_s": t_wall,
                    "sync_call_p50_ms": float(np.percentile(e2e_lat, 50) * 1e3),
                    "sync_call_p99_ms": float(np.percentile(e2e_lat, 99) * 1e3)},
            "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak,
                         "unit": "GB/s", "frac": achieved_gbs / hbm_peak, "traffic": traffic,
                         "traffic_source": "profiles/r02_ncu_traffic.json (ncu --set full)",
                         "kernel": kname + ": recompute of A (pre-batch memory) + V_direct "
                                           "(post-batch memory), one launch",
                         "avg_launch_ms": a_ms, "algorithmic_bytes": float(np.mean(attn_bytes)),
                         "flops": float(np.mean(attn_flops)),
                         "tflops": float(np.mean(attn_flops)) / (a_ms / 1e3) / 1e12,
                         "peak_source": peak_src, "rows_per_launch": float(np.mean(nA_list)),
                         "entries_per_launch": float(np.mean(eA_list))},
            "stage_ms": stage_ms,
            "affected_per_batch": rep_nA,
            "gpu_launches": (int(launches) + 1) * K,  # + k_set_hdr per batch
            "clocks": clk,
            "engine": info,
            "window": win,
            "latency": lat,
            "sweep": sweep_out,
            "configs": cfg_legs,
            "operator_pipeline_many": op_leg,
            "dysat": dy_leg,
            "full_rebuild": rb,
            # the paper's "index refresh" comparison: one full recompute of
            # every node (the TGL-style / OracleEngine baseline) vs one incremental batch
            "refresh_vs_full_recompute": None if rb is None else {
                "full_recompute_ms": rb["ms"], "incremental_ms": total_ms / K,
                "speedup": rb["ms"] / (total_ms / K),
                "direct_scope_speedup": (rb["ms"] / direct["p50_ms"]) if direct else None},
            "direct_scope": direct,
            "delta_mode": delta,
            "setup_s": {"generate": t_gen, "fast_forward": t_ff},
        }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cv, ctimes, sample, kind = cpu_reference(args, max(1, args.cpu_batches))
        line["cpu_baseline"] = {"value": cv, "unit": UNIT, "cores": 1, "kind": kind,
                                "sample": sample, "p50_ms": float(np.median(ctimes) * 1e3),
                                "host_nproc": os.cpu_count()}
    if line is not None:
        print(json.dumps(line), flush=True)


def recompute_bytes(g, rows, entries, time_basis=False):
    """Algorithmic HBM bytes of one recompute launch, SURVEY.md §8d's per-unit
    figure: per row the query row (4 d_s), the K*d output and 16 B of ring
    meta; per ring entry the K*d frozen payload, d_e features and 16 B
    (timestamp + ids). `time_basis` is accepted for the record but does not
    change the count: the bf16x3 kernel's stored time basis (4*d_t bytes per
    entry and layer) is an implementation choice that trades bytes for
    instructions, and shows up in `roofline.traffic` (ncu DRAM bytes), not here."""
    del time_basis
    return rows * (4 * g.d_s + 4 * g.layers * g.d + 16) + \
        entries * (4 * g.layers * g.d + 4 * g.d_e + 16)


def recompute_flops(g, rows, entries):
    """FLOPs of the folded formulation the kernel executes."""
    per_node_l = 2 * (g.query_in * g.heads * g.d_k + g.heads * g.d_k * g.key_in +
                      g.heads * g.key_in * g.d_k + g.heads * g.d_k * g.d)
    per_entry_l = 2 * (2 * g.heads * g.key_in)
    return g.layers * (rows * per_node_l + entries * per_entry_l)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        if args.impl == "ours":
            import torch
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl")
        else:
            if rank != 0:
                return
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local_rank)
    if world > 1 and args.impl == "ours":
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
