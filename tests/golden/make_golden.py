"""Write golden fixtures by running the REFERENCE itself (run in the build
container, where /root/reference exists; the fixtures travel, the
reference does not).

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py

Outputs (tests/golden/):
  engine_<name>.npz   per-batch predictions, direct/affected sets,
                      counters, rebuild decisions; final memory,
                      last_interaction, version, layer cache h, valid_at,
                      neighbour-cache lists (nbr, t, eid) of every node.
  pipeline_<name>.npz operator-level pipeline_many inputs and outputs.
  params_seed.npz     init_params tensors for two dims (init pinning).
  streams.npz         generate_stream outputs (generator pinning).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from streamtgn import kernels  # noqa: E402
from streamtgn.config import Dims, RunConfig  # noqa: E402
from streamtgn.engine import IncrementalEngine  # noqa: E402
from streamtgn.graph_store import TemporalEdge  # noqa: E402
from streamtgn.params import init_params  # noqa: E402
from streamtgn.streamio import generate_stream  # noqa: E402

# (name, dims kwargs, cfg kwargs, params seed, randomize biases,
#  stream kwargs | explicit edge list, batch size)
ENGINE_CASES = [
    ("small_mean", dict(d_s=6, d_e=3, d_t=6, d_m=5, d_k=4, heads=2, layers=1),
     dict(fanout=4, nodes=25, aggregator="mean"), 3, True,
     dict(seed=21, n=25, m=250, attachment="uniform", d_e=3), 7),
    ("k2_last_adaptive", dict(d_s=8, d_e=4, d_t=8, d_m=8, d_k=4, heads=2, layers=2),
     dict(fanout=5, nodes=60, aggregator="last", rebuild="adaptive",
          gamma=0.9, delta_max=0.5, alpha=0.1), 5, True,
     dict(seed=7, n=60, m=900, attachment="preferential", burstiness=2.0, d_e=4), 16),
    ("k2_sum_window", dict(d_s=6, d_e=2, d_t=4, d_m=5, d_k=3, heads=2, layers=2),
     dict(fanout=3, nodes=30, aggregator="sum", window=5.0), 9, True,
     dict(seed=4, n=30, m=300, attachment="uniform", d_e=2), 5),
    ("k1_fixed_de0", dict(d_s=8, d_e=0, d_t=8, d_m=8, d_k=4, heads=2, layers=1),
     dict(fanout=10, nodes=0, aggregator="last", rebuild="fixed", rebuild_interval=7),
     11, False, dict(seed=12, n=200, m=1500, attachment="preferential", d_e=0), 20),
    ("k2_wide_adaptive", dict(d_s=16, d_e=0, d_t=16, d_m=16, d_k=8, heads=2, layers=2),
     dict(fanout=10, nodes=500, aggregator="last", rebuild="adaptive",
          gamma=0.9, delta_max=0.3, alpha=0.1), 0, False,
     dict(seed=2, n=500, m=4000, attachment="preferential", d_e=0), 50),
    ("k2_mean_b1", dict(d_s=6, d_e=3, d_t=6, d_m=5, d_k=4, heads=2, layers=2),
     dict(fanout=4, nodes=20, aggregator="mean"), 13, True,
     dict(seed=13, n=20, m=150, attachment="uniform", d_e=3), 1),
    ("selfloops_dups", dict(d_s=6, d_e=3, d_t=6, d_m=5, d_k=4, heads=2, layers=2),
     dict(fanout=3, nodes=6, aggregator="last"), 17, True, "handmade", 4),
    ("c4_shape_tiny", dict(d_s=100, d_e=0, d_t=100, d_m=100, d_k=50, heads=2, layers=2),
     dict(fanout=10, nodes=3000, aggregator="last"), 0, False,
     dict(seed=2, n=3000, m=3000, attachment="preferential", d_e=0), 600),
    # round 2: the C2 / C1 widths (d_e = 172, k_in = 372), heads 1 / 3 / 4, a B = 3,000
    # batch, and the C3 memoryless (TGAT) emulation at the C4 widths
    ("c2_widths", dict(d_s=100, d_e=172, d_t=100, d_m=100, d_k=50, heads=2, layers=2),
     dict(fanout=10, nodes=800, aggregator="last", rebuild="adaptive",
          gamma=0.9, delta_max=0.5, alpha=0.1), 0, False,
     dict(seed=1, n=800, m=6000, attachment="preferential", d_e=172), 600),
    ("c1_widths", dict(d_s=100, d_e=172, d_t=100, d_m=100, d_k=50, heads=2, layers=1),
     dict(fanout=10, nodes=1500, aggregator="last", rebuild="adaptive",
          gamma=0.9, delta_max=0.5, alpha=0.1), 0, False,
     dict(seed=0, n=1500, m=6000, attachment="preferential", d_e=172), 200),
    ("heads1_k2", dict(d_s=8, d_e=2, d_t=8, d_m=8, d_k=6, heads=1, layers=2),
     dict(fanout=5, nodes=80, aggregator="last", rebuild="adaptive",
          gamma=0.9, delta_max=1.5, alpha=0.1), 21, True,
     dict(seed=31, n=80, m=1200, attachment="preferential", d_e=2), 20),
    ("heads4_k2", dict(d_s=12, d_e=3, d_t=8, d_m=8, d_k=4, heads=4, layers=2),
     dict(fanout=6, nodes=80, aggregator="mean"), 22, True,
     dict(seed=32, n=80, m=1200, attachment="preferential", d_e=3), 24),
    ("heads3_k1", dict(d_s=10, d_e=0, d_t=6, d_m=7, d_k=5, heads=3, layers=1),
     dict(fanout=7, nodes=60, aggregator="sum", rebuild="fixed", rebuild_interval=9), 23, True,
     dict(seed=33, n=60, m=900, attachment="uniform", d_e=0), 15),
    ("b3000", dict(d_s=16, d_e=0, d_t=16, d_m=16, d_k=8, heads=2, layers=2),
     dict(fanout=10, nodes=20000, aggregator="last"), 0, False,
     dict(seed=2, n=20000, m=15000, attachment="preferential", d_e=0), 3000),
    ("c3_memoryless", dict(d_s=100, d_e=0, d_t=100, d_m=100, d_k=50, heads=2, layers=2),
     dict(fanout=10, nodes=3000, aggregator="last"), "memoryless", False,
     dict(seed=2, n=3000, m=6000, attachment="preferential", d_e=0), 600),
]

GRU_TENSORS = ("w_z", "u_z", "b_z", "w_r", "u_r", "b_r", "w_h", "u_h", "b_h")


def memoryless_params(dims):
    """TGAT emulation: every GRU tensor zero, so s' = 0.5 s + 0.5 tanh(0)
    and the memory stays 0 (S/kernels/reference.py:87-90, S/engine_base.py:237-241)."""
    p = init_params(0, dims)
    for name in GRU_TENSORS:
        getattr(p, name)[...] = 0.0
    return p


def random_params(seed, dims):
    """Same as the reference's tests/conftest.py:18-26 (biases random too)."""
    p = init_params(seed, dims)
    rng = np.random.default_rng(seed + 1)
    for name, t in p.tensors().items():
        if name.startswith("b_") and name != "b_pred":
            t[...] = rng.standard_normal(t.shape)
    p.b_pred = float(rng.standard_normal())
    return p


def handmade_stream(d_e):
    rng = np.random.default_rng(99)
    rows = [(0, 0, 1.0), (0, 1, 1.0), (0, 1, 1.0), (2, 2, 2.0), (1, 2, 2.0), (3, 0, 3.0),
            (3, 3, 3.0), (4, 5, 3.0), (5, 4, 4.0), (0, 5, 4.0), (0, 0, 4.0), (1, 1, 5.0),
            (2, 3, 5.0), (3, 2, 5.0), (4, 0, 6.0), (0, 4, 6.0), (5, 5, 6.0), (1, 3, 7.0),
            (2, 4, 7.0), (0, 2, 7.0), (0, 3, 7.0), (0, 4, 8.0), (0, 5, 8.0), (0, 1, 8.0)]
    return [TemporalEdge(s, d, t, rng.standard_normal(d_e)) for (s, d, t) in rows]


COUNTER_KEYS = ("nbr_hit", "nbr_miss", "embed_refresh", "embed_predict", "gru_steps",
                "messages", "macs_attention", "macs_gru", "rows_gathered",
                "rebuild_pipelines", "direct", "affected", "rebuilds")


def run_engine_case(name, dkw, ckw, pseed, rand_bias, skw, B):
    dims = Dims(**dkw)
    cfg = RunConfig(dims=dims, batch_size=B, **ckw)
    if pseed == "memoryless":
        params = memoryless_params(dims)
    else:
        params = random_params(pseed, dims) if rand_bias else init_params(pseed, dims)
    stream = handmade_stream(dims.d_e) if skw == "handmade" else generate_stream(**skw)
    eng = IncrementalEngine(cfg, params)
    preds, direct, affected, a_off, d_off = [], [], [], [0], [0]
    counters, rebuild_kind, rebuild_cnt = [], [], []
    # delta mode: per-update error-bound records (S/engine.py:333-353) and the running
    # max value norm, per batch
    ev = {k: [] for k in ("node", "bound", "dn", "nv", "max_v", "z_dev", "emb")}
    ev_off, mvn = [0], []
    for i in range(0, len(stream), B):
        preds.extend(eng.process_batch(stream[i:i + B]))
        for e in eng.delta_events:
            ev["node"].append(e.node)
            ev["bound"].append(e.bound)
            ev["dn"].append(e.dn)
            ev["nv"].append(e.nv)
            ev["max_v"].append(e.max_v)
            ev["z_dev"].append(e.z_dev)
            ev["emb"].append(e.embedding)
        ev_off.append(len(ev["node"]))
        mvn.append(eng.max_value_norm_seen)
        aff = eng.last_affected
        affected.extend(sorted(aff.all))
        direct.extend(sorted(aff.direct))
        a_off.append(len(affected))
        d_off.append(len(direct))
        counters.append([eng.counters.get(k) for k in COUNTER_KEYS])
        rebuild_kind.append({"none": 0, "partial": 1, "full": 2}[eng.last_report.rebuild])
        rebuild_cnt.append(eng.last_report.rebuild_nodes)
    n = eng.node_count
    L, K = cfg.fanout, dims.layers
    c_cnt = np.full(n, -1, dtype=np.int64)
    c_nbr = np.zeros((n, L), dtype=np.int64)
    c_eid = np.zeros((n, L), dtype=np.int64)
    c_t = np.zeros((n, L))
    for v in range(n):
        lst = eng.nbr_cache.get(v)
        if lst is None:
            continue
        c_cnt[v] = len(lst)
        for j, e in enumerate(lst):
            c_nbr[v, j], c_t[v, j], c_eid[v, j] = e.nbr, e.t, e.edge_id
    src = np.array([e.src for e in stream], dtype=np.int64)
    dst = np.array([e.dst for e in stream], dtype=np.int64)
    ts = np.array([e.t for e in stream])
    feat = np.array([e.feat for e in stream]).reshape(len(stream), dims.d_e)
    out = dict(
        dims=np.array([getattr(dims, k) for k in
                       ("d_s", "d_e", "d_t", "d_x", "d_m", "d_k", "heads", "layers")]),
        batch_size=B, fanout=L, nodes=cfg.nodes, aggregator=cfg.aggregator,
        rebuild=cfg.rebuild, rebuild_interval=cfg.rebuild_interval,
        gamma=cfg.gamma, delta_max=cfg.delta_max, alpha=cfg.alpha, window=cfg.window,
        src=src, dst=dst, t=ts, feat=feat,
        **{f"param_{k}": v for k, v in params.tensors().items()},
        preds=np.array(preds), affected=np.array(affected, dtype=np.int64),
        direct=np.array(direct, dtype=np.int64), a_off=np.array(a_off), d_off=np.array(d_off),
        counters=np.array(counters, dtype=np.float64), counter_keys=np.array(COUNTER_KEYS),
        rebuild_kind=np.array(rebuild_kind), rebuild_cnt=np.array(rebuild_cnt),
        memory=eng.memory.states[:n].copy(), last=eng.memory.last_interaction[:n].copy(),
        version=eng.memory.version[:n].copy(), h=eng.cache.h[:n].copy(),
        valid=eng.cache.valid[:n].copy(), valid_at=eng.cache.valid_at[:n].copy(),
        cache_cnt=c_cnt, cache_nbr=c_nbr, cache_eid=c_eid, cache_t=c_t,
        full_reference=eng.full_reference(), node_count=n,
        global_drift=eng.scheduler.global_drift(), tau=eng.scheduler.tau,
        ev_off=np.array(ev_off), ev_node=np.array(ev["node"], dtype=np.int64),
        ev_bound=np.array(ev["bound"]), ev_dn=np.array(ev["dn"], dtype=np.int64),
        ev_nv=np.array(ev["nv"], dtype=np.int64), ev_max_v=np.array(ev["max_v"]),
        ev_z_dev=np.array(ev["z_dev"]),
        ev_emb=np.array(ev["emb"]).reshape(len(ev["node"]), dims.d),
        max_value_norm_seen=np.array(mvn),
    )
    np.savez_compressed(os.path.join(HERE, f"engine_{name}.npz"), **out)
    print(f"engine_{name}: {len(stream)} edges, {len(a_off) - 1} batches, n={n}, "
          f"rebuilds={sum(1 for k in rebuild_kind if k)}")


def run_pipeline_case(name, dims, pseed, n_nodes, max_entries, case_seed):
    p = random_params(pseed, dims)
    rng = np.random.default_rng(case_seed)
    counts = rng.integers(0, max_entries + 1, size=n_nodes)
    offsets = np.zeros(n_nodes + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(counts)
    E = int(offsets[-1])
    qbase = rng.standard_normal((n_nodes, dims.d))
    payload = rng.standard_normal((E, dims.layers, dims.d))
    feat = rng.standard_normal((E, dims.d_e))
    dt = rng.uniform(0, 20, size=E)
    phi0 = kernels.time_encode(0.0, p)
    outs = kernels.backend_for("numba").pipeline_many(
        qbase, offsets, payload, feat, dt, p.omega, phi0, p.w_q, p.w_k, p.w_v, p.w_o)
    names = ("out", "scores", "values", "maxlog", "zsum", "qvecs")
    np.savez_compressed(os.path.join(HERE, f"pipeline_{name}.npz"),
                        qbase=qbase, offsets=offsets, payload=payload, feat=feat, dt=dt,
                        omega=p.omega, phi0=phi0, wq=p.w_q, wk=p.w_k, wv=p.w_v, wo=p.w_o,
                        **dict(zip(names, outs)))
    print(f"pipeline_{name}: N={n_nodes} E={E}")


def main():
    only = [a for a in sys.argv[1:] if not a.startswith("-")]
    if only:  # regenerate the named engine fixtures only
        for case in ENGINE_CASES:
            if case[0] in only:
                run_engine_case(*case)
        return
    for case in ENGINE_CASES:
        run_engine_case(*case)
    run_pipeline_case("k1", Dims(d_s=6, d_e=3, d_t=6, d_m=5, d_k=4, heads=2, layers=1),
                      1, 40, 7, 17)
    run_pipeline_case("k2", Dims(d_s=6, d_e=3, d_t=6, d_m=5, d_k=4, heads=2, layers=2),
                      2, 40, 7, 18)
    run_pipeline_case("c1dims", Dims(d_s=100, d_e=172, d_t=100, d_m=100, d_k=50, heads=2,
                                     layers=1), 0, 64, 10, 19)
    run_pipeline_case("c4dims", Dims(d_s=100, d_e=0, d_t=100, d_m=100, d_k=50, heads=2,
                                     layers=2), 0, 64, 10, 20)
    pz = {}
    for tag, dims in (("a", Dims(d_s=6, d_e=3, d_t=6, d_m=5, d_k=4, heads=2, layers=1)),
                      ("b", Dims(d_s=100, d_e=172, d_t=100, d_m=100, d_k=50, heads=2,
                                 layers=2))):
        for k, v in init_params(12345, dims).tensors().items():
            pz[f"{tag}_{k}"] = v
    np.savez_compressed(os.path.join(HERE, "params_seed.npz"), **pz)
    sz = {}
    for i, kw in enumerate([dict(seed=0, n=50, m=400, attachment="uniform", d_e=3),
                            dict(seed=1, n=100, m=1500, attachment="preferential",
                                 burstiness=2.0, d_e=4),
                            dict(seed=2, n=2000, m=5000, attachment="preferential", d_e=0)]):
        s = generate_stream(**kw)
        sz[f"s{i}_src"] = np.array([e.src for e in s])
        sz[f"s{i}_dst"] = np.array([e.dst for e in s])
        sz[f"s{i}_t"] = np.array([e.t for e in s])
        sz[f"s{i}_feat"] = np.array([e.feat for e in s]).reshape(len(s), kw["d_e"])
    np.savez_compressed(os.path.join(HERE, "streams.npz"), **sz)
    print("params_seed.npz, streams.npz written")


if __name__ == "__main__":
    main()
