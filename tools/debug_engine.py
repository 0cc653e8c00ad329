"""Batch-by-batch engine-vs-oracle comparison with a detailed report of the
first divergence (developer tool; run under gpurun)."""

import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")

from golden_util import batches, case_setup, load  # noqa: E402
from oracle.stgn_oracle import Oracle  # noqa: E402
from paper_2603_21090_b200.engine import IncrementalEngine  # noqa: E402


def main(name, limit=5):
    z = load("engine_" + name)
    cfg, params, stream = case_setup(z)
    eng = IncrementalEngine(cfg, params)
    orc = Oracle(cfg, params)
    shown = 0
    for bi, b in enumerate(batches(stream, cfg.batch_size)):
        p = eng.process_batch_arrays(b.src, b.dst, b.t, b.feat)
        q = np.array(orc.process_batch(b.src, b.dst, b.t, b.feat))
        la = eng.last_affected
        msgs = []
        if la.direct != orc.last_direct:
            msgs.append(f"direct: gpu-only {sorted(la.direct - orc.last_direct)} "
                        f"orc-only {sorted(orc.last_direct - la.direct)}")
        if la.all != orc.last_all:
            msgs.append(f"A: gpu-only {sorted(la.all - orc.last_all)[:20]} "
                        f"orc-only {sorted(orc.last_all - la.all)[:20]}")
        n = orc.node_count
        for v in range(n):
            a = eng.nbr_cache.get(v)
            o = orc.neighbor_list(v)
            if (a is None) != (o is None) or (a is not None and
                                               [(e.nbr, e.edge_id) for e in a] != [(x[0], x[2]) for x in o]):
                msgs.append(f"ring v={v}: gpu {None if a is None else [(e.nbr, e.edge_id) for e in a]} "
                            f"orc {None if o is None else [(x[0], x[2]) for x in o]}")
                break
        dp = float(np.max(np.abs(p - q)))
        if dp > 1e-5:
            msgs.append(f"pred dev {dp:.3e}")
        dm = float(np.max(np.abs(eng.memory.states[:n] - orc.mem[:n])))
        if dm > 1e-4:
            bad = np.nonzero(np.abs(eng.memory.states[:n] - orc.mem[:n]).max(axis=1) > 1e-4)[0]
            msgs.append(f"mem dev {dm:.3e} rows {bad[:10]}")
        dl = float(np.max(np.abs(eng.memory.last_interaction[:n] - orc.last[:n])))
        if dl > 0:
            msgs.append(f"last dev {dl}")
        dh = np.abs(eng.cache.h[:n] - orc.h[:n]).reshape(n, -1).max(axis=1)
        if dh.max() > 1e-4:
            bad = np.nonzero(dh > 1e-4)[0]
            msgs.append(f"h dev {dh.max():.3e} rows {bad[:10]} (direct={sorted(orc.last_direct)[:10]})")
        rep = eng.last_report
        if rep.rebuild != orc.last_report["rebuild"] or rep.rebuild_nodes != orc.last_report["rebuild_nodes"]:
            msgs.append(f"rebuild gpu {rep.rebuild}/{rep.rebuild_nodes} orc {orc.last_report}")
        if msgs:
            print(f"== batch {bi} (B={len(b)}) src={b.src.tolist()[:12]} dst={b.dst.tolist()[:12]}")
            for m in msgs:
                print("  ", m)
            shown += 1
            if shown >= limit:
                break
    print("done", name)


if __name__ == "__main__":
    for nm in sys.argv[1:]:
        main(nm)
