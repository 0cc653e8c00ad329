"""Phase timeline of CTA 0 of attn4 at the C4 end-of-stream state (needs a
library built with -DA4_PROF). Tags: 0 layer start, 1 after Q(+q epilogue),
2 walk start (after K_1), 3 walk end, 4 after V(+c epilogue), 5 after O."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_21090_b200 import _lib  # noqa: E402
from paper_2603_21090_b200.config import Dims, RunConfig  # noqa: E402
from paper_2603_21090_b200.engine import IncrementalEngine  # noqa: E402
from paper_2603_21090_b200.feeder import DeviceStream  # noqa: E402
from paper_2603_21090_b200.params import init_params  # noqa: E402
from paper_2603_21090_b200.streamio import generate_stream  # noqa: E402

edges = int(sys.argv[1]) if len(sys.argv) > 1 else 30_000_000
dims = Dims(d_s=100, d_e=0, d_t=100, d_m=100, d_k=50, heads=2, layers=2)
cfg = RunConfig(dims=dims, batch_size=600, fanout=10, nodes=2_600_000, aggregator="last",
                rebuild="adaptive")
st = generate_stream(2, 2_600_000, edges + 600, attachment="preferential", d_e=0)
eng = IncrementalEngine(cfg, init_params(0, dims))
eng.reserve(nodes=2_600_000, edges=edges + 1200, batch=600, batches=edges // 600 + 8)
DeviceStream(eng, st, 600, 0, edges).run()
torch.cuda.synchronize()
L = _lib.lib()
buf = (C.c_uint64 * 8192)()
L.stgn_debug_a4_prof(buf, 8192)  # drop the fast-forward marks
L.stgn_debug_a4_cta((C.c_uint64 * 4096)(), 4096)
eng.set_profiling(True)
eng.process_batch_arrays(st.src[edges:edges + 600], st.dst[edges:edges + 600], st.t[edges:edges + 600])
torch.cuda.synchronize()
n = L.stgn_debug_a4_prof(buf, 8192)
a = np.array(buf[:n], dtype=np.uint64)
t = (a >> 4).astype(np.int64)
tag = (a & 15).astype(np.int64)
print("marks", n, "rows", eng._rep.affected, "span_us", (t[-1] - t[0]) / 1e3 if n else 0)
names = {0: "Q+q", 1: "K0/K1", 2: "walk (thread 0)", 3: "walk tail (CTA barrier)",
         6: "V weights staged + V_0", 7: "V_1 + c", 4: "O+out", 5: "->next"}
acc = {}
keep = tag < 8  # attn4 marks only (mem4 uses 8..15)
t, tag = t[keep], tag[keep]
n = len(t)
for i in range(n - 1):
    acc.setdefault(int(tag[i]), []).append((t[i + 1] - t[i]) / 1e3)
tot = sum(sum(v) for v in acc.values())
for k in sorted(acc):
    v = acc[k]
    print(f"after tag {k} ({names.get(k)}): n={len(v)} total_us={sum(v):8.1f} share={100 * sum(v) / tot:5.1f}% mean_us={np.mean(v):7.2f}")

# per-CTA balance of the same launch(es): start/end spread, ring entries per CTA
buf2 = (C.c_uint64 * 4096)()
L.stgn_debug_a4_cta(buf2, 4096)
c = np.array(buf2[:4096], dtype=np.uint64).reshape(1024, 4).astype(np.int64)
c = c[(c[:, 3] & 0xFFFF) > 0]
if len(c):
    sm = c[:, 3] >> 16
    c[:, 3] &= 0xFFFF
    t0 = c[:, 0].min()
    st_us, en_us = (c[:, 0] - t0) / 1e3, (c[:, 1] - t0) / 1e3
    dur = en_us - st_us
    print(f"CTAs {len(c)} tiles/CTA {np.unique(c[:, 3]).tolist()}")
    print(f"start us: min {st_us.min():.1f} p50 {np.median(st_us):.1f} max {st_us.max():.1f}")
    print(f"end   us: min {en_us.min():.1f} p50 {np.median(en_us):.1f} mean {en_us.mean():.1f} max {en_us.max():.1f}")
    print(f"busy  us: min {dur.min():.1f} p50 {np.median(dur):.1f} max {dur.max():.1f}")
    e = c[:, 2].astype(np.float64)
    print(f"entries/CTA: min {e.min():.0f} p50 {np.median(e):.0f} max {e.max():.0f}; corr(entries, busy) {np.corrcoef(e, dur)[0, 1]:.3f}")
    print(f"us per 1K entries (fit): {1e3 * np.polyfit(e, dur, 1)[0]:.3f}, intercept {np.polyfit(e, dur, 1)[1]:.1f} us")
    for name, m in (("SM id < 74", sm < 74), ("SM id >= 74", sm >= 74), ("even SM", sm % 2 == 0), ("odd SM", sm % 2 == 1)):
        if m.any():
            print(f"  {name}: n {m.sum()} mean end {en_us[m].mean():.1f} max {en_us[m].max():.1f}")
    # a tile's rows' entries: the slowest CTAs vs the fastest
    q = np.argsort(dur)
    print(f"fastest 20 CTAs mean entries {e[q[:20]].mean():.0f}, slowest 20 {e[q[-20:]].mean():.0f}")
    order = np.argsort(-en_us)[:5]
    print("latest CTAs (idx, start, end, entries):", [(int(i), round(st_us[i], 1), round(en_us[i], 1), int(e[i])) for i in order])
