"""Phase timeline of CTA 0 of mem4_kernel (and attn4) for one profiled batch at the
C4 window state (needs a library built with -DA4_PROF). mem4 tags: 8 header,
9 X2 chunk 0, 10 message GEMMs, 11 A2 pack, 12 ZR GEMMs, 13 ZR epilogue,
14 H GEMMs + final epilogue, 15 tile end."""
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

edges = int(sys.argv[1]) if len(sys.argv) > 1 else 120_000
dims = Dims(d_s=100, d_e=0, d_t=100, d_m=100, d_k=50, heads=2, layers=2)
cfg = RunConfig(dims=dims, batch_size=600, fanout=10, nodes=2_600_000, aggregator="last",
                rebuild="adaptive")
st = generate_stream(2, 2_600_000, edges + 1800, attachment="preferential", d_e=0)
eng = IncrementalEngine(cfg, init_params(0, dims))
eng.reserve(nodes=2_600_000, edges=edges + 2400, batch=600, batches=edges // 600 + 8)
DeviceStream(eng, st, 600, 0, edges).run()
torch.cuda.synchronize()
L = _lib.lib()
buf = (C.c_uint64 * 8192)()
eng.set_profiling(True)
for k in range(3):
    L.stgn_debug_a4_prof(buf, 8192)
    lo = edges + 600 * k
    eng.process_batch_arrays(st.src[lo:lo + 600], st.dst[lo:lo + 600], st.t[lo:lo + 600])
    torch.cuda.synchronize()
n = L.stgn_debug_a4_prof(buf, 8192)
a = np.array(buf[:n], dtype=np.uint64)
t = (a >> 4).astype(np.int64)
tag = (a & 15).astype(np.int64)
sel = tag >= 8
t, tag = t[sel], tag[sel]
print("mem4 marks", len(t), "direct", eng._rep.direct)
for i in range(len(t) - 1):
    print(f"  after tag {tag[i]:2d}: {(t[i + 1] - t[i]) / 1e3:7.2f} us")
