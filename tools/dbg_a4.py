import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
from golden_util import load, case_setup
from paper_2603_21090_b200.engine import IncrementalEngine
from paper_2603_21090_b200 import _lib
for n in ['c4_shape_tiny','k2_sum_window','selfloops_dups']:
    z=load('engine_'+n); cfg,p,s=case_setup(z)
    e=IncrementalEngine(cfg,p)
    print(n, e.info(), sorted(e._w.keys()), _lib.lib().stgn_last_error())
