"""Quick K11 check: paired vs single-pass builds, bitwise, then timing at C3/C4."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2512_07311_b200 as rcs
from rcs_workload import config_qasm
ctx = rcs.Context(0)
for cfg in sys.argv[1:]:
    c = rcs.Circuit.from_qasm(config_qasm(cfg))
    os.environ["RCS_TC_PAIR"] = "1"
    a = rcs.State.build(ctx, c, fuse_k=6, timing=True)
    ra = dict(a.report)
    big = a.n > 30
    ha = a.copy_out(0, 1 << 20) if big else a.copy_out()
    del a
    os.environ["RCS_TC_PAIR"] = "0"
    b = rcs.State.build(ctx, c, fuse_k=6, timing=True)
    rb = dict(b.report)
    hb = b.copy_out(0, 1 << 20) if big else b.copy_out()
    del b
    print(cfg, "paired", ra["n_paired"], "bitwise_equal", bool(np.array_equal(ha, hb)),
          "build_ms paired %.1f single %.1f" % (ra["build_ms"], rb["build_ms"]),
          "pass_ms %.1f vs %.1f" % (ra["pass_ms"], rb["pass_ms"]), "norm", ra["norm"], rb["norm"], flush=True)
