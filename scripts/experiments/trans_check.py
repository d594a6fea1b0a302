"""K12 (transposed TC pass) vs K9: bitwise state comparison and build times."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2512_07311_b200 as rcs
from rcs_workload import config_qasm, random_qasm
ctx = rcs.Context(0)
for cfg in sys.argv[1:]:
    text = random_qasm(22, 300, 7) if cfg == "rand22" else config_qasm(cfg)
    c = rcs.Circuit.from_qasm(text)
    os.environ.pop("RCS_TC_NOTRANS", None)
    a = rcs.State.build(ctx, c, fuse_k=6, timing=True)
    ra = dict(a.report)
    big = a.n > 30
    ha = a.copy_out(0, 1 << 22) if big else a.copy_out()
    ta = a.copy_out((1 << a.n) - (1 << 22), 1 << 22) if big else None
    del a
    os.environ["RCS_TC_NOTRANS"] = "1"
    b = rcs.State.build(ctx, c, fuse_k=6, timing=True)
    rb = dict(b.report)
    hb = b.copy_out(0, 1 << 22) if big else b.copy_out()
    tb = b.copy_out((1 << b.n) - (1 << 22), 1 << 22) if big else None
    del b
    eq = bool(np.array_equal(ha, hb)) and (ta is None or bool(np.array_equal(ta, tb)))
    md = float(np.abs(ha.astype(np.complex128) - hb).max())
    print(cfg, "bitwise_equal", eq, "maxdiff %.3g" % md, "build_ms K12 %.1f K9 %.1f" % (ra["build_ms"], rb["build_ms"]),
          "norm", ra["norm"], rb["norm"], flush=True)
