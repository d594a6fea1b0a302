#!/usr/bin/env python
"""Build one config's state twice (the second build is the one to profile) and print its per-pass
times: python scripts/c3_build.py [config] [--tma auto|bulk] [--k9]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_07311_b200 as rcs  # noqa: E402
from rcs_workload import config_qasm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="c3")
ap.add_argument("--tma", default="auto")
ap.add_argument("--k9", action="store_true")
a = ap.parse_args()
c = rcs.Circuit.from_qasm(config_qasm(a.config))
ctx = rcs.Context(0)
kw = dict(fuse_k=6, timing=True, tc_tma=a.tma, tc_kernel="k9" if a.k9 else "auto")
st = rcs.State.build(ctx, c, **kw)
amps, scratch = st.amps, st.scratch
st.free()
st = rcs.State.build(ctx, c, amps=amps, scratch=scratch, **kw)
t = st.pass_times()
print(a.config, a.tma, "passes", len(t), "sum ms %.2f" % t.sum(), " ".join("%.2f" % x for x in t))
