"""CUDA-graph replay of a whole pipeline vs the eager run (paper_2412_15126_b200.graphs).

usage: python tools/graph_pipe.py rank|argmin|sort256|sort1024"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_15126_b200 as M  # noqa: E402
from paper_2412_15126_b200.graphs import CapturedPipeline  # noqa: E402
from paper_2412_15126_b200.params import preset  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "rank"
if what == "rank":
    eng = M.B200Engine(preset("cfg3"))
    v = np.random.default_rng(0).choice(1024, 128, replace=False) / 1024
    cfg = M.KernelConfig(mode="composite", composite=(4, 2))
    x = eng.encrypt(v)
    fn = lambda c: M.rank(eng, c, 128, cfg).ranks  # noqa: E731
elif what == "argmin":
    eng = M.B200Engine(preset("long"))
    v = np.random.default_rng(0).choice(1024, 128, replace=False) / 1024
    cfg = M.KernelConfig(mode="composite", composite=(4, 2), indicator_composite=(4, 2))
    x = eng.encrypt(v)
    fn = lambda c: M.order_statistic_mask(eng, c, 128, M.StatisticQuery("min"), cfg)  # noqa: E731
else:
    nv = int(what[4:] or 256)
    eng = M.B200Engine(preset("long"))
    v = np.random.default_rng(0).choice(8 * nv, nv, replace=False) / (8 * nv)
    cfg = M.SortConfig(kernel=M.KernelConfig(mode="composite", composite=(6, 2), indicator_composite=(6, 2)),
                       tie_correction=False)
    x = M.block_split(eng, v)
    fn = lambda c: M.multi_sort(eng, c, cfg)  # noqa: E731

ref = [d.clone() for d in __import__("paper_2412_15126_b200.graphs", fromlist=["_datas"])._datas(fn(x))]
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    fn(x)
torch.cuda.synchronize()
eager = (time.perf_counter() - t0) / 3
cap = CapturedPipeline(eng, fn, x, release_cache=what.startswith("sort"))
cap.replay()
torch.cuda.synchronize()
from paper_2412_15126_b200.graphs import _datas  # noqa: E402
assert all(torch.equal(a, b) for a, b in zip(_datas(cap.output), ref)), "graph replay differs"
t0 = time.perf_counter()
for _ in range(5):
    cap.replay(x)
torch.cuda.synchronize()
gr = (time.perf_counter() - t0) / 5
print(f"{what}: eager {eager * 1e3:.2f} ms, graph replay {gr * 1e3:.2f} ms, bit-identical")
