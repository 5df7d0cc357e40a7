"""Latency of rank N=128 with the reference's Chebyshev comparison (d=1024), eager and graph."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_15126_b200 as M  # noqa: E402
from paper_2412_15126_b200.graphs import CapturedPipeline  # noqa: E402
from paper_2412_15126_b200.params import preset  # noqa: E402

eng = M.B200Engine(preset("cfg3"))
v = np.random.default_rng(0).choice(1024, 128, replace=False) / 1024
cfg = M.KernelConfig(mode="chebyshev", degree=1024)
x = eng.encrypt(v)
fn = lambda c: M.rank(eng, c, 128, cfg).ranks  # noqa: E731
fn(x)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    fn(x)
torch.cuda.synchronize()
eager = (time.perf_counter() - t0) / 3
cap = CapturedPipeline(eng, fn, x)
cap.replay()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    cap.replay()
torch.cuda.synchronize()
print(f"rank N=128 chebyshev d=1024: eager {eager * 1e3:.2f} ms, graph {(time.perf_counter() - t0) / 3 * 1e3:.2f} ms")
