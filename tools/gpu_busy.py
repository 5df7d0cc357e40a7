"""GPU busy time vs wall time of a pipeline (torch.profiler / CUPTI kernel records).

usage: python tools/gpu_busy.py rank|sort256|argmin"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_15126_b200 as M  # noqa: E402
from paper_2412_15126_b200.params import preset  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "rank"
if what == "rank":
    eng = M.B200Engine(preset("cfg3"))
    v = np.random.default_rng(0).choice(1024, 128, replace=False) / 1024
    cfg = M.KernelConfig(mode="composite", composite=(4, 2))
    ct = eng.encrypt(v)
    run = lambda: M.rank(eng, ct, 128, cfg).ranks  # noqa: E731
else:
    nv = int(what[4:] or 256)
    eng = M.B200Engine(preset("long"))
    v = np.random.default_rng(0).choice(8 * nv, nv, replace=False) / (8 * nv)
    cfg = M.SortConfig(kernel=M.KernelConfig(mode="composite", composite=(6, 2), indicator_composite=(6, 2)),
                       tie_correction=False)
    bv = M.block_split(eng, v)
    run = lambda: M.multi_sort(eng, bv, cfg)  # noqa: E731
run()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    run()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
iv = sorted((e.time_range.start, e.time_range.end) for e in ev)
busy, cur_s, cur_e = 0.0, None, None
for s, e in iv:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
if cur_e is not None:
    busy += cur_e - cur_s
span = (iv[-1][1] - iv[0][0]) if iv else 0
print(f"{what}: wall {wall * 1e3:.2f} ms, GPU span {span / 1e3:.2f} ms, GPU busy (union of kernels) {busy / 1e3:.2f} ms, "
      f"{len(iv)} device records, sum of durations {sum(e - s for s, e in iv) / 1e3:.2f} ms")
