import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2412_15126_b200 as M
from paper_2412_15126_b200.params import preset
eng = M.B200Engine(preset("long"))
v = np.random.default_rng(0).choice(1024, 128, replace=False) / 1024
cfg = M.KernelConfig(mode="composite", composite=(4, 2), indicator_composite=(4, 2), tie_margin=2.0 ** -11)
ct = eng.encrypt(v)
M.order_statistic_mask(eng, ct, 128, M.StatisticQuery("min"), cfg)
torch.cuda.synchronize()
torch.cuda.profiler.start()
M.order_statistic_mask(eng, ct, 128, M.StatisticQuery("min"), cfg)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(eng.cost_snapshot())
