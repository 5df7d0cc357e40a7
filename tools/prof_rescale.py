"""ncu driver: one batched rescale of 64 cfg2 ciphertexts (the fused FP64 rescale passes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

step = bench.PrimitiveStep(torch, 0, n_ct=64)
p = step.p
L = step.nl - 1
ct = 2 * step.nl * p.ring_degree
s = step.be.stream()
run = lambda: step._c("srk_rescale_batch", step.prod.data_ptr(), ct, step.res.data_ptr(),  # noqa: E731
                      2 * L * p.ring_degree, step.n_ct, L, step.ws, s)
run()
torch.cuda.synchronize()
torch.cuda.profiler.start()
run()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
