"""Small driver for ncu: a few cfg2 primitive calls on one GPU (no timing)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "keyswitch"
n_ct = int(sys.argv[2]) if len(sys.argv) > 2 else 4
step = bench.PrimitiveStep(torch, 0, n_ct=n_ct)
for _ in range(2):
    if what == "ntt":
        step.ntt(step.x, False)
        step.ntt(step.x, True)
    elif what == "keyswitch":
        step.relin_batch()
    elif what == "rot":
        step.rotations(step.x)
    elif what == "step":
        step.step()
torch.cuda.synchronize()
print("done", what)
