"""Small driver for ncu: a few cfg2 primitive calls on one GPU (no timing).

The calls of interest run between cudaProfilerStart/Stop, so
``ncu --profile-from-start off`` sees only them (not the key generation).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "keyswitch"
n_ct = int(sys.argv[2]) if len(sys.argv) > 2 else 4
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
step = bench.PrimitiveStep(torch, 0, n_ct=n_ct)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(reps):
    if what == "ntt":
        step.ntt(step.x, False)
        step.ntt(step.x, True)
    elif what == "fwd":
        step.ntt(step.x, False)
    elif what == "keyswitch":
        step.relin_batch()
    elif what == "rot":
        step.rotations(step.x)
    elif what == "step":
        step.step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done", what)
