"""Time the 64-ciphertext forward/inverse NTT and 64 HMult+relin for the library at $SRK_LIB."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

step = bench.PrimitiveStep(torch, 0)
for _ in range(3):
    step.ntt(step.x, False)
f = bench.time_region(torch, lambda: step.ntt(step.x, False), 5)
i = bench.time_region(torch, lambda: step.ntt(step.x, True), 5)
r = bench.time_region(torch, step.relin_batch, 3)
rot = bench.time_region(torch, lambda: step.rotations(step.x), 2)
print(f"{os.environ.get('SRK_LIB', 'default')} pipe={os.environ.get('SRK_NTT_PIPE', '0')}: "
      f"fwd {f:.3f} ms inv {i:.3f} ms relin64 {r:.3f} ms rot15x64 {rot:.3f} ms")
