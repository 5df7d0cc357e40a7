"""Latency of one ciphertext's rotations at a given level: n sequential srk_rotate calls
against one srk_rotate_hoisted call with n outputs (cfg3 chain, CUDA events)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2412_15126_b200 import _lib  # noqa: E402
from paper_2412_15126_b200.backend_cuda import CudaBackend  # noqa: E402
from paper_2412_15126_b200.keys import sample_secret  # noqa: E402
from paper_2412_15126_b200.params import preset  # noqa: E402

p = preset("cfg3")
be = CudaBackend(p, 0)
be.set_secret(sample_secret(p))
N = p.ring_degree
gal = [pow(5, k, 2 * N) for k in range(1, 16)]
keys = [be.galois_key(g) for g in gal]
ws, s = be.workspace(), be.stream()


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


for level in (29, 20, 12, 5):
    nl = level + 1
    x = torch.randint(0, 1 << 30, (2, nl, N), dtype=torch.int64, device=be.device)
    outs = [torch.empty_like(x) for _ in gal]

    def seq(n):
        for i in range(n):
            _lib.check(be.lib.srk_rotate(be.ctx, x.data_ptr(), keys[i].data_ptr(), outs[i].data_ptr(), level, gal[i], ws, s))

    def hoist(n):
        k = (ctypes.c_void_p * n)(*[keys[i].data_ptr() for i in range(n)])
        g = (ctypes.c_uint64 * n)(*gal[:n])
        o = (ctypes.c_void_p * n)(*[outs[i].data_ptr() for i in range(n)])
        _lib.check(be.lib.srk_rotate_hoisted(be.ctx, x.data_ptr(), 2 * nl * N, 1, n, k, g, o, 2 * nl * N, level, ws, s))

    one = timed(lambda: seq(1))
    print(f"level {level}: one rotation {one:.0f} us; hoisted n=3 {timed(lambda: hoist(3)):.0f} us, "
          f"n=7 {timed(lambda: hoist(7)):.0f} us, n=15 {timed(lambda: hoist(15)):.0f} us")
