import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
sys.path.insert(0, '/root/repo/tests')
from test_gpu_primitives import rand_limbs, dev, host, call, ptr, rot_layout, _key
from paper_2412_15126_b200.params import preset
from paper_2412_15126_b200.backend_cuda import CudaBackend
from oracle.oracle import OracleCKKS
for name in ["cfg1", "toy"]:
    p = preset(name); gb = CudaBackend(p); orc = OracleCKKS(p)
    lvl = p.max_level; n = p.ring_degree; ps = (lvl + 1) * n
    key = _key(p, 42); g = pow(5, 5, 2 * n); tr = rot_layout(gb, key, g)
    for B in (1, 2, 3, 8, 9):
        a = rand_limbs(p, (B, 2), lvl, 40); ta = dev(gb, a)
        out = gb.empty_ct(lvl, polys=2 * B)
        call(gb, "srk_rotate_batch", ptr(ta), 2 * ps, ptr(tr), ptr(out), 2 * ps, B, lvl, g, gb.workspace(), gb.stream())
        got = host(gb, out).reshape(B, 2, lvl + 1, n)
        bad = [i for i in range(B) if not np.array_equal(got[i], orc.rotate_raw(a[i], key, g, lvl))]
        print(name, B, "bad:", bad)
    # relin batch
    for B in (1, 2):
        a = rand_limbs(p, (B, 2), lvl, 40); b = rand_limbs(p, (B, 2), lvl, 41)
        ta, tb, tk = dev(gb, a), dev(gb, b), dev(gb, key)
        out = gb.empty_ct(lvl, polys=2 * B)
        call(gb, "srk_mul_relin_batch", ptr(ta), ptr(tb), 2 * ps, ptr(tk), ptr(out), 2 * ps, B, lvl, 0, gb.workspace(), gb.stream())
        got = host(gb, out).reshape(B, 2, lvl + 1, n)
        bad = [i for i in range(B) if not np.array_equal(got[i], orc.mul_relin(a[i], b[i], key, lvl))]
        print(name, 'relin', B, "bad:", bad)
