"""ctypes wrapper of the CPU RNS-CKKS oracle (oracle/ckks_oracle.c).

TEST INFRASTRUCTURE.  Only tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs may import this module, as the
checker or the CPU baseline; the product (``paper_2412_15126_b200``) never
imports it.

``OracleBackend`` implements the same backend surface as the product's
``CudaBackend`` on host numpy arrays, so ``oracle_engine(params)`` runs the
product's own engine bookkeeping (levels, scales, counters) over the CPU
restatement of every primitive -- the GPU limbs must match it bit for bit.
Parity status: ciphertext level "parity unpinned" (see ckks_oracle.c header);
slot level pinned against the reference simulator through tests/golden/.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from ctypes import POINTER, c_int, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libckks_oracle.so")

_u64 = np.uint64
_lib = None
_lock = threading.Lock()


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                build()
            L = ctypes.CDLL(LIB_PATH)
            P = c_void_p
            sig = {
                "orc_create": ([c_int, P, P, c_int, c_int, c_int], c_void_p),
                "orc_destroy": ([P], None),
                "orc_ntt": ([P, P, c_int, P, c_int], None),
                "orc_addsub": ([P, P, P, P, c_int, c_int], None),
                "orc_add_const": ([P, P, P, P, c_int], None),
                "orc_mul_const": ([P, P, c_int, P, P, c_int], None),
                "orc_mul_plain": ([P, P, P, P, c_int], None),
                "orc_tensor": ([P, P, P, P, c_int], None),
                "orc_rescale": ([P, P, P, c_int], None),
                "orc_automorph": ([P, P, P, c_int, c_uint64], None),
                "orc_keyswitch": ([P, P, P, P, P, c_int], None),
                "orc_mul_relin": ([P, P, P, P, P, c_int], None),
                "orc_mul_relin_rescale": ([P, P, P, P, P, c_int], None),
                "orc_rotate": ([P, P, P, P, c_int, c_uint64], None),
                "orc_rotate_hoisted": ([P, P, P, P, c_int, P, c_int], None),
                "orc_uniform_poly": ([P, P, c_int, P, c_uint64, c_uint64], None),
                "orc_small_to_ntt": ([P, P, P, c_int, P], None),
                "orc_keygen": ([P, P, P, P, c_uint64, c_uint64, P], None),
                "orc_encrypt": ([P, P, P, P, c_uint64, c_uint64, P, c_int], None),
                "orc_decrypt_limb0": ([P, P, P, P, c_int], None),
            }
            for name, (args, res) in sig.items():
                fn = getattr(L, name)
                fn.argtypes = args
                fn.restype = res
            _lib = L
        return _lib


def _p(a: np.ndarray) -> int:
    assert a.flags.c_contiguous
    return a.ctypes.data


def _ids(ids) -> np.ndarray:
    return np.ascontiguousarray(ids, dtype=np.int32)


class OracleCKKS:
    """Thin object wrapper: one C context per parameter set."""

    def __init__(self, params):
        self.params = params
        self.n = params.ring_degree
        primes = np.array(params.all_primes, dtype=_u64)
        roots = np.array(params.roots, dtype=_u64)
        self.L = lib()
        self.ctx = self.L.orc_create(params.log_n, _p(primes), _p(roots), len(params.q_primes),
                                     len(params.p_primes), params.dnum)
        if not self.ctx:
            raise RuntimeError("orc_create failed")
        self.n_q = len(params.q_primes)
        self.n_all = len(params.all_primes)

    def __del__(self):
        try:
            if self.ctx:
                self.L.orc_destroy(self.ctx)
        except Exception:
            pass

    # raw primitives ---------------------------------------------------
    def ntt(self, a: np.ndarray, prime_ids, inverse=False) -> np.ndarray:
        out = np.ascontiguousarray(a, dtype=_u64).copy()
        ids = _ids(prime_ids)
        self.L.orc_ntt(self.ctx, _p(out), len(ids), _p(ids), int(inverse))
        return out

    def tensor(self, a, b, level):
        d = np.empty((3, level + 1, self.n), dtype=_u64)
        self.L.orc_tensor(self.ctx, _p(a), _p(b), _p(d), level)
        return d

    def rescale(self, a, level):
        out = np.empty((2, level, self.n), dtype=_u64)
        self.L.orc_rescale(self.ctx, _p(a), _p(out), level)
        return out

    def keyswitch(self, d, key, level):
        out = np.empty((2, level + 1, self.n), dtype=_u64)
        self.L.orc_keyswitch(self.ctx, _p(d), _p(key), _p(out[0]), _p(out[1]), level)
        return out

    def mul_relin(self, a, b, rlk, level):
        out = np.empty((2, level + 1, self.n), dtype=_u64)
        self.L.orc_mul_relin(self.ctx, _p(a), _p(b), _p(rlk), _p(out), level)
        return out

    def mul_relin_rescale(self, a, b, rlk, level):
        """HMult + relinearisation with the rescale fused into the ModDown."""
        out = np.empty((2, level, self.n), dtype=_u64)
        self.L.orc_mul_relin_rescale(self.ctx, _p(a), _p(b), _p(rlk), _p(out), level)
        return out

    def automorph(self, a, galois):
        out = np.empty_like(a)
        nl = a.size // self.n
        self.L.orc_automorph(self.ctx, _p(a), _p(out), nl, galois)
        return out

    def rotate_raw(self, a, gkey, galois, level):
        out = np.empty((2, level + 1, self.n), dtype=_u64)
        self.L.orc_rotate(self.ctx, _p(a), _p(gkey), _p(out), level, galois)
        return out

    def rotate_hoisted_raw(self, a, gkeys, galois, level):
        """Rotations of one ciphertext sharing one base extension; each output
        is bit-identical to rotate_raw (ckks_oracle.c orc_rotate_hoisted)."""
        r = len(galois)
        outs = [np.empty((2, level + 1, self.n), dtype=_u64) for _ in range(r)]
        kp = np.array([_p(k) for k in gkeys], dtype=_u64)
        op = np.array([_p(o) for o in outs], dtype=_u64)
        g = np.array([int(x) for x in galois], dtype=_u64)
        self.L.orc_rotate_hoisted(self.ctx, _p(a), _p(kp), _p(g), r, _p(op), level)
        return outs

    def uniform(self, n_limbs, prime_ids, seed, stream_base):
        out = np.empty((n_limbs, self.n), dtype=_u64)
        ids = _ids(prime_ids)
        self.L.orc_uniform_poly(self.ctx, _p(out), n_limbs, _p(ids), seed, stream_base)
        return out

    def small_to_ntt(self, v, prime_ids):
        v = np.ascontiguousarray(v, dtype=np.int64)
        ids = _ids(prime_ids)
        out = np.empty((len(ids), self.n), dtype=_u64)
        self.L.orc_small_to_ntt(self.ctx, _p(v), _p(out), len(ids), _p(ids))
        return out

    def keygen(self, s_ntt, sfrom_ntt, e, seed, key_id):
        key = np.empty((self.params.dnum, 2, self.n_all, self.n), dtype=_u64)
        e = np.ascontiguousarray(e, dtype=np.int64)
        self.L.orc_keygen(self.ctx, _p(s_ntt), _p(sfrom_ntt), _p(e), seed, key_id, _p(key))
        return key


def _batched(fn):
    """Run a single-ciphertext oracle op over a batch (leading axis) element by element."""

    def wrapper(self, a, *args, batch=None, each=False, **kw):
        if batch is None:
            return fn(self, a, *args, **kw)
        outs = []
        for i in range(batch):
            rest = list(args)
            if rest and isinstance(rest[0], np.ndarray) and rest[0].ndim == a.ndim:
                rest[0] = rest[0][i]  # second ciphertext operand (add/sub/mul)
            elif each and rest and isinstance(rest[0], np.ndarray):
                rest[0] = rest[0][i]  # per-ciphertext plaintext
            outs.append(fn(self, np.ascontiguousarray(a[i]), *rest, **kw))
        return np.stack(outs)

    return wrapper


class OracleBackend:
    """CPU restatement of ``CudaBackend``'s surface (numpy uint64 arrays)."""

    kind = "oracle"

    def __init__(self, params):
        from paper_2412_15126_b200.keys import KEY_RELIN

        self.params = params
        self.o = OracleCKKS(params)
        self.n = params.ring_degree
        self._keys = {}
        self._key_relin = KEY_RELIN
        self._lock = threading.Lock()
        self.launches = 0

    def set_secret(self, s):
        self.sk = self.o.small_to_ntt(s, range(self.o.n_all))

    def _keygen(self, key_id, sfrom):
        from paper_2412_15126_b200.keys import sample_error

        e = sample_error(self.params, (2, key_id), self.params.dnum)
        return self.o.keygen(self.sk, sfrom, e, self.params.seed, key_id)

    def relin_key(self):
        with self._lock:
            if self._key_relin not in self._keys:
                q = np.array(self.params.all_primes, dtype=object)
                s2 = np.empty_like(self.sk)
                for i, p in enumerate(self.params.all_primes):
                    s2[i] = ((self.sk[i].astype(object) ** 2) % p).astype(_u64)
                self._keys[self._key_relin] = self._keygen(self._key_relin, s2)
            return self._keys[self._key_relin]

    def galois_key(self, galois):
        from paper_2412_15126_b200.keys import galois_key_id

        kid = galois_key_id(galois)
        with self._lock:
            if kid not in self._keys:
                sg = self.o.automorph(self.sk, galois)
                self._keys[kid] = self._keygen(kid, sg)
            return self._keys[kid]

    def to_host(self, data):
        return data

    def encrypt(self, m, e, seq, level):
        ids = range(level + 1)
        m_ntt = self.o.small_to_ntt(m, ids)
        out = np.empty((2, level + 1, self.n), dtype=_u64)
        e = np.ascontiguousarray(e, dtype=np.int64)
        self.o.L.orc_encrypt(self.o.ctx, _p(m_ntt), _p(self.sk), _p(e), self.params.seed, seq,
                             _p(out), level)
        return out

    def decrypt_limb0(self, data, level):
        m = np.empty(self.n, dtype=np.int64)
        self.o.L.orc_decrypt_limb0(self.o.ctx, _p(data), _p(self.sk), _p(m), level)
        return m

    def encode_plain(self, coeffs, level):
        return self.o.small_to_ntt(coeffs, range(level + 1))

    @_batched
    def addsub(self, a, b, level, op):
        out = np.empty((2, level + 1, self.n), dtype=_u64)
        self.o.L.orc_addsub(self.o.ctx, _p(a), _p(b) if b is not None else _p(a), _p(out), level, op)
        return out

    @_batched
    def add_const(self, a, residues, level):
        out = np.empty_like(a)
        k = np.array([int(r) for r in residues], dtype=_u64)
        self.o.L.orc_add_const(self.o.ctx, _p(a), _p(k), _p(out), level)
        return out

    @_batched
    def add_plain(self, a, pt, level):
        out = a.copy()
        q = np.array(self.params.q_primes[: level + 1], dtype=_u64)[:, None]
        s = out[0] + pt
        out[0] = np.where(s >= q, s - q, s)
        return out

    @_batched
    def mul_const_rescale(self, a, src_level, residues, level):
        k = np.array([int(r) for r in residues], dtype=_u64)
        tmp = np.empty((2, level + 1, self.n), dtype=_u64)
        self.o.L.orc_mul_const(self.o.ctx, _p(a), src_level + 1, _p(k), _p(tmp), level)
        return self.o.rescale(tmp, level)

    @_batched
    def mul_plain_rescale(self, a, pt, level):
        tmp = np.empty_like(a)
        self.o.L.orc_mul_plain(self.o.ctx, _p(a), _p(pt), _p(tmp), level)
        return self.o.rescale(tmp, level)

    @_batched
    def mul_relin_rescale(self, a, b, level):
        return self.o.mul_relin_rescale(np.ascontiguousarray(a), np.ascontiguousarray(b), self.relin_key(),
                                        level)

    def mul_relin_rescale_pairs(self, pairs, level):
        return np.stack([self.mul_relin_rescale(a, b, level) for a, b in pairs])

    @_batched
    def rotate(self, a, galois, level):
        return self.o.rotate_raw(a, self.galois_key(galois), galois, level)

    @_batched
    def rescale(self, a, level):
        return self.o.rescale(np.ascontiguousarray(a), level)

    def lincomb(self, terms, term_levels, residues, level, batch=None):
        """sum_i k_i T_i over limbs 0..level, term by term (mul_const + add)."""
        if batch is not None:
            return np.stack([self.lincomb([t[i] for t in terms], term_levels, residues, level)
                             for i in range(batch)])
        acc = None
        for t, lv, res in zip(terms, term_levels, residues):
            k = np.array([int(r) for r in res], dtype=_u64)
            prod = np.empty((2, level + 1, self.n), dtype=_u64)
            self.o.L.orc_mul_const(self.o.ctx, _p(np.ascontiguousarray(t)), lv + 1, _p(k), _p(prod), level)
            if acc is None:
                acc = prod
            else:
                nxt = np.empty_like(acc)
                self.o.L.orc_addsub(self.o.ctx, _p(acc), _p(prod), _p(nxt), level, 0)
                acc = nxt
        return acc

    def stack(self, datas):
        return np.stack(datas)

    def index(self, data, i):
        return np.ascontiguousarray(data[i])

    def slice(self, data, a, b):
        return np.ascontiguousarray(data[a:b])

    def stack_plain(self, pts):
        return np.stack(pts)

    # collectives (paper_2412_15126_b200/shard.py) over gloo
    def as_tensor(self, data):
        import torch

        return torch.from_numpy(np.ascontiguousarray(data).view(np.int64).copy())

    def zeros_tensor(self, level):
        import torch

        return torch.zeros((2, level + 1, self.n), dtype=torch.int64)

    def from_tensor(self, t, level):
        return t.numpy().view(np.uint64).copy()

    def reduce_mod_tensor(self, t, level):
        q = np.array(self.params.q_primes[: level + 1], dtype=np.uint64)[None, :, None]
        return t.numpy().view(np.uint64) % q


def oracle_engine(params):
    """The product's engine bookkeeping over the CPU oracle backend (tests only)."""
    from paper_2412_15126_b200.engine import CKKSEngineCore

    return CKKSEngineCore(params, OracleBackend(params))
