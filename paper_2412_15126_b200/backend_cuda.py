"""Device-resident RNS-CKKS backend: torch owns HBM, libslotrank_b200 computes.

Ciphertexts are ``torch.int64`` tensors of shape [2, level+1, N] holding the
uint64 limbs bit for bit (torch has no unsigned 64-bit arithmetic; the kernels
reinterpret the storage).  Evaluation keys are [dnum, 2, n_q+n_p, N] tensors
generated on the device the first time a Galois element is used and kept
for the engine's lifetime (keys are read-only, shared by every stream).
All launches go to the caller's current torch CUDA stream; the engine's
workspace is used stream-ordered, one workspace per stream.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np
import torch

from . import _lib
from .keys import KEY_RELIN, galois_key_id, sample_error
from .params import CKKSParams

__all__ = ["CudaBackend"]


def _ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


def _u64_array(values) -> ctypes.Array:
    arr = (ctypes.c_uint64 * len(values))()
    for i, v in enumerate(values):
        arr[i] = int(v)
    return arr


class CudaBackend:
    """One CUDA context (tables, keys, workspaces) per parameter set and device."""

    kind = "cuda"

    def __init__(self, params: CKKSParams, device: int | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("B200 backend needs a CUDA device; none is visible")
        self.params = params
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.lib = _lib.lib()
        primes = params.all_primes
        roots = params.roots
        ctx = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(
                self.lib.srk_ctx_create(
                    self.device.index,
                    params.log_n,
                    _u64_array(primes),
                    _u64_array(roots),
                    len(params.q_primes),
                    len(params.p_primes),
                    params.dnum,
                    ctypes.byref(ctx),
                )
            )
        self.ctx = ctx
        self.n = params.ring_degree
        self._ws_bytes = int(self.lib.srk_workspace_bytes(self.ctx))
        self._ws: dict[int, torch.Tensor] = {}
        self._keys: dict[int, torch.Tensor] = {}
        self._capture_keepalive: list = []  # pinned sources of copies captured in CUDA graphs
        self._key_lock = threading.Lock()
        self._call_lock = threading.RLock()
        self._branch = None  # second stream for engine.parallel (run_parallel)
        self._tls = threading.local()
        self.launches = 0
        self._sk_ntt = None

    def __del__(self):
        try:
            if getattr(self, "ctx", None) is not None and self.ctx.value:
                torch.cuda.synchronize(self.device)
                self.lib.srk_ctx_destroy(self.ctx)
                self.ctx = None
        except Exception:
            pass

    # ------------------------------------------------------------------
    # plumbing
    # ------------------------------------------------------------------
    def stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def workspace(self) -> int:
        s = self.stream()
        ws = self._ws.get(s)
        if ws is None:
            ws = torch.empty(self._ws_bytes, dtype=torch.uint8, device=self.device)
            self._ws[s] = ws
        return _ptr(ws)

    def run_parallel(self, first, second):
        """first() on the current stream, second() on the backend's branch stream (forked
        before first's work is enqueued, joined after second's), each with its own
        key-switch workspace.  Every use of the branch stream starts by waiting on the
        current stream's tail and ends joined into it, so tensors crossing the two
        streams are never recycled by the caching allocator while the other stream
        can still touch them; also valid inside a CUDA-graph capture (fork / join
        edges).  Nested calls (already on the branch stream) run in turn."""
        if getattr(self._tls, "in_branch", False) or os.environ.get("SRK_BRANCH", "1") == "0":
            return first(), second()
        main = torch.cuda.current_stream(self.device)
        if self._branch is None:
            self._branch = torch.cuda.Stream(self.device)
            _lib.check(self.lib.srk_ctx_set_branch_stream(self.ctx, self._branch.cuda_stream))
        side = self._branch
        side.wait_stream(main)
        a = first()
        self._tls.in_branch = True
        try:
            with torch.cuda.stream(side):
                b = second()
        finally:
            self._tls.in_branch = False
        main.wait_stream(side)
        return a, b

    def release_workspace(self, stream_handle: int) -> None:
        """Drop the key-switch workspace cached for a stream that is going away."""
        self._ws.pop(stream_handle, None)

    def empty_ct(self, level: int, polys: int = 2) -> torch.Tensor:
        return torch.empty((polys, level + 1, self.n), dtype=torch.int64, device=self.device)

    def _h2d(self, arr: np.ndarray) -> torch.Tensor:
        """Host array -> device.  Under CUDA-graph capture the source is pinned and
        kept alive with the backend (the captured copy node re-reads it on replay)."""
        t = torch.from_numpy(np.ascontiguousarray(arr))
        if torch.cuda.is_current_stream_capturing():
            t = t.pin_memory()
            self._capture_keepalive.append(t)
            return t.to(self.device, non_blocking=True)
        return t.to(self.device)

    def to_host(self, data: torch.Tensor) -> np.ndarray:
        return data.cpu().numpy().view(np.uint64)

    def from_host(self, arr: np.ndarray) -> torch.Tensor:
        return self._h2d(np.ascontiguousarray(arr).view(np.int64))

    def _call(self, name: str, *args):
        # one C-ABI call enqueues a whole op (several kernels, the context's side
        # streams and events); ctypes releases the GIL, so concurrent host threads
        # (ops on distinct inputs may run concurrently, reference SPEC.md:121) are
        # serialised here -- each op's launch sequence stays contiguous
        with self._call_lock:
            self.launches += 1
            _lib.check(getattr(self.lib, name)(self.ctx, *args))

    # ------------------------------------------------------------------
    # keys
    # ------------------------------------------------------------------
    def set_secret(self, s: np.ndarray):
        np_all = len(self.params.all_primes)
        s_dev = torch.from_numpy(s.astype(np.int64)).to(self.device)
        sk = torch.empty((np_all, self.n), dtype=torch.int64, device=self.device)
        self._call("srk_small_to_ntt", _ptr(s_dev), _ptr(sk), np_all, 0, self.stream())
        self._sk_ntt = sk

    def _keygen(self, key_id: int, sfrom: torch.Tensor) -> torch.Tensor:
        p = self.params
        np_all = len(p.all_primes)
        e = sample_error(p, (2, key_id), p.dnum)
        e_dev = torch.from_numpy(e).to(self.device)
        key = torch.empty((p.dnum, 2, np_all, self.n), dtype=torch.int64, device=self.device)
        self._call("srk_keygen", _ptr(self._sk_ntt), _ptr(sfrom), _ptr(e_dev), p.seed, key_id,
                   _ptr(key), self.workspace(), self.stream())
        return key

    def relin_key(self) -> torch.Tensor:
        with self._key_lock:
            k = self._keys.get(KEY_RELIN)
            if k is None:
                np_all = len(self.params.all_primes)
                s2 = torch.empty_like(self._sk_ntt)
                self._call("srk_square", _ptr(self._sk_ntt), _ptr(s2), np_all, self.stream())
                k = self._keygen(KEY_RELIN, s2)
                self._keys[KEY_RELIN] = k
            return k

    def galois_key(self, galois: int) -> torch.Tensor:
        kid = galois_key_id(galois)
        with self._key_lock:
            k = self._keys.get(kid)
            if k is None:
                # rotation layout: sigma_g(s) -> s switching key, limbs permuted by sigma_g^-1
                p = self.params
                np_all = len(p.all_primes)
                e = sample_error(p, (2, kid), p.dnum)
                e_dev = torch.from_numpy(e).to(self.device)
                k = torch.empty((p.dnum, 2, np_all, self.n), dtype=torch.int64, device=self.device)
                self._call("srk_keygen_galois", _ptr(self._sk_ntt), _ptr(e_dev), p.seed, kid, galois,
                           _ptr(k), self.workspace(), self.stream())
                self._keys[kid] = k
            return k

    def key_bytes(self) -> int:
        return sum(k.numel() * 8 for k in self._keys.values())

    # ------------------------------------------------------------------
    # ciphertext primitives (see engine.py for the level/scale policy)
    # ------------------------------------------------------------------
    def encrypt(self, m: np.ndarray, e: np.ndarray, seq: int, level: int) -> torch.Tensor:
        out = self.empty_ct(level)
        m_dev = torch.from_numpy(np.ascontiguousarray(m, dtype=np.int64)).to(self.device)
        e_dev = torch.from_numpy(np.ascontiguousarray(e, dtype=np.int64)).to(self.device)
        self._call("srk_encrypt", _ptr(m_dev), _ptr(self._sk_ntt), _ptr(e_dev), self.params.seed,
                   seq, _ptr(out), level, self.workspace(), self.stream())
        return out

    def decrypt_limb0(self, data: torch.Tensor, level: int) -> np.ndarray:
        m = torch.empty(self.n, dtype=torch.int64, device=self.device)
        self._call("srk_decrypt_limb0", _ptr(data), _ptr(self._sk_ntt), _ptr(m), level,
                   self.workspace(), self.stream())
        return m.cpu().numpy()

    def encode_plain(self, coeffs: np.ndarray, level: int) -> torch.Tensor:
        c = self._h2d(np.ascontiguousarray(coeffs, dtype=np.int64))
        pt = torch.empty((level + 1, self.n), dtype=torch.int64, device=self.device)
        self._call("srk_encode_plain", _ptr(c), _ptr(pt), level, self.stream())
        return pt

    # batched ciphertexts: data [B][2][level+1][N]; batch=None -> [2][level+1][N]
    def _out(self, level: int, batch) -> torch.Tensor:
        shape = (2, level + 1, self.n) if batch is None else (batch, 2, level + 1, self.n)
        return torch.empty(shape, dtype=torch.int64, device=self.device)

    def stack(self, datas) -> torch.Tensor:
        return torch.stack(datas)

    def index(self, data, i: int) -> torch.Tensor:
        return data[i]

    def slice(self, data, a: int, b: int) -> torch.Tensor:
        return data[a:b]  # contiguous view: the C-ABI sees data_ptr() of row a

    def stack_plain(self, pts) -> torch.Tensor:
        return torch.stack(pts)

    def addsub(self, a, b, level: int, op: int, batch=None) -> torch.Tensor:
        out = self._out(level, batch)
        self._call("srk_addsub_batch", _ptr(a), _ptr(b) if b is not None else 0, _ptr(out), batch or 1,
                   level, op, self.stream())
        return out

    def add_const(self, a, residues, level: int, batch=None) -> torch.Tensor:
        out = self._out(level, batch)
        self._call("srk_add_plain_batch", _ptr(a), 0, 0, _u64_array(residues), _ptr(out), batch or 1,
                   level, self.stream())
        return out

    def add_plain(self, a, pt, level: int, batch=None, each=False) -> torch.Tensor:
        out = self._out(level, batch)
        pt_ct = (level + 1) * self.n if each else 0
        self._call("srk_add_plain_batch", _ptr(a), _ptr(pt), pt_ct, None, _ptr(out), batch or 1, level,
                   self.stream())
        return out

    def mul_const_rescale(self, a, src_level: int, residues, level: int, batch=None) -> torch.Tensor:
        """rescale(view_level(a) * k): output at level-1."""
        out = self._out(level - 1, batch)
        self._call("srk_mul_const_rescale_batch", _ptr(a), 2 * (src_level + 1) * self.n, src_level + 1,
                   _u64_array(residues), _ptr(out), batch or 1, level, self.workspace(), self.stream())
        return out

    def mul_plain_rescale(self, a, pt, level: int, batch=None, each=False) -> torch.Tensor:
        out = self._out(level - 1, batch)
        pt_ct = (level + 1) * self.n if each else 0
        self._call("srk_mul_plain_rescale_batch", _ptr(a), _ptr(pt), pt_ct, _ptr(out), batch or 1, level,
                   self.workspace(), self.stream())
        return out

    def mul_relin_rescale(self, a, b, level: int, batch=None) -> torch.Tensor:
        out = self._out(level - 1, batch)
        ct = 2 * (level + 1) * self.n
        self._call("srk_mul_relin_batch", _ptr(a), _ptr(b), ct, _ptr(self.relin_key()), _ptr(out),
                   2 * level * self.n, batch or 1, level, 1, self.workspace(), self.stream())
        return out

    def mul_relin_rescale_pairs(self, pairs, level: int) -> torch.Tensor:
        """a_i x b_i for every (a_i, b_i) in ``pairs`` (each a [2][level+1][N] ciphertext,
        operands may repeat), relinearised and rescaled, packed [len][2][level][N]:
        one pointer table, no copy of the operands into a batch first."""
        n = len(pairs)
        out = self._out(level - 1, n)
        ta = (ctypes.c_void_p * n)(*[_ptr(a) for a, _ in pairs])
        tb = (ctypes.c_void_p * n)(*[_ptr(b) for _, b in pairs])
        self._call("srk_mul_relin_ptrs", ta, tb, n, _ptr(self.relin_key()), _ptr(out), 2 * level * self.n,
                   level, 1, self.workspace(), self.stream())
        return out

    def rescale(self, a, level: int, batch=None) -> torch.Tensor:
        out = self._out(level - 1, batch)
        self._call("srk_rescale_batch", _ptr(a), 2 * (level + 1) * self.n, _ptr(out),
                   2 * level * self.n, batch or 1, level, self.workspace(), self.stream())
        return out

    def lincomb(self, terms, term_levels, residues, level: int, batch=None) -> torch.Tensor:
        """sum_i k_i T_i over limbs 0..level (no rescale); residues: [n_terms][level+1] ints."""
        n_t = len(terms)
        out = self._out(level, batch)
        k = np.array([[int(r) for r in row] for row in residues], dtype=np.uint64).view(np.int64)
        k_dev = self._h2d(k)
        ptrs = (ctypes.c_void_p * n_t)(*[_ptr(t) for t in terms])
        limbs = (ctypes.c_int * n_t)(*[lv + 1 for lv in term_levels])
        self._call("srk_lincomb", ptrs, limbs, n_t, _ptr(k_dev), _ptr(out), batch or 1, level,
                   self.stream())
        return out

    def lincomb_multi(self, terms, term_levels, residues_rows, level: int, batch=None) -> list:
        """Several sums over the SAME terms: out_l = sum_i k[l][i] T_i (no rescale);
        residues_rows: [n_out][n_terms][level+1] ints.  One pass over the terms per
        eight outputs (srk_lincomb_multi).  Unbatched terms: ONE tensor [n_out][2][level+1][N];
        batched terms: a list of n_out tensors."""
        n_t, n_o = len(terms), len(residues_rows)
        if batch is None:  # one stacked tensor: the caller rescales all sums in one batched call
            block = self._out(level, n_o)
            outs = [block[i] for i in range(n_o)]
        else:
            block, outs = None, [self._out(level, batch) for _ in range(n_o)]
        k = np.array([[[int(r) for r in row] for row in rows] for rows in residues_rows],
                     dtype=np.uint64).view(np.int64)
        k_dev = self._h2d(k)
        # k / q_j for the FP64 path of the limbs under primes < 2^41 (exact there: k < 2^41)
        q = np.array(self.params.q_primes[: level + 1], dtype=np.float64)
        kf_dev = self._h2d(np.ascontiguousarray(k.view(np.uint64).astype(np.float64) / q).view(np.int64))
        ptrs = (ctypes.c_void_p * n_t)(*[_ptr(t) for t in terms])
        limbs = (ctypes.c_int * n_t)(*[lv + 1 for lv in term_levels])
        optrs = (ctypes.c_void_p * n_o)(*[_ptr(o) for o in outs])
        self._call("srk_lincomb_multi", ptrs, limbs, n_t, _ptr(k_dev), _ptr(kf_dev), optrs, n_o, batch or 1,
                   level, self.stream())
        return outs if block is None else block

    def rotate(self, a, galois: int, level: int, batch=None) -> torch.Tensor:
        key = self.galois_key(galois)
        out = self._out(level, batch)
        ct = 2 * (level + 1) * self.n
        self._call("srk_rotate_batch", _ptr(a), ct, _ptr(key), _ptr(out), ct, batch or 1, level, galois,
                   self.workspace(), self.stream())
        return out

    def mod_drop(self, a, src_level: int, level: int) -> torch.Tensor:
        return a[:, : level + 1, :].contiguous()

    # collectives (shard.py): limbs travel as int64 tensors on this device
    def as_tensor(self, data) -> torch.Tensor:
        return data.clone()

    def zeros_tensor(self, level: int) -> torch.Tensor:
        return torch.zeros((2, level + 1, self.n), dtype=torch.int64, device=self.device)

    def from_tensor(self, t, level: int) -> torch.Tensor:
        return t

    def reduce_mod_tensor(self, t, level: int) -> torch.Tensor:
        self._call("srk_reduce_mod", _ptr(t), 2, level, self.stream())
        return t
