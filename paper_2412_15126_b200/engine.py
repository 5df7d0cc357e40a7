"""B200Engine -- RNS-CKKS drop-in for the reference ``HESimulator``.

The reference's algorithm modules talk to their engine only through the
method surface of ``HESimulator`` (reference ``pkg/src/slotrank/engine.py:
133-328``).  ``B200Engine`` exposes exactly that surface
-- ``encrypt/decrypt/plain/add/sub/negate/add_plain/mul/mul_plain/rotate/
ideal_map/note_*/cost_*/rotation_offsets`` plus ``params.slot_count`` /
``params.max_level`` -- with identical level semantics, counters, trace and
exceptions, but every ciphertext is a real RNS-CKKS ciphertext in HBM and
every operation runs on the hand-written sm_100a kernels of
``libslotrank_b200.so``.

Level / scale policy (shared by every backend, so results are bit-identical
between the GPU and the CPU oracle for the same op sequence):

* a level-l ciphertext has nominal scale ``params.scales[l]``;
* ``mul`` aligns both operands to min level l, multiplies, relinearises and
  rescales by q_l -> level l-1, scale scales[l]^2/q_l == scales[l-1];
* ``mul_plain`` multiplies by the plaintext encoded at scale
  scales[l-1] q_l / scales[l] and rescales -> level l-1, scale scales[l-1];
  a scalar (or constant vector) is the integer round(c * that scale), no
  encoding at all;
* ``add``/``sub`` bring the higher-level operand down with one fused
  "multiply by round(scales[t] q_{t+1} / scales[l]) and rescale" step
  (the simulator's ``min(level)`` rule, reference ``engine.py:195``);
* ``rotate(x, k)`` is the Galois automorphism X -> X^(5^k mod 2N) followed by
  hybrid key switching; k = 0 (mod slots) returns ``x`` itself uncounted
  (reference ``engine.py:234-251``).

Decryption reads limb 0 only (the 60-bit base prime), which represents any
slot magnitude below 2^(59 - log_scale) exactly -- ranks, masks and values
of every pipeline here are far below that.
"""

from __future__ import annotations

import math
import threading
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

from .encoder import get_encoder
from .keys import sample_error, sample_secret
from .params import CKKSParams

__all__ = [
    "EngineError",
    "CapacityError",
    "IncompatibleParamsError",
    "DepthBudgetError",
    "Ciphertext",
    "CostReport",
    "CKKSEngineCore",
    "B200Engine",
]


class EngineError(Exception):
    """Base class for engine failures (reference ``engine.py:43``)."""


class CapacityError(EngineError):
    """Data does not fit in the available slots."""


class IncompatibleParamsError(EngineError):
    """Operands belong to differently parametrised engines."""


class DepthBudgetError(EngineError):
    """An operation would drop the remaining level below zero (``engine.py:55-65``)."""

    def __init__(self, site: str, available: int, needed: int = 1):
        self.site = site
        self.available = available
        self.needed = needed
        super().__init__(
            f"depth budget exhausted at '{site}': "
            f"{needed} level(s) needed, {available} available"
        )


class Ciphertext:
    """Device limbs + remaining level + rotation-chain tag.  Immutable by contract.

    ``batch`` is None for one ciphertext (limbs [2][level+1][N]) or B for a
    stack of B ciphertexts evaluated in lock step (limbs [B][2][level+1][N]):
    every engine op then runs as ONE batched kernel sequence and is counted B
    times, exactly as B separate calls would be (``CKKSEngineCore.stack``).
    """

    __slots__ = ("data", "level", "rot_chain", "params", "batch")

    def __init__(self, data, level: int, rot_chain: int, params: CKKSParams, batch: int | None = None):
        self.data = data
        self.level = level
        self.rot_chain = rot_chain
        self.params = params
        self.batch = batch

    def __repr__(self):
        b = "" if self.batch is None else f", batch={self.batch}"
        return f"Ciphertext(level={self.level}, ring=2^{self.params.log_n}, rot_chain={self.rot_chain}{b})"


@dataclass(frozen=True)
class CostReport:
    """Snapshot of the engine counters (reference ``engine.py:119-130``)."""

    rotations: int = 0
    ctct_mults: int = 0
    ctpt_mults: int = 0
    additions: int = 0
    cmp_evals: int = 0
    ind_evals: int = 0
    levels_consumed: int = 0
    critical_rotations: int = 0


_PT_CACHE_BYTES = 4 << 30


class CKKSEngineCore:
    """Backend-independent engine logic: levels, scales, counters, plaintext cache.

    ``backend`` supplies the ciphertext primitives (``encrypt``,
    ``decrypt_limb0``, ``addsub``, ``add_const``, ``add_plain``,
    ``mul_const_rescale``, ``mul_plain_rescale``, ``mul_relin_rescale``,
    ``rotate``, ``encode_plain``).  The product engine is ``B200Engine``; the
    CPU oracle reuses this class with its own backend only inside tests.
    """

    def __init__(self, params: CKKSParams, backend):
        self.params = params
        self.backend = backend
        self.encoder = get_encoder(params.log_n)
        self._lock = threading.Lock()
        self.trace: list[tuple[str, int]] = []
        self._reset_counters()
        self._enc_seq = 0
        self._pt_cache: OrderedDict = OrderedDict()
        self._pt_bytes = 0
        backend.set_secret(sample_secret(params))

    def use_secret(self, secret: np.ndarray) -> None:
        """Switch to another ternary secret (e.g. one read by ``wire.load_secret``):
        evaluation keys are regenerated from it on first use."""
        s = np.asarray(secret, dtype=np.int64)
        if s.shape != (self.params.ring_degree,) or np.any(np.abs(s) > 1):
            raise ValueError("secret must be a ternary vector of ring-degree length")
        self.backend.set_secret(s)
        keys = getattr(self.backend, "_keys", None)
        if keys is not None:
            keys.clear()

    # ------------------------------------------------------------------
    # counters
    # ------------------------------------------------------------------
    def _reset_counters(self):
        self._rotations = 0
        self._ctct = 0
        self._ctpt = 0
        self._adds = 0
        self._cmp_evals = 0
        self._ind_evals = 0
        self._levels = 0
        self._critical = 0

    def note_compare_eval(self):
        with self._lock:
            self._cmp_evals += 1

    def note_indicator_eval(self):
        with self._lock:
            self._ind_evals += 1

    def cost_snapshot(self) -> CostReport:
        with self._lock:
            return CostReport(
                rotations=self._rotations,
                ctct_mults=self._ctct,
                ctpt_mults=self._ctpt,
                additions=self._adds,
                cmp_evals=self._cmp_evals,
                ind_evals=self._ind_evals,
                levels_consumed=self._levels,
                critical_rotations=self._critical,
            )

    def cost_reset(self):
        with self._lock:
            self._reset_counters()
            self.trace = []

    def rotation_offsets(self) -> list[int]:
        with self._lock:
            return [k for op, k in self.trace if op == "rotate"]

    # ------------------------------------------------------------------
    # helpers
    # ------------------------------------------------------------------
    def _check(self, *cts: Ciphertext):
        for c in cts:
            if c.params != self.params:
                raise IncompatibleParamsError(
                    f"ciphertext parameters {c.params.name} do not match engine {self.params.name}"
                )

    def _emit(self, data, level: int, rot_chain: int, batch: int | None = None) -> Ciphertext:
        consumed = self.params.max_level - level
        with self._lock:
            if consumed > self._levels:
                self._levels = consumed
        return Ciphertext(data, level, rot_chain, self.params, batch)

    @staticmethod
    def _nb(*cts) -> int | None:
        """Common batch size of the operands (None = single ciphertexts)."""
        sizes = {c.batch for c in cts}
        if len(sizes) != 1:
            raise ValueError(f"mixed batch sizes {sorted(map(str, sizes))}")
        return sizes.pop()

    # ------------------------------------------------------------------
    # batches of ciphertexts evaluated in lock step
    # ------------------------------------------------------------------
    def stack(self, cts) -> Ciphertext:
        """One batched ciphertext from single ones (aligned to their min level)."""
        cts = list(cts)
        self._check(*cts)
        if any(c.batch is not None for c in cts):
            raise ValueError("stack takes single ciphertexts")
        level = min(c.level for c in cts)
        datas = [self._align(c, level) for c in cts]
        return self._emit(self.backend.stack(datas), level, max(c.rot_chain for c in cts), len(cts))

    def unstack(self, ct: Ciphertext) -> list:
        """Single ciphertexts viewing the limbs of a batched one."""
        if ct.batch is None:
            return [ct]
        return [Ciphertext(self.backend.index(ct.data, i), ct.level, ct.rot_chain, self.params)
                for i in range(ct.batch)]

    def split(self, ct: Ciphertext, parts: int) -> list:
        """``parts`` equal consecutive sub-batches of a batched ciphertext, as views
        of its limbs (no copy); parts of size 1 come back as single ciphertexts."""
        if ct.batch is None or ct.batch % parts:
            raise ValueError(f"cannot split a batch of {ct.batch} into {parts} parts")
        b = ct.batch // parts
        if b == 1:
            return self.unstack(ct)
        return [Ciphertext(self.backend.slice(ct.data, i * b, (i + 1) * b), ct.level, ct.rot_chain,
                           self.params, b) for i in range(parts)]

    def concat(self, cts) -> Ciphertext:
        """One batch from single and/or batched ciphertexts (in order)."""
        singles = []
        for c in cts:
            singles.extend(self.unstack(c))
        return self.stack(singles)

    def _residues(self, k: int, level: int) -> list[int]:
        return [k % q for q in self.params.q_primes[: level + 1]]

    def _align(self, ct: Ciphertext, level: int):
        """Limbs of ``ct`` brought down to ``level`` at scale scales[level]."""
        if ct.level == level:
            return ct.data
        p = self.params
        k = int(round(p.scales[level] * p.q_primes[level + 1] / p.scales[ct.level]))
        return self.backend.mul_const_rescale(ct.data, ct.level, self._residues(k, level + 1), level + 1,
                                              batch=ct.batch)

    def at_level(self, ct: Ciphertext, level: int) -> Ciphertext:
        """``ct`` brought down to ``level`` (scale-preserving; not counted, like the min rule)."""
        return self._emit(self._align(ct, level), level, ct.rot_chain, ct.batch)

    def wrap(self, data, level: int, rot_chain: int = 0) -> Ciphertext:
        """Ciphertext around backend limbs produced outside the engine (collectives)."""
        return self._emit(data, level, rot_chain)

    @staticmethod
    def _as_constant(p):
        """Return the float if ``p`` is a scalar or a constant vector, else None."""
        if np.isscalar(p):
            return float(p)
        arr = np.asarray(p, dtype=np.float64)
        if arr.ndim == 0:
            return float(arr)
        if arr.size and arr.min() == arr.max():
            return float(arr.flat[0])
        return None

    def _batch_plain(self, p, batch):
        """('const', c) | ('vec', vector) | ('each', [B, slots] array) for plaintext p."""
        if batch is not None and not np.isscalar(p):
            arr = np.asarray(p, dtype=np.float64)
            if arr.ndim == 2:
                if arr.shape != (batch, self.params.slot_count):
                    raise ValueError(f"per-ciphertext plaintexts must be [{batch}, {self.params.slot_count}]")
                return "each", arr
        c = self._as_constant(p)
        if c is not None:
            if isinstance(p, np.ndarray) and p.size != self.params.slot_count:
                self.plain(p)
            return "const", c
        return "vec", self.plain(p)

    def _encode_each(self, arr: np.ndarray, scale: float, level: int):
        return self.backend.stack_plain([self._encode_cached(np.ascontiguousarray(v), scale, level)
                                         for v in arr])

    def _encode_cached(self, vec: np.ndarray, scale: float, level: int):
        if vec.flags.writeable:
            ident = ("h", hash(vec.tobytes()))
        else:
            ident = ("id", id(vec))
        key = (ident, level, scale)
        with self._lock:
            hit = self._pt_cache.get(key)
            if hit is not None and (ident[0] == "h" or hit[0] is vec):
                self._pt_cache.move_to_end(key)
                return hit[1]
        coeffs = self.encoder.encode(vec, scale)
        pt = self.backend.encode_plain(coeffs, level)
        nbytes = (level + 1) * self.params.ring_degree * 8
        with self._lock:
            self._pt_cache[key] = (vec, pt, nbytes)
            self._pt_bytes += nbytes
            while self._pt_bytes > _PT_CACHE_BYTES and len(self._pt_cache) > 1:
                _, (_, _, nb) = self._pt_cache.popitem(last=False)
                self._pt_bytes -= nb
        return pt

    # ------------------------------------------------------------------
    # data movement
    # ------------------------------------------------------------------
    def encrypt(self, values, level: int | None = None) -> Ciphertext:
        """Pack ``values`` into the slots (zero padded) at full level.

        ``level`` (extension; the reference's ``encrypt`` has no such argument)
        starts the ciphertext lower in the chain: a circuit of depth d needs only
        level d, and every operation's cost grows with the level it runs at
        (``circuit_depth`` measures d without touching ciphertext data)."""
        arr = np.asarray(values, dtype=np.float64).ravel()
        n = self.params.slot_count
        if arr.size > n:
            raise CapacityError(f"{arr.size} values do not fit in {n} slots")
        if level is None:
            level = self.params.max_level
        if not 0 <= level <= self.params.max_level:
            raise EngineError(f"level {level} outside the chain [0, {self.params.max_level}]")
        return self._encrypt_at(arr, int(level))

    def parallel(self, first, second):
        """``(first(), second())`` for two independent op sequences (the ReplR and
        TransR + ReplC branches of a rank).  Host order, counters and trace are those
        of calling them in turn; a backend with streams (``CudaBackend.run_parallel``)
        issues the second on its branch stream, so at one ciphertext per op -- where
        the kernels are latency-bound and leave most of the GPU idle -- the two
        run side by side.  Results are bit-identical either way."""
        run = getattr(self.backend, "run_parallel", None)
        return run(first, second) if run is not None else (first(), second())

    def fit_depth(self, ct: Ciphertext, circuit) -> Ciphertext:
        """``ct`` dropped to the level ``circuit`` needs (one fused multiply-and-rescale
        that discards the unused limbs, scale kept exact; ``at_level``): a ciphertext
        encrypted at the top of a long chain runs a shallow circuit at the shallow
        circuit's cost.  Unchanged when the circuit needs every level ``ct`` has."""
        d = circuit if isinstance(circuit, int) else self.circuit_depth(circuit)  # a known depth, or trace it
        return ct if ct.level <= d else self.at_level(ct, d)

    def circuit_depth(self, circuit) -> int:
        """Levels ``circuit(engine, ciphertext)`` consumes from a fresh ciphertext,
        found on the level tracer (host bookkeeping only; ``levels.py``)."""
        from .levels import level_tracer

        t = level_tracer(self)
        top = self.params.max_level
        out = circuit(t, t.token(top))
        outs = out if isinstance(out, (list, tuple)) else [out]
        return top - min(o.level for o in outs)

    def _encrypt_at(self, arr: np.ndarray, level: int) -> Ciphertext:
        p = self.params
        with self._lock:
            seq = self._enc_seq
            self._enc_seq += 1
        m = self.encoder.encode(arr, p.scales[level])
        e = sample_error(p, (1, seq))[0]
        data = self.backend.encrypt(m, e, seq, level)
        return Ciphertext(data, level, 0, p)

    def decrypt(self, ct: Ciphertext) -> np.ndarray:
        """Slot vector (or [B, slots] for a batched ciphertext)."""
        self._check(ct)
        if ct.batch is not None:
            return np.stack([self.decrypt(c) for c in self.unstack(ct)])
        coeffs = self.backend.decrypt_limb0(ct.data, ct.level)
        return self.encoder.decode(coeffs.astype(np.float64) / self.params.scales[ct.level])

    def plain(self, values) -> np.ndarray:
        """Coerce a scalar or full-width sequence to a plaintext vector."""
        if np.isscalar(values):
            return np.full(self.params.slot_count, float(values))
        arr = np.asarray(values, dtype=np.float64).ravel()
        if arr.size != self.params.slot_count:
            raise ValueError(
                f"plain vector must have exactly {self.params.slot_count} slots, got {arr.size}"
            )
        return arr

    # ------------------------------------------------------------------
    # arithmetic
    # ------------------------------------------------------------------
    def _addsub(self, x: Ciphertext, y: Ciphertext, op: int) -> Ciphertext:
        self._check(x, y)
        nb = self._nb(x, y)
        level = min(x.level, y.level)
        data = self.backend.addsub(self._align(x, level), self._align(y, level), level, op, batch=nb)
        with self._lock:
            self._adds += nb or 1
        return self._emit(data, level, max(x.rot_chain, y.rot_chain), nb)

    def add(self, x: Ciphertext, y: Ciphertext) -> Ciphertext:
        return self._addsub(x, y, 0)

    def sub(self, x: Ciphertext, y: Ciphertext) -> Ciphertext:
        return self._addsub(x, y, 1)

    def negate(self, x: Ciphertext) -> Ciphertext:
        self._check(x)
        data = self.backend.addsub(x.data, None, x.level, 2, batch=x.batch)
        return self._emit(data, x.level, x.rot_chain, x.batch)

    def add_plain(self, x: Ciphertext, p) -> Ciphertext:
        """x + p; for a batched x, p may also be a [B, slots] array (one plaintext each)."""
        self._check(x)
        level, nb = x.level, x.batch
        kind, val = self._batch_plain(p, nb)
        if kind == "const":
            k = int(round(val * self.params.scales[level]))
            data = self.backend.add_const(x.data, self._residues(k, level), level, batch=nb)
        elif kind == "vec":
            pt = self._encode_cached(val, self.params.scales[level], level)
            data = self.backend.add_plain(x.data, pt, level, batch=nb)
        else:
            pts = self._encode_each(val, self.params.scales[level], level)
            data = self.backend.add_plain(x.data, pts, level, batch=nb, each=True)
        with self._lock:
            self._adds += nb or 1
        return self._emit(data, level, x.rot_chain, nb)

    def mul(self, x: Ciphertext, y: Ciphertext, site: str = "mul") -> Ciphertext:
        self._check(x, y)
        nb = self._nb(x, y)
        level = min(x.level, y.level)
        if level < 1:
            raise DepthBudgetError(site, level)
        a = self._align(x, level)
        b = a if y is x else self._align(y, level)
        data = self.backend.mul_relin_rescale(a, b, level, batch=nb)
        with self._lock:
            self._ctct += nb or 1
        return self._emit(data, level - 1, max(x.rot_chain, y.rot_chain), nb)

    def mul_pairs(self, pairs, site: str = "mul") -> Ciphertext:
        """[x_i * y_i for (x_i, y_i) in pairs] as ONE batched ciphertext (batched operands
        expand to their members; a single operand broadcasts over a batched partner).
        Counted as one ct x ct multiplication per member; the operands are handed to
        the kernels through a pointer table (no batch assembled by copying)."""
        if not hasattr(self.backend, "mul_relin_rescale_pairs"):
            prods = [self.mul(x, y, site=site) for x, y in pairs]
            return self.concat(prods)
        singles = []
        for x, y in pairs:
            self._check(x, y)
            xs, ys = self.unstack(x), self.unstack(y)
            if len(xs) != len(ys):
                if len(xs) == 1:
                    xs = xs * len(ys)
                elif len(ys) == 1:
                    ys = ys * len(xs)
                else:
                    raise ValueError("batched operands of different sizes")
            singles.extend(zip(xs, ys))
        level = min(min(x.level, y.level) for x, y in singles)
        if level < 1:
            raise DepthBudgetError(site, level)
        aligned = {}

        def al(ct):
            key = id(ct)
            if key not in aligned:
                aligned[key] = (ct, self._align(ct, level))
            return aligned[key][1]

        data = self.backend.mul_relin_rescale_pairs([(al(x), al(y)) for x, y in singles], level)
        with self._lock:
            self._ctct += len(singles)
        chain = max(max(x.rot_chain, y.rot_chain) for x, y in singles)
        return self._emit(data, level - 1, chain, len(singles))

    supports_mul_plain_level = True

    def mul_plain(self, x: Ciphertext, p, site: str = "mul_plain", level: int | None = None) -> Ciphertext:
        """x * p, one level down -- or, for a scalar p and ``level`` < x.level - 1,
        straight to ``level`` in the same single rescale (the simulator's
        mul_plain followed by the min-level rule of a later add).  A batched x
        may take a [B, slots] array of per-ciphertext plaintexts."""
        self._check(x)
        if x.level < 1:
            raise DepthBudgetError(site, x.level)
        pr = self.params
        nb = x.batch
        kind, val = self._batch_plain(p, nb)
        if level is not None and level < x.level - 1:
            if kind != "const":
                raise ValueError("mul_plain(level=...) takes a scalar plaintext")
            if level < 0:
                raise DepthBudgetError(site, x.level, x.level - level)
            # drop to level+1 limbs, multiply by round(c * scales[level] q_{level+1} / scales[x]),
            # rescale by q_{level+1}  -> scale scales[level]
            k = int(round(val * pr.scales[level] * pr.q_primes[level + 1] / pr.scales[x.level]))
            data = self.backend.mul_const_rescale(x.data, x.level, self._residues(k, level + 1), level + 1,
                                                  batch=nb)
            with self._lock:
                self._ctpt += nb or 1
            return self._emit(data, level, x.rot_chain, nb)
        level = x.level
        pt_scale = pr.scales[level - 1] * pr.q_primes[level] / pr.scales[level]
        if kind == "const":
            k = int(round(val * pt_scale))
            data = self.backend.mul_const_rescale(x.data, level, self._residues(k, level), level, batch=nb)
        elif kind == "vec":
            pt = self._encode_cached(val, pt_scale, level)
            data = self.backend.mul_plain_rescale(x.data, pt, level, batch=nb)
        else:
            pts = self._encode_each(val, pt_scale, level)
            data = self.backend.mul_plain_rescale(x.data, pts, level, batch=nb, each=True)
        with self._lock:
            self._ctpt += nb or 1
        return self._emit(data, level - 1, x.rot_chain, nb)

    def linear_combination(self, terms, site: str = "lincomb") -> Ciphertext:
        """sum_i c_i * ct_i with ONE rescale (the BSGS leaf sum).

        Counted as the reference counts the unfused form -- len(terms)
        plaintext multiplications and len(terms)-1 additions -- and lands at
        min(level_i) - 1 like it.  Each term is multiplied by the integer
        round(c_i scales[o] q_{o+1} / scales[l_i]) on its first o+2 limbs, the
        products are summed (U128, one reduction per word) and rescaled once.
        """
        cts = [t for t, _ in terms]
        self._check(*cts)
        nb = self._nb(*cts)
        lo = min(t.level for t in cts)
        if lo < 1:
            raise DepthBudgetError(site, lo)
        o = lo - 1
        pr = self.params
        res = []
        for ct, c in terms:
            k = int(round(float(c) * pr.scales[o] * pr.q_primes[o + 1] / pr.scales[ct.level]))
            res.append(self._residues(k, o + 1))
        summed = self.backend.lincomb([t.data for t in cts], [t.level for t in cts], res, o + 1, batch=nb)
        data = self.backend.rescale(summed, o + 1, batch=nb)
        with self._lock:
            self._ctpt += len(terms) * (nb or 1)
            self._adds += (len(terms) - 1) * (nb or 1)
        return self._emit(data, o, max(t.rot_chain for t in cts), nb)

    def linear_combinations(self, cts, coeff_rows, site: str = "lincomb") -> list:
        """``[linear_combination(zip(cts, row)) for row in coeff_rows]`` -- the leaf sums of
        one BSGS evaluation share their baby-step ciphertexts.  Same results, levels and
        counters; a backend with ``lincomb_multi`` reads every term once per eight sums
        instead of once per sum."""
        multi = getattr(self.backend, "lincomb_multi", None)
        if multi is None or len(coeff_rows) < 2:
            return [self.linear_combination(list(zip(cts, row)), site=site) for row in coeff_rows]
        self._check(*cts)
        nb = self._nb(*cts)
        lo = min(t.level for t in cts)
        if lo < 1:
            raise DepthBudgetError(site, lo)
        o = lo - 1
        pr = self.params
        rows = [[self._residues(int(round(float(c) * pr.scales[o] * pr.q_primes[o + 1] / pr.scales[ct.level])),
                                o + 1) for ct, c in zip(cts, row)] for row in coeff_rows]
        sums = multi([t.data for t in cts], [t.level for t in cts], rows, o + 1, batch=nb)
        if nb is None:  # the sums come stacked: one batched rescale, then views of its rows
            scaled = self.backend.rescale(sums, o + 1, batch=len(rows))
            datas = [self.backend.index(scaled, i) for i in range(len(rows))]
        else:
            datas = [self.backend.rescale(summed, o + 1, batch=nb) for summed in sums]
        out = []
        for data in datas:
            with self._lock:
                self._ctpt += len(cts) * (nb or 1)
                self._adds += (len(cts) - 1) * (nb or 1)
            out.append(self._emit(data, o, max(t.rot_chain for t in cts), nb))
        return out

    def rotate(self, x: Ciphertext, k: int) -> Ciphertext:
        """Cyclic rotation of the slot vector; k > 0 rotates left (``engine.py:234``)."""
        self._check(x)
        slots = self.params.slot_count
        k_eff = int(k) % slots
        if k_eff == 0:
            return x
        galois = pow(5, k_eff, 2 * self.params.ring_degree)
        data = self.backend.rotate(x.data, galois, x.level, batch=x.batch)
        chain = x.rot_chain + 1
        with self._lock:
            self._rotations += x.batch or 1
            if chain > self._critical:
                self._critical = chain
            self.trace.extend([("rotate", k_eff)] * (x.batch or 1))
        return self._emit(data, x.level, chain, x.batch)

    def ideal_map(self, fn, *cts: Ciphertext, levels: int = 0, site: str = "ideal_map") -> Ciphertext:
        """Only constant slot functions have an encrypted realisation.

        The reference's Chebyshev evaluator uses ``ideal_map`` solely to
        materialise a degree-0 polynomial (reference ``chebyshev.py:267``,
        ``chebyshev.py:279``); that case is served by encrypting the constant
        at the target level.  Anything else needs the cleartext and raises.
        """
        self._check(*cts)
        level = min(c.level for c in cts) - levels
        if level < 0:
            raise DepthBudgetError(site, min(c.level for c in cts), levels)
        n = self.params.slot_count
        rng = np.random.default_rng(0)
        probes = [rng.uniform(-1, 1, n) for _ in cts]
        out1 = np.asarray(fn(*probes), dtype=np.float64)
        out2 = np.asarray(fn(*[-q for q in probes]), dtype=np.float64)
        if out1.shape != (n,) or not np.all(out1 == out1[0]) or not np.array_equal(out1, out2):
            raise EngineError(
                f"ideal_map at '{site}' needs cleartext slots; only constant maps run encrypted"
            )
        top = self._encrypt_at(np.full(n, out1[0]), self.params.max_level)
        data = self._align(top, level)
        return self._emit(data, level, max(c.rot_chain for c in cts))


class B200Engine(CKKSEngineCore):
    """RNS-CKKS engine on one B200: the product drop-in for ``HESimulator``.

    ``B200Engine(params)`` with a ``CKKSParams`` (see ``params.preset``) or an
    object with ``slot_count``/``max_level`` (a reference ``HEParams``), which
    selects the smallest preset with at least that many slots and levels.
    """

    def __init__(self, params, device: int | None = None):
        from .backend_cuda import CudaBackend  # needs torch + CUDA, fails loudly

        if not isinstance(params, CKKSParams):
            params = params_for(params.slot_count, params.max_level)
        super().__init__(params, CudaBackend(params, device))

    @property
    def launches(self) -> int:
        return self.backend.launches


def params_for(slot_count: int, max_level: int) -> CKKSParams:
    """Smallest repo preset-style chain with ``slot_count`` slots and ``max_level`` levels."""
    from .params import make_params

    log_n = int(math.log2(slot_count)) + 1
    if (1 << (log_n - 1)) != slot_count:
        raise ValueError(f"slot_count must be a power of two, got {slot_count}")
    log_n = max(log_n, 10)
    levels = max_level
    alpha = 8 if levels >= 24 else 4
    dnum = -(-(levels + 1) // alpha)
    digit_bits = 60 + 40 * (alpha - 1)
    special = -(-(digit_bits + 60) // 60)
    return make_params(
        f"auto{log_n}x{levels}", log_n, levels, special=special, dnum=dnum,
        hamming_weight=min(192, (1 << log_n) // 8),
    )
