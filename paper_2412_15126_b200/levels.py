"""Level tracing: the engine's level bookkeeping without any ciphertext data.

``level_tracer(engine)`` is a ``CKKSEngineCore`` over ``LevelBackend``, whose
"limbs" are tokens carrying only a batch size.  Every engine method therefore
applies exactly the product engine's level rules (min-level alignment, the
level argument of ``mul_plain``, rescales, stacking) -- it *is* that code --
while costing only host bookkeeping.  ``shard.py`` runs a pipeline phase on
the tracer over ALL units to learn, on every rank and without communication,
the level each exchanged ciphertext will have, so its collectives need no
level exchange (no host synchronisation) and the sharded pipeline can be
captured as one CUDA graph.
"""

from __future__ import annotations

from .engine import CKKSEngineCore

__all__ = ["LevelBackend", "level_tracer"]


class _Tok:
    """Stand-in for a backend limb array: only the batch size is kept."""

    __slots__ = ("n",)

    def __init__(self, n: int = 1):
        self.n = n


def _tok(batch=None, **_):
    return _Tok(batch or 1)


class LevelBackend:
    """Backend surface of ``CudaBackend`` / ``OracleBackend`` returning tokens."""

    kind = "levels"
    launches = 0

    def __init__(self, params):
        self.params = params

    def set_secret(self, s):
        pass

    def encrypt(self, m, e, seq, level):
        return _Tok()

    def decrypt_limb0(self, data, level):
        raise RuntimeError("the level tracer holds no ciphertext data")

    def encode_plain(self, coeffs, level):
        return _Tok()

    def stack(self, datas):
        return _Tok(sum(d.n for d in datas))

    def index(self, data, i):
        return _Tok()

    def slice(self, data, a, b):
        return _Tok(b - a)

    def stack_plain(self, pts):
        return _Tok(len(pts))

    def addsub(self, a, b, level, op, batch=None):
        return _tok(batch)

    def add_const(self, a, residues, level, batch=None):
        return _tok(batch)

    def add_plain(self, a, pt, level, batch=None, each=False):
        return _tok(batch)

    def mul_const_rescale(self, a, src_level, residues, level, batch=None):
        return _tok(batch)

    def mul_plain_rescale(self, a, pt, level, batch=None, each=False):
        return _tok(batch)

    def mul_relin_rescale(self, a, b, level, batch=None):
        return _tok(batch)

    def mul_relin_rescale_pairs(self, pairs, level):
        return _Tok(len(pairs))

    def rescale(self, a, level, batch=None):
        return _tok(batch)

    def lincomb(self, terms, term_levels, residues, level, batch=None):
        return _tok(batch)

    def rotate(self, a, galois, level, batch=None):
        return _tok(batch)


class _Tracer(CKKSEngineCore):
    def token(self, level: int, batch: int | None = None):
        """A traced ciphertext at ``level`` (``batch`` members or a single one)."""
        return self._emit(_Tok(batch or 1), level, 0, batch)


def level_tracer(engine) -> _Tracer:
    """The (cached) tracer twin of ``engine``: same parameters, same level rules."""
    t = engine.__dict__.get("_level_tracer")
    if t is None:
        t = _Tracer(engine.params, LevelBackend(engine.params))
        engine.__dict__["_level_tracer"] = t
    return t
