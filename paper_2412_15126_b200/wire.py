"""Ciphertext / key-material wire format shared by the GPU engine, the CPU
oracle engine and the tests.

One ``.npz`` file per object:

* ciphertext: ``format`` = ``slotrank-b200-ct/1``, ``params`` (JSON of the
  parameter set, compared by value like the reference's ``_check``,
  ``engine.py:309-314``), ``limbs`` (``uint64[(B,) 2, level + 1, N]``: RNS
  limbs, NTT form, canonical residues, limb i under prime i), ``level``,
  ``rot_chain``, ``batch`` (-1 = a single ciphertext);
* secret: ``format`` = ``slotrank-b200-sk/1``, ``params``, ``secret``
  (ternary ``int8[N]``).  Evaluation keys are a deterministic function of the
  secret and ``params.seed`` (``keys.py``), so the secret is the whole key
  material: an engine given the same secret regenerates bit-identical relin
  and Galois keys.

The limbs are exactly what every backend computes on, so a ciphertext written
by ``B200Engine`` and read by the oracle engine (or the other way round) is
the same ciphertext bit for bit -- the GPU tests use this to check GPU
results on the CPU oracle.
"""

from __future__ import annotations

import json

import numpy as np

from .engine import Ciphertext, IncompatibleParamsError
from .params import CKKSParams

CT_FORMAT = "slotrank-b200-ct/1"
SK_FORMAT = "slotrank-b200-sk/1"

_FIELDS = ("name", "log_n", "q_primes", "p_primes", "dnum", "log_scale", "hamming_weight", "sigma",
           "seed", "secure")


def params_json(p: CKKSParams) -> str:
    """Canonical JSON of every field that takes part in parameter equality."""
    d = {k: getattr(p, k) for k in _FIELDS}
    d["q_primes"] = [int(x) for x in p.q_primes]
    d["p_primes"] = [int(x) for x in p.p_primes]
    return json.dumps(d, sort_keys=True)


def _check_params(stored: str, engine) -> None:
    mine = params_json(engine.params)
    if json.loads(stored) != json.loads(mine):
        raise IncompatibleParamsError("wire object was written under different CKKS parameters")


def _open(path, fmt: str):
    with np.load(path, allow_pickle=False) as z:
        d = {k: z[k] for k in z.files}
    got = str(d.get("format", ""))
    if got != fmt:
        raise ValueError(f"{path}: not a {fmt} file (format={got!r})")
    return d


def save_ciphertext(path, engine, ct: Ciphertext) -> None:
    """Write ``ct`` (device or host limbs) to ``path`` (.npz)."""
    engine._check(ct)
    limbs = np.asarray(engine.backend.to_host(ct.data)).view(np.uint64)
    np.savez(path, format=np.array(CT_FORMAT), params=np.array(params_json(engine.params)),
             limbs=limbs, level=np.int64(ct.level), rot_chain=np.int64(ct.rot_chain),
             batch=np.int64(-1 if ct.batch is None else ct.batch))


def load_ciphertext(path, engine) -> Ciphertext:
    """Read a ciphertext written by ``save_ciphertext`` into ``engine``'s memory.

    Raises ``IncompatibleParamsError`` when the file's parameters differ from the
    engine's and ``ValueError`` for a malformed file."""
    d = _open(path, CT_FORMAT)
    _check_params(str(d["params"]), engine)
    level, batch = int(d["level"]), int(d["batch"])
    limbs = d["limbs"].astype(np.uint64, copy=False)
    n = engine.params.ring_degree
    want = (2, level + 1, n) if batch < 0 else (batch, 2, level + 1, n)
    if limbs.shape != want or not 0 <= level <= engine.params.max_level:
        raise ValueError(f"{path}: limbs of shape {limbs.shape} do not match level {level}")
    q = np.array(engine.params.q_primes[: level + 1], dtype=np.uint64)
    if np.any(limbs >= q[:, None]):
        raise ValueError(f"{path}: limbs are not canonical residues")
    from_host = getattr(engine.backend, "from_host", None)
    data = from_host(limbs) if from_host is not None else limbs
    return engine._emit(data, level, int(d["rot_chain"]), None if batch < 0 else batch)


def save_secret(path, engine, secret: np.ndarray) -> None:
    """Write the ternary secret that generated ``engine``'s keys."""
    s = np.asarray(secret)
    if s.shape != (engine.params.ring_degree,) or np.any(np.abs(s) > 1):
        raise ValueError("secret must be a ternary vector of ring-degree length")
    np.savez(path, format=np.array(SK_FORMAT), params=np.array(params_json(engine.params)),
             secret=s.astype(np.int8))


def load_secret(path, engine) -> np.ndarray:
    """Read a secret written by ``save_secret`` (checked against ``engine.params``)."""
    d = _open(path, SK_FORMAT)
    _check_params(str(d["params"]), engine)
    return d["secret"].astype(np.int64)
