"""Composite sign polynomials (Cheon-Kim-Kim, ASIACRYPT 2020) as an engine kernel.

BASELINE.json asks for sign(x) ~ f_3^(o2) o g_3^(o4) (g applied first, then f),
mapped to 0.5 (sign + 1).  The reference only has Chebyshev interpolants
(reference ``chebyshev.py:296-334``; SPEC.md:229 leaves composites out), so
this module is new: it is written against the engine method surface, runs on
any engine (B200, the CPU oracle, the slot simulator) and costs O(1)
comparison depth independent of the input gap's resolution target:

* f_n(x) = sum_{i<=n} 4^-i C(2i, i) x (1 - x^2)^i: odd, f(+-1) = +-1,
  f'(+-1) = ... = f^(n)(+-1) = 0 -- for n = 3,
  f_3(x) = (35 x - 35 x^3 + 21 x^5 - 5 x^7) / 2^4;
* g_n is the published heuristic minimax companion with a steep slope at 0
  that maps [tau, 1] into [1 - tau, 1] (tau = 1/4) -- for n = 3,
  g_3(x) = (4589 x - 16577 x^3 + 25614 x^5 - 12860 x^7) / 2^10.

Each odd degree-7 polynomial is evaluated in multiplicative depth 3 with
4 ct x ct and 4 ct x pt multiplications (4 non-scalar products is the
Paterson-Stockmeyer count for degree 7):

    y = x^2,  z = y^2,  t7 = (a7 x) y
    p(x) = a1 x + (a3 / a7) t7 + [a5 x + t7] z

The cubic term reuses t7 = a7 x^3 through one scalar product -- which also lands
it on the level of the sum -- so a polynomial costs four key switches; the LAST
polynomial of a composite keeps the five-product form a1 x + (a3 x) y +
[a5 x + (a7 x) y] z, because the scalar a3 / a7 (7 for f_3) would multiply t7's
noise straight into the output.  The scalar products are issued directly at the
level their sum needs (``mul_plain(..., level=...)`` on engines that support
it); on engines with ``linear_combination`` the two scalar terms a1 x and
(a3 / a7) t7 are summed before ONE rescale.  A sign evaluation with (g, f)
iterations uses 3 (g + f) levels and 4 (g + f) + 1 ct x ct products.
"""

from __future__ import annotations

from fractions import Fraction

__all__ = ["F3", "G3", "odd_poly_eval", "composite_sign", "composite_step", "composite_depth",
           "sign_value"]

F3 = tuple(Fraction(c, 16) for c in (35, -35, 21, -5))
G3 = tuple(Fraction(c, 1024) for c in (4589, -16577, 25614, -12860))


def _mul_plain_at(engine, x, c: float, level: int, site: str):
    if getattr(engine, "supports_mul_plain_level", False):
        return engine.mul_plain(x, c, site=site, level=level)
    return engine.mul_plain(x, c, site=site)


def _products(engine, pairs, site):
    """[a*b for (a, b) in pairs]: one lock-step batch on engines that stack ciphertexts
    (the pairs go to the kernels as a pointer table: shared operands are not copied)."""
    n = len(pairs)
    y = pairs[0][0]
    mul_pairs = getattr(engine, "mul_pairs", None)
    if mul_pairs is not None:
        prod = mul_pairs(list(pairs), site=f"{site}-quad")
    else:
        concat = getattr(engine, "concat", None)
        if concat is None:
            return tuple(engine.mul(a, b, site=f"{site}-quad") for a, b in pairs)
        prod = engine.mul(concat([a for a, _ in pairs]), concat([b for _, b in pairs]), site=f"{site}-quad")
    if y.batch is None:
        return tuple(engine.unstack(prod))
    return tuple(engine.split(prod, n))  # views: no copies


def odd_poly_eval(engine, x, coeffs, site: str = "composite", lean: bool = True):
    """a1 x + a3 x^3 + a5 x^5 + a7 x^7 on ``x`` in depth 3 (coeffs = (a1, a3, a5, a7)).

    ``lean``: four ct x ct products -- the cubic term is (a3 / a7) t7, a scalar
    multiple of t7 = (a7 x) x^2, instead of its own product (a3 x) x^2.  The scalar
    also multiplies t7's key-switch / rescale noise (7x for f3, 1.3x for g3), which
    is harmless wherever another polynomial follows (its flat regions squash it) and
    is why the last polynomial of a composite is evaluated with five products.
    """
    a1, a3, a5, a7 = (float(c) for c in coeffs)
    lvl = x.level
    lean = lean and a7 != 0.0
    y = engine.mul(x, x, site=f"{site}-sq")
    u7 = engine.mul_plain(x, a7, site=f"{site}-c7")
    if lean:
        z, t7 = _products(engine, [(y, y), (u7, y)], site)  # x^4, a7 x^3 at level lvl - 2
    else:
        u3 = engine.mul_plain(x, a3, site=f"{site}-c3")
        z, t3, t7 = _products(engine, [(y, y), (u3, y), (u7, y)], site)
    w = _mul_plain_at(engine, x, a5, lvl - 2, f"{site}-c5")
    t57 = engine.mul(engine.add(w, t7), z, site=f"{site}-x5")
    lincomb = getattr(engine, "linear_combination", None)
    if lean and lincomb is not None:
        # a1 x + (a3 / a7) t7 summed before ONE rescale, landing at level lvl - 3
        return engine.add(lincomb([(x, a1), (t7, a3 / a7)], site=f"{site}-c13"), t57)
    if lean:
        t3 = engine.mul_plain(t7, a3 / a7, site=f"{site}-c3")  # a3 x^3 at level lvl - 3
    t1 = _mul_plain_at(engine, x, a1, lvl - 3, f"{site}-c1")
    return engine.add(engine.add(t1, t3), t57)


def composite_sign(engine, x, g_iters: int, f_iters: int, out_scale: float = 1.0,
                   site: str = "sign"):
    """sign(x) for x in [-1, 1] as f^(f_iters) o g^(g_iters), times ``out_scale``.

    ``out_scale`` is folded into the last polynomial's coefficients.
    """
    chain = [G3] * g_iters + [F3] * f_iters
    if not chain:
        raise ValueError("composite sign needs at least one polynomial")
    for idx, poly in enumerate(chain):
        coeffs = poly if idx < len(chain) - 1 else tuple(c * Fraction(out_scale) for c in poly)
        x = odd_poly_eval(engine, x, coeffs, site=f"{site}-{idx}", lean=idx < len(chain) - 1)
    return x


def composite_step(engine, x, g_iters: int, f_iters: int, site: str = "step"):
    """0.5 (1 + sign(x)): 1 for x > 0, 0.5 at 0, 0 for x < 0."""
    s = composite_sign(engine, x, g_iters, f_iters, out_scale=0.5, site=site)
    return engine.add_plain(s, 0.5)


def composite_depth(g_iters: int, f_iters: int) -> int:
    return 3 * (g_iters + f_iters)


def sign_value(t, g_iters: int, f_iters: int):
    """Plaintext evaluation of the same composite (numpy), for tests and fits."""
    import numpy as np

    v = np.asarray(t, dtype=np.float64)
    for poly in [G3] * g_iters + [F3] * f_iters:
        a1, a3, a5, a7 = (float(c) for c in poly)
        y = v * v
        v = v * (a1 + y * (a3 + y * (a5 + y * a7)))
    return v
