"""The golden circuits, written against a slotrank-compatible package ``R``.

TEST INFRASTRUCTURE.  ``oracle/gen_golden.py`` runs them with ``R = slotrank``
(the reference, on its own HESimulator) to produce tests/golden/circuits.json;
the tests replay them with ``R = paper_2412_15126_b200`` on oracle/slotsim.py
(bit-identical expected) and on B200Engine (CKKS tolerance expected).  Each
circuit is a known-answer case from the reference's own tests.
"""

from __future__ import annotations

import numpy as np

IDEAL = {"mode": "ideal", "degree": 256}


def cheb(d, **kw):
    return {"mode": "chebyshev", "degree": d, **kw}


def kc(R, kernel):
    return R.KernelConfig(**{k: (tuple(v) if isinstance(v, list) else v) for k, v in kernel.items()})


def inputs():
    rng = np.random.default_rng(0)
    v16 = rng.choice(64, 16, replace=False) / 64
    w40 = rng.uniform(size=40)
    v8 = np.array([0.15, 0.55, 0.35, 0.95, 0.05, 0.75, 0.25, 0.85])
    return {"v16": v16, "v8": v8, "w40": w40}


def circuits():
    X = inputs()
    v16, v8, w40 = X["v16"], X["v8"], X["w40"]
    out = []

    def add(name, slots, max_level, kernel, fn, keep, gpu=False):
        out.append(dict(name=name, slot_count=slots, max_level=max_level, kernel=kernel, fn=fn,
                        keep=keep, gpu=gpu))

    # Fig. 3 / section 3.1 / section 4 (ideal mode; reference tests/test_ranking.py:41-140)
    for name, v, slots in (("fig3_rank", [20, 30, 10, 40], 16),
                           ("sec31_rank_ties", [50, 10, 20, 20, 40], 64),
                           ("sec4_ties", [10, 20, 20, 40], 16),
                           ("all_equal", [7, 7, 7, 7], 16)):
        n = len(v)
        add(name, slots, 48, IDEAL,
            lambda e, R, k, v=v, n=n: R.read_row(e, R.rank(e, e.encrypt(v), n, kc(R, k)).ranks, n), n)
        add(name + "_corrected", slots, 48, IDEAL,
            lambda e, R, k, v=v, n=n: R.read_row(e, R.rank_corrected(e, e.encrypt(v), n, kc(R, k)).ranks, n), n)
    # Fig. 5 (reference tests/test_sorting.py:29-43, tests/test_select.py:36-42)
    add("fig5_sort", 16, 48, IDEAL,
        lambda e, R, k: R.read_row(e, R.sort(e, e.encrypt([20, 30, 10, 40]), 4,
                                           R.SortConfig(kernel=kc(R, k), tie_correction=False)), 4), 4)

    def fig5_selection(e, R, k):
        res = R.sorting.sort_full(e, e.encrypt([20, 30, 10, 40]), 4,
                                  R.SortConfig(kernel=kc(R, k), tie_correction=False, optimized_layout=False))
        return e.decrypt(res.selection)[:16]

    add("fig5_selection_matrix", 16, 48, IDEAL, fig5_selection, 16)
    for kind, kk in (("min", None), ("max", None), ("kth", 1), ("kth", 4)):
        add(f"fig5_mask_{kind}{kk or ''}", 16, 48, IDEAL,
            lambda e, R, k, kind=kind, kk=kk: e.decrypt(R.order_statistic_mask(
                e, e.encrypt([20, 30, 10, 40]), 4, R.StatisticQuery(kind, k=kk), kc(R, k)))[:4], 4)

    # Fig. 2 transpose (reference tests/test_matrix.py:104-112: trace [28, 14, 7])
    def transpose_n8(e, R, k):
        return e.decrypt(R.transpose_vector(e, e.encrypt(np.arange(1, 9)), R.MatrixLayout(8, 64),
                                            "row_to_col"))[:64]

    add("fig2_transpose_n8", 64, 48, IDEAL, transpose_n8, 64)
    # rotation direction (reference tests/test_engine.py:120-143)
    add("rotate_left_1", 4, 8, IDEAL, lambda e, R, k: e.decrypt(e.rotate(e.encrypt([1, 2, 3, 4]), 1)), 4)
    add("rotate_right_1", 4, 8, IDEAL, lambda e, R, k: e.decrypt(e.rotate(e.encrypt([1, 2, 3, 4]), -1)), 4)

    # Chebyshev mode: the circuits the CKKS engine can run (no ideal_map)
    for d in (64, 256):
        add(f"cheb_rank_n16_d{d}", 2048, 40, cheb(d),
            lambda e, R, k: R.read_row(e, R.rank(e, e.encrypt(v16), 16, kc(R, k)).ranks, 16), 16, gpu=True)
    add("cheb_sort_n8_d512", 64, 64, cheb(512),
        lambda e, R, k: R.read_row(e, R.sort(e, e.encrypt(v8), 8,
                                           R.SortConfig(kernel=kc(R, k), tie_correction=False)), 8), 8)
    for kind, kk in (("min", None), ("max", None), ("kth", 5)):
        add(f"cheb_mask_{kind}{kk or ''}_n16", 2048, 60, cheb(128, tie_margin=2.0 ** -7),
            lambda e, R, k, kind=kind, kk=kk: e.decrypt(R.order_statistic_mask(
                e, e.encrypt(v16), 16, R.StatisticQuery(kind, k=kk), kc(R, k)))[:16], 16, gpu=True)
        add(f"cheb_value_{kind}{kk or ''}_n16", 2048, 60, cheb(128, tie_margin=2.0 ** -7),
            lambda e, R, k, kind=kind, kk=kk: e.decrypt(R.order_statistic_value(
                e, e.encrypt(v16), 16, R.StatisticQuery(kind, k=kk), kc(R, k)))[:1], 1)
    add("cheb_multisort_n40_b16", 256, 60, cheb(256),
        lambda e, R, k: R.block_merge(e, R.multi_sort(e, R.block_split(e, w40),
                                                      R.SortConfig(kernel=kc(R, k), tie_correction=False))), 40)
    add("ideal_multisort_ties_n11", 16, 48, IDEAL,
        lambda e, R, k: R.block_merge(e, R.multi_sort(e, R.block_split(e, [5, 1, 4, 1, 3, 9, 2, 6, 5, 3, 5]),
                                                      R.SortConfig(kernel=kc(R, k)))), 11)
    add("cheb_rank_corrected_ties_n8", 64, 40, cheb(256),
        lambda e, R, k: R.read_row(e, R.rank_corrected(
            e, e.encrypt([0.5, 0.25, 0.5, 0.75, 0.25, 0.5, 0.125, 1.0]), 8, kc(R, k)).ranks, 8), 8)
    return out
