"""Degree study on the B200 engine (reference ``cli.py:269-326``).

``degree_sweep`` restates the reference's ``bench_sweep``: one record per
comparison degree (and indicator degree) with the error averaged over
``seeds`` seeded inputs, the CostReport of one run and the wall time -- but
every run is an encrypted pipeline on the GPU.  It also sweeps BASELINE's
composite sign by its (g, f) iteration counts, the axis of the paper's
runtime-vs-comparison-depth study.

    python -m paper_2412_15126_b200.sweep --task rank --count 128 \\
        --degrees 64 128 256 512 1024 --seeds 3 --json out.json
    python -m paper_2412_15126_b200.sweep --task rank --count 128 --composite 2,2 3,2 4,2
"""

from __future__ import annotations

import argparse
import json
import time

import numpy as np

from .chebyshev import KernelConfig
from .ranking import rank_pipeline, read_row
from .select import StatisticQuery, order_statistic_value
from .sorting import SortConfig, sort

__all__ = ["generate_values", "degree_sweep"]

TASKS = ("rank", "sort", "min", "max")


def generate_values(count: int, seed: int, tie_fraction: float = 0.0) -> np.ndarray:
    """Seeded uniform values in [0, 1) with a fraction of copied entries (ties),
    as the reference's workload generator (``cli.py:89-99``)."""
    rng = np.random.default_rng(seed)
    values = rng.uniform(0.0, 1.0, count)
    n_ties = int(round(tie_fraction * count))
    if n_ties:
        for t in rng.choice(count, size=n_ties, replace=False):
            donor = int(rng.integers(0, count))
            if donor != t:
                values[t] = values[donor]
    return values


def _fractional_ranks(v: np.ndarray) -> np.ndarray:
    """Rank with ties sharing the mean position (1-based)."""
    less = (v[None, :] < v[:, None]).sum(axis=1)
    equal = (v[None, :] == v[:, None]).sum(axis=1)
    return less + (equal + 1) / 2.0


def _run(engine, task: str, values: np.ndarray, cfg: KernelConfig, tie_correction: bool):
    n = values.size
    ct = engine.encrypt(values)
    if task == "rank":
        est = read_row(engine, rank_pipeline(engine, ct, n, cfg).result.ranks, n)
        return np.abs(est - _fractional_ranks(values))
    if task == "sort":
        out = read_row(engine, sort(engine, ct, n, SortConfig(kernel=cfg, tie_correction=tie_correction)), n)
        return np.abs(out - np.sort(values))
    val = engine.decrypt(order_statistic_value(engine, ct, n, StatisticQuery(task), cfg))[0]
    return np.abs(val - (values.min() if task == "min" else values.max()))


def degree_sweep(engine, task: str, count: int, configs, seeds: int = 3, seed: int = 0,
                 tie_fraction: float = 0.0, tie_correction: bool = True) -> tuple[list[dict], bool]:
    """One record per kernel configuration in ``configs`` (``KernelConfig``s):
    error over ``seeds`` inputs, the CostReport of one run, mean wall ms (device
    synchronised).  Second value: the reference's monotone-trend flag (each
    configuration's mean error within 10% of, or below, the previous one's)."""
    try:
        import torch

        sync = torch.cuda.synchronize if torch.cuda.is_available() else (lambda: None)
    except ImportError:  # CPU engines (tests)
        sync = lambda: None  # noqa: E731
    if task not in TASKS:
        raise ValueError(f"task must be one of {TASKS}")
    records = []
    for cfg in configs:
        _run(engine, task, generate_values(count, seed, tie_fraction), cfg, tie_correction)  # keys, caches
        errs, wall, report = [], 0.0, None
        for s in range(seeds):
            values = generate_values(count, seed + s, tie_fraction)
            engine.cost_reset()
            sync()
            t0 = time.perf_counter()
            errs.append(np.atleast_1d(_run(engine, task, values, cfg, tie_correction)))
            sync()
            wall += (time.perf_counter() - t0) * 1e3
            report = engine.cost_snapshot()
        flat = np.concatenate(errs)
        records.append({
            "kernel": {"mode": cfg.mode, "degree": cfg.degree, "indicator_degree": cfg.indicator_degree,
                       "composite": cfg.composite, "indicator_composite": cfg.indicator_composite},
            "avg_err": float(flat.mean()), "max_err": float(flat.max()),
            "report": report.__dict__, "wall_ms": wall / seeds})
    errs = [r["avg_err"] for r in records]
    monotone = all(b <= a * 1.10 for a, b in zip(errs, errs[1:]))
    return records, monotone


def main(argv=None) -> int:
    from .engine import B200Engine
    from .params import preset

    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--task", choices=TASKS, default="rank")
    ap.add_argument("--count", type=int, default=128)
    ap.add_argument("--degrees", type=int, nargs="*", default=[])
    ap.add_argument("--ind-degree", type=int, default=None)
    ap.add_argument("--composite", nargs="*", default=[], help="g,f pairs, e.g. 3,2 4,2")
    ap.add_argument("--seeds", type=int, default=3)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--tie-fraction", type=float, default=0.0)
    ap.add_argument("--params", default=None, help="preset (default: cfg3 for rank, long otherwise)")
    ap.add_argument("--json", default=None)
    args = ap.parse_args(argv)
    configs = [KernelConfig(mode="chebyshev", degree=d, indicator_degree=args.ind_degree or d)
               for d in args.degrees]
    for gf in args.composite:
        g, f = (int(x) for x in gf.split(","))
        configs.append(KernelConfig(mode="composite", composite=(g, f), indicator_composite=(g, f)))
    if not configs:
        ap.error("give --degrees and/or --composite")
    eng = B200Engine(preset(args.params or ("cfg3" if args.task == "rank" else "long")))
    records, monotone = degree_sweep(eng, args.task, args.count, configs, args.seeds, args.seed,
                                     args.tie_fraction)
    out = {"task": args.task, "count": args.count, "params": eng.params.name, "seeds": args.seeds,
           "monotone": monotone, "records": records}
    for r in records:
        k = r["kernel"]
        name = f"cheb d={k['degree']}" if k["mode"] == "chebyshev" else f"composite {tuple(k['composite'])}"
        print(f"{name:22s} avg_err={r['avg_err']:.4g} max_err={r['max_err']:.4g} wall={r['wall_ms']:.2f} ms "
              f"ctct={r['report']['ctct_mults']} levels={r['report']['levels_consumed']}")
    if args.json:
        with open(args.json, "w") as fh:
            json.dump(out, fh, indent=1)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
