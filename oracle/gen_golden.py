"""Generate tests/golden/*.json from the REAL reference package (run here only).

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden.py

Imports ``slotrank`` from /root/reference (read-only, never copied), runs the
reference's own circuits on its own ``HESimulator`` and records inputs,
decrypted outputs, CostReports and rotation traces.  The fixtures pin:

* oracle/slotsim.py + the product's pipeline mirror (bit-identical slots and
  identical CostReports on every circuit below), and, on the GPU box, the
  B200 pipelines after decryption (within the CKKS tolerance);
* oracle/plain.py against ``slotrank.reference`` (plain.json).

Circuits follow the reference's own known-answer tests: Fig. 3 rank, the
section 3.1 tie example, section 4 tie offsets, Fig. 5 sort and selection
matrix, the Fig. 2 transpose trace, rotation direction, plus Chebyshev-mode
rank / sort / order statistics / multi_sort at small degrees.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def _f(a):
    return [float(x) for x in np.asarray(a, dtype=np.float64).ravel()]


def main():
    sys.path.insert(0, REF)
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import slotrank as R
    from slotrank import reference as ref

    os.makedirs(OUT, exist_ok=True)
    from oracle.circuits import circuits, inputs

    cases = []
    for c in circuits():
        eng = R.HESimulator(R.HEParams(slot_count=c["slot_count"], max_level=c["max_level"]))
        out = c["fn"](eng, R, c["kernel"])
        cases.append({
            "name": c["name"],
            "slot_count": c["slot_count"],
            "max_level": c["max_level"],
            "kernel": c["kernel"],
            "output": _f(np.asarray(out)[: c["keep"]]),
            "cost": eng.cost_snapshot().__dict__,
            "trace": eng.rotation_offsets(),
        })
    X = inputs()
    v16, v8, w40 = X["v16"], X["v8"], X["w40"]

    with open(os.path.join(OUT, "circuits.json"), "w") as fh:
        json.dump({"generator": "oracle/gen_golden.py", "reference": "slotrank " + R.__version__,
                   "inputs": {"v16": _f(v16), "v8": _f(v8), "w40": _f(w40)}, "cases": cases}, fh, indent=0)

    # --- plaintext oracle fixtures ------------------------------------------------
    vecs = [[20, 30, 10, 40], [50, 10, 20, 20, 40], [10, 20, 20, 40], [7, 7, 7, 7],
            list(np.random.default_rng(3).integers(0, 6, 20).astype(float))]
    plain = []
    for v in vecs:
        plain.append({
            "values": _f(v),
            "fractional": _f(ref.fractional_ranks(v)),
            "corrected": _f(ref.corrected_ranks(v)),
            "offsets": _f(ref.tie_offsets(v)),
            "sorted": _f(ref.sorted_values(v)),
            "median": ref.median_value(v),
            "p25": ref.percentile_value(v, 25.0),
            "p90": ref.percentile_value(v, 90.0),
            "k2": ref.kth_smallest(v, 2),
        })
    with open(os.path.join(OUT, "plain.json"), "w") as fh:
        json.dump(plain, fh, indent=0)
    print(f"wrote {len(cases)} circuits, {len(plain)} plaintext vectors to {OUT}")


if __name__ == "__main__":
    main()
