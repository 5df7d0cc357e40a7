"""Two blocks per ciphertext: the opt-in packed layout of multi_rank / multi_sort.

The reference's multi-ciphertext layout (``ranking.py:240-285, 307-392``,
``sorting.py:106-142``) gives every B x B block its own ciphertext: at 2^15
slots and B = 128 a block fills half the slots, so the N = 1024 sort's 36
block-pair comparisons and 64 indicator placements run on 100 half-empty
ciphertexts.  BASELINE config 5 counts the 1024 x 1024 matrix as 32 full
ciphertexts; this module packs two blocks into one ciphertext (block A in
slots [0, H), block B in [H, 2H), H = slots / 2) for exactly the two
slotwise-heavy stages, which halves their composite-polynomial evaluations:

* comparisons: pairs p, p' are evaluated together on
  X = ReplR_i + rot_H(ReplR_i'), Y = ReplC_j + rot_H(ReplC_j') (the replicated
  blocks are zero above slot H, so the halves never mix); 18 comparison
  evaluations instead of 36 at N = 1024;
* placements: for output block i, placements (i, j), (i, j') share one
  ciphertext: the rank spreads and the replicated inputs are packed once per
  j-pair and the target plaintext holds block i's targets in both halves;
  32 indicator evaluations instead of 64.

Unpacking costs no level: the halves of a packed partial sum are folded with
one rotation by H (rot_H(U) moves the upper half onto the lower), and every
later operation (SumR / SumC / TransC) reads only the lower half for the
cells its mask keeps.  Rotations added: at most 2 L (pack the comparison
operands) + 2 L (fold the rank partials) + L (pack spreads / inputs) + L (fold
the placements), all batched.

This changes the circuit (op counts and rotation trace differ from the
reference), so it is opt-in (``SortConfig(packed=True)``); the decrypted
sort must equal the reference layout's (tests/test_packing.py on the slot
oracle, tests/test_gpu_baseline_configs.py on the GPU).  Tie correction is
not packed (its triangle masks are per block): ``packed`` requires
``tie_correction=False``.
"""

from __future__ import annotations

import numpy as np

from .chebyshev import KernelConfig, compare_kernel, indicator_kernel, with_input_range
from .matrix import MatrixLayout, replicate, sum_axis, transpose_vector
from .ranking import (
    BlockVector,
    MultiRankPipeline,
    _row_band_mask,
    batched,
    block_pairs,
    finish_block_rank,
    replicated_blocks,
)

__all__ = ["can_pack", "multi_rank_packed", "multi_sort_packed"]


def can_pack(engine, block_size: int) -> bool:
    """Two B x B blocks fit one ciphertext (B^2 <= slots / 2)."""
    return 2 * block_size * block_size <= engine.params.slot_count


def _add(engine, a, b):
    if a is None:
        return b
    return a if b is None else engine.add(a, b)


def _rot_many(engine, cts, k):
    """rotate(c, k) for each c (one lock-step batch on engines that have one)."""
    cts = list(cts)
    if not cts:
        return []
    if batched(engine) and len(cts) > 1:
        lvl = min(c.level for c in cts)
        same = [c if c.level == lvl else engine.at_level(c, lvl) for c in cts]
        return engine.unstack(engine.rotate(engine.stack(same), k))
    return [engine.rotate(c, k) for c in cts]


def _two_halves(lo: np.ndarray, hi: np.ndarray, half: int) -> np.ndarray:
    v = np.concatenate([lo[:half], hi[:half]])
    v.setflags(write=False)
    return v


def multi_rank_packed(engine, bv: BlockVector, cfg: KernelConfig) -> MultiRankPipeline:
    """``multi_rank_pipeline`` (no tie correction) with two block pairs per comparison."""
    b, count = bv.block_size, len(bv.blocks)
    slots = engine.params.slot_count
    half = slots // 2
    if not can_pack(engine, b):
        raise ValueError(f"two {b}x{b} blocks do not fit {slots} slots")
    layout = MatrixLayout(b, slots)
    valid_last = bv.valid_in(count - 1)
    rows, cols = replicated_blocks(engine, bv, layout)
    pairs = block_pairs(count)
    packs = [(pairs[k], pairs[k + 1] if k + 1 < len(pairs) else None) for k in range(0, len(pairs), 2)]
    hi_i = sorted({p[1][0] for p in packs if p[1] is not None})
    hi_j = sorted({p[1][1] for p in packs if p[1] is not None})
    rot_rows = dict(zip(hi_i, _rot_many(engine, [rows[i] for i in hi_i], half)))
    rot_cols = dict(zip(hi_j, _rot_many(engine, [cols[j] for j in hi_j], half)))
    xs = [_add(engine, rows[lo[0]], rot_rows[hi[0]] if hi else None) for lo, hi in packs]
    ys = [_add(engine, cols[lo[1]], rot_cols[hi[1]] if hi else None) for lo, hi in packs]
    if batched(engine) and len(packs) > 1:
        cmp_packed = engine.unstack(compare_kernel(engine, engine.stack(xs), engine.stack(ys), cfg))
        for _ in range(len(packs) - 1):  # one evaluation per packed ciphertext
            engine.note_compare_eval()
    else:
        cmp_packed = [compare_kernel(engine, x, y, cfg) for x, y in zip(xs, ys)]
    # pad rows of the last block (per half)
    if valid_last < b:
        band = _row_band_mask(slots, b, valid_last)
        ones = np.ones(slots)
        for k, (lo, hi) in enumerate(packs):
            lo_pad = lo[1] == count - 1
            hi_pad = hi is not None and hi[1] == count - 1
            if lo_pad or hi_pad:
                m = _two_halves(band if lo_pad else ones, band if hi_pad else ones, half)
                cmp_packed[k] = engine.mul_plain(cmp_packed[k], m, site="block-pad-mask")
    where = {}
    for k, (lo, hi) in enumerate(packs):
        where[lo] = (k, 0)
        if hi is not None:
            where[hi] = (k, 1)
    # per-block partials, split by the half each contribution sits in
    up = [[None, None] for _ in range(count)]
    low = [[None, None] for _ in range(count)]
    for (i, j), (k, h) in where.items():
        c = cmp_packed[k]
        up[i][h] = _add(engine, up[i][h], c)
        if j > i:  # complement C(j, i) = 1 - C(i, j)^T feeds block j's lower part
            low[j][h] = _add(engine, low[j][h], engine.add_plain(engine.negate(c), 1.0))
    # fold the upper-half contributions onto the lower half: one batched rotation
    uppers = [(("u", i), up[i][1]) for i in range(count) if up[i][1] is not None]
    uppers += [(("l", i), low[i][1]) for i in range(count) if low[i][1] is not None]
    folded = dict(zip([key for key, _ in uppers], _rot_many(engine, [c for _, c in uppers], half)))
    blocks = []
    for i in range(count):
        upper = _add(engine, up[i][0], folded.get(("u", i)))
        lower = _add(engine, low[i][0], folded.get(("l", i))) if i > 0 else None
        blocks.append(finish_block_rank(engine, upper, lower, i, bv, layout, None))
    return MultiRankPipeline(
        ranks=BlockVector(blocks=tuple(blocks), block_size=b, total_len=bv.total_len),
        comparisons={"packed": cmp_packed, "where": where},
        row_replicated=rows,
        col_replicated=cols,
        layout=layout,
    )


def multi_sort_packed(engine, bv: BlockVector, kcfg: KernelConfig) -> BlockVector:
    """``multi_sort`` (no tie correction) with two placements per indicator evaluation."""
    from .sorting import _neg_rank_targets, common_level

    ranking = multi_rank_packed(engine, bv, kcfg)
    layout = ranking.layout
    b, count = bv.block_size, len(bv.blocks)
    slots = engine.params.slot_count
    half = slots // 2
    window = with_input_range(kcfg, -float(b * count), float(b * count))
    rank_blocks = common_level(engine, ranking.ranks.blocks)
    if batched(engine) and count > 1:
        spreads = engine.unstack(replicate(engine, engine.stack(rank_blocks), layout, "row"))
    else:
        spreads = [replicate(engine, blk, layout, "row") for blk in rank_blocks]
    jpairs = [(j, j + 1 if j + 1 < count else None) for j in range(0, count, 2)]
    his = [j2 for _, j2 in jpairs if j2 is not None]
    rot = _rot_many(engine, [spreads[j] for j in his] + [ranking.row_replicated[j] for j in his], half)
    rot_spread = dict(zip(his, rot[: len(his)]))
    rot_rowrep = dict(zip(his, rot[len(his):]))
    spread_p = [_add(engine, spreads[j1], rot_spread.get(j2)) for j1, j2 in jpairs]
    rowrep_p = [_add(engine, ranking.row_replicated[j1], rot_rowrep.get(j2)) for j1, j2 in jpairs]
    units = [(i, m) for i in range(count) for m in range(len(jpairs))]

    def targets(i):
        t = _neg_rank_targets(slots, b, "row", b * i + 1)
        return _two_halves(t, t, half)

    if batched(engine) and len(units) > 1:
        tg = np.stack([targets(i) for i, _ in units])
        shifted = engine.add_plain(engine.stack([spread_p[m] for _, m in units]), tg)
        sel = indicator_kernel(engine, shifted, -0.5, 0.5, window, boundary="open")
        for _ in range(len(units) - 1):
            engine.note_indicator_eval()
        placed = engine.unstack(engine.mul(sel, engine.stack([rowrep_p[m] for _, m in units]),
                                           site="sort-place"))
    else:
        placed = []
        for i, m in units:
            sel = indicator_kernel(engine, engine.add_plain(spread_p[m], targets(i)), -0.5, 0.5, window,
                                   boundary="open")
            placed.append(engine.mul(sel, rowrep_p[m], site="sort-place"))
    accs = [None] * count
    for (i, _), p in zip(units, placed):
        accs[i] = _add(engine, accs[i], p)
    # lower half + upper half: one rotation per output block (batched)
    halves = _rot_many(engine, accs, half)
    folded = [engine.add(a, h) for a, h in zip(accs, halves)]
    if batched(engine) and count > 1:
        out = engine.unstack(transpose_vector(engine, sum_axis(engine, engine.stack(folded), layout, "col"),
                                              layout, "col_to_row"))
    else:
        out = [transpose_vector(engine, sum_axis(engine, f, layout, "col"), layout, "col_to_row")
               for f in folded]
    return BlockVector(blocks=tuple(out), block_size=b, total_len=bv.total_len)
