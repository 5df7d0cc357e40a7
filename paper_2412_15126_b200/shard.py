"""Multi-GPU sharding of the multi-ciphertext pipelines (N >= 256).

Restates reference ``multi_rank_pipeline`` / ``multi_sort``
(``pkg/src/slotrank/ranking.py:307-392``, ``sorting.py:106-142``) with the
independent units spread over ranks, in five phases,
each ONE collective on the stacked ciphertexts of the phase.  The level every
exchanged ciphertext will have is known in advance on every rank: the first
call of a configuration traces the single-GPU circuit on the level tracer
(``levels.py``: the engine's own level rules over data-free tokens) and caches
the level vectors, so no level is ever exchanged and nothing synchronises the
host (the pipeline can be captured as one CUDA graph with its collectives):

0. ReplR(block) and ReplC(TransR(block)) for blocks i with i % world == rank,
   batched; all-gather of the stacked results (every rank needs every block);
1. the L(L+1)/2 block-pair comparisons C(i, j), i <= j, dealt round-robin;
   each rank folds its own pairs into per-block partial sums
   U_i = sum_{j>=i} C(i, j), D_i = sum_{j<i} (1 - C(j, i)) (and the tie-offset
   pieces); all partials of all blocks go through one all-reduce of their RNS
   limbs (int64 sum -- limbs are < 2^60 and world <= 8, so no overflow)
   followed by one mod-q fix-up launch;
2. block i is finished (SumR / SumC / TransC / +1/2) by rank i % world; the
   finished blocks are all-gathered;
3. the L^2 indicator placements (i, j) of the sort are dealt round-robin and
   folded into per-output-block partial sums: one all-reduce + fix-up;
4. output block i is finished (SumC + TransC) by its owner; one all-gather.

Modular addition is exact and associative, so the ciphertexts every rank ends
with are bit-identical to the single-GPU pipeline's for any world size whenever
the partial sums sit at one level (every BASELINE configuration; with a padded
last block the min-level alignment is applied per rank, as in the single-GPU
``engine.add``).  tests/test_shard_gloo.py checks it with 2 gloo ranks on the
CPU oracle.  Evaluation keys are replicated (every rank generates them from the
shared seed); only ciphertexts cross NVLink.  With world == 1 every collective
is skipped and this is exactly the single-GPU pipeline.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .chebyshev import KernelConfig, equality_from_compare, indicator_kernel, with_input_range
from .matrix import MatrixLayout, replicate, sum_axis, transpose_vector
from .ranking import (
    BlockVector,
    MultiRankPipeline,
    _prefix_vector,
    _triangle_mask,
    batched,
    block_pairs,
    compare_block_pairs,
    finish_block_rank,
    lower_partial,
    replicated_blocks,
    upper_partial,
)
from .sorting import SortConfig, _neg_rank_targets, common_level, place_block

__all__ = ["Comm", "ProjectedComm", "multi_rank_sharded", "multi_sort_sharded"]

# The packed layout (packing.py, two blocks per ciphertext) shards the same way:
# packed comparisons / placements are the units dealt round-robin, the
# per-half partial sums go through the phase's all-reduce, and the owner folds
# the halves (one rotation by slots/2) -- after the reduction, so the result is
# bit-identical to the single-GPU packed run.

_NO_LEVEL = 1 << 20
MAX_WORLD = 8  # int64 sums of world residues < 2^60 must not overflow


@dataclass
class Comm:
    """torch.distributed process group wrapper (NCCL on GPUs, gloo on CPU)."""

    group: object = None

    def __post_init__(self):
        import torch.distributed as dist

        self.dist = dist
        self.rank = dist.get_rank(self.group)
        self.world = dist.get_world_size(self.group)
        if self.world > MAX_WORLD:
            raise ValueError(f"shard.py sums int64 limbs (< 2^60) over ranks: world <= {MAX_WORLD}")
        self.collectives = 0  # data collectives issued (tests assert O(1) per phase)
        self.level_syncs = 0  # host syncs (level exchanges: 0 once a level plan is cached)
        self.planned = None   # level vectors of the coming exchanges, in order (levels.py trace)
        self.recorder = None  # list collecting each exchange's level vector (tracing)

    def owner(self, unit_index: int) -> int:
        return unit_index % self.world

    def device(self):
        import torch

        if self.dist.get_backend(self.group) == "nccl":
            return torch.device("cuda", torch.cuda.current_device())
        return "cpu"

    def exchange_levels(self, levels: list[int]) -> list[int]:
        """The levels the items of this exchange will have on every rank: the next
        planned vector (no communication), else one MIN all-reduce (a host sync)."""
        if self.recorder is not None:
            self.recorder.append(list(levels))
        if self.world == 1:
            return list(levels)
        if self.planned:
            return self.planned.pop(0)
        return self.min_levels(levels)

    def min_levels(self, levels: list[int]) -> list[int]:
        """Element-wise MIN over ranks of a level vector (_NO_LEVEL = absent)."""
        import torch

        t = torch.tensor(levels, dtype=torch.int64, device=self.device())
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        self.level_syncs += 1
        return [int(x) for x in t.cpu().tolist()]

    def all_reduce(self, t):
        self.dist.all_reduce(t, group=self.group)
        self.collectives += 1

    def all_gather(self, t):
        """[world * k, ...] from every rank's [k, ...] (rank-major)."""
        import torch

        parts = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t.contiguous(), group=self.group)
        self.collectives += 1
        return torch.cat(parts)


class ProjectedComm:
    """ONE rank's share of a ``world``-rank run inside a single process, for timing
    that rank's kernels when the other GPUs are absent.  The collectives move no
    data -- ``all_reduce`` leaves the local partial sums, ``all_gather`` tiles the
    local rows -- so the ciphertexts that come out are NOT the pipeline's result
    (the multi-rank result is checked by the gloo / NCCL tests); the kernel work
    of rank ``rank`` and the bytes each collective would move are exactly those of
    the real run (levels come from the same cached plan).  ``bench.py`` reports
    them as a projection, never as a measured multi-GPU latency."""

    def __init__(self, rank: int, world: int):
        if not 0 <= rank < world <= MAX_WORLD:
            raise ValueError(f"need 0 <= rank < world <= {MAX_WORLD}")
        self.rank, self.world = rank, world
        self.collectives = self.level_syncs = 0
        self.planned = self.recorder = None
        self.all_reduce_bytes = self.all_gather_bytes = 0  # payload per rank / gathered total

    def owner(self, unit_index: int) -> int:
        return unit_index % self.world

    def exchange_levels(self, levels):
        if self.recorder is not None:
            self.recorder.append(list(levels))
        if not self.planned:
            raise RuntimeError("ProjectedComm needs the cached level plan (_with_plan)")
        return self.planned.pop(0)

    def all_reduce(self, t):
        self.collectives += 1
        self.all_reduce_bytes += t.numel() * t.element_size()

    def all_gather(self, t):
        import torch

        self.collectives += 1
        self.all_gather_bytes += self.world * t.numel() * t.element_size()
        return torch.cat([t] * self.world)


class _TraceComm:
    """world-1 stand-in for ``Comm`` that records every exchange's level vector."""

    rank, world = 0, 1

    def __init__(self):
        self.recorder, self.planned = [], None
        self.collectives = self.level_syncs = 0

    def owner(self, unit_index: int) -> int:
        return 0

    def exchange_levels(self, levels):
        self.recorder.append(list(levels))
        return list(levels)


def _with_plan(engine, comm, key, bv: BlockVector, run):
    """Run ``run(eng, bv, comm)`` with the level vector of every exchange known in
    advance: the first call traces the single-GPU circuit on the level tracer
    (levels.py, no data, no communication) and caches the vectors on the engine."""
    if comm.world == 1:
        return run(engine, bv, comm)
    from .levels import level_tracer

    plans = engine.__dict__.setdefault("_shard_level_plans", {})
    full = key + (bv.block_size, bv.total_len, tuple(b.level for b in bv.blocks))
    if full not in plans:
        tr = level_tracer(engine)
        tbv = BlockVector(blocks=tuple(tr.token(b.level) for b in bv.blocks), block_size=bv.block_size,
                          total_len=bv.total_len)
        tc = _TraceComm()
        run(tr, tbv, tc)
        plans[full] = tc.recorder
    comm.planned = [list(v) for v in plans[full]]
    try:
        return run(engine, bv, comm)
    finally:
        comm.planned = None


def _lv(ct) -> int:
    return _NO_LEVEL if ct is None else ct.level


def _stacked(engine, cts, levels):
    """int64 tensor [k][2][max level + 1][N] of ciphertexts brought to ``levels``
    (zeros for None; shorter limb counts zero-padded)."""
    import torch

    be = engine.backend
    top = max(lv for lv in levels if lv != _NO_LEVEL)
    rows = []
    for ct, lv in zip(cts, levels):
        if ct is None or lv == _NO_LEVEL:
            rows.append(be.zeros_tensor(top))
            continue
        if ct.level != lv:
            ct = engine.at_level(ct, lv)
        t = be.as_tensor(ct.data)
        if lv < top:
            pad = be.zeros_tensor(top)
            pad[:, : lv + 1] = t
            t = pad
        rows.append(t)
    return torch.stack(rows)


def _unstacked(engine, t, levels, reduce_mod: bool):
    """Ciphertexts (None where absent) from a stacked tensor at ``levels``."""
    be = engine.backend
    out = []
    for k, lv in enumerate(levels):
        if lv == _NO_LEVEL:
            out.append(None)
            continue
        x = t[k, :, : lv + 1].contiguous()
        data = be.reduce_mod_tensor(x, lv) if reduce_mod else be.from_tensor(x, lv)
        out.append(engine.wrap(data, lv, 0))
    return out


def _sum_all(engine, cts, comm: Comm):
    """Modular sums over ranks of a list of ciphertexts (one all-reduce): each
    rank's item is brought to the minimum level over ranks first."""
    levels = comm.exchange_levels([_lv(c) for c in cts])
    if comm.world == 1:
        return list(cts)
    if all(lv == _NO_LEVEL for lv in levels):
        return [None] * len(cts)
    t = _stacked(engine, cts, levels)
    comm.all_reduce(t)
    return _unstacked(engine, t, levels, reduce_mod=True)


def _gather_owned(engine, owned: dict, count: int, comm: Comm):
    """Every rank ends with all ``count`` items; item i is computed by rank
    comm.owner(i) (``owned`` maps its indices to ciphertexts): one all-gather."""
    levels = comm.exchange_levels([_lv(owned.get(i)) for i in range(count)])
    if comm.world == 1:
        return [owned[i] for i in range(count)]
    per = -(-count // comm.world)
    # slot s of rank r holds item r + s * world
    local = [owned.get(comm.rank + s * comm.world) for s in range(per)]
    local_lv = [levels[comm.rank + s * comm.world] if comm.rank + s * comm.world < count else _NO_LEVEL
                for s in range(per)]
    top = max(lv for lv in levels if lv != _NO_LEVEL)
    t = _stacked(engine, local + [None], local_lv + [top])[:per]  # pad row fixes the limb count
    g = comm.all_gather(t)  # [world * per], rank-major
    out = []
    for i in range(count):
        r, s = i % comm.world, i // comm.world
        lv = levels[i]
        out.append(None if lv == _NO_LEVEL else
                   engine.wrap(engine.backend.from_tensor(g[r * per + s, :, : lv + 1].contiguous(), lv), lv, 0))
    return out


def _replicated_sharded(engine, bv: BlockVector, layout: MatrixLayout, comm: Comm):
    """Phase 0: (rows, cols) of every block, each computed once over the world."""
    count = len(bv.blocks)
    if comm.world == 1:
        rows, cols = replicated_blocks(engine, bv, layout)
        comm.exchange_levels([c.level for pair in zip(rows, cols) for c in pair])
        return rows, cols
    mine = [i for i in range(count) if comm.owner(i) == comm.rank]
    owned = {}
    if mine:
        sub = BlockVector(blocks=tuple(bv.blocks[i] for i in mine), block_size=bv.block_size,
                          total_len=bv.total_len)
        rows, cols = replicated_blocks(engine, sub, layout)
        for i, r, c in zip(mine, rows, cols):
            owned[2 * i], owned[2 * i + 1] = r, c
    both = _gather_pairs(engine, owned, count, comm)  # items 2i (row), 2i + 1 (col)
    return [both[2 * i] for i in range(count)], [both[2 * i + 1] for i in range(count)]


def _gather_pairs(engine, owned2: dict, count: int, comm: Comm):
    """All-gather of 2 items per block (row, col) -- block i's pair computed by
    comm.owner(i), stacked along a second axis -- in one collective."""
    import torch

    lv = comm.exchange_levels([_lv(owned2.get(k)) for k in range(2 * count)])
    if comm.world == 1:
        return [owned2[k] for k in range(2 * count)]
    per = -(-count // comm.world)
    top = max(x for x in lv if x != _NO_LEVEL)
    rows = []
    for s in range(per):
        i = comm.rank + s * comm.world
        pair = [owned2.get(2 * i), owned2.get(2 * i + 1)] if i < count else [None, None]
        pl = [lv[2 * i], lv[2 * i + 1]] if i < count else [_NO_LEVEL, _NO_LEVEL]
        rows.append(_stacked(engine, pair + [None], pl + [top])[:2])
    t = torch.stack(rows)  # [per][2][2][top+1][N]
    g = comm.all_gather(t)  # [world * per][2]...
    out = []
    for k in range(2 * count):
        i, c = divmod(k, 2)
        r, s = i % comm.world, i // comm.world
        x = lv[k]
        out.append(None if x == _NO_LEVEL else
                   engine.wrap(engine.backend.from_tensor(g[r * per + s, c, :, : x + 1].contiguous(), x), x, 0))
    return out


def multi_rank_sharded(engine, bv: BlockVector, cfg: KernelConfig, comm: Comm, *,
                       tie_correction: bool = False, packed: bool = False) -> MultiRankPipeline:
    """``multi_rank_pipeline`` with blocks, block pairs and block finishes dealt over
    ``comm``'s ranks (phases 0-2 of the module docstring); every exchange's levels
    come from a cached trace of the circuit (no host synchronisation)."""
    return _with_plan(engine, comm, ("rank", cfg, tie_correction, packed), bv,
                      lambda e, v, c: _multi_rank_sharded(e, v, cfg, c, tie_correction=tie_correction,
                                                          packed=packed))


def _multi_rank_sharded(engine, bv: BlockVector, cfg: KernelConfig, comm: Comm, *,
                        tie_correction: bool = False, packed: bool = False) -> MultiRankPipeline:
    if packed:
        if tie_correction:
            raise ValueError("the packed layout has no tie correction")
        return _multi_rank_sharded_packed(engine, bv, cfg, comm)
    b, count = bv.block_size, len(bv.blocks)
    layout = MatrixLayout(b, engine.params.slot_count)
    valid_last = bv.valid_in(count - 1)
    rows, cols = _replicated_sharded(engine, bv, layout, comm)
    pairs = block_pairs(count)
    mine = [p for idx, p in enumerate(pairs) if comm.owner(idx) == comm.rank]
    comparisons = compare_block_pairs(engine, mine, rows, cols, cfg, layout, count, valid_last) if mine else {}
    equalities = {p: equality_from_compare(engine, c) for p, c in comparisons.items()} if tie_correction else {}
    # phase 1: every partial of every block in one all-reduce
    parts = []
    for i in range(count):
        parts.append(upper_partial(engine, comparisons, i, count))
        parts.append(lower_partial(engine, comparisons, i) if i > 0 else None)
        if tie_correction:
            tp = _tie_partials(engine, equalities, i, count, layout)
            parts.extend([tp["cross"], tp["diag"], tp["total"]])
    stride = 5 if tie_correction else 2
    summed = _sum_all(engine, parts, comm)
    # phase 2: owners finish their blocks; one all-gather
    owned = {}
    for i in range(count):
        if comm.owner(i) != comm.rank:
            continue
        upper, lower = summed[stride * i], summed[stride * i + 1]
        tie = None
        if tie_correction:
            tp = {"cross": summed[stride * i + 2], "diag": summed[stride * i + 3], "total": summed[stride * i + 4]}

            def tie(i=i, tp=tp):
                return _finish_tie(engine, tp, i, bv.valid_in(i), layout)
        owned[i] = finish_block_rank(engine, upper, lower, i, bv, layout, tie)
    blocks = _gather_owned(engine, owned, count, comm)
    return MultiRankPipeline(
        ranks=BlockVector(blocks=tuple(blocks), block_size=b, total_len=bv.total_len),
        comparisons=comparisons,
        row_replicated=rows,
        col_replicated=cols,
        layout=layout,
    )


def _tie_partials(engine, equalities, i, count, layout):
    """Per-rank pieces of the blockwise tie offset (reference ranking.py:395-423)."""
    cross = None
    for j in range(i):
        e = equalities.get((j, i))
        if e is not None:
            cross = e if cross is None else engine.add(cross, e)
    own = equalities.get((i, i))
    diag_in = None
    if own is not None:
        diag_in = engine.mul_plain(own, _triangle_mask(layout.slot_count, layout.n_dim, "upper", 1.0),
                                   site="tie-triangle")
    total = own
    for j in range(i + 1, count):
        e = equalities.get((i, j))
        if e is not None:
            total = e if total is None else engine.add(total, e)
    return {"cross": cross, "diag": diag_in, "total": total}


def _finish_tie(engine, parts, i, valid_i, layout):
    slots, b = layout.slot_count, layout.n_dim
    cross_row = None
    if parts["cross"] is not None and i > 0:
        cross_row = transpose_vector(engine, sum_axis(engine, parts["cross"], layout, "col"), layout,
                                     "col_to_row")
    diag = sum_axis(engine, parts["diag"], layout, "row")
    total_row = sum_axis(engine, parts["total"], layout, "row")
    position = diag if cross_row is None else engine.add(diag, cross_row)
    total = total_row if cross_row is None else engine.add(total_row, cross_row)
    offset = engine.sub(position, engine.mul_plain(total, 0.5, site="tie-total"))
    return engine.add_plain(offset, _prefix_vector(slots, b, valid_i, -0.5, "row"))


def multi_sort_sharded(engine, bv: BlockVector, cfg: SortConfig, comm: Comm) -> BlockVector:
    """``multi_sort`` with the ranking sharded as above and the L^2 placements dealt
    over ranks (phases 3-4 of the module docstring); no host synchronisation once
    the level plan of this configuration is cached."""
    return _with_plan(engine, comm, ("sort", cfg), bv, lambda e, v, c: _multi_sort_sharded(e, v, cfg, c))


def _multi_sort_sharded(engine, bv: BlockVector, cfg: SortConfig, comm: Comm) -> BlockVector:
    if getattr(cfg, "packed", False):
        if cfg.tie_correction:
            raise ValueError("the packed layout has no tie correction")
        return _multi_sort_sharded_packed(engine, bv, cfg.kernel, comm)
    ranking = _multi_rank_sharded(engine, bv, cfg.kernel, comm, tie_correction=cfg.tie_correction)
    layout = ranking.layout
    b, count = bv.block_size, len(bv.blocks)
    window = with_input_range(cfg.kernel, -float(b * count), float(b * count))
    units = [(i, j) for i in range(count) for j in range(count)]
    mine = [u for idx, u in enumerate(units) if comm.owner(idx) == comm.rank]
    rank_blocks = common_level(engine, ranking.ranks.blocks)
    needed = sorted({j for _, j in mine})
    if batched(engine) and len(needed) > 1:
        spread_list = engine.unstack(replicate(engine, engine.stack([rank_blocks[j] for j in needed]),
                                               layout, "row"))
        spreads = dict(zip(needed, spread_list))
    else:
        spreads = {j: replicate(engine, rank_blocks[j], layout, "row") for j in needed}
    placed_all = {}
    if batched(engine) and len(mine) > 1:
        targets = np.stack([_neg_rank_targets(layout.slot_count, b, "row", b * i + 1) for i, _ in mine])
        shifted = engine.add_plain(engine.stack([spreads[j] for _, j in mine]), targets)
        sel = indicator_kernel(engine, shifted, -0.5, 0.5, window, boundary="open")
        for _ in range(len(mine) - 1):
            engine.note_indicator_eval()
        prod = engine.mul(sel, engine.stack([ranking.row_replicated[j] for _, j in mine]), site="sort-place")
        placed_all = dict(zip(mine, engine.unstack(prod)))
    # phase 3: per-output-block partial sums, one all-reduce
    partial = []
    for i in range(count):
        acc = None
        for (ii, j) in mine:
            if ii != i:
                continue
            placed = placed_all.get((ii, j))
            if placed is None:
                placed = place_block(engine, spreads[j], ranking.row_replicated[j], i, layout, window)
            acc = placed if acc is None else engine.add(acc, placed)
        partial.append(acc)
    summed = _sum_all(engine, partial, comm)
    # phase 4: owners finish (SumC + TransC); one all-gather
    owned = {i: transpose_vector(engine, sum_axis(engine, summed[i], layout, "col"), layout, "col_to_row")
             for i in range(count) if comm.owner(i) == comm.rank}
    out = _gather_owned(engine, owned, count, comm)
    return BlockVector(blocks=tuple(out), block_size=b, total_len=bv.total_len)


# ---------------------------------------------------------------------------
# packed layout (packing.py) over ranks
# ---------------------------------------------------------------------------
def _multi_rank_sharded_packed(engine, bv: BlockVector, cfg: KernelConfig, comm: Comm) -> MultiRankPipeline:
    from .packing import _add, _rot_many, _two_halves, can_pack
    from .chebyshev import compare_kernel
    from .ranking import _row_band_mask

    b, count = bv.block_size, len(bv.blocks)
    slots = engine.params.slot_count
    half = slots // 2
    if not can_pack(engine, b):
        raise ValueError(f"two {b}x{b} blocks do not fit {slots} slots")
    layout = MatrixLayout(b, slots)
    valid_last = bv.valid_in(count - 1)
    rows, cols = _replicated_sharded(engine, bv, layout, comm)
    pairs = block_pairs(count)
    packs = [(pairs[k], pairs[k + 1] if k + 1 < len(pairs) else None) for k in range(0, len(pairs), 2)]
    mine = [k for k in range(len(packs)) if comm.owner(k) == comm.rank]
    hi_i = sorted({packs[k][1][0] for k in mine if packs[k][1] is not None})
    hi_j = sorted({packs[k][1][1] for k in mine if packs[k][1] is not None})
    rot_rows = dict(zip(hi_i, _rot_many(engine, [rows[i] for i in hi_i], half)))
    rot_cols = dict(zip(hi_j, _rot_many(engine, [cols[j] for j in hi_j], half)))
    xs = [_add(engine, rows[packs[k][0][0]], rot_rows[packs[k][1][0]] if packs[k][1] else None) for k in mine]
    ys = [_add(engine, cols[packs[k][0][1]], rot_cols[packs[k][1][1]] if packs[k][1] else None) for k in mine]
    cmp_mine = []
    if len(mine) > 1 and batched(engine):
        cmp_mine = engine.unstack(compare_kernel(engine, engine.stack(xs), engine.stack(ys), cfg))
        for _ in range(len(mine) - 1):
            engine.note_compare_eval()
    elif mine:
        cmp_mine = [compare_kernel(engine, x, y, cfg) for x, y in zip(xs, ys)]
    if valid_last < b:
        band, ones = _row_band_mask(slots, b, valid_last), np.ones(slots)
        for idx, k in enumerate(mine):
            lo, hi = packs[k]
            lo_pad, hi_pad = lo[1] == count - 1, hi is not None and hi[1] == count - 1
            if lo_pad or hi_pad:
                m = _two_halves(band if lo_pad else ones, band if hi_pad else ones, half)
                cmp_mine[idx] = engine.mul_plain(cmp_mine[idx], m, site="block-pad-mask")
    up = [[None, None] for _ in range(count)]
    low = [[None, None] for _ in range(count)]
    for c, k in zip(cmp_mine, mine):
        for h, pair in enumerate(packs[k]):
            if pair is None:
                continue
            i, j = pair
            up[i][h] = _add(engine, up[i][h], c)
            if j > i:
                low[j][h] = _add(engine, low[j][h], engine.add_plain(engine.negate(c), 1.0))
    parts = []
    for i in range(count):
        parts.extend([up[i][0], up[i][1], low[i][0], low[i][1]])
    summed = _sum_all(engine, parts, comm)
    owned = {}
    for i in range(count):
        if comm.owner(i) != comm.rank:
            continue
        u0, u1, l0, l1 = summed[4 * i: 4 * i + 4]
        upper = _add(engine, u0, engine.rotate(u1, half) if u1 is not None else None)
        lower = None
        if i > 0:
            lower = _add(engine, l0, engine.rotate(l1, half) if l1 is not None else None)
        owned[i] = finish_block_rank(engine, upper, lower, i, bv, layout, None)
    blocks = _gather_owned(engine, owned, count, comm)
    return MultiRankPipeline(
        ranks=BlockVector(blocks=tuple(blocks), block_size=b, total_len=bv.total_len),
        comparisons={"packed_mine": cmp_mine},
        row_replicated=rows,
        col_replicated=cols,
        layout=layout,
    )


def _multi_sort_sharded_packed(engine, bv: BlockVector, kcfg: KernelConfig, comm: Comm) -> BlockVector:
    from .packing import _add, _rot_many, _two_halves

    ranking = _multi_rank_sharded_packed(engine, bv, kcfg, comm)
    layout = ranking.layout
    b, count = bv.block_size, len(bv.blocks)
    slots = engine.params.slot_count
    half = slots // 2
    window = with_input_range(kcfg, -float(b * count), float(b * count))
    rank_blocks = common_level(engine, ranking.ranks.blocks)
    jpairs = [(j, j + 1 if j + 1 < count else None) for j in range(0, count, 2)]
    units = [(i, m) for i in range(count) for m in range(len(jpairs))]
    mine = [u for idx, u in enumerate(units) if comm.owner(idx) == comm.rank]
    ms = sorted({m for _, m in mine})
    need = sorted({j for m in ms for j in jpairs[m] if j is not None})
    if batched(engine) and len(need) > 1:
        spreads = dict(zip(need, engine.unstack(replicate(engine, engine.stack([rank_blocks[j] for j in need]),
                                                               layout, "row"))))
    else:
        spreads = {j: replicate(engine, rank_blocks[j], layout, "row") for j in need}
    his = [jpairs[m][1] for m in ms if jpairs[m][1] is not None]
    rot = _rot_many(engine, [spreads[j] for j in his] + [ranking.row_replicated[j] for j in his], half)
    rot_spread, rot_rowrep = dict(zip(his, rot[: len(his)])), dict(zip(his, rot[len(his):]))
    spread_p = {m: _add(engine, spreads[jpairs[m][0]], rot_spread.get(jpairs[m][1])) for m in ms}
    rowrep_p = {m: _add(engine, ranking.row_replicated[jpairs[m][0]], rot_rowrep.get(jpairs[m][1])) for m in ms}

    def targets(i):
        t = _neg_rank_targets(slots, b, "row", b * i + 1)
        return _two_halves(t, t, half)

    placed = []
    if batched(engine) and len(mine) > 1:
        tg = np.stack([targets(i) for i, _ in mine])
        shifted = engine.add_plain(engine.stack([spread_p[m] for _, m in mine]), tg)
        sel = indicator_kernel(engine, shifted, -0.5, 0.5, window, boundary="open")
        for _ in range(len(mine) - 1):
            engine.note_indicator_eval()
        placed = engine.unstack(engine.mul(sel, engine.stack([rowrep_p[m] for _, m in mine]), site="sort-place"))
    else:
        for i, m in mine:
            sel = indicator_kernel(engine, engine.add_plain(spread_p[m], targets(i)), -0.5, 0.5, window,
                                   boundary="open")
            placed.append(engine.mul(sel, rowrep_p[m], site="sort-place"))
    accs = [None] * count
    for (i, _), p in zip(mine, placed):
        accs[i] = _add(engine, accs[i], p)
    summed = _sum_all(engine, accs, comm)
    owned = {}
    for i in range(count):
        if comm.owner(i) != comm.rank:
            continue
        f = engine.add(summed[i], engine.rotate(summed[i], half))
        owned[i] = transpose_vector(engine, sum_axis(engine, f, layout, "col"), layout, "col_to_row")
    out = _gather_owned(engine, owned, count, comm)
    return BlockVector(blocks=tuple(out), block_size=b, total_len=bv.total_len)
