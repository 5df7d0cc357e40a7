"""Multi-GPU sharding of the multi-ciphertext pipelines (N >= 256).

Restates reference ``multi_rank_pipeline`` / ``multi_sort``
(``pkg/src/slotrank/ranking.py:307-392``, ``sorting.py:106-142``) with the
independent units spread over ranks:

* the L(L+1)/2 block-pair comparisons C(i, j), i <= j, are dealt
  round-robin over ranks; each rank folds its own pairs into per-block
  partial sums  U_i = sum_{j>=i} C(i, j)  and  D_i = sum_{j<i} (1 - C(j, i));
* the L^2 indicator placements (i, j) of the sort are dealt the same way and
  folded into per-output-block partial sums;
* every partial sum is combined with ONE all-reduce of its RNS limbs
  (int64 sum -- limbs are < 2^60 and world <= 8, so no overflow) followed
  by a mod-q fix-up (``srk_reduce_mod`` on the GPU); block i is then finished
  (SumR / SumC / TransC / +1/2) by rank i % world and broadcast.

Modular addition is exact and associative, so the ciphertexts every rank
ends with are bit-identical to the single-GPU pipeline's for any world size
(tests/test_shard_gloo.py checks it with 2 gloo ranks on the CPU oracle).
Evaluation keys are replicated (every rank generates them from the shared
seed); only ciphertexts cross NVLink.  With world == 1 this is exactly the
single-GPU pipeline.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .chebyshev import KernelConfig, equality_from_compare, with_input_range
from .matrix import MatrixLayout, replicate, sum_axis, transpose_vector
from .ranking import (
    BlockVector,
    MultiRankPipeline,
    _triangle_mask,
    _prefix_vector,
    block_pairs,
    compare_block_pairs,
    finish_block_rank,
    lower_partial,
    replicated_blocks,
    upper_partial,
)
from .chebyshev import indicator_kernel
from .ranking import batched
from .sorting import SortConfig, _neg_rank_targets, common_level, place_block

__all__ = ["Comm", "multi_rank_sharded", "multi_sort_sharded"]

_NO_LEVEL = 1 << 20


@dataclass
class Comm:
    """torch.distributed process group wrapper (NCCL on GPUs, gloo on CPU)."""

    group: object = None

    def __post_init__(self):
        import torch.distributed as dist

        self.dist = dist
        self.rank = dist.get_rank(self.group)
        self.world = dist.get_world_size(self.group)

    def owner(self, unit_index: int) -> int:
        return unit_index % self.world

    def min_int(self, v: int) -> int:
        import torch

        t = torch.tensor([v], dtype=torch.int64, device=self._device())
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        return int(t.item())

    def _device(self):
        import torch

        return torch.device("cuda", torch.cuda.current_device()) if self.dist.get_backend(self.group) == "nccl" else "cpu"


def _sum_across(engine, ct, comm: Comm):
    """Modular sum over ranks of one ciphertext per rank (None = zero)."""
    if comm.world == 1:
        return ct
    level = comm.min_int(ct.level if ct is not None else _NO_LEVEL)
    if level == _NO_LEVEL:
        return None
    if ct is not None and ct.level != level:
        ct = engine.at_level(ct, level)
    t = engine.backend.as_tensor(ct.data) if ct is not None else engine.backend.zeros_tensor(level)
    comm.dist.all_reduce(t, group=comm.group)
    data = engine.backend.reduce_mod_tensor(t, level)
    return engine.wrap(data, level, ct.rot_chain if ct is not None else 0)


def _broadcast(engine, ct, src: int, comm: Comm):
    """Ciphertext held by rank ``src`` on every rank (level broadcast first)."""
    if comm.world == 1:
        return ct
    import torch

    lvl = torch.tensor([ct.level if comm.rank == src else 0], dtype=torch.int64, device=comm._device())
    comm.dist.broadcast(lvl, src, group=comm.group)
    level = int(lvl.item())
    t = engine.backend.as_tensor(ct.data) if comm.rank == src else engine.backend.zeros_tensor(level)
    comm.dist.broadcast(t, src, group=comm.group)
    return ct if comm.rank == src else engine.wrap(engine.backend.from_tensor(t, level), level, 0)


def multi_rank_sharded(engine, bv: BlockVector, cfg: KernelConfig, comm: Comm, *,
                       tie_correction: bool = False) -> MultiRankPipeline:
    """``multi_rank_pipeline`` with the block pairs dealt over ``comm``'s ranks."""
    b, count = bv.block_size, len(bv.blocks)
    layout = MatrixLayout(b, engine.params.slot_count)
    valid_last = bv.valid_in(count - 1)
    rows, cols = replicated_blocks(engine, bv, layout)
    pairs = block_pairs(count)
    mine = [p for idx, p in enumerate(pairs) if comm.owner(idx) == comm.rank]
    comparisons = compare_block_pairs(engine, mine, rows, cols, cfg, layout, count, valid_last)
    equalities = {p: equality_from_compare(engine, c) for p, c in comparisons.items()} if tie_correction else {}
    blocks = []
    for i in range(count):
        upper = _sum_across(engine, upper_partial(engine, comparisons, i, count), comm)
        lower = _sum_across(engine, lower_partial(engine, comparisons, i), comm) if i > 0 else None
        tie = None
        if tie_correction:
            parts = _tie_partials(engine, equalities, i, count, layout)
            parts = {k: _sum_across(engine, v, comm) for k, v in parts.items()}
        owner = comm.owner(i)
        if comm.rank == owner:
            if tie_correction:
                def tie(i=i, parts=parts):
                    return _finish_tie(engine, parts, i, bv.valid_in(i), layout)
            ranks_i = finish_block_rank(engine, upper, lower, i, bv, layout, tie)
        else:
            ranks_i = None
        blocks.append(_broadcast(engine, ranks_i, owner, comm))
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
    """``multi_sort`` with pairs and the L^2 placements dealt over ranks."""
    ranking = multi_rank_sharded(engine, bv, cfg.kernel, comm, tie_correction=cfg.tie_correction)
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
    out = []
    for i in range(count):
        acc = None
        for (ii, j) in mine:
            if ii != i:
                continue
            placed = placed_all.get((ii, j))
            if placed is None:
                placed = place_block(engine, spreads[j], ranking.row_replicated[j], i, layout, window)
            acc = placed if acc is None else engine.add(acc, placed)
        acc = _sum_across(engine, acc, comm)
        owner = comm.owner(i)
        blk = None
        if comm.rank == owner:
            blk = transpose_vector(engine, sum_axis(engine, acc, layout, "col"), layout, "col_to_row")
        out.append(_broadcast(engine, blk, owner, comm))
    return BlockVector(blocks=tuple(out), block_size=b, total_len=bv.total_len)
