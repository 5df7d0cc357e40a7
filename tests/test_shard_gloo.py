"""Multi-rank sharding of multi_rank / multi_sort (shard.py) with 2 gloo ranks
on the CPU oracle: every rank ends with ciphertext limbs bit-identical to the
single-process pipeline (modular sums are exact), for ranks and sort."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_2412_15126_b200 as M
from paper_2412_15126_b200.params import preset

KCFG = M.KernelConfig(mode="composite", composite=(3, 2), indicator_composite=(4, 2))
VALUES = np.random.default_rng(5).choice(256, 40, replace=False) / 256  # 3 blocks of 16


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _params(pname):
    # ring 2^12 (2048 slots, blocks of 32): two blocks fit one ciphertext (packing.py)
    return preset("toy_sort", log_n=12) if pname == "toy_sort12" else preset(pname)


def _worker(rank, world, port, what, out_dir, values=None, tie=False, packed=False, pname="toy_sort"):
    import torch.distributed as dist

    from oracle.oracle import oracle_engine
    from paper_2412_15126_b200.shard import Comm, multi_rank_sharded, multi_sort_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    eng = oracle_engine(_params(pname))
    bv = M.block_split(eng, VALUES if values is None else values)
    comm = Comm()
    if what == "rank":
        res = multi_rank_sharded(eng, bv, KCFG, comm, tie_correction=tie, packed=packed).ranks
    else:
        res = multi_sort_sharded(eng, bv, M.SortConfig(kernel=KCFG, tie_correction=tie, packed=packed), comm)
    np.savez(os.path.join(out_dir, f"{what}_{rank}.npz"), *[b.data for b in res.blocks],
             counts=np.array([comm.collectives, comm.level_syncs]))
    dist.destroy_process_group()


def _single(what):
    from oracle.oracle import oracle_engine

    eng = oracle_engine(preset("toy_sort"))
    bv = M.block_split(eng, VALUES)
    if what == "rank":
        res = M.multi_rank(eng, bv, KCFG)
    else:
        res = M.multi_sort(eng, bv, M.SortConfig(kernel=KCFG, tie_correction=False))
    return eng, res


@pytest.mark.slow
@pytest.mark.parametrize("what", ["rank", "sort"])
def test_two_rank_shards_are_bit_identical(tmp_path, what):
    mp.spawn(_worker, args=(2, _port(), what, str(tmp_path)), nprocs=2, join=True)
    eng, res = _single(what)
    for r in range(2):
        got = np.load(tmp_path / f"{what}_{r}.npz")
        assert len([f for f in got.files if f.startswith('arr_')]) == len(res.blocks)
        for i, blk in enumerate(res.blocks):
            assert np.array_equal(got[f"arr_{i}"], blk.data), (r, i)
    vals = M.block_merge(eng, res)
    if what == "rank":
        from oracle.plain import fractional_ranks

        assert np.array_equal(np.rint(vals), fractional_ranks(VALUES))
    else:
        assert np.abs(vals - np.sort(VALUES)).max() < 5e-3


TIES = np.repeat(np.random.default_rng(9).choice(64, 48, replace=False) / 64, 2)  # 96 values, all tied


@pytest.mark.slow
def test_three_rank_tie_corrected_sort_bit_identical_and_o1_collectives(tmp_path):
    """3 ranks, 3 unpadded blocks, tie correction (block tie offsets,
    reference ranking.py:395-423): bit-identical blocks, exactly one data
    collective per phase (5 phases) and no level exchange: every exchange's
    levels come from the cached level-tracer plan (levels.py)."""
    mp.spawn(_worker, args=(3, _port(), "sort", str(tmp_path), TIES, True), nprocs=3, join=True)
    from oracle.oracle import oracle_engine

    eng = oracle_engine(preset("toy_sort"))
    res = M.multi_sort(eng, M.block_split(eng, TIES), M.SortConfig(kernel=KCFG, tie_correction=True))
    for r in range(3):
        got = np.load(tmp_path / f"sort_{r}.npz")
        assert list(got["counts"]) == [5, 0]  # 5 collectives, no level exchange (levels.py plan)
        for i, blk in enumerate(res.blocks):
            assert np.array_equal(got[f"arr_{i}"], blk.data), (r, i)
    assert np.abs(M.block_merge(eng, res) - np.sort(TIES)).max() < 5e-2


PACKVALS = np.random.default_rng(11).choice(128, 96, replace=False) / 128  # 3 blocks of 32


@pytest.mark.slow
def test_three_rank_packed_sort_bit_identical(tmp_path):
    """The packed layout (packing.py) sharded over 3 ranks: packed comparisons and
    placements dealt round-robin, halves folded after the all-reduce -- the same
    limbs as the single-process packed sort."""
    mp.spawn(_worker, args=(3, _port(), "sort", str(tmp_path), PACKVALS, False, True, "toy_sort12"),
             nprocs=3, join=True)
    from oracle.oracle import oracle_engine

    eng = oracle_engine(_params("toy_sort12"))
    res = M.multi_sort(eng, M.block_split(eng, PACKVALS),
                       M.SortConfig(kernel=KCFG, tie_correction=False, packed=True))
    for r in range(3):
        got = np.load(tmp_path / f"sort_{r}.npz")
        assert list(got["counts"]) == [5, 0]  # 5 collectives, no level exchange (levels.py plan)
        for i, blk in enumerate(res.blocks):
            assert np.array_equal(got[f"arr_{i}"], blk.data), (r, i)
    assert np.abs(M.block_merge(eng, res) - np.sort(PACKVALS)).max() < 5e-3


def test_projected_comm_runs_one_ranks_share():
    """shard.ProjectedComm (bench.py's one-GPU projection of the W-rank sort): rank r's
    share runs through the real sharded code path with data-free collectives -- five
    collectives, no level exchange, and over all ranks exactly the single-process
    pipeline's ct x ct products (no unit is computed twice)."""
    from oracle.oracle import oracle_engine
    from paper_2412_15126_b200.shard import ProjectedComm, multi_sort_sharded

    eng = oracle_engine(preset("toy_sort"))
    bv = M.block_split(eng, VALUES)
    scfg = M.SortConfig(kernel=KCFG, tie_correction=False)
    eng.cost_reset()
    M.multi_sort(eng, bv, scfg)
    total = eng.cost_snapshot()
    world, ctct, cmps = 2, 0, 0
    for r in range(world):
        comm = ProjectedComm(r, world)
        eng.cost_reset()
        out = multi_sort_sharded(eng, bv, scfg, comm)
        c = eng.cost_snapshot()
        assert len(out.blocks) == len(bv.blocks)
        assert comm.collectives == 5 and comm.level_syncs == 0
        assert comm.all_reduce_bytes > 0 and comm.all_gather_bytes > 0
        assert c.ctct_mults < total.ctct_mults
        ctct += c.ctct_mults
        cmps += c.cmp_evals
    assert ctct == total.ctct_mults and cmps == total.cmp_evals
