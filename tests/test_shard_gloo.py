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


def _worker(rank, world, port, what, out_dir):
    import torch.distributed as dist

    from oracle.oracle import oracle_engine
    from paper_2412_15126_b200.shard import Comm, multi_rank_sharded, multi_sort_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    eng = oracle_engine(preset("toy_sort"))
    bv = M.block_split(eng, VALUES)
    comm = Comm()
    if what == "rank":
        res = multi_rank_sharded(eng, bv, KCFG, comm).ranks
    else:
        res = multi_sort_sharded(eng, bv, M.SortConfig(kernel=KCFG, tie_correction=False), comm)
    np.savez(os.path.join(out_dir, f"{what}_{rank}.npz"), *[b.data for b in res.blocks])
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
        assert len(got.files) == len(res.blocks)
        for i, blk in enumerate(res.blocks):
            assert np.array_equal(got[f"arr_{i}"], blk.data), (r, i)
    vals = M.block_merge(eng, res)
    if what == "rank":
        from oracle.plain import fractional_ranks

        assert np.array_equal(np.rint(vals), fractional_ranks(VALUES))
    else:
        assert np.abs(vals - np.sort(VALUES)).max() < 5e-3
