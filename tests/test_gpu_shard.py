"""shard.py on the CUDA backend: 2 ranks (gloo collectives, both ranks on
cuda:0) run the sharded multi_rank / multi_sort and end with ciphertext limbs
bit-identical to the single-process GPU pipeline.  On an 8-GPU box the same
code runs one rank per GPU over NCCL (bench.py --gpus N)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_2412_15126_b200 as M
from paper_2412_15126_b200.params import preset

KCFG = M.KernelConfig(mode="composite", composite=(3, 2), indicator_composite=(4, 2))
VALUES = np.random.default_rng(7).choice(512, 40, replace=False) / 512  # 3 blocks of 16


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, what, out_dir, backend="gloo"):
    import torch
    import torch.distributed as dist

    from paper_2412_15126_b200.shard import Comm, multi_rank_sharded, multi_sort_sharded

    dev = rank if backend == "nccl" else 0
    torch.cuda.set_device(dev)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    eng = M.B200Engine(preset("toy_sort"))
    bv = M.block_split(eng, VALUES)
    comm = Comm()
    if what == "rank":
        res = multi_rank_sharded(eng, bv, KCFG, comm).ranks
    else:
        res = multi_sort_sharded(eng, bv, M.SortConfig(kernel=KCFG, tie_correction=False), comm)
    np.savez(os.path.join(out_dir, f"{what}_{rank}.npz"),
             *[b.data.cpu().numpy().view(np.uint64) for b in res.blocks])
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("backend", ["gloo", "nccl"])
@pytest.mark.parametrize("what", ["rank", "sort"])
def test_two_rank_gpu_shards_are_bit_identical(tmp_path, what, backend, require_cuda):
    import torch

    if backend == "nccl" and torch.cuda.device_count() < 2:
        pytest.skip("NCCL sharding needs 2 GPUs (one rank per GPU)")
    mp.spawn(_worker, args=(2, _port(), what, str(tmp_path), backend), nprocs=2, join=True)
    eng = M.B200Engine(preset("toy_sort"))
    bv = M.block_split(eng, VALUES)
    if what == "rank":
        res = M.multi_rank(eng, bv, KCFG)
    else:
        res = M.multi_sort(eng, bv, M.SortConfig(kernel=KCFG, tie_correction=False))
    for r in range(2):
        got = np.load(tmp_path / f"{what}_{r}.npz")
        assert len(got.files) == len(res.blocks)
        for i, blk in enumerate(res.blocks):
            assert np.array_equal(got[f"arr_{i}"], blk.data.cpu().numpy().view(np.uint64)), (r, i)
    vals = M.block_merge(eng, res)
    if what == "rank":
        from oracle.plain import fractional_ranks

        assert np.array_equal(np.rint(vals), fractional_ranks(VALUES))
    else:
        assert np.abs(vals - np.sort(VALUES)).max() < 5e-3
