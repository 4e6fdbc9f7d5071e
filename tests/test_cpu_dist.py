"""N>1 bench plumbing on CPU (gloo, world_size 2): every rank reports its own
replica time, the job time is the max over ranks, and only rank 0 prints."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = 10.0 + 5.0 * rank
    out[rank] = bench.max_over_ranks(mine, dist, torch.device("cpu"))
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    port = _free_port()
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        out = mgr.dict()
        mp.start_processes(_worker, args=(2, port, out), nprocs=2, join=True, start_method="spawn")
        assert dict(out) == {0: 15.0, 1: 15.0}


def test_max_over_ranks_single_process():
    assert bench.max_over_ranks(3.5) == 3.5


def test_reference_arm_nonzero_rank_exits_quietly(monkeypatch, capsys):
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "2")

    class A:
        n, steps, warmup = 64, 1, 0
    assert bench.run_reference(A()) == 0
    assert capsys.readouterr().out == ""


# ---------------------------------------------------------------------------
# Column-sharded solve: host-side logic (partition, host-staged broadcast)

def test_shard_range_matches_c_abi_and_partitions():
    import ctypes as C

    from paper_1501_03830_b200 import _lib
    from paper_1501_03830_b200.distributed import shard_range
    lib = _lib.load()
    for n in (0, 1, 2, 3, 7, 64, 301, 16384):
        for world in (1, 2, 3, 4, 8):
            cover = []
            for r in range(world):
                c0, c1 = C.c_int64(), C.c_int64()
                assert lib.bse_shard_range(n, world, r, C.byref(c0), C.byref(c1)) == 0
                assert (c0.value, c1.value) == shard_range(n, world, r)
                cover += list(range(c0.value, c1.value))
            assert cover == list(range(n))
    c0, c1 = C.c_int64(), C.c_int64()
    assert lib.bse_shard_range(10, 2, 2, C.byref(c0), C.byref(c1)) == _lib.BSE_BAD_ARGUMENT


def _shard_worker(rank, world, port, out):
    import numpy as np

    from oracle import bse_oracle as orc
    from paper_1501_03830_b200 import configs
    from paper_1501_03830_b200.distributed import allgather_cols_host, make_host_bcast, shard_range
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b, _ = configs.config_operator(0, n=37)
    lam, x1, x2 = orc.solve_complex(a, b)
    n = lam.size
    # each rank keeps only its own column block, then the blocks are
    # broadcast from their owners exactly as the device transport does
    c0, c1 = shard_range(n, world, rank)
    mine = np.zeros((2 * n, n))
    mine[:, c0:c1] = np.vstack([x1.real, x2.real])[:, c0:c1]
    full = allgather_cols_host(mine, world, rank, make_host_bcast())
    out[rank] = float(np.max(np.abs(full - np.vstack([x1.real, x2.real]))))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_columns_allgather_gloo_world2():
    port = _free_port()
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        out = mgr.dict()
        mp.start_processes(_shard_worker, args=(2, port, out), nprocs=2, join=True,
                           start_method="spawn")
        assert dict(out) == {0: 0.0, 1: 0.0}


# ---------------------------------------------------------------------------
# Block-cyclic column layout of the memory-distributed solve (csrc/dist.cuh)

def test_bc_index_maps_match_the_library():
    """bse_bc_local_cols / bse_bc_global_col (C ABI) against the Python mirror
    and a brute-force owner map, ragged and degenerate shapes included."""
    from paper_1501_03830_b200 import _lib
    from paper_1501_03830_b200.distributed import bc_local_cols, bc_owner
    lib = _lib.load()
    for n, nb, world in [(0, 64, 2), (1, 64, 3), (100, 64, 3), (1100, 128, 2), (4096, 512, 8),
                         (4097, 512, 8), (65536, 1024, 8), (700, 128, 1)]:
        seen = np.zeros(n, dtype=int)
        for r in range(world):
            cols = bc_local_cols(n, nb, world, r)
            assert lib.bse_bc_local_cols(n, nb, world, r) == len(cols)
            for lc in (0, len(cols) // 2, len(cols) - 1):
                if 0 <= lc < len(cols):
                    assert lib.bse_bc_global_col(lc, nb, world, r) == cols[lc]
            assert all(bc_owner(c // nb, world) == r for c in cols[:: max(1, len(cols) // 50)])
            assert np.all(np.diff(cols) > 0)
            seen[cols] += 1
        assert np.all(seen == 1)
    assert lib.bse_bc_local_cols(100, 100, 2, 0) == -1  # nb must be a multiple of 64


def _bc_gloo_worker(rank, world, port, out):
    import torch.distributed as dist
    from paper_1501_03830_b200.distributed import bc_gather, bc_local_cols, bc_scatter
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, nb = 300, 64
    a = np.arange(7 * n, dtype=np.float64).reshape(7, n)
    mine = np.ascontiguousarray(bc_scatter(a, nb, world, rank))
    blocks = [None] * world
    dist.all_gather_object(blocks, mine)
    back = bc_gather(blocks, n, nb)
    out[rank] = bool(np.array_equal(back, a)) and len(bc_local_cols(n, nb, world, rank)) == mine.shape[1]
    dist.barrier()
    dist.destroy_process_group()


def test_bc_scatter_gather_gloo_world2():
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        out = mgr.dict()
        mp.start_processes(_bc_gloo_worker, args=(2, port, out), nprocs=2, join=True,
                           start_method="spawn")
        assert dict(out) == {0: True, 1: True}
