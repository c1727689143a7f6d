"""Multi-rank host logic on the CPU (gloo, world size 2 and 3): partitions,
the row-block all-gather and its bit-identity with the single-rank image,
the transmit-block trace all-gather of sharded stage 1.
The per-rank compute is the oracle here (no GPU in this container); on the
GPU the same partition drives the K5 kernel (tests/test_gpu_shard.py)."""

import os
import socket

import numpy as np
import pytest

from conftest import golden

from paper_2603_22496_b200 import shard


def test_balanced_ranges_cover_exactly():
    for count in (0, 1, 7, 400, 1024):
        for world in (1, 2, 3, 4, 8):
            got = [shard.balanced_range(count, r, world) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == count
            for (b0, e0), (b1, e1) in zip(got, got[1:]):
                assert e0 == b1
            sizes = [e - b for b, e in got]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard.balanced_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    from oracle import kkbeam_oracle as O

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = golden("config1")
        luts = [g[k] for k in ("ltx", "ltz", "lrx", "lrz")]
        nx, nz = luts[0].shape[0], luts[1].shape[0]
        fs, t0 = 20e6, 6e-6
        ix0, ix1 = shard.row_block_range(nx, rank, world)
        part = O.kk_kernel(g["compressed"], *luts, np.ones(11), fs, (0.0 - t0) * fs,
                           p_range=(ix0 * nz, ix1 * nz), threads=1)
        block = torch.from_numpy(part.astype(np.complex64).reshape(ix1 - ix0, nz))
        full = shard.gather_row_blocks(block, nx, nz)
        # P2P transport plumbing: every rank receives all 64-byte handles in rank order
        hs = shard.exchange_handles(bytes([rank]) * 64)
        assert hs == [bytes([r]) * 64 for r in range(world)]
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), full.numpy())
        # transmit-sharded stage 1 (NCCL-form fallback): each rank holds the
        # traces of its transmit block; the all-gather rebuilds (N, M, T)
        comp = g["compressed"].astype(np.complex64)
        n0, n1 = shard.balanced_range(comp.shape[0], rank, world)
        tr = shard.gather_transmit_blocks(torch.from_numpy(comp[n0:n1].copy()), comp.shape[0])
        assert np.array_equal(tr.numpy(), comp)
        # frame sharding: each rank sums its frames' ids; all-reduce checks coverage
        b, e = shard.frame_range(400, rank, world)
        t = torch.tensor([float(sum(range(b, e)))])
        dist.all_reduce(t)
        np.save(os.path.join(out_dir, f"frames{rank}.npy"), t.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_block_gather_is_bit_identical(tmp_path, world):
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    ref = golden("config1")["image"].astype(np.complex64)
    for r in range(world):
        got = np.load(tmp_path / f"rank{r}.npy")
        assert got.shape == ref.shape
        assert np.array_equal(got, ref), r
        assert float(np.load(tmp_path / f"frames{r}.npy")[0]) == sum(range(400))
