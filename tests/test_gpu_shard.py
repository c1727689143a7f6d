"""Row-block sharding on one GPU: the blocks every rank would compute,
concatenated, are bit-identical to the single-GPU image (the all-gather
itself is covered by tests/test_multirank_gloo.py)."""

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu

import paper_2603_22496_b200 as kb  # noqa: E402
from paper_2603_22496_b200 import configs, shard  # noqa: E402


@pytest.mark.parametrize("cfg,worlds", [(1, (2, 3)), (5, (8,))])
def test_row_blocks_concatenate_to_full_image(cfg, worlds):
    import torch

    w = configs.CONFIGS[cfg]()
    p, arr = w.params, w.array
    rf = configs.noise_rf(p.num_transmits, arr.num_elements, p.num_samples, seed=21)
    rf_d = torch.from_numpy(rf).cuda()
    full_eng = kb.KKEngine(arr, p, w.receive, w.grid, frames=1, want_db=False)
    full = full_eng.run(rf_d[None]).clone()[0]
    torch.cuda.synchronize()
    for world in worlds:
        blocks = []
        for r in range(world):
            rb = shard.RowBlockKK(arr, p, w.receive, w.grid, r, world)
            blocks.append(rb.beamform_block(rf_d).clone())
            torch.cuda.synchronize()
            rb.close()
        got = torch.cat(blocks, dim=0)
        assert got.shape == full.shape
        assert torch.equal(got, full), world
    full_eng.close()


def test_scatter_epilogue_assembles_every_image_buffer():
    # the fused row-block all-gather on one GPU: three "ranks" run their row
    # blocks one after another, each storing its rows into all three image
    # buffers (in a multi-GPU run these are peers' buffers mapped over NVLink)
    import ctypes

    import torch

    from paper_2603_22496_b200 import _device as dev
    from paper_2603_22496_b200 import _lib

    w = configs.config1()
    p, arr, g = w.params, w.array, w.grid
    rf = torch.from_numpy(configs.noise_rf(p.num_transmits, arr.num_elements, p.num_samples,
                                           seed=3)).cuda()
    full_eng = kb.KKEngine(arr, p, w.receive, g, frames=1, want_db=False)
    full = full_eng.run(rf[None]).clone()[0]
    imgs = [torch.full((g.nx, g.nz), complex(7, 7), dtype=torch.complex64, device="cuda")
            for _ in range(3)]
    dsts = (ctypes.c_void_p * 3)(*[x.data_ptr() for x in imgs])
    for r in range(3):
        rb = shard.RowBlockKK(arr, p, w.receive, g, r, 3, transport="nccl")
        rb.engine.decompose(rf[None], n_frames=1)
        _lib.call("kkb_kk_plan_run_scatter", rb._plan, dev.ptr(rb.engine.traces), 1, 0, dsts, 3,
                  rb.ix0 * g.nz, _lib.KKB_OUT_C64, 0, dev.stream_handle())
        torch.cuda.synchronize()
        rb.close()
    for x in imgs:
        assert torch.equal(x, full)
    full_eng.close()


def test_p2p_transport_single_rank_is_the_full_image():
    import torch

    w = configs.config1()
    p, arr = w.params, w.array
    rf = torch.from_numpy(configs.noise_rf(p.num_transmits, arr.num_elements, p.num_samples,
                                           seed=4)).cuda()
    full_eng = kb.KKEngine(arr, p, w.receive, w.grid, frames=1, want_db=False)
    full = full_eng.run(rf[None]).clone()[0]
    rb = shard.RowBlockKK(arr, p, w.receive, w.grid, 0, 1, transport="p2p")
    assert rb.transport == "p2p"
    rb.beamform_block(rf)
    assert torch.equal(rb.gather(), full)
    rb.close()
    full_eng.close()
