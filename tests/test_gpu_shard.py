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
    first = rb.gather()
    assert torch.equal(first, full)
    # the next frame lands in the other half of the double-buffered IPC image,
    # so the previous image stays intact until the next gather()
    rf2 = torch.from_numpy(configs.noise_rf(p.num_transmits, arr.num_elements, p.num_samples,
                                            seed=5)).cuda()
    full2 = full_eng.run(rf2[None]).clone()[0]
    rb.beamform_block(rf2)
    torch.cuda.synchronize()
    assert torch.equal(first, full)
    assert torch.equal(rb.gather(), full2)
    rb.beamform_block(rf)
    assert torch.equal(rb.gather(), full)
    rb.close()
    full_eng.close()


def _full_traces(w, rf, frames):
    eng = kb.KKEngine(w.array, w.params, w.receive, w.grid, frames=frames, want_db=False)
    tr = eng.decompose(rf).clone()
    eng.close()
    return tr


@pytest.mark.parametrize("cfg,T,frames,world,odd_l", [(4, None, 2, 3, False), (5, None, 1, 8, False),
                                                      (1, 1000, 2, 3, False), (1, None, 2, 3, True),
                                                      (1, 1000, 3, 2, True)])
def test_transmit_sharded_stage1_scatter_assembles_every_trace_buffer(cfg, T, frames, world, odd_l):
    # transmit-sharded stage 1 on one GPU: `world` "ranks" each decompose their
    # transmit block and the inverse FFT's epilogue stores the rows into all
    # ranks' full trace buffers (fused for the compile-time lengths, strided
    # copies after the transform for T = 1000); every buffer must equal the
    # single-plan decomposition bit for bit
    import ctypes

    import torch

    from paper_2603_22496_b200 import _device as dev
    from paper_2603_22496_b200 import _lib

    w = configs.CONFIGS[cfg]()
    p, arr = w.params, w.array
    if T is not None:
        p = kb.AcquisitionParams(p.sound_speed, p.transmit_angles, T, start_time=p.start_time)
        w = configs.Workload(w.name, arr, p, w.receive, w.grid)
    if odd_l:  # 63 elements: rows pair only within one (frame, transmit)
        arr = kb.TransducerArray(63, arr.pitch, arr.center_frequency, arr.sampling_frequency,
                                 arr.fractional_bandwidth)
        w = configs.Workload(w.name, arr, p, w.receive, w.grid)
    N, M, L, TT = p.num_transmits, w.receive.num_angles, arr.num_elements, p.num_samples
    rf = torch.from_numpy(np.stack([configs.noise_rf(N, L, TT, seed=30 + f)
                                    for f in range(frames)])).cuda()
    full = _full_traces(w, rf, frames)
    bufs = [torch.full((frames, N, M, TT), complex(5, 5), dtype=torch.complex64, device="cuda")
            for _ in range(world)]
    dsts = (ctypes.c_void_p * world)(*[b.data_ptr() for b in bufs])
    pos = np.ascontiguousarray(arr.positions, dtype=np.float64)
    ang = np.ascontiguousarray(w.receive.angles, dtype=np.float64)
    for r in range(world):
        n0, n1 = shard.balanced_range(N, r, world)
        h = ctypes.c_void_p()
        _lib.call("kkb_decomposer_create", n1 - n0, L, TT, pos.ctypes.data, ang.ctypes.data, M,
                  float(arr.sampling_frequency), float(p.sound_speed), frames, ctypes.byref(h))
        sub = rf[:, n0:n1].contiguous()
        _lib.call("kkb_decomposer_run_scatter", h, dev.ptr(sub), 0, frames, dsts, world,
                  n0 * M * TT, N * M * TT, dev.stream_handle())
        torch.cuda.synchronize()
        _lib.load().kkb_decomposer_destroy(h)
    for b in bufs:
        assert torch.equal(b, full)


def test_decomposer_scatter_rejects_bad_arguments():
    import ctypes

    from paper_2603_22496_b200 import _lib
    from paper_2603_22496_b200.errors import ConfigError

    w = configs.config1()
    p, arr = w.params, w.array
    pos = np.ascontiguousarray(arr.positions, dtype=np.float64)
    ang = np.ascontiguousarray(w.receive.angles, dtype=np.float64)
    h = ctypes.c_void_p()
    N, M, T = p.num_transmits, w.receive.num_angles, p.num_samples
    _lib.call("kkb_decomposer_create", N, arr.num_elements, T, pos.ctypes.data, ang.ctypes.data, M,
              float(arr.sampling_frequency), float(p.sound_speed), 1, ctypes.byref(h))
    one = (ctypes.c_void_p * 1)(16)
    nine = (ctypes.c_void_p * 9)(*([16] * 9))
    for dsts, n, stride in ((one, 0, N * M * T), (nine, 9, N * M * T), (one, 1, N * M * T - 1)):
        with pytest.raises(ConfigError):
            _lib.call("kkb_decomposer_run_scatter", h, None, 0, 1, dsts, n, 0, stride, None)
    _lib.load().kkb_decomposer_destroy(h)


@pytest.mark.parametrize("transport", ["p2p", "nccl"])
@pytest.mark.parametrize("cfg", [1, 5])
def test_sharded_stage1_single_rank_is_the_full_image(cfg, transport):
    import torch

    w = configs.CONFIGS[cfg]()
    p, arr = w.params, w.array
    rf = torch.from_numpy(configs.noise_rf(p.num_transmits, arr.num_elements, p.num_samples,
                                           seed=6)).cuda()
    full_eng = kb.KKEngine(arr, p, w.receive, w.grid, frames=1, want_db=False)
    full = full_eng.run(rf[None]).clone()[0]
    rb = shard.RowBlockKK(arr, p, w.receive, w.grid, 0, 1, transport=transport, stage1="sharded")
    assert rb.transport == transport and rb.engine is None
    rb.beamform_block(rf)
    assert torch.equal(rb.gather(), full)
    rb.beamform_block(rf)  # rerun: identical
    assert torch.equal(rb.gather(), full)
    rb.close()
    full_eng.close()
