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
