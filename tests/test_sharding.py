"""Multi-rank frame sharding (CPU, gloo, world size 2): the N>1 path has no data-path collective;
ranks score disjoint contiguous frame blocks and the per-frame scores are gathered in frame
order after scoring (the reference's ordered frame loop, src/pipeline.py:319-328)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2101_06354_b200.video import shard_bounds


def test_shard_bounds_partition():
    for n in (0, 1, 7, 64, 300, 4800):
        for world in (1, 2, 3, 4, 8):
            blocks = [shard_bounds(n, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            for (a0, a1), (b0, b1) in zip(blocks, blocks[1:]):
                assert a1 == b0
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(Exception):
        shard_bounds(10, 2, 2)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, n_frames: int, out_dir: str):
    import torch.distributed as dist

    from oracle import ssim_oracle as O
    from paper_2101_06354_b200.video import gather_frame_scores, shard_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    start, stop = shard_bounds(n_frames, rank, world)
    # each rank "scores" its own frames (the CPU oracle stands in for the GPU kernel here)
    rng = np.random.default_rng(1234)
    frames = [(rng.integers(0, 256, (24, 30)).astype(np.uint8), rng.integers(0, 256, (24, 30)).astype(np.uint8))
              for _ in range(n_frames)]
    local = np.array([O.ssim_score(*frames[i], shape="rect", k=7) for i in range(start, stop)])
    allv = gather_frame_scores(local, n_frames)
    if rank == 0:
        np.save(os.path.join(out_dir, "gathered.npy"), allv)
    dist.destroy_process_group()


def test_gloo_two_ranks_gather_in_frame_order(tmp_path):
    from oracle import ssim_oracle as O

    n = 7
    mp.spawn(_worker, args=(2, _free_port(), n, str(tmp_path)), nprocs=2, join=True)
    got = np.load(tmp_path / "gathered.npy")
    rng = np.random.default_rng(1234)
    frames = [(rng.integers(0, 256, (24, 30)).astype(np.uint8), rng.integers(0, 256, (24, 30)).astype(np.uint8))
              for _ in range(n)]
    want = np.array([O.ssim_score(a, b, shape="rect", k=7) for a, b in frames])
    assert np.array_equal(got, want)
