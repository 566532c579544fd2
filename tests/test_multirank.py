"""World-size-2 gloo tests of the multi-GPU host logic (CPU only).

Each rank takes its frame shard (weak and strong schemes), computes masks
for its frames (here with the CPU oracle standing in for the GPU kernels,
which these tests cannot run), reduces its timing with max-over-ranks and
gathers the masks to rank 0, which checks them against a single-process run.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2408_14050_b200 import shard


def test_weak_and_strong_shards():
    assert shard.weak_shard(256, 0) == (0, 256)
    assert shard.weak_shard(256, 3) == (768, 256)
    blocks = [shard.strong_shard(10, 4, r) for r in range(4)]
    assert blocks == [(0, 3), (3, 3), (6, 2), (8, 2)]
    assert sum(n for _, n in blocks) == 10
    for total in (0, 1, 7, 256):
        for world in (1, 2, 3, 8):
            spans = [shard.strong_shard(total, world, r) for r in range(world)]
            covered = [f for a, n in spans for f in range(a, a + n)]
            assert covered == list(range(total))
    with pytest.raises(ValueError):
        shard.strong_shard(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2408_14050_b200 import scenes
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    first, n = shard.strong_shard(5, world, rank)
    views = scenes.VIEWS_3X3
    frames = [scenes.make_scene(2, 0, f)[:96, :128].copy() for f in range(first, first + n)]
    masks = np.stack([oracle.detect(D, views) for D in frames]) if n else np.zeros((0, 8, 96, 128), np.uint8)
    # pad to equal shapes for gather (3 + 2 frames)
    pad = np.zeros((3, 8, 96, 128), np.uint8)
    pad[:n] = masks
    t = shard.max_over_ranks(float(rank + 1))
    got = shard.gather_to_rank0(torch.from_numpy(pad))
    dist.barrier()
    if rank == 0:
        allm = []
        for r, m in enumerate(got):
            a, k = shard.strong_shard(5, world, r)
            allm.append(m.numpy()[:k])
        np.save(os.path.join(out_dir, "masks.npy"), np.concatenate(allm))
        with open(os.path.join(out_dir, "t.txt"), "w") as f:
            f.write(str(t))
    dist.destroy_process_group()


def test_two_rank_gloo_shard_gather(tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    import oracle
    from paper_2408_14050_b200 import scenes
    got = np.load(tmp_path / "masks.npy")
    ref = np.stack([oracle.detect(scenes.make_scene(2, 0, f)[:96, :128].copy(), scenes.VIEWS_3X3)
                    for f in range(5)])
    assert got.shape == ref.shape and (got == ref).all()
    assert float((tmp_path / "t.txt").read_text()) == 2.0    # max over ranks


def _view_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2408_14050_b200 import scenes
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    views = scenes.config_views(4)                      # 24 views of the 5x5 array
    D = scenes.make_scene(4)[:64, :96].copy()
    mine = shard.view_shard(views, world, rank)
    m = oracle.detect(D, [b for _, b in mine])
    pad = np.zeros((8, 64, 96), np.uint8)                # 24 views / 3 ranks
    pad[:len(mine)] = m
    got = shard.gather_to_rank0(torch.from_numpy(pad))
    if rank == 0:
        allm = [g.numpy()[:len(shard.view_shard(views, world, r))] for r, g in enumerate(got)]
        np.save(os.path.join(out_dir, "views.npy"), np.concatenate(allm))
    dist.destroy_process_group()


def test_view_shards_cover_all_views():
    from paper_2408_14050_b200 import scenes
    views = scenes.config_views(4)
    for world in (1, 2, 3, 8, 24):
        got = [i for r in range(world) for i, _ in shard.view_shard(views, world, r)]
        assert got == list(range(24))


def test_three_rank_gloo_view_shards(tmp_path):
    import oracle
    from paper_2408_14050_b200 import scenes
    mp.spawn(_view_worker, args=(3, _free_port(), str(tmp_path)), nprocs=3, join=True)
    D = scenes.make_scene(4)[:64, :96].copy()
    ref = oracle.detect(D, scenes.config_views(4))
    assert (np.load(tmp_path / "views.npy") == ref).all()
