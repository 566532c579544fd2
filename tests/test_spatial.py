"""Single-frame spatial sharding (paper_2408_14050_b200/spatial.py, NEXT #4):
row bands + all-reduced Eq. 3 statistics + 2h+2 halo rows exchanged
point-to-point, world sizes 2 and 3 over gloo on CPU.  Each rank's band is
detected by the oracle with the imposed whole-frame range (orc_detect_range,
standing in for the GPU kernels these tests cannot run); rank 0 gathers the
interior rows and the result must equal the oracle on the whole frame, for
N = infinity and N = 8.  Also pins orc_detect_range itself."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2408_14050_b200 import scenes, spatial

VIEWS = [(1, 0), (-1, 0), (0, 1), (0, -1), (1, 1), (-1, 1), (2, 1), (0, 2)]


def frame(seed, H=90, W=120):
    rng = scenes.SplitMix64(4101, seed)
    y = np.arange(H, dtype=np.float64)[:, None]
    img = np.broadcast_to(1.0 + 2.0 * y / (H - 1), (H, W)).copy()
    shapes = []
    for i in range(9):
        u = rng.uniform(5)
        shapes.append((1.0 + 11.0 * u[4], i, u[0] * (W - 1), u[1] * (H - 1), 2 + u[2] * W / 5, 2 + u[3] * H / 5))
    for d, _, cx, cy, ax, ay in sorted(shapes):
        img[max(0, int(cy - ay)):min(H, int(cy + ay) + 1), max(0, int(cx - ax)):min(W, int(cx + ax) + 1)] = d
    img += 0.25 * rng.normal(H * W).reshape(H, W)
    return img.astype(np.float32)


def test_bands_and_halo():
    assert spatial.bands(10, 3) == [(0, 4), (4, 7), (7, 10)]
    for H in (2, 7, 90, 1080):
        for world in (1, 2, 3, 8):
            if world > H:
                continue
            b = spatial.bands(H, world)
            assert b[0][0] == 0 and b[-1][1] == H and all(b[i][1] == b[i + 1][0] for i in range(world - 1))
    with pytest.raises(ValueError):
        spatial.bands(2, 3)
    assert spatial.halo_rows([3, 9, 4]) == 20
    assert spatial.extended(10, 20, 15, 40) == (0, 35)


def oracle_h(lo, hi, views=None):
    """Eq. 3's h per view from the oracle's scan length (test infrastructure)."""
    import oracle
    return [oracle.scan_length(lo, hi, max(abs(bx), abs(by))) // 2 for bx, by in (views or VIEWS)]


def test_detect_range_pins(orc):
    D = frame(0)
    lo, hi, _ = orc.stats(D)
    # the frame's own statistics: identical to orc_detect / orc_detect_n
    assert (orc.detect_range(D, VIEWS, lo, hi) == orc.detect(D, VIEWS)).all()
    assert (orc.detect_range(D, VIEWS, lo, hi, neighbors=8) == orc.detect(D, VIEWS, neighbors=8)).all()
    # a constant band of a non-constant frame: h > 0 but no candidates -> zero
    assert orc.detect_range(np.full((12, 16), 3.0, np.float32), VIEWS, 1.0, 9.0).sum() == 0
    with pytest.raises(ValueError):
        orc.detect_range(D, VIEWS, 2.0, 1.0)
    # a band with the whole frame's range equals the whole frame's rows when
    # the band holds every window of those rows (2h + 2 halo rows)
    halo = spatial.halo_rows(oracle_h(lo, hi))
    full = orc.detect(D, VIEWS)
    e0, e1 = spatial.extended(40, 50, halo, D.shape[0])
    part = orc.detect_range(D[e0:e1], VIEWS, lo, hi)
    assert (part[:, 40 - e0:50 - e0] == full[:, 40:50]).all()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir, N, bad):
    import torch
    import torch.distributed as dist

    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    D = frame(7)
    if bad:
        D[D.shape[0] - 3, 5] = np.nan         # only the last rank sees it
    H = D.shape[0]
    r0, r1 = spatial.bands(H, world)[rank]
    band = torch.from_numpy(D[r0:r1].copy())

    def stats_fn(b):
        lo, hi, nb = oracle.stats(b.numpy())
        return lo, hi, nb

    def detect_fn(ext, dmin, dmax, nbad):
        if nbad:
            return np.zeros((len(VIEWS),) + tuple(ext.shape), np.uint8)
        return oracle.detect_range(ext.numpy(), VIEWS, dmin, dmax, neighbors=N)

    part, st = spatial.detect_band(band, r0, r1, H, VIEWS, rank, world, stats_fn, detect_fn, oracle_h)
    full = spatial.gather_rows(torch.from_numpy(np.ascontiguousarray(part)), r0, r1, H, world, rank)
    if rank == 0:
        np.save(os.path.join(out_dir, "masks.npy"), full.numpy())
        np.save(os.path.join(out_dir, "stats.npy"), np.array(st, np.float64))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,N", [(2, 0), (3, 0), (3, 8), (4, 2)])
def test_gloo_row_bands_equal_whole_frame(tmp_path, world, N):
    import oracle
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), N, False), nprocs=world, join=True)
    D = frame(7)
    got = np.load(tmp_path / "masks.npy")
    ref = oracle.detect(D, VIEWS, neighbors=N)
    assert got.shape == ref.shape and (got == ref).all()
    lo, hi, nb = oracle.stats(D)
    st = np.load(tmp_path / "stats.npy")
    assert st[0] == lo and st[1] == hi and st[2] == 0
    # the halo exceeds a band here (bands of 30 or 22 rows): rows come from
    # ranks two bands away as well
    assert spatial.halo_rows(oracle_h(lo, hi)) > D.shape[0] // world


def test_gloo_nonfinite_rejects_whole_frame(tmp_path):
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), 0, True), nprocs=2, join=True)
    assert np.load(tmp_path / "masks.npy").sum() == 0
    assert np.load(tmp_path / "stats.npy")[2] == 1
