"""Single-frame spatial sharding: one frame split into
row bands across ranks, for frames larger than one GPU's share.

Why it is exact.  A pixel's mark depends on the frame only through
  * Eq. 3's min / max: the ranks all-reduce their band
    statistics (MAX of -dmin and dmax, SUM of the non-finite count) and impose
    the result with occ_set_frame_stats;
  * the samples of the scan windows that contain it (Eq. 4):
    a window is centred on a candidate within h of the pixel along its line
    and reaches h further, so every relevant sample lies within 2h line steps,
    i.e. within 2h rows for any line family; the candidates themselves need
    E_y, one row further down (Eq. 1).  A band extended by 2h + 2 rows on each
    side (clipped to the frame) therefore holds every window of its interior
    pixels complete, with the frame's own border clipping where the band
    touches it.
The halo rows come from the ranks that own them (point-to-point send/recv:
NCCL for device tensors, gloo for host tensors in the CPU tests).  The
per-band detection itself is the library's (occ_detect on the extended band
with the imposed statistics); nothing here computes masks.
"""
from __future__ import annotations

from typing import Callable, List, Sequence, Tuple

import numpy as np


def bands(H: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous near-equal row bands [r0, r1) of an H-row frame."""
    if world < 1 or H < world:
        raise ValueError("need 1 <= world <= H")
    base, extra = divmod(H, world)
    out, r = [], 0
    for k in range(world):
        n = base + (1 if k < extra else 0)
        out.append((r, r + n))
        r += n
    return out


def halo_rows(h_per_view: Sequence[int]) -> int:
    """Rows of halo each side of a band: 2 max(h) + 2 (see the module doc).
    h_per_view: Eq. 3's scan half-lengths under the whole frame's statistics
    (occ_scan_half_lengths through device_fns' h_fn; this module computes no
    part of the method)."""
    return 2 * max(h_per_view) + 2


def extended(r0: int, r1: int, halo: int, H: int) -> Tuple[int, int]:
    return max(0, r0 - halo), min(H, r1 + halo)


def global_stats(dmin: float, dmax: float, nonfinite: int, device=None) -> Tuple[float, float, int]:
    """All-reduce of band statistics (identity without torch.distributed)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(dmin), float(dmax), int(nonfinite)
    t = torch.tensor([-float(dmin), float(dmax)], dtype=torch.float32, device=device)
    n = torch.tensor([int(nonfinite)], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(n, op=dist.ReduceOp.SUM)
    return -float(t[0]), float(t[1]), int(n[0])


def exchange_halos(band, r0: int, r1: int, halo: int, H: int, all_bands: List[Tuple[int, int]], rank: int):
    """Assemble rows [e0, e1) = extended(r0, r1, halo, H) from the owning ranks.

    band: this rank's rows [r0, r1) as a torch tensor [r1 - r0, W] (device or
    host).  Every rank calls this with the same halo and band table."""
    import torch
    import torch.distributed as dist
    e0, e1 = extended(r0, r1, halo, H)
    ext = torch.empty((e1 - e0,) + tuple(band.shape[1:]), dtype=band.dtype, device=band.device)
    ext[r0 - e0:r1 - e0] = band
    ops, bufs = [], []
    for q, (q0, q1) in enumerate(all_bands):
        if q == rank:
            continue
        # rows of q's band that this rank needs
        a, b = max(e0, q0), min(e1, q1)
        if a < b:
            buf = torch.empty((b - a,) + tuple(band.shape[1:]), dtype=band.dtype, device=band.device)
            ops.append(("recv", q, buf))
            bufs.append((a, b, buf))
        # rows of this band that q needs
        f0, f1 = extended(q0, q1, halo, H)
        a, b = max(f0, r0), min(f1, r1)
        if a < b:
            ops.append(("send", q, band[a - r0:b - r0].contiguous()))
    if ops:
        if band.is_cuda:
            p2p = [dist.P2POp(dist.isend if k == "send" else dist.irecv, t, q) for k, q, t in ops]
            for w in dist.batch_isend_irecv(p2p):
                w.wait()
        else:
            works = [dist.isend(t, q) if k == "send" else dist.irecv(t, q) for k, q, t in ops]
            for w in works:
                w.wait()
    for a, b, buf in bufs:
        ext[a - e0:b - e0] = buf
    return ext, e0, e1


def detect_band(band, r0: int, r1: int, H: int, views, rank: int, world: int,
                stats_fn: Callable, detect_fn: Callable, h_fn: Callable):
    """One rank's part of a sharded frame.

    stats_fn(band) -> (dmin, dmax, nonfinite) of the band;
    h_fn(dmin, dmax) -> Eq. 3's h per view under those statistics;
    detect_fn(ext, dmin, dmax, nonfinite) -> masks [V, e1 - e0, W] of the
    extended band under the imposed whole-frame statistics.
    Returns (interior masks [V, r1 - r0, W], (dmin, dmax, nonfinite))."""
    lo, hi, bad = stats_fn(band)
    dmin, dmax, nbad = global_stats(lo, hi, bad, device=band.device)
    all_bands = bands(H, world)
    assert all_bands[rank] == (r0, r1)
    halo = 0 if nbad else halo_rows(h_fn(dmin, dmax))
    ext, e0, e1 = exchange_halos(band, r0, r1, halo, H, all_bands, rank)
    m = detect_fn(ext, dmin, dmax, nbad)
    return m[:, r0 - e0:r1 - e0], (dmin, dmax, nbad)


def gather_rows(part, r0: int, r1: int, H: int, world: int, rank: int, dst: int = 0):
    """Collect the ranks' interior masks [V, r1 - r0, ...] into [V, H, ...] on dst
    (None elsewhere) by point-to-point transfers."""
    import torch
    import torch.distributed as dist
    all_bands = bands(H, world)
    if rank != dst:
        dist.send(part.contiguous(), dst)
        return None
    out = torch.empty((part.shape[0], H) + tuple(part.shape[2:]), dtype=part.dtype, device=part.device)
    out[:, r0:r1] = part
    for q, (q0, q1) in enumerate(all_bands):
        if q == dst:
            continue
        buf = torch.empty((part.shape[0], q1 - q0) + tuple(part.shape[2:]), dtype=part.dtype, device=part.device)
        dist.recv(buf, q)
        out[:, q0:q1] = buf
    return out


def device_fns(views, **detector_kw):
    """stats_fn / detect_fn / h_fn over libocc: occ_frame_stats on the band,
    occ_detect with occ_set_frame_stats on the extended band (a Detector per
    band shape, created on first use; detector_kw as for Detector) and
    occ_scan_half_lengths."""
    from .occ import Detector
    cache = {}

    def det_for(rows, W):
        if (rows, W) not in cache:
            cache[(rows, W)] = Detector(rows, W, views, **detector_kw)
        return cache[(rows, W)]

    def stats_fn(band):
        lo, hi, bad = det_for(*band.shape).frame_stats(band)
        return float(lo[0]), float(hi[0]), int(bad[0])

    def detect_fn(ext, dmin, dmax, nbad):
        det = det_for(*ext.shape)
        det.set_frame_stats([dmin], [dmax], [nbad])
        m = det.detect(ext)
        det.set_frame_stats()
        return m[0]

    def h_fn(dmin, dmax):
        return det_for(2, 2).scan_half_lengths(dmin, dmax)

    def close():
        for d in cache.values():
            d.close()
        cache.clear()
    return stats_fn, detect_fn, h_fn, close
