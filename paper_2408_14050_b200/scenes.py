"""Seeded synthetic disparity scenes for the five BASELINE.json configs.

This module is INPUT INFRASTRUCTURE shared by the oracle tests, the GPU
parity tests and ``bench.py``.  It contains none of the method's arithmetic
(no edges, candidates, scan lines, warps or occlusion tests) -- only the
recipe that paints layered disparity maps, stated in DESIGN.md §3
("Input recipe") and SURVEY.md §8(d) "Synthetic inputs".

PRNG: SplitMix64 (Steele, Lea, Flood 2014), counter based, so every draw is
addressed by (stream, index) and the maps are bit-identical on every host.
Geometry is evaluated in fp64; each pixel is rounded to fp32 exactly once.

The paper's datasets (SceneFlow, the hyperspectral video DB, CAMSI;
PAPER.md §4) are not available; these scenes stand in for them with the
shapes, disparity ranges, layering and noise BASELINE.json names.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Sequence, Tuple

import numpy as np

_GOLD = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix(z: np.ndarray) -> np.ndarray:
    """SplitMix64 output function (vectorised, wrapping uint64 arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


class SplitMix64:
    """Counter-based SplitMix64 stream: draw i = mix(key + (i+1)*golden)."""

    def __init__(self, *key: int):
        k = np.uint64(0x6A09E667F3BCC909)
        for part in key:
            with np.errstate(over="ignore"):
                k = _mix(np.uint64(k) ^ np.uint64(int(part) & 0xFFFFFFFFFFFFFFFF))
        self.key = np.uint64(k)
        self.n = 0

    def raw(self, count: int) -> np.ndarray:
        idx = np.arange(self.n + 1, self.n + 1 + count, dtype=np.uint64)
        self.n += count
        with np.errstate(over="ignore"):
            return _mix(self.key + idx * _GOLD)

    def uniform(self, count: int = 1) -> np.ndarray:
        """Uniform doubles in [0, 1) with 53 random bits."""
        return (self.raw(count) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)

    def uniform_range(self, lo: float, hi: float) -> float:
        return float(lo + (hi - lo) * self.uniform(1)[0])

    def randint(self, lo: int, hi: int) -> int:
        """Integer uniform in [lo, hi] (inclusive)."""
        return int(lo + math.floor(self.uniform(1)[0] * (hi - lo + 1)))

    def normal(self, count: int) -> np.ndarray:
        """Standard normals via Box-Muller, two per uniform pair."""
        m = (count + 1) // 2
        u = self.uniform(2 * m).reshape(m, 2)
        r = np.sqrt(-2.0 * np.log1p(-u[:, 0]))  # 1-u in (0, 1]
        th = 2.0 * math.pi * u[:, 1]
        out = np.empty(2 * m, dtype=np.float64)
        out[0::2] = r * np.cos(th)
        out[1::2] = r * np.sin(th)
        return out[:count]


# --------------------------------------------------------------------------
# Config table (BASELINE.json "configs")
# --------------------------------------------------------------------------

VIEWS_3X3: List[Tuple[int, int]] = [(1, 0), (-1, 0), (0, 1), (0, -1),
                                    (1, 1), (-1, -1), (1, -1), (-1, 1)]
VIEWS_5X5: List[Tuple[int, int]] = [(bx, by) for by in range(-2, 3) for bx in range(-2, 3)
                                    if (bx, by) != (0, 0)]


@dataclass(frozen=True)
class SceneConfig:
    name: str
    H: int
    W: int
    views: Tuple[Tuple[int, int], ...]
    n_shapes: int
    half_lo: float
    half_hi: float
    disp_lo: float
    disp_hi: float
    kinds: int          # 1: rect only, 2: rect/ellipse, 3: rect/ellipse/slanted patch
    noise_sigma: float
    frames: int = 1


CONFIGS = {
    1: SceneConfig("C1", 48, 64, ((1, 0),), 1, 0, 0, 8.0, 8.0, 1, 0.0),
    2: SceneConfig("C2", 480, 640, tuple(VIEWS_3X3), 20, 8.0, 64.0, 4.0, 32.0, 2, 0.0),
    3: SceneConfig("C3", 1080, 1920, tuple(VIEWS_3X3), 50, 16.0, 192.0, 1.0, 64.0, 3, 0.25),
    4: SceneConfig("C4", 3072, 4096, tuple(VIEWS_5X5), 200, 32.0, 384.0, 1.0, 48.0, 3, 0.0),
    5: SceneConfig("C5", 1080, 1920, tuple(VIEWS_3X3), 50, 16.0, 192.0, 1.0, 64.0, 3, 0.25, 256),
}


def config_views(cfg: int) -> List[Tuple[int, int]]:
    return list(CONFIGS[cfg].views)


def _background(H: int, W: int) -> np.ndarray:
    """Slanted ground plane d = 1 + 3*y/(H-1)."""
    y = np.arange(H, dtype=np.float64)[:, None]
    return np.broadcast_to(1.0 + 3.0 * y / (H - 1), (H, W)).copy()


def _paint_layers(img: np.ndarray, rng: SplitMix64, c: SceneConfig) -> None:
    H, W = img.shape
    shapes = []
    for i in range(c.n_shapes):
        # fixed draw order per shape: kind, cx, cy, ax, ay, disparity, gx, gy
        u_kind, ucx, ucy, uax, uay, ud, ugx, ugy = rng.uniform(8)
        kind = min(int(u_kind * c.kinds), c.kinds - 1)
        cx = ucx * (W - 1)
        cy = ucy * (H - 1)
        ax = c.half_lo + (c.half_hi - c.half_lo) * uax
        ay = c.half_lo + (c.half_hi - c.half_lo) * uay
        d0 = c.disp_lo + (c.disp_hi - c.disp_lo) * ud
        gx = -0.1 + 0.2 * ugx
        gy = -0.1 + 0.2 * ugy
        shapes.append((d0, i, kind, cx, cy, ax, ay, gx, gy))
    # painter's order: far (small disparity) first, nearer shapes overwrite
    shapes.sort(key=lambda s: (s[0], s[1]))
    for d0, _, kind, cx, cy, ax, ay, gx, gy in shapes:
        x0 = max(0, int(math.floor(cx - ax)))
        x1 = min(W - 1, int(math.ceil(cx + ax)))
        y0 = max(0, int(math.floor(cy - ay)))
        y1 = min(H - 1, int(math.ceil(cy + ay)))
        if x0 > x1 or y0 > y1:
            continue
        xs = np.arange(x0, x1 + 1, dtype=np.float64)[None, :]
        ys = np.arange(y0, y1 + 1, dtype=np.float64)[:, None]
        if kind == 1:   # ellipse, inside test at pixel centres
            inside = ((xs - cx) / ax) ** 2 + ((ys - cy) / ay) ** 2 <= 1.0
        else:           # rectangle footprint (also for slanted patches)
            inside = (np.abs(xs - cx) <= ax) & (np.abs(ys - cy) <= ay)
        if kind == 2:   # slanted planar patch, clamped to the disparity range
            val = np.clip(d0 + gx * (xs - cx) + gy * (ys - cy), c.disp_lo, c.disp_hi)
            val = np.broadcast_to(val, inside.shape)
        else:
            val = np.full(inside.shape, d0)
        sub = img[y0:y1 + 1, x0:x1 + 1]
        sub[inside] = val[inside]


def make_scene(cfg: int, seed: int = 0, frame: int = 0) -> np.ndarray:
    """One fp32 [H, W] disparity map of config ``cfg`` (1..5)."""
    c = CONFIGS[cfg]
    if cfg == 1:
        rng = SplitMix64(1, seed, frame)
        x0 = rng.randint(7, 44)
        y0 = rng.randint(0, 32)
        img = np.full((c.H, c.W), 2.0, dtype=np.float64)
        img[y0:y0 + 16, x0:x0 + 20] = 8.0
        return img.astype(np.float32)
    return make_scene_scaled(cfg, 1.0, seed, frame)


def make_scene_scaled(cfg: int, scale: float, seed: int = 0, frame: int = 0) -> np.ndarray:
    """The config-``cfg`` scene (2..5) with the layered, noise-free disparities
    mapped d -> 1 + scale*(d - 1) BEFORE the config's estimation noise is added
    (the noise stays sigma pixels: a stereo matcher's error does not grow with
    the disparity).  scale = 1 is make_scene bit for bit (d - 1 + 1 is exact).
    bench.py's h sweep uses it to set Eq. 3's h (about 66*scale for C3)."""
    c = CONFIGS[cfg]
    base = 3 if cfg == 5 else cfg       # C5 frames are C3 scenes from seed+frame
    rng = SplitMix64(base, seed + frame)
    img = _background(c.H, c.W)
    _paint_layers(img, rng, c)
    if scale != 1.0:
        img = 1.0 + float(scale) * (img - 1.0)
    if c.noise_sigma > 0:
        noise = SplitMix64(base, seed + frame, 0x4E4F495345).normal(c.H * c.W)
        img = img + c.noise_sigma * noise.reshape(c.H, c.W)
    return img.astype(np.float32)


def scale_disparity(D: np.ndarray, scale: float) -> np.ndarray:
    """The same layered scene with every disparity mapped d -> 1 + scale*(d - 1)
    (fp64, one fp32 rounding).  Scaling the C3 recipe sets the frame's
    disparity range, and with it Eq. 3's scan half-length h (about 66*scale
    for C3 frames); bench.py's h sweep and the GPU h tests use it."""
    return (1.0 + float(scale) * (np.asarray(D, dtype=np.float64) - 1.0)).astype(np.float32)


def c1_rect_origin(seed: int = 0, frame: int = 0) -> Tuple[int, int]:
    rng = SplitMix64(1, seed, frame)
    x0 = rng.randint(7, 44)
    y0 = rng.randint(0, 32)
    return x0, y0


def make_batch(cfg: int, frames: int, seed: int = 0, first_frame: int = 0) -> np.ndarray:
    """[frames, H, W] fp32; frame f is generated from seed + (first_frame + f)."""
    maps = [make_scene(cfg, seed, first_frame + f) for f in range(frames)]
    return np.stack(maps, axis=0)


# --------------------------------------------------------------------------
# Small structured maps for tests (SPEC.md:60-68 synth_scene)
# --------------------------------------------------------------------------

def step_scene(H: int, W: int, bg: float, fg: float, col: int, axis: int = 0,
               fg_first: bool = True) -> np.ndarray:
    """Vertical (axis=0) or horizontal (axis=1) step; fg on the low-index side
    when ``fg_first`` (D=fg for x<col, bg for x>=col)."""
    img = np.full((H, W), bg, dtype=np.float64)
    if axis == 0:
        if fg_first:
            img[:, :col] = fg
        else:
            img[:, col:] = fg
    else:
        if fg_first:
            img[:col, :] = fg
        else:
            img[col:, :] = fg
    return img.astype(np.float32)


def square_scene(H: int, W: int, bg: float, fg: float, rect: Tuple[int, int, int, int]) -> np.ndarray:
    """Constant fg inside rect=(x0, y0, x1, y1) (exclusive ends), bg outside."""
    x0, y0, x1, y1 = rect
    img = np.full((H, W), bg, dtype=np.float64)
    img[y0:y1, x0:x1] = fg
    return img.astype(np.float32)


def random_tiny_map(rng: SplitMix64, H: int, W: int, mode: str) -> np.ndarray:
    """Tiny random maps for brute-force and parity sweeps.

    mode: 'int'    -- piecewise-constant even integers (all jumps >= 2)
          'half'   -- half-integer rectangles on an integer background
          'noisy'  -- layered rectangles plus N(0, 0.25^2) fp32 noise
          'uniform'-- i.i.d. uniform values in [0, 8)
    """
    img = np.zeros((H, W), dtype=np.float64)
    if mode == "uniform":
        return (8.0 * rng.uniform(H * W).reshape(H, W)).astype(np.float32)
    nrect = rng.randint(1, 4)
    base = 2.0 * rng.randint(0, 2)
    img[:] = base
    for _ in range(nrect):
        x0 = rng.randint(0, W - 1)
        y0 = rng.randint(0, H - 1)
        x1 = rng.randint(x0 + 1, W)
        y1 = rng.randint(y0 + 1, H)
        if mode == "int":
            v = 2.0 * rng.randint(0, 5)
        elif mode == "half":
            v = 0.5 * rng.randint(0, 16)
        else:
            v = rng.uniform_range(0.0, 8.0)
        img[y0:y1, x0:x1] = v
    if mode == "noisy":
        img = img + 0.25 * rng.normal(H * W).reshape(H, W)
    return img.astype(np.float32)


def all_small_baselines(maxc: int = 2) -> List[Tuple[int, int]]:
    return [(bx, by) for by in range(-maxc, maxc + 1) for bx in range(-maxc, maxc + 1)
            if (bx, by) != (0, 0)]


def describe(cfg: int) -> str:
    c = CONFIGS[cfg]
    return f"{c.name}: {c.W}x{c.H}, {len(c.views)} views, {c.frames} frame(s)"


__all__: Sequence[str] = [
    "SplitMix64", "CONFIGS", "SceneConfig", "config_views", "make_scene", "make_batch",
    "c1_rect_origin", "step_scene", "square_scene", "random_tiny_map", "all_small_baselines",
    "VIEWS_3X3", "VIEWS_5X5", "describe",
]
