"""Thin Python binding of libocc's C ABI (include/occ.h) -- marshalling only.

Every step of the detector runs in libocc's sm_100a CUDA kernels; this module
only passes pointers, sizes and the current torch CUDA stream.  There is no
CPU or PyTorch fallback: if ``libocc.so`` is missing or cannot be loaded the
import of :class:`Detector` fails loudly.
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
def _lib_path() -> str:
    """libocc.so, or an A/B build: OCC_LIB names a library, OCC_DEFINES (and
    OCC_LINE_STATS) select the instrumented build of build.lib_path()."""
    if os.environ.get("OCC_LIB"):
        return os.environ["OCC_LIB"]
    if os.environ.get("OCC_DEFINES") or os.environ.get("OCC_LINE_STATS"):
        from . import build
        return build.lib_path()
    return os.path.join(_HERE, "libocc.so")


LIB_PATH = _lib_path()

OCC_OK = 0
OCC_ERR_INVALID_ARG = -1
OCC_ERR_CUDA = -2
OCC_ERR_OOM = -3
OCC_ERR_NONFINITE = -4
OCC_ERR_UNSUPPORTED = -5
PATHS = {"auto": 0, "tiled": 1, "direct": 2}

# every function include/occ.h declares (checked against the header by tests)
EXPORTS = ["occ_default_params", "occ_create", "occ_detect", "occ_detect_host", "occ_status",
           "occ_frame_info", "occ_set_path", "occ_last_launches", "occ_destroy", "occ_strerror",
           "occ_version", "occ_profile", "occ_profile_read", "occ_fuse_median", "occ_set_mask_format",
           "occ_mask_bytes", "occ_set_neighbors", "occ_get_neighbors", "occ_frame_stats",
           "occ_set_frame_stats", "occ_create_dirs", "occ_scan_half_lengths"]
MASK_FORMATS = {"u8": 0, "bits": 1}
KERNEL_KINDS = {"init": 0, "stats": 1, "tile": 2, "direct": 3, "cand": 4, "line": 5, "nwin": 6, "hard": 7}


class occ_baseline(ctypes.Structure):
    _fields_ = [("bx", ctypes.c_int32), ("by", ctypes.c_int32)]


class occ_direction(ctypes.Structure):
    _fields_ = [("baseline_angle", ctypes.c_double), ("baseline_length", ctypes.c_double)]


class occ_params(ctypes.Structure):
    _fields_ = [("t_edge", ctypes.c_float), ("t_dist", ctypes.c_float),
                ("t_disp", ctypes.c_float), ("max_scan", ctypes.c_int32)]


class OccError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: {strerror(code)} ({code})")
        self.code = code


_lib: Optional[ctypes.CDLL] = None


def lib() -> ctypes.CDLL:
    """Load libocc.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libocc.so not found at {LIB_PATH}: run `python -c "
                               f"'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32 = ctypes.c_void_p, ctypes.c_int32
        L.occ_default_params.argtypes = [ctypes.POINTER(occ_params)]
        L.occ_default_params.restype = None
        L.occ_create.argtypes = [i32, i32, ctypes.POINTER(occ_baseline), i32,
                                 ctypes.POINTER(occ_params), i32, ctypes.POINTER(vp)]
        L.occ_create.restype = ctypes.c_int
        L.occ_detect.argtypes = [vp, vp, vp, i32, vp]
        L.occ_detect.restype = ctypes.c_int
        L.occ_detect_host.argtypes = [vp, vp, vp, i32, vp]
        L.occ_detect_host.restype = ctypes.c_int
        L.occ_status.argtypes = [vp, ctypes.POINTER(i32)]
        L.occ_status.restype = ctypes.c_int
        L.occ_frame_info.argtypes = [vp, i32, ctypes.POINTER(ctypes.c_float),
                                     ctypes.POINTER(ctypes.c_float), ctypes.POINTER(i32)]
        L.occ_frame_info.restype = ctypes.c_int
        L.occ_set_path.argtypes = [vp, i32]
        L.occ_set_path.restype = ctypes.c_int
        L.occ_last_launches.argtypes = [vp]
        L.occ_last_launches.restype = i32
        L.occ_destroy.argtypes = [vp]
        L.occ_destroy.restype = ctypes.c_int
        L.occ_strerror.argtypes = [ctypes.c_int]
        L.occ_strerror.restype = ctypes.c_char_p
        L.occ_profile.argtypes = [vp, i32]
        L.occ_profile.restype = ctypes.c_int
        L.occ_profile_read.argtypes = [vp, i32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i32)]
        L.occ_profile_read.restype = ctypes.c_int
        L.occ_version.argtypes = []
        L.occ_version.restype = i32
        L.occ_fuse_median.argtypes = [vp, i32, ctypes.c_int64, vp, vp]
        L.occ_fuse_median.restype = ctypes.c_int
        L.occ_set_mask_format.argtypes = [vp, i32]
        L.occ_set_mask_format.restype = ctypes.c_int
        L.occ_mask_bytes.argtypes = [vp, i32]
        L.occ_mask_bytes.restype = ctypes.c_int64
        L.occ_set_neighbors.argtypes = [vp, i32]
        L.occ_set_neighbors.restype = ctypes.c_int
        L.occ_get_neighbors.argtypes = [vp]
        L.occ_get_neighbors.restype = i32
        L.occ_create_dirs.argtypes = [i32, i32, vp, i32, vp, i32, vp]
        L.occ_create_dirs.restype = ctypes.c_int
        L.occ_frame_stats.argtypes = [vp, vp, i32, vp, vp, vp, vp]
        L.occ_frame_stats.restype = ctypes.c_int
        L.occ_set_frame_stats.argtypes = [vp, vp, vp, vp, i32]
        L.occ_set_frame_stats.restype = ctypes.c_int
        L.occ_scan_half_lengths.argtypes = [vp, ctypes.c_float, ctypes.c_float, vp]
        L.occ_scan_half_lengths.restype = ctypes.c_int
        _lib = L
    return _lib


def strerror(code: int) -> str:
    try:
        return lib().occ_strerror(code).decode()
    except Exception:  # pragma: no cover - message formatting only
        return str(code)


def default_params() -> occ_params:
    p = occ_params()
    lib().occ_default_params(ctypes.byref(p))
    return p


def create_raw(H: int, W: int, baselines: Sequence[Tuple[int, int]], params: Optional[occ_params],
               max_batch: int = 1) -> Tuple[int, Optional[int]]:
    """Call occ_create; returns (rc, handle or None).  Used by ABI tests."""
    arr = (occ_baseline * max(1, len(baselines)))(*[occ_baseline(int(a), int(b)) for a, b in baselines])
    h = ctypes.c_void_p()
    rc = lib().occ_create(int(H), int(W), arr if len(baselines) else None, len(baselines),
                          ctypes.byref(params) if params is not None else None, int(max_batch),
                          ctypes.byref(h))
    return rc, (h.value if rc == OCC_OK else None)


def create_dirs_raw(H: int, W: int, dirs, params: Optional[occ_params], max_batch: int = 1):
    """Call occ_create_dirs with [(baseline_angle, baseline_length), ...]."""
    arr = (occ_direction * max(1, len(dirs)))(*[occ_direction(float(a), float(r)) for a, r in dirs])
    h = ctypes.c_void_p()
    rc = lib().occ_create_dirs(int(H), int(W), ctypes.addressof(arr) if len(dirs) else None, len(dirs),
                               ctypes.addressof(params) if params is not None else None, int(max_batch),
                               ctypes.addressof(h))
    return rc, (h.value if rc == OCC_OK else None)


class Detector:
    """``Detector(H, W, baselines).detect(D)`` -> uint8 masks [B, V, H, W].

    D: torch.float32 CUDA tensor [B, H, W] (or [H, W]), contiguous.  The call
    is enqueued on the current torch CUDA stream and does not synchronise.
    """

    def __init__(self, H: int, W: int, baselines: Optional[Sequence[Tuple[int, int]]] = None, t_edge: float = 1.0,
                 t_dist: float = 2.0, t_disp: float = 0.5, max_scan: int = 4096, max_batch: int = 1,
                 path: str = "auto", mask_format: str = "u8", neighbors: int = 0,
                 directions: Optional[Sequence[Tuple[float, float]]] = None):
        """baselines: integer grid offsets (occ_create); or directions:
        [(baseline_angle_rad, baseline_length), ...] (occ_create_dirs, NEXT #2)."""
        self.H, self.W = int(H), int(W)
        self.max_batch = int(max_batch)
        p = occ_params(t_edge, t_dist, t_disp, max_scan)
        if (baselines is None) == (directions is None):
            raise ValueError("give exactly one of baselines / directions")
        if directions is not None:
            self.directions = [(float(a), float(r)) for a, r in directions]
            self.baselines = []
            self.V = len(self.directions)
            rc, h = create_dirs_raw(self.H, self.W, self.directions, p, self.max_batch)
            what = "occ_create_dirs"
        else:
            self.directions = None
            self.baselines: List[Tuple[int, int]] = [(int(a), int(b)) for a, b in baselines]
            self.V = len(self.baselines)
            rc, h = create_raw(self.H, self.W, self.baselines, p, self.max_batch)
            what = "occ_create"
        if rc != OCC_OK:
            raise OccError(rc, what)
        self._h = h
        self._last_batch = 0
        self.set_path(path)
        self.mask_format = mask_format
        rc = lib().occ_set_mask_format(self._h, MASK_FORMATS[mask_format])
        if rc != OCC_OK:
            raise OccError(rc, "occ_set_mask_format")
        self.Wb = (self.W + 31) // 32
        self.set_neighbors(neighbors)

    def scan_half_lengths(self, dmin: float, dmax: float) -> List[int]:
        """Eq. 3's h per view for the given frame statistics (occ_scan_half_lengths)."""
        h = np.zeros(self.V, np.int32)
        rc = lib().occ_scan_half_lengths(self._h, float(dmin), float(dmax), h.ctypes.data)
        if rc != OCC_OK:
            raise OccError(rc, "occ_scan_half_lengths")
        return [int(x) for x in h]

    def frame_stats(self, D, stream=None):
        """Exact per-frame (dmin, dmax, nonfinite) numpy arrays of device frames
        D [B, H, W] (occ_frame_stats; synchronises)."""
        import torch
        if D.dim() == 2:
            D = D.unsqueeze(0)
        assert D.is_cuda and D.dtype == torch.float32 and D.is_contiguous()
        B = D.shape[0]
        lo, hi = np.empty(B, np.float32), np.empty(B, np.float32)
        bad = np.empty(B, np.int32)
        s = stream if stream is not None else torch.cuda.current_stream(D.device).cuda_stream
        rc = lib().occ_frame_stats(self._h, D.data_ptr(), B, lo.ctypes.data, hi.ctypes.data, bad.ctypes.data, s)
        if rc != OCC_OK:
            raise OccError(rc, "occ_frame_stats")
        return lo, hi, bad

    def set_frame_stats(self, dmin=None, dmax=None, nonfinite=None) -> None:
        """Impose whole-frame statistics on subsequent calls (occ_set_frame_stats);
        no arguments: back to the data's own statistics."""
        if dmin is None:
            rc = lib().occ_set_frame_stats(self._h, None, None, None, 0)
        else:
            lo = np.ascontiguousarray(dmin, np.float32).ravel()
            hi = np.ascontiguousarray(dmax, np.float32).ravel()
            bad = np.ascontiguousarray(nonfinite if nonfinite is not None else np.zeros(len(lo)), np.int32).ravel()
            rc = lib().occ_set_frame_stats(self._h, lo.ctypes.data, hi.ctypes.data, bad.ctypes.data, len(lo))
        if rc != OCC_OK:
            raise OccError(rc, "occ_set_frame_stats")

    def set_neighbors(self, N: int) -> None:
        """Eq. 5's neighbour count N (0 = infinity; see occ_set_neighbors)."""
        rc = lib().occ_set_neighbors(self._h, int(N))
        if rc != OCC_OK:
            raise OccError(rc, "occ_set_neighbors")
        self.neighbors = int(N)

    def set_path(self, path: str) -> None:
        rc = lib().occ_set_path(self._h, PATHS[path])
        if rc != OCC_OK:
            raise OccError(rc, "occ_set_path")

    def detect(self, D, out=None, stream=None):
        import torch
        if D.dim() == 2:
            D = D.unsqueeze(0)
        if D.dtype != torch.float32 or not D.is_cuda or not D.is_contiguous():
            raise ValueError("D must be a contiguous float32 CUDA tensor [B, H, W]")
        B = D.shape[0]
        if tuple(D.shape[1:]) != (self.H, self.W):
            raise ValueError(f"expected [B, {self.H}, {self.W}], got {tuple(D.shape)}")
        if out is None:
            out = torch.empty(self.mask_shape(B), dtype=self.mask_dtype(torch), device=D.device)
        elif (out.dtype != self.mask_dtype(torch) or not out.is_contiguous()
              or out.numel() * out.element_size() < lib().occ_mask_bytes(self._h, B)):
            raise ValueError(f"out must be a contiguous {self.mask_dtype(torch)} CUDA tensor {self.mask_shape(B)}")
        s = stream if stream is not None else torch.cuda.current_stream(D.device)
        rc = lib().occ_detect(self._h, D.data_ptr(), out.data_ptr(), B, s.cuda_stream)
        if rc != OCC_OK:
            raise OccError(rc, "occ_detect")
        self._last_batch = B
        return out

    def detect_host(self, D: np.ndarray, out: Optional[np.ndarray] = None, stream=None) -> np.ndarray:
        """Host buffers in, host masks out; copies and synchronisation inside."""
        D = np.ascontiguousarray(D, dtype=np.float32)
        if D.ndim == 2:
            D = D[None]
        if D.ndim != 3 or tuple(D.shape[1:]) != (self.H, self.W):
            raise ValueError(f"expected D [B, {self.H}, {self.W}], got {tuple(D.shape)}")
        B = D.shape[0]
        mdt = np.uint8 if self.mask_format == "u8" else np.uint32
        if out is None:
            out = np.empty(self.mask_shape(B), dtype=mdt)
        elif (out.dtype != mdt or not out.flags["C_CONTIGUOUS"] or not out.flags["WRITEABLE"]
              or out.nbytes < lib().occ_mask_bytes(self._h, B)):
            raise ValueError(f"out must be a writeable C-contiguous {np.dtype(mdt).name} array {self.mask_shape(B)}")
        sp = 0
        if stream is not None:
            sp = stream.cuda_stream
        else:
            try:
                import torch
                sp = torch.cuda.current_stream().cuda_stream
            except Exception:
                sp = 0
        rc = lib().occ_detect_host(self._h, D.ctypes.data, out.ctypes.data, B, sp)
        if rc != OCC_OK:
            raise OccError(rc, "occ_detect_host")
        self._last_batch = B
        return out

    def mask_shape(self, B: int):
        """[B, V, H, W] for uint8 masks, [B, V, H, ceil(W/32)] words for bit-packed ones."""
        return (B, self.V, self.H, self.W if self.mask_format == "u8" else self.Wb)

    def mask_dtype(self, torch):
        return torch.uint8 if self.mask_format == "u8" else torch.int32

    def detect_host_ptr(self, d_ptr: int, m_ptr: int, batch: int, stream_ptr: int = 0) -> None:
        rc = lib().occ_detect_host(self._h, d_ptr, m_ptr, batch, stream_ptr)
        if rc != OCC_OK:
            raise OccError(rc, "occ_detect_host")
        self._last_batch = batch

    def status(self) -> List[int]:
        st = (ctypes.c_int32 * max(1, self._last_batch))()
        rc = lib().occ_status(self._h, st)
        if rc != OCC_OK:
            raise OccError(rc, "occ_status")
        return list(st)[: self._last_batch]

    def frame_info(self, frame: int = 0):
        lo, hi = ctypes.c_float(), ctypes.c_float()
        hv = (ctypes.c_int32 * self.V)()
        rc = lib().occ_frame_info(self._h, frame, ctypes.byref(lo), ctypes.byref(hi), hv)
        if rc != OCC_OK:
            raise OccError(rc, "occ_frame_info")
        return lo.value, hi.value, list(hv)

    def profile(self, enable: bool) -> None:
        rc = lib().occ_profile(self._h, 1 if enable else 0)
        if rc != OCC_OK:
            raise OccError(rc, "occ_profile")

    def profile_read(self) -> dict:
        """{kind: (total_ms, launches)} since the last occ_profile call (syncs)."""
        out = {}
        for name, k in KERNEL_KINDS.items():
            ms, n = ctypes.c_double(), ctypes.c_int32()
            rc = lib().occ_profile_read(self._h, k, ctypes.byref(ms), ctypes.byref(n))
            if rc != OCC_OK:
                raise OccError(rc, "occ_profile_read")
            out[name] = (ms.value, n.value)
        return out

    @property
    def last_launches(self) -> int:
        return int(lib().occ_last_launches(self._h))

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().occ_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fuse_median(stack, out=None, stream=None):
    """Pixel-wise median of K disparity estimates (occ_fuse_median).

    stack: contiguous fp32 CUDA tensor [K, ...]; returns fp32 [...] (or fills
    ``out``).  Marshalling only: the median runs in libocc's k_fuse kernel."""
    import torch
    if not (stack.is_cuda and stack.dtype == torch.float32 and stack.is_contiguous()):
        raise ValueError("stack must be a contiguous float32 CUDA tensor [K, ...]")
    K = int(stack.shape[0])
    n = stack.numel() // max(1, K)
    if out is None:
        out = torch.empty(stack.shape[1:], dtype=torch.float32, device=stack.device)
    elif not (out.is_cuda and out.dtype == torch.float32 and out.is_contiguous() and out.numel() >= n
              and out.device == stack.device):
        raise ValueError(f"out must be a contiguous float32 CUDA tensor of {n} elements on {stack.device}")
    s = stream or torch.cuda.current_stream(stack.device)
    rc = lib().occ_fuse_median(stack.data_ptr(), K, n, out.data_ptr(), s.cuda_stream)
    if rc != OCC_OK:
        raise OccError(rc, "occ_fuse_median")
    return out


def unpack_masks(words: np.ndarray, W: int) -> np.ndarray:
    """Bit-packed masks (OCC_MASK_BITS: [..., H, ceil(W/32)] 32-bit words, bit
    x & 31 of word x >> 5) -> uint8 0/1 masks [..., H, W] (host-side view helper)."""
    w = np.ascontiguousarray(words).view(np.uint32)
    b = np.unpackbits(w.view(np.uint8), axis=-1, bitorder="little")
    return b[..., :W]
