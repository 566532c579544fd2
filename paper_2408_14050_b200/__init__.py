"""B200-native fast edge-aware occlusion detection (arXiv 2408.14050).

``Detector`` (paper_2408_14050_b200.occ) wraps the C ABI of libocc
(include/occ.h); every step runs in libocc's sm_100a CUDA kernels.
``scenes`` holds the seeded synthetic inputs shared by tests and bench.
"""

__all__ = ["Detector", "scenes"]


def __getattr__(name):
    if name == "Detector":
        from .occ import Detector
        return Detector
    raise AttributeError(name)
