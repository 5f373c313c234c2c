"""B200-native (sm_100a) real-time NOMA detector -- the hot path of
arxiv 2206.05998 ("noma-detect"): LLS initialiser, fused online training of
the hybrid linear + ReLU-MLP network with IQ-symmetry augmentation, and
streaming detection with fused hard decisions and BER counters.

Layers: include/noma_cuda.h (C-ABI) <- csrc/*.cu (sm_100a kernels) ;
native.py (ctypes plumbing) ; api.py (reference-named Python mirror) ;
host/ (C++ noma:: API over the C-ABI).
"""
from .native import LIB_PATH, load  # noqa: F401

__all__ = ["LIB_PATH", "load"]
