"""B200-native ASSE hot path (arXiv 1807.01527): sliding-window super-point
detection with asynchronous timestamps. The compute path is the C-ABI library
libasse.so (hand-written CUDA for sm_100a); `asse.py` is a thin ctypes binding.
"""
__all__ = ["asse", "dist"]
