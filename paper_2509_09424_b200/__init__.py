"""B200-native (sm_100a) engine for ENSI's ternary PCMM hot path (arXiv 2509.09424, Algorithm 1).

The CUDA kernels and the C ABI live in csrc/ and are built into libensi.so (see build.py);
``ensi`` is the ctypes binding.  The multi-GPU driver is ``dist``.
"""
from .ensi import Context, Weights, EnsiError, galois_elt, lib  # noqa: F401
