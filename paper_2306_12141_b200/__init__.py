"""B200-native Recoil (arXiv 2306.12141): parallel decoding of one interleaved rANS
bitstream from split points.  The product is ``librecoil.so`` (C ABI in
``include/recoil.h``: host C++ encoder/metadata + sm_100a CUDA decode kernels);
``paper_2306_12141_b200.recoil`` is its thin ctypes binding (same names)."""
from .recoil import *  # noqa: F401,F403
