"""B200-native explicit time step of the grand-potential phase-field model
(Bauer et al., arXiv 1506.01684).  The product is libpf.so (CUDA, sm_100a)
behind the C ABI of include/pf.h; ``pf`` is its thin ctypes binding."""
from . import pf  # noqa: F401
