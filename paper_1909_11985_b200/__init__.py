"""B200-native elastic data-parallel SGD hot path of EDL (arXiv 1909.11985).

Host mirror of the reference interfaces (proj/include/edl/*.hpp) over the C ABI in
include/edl_b200.h; the compute path is hand-written sm_100a CUDA in csrc/.
"""
__version__ = "0.1.0"
