"""B200-native coherent-likelihood engine for Coherent Direct Multipath SLAM (arxiv 2604.19723).

The compute path is libcdms.so (hand-written CUDA for sm_100a behind the C ABI in include/cdms.h);
``paper_2604_19723_b200.cdms`` is the thin ctypes binding.  ``scenes`` draws the seeded synthetic
inputs.  Importing this package does not load the CUDA library.
"""
__all__ = ["scenes"]
