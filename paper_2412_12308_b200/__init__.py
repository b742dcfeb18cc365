"""fftpde: B200-native 2D FFT-PDE hot path (arXiv 2412.12308).

The compute path is the C-ABI library ``libfftpde.so`` (hand-written sm_100a
CUDA kernels); ``paper_2412_12308_b200.fftpde`` is the thin ctypes binding.
Importing this package does not load the library; ``fftpde`` does, and fails
loudly if it is missing.  ``inputs`` holds the seeded synthetic generators.
"""
__all__ = ["fftpde", "inputs"]
