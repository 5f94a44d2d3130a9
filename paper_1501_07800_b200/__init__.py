"""B200-native block-sparse quadtree matrix multiply (arXiv 1501.07800 hot path).

The product is ``libqtmm.so`` (C ABI in ``include/qt.h``, CUDA sources in
``csrc/``); ``qtmm`` is its thin ctypes binding.  Importing ``qtmm`` fails if
the library is not built: there is no CPU fallback.
"""
