"""B200-native Anderson-acceleration hot path of arXiv 2110.09667 (low-synchronisation
QR updates: MGS, ICWY-MGS, CGS-2, DCGS-2), behind the C ABI of include/aa.h.

``from paper_2110_09667_b200 import aa`` loads libaa.so (built in-tree by
``python -m paper_2110_09667_b200.build``); it raises if the library is missing.
"""
__all__ = ["aa", "build"]
