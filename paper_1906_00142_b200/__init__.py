"""B200-native rational-program evaluator (arXiv 1906.00142 / KLARAPTOR).

Host-side mirror of the reference ``ratprog`` hot path over the C ABI of
``librpgpu.so`` (include/rpg.h): batched MWP-CWP evaluation of every
(data tuple, block configuration) point and the per-tuple argmin, on sm_100a.
"""
__version__ = "0.1.0"
