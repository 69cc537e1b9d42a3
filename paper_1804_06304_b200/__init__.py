"""paper_1804_06304_b200 — B200-native (sm_100a) hot path of arXiv 1804.06304:
batched Monte-Carlo evolution of 3D snakuscules ("Three-Dimensional
GPU-Accelerated Active Contours for Automated Localization of Cells in Large
Images") plus resampling, Q14 blur, gradient magnitude, seeds, culling and
the label map, behind the C ABI in include/snk.h (libsnk.so).

Importing ``paper_1804_06304_b200.snk`` loads libsnk.so and raises if it is
missing: there is no CPU fallback.
"""
__all__ = ["snk", "pipeline", "dist"]
