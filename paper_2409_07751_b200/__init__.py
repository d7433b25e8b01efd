"""B200-native RNS-CKKS engine for encrypted KAN inference (arXiv 2409.07751).

Drop-in for the reference package `hekan`'s encrypted path: the HeBackend
plugin contract (`backend`), the HE polynomial evaluator and comparator
(`approx`), the encrypted B-spline machinery (`bspline`) and the encrypted KAN
pipeline (`inference`), with every homomorphic op executed by hand-written
sm_100a kernels (libhekan_gpu.so, C ABI in include/hekan.h).
"""

__version__ = "0.1.0"
