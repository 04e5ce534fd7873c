"""B200-native TRMC-R (recursive Time-Relaxed Monte Carlo, arXiv:1009.2768).

The hot path is CUDA (sm_100a) behind the C ABI in include/trmcr.h;
`paper_1009_2768_b200.api` is the thin Python binding and
`paper_1009_2768_b200.build` compiles the library.  Submodules are imported
explicitly so that `build` works on a machine without the built library.
"""
