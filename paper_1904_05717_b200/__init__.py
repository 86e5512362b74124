"""B200-native MOMMS GEMM (arXiv 1904.05717): multilevel-blocked C += A·B with
the reference toolkit's algorithm-composition surface, executed by
hand-written sm_100a kernels through the C ABI in include/tilemul_b200.h.

`paper_1904_05717_b200.tilemul` mirrors the reference's interface for the
execution path; the native library is required (no fallback).
"""
from . import tilemul  # noqa: F401
from ._native import LIB_PATH, lib  # noqa: F401

__all__ = ["tilemul", "lib", "LIB_PATH"]
