"""paper_2502_20969_b200 — B200-native lookahead IVF retrieval (TeleRAG, arXiv 2502.20969).

The product is liblaivg.so (CUDA kernels for sm_100a + C++ host runtime behind
the C ABI in include/laivg.h). ``laiv`` mirrors the reference `laiv` C++ API
over that ABI. Nothing here imports the test oracle under oracle/.
"""
from . import laiv  # noqa: F401
from ._lib import LIB_PATH, lib  # noqa: F401

__all__ = ["laiv", "lib", "LIB_PATH"]
