"""B200-native numeric phase of the Crout-type block ILU (arXiv:1908.10169).

The product path is libbilu.so (csrc/, include/bilu.h) driven through the thin
ctypes binding in bilu.py.  Importing this package never falls back to a CPU
implementation: a missing library raises at first use.
"""
from .bilu import BILU, BiluError, Factor, default_options, load_library, ABI_SYMBOLS, ilu1_blocks, cosine_blocks, mwm  # noqa: F401

__all__ = ["BILU", "BiluError", "Factor", "default_options", "load_library", "ABI_SYMBOLS", "ilu1_blocks", "cosine_blocks", "mwm"]
