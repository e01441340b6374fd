"""B200-native ParamSpMM hot path (arXiv 2605.15695).

The product is the C-ABI library libpspmm.so (include/pspmm.h) built from
csrc/ for sm_100a; `api` is its thin Python binding.  Importing `api` fails
loudly if the library is not built — there is no CPU or PyTorch fallback.
"""
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpspmm.so")
__all__ = ["LIB_PATH"]
