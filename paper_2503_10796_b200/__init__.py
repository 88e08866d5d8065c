"""B200-native (sm_100a) mechanics hot path of BioDynaMo/TeraAgent (arXiv 2503.10796).

The product is libbdm.so (C ABI, include/bdm.h); ``bdm`` is its thin ctypes binding.
"""
from .bdm import (Agents, BdmError, CGrid3, COncoParams, Engine, Params, load_library, EXPORTS,  # noqa: F401
                  FLAG_ADDED, FLAG_GREW, FLAG_MOVED, FLAG_STATIC, NNZ_SHIFT, tile_curve)

__version__ = "0.1.0"
