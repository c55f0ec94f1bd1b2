"""B200-native projected star-Q product and truncated tSVDQ (arXiv 2409.19402).

The engine is libppc.so (CUDA, sm_100a) behind the C-ABI in include/ppc.h;
`projprod` mirrors the reference's Python module on top of it.
"""
from . import projprod
from .projprod import *  # noqa: F401,F403

__version__ = "0.1.0"
