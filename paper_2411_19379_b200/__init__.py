"""B200-native (sm_100a) α-grid trace replay of Marconi's hybrid prefix cache (arXiv 2411.19379).

Product path: libmarconi.so (paper_2411_19379_b200/csrc, C ABI in include/marconi.h)
driven through the ctypes binding in `marconi` and the α-grid driver in `grid`.
PyTorch supplies device memory, streams and the NCCL process group only.
"""
from . import marconi  # noqa: F401
from .marconi import Context, MarconiError  # noqa: F401
from .grid import AlphaGrid, LiveTuner, lpt_shard, select_alpha  # noqa: F401
