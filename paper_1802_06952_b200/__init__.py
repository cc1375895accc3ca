"""B200-native hot path of the partitioned simulator of arXiv:1802.06952.

The product is the C-ABI library ``libqsim.so`` (CUDA kernels for sm_100a + host
executor, declared in ``include/qsim.h``); ``qsim`` is its thin ctypes binding.
"""
from .qsim import *  # noqa: F401,F403
from .qsim import Simulator, QsimError, EXPORTED, LIB_PATH  # noqa: F401
