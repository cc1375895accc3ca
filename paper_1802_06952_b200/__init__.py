"""B200-native hot path of the partitioned simulator of arXiv:1802.06952.

The product is the C-ABI library ``libqsim.so`` (CUDA kernels for sm_100a + host
executor, declared in ``include/qsim.h``); ``qsim`` is its thin ctypes binding.
The binding is loaded on first use (``from paper_1802_06952_b200 import qsim``) so that
``python -m paper_1802_06952_b200.build`` works before the library exists; using it
without a built library raises ImportError (there is no CPU fallback).
"""
import importlib


def __getattr__(name):
    if name in ("qsim", "build"):
        return importlib.import_module("." + name, __name__)
    if name.startswith("__"):
        raise AttributeError(name)
    mod = importlib.import_module(".qsim", __name__)
    if hasattr(mod, name):
        return getattr(mod, name)
    raise AttributeError(name)
