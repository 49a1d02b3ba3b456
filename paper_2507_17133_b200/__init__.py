"""B200-native brownout MoE-layer forward (BrownoutServe, arXiv 2507.17133).

The compute path is libbrownout.so (hand-written sm_100a CUDA behind the C ABI
of include/brownout.h); ``paper_2507_17133_b200.brownout`` is its thin ctypes
binding.  The binding is loaded lazily so that ``paper_2507_17133_b200.build``
can (re)build the library first; loading it fails loudly if it is missing.
"""
import importlib

__all__ = ["BrownoutMoE", "BrownoutError", "UnitedDistiller", "LIB_PATH", "lib", "STATS_FIELDS"]


def __getattr__(name):
    if name.startswith("__") or name in ("brownout", "build"):
        raise AttributeError(name)
    mod = importlib.import_module(__name__ + ".brownout")
    return getattr(mod, name)
