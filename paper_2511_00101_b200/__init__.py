"""B200-native Segmented Multi-LoRA Multiplication (SMLM), after Loquetier (arXiv 2511.00101).

The product is `libsmlm.so` (C ABI in include/smlm.h, CUDA kernels for sm_100a in csrc/).
`paper_2511_00101_b200.smlm` is its thin Python binding; it raises ImportError if the library is
not built (there is no CPU fallback).  Attribute access on this package loads the binding lazily
so that `python -m paper_2511_00101_b200.build` works before the library exists.
"""
import importlib

_SUBMODULES = ("build", "smlm", "dp")


def __getattr__(name):
    if name in _SUBMODULES:
        return importlib.import_module("." + name, __name__)
    if name.startswith("__"):
        raise AttributeError(name)
    mod = importlib.import_module(".smlm", __name__)
    return getattr(mod, name)
