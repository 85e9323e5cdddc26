"""B200-native hot path of SeCO / SpaCO (arXiv 2505.16710): chunked causal GQA
attention forward + chunk-local backward with in-place checkpoint-gradient
accumulation, on sm_100a tensor cores (tcgen05 / TMEM / TMA), behind the C ABI
of include/seco.h (libseco.so).  See DESIGN.md."""
from . import flops  # noqa: F401

__all__ = ["ops", "step", "flops"]


def __getattr__(name):
    # lazy: importing the package does not require torch or the built library
    if name in ("ops", "step"):
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
