"""B200-native quadratic-neuron layers (QuadraLib hot path, arXiv 2204.01701).

Drop-in for the reference's quadratic-layer API (``quadra.neurons``), backed
by hand-written sm_100a kernels in ``libquadra_b200.so``.
"""

from . import errors, spec
from .spec import QuadraticLayerSpec

__version__ = "0.1.0"

__all__ = ["errors", "spec", "QuadraticLayerSpec", "neurons", "nn"]


def __getattr__(name):  # lazy: importing torch-backed modules only when used
    if name in ("neurons", "nn", "train"):
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
