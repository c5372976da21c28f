"""B200-native eddy hot path of Hydro (arXiv 2403.14902): C-ABI library libhydro.so
(csrc/, include/hydro.h) and its thin ctypes binding (hydro.py)."""
from .hydro import (Eddy, EXPORTS, HydroError, hydro_version, lib)  # noqa: F401
