"""B200-native FlashRNN engine (arXiv 2412.07752), Python plumbing.

The product is ``libflashrnn.so`` (C ABI in ``include/flashrnn.h``; C++ drop-in
shim in ``include/flashrnn/engine.hpp``).  This package only loads it through
ctypes and hands it device buffers (torch tensors) -- it contains no compute.
If the library or an sm_100 GPU is missing, calls fail loudly; there is no CPU
fallback.
"""
from .abi import (ALGO, CLIP, DTYPE, PASS, VARIANTS, FlashRNN, FrnnError, cell_spec, lib_path,
                  load)

__all__ = ["ALGO", "CLIP", "DTYPE", "PASS", "VARIANTS", "FlashRNN", "FrnnError", "cell_spec",
           "lib_path", "load"]
