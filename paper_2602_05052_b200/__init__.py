"""B200-native P1 Galerkin assembly engine (TensorGalerkin hot path, arXiv 2602.05052).

Layers
  include/tgk.h          C ABI (the drop-in boundary), implemented by lib/libtgk.so
  _native                ctypes binding of that ABI
  engine                 device-resident API (torch tensors as buffers)
  tgfem                  drop-in for the reference's Python module (NumPy in/out)
"""
from ._native import CudaError, InputError, NumericalError  # noqa: F401

__version__ = "0.1.0"
