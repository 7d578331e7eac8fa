"""TEST INFRASTRUCTURE ONLY — the reference library with the GPU drop-in.

oracle/_ref/libtgref_gpu.so (oracle/Makefile `refgpu`) is the unmodified
reference library whose tg::assemble is replaced by adapter/physics_gpu.cpp
(physics.cpp's own symbol renamed to tg::assemble_cpu).  This module is
oracle/ref.py loaded a second time against that library, so tests can drive
the reference's own C++ API — ProblemSpec, Mesh, DofMap, RoutingMatrices,
CoefficientField (Analytic included) — through the GPU drop-in and compare
with the CPU library side by side.
"""
import importlib.util
import os
import sys

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libtgref_gpu.so")

_spec = importlib.util.spec_from_file_location("oracle._ref_gpu_impl", os.path.join(_HERE, "ref.py"))
_mod = importlib.util.module_from_spec(_spec)
_mod.__package__ = "oracle"
_old = os.environ.get("_TGREF_LIB_OVERRIDE")
os.environ["_TGREF_LIB_OVERRIDE"] = LIB_PATH
try:
    _spec.loader.exec_module(_mod)
finally:
    if _old is None:
        os.environ.pop("_TGREF_LIB_OVERRIDE", None)
    else:
        os.environ["_TGREF_LIB_OVERRIDE"] = _old
sys.modules["oracle._ref_gpu_impl"] = _mod
globals().update({k: v for k, v in vars(_mod).items() if not k.startswith("__")})
LIB_PATH = _mod.LIB_PATH
