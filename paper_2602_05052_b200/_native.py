"""ctypes binding of libtgk.so (include/tgk.h).

Loads the in-tree library built by ``paper_2602_05052_b200/build.py``.  There
is no fallback: if the library is missing, import of the compute API raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TGK_LIB") or os.path.join(_HERE, "lib", "libtgk.so")  # TGK_LIB: A/B builds

TGK_OK, TGK_ERR_NUMERICAL, TGK_ERR_INPUT, TGK_ERR_CUDA = 0, 1, 2, 3
TRI3, QUAD4, TET4 = 0, 1, 2
POISSON, ELASTICITY, MASS = 0, 1, 2
FIELD_CONSTANT, FIELD_ELEMENT, FIELD_NODAL = 0, 1, 2
MODE_EXACT = 0
MODE_FAST = 1
ROUTING_SEGMENTS = 1
KINDS = {"tri3": TRI3, "quad4": QUAD4, "tet4": TET4}
KIND_NAMES = {v: k.upper() for k, v in KINDS.items()}


class InputError(RuntimeError):
    """tg::InputError (errors.hpp:9-11)."""


class NumericalError(RuntimeError):
    """tg::NumericalError (errors.hpp:13-16)."""


class CudaError(RuntimeError):
    """CUDA / runtime failure inside libtgk (no CPU fallback exists)."""


class Field(C.Structure):
    _fields_ = [("type", C.c_int), ("value", C.c_double), ("data", C.c_void_p), ("n", C.c_int64)]


class Problem(C.Structure):
    _fields_ = [("kind", C.c_int), ("diffusion", Field), ("lam", Field), ("mu", Field),
                ("plane_stress", C.c_int), ("n_source", C.c_int), ("source", Field * 3),
                ("with_mass", C.c_int), ("mode", C.c_int)]


class FieldBatch(C.Structure):
    _fields_ = [("slot", C.c_int), ("data", C.c_void_p), ("stride", C.c_int64)]


SLOTS = {"diffusion": 0, "lam": 1, "mu": 2, "source0": 3, "source1": 4, "source2": 5}


class RoutingView(C.Structure):
    _fields_ = [("N", C.c_int64), ("E", C.c_int64), ("nnz", C.c_int64), ("k", C.c_int),
                ("components", C.c_int), ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p),
                ("slot_of", C.c_void_p), ("vec_offsets", C.c_void_p), ("vec_slots", C.c_void_p),
                ("mat_offsets", C.c_void_p), ("mat_slots", C.c_void_p)]


_lib = None

_P = C.c_void_p
_I = C.c_int
_I64 = C.c_int64
_D = C.c_double
_SIGS = {
    "tgk_last_error": (C.c_char_p, []),
    "tgk_version": (_I, []),
    "tgk_device_count": (_I, []),
    "tgk_set_thread_count": (None, [_I]),
    "tgk_thread_count": (_I, []),
    "tgk_grid_sizes": (_I, [_I, _P, _P, _P]),
    "tgk_generate_grid": (_I, [_I, _P, _P, _P, _P]),
    "tgk_content_hash": (C.c_uint64, [_I, _P, _I64, _P, _I64]),
    "tgk_topological_boundary": (_I64, [_I, _P, _I64, _I64, _P]),
    "tgk_validate": (_I, [_I, _P, _I64, _P, _I64]),
    "tgk_default_degree": (_I, [_I, _I]),
    "tgk_tables": (_I, [_I, _I, _P, _P, _P, _P, _P]),
    "tgk_mesh_create": (_I, [_I, _P, _I64, _P, _I64, _P]),
    "tgk_mesh_create_d": (_I, [_I, _P, _I64, _P, _I64, _P]),
    "tgk_mesh_upload": (_I, [_P, _P, _P, _P]),
    "tgk_mesh_destroy": (None, [_P]),
    "tgk_mesh_info": (_I, [_P, _P, _P, _P, _P, _P]),
    "tgk_routing_build": (_I, [_P, _I, _I, _P, _P]),
    "tgk_routing_destroy": (None, [_P]),
    "tgk_routing_get_view": (_I, [_P, _P]),
    "tgk_routing_copy": (_I, [_P, _P, _P, _P, _P, _P, _P, _P]),
    "tgk_routing_set_owned_rows": (_I, [_P, _I64, _I64]),
    "tgk_routing_set_element_range": (_I, [_P, _I64, _I64]),
    "tgk_interface_combine_d": (_I, [_P, _P, _I64, _P]),
    "tgk_allen_cahn_d": (_I, [_P, _P, _P, _D, _P, _P, _P]),
    "tgk_assemble_f32_d": (_I, [_P, _P, _P, _P, _P, _P, _P, _P]),
    "tgk_routing_load": (_I, [_P, _I, C.c_uint64, C.c_char_p, _P, _P, _P]),
    "tgk_spmv_d": (_I, [_I64, _P, _P, _P, _P, _P, _P]),
    "tgk_condense_d": (_I, [_I64, _P, _P, _P, _P, _I64, _P, _P, _P, _P]),
    "tgk_condensed_info": (_I, [_P] * 11),
    "tgk_restrict_to_free_d": (_I, [_P, _P, _P, _P, _P, _P]),
    "tgk_expand_d": (_I, [_P, _P, _P, _P]),
    "tgk_condensed_copy": (_I, [_P] * 8),
    "tgk_condensed_destroy": (None, [_P]),
    "tgk_bicgstab_d": (_I, [_I64, _P, _P, _P, _P, _P, _D, _D, _I64, _P, _P, _P, _P]),
    "tgk_copy_d2d": (_I, [_P, _P, _I64, _P]),
    "tgk_alloc_d": (_I, [_P, _I64]),
    "tgk_scatter_add": (_I, [_P, _P, _P, _P, _P, _P, _P, _P]),
    "tgk_mesh_coordinates_changed": (_I, [_P]),
    "tgk_free_d": (_I, [_P]),
    "tgk_copy_d2h": (_I, [_P, _P, _I64]),
    "tgk_copy_h2d": (_I, [_P, _P, _I64]),
    "tgk_mesh_upload_async": (_I, [_P, _P, _P, _P]),
    "tgk_mesh_upload_check": (_I, [_P]),
    "tgk_routing_create_host": (_I, [_P, _I, _I64, _I64, _I, _I64, _P, _P, _P, _P, _P, _P, _P, _P]),
    "tgk_routing_plan_stats": (_I, [_P, _I, _P, _P, _P, _P]),
    "tgk_routing_fast_plan_info": (_I, [_P, _P, _P, _P, _P, _P, _P]),
    "tgk_routing_save": (_I, [_P, C.c_uint64, C.c_char_p]),
    "tgk_geometry_d": (_I, [_P, _I, _P, _P, _P, _P, _P, _P]),
    "tgk_local_stiffness_diffusion_d": (_I, [_P, _I, _P, _P, _P]),
    "tgk_local_stiffness_elasticity_d": (_I, [_P, _I, _P, _P, _P, _P]),
    "tgk_local_mass_d": (_I, [_P, _I, _P, _P, _P]),
    "tgk_local_load_d": (_I, [_P, _I, _P, _P, _P]),
    "tgk_local_load_vector_d": (_I, [_P, _I, _P, _P, _P]),
    "tgk_evaluate_field_d": (_I, [_P, _I, _P, _P, _P]),
    "tgk_reduce_matrix_d": (_I, [_P, _P, _P, _P]),
    "tgk_reduce_vector_d": (_I, [_P, _P, _P, _P]),
    "tgk_assemble_d": (_I, [_P, _P, _P, _P, _P, _P, _P]),
    "tgk_assemble_async_d": (_I, [_P, _P, _P, _P, _P, _P, _P, _P]),
    "tgk_assemble": (_I, [_P, _P, _P, _P, _P, _P]),
    "tgk_assemble_batched_d": (_I, [_P, _P, _I64, _P, _D, _P, _P, _I, _P]),
    "tgk_assemble_fields_batched_d": (_I, [_P, _P, _P, _I64, _P, _I, _P, _P, _P, _P]),
    "tgk_gradient_products_d": (_I, [_P, _I64, _P, _P, _P, _P, _P]),
    "tgk_adjoint_gather_d": (_I, [_P, _P, _I64, _P, _P, _P, _I, _P]),
    "tgk_simp_sensitivity_d": (_I, [_I64, _I, _P, _P, _D, _D, _D, _P, _P, _I64, _P, _P]),
}
EXPORTS = tuple(_SIGS)


def lib():
    """The loaded libtgk.so (raises OSError when it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OSError(f"{LIB_PATH} not built: run `python -m paper_2602_05052_b200.build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc):
    if rc == TGK_OK:
        return
    msg = lib().tgk_last_error().decode()
    if rc == TGK_ERR_INPUT:
        raise InputError(msg)
    if rc == TGK_ERR_NUMERICAL:
        raise NumericalError(msg)
    raise CudaError(msg)
