"""ctypes binding of the in-tree C ABI (include/peps_b200.h, lib/libpeps_b200.so).

There is no fallback: if the shared library or an sm_100 device is missing,
every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libpeps_b200.so")

_lib = None


class PepsError(RuntimeError):
    KINDS = {1: "ShapeError", 2: "ValidationError", 3: "ResourceError", 4: "NumericalError",
             5: "ConfigError", 6: "CudaError", 9: "Error"}

    def __init__(self, kind: int, msg: str):
        self.kind = self.KINDS.get(kind, "Error")
        super().__init__(f"{self.kind}: {msg}")


class Trunc(C.Structure):
    _fields_ = [("max_rank", C.c_uint64), ("rel_cutoff", C.c_double)]


class Rsvd(C.Structure):
    _fields_ = [("power_iters", C.c_int32), ("oversample", C.c_int32), ("seed", C.c_uint64)]


class ContractOpt(C.Structure):
    _fields_ = [("trunc", Trunc), ("strategy", C.c_int32), ("rsvd", Rsvd), ("canonicalize", C.c_int32),
                ("seed", C.c_uint64)]


class ExpectationOpt(C.Structure):
    _fields_ = [("contract", ContractOpt), ("use_cache", C.c_int32), ("shared_environments", C.c_int32),
                ("allow_complex", C.c_int32)]


class ExpectationResult(C.Structure):
    _fields_ = [("value", C.c_double), ("norm_sq", C.c_double), ("raw_sum", C.c_double * 2),
                ("complex_value", C.c_double * 2), ("full_sweeps", C.c_uint64), ("band_contractions", C.c_uint64),
                ("flops", C.c_uint64)]


_VP = C.c_void_p
_SIGS = {
    "pepsb_last_error": (C.c_char_p, []),
    "pepsb_last_error_kind": (C.c_int, []),
    "pepsb_ctx_create": (C.c_int, [C.c_int, C.POINTER(_VP)]),
    "pepsb_ctx_destroy": (C.c_int, [_VP]),
    "pepsb_ctx_sync": (C.c_int, [_VP]),
    "pepsb_ctx_set_option": (C.c_int, [_VP, C.c_char_p, C.c_int64]),
    "pepsb_ctx_counters": (C.c_int, [_VP, C.POINTER(C.c_uint64)]),
    "pepsb_ctx_get_counter": (C.c_int, [_VP, C.c_char_p, C.POINTER(C.c_uint64)]),
    "pepsb_ctx_reset_counters": (C.c_int, [_VP]),
    "pepsb_ctx_stream": (_VP, [_VP]),
    "pepsb_ctx_profile_timeline": (C.c_int, [_VP, C.POINTER(C.c_double), C.c_int]),
    "pepsb_ctx_debug_word": (C.c_int, [_VP, C.c_int, C.c_int]),
    "pepsb_ctx_profile_records": (C.c_int, [_VP, C.POINTER(C.c_double), C.c_int]),
    "pepsb_ctx_profile": (C.c_int, [_VP, C.c_int]),
    "pepsb_ctx_profile_report": (C.c_int, [_VP, C.POINTER(C.c_double)]),
    "pepsb_ctx_profile_report_ex": (C.c_int, [_VP, C.POINTER(C.c_double)]),
    "pepsb_tensor_from_host": (C.c_int, [_VP, C.c_int, C.POINTER(C.c_int64), _VP, C.POINTER(_VP)]),
    "pepsb_tensor_from_device": (C.c_int, [_VP, C.c_int, C.POINTER(C.c_int64), _VP, C.POINTER(_VP)]),
    "pepsb_tensor_ndim": (C.c_int, [_VP]),
    "pepsb_tensor_shape": (C.c_int, [_VP, C.POINTER(C.c_int64)]),
    "pepsb_tensor_to_host": (C.c_int, [_VP, _VP, _VP]),
    "pepsb_tensor_to_host_async": (C.c_int, [_VP, _VP, _VP]),
    "pepsb_tensor_to_device": (C.c_int, [_VP, _VP, _VP]),
    "pepsb_tensor_free": (None, [_VP]),
    "pepsb_random_tensor": (C.c_int, [_VP, C.c_int, C.POINTER(C.c_int64), C.c_uint64, C.c_int, C.POINTER(_VP)]),
    "pepsb_contract": (C.c_int, [_VP, C.c_char_p, C.c_int, C.POINTER(_VP), C.POINTER(_VP)]),
    "pepsb_implicit": (C.c_int, [_VP, C.c_int, C.POINTER(_VP), C.c_char_p, C.c_char_p, C.c_char_p, _VP, C.c_int,
                                 C.POINTER(_VP)]),
    "pepsb_gram_orthogonalize": (C.c_int, [_VP, _VP, C.c_int, C.POINTER(_VP), C.POINTER(_VP)]),
    "pepsb_eigh": (C.c_int, [_VP, _VP, C.POINTER(C.c_double), C.c_int64, C.POINTER(_VP)]),
    "pepsb_random_slice": (C.c_int, [_VP, C.c_int, C.POINTER(C.c_int64), C.c_int, C.c_int64, C.c_int64, C.c_uint64,
                                     C.c_int, C.POINTER(_VP)]),
    "pepsb_tensor_conj": (C.c_int, [_VP, _VP, C.POINTER(_VP)]),
    "pepsb_tensor_slice": (C.c_int, [_VP, _VP, C.c_int, C.c_int64, C.c_int64, C.POINTER(_VP)]),
    "pepsb_tensor_reshape": (C.c_int, [_VP, C.c_int, C.POINTER(C.c_int64), C.POINTER(_VP)]),
    "pepsb_tensor_data_ptr": (C.c_int, [_VP, C.POINTER(_VP)]),
    "pepsb_gram": (C.c_int, [_VP, _VP, C.POINTER(_VP)]),
    "pepsb_gram_factors": (C.c_int, [_VP, _VP, C.POINTER(_VP), C.POINTER(_VP), C.POINTER(_VP), C.POINTER(C.c_double),
                                     C.POINTER(C.c_int), C.c_int64]),
    "pepsb_projected_svd": (C.c_int, [_VP, _VP, C.c_int64, C.POINTER(_VP), C.POINTER(C.c_double), C.c_int64]),
    "pepsb_svd": (C.c_int, [_VP, _VP, C.c_int, C.POINTER(_VP), C.POINTER(C.c_double), C.c_int64,
                            C.POINTER(C.c_int64), C.POINTER(_VP)]),
    "pepsb_randomized_svd": (C.c_int, [_VP, C.c_int, C.POINTER(_VP), C.c_char_p, C.c_char_p, C.c_char_p,
                                       C.POINTER(Trunc), C.POINTER(Rsvd), C.POINTER(_VP), C.POINTER(C.c_double),
                                       C.c_int64, C.POINTER(C.c_int64), C.POINTER(_VP), C.POINTER(C.c_int)]),
    "pepsb_einsumsvd": (C.c_int, [_VP, C.c_int, C.POINTER(_VP), C.c_char_p, C.c_char_p, C.c_char_p,
                                  C.POINTER(Trunc), C.c_int, C.c_int, C.POINTER(Rsvd), C.POINTER(_VP),
                                  C.POINTER(_VP), C.POINTER(C.c_double), C.c_int64, C.POINTER(C.c_int64),
                                  C.POINTER(C.c_int)]),
    "pepsb_state_create": (C.c_int, [_VP, C.c_int, C.c_int, C.c_int, C.POINTER(_VP), C.POINTER(_VP)]),
    "pepsb_state_site": (C.c_int, [_VP, C.c_int, C.c_int, C.POINTER(_VP)]),
    "pepsb_state_free": (None, [_VP]),
    "pepsb_boundary_create": (C.c_int, [_VP, C.c_int, C.POINTER(_VP), C.POINTER(C.c_int64), C.POINTER(_VP)]),
    "pepsb_boundary_length": (C.c_int, [_VP]),
    "pepsb_boundary_site": (C.c_int, [_VP, C.c_int, C.POINTER(_VP)]),
    "pepsb_boundary_phys": (C.c_int, [_VP, C.POINTER(C.c_int64)]),
    "pepsb_boundary_free": (None, [_VP]),
    "pepsb_two_layer_first_row": (C.c_int, [_VP, _VP, _VP, C.POINTER(_VP)]),
    "pepsb_two_layer_apply_row": (C.c_int, [_VP, _VP, _VP, _VP, C.c_int, C.POINTER(ContractOpt), C.c_uint64,
                                            C.POINTER(_VP)]),
    "pepsb_comm_unique_id": (C.c_int, [C.c_char_p]),
    "pepsb_comm_init": (C.c_int, [_VP, C.c_char_p, C.c_int, C.c_int]),
    "pepsb_comm_destroy": (C.c_int, [_VP]),
    "pepsb_two_layer_apply_row_sharded": (C.c_int, [_VP, _VP, _VP, _VP, C.c_int, C.POINTER(ContractOpt),
                                                    C.c_uint64, C.POINTER(_VP)]),
    "pepsb_contract_two_layer_sharded": (C.c_int, [_VP, _VP, _VP, C.POINTER(ContractOpt), C.POINTER(C.c_double),
                                                   C.POINTER(C.c_double)]),
    "pepsb_contract_two_layer": (C.c_int, [_VP, _VP, _VP, C.POINTER(ContractOpt), C.POINTER(C.c_double),
                                           C.POINTER(C.c_double)]),
    "pepsb_chain_scalar": (C.c_int, [_VP, _VP, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "pepsb_build_row_cache": (C.c_int, [_VP, _VP, C.POINTER(ContractOpt), C.POINTER(_VP)]),
    "pepsb_flip_vertical": (C.c_int, [_VP, _VP, C.POINTER(_VP)]),
    "pepsb_row_cache_get": (C.c_int, [_VP, C.c_int, C.c_int, C.POINTER(_VP)]),
    "pepsb_row_cache_free": (None, [_VP]),
    "pepsb_band_environment": (C.c_int, [_VP, _VP, _VP, _VP, C.c_int, C.c_int, _VP, C.POINTER(_VP)]),
    "pepsb_band_splice": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _VP, C.c_int, C.POINTER(C.c_int), C.POINTER(_VP),
                                    C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_int, C.c_int,
                                    C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "pepsb_band_value": (C.c_int, [_VP, _VP, _VP, _VP, C.c_int, C.c_int, _VP, C.c_int, C.POINTER(C.c_int),
                                   C.POINTER(_VP), C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_double),
                                   C.POINTER(C.c_double)]),
    "pepsb_band_env_free": (None, [_VP]),
    "pepsb_save_peps": (C.c_int, [_VP, _VP, C.c_char_p]),
    "pepsb_state_dims": (C.c_int, [_VP, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "pepsb_load_peps": (C.c_int, [_VP, C.c_char_p, C.POINTER(_VP)]),
    "pepsb_approx_apply_mpo": (C.c_int, [_VP, C.c_int, C.POINTER(_VP), C.POINTER(_VP), C.POINTER(Trunc), C.c_int,
                                         C.c_int, C.POINTER(Rsvd), C.c_uint64, C.POINTER(_VP)]),
    "pepsb_contract_one_layer": (C.c_int, [_VP, C.c_int, C.c_int, C.POINTER(_VP), C.c_int, C.POINTER(ContractOpt),
                                           C.c_uint64, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "pepsb_expectation": (C.c_int, [_VP, _VP, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int),
                                    C.POINTER(C.c_int), C.POINTER(_VP), C.POINTER(ExpectationOpt),
                                    C.POINTER(ExpectationResult)]),
    "pepsb_hermitian_exp": (C.c_int, [_VP, _VP, C.c_double, C.c_double, C.POINTER(_VP)]),
    "pepsb_apply_one_site": (C.c_int, [_VP, _VP, _VP, C.c_int, C.POINTER(C.c_int), C.POINTER(_VP)]),
    "pepsb_apply_two_site": (C.c_int, [_VP, _VP, _VP, C.c_int, C.POINTER(C.c_int), C.POINTER(Trunc),
                                       C.POINTER(_VP)]),
    "pepsb_ite_tfim": (C.c_int, [_VP, _VP, C.c_double, C.c_double, C.c_double, C.c_int, C.c_uint64,
                                 C.POINTER(_VP)]),
}


def exported_symbols():
    return list(_SIGS)


def lib():
    """Loads the shared library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(
                f"{LIB_PATH} missing: build it with __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int):
    if rc != 0:
        L = lib()
        raise PepsError(L.pepsb_last_error_kind(), L.pepsb_last_error().decode())
