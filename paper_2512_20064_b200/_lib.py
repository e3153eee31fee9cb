"""ctypes binding of libmpsg.so (include/mpsg.h).  The CUDA library is the only compute path:
if it is missing or no B200 is visible, calls fail loudly — there is no CPU fallback."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MPSG_LIB_PATH") or os.path.join(HERE, "libmpsg.so")

ABI_VERSION = 5  # include/mpsg.h MPSG_ABI_VERSION
MPSG_OK, MPSG_ERR_INTERNAL, MPSG_ERR_CONFIG, MPSG_ERR_NUMERIC, MPSG_ERR_IO, MPSG_ERR_CUDA = 0, 1, 2, 3, 4, 5

_u64, _int, _dbl = C.c_uint64, C.c_int, C.c_double
_pd = C.POINTER(C.c_double)
_pu8 = C.POINTER(C.c_uint8)
_pu64 = C.POINTER(C.c_uint64)


class MpsView(C.Structure):
    _fields_ = [("num_sites", _u64), ("phys_dim", _u64), ("bond_dims", _pu64),
                ("gamma", C.POINTER(_pd)), ("lambda_", C.POINTER(_pd))]


class Policy(C.Structure):
    _fields_ = [("compute", _int), ("storage", _int), ("scaling", _int)]


class Options(C.Structure):
    _fields_ = [("mode", _int), ("pass_samples", _u64), ("record_site_times", _int),
                ("tp_size", _int), ("tp_rank", _int), ("host_stream_slots", _int),
                ("record_decay_trace", _int), ("scheme", _int), ("slice", _int)]


class Stats(C.Structure):
    _fields_ = [("contraction_macs", _u64), ("measure_weight_macs", _u64), ("dead_samples", _u64),
                ("seconds", _dbl), ("site_seconds", _pd), ("issued_mma_flops", _u64),
                ("h2d_bytes", _u64), ("d2h_bytes", _u64), ("gemm_seconds", _dbl),
                ("gemm_flops", _u64), ("kernel_launches", _u64), ("device_seconds", _dbl),
                ("decay_trace", _pd), ("displacement_macs", _u64), ("measure_pipeline_ops", _u64),
                ("near_boundary_draws", _u64)]


# (name, restype, argtypes) for every entry point of include/mpsg.h
SIGNATURES = [
    ("mpsg_abi_version", _int, []),
    ("mpsg_last_error", C.c_char_p, []),
    ("mpsg_device_count", _int, []),
    ("mpsg_create", _int, [C.POINTER(MpsView), C.POINTER(Policy), C.POINTER(Options),
                           C.POINTER(_int), _int, C.POINTER(C.c_void_p)]),
    ("mpsg_builder_begin", _int, [_u64, _u64, _pu64, C.POINTER(Policy), C.POINTER(Options),
                                  C.POINTER(_int), _int, C.POINTER(C.c_void_p)]),
    ("mpsg_builder_set_site", _int, [C.c_void_p, _u64, C.c_void_p, _int, _int, _pd]),
    ("mpsg_builder_finish", _int, [C.c_void_p]),
    ("mpsg_destroy", None, [C.c_void_p]),
    ("mpsg_state_bytes", _u64, [C.c_void_p]),
    ("mpsg_scheme", _int, [C.c_void_p]),
    ("mpsg_mode", _int, [C.c_void_p]),
    ("mpsg_gamma_store", _int, [C.c_void_p]),
    ("mpsg_decoded_gamma", _int, [C.c_void_p, _u64, _pd]),
    ("mpsg_sample", _int, [C.c_void_p, _u64, _u64, _u64, _pu8, C.POINTER(Stats)]),
    ("mpsg_sample_device", _int, [C.c_void_p, _u64, _u64, _u64, C.c_void_p, C.POINTER(Stats)]),
    ("mpsg_marginals", _int, [C.c_void_p, _u64, _u64, _pu8, _pd]),
    ("mpsg_sample_displaced", _int, [C.c_void_p, _u64, _u64, _u64, _pd, _pu8, C.POINTER(Stats)]),
    ("mpsg_marginals_displaced", _int, [C.c_void_p, _u64, _u64, _pu8, _pd, _pd]),
    ("mpsg_displacement_matrix", _int, [_dbl, _dbl, _u64, _pd]),
    ("mpsg_device_draws", _int, [_u64, _u64, _u64, _u64, _pd]),
    ("mpsg_contract_site", _int, [C.c_void_p, _u64, _pd, _u64, _pd]),
    ("mpsg_create_from_file", _int, [C.c_char_p, C.POINTER(Policy), C.POINTER(Options),
                                     C.POINTER(_int), _int, C.POINTER(C.c_void_p)]),
    ("mpsg_generated_site_values", _int, [C.c_void_p, _u64, _pd]),
    ("mpsg_create_from_file_streamed", _int, [C.c_char_p, C.POINTER(Policy), C.POINTER(Options),
                                     C.POINTER(_int), _int, C.POINTER(C.c_void_p)]),
    ("mpsg_save_file", _int, [C.c_void_p, C.c_char_p, _int]),
    ("mpsg_nccl_unique_id", _int, [C.POINTER(C.c_uint8)]),
    ("mpsg_tp_connect_nccl", _int, [C.c_void_p, C.POINTER(C.c_uint8)]),
    ("mpsg_tp_connect_local", _int, [C.POINTER(C.c_void_p), _int]),
    ("mpsg_generated_begin", _int, [_u64, _u64, _pu64, C.POINTER(Policy), C.POINTER(Options),
                                    C.POINTER(_int), _int, _u64, C.POINTER(C.c_void_p)]),
    ("mpsg_generated_add_base", _int, [C.c_void_p, C.c_void_p, _int, _u64, _u64, C.POINTER(_int)]),
    ("mpsg_generated_set_site", _int, [C.c_void_p, _u64, _int, _pd]),
    ("mpsg_synthetic_site", _int, [C.c_void_p, _u64, _u64, _u64, _u64, _pd, _pd, _u64, _u64, C.c_void_p]),
]

_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "csrc")], check=True)


def lib():
    """Load the in-tree libmpsg.so (building it if a toolchain is present)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            try:
                build()
            except Exception as e:  # pragma: no cover
                raise RuntimeError(f"libmpsg.so missing and could not be built: {e}") from e
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        if L.mpsg_abi_version() != ABI_VERSION:
            raise RuntimeError("libmpsg ABI mismatch")
        _lib = L
    return _lib


def last_error() -> str:
    return lib().mpsg_last_error().decode(errors="replace")
