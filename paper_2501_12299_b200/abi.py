"""ctypes binding of libvmfa_b200.so (include/vmfa_b200.h).

Loads the in-tree library built by ``paper_2501_12299_b200.build`` and raises
``VmfaError`` when it is missing -- there is no fallback implementation.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "_lib", "libvmfa_b200.so")
_lib = None

STATUS = {
    0: "OK", 1: "InvalidArgument", 2: "CholeskyFailure", 3: "EmptyKSet",
    4: "InsufficientCandidates", 5: "SingularEc", 6: "MaxIterExceeded",
    7: "TargetUnreachable", 8: "DegenerateData", 9: "BadMagic", 10: "TruncatedFile",
    11: "UnsupportedVersion", 12: "IoError", 100: "CudaError", 101: "NoDevice", 102: "Unsupported",
}


class VmfaError(RuntimeError):
    """A non-zero vmfa_status; ``code`` maps 1:1 onto the reference's
    exception types (errors.hpp:9-62)."""

    def __init__(self, code: int, msg: str):
        self.code = code
        self.kind = STATUS.get(code, str(code))
        super().__init__(f"{self.kind}: {msg}")


def library_path() -> str:
    return _LIB


class IterReport(C.Structure):
    _fields_ = [("free_energy_estep", C.c_double), ("free_energy", C.c_double),
                ("joints", C.c_uint64), ("empty_components", C.c_int32),
                ("failed_component", C.c_int32)]


class SynthSpec(C.Structure):
    _fields_ = [("kind", C.c_int), ("n_total", C.c_int64), ("D", C.c_int), ("C_true", C.c_int),
                ("H_true", C.c_int), ("dirichlet", C.c_int), ("mu_std", C.c_double),
                ("lam_std", C.c_double), ("psi_lo", C.c_double), ("psi_hi", C.c_double),
                ("noise_std", C.c_double), ("img_w", C.c_int), ("img_h", C.c_int),
                ("img_c", C.c_int), ("blur_sigma", C.c_double), ("data_seed", C.c_uint64)]


_P = C.c_void_p
_I, _I64, _U64, _D = C.c_int, C.c_int64, C.c_uint64, C.c_double
_SIGS = {
    "vmfa_abi_version": (_I, []),
    "vmfa_last_error": (C.c_char_p, []),
    "vmfa_device_available": (_I, []),
    "vmfa_ctx_create": (_I, [C.POINTER(_P), _I, _I, _I, _I, _I, _I, _I64, _I64, _I64, _P]),
    "vmfa_ctx_destroy": (_I, [_P]),
    "vmfa_ctx_device_bytes": (_I, [_P, C.POINTER(C.c_size_t)]),
    "vmfa_upload_data": (_I, [_P, _P, _I64, _I64]),
    "vmfa_upload_data_async": (_I, [_P, _P, _I64, _I64]),
    "vmfa_stage_data_async": (_I, [_P, _P, _I64, _I64]),
    "vmfa_swap_data": (_I, [_P]),
    "vmfa_set_lookahead": (_I, [_P, _I]),
    "vmfa_save_dataset": (_I, [C.c_char_p, _P, _I64, _I]),
    "vmfa_dataset_info": (_I, [C.c_char_p, _P, _P]),
    "vmfa_load_dataset": (_I, [C.c_char_p, _I64, _I64, _I, _P]),
    "vmfa_save_checkpoint": (_I, [C.c_char_p, _I, _I, _I, _P, _P, _P, _P]),
    "vmfa_checkpoint_info": (_I, [C.c_char_p, _P, _P, _P]),
    "vmfa_load_checkpoint": (_I, [C.c_char_p, _I, _I, _I, _P, _P, _P, _P]),
    "vmfa_save_state": (_I, [C.c_char_p, _I64, _I, _I, _I, _P, _P, _P]),
    "vmfa_state_info": (_I, [C.c_char_p, _P, _P, _P, _P]),
    "vmfa_load_state": (_I, [C.c_char_p, _I64, _I64, _I, _I, _I, _P, _P, _P]),
    "vmfa_set_floor": (_I, [_P, _P]),
    "vmfa_upload_params": (_I, [_P, _P, _P, _P, _P]),
    "vmfa_download_params": (_I, [_P, _P, _P, _P, _P]),
    "vmfa_precompute": (_I, [_P, C.POINTER(_I)]),
    "vmfa_download_caches": (_I, [_P, _P, _P, _P, _P, _P, _P, _P]),
    "vmfa_upload_state": (_I, [_P, _P, _P, _P]),
    "vmfa_download_state": (_I, [_P, _P, _P, _P, _P]),
    "vmfa_estep": (_I, [_P, _U64, _U64, _I, C.POINTER(_D), C.POINTER(_U64)]),
    "vmfa_download_estep": (_I, [_P, _P, _P, _P, _P]),
    "vmfa_download_distances": (_I, [_P, _I64, _P, _P, _P, _P, C.POINTER(_I64)]),
    "vmfa_accumulate_suffstats": (_I, [_P]),
    "vmfa_download_suffstats": (_I, [_P, _P, _P, _P, _P]),
    "vmfa_upload_suffstats": (_I, [_P, _P, _P, _P, _P]),
    "vmfa_update_params": (_I, [_P, C.POINTER(_I)]),
    "vmfa_truncated_free_energy": (_I, [_P, C.POINTER(_D)]),
    "vmfa_exact_log_likelihood": (_I, [_P, C.POINTER(_D)]),
    "vmfa_em_full_step": (_I, [_P, C.POINTER(_D), C.POINTER(_U64)]),
    "vmfa_afkmc2_seed": (_I, [_P, _I, _I, _U64, _P, _P, C.POINTER(_U64)]),
    "vmfa_iterate": (_I, [_P, _U64, _U64, _I, C.POINTER(IterReport)]),
    "vmfa_exchange_buffer": (_I, [_P, _I, C.POINTER(_P), C.POINTER(C.c_size_t), C.POINTER(_I)]),
    "vmfa_phase_estep_local": (_I, [_P, _U64, _U64, _I]),
    "vmfa_phase_estep_finish": (_I, [_P]),
    "vmfa_phase_stats_local": (_I, [_P]),
    "vmfa_phase_update": (_I, [_P, C.POINTER(_I)]),
    "vmfa_phase_free_energy_local": (_I, [_P]),
    "vmfa_phase_scalars": (_I, [_P, C.POINTER(_D), C.POINTER(_U64), C.POINTER(_D)]),
    "vmfa_cooc_sparse": (_I, [_P, C.POINTER(_I)]),
    "vmfa_cooc_local_list": (_I, [_P, _I, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P), C.POINTER(_P), _P]),
    "vmfa_cooc_select": (_I, [_P, _P, _P, _P, _P, C.c_int64, _I, _I]),
    "vmfa_profile_enable": (_I, [_P, _I]),
    "vmfa_scoring_work": (_I, [_P, _P, _I]),
    "vmfa_accumulate_suffstats_k": (_I, [_P, _P, _P]),
    "vmfa_truncated_free_energy_k": (_I, [_P, _P, C.POINTER(_D)]),
    "vmfa_log_joint": (_I, [_P, _P, _I64, _P, _P]),
    "vmfa_build_search_space": (_I, [_P, _U64, _U64, _P, _P, _P]),
    "vmfa_update_k": (_I, [_P, _P, _P, _P, _P]),
    "vmfa_hard_partition": (_I, [_P, _P, _P, _P, _P, _P, _P, _P]),
    "vmfa_accumulate_distances": (_I, [_P, _I, _P, _P, _P, _P, _P, _P, _I64, _P, _P, _P, _P, C.POINTER(_I64)]),
    "vmfa_update_g": (_I, [_P, _I64, _P, _P, _P, _P, _P, _P]),
    "vmfa_responsibilities": (_I, [_P, _I64, _I, _P, _P]),
    "vmfa_kernel_times": (_I, [_P, _I, _P, _P, _P, C.POINTER(_I)]),
    "vmfa_kernel_name": (C.c_char_p, [_I]),
    "vmfa_ctx_stream": (_P, [_P]),
    "vmfa_diag_scorer_cycles": (_I, [_I, _P, _I]),
    "vmfa_diag_radix_sort": (_I, [_P, _I64, _I, _P, _P, _I]),
    "vmfa_synchronize": (_I, [_P]),
    "vmfa_gen_synthetic": (_I, [C.POINTER(SynthSpec), _I64, _I64, _P, _P, _I]),
    "vmfa_host_initialize": (_I, [_P, _I64, _I, _I, _I, _I, _I, _U64, _D, _I, _P, _P, _P, _P,
                                  _P, _P, _P, _P, _P]),
    "vmfa_host_moments": (_I, [_P, _I64, _I, _P, _P, _I]),
    "vmfa_seed_draws": (_I, [_U64, _I64, _I64, _I64, _P]),
    "vmfa_host_distinct_hashes": (_I, [_P, _I64, _I, _I64, _P, C.POINTER(_I64)]),
    "vmfa_host_init_shard": (_I, [_I64, _I, _I, _I, _I, _I, _U64, _D, _I, _P, _P, _P, _P, _I64, _I64, _I64,
                                  _P, _P, _P, _P, _P, _P, _P]),
}


def lib():
    """Load libvmfa_b200.so (raises VmfaError if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise VmfaError(101, f"{_LIB} not built: run `python -m paper_2501_12299_b200.build` "
                                 "(there is no CPU fallback)")
        L = C.CDLL(_LIB)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(code: int):
    if code != 0:
        msg = lib().vmfa_last_error()
        raise VmfaError(code, msg.decode() if msg else "")


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays passed to the C-ABI must be C-contiguous"
    return a.ctypes.data_as(C.c_void_p)
