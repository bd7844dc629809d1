"""ctypes binding of the C-ABI library ``libhv_b200.so`` (include/hv_b200.h).

There is no CPU fallback anywhere in the product: if the library is missing,
fails to load, or no CUDA device is present, every operator raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["HV_LIB"]) if os.environ.get("HV_LIB") else _HERE / "libhv_b200.so"

HV_OK = 0
HV_ERR_INVALID = 1
HV_ERR_DEGENERATE = 2
HV_ERR_NONCONFORMING = 3
HV_ERR_CUDA = 4
HV_ERR_NCCL = 5
HV_ERR_UNSUPPORTED = 6

_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32
_D = C.c_double


class LapPlan(C.Structure):
    """Mirror of ``hv_lap_plan`` (include/hv_b200.h)."""

    _fields_ = [
        ("N", C.c_int),
        ("D", C.c_double * 81),
        ("nelem", _I64),
        ("nglobal", _I64),
        ("d_gid", _P),
        ("d_off", _P),
        ("d_idx", _P),
        ("d_W", _P),
        ("d_Minv", _P),
        ("d_work", _P),
        ("d_y", _P),
        ("TX", C.c_int),
        ("TY", C.c_int),
        ("nlay", C.c_int),
        ("n_z", C.c_int),
        ("ntiles", _I64),
        ("nslot", _I64),
        ("d_gt", _P),
        ("d_code", _P),
        ("d_tmeta", _P),
        ("d_slot_col", _P),
        ("d_slot_row0", _P),
        ("d_slot_nc", _P),
        ("d_col_gid", _P),
        ("d_Wt", _P),
        ("d_Mt", _P),
        ("d_part", _P),
        ("kernel", C.c_int),
        ("d_slot_ext", _P),
        ("d_ext_slots", _P),
        ("next", _I64),
        ("face", C.c_int),
        ("d_send", _P),
        ("d_recv", _P),
        ("wform", C.c_int),
        ("kh", C.c_double),
        ("kd", C.c_double),
        ("d_Ms", _P),
        ("d_tper", _P),
        ("d_yt", _P),
        ("d_tchunk", _P),
        ("d_sv", _P),
        ("seg", C.c_int),
        ("d_bnd", _P),
        ("d_prow", _P),
    ]


# name -> (restype, argtypes)
_SIGS = {
    "hv_abi_version": (C.c_int, []),
    "hv_last_error": (C.c_char_p, []),
    "hv_launch_count": (C.c_int64, []),
    "hv_probe_dfma": (C.c_int, [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_void_p]),
    "hv_probe_pow": (C.c_int, [C.c_int64, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p]),
    "hv_probe_div": (C.c_int, [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "hv_rows_minv": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int, C.c_int,
                               C.c_void_p]),
    "hv_number_gridpoints": (C.c_int, [_P, _I64, C.c_int, C.c_int, C.c_int, _D, _P, _P]),
    "hv_last_writer_coords": (C.c_int, [_P, _P, _I64, C.c_int, C.c_int, C.c_int, _I64, _P]),
    "hv_build_columns": (C.c_int, [_P, _I64, C.c_int, C.c_int, C.c_int, _P, _P, _I64, _I64, _P, _P, _P, _P, _P]),
    "hv_build_dss_csr": (C.c_int, [_P, _I64, _I64, _P, _P]),
    "hv_metric_terms": (C.c_int, [C.c_int, C.c_int, _P, _P, _I64, _P, _P, _P, _P]),
    "hv_dss_csr": (C.c_int, [_P, C.c_int, _I64, _P, _P, _I64, _P, _P]),
    "hv_mass_and_projection": (C.c_int, [C.c_int, _P, _P, _P, _I64, _P, _P, _I64, _P, _P, _P, _P, _P]),
    "hv_mass_proj_sums": (C.c_int, [C.c_int, _P, _P, _P, _I64, _P, _P, _I64, _P, _P]),
    "hv_mass_proj_finalize": (C.c_int, [_I64, _P, _P, _P, _P, _P, _P]),
    "hv_viscous_metric": (C.c_int, [C.c_int, C.c_int, _P, _D, _P, _P, _I64, _P, _P, _P, _P, _P, _P, _P, _P]),
    "hv_laplacian": (C.c_int, [C.POINTER(LapPlan), _P, _I64, C.c_int, _P, _P, _I64, _P, _D, _P]),
    "hv_tile_pack_minv": (C.c_int, [_I64, C.c_int, C.c_int, _P, _P, _P, _P]),
    "hv_viscous_axis": (C.c_int, [C.c_int, _P, _I64, _P, _P, _P, C.c_int, _D, _P, _P]),
    "hv_plane_metric_doubles": (_I64, [C.c_int, C.c_int, C.c_int, C.c_int]),
    "hv_plane_yt_layout": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _P]),
    "hv_plane_chunk_rows": (C.c_int, [C.c_int, C.c_int, C.c_int]),
    "hv_tile_pack_metric": (C.c_int, [C.c_int, C.c_int, C.c_int, _I64, C.c_int, _P, _P, _I64, C.c_int, _P, _P]),
    "hv_lap_local": (C.c_int, [C.POINTER(LapPlan), _P, _I64, C.c_int, _P, _P, _I64, _P, _D, C.c_uint32, C.c_int,
                               _P]),
    "hv_lap_finish": (C.c_int, [C.POINTER(LapPlan), _P, _I64, C.c_int, _P, _D, C.c_uint32, C.c_int, _P]),
    "hv_hyperdiffusion": (C.c_int, [C.POINTER(LapPlan), _P, _I64, C.c_int, _P, C.c_int, _P, _I64, C.c_int, _P]),
    "hv_hyperdiffusion_stage": (C.c_int, [C.POINTER(LapPlan), _P, _I64, C.c_int, _P, _P, _I64, C.c_int, _P]),
    "hv_euler_setup": (C.c_int, [C.c_int, _P, _I64, _P, _P, _P, _P, _P, _P, _P, C.c_int, _P, _P]),
    "hv_euler_vertical": (C.c_int, [C.c_int, _P, _P, C.c_int, _D, _D, _D, _I64, C.c_int, C.c_int, _P, _P, _P, _P, _P,
                                    _P, _I64, _P, _I64, C.c_int, _P]),
    "hv_column_jacobian": (C.c_int, [C.c_int, _P, _P, C.c_int, _D, _D, _D, _D, _I64, C.c_int, C.c_int, _P, _P,
                                     _P, _P, _P, _P, _P, _P]),
    "hv_band_lu_factor": (C.c_int, [_P, _I64, C.c_int, C.c_int, C.c_int, _P, _P, _P]),
    "hv_band_solve": (C.c_int, [_P, _P, _I64, C.c_int, C.c_int, C.c_int, _P, _P]),
    "hv_euler_diagnostics": (C.c_int, [C.c_int, _D, _D, _D, _D, C.c_int, _I64, _P, _P, _P, _P, _I64, C.c_int, _P,
                                       _P, _P, _P]),
    "hv_elem_deriv": (C.c_int, [C.c_int, _P, _P, _I64, _P, C.c_int, C.c_int, _P, _P]),
    "hv_lap_local_tiles": (C.c_int, [C.POINTER(LapPlan), _P, _I64, C.c_int, _P, _P, _I64, _P, _D, C.c_uint32,
                                     C.c_int, _I64, _I64, C.c_int, _P]),
    "hv_euler_rhs_tiles": (C.c_int, [C.POINTER(LapPlan), _P, _P, C.c_int, C.c_int, C.c_int, _D, _D, _D, _D, _P, _P,
                                     _I64, _P, _I64, C.c_int, _P]),
    "hv_euler_rhs": (C.c_int, [C.c_int, _P, C.c_int, C.c_int, C.c_int, _D, _D, _D, _D, _I64, _I64, _P, _P, C.c_int,
                               _P, _P, _P, _P, _P, _P, _I64, _P, _P, _I64, C.c_int, _P]),
    # test hook (host build of the metric arithmetic); never used by the product path
    "hv_debug_metric_terms_host": (C.c_int, [C.c_int, C.c_int, _P, _P, _I64, _P, _P, _P]),
}

_lib = None
ABI_VERSION = 6          # include/hv_b200.h HV_ABI_VERSION (LapPlan layout above)


def lib():
    """Load (once) and return the ctypes handle; raises if the library is absent."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2311_11425_b200.build` "
                "(there is no CPU fallback)")
        h = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        if h.hv_abi_version() != ABI_VERSION:
            raise RuntimeError(f"{LIB_PATH}: ABI {h.hv_abi_version()} != {ABI_VERSION}: rebuild the library")
        _lib = h
    return _lib


class HVError(RuntimeError):
    pass


def check(rc):
    """Map an HV_* status onto the reference's exception types."""
    if rc == HV_OK:
        return
    msg = lib().hv_last_error().decode(errors="replace")
    if rc in (HV_ERR_INVALID, HV_ERR_DEGENERATE):
        raise ValueError(msg)
    if rc == HV_ERR_NONCONFORMING:
        raise RuntimeError(msg)
    if rc == HV_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise HVError(f"hv_b200 error {rc}: {msg}")


def ptr(a):
    """Data pointer of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


def stream_handle(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def exported_symbols():
    """Names of the C-ABI functions the header declares (for the symbol test)."""
    return [n for n in _SIGS]
