"""ctypes binding of include/gentree_ar.h — argument marshalling only.

Every computation happens inside `libgentree_ar.so` (host planning core + sm_100a kernels).
There is no Python or CPU fallback: if the library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgentree_ar.so")

AR_OK, AR_EINVAL, AR_ESYS = 0, 1, 2
AR_F32, AR_BF16 = 0, 1
AR_MAX_RANKS = 64
AR_BLOB_BYTES = 512
DTYPES = {"f32": AR_F32, "bf16": AR_BF16}
ESIZE = {AR_F32: 4, AR_BF16: 2}

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2409_04202_b200.build` "
                      "(or __graft_entry__.build()); there is no fallback implementation")

lib = ctypes.CDLL(LIB_PATH)


class ArError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{ {1: 'AR_EINVAL', 2: 'AR_ESYS'}.get(code, code)}] {msg}")
        self.code = code


class ArInvalid(ArError, ValueError):
    pass


class GmParams(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_double), ("beta", ctypes.c_double), ("gamma", ctypes.c_double),
                ("delta", ctypes.c_double), ("epsilon", ctypes.c_double), ("w_t", ctypes.c_int32),
                ("has_combined", ctypes.c_int32), ("combined", ctypes.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class GmBreakdown(ctypes.Structure):
    _fields_ = [(k, ctypes.c_double) for k in ("latency", "bandwidth", "compute", "memory", "incast", "total")]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class GmMeasurement(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("reserved", ctypes.c_int32), ("bytes", ctypes.c_uint64),
                ("seconds", ctypes.c_double)]


P = ctypes.c_void_p
I32 = ctypes.c_int32
U64 = ctypes.c_uint64
SZ = ctypes.c_size_t

_SIGS = {
    "ar_last_error": (ctypes.c_char_p, []),
    "ar_version": (ctypes.c_char_p, []),
    "genmodel_fit": (I32, [ctypes.POINTER(GmMeasurement), SZ, I32, I32, ctypes.c_double,
                           ctypes.POINTER(GmParams), ctypes.POINTER(ctypes.c_double)]),
    "genmodel_fit_nvls": (I32, [ctypes.POINTER(GmMeasurement), SZ, ctypes.POINTER(GmParams),
                                ctypes.POINTER(ctypes.c_double)]),
    "genmodel_fit_row": (I32, [ctypes.c_char_p, ctypes.POINTER(GmMeasurement), SZ, ctypes.POINTER(GmParams),
                               ctypes.POINTER(ctypes.c_double)]),
    "genmodel_choose_nvls": (I32, [P, ctypes.POINTER(GmParams), ctypes.POINTER(GmParams), ctypes.POINTER(I32),
                                   ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
    "gt_plan_simulate": (I32, [P, ctypes.c_char_p, ctypes.POINTER(GmParams), ctypes.POINTER(GmBreakdown),
                               ctypes.POINTER(ctypes.c_double), SZ, ctypes.POINTER(SZ)]),
    "genmodel_closed_form": (I32, [ctypes.c_char_p, I32, U64, ctypes.POINTER(GmParams),
                                   ctypes.POINTER(GmBreakdown)]),
    "gentree_plan": (I32, [ctypes.c_char_p, U64, I32, ctypes.POINTER(GmParams), ctypes.c_char_p,
                           ctypes.POINTER(P)]),
    "gentree_plan_single_switch": (I32, [I32, U64, I32, ctypes.POINTER(GmParams), ctypes.c_char_p,
                                         ctypes.POINTER(P)]),
    "gt_plan_to_json": (I32, [P, ctypes.c_char_p, SZ, ctypes.POINTER(SZ)]),
    "gt_plan_report_json": (I32, [P, ctypes.c_char_p, SZ, ctypes.POINTER(SZ)]),
    "gt_plan_info": (I32, [P, ctypes.POINTER(I32), ctypes.POINTER(I32), ctypes.POINTER(U64),
                           ctypes.POINTER(I32)]),
    "genmodel_predict": (I32, [P, ctypes.POINTER(GmParams), ctypes.POINTER(GmBreakdown)]),
    "gt_plan_free": (None, [P]),
    "gt_plan_from_json": (I32, [ctypes.c_char_p, ctypes.POINTER(P), ctypes.POINTER(I32)]),
    "genmodel_predict_executed": (I32, [P, ctypes.POINTER(GmParams), ctypes.POINTER(GmBreakdown)]),
    "genmodel_predict_executed_shared": (I32, [P, ctypes.POINTER(GmParams), ctypes.POINTER(GmBreakdown)]),
    "ar_comm_create": (I32, [I32, I32, I32, ctypes.POINTER(P)]),
    "ar_comm_create_multi": (I32, [I32, I32, I32, I32, ctypes.POINTER(P)]),
    "ar_comm_create_local": (I32, [I32, I32, ctypes.POINTER(P)]),
    "ar_comm_set_ctas": (I32, [P, I32]),
    "ar_comm_register": (I32, [P, P, SZ, ctypes.c_char_p]),
    "ar_comm_open_peers": (I32, [P, ctypes.c_char_p]),
    "ar_comm_get_async_error": (I32, [P]),
    "ar_comm_destroy": (I32, [P]),
    "ar_comm_last_launch_count": (I32, [P, ctypes.POINTER(I32)]),
    "ar_plan_lowering_json": (I32, [P, ctypes.c_char_p, SZ, ctypes.POINTER(SZ)]),
    "ar_nvls_create": (I32, [I32, I32, I32, U64, ctypes.POINTER(P), ctypes.c_char_p]),
    "ar_nvls_attach": (I32, [P, ctypes.c_char_p]),
    "ar_nvls_bind": (I32, [P, ctypes.POINTER(P)]),
    "allreduce_exec_nvls": (I32, [P, U64, I32, P]),
    "ar_comm_attach_nvls": (I32, [P, P]),
    "gentree_plan_nvls": (I32, [ctypes.c_char_p, U64, I32, ctypes.POINTER(GmParams), ctypes.POINTER(GmParams),
                                ctypes.POINTER(GmParams), U64, ctypes.POINTER(GmParams), U64, U64, ctypes.POINTER(P)]),
    "ar_nvls_get_async_error": (I32, [P]),
    "ar_nvls_destroy": (I32, [P]),
    "ar_comm_set_trace": (I32, [P, I32]),
    "ar_comm_read_trace": (I32, [P, ctypes.POINTER(U64), SZ, ctypes.POINTER(SZ), ctypes.POINTER(I32),
                                 ctypes.POINTER(I32)]),
    "ar_rank_stride_bytes": (U64, [U64, I32]),
    "allreduce_exec": (I32, [P, P, P, U64, I32, P]),
    "allreduce_exec_op": (I32, [P, P, P, U64, I32, I32, P]),
    "ar_exec_movement_plan": (I32, [P, P, P, U64, I32, P]),
    "ar_comm_last_kernel": (ctypes.c_char_p, [P]),
    "ar_comm_set_oneshot_max": (I32, [P, U64]),
    "ar_default_paths": (I32, [I32, ctypes.POINTER(U64), ctypes.POINTER(U64), ctypes.POINTER(U64)]),
    "ar_comm_get_paths": (I32, [P, ctypes.POINTER(U64), ctypes.POINTER(U64), ctypes.POINTER(U64)]),
    "allreduce_exec_host": (I32, [P, P, P, P, U64, I32, P]),
    "ar_fill_synthetic": (I32, [P, U64, I32, U64, I32, I32, U64, P]),
    "ar_local_reduce": (I32, [ctypes.POINTER(P), I32, P, U64, I32, P]),
}

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def exported_symbols():
    return list(_SIGS)


def check(rc: int):
    if rc != AR_OK:
        msg = lib.ar_last_error().decode(errors="replace")
        if rc == AR_EINVAL:
            raise ArInvalid(rc, msg)
        raise ArError(rc, msg)
