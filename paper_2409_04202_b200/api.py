"""Python API over the C-ABI (same names as include/gentree_ar.h; marshalling only).

    plan = Plan.single_switch(world=8, count=n, dtype="bf16", params=p)      # GenTree
    comm = Comm.local(world=8, device=0)                                     # 8 ranks, 1 GPU
    allreduce_exec(plan, comm, buf)                                          # sm_100a kernels

Multi-process (one process per GPU, torch.distributed for the handle exchange):

    comm = Comm.from_process_group(device=local_rank)
    comm.register(tensor)                     # collective
    allreduce_exec(plan, comm, tensor)
"""
from __future__ import annotations

import ctypes
import json

from . import _lib as L
from ._lib import AR_BF16, AR_F32, GmBreakdown, GmMeasurement, GmParams, check, lib

__all__ = ["GmParams", "params", "genmodel_fit", "genmodel_fit_nvls", "genmodel_fit_row", "genmodel_closed_form", "Plan", "Comm",
           "allreduce_exec", "allreduce_exec_host", "fill_synthetic", "local_reduce",
           "rank_stride_bytes", "dtype_code"]


def dtype_code(dtype) -> int:
    if isinstance(dtype, int):
        return dtype
    if dtype in L.DTYPES:
        return L.DTYPES[dtype]
    s = str(dtype)
    if s.endswith("float32"):
        return AR_F32
    if s.endswith("bfloat16"):
        return AR_BF16
    raise ValueError(f"unsupported dtype {dtype!r}")


def params(alpha=0.0, beta=0.0, gamma=0.0, delta=0.0, epsilon=0.0, w_t=1, combined=None) -> GmParams:
    """GenModel parameters per byte (seconds, seconds/byte)."""
    p = GmParams(alpha, beta, gamma, delta, epsilon, int(w_t), 0, 0.0)
    if combined is not None:
        p.has_combined = 1
        p.combined = combined
    return p


def genmodel_fit(rows, wt_min: int, wt_max: int, link_bytes_per_s: float = 0.0):
    """rows: iterable of (n, bytes, seconds).  Returns (GmParams, sse)."""
    rows = list(rows)
    arr = (GmMeasurement * max(1, len(rows)))()
    for i, (n, b, t) in enumerate(rows):
        arr[i] = GmMeasurement(int(n), 0, int(b), float(t))
    out = GmParams()
    sse = ctypes.c_double()
    check(lib.genmodel_fit(arr, len(rows), wt_min, wt_max, float(link_bytes_per_s), ctypes.byref(out),
                           ctypes.byref(sse)))
    return out, sse.value


def genmodel_fit_nvls(rows):
    """NVLS plan row fit (reading NV1).  rows: iterable of (n, bytes, seconds).
    Returns (GmParams with alpha, beta; sse)."""
    rows = list(rows)
    arr = (GmMeasurement * max(1, len(rows)))()
    for i, (n, b, t) in enumerate(rows):
        arr[i] = GmMeasurement(int(n), 0, int(b), float(t))
    out = GmParams()
    sse = ctypes.c_double()
    check(lib.genmodel_fit_nvls(arr, len(rows), ctypes.byref(out), ctypes.byref(sse)))
    return out, sse.value


def genmodel_fit_row(kind: str, rows):
    """(α, β) of the "nvls" or "oneshot" row (genmodel_fit_row).  Returns (GmParams, sse)."""
    rows = list(rows)
    arr = (GmMeasurement * max(1, len(rows)))()
    for i, (n, b, t) in enumerate(rows):
        arr[i] = GmMeasurement(int(n), 0, int(b), float(t))
    out = GmParams()
    sse = ctypes.c_double()
    check(lib.genmodel_fit_row(kind.encode(), arr, len(rows), ctypes.byref(out), ctypes.byref(sse)))
    return out, sse.value


def genmodel_closed_form(kind: str, n: int, nbytes: int, p: GmParams) -> dict:
    out = GmBreakdown()
    check(lib.genmodel_closed_form(kind.encode(), n, nbytes, ctypes.byref(p), ctypes.byref(out)))
    return out.as_dict()


class Plan:
    """Immutable AllReduce plan (opaque gt_plan*)."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def from_topology(cls, topology_json: str, count: int, dtype="f32", params: GmParams | None = None,
                      force: str | None = None) -> "Plan":
        h = ctypes.c_void_p()
        check(lib.gentree_plan(topology_json.encode(), count, dtype_code(dtype),
                               ctypes.byref(params) if params is not None else None,
                               force.encode() if force else None, ctypes.byref(h)))
        return cls(h)

    @classmethod
    def from_topology_nvls(cls, topology_json: str, count: int, dtype, params: GmParams,
                           nvls_params: GmParams, oneshot_params: GmParams | None = None,
                           oneshot_max_bytes: int = 0, ll128_params: GmParams | None = None,
                           ll128_max_bytes: int = 0, ll128_min_bytes: int = 0) -> "Plan":
        """GenTree with the NVLS kind as a candidate (gentree_plan_nvls, reading NV1); the plan
        side is predicted on the row of the path the executor takes (LL128, one-shot, steps;
        cut-offs as default_paths() / Comm.paths())."""
        h = ctypes.c_void_p()
        check(lib.gentree_plan_nvls(topology_json.encode(), count, dtype_code(dtype), ctypes.byref(params),
                                    ctypes.byref(nvls_params),
                                    ctypes.byref(oneshot_params) if oneshot_params is not None else None,
                                    int(oneshot_max_bytes),
                                    ctypes.byref(ll128_params) if ll128_params is not None else None,
                                    int(ll128_min_bytes), int(ll128_max_bytes), ctypes.byref(h)))
        return cls(h)

    @property
    def switch_reduce(self) -> bool:
        """True for an NVLS plan (the reduce happens in the NVSwitch)."""
        return '"switch_reduce":true' in self.to_json()

    @classmethod
    def single_switch(cls, world: int, count: int, dtype="f32", params: GmParams | None = None,
                      force: str | None = None) -> "Plan":
        h = ctypes.c_void_p()
        if params is None:
            params = GmParams(1e-6, 1.0 / 900e9, 0.0, 1.0 / 6.5e12, 0.0, 64, 0, 0.0)
        check(lib.gentree_plan_single_switch(world, count, dtype_code(dtype), ctypes.byref(params),
                                             force.encode() if force else None, ctypes.byref(h)))
        return cls(h)

    @classmethod
    def from_json(cls, plan_json: str) -> "Plan":
        """Plan from canonical plan JSON (any data-movement plan; `.is_allreduce` tells)."""
        h, flag = ctypes.c_void_p(), ctypes.c_int32()
        check(lib.gt_plan_from_json(plan_json.encode(), ctypes.byref(h), ctypes.byref(flag)))
        p = cls(h)
        p.is_allreduce = bool(flag.value)
        return p

    def _str(self, fn) -> str:
        need = ctypes.c_size_t()
        fn(self._h, None, 0, ctypes.byref(need))
        buf = ctypes.create_string_buffer(need.value)
        check(fn(self._h, buf, need.value, None))
        return buf.value.decode()

    def to_json(self) -> str:
        return self._str(lib.gt_plan_to_json)

    def report(self) -> list:
        return json.loads(self._str(lib.gt_plan_report_json))

    def lowering(self) -> dict:
        """Device step tables allreduce_exec runs for this plan (host-only inspection)."""
        return json.loads(self._str(lib.ar_plan_lowering_json))

    def info(self) -> dict:
        n, s, c, d = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_uint64(), ctypes.c_int32()
        check(lib.gt_plan_info(self._h, ctypes.byref(n), ctypes.byref(s), ctypes.byref(c), ctypes.byref(d)))
        return {"n": n.value, "steps": s.value, "count": c.value, "dtype": d.value}

    def predict(self, params: GmParams | None = None) -> dict:
        out = GmBreakdown()
        check(lib.genmodel_predict(self._h, ctypes.byref(params) if params is not None else None,
                                   ctypes.byref(out)))
        return out.as_dict()

    def predict_executed(self, params: GmParams) -> dict:
        """GenModel of the lowered (fused, full-duplex) step structure the executor runs."""
        out = GmBreakdown()
        check(lib.genmodel_predict_executed(self._h, ctypes.byref(params), ctypes.byref(out)))
        return out.as_dict()

    def predict_executed_shared(self, params: GmParams) -> dict:
        """Executed-plan GenModel with all ranks on one GPU (reading A6e)."""
        out = GmBreakdown()
        check(lib.genmodel_predict_executed_shared(self._h, ctypes.byref(params), ctypes.byref(out)))
        return out.as_dict()

    def simulate(self, params: GmParams | None = None, topology_json: str | None = None) -> dict:
        """Incast-aware flow-level simulation (gt_plan_simulate; NEXT #2), on the plan's own
        topology or on `topology_json`.  Adds "steps"."""
        out = GmBreakdown()
        n = ctypes.c_size_t()
        pp = ctypes.byref(params) if params is not None else None
        doc = topology_json.encode() if topology_json is not None else None
        check(lib.gt_plan_simulate(self._h, doc, pp, ctypes.byref(out), None, 0, ctypes.byref(n)))
        steps = (ctypes.c_double * max(1, n.value))()
        check(lib.gt_plan_simulate(self._h, doc, pp, ctypes.byref(out), steps, n.value, None))
        d = out.as_dict()
        d["steps"] = list(steps)[: n.value]
        return d

    def choose_nvls(self, params: GmParams, nvls_params: GmParams) -> dict:
        """GenModel's plan-vs-NVLS choice at this plan's (n, bytes) (genmodel_choose_nvls)."""
        use = ctypes.c_int32()
        tp, tn = ctypes.c_double(), ctypes.c_double()
        check(lib.genmodel_choose_nvls(self._h, ctypes.byref(params), ctypes.byref(nvls_params), ctypes.byref(use),
                                       ctypes.byref(tp), ctypes.byref(tn)))
        return {"use_nvls": bool(use.value), "t_plan": tp.value, "t_nvls": tn.value}

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            lib.gt_plan_free(h)


def rank_stride_bytes(count: int, dtype) -> int:
    return int(lib.ar_rank_stride_bytes(count, dtype_code(dtype)))


def _ptr(x) -> int:
    if isinstance(x, int):
        return x
    return int(x.data_ptr())


class Comm:
    """Communicator (opaque ar_comm*)."""

    def __init__(self, handle, world: int, rank: int, local: bool, device: int, nproc: int | None = None,
                 ranks_per_proc: int = 1):
        self._h = handle
        self.world, self.rank, self.local, self.device = world, rank, local, device
        self.ranks_per_proc = ranks_per_proc
        self.nproc = world // ranks_per_proc if nproc is None else nproc

    @classmethod
    def create(cls, rank: int, world: int, device: int) -> "Comm":
        h = ctypes.c_void_p()
        check(lib.ar_comm_create(rank, world, device, ctypes.byref(h)))
        return cls(h, world, rank, False, device)

    @classmethod
    def create_multi(cls, proc: int, nproc: int, ranks_per_proc: int, device: int) -> "Comm":
        """ranks_per_proc consecutive ranks per process (ar_comm_create_multi; NEXT #3)."""
        h = ctypes.c_void_p()
        check(lib.ar_comm_create_multi(proc, nproc, ranks_per_proc, device, ctypes.byref(h)))
        return cls(h, nproc * ranks_per_proc, proc * ranks_per_proc, False, device, nproc, ranks_per_proc)

    @classmethod
    def local(cls, world: int, device: int = 0) -> "Comm":
        h = ctypes.c_void_p()
        check(lib.ar_comm_create_local(world, device, ctypes.byref(h)))
        return cls(h, world, 0, True, device)

    @classmethod
    def from_process_group(cls, device: int, group=None) -> "Comm":
        import torch.distributed as dist
        return cls.create(dist.get_rank(group), dist.get_world_size(group), device)

    def set_ctas(self, ctas: int):
        check(lib.ar_comm_set_ctas(self._h, ctas))

    def export(self, buf, nbytes: int | None = None) -> bytes:
        if nbytes is None:
            nbytes = buf.numel() * buf.element_size()
        blob = ctypes.create_string_buffer(L.AR_BLOB_BYTES)
        check(lib.ar_comm_register(self._h, _ptr(buf), nbytes, blob))
        return blob.raw

    def open_peers(self, blobs: list):
        assert len(blobs) == self.nproc
        data = b"".join(blobs)
        check(lib.ar_comm_open_peers(self._h, data))

    def register(self, tensor, group=None):
        """Collective over torch.distributed: export + all_gather_object + open_peers."""
        import torch.distributed as dist
        blob = self.export(tensor)
        blobs = [None] * self.nproc
        dist.all_gather_object(blobs, blob, group=group)
        self.open_peers(blobs)

    def attach_nvls(self, nvls: "Nvls"):
        """Run NVLS plans on this comm with `nvls`'s buffer (ar_comm_attach_nvls)."""
        check(lib.ar_comm_attach_nvls(self._h, nvls._h))
        self._nvls = nvls

    def set_trace(self, enable: bool = True):
        check(lib.ar_comm_set_trace(self._h, 1 if enable else 0))

    def read_trace(self):
        """globaltimer stamps (ns) of the last call: array [local ranks, ctas, slots]."""
        import numpy as np
        n, slots, ctas = ctypes.c_size_t(), ctypes.c_int32(), ctypes.c_int32()
        lib.ar_comm_read_trace(self._h, None, 0, ctypes.byref(n), ctypes.byref(slots), ctypes.byref(ctas))
        out = np.zeros(n.value, dtype=np.uint64)
        check(lib.ar_comm_read_trace(self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), n.value,
                                     None, None, None))
        return out.reshape(-1, ctas.value, slots.value)

    def async_error(self):
        check(lib.ar_comm_get_async_error(self._h))

    def paths(self) -> dict:
        """The communicator's path cut-offs (ar_comm_get_paths), bytes per rank."""
        a, b, c = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        check(lib.ar_comm_get_paths(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return {"oneshot_max": a.value, "ll128_min": b.value, "ll128_max": c.value}

    def set_oneshot_max(self, nbytes: int):
        """Cut-off of the one-shot small-message path (ar_comm_set_oneshot_max)."""
        check(lib.ar_comm_set_oneshot_max(self._h, int(nbytes)))

    def last_kernel(self) -> str:
        return lib.ar_comm_last_kernel(self._h).decode()

    def last_launch_count(self) -> int:
        k = ctypes.c_int32()
        check(lib.ar_comm_last_launch_count(self._h, ctypes.byref(k)))
        return k.value

    @property
    def handle(self):
        return self._h

    def destroy(self):
        h, self._h = self._h, None
        if h:
            lib.ar_comm_destroy(h)

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


class _CudaArray:
    """__cuda_array_interface__ wrapper so torch can view library-owned device memory."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}


class Nvls:
    """NVLS (in-switch reduction) buffer of `nbytes` per rank over torch.distributed (collective
    construction; see include/gentree_ar.h "NVLS plan kind").  `.tensor` is this rank's buffer."""

    def __init__(self, nbytes: int, device: int, group=None):
        import torch
        import torch.distributed as dist
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.device, self.nbytes = device, nbytes
        h = ctypes.c_void_p()
        blob = ctypes.create_string_buffer(L.AR_BLOB_BYTES)
        check(lib.ar_nvls_create(self.rank, self.world, device, nbytes, ctypes.byref(h), blob))
        self._h = h
        blobs = [None] * self.world
        dist.all_gather_object(blobs, blob.raw, group=group)
        check(lib.ar_nvls_attach(self._h, b"".join(blobs)))
        dist.barrier(group=group)
        ptr = ctypes.c_void_p()
        check(lib.ar_nvls_bind(self._h, ctypes.byref(ptr)))
        dist.barrier(group=group)
        self.ptr = ptr.value
        self.tensor = torch.as_tensor(_CudaArray(self.ptr, nbytes), device=f"cuda:{device}")

    def allreduce(self, count: int, dtype, stream=None):
        check(lib.allreduce_exec_nvls(self._h, count, dtype_code(dtype), _stream(stream)))

    def async_error(self):
        check(lib.ar_nvls_get_async_error(self._h))

    def destroy(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            lib.ar_nvls_destroy(h)

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def _stream(stream) -> int | None:
    if stream is None:
        try:
            import torch
            return int(torch.cuda.current_stream().cuda_stream) or None
        except Exception:
            return None
    if isinstance(stream, int):
        return stream or None
    return int(stream.cuda_stream) or None


class Executor:
    """allreduce_exec(plan, comm, buf) with the arguments marshalled once, for repeated calls
    (e.g. every training step, or inside torch.cuda.graph capture: the kernel launch carries no
    per-call host state, the call epoch lives on the device)."""

    def __init__(self, plan: Plan, comm: Comm, buf, stream=None, op: str = "sum", movement: bool = False):
        info = plan.info()
        self._keep = (plan, comm, buf)
        if movement:   # data-movement probe plan (ar_exec_movement_plan)
            self._args = (plan.handle, comm.handle, ctypes.c_void_p(_ptr(buf)), info["count"], info["dtype"],
                          ctypes.c_void_p(_stream(stream)))
            self._f = lib.ar_exec_movement_plan
            return
        self._args = (plan.handle, comm.handle, ctypes.c_void_p(_ptr(buf)), info["count"], info["dtype"],
                      OPS[op], ctypes.c_void_p(_stream(stream)))
        self._f = lib.allreduce_exec_op

    def __call__(self):
        rc = self._f(*self._args)
        if rc:
            check(rc)


OPS = {"sum": 0, "avg": 1}


def default_paths(world: int) -> dict:
    """Default path cut-offs of a one-rank-per-GPU communicator of `world` ranks
    (ar_default_paths), bytes per rank."""
    a, b, c = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    check(lib.ar_default_paths(world, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
    return {"oneshot_max": a.value, "ll128_min": b.value, "ll128_max": c.value}


def allreduce_exec(plan: Plan, comm: Comm, buf, count: int | None = None, dtype=None, stream=None, op: str = "sum"):
    """In-place AllReduce of `buf` (torch tensor or device pointer) with `plan`; op "sum" or
    "avg" (allreduce_exec_op, reading AV1)."""
    info = None
    if count is None or dtype is None:
        info = plan.info()
    count = info["count"] if count is None else count
    dt = info["dtype"] if dtype is None else dtype_code(dtype)
    if comm.local and not isinstance(buf, int):   # world rank buffers at the emulated stride
        need = rank_stride_bytes(count, dt) * (comm.world - 1) + count * (2 if dt == AR_BF16 else 4)
        if buf.numel() * buf.element_size() < need:
            raise ValueError(f"buffer holds {buf.numel() * buf.element_size()} bytes; an emulated "
                             f"communicator of {comm.world} ranks needs {need}")
    if op == "sum":
        check(lib.allreduce_exec(plan.handle, comm.handle, _ptr(buf), count, dt, _stream(stream)))
    else:
        check(lib.allreduce_exec_op(plan.handle, comm.handle, _ptr(buf), count, dt, OPS[op], _stream(stream)))


def allreduce_exec_host(plan: Plan, comm: Comm, dbuf, host_ptr: int, count: int, dtype, stream=None):
    check(lib.allreduce_exec_host(plan.handle, comm.handle, _ptr(dbuf), host_ptr, count, dtype_code(dtype),
                                  _stream(stream)))


def fill_synthetic(buf, count: int, dtype, seed: int, rank: int, mode: int = 0, start: int = 0, stream=None):
    check(lib.ar_fill_synthetic(_ptr(buf), count, dtype_code(dtype), seed, rank, mode, start, _stream(stream)))


def local_reduce(inputs, out, count: int, dtype, stream=None):
    arr = (ctypes.c_void_p * len(inputs))(*[_ptr(x) for x in inputs])
    check(lib.ar_local_reduce(arr, len(inputs), _ptr(out), count, dtype_code(dtype), _stream(stream)))
