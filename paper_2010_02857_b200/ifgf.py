"""Thin ctypes binding of libifgf.so (include/ifgf.h).

Argument marshalling only: every step of the IFGF path runs in the library's
CUDA kernels.  PyTorch supplies device memory, streams and (for multi-GPU) the
``torch.distributed`` broadcast of the NCCL unique id; the all-reduce of the
ranks' partial fields runs inside ``ifgf_apply`` on a communicator the library
creates (``NcclComm``).  There is no CPU fallback -- importing this module on a
box without the built library raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libifgf.so")

IFGF_STAGE_NEAR, IFGF_STAGE_COUSIN, IFGF_STAGE_UPWARD, IFGF_STAGE_ALL = 1, 2, 4, 7
MAX_LEVELS = 22
NUM_KCLASS = 7
KCLASS_NAMES = ["permute", "near", "s2c", "fit", "cousin", "upward", "unpermute"]

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libifgf.so not built ({LIB_PATH}); run __graft_entry__.build()")

_lib = ctypes.CDLL(LIB_PATH)


class IfgfOpts(ctypes.Structure):
    _fields_ = [
        ("leaf_ns", ctypes.c_int), ("leaf_nc", ctypes.c_int),
        ("has_root", ctypes.c_int), ("root_center", ctypes.c_double * 3), ("root_side", ctypes.c_double),
        ("stage_mask", ctypes.c_uint), ("device", ctypes.c_int),
        ("rank", ctypes.c_int), ("nranks", ctypes.c_int),
        ("nccl_comm", ctypes.c_void_p), ("no_graph", ctypes.c_int),
        ("reserved", ctypes.c_int * 7),
    ]


_L1 = MAX_LEVELS + 1


class IfgfStats(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("levels", ctypes.c_int), ("P_s", ctypes.c_int), ("P_ang", ctypes.c_int), ("P", ctypes.c_int),
        ("k", ctypes.c_double), ("root_center", ctypes.c_double * 3), ("root_side", ctypes.c_double),
        ("owned_leaf_begin", ctypes.c_int64), ("owned_leaf_end", ctypes.c_int64),
        ("nbox", ctypes.c_int64 * _L1), ("nseg", ctypes.c_int64 * _L1),
        ("ns", ctypes.c_int * _L1), ("nC", ctypes.c_int * _L1),
        ("near_pairs", ctypes.c_int64), ("s2c_pairs", ctypes.c_int64),
        ("cousin_evals", ctypes.c_int64 * _L1), ("upward_evals", ctypes.c_int64 * _L1),
        ("segment_bytes", ctypes.c_int64 * _L1),
        ("plan_device_bytes", ctypes.c_int64), ("plan_ms", ctypes.c_double),
        ("upward_kernel", ctypes.c_int * _L1),
        ("owned_morton_begin", ctypes.c_uint64), ("owned_morton_end", ctypes.c_uint64),
        ("graph_applies", ctypes.c_int64),
        ("partition_weight_total", ctypes.c_double), ("partition_weight_owned", ctypes.c_double),
    ]


_c_p, _c_i, _c_i64, _c_d = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
_SIGS = {
    "ifgf_opts_init": ([ctypes.POINTER(IfgfOpts)], _c_i),
    "ifgf_plan": ([_c_p, _c_i64, _c_d, _c_i, _c_i, _c_i, ctypes.POINTER(IfgfOpts), ctypes.POINTER(_c_p)], _c_i),
    "ifgf_apply": ([_c_p, _c_p, _c_p, _c_p], _c_i),
    "ifgf_apply_host": ([_c_p, _c_p, _c_p, _c_p], _c_i),
    "ifgf_plan_destroy": ([_c_p], _c_i),
    "ifgf_plan_stats": ([_c_p, ctypes.POINTER(IfgfStats)], _c_i),
    "ifgf_plan_level_segments": ([_c_p, _c_i, _c_p, _c_i64, ctypes.POINTER(_c_i64)], _c_i),
    "ifgf_profile_enable": ([_c_p, _c_i], _c_i),
    "ifgf_profile_read": ([_c_p, _c_p, _c_p, _c_i], _c_i),
    "ifgf_direct": ([_c_p, _c_i64, _c_d, _c_p, _c_p, _c_i64, _c_p, _c_p], _c_i),
    "ifgf_partition": ([_c_p, _c_i64, _c_i, _c_p], _c_i),
    "ifgf_bench_dfma": ([_c_i64, ctypes.POINTER(_c_d), ctypes.POINTER(_c_d), _c_p], _c_i),
    "ifgf_bench_dmma": ([_c_i64, ctypes.POINTER(_c_d), ctypes.POINTER(_c_d), _c_p], _c_i),
    "ifgf_status_string": ([_c_i], ctypes.c_char_p),
    "ifgf_last_error_message": ([], ctypes.c_char_p),
    "ifgf_version": ([], ctypes.c_char_p),
    "ifgf_debug_level_pass": ([_c_p, _c_i, _c_p, ctypes.c_uint, _c_p, _c_p], _c_i),
    "ifgf_nccl_unique_id": ([_c_p], _c_i),
    "ifgf_nccl_comm_create": ([_c_p, _c_i, _c_i, _c_i, ctypes.POINTER(_c_p)], _c_i),
    "ifgf_nccl_comm_destroy": ([_c_p], _c_i),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_SIGS)


class IfgfError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        msg = _lib.ifgf_last_error_message().decode()
        super().__init__(f"{where}: {_lib.ifgf_status_string(code).decode()}: {msg}")


def _check(code: int, where: str):
    if code != 0:
        raise IfgfError(code, where)


def _stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _f64_cuda(x: torch.Tensor, name: str) -> torch.Tensor:
    if not (isinstance(x, torch.Tensor) and x.is_cuda):
        raise TypeError(f"{name} must be a CUDA tensor")
    if x.dtype != torch.float64:
        raise TypeError(f"{name} must be float64")
    return x.contiguous()


def _c128_cuda(x: torch.Tensor, name: str) -> torch.Tensor:
    if not (isinstance(x, torch.Tensor) and x.is_cuda):
        raise TypeError(f"{name} must be a CUDA tensor")
    if x.dtype != torch.complex128:
        raise TypeError(f"{name} must be complex128")
    return x.contiguous()


class NcclComm:
    """An NCCL communicator created by the library (ifgf_nccl_comm_create) from a
    unique id that rank 0 draws and ``torch.distributed`` broadcasts; passed to
    ``Plan(comm=...)`` it makes ``apply`` return the full field on every rank
    (in-library ncclAllReduce of the partial fields)."""

    ID_BYTES = 128

    def __init__(self, nranks: int, rank: int, device: int, unique_id: bytes):
        if len(unique_id) != self.ID_BYTES:
            raise ValueError("unique_id must be 128 bytes")
        self.nranks, self.rank, self.device = int(nranks), int(rank), int(device)
        buf = ctypes.create_string_buffer(bytes(unique_id), self.ID_BYTES)
        h = ctypes.c_void_p()
        _check(_lib.ifgf_nccl_comm_create(buf, self.nranks, self.rank, self.device, ctypes.byref(h)),
               "ifgf_nccl_comm_create")
        self._h = h

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(NcclComm.ID_BYTES)
        _check(_lib.ifgf_nccl_unique_id(buf), "ifgf_nccl_unique_id")
        return buf.raw

    @classmethod
    def from_group(cls, group=None, device: int | None = None) -> "NcclComm":
        """Collective over a torch.distributed group (any backend): rank 0's unique
        id is broadcast with broadcast_object_list."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        dev = torch.cuda.current_device() if device is None else int(device)
        return cls(world, rank, dev, obj[0])

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.ifgf_nccl_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Plan:
    """IFGF plan: ``ifgf_plan(points, k, levels, P_s, P_ang)`` (C ABI).

    points: float64 [N, 3] CUDA tensor.  ``rank``/``nranks`` select this
    process's source partition; with ``comm`` (an ``NcclComm`` of the nranks
    processes) ``apply`` returns the full field on every rank, without it this
    rank's partial field.  ``graph=False`` launches the kernels one by one
    instead of replaying the plan's CUDA graph.
    """

    def __init__(self, points: torch.Tensor, k: float, levels: int, P_s: int = 3, P_ang: int = 5, *,
                 leaf_ns: int = 0, leaf_nc: int = 0, root=None, stage_mask: int = 0, rank: int = 0,
                 nranks: int = 1, comm: NcclComm | None = None, graph: bool = True):
        pts = _f64_cuda(points, "points")
        if pts.dim() != 2 or pts.shape[1] != 3:
            raise ValueError("points must be [N, 3]")
        self.n = int(pts.shape[0])
        self.device = pts.device
        self.comm = comm  # borrowed by the library plan: keep it alive as long as the plan
        o = IfgfOpts()
        _check(_lib.ifgf_opts_init(ctypes.byref(o)), "ifgf_opts_init")
        o.leaf_ns, o.leaf_nc = int(leaf_ns), int(leaf_nc)
        if root is not None:
            o.has_root = 1
            for a in range(3):
                o.root_center[a] = float(root[0][a])
            o.root_side = float(root[1])
        o.stage_mask = int(stage_mask)
        o.device = pts.device.index if pts.device.index is not None else torch.cuda.current_device()
        o.rank, o.nranks = int(rank), int(nranks)
        o.nccl_comm = comm.handle.value if comm is not None else None
        o.no_graph = 0 if graph else 1
        h = ctypes.c_void_p()
        _check(_lib.ifgf_plan(pts.data_ptr(), self.n, float(k), int(levels), int(P_s), int(P_ang), ctypes.byref(o),
                              ctypes.byref(h)), "ifgf_plan")
        self._h = h
        self.k, self.levels, self.P_s, self.P_ang = float(k), int(levels), int(P_s), int(P_ang)

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.ifgf_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check_dev(self, x: torch.Tensor, name: str):
        if x.device != self.device:
            raise ValueError(f"{name} is on {x.device}, the plan on {self.device}")

    def apply(self, a: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """out = I(a) (complex128 [N] CUDA tensors on the plan's device, caller's
        point order), enqueued on ``stream`` (default: the current stream)."""
        a = _c128_cuda(a, "densities")
        self._check_dev(a, "densities")
        if a.shape != (self.n,):
            raise ValueError("densities must be [N]")
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        if out is None:
            with torch.cuda.stream(s):
                out = torch.empty(self.n, dtype=torch.complex128, device=self.device)
        elif not out.is_contiguous() or out.dtype != torch.complex128 or out.shape != (self.n,):
            raise ValueError("out must be a contiguous complex128 [N] tensor")
        self._check_dev(out, "out")
        if s != torch.cuda.current_stream(self.device):
            a.record_stream(s)  # the contiguous copy (if any) lives until the library's work on s is done
            out.record_stream(s)
        _check(_lib.ifgf_apply(self._h, a.data_ptr(), out.data_ptr(), s.cuda_stream), "ifgf_apply")
        return out

    def apply_host(self, a_host: np.ndarray | torch.Tensor, out_host=None, stream=None):
        """End-to-end apply from host buffers (ifgf_apply_host): H2D, apply, D2H, sync.
        a_host / out_host: complex128 [N] host arrays (numpy or CPU tensors; pinned
        memory is faster)."""
        def host_buf(x, name):
            if isinstance(x, torch.Tensor):
                if x.is_cuda or x.dtype != torch.complex128 or x.shape != (self.n,) or not x.is_contiguous():
                    raise ValueError(f"{name} must be a contiguous complex128 [N] host tensor")
                return x, x.data_ptr()
            x = np.asarray(x)
            if x.dtype != np.complex128 or x.shape != (self.n,) or not x.flags.c_contiguous:
                raise ValueError(f"{name} must be a contiguous complex128 [N] array")
            return x, x.ctypes.data
        a, ptr = host_buf(a_host, "densities")
        if out_host is None:
            out_host = torch.empty(self.n, dtype=torch.complex128, pin_memory=True)
        if isinstance(out_host, np.ndarray) and not out_host.flags.writeable:
            raise ValueError("out must be writeable")
        out_host, optr = host_buf(out_host, "out")
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        _check(_lib.ifgf_apply_host(self._h, ptr, optr, s.cuda_stream), "ifgf_apply_host")
        return out_host

    def stats(self) -> dict:
        s = IfgfStats()
        _check(_lib.ifgf_plan_stats(self._h, ctypes.byref(s)), "ifgf_plan_stats")
        D = s.levels
        lv = range(1, D + 1)
        return dict(
            n=s.n, levels=D, P_s=s.P_s, P_ang=s.P_ang, P=s.P, k=s.k,
            root_center=list(s.root_center), root_side=s.root_side,
            owned_leaf_range=(s.owned_leaf_begin, s.owned_leaf_end),
            owned_morton_range=(s.owned_morton_begin, s.owned_morton_end),
            nbox={d: s.nbox[d] for d in lv}, nseg={d: s.nseg[d] for d in lv},
            grid={d: (s.ns[d], s.nC[d]) for d in lv},
            near_pairs=s.near_pairs, s2c_pairs=s.s2c_pairs,
            cousin_evals={d: s.cousin_evals[d] for d in lv}, upward_evals={d: s.upward_evals[d] for d in lv},
            segment_bytes={d: s.segment_bytes[d] for d in lv},
            plan_device_bytes=s.plan_device_bytes, plan_ms=s.plan_ms,
            upward_kernel={d: s.upward_kernel[d] for d in lv},
            graph_applies=s.graph_applies,
            partition_weight=(s.partition_weight_owned, s.partition_weight_total),
        )

    def level_segments(self, d: int) -> np.ndarray:
        cnt = ctypes.c_int64()
        _check(_lib.ifgf_plan_level_segments(self._h, d, None, 0, ctypes.byref(cnt)), "ifgf_plan_level_segments")
        out = np.zeros((cnt.value, 4), dtype=np.int64)
        if cnt.value:
            _check(_lib.ifgf_plan_level_segments(self._h, d, out.ctypes.data, cnt.value, ctypes.byref(cnt)),
                   "ifgf_plan_level_segments")
        return out

    def debug_level_pass(self, d: int, values: np.ndarray, cousin: bool = True, upward: bool = True):
        """Test hook (ifgf_debug_level_pass): K5 + K6 and/or K7 of level d alone on
        the given node values (complex128 [nseg_d, P], plan segment order).
        Returns (field [N] or None, parent coefficients [nseg_{d-1}, P] or None)."""
        st = self.stats()
        v = np.ascontiguousarray(values, dtype=np.complex128)
        if v.shape != (st["nseg"][d], st["P"]):
            raise ValueError("values must be [nseg_d, P]")
        what = (1 if cousin else 0) | (2 if upward and d > 3 else 0)
        field = np.zeros(self.n, dtype=np.complex128) if cousin else None
        parent = np.zeros((st["nseg"][d - 1], st["P"]), dtype=np.complex128) if what & 2 else None
        _check(_lib.ifgf_debug_level_pass(self._h, int(d), v.ctypes.data, what,
                                          field.ctypes.data if field is not None else None,
                                          parent.ctypes.data if parent is not None else None),
               "ifgf_debug_level_pass")
        return field, parent

    def profile_enable(self, on: bool = True):
        _check(_lib.ifgf_profile_enable(self._h, 1 if on else 0), "ifgf_profile_enable")

    def profile_read(self, reset: bool = True) -> dict:
        ms = np.zeros(NUM_KCLASS)
        ln = np.zeros(NUM_KCLASS, dtype=np.int64)
        _check(_lib.ifgf_profile_read(self._h, ms.ctypes.data, ln.ctypes.data, 1 if reset else 0),
               "ifgf_profile_read")
        return {KCLASS_NAMES[c]: (float(ms[c]), int(ln[c])) for c in range(NUM_KCLASS)}


def direct(points: torch.Tensor, k: float, a: torch.Tensor, targets: torch.Tensor, stream=None) -> torch.Tensor:
    """GPU direct sum at target indices (measurement harness; eq. field1)."""
    pts = _f64_cuda(points, "points")
    a = _c128_cuda(a, "densities")
    t = targets.to(device=pts.device, dtype=torch.int64).contiguous()
    out = torch.empty(t.shape[0], dtype=torch.complex128, device=pts.device)
    _check(_lib.ifgf_direct(pts.data_ptr(), pts.shape[0], float(k), a.data_ptr(), t.data_ptr(), t.shape[0],
                            out.data_ptr(), _stream_ptr(stream)), "ifgf_direct")
    return out


def partition(weights, nranks: int) -> np.ndarray:
    """Host-only work-weighted contiguous partition (ifgf_partition)."""
    w = np.ascontiguousarray(weights, dtype=np.float64)
    b = np.zeros(nranks + 1, dtype=np.int64)
    _check(_lib.ifgf_partition(w.ctypes.data, w.shape[0], int(nranks), b.ctypes.data), "ifgf_partition")
    return b


def bench_dfma(iters: int = 20000, stream=None):
    """Measured FP64 FMA throughput (FLOP/s) and kernel ms on the current device."""
    f, ms = ctypes.c_double(), ctypes.c_double()
    _check(_lib.ifgf_bench_dfma(int(iters), ctypes.byref(f), ctypes.byref(ms), _stream_ptr(stream)),
           "ifgf_bench_dfma")
    return f.value, ms.value


def bench_dmma(iters: int = 20000, stream=None):
    """Measured FP64 tensor-core (DMMA m8n8k4) throughput (FLOP/s) and kernel ms."""
    f, ms = ctypes.c_double(), ctypes.c_double()
    _check(_lib.ifgf_bench_dmma(int(iters), ctypes.byref(f), ctypes.byref(ms), _stream_ptr(stream)),
           "ifgf_bench_dmma")
    return f.value, ms.value


def version() -> str:
    return _lib.ifgf_version().decode()
