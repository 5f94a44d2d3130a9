"""Python binding of libqtmm (include/qt.h): argument marshalling only.

Every step of the multiply runs in the CUDA kernels of libqtmm.so; this module
turns numpy arrays / torch tensors into pointers, calls the C ABI and wraps the
handles.  There is no fallback: if libqtmm.so is missing or fails to load, the
import raises.  PyTorch is used only for streams and torch.distributed (the
NCCL unique id broadcast).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QTMM_LIB_DEV") or os.path.join(_HERE, "lib", "libqtmm.so")  # dev A/B override

QT_F64, QT_F32 = 0, 1
STATUS = {0: "QT_OK", 1: "QT_EINVAL", 2: "QT_ERANGE", 3: "QT_EDUP", 4: "QT_EDIM", 5: "QT_EBS",
          6: "QT_EDTYPE", 7: "QT_ENOMEM", 8: "QT_ECUDA", 9: "QT_ENCCL", 10: "QT_ESTATE"}
MAX_LEVELS = 40


class QtError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class Stats(ctypes.Structure):
    _fields_ = [
        ("nlevels", ctypes.c_int32),
        ("leaf_level", ctypes.c_int32),
        ("level_tasks", ctypes.c_int64 * MAX_LEVELS),
        ("level_c_nodes", ctypes.c_int64 * MAX_LEVELS),
        ("block_products", ctypes.c_int64),
        ("c_blocks", ctypes.c_int64),
        ("bytes_recv_payload", ctypes.c_int64),
        ("bytes_recv_meta", ctypes.c_int64),
        ("bytes_sent_payload", ctypes.c_int64),
        ("bytes_sent_meta", ctypes.c_int64),
        ("blocks_recv", ctypes.c_int64),
        ("ms_exchange", ctypes.c_float),
        ("ms_symbolic", ctypes.c_float),
        ("ms_numeric", ctypes.c_float),
        ("ms_total", ctypes.c_float),
        ("tiles_overlapped", ctypes.c_int64),
        ("tiles_after", ctypes.c_int64),
        ("ms_payload", ctypes.c_float),
    ]

    def as_dict(self) -> dict:
        n = self.nlevels
        d = {f: getattr(self, f) for f, _ in self._fields_ if f not in ("level_tasks", "level_c_nodes")}
        d["level_tasks"] = list(self.level_tasks[:n])
        d["level_c_nodes"] = list(self.level_c_nodes[:n])
        return d


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_1501_07800_b200.build`")
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    P, i32, i64, st = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int
    sig = {
        "qt_ctx_create": [ctypes.c_int, P, ctypes.c_int, ctypes.c_int, P, P],
        "qt_ctx_destroy": [P],
        "qt_ctx_info": [P, P, P, P, P],
        "qt_ctx_set_timing": [P, i32],
        "qt_nccl_unique_id": [P],
        "qt_create": [P, i64, i32, i32, ctypes.c_int, i64, P, P, P, P, P],
        "qt_multiply": [P, P, P, P],
        "qt_multiply_async": [P, P, P, P],
        "qt_multiply_ex": [P, P, i32, i32, P, P],
        "qt_symm_square": [P, P, P],
        "qt_multiply_screened": [P, P, ctypes.c_double, P, P],
        "qt_multiply_virtual": [P, P, i32, i32, P, P, P],
        "qt_symm_square_virtual": [P, i32, i32, P, P, P],
        "qt_plan_strips": [P, i64, i32, i32, i64, P, P, i64, P, i32, P, P],
        "qt_multiply_plan": [P, P, i32, i32, P, P, P],
        "qt_plan_execute": [P],
        "qt_symm_square_plan": [P, P, P, P],
        "qt_plan_destroy": [P],
        "qt_update_values": [P, P],
        "qt_gather": [P, i32, P, P, P, P],
        "qt_truncate": [P, ctypes.c_double, P],
        "qt_info": [P, P, P, P, P, P, P, P, P],
        "qt_level_nodes": [P, P, i32, P],
        "qt_read_back": [P, P, P, P],
        "qt_read_back_async": [P, P, P, P],
        "qt_ctx_synchronize": [P],
        "qt_destroy": [P],
        "qt_fp64_peak": [P, ctypes.c_int, ctypes.c_float, P],
        "qt_loopback_hub_create": [i32, P],
        "qt_loopback_hub_destroy": [P],
        "qt_ctx_create_loopback": [ctypes.c_int, P, ctypes.c_int, ctypes.c_int, P, P],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = st
    lib.qt_last_error.restype = ctypes.c_char_p
    lib.qt_last_error.argtypes = []
    lib.qt_kernel_launches.restype = i64
    lib.qt_kernel_launches.argtypes = [P]
    return lib


_lib = _load()
EXPORTED = ("qt_ctx_create", "qt_ctx_destroy", "qt_ctx_info", "qt_ctx_set_timing", "qt_nccl_unique_id", "qt_create", "qt_multiply",
            "qt_multiply_async",
            "qt_multiply_ex", "qt_symm_square", "qt_multiply_screened",
            "qt_multiply_virtual", "qt_symm_square_virtual", "qt_plan_strips", "qt_multiply_plan",
            "qt_symm_square_plan", "qt_plan_execute", "qt_plan_destroy", "qt_update_values", "qt_gather", "qt_truncate", "qt_info", "qt_level_nodes", "qt_read_back",
            "qt_read_back_async", "qt_ctx_synchronize", "qt_destroy", "qt_last_error", "qt_kernel_launches", "qt_fp64_peak",
            "qt_loopback_hub_create", "qt_loopback_hub_destroy", "qt_ctx_create_loopback")


def _check(status: int):
    if status != 0:
        raise QtError(status, _lib.qt_last_error().decode(errors="replace"))


def _ptr(x):
    """Pointer of a numpy array or torch tensor (must be contiguous)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return ctypes.c_void_p(x.ctypes.data)
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return ctypes.c_void_p(x.data_ptr())
    raise TypeError(f"unsupported buffer {type(x)}")


def _dtype_code(vals) -> int:
    dt = str(vals.dtype)
    if dt in ("float64", "torch.float64"):
        return QT_F64
    if dt in ("float32", "torch.float32"):
        return QT_F32
    raise TypeError(f"values must be float64 or float32, got {dt}")


class Context:
    """One per process (rank): device, stream and (world > 1) NCCL communicator."""

    def __init__(self, device: int = 0, stream=None, process_group=None, loopback=None, nccl_self=False):
        """``loopback=(hub, rank, world)``: a rank thread of the single-device
        loopback transport (testing only, see LoopbackHub).  ``nccl_self``: a
        single-rank context that still builds its own one-rank NCCL
        communicator (qt_ctx_create with world 1 and a unique id)."""
        import torch
        self.device = device
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        sptr = ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
        rank, world = 0, 1
        uid = None
        if loopback is not None:
            hub, rank, world = loopback
            h = ctypes.c_void_p()
            _check(_lib.qt_ctx_create_loopback(device, sptr, rank, world, hub.handle, ctypes.byref(h)))
            self.rank, self.world, self._h = rank, world, h
            return
        if process_group is not None or (torch.distributed.is_available() and torch.distributed.is_initialized()):
            import torch.distributed as dist
            world = dist.get_world_size(process_group)
            rank = dist.get_rank(process_group)
            if world > 1:
                buf = ctypes.create_string_buffer(128)
                if rank == 0:
                    _check(_lib.qt_nccl_unique_id(buf))
                obj = [bytes(buf.raw)]
                src = dist.get_global_rank(process_group, 0) if process_group is not None else 0
                dist.broadcast_object_list(obj, src=src, group=process_group)
                uid = ctypes.create_string_buffer(obj[0], 128)
        if nccl_self and world == 1:
            uid = ctypes.create_string_buffer(128)
            _check(_lib.qt_nccl_unique_id(uid))
        self.rank, self.world = rank, world
        h = ctypes.c_void_p()
        _check(_lib.qt_ctx_create(device, sptr, rank, world, uid, ctypes.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    @property
    def kernel_launches(self) -> int:
        return int(_lib.qt_kernel_launches(self._h))

    def info(self) -> dict:
        """qt_ctx_info: rank, world, the library communicator's rank count and transport."""
        r, w, n, t = (ctypes.c_int32() for _ in range(4))
        _check(_lib.qt_ctx_info(self._h, ctypes.byref(r), ctypes.byref(w), ctypes.byref(n), ctypes.byref(t)))
        return {"rank": r.value, "world": w.value, "comm_ranks": n.value,
                "transport": {0: "none", 1: "nccl", 2: "loopback"}[t.value]}

    def set_timing(self, on: bool):
        """qt_ctx_set_timing: CUDA-event phase timings in the stats (default on)."""
        _check(_lib.qt_ctx_set_timing(self._h, int(bool(on))))

    def synchronize(self):
        """Wait for all enqueued work, including qt_read_back_async copies."""
        _check(_lib.qt_ctx_synchronize(self._h))

    def fp64_peak(self, kind: str = "dmma", ms: float = 50.0) -> float:
        out = ctypes.c_double()
        _check(_lib.qt_fp64_peak(self._h, 0 if kind == "dmma" else 1, ms, ctypes.byref(out)))
        return out.value

    def close(self):
        if getattr(self, "_h", None):
            _check(_lib.qt_ctx_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def plan_strips(n: int, block_size: int, parts: int, a_rc, b_rows, align_rows: int = 1, ctx=None):
    """Product-balanced block-row strips of C = A·B (qt_plan_strips).
    ``a_rc`` = (brow, bcol) of A's blocks, ``b_rows`` = B's block rows; with a
    multi-rank ``ctx`` each rank passes its own blocks (collective).  Returns
    (bounds[parts+1], products per strip)."""
    ar = np.ascontiguousarray(np.asarray(a_rc[0], dtype=np.int32))
    ac = np.ascontiguousarray(np.asarray(a_rc[1], dtype=np.int32))
    br = np.ascontiguousarray(np.asarray(b_rows, dtype=np.int32))
    bounds = np.zeros(parts + 1, np.int32)
    prods = np.zeros(parts, np.int64)
    _check(_lib.qt_plan_strips(ctx.handle if ctx is not None else None, int(n), int(block_size), int(align_rows),
                               ar.shape[0], _ptr(ar) if ar.size else None, _ptr(ac) if ac.size else None,
                               br.shape[0], _ptr(br) if br.size else None, int(parts), _ptr(bounds), _ptr(prods)))
    return bounds, prods


class Plan:
    """A multiply whose numeric pass can be re-run (qt_multiply_plan)."""

    def __init__(self, ctx, handle):
        self.ctx, self._h = ctx, handle

    def execute(self):
        """Recompute C from the current values of A and B (enqueue only; CUDA-graph capturable)."""
        _check(_lib.qt_plan_execute(self._h))

    def close(self):
        if getattr(self, "_h", None):
            _check(_lib.qt_plan_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LoopbackHub:
    """Shared state of the single-device loopback transport (testing the
    multi-rank path with rank threads on one GPU)."""

    def __init__(self, world: int):
        h = ctypes.c_void_p()
        _check(_lib.qt_loopback_hub_create(world, ctypes.byref(h)))
        self.handle = h
        self.world = world

    def close(self):
        if getattr(self, "handle", None):
            _check(_lib.qt_loopback_hub_destroy(self.handle))
            self.handle = None


class Matrix:
    """Immutable quadtree matrix handle (the rank-local part when world > 1)."""

    def __init__(self, ctx: Context, handle):
        self.ctx = ctx
        self._h = handle

    @classmethod
    def from_blocks(cls, ctx: Context, n: int, leaf_dim: int, bs: int, brow, bcol, vals,
                    row_bounds=None) -> "Matrix":
        nb = int(brow.shape[0])
        if nb:
            if isinstance(brow, np.ndarray):
                brow = np.ascontiguousarray(brow, dtype=np.int32)
                bcol = np.ascontiguousarray(bcol, dtype=np.int32)
            if isinstance(vals, np.ndarray):
                vals = np.ascontiguousarray(vals)
            if tuple(vals.shape[-2:]) != (bs, bs) or int(vals.shape[0]) != nb:
                raise ValueError("vals must have shape [nblocks, bs, bs]")
        code = _dtype_code(vals) if nb or hasattr(vals, "dtype") else QT_F64
        rb = None
        if row_bounds is not None:
            rb = np.ascontiguousarray(np.asarray(row_bounds, dtype=np.int32))
        h = ctypes.c_void_p()
        _check(_lib.qt_create(ctx.handle, n, leaf_dim, bs, code, nb, _ptr(brow) if nb else None,
                              _ptr(bcol) if nb else None, _ptr(vals) if nb else None,
                              _ptr(rb), ctypes.byref(h)))
        return cls(ctx, h)

    def multiply(self, other: "Matrix", wait: bool = True):
        """C = self * other.  ``wait=False`` (qt_multiply_async): returns once
        the numeric kernel is enqueued (stats without timings)."""
        st = Stats()
        h = ctypes.c_void_p()
        fn = _lib.qt_multiply if wait else _lib.qt_multiply_async
        _check(fn(self._h, other._h, ctypes.byref(h), ctypes.byref(st)))
        return Matrix(self.ctx, h), st

    def multiply_ex(self, other: "Matrix", trans_a: bool = False, trans_b: bool = False):
        """C = op(self) op(other), op = transpose when the flag is set."""
        st = Stats()
        h = ctypes.c_void_p()
        _check(_lib.qt_multiply_ex(self._h, other._h, int(trans_a), int(trans_b), ctypes.byref(h),
                                   ctypes.byref(st)))
        return Matrix(self.ctx, h), st

    def multiply_screened(self, other: "Matrix", tau: float):
        """C~ = sum of the block products with ||A_ik|| ||B_kj|| >= tau."""
        st = Stats()
        h = ctypes.c_void_p()
        _check(_lib.qt_multiply_screened(self._h, other._h, float(tau), ctypes.byref(h), ctypes.byref(st)))
        return Matrix(self.ctx, h), st

    def symm_square(self):
        """C = A^2 for symmetric A stored as its upper block triangle; C upper."""
        st = Stats()
        h = ctypes.c_void_p()
        _check(_lib.qt_symm_square(self._h, ctypes.byref(h), ctypes.byref(st)))
        return Matrix(self.ctx, h), st

    def __matmul__(self, other: "Matrix") -> "Matrix":
        return self.multiply(other)[0]

    def multiply_virtual(self, other: "Matrix", P: int, g: int, row_bounds):
        st = Stats()
        h = ctypes.c_void_p()
        rb = np.ascontiguousarray(np.asarray(row_bounds, dtype=np.int32))
        _check(_lib.qt_multiply_virtual(self._h, other._h, P, g, _ptr(rb), ctypes.byref(h),
                                        ctypes.byref(st)))
        return Matrix(self.ctx, h), st

    def symm_square_virtual(self, P: int, g: int, row_bounds):
        """Rank g of the P-rank symmetric square, on one device (self = the whole U)."""
        st = Stats()
        h = ctypes.c_void_p()
        rb = np.ascontiguousarray(np.asarray(row_bounds, dtype=np.int32))
        _check(_lib.qt_symm_square_virtual(self._h, P, g, _ptr(rb), ctypes.byref(h), ctypes.byref(st)))
        return Matrix(self.ctx, h), st

    def multiply_plan(self, other: "Matrix", trans_a: bool = False, trans_b: bool = False):
        """C = op(A) op(B) plus a Plan that recomputes C after qt_update_values."""
        st = Stats()
        h, p = ctypes.c_void_p(), ctypes.c_void_p()
        _check(_lib.qt_multiply_plan(self._h, other._h, int(trans_a), int(trans_b), ctypes.byref(p),
                                     ctypes.byref(h), ctypes.byref(st)))
        return Plan(self.ctx, p), Matrix(self.ctx, h), st

    def gather(self, root: int = 0):
        """Collective: every rank's blocks on `root` in (brow, bcol) order
        (qt_gather); returns (brow, bcol, vals) on the root, None elsewhere."""
        total = ctypes.c_int64()
        _check(_lib.qt_gather(self._h, root, None, None, None, ctypes.byref(total)))
        n = total.value
        if self.ctx.world > 1 and self.ctx.rank != root:
            _check(_lib.qt_gather(self._h, root, None, None, None, None))
            return None
        inf = self.info()
        bs = inf["bs"]
        dt = np.float64 if inf["dtype"] == "f64" else np.float32
        out = (np.empty(n, np.int32), np.empty(n, np.int32), np.empty((n, bs, bs), dt))
        _check(_lib.qt_gather(self._h, root, _ptr(out[0]) if n else None, _ptr(out[1]) if n else None,
                              _ptr(out[2]) if n else None, None))
        return out

    def symm_square_plan(self):
        """C = A^2 (upper-triangular storage) plus a Plan that recomputes C after qt_update_values."""
        st = Stats()
        h, p = ctypes.c_void_p(), ctypes.c_void_p()
        _check(_lib.qt_symm_square_plan(self._h, ctypes.byref(p), ctypes.byref(h), ctypes.byref(st)))
        return Plan(self.ctx, p), Matrix(self.ctx, h), st

    def update_values(self, vals):
        """New values (same pattern) in to_blocks order: [nblocks, bs, bs]."""
        if isinstance(vals, np.ndarray):
            vals = np.ascontiguousarray(vals)
        _check(_lib.qt_update_values(self._h, _ptr(vals)))

    def truncate(self, tau: float) -> "Matrix":
        h = ctypes.c_void_p()
        _check(_lib.qt_truncate(self._h, float(tau), ctypes.byref(h)))
        return Matrix(self.ctx, h)

    def info(self) -> dict:
        n, nl, nglob = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        leaf, bs, lo, hi = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        dt = ctypes.c_int()
        _check(_lib.qt_info(self._h, ctypes.byref(n), ctypes.byref(leaf), ctypes.byref(bs),
                            ctypes.byref(dt), ctypes.byref(nl), ctypes.byref(nglob),
                            ctypes.byref(lo), ctypes.byref(hi)))
        return {"n": n.value, "leaf_dim": leaf.value, "bs": bs.value,
                "dtype": "f64" if dt.value == QT_F64 else "f32", "local_nblocks": nl.value,
                "global_nblocks": nglob.value, "row_lo": lo.value, "row_hi": hi.value}

    @property
    def nblocks(self) -> int:
        return self.info()["local_nblocks"]

    def level_nodes(self):
        buf = (ctypes.c_int64 * MAX_LEVELS)()
        nl = ctypes.c_int32()
        _check(_lib.qt_level_nodes(self._h, buf, MAX_LEVELS, ctypes.byref(nl)))
        return list(buf[: nl.value])

    def to_blocks(self, out=None, wait=True):
        """(brow, bcol, vals) sorted by (brow, bcol).  Default: new numpy arrays.
        ``out=(brow, bcol, vals)`` writes into caller buffers (numpy or torch,
        host or device).  ``wait=False`` (qt_read_back_async): host copies run
        on the context's copy stream and are valid after ``ctx.synchronize()``."""
        inf = self.info()
        nb, bs = inf["local_nblocks"], inf["bs"]
        if out is None:
            dt = np.float64 if inf["dtype"] == "f64" else np.float32
            out = (np.empty(nb, np.int32), np.empty(nb, np.int32), np.empty((nb, bs, bs), dt))
        if nb:
            fn = _lib.qt_read_back if wait else _lib.qt_read_back_async
            _check(fn(self._h, _ptr(out[0]), _ptr(out[1]), _ptr(out[2])))
        return out

    def close(self):
        if getattr(self, "_h", None):
            _check(_lib.qt_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
