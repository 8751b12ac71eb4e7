"""paper_2601_19092_b200 -- thin Python binding of libaxe (include/axe.h).

Argument marshalling only: every step of the data path runs inside libaxe.so
(host planner in C++, kernels in CUDA for sm_100a).  There is no Python or CPU
fallback: importing this package fails loudly if libaxe.so is missing.

Layouts / storages are accepted as the plain-data dicts of synth.py:
  layout  = {"D": [(extent, stride, axis)], "R": [...], "O": {axis: value}}
  storage = {"digits": [(axis, extent, divisor)], "swizzle": (B, M, S)}
Device buffers are torch CUDA tensors (or raw device pointers as ints).
"""
from __future__ import annotations

import ctypes as C
import json
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.environ.get("AXE_LIBAXE") or os.path.join(_HERE, "libaxe.so")  # AXE_LIBAXE: A/B builds only

if not os.path.exists(_SO):
    raise ImportError(f"libaxe.so not built ({_SO}); run __graft_entry__.build() or "
                      f"python paper_2601_19092_b200/build.py")

_lib = C.CDLL(_SO, mode=C.RTLD_GLOBAL)

# --------------------------------------------------------------------------- C types
AXE_OK = 0
ERRORS = {0: "AXE_OK", 1: "AXE_ERR_INVALID_ARG", 2: "AXE_ERR_OVERFLOW", 3: "AXE_ERR_DOMAIN", 4: "AXE_ERR_CAPACITY",
          5: "AXE_ERR_SIZE_MISMATCH", 6: "AXE_ERR_NONINJECTIVE", 7: "AXE_ERR_BOUNDS",
          8: "AXE_ERR_UNSUPPORTED_AXIS", 9: "AXE_ERR_ALIGNMENT", 10: "AXE_ERR_ALIAS", 11: "AXE_ERR_CUDA",
          12: "AXE_ERR_NCCL", 13: "AXE_ERR_UNSUPPORTED", 14: "AXE_ERR_TIMEOUT"}
KERNELS = {"auto": 0, "generic": 1, "vector": 2, "tma": 3, "tile": 4, "register": 5, "shuffle": 7, "transpose": 8,
           "lowered": 9, "dual": 10}


class axe_iter(C.Structure):
    _fields_ = [("extent", C.c_int64), ("stride", C.c_int64), ("axis", C.c_char_p)]


class axe_axis_coord(C.Structure):
    _fields_ = [("axis", C.c_char_p), ("value", C.c_int64)]


class axe_storage_digit(C.Structure):
    _fields_ = [("axis", C.c_char_p), ("extent", C.c_int64), ("divisor", C.c_int64)]


class axe_tma_desc(C.Structure):
    _fields_ = [("rank", C.c_int), ("dims", C.c_uint64 * 5), ("strides", C.c_uint64 * 5), ("box", C.c_uint32 * 5),
                ("logical_dim", C.c_int * 5), ("swizzle_bytes", C.c_int), ("base_bytes", C.c_int64), ("atoms", C.c_int64),
                ("fused_rows", C.c_uint32)]


class axe_storage(C.Structure):
    _fields_ = [("n", C.c_int), ("digits", C.POINTER(axe_storage_digit)), ("swz_bits", C.c_int),
                ("swz_base", C.c_int), ("swz_shift", C.c_int)]


_vp, _i64, _pi64 = C.c_void_p, C.c_int64, C.POINTER(C.c_int64)
_SIGS = {
    "axe_last_error": ([], C.c_char_p),
    "axe_version": ([], C.c_char_p),
    "axe_kernel_launch_count": ([], C.c_int64),
    "axe_layout_create": ([C.POINTER(axe_iter), C.c_int, C.POINTER(axe_iter), C.c_int, C.POINTER(axe_axis_coord),
                           C.c_int, C.POINTER(_vp)], C.c_int),
    "axe_layout_destroy": ([_vp], None),
    "axe_layout_info": ([_vp, _pi64, _pi64, C.POINTER(C.c_int)], C.c_int),
    "axe_layout_axis_name": ([_vp, C.c_int, C.POINTER(C.c_char_p)], C.c_int),
    "axe_layout_iters": ([_vp, C.c_int, C.POINTER(axe_iter), C.c_int, C.POINTER(C.c_int)], C.c_int),
    "axe_layout_offset": ([_vp, C.POINTER(axe_axis_coord), C.c_int, C.POINTER(C.c_int)], C.c_int),
    "axe_layout_eval": ([_vp, _i64, _pi64, _i64], C.c_int),
    "axe_layout_canonicalize": ([_vp, C.POINTER(_vp), C.POINTER(C.c_int)], C.c_int),
    "axe_layout_bounds": ([_vp, C.c_char_p, _pi64, _pi64], C.c_int),
    "axe_layout_group": ([_vp, _pi64, C.c_int, C.POINTER(_vp), C.POINTER(C.c_int)], C.c_int),
    "axe_layout_span": ([_vp, C.c_char_p, _pi64], C.c_int),
    "axe_layout_tile": ([_vp, _pi64, _vp, _pi64, C.c_int, C.POINTER(_vp)], C.c_int),
    "axe_layout_tile_of": ([_vp, _pi64, _vp, _pi64, C.c_int, C.POINTER(_vp), _pi64], C.c_int),
    "axe_layout_direct_sum": ([_vp, _pi64, _vp, _pi64, C.c_int, C.POINTER(_vp)], C.c_int),
    "axe_layout_slice": ([_vp, _pi64, C.c_int, _pi64, _pi64, C.POINTER(_vp)], C.c_int),
    "axe_layout_parse": ([C.c_char_p, C.POINTER(_vp), C.POINTER(C.c_int)], C.c_int),
    "axe_layout_format": ([_vp, C.c_char_p, C.c_int], C.c_int),
    "axe_layout_to_json": ([_vp, C.c_char_p, C.c_int], C.c_int),
    "axe_layout_equivalent": ([_vp, _vp, _i64, C.POINTER(C.c_int)], C.c_int),
    "axe_tma_lower": ([_vp, _pi64, _pi64, _pi64, _vp, _pi64, C.c_int, C.c_int, C.c_int, C.POINTER(axe_tma_desc),
                       C.POINTER(_vp)], C.c_int),
    "axe_copy_plan_create": ([_vp, C.POINTER(axe_storage), _vp, C.POINTER(axe_storage), C.c_int, C.c_int,
                              C.POINTER(_vp)], C.c_int),
    "axe_copy_plan_create_ex": ([_vp, C.POINTER(axe_storage), _vp, C.POINTER(axe_storage), C.c_int, C.c_int, C.c_int,
                                 C.POINTER(_vp)], C.c_int),
    "axe_copy_plan_execute": ([_vp, _vp, _vp, _vp], C.c_int),
    "axe_copy_plan_execute_host": ([_vp, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "axe_copy_plan_sizes": ([_vp, _pi64, _pi64], C.c_int),
    "axe_copy_plan_describe": ([_vp, C.c_char_p, C.c_int], C.c_int),
    "axe_copy_plan_destroy": ([_vp], None),
    "axe_tma_plan_create": ([C.POINTER(axe_tma_desc), _vp, C.POINTER(_vp)], C.c_int),
    "axe_tma_plan_sizes": ([_vp, _pi64, _pi64, _pi64], C.c_int),
    "axe_tma_plan_execute": ([_vp, _vp, _vp, _vp], C.c_int),
    "axe_tma_plan_execute_store": ([_vp, _vp, _vp, _vp], C.c_int),
    "axe_tma_plan_destroy": ([_vp], None),
    "axe_copy": ([_vp, C.POINTER(axe_storage), _vp, _vp, C.POINTER(axe_storage), _vp, C.c_int, _vp], C.c_int),
    "axe_get_unique_id": ([C.c_char_p], C.c_int),
    "axe_comm_create": ([C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(_vp)], C.c_int),
    "axe_comm_destroy": ([_vp], None),
    "axe_comm_wait": ([_vp, _vp, C.c_int], C.c_int),
    "axe_ipc_export": ([_vp, C.c_char_p], C.c_int),
    "axe_ipc_import": ([C.c_char_p, C.POINTER(_vp)], C.c_int),
    "axe_ipc_close": ([_vp], C.c_int),
    "axe_redist_plan_create": ([_vp, C.POINTER(axe_storage), _vp, C.POINTER(axe_storage), C.c_int, C.c_int, C.c_int,
                                C.POINTER(_vp)], C.c_int),
    "axe_redist_plan_execute": ([_vp, _vp, _vp, _vp, _vp], C.c_int),
    "axe_redist_plan_describe": ([_vp, C.c_char_p, C.c_int], C.c_int),
    "axe_redist_plan_execute_peers": ([_vp, _vp, C.POINTER(_vp), _vp], C.c_int),
    "axe_redist_plan_counts": ([_vp, C.c_int, _pi64, _pi64], C.c_int),
    "axe_redist_plan_map": ([_vp, C.c_int, C.c_int, _i64, _pi64, _pi64], C.c_int),
    "axe_redist_plan_destroy": ([_vp], None),
    "axe_redistribute": ([_vp, C.POINTER(axe_storage), _vp, _vp, C.POINTER(axe_storage), _vp, C.c_int, _vp, _vp],
                         C.c_int),
    "axe_redist_emulate": ([C.POINTER(_vp), C.c_int, C.POINTER(_vp), C.POINTER(_vp), _vp], C.c_int),
    "axe_reduce_plan_create": ([_vp, C.POINTER(axe_storage), _vp, C.POINTER(axe_storage), C.c_int, C.POINTER(_vp)],
                               C.c_int),
    "axe_reduce_plan_execute": ([_vp, _vp, _vp, _vp], C.c_int),
    "axe_reduce_plan_sizes": ([_vp, _pi64, _pi64], C.c_int),
    "axe_reduce_plan_describe": ([_vp, C.c_char_p, C.c_int], C.c_int),
    "axe_reduce_plan_destroy": ([_vp], None),
    "axe_reduce": ([_vp, C.POINTER(axe_storage), _vp, _vp, C.POINTER(axe_storage), _vp, C.c_int, _vp], C.c_int),
    "axe_redist_reduce_plan_create": ([_vp, C.POINTER(axe_storage), _vp, C.POINTER(axe_storage), C.c_int, C.c_int,
                                       C.c_int, C.POINTER(_vp)], C.c_int),
    "axe_redist_plan_phase": ([_vp, C.c_int, C.POINTER(_vp)], C.c_int),
    "axe_redist_plan_execute_peers_reduce": ([_vp, C.POINTER(_vp), _vp, _vp], C.c_int),
    "axe_redist_plan_execute_multicast_reduce": ([_vp, _vp, _vp, _vp], C.c_int),
    "axe_redistribute_reduce": ([_vp, C.POINTER(axe_storage), _vp, _vp, C.POINTER(axe_storage), _vp, C.c_int, _vp,
                                 _vp], C.c_int),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = sorted(_SIGS)


class AxeError(RuntimeError):
    def __init__(self, code: int, what: str):
        self.code = code
        self.name = ERRORS.get(code, str(code))
        msg = _lib.axe_last_error()
        super().__init__(f"{what}: {self.name}: {msg.decode() if msg else ''}")


def _check(code: int, what: str):
    if code != AXE_OK:
        raise AxeError(code, what)


def version() -> str:
    return _lib.axe_version().decode()


def kernel_launch_count() -> int:
    return int(_lib.axe_kernel_launch_count())


# --------------------------------------------------------------------------- marshalling
def _iters(lst, keep):
    arr = (axe_iter * max(1, len(lst)))()
    for i, it in enumerate(lst):
        e, s = int(it[0]), int(it[1])
        a = it[2] if len(it) > 2 and it[2] is not None else "m"
        b = a.encode()
        keep.append(b)
        arr[i] = axe_iter(e, s, b)
    keep.append(arr)
    return arr


def make_storage(st) -> tuple:
    """plain-data storage dict -> (axe_storage, keepalive)."""
    keep = []
    d = st["digits"]
    arr = (axe_storage_digit * max(1, len(d)))()
    for i, dg in enumerate(d):
        b = dg[0].encode()
        keep.append(b)
        arr[i] = axe_storage_digit(b, int(dg[1]), int(dg[2]) if len(dg) > 2 else 1)
    keep.append(arr)
    sw = tuple(st.get("swizzle", (0, 0, 0)))
    return axe_storage(len(d), arr, sw[0], sw[1], sw[2]), keep


def _ptr(x):
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "ctypes"):
        return x.ctypes.data
    raise TypeError(f"cannot take a pointer of {type(x)}")


def _stream(s):
    if s is None:
        try:
            import torch
            return torch.cuda.current_stream().cuda_stream
        except Exception:
            return None
    if isinstance(s, int):
        return s
    return s.cuda_stream


# --------------------------------------------------------------------------- layouts
class Layout:
    """An immutable Axe layout L = (D, R, O) owned by libaxe."""

    def __init__(self, D=None, R=(), O=None, *, spec=None, _handle=None):
        if _handle is not None:
            self._h = _handle
            return
        if spec is not None:
            D, R, O = spec["D"], spec.get("R", []), spec.get("O", {})
        keep = []
        O = dict(O or {})
        oarr = (axe_axis_coord * max(1, len(O)))()
        for i, (a, v) in enumerate(O.items()):
            b = a.encode()
            keep.append(b)
            oarr[i] = axe_axis_coord(b, int(v))
        h = C.c_void_p()
        _check(_lib.axe_layout_create(_iters(list(D), keep), len(D), _iters(list(R), keep), len(R), oarr, len(O),
                                      C.byref(h)), "axe_layout_create")
        self._h = h

    @classmethod
    def of(cls, spec) -> "Layout":
        return spec if isinstance(spec, Layout) else cls(spec=spec)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:  # (module globals may be gone at interpreter exit)
            _lib.axe_layout_destroy(h)
        self._h = None

    @property
    def handle(self):
        return self._h

    def info(self):
        ed, er, na = C.c_int64(), C.c_int64(), C.c_int()
        _check(_lib.axe_layout_info(self._h, C.byref(ed), C.byref(er), C.byref(na)), "axe_layout_info")
        return ed.value, er.value, na.value

    @property
    def E_D(self):
        return self.info()[0]

    @property
    def E_R(self):
        return self.info()[1]

    def axes(self):
        n = self.info()[2]
        out = []
        for i in range(n):
            p = C.c_char_p()
            _check(_lib.axe_layout_axis_name(self._h, i, C.byref(p)), "axe_layout_axis_name")
            out.append(p.value.decode())
        return out

    def iters(self, which: int = 0):
        n = C.c_int()
        arr = (axe_iter * 64)()
        _check(_lib.axe_layout_iters(self._h, which, arr, 64, C.byref(n)), "axe_layout_iters")
        return [(arr[i].extent, arr[i].stride, arr[i].axis.decode()) for i in range(n.value)]

    def offset(self):
        n = C.c_int()
        arr = (axe_axis_coord * 64)()
        _check(_lib.axe_layout_offset(self._h, arr, 64, C.byref(n)), "axe_layout_offset")
        return {arr[i].axis.decode(): arr[i].value for i in range(n.value)}

    def spec(self):
        return {"D": self.iters(0), "R": self.iters(1), "O": self.offset()}

    def eval(self, x: int):
        """f_L(x): list of E_R dicts {axis: value}."""
        ed, er, na = self.info()
        buf = (C.c_int64 * max(1, er * na))()
        _check(_lib.axe_layout_eval(self._h, x, buf, er * na), "axe_layout_eval")
        ax = self.axes()
        return [{ax[i]: buf[r * na + i] for i in range(na)} for r in range(er)]

    def canonicalize(self):
        h = C.c_void_p()
        gc = C.c_int()
        _check(_lib.axe_layout_canonicalize(self._h, C.byref(h), C.byref(gc)), "axe_layout_canonicalize")
        return Layout(_handle=h), bool(gc.value)

    def bounds(self, axis: str):
        lo, hi = C.c_int64(), C.c_int64()
        _check(_lib.axe_layout_bounds(self._h, axis.encode(), C.byref(lo), C.byref(hi)), "axe_layout_bounds")
        return lo.value, hi.value

    # ---- layout operators (§3.3, Apps. B-F) ----
    @staticmethod
    def _shape(S):
        return (C.c_int64 * len(S))(*[int(v) for v in S])

    def span(self, axis: str) -> int:
        v = C.c_int64()
        _check(_lib.axe_layout_span(self._h, axis.encode(), C.byref(v)), "axe_layout_span")
        return v.value

    def group(self, S):
        """Group-By-Shape (Alg. 1): (grouped layout, block boundaries)."""
        h = C.c_void_p()
        b = (C.c_int * (len(S) + 1))()
        _check(_lib.axe_layout_group(self._h, self._shape(S), len(S), C.byref(h), b), "axe_layout_group")
        return Layout(_handle=h), list(b)

    def tile(self, SA, B, SB):
        """self (x) B (Alg. 2), grouped by the interleaved shape."""
        h = C.c_void_p()
        _check(_lib.axe_layout_tile(self._h, self._shape(SA), Layout.of(B).handle, self._shape(SB), len(SA),
                                    C.byref(h)), "axe_layout_tile")
        return Layout(_handle=h)

    def tile_of(self, SA, B, SB):
        """TileOf_AndRecoverC (Alg. 3): (C, S_C) with self = C (x) B."""
        h = C.c_void_p()
        sc = (C.c_int64 * len(SA))()
        _check(_lib.axe_layout_tile_of(self._h, self._shape(SA), Layout.of(B).handle, self._shape(SB), len(SA),
                                       C.byref(h), sc), "axe_layout_tile_of")
        return Layout(_handle=h), list(sc)

    def direct_sum(self, SA, B, SB):
        h = C.c_void_p()
        _check(_lib.axe_layout_direct_sum(self._h, self._shape(SA), Layout.of(B).handle, self._shape(SB), len(SA),
                                          C.byref(h)), "axe_layout_direct_sum")
        return Layout(_handle=h)

    @classmethod
    def parse(cls, text: str) -> "Layout":
        """axe_layout_parse: "(e0,e1):(s0@a0,s1) + [(r):(t@b)] + o@c" (axis m by default)."""
        h, pos = C.c_void_p(), C.c_int(-1)
        code = _lib.axe_layout_parse(text.encode(), C.byref(h), C.byref(pos))
        if code != AXE_OK:
            err = AxeError(code, "axe_layout_parse")
            err.pos = pos.value
            raise err
        return Layout(_handle=h)

    def format(self) -> str:
        buf = C.create_string_buffer(1 << 14)
        _check(_lib.axe_layout_format(self._h, buf, len(buf)), "axe_layout_format")
        return buf.value.decode()

    def __str__(self):
        return self.format()

    def to_json(self) -> dict:
        buf = C.create_string_buffer(1 << 15)
        _check(_lib.axe_layout_to_json(self._h, buf, len(buf)), "axe_layout_to_json")
        return json.loads(buf.value.decode())

    def equivalent(self, other, threshold: int = -1):
        """True / False, or None when undecidable (no gap condition and too large to enumerate)."""
        r = C.c_int()
        _check(_lib.axe_layout_equivalent(self._h, Layout.of(other).handle, threshold, C.byref(r)),
               "axe_layout_equivalent")
        return None if r.value < 0 else bool(r.value)

    def slice(self, S, begin, extent):
        """L[R:S] (Alg. 4 per block) for the region [begin, begin + extent)."""
        h = C.c_void_p()
        _check(_lib.axe_layout_slice(self._h, self._shape(S), len(S), self._shape(begin), self._shape(extent),
                                     C.byref(h)), "axe_layout_slice")
        return Layout(_handle=h)


# --------------------------------------------------------------------------- copy
class CopyPlan:
    """axe_copy_plan_create / _execute / _describe (include/axe.h)."""

    def __init__(self, src, src_st, dst, dst_st, elem_size: int, kernel: str = "auto", host_slabs: int = 0):
        self.src, self.dst = Layout.of(src), Layout.of(dst)
        ss, k1 = make_storage(src_st)
        ds, k2 = make_storage(dst_st)
        h = C.c_void_p()
        if host_slabs:
            _check(_lib.axe_copy_plan_create_ex(self.src.handle, C.byref(ss), self.dst.handle, C.byref(ds),
                                                elem_size, KERNELS[kernel], host_slabs, C.byref(h)),
                   "axe_copy_plan_create_ex")
        else:
            _check(_lib.axe_copy_plan_create(self.src.handle, C.byref(ss), self.dst.handle, C.byref(ds), elem_size,
                                             KERNELS[kernel], C.byref(h)), "axe_copy_plan_create")
        self._h = h
        self.elem_size = elem_size

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:  # (module globals may be gone at interpreter exit)
            _lib.axe_copy_plan_destroy(h)
        self._h = None

    def execute(self, src, dst, stream=None):
        _check(_lib.axe_copy_plan_execute(self._h, _ptr(src), _ptr(dst), _stream(stream)), "axe_copy_plan_execute")

    def execute_host(self, host_src, host_dst, dev_src, dev_dst, stream=None):
        _check(_lib.axe_copy_plan_execute_host(self._h, _ptr(host_src), _ptr(host_dst), _ptr(dev_src), _ptr(dev_dst),
                                               _stream(stream)), "axe_copy_plan_execute_host")

    def sizes(self):
        a, b = C.c_int64(), C.c_int64()
        _check(_lib.axe_copy_plan_sizes(self._h, C.byref(a), C.byref(b)), "axe_copy_plan_sizes")
        return a.value, b.value

    def describe(self) -> dict:
        buf = C.create_string_buffer(1 << 16)
        _check(_lib.axe_copy_plan_describe(self._h, buf, len(buf)), "axe_copy_plan_describe")
        return json.loads(buf.value.decode())


def axe_copy(src, src_st, src_buf, dst, dst_st, dst_buf, elem_size: int, stream=None):
    """One-shot stream-ordered copy dst <- src (include/axe.h axe_copy)."""
    s, d = Layout.of(src), Layout.of(dst)
    ss, k1 = make_storage(src_st)
    ds, k2 = make_storage(dst_st)
    _check(_lib.axe_copy(s.handle, C.byref(ss), _ptr(src_buf), d.handle, C.byref(ds), _ptr(dst_buf), elem_size,
                         _stream(stream)), "axe_copy")


# --------------------------------------------------------------------------- redistribute
def get_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib.axe_get_unique_id(buf), "axe_get_unique_id")
    return buf.raw


class Comm:
    """axe_comm_create: an NCCL communicator owned by libaxe.  The 128-byte id is created on rank 0
    (get_unique_id) and broadcast by the caller, e.g. over a torch.distributed process group."""

    def __init__(self, uid: bytes, nranks: int, rank: int, device: int):
        h = C.c_void_p()
        _check(_lib.axe_comm_create(uid, nranks, rank, device, C.byref(h)), "axe_comm_create")
        self._h, self.nranks, self.rank = h, nranks, rank

    @classmethod
    def from_process_group(cls, device: int, group=None) -> "Comm":
        import torch
        import torch.distributed as dist
        rank, ws = dist.get_rank(group), dist.get_world_size(group)
        obj = [get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(obj[0], ws, rank, device)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:  # (module globals may be gone at interpreter exit)
            _lib.axe_comm_destroy(h)
        self._h = None

    @property
    def handle(self):
        return self._h

    def wait(self, stream=None, timeout_ms: int = -1):
        """axe_comm_wait: block until the stream is done, polling NCCL's asynchronous errors; on an error or
        a timeout the communicator is aborted and AxeError (AXE_ERR_NCCL / AXE_ERR_TIMEOUT) raised."""
        _check(_lib.axe_comm_wait(self._h, _stream(stream), int(timeout_ms)), "axe_comm_wait")


def ipc_export(buf) -> bytes:
    """axe_ipc_export: a 128-byte CUDA IPC handle for the device buffer (tensor or pointer)."""
    h = C.create_string_buffer(128)
    _check(_lib.axe_ipc_export(_ptr(buf), h), "axe_ipc_export")
    return h.raw


def ipc_import(handle: bytes) -> int:
    """axe_ipc_import: map another process's exported buffer; returns the device pointer (int)."""
    assert len(handle) == 128
    p = C.c_void_p()
    _check(_lib.axe_ipc_import(handle, C.byref(p)), "axe_ipc_import")
    return int(p.value)


def ipc_close(ptr: int) -> None:
    _check(_lib.axe_ipc_close(C.c_void_p(ptr)), "axe_ipc_close")


class RedistPlan:
    """axe_redist_plan_create / _execute / _describe / _counts / _map (include/axe.h).
    With reduce_dtype set: axe_redist_reduce_plan_create (the source's leading logical dimension
    is summed away; elem_size is then the dtype's size)."""

    def __init__(self, src, src_st, dst, dst_st, elem_size: int, nranks: int, rank: int, reduce_dtype=None):
        self.src, self.dst = Layout.of(src), Layout.of(dst)
        ss, k1 = make_storage(src_st)
        ds, k2 = make_storage(dst_st)
        h = C.c_void_p()
        if reduce_dtype is None:
            _check(_lib.axe_redist_plan_create(self.src.handle, C.byref(ss), self.dst.handle, C.byref(ds), elem_size,
                                               nranks, rank, C.byref(h)), "axe_redist_plan_create")
        else:
            _check(_lib.axe_redist_reduce_plan_create(self.src.handle, C.byref(ss), self.dst.handle, C.byref(ds),
                                                      DTYPES[reduce_dtype], nranks, rank, C.byref(h)),
                   "axe_redist_reduce_plan_create")
            elem_size = DTYPE_SIZE[reduce_dtype]
        self._h, self.nranks, self.rank, self.elem_size = h, nranks, rank, elem_size

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and getattr(self, "_owned", True) and _lib is not None:
            _lib.axe_redist_plan_destroy(h)
        self._h = None

    def phase(self, i: int) -> "RedistPlan":
        """Sub-plan i (0: reduce-scatter, 1: gather) of a two-phase reduction plan (owned by this plan)."""
        h = C.c_void_p()
        _check(_lib.axe_redist_plan_phase(self._h, i, C.byref(h)), "axe_redist_plan_phase")
        sub = RedistPlan.__new__(RedistPlan)
        sub._h, sub._owned, sub._parent = h, False, self
        sub.nranks, sub.rank, sub.elem_size = self.nranks, self.rank, self.elem_size
        return sub

    @property
    def handle(self):
        return self._h

    def execute(self, comm: Comm, src_local, dst_local, stream=None):
        _check(_lib.axe_redist_plan_execute(self._h, comm.handle, _ptr(src_local), _ptr(dst_local), _stream(stream)),
               "axe_redist_plan_execute")

    def describe(self) -> dict:
        buf = C.create_string_buffer(1 << 14)
        _check(_lib.axe_redist_plan_describe(self._h, buf, len(buf)), "axe_redist_plan_describe")
        return json.loads(buf.value.decode())

    def execute_peers(self, src_local, dst_peers, stream=None):
        """One-sided: copy kernels from src_local straight into every receiver's dst (peer pointers)."""
        arr = (C.c_void_p * len(dst_peers))(*[_ptr(d) for d in dst_peers])
        _check(_lib.axe_redist_plan_execute_peers(self._h, _ptr(src_local), arr, _stream(stream)),
               "axe_redist_plan_execute_peers")

    def execute_peers_reduce(self, src_peers, dst_local, stream=None):
        """One-sided pull reduction: K4 kernels read every partial straight from src_peers[owner]."""
        arr = (C.c_void_p * len(src_peers))(*[_ptr(x) for x in src_peers])
        _check(_lib.axe_redist_plan_execute_peers_reduce(self._h, arr, _ptr(dst_local), _stream(stream)),
               "axe_redist_plan_execute_peers_reduce")

    def execute_multicast_reduce(self, src_multicast, dst_local, stream=None):
        """NVLS reduction: one multimem.ld_reduce per 16-byte output vector on the multicast address."""
        _check(_lib.axe_redist_plan_execute_multicast_reduce(self._h, _ptr(src_multicast), _ptr(dst_local),
                                                             _stream(stream)),
               "axe_redist_plan_execute_multicast_reduce")

    def counts(self, peer: int):
        a, b = C.c_int64(), C.c_int64()
        _check(_lib.axe_redist_plan_counts(self._h, peer, C.byref(a), C.byref(b)), "axe_redist_plan_counts")
        return a.value, b.value

    def map(self, kind: int, peer: int, k: int):
        a, b = C.c_int64(), C.c_int64()
        _check(_lib.axe_redist_plan_map(self._h, kind, peer, k, C.byref(a), C.byref(b)), "axe_redist_plan_map")
        return a.value, b.value


def axe_redistribute(src, src_st, src_local, dst, dst_st, dst_local, elem_size: int, comm: Comm, stream=None):
    s, d = Layout.of(src), Layout.of(dst)
    ss, k1 = make_storage(src_st)
    ds, k2 = make_storage(dst_st)
    _check(_lib.axe_redistribute(s.handle, C.byref(ss), _ptr(src_local), d.handle, C.byref(ds), _ptr(dst_local),
                                 elem_size, comm.handle, _stream(stream)), "axe_redistribute")


# --------------------------------------------------------------------------- reduction (§8(f) f3)
DTYPES = {"f32": 1, "f64": 2, "f16": 3, "bf16": 4, "i32": 5, "i64": 6}
DTYPE_SIZE = {"f32": 4, "f64": 8, "f16": 2, "bf16": 2, "i32": 4, "i64": 8}


class ReducePlan:
    """axe_reduce_plan_create / _execute / _sizes / _describe: dst(y) = sum_k src(k * E_D(dst) + y)."""

    def __init__(self, src, src_st, dst, dst_st, dtype: str):
        self.src, self.dst = Layout.of(src), Layout.of(dst)
        ss, k1 = make_storage(src_st)
        ds, k2 = make_storage(dst_st)
        h = C.c_void_p()
        _check(_lib.axe_reduce_plan_create(self.src.handle, C.byref(ss), self.dst.handle, C.byref(ds), DTYPES[dtype],
                                           C.byref(h)), "axe_reduce_plan_create")
        self._h, self.dtype = h, dtype

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:  # (module globals may be gone at interpreter exit)
            _lib.axe_reduce_plan_destroy(h)
        self._h = None

    def execute(self, src, dst, stream=None):
        _check(_lib.axe_reduce_plan_execute(self._h, _ptr(src), _ptr(dst), _stream(stream)), "axe_reduce_plan_execute")

    def sizes(self):
        a, b = C.c_int64(), C.c_int64()
        _check(_lib.axe_reduce_plan_sizes(self._h, C.byref(a), C.byref(b)), "axe_reduce_plan_sizes")
        return a.value, b.value

    def describe(self) -> dict:
        buf = C.create_string_buffer(1 << 14)
        _check(_lib.axe_reduce_plan_describe(self._h, buf, len(buf)), "axe_reduce_plan_describe")
        return json.loads(buf.value.decode())


def axe_reduce(src, src_st, src_buf, dst, dst_st, dst_buf, dtype: str, stream=None):
    """One-shot stream-ordered reduction over the leading logical dimension (include/axe.h axe_reduce)."""
    s, d = Layout.of(src), Layout.of(dst)
    ss, k1 = make_storage(src_st)
    ds, k2 = make_storage(dst_st)
    _check(_lib.axe_reduce(s.handle, C.byref(ss), _ptr(src_buf), d.handle, C.byref(ds), _ptr(dst_buf), DTYPES[dtype],
                           _stream(stream)), "axe_reduce")


def axe_redistribute_reduce(src, src_st, src_local, dst, dst_st, dst_local, dtype: str, comm: Comm, stream=None):
    s, d = Layout.of(src), Layout.of(dst)
    ss, k1 = make_storage(src_st)
    ds, k2 = make_storage(dst_st)
    _check(_lib.axe_redistribute_reduce(s.handle, C.byref(ss), _ptr(src_local), d.handle, C.byref(ds),
                                        _ptr(dst_local), DTYPES[dtype], comm.handle, _stream(stream)),
           "axe_redistribute_reduce")


def redist_emulate(plans, src_locals, dst_locals, stream=None):
    """axe_redist_emulate: every rank's plan on the current device, device-to-device copies as the wire."""
    n = len(plans)
    hp = (C.c_void_p * n)(*[p.handle.value for p in plans])
    sp = (C.c_void_p * n)(*[_ptr(x) for x in src_locals])
    dp = (C.c_void_p * n)(*[_ptr(x) for x in dst_locals])
    _check(_lib.axe_redist_emulate(hp, n, sp, dp, _stream(stream)), "axe_redist_emulate")


def tma_lower(LG, EG, LS, ES, elem_size: int, swizzle_bytes: int, begin=None, extent=None) -> dict:
    """axe_tma_lower: the paper's TMA lowering -> CuTensorMap encoding + the atom tiler T."""
    G, S = Layout.of(LG), Layout.of(LS)
    r = len(EG)
    arr = lambda v: (C.c_int64 * r)(*v) if v is not None else None
    d = axe_tma_desc()
    t = C.c_void_p()
    _check(_lib.axe_tma_lower(G.handle, arr(EG), arr(begin), arr(extent), S.handle, arr(ES), r, elem_size,
                              swizzle_bytes, C.byref(d), C.byref(t)), "axe_tma_lower")
    n = d.rank
    return {"rank": n, "dims": list(d.dims[:n]), "strides": list(d.strides[:n]), "box": list(d.box[:n]),
            "logical_dim": list(d.logical_dim[:n]),
            "swizzle_bytes": d.swizzle_bytes, "base_bytes": d.base_bytes, "atoms": d.atoms,
            "fused_rows": d.fused_rows, "tiler": Layout(_handle=t), "_desc": d}


class TmaPlan:
    """axe_tma_plan_create / _sizes / _execute: the lowering of tma_lower() run on the device -- one TMA
    tensor load + one bulk store per swizzle atom, into an HBM image of the shared-memory tensor L_S."""

    def __init__(self, LG, EG, LS, ES, elem_size: int, swizzle_bytes: int, begin=None, extent=None):
        self.lowering = tma_lower(LG, EG, LS, ES, elem_size, swizzle_bytes, begin, extent)
        h = C.c_void_p()
        _check(_lib.axe_tma_plan_create(C.byref(self.lowering["_desc"]), self.lowering["tiler"].handle, C.byref(h)),
               "axe_tma_plan_create")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.axe_tma_plan_destroy(h)
        self._h = None

    def sizes(self):
        a, b = C.c_int64(), C.c_int64()
        _check(_lib.axe_tma_plan_sizes(self._h, C.byref(a), None, C.byref(b)), "axe_tma_plan_sizes")
        return a.value, b.value   # atoms, image bytes

    def boxes(self) -> int:
        n = C.c_int64()
        _check(_lib.axe_tma_plan_sizes(self._h, None, C.byref(n), None), "axe_tma_plan_sizes")
        return n.value

    def execute(self, g_base, s_image, stream=None):
        _check(_lib.axe_tma_plan_execute(self._h, _ptr(g_base), _ptr(s_image), _stream(stream)), "axe_tma_plan_execute")

    def execute_store(self, g_base, s_image, stream=None):
        """The reverse: the L_S image back into the region of the global tensor (TMA tensor stores)."""
        _check(_lib.axe_tma_plan_execute_store(self._h, _ptr(g_base), _ptr(s_image), _stream(stream)),
               "axe_tma_plan_execute_store")


def axe_layout_create(D, R=(), O=None) -> Layout:
    return Layout(D, R, O)


def axe_layout_eval(layout, x: int):
    return Layout.of(layout).eval(x)


def axe_copy_plan_create(src, src_st, dst, dst_st, elem_size: int, kernel: str = "auto") -> CopyPlan:
    return CopyPlan(src, src_st, dst, dst_st, elem_size, kernel)
