"""ctypes wrapper around oracle/axe_oracle.c -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product library never does, and
this package never imports the product (paper_2601_19092_b200).

Layouts and storage descriptors are the plain-data dicts of synth.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "axe_oracle.c")
_LIB = os.environ.get("AXE_ORACLE_LIB") or os.path.join(_HERE, "liboracle.so")  # (tools/asan_host.sh build)

OK, EINVAL, EDOMAIN, ESIZE, EBOUNDS, ECOLLIDE, ECAPACITY, ENOMEM = range(8)
STATUS = {OK: "ok", EINVAL: "invalid", EDOMAIN: "domain", ESIZE: "size", EBOUNDS: "bounds",
          ECOLLIDE: "collide", ECAPACITY: "capacity", ENOMEM: "nomem"}


class OracleError(RuntimeError):
    def __init__(self, code, what=""):
        super().__init__(f"oracle {what}: {STATUS.get(code, code)}")
        self.code = code
        self.status = STATUS.get(code, str(code))


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (no shared code with the product build)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread", "-Wall",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Iter(C.Structure):
    _fields_ = [("extent", C.c_int64), ("stride", C.c_int64), ("axis", C.c_char_p)]


class _Coord(C.Structure):
    _fields_ = [("axis", C.c_char_p), ("value", C.c_int64)]


class _SDigit(C.Structure):
    _fields_ = [("axis", C.c_char_p), ("extent", C.c_int64), ("divisor", C.c_int64)]


class _Storage(C.Structure):
    _fields_ = [("n", C.c_int), ("digits", C.POINTER(_SDigit)), ("swz_b", C.c_int), ("swz_m", C.c_int),
                ("swz_s", C.c_int)]


class _Layout(C.Structure):
    _fields_ = [("nD", C.c_int), ("D", C.POINTER(_Iter)), ("nR", C.c_int), ("R", C.POINTER(_Iter)),
                ("nO", C.c_int), ("O", C.POINTER(_Coord))]


_lib = None
_lock = threading.Lock()


def _L():
    global _lib
    with _lock:
        if _lib is None:
            lib = C.CDLL(build())
            P = C.POINTER
            lib.ora_sizes.argtypes = [P(_Layout), P(C.c_int64), P(C.c_int64)]
            lib.ora_eval.argtypes = [P(_Layout), C.c_int64, P(C.c_char_p), P(C.c_int), P(C.c_int64), C.c_int64]
            lib.ora_bounds.argtypes = [P(_Layout), C.c_char_p, P(C.c_int64), P(C.c_int64)]
            lib.ora_storage_check.argtypes = [P(_Storage)]
            lib.ora_storage_cells.argtypes = [P(_Storage)]
            lib.ora_storage_cells.restype = C.c_int64
            lib.ora_storage_byte.argtypes = [P(_Storage), C.c_int, P(C.c_char_p), P(C.c_int64), C.c_int]
            lib.ora_storage_byte.restype = C.c_int64
            lib.ora_copy.argtypes = [P(_Layout), P(_Storage), C.c_void_p, C.c_int64, P(_Layout), P(_Storage),
                                     C.c_void_p, C.c_int64, C.c_int, C.c_int]
            lib.ora_redistribute.argtypes = [P(_Layout), P(_Storage), P(C.c_void_p), C.c_int64, P(_Layout),
                                             P(_Storage), P(C.c_void_p), C.c_int64, C.c_int, C.c_int, C.c_int,
                                             C.c_int]
            lib.ora_reduce.argtypes = [P(_Layout), P(_Storage), P(C.c_void_p), C.c_int64, P(_Layout), P(_Storage),
                                       P(C.c_void_p), C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int]
            _lib = lib
    return _lib


class _Keep:
    """Holds ctypes objects alive for the duration of a call."""

    def __init__(self):
        self.objs = []

    def add(self, o):
        self.objs.append(o)
        return o


def _mk_layout(L, keep: _Keep) -> _Layout:
    def iters(lst):
        arr = keep.add((_Iter * max(1, len(lst)))())
        for i, (e, s, a) in enumerate(lst):
            arr[i].extent, arr[i].stride = e, s
            arr[i].axis = keep.add(a.encode())
        return arr
    O = list(L.get("O", {}).items())
    oarr = keep.add((_Coord * max(1, len(O)))())
    for i, (a, v) in enumerate(O):
        oarr[i].axis = keep.add(a.encode())
        oarr[i].value = v
    lay = _Layout(len(L["D"]), iters(L["D"]), len(L.get("R", [])), iters(L.get("R", [])), len(O), oarr)
    return keep.add(lay)


def _mk_storage(st, keep: _Keep) -> _Storage:
    d = st["digits"]
    arr = keep.add((_SDigit * max(1, len(d)))())
    for i, (a, e, dv) in enumerate(d):
        arr[i].axis = keep.add(a.encode())
        arr[i].extent, arr[i].divisor = e, dv
    b, m, s = st.get("swizzle", (0, 0, 0))
    return keep.add(_Storage(len(d), arr, b, m, s))


def sizes(L):
    k = _Keep()
    ed, er = C.c_int64(), C.c_int64()
    st = _L().ora_sizes(C.byref(_mk_layout(L, k)), C.byref(ed), C.byref(er))
    if st:
        raise OracleError(st, "sizes")
    return ed.value, er.value


def eval(L, x: int):
    """f_L(x) as a list of E_R dicts {axis: value} in lexicographic replica order."""
    k = _Keep()
    lay = _mk_layout(L, k)
    ed, er = sizes(L)
    axes = (C.c_char_p * 32)()
    n = C.c_int()
    cap = er * 32
    rows = (C.c_int64 * cap)()
    st = _L().ora_eval(C.byref(lay), x, axes, C.byref(n), rows, cap)
    if st:
        raise OracleError(st, "eval")
    names = [axes[i].decode() for i in range(n.value)]
    return [{names[i]: rows[r * n.value + i] for i in range(n.value)} for r in range(er)]


def eval_set(L, x: int):
    """f_L(x) as a frozenset of coordinates with zero components dropped (sparse ZA)."""
    return frozenset(frozenset((a, v) for a, v in c.items() if v != 0) for c in eval(L, x))


def bounds(L, axis: str):
    """Brute-force (min, max) of the axis over every coordinate of every f_L(x); None if absent."""
    k = _Keep()
    lo, hi = C.c_int64(), C.c_int64()
    st = _L().ora_bounds(C.byref(_mk_layout(L, k)), axis.encode(), C.byref(lo), C.byref(hi))
    if st == EBOUNDS:
        return None
    if st:
        raise OracleError(st, "bounds")
    return lo.value, hi.value


def storage_check(st) -> int:
    k = _Keep()
    return _L().ora_storage_check(C.byref(_mk_storage(st, k)))


def storage_byte(st, coord: dict, es: int) -> int:
    """Byte offset of a coordinate in the storage (after swizzle), -1 if outside the bound box."""
    k = _Keep()
    names = (C.c_char_p * max(1, len(coord)))(*[k.add(a.encode()) for a in coord])
    vals = (C.c_int64 * max(1, len(coord)))(*coord.values())
    return _L().ora_storage_byte(C.byref(_mk_storage(st, k)), len(coord), names, vals, es)


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


def copy(src, src_st, sbuf: np.ndarray, dst, dst_st, dbuf: np.ndarray, es: int, nthreads: int = 1) -> None:
    """dst cells of f_L^dst(x) <- src cell f_D^src(x) + O^src, for every x; dbuf updated in place."""
    k = _Keep()
    st = _L().ora_copy(C.byref(_mk_layout(src, k)), C.byref(_mk_storage(src_st, k)), _ptr(sbuf), sbuf.nbytes,
                       C.byref(_mk_layout(dst, k)), C.byref(_mk_storage(dst_st, k)), _ptr(dbuf), dbuf.nbytes,
                       es, nthreads)
    if st:
        raise OracleError(st, "copy")


def redistribute(src, src_st, sbufs, dst, dst_st, dbufs, es: int, only_rank: int = -1, nthreads: int = 1) -> None:
    """Per-rank buffers; the gpuid coordinate selects the rank.  dbufs[g] may be None
    for g != only_rank when only_rank >= 0."""
    k = _Keep()
    n = len(sbufs)
    assert len(dbufs) == n
    sp = (C.c_void_p * n)(*[_ptr(b).value for b in sbufs])
    dp = (C.c_void_p * n)(*[(_ptr(b).value if b is not None else None) for b in dbufs])
    sbytes = sbufs[0].nbytes
    dbytes = next(b.nbytes for b in dbufs if b is not None)
    st = _L().ora_redistribute(C.byref(_mk_layout(src, k)), C.byref(_mk_storage(src_st, k)), sp, sbytes,
                               C.byref(_mk_layout(dst, k)), C.byref(_mk_storage(dst_st, k)), dp, dbytes, es, n,
                               only_rank, nthreads)
    if st:
        raise OracleError(st, "redistribute")


def scatter_logical(L, st, values_bytes: np.ndarray, es: int, fill: np.ndarray, nthreads: int = 1) -> np.ndarray:
    """Materialise a tensor in layout L: copy from the identity layout (E_D):(1) over the
    logical values into every replica of L (test-input preparation, SURVEY §3 parity test)."""
    ed, _ = sizes(L)
    ident = {"D": [(ed, 1, "m")], "R": [], "O": {}}
    ident_st = {"digits": [("m", ed, 1)], "swizzle": (0, 0, 0)}
    buf = fill.copy()
    copy(ident, ident_st, values_bytes, L, st, buf, es, nthreads)
    return buf


def scatter_ranks(L, st, values_bytes: np.ndarray, es: int, nranks: int, fill: np.ndarray, nthreads: int = 1):
    """Per-rank materialisation of a distributed tensor in layout L (its gpuid coordinate selects
    the rank); every replica is written, so source replicas are consistent (reading R4)."""
    ed, _ = sizes(L)
    ident = {"D": [(ed, 1, "m")], "R": [], "O": {}}
    ident_st = {"digits": [("m", ed, 1)], "swizzle": (0, 0, 0)}
    bufs = [fill.copy() for _ in range(nranks)]
    redistribute(ident, ident_st, [values_bytes] * nranks, L, st, bufs, es, -1, nthreads)
    return bufs


# element types of the reduction (the oracle's own codes; ints add modulo 2^bits)
DTYPES = {"f32": 1, "f64": 2, "f16": 3, "bf16": 4, "i32": 5, "i64": 6}
DTYPE_SIZE = {"f32": 4, "f64": 8, "f16": 2, "bf16": 2, "i32": 4, "i64": 8}


def reduce(src, src_st, sbufs, dst, dst_st, dbufs, dtype: str, nranks: int = 0, only_rank: int = -1,
           nthreads: int = 1) -> None:
    """dst(y) = sum_k src(k * E_D(dst) + y) (reading R24): fp64 sum in k order,
    rounded once to dtype; ints modulo 2^bits.  nranks = 0: sbufs / dbufs are single arrays;
    else per-rank lists selected by the gpuid coordinate (as redistribute)."""
    k = _Keep()
    if nranks == 0:
        sbufs, dbufs = [sbufs], [dbufs]
    n = len(sbufs)
    sp = (C.c_void_p * n)(*[_ptr(b).value for b in sbufs])
    dp = (C.c_void_p * n)(*[(_ptr(b).value if b is not None else None) for b in dbufs])
    dbytes = next(b.nbytes for b in dbufs if b is not None)
    st = _L().ora_reduce(C.byref(_mk_layout(src, k)), C.byref(_mk_storage(src_st, k)), sp, sbufs[0].nbytes,
                         C.byref(_mk_layout(dst, k)), C.byref(_mk_storage(dst_st, k)), dp, dbytes, DTYPES[dtype],
                         nranks, only_rank, nthreads)
    if st:
        raise OracleError(st, "reduce")
