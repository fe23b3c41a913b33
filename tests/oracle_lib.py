"""TEST INFRASTRUCTURE — ctypes bindings for the two CPU checkers.

* ``Oracle``  : oracle/liboracle.so, our plain-C restatement of the reference
  (oracle/h3d_oracle.c).
* ``RefLib``  : oracle/_ref/libh3dref.so, the unmodified reference sources
  compiled in place against oracle/shim (oracle/Makefile, target ``ref``).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
leg import this module, and only as the checker.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE_SO = ROOT / "oracle" / "liboracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libh3dref.so"
# the same reference sources with release flags for an AVX-512 host (timing only)
REF_REL_SO = ROOT / "oracle" / "_ref" / "libh3dref_rel.so"


def host_has_avx512() -> bool:
    try:
        flags = next(l for l in open("/proc/cpuinfo") if l.startswith("flags")).split()
    except (OSError, StopIteration):
        return False
    return all(f in flags for f in ("avx512f", "avx512dq", "avx512cd", "avx512bw", "avx512vl"))

KERNELS = {"laplace3d": 0, "r4": 1, "helmholtz-re": 2}
VARIANTS = {"hodlr3d": 0, "hodlr": 1, "hstrong": 2}  # h3d::Variant order (octree.hpp:80)


def _variant(v) -> int:
    return VARIANTS[v] if isinstance(v, str) else int(v)

_P = C.c_void_p
_D = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_I32 = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_I64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_U64 = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")


class CheckerError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _ptr_or_null(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Oracle:
    """Plain-C restatement (always buildable: `make -C oracle oracle`)."""

    def __init__(self, path: Path = ORACLE_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle oracle`")
        L = C.CDLL(str(path))
        self.L = L
        L.orc_last_error.restype = C.c_char_p
        L.orc_generate_points.argtypes = [C.c_int64, C.c_uint64, _D]
        L.orc_random_vector.argtypes = [C.c_int64, C.c_uint64, _D]
        L.orc_initialize.argtypes = [_D, C.c_int64, C.c_int, C.c_double, C.c_int, C.c_double,
                                     C.c_int, C.c_int64, C.c_int, C.POINTER(_P)]
        L.orc_free.argtypes = [_P]
        L.orc_matvec.argtypes = [_P, _D, _D]
        L.orc_depth.argtypes = [_P]
        L.orc_export_perm.argtypes = [_P, _I32]
        L.orc_export_offsets.argtypes = [_P, C.c_int, _I64]
        L.orc_export_list.argtypes = [_P, C.c_int, C.c_int, _P, _P]
        L.orc_export_list.restype = C.c_int64
        L.orc_lr_blocks.argtypes = [_P, C.c_int, _P, _P, _P]
        L.orc_lr_blocks.restype = C.c_int64
        L.orc_lr_block_detail.argtypes = [_P, C.c_int, C.c_int64, _I32, _I32, _D]
        L.orc_stats.argtypes = [_P, _U64]
        L.orc_reference_error.argtypes = [_P, _D, _D]
        L.orc_reference_error.restype = C.c_double
        L.orc_aca_block.argtypes = [_D, C.c_int64, _D, C.c_int64, C.c_int, C.c_double, C.c_int64,
                                    _I32, _I32, _D, C.c_int64, C.POINTER(C.c_int)]
        L.orc_dense_matvec.argtypes = [_D, C.c_int64, C.c_int, C.c_double, _D, _D]
        L.orc_exact_rows.argtypes = [_D, C.c_int64, C.c_int, C.c_double, _D, _I64, C.c_int64, _D]
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_uniform_stream.argtypes = [C.c_int64, C.c_uint64, _D]
        L.orc_tree_lists.argtypes = [_D, C.c_int64, C.c_int, C.c_int, C.c_int, C.POINTER(_P)]

    def _check(self, st):
        if st != 0:
            raise CheckerError(st, self.L.orc_last_error().decode())

    def uniform_stream(self, n: int, seed: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        self.L.orc_uniform_stream(n, seed, out)
        return out

    def tree_lists(self, pts, n_max=216, depth_cap=12, variant="hodlr3d") -> "OracleRep":
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1)
        h = _P()
        self._check(self.L.orc_tree_lists(pts, len(pts) // 3, n_max, depth_cap, _variant(variant),
                                          C.byref(h)))
        return OracleRep(self, h, len(pts) // 3)

    def set_threads(self, n: int):
        self.L.orc_set_threads(n)

    def generate_points(self, n: int, seed: int) -> np.ndarray:
        out = np.empty(3 * n, dtype=np.float64)
        self._check(self.L.orc_generate_points(n, seed, out))
        return out.reshape(n, 3)

    def random_vector(self, n: int, seed: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        self.L.orc_random_vector(n, seed, out)
        return out

    def dense_matvec(self, pts, x, kernel="laplace3d", diag=0.0):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1)
        x = np.ascontiguousarray(x, dtype=np.float64)
        b = np.empty_like(x)
        self._check(self.L.orc_dense_matvec(pts, len(x), KERNELS[kernel], diag, x, b))
        return b

    def exact_rows(self, pts, x, rows, kernel="laplace3d", diag=0.0):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1)
        x = np.ascontiguousarray(x, dtype=np.float64)
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        out = np.empty(len(rows), dtype=np.float64)
        self._check(self.L.orc_exact_rows(pts, len(x), KERNELS[kernel], diag, x, rows, len(rows), out))
        return out

    def aca_block(self, xs, ys, kernel="laplace3d", eps=1e-7, max_rank=0):
        xs = np.ascontiguousarray(xs, dtype=np.float64).reshape(-1)
        ys = np.ascontiguousarray(ys, dtype=np.float64).reshape(-1)
        m, n = len(xs) // 3, len(ys) // 3
        cap = min(m, n)
        rp = np.empty(cap, np.int32)
        cp = np.empty(cap, np.int32)
        lu = np.empty(cap * cap, np.float64)
        r = C.c_int(0)
        self._check(self.L.orc_aca_block(xs, m, ys, n, KERNELS[kernel], eps, max_rank, rp, cp, lu,
                                         cap, C.byref(r)))
        k = r.value
        return rp[:k].copy(), cp[:k].copy(), lu[: k * k].reshape(k, k).copy()

    def initialize(self, pts, kernel="laplace3d", n_max=216, eps=1e-7, depth_cap=12,
                   max_rank=0, diag=0.0, variant="hodlr3d") -> "OracleRep":
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1)
        h = _P()
        self._check(self.L.orc_initialize(pts, len(pts) // 3, KERNELS[kernel], diag, n_max, eps,
                                          depth_cap, max_rank, _variant(variant), C.byref(h)))
        return OracleRep(self, h, len(pts) // 3)


class OracleRep:
    def __init__(self, lib: Oracle, h, n: int):
        self.lib, self.h, self.n = lib, h, n

    def __del__(self):
        try:
            self.lib.L.orc_free(self.h)
        except Exception:
            pass

    @property
    def depth(self) -> int:
        return self.lib.L.orc_depth(self.h)

    def matvec(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        b = np.empty_like(x)
        self.lib._check(self.lib.L.orc_matvec(self.h, x, b))
        return b

    def perm(self):
        p = np.empty(self.n, np.int32)
        self.lib.L.orc_export_perm(self.h, p)
        return p

    def offsets(self, level):
        o = np.empty((1 << (3 * level)) + 1, np.int64)
        self.lib.L.orc_export_offsets(self.h, level, o)
        return o

    def list(self, level, kind):
        nn = 1 << (3 * level)
        off = np.empty(nn + 1, np.int32)
        tot = self.lib.L.orc_export_list(self.h, level, kind, _ptr_or_null(off), None)
        ids = np.empty(max(tot, 1), np.int32)
        self.lib.L.orc_export_list(self.h, level, kind, _ptr_or_null(off), _ptr_or_null(ids))
        return off, ids[:tot]

    def lr_blocks(self, level):
        k = self.lib.L.orc_lr_blocks(self.h, level, None, None, None)
        t, s, r = (np.empty(max(k, 1), np.int32) for _ in range(3))
        self.lib.L.orc_lr_blocks(self.h, level, _ptr_or_null(t), _ptr_or_null(s), _ptr_or_null(r))
        return t[:k], s[:k], r[:k]

    def lr_block_detail(self, level, k, rank):
        rp = np.empty(max(rank, 1), np.int32)
        cp = np.empty(max(rank, 1), np.int32)
        lu = np.empty(max(rank * rank, 1), np.float64)
        self.lib.L.orc_lr_block_detail(self.h, level, k, rp, cp, lu)
        return rp[:rank], cp[:rank], lu[: rank * rank].reshape(rank, rank)

    def stats(self):
        o = np.empty(5, np.uint64)
        self.lib.L.orc_stats(self.h, o)
        return dict(float_count=int(o[0]), int_count=int(o[1]), memory_bytes=int(o[2]),
                    max_rank=int(o[3]), depth=int(o[4]))

    def reference_error(self, x, b):
        return self.lib.L.orc_reference_error(self.h, np.ascontiguousarray(x, np.float64),
                                              np.ascontiguousarray(b, np.float64))


class RefLib:
    """The unmodified reference compiled in place (oracle/_ref)."""

    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    "/root/reference is mounted")
        L = C.CDLL(str(path))
        self.L = L
        L.h3dref_last_error.restype = C.c_char_p
        L.h3dref_set_threads.argtypes = [C.c_int]
        L.h3dref_generate_points.argtypes = [C.c_int, C.c_int64, C.c_uint64, _D]
        L.h3dref_random_vector.argtypes = [C.c_int64, C.c_uint64, _D]
        L.h3dref_initialize.argtypes = [_D, C.c_int64, C.c_int, C.c_double, C.c_int, C.c_int,
                                        C.c_double, C.c_int, C.c_int, C.c_int64, C.POINTER(_P)]
        L.h3dref_free.argtypes = [_P]
        L.h3dref_tree_lists.argtypes = [_D, C.c_int64, C.c_int, C.c_int, C.POINTER(_P)]
        L.h3dref_matvec.argtypes = [_P, _D, _D, _P]
        L.h3dref_parallel_matvec.argtypes = [_P, _D, C.c_int, _D, _P]
        L.h3dref_reference_error.argtypes = [_P, _D, _D, C.POINTER(C.c_double)]
        L.h3dref_stats.argtypes = [_P, _U64, _P]
        L.h3dref_depth.argtypes = [_P]
        L.h3dref_export_perm.argtypes = [_P, _I32]
        L.h3dref_export_ranges.argtypes = [_P, C.c_int, _I64]
        L.h3dref_export_list.argtypes = [_P, C.c_int, C.c_int, _P, _P]
        L.h3dref_export_list.restype = C.c_int64
        L.h3dref_lr_blocks.argtypes = [_P, C.c_int, _P, _P, _P]
        L.h3dref_lr_blocks.restype = C.c_int64
        L.h3dref_lr_block_detail.argtypes = [_P, C.c_int, C.c_int64, _I32, _I32, _D]
        L.h3dref_dense_blocks.argtypes = [_P, _P, _P, _P]
        L.h3dref_dense_blocks.restype = C.c_int64
        L.h3dref_aca_block.argtypes = [_D, C.c_int64, _D, C.c_int64, C.c_int, C.c_double,
                                       C.c_int64, _I32, _I32, _D, C.c_int64, C.POINTER(C.c_int)]
        L.h3dref_census.argtypes = [_P, _U64]
        L.h3dref_dense_matvec.argtypes = [_D, C.c_int64, C.c_int, C.c_double, _D, _D]
        L.h3dref_cell_self_integral.argtypes = [C.c_double]
        L.h3dref_cell_self_integral.restype = C.c_double
        L.h3dref_ie_experiment.argtypes = [C.c_int, C.c_double, C.c_int, C.c_uint64, C.c_double,
                                           C.c_int, C.c_int, C.POINTER(C.c_int),
                                           C.POINTER(C.c_int), C.POINTER(C.c_double)]
        L.h3dref_max_threads.restype = C.c_int

    def _check(self, st):
        if st != 0:
            raise CheckerError(st, self.L.h3dref_last_error().decode())

    def set_threads(self, n: int):
        self.L.h3dref_set_threads(n)

    def max_threads(self) -> int:
        return self.L.h3dref_max_threads()

    def generate_points(self, n: int, seed: int, dist: int = 0) -> np.ndarray:
        out = np.empty(3 * n, dtype=np.float64)
        self._check(self.L.h3dref_generate_points(dist, n, seed, out))
        return out.reshape(n, 3)

    def random_vector(self, n: int, seed: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        self.L.h3dref_random_vector(n, seed, out)
        return out

    def cell_self_integral(self, h: float) -> float:
        return float(self.L.h3dref_cell_self_integral(float(h)))

    def ie_experiment(self, grid_n: int, eps: float, n_max: int = 216, seed: int = 0,
                      tol: float = 1e-10, restart: int = 0, max_iter: int = 500) -> dict:
        """reference solver.cpp:243-300 (HODLR3D, laplace3d)."""
        it, cv, fe = C.c_int(0), C.c_int(0), C.c_double(0.0)
        self._check(self.L.h3dref_ie_experiment(grid_n, eps, n_max, seed, tol, restart, max_iter,
                                                C.byref(it), C.byref(cv), C.byref(fe)))
        return {"iterations": it.value, "converged": bool(cv.value), "forward_error": fe.value}

    def dense_matvec(self, pts, x, kernel="laplace3d", diag=0.0):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1)
        x = np.ascontiguousarray(x, dtype=np.float64)
        b = np.empty_like(x)
        self._check(self.L.h3dref_dense_matvec(pts, len(x), KERNELS[kernel], diag, x, b))
        return b

    def aca_block(self, xs, ys, kernel="laplace3d", eps=1e-7, max_rank=0):
        xs = np.ascontiguousarray(xs, dtype=np.float64).reshape(-1)
        ys = np.ascontiguousarray(ys, dtype=np.float64).reshape(-1)
        m, n = len(xs) // 3, len(ys) // 3
        cap = min(m, n)
        rp = np.empty(cap, np.int32)
        cp = np.empty(cap, np.int32)
        lu = np.empty(cap * cap, np.float64)
        r = C.c_int(0)
        self._check(self.L.h3dref_aca_block(xs, m, ys, n, KERNELS[kernel], eps, max_rank, rp, cp,
                                            lu, cap, C.byref(r)))
        k = r.value
        return rp[:k].copy(), cp[:k].copy(), lu[: k * k].reshape(k, k).copy()

    def tree_lists(self, pts, n_max=216, variant=0) -> "RefRep":
        """build_tree + build_interaction_lists only (octree.cpp:76-260)."""
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1)
        h = _P()
        self._check(self.L.h3dref_tree_lists(pts, len(pts) // 3, n_max, _variant(variant), C.byref(h)))
        return RefRep(self, h, len(pts) // 3)

    def initialize(self, pts, kernel="laplace3d", n_max=216, eps=1e-7, depth_cap=12,
                   max_rank=0, diag=0.0, variant=0, cached=False) -> "RefRep":
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1)
        h = _P()
        self._check(self.L.h3dref_initialize(pts, len(pts) // 3, KERNELS[kernel], diag,
                                             _variant(variant),
                                             n_max, eps, int(cached), depth_cap, max_rank,
                                             C.byref(h)))
        return RefRep(self, h, len(pts) // 3)


class RefRep:
    def __init__(self, lib: RefLib, h, n: int):
        self.lib, self.h, self.n = lib, h, n

    def __del__(self):
        try:
            self.lib.L.h3dref_free(self.h)
        except Exception:
            pass

    @property
    def depth(self) -> int:
        return self.lib.L.h3dref_depth(self.h)

    def matvec(self, x, timing=False):
        x = np.ascontiguousarray(x, dtype=np.float64)
        b = np.empty_like(x)
        t = np.zeros(3, np.float64)
        self.lib._check(self.lib.L.h3dref_matvec(self.h, x, b, t.ctypes.data_as(C.c_void_p)))
        return (b, t) if timing else b

    def parallel_matvec(self, x, n_p):
        x = np.ascontiguousarray(x, dtype=np.float64)
        b = np.empty_like(x)
        led = np.zeros(3, np.uint64)
        self.lib._check(self.lib.L.h3dref_parallel_matvec(self.h, x, n_p, b,
                                                          led.ctypes.data_as(C.c_void_p)))
        return b, led

    def perm(self):
        p = np.empty(self.n, np.int32)
        self.lib.L.h3dref_export_perm(self.h, p)
        return p

    def offsets(self, level):
        nn = 1 << (3 * level)
        r = np.empty(2 * nn, np.int64)
        self.lib.L.h3dref_export_ranges(self.h, level, r)
        r = r.reshape(nn, 2)
        assert np.all(r[1:, 0] == r[:-1, 1])
        return np.concatenate([r[:, 0], r[-1:, 1]])

    def list(self, level, kind):
        nn = 1 << (3 * level)
        off = np.empty(nn + 1, np.int32)
        tot = self.lib.L.h3dref_export_list(self.h, level, kind, _ptr_or_null(off), None)
        ids = np.empty(max(tot, 1), np.int32)
        self.lib.L.h3dref_export_list(self.h, level, kind, _ptr_or_null(off), _ptr_or_null(ids))
        return off, ids[:tot]

    def lr_blocks(self, level):
        k = self.lib.L.h3dref_lr_blocks(self.h, level, None, None, None)
        t, s, r = (np.empty(max(k, 1), np.int32) for _ in range(3))
        self.lib.L.h3dref_lr_blocks(self.h, level, _ptr_or_null(t), _ptr_or_null(s), _ptr_or_null(r))
        return t[:k], s[:k], r[:k]

    def lr_block_detail(self, level, k, rank):
        rp = np.empty(max(rank, 1), np.int32)
        cp = np.empty(max(rank, 1), np.int32)
        lu = np.empty(max(rank * rank, 1), np.float64)
        self.lib.L.h3dref_lr_block_detail(self.h, level, k, rp, cp, lu)
        return rp[:rank], cp[:rank], lu[: rank * rank].reshape(rank, rank)

    def dense_blocks(self):
        k = self.lib.L.h3dref_dense_blocks(self.h, None, None, None)
        t, s, c = (np.empty(max(k, 1), np.int32) for _ in range(3))
        self.lib.L.h3dref_dense_blocks(self.h, _ptr_or_null(t), _ptr_or_null(s), _ptr_or_null(c))
        return t[:k], s[:k], c[:k]

    def stats(self):
        o = np.empty(5, np.uint64)
        secs = np.zeros(3, np.float64)
        self.lib.L.h3dref_stats(self.h, o, secs.ctypes.data_as(C.c_void_p))
        return dict(float_count=int(o[0]), int_count=int(o[1]), memory_bytes=int(o[2]),
                    max_rank=int(o[3]), depth=int(o[4]), init_seconds=float(secs[0]),
                    aca_seconds=float(secs[1]), dense_form_seconds=float(secs[2]))

    def census(self):
        o = np.empty(8, np.uint64)
        self.lib.L.h3dref_census(self.h, o)
        keys = ["dense", "lowrank", "ws", "vertex", "edge", "face", "coverage_area", "n_squared"]
        return {k: int(v) for k, v in zip(keys, o)}

    def reference_error(self, x, b):
        out = C.c_double(0.0)
        self.lib._check(self.lib.L.h3dref_reference_error(
            self.h, np.ascontiguousarray(x, np.float64), np.ascontiguousarray(b, np.float64),
            C.byref(out)))
        return out.value


def have_ref() -> bool:
    return REF_SO.exists()


def have_oracle() -> bool:
    return ORACLE_SO.exists()
