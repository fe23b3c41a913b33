"""Python host mirror of the reference HODLR3D C++ API over the C-ABI.

The reference operator surface for this path (proj/include/h3d/hmatrix.hpp)::

    HMatrixRep initialize(const PointSet&, const KernelSpec&, Variant, const HmatOptions&)
    std::vector<double> matvec(const HMatrixRep&, std::span<const double> x, MatvecTiming*)
    RepStats stats(const HMatrixRep&)

is mirrored here with the same names, argument meaning and error behaviour
(``std::invalid_argument`` -> ``ValueError``; ``DegenerateGeometryError`` and
``DegenerateDistributionError`` keep their names). Everything runs through
``lib/libh3d_b200.so`` (include/h3d_b200.h); there is no CPU fallback: without
the built library, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from pathlib import Path
from typing import Optional

import numpy as np

# H3D_LIB_PATH: developer override (tuning builds of the same library)
_LIB_PATH = Path(os.environ.get("H3D_LIB_PATH") or
                 Path(__file__).resolve().parent / "lib" / "libh3d_b200.so")

KERNELS = {"laplace3d": 0, "r4": 1, "helmholtz-re": 2}
VARIANTS = {"hodlr3d": 0, "hodlr": 1, "hstrong": 2}  # h3d::Variant order (octree.hpp:80)
NEAR_STORED, NEAR_MATRIX_FREE = 0, 1


class DegenerateGeometryError(RuntimeError):
    """Coincident distinct points (reference kernel.hpp:64-66)."""


class DegenerateDistributionError(RuntimeError):
    """Depth cap exceeded (reference octree.hpp:41-43)."""


class DeviceError(RuntimeError):
    """CUDA / NCCL / allocation failure inside the engine."""


class _Options(C.Structure):
    _fields_ = [
        ("kernel_id", C.c_int),
        ("diagonal", C.c_double),
        ("n_max", C.c_int),
        ("epsilon", C.c_double),
        ("depth_cap", C.c_int),
        ("max_rank", C.c_int64),
        ("near_mode", C.c_int),
        ("device", C.c_int),
        ("shard_rank", C.c_int),
        ("shard_world", C.c_int),
        ("mode_policy", C.c_int),
        ("level_modes", C.c_int * 16),
        ("variant", C.c_int),
        ("gather_b", C.c_int64),
        ("reserved", C.c_int64 * 3),
    ]


class _CommLedger(C.Structure):
    _fields_ = [
        ("x_gather_doubles", C.c_int64),
        ("b_gather_doubles", C.c_int64),
        ("collectives", C.c_int64),
        ("matvecs", C.c_int64),
        ("reserved", C.c_int64 * 4),
    ]


class _Timing(C.Structure):
    _fields_ = [
        ("total_ms", C.c_double),
        ("h2d_ms", C.c_double),
        ("gather_ms", C.c_double),
        ("exchange_ms", C.c_double),
        ("phase1_ms", C.c_double),
        ("phase2_ms", C.c_double),
        ("d2h_ms", C.c_double),
        ("launches", C.c_int64),
        ("device_ms", C.c_double),
    ]


class _Stats(C.Structure):
    _fields_ = [
        ("depth", C.c_int),
        ("max_rank", C.c_int),
        ("n", C.c_int64),
        ("lowrank_blocks", C.c_int64),
        ("aca_pairs", C.c_int64),
        ("sum_rank", C.c_int64),
        ("factor_doubles", C.c_int64),
        ("factor_bytes_alloc", C.c_int64),
        ("tvec_doubles", C.c_int64),
        ("near_blocks", C.c_int64),
        ("near_entries", C.c_int64),
        ("near_bytes_stored", C.c_int64),
        ("ref_float_count", C.c_uint64),
        ("ref_int_count", C.c_uint64),
        ("compression_ratio", C.c_double),
        ("build_ms_tree", C.c_double),
        ("build_ms_lists", C.c_double),
        ("build_ms_aca_rank", C.c_double),
        ("build_ms_aca_write", C.c_double),
        ("build_ms_total", C.c_double),
        ("phase1_items", C.c_int64),
        ("owned_row_begin", C.c_int64),
        ("owned_row_end", C.c_int64),
        ("level_modes", C.c_int * 16),
        ("proxy_units", C.c_int64),
        ("direct_evals", C.c_int64),
        ("lu_doubles", C.c_int64),
        ("level_units", C.c_int64 * 16),
        ("level_aca_ms", C.c_double * 16),
        ("build_ms_plan", C.c_double),
        ("build_ms_post", C.c_double),
        ("build_ms_near", C.c_double),
        ("half_units", C.c_int64),
    ]


_EXPORTS = [
    "h3d_last_error", "h3d_abi_version", "h3d_default_options", "h3d_generate_points",
    "h3d_random_vector", "h3d_dev_create", "h3d_dev_destroy", "h3d_dev_matvec",
    "h3d_dev_stats", "h3d_dev_export_tree", "h3d_dev_export_list", "h3d_dev_export_pairs",
    "h3d_nccl_get_id", "h3d_dev_attach_nccl", "h3d_dev_matvec_async", "h3d_dev_profile",
    "h3d_dev_profile_read", "h3d_dev_profile_kernels", "h3d_plan_create", "h3d_plan_destroy", "h3d_plan_pairs",
    "h3d_plan_set_ranks", "h3d_plan_set_mode", "h3d_plan_layout", "h3d_plan_array",
    "h3d_dev_gmres", "h3d_dev_direct_matvec", "h3d_generate_grid_points", "h3d_cell_self_integral",
    "h3d_dev_reference_error", "h3d_dev_comm_ledger",
]


class _GmresInfo(C.Structure):
    _fields_ = [
        ("iterations", C.c_int),
        ("converged", C.c_int),
        ("history_len", C.c_int),
        ("reserved", C.c_int),
        ("solve_ms", C.c_double),
        ("final_relres", C.c_double),
    ]


def _load():
    if not _LIB_PATH.exists():
        raise ImportError(
            f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (or `make -C paper_2307_16303_b200/csrc`). There is no CPU fallback.")
    L = C.CDLL(str(_LIB_PATH))
    P = C.c_void_p
    L.h3d_last_error.restype = C.c_char_p
    L.h3d_default_options.argtypes = [C.POINTER(_Options)]
    L.h3d_generate_points.argtypes = [C.c_int64, C.c_uint64, P]
    L.h3d_random_vector.argtypes = [C.c_int64, C.c_uint64, P]
    L.h3d_dev_create.argtypes = [P, C.c_int64, C.POINTER(_Options), C.POINTER(P)]
    L.h3d_dev_destroy.argtypes = [P]
    L.h3d_dev_matvec.argtypes = [P, P, P, C.c_int, C.POINTER(_Timing)]
    L.h3d_dev_stats.argtypes = [P, C.POINTER(_Stats)]
    L.h3d_dev_export_tree.argtypes = [P, P, C.c_int, P]
    L.h3d_dev_export_list.argtypes = [P, C.c_int, C.c_int, P, P, C.POINTER(C.c_int64)]
    L.h3d_dev_export_pairs.argtypes = [P, C.c_int, P, P, P, C.POINTER(C.c_int64)]
    L.h3d_dev_matvec_async.argtypes = [P, P, P, P]
    L.h3d_dev_profile.argtypes = [P, C.c_int, C.c_int64]
    L.h3d_dev_profile_read.argtypes = [P, C.POINTER(_Timing), C.POINTER(C.c_int64)]
    L.h3d_dev_profile_kernels.argtypes = [P, P, P, P, C.c_int]
    L.h3d_plan_create.argtypes = [C.c_int, C.c_int64, P, P, P, P, C.c_int, C.c_int, P,
                                  C.POINTER(P)]
    L.h3d_plan_destroy.argtypes = [P]
    L.h3d_plan_pairs.argtypes = [P, C.c_int, P, P, C.POINTER(C.c_int64)]
    L.h3d_plan_set_ranks.argtypes = [P, C.c_int, P]
    L.h3d_plan_set_mode.argtypes = [P, C.c_int, C.c_int]
    L.h3d_plan_layout.argtypes = [P]
    L.h3d_plan_array.argtypes = [P, C.c_char_p, C.c_int, P, C.POINTER(C.c_int64)]
    L.h3d_nccl_get_id.argtypes = [P]
    L.h3d_dev_attach_nccl.argtypes = [P, P, C.c_int, C.c_int]
    L.h3d_dev_gmres.argtypes = [P, P, P, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int,
                                C.c_int, P, C.c_int, C.POINTER(_GmresInfo)]
    L.h3d_dev_direct_matvec.argtypes = [P, P, P, C.c_int]
    L.h3d_dev_comm_ledger.argtypes = [P, C.POINTER(_CommLedger)]
    L.h3d_dev_reference_error.argtypes = [P, P, P, C.c_int, C.c_int64, C.c_int64, C.c_uint64,
                                          C.POINTER(C.c_double)]
    L.h3d_generate_grid_points.argtypes = [C.c_int64, P]
    L.h3d_cell_self_integral.argtypes = [C.c_double]
    L.h3d_cell_self_integral.restype = C.c_double
    return L


_L = _load()


def library_path() -> str:
    return str(_LIB_PATH)


def exported_symbols():
    return list(_EXPORTS)


def _raise(code: int):
    msg = _L.h3d_last_error().decode()
    if code == 1 or code == 7:
        raise ValueError(msg)
    if code == 2:
        raise DegenerateGeometryError(msg)
    if code == 3:
        raise DegenerateDistributionError(msg)
    raise DeviceError(f"[status {code}] {msg}")


def _check(code: int):
    if code != 0:
        _raise(code)


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


# ---------------------------------------------------------------- inputs
def generate_points(n: int, seed: int) -> np.ndarray:
    """generate_points(UniformRandom, n, seed) (reference kernel.cpp:88-95), (n, 3)."""
    out = np.empty((n, 3), dtype=np.float64)
    _check(_L.h3d_generate_points(n, seed, _ptr(out)))
    return out


def random_vector(n: int, seed: int) -> np.ndarray:
    """mt19937_64(seed), 2u-1 (reference tools/h3d.cpp:135-137)."""
    out = np.empty(n, dtype=np.float64)
    _L.h3d_random_vector(n, seed, _ptr(out))
    return out


# ---------------------------------------------------------------- options
@dataclasses.dataclass
class KernelSpec:
    """Built-in radial kernel (reference kernel.hpp:46-53)."""

    name: str = "laplace3d"
    diagonal: float = 0.0

    @property
    def id(self) -> int:
        if self.name not in KERNELS:
            raise ValueError(f"unknown kernel: {self.name}")
        return KERNELS[self.name]


def make_kernel(name: str, diagonal: float = 0.0) -> KernelSpec:
    """parse_kernel (reference kernel.cpp:52-57): laplace3d, r4, helmholtz-re."""
    if name not in KERNELS:
        raise ValueError(f"unknown kernel: {name}")
    return KernelSpec(name, diagonal)


@dataclasses.dataclass
class HmatOptions:
    """Reference hmatrix.hpp:16-22. dense_mode: "cached" stores the near field,
    "on-the-fly" recomputes it every matvec (matrix-free)."""

    n_max: int = 216
    epsilon: float = 1e-7
    dense_mode: str = "on-the-fly"
    depth_cap: int = 12
    max_rank: int = 0
    # B200 extension: "auto" (cost model), "stream"
    # (explicit factors everywhere) or "explicit" (level_modes[l]: 0 stream,
    # 1 proxy, 2 direct at the leaf level, 3 pair = explicit factors applied in
    # one fused read per pair, 4 fused, 5 half = U' = K(X, tau) (LR)^-1
    # streamed and K(sigma, Y) regenerated, laplace3d / r4 only, 6 split =
    # proxy storage, the Y-role entries evaluated once for both uses)
    mode_policy: str = "auto"
    level_modes: tuple = ()
    # multi-GPU (B200 extension): every rank returns the full b, all-gathered
    # over NCCL after the matvec (parallel_matvec's final gather, parallel.cpp:284-290)
    gather_b: bool = False


@dataclasses.dataclass
class MatvecTiming:
    total_ms: float = 0.0
    h2d_ms: float = 0.0
    gather_ms: float = 0.0
    exchange_ms: float = 0.0
    phase1_ms: float = 0.0
    phase2_ms: float = 0.0
    d2h_ms: float = 0.0
    launches: int = 0
    device_ms: float = 0.0  # graph replay: the device time (no per-phase split)


class HMatrixRep:
    """Device-resident HODLR3D representation (reference hmatrix.hpp:37-55)."""

    def __init__(self, points, kernel: KernelSpec, options: HmatOptions, device: int = 0,
                 shard_rank: int = 0, shard_world: int = 1, variant: str = "hodlr3d"):
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        o = _Options()
        _L.h3d_default_options(C.byref(o))
        o.kernel_id = kernel.id
        o.diagonal = float(kernel.diagonal)
        o.n_max = int(options.n_max)
        o.epsilon = float(options.epsilon)
        o.depth_cap = int(options.depth_cap)
        o.max_rank = int(options.max_rank)
        if options.dense_mode not in ("cached", "on-the-fly"):
            raise ValueError(f"unknown dense_mode: {options.dense_mode}")
        o.near_mode = NEAR_STORED if options.dense_mode == "cached" else NEAR_MATRIX_FREE
        o.device = int(device)
        o.shard_rank = int(shard_rank)
        o.shard_world = int(shard_world)
        policies = {"stream": 0, "auto": 1, "explicit": 2}
        if options.mode_policy not in policies:
            raise ValueError(f"unknown mode_policy: {options.mode_policy}")
        o.mode_policy = policies[options.mode_policy]
        for l, m in enumerate(options.level_modes):
            if l < 16:
                o.level_modes[l] = int(m)
        if variant not in VARIANTS:
            raise ValueError(f"unknown variant: {variant}")
        o.variant = VARIANTS[variant]
        o.gather_b = 1 if options.gather_b else 0
        h = C.c_void_p()
        self._h = None
        _check(_L.h3d_dev_create(_ptr(pts), len(pts), C.byref(o), C.byref(h)))
        self._h = h
        self.kernel = kernel
        self.options = options
        self.variant = variant
        self.n = len(pts)
        self.device = device
        self.shard_rank, self.shard_world = shard_rank, shard_world

    def close(self):
        if getattr(self, "_h", None):
            _L.h3d_dev_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- matvec -------------------------------------------------------------
    def matvec(self, x, out: Optional[np.ndarray] = None, timing: Optional[MatvecTiming] = None):
        """b = A~ x in original point order (reference hmatrix.cpp:153-226)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.ndim != 1 or len(x) != self.n:
            raise ValueError("matvec: vector length != N")
        b = out if out is not None else np.empty(self.n, dtype=np.float64)
        t = _Timing()
        _check(_L.h3d_dev_matvec(self._h, _ptr(x), _ptr(b), 0, C.byref(t)))
        if timing is not None:
            for f, _ in _Timing._fields_:
                setattr(timing, f, getattr(t, f))
        return b

    def matvec_ptr(self, x_ptr: int, b_ptr: int, host: bool, timing: Optional[MatvecTiming] = None):
        """Raw-pointer matvec (device pointers for torch CUDA tensors, or pinned host)."""
        t = _Timing()
        _check(_L.h3d_dev_matvec(self._h, C.c_void_p(x_ptr), C.c_void_p(b_ptr), 0 if host else 1,
                                 C.byref(t)))
        if timing is not None:
            for f, _ in _Timing._fields_:
                setattr(timing, f, getattr(t, f))
        return t

    def matvec_async(self, x_ptr: int, b_ptr: int, stream: int = 0):
        """Enqueue b = A~ x on a CUDA stream (device pointers, no sync)."""
        _check(_L.h3d_dev_matvec_async(self._h, C.c_void_p(x_ptr), C.c_void_p(b_ptr),
                                       C.c_void_p(stream)))

    def profile(self, enable: bool, capacity: int = 1024):
        _check(_L.h3d_dev_profile(self._h, int(enable), int(capacity)))

    def profile_read(self):
        """(summed MatvecTiming over recorded async calls, number of calls)."""
        t = _Timing()
        steps = C.c_int64(0)
        _check(_L.h3d_dev_profile_read(self._h, C.byref(t), C.byref(steps)))
        out = MatvecTiming()
        for f, _ in _Timing._fields_:
            setattr(out, f, getattr(t, f))
        return out, steps.value

    def profile_kernels(self) -> dict:
        """Per-kernel (summed ms, launches, summed start offset ms) of the calls
        read by the last profile_read, keyed by KERNEL_SLOTS (kernels of
        different lanes overlap)."""
        ms = np.zeros(len(KERNEL_SLOTS))
        cnt = np.zeros(len(KERNEL_SLOTS), np.int64)
        st = np.zeros(len(KERNEL_SLOTS))
        _check(_L.h3d_dev_profile_kernels(self._h, _ptr(ms), _ptr(cnt), _ptr(st), len(KERNEL_SLOTS)))
        return {k: (float(ms[i]), int(cnt[i]), float(st[i])) for i, k in enumerate(KERNEL_SLOTS)}

    # --- introspection ------------------------------------------------------
    def stats(self) -> dict:
        s = _Stats()
        _check(_L.h3d_dev_stats(self._h, C.byref(s)))
        out = {}
        for f, _ in _Stats._fields_:
            if f == "reserved":
                continue
            v = getattr(s, f)
            out[f] = list(v) if f in ("level_modes", "level_units", "level_aca_ms") else v
        L = out["depth"]
        for f in ("level_modes", "level_units", "level_aca_ms"):
            out[f] = out[f][: L + 1]
        return out

    @property
    def depth(self) -> int:
        return self.stats()["depth"]

    def perm(self) -> np.ndarray:
        p = np.empty(self.n, np.int32)
        _check(_L.h3d_dev_export_tree(self._h, _ptr(p), -1, None))
        return p

    def offsets(self, level: int) -> np.ndarray:
        o = np.empty((1 << (3 * level)) + 1, np.int64)
        _check(_L.h3d_dev_export_tree(self._h, None, level, _ptr(o)))
        return o

    def list(self, level: int, kind: int):
        """Interaction list CSR (kind 0 inter, 1 near_edge, 2 near_face, 3 near_vertex)."""
        nn = 1 << (3 * level)
        off = np.empty(nn + 1, np.int32)
        cnt = C.c_int64(0)
        _check(_L.h3d_dev_export_list(self._h, level, kind, _ptr(off), None, C.byref(cnt)))
        ids = np.empty(max(cnt.value, 1), np.int32)
        _check(_L.h3d_dev_export_list(self._h, level, kind, _ptr(off), _ptr(ids), C.byref(cnt)))
        return off, ids[: cnt.value]

    def pairs(self, level: int):
        cnt = C.c_int64(0)
        _check(_L.h3d_dev_export_pairs(self._h, level, None, None, None, C.byref(cnt)))
        k = cnt.value
        x, y, r = (np.empty(max(k, 1), np.int32) for _ in range(3))
        _check(_L.h3d_dev_export_pairs(self._h, level, _ptr(x), _ptr(y), _ptr(r), C.byref(cnt)))
        return x[:k], y[:k], r[:k]

    # --- multi-GPU ----------------------------------------------------------
    def attach_nccl(self, unique_id: bytes, rank: int, world: int):
        buf = (C.c_char * 128).from_buffer_copy(unique_id)
        _check(_L.h3d_dev_attach_nccl(self._h, C.cast(buf, C.c_void_p), rank, world))


    def comm_ledger(self) -> dict:
        """Per-rank exchange volume per matvec (analogue of h3d::CommLedger,
        parallel.hpp:38-51)."""
        c = _CommLedger()
        _check(_L.h3d_dev_comm_ledger(self._h, C.byref(c)))
        return {f: getattr(c, f) for f, _ in _CommLedger._fields_ if f != "reserved"}

    # --- solver -------------------------------------------------------------
    def gmres(self, rhs, alpha: float = 0.0, beta: float = 1.0,
              options: Optional["GmresOptions"] = None) -> "GmresResult":
        """Device GMRES on (alpha I + beta A~) x = rhs (reference solver.cpp:22-125
        over IEOperator::apply, solver.cpp:199-206). Host vectors, original order."""
        opt = options or GmresOptions()
        f = np.ascontiguousarray(rhs, dtype=np.float64)
        if f.ndim != 1 or len(f) != self.n:
            raise ValueError("gmres: rhs length != N")
        x = np.empty(self.n, dtype=np.float64)
        cap = max(int(opt.max_iter), 1)
        hist = np.zeros(cap, dtype=np.float64)
        info = _GmresInfo()
        _check(_L.h3d_dev_gmres(self._h, _ptr(f), _ptr(x), 0, float(alpha), float(beta),
                                float(opt.tol), int(opt.restart), int(opt.max_iter), _ptr(hist), cap,
                                C.byref(info)))
        return GmresResult(x=x, iterations=info.iterations, converged=bool(info.converged),
                           residual_history=hist[: min(info.history_len, cap)].copy(),
                           solve_ms=info.solve_ms, final_relres=info.final_relres)

    def direct_matvec(self, x) -> np.ndarray:
        """Exact dense b = K x on the device, O(N^2) (reference solver.cpp:247-258)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.ndim != 1 or len(x) != self.n:
            raise ValueError("direct_matvec: vector length != N")
        b = np.empty(self.n, dtype=np.float64)
        _check(_L.h3d_dev_direct_matvec(self._h, _ptr(x), _ptr(b), 0))
        return b


    def reference_error(self, x, b_approx, exact_limit: int = 4096, sample_rows: int = 2000,
                        seed: int = 7) -> float:
        """Relative 2-norm error of b_approx against exact row sums, rows drawn
        as the reference does (hmatrix.hpp:87-93, hmatrix.cpp:253-291)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        b = np.ascontiguousarray(b_approx, dtype=np.float64)
        if x.shape != (self.n,) or b.shape != (self.n,):
            raise ValueError("reference_error: length mismatch")
        out = C.c_double(0.0)
        _check(_L.h3d_dev_reference_error(self._h, _ptr(x), _ptr(b), 0, int(exact_limit),
                                          int(sample_rows), int(seed), C.byref(out)))
        return out.value


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(_L.h3d_nccl_get_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


def initialize(points, kernel: KernelSpec, variant: str = "hodlr3d",
               options: Optional[HmatOptions] = None, device: int = 0, shard_rank: int = 0,
               shard_world: int = 1) -> HMatrixRep:
    """Reference hmatrix.hpp:57-58; variant "hodlr3d", "hodlr" or "hstrong"
    (parse_variant, octree.cpp:180-185)."""
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant: {variant}")
    if len(np.asarray(points).reshape(-1, 3)) == 0:
        raise ValueError("initialize: empty point set")
    return HMatrixRep(points, kernel, options or HmatOptions(), device, shard_rank, shard_world,
                      variant)


def matvec(rep: HMatrixRep, x, timing: Optional[MatvecTiming] = None) -> np.ndarray:
    return rep.matvec(x, timing=timing)


def stats(rep: HMatrixRep) -> dict:
    return rep.stats()


def reference_error(rep: HMatrixRep, x, b_approx, exact_limit: int = 4096, sample_rows: int = 2000,
                    seed: int = 7) -> float:
    """Reference hmatrix.hpp:87-93."""
    return rep.reference_error(x, b_approx, exact_limit, sample_rows, seed)


# ---------------------------------------------------------------- IE solver
@dataclasses.dataclass
class GmresOptions:
    """Reference solver.hpp:10-14."""

    tol: float = 1e-10
    restart: int = 0
    max_iter: int = 500


@dataclasses.dataclass
class GmresResult:
    """Reference solver.hpp:16-21 (+ device timing and the true final residual)."""

    x: np.ndarray
    iterations: int = 0
    converged: bool = False
    residual_history: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(0))
    solve_ms: float = 0.0
    final_relres: float = 0.0


def generate_grid_points(n: int) -> np.ndarray:
    """generate_points(TensorGrid, n) (reference kernel.cpp:96-109): cell centres
    of the side^3 partition of [-1,1]^3 (n must be a perfect cube), z fastest, (n, 3)."""
    out = np.empty((n, 3), dtype=np.float64)
    _check(_L.h3d_generate_grid_points(int(n), _ptr(out)))
    return out


def cell_self_integral(h: float) -> float:
    """Integral of 1/r over a cube of side h about its centre (reference solver.cpp:127-197)."""
    return float(_L.h3d_cell_self_integral(float(h)))


class IEOperator:
    """d I + w K_offdiag on the grid_n^3 collocation grid (reference solver.hpp:35-53)."""

    def __init__(self, n: int, kernel: KernelSpec, eps: float, variant: str = "hodlr3d",
                 base: Optional[HmatOptions] = None, device: int = 0):
        if n < 2:
            raise ValueError("discretize_ie: n must be >= 2")
        if kernel.name != "laplace3d":
            raise ValueError("discretize_ie: unsupported kernel (only laplace3d has the singular "
                             "cell quadrature wired)")
        self.grid_n = n
        self.size = n * n * n
        h = 2.0 / n
        self.cell_volume = h * h * h
        self.diagonal = 1.0 + cell_self_integral(h)
        self.collocation = generate_grid_points(self.size)
        opts = dataclasses.replace(base or HmatOptions(), epsilon=eps)
        self.rep = initialize(self.collocation, kernel, variant, opts, device=device)

    def apply(self, x) -> np.ndarray:
        """solver.cpp:199-206: d x + w A~ x."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        return self.diagonal * x + self.cell_volume * self.rep.matvec(x)

    def dense_matrix(self, max_n: int = 24) -> np.ndarray:
        """Dense assembly for cross-checks, guarded to small grids (reference
        solver.cpp:208-216; host numpy, not the device path)."""
        if self.grid_n > max_n:
            raise ValueError("dense_matrix: grid too large for dense assembly")
        p = self.collocation
        d = p[:, None, :] - p[None, :, :]
        r = np.sqrt(np.einsum("ijk,ijk->ij", d, d))
        np.fill_diagonal(r, 1.0)
        a = self.cell_volume / r
        np.fill_diagonal(a, self.diagonal)
        return a

    def solve(self, f, options: Optional[GmresOptions] = None) -> GmresResult:
        return self.rep.gmres(f, alpha=self.diagonal, beta=self.cell_volume, options=options)

    def close(self):
        self.rep.close()


def discretize_ie(n: int, kernel: KernelSpec, eps: float, variant: str = "hodlr3d",
                  base: Optional[HmatOptions] = None, device: int = 0) -> IEOperator:
    """Reference solver.cpp:218-240."""
    return IEOperator(n, kernel, eps, variant, base, device)


@dataclasses.dataclass
class IeReport:
    """Reference solver.hpp:55-65 (solve time in seconds, device-resident GMRES)."""

    variant: str = "hodlr3d"
    grid_n: int = 0
    size: int = 0
    epsilon: float = 0.0
    iterations: int = 0
    converged: bool = False
    solve_seconds: float = 0.0
    forward_error: float = 0.0
    seed: int = 0


def ie_experiment(n: int, kernel: KernelSpec, eps: float, variant: str = "hodlr3d", seed: int = 0,
                  base: Optional[HmatOptions] = None,
                  gmres_opt: Optional[GmresOptions] = None, device: int = 0) -> IeReport:
    """Manufactured-solution protocol (reference solver.cpp:243-300): sigma from
    mt19937_64(seed), f = d sigma + w (K sigma) by exact dense row sums on the
    device, GMRES over the hierarchical operator, relative forward error."""
    op = discretize_ie(n, kernel, eps, variant, base, device)
    try:
        sigma = random_vector(op.size, seed)
        f = op.diagonal * sigma + op.cell_volume * op.rep.direct_matvec(sigma)
        sol = op.solve(f, gmres_opt)
    finally:
        op.close()
    err = float(np.sqrt(np.sum((sol.x - sigma) ** 2) / np.sum(sigma * sigma)))
    return IeReport(variant=variant, grid_n=n, size=op.size, epsilon=eps,
                    iterations=sol.iterations, converged=sol.converged,
                    solve_seconds=sol.solve_ms * 1e-3, forward_error=err, seed=seed)


# ---------------------------------------------------------------- host planner
# h3d_kernel_slot order (include/h3d_b200.h)
KERNEL_SLOTS = ("gather", "p1_stream", "red_stream", "p2_stream", "p1_proxy", "red_proxy", "solve",
                "p2_proxy", "near", "combine", "pair", "fused", "half")

_PLAN_DTYPES = {
    "woff": np.int64, "soff": np.int64, "rowbeg": np.int64, "rpad": np.int32, "rows": np.int32,
    "spos": np.int32, "pair_wx": np.int64, "pair_wy": np.int64, "pair_rx": np.int32,
    "pair_ry": np.int32, "pair_cx": np.int32, "pair_cy": np.int32, "pair_piv": np.int64, "pair_lu": np.int64, "near_off": np.int32,
    "near_ids": np.int32, "near_dense": np.int32, "sym_off": np.int32, "sym_ids": np.int32,
    "sym_cnt": np.int32, "out_off": np.int64, "in_off": np.int32, "in_pos": np.int64, "node_base": np.int64, "vbase": np.int64, "modes": np.int32, "ranges": np.int64,
    "rank_rows": np.int64, "sizes": np.int64,
    # structs, decoded as int64 fields (see csrc/planner.h)
    "h2_items": np.dtype([("node", np.int32), ("row0", np.int32), ("nrows", np.int32), ("slot", np.int32),
                          ("pslot", np.int64)]),
    "proxy_segs": np.dtype([("so", np.int64), ("base", np.int64), ("piv_off", np.int64),
                            ("lu_off", np.int64), ("r", np.int32), ("side", np.int32),
                            ("solve", np.int32), ("pad", np.int32)]),
    "items": np.dtype([("node", np.int32), ("row0", np.int32), ("nrows", np.int32),
                       ("col0", np.int32), ("ncols", np.int32), ("kind", np.int32),
                       ("pslot", np.int64)]),
    "reds": np.dtype([("node", np.int32), ("ncols", np.int32), ("nchunks", np.int32),
                      ("kind", np.int32), ("pbase", np.int64)]),
    "pair_descs": np.dtype([("woff", np.int64), ("xrow", np.int64), ("yrow", np.int64),
                            ("out", np.int64), ("m", np.int32), ("n", np.int32), ("rp", np.int32),
                            ("own", np.int32)]),
    "pd_level": np.int64, "pc_off": np.int32, "pc_pos": np.int64,
    "fused_descs": np.dtype([("piv_off", np.int64), ("lu_off", np.int64), ("xrow", np.int64),
                             ("yrow", np.int64), ("out", np.int64), ("m", np.int32), ("n", np.int32),
                             ("r", np.int32), ("own", np.int32), ("touch", np.int32), ("pad", np.int32),
                             ("cx", np.float64), ("cy", np.float64), ("cz", np.float64),
                             ("pad2", np.float64)]),
    "fd_level": np.int64, "pg_level": np.int64,
    "pg_items": np.dtype([("node", np.int32), ("row0", np.int32), ("nrows", np.int32),
                          ("slot", np.int32)]),
    "p2_items": np.dtype([("node", np.int32), ("row0", np.int32), ("nrows", np.int32),
                          ("slot", np.int32)]),
    "p2s_items": np.dtype([("node", np.int32), ("row0", np.int32), ("nrows", np.int32),
                           ("slot", np.int32)]),
}


class Plan:
    """The engine's host planner (csrc/planner.cpp) driven from Python: shard
    ownership, pair selection, column layout, phase-1 items, proxy segments and
    leaf lists, without a GPU. `offsets[l]` / `lists[l][k]` = (off, ids) as
    exported by the tree/list builders (bit-identical to the reference)."""

    def __init__(self, depth, n, offsets, lists, shard_rank=0, shard_world=1, modes=None):
        off = np.ascontiguousarray(np.concatenate([np.asarray(offsets[l], np.int64)
                                                   for l in range(depth + 1)]))
        lo, li, counts = [], [], np.zeros(4 * (depth + 1), np.int64)
        for l in range(1, depth + 1):
            for k in range(4):
                if k < len(lists[l]):
                    o, ids = lists[l][k]
                else:  # no near_vertex kind given: empty (HODLR3D / HODLR)
                    o, ids = np.zeros((1 << (3 * l)) + 1, np.int32), np.zeros(0, np.int32)
                lo.append(np.asarray(o, np.int32))
                li.append(np.asarray(ids, np.int32))
                counts[4 * l + k] = len(ids)
        lo = np.ascontiguousarray(np.concatenate(lo) if lo else np.zeros(1, np.int32))
        li = np.ascontiguousarray(np.concatenate(li) if li else np.zeros(1, np.int32))
        md = None if modes is None else np.ascontiguousarray(np.asarray(modes, np.int32))
        h = C.c_void_p()
        self._h = None
        _check(_L.h3d_plan_create(depth, n, _ptr(off), _ptr(lo), _ptr(li), _ptr(counts),
                                  shard_rank, shard_world, None if md is None else _ptr(md),
                                  C.byref(h)))
        self._h = h
        self.depth = depth

    def __del__(self):
        if getattr(self, "_h", None):
            _L.h3d_plan_destroy(self._h)

    def pairs(self, level):
        cnt = C.c_int64(0)
        _check(_L.h3d_plan_pairs(self._h, level, None, None, C.byref(cnt)))
        x = np.empty(max(cnt.value, 1), np.int32)
        y = np.empty(max(cnt.value, 1), np.int32)
        _check(_L.h3d_plan_pairs(self._h, level, _ptr(x), _ptr(y), C.byref(cnt)))
        return x[: cnt.value], y[: cnt.value]

    def set_ranks(self, level, ranks):
        r = np.ascontiguousarray(ranks, np.int32)
        _check(_L.h3d_plan_set_ranks(self._h, level, _ptr(r)))

    def set_mode(self, level, mode):
        _check(_L.h3d_plan_set_mode(self._h, level, int(mode)))

    def layout(self):
        _check(_L.h3d_plan_layout(self._h))

    def array(self, name, level=0):
        dt = np.dtype(_PLAN_DTYPES[name])
        cnt = C.c_int64(0)
        _check(_L.h3d_plan_array(self._h, name.encode(), level, None, C.byref(cnt)))
        out = np.zeros(max(cnt.value, 1), dt)
        _check(_L.h3d_plan_array(self._h, name.encode(), level, _ptr(out), C.byref(cnt)))
        return out[: cnt.value]
