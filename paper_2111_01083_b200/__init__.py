"""periwave-b200: B200-native periodic evaluation (arXiv 2111.01083).

Python host mirror of the reference's C++ API (/root/reference/proj/include/periwave/),
bound to the C-ABI in include/periwave_b200.h through ctypes. Every compute
call runs the sm_100a kernels in libperiwave_b200.so; there is no CPU fallback:
if the shared library is missing, importing the compute entry points raises.

Arrays: host data is numpy (float64, C-contiguous; points shaped (n, 2));
device data is torch CUDA tensors (float64), passed by pointer with no copy.
"""
from __future__ import annotations

import ctypes
import enum
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libperiwave_b200.so")
INCLUDE_DIR = os.path.join(os.path.dirname(_HERE), "include")


class ErrorCode(enum.IntEnum):
    """periwave::ErrorCode (reference include/periwave/errors.hpp:8-28), same ordinals."""

    NonPositiveDimension = 0
    OrientationViolation = 1
    CoincidentPoints = 2
    CoincidentSourceTarget = 3
    MissingBeta = 4
    InvalidOrder = 5
    OrderOutOfRange = 6
    PrecisionOutOfRange = 7
    RuleMismatch = 8
    NotDoubly = 9
    LengthMismatch = 10
    DimensionMismatch = 11
    NotNeutral = 12
    GridTooCoarse = 13
    OutOfInterval = 14
    NonUnitNormal = 15
    NotConverged = 16
    ParseError = 17
    Unsupported = 18


class PeriwaveError(RuntimeError):
    """periwave::Error: carries the reference ErrorCode (or a library status >= 64)."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.code = ErrorCode(status - 1) if 1 <= status <= 19 else None
        super().__init__(f"[{self.code.name if self.code is not None else status}] {message}")


class Pde(enum.IntEnum):
    Poisson = 0
    ModHelmholtz = 1
    Stokes = 2
    ModStokes = 3


class Periodicity(enum.IntEnum):
    Singly = 1
    Doubly = 2


class ApplyPath(enum.IntEnum):
    Auto = 0
    Direct = 1
    Accelerated = 2


class NufftBackend(enum.IntEnum):
    Reference = 0
    Accelerated = 1


PART_SCALAR, PART_BLOCK, PART_PRESSURE, PART_STRESSLET = 0, 1, 2, 3
MEM_HOST, MEM_DEVICE = 0, 1


# ---------------------------------------------------------------- ctypes mirror of periwave_b200.h
class _Cell(ctypes.Structure):
    _fields_ = [("d", ctypes.c_double), ("xi", ctypes.c_double), ("eta", ctypes.c_double),
                ("periodicity", ctypes.c_int), ("m0", ctypes.c_int)]


class _Info(ctypes.Structure):
    _fields_ = [("pde", ctypes.c_int), ("beta", ctypes.c_double), ("cell", _Cell), ("eps", ctypes.c_double),
                ("dlp", ctypes.c_int), ("multipole_order", ctypes.c_int), ("requires_neutrality", ctypes.c_int),
                ("n_parts", ctypes.c_int * 4)]


_DP = ctypes.POINTER(ctypes.c_double)


class _Part(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("axis", ctypes.c_int), ("dir", ctypes.c_int), ("flag", ctypes.c_int),
                ("has_m0", ctypes.c_int), ("size", ctypes.c_size_t),
                ("phase", _DP), ("decay_t", _DP), ("decay_s", _DP), ("shift_t", _DP), ("shift_s", _DP),
                ("t", _DP * 6), ("m0", ctypes.c_double * 4)]


class _System(ctypes.Structure):
    _fields_ = [("n_src", ctypes.c_size_t), ("n_tgt", ctypes.c_size_t), ("sources", ctypes.c_void_p),
                ("charges", ctypes.c_void_p), ("forces", ctypes.c_void_p), ("normals", ctypes.c_void_p),
                ("coefficients", ctypes.c_void_p), ("targets", ctypes.c_void_p), ("memory", ctypes.c_int)]


class _Options(ctypes.Structure):
    _fields_ = [("path", ctypes.c_int), ("threads", ctypes.c_int), ("with_pressure", ctypes.c_int),
                ("nufft_eps", ctypes.c_double), ("with_gradient", ctypes.c_int), ("device", ctypes.c_int),
                ("stream", ctypes.c_void_p)]


class _Field(ctypes.Structure):
    _fields_ = [("scalar", ctypes.c_void_p), ("velocity", ctypes.c_void_p), ("pressure", ctypes.c_void_p),
                ("complex_scalar", ctypes.c_void_p), ("gradient", ctypes.c_void_p), ("accelerated", ctypes.c_int),
                ("memory", ctypes.c_int)]


# Every symbol declared in include/periwave_b200.h (checked by tests/test_abi.py).
EXPORTED = [
    "pwb_last_error", "pwb_version", "pwb_device_count", "pwb_make_unit_cell", "pwb_near_translations",
    "pwb_make_periodizer", "pwb_make_stokes_dlp_periodizer", "pwb_make_multipole_periodizer",
    "pwb_periodizer_free", "pwb_periodizer_rank", "pwb_truncation_order", "pwb_periodizer_get_info",
    "pwb_periodizer_get_part", "pwb_periodizer_new", "pwb_periodizer_add_part", "pwb_options_default",
    "pwb_total_field", "pwb_apply_far", "pwb_accumulate", "pwb_near_field", "pwb_choose_path",
    "pwb_far_coeff_size", "pwb_far_source_pass", "pwb_far_target_pass", "pwb_validate",
    "pwb_nufft_type1", "pwb_nufft_type2", "pwb_nufft_type3", "pwb_fast_nufft_available",
    "pwb_eval_kernel", "pwb_rng_uniform", "pwb_launch_count", "pwb_last_phase_ms", "pwb_fp64_peak_probe",
    "pwb_near_sym_items", "pwb_near_sym_partial", "pwb_near_sym_split", "pwb_fixed_to_field",
    "pwb_brute_force_far", "pwb_periodicity_residual",
]

_lib = None


def lib() -> ctypes.CDLL:
    """The loaded product library; raises if it was not built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (make -C paper_2111_01083_b200)")
    L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_LOCAL)
    vp, sz, i, d = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_double
    L.pwb_last_error.restype = ctypes.c_char_p
    L.pwb_version.restype = ctypes.c_char_p
    L.pwb_make_unit_cell.argtypes = [d, d, d, i, ctypes.POINTER(_Cell)]
    L.pwb_near_translations.argtypes = [ctypes.POINTER(_Cell), sz, vp, vp, ctypes.POINTER(sz)]
    L.pwb_make_periodizer.argtypes = [i, d, ctypes.POINTER(_Cell), d, ctypes.POINTER(vp)]
    L.pwb_make_stokes_dlp_periodizer.argtypes = [ctypes.POINTER(_Cell), d, ctypes.POINTER(vp)]
    L.pwb_make_multipole_periodizer.argtypes = [i, d, i, ctypes.POINTER(_Cell), d, ctypes.POINTER(vp)]
    L.pwb_periodizer_free.argtypes = [vp]
    L.pwb_periodizer_free.restype = None
    L.pwb_periodizer_rank.argtypes = [vp]
    L.pwb_periodizer_rank.restype = sz
    L.pwb_truncation_order.argtypes = [ctypes.POINTER(_Cell), d, ctypes.POINTER(i)]
    L.pwb_periodizer_get_info.argtypes = [vp, ctypes.POINTER(_Info)]
    L.pwb_periodizer_get_part.argtypes = [vp, i, i, ctypes.POINTER(_Part)]
    L.pwb_periodizer_new.argtypes = [i, d, ctypes.POINTER(_Cell), d, i, i, i, ctypes.POINTER(vp)]
    L.pwb_periodizer_add_part.argtypes = [vp, ctypes.POINTER(_Part)]
    L.pwb_options_default.argtypes = [ctypes.POINTER(_Options)]
    L.pwb_options_default.restype = None
    for name in ("pwb_total_field", "pwb_apply_far", "pwb_near_field"):
        getattr(L, name).argtypes = [vp, ctypes.POINTER(_System), ctypes.POINTER(_Options), ctypes.POINTER(_Field)]
    L.pwb_accumulate.argtypes = [vp, ctypes.POINTER(_System), d, d, i, ctypes.POINTER(_Options),
                                 ctypes.POINTER(_Field)]
    L.pwb_choose_path.argtypes = [vp, sz, sz, ctypes.POINTER(i)]
    L.pwb_far_coeff_size.argtypes = [vp, ctypes.POINTER(_Options), sz, sz, ctypes.POINTER(sz)]
    L.pwb_far_source_pass.argtypes = [vp, ctypes.POINTER(_System), ctypes.POINTER(_Options), sz, sz, vp]
    L.pwb_far_target_pass.argtypes = [vp, ctypes.POINTER(_System), ctypes.POINTER(_Options), sz, sz, vp,
                                      ctypes.POINTER(_Field)]
    L.pwb_validate.argtypes = [vp, ctypes.POINTER(_System), ctypes.POINTER(_Options)]
    L.pwb_nufft_type1.argtypes = [i, d, sz, vp, vp, sz, vp, i, vp]
    L.pwb_nufft_type2.argtypes = [i, d, sz, vp, sz, vp, vp, i, vp]
    L.pwb_nufft_type3.argtypes = [i, d, sz, vp, vp, sz, vp, vp, i, vp]
    L.pwb_eval_kernel.argtypes = [i, i, d, i, sz, vp, vp]
    L.pwb_rng_uniform.argtypes = [ctypes.c_uint64, sz, vp]
    L.pwb_device_count.argtypes = [ctypes.POINTER(i)]
    L.pwb_launch_count.argtypes = [ctypes.POINTER(ctypes.c_long)]
    L.pwb_last_phase_ms.argtypes = [vp, i, ctypes.POINTER(d), ctypes.POINTER(d)]
    L.pwb_fp64_peak_probe.argtypes = [i, ctypes.POINTER(d)]
    L.pwb_near_sym_items.argtypes = [vp, sz, ctypes.POINTER(_Options), ctypes.POINTER(ctypes.c_long),
                                     ctypes.POINTER(i)]
    L.pwb_near_sym_partial.argtypes = [vp, ctypes.POINTER(_System), ctypes.POINTER(_Options), ctypes.c_long,
                                       ctypes.c_long, vp, ctypes.POINTER(i), ctypes.POINTER(i)]
    L.pwb_near_sym_split.argtypes = [vp, ctypes.POINTER(_System), ctypes.POINTER(_Options), i,
                                     ctypes.POINTER(ctypes.c_long)]
    L.pwb_fixed_to_field.argtypes = [vp, ctypes.POINTER(_Options), vp, sz, i, ctypes.POINTER(_Field)]
    L.pwb_brute_force_far.argtypes = [vp, ctypes.POINTER(_System), i, ctypes.POINTER(_Options),
                                      ctypes.POINTER(_Field)]
    L.pwb_periodicity_residual.argtypes = [vp, ctypes.POINTER(_System), i, ctypes.POINTER(_Options),
                                           ctypes.POINTER(d), ctypes.POINTER(d), ctypes.POINTER(d)]
    _lib = L
    return L


def _check(status: int) -> None:
    if status != 0:
        raise PeriwaveError(status, lib().pwb_last_error().decode())


def device_count() -> int:
    n = ctypes.c_int(0)
    _check(lib().pwb_device_count(ctypes.byref(n)))
    return n.value


# ---------------------------------------------------------------- cells
@dataclass(frozen=True)
class UnitCell:
    """periwave::UnitCell (reference include/periwave/cell.hpp:17-29)."""

    d: float
    xi: float
    eta: float
    periodicity: Periodicity
    m0: int

    def _c(self) -> _Cell:
        return _Cell(self.d, self.xi, self.eta, int(self.periodicity), self.m0)

    def e1(self):
        return (self.d, 0.0)

    def e2(self):
        return (self.xi, self.eta)


def make_unit_cell(d: float, xi: float, eta: float, periodicity: Periodicity = Periodicity.Doubly) -> UnitCell:
    c = _Cell()
    _check(lib().pwb_make_unit_cell(float(d), float(xi), float(eta), int(periodicity), ctypes.byref(c)))
    return UnitCell(c.d, c.xi, c.eta, Periodicity(c.periodicity), c.m0)


def near_translations(cell: UnitCell):
    """[(m, n, (sx, sy)), ...] in the reference order (cell.cpp:47-58)."""
    cnt = ctypes.c_size_t(0)
    shifts = np.zeros((32, 2))
    mn = np.zeros((32, 2), dtype=np.int32)
    _check(lib().pwb_near_translations(ctypes.byref(cell._c()), 32, shifts.ctypes.data, mn.ctypes.data,
                                       ctypes.byref(cnt)))
    return [(int(mn[i, 0]), int(mn[i, 1]), (float(shifts[i, 0]), float(shifts[i, 1]))) for i in range(cnt.value)]


def truncation_order(cell: UnitCell, eps: float) -> int:
    out = ctypes.c_int(0)
    _check(lib().pwb_truncation_order(ctypes.byref(cell._c()), float(eps), ctypes.byref(out)))
    return out.value


def rng_uniform(seed: int, n: int) -> np.ndarray:
    """The reference Rng::uniform stream (util.hpp:83-98)."""
    out = np.empty(n, dtype=np.float64)
    _check(lib().pwb_rng_uniform(ctypes.c_uint64(seed), n, out.ctypes.data))
    return out


# ---------------------------------------------------------------- periodizers
@dataclass
class Part:
    kind: int
    axis: int
    dir: int
    flag: int
    has_m0: int
    phase: np.ndarray
    decay_t: np.ndarray
    decay_s: np.ndarray
    shift_t: np.ndarray
    shift_s: np.ndarray
    tables: list
    m0: np.ndarray

    @property
    def size(self) -> int:
        return len(self.phase)


# doubles per mode of each table, by part kind (periwave_b200.h pwb_part)
_TABLE_WIDTHS = {PART_SCALAR: [2], PART_BLOCK: [8, 8], PART_PRESSURE: [2, 4], PART_STRESSLET: [8, 8, 8, 2, 2, 2]}


class Periodizer:
    """Owning handle for a pwb_periodizer (periwave::Periodizer, periodize.hpp:99-112)."""

    def __init__(self, handle: int):
        self._h = ctypes.c_void_p(handle)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value and _lib is not None:
            _lib.pwb_periodizer_free(h)
            self._h = ctypes.c_void_p(None)

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    def rank(self) -> int:
        return int(lib().pwb_periodizer_rank(self._h))

    def info(self) -> dict:
        inf = _Info()
        _check(lib().pwb_periodizer_get_info(self._h, ctypes.byref(inf)))
        return {"pde": Pde(inf.pde), "beta": inf.beta, "eps": inf.eps, "dlp": bool(inf.dlp),
                "multipole_order": inf.multipole_order, "requires_neutrality": bool(inf.requires_neutrality),
                "cell": UnitCell(inf.cell.d, inf.cell.xi, inf.cell.eta, Periodicity(inf.cell.periodicity),
                                 inf.cell.m0),
                "n_parts": list(inf.n_parts)}

    @property
    def cell(self) -> UnitCell:
        return self.info()["cell"]

    def part(self, kind: int, index: int) -> Part:
        p = _Part()
        _check(lib().pwb_periodizer_get_part(self._h, kind, index, ctypes.byref(p)))
        n = p.size

        def arr(ptr, count):
            if count == 0 or not ptr:
                return np.zeros(0)
            return np.ctypeslib.as_array(ptr, shape=(count,)).copy()

        tables = [arr(p.t[k], w * n) for k, w in enumerate(_TABLE_WIDTHS[kind])]
        return Part(kind, p.axis, p.dir, p.flag, p.has_m0, arr(p.phase, n), arr(p.decay_t, n), arr(p.decay_s, n),
                    arr(p.shift_t, n), arr(p.shift_s, n), tables, np.array(list(p.m0)))

    def parts(self, kind: int):
        return [self.part(kind, i) for i in range(self.info()["n_parts"][kind])]

    @staticmethod
    def from_tables(pde: Pde, beta: float, cell: UnitCell, eps: float, parts, dlp=False, multipole_order=0,
                    requires_neutrality=False) -> "Periodizer":
        """Build a periodizer from explicit tables (pwb_periodizer_new + add_part)."""
        h = ctypes.c_void_p()
        _check(lib().pwb_periodizer_new(int(pde), float(beta), ctypes.byref(cell._c()), float(eps), int(dlp),
                                        int(multipole_order), int(requires_neutrality), ctypes.byref(h)))
        pz = Periodizer(h.value)
        for part in parts:
            keep = [np.ascontiguousarray(a, dtype=np.float64) for a in
                    (part.phase, part.decay_t, part.decay_s, part.shift_t, part.shift_s)]
            tabs = [np.ascontiguousarray(t, dtype=np.float64) for t in part.tables]
            c = _Part()
            c.kind, c.axis, c.dir, c.flag, c.has_m0 = part.kind, part.axis, part.dir, part.flag, part.has_m0
            c.size = len(keep[0])
            c.phase, c.decay_t, c.decay_s, c.shift_t, c.shift_s = [a.ctypes.data_as(_DP) for a in keep]
            for k, t in enumerate(tabs):
                c.t[k] = t.ctypes.data_as(_DP)
            for k in range(4):
                c.m0[k] = float(part.m0[k]) if k < len(part.m0) else 0.0
            _check(lib().pwb_periodizer_add_part(pz._h, ctypes.byref(c)))
        return pz


def make_periodizer(pde: Pde, beta: float, cell: UnitCell, eps: float) -> Periodizer:
    h = ctypes.c_void_p()
    _check(lib().pwb_make_periodizer(int(pde), float(beta), ctypes.byref(cell._c()), float(eps), ctypes.byref(h)))
    return Periodizer(h.value)


def make_stokes_dlp_periodizer(cell: UnitCell, eps: float) -> Periodizer:
    h = ctypes.c_void_p()
    _check(lib().pwb_make_stokes_dlp_periodizer(ctypes.byref(cell._c()), float(eps), ctypes.byref(h)))
    return Periodizer(h.value)


def make_multipole_periodizer(pde: Pde, beta: float, l: int, cell: UnitCell, eps: float) -> Periodizer:
    h = ctypes.c_void_p()
    _check(lib().pwb_make_multipole_periodizer(int(pde), float(beta), int(l), ctypes.byref(cell._c()), float(eps),
                                               ctypes.byref(h)))
    return Periodizer(h.value)


# ---------------------------------------------------------------- systems and results
def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def _ptr_mem(a, n_expected: int, width: int, name: str):
    """(pointer, memory) of a float64 array of n_expected*width values, or (None, None)."""
    if a is None:
        return None, None
    if _is_torch(a):
        if a.dtype.itemsize != 8 or not a.is_contiguous():
            raise ValueError(f"{name}: need a contiguous float64 tensor")
        if a.numel() != n_expected * width:
            raise PeriwaveError(1 + ErrorCode.LengthMismatch, f"{name} length does not match")
        return a.data_ptr(), (MEM_DEVICE if a.is_cuda else MEM_HOST)
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous):
        raise ValueError(f"{name}: need a C-contiguous float64 numpy array")
    if a.size != n_expected * width:
        raise PeriwaveError(1 + ErrorCode.LengthMismatch, f"{name} length does not match")
    return a.ctypes.data, MEM_HOST


@dataclass
class ParticleSystem:
    """periwave::ParticleSystem (cell.hpp:58-65). Points are (n, 2) float64; complex
    coefficients are (n, 2) (re, im). numpy (host) or torch CUDA tensors (device)."""

    sources: object = None
    charges: object = None
    forces: object = None
    normals: object = None
    coefficients: object = None
    targets: object = None

    def _n(self, a):
        if a is None:
            return 0
        return int(a.shape[0])

    def _c(self):
        ns, nt = self._n(self.sources), self._n(self.targets)
        fields = [("sources", self.sources, ns, 2), ("charges", self.charges, ns, 1), ("forces", self.forces, ns, 2),
                  ("normals", self.normals, ns, 2), ("coefficients", self.coefficients, ns, 2),
                  ("targets", self.targets, nt, 2)]
        ptrs, mems = {}, set()
        for name, a, n, w in fields:
            p, m = _ptr_mem(a, n, w, name)
            ptrs[name] = p
            if m is not None and n > 0:
                mems.add(m)
        if len(mems) > 1:
            raise ValueError("all arrays of a system must live in the same memory (host or device)")
        mem = mems.pop() if mems else MEM_HOST
        s = _System(ns, nt, ptrs["sources"], ptrs["charges"], ptrs["forces"], ptrs["normals"], ptrs["coefficients"],
                    ptrs["targets"], mem)
        return s, mem


@dataclass
class ApplyOptions:
    """periwave::ApplyOptions (apply.hpp:15-20) plus the gradient/device/stream extensions."""

    path: ApplyPath = ApplyPath.Auto
    threads: int = 1
    with_pressure: bool = False
    nufft_eps: float = 0.0
    with_gradient: bool = False
    device: int = -1
    stream: Optional[int] = None

    def _c(self) -> _Options:
        o = _Options()
        lib().pwb_options_default(ctypes.byref(o))
        o.path, o.threads, o.with_pressure = int(self.path), int(self.threads), int(self.with_pressure)
        o.nufft_eps, o.with_gradient, o.device = float(self.nufft_eps), int(self.with_gradient), int(self.device)
        o.stream = self.stream
        return o


@dataclass
class FieldResult:
    """periwave::FieldResult (apply.hpp:25-31) plus `gradient`."""

    scalar: object = None
    velocity: object = None
    pressure: object = None
    complex_scalar: object = None
    gradient: object = None
    accelerated: bool = False


def _kind(pz: Periodizer) -> str:
    k = getattr(pz, "_kind_cache", None)  # the tables are immutable: one info() per periodizer
    if k is None:
        inf = pz.info()
        k = ("multipole" if inf["multipole_order"] >= 1 else
             "velocity" if inf["pde"] in (Pde.Stokes, Pde.ModStokes) else "scalar")
        pz._kind_cache = k
    return k


def _alloc(like_device: bool, shape, ref=None, zero=True):
    if like_device:
        import torch
        dev = ref.device if ref is not None else "cuda"
        # overwriting entry points fill every element: no zero-fill kernel
        return (torch.zeros if zero else torch.empty)(shape, dtype=torch.float64, device=dev)
    return np.zeros(shape)


def _field_for(pz: Periodizer, opt: ApplyOptions, nt: int, device: bool, ref, out: Optional[FieldResult],
               zero: bool = True):
    k = _kind(pz)
    res = out if out is not None else FieldResult()
    f = _Field()
    f.memory = MEM_DEVICE if device else MEM_HOST

    def ensure(name, shape):
        cur = getattr(res, name)
        if cur is None:
            cur = _alloc(device, shape, ref, zero)
            setattr(res, name, cur)
        p, _ = _ptr_mem(cur, nt, int(np.prod(shape[1:])) if len(shape) > 1 else 1, name)
        return p

    if k == "multipole":
        f.complex_scalar = ensure("complex_scalar", (nt, 2))
    elif k == "velocity":
        f.velocity = ensure("velocity", (nt, 2))
        if opt.with_pressure:
            f.pressure = ensure("pressure", (nt,))
    else:
        f.scalar = ensure("scalar", (nt,))
        if opt.with_gradient:
            f.gradient = ensure("gradient", (nt, 2))
    return res, f


def _apply(fn, pz: Periodizer, sys: ParticleSystem, opt: Optional[ApplyOptions], out=None, extra=(), zero=True):
    opt = opt or ApplyOptions()
    s, mem = sys._c()
    res, f = _field_for(pz, opt, s.n_tgt, mem == MEM_DEVICE, sys.targets if mem == MEM_DEVICE else None, out, zero)
    o = opt._c()
    _check(fn(pz.handle, ctypes.byref(s), *extra, ctypes.byref(o), ctypes.byref(f)))
    res.accelerated = bool(f.accelerated)
    return res


def total_field(pz: Periodizer, sys: ParticleSystem, opt: Optional[ApplyOptions] = None) -> FieldResult:
    """Far apply + fused near images (reference apply.cpp:548-556)."""
    return _apply(lib().pwb_total_field, pz, sys, opt, zero=False)


def apply_far(pz: Periodizer, sys: ParticleSystem, opt: Optional[ApplyOptions] = None) -> FieldResult:
    """Low-rank plane-wave far field (reference apply.cpp:417-479)."""
    return _apply(lib().pwb_apply_far, pz, sys, opt, zero=False)


def accumulate(pz: Periodizer, sys: ParticleSystem, shift, identity_shift: bool, opt: Optional[ApplyOptions],
               out: FieldResult) -> FieldResult:
    """FreeSpaceEvaluator::accumulate (reference apply.cpp:481-546): ADDS one image into `out`."""
    return _apply(lib().pwb_accumulate, pz, sys, opt, out,
                  (ctypes.c_double(shift[0]), ctypes.c_double(shift[1]), ctypes.c_int(int(identity_shift))))


def near_field(pz: Periodizer, sys: ParticleSystem, opt: Optional[ApplyOptions] = None,
               out: Optional[FieldResult] = None) -> FieldResult:
    """Adds every near image (one fused launch)."""
    return _apply(lib().pwb_near_field, pz, sys, opt, out)


def choose_path(pz: Periodizer, n_src: int, n_tgt: int) -> ApplyPath:
    out = ctypes.c_int(0)
    _check(lib().pwb_choose_path(pz.handle, n_src, n_tgt, ctypes.byref(out)))
    return ApplyPath(out.value)


def fast_nufft_available() -> bool:
    return bool(lib().pwb_fast_nufft_available())


def _cplx(a) -> np.ndarray:
    """Any 1-D real/complex array -> interleaved (re, im) float64 of shape (n, 2)."""
    a = np.asarray(a)
    return np.ascontiguousarray(np.stack([a.real, a.imag], axis=-1), dtype=np.float64)


def nufft_type1(backend: NufftBackend, eps: float, x, c, nmodes: int) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    cc = _cplx(c)
    f = np.zeros((nmodes, 2))
    _check(lib().pwb_nufft_type1(int(backend), float(eps), len(x), x.ctypes.data, cc.ctypes.data, nmodes,
                                 f.ctypes.data, MEM_HOST, None))
    return f[:, 0] + 1j * f[:, 1]


def nufft_type2(backend: NufftBackend, eps: float, x, fm) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    ff = _cplx(fm)
    c = np.zeros((len(x), 2))
    _check(lib().pwb_nufft_type2(int(backend), float(eps), len(x), x.ctypes.data, ff.shape[0], ff.ctypes.data,
                                 c.ctypes.data, MEM_HOST, None))
    return c[:, 0] + 1j * c[:, 1]


def nufft_type3(backend: NufftBackend, eps: float, x, c, s) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    s = np.ascontiguousarray(s, dtype=np.float64)
    cc = _cplx(c)
    f = np.zeros((len(s), 2))
    _check(lib().pwb_nufft_type3(int(backend), float(eps), len(x), x.ctypes.data, cc.ctypes.data, len(s),
                                 s.ctypes.data, f.ctypes.data, MEM_HOST, None))
    return f[:, 0] + 1j * f[:, 1]


def eval_kernel(which: int, pde: int, beta: float, l: int, inputs: np.ndarray) -> np.ndarray:
    """Device pair math at host points (pwb_eval_kernel)."""
    widths_in = {0: 1, 1: 2, 2: 2, 3: 2, 4: 2, 5: 4, 6: 1, 7: 1, 8: 1, 9: 1, 10: 1, 11: 1, 12: 1}
    widths_out = {0: 1, 1: 1, 2: 4, 3: 2, 4: 2, 5: 4, 6: 6, 7: 4, 8: 1, 9: 2, 10: 1, 11: 1, 12: 1}
    a = np.ascontiguousarray(inputs, dtype=np.float64).reshape(-1)
    n = a.size // widths_in[which]
    out = np.zeros(n * widths_out[which])
    _check(lib().pwb_eval_kernel(which, pde, float(beta), int(l), n, a.ctypes.data, out.ctypes.data))
    return out.reshape(n, widths_out[which]) if widths_out[which] > 1 else out


# ---------------------------------------------------------------- sharded far field (multi-GPU)
def far_coeff_size(pz: Periodizer, opt: Optional[ApplyOptions] = None, n_src_total: int = 0,
                   n_tgt_total: int = 0) -> int:
    """Doubles in the plane-wave coefficient buffer (the allreduce operand); the path is
    resolved from the global counts (0: the local system is the whole problem)."""
    n = ctypes.c_size_t(0)
    o = (opt or ApplyOptions())._c()
    _check(lib().pwb_far_coeff_size(pz.handle, ctypes.byref(o), n_src_total, n_tgt_total, ctypes.byref(n)))
    return n.value


def far_source_pass(pz: Periodizer, sys: ParticleSystem, coeff, opt: Optional[ApplyOptions] = None,
                    n_src_total: int = 0, n_tgt_total: int = 0) -> None:
    s, mem = sys._c()
    if mem != MEM_DEVICE:
        raise ValueError("far_source_pass takes device tensors")
    o = (opt or ApplyOptions())._c()
    _check(lib().pwb_far_source_pass(pz.handle, ctypes.byref(s), ctypes.byref(o), n_src_total, n_tgt_total,
                                     coeff.data_ptr()))


def far_target_pass(pz: Periodizer, sys: ParticleSystem, coeff, opt: Optional[ApplyOptions] = None,
                    out: Optional[FieldResult] = None, n_src_total: int = 0, n_tgt_total: int = 0) -> FieldResult:
    opt = opt or ApplyOptions()
    s, mem = sys._c()
    if mem != MEM_DEVICE:
        raise ValueError("far_target_pass takes device tensors")
    res, f = _field_for(pz, opt, s.n_tgt, True, sys.targets, out, zero=False)
    o = opt._c()
    _check(lib().pwb_far_target_pass(pz.handle, ctypes.byref(s), ctypes.byref(o), n_src_total, n_tgt_total,
                                     coeff.data_ptr(), ctypes.byref(f)))
    res.accelerated = bool(f.accelerated)
    return res


def brute_force_far(pz: Periodizer, sys: ParticleSystem, shells: int,
                    opt: Optional[ApplyOptions] = None) -> FieldResult:
    """Shell-by-shell lattice sum of the far images (reference oracle.cpp:83-110), on the GPU."""
    opt = opt or ApplyOptions()
    s, mem = sys._c()
    if mem != MEM_HOST:
        raise ValueError("brute_force_far takes host arrays")
    res, f = _field_for(pz, opt, s.n_tgt, False, None, None)
    o = opt._c()
    _check(lib().pwb_brute_force_far(pz.handle, ctypes.byref(s), int(shells), ctypes.byref(o), ctypes.byref(f)))
    return res


def periodicity_residual(pz: Periodizer, sys: ParticleSystem, samples_per_side: int,
                         opt: Optional[ApplyOptions] = None) -> dict:
    """Face-jump residual of total_field (reference oracle.cpp:112-173): {e1, e2, scale, rel}."""
    s, mem = sys._c()
    if mem != MEM_HOST:
        raise ValueError("periodicity_residual takes host arrays")
    e1, e2, sc = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    o = (opt or ApplyOptions())._c()
    _check(lib().pwb_periodicity_residual(pz.handle, ctypes.byref(s), int(samples_per_side), ctypes.byref(o),
                                          ctypes.byref(e1), ctypes.byref(e2), ctypes.byref(sc)))
    rel = max(e1.value, e2.value) / max(sc.value, 1e-300)
    return {"e1": e1.value, "e2": e2.value, "scale": sc.value, "rel": rel}


def near_sym_items(pz: Periodizer, n: int, opt: Optional[ApplyOptions] = None):
    """(work items, outputs per target) of the symmetric near decomposition (host only)."""
    items, nout = ctypes.c_long(0), ctypes.c_int(0)
    o = (opt or ApplyOptions())._c()
    _check(lib().pwb_near_sym_items(pz.handle, n, ctypes.byref(o), ctypes.byref(items), ctypes.byref(nout)))
    return items.value, nout.value


# status bits of near_sym_partial (include/periwave_b200.h)
SYM_COINCIDENT = 1
SYM_OVERFLOW = 2


def near_sym_partial(pz: Periodizer, sys: ParticleSystem, acc, item_begin: int, item_end: int,
                     opt: Optional[ApplyOptions] = None):
    """Adds work items [begin, end) of the symmetric near field into the int64 accumulator
    `acc` (device, n * nout * 3, target-major). sys.targets must be sys.sources.

    Returns (scale_exp, status): the accumulator holds the field times 2**scale_exp (pass
    it to fixed_to_field); status bit SYM_COINCIDENT / SYM_OVERFLOW is NOT raised here, so
    the ranks can agree on it before the reduce-scatter (raise_sym_status)."""
    s, mem = sys._c()
    if mem != MEM_DEVICE:
        raise ValueError("near_sym_partial takes device tensors")
    o = (opt or ApplyOptions())._c()
    k, st = ctypes.c_int(0), ctypes.c_int(0)
    _check(lib().pwb_near_sym_partial(pz.handle, ctypes.byref(s), ctypes.byref(o), item_begin, item_end,
                                      acc.data_ptr(), ctypes.byref(k), ctypes.byref(st)))
    return k.value, st.value


def raise_sym_status(status: int) -> None:
    """The error the reference raises for a combined near_sym_partial status word."""
    if status & SYM_COINCIDENT:  # apply.cpp:544-545
        raise PeriwaveError(1 + ErrorCode.CoincidentSourceTarget,
                            "a target coincides with a lattice image of a source")
    if status & SYM_OVERFLOW:
        raise PeriwaveError(1 + ErrorCode.Unsupported,
                            "symmetric near field: strengths or kernel values exceed the fixed-point range")


def near_sym_split(pz: Periodizer, sys: ParticleSystem, world: int, opt: Optional[ApplyOptions] = None):
    """Item boundaries (world + 1 ints) of a balanced split of the symmetric work items
    (pwb_near_sym_split: cost-balanced for the screened kernels, by count otherwise)."""
    s, mem = sys._c()
    if mem != MEM_DEVICE:
        raise ValueError("near_sym_split takes device tensors")
    b = (ctypes.c_long * (world + 1))()
    o = (opt or ApplyOptions())._c()
    _check(lib().pwb_near_sym_split(pz.handle, ctypes.byref(s), ctypes.byref(o), int(world), b))
    return [int(v) for v in b]


def fixed_to_field(pz: Periodizer, acc, n_targets: int, out: FieldResult, opt: Optional[ApplyOptions] = None,
                   like=None, scale_exp: int = 0) -> FieldResult:
    """out += 2**-scale_exp times the fp64 value of a fixed-point accumulator slice (device)."""
    opt = opt or ApplyOptions()
    res, f = _field_for(pz, opt, n_targets, True, like if like is not None else acc, out)
    o = opt._c()
    _check(lib().pwb_fixed_to_field(pz.handle, ctypes.byref(o), acc.data_ptr(), n_targets, int(scale_exp),
                                    ctypes.byref(f)))
    return res


__all__ = [
    "ErrorCode", "PeriwaveError", "Pde", "Periodicity", "ApplyPath", "NufftBackend", "UnitCell", "make_unit_cell",
    "near_translations", "truncation_order", "rng_uniform", "Periodizer", "make_periodizer",
    "make_stokes_dlp_periodizer", "make_multipole_periodizer", "ParticleSystem", "ApplyOptions", "FieldResult",
    "total_field", "apply_far", "accumulate", "near_field", "choose_path", "fast_nufft_available", "nufft_type1",
    "nufft_type2", "nufft_type3", "eval_kernel", "far_coeff_size", "far_source_pass", "far_target_pass",
    "near_sym_split",
    "device_count", "lib", "EXPORTED",
]
