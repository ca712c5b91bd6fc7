"""TEST INFRASTRUCTURE: ctypes wrappers of the two CPU checkers (see oracle/__init__.py)."""
from __future__ import annotations

import ctypes
import os
from types import SimpleNamespace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libperiwave_ref.so")
PORT_SO = os.path.join(HERE, "_build", "libperiwave_port.so")

_vp, _sz, _i, _d = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_double


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def port_available() -> bool:
    return os.path.exists(PORT_SO)


def _p(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64).ctypes.data


_rng_src = None


def rng_uniform(seed: int, n: int) -> np.ndarray:
    """The reference's Rng::uniform stream from the checkers, never the product library:
    oracle/_ref's own periwave::Rng, else the C restatement in oracle/port."""
    global _rng_src
    if _rng_src is None:
        _rng_src = Ref() if ref_available() else Port()
    return _rng_src.rng_uniform(seed, n)


class RefError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        super().__init__(f"reference error {status}: {msg}")


class Ref:
    """The compiled reference library (oracle/_ref)."""

    def __init__(self):
        if not ref_available():
            raise FileNotFoundError(REF_SO)
        L = ctypes.CDLL(REF_SO, mode=ctypes.RTLD_LOCAL)
        L.ref_last_error.restype = ctypes.c_char_p
        for name in ("ref_make_periodizer",):
            getattr(L, name).restype = _vp
            getattr(L, name).argtypes = [_i, _d, _d, _d, _d, _i, _d, ctypes.POINTER(_i)]
        L.ref_make_multipole_periodizer.restype = _vp
        L.ref_make_multipole_periodizer.argtypes = [_i, _d, _i, _d, _d, _d, _i, _d, ctypes.POINTER(_i)]
        L.ref_make_stokes_dlp_periodizer.restype = _vp
        L.ref_make_stokes_dlp_periodizer.argtypes = [_d, _d, _d, _i, _d, ctypes.POINTER(_i)]
        L.ref_free_periodizer.argtypes = [_vp]
        L.ref_rank.restype = _sz
        L.ref_rank.argtypes = [_vp]
        L.ref_requires_neutrality.argtypes = [_vp]
        L.ref_num_parts.argtypes = [_vp, _i]
        L.ref_part_info.argtypes = [_vp, _i, _i, _vp, _vp]
        L.ref_part_modes.argtypes = [_vp, _i, _i, _vp, _vp, _vp, _vp, _vp]
        L.ref_part_table.argtypes = [_vp, _i, _i, _i, _vp]
        L.ref_apply.argtypes = [_vp, _i, _sz, _vp, _vp, _vp, _vp, _vp, _sz, _vp, _i, _i, _i, _d, _vp, _vp, _vp, _vp,
                                ctypes.POINTER(_i)]
        L.ref_accumulate.argtypes = [_vp, _sz, _vp, _vp, _vp, _vp, _vp, _sz, _vp, _d, _d, _i, _i, _i, _vp, _vp, _vp,
                                     _vp]
        L.ref_choose_path.argtypes = [_vp, _sz, _sz]
        L.ref_brute_force_far.argtypes = [_vp, _i, _sz, _vp, _vp, _vp, _vp, _vp, _sz, _vp, _i, _vp, _vp, _vp]
        L.ref_periodicity_residual.argtypes = [_vp, _i, _sz, _vp, _vp, _vp, _vp, _vp, _i, _i, _vp, _vp, _vp]
        L.ref_nufft_type1.argtypes = [_i, _d, _sz, _vp, _vp, _sz, _vp]
        L.ref_nufft_type2.argtypes = [_i, _d, _sz, _vp, _sz, _vp, _vp]
        L.ref_nufft_type3.argtypes = [_i, _d, _sz, _vp, _vp, _sz, _vp, _vp]
        L.ref_bessel_kn.argtypes = [_i, _d, _vp]
        L.ref_greens_scalar.argtypes = [_i, _d, _d, _d, _vp]
        L.ref_greens_block.argtypes = [_i, _d, _d, _d, _vp]
        L.ref_multipole_kernel.argtypes = [_i, _d, _i, _d, _d, _vp]
        L.ref_stresslet_dlp.argtypes = [_d, _d, _d, _d, _vp]
        L.ref_pressurelet.argtypes = [_d, _d, _vp]
        L.ref_truncation_order.argtypes = [_d, _d, _d, _i, _d, _vp]
        L.ref_gauss_legendre.argtypes = [_i, _vp, _vp]
        L.ref_sommerfeld_rule.argtypes = [_i, _d, _d, _d, _d, _i, _d, _d, _sz, _vp, _vp, ctypes.POINTER(_sz), _vp, _vp]
        L.ref_interp_coeffs.argtypes = [_d, _d, _i, _d, _vp]
        L.ref_unit_cell_m0.argtypes = [_d, _d, _d, _i, ctypes.POINTER(_i)]
        L.ref_rng_uniform.argtypes = [ctypes.c_ulonglong, _sz, _vp]
        self.L = L

    def rng_uniform(self, seed, n):
        out = np.empty(n, dtype=np.float64)
        self.L.ref_rng_uniform(int(seed), int(n), out.ctypes.data)
        return out

    def _chk(self, st):
        if st != 0:
            raise RefError(st, self.L.ref_last_error().decode())

    # periodizers -----------------------------------------------------------------
    def make_periodizer(self, pde, beta, cell, eps):
        err = _i(0)
        d, xi, eta, per = cell
        h = self.L.ref_make_periodizer(int(pde), float(beta), d, xi, eta, int(per), float(eps), ctypes.byref(err))
        self._chk(err.value)
        return RefPeriodizer(self, h)

    def make_multipole_periodizer(self, pde, beta, l, cell, eps):
        err = _i(0)
        d, xi, eta, per = cell
        h = self.L.ref_make_multipole_periodizer(int(pde), float(beta), int(l), d, xi, eta, int(per), float(eps),
                                                 ctypes.byref(err))
        self._chk(err.value)
        return RefPeriodizer(self, h)

    def make_stokes_dlp_periodizer(self, cell, eps):
        err = _i(0)
        d, xi, eta, per = cell
        h = self.L.ref_make_stokes_dlp_periodizer(d, xi, eta, int(per), float(eps), ctypes.byref(err))
        self._chk(err.value)
        return RefPeriodizer(self, h)

    # kernels ---------------------------------------------------------------------
    def bessel_kn(self, l, x):
        out = np.zeros(1)
        self._chk(self.L.ref_bessel_kn(int(l), float(x), out.ctypes.data))
        return out[0]

    def greens_scalar(self, pde, beta, r):
        out = np.zeros(1)
        self._chk(self.L.ref_greens_scalar(int(pde), float(beta), float(r[0]), float(r[1]), out.ctypes.data))
        return out[0]

    def greens_block(self, pde, beta, r):
        out = np.zeros(4)
        self._chk(self.L.ref_greens_block(int(pde), float(beta), float(r[0]), float(r[1]), out.ctypes.data))
        return out

    def multipole_kernel(self, pde, beta, l, r):
        out = np.zeros(2)
        self._chk(self.L.ref_multipole_kernel(int(pde), float(beta), int(l), float(r[0]), float(r[1]),
                                              out.ctypes.data))
        return out[0] + 1j * out[1]

    def stresslet_dlp(self, r, n):
        out = np.zeros(4)
        self._chk(self.L.ref_stresslet_dlp(float(r[0]), float(r[1]), float(n[0]), float(n[1]), out.ctypes.data))
        return out

    def pressurelet(self, r):
        out = np.zeros(2)
        self._chk(self.L.ref_pressurelet(float(r[0]), float(r[1]), out.ctypes.data))
        return out

    # quadrature ------------------------------------------------------------------
    def truncation_order(self, cell, eps):
        out = np.zeros(1, dtype=np.int32)
        d, xi, eta, per = cell
        self._chk(self.L.ref_truncation_order(d, xi, eta, int(per), float(eps), out.ctypes.data))
        return int(out[0])

    def unit_cell_m0(self, cell):
        out = _i(0)
        d, xi, eta, per = cell
        self._chk(self.L.ref_unit_cell_m0(d, xi, eta, int(per), ctypes.byref(out)))
        return out.value

    def gauss_legendre(self, n):
        x, w = np.zeros(n), np.zeros(n)
        self._chk(self.L.ref_gauss_legendre(n, x.ctypes.data, w.ctypes.data))
        return x, w

    def sommerfeld_rule(self, pde, beta, cell, eps, min_upper=0.0):
        cap = 20000
        x, w = np.zeros(cap), np.zeros(cap)
        cnt = _sz(0)
        up, cert = np.zeros(1), np.zeros(1)
        d, xi, eta, per = cell
        self._chk(self.L.ref_sommerfeld_rule(int(pde), float(beta), d, xi, eta, int(per), float(eps),
                                             float(min_upper), cap, x.ctypes.data, w.ctypes.data, ctypes.byref(cnt),
                                             up.ctypes.data, cert.ctypes.data))
        n = cnt.value
        return x[:n].copy(), w[:n].copy(), up[0], cert[0]

    def interp_coeffs(self, lo, hi, m, x):
        out = np.zeros(m)
        self._chk(self.L.ref_interp_coeffs(float(lo), float(hi), int(m), float(x), out.ctypes.data))
        return out

    # nufft -------------------------------------------------------------------------
    def nufft_type1(self, backend, eps, x, c, nmodes):
        x = np.ascontiguousarray(x, dtype=np.float64)
        cc = np.ascontiguousarray(np.stack([np.real(c), np.imag(c)], -1), dtype=np.float64)
        f = np.zeros((nmodes, 2))
        self._chk(self.L.ref_nufft_type1(int(backend), float(eps), len(x), x.ctypes.data, cc.ctypes.data, nmodes,
                                         f.ctypes.data))
        return f[:, 0] + 1j * f[:, 1]

    def nufft_type2(self, backend, eps, x, fm):
        x = np.ascontiguousarray(x, dtype=np.float64)
        ff = np.ascontiguousarray(np.stack([np.real(fm), np.imag(fm)], -1), dtype=np.float64)
        c = np.zeros((len(x), 2))
        self._chk(self.L.ref_nufft_type2(int(backend), float(eps), len(x), x.ctypes.data, len(fm), ff.ctypes.data,
                                         c.ctypes.data))
        return c[:, 0] + 1j * c[:, 1]

    def nufft_type3(self, backend, eps, x, c, s):
        x = np.ascontiguousarray(x, dtype=np.float64)
        s = np.ascontiguousarray(s, dtype=np.float64)
        cc = np.ascontiguousarray(np.stack([np.real(c), np.imag(c)], -1), dtype=np.float64)
        f = np.zeros((len(s), 2))
        self._chk(self.L.ref_nufft_type3(int(backend), float(eps), len(x), x.ctypes.data, cc.ctypes.data, len(s),
                                         s.ctypes.data, f.ctypes.data))
        return f[:, 0] + 1j * f[:, 1]


class RefPeriodizer:
    KINDS = (0, 1, 2, 3)
    WIDTHS = {0: [2], 1: [8, 8], 2: [2, 4], 3: [8, 8, 8, 2, 2, 2]}

    def __init__(self, ref: Ref, h):
        self.ref, self.h = ref, _vp(h)

    def __del__(self):
        try:
            self.ref.L.ref_free_periodizer(self.h)
        except Exception:
            pass

    def rank(self):
        return int(self.ref.L.ref_rank(self.h))

    def requires_neutrality(self):
        return bool(self.ref.L.ref_requires_neutrality(self.h))

    def parts(self, kind):
        """Parts as SimpleNamespace with the product's Part field names."""
        L = self.ref.L
        out = []
        for idx in range(L.ref_num_parts(self.h, kind)):
            info = np.zeros(5, dtype=np.int64)
            m0 = np.zeros(4)
            self.ref._chk(L.ref_part_info(self.h, kind, idx, info.ctypes.data, m0.ctypes.data))
            n = int(info[4])
            arrs = [np.zeros(max(n, 1)) for _ in range(5)]
            self.ref._chk(L.ref_part_modes(self.h, kind, idx, *[a.ctypes.data for a in arrs]))
            arrs = [a[:n] for a in arrs]
            tables = []
            for which, w in enumerate(self.WIDTHS[kind]):
                t = np.zeros(max(w * n, 1))
                if kind == 1 and which == 1 and not info[2]:
                    tables.append(np.zeros(w * n))
                    continue
                self.ref._chk(L.ref_part_table(self.h, kind, idx, which, t.ctypes.data))
                tables.append(t[:w * n])
            flag = int(info[2])
            if kind == 1:  # block: take_real (always true upstream) | three_term << 1
                flag = 1 | (2 if info[2] else 0)
            out.append(SimpleNamespace(kind=kind, axis=int(info[0]), dir=int(info[1]), flag=flag,
                                       has_m0=int(info[3]), phase=arrs[0], decay_t=arrs[1], decay_s=arrs[2],
                                       shift_t=arrs[3], shift_s=arrs[4], tables=tables, m0=m0))
        return out

    def all_parts(self):
        return [p for k in self.KINDS for p in self.parts(k)]

    def choose_path(self, ns, nt):
        return int(self.ref.L.ref_choose_path(self.h, ns, nt))

    def apply(self, mode, sources, targets, charges=None, forces=None, normals=None, coefficients=None, path=1,
              threads=1, with_pressure=False, nufft_eps=0.0, kind="scalar"):
        """mode 0 total_field, 1 apply_far, 2 near images. Returns dict of outputs."""
        ns, nt = len(sources), len(targets)
        out = {"scalar": np.zeros(nt), "velocity": np.zeros((nt, 2)), "pressure": np.zeros(nt),
               "complex": np.zeros((nt, 2))}
        acc = _i(0)
        keep = [np.ascontiguousarray(a, dtype=np.float64) if a is not None else None
                for a in (sources, charges, forces, normals, coefficients, targets)]
        self.ref._chk(self.ref.L.ref_apply(self.h, mode, ns, *[_p(a) for a in keep[:5]], nt, _p(keep[5]), path,
                                           threads, int(with_pressure), float(nufft_eps), out["scalar"].ctypes.data,
                                           out["velocity"].ctypes.data, out["pressure"].ctypes.data,
                                           out["complex"].ctypes.data, ctypes.byref(acc)))
        out["accelerated"] = bool(acc.value)
        return out

    def accumulate(self, sources, targets, shift, identity, charges=None, forces=None, normals=None,
                   coefficients=None, threads=1, with_pressure=False, init=None):
        nt = len(targets)
        out = init or {"scalar": np.zeros(nt), "velocity": np.zeros((nt, 2)), "pressure": np.zeros(nt),
                       "complex": np.zeros((nt, 2))}
        keep = [np.ascontiguousarray(a, dtype=np.float64) if a is not None else None
                for a in (sources, charges, forces, normals, coefficients, targets)]
        self.ref._chk(self.ref.L.ref_accumulate(self.h, len(sources), *[_p(a) for a in keep[:5]], nt, _p(keep[5]),
                                                float(shift[0]), float(shift[1]), int(identity), threads,
                                                int(with_pressure), out["scalar"].ctypes.data,
                                                out["velocity"].ctypes.data, out["pressure"].ctypes.data,
                                                out["complex"].ctypes.data))
        return out

    def brute_force_far(self, shells, sources, targets, charges=None, forces=None, coefficients=None, threads=1):
        nt = len(targets)
        out = {"scalar": np.zeros(nt), "velocity": np.zeros((nt, 2)), "complex": np.zeros((nt, 2))}
        keep = [np.ascontiguousarray(a, dtype=np.float64) if a is not None else None
                for a in (sources, charges, forces, None, coefficients, targets)]
        self.ref._chk(self.ref.L.ref_brute_force_far(self.h, shells, len(sources), *[_p(a) for a in keep[:5]], nt,
                                                     _p(keep[5]), threads, out["scalar"].ctypes.data,
                                                     out["velocity"].ctypes.data, out["complex"].ctypes.data))
        return out


class Port:
    """The plain-C restatement (oracle/port)."""

    LAPLACE, MODHELM, STOKES, MODSTOKES, MP_LAPLACE, MP_MODHELM, STRESSLET = range(7)

    def __init__(self):
        if not port_available():
            raise FileNotFoundError(PORT_SO)
        L = ctypes.CDLL(PORT_SO, mode=ctypes.RTLD_LOCAL)
        L.port_bessel_kn.restype = _d
        L.port_bessel_kn.argtypes = [_i, _d]
        L.port_near.argtypes = [_i, _d, _i, _sz, _vp, _vp, _vp, _vp, _sz, _vp, _i, _vp, _i, _i, _i, _vp, _i]
        L.port_far_scalar.argtypes = [_sz, _i, _vp, _vp, _vp, _vp, _vp, _vp, _i, _d, _sz, _vp, _vp, _sz, _vp, _vp,
                                      _vp, _i]
        L.port_far_block.argtypes = [_sz, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _vp, _sz, _vp, _vp, _sz, _vp,
                                     _vp, _i]
        L.port_nufft_type1.argtypes = [_sz, _vp, _vp, _sz, _vp]
        L.port_nufft_type2.argtypes = [_sz, _vp, _sz, _vp, _vp]
        L.port_nufft_type3.argtypes = [_sz, _vp, _vp, _sz, _vp, _vp]
        L.port_rng_uniform.argtypes = [ctypes.c_ulonglong, _sz, _vp]
        self.L = L

    def rng_uniform(self, seed, n):
        out = np.empty(n, dtype=np.float64)
        self.L.port_rng_uniform(int(seed), int(n), out.ctypes.data)
        return out

    def bessel_kn(self, l, x):
        return self.L.port_bessel_kn(int(l), float(x))

    def near(self, kind, sources, targets, shifts, id_img, q=None, vec=None, nrm=None, beta=0.0, order=0,
             with_pressure=False, with_gradient=False, threads=1):
        nout = {0: 3 if with_gradient else 1, 1: 3 if with_gradient else 1, 2: 3 if with_pressure else 2,
                3: 3 if with_pressure else 2}.get(kind, 2)
        nt = len(targets)
        out = np.zeros((nt, nout))
        keep = [np.ascontiguousarray(a, dtype=np.float64) if a is not None else None
                for a in (sources, q, vec, nrm, targets, shifts)]
        coinc = self.L.port_near(kind, float(beta), int(order), len(sources), _p(keep[0]), _p(keep[1]), _p(keep[2]),
                                 _p(keep[3]), nt, _p(keep[4]), len(shifts), _p(keep[5]), int(id_img),
                                 int(with_pressure), int(with_gradient), out.ctypes.data, int(threads))
        return out, bool(coinc)

    def far(self, parts, sources, targets, charges=None, forces=None, coefficients=None, gradient=False, threads=1):
        """Sum of the direct far apply over scalar (kind 0) or block (kind 1) parts; complex accumulators."""
        ns, nt = len(sources), len(targets)
        src = np.ascontiguousarray(sources, dtype=np.float64)
        tgt = np.ascontiguousarray(targets, dtype=np.float64)
        acc_s = np.zeros((nt, 2))
        acc_v = np.zeros((nt, 4))
        grad = np.zeros((nt, 4)) if gradient else None
        if coefficients is not None:
            w = np.ascontiguousarray(coefficients, dtype=np.float64)
        elif charges is not None:
            w = np.ascontiguousarray(np.stack([charges, np.zeros(ns)], -1), dtype=np.float64)
        else:
            w = None
        f = None if forces is None else np.ascontiguousarray(forces, dtype=np.float64)
        for p in parts:
            arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
                    (p.phase, p.decay_t, p.decay_s, p.shift_t, p.shift_s)]
            if p.kind == 0:
                diag = np.ascontiguousarray(p.tables[0], dtype=np.float64)
                self.L.port_far_scalar(len(arrs[0]), p.axis, *[a.ctypes.data for a in arrs], diag.ctypes.data,
                                       int(p.has_m0), float(p.m0[0]), ns, src.ctypes.data, w.ctypes.data, nt,
                                       tgt.ctypes.data, acc_s.ctypes.data, _p(grad) if grad is not None else None,
                                       int(threads))
            elif p.kind == 1:
                da = np.ascontiguousarray(p.tables[0], dtype=np.float64)
                db = np.ascontiguousarray(p.tables[1], dtype=np.float64)
                m0 = np.ascontiguousarray(p.m0, dtype=np.float64)
                self.L.port_far_block(len(arrs[0]), p.axis, *[a.ctypes.data for a in arrs], da.ctypes.data,
                                      db.ctypes.data if db.size else None, int(bool(p.flag & 2)), int(p.has_m0),
                                      m0.ctypes.data, ns, src.ctypes.data, f.ctypes.data, nt, tgt.ctypes.data,
                                      acc_v.ctypes.data, int(threads))
        return SimpleNamespace(scalar=acc_s, velocity=acc_v, gradient=grad)

    def nufft_type1(self, x, c, nmodes):
        x = np.ascontiguousarray(x, dtype=np.float64)
        cc = np.ascontiguousarray(np.stack([np.real(c), np.imag(c)], -1), dtype=np.float64)
        f = np.zeros((nmodes, 2))
        self.L.port_nufft_type1(len(x), x.ctypes.data, cc.ctypes.data, nmodes, f.ctypes.data)
        return f[:, 0] + 1j * f[:, 1]

    def nufft_type2(self, x, fm):
        x = np.ascontiguousarray(x, dtype=np.float64)
        ff = np.ascontiguousarray(np.stack([np.real(fm), np.imag(fm)], -1), dtype=np.float64)
        c = np.zeros((len(x), 2))
        self.L.port_nufft_type2(len(x), x.ctypes.data, len(fm), ff.ctypes.data, c.ctypes.data)
        return c[:, 0] + 1j * c[:, 1]

    def nufft_type3(self, x, c, s):
        x = np.ascontiguousarray(x, dtype=np.float64)
        s = np.ascontiguousarray(s, dtype=np.float64)
        cc = np.ascontiguousarray(np.stack([np.real(c), np.imag(c)], -1), dtype=np.float64)
        f = np.zeros((len(s), 2))
        self.L.port_nufft_type3(len(x), x.ctypes.data, cc.ctypes.data, len(s), s.ctypes.data, f.ctypes.data)
        return f[:, 0] + 1j * f[:, 1]


def near_shifts(cell):
    """Near images in the reference order (cell.cpp:47-58): (shifts (k,2), identity index)."""
    d, xi, eta, per = cell
    sh = []
    if int(per) == 2:
        d_, xi_, eta_ = d, xi, eta
        m0 = 1 if xi == 0.0 else min(3, max(1, int(np.ceil(1.0 + 2.0 * abs(xi) / d))))
        for n in (-1, 0, 1):
            for m in range(-m0, m0 + 1):
                sh.append((m * d_ + n * xi_, n * eta_))
        ident = (len(sh) - 1) // 2
    else:
        for m in (-1, 0, 1):
            sh.append((m * d, 0.0))
        ident = 1
    return np.array(sh), ident
