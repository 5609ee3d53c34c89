"""Python handle on the fp64 CPU oracle (liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs — never by the product
package ``paper_2503_17743_b200``.  This wrapper marshals a problem dict from
``problems`` into the oracle's own ``or_problem`` struct (it shares no code with
the product binding).

Functions implemented in moc_oracle.cpp, each citing the passage it follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "moc_oracle.cpp")


def build(force: bool = False) -> str:
    """Compile liboracle.so (g++ -O2 -fopenmp, no fast-math, no FP contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "moc_oracle.h"))):
        cmd = ["g++", "-std=c++17", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-fPIC", "-shared", "-o", _SO + ".tmp", _SRC]
        subprocess.check_call(cmd)
        os.replace(_SO + ".tmp", _SO)
    return _SO


class _Problem(C.Structure):
    _fields_ = [
        ("nx", C.c_int32), ("ny", C.c_int32),
        ("pitch_x", C.c_double), ("pitch_y", C.c_double),
        ("cell_type", C.POINTER(C.c_int32)),
        ("n_types", C.c_int32), ("max_rings", C.c_int32),
        ("n_rings", C.POINTER(C.c_int32)),
        ("radii", C.POINTER(C.c_double)),
        ("n_layers", C.c_int32),
        ("planes", C.POINTER(C.c_double)),
        ("n_zones", C.c_int32),
        ("zone_of_layer", C.POINTER(C.c_int32)),
        ("material", C.POINTER(C.c_int32)),
        ("bc", C.c_int32 * 6),
        ("n_mat", C.c_int32), ("G", C.c_int32),
        ("sigma_t", C.POINTER(C.c_double)),
        ("sigma_s", C.POINTER(C.c_double)),
        ("nu_sigma_f", C.POINTER(C.c_double)),
        ("chi", C.POINTER(C.c_double)),
        ("num_azim", C.c_int32), ("num_polar", C.c_int32),
        ("radial_spacing", C.c_double), ("axial_spacing", C.c_double),
    ]


class _Counts(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("n_fsr", "n_regions", "n_tracks2d", "n_segs2d", "n_stacks",
                                         "n_tracks3d", "n_cycles", "n_degenerate")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        vp, i64, i32, dbl = C.c_void_p, C.c_int64, C.c_int32, C.c_double
        P = C.POINTER
        L.or_create.restype = vp
        L.or_create.argtypes = [P(_Problem), C.c_char_p, i64]
        L.or_destroy.argtypes = [vp]
        L.or_get_counts.argtypes = [vp, P(_Counts)]
        L.or_trace3d.restype = i64
        L.or_trace3d.argtypes = [vp, i64, vp, vp, i64]
        L.or_track_checksums.argtypes = [vp, i64, i64, vp, vp, vp, vp, vp]
        L.or_total_segments3d.restype = i64
        L.or_total_segments3d.argtypes = [vp]
        L.or_links3d.restype = C.c_int
        L.or_links3d.argtypes = [vp, vp, C.c_char_p, i64]
        L.or_volumes.argtypes = [vp, vp, vp]
        L.or_fsr_material.argtypes = [vp, vp]
        L.or_get_tracks2d.argtypes = [vp] + [vp] * 12
        L.or_get_segments2d.argtypes = [vp, vp, vp]
        L.or_get_azim.argtypes = [vp, vp, vp, vp, vp, vp]
        L.or_get_polar.argtypes = [vp, vp, vp, vp, vp]
        L.or_get_polar_gl.argtypes = [vp, vp, vp]
        L.or_get_stacks.argtypes = [vp, vp, vp, vp]
        L.or_solve.restype = C.c_int
        L.or_solve.argtypes = [vp, C.c_int, C.c_int, dbl, dbl, P(dbl), vp, vp, vp, P(dbl), P(dbl),
                               P(dbl), C.c_char_p, i64]
        L.or_time_sample_sweep.restype = dbl
        L.or_time_sample_sweep.argtypes = [vp, i64, C.c_int, P(i64)]
        L.or_num_threads.restype = C.c_int
        L.or_segment_line.restype = i64
        L.or_segment_line.argtypes = [vp, dbl, dbl, dbl, dbl, dbl, vp, vp, i64]
        L.or_region_of.restype = i64
        L.or_region_of.argtypes = [vp, dbl, dbl]
        L.or_attenuate.restype = dbl
        L.or_attenuate.argtypes = [dbl, dbl, dbl, dbl, P(dbl)]
        L.or_source.argtypes = [C.c_int, vp, vp, vp, vp, vp, dbl, vp]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def attenuate(psi_in, q_over_sigma, sigma_t, s):
    """Eq. 3 for one segment and group; returns (psi_out, delta_psi)."""
    d = C.c_double()
    out = lib().or_attenuate(psi_in, q_over_sigma, sigma_t, s, C.byref(d))
    return out, d.value


def source(phi, sigma_t, sigma_s, nu_sigma_f, chi, k):
    """Reduced source qtilde_g = Q_g / Sigma_t,g with Q from S:301 (reading Q2)."""
    phi = np.ascontiguousarray(phi, np.float64)
    G = phi.size
    arrs = [np.ascontiguousarray(x, np.float64).ravel() for x in (sigma_t, sigma_s, nu_sigma_f, chi)]
    out = np.zeros(G)
    lib().or_source(G, _ptr(phi), *[_ptr(a) for a in arrs], float(k), _ptr(out))
    return out


class Oracle:
    """One problem laid down by the oracle (2D/3D tracks, segments, stacks)."""

    def __init__(self, prob: dict):
        self.prob = prob
        keep = []

        def arr(x, dt):
            a = np.ascontiguousarray(np.array(x, dtype=dt).ravel())
            keep.append(a)
            return a.ctypes.data_as(C.POINTER(C.c_int32 if dt == np.int32 else C.c_double))

        lat = prob["lattice"]
        types = prob["cell_types"]
        max_rings = max([len(t["radii"]) for t in types] + [0])
        n_zones = max(prob["axial"]["zone_of_layer"]) + 1
        radii = np.zeros((len(types), max(max_rings, 1)))
        mat = np.zeros((len(types), max_rings + 1, n_zones), np.int32)
        for i, t in enumerate(types):
            nr = len(t["radii"])
            radii[i, :nr] = t["radii"]
            for loc in range(nr + 1):
                src = t["material"][loc] if loc < nr else t["material"][-1]
                row = list(src) if isinstance(src, (list, tuple)) else [src]
                if len(row) == 1:
                    row = row * n_zones
                mat[i, loc, :] = row
            for loc in range(nr + 1, max_rings + 1):
                mat[i, loc, :] = mat[i, nr, :]
        mats = prob["materials"]
        G = len(mats[0]["sigma_t"])
        p = _Problem()
        p.nx, p.ny = lat["nx"], lat["ny"]
        p.pitch_x, p.pitch_y = lat["pitch_x"], lat["pitch_y"]
        p.cell_type = arr(lat["cell_type"], np.int32)
        p.n_types = len(types)
        p.max_rings = max_rings
        p.n_rings = arr([len(t["radii"]) for t in types], np.int32)
        p.radii = arr(radii[:, :max(max_rings, 1)] if max_rings else np.zeros(1), np.float64)
        p.n_layers = len(prob["axial"]["planes"]) - 1
        p.planes = arr(prob["axial"]["planes"], np.float64)
        p.n_zones = n_zones
        p.zone_of_layer = arr(prob["axial"]["zone_of_layer"], np.int32)
        p.material = arr(mat, np.int32)
        for f in range(6):
            p.bc[f] = int(prob["bc"][f])
        p.n_mat, p.G = len(mats), G
        p.sigma_t = arr([m["sigma_t"] for m in mats], np.float64)
        p.sigma_s = arr([m["sigma_s"] for m in mats], np.float64)
        p.nu_sigma_f = arr([m["nu_sigma_f"] for m in mats], np.float64)
        p.chi = arr([m["chi"] for m in mats], np.float64)
        q = prob["quadrature"]
        p.num_azim, p.num_polar = q["num_azim"], q["num_polar"]
        p.radial_spacing, p.axial_spacing = q["radial_spacing"], q["axial_spacing"]
        err = C.create_string_buffer(512)
        self._h = lib().or_create(C.byref(p), err, 512)
        if not self._h:
            raise ValueError("oracle: " + err.value.decode())
        c = _Counts()
        lib().or_get_counts(self._h, C.byref(c))
        self.counts = {f: getattr(c, f) for f, _ in _Counts._fields_}
        self.G = G
        self.N = q["num_polar"]
        self.M = q["num_azim"]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.or_destroy(h)
            self._h = None

    # --- laydown exports ---
    def tracks2d(self):
        n = self.counts["n_tracks2d"]
        out = dict(azim=np.zeros(n, np.int32), xy0=np.zeros((n, 2)), xy1=np.zeros((n, 2)), length=np.zeros(n),
                   seg_off=np.zeros(n + 1, np.int64), link_fwd=np.zeros(n, np.int64),
                   link_fwd_enters_fwd=np.zeros(n, np.int32), link_bwd=np.zeros(n, np.int64),
                   link_bwd_enters_fwd=np.zeros(n, np.int32), cycle=np.zeros(n, np.int64),
                   ltilde=np.zeros(n), sigma=np.zeros(n, np.int32))
        keys = ["azim", "xy0", "xy1", "length", "seg_off", "link_fwd", "link_fwd_enters_fwd", "link_bwd",
                "link_bwd_enters_fwd", "cycle", "ltilde", "sigma"]
        lib().or_get_tracks2d(self._h, *[_ptr(out[k]) for k in keys])
        return out

    def segments2d(self):
        n = self.counts["n_segs2d"]
        region, s_end = np.zeros(n, np.int64), np.zeros(n)
        lib().or_get_segments2d(self._h, _ptr(region), _ptr(s_end))
        return region, s_end

    def azim(self):
        m = self.M // 2
        phi, nx, ny, delta, omega = np.zeros(m), np.zeros(m, np.int32), np.zeros(m, np.int32), np.zeros(m), np.zeros(m)
        lib().or_get_azim(self._h, _ptr(phi), _ptr(nx), _ptr(ny), _ptr(delta), _ptr(omega))
        return dict(phi=phi, nx=nx, ny=ny, delta=delta, omega=omega)

    def polar(self):
        m = (self.M // 2) * self.N
        th, dz, w, ap = np.zeros(m), np.zeros(m), np.zeros(m), np.zeros(m)
        lib().or_get_polar(self._h, _ptr(th), _ptr(dz), _ptr(w), _ptr(ap))
        mu, wg = np.zeros(self.N), np.zeros(self.N)
        lib().or_get_polar_gl(self._h, _ptr(mu), _ptr(wg))
        shp = (self.M // 2, self.N)
        return dict(theta=th.reshape(shp), dz=dz.reshape(shp), weight=w.reshape(shp), aperp=ap.reshape(shp),
                    mu=mu, w_gl=wg)

    def stacks(self):
        ns = self.counts["n_stacks"]
        z0, cnt, first = np.zeros(ns), np.zeros(ns, np.int64), np.zeros(ns + 1, np.int64)
        lib().or_get_stacks(self._h, _ptr(z0), _ptr(cnt), _ptr(first))
        return dict(z0=z0, count=cnt, first=first)

    def trace3d(self, track: int):
        cap = 4096
        while True:
            f, l = np.zeros(cap, np.int64), np.zeros(cap)
            n = lib().or_trace3d(self._h, int(track), _ptr(f), _ptr(l), cap)
            if n >= 0:
                return f[:n], l[:n]
            cap = -n

    def checksums(self, first=0, n=None):
        if n is None:
            n = self.counts["n_tracks3d"] - first
        nseg, h, sl, ch = np.zeros(n, np.int32), np.zeros(n, np.uint64), np.zeros(n), np.zeros(n)
        rh = np.zeros(n, np.uint64)
        lib().or_track_checksums(self._h, int(first), int(n), _ptr(nseg), _ptr(h), _ptr(sl), _ptr(ch), _ptr(rh))
        return dict(nseg=nseg, hash=h, suml=sl, chord=ch, rhash=rh)

    def total_segments3d(self):
        return int(lib().or_total_segments3d(self._h))

    def links3d(self):
        link = np.zeros(2 * self.counts["n_tracks3d"], np.int64)
        err = C.create_string_buffer(512)
        if lib().or_links3d(self._h, _ptr(link), err, 512) != 0:
            raise RuntimeError("oracle links: " + err.value.decode())
        return link

    def volumes(self):
        J = self.counts["n_fsr"]
        vt, va = np.zeros(J), np.zeros(J)
        lib().or_volumes(self._h, _ptr(vt), _ptr(va))
        return vt, va

    def fsr_material(self):
        m = np.zeros(self.counts["n_fsr"], np.int32)
        lib().or_fsr_material(self._h, _ptr(m))
        return m

    def solve(self, fixed_iters=0, max_iter=2000, tol_k=1e-7, tol_src=1e-6):
        """Power iteration.  Returns a dict with k, iterations,
        k/residual histories, phi[J][G] (normalised sum V F = 1), leakage,
        production and absorption (for the balance pin P15)."""
        J, G = self.counts["n_fsr"], self.G
        lim = fixed_iters if fixed_iters > 0 else max_iter
        kh, rh = np.zeros(lim), np.zeros(lim)
        phi = np.zeros((J, G))
        k, leak, prod, absn = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        err = C.create_string_buffer(512)
        it = lib().or_solve(self._h, int(fixed_iters), int(max_iter), float(tol_k), float(tol_src), C.byref(k),
                            _ptr(kh), _ptr(rh), _ptr(phi), C.byref(leak), C.byref(prod), C.byref(absn), err, 512)
        if it < 0:
            raise RuntimeError("oracle solve: " + err.value.decode())
        return dict(k=k.value, iterations=it, k_hist=kh[:it], res_hist=rh[:it], phi=phi, leakage=leak.value,
                    production=prod.value, absorption=absn.value)

    def segment_line(self, x0, y0, ux, uy, L):
        reg, se = np.zeros(4096, np.int64), np.zeros(4096)
        n = lib().or_segment_line(self._h, x0, y0, ux, uy, L, _ptr(reg), _ptr(se), 4096)
        assert n >= 0
        return reg[:n], se[:n]

    def region_of(self, x, y):
        return int(lib().or_region_of(self._h, x, y))

    def time_sample_sweep(self, stride: int, nthreads: int = 0):
        nint = C.c_int64()
        sec = lib().or_time_sample_sweep(self._h, int(stride), int(nthreads), C.byref(nint))
        return sec, nint.value


def num_threads() -> int:
    return int(lib().or_num_threads())
