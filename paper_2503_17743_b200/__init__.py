"""Thin Python binding of libmoc3d.so (include/moc3d.h) — argument marshalling only.

Every step of the hot path runs in the library's host C++ (laydown, once) and
CUDA kernels (sweep and power iteration).  There is no Python or CPU fallback:
if ``libmoc3d.so`` cannot be loaded, importing the binding raises.

``Problem`` marshals a problem dict (schema in ``problems/__init__.py``) into
``moc_set_materials`` / ``moc_set_geometry`` / ``moc_generate_tracks``;
``Solver`` wraps ``moc_solver_create`` .. ``moc_get_timings``.  Raw ABI
functions are available under the same names via ``lib()``.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MOC3D_LIB selects an in-tree variant build (A/B performance runs); default is the product build
SO_PATH = os.environ.get("MOC3D_LIB") or os.path.join(_HERE, "libmoc3d.so")

MOC_OK = 0
ERRORS = {
    -1: "MOC_E_INVALID_ARG", -2: "MOC_E_GEOMETRY", -3: "MOC_E_REFERENCE", -4: "MOC_E_MESH",
    -5: "MOC_E_PARAM", -6: "MOC_E_TRACE", -7: "MOC_E_CAPACITY", -8: "MOC_E_EIGEN", -9: "MOC_E_NUMERIC",
    -10: "MOC_E_NOCONV", -11: "MOC_E_CUDA", -12: "MOC_E_NCCL", -13: "MOC_E_STATE",
}


class MocError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class moc_geometry_desc(C.Structure):
    _fields_ = [
        ("nx", C.c_int32), ("ny", C.c_int32), ("pitch_x", C.c_double), ("pitch_y", C.c_double),
        ("cell_type", C.c_void_p), ("n_types", C.c_int32), ("max_rings", C.c_int32),
        ("n_rings", C.c_void_p), ("radii", C.c_void_p), ("n_layers", C.c_int32), ("planes", C.c_void_p),
        ("n_zones", C.c_int32), ("zone_of_layer", C.c_void_p), ("material", C.c_void_p), ("bc", C.c_int32 * 6),
    ]


class moc_track_params(C.Structure):
    _fields_ = [("num_azim", C.c_int32), ("num_polar", C.c_int32), ("radial_spacing", C.c_double),
                ("axial_spacing", C.c_double)]


class moc_track_stats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("n_fsr", "n_regions", "n_tracks2d", "n_segs2d", "n_stacks", "n_tracks3d",
                                         "n_cycles", "n_segs3d_raw")]


MOC_COMM_CALLER, MOC_COMM_NCCL = 0, 1
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p)


class moc_comm_desc(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("backend", C.c_int32),
                ("nccl_id", C.c_uint8 * 128)]


class moc_solver_opts(C.Structure):
    _fields_ = [("schedule", C.c_int32), ("threads", C.c_int32), ("blocks", C.c_int32),
                ("deterministic", C.c_int32), ("tile_cells", C.c_int32), ("exp_mode", C.c_int32),
                ("exp_budget_mb", C.c_int32), ("exp_fraction", C.c_double),
                ("sc_lanes_per_cell", C.c_int32), ("sc_psi_cap", C.c_int32), ("v2_lane_stride", C.c_int32),
                ("no_graph", C.c_int32), ("gauss_seidel", C.c_int32), ("sc_ctas_per_sm", C.c_int32)]


class moc_solve_opts(C.Structure):
    _fields_ = [("tol_k", C.c_double), ("tol_src", C.c_double), ("max_iter", C.c_int32),
                ("check_every", C.c_int32)]


class moc_result(C.Structure):
    _fields_ = [("k", C.c_double), ("residual", C.c_double), ("iterations", C.c_int32), ("converged", C.c_int32)]


class moc_timings(C.Structure):
    _fields_ = [("n_segs3d", C.c_int64), ("n_integrations", C.c_int64), ("sweep_ms_last", C.c_double),
                ("iter_ms_last", C.c_double), ("launches_per_iter", C.c_int64), ("setup_ms", C.c_double),
                ("device_bytes", C.c_int64), ("exp_segments", C.c_int64), ("exp_bytes", C.c_int64),
                ("emitted_last", C.c_int64), ("sc_units", C.c_int64 * 3)]


class moc_comm_buffers(C.Structure):
    _fields_ = [("tally", C.c_void_p), ("tally_elems", C.c_int64), ("halo_send", C.c_void_p),
                ("halo_recv", C.c_void_p), ("halo_elems", C.c_int64)]


# name -> (restype, argtypes); every symbol declared in include/moc3d.h
_vp, _i32, _i64, _d = C.c_void_p, C.c_int32, C.c_int64, C.c_double
_P = C.POINTER
SIGNATURES = {
    "moc_problem_create": (C.c_int, [_P(_vp)]),
    "moc_problem_destroy": (None, [_vp]),
    "moc_last_error": (C.c_char_p, [_vp]),
    "moc_set_materials": (C.c_int, [_vp, _i32, _i32, _vp, _vp, _vp, _vp]),
    "moc_set_geometry": (C.c_int, [_vp, _P(moc_geometry_desc)]),
    "moc_num_fsrs": (C.c_int, [_vp, _P(_i64)]),
    "moc_fsr_of_point": (C.c_int, [_vp, _d, _d, _d, _P(_i64)]),
    "moc_generate_tracks": (C.c_int, [_vp, _P(moc_track_params)]),
    "moc_get_track_stats": (C.c_int, [_vp, _P(moc_track_stats)]),
    "moc_get_tracks2d": (C.c_int, [_vp] + [_vp] * 9),
    "moc_get_segments2d": (C.c_int, [_vp, _vp, _vp]),
    "moc_get_stacks": (C.c_int, [_vp, _vp, _vp, _vp]),
    "moc_get_polar": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "moc_get_links3d": (C.c_int, [_vp, _vp]),
    "moc_trace_track_3d": (C.c_int, [_vp, _i64, _vp, _vp, _i64, _P(_i64)]),
    "moc_z_of": (_d, [_d, _d, _i64, _d, _d]),
    "moc_intersecting_range": (None, [_d, _d, _d, _d, _d, _P(_i64), _P(_i64)]),
    "moc_full_crossing_range": (None, [_d, _d, _d, _d, _d, _P(_i64), _P(_i64)]),
    "moc_flat_index": (_i64, [_vp, _i64, _i64, _i64, _i64]),
    "moc_serpentine_order": (C.c_int, [_vp, _i64, _i64, _vp]),
    "moc_partition_exp_otf": (C.c_int, [_vp, _i64, _d, _d, _vp]),
    "moc_partition_stacks": (C.c_int, [_vp, _i32, _vp, _vp]),
    "moc_halo_plan": (C.c_int, [_vp, _i32, _vp, _i32, _i32, _vp, _i64, _P(_i64)]),
    "moc_solver_create": (C.c_int, [_P(_vp), _vp, C.c_int, _vp, _P(moc_comm_desc), _P(moc_solver_opts)]),
    "moc_solver_destroy": (C.c_int, [_vp]),
    "moc_solver_last_error": (C.c_char_p, [_vp]),
    "moc_iterate": (C.c_int, [_vp, _i32, _P(_d), _P(_d)]),
    "moc_solve": (C.c_int, [_vp, _P(moc_solve_opts), _P(moc_result)]),
    "moc_reset": (C.c_int, [_vp]),
    "moc_solver_update_materials": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "moc_get_scalar_flux": (C.c_int, [_vp, _vp]),
    "moc_get_fsr_volumes": (C.c_int, [_vp, _vp, _vp]),
    "moc_get_history": (C.c_int, [_vp, _vp, _vp, _i32, _P(_i32)]),
    "moc_get_balance": (C.c_int, [_vp, _P(_d), _P(_d), _P(_d)]),
    "moc_device_trace_checksums": (C.c_int, [_vp, _i64, _i64, _vp, _vp, _vp]),
    "moc_get_timings": (C.c_int, [_vp, _P(moc_timings)]),
    "moc_solver_comm_buffers": (C.c_int, [_vp, _P(moc_comm_buffers)]),
    "moc_solver_halo_counts": (C.c_int, [_vp, _vp, _vp]),
    "moc_attenuation_probe": (C.c_int, [C.c_int, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "moc_sweep_checksums": (C.c_int, [_vp, _vp, _vp]),
    "moc_iteration_sweep": (C.c_int, [_vp]),
    "moc_rank_layout": (C.c_int, [_vp, C.c_int32, _vp, C.c_int32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "moc_problem_fsr_volumes": (C.c_int, [_vp, _vp, _vp]),
    "moc_nccl_unique_id": (C.c_int, [_vp]),
    "moc_solver_set_exchange": (C.c_int, [_vp, EXCHANGE_FN, _vp]),
    "moc_iteration_finish": (C.c_int, [_vp]),
}
# host-only test hook (not in the public header): backward OTF walk of one track
_EXTRA = {"moc_trace_track_3d_backward": (C.c_int, [_vp, _i64, _vp, _vp, _i64, _P(_i64)])}

_lib = None


def lib():
    """Load libmoc3d.so (raises if it is missing: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise ImportError(f"{SO_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(SO_PATH)
        for name, (res, args) in {**SIGNATURES, **_EXTRA}.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _check(rc, h, errf):
    if rc != MOC_OK:
        msg = errf(h).decode() if h else ""
        raise MocError(rc, msg)


class Problem:
    """Geometry + materials + host laydown."""

    def __init__(self, prob: dict, generate: bool = True):
        L = lib()
        self._h = C.c_void_p()
        _check(L.moc_problem_create(C.byref(self._h)), None, None)
        self.prob = prob
        self._keep = []
        mats = prob["materials"]
        G = len(mats[0]["sigma_t"])
        self.G = G
        st = np.ascontiguousarray([m["sigma_t"] for m in mats], np.float64)
        ss = np.ascontiguousarray([m["sigma_s"] for m in mats], np.float64)
        nf = np.ascontiguousarray([m["nu_sigma_f"] for m in mats], np.float64)
        ch = np.ascontiguousarray([m["chi"] for m in mats], np.float64)
        self._call(L.moc_set_materials, len(mats), G, _p(st), _p(ss), _p(nf), _p(ch))
        self._set_geometry(prob)
        if generate:
            q = prob["quadrature"]
            tp = moc_track_params(q["num_azim"], q["num_polar"], q["radial_spacing"], q["axial_spacing"])
            self._call(L.moc_generate_tracks, C.byref(tp))

    def _call(self, f, *args):
        _check(f(self._h, *args), self._h, lib().moc_last_error)

    def _set_geometry(self, prob):
        lat, types, ax = prob["lattice"], prob["cell_types"], prob["axial"]
        max_rings = max([len(t["radii"]) for t in types] + [0])
        n_zones = max(ax["zone_of_layer"]) + 1
        radii = np.zeros((len(types), max(max_rings, 1)))
        mat = np.zeros((len(types), max_rings + 1, n_zones), np.int32)
        for i, t in enumerate(types):
            nr = len(t["radii"])
            radii[i, :nr] = t["radii"]
            for loc in range(max_rings + 1):
                src = t["material"][min(loc, nr)]
                row = list(src) if isinstance(src, (list, tuple)) else [src]
                mat[i, loc, :] = row * n_zones if len(row) == 1 else row
        arrs = dict(
            cell_type=np.ascontiguousarray(lat["cell_type"], np.int32),
            n_rings=np.ascontiguousarray([len(t["radii"]) for t in types], np.int32),
            radii=np.ascontiguousarray(radii[:, :max_rings] if max_rings else np.zeros(1)),
            planes=np.ascontiguousarray(ax["planes"], np.float64),
            zone_of_layer=np.ascontiguousarray(ax["zone_of_layer"], np.int32),
            material=np.ascontiguousarray(mat, np.int32),
        )
        self._keep.append(arrs)
        d = moc_geometry_desc()
        d.nx, d.ny, d.pitch_x, d.pitch_y = lat["nx"], lat["ny"], lat["pitch_x"], lat["pitch_y"]
        d.cell_type = arrs["cell_type"].ctypes.data
        d.n_types, d.max_rings = len(types), max_rings
        d.n_rings = arrs["n_rings"].ctypes.data
        d.radii = arrs["radii"].ctypes.data
        d.n_layers = len(ax["planes"]) - 1
        d.planes = arrs["planes"].ctypes.data
        d.n_zones = n_zones
        d.zone_of_layer = arrs["zone_of_layer"].ctypes.data
        d.material = arrs["material"].ctypes.data
        for f in range(6):
            d.bc[f] = int(prob["bc"][f])
        self._call(lib().moc_set_geometry, C.byref(d))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.moc_problem_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def stats(self) -> dict:
        s = moc_track_stats()
        self._call(lib().moc_get_track_stats, C.byref(s))
        return {f: getattr(s, f) for f, _ in moc_track_stats._fields_}

    def num_fsrs(self) -> int:
        J = C.c_int64()
        self._call(lib().moc_num_fsrs, C.byref(J))
        return J.value

    def fsr_of_point(self, x, y, z) -> int:
        j = C.c_int64()
        self._call(lib().moc_fsr_of_point, float(x), float(y), float(z), C.byref(j))
        return j.value

    def tracks2d(self) -> dict:
        n = self.stats()["n_tracks2d"]
        o = dict(azim=np.zeros(n, np.int32), xy0=np.zeros((n, 2)), xy1=np.zeros((n, 2)), length=np.zeros(n),
                 seg_off=np.zeros(n + 1, np.int64), link_fwd=np.zeros(n, np.int64),
                 link_fwd_enters_fwd=np.zeros(n, np.int32), link_bwd=np.zeros(n, np.int64),
                 link_bwd_enters_fwd=np.zeros(n, np.int32))
        self._call(lib().moc_get_tracks2d, *[_p(o[k]) for k in ("azim", "xy0", "xy1", "length", "seg_off", "link_fwd",
                                                                 "link_fwd_enters_fwd", "link_bwd",
                                                                 "link_bwd_enters_fwd")])
        return o

    def segments2d(self):
        n = self.stats()["n_segs2d"]
        r, s = np.zeros(n, np.int64), np.zeros(n)
        self._call(lib().moc_get_segments2d, _p(r), _p(s))
        return r, s

    def stacks(self) -> dict:
        ns = self.stats()["n_stacks"]
        z0, cnt, first = np.zeros(ns), np.zeros(ns, np.int64), np.zeros(ns + 1, np.int64)
        self._call(lib().moc_get_stacks, _p(z0), _p(cnt), _p(first))
        return dict(z0=z0, count=cnt, first=first)

    def polar(self) -> dict:
        q = self.prob["quadrature"]
        shp = (q["num_azim"] // 2, q["num_polar"])
        a = [np.zeros(shp) for _ in range(4)]
        self._call(lib().moc_get_polar, *[_p(x) for x in a])
        return dict(theta=a[0], dz=a[1], weight=a[2], aperp=a[3])

    def links3d(self) -> np.ndarray:
        n = self.stats()["n_tracks3d"]
        link = np.zeros(2 * n, np.int64)
        self._call(lib().moc_get_links3d, _p(link))
        return link

    def partition(self, world: int):
        """Stack owner per rank and raw segment cost per rank."""
        S = self.stats()["n_stacks"]
        owner, cost = np.zeros(S, np.int32), np.zeros(world)
        self._call(lib().moc_partition_stacks, int(world), _p(owner), _p(cost))
        return owner, cost

    def halo_plan(self, world: int, owner, rank: int, peer: int):
        own = np.ascontiguousarray(owner, np.int32)
        n = C.c_int64()
        self._call(lib().moc_halo_plan, int(world), _p(own), int(rank), int(peer), None, 0, C.byref(n))
        out = np.zeros(n.value, np.int64)
        self._call(lib().moc_halo_plan, int(world), _p(own), int(rank), int(peer), _p(out), n.value, C.byref(n))
        return out

    def fsr_volumes(self):
        """(track-estimated, analytic) FSR volumes [J] from the host walk (no GPU)."""
        J = self.num_fsrs()
        vt, va = np.zeros(J), np.zeros(J)
        self._call(lib().moc_problem_fsr_volumes, _p(vt), _p(va))
        return vt, va

    def rank_layout(self, world: int, owner, rank: int) -> dict:
        """The solver's per-rank track numbering, local link table and halo layout."""
        own = np.ascontiguousarray(owner, np.int32)
        sz = np.zeros(3, np.int64)
        L = lib()
        self._call(L.moc_rank_layout, int(world), _p(own), int(rank), _p(sz), None, None, None, None, None)
        S = self.stats()["n_stacks"]
        sf, lk, rs = np.zeros(S + 1, np.int64), np.zeros(2 * sz[0], np.int64), np.zeros(sz[2], np.int64)
        sc, rc = np.zeros(world, np.int64), np.zeros(world, np.int64)
        self._call(L.moc_rank_layout, int(world), _p(own), int(rank), _p(sz), _p(sf), _p(lk), _p(rs), _p(sc), _p(rc))
        return dict(T3_local=int(sz[0]), n_send=int(sz[1]), slot_first=sf, link=lk, recv_slots=rs, send_counts=sc,
                    recv_counts=rc)

    def trace_track_3d(self, track: int, backward: bool = False):
        nseg = C.c_int64()
        f = lib().moc_trace_track_3d_backward if backward else lib().moc_trace_track_3d
        rc = f(self._h, int(track), None, None, 0, C.byref(nseg))
        if rc not in (MOC_OK, -1):
            _check(rc, self._h, lib().moc_last_error)
        fsr, ln = np.zeros(nseg.value, np.int64), np.zeros(nseg.value)
        self._call(f, int(track), _p(fsr), _p(ln), nseg.value, C.byref(nseg))
        return fsr, ln


class _DeviceArray:
    """Minimal __cuda_array_interface__ holder so torch can view a library-owned buffer."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f4", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class Solver:
    """Device state + power iteration on one GPU (one rank)."""

    def __init__(self, problem: Problem, device: int = 0, stream=None, schedule: int = 3, threads: int = 0,
                 blocks: int = 0, rank: int = 0, world: int = 1, tile_cells: int = 0, exp_mode: int = 0,
                 exp_budget_mb: int = 0, exp_fraction: float = 0.0, sc_lanes_per_cell: int = 0,
                 sc_psi_cap: int = 0, v2_lane_stride: int = 0, no_graph: bool = False, backend: str | None = None,
                 gauss_seidel: bool = False, sc_ctas_per_sm: int = 0):
        """world > 1: one rank of a torch.distributed job.  backend "nccl"
        (default when the process group is NCCL): the library owns an NCCL communicator
        and runs the whole iteration on the device; "gloo": the exchange is staged through
        host memory by a Python callback (tests, several ranks on one GPU)."""
        L = lib()
        self.problem = problem
        self._h = C.c_void_p()
        self._xfn = None
        if stream is None:
            try:
                import torch
                stream = torch.cuda.current_stream(device).cuda_stream
            except Exception:  # torch without CUDA: legacy default stream
                stream = 0
        opts = moc_solver_opts(schedule, threads, blocks, 0, tile_cells, exp_mode, exp_budget_mb, exp_fraction,
                               sc_lanes_per_cell, sc_psi_cap, v2_lane_stride, int(bool(no_graph)),
                               int(bool(gauss_seidel)), sc_ctas_per_sm)
        comm = moc_comm_desc(rank, world, MOC_COMM_CALLER)
        if world == 1 and backend == "nccl":  # 1-rank communicator (tests the NCCL path on one GPU)
            comm.backend = MOC_COMM_NCCL
            _check(L.moc_nccl_unique_id(comm.nccl_id), None, None)
        if world > 1:
            import torch.distributed as dist
            backend = backend or ("nccl" if dist.get_backend() == "nccl" else "gloo")
            if backend == "nccl":
                comm.backend = MOC_COMM_NCCL
                uid = (C.c_uint8 * 128)()
                if rank == 0:
                    _check(L.moc_nccl_unique_id(uid), None, None)
                obj = [bytes(uid)]
                dist.broadcast_object_list(obj, src=0)
                C.memmove(comm.nccl_id, obj[0], 128)
        self.backend = backend if world > 1 else None
        rc = L.moc_solver_create(C.byref(self._h), problem.handle, device, C.c_void_p(stream), C.byref(comm),
                                 C.byref(opts))
        if rc != MOC_OK:
            raise MocError(rc, L.moc_last_error(problem.handle).decode())
        self.G = problem.G
        self.J = problem.num_fsrs()
        self.world, self.rank, self.device = world, rank, device
        self._comm = None
        if world > 1 and self.backend != "nccl":
            self._xfn = EXCHANGE_FN(self._host_exchange)
            self._call(L.moc_solver_set_exchange, self._xfn, None)

    def _host_exchange(self, _ctx):
        """Exchange callback (backend gloo): sum all-reduce of the tally and all-to-all of
        the cut-crossing boundary psi, staged through host memory.  Every rank takes part
        in both collectives every iteration (an empty halo still participates)."""
        try:
            import torch.distributed as dist
            c = self._comm_tensors()
            t = c["tally"].cpu()
            dist.all_reduce(t)
            c["tally"].copy_(t)
            rbuf = c["recv"].cpu()
            dist.all_to_all_single(rbuf, c["send"].cpu(), c["recv_splits"], c["send_splits"])
            c["recv"].copy_(rbuf)
            import torch
            torch.cuda.current_stream(self.device).synchronize()
            return 0
        except Exception:  # reported by the library as MOC_E_NCCL
            import traceback
            traceback.print_exc()
            return 1

    def _comm_tensors(self):
        """torch views (via __cuda_array_interface__) of the library's tally and halo
        buffers, for the caller-driven NCCL all-reduce / all-to-all."""
        if self._comm is None:
            import torch
            b = self.comm_buffers()
            se, re = np.zeros(self.world, np.int64), np.zeros(self.world, np.int64)
            self._call(lib().moc_solver_halo_counts, _p(se), _p(re))
            dev = torch.device("cuda", self.device)

            def view(ptr, n):
                if n == 0 or not ptr:
                    return torch.zeros(0, dtype=torch.float32, device=dev)
                return torch.as_tensor(_DeviceArray(ptr, n), device=dev)

            self._comm = dict(tally=view(b["tally"], b["tally_elems"]),
                              send=view(b["halo_send"], int(se.sum())), recv=view(b["halo_recv"], int(re.sum())),
                              send_splits=se.tolist(), recv_splits=re.tolist())
        return self._comm

    def _call(self, f, *args):
        _check(f(self._h, *args), self._h, lib().moc_solver_last_error)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.moc_solver_destroy(h)
            self._h = None

    def close(self):
        self.__del__()

    def iterate(self, n: int):
        """n power iterations (multi-rank: the exchange runs inside the library)."""
        k, r = C.c_double(), C.c_double()
        self._call(lib().moc_iterate, int(n), C.byref(k), C.byref(r))
        return k.value, r.value

    def iterate_split(self, n: int):
        """Caller-driven multi-rank iteration (moc_iteration_sweep / _finish with the
        collectives issued from Python on torch's stream); the reference for the in-library
        exchange in tests."""
        import torch.distributed as dist
        c = self._comm_tensors()
        host = dist.get_backend() != "nccl"
        for _ in range(int(n)):
            self._call(lib().moc_iteration_sweep)
            if host:
                t = c["tally"].cpu()
                dist.all_reduce(t)
                c["tally"].copy_(t)
                rbuf = c["recv"].cpu()
                dist.all_to_all_single(rbuf, c["send"].cpu(), c["recv_splits"], c["send_splits"])
                c["recv"].copy_(rbuf)
            else:
                dist.all_reduce(c["tally"])
                dist.all_to_all_single(c["recv"], c["send"], c["recv_splits"], c["send_splits"])
            self._call(lib().moc_iteration_finish)
        return self.iterate(0)

    def solve(self, tol_k=1e-7, tol_src=1e-6, max_iter=5000, check_every=10):
        o = moc_solve_opts(tol_k, tol_src, max_iter, check_every)
        r = moc_result()
        self._call(lib().moc_solve, C.byref(o), C.byref(r))
        return dict(k=r.k, residual=r.residual, iterations=r.iterations, converged=bool(r.converged))

    def reset(self):
        self._call(lib().moc_reset)

    def update_materials(self, sigma_t, sigma_s, nu_sigma_f, chi):
        """Host fp64 arrays [n_mat][G] / [n_mat][G][G]; copied H2D on the solver stream."""
        a = [np.ascontiguousarray(x, np.float64) for x in (sigma_t, sigma_s, nu_sigma_f, chi)]
        self._call(lib().moc_solver_update_materials, *[_p(x) for x in a])

    def scalar_flux(self) -> np.ndarray:
        phi = np.zeros((self.J, self.G))
        self._call(lib().moc_get_scalar_flux, _p(phi))
        return phi

    def fsr_volumes(self, analytic: bool = False):
        """Track-estimated FSR volumes [J]; with analytic=True also the analytic ones
         as a second array."""
        v = np.zeros(self.J)
        if not analytic:
            self._call(lib().moc_get_fsr_volumes, _p(v), None)
            return v
        va = np.zeros(self.J)
        self._call(lib().moc_get_fsr_volumes, _p(v), _p(va))
        return v, va

    def history(self):
        n = C.c_int32()
        self._call(lib().moc_get_history, None, None, 0, C.byref(n))
        k, r = np.zeros(max(n.value, 1)), np.zeros(max(n.value, 1))
        self._call(lib().moc_get_history, _p(k), _p(r), n.value, C.byref(n))
        return k[:n.value], r[:n.value]

    def balance(self):
        p, a, l = C.c_double(), C.c_double(), C.c_double()
        self._call(lib().moc_get_balance, C.byref(p), C.byref(a), C.byref(l))
        return dict(production=p.value, absorption=a.value, leakage=l.value)

    def checksums(self, first: int = 0, n: int | None = None):
        if n is None:
            n = self.problem.stats()["n_tracks3d"] - first
        nseg, h, sl = np.zeros(n, np.int32), np.zeros(n, np.uint64), np.zeros(n)
        self._call(lib().moc_device_trace_checksums, int(first), int(n), _p(nseg), _p(h), _p(sl))
        return dict(nseg=nseg, hash=h, suml=sl)

    def sweep_checksums(self):
        """Schedule 3: one checksum-mode sweep; per slot (2*track + dir) the number of
        segments the kernel applied and the FNV-1a-64 of their FSR ids in travel order."""
        n = 2 * self.problem.stats()["n_tracks3d"]
        nseg, h = np.zeros(n, np.int32), np.zeros(n, np.uint64)
        self._call(lib().moc_sweep_checksums, _p(nseg), _p(h))
        return nseg, h

    def timings(self) -> dict:
        t = moc_timings()
        self._call(lib().moc_get_timings, C.byref(t))
        return {f: (list(getattr(t, f)) if isinstance(getattr(t, f), C.Array) else getattr(t, f))
                for f, _ in moc_timings._fields_}

    def comm_buffers(self) -> dict:
        b = moc_comm_buffers()
        self._call(lib().moc_solver_comm_buffers, C.byref(b))
        return {f: getattr(b, f) for f, _ in moc_comm_buffers._fields_}


# module-level aliases with the ABI names (Eqs. 5-7, 9-10, 13; §4.2, §4.3)
def moc_z_of(z0, dz, i, theta, s):
    return lib().moc_z_of(z0, dz, int(i), theta, s)


def moc_intersecting_range(z0s, z0e, dz, zmin, zmax):
    a, b = C.c_int64(), C.c_int64()
    lib().moc_intersecting_range(z0s, z0e, dz, zmin, zmax, C.byref(a), C.byref(b))
    return a.value, b.value


def moc_full_crossing_range(z0s, z0e, dz, zmin, zmax):
    a, b = C.c_int64(), C.c_int64()
    lib().moc_full_crossing_range(z0s, z0e, dz, zmin, zmax, C.byref(a), C.byref(b))
    return a.value, b.value


def moc_flat_index(offsets, c, i, j, k):
    off = np.ascontiguousarray(offsets, np.int64)
    return int(lib().moc_flat_index(_p(off), int(c), int(i), int(j), int(k)))


def moc_attenuation_probe(psi, q, sigma_t, length, device=0):
    """The sweep kernel's Eq. 3 arithmetic on the device; returns (psi_out, dpsi) fp32."""
    a = [np.ascontiguousarray(x, np.float32).ravel() for x in (psi, q, sigma_t, length)]
    n = a[0].size
    po, dp = np.zeros(n, np.float32), np.zeros(n, np.float32)
    _check(lib().moc_attenuation_probe(int(device), n, *[_p(x) for x in a], _p(po), _p(dp)), None, None)
    return po, dp


def moc_serpentine_order(counts, chunk):
    c = np.ascontiguousarray(counts, np.int64)
    out = np.zeros(len(c), np.int64)
    _check(lib().moc_serpentine_order(_p(c), len(c), int(chunk), _p(out)), None, None)
    return out


def moc_partition_exp_otf(estimates, budget, fraction):
    e = np.ascontiguousarray(estimates, np.int64)
    out = np.zeros(len(e), np.int32)
    _check(lib().moc_partition_exp_otf(_p(e), len(e), float(budget), float(fraction), _p(out)), None, None)
    return out.astype(bool)
