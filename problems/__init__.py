"""Seeded synthetic problem generators shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no tracking, no attenuation, no
source, no eigenvalue math).  It only writes down problem descriptions — pin
lattices, axial meshes, boundary conditions, quadrature parameters and
cross-section tables — as plain Python dicts.  Both ``oracle/`` and
``paper_2503_17743_b200`` marshal these dicts into their own C structures with
their own code.

Configs follow BASELINE.json ``configs`` as made concrete in SURVEY.md §8(d)
(table "Configs as concrete synthetic inputs") and Appendix B (cross sections).

Dict schema::

    {
      "name": str,
      "materials": [{"name", "sigma_t"[G], "sigma_s"[G][G] (from->to),
                     "nu_sigma_f"[G], "chi"[G]}],
      "lattice": {"nx", "ny", "pitch_x", "pitch_y",
                  "cell_type": [ny*nx] row-major from (x_min, y_min)},
      "cell_types": [{"radii": [...ascending...],
                      "material": [[mat per zone] per local region]}],
                      # local region 0..n_rings-1 = rings inner->outer, last = moderator
      "axial": {"planes": [NL+1] starting at 0, "zone_of_layer": [NL]},
      "bc": [x-, x+, y-, y+, z-, z+]   (0 vacuum, 1 reflective),
      "quadrature": {"num_azim", "num_polar", "radial_spacing", "axial_spacing"},
    }
"""
from __future__ import annotations

import copy

import numpy as np

SEED = 17743  # XS generator seed (numpy PCG64)
PITCH = 1.26  # C5G7 pin pitch (cm)
FUEL_R = 0.54  # C5G7 fuel radius (cm)

VACUUM, REFLECTIVE = 0, 1


# ----------------------------------------------------------------------------
# cross sections
# ----------------------------------------------------------------------------
def xs_one_group():
    """1G: Sigma_t 1.0, Sigma_s 0.8, nuSigma_f 0.3, chi 1 (k_inf = 1.5)."""
    return [dict(name="mat1g", sigma_t=[1.0], sigma_s=[[0.8]], nu_sigma_f=[0.3], chi=[1.0])]


def xs_two_group():
    """2G set of App. B (fuel k_inf = 1.1, moderator non-fissile)."""
    fuel = dict(name="fuel2g", sigma_t=[0.5, 1.3], sigma_s=[[0.45, 0.02], [0.0, 1.10]],
                nu_sigma_f=[0.02, 0.35], chi=[1.0, 0.0])
    mod = dict(name="mod2g", sigma_t=[0.6, 2.0], sigma_s=[[0.55, 0.049], [0.0, 1.98]],
               nu_sigma_f=[0.0, 0.0], chi=[0.0, 0.0])
    return [fuel, mod]


C5G7_NAMES = ["UO2", "MOX4.3", "MOX7.0", "MOX8.7", "FC", "GT", "MOD", "CR"]
_FUEL_SHAPE = [0.18, 0.33, 0.48, 0.56, 0.31, 0.40, 0.57]
_MOD_SHAPE = [0.16, 0.41, 0.59, 0.58, 0.72, 1.25, 2.65]
_CR_SHAPE = [0.22, 0.48, 0.89, 0.97, 0.91, 1.14, 1.84]
_CHI = [0.58791, 0.41176, 3.3906e-4, 1.1761e-7, 0.0, 0.0, 0.0]


def xs_c5g7_synthetic(seed: int = SEED):
    """7-group C5G7-shaped synthetic set (App. B), deterministic in ``seed``.

    Sigma_t,g = shape_g (1 + 0.05 U(-1,1)); scattering ratio in [0.55, 0.999];
    downscatter up to 3 groups below, upscatter only among groups 5-7 (1-based)
    at 1-5% of the row; nuSigma_f > 0 only in the four fuels, MOX thermal
    groups 1.5-2.5x UO2; chi = normalised C5G7 shape.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    G = 7
    chi = np.array(_CHI) / np.sum(_CHI)
    mats = []
    for name in C5G7_NAMES:
        if name in ("UO2", "MOX4.3", "MOX7.0", "MOX8.7"):
            shape = np.array(_FUEL_SHAPE)
        elif name == "MOD":
            shape = np.array(_MOD_SHAPE)
        elif name in ("FC", "GT"):
            shape = 0.98 * np.array(_MOD_SHAPE)
        else:
            shape = np.array(_CR_SHAPE)
        st = shape * (1.0 + 0.05 * rng.uniform(-1.0, 1.0, G))
        if name in ("UO2", "MOX4.3", "MOX7.0", "MOX8.7"):
            ratio = rng.uniform(0.55, 0.80, G)
        elif name == "CR":
            ratio = rng.uniform(0.55, 0.70, G)
        else:
            ratio = rng.uniform(0.90, 0.999, G)
        ss = np.zeros((G, G))
        for g in range(G):
            row_total = ratio[g] * st[g]
            targets = list(range(g, min(G, g + 4)))  # self + up to 3 groups below
            w = rng.uniform(0.2, 1.0, len(targets))
            w[0] *= 4.0  # within-group dominant
            up = []
            if g >= 5:  # upscatter among groups 5..7 (0-based 4..6)
                up = [gp for gp in range(4, g)]
            if up:
                frac_up = rng.uniform(0.01, 0.05)
                wu = rng.uniform(0.5, 1.0, len(up))
                for gp, x in zip(up, wu):
                    ss[g, gp] = row_total * frac_up * x / wu.sum()
                row_total *= (1.0 - frac_up)
            for gp, x in zip(targets, w):
                ss[g, gp] += row_total * x / w.sum()
        nsf = np.zeros(G)
        if name in ("UO2", "MOX4.3", "MOX7.0", "MOX8.7"):
            base = rng.uniform(0.005, 0.02, G)
            base[4:] = rng.uniform(0.1, 0.3, 3)
            mult = {"UO2": 1.0, "MOX4.3": 1.5, "MOX7.0": 2.0, "MOX8.7": 2.5}[name]
            base[4:] *= mult
            nsf = np.clip(base, 0.005, 0.8)
            c = chi.copy()
        else:
            c = np.zeros(G)
        mats.append(dict(name=name, sigma_t=st.tolist(), sigma_s=ss.tolist(),
                         nu_sigma_f=nsf.tolist(), chi=c.tolist()))
    return mats


def load_xs_table(path: str, normalise_chi: bool = True):
    """Real NEA C5G7 cross sections from a user-supplied table (SURVEY §8(f) unranked item,
    P19: k-eff context against the published MCNP values; not a parity target).  JSON:

        {"materials": [{"name": "UO2", "sigma_tr": [7], "nu_sigma_f": [7], "chi": [7],
                        "sigma_s": [7][7] (from -> to)}, ...]}

    with the eight C5G7 materials (C5G7_NAMES; NEA/NSC/DOC(2003)16 tables typed in by the
    user: no data ships here).  sigma_t = the transport-corrected total sigma_tr (S:96,
    reading Q13: Sigma_a = sigma_tr - sum sigma_s may be slightly negative).  A fissile chi
    is renormalised to sum 1 (the published chi sums to 1.0000092; S:33 needs 1 +- 1e-9).
    Returns the materials list in C5G7_NAMES order (the index order configs 3-5 use)."""
    import json
    with open(path) as f:
        tab = json.load(f)
    by = {m["name"]: m for m in tab["materials"]}
    missing = [n for n in C5G7_NAMES if n not in by]
    if missing:
        raise ValueError(f"C5G7 table {path}: missing materials {missing}")
    out = []
    for name in C5G7_NAMES:
        m = by[name]
        st = np.asarray(m["sigma_tr"], np.float64)
        ss = np.asarray(m["sigma_s"], np.float64)
        nsf = np.asarray(m.get("nu_sigma_f", np.zeros(st.size)), np.float64)
        chi = np.asarray(m.get("chi", np.zeros(st.size)), np.float64)
        G = st.size
        if ss.shape != (G, G) or nsf.size != G or chi.size != G:
            raise ValueError(f"{name}: inconsistent group counts")
        if not (st > 0).all() or (ss < 0).any() or (nsf < 0).any() or (chi < 0).any():
            raise ValueError(f"{name}: sigma_tr must be > 0 and sigma_s, nu_sigma_f, chi >= 0")
        if nsf.sum() > 0:
            if abs(chi.sum() - 1.0) > 1e-4:
                raise ValueError(f"{name}: chi sums to {chi.sum()}")
            if normalise_chi:
                chi = chi / chi.sum()
        out.append(dict(name=name, sigma_t=st.tolist(), sigma_s=ss.tolist(), nu_sigma_f=nsf.tolist(),
                        chi=chi.tolist()))
    return out


def dump_xs_table(mats, path: str):
    """Write a materials list in load_xs_table's format (round-trip tests, templates)."""
    import json
    tab = {"materials": [dict(name=m["name"], sigma_tr=list(m["sigma_t"]), nu_sigma_f=list(m["nu_sigma_f"]),
                              chi=list(m["chi"]), sigma_s=[list(r) for r in m["sigma_s"]]) for m in mats]}
    with open(path, "w") as f:
        json.dump(tab, f, indent=1)


def with_xs(prob, mats):
    """Copy of ``prob`` with its materials list replaced (same order and count)."""
    if len(mats) != len(prob["materials"]):
        raise ValueError("material count differs")
    p = copy.deepcopy(prob)
    p["materials"] = copy.deepcopy(mats)
    return p


# ----------------------------------------------------------------------------
# geometry helpers
# ----------------------------------------------------------------------------
def xs_synthetic(G: int, n_mat: int = 7, seed: int = SEED):
    """G-group synthetic set with ``n_mat`` materials (tests of other group counts):
    material 0 and 1 fissile (fuel-like), the rest moderator / absorber-like.
    Sigma_t in [0.2, 2.5], scattering ratio 0.5-0.95 (fuel) / 0.85-0.99 (others),
    downscatter to up to 2 groups below plus within-group, chi on the fastest
    groups; deterministic in ``seed``."""
    rng = np.random.Generator(np.random.PCG64(seed + 1000 * G + n_mat))
    chi = np.zeros(G)
    chi[: max(1, (G + 1) // 2)] = rng.uniform(0.2, 1.0, max(1, (G + 1) // 2))
    chi /= chi.sum()
    mats = []
    for m in range(n_mat):
        fis = m < 2
        st = rng.uniform(0.2, 2.5, G)
        ratio = rng.uniform(0.5, 0.95, G) if fis else rng.uniform(0.85, 0.99, G)
        ss = np.zeros((G, G))
        for g in range(G):
            tg = list(range(g, min(G, g + 3)))
            w = rng.uniform(0.2, 1.0, len(tg))
            w[0] *= 3.0
            ss[g, tg] = ratio[g] * st[g] * w / w.sum()
        nf = rng.uniform(0.01, 0.3, G) * st if fis else np.zeros(G)
        mats.append(dict(name=f"syn{G}g{m}", sigma_t=st.tolist(), sigma_s=ss.tolist(), nu_sigma_f=nf.tolist(),
                         chi=(chi if fis else np.zeros(G)).tolist()))
    return mats


def _uniform_planes(n, h):
    return [round(i * h, 12) for i in range(n + 1)]


def homogeneous_cube(side=4.0, ncell=2, nlayers=2, xs=None, bc=None, quad=None, name="cube"):
    xs = xs if xs is not None else xs_one_group()
    p = side / ncell
    return dict(
        name=name,
        materials=xs,
        lattice=dict(nx=ncell, ny=ncell, pitch_x=p, pitch_y=p, cell_type=[0] * (ncell * ncell)),
        cell_types=[dict(radii=[], material=[[0]])],
        axial=dict(planes=_uniform_planes(nlayers, side / nlayers), zone_of_layer=[0] * nlayers),
        bc=bc if bc is not None else [REFLECTIVE] * 6,
        quadrature=quad if quad is not None else dict(num_azim=4, num_polar=2, radial_spacing=0.5,
                                                      axial_spacing=0.5),
    )


def config1(variant: str = "1g"):
    """Config 1: 4x4x4 cm reflective cube, 2x2 cells x 2 layers, one material;
    M=4, N=2, delta_r = delta_z = 0.5."""
    if variant == "1g":
        xs = xs_one_group()
    elif variant == "7g":
        xs = [xs_c5g7_synthetic()[0]]  # synthetic UO2 only (variant 1b)
    elif variant == "2g":
        xs = [xs_two_group()[0]]
    else:
        raise ValueError(variant)
    return homogeneous_cube(xs=xs, name=f"cfg1-{variant}")


def config2(variant: str = "pin"):
    """Config 2: UO2 pin cell 1.26x1.26x10 cm, fuel r=0.54 + moderator, 10 x 1 cm
    layers, 2 groups; x/y reflective, z vacuum; M=8, N=4, delta_r 0.05,
    delta_z 0.1.  Variant 'homog' is all-fuel (1D slab reduction, P13)."""
    xs = xs_two_group()
    if variant == "pin":
        ct = [dict(radii=[FUEL_R], material=[[0], [1]])]
    elif variant == "homog":
        ct = [dict(radii=[], material=[[0]])]
    else:
        raise ValueError(variant)
    return dict(
        name=f"cfg2-{variant}",
        materials=xs,
        lattice=dict(nx=1, ny=1, pitch_x=PITCH, pitch_y=PITCH, cell_type=[0]),
        cell_types=ct,
        axial=dict(planes=_uniform_planes(10, 1.0), zone_of_layer=[0] * 10),
        bc=[REFLECTIVE, REFLECTIVE, REFLECTIVE, REFLECTIVE, VACUUM, VACUUM],
        quadrature=dict(num_azim=8, num_polar=4, radial_spacing=0.05, axial_spacing=0.1),
    )


# C5G7 17x17 assembly guide-tube positions (0-based row, col) and the central fission chamber
_GT = [(2, 5), (2, 8), (2, 11), (3, 3), (3, 13), (5, 2), (5, 5), (5, 8), (5, 11), (5, 14),
       (8, 2), (8, 5), (8, 11), (8, 14), (11, 2), (11, 5), (11, 8), (11, 11), (11, 14),
       (13, 3), (13, 13), (14, 5), (14, 8), (14, 11)]
_FC = (8, 8)


def _mox_pin(r, c):
    """C5G7 MOX assembly enrichment zoning (outer ring 4.3%, next 7.0%, inner 8.7%)."""
    if r in (0, 16) or c in (0, 16):
        return "MOX4.3"
    if r in (1, 15) or c in (1, 15):
        return "MOX7.0"
    if (r in (2, 14) and c in (2, 3, 13, 14)) or (c in (2, 14) and r in (2, 3, 13, 14)):
        return "MOX7.0"
    if (r in (3, 13) and c in (2, 14)) or (c in (3, 13) and r in (2, 14)):
        return "MOX7.0"
    return "MOX8.7"


def _assembly_layout(kind):
    """17x17 list of pin kinds for an assembly: 'UO2'/'MOX4.3'/.../'GT'/'FC'/'REFL'."""
    rows = []
    for r in range(17):
        row = []
        for c in range(17):
            if kind == "REFL":
                row.append("REFL")
            elif (r, c) == _FC:
                row.append("FC")
            elif (r, c) in _GT:
                row.append("GT")
            elif kind == "UO2":
                row.append("UO2")
            else:
                row.append(_mox_pin(r, c))
        rows.append(row)
    return rows


def _c5g7_lattice(assemblies, zones_rod, n_layers, zone_of_layer, top_water_zone):
    """Build lattice + cell types.

    assemblies: 2D list (rows from y_min) of assembly kinds.
    zones_rod: dict assembly-index -> set of zones where guide tubes hold control rods.
    top_water_zone: zone index of the upper water reflector (pins become water,
    rodded guide tubes keep CR)."""
    mats = {n: i for i, n in enumerate(C5G7_NAMES)}
    na_y, na_x = len(assemblies), len(assemblies[0])
    nx, ny = 17 * na_x, 17 * na_y
    n_zones = max(zone_of_layer) + 1
    type_index = {}
    types = []
    cell_type = [0] * (nx * ny)
    for ay in range(na_y):
        for ax in range(na_x):
            kind = assemblies[ay][ax]
            rod_zones = zones_rod.get((ay, ax), set())
            lay = _assembly_layout(kind)
            for r in range(17):
                for c in range(17):
                    pk = lay[r][c]
                    if pk == "REFL":
                        key = ("REFL",)
                        spec = dict(radii=[], material=[[mats["MOD"]] * n_zones])
                    else:
                        ring = []
                        for z in range(n_zones):
                            if pk == "GT":
                                ring.append(mats["CR"] if z in rod_zones else mats["GT"])
                            elif z == top_water_zone:
                                ring.append(mats["MOD"])
                            else:
                                ring.append(mats[pk])
                        key = (pk, tuple(ring))
                        spec = dict(radii=[FUEL_R], material=[ring, [mats["MOD"]] * n_zones])
                    if key not in type_index:
                        type_index[key] = len(types)
                        types.append(spec)
                    # rows of the assembly counted from y_min upward
                    gy = ay * 17 + r
                    gx = ax * 17 + c
                    cell_type[gy * nx + gx] = type_index[key]
    lattice = dict(nx=nx, ny=ny, pitch_x=PITCH, pitch_y=PITCH, cell_type=cell_type)
    return lattice, types


def config3():
    """Config 3: single C5G7 UO2 assembly 21.42x21.42x214.2 cm, fuel 0-192.78 in
    3 zones, water 192.78-214.2; 100 layers x 2.142; 7G synthetic; M=16, N=6;
    delta_r 0.1, delta_z 0.5; radial reflective, z- reflective, z+ vacuum."""
    h = 2.142
    zone_of_layer = [min(l // 30, 3) for l in range(100)]  # 3 fuel zones of 30 layers, top water
    lattice, types = _c5g7_lattice([["UO2"]], {}, 100, zone_of_layer, top_water_zone=3)
    return dict(
        name="cfg3-c5g7-uo2-assembly",
        materials=xs_c5g7_synthetic(),
        lattice=lattice,
        cell_types=types,
        axial=dict(planes=_uniform_planes(100, h), zone_of_layer=zone_of_layer),
        bc=[REFLECTIVE, REFLECTIVE, REFLECTIVE, REFLECTIVE, REFLECTIVE, VACUUM],
        quadrature=dict(num_azim=16, num_polar=6, radial_spacing=0.1, axial_spacing=0.5),
    )


def config4(radial_spacing=0.1, axial_spacing=0.5, name="cfg4-c5g7-rodded-b"):
    """Config 4: C5G7 3D Rodded B, 64.26x64.26x214.2 cm: [UO2_in, MOX; MOX, UO2]
    quarter core (inner UO2 at the reflective x-/y- corner) + L-shaped water
    reflector; fuel in 3 axial zones + 21.42 cm top water; control rods in
    UO2_in zones 2-3 (+ top water) and in MOX zone 3 (+ top water).
    x-, y-, z- reflective; x+, y+, z+ vacuum."""
    h = 2.142
    zone_of_layer = [min(l // 30, 3) for l in range(100)]
    assemblies = [["UO2", "MOX", "REFL"],
                  ["MOX", "UO2", "REFL"],
                  ["REFL", "REFL", "REFL"]]
    rods = {(0, 0): {1, 2, 3}, (0, 1): {2, 3}, (1, 0): {2, 3}}
    lattice, types = _c5g7_lattice(assemblies, rods, 100, zone_of_layer, top_water_zone=3)
    return dict(
        name=name,
        materials=xs_c5g7_synthetic(),
        lattice=lattice,
        cell_types=types,
        axial=dict(planes=_uniform_planes(100, h), zone_of_layer=zone_of_layer),
        bc=[REFLECTIVE, VACUUM, REFLECTIVE, VACUUM, REFLECTIVE, VACUUM],
        quadrature=dict(num_azim=16, num_polar=6, radial_spacing=radial_spacing,
                        axial_spacing=axial_spacing),
    )


def config5():
    """Config 5: as config 4 with fine tracking (0.05 cm radial, 0.1 cm axial)."""
    return config4(radial_spacing=0.05, axial_spacing=0.1, name="cfg5-c5g7-rodded-b-fine")


def config(n: int, variant: str | None = None):
    if n == 1:
        return config1(variant or "1g")
    if n == 2:
        return config2(variant or "pin")
    if n == 3:
        return config3()
    if n == 4:
        return config4()
    if n == 5:
        return config5()
    raise ValueError(n)


def with_quadrature(prob, **kw):
    """Copy of ``prob`` with quadrature fields replaced (e.g. coarser tracking)."""
    p = copy.deepcopy(prob)
    p["quadrature"].update(kw)
    return p


def with_bc(prob, bc):
    p = copy.deepcopy(prob)
    p["bc"] = list(bc)
    return p


def small_lattice(nx=3, ny=3, nlayers=5, xs=None, bc=None, quad=None, seed=1, name="small-lattice"):
    """Seeded small heterogeneous pin lattice (tests): random fuel/GT/refl mix,
    1.26 cm pins, ``nlayers`` 1 cm layers in two zones."""
    rng = np.random.Generator(np.random.PCG64(seed))
    xs = xs if xs is not None else xs_c5g7_synthetic()
    nm = len(xs)
    types = [
        dict(radii=[FUEL_R], material=[[0, 6 if nm > 6 else nm - 1], [6 if nm > 6 else nm - 1] * 2]),
        dict(radii=[FUEL_R], material=[[1 if nm > 1 else 0, 6 if nm > 6 else nm - 1], [6 if nm > 6 else nm - 1] * 2]),
        dict(radii=[0.3, FUEL_R], material=[[5 if nm > 5 else 0] * 2, [0, 0], [6 if nm > 6 else nm - 1] * 2]),
        dict(radii=[], material=[[6 if nm > 6 else nm - 1] * 2]),
    ]
    cell_type = rng.integers(0, len(types), nx * ny).tolist()
    cell_type[0] = 0
    zone_of_layer = [0 if l < max(1, nlayers - 1) else 1 for l in range(nlayers)]
    return dict(
        name=name,
        materials=xs,
        lattice=dict(nx=nx, ny=ny, pitch_x=PITCH, pitch_y=PITCH, cell_type=cell_type),
        cell_types=types,
        axial=dict(planes=_uniform_planes(nlayers, 1.0), zone_of_layer=zone_of_layer),
        bc=bc if bc is not None else [REFLECTIVE, VACUUM, REFLECTIVE, VACUUM, REFLECTIVE, VACUUM],
        quadrature=quad if quad is not None else dict(num_azim=8, num_polar=4, radial_spacing=0.2,
                                                      axial_spacing=0.4),
    )
