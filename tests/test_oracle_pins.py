"""Pins for the fp64 CPU oracle (SURVEY.md §8(c) table "What pins each part").

Every test checks the oracle against something other than itself: a value the
paper/SPEC prints (tests/golden/worked_examples.json, cited), a closed form,
an invariant, a special case that reduces to a textbook solver written here
(1D slab step characteristics, 2D MOC), or brute force on tiny inputs.
CPU only.
"""
import json
import math
import os

import numpy as np
import pytest

import problems as P

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


# --------------------------------------------------------------------- P1, P2
def test_attenuate_worked_example(oracle_mod):
    g = GOLD["attenuate_e_minus_1"]
    out, d = oracle_mod.attenuate(g["psi_in"], g["q_over_sigma"], g["sigma_t"], g["s"])
    assert out == pytest.approx(g["psi_out"], abs=1e-10)
    assert out == pytest.approx(math.exp(-1.0), rel=1e-15)
    assert d == pytest.approx(1.0 - math.exp(-1.0), rel=1e-15)


def test_attenuate_identities(oracle_mod):
    # s = 0 -> identity; psi_in = Q/Sigma -> fixed point
    out, d = oracle_mod.attenuate(0.7, 0.3, 1.3, 0.0)
    assert out == 0.7 and d == 0.0
    out, d = oracle_mod.attenuate(0.3, 0.3, 1.3, 2.5)
    assert out == pytest.approx(0.3, rel=1e-15) and abs(d) < 1e-16
    # small tau: exact expansion psi_out = psi_in(1 - tau) + q tau + O(tau^2)
    tau = 1e-8
    out, d = oracle_mod.attenuate(2.0, 0.5, 1.0, tau)
    assert d == pytest.approx((2.0 - 0.5) * tau, rel=1e-7)


def test_source_worked_examples(oracle_mod):
    g = GOLD["source_fission_only"]
    q = oracle_mod.source([g["phi"]], [g["sigma_t"]], [[0.0]], [g["nu_sigma_f"]], [g["chi"]], g["k"])
    assert q[0] == pytest.approx(g["Q"], abs=1e-12)
    g2 = GOLD["source_scatter_add"]
    q2 = oracle_mod.source([g2["phi"]], [g2["sigma_t"]], [[g2["sigma_s"]]], [0.0], [0.0], 1.0)
    assert q2[0] == pytest.approx(g2["Q_added"], abs=1e-12)
    # zero flux -> zero source
    assert oracle_mod.source([0.0, 0.0], [1, 1], [[.5, .1], [0, .5]], [.1, .2], [1, 0], 1.0).tolist() == [0, 0]


# --------------------------------------------------------------- quadrature
@pytest.mark.parametrize("N", [2, 4, 6, 8])
def test_gauss_legendre_matches_numpy(oracle_mod, N):
    prob = P.homogeneous_cube(quad=dict(num_azim=4, num_polar=N, radial_spacing=1.0, axial_spacing=1.0))
    o = oracle_mod.Oracle(prob)
    pol = o.polar()
    x, w = np.polynomial.legendre.leggauss(N)
    order = np.argsort(-x)
    np.testing.assert_allclose(pol["mu"], x[order], atol=1e-14)
    np.testing.assert_allclose(pol["w_gl"], w[order], atol=1e-14)


# --------------------------------------------------------------- 2D laydown
def test_cfg1_counts_and_angles(oracle_mod):
    o = oracle_mod.Oracle(P.config(1))
    g = GOLD["cfg1_counts"]
    assert o.counts["n_tracks2d"] == g["tracks2d"]
    assert o.counts["n_tracks3d"] == g["tracks3d"]
    assert o.counts["n_fsr"] == g["J"]
    az = o.azim()
    assert az["nx"].tolist() == [6, 6] and az["ny"].tolist() == [6, 6]
    assert az["phi"][0] == pytest.approx(math.pi / 4, abs=1e-15)


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_laydown_rational_angles_cycles(oracle_mod, n):
    prob = P.config(n)
    o = oracle_mod.Oracle(prob)
    W = prob["lattice"]["nx"] * prob["lattice"]["pitch_x"]
    Y = prob["lattice"]["ny"] * prob["lattice"]["pitch_y"]
    az = o.azim()
    t = o.tracks2d()
    M = prob["quadrature"]["num_azim"]
    assert o.counts["n_degenerate"] == 0
    for a in range(M // 2):
        nx, ny = int(az["nx"][a]), int(az["ny"][a])
        phi = az["phi"][a]
        # rational-angle condition (S:136 after renaming, reading Q6)
        assert abs(math.tan(phi)) == pytest.approx(Y * nx / (W * ny), rel=1e-13)
        fam = np.where(t["azim"] == a)[0]
        assert len(fam) == nx + ny
        # exact 2D track area per family: sum delta_a L_t = W Y
        assert az["delta"][a] * t["length"][fam].sum() == pytest.approx(W * Y, rel=1e-13)
    # cycles: gcd(nx, ny) per complementary pair, each of length hypot(2W ny/g, 2Y nx/g) (App. A.2)
    for a in range(M // 4):
        nx, ny = int(az["nx"][a]), int(az["ny"][a])
        g = math.gcd(nx, ny)
        fam = np.where((t["azim"] == a) | (t["azim"] == M // 2 - 1 - a))[0]
        cyc = np.unique(t["cycle"][fam])
        assert len(cyc) == g
        LC = math.hypot(2 * W * ny / g, 2 * Y * nx / g)
        for c in cyc:
            members = np.where(t["cycle"] == c)[0]
            assert t["length"][members].sum() == pytest.approx(LC, rel=1e-12)
    assert o.counts["n_cycles"] == sum(math.gcd(int(az["nx"][a]), int(az["ny"][a])) for a in range(M // 4))


def _region_brute(prob, x, y):
    """Independent point location (test's own): cell by floor, ring by radius."""
    lat = prob["lattice"]
    px, py, nx, ny = lat["pitch_x"], lat["pitch_y"], lat["nx"], lat["ny"]
    cx = min(max(int(math.floor(x / px)), 0), nx - 1)
    cy = min(max(int(math.floor(y / py)), 0), ny - 1)
    pref = 0
    for c in range(cy * nx + cx):
        pref += len(prob["cell_types"][lat["cell_type"][c]]["radii"]) + 1
    radii = prob["cell_types"][lat["cell_type"][cy * nx + cx]]["radii"]
    d = math.hypot(x - (cx + 0.5) * px, y - (cy + 0.5) * py)
    for q, r in enumerate(radii):
        if d < r:
            return pref + q
    return pref + len(radii)


@pytest.mark.parametrize("n", [2, 3])
def test_2d_segments_closure_and_midpoints(oracle_mod, n):
    prob = P.config(n) if n != 3 else P.small_lattice(4, 3, 3, quad=dict(num_azim=8, num_polar=2,
                                                                          radial_spacing=0.15, axial_spacing=1.0))
    o = oracle_mod.Oracle(prob)
    t = o.tracks2d()
    reg, send = o.segments2d()
    rng = np.random.default_rng(0)
    for tr in range(len(t["length"])):
        a, b = t["seg_off"][tr], t["seg_off"][tr + 1]
        assert send[b - 1] == t["length"][tr]
        s0 = np.concatenate([[0.0], send[a:b - 1]])
        L = send[a:b] - s0
        assert (L >= 1e-6).all() or b - a == 1
        ux = (t["xy1"][tr, 0] - t["xy0"][tr, 0]) / t["length"][tr]
        uy = (t["xy1"][tr, 1] - t["xy0"][tr, 1]) / t["length"][tr]
        for q in rng.choice(b - a, size=min(6, b - a), replace=False):
            sm = 0.5 * (s0[q] + send[a + q])
            x, y = t["xy0"][tr, 0] + sm * ux, t["xy0"][tr, 1] + sm * uy
            assert reg[a + q] == _region_brute(prob, x, y)


def test_chord_ring_worked_example(oracle_mod):
    g = GOLD["chord_ring"]
    prob = P.homogeneous_cube(side=1.0, ncell=1, nlayers=1)
    prob["cell_types"] = [dict(radii=[g["radius"]], material=[[0], [0]])]
    o = oracle_mod.Oracle(prob)
    reg, send = o.segment_line(0.0, 0.5, 1.0, 0.0, 1.0)
    L = np.diff(np.concatenate([[0.0], send]))
    np.testing.assert_allclose(L, g["segments"], atol=1e-12)
    assert reg.tolist() == [1, 0, 1]
    # tangent line: chord 2 sqrt(r^2 - d^2) <= eps_L is not a crossing (App. A.7)
    # (the single segment's region then follows the midpoint rule)
    reg, send = o.segment_line(0.0, 0.5 + g["radius"] - 1e-14, 1.0, 0.0, 1.0)
    assert len(reg) == 1 and send[0] == 1.0
    reg, send = o.segment_line(0.0, 0.5 + g["radius"] - 1e-12, 1.0, 0.0, 0.4)
    assert reg.tolist() == [1]


# --------------------------------------------------------------- volumes
def test_volume_worked_examples(oracle_mod):
    gc, gm, gj = GOLD["volume_cube"], GOLD["volume_moderator"], GOLD["fsr_count_lattice"]
    prob = P.homogeneous_cube(side=1.0, ncell=1, nlayers=1,
                              quad=dict(num_azim=4, num_polar=2, radial_spacing=0.1, axial_spacing=0.1))
    prob["axial"]["planes"] = [0.0, gc["height"]]
    o = oracle_mod.Oracle(prob)
    vt, va = o.volumes()
    assert va[0] == pytest.approx(gc["volume"], abs=1e-12)
    assert vt[0] == pytest.approx(gc["volume"], rel=1e-12)
    prob["cell_types"] = [dict(radii=[gm["radius"]], material=[[0], [0]])]
    prob["axial"]["planes"] = [0.0, gm["height"]]
    o = oracle_mod.Oracle(prob)
    vt, va = o.volumes()
    assert va[1] == pytest.approx(gm["volume"], abs=1e-9)
    lat = P.small_lattice(3, 3, 5)
    lat["cell_types"] = [dict(radii=[0.54], material=[[0, 0], [6, 6]])]
    lat["lattice"]["cell_type"] = [0] * 9
    assert oracle_mod.Oracle(lat).counts["n_fsr"] == gj["J"]


@pytest.mark.parametrize("which", ["cfg1", "cfg2", "lattice", "lattice_odd"])
def test_total_track_volume_exact(oracle_mod, which):
    """sum_j V_j = W Y Z exactly (per reflective component)."""
    if which == "cfg1":
        prob = P.config(1)
    elif which == "cfg2":
        prob = P.config(2)
    elif which == "lattice":
        prob = P.small_lattice(3, 2, 4)
    else:
        prob = P.small_lattice(2, 3, 3, quad=dict(num_azim=12, num_polar=6, radial_spacing=0.13,
                                                  axial_spacing=0.37))
    o = oracle_mod.Oracle(prob)
    vt, va = o.volumes()
    W = prob["lattice"]["nx"] * prob["lattice"]["pitch_x"]
    Y = prob["lattice"]["ny"] * prob["lattice"]["pitch_y"]
    Z = prob["axial"]["planes"][-1]
    assert vt.sum() == pytest.approx(W * Y * Z, rel=1e-12)
    assert va.sum() == pytest.approx(W * Y * Z, rel=1e-12)


def test_track_volume_vs_analytic_pin(oracle_mod):
    """S:265 / SURVEY P10: <= 2% at (0.05, 0.1) on the pin cell."""
    o = oracle_mod.Oracle(P.config(2))
    vt, va = o.volumes()
    assert np.max(np.abs(vt / va - 1)) < 0.02


def test_chord_closure_and_3d_bruteforce_sampling(oracle_mod):
    """S:260 chord closure; and the FSR sequence agrees with dense point sampling
    (test's own point location) along sampled 3D tracks."""
    prob = P.small_lattice(2, 2, 3, quad=dict(num_azim=8, num_polar=4, radial_spacing=0.3, axial_spacing=0.4))
    o = oracle_mod.Oracle(prob)
    cs = o.checksums()
    np.testing.assert_allclose(cs["suml"], cs["chord"], rtol=1e-12, atol=1e-13)
    t = o.tracks2d()
    st = o.stacks()
    pol = o.polar()
    planes = np.array(prob["axial"]["planes"])
    NL = len(planes) - 1
    N = prob["quadrature"]["num_polar"]
    rng = np.random.default_rng(3)
    for tid in rng.choice(o.counts["n_tracks3d"], 40, replace=False):
        s = np.searchsorted(st["first"], tid, side="right") - 1
        t2, n, i = s // N, s % N, tid - st["first"][s]
        a = t["azim"][t2]
        th, dz = pol["theta"][a, n], pol["dz"][a, n]
        z0 = st["z0"][s] + i * dz
        fsr, ln = o.trace3d(tid)
        ux = (t["xy1"][t2] - t["xy0"][t2]) / t["length"][t2]
        # walk the segments: sample interior points of each segment (away from ends)
        u_hi = t["length"][t2] / math.sin(th)
        if math.cos(th) > 0:
            ua = -z0 / math.cos(th)
        else:
            ua = (planes[-1] - z0) / math.cos(th)
        u = max(0.0, ua)
        for f, l in zip(fsr, ln):
            if l > 1e-4:
                for frac in (0.25, 0.5, 0.75):
                    uu = u + frac * l
                    sxy = t["xy0"][t2] + uu * math.sin(th) * ux
                    z = z0 + uu * math.cos(th)
                    layer = min(int(np.searchsorted(planes, z, side="right")) - 1, NL - 1)
                    assert f == _region_brute(prob, *sxy) * NL + layer
            u += l
        assert u == pytest.approx(min(u_hi, u), rel=1e-12)


# --------------------------------------------------------------- links
def test_links_reflective_bijection(oracle_mod):
    prob = P.small_lattice(2, 2, 3, bc=[1] * 6, quad=dict(num_azim=8, num_polar=4, radial_spacing=0.3,
                                                           axial_spacing=0.4))
    o = oracle_mod.Oracle(prob)
    link = o.links3d()
    assert (link >= 0).all()
    assert len(np.unique(link)) == len(link)  # a permutation of slots
    # physical involution: (A,d) -> (B,d') implies (B, not d') -> (A, not d)
    for s in range(0, len(link), 7):
        tgt = int(link[s])
        back = int(link[tgt ^ 1])
        assert back == (s ^ 1)


def test_links_vacuum_terminal(oracle_mod):
    prob = P.small_lattice(2, 2, 3, bc=[0] * 6, quad=dict(num_azim=8, num_polar=4, radial_spacing=0.3,
                                                           axial_spacing=0.4))
    o = oracle_mod.Oracle(prob)
    assert (o.links3d() == -1).all()
    t = o.tracks2d()
    assert (t["link_fwd"] == -1).all() and (t["link_bwd"] == -1).all()


# --------------------------------------------------------------- eigenvalue
def test_k_inf_one_group(oracle_mod):
    """k = nuSf/Sa = 1.5, flat flux."""
    o = oracle_mod.Oracle(P.config(1))
    r = o.solve(max_iter=500, tol_k=1e-11, tol_src=1e-10)
    assert r["k"] == pytest.approx(GOLD["k_inf_1g"]["k"], abs=1e-9)
    phi = r["phi"][:, 0]
    assert np.ptp(phi) / phi.mean() < 1e-9


def _kinf_dense(m):
    G = len(m["sigma_t"])
    A = np.diag(m["sigma_t"]) - np.array(m["sigma_s"]).T
    Fm = np.outer(m["chi"], m["nu_sigma_f"])
    return max(abs(np.linalg.eigvals(np.linalg.solve(A, Fm))))


@pytest.mark.parametrize("variant", ["7g", "2g"])
def test_k_inf_multigroup(oracle_mod, variant):
    """homogeneous reflective box -> dominant eigenvalue of the dense G x G matrix."""
    prob = P.config1(variant)
    o = oracle_mod.Oracle(prob)
    r = o.solve(max_iter=3000, tol_k=1e-12, tol_src=1e-11)
    kd = _kinf_dense(prob["materials"][0])
    assert r["k"] == pytest.approx(kd, abs=1e-9)
    if variant == "2g":
        assert kd == pytest.approx(GOLD["k_inf_2g_fuel"]["k"], abs=1e-12)


@pytest.mark.parametrize("G", [3, 8])
def test_k_inf_other_group_counts(oracle_mod, G):
    """SURVEY P12 for the other group counts the GPU instantiates (G = 3 pads to 4, G = 8
    has no pad slot): homogeneous reflective cube of a synthetic fissile material."""
    m = P.xs_synthetic(G)[0]
    prob = P.homogeneous_cube(side=2.0, ncell=1, nlayers=2, xs=[m])
    o = oracle_mod.Oracle(prob)
    r = o.solve(max_iter=4000, tol_k=1e-12, tol_src=1e-11)
    assert r["k"] == pytest.approx(_kinf_dense(m), abs=1e-9)


def _slab_1d(prob, pol):
    """Independent 1D step-characteristics power iteration (test's own) with the
    oracle's corrected polar cosines and weights: directions +-mu_{a,n} for
    a < M/4, n < N/2 with weight 4 W_{a,n} each."""
    m = prob["materials"][0]
    G = len(m["sigma_t"])
    st, ss, nsf, chi = (np.array(m[k]) for k in ("sigma_t", "sigma_s", "nu_sigma_f", "chi"))
    planes = np.array(prob["axial"]["planes"])
    h = np.diff(planes)
    NL = len(h)
    M, N = prob["quadrature"]["num_azim"], prob["quadrature"]["num_polar"]
    dirs = []
    for a in range(M // 4):
        for n in range(N // 2):
            mu = math.cos(pol["theta"][a, n])
            dirs.append((mu, 4 * pol["weight"][a, n]))
    phi = np.ones((NL, G))
    k = 1.0
    for it in range(20000):
        F = phi @ nsf
        q = (np.outer(F, chi) / k + phi @ ss) / (4 * math.pi * st)
        T = np.zeros((NL, G))
        for mu, w in dirs:
            for order in (range(NL), range(NL - 1, -1, -1)):
                psi = np.zeros(G)
                for l in order:
                    Fa = -np.expm1(-st * h[l] / mu)
                    d = (psi - q[l]) * Fa
                    psi = psi - d
                    T[l] += w * mu * d
        phin = 4 * math.pi * q + T / (st * h[:, None])
        Fn = phin @ nsf
        kn = k * (Fn * h).sum() / (F * h).sum()
        phin /= (Fn * h).sum()
        done = abs(kn - k) < 1e-13 and np.max(np.abs(phin - phi)) < 1e-12 * phin.max()
        phi, k = phin, kn
        if done:
            break
    return k


def test_slab_reduction(oracle_mod):
    """SURVEY P13 (and S:343/S:503 slab vs independent Sn): homogeneous box, radial
    reflective, axial vacuum -> 3D MOC k equals the 1D step-characteristics k."""
    prob = P.config2("homog")
    prob = P.with_quadrature(prob, radial_spacing=0.2, axial_spacing=0.25)
    o = oracle_mod.Oracle(prob)
    r = o.solve(max_iter=20000, tol_k=1e-13, tol_src=1e-12)
    k1 = _slab_1d(prob, o.polar())
    assert r["k"] == pytest.approx(k1, abs=1e-9)


def _moc_2d(prob, o):
    """Independent 2D MOC (test's own) on the oracle's exported 2D tracks, segments
    and links, with polar factor 1/sin(theta_{a,n}) and weights W_{a,n} delta_a h
    sin(theta) per 2D crossing."""
    mats = prob["materials"]
    G = len(mats[0]["sigma_t"])
    t = o.tracks2d()
    reg, send = o.segments2d()
    az, pol = o.azim(), o.polar()
    h = prob["axial"]["planes"][1] - prob["axial"]["planes"][0]
    nreg = o.counts["n_regions"]
    mat_r = o.fsr_material()  # one layer: FSR id == region id
    st = np.array([mats[m]["sigma_t"] for m in mat_r])
    ss = np.array([mats[m]["sigma_s"] for m in mat_r])
    nsf = np.array([mats[m]["nu_sigma_f"] for m in mat_r])
    chi = np.array([mats[m]["chi"] for m in mat_r])
    N = prob["quadrature"]["num_polar"]
    T2 = len(t["length"])
    segs = []
    for tr in range(T2):
        a, b = t["seg_off"][tr], t["seg_off"][tr + 1]
        s0 = np.concatenate([[0.0], send[a:b - 1]])
        segs.append((reg[a:b], send[a:b] - s0))
    wfac = np.zeros((T2, N))
    sth = np.zeros((T2, N))
    V = np.zeros(nreg)
    for tr in range(T2):
        a = t["azim"][tr]
        for n in range(N):
            sth[tr, n] = math.sin(pol["theta"][a, n])
            wfac[tr, n] = pol["weight"][a, n] * az["delta"][a] * h * sth[tr, n]
            r_, L_ = segs[tr]
            np.add.at(V, r_, pol["weight"][a, n] / (2 * math.pi) * az["delta"][a] * h * L_)
    psi_in = np.zeros((T2, 2, N, G))
    phi = np.ones((nreg, G))
    k = 1.0
    for it in range(20000):
        F = (nsf * phi).sum(1)
        q = (chi * F[:, None] / k + np.einsum("rg,rgh->rh", phi, ss)) / (4 * math.pi * st)
        T = np.zeros((nreg, G))
        psi_out = np.zeros_like(psi_in)
        for tr in range(T2):
            r_, L_ = segs[tr]
            for d in (0, 1):
                psi = psi_in[tr, d].copy()
                idx = range(len(r_)) if d == 0 else range(len(r_) - 1, -1, -1)
                for qq in idx:
                    rr = r_[qq]
                    Fa = -np.expm1(-np.outer(L_[qq] / sth[tr], st[rr]))
                    dd = (psi - q[rr]) * Fa
                    psi = psi - dd
                    T[rr] += (wfac[tr][:, None] * dd).sum(0)
                psi_out[tr, d] = psi
        psi_in = np.zeros_like(psi_in)
        phin = 4 * math.pi * q + T / (st * V[:, None])
        Fn = (nsf * phin).sum(1)
        kn = k * (V * Fn).sum() / (V * F).sum()
        sc = 1.0 / (V * Fn).sum()
        phin *= sc
        for tr in range(T2):
            for d, (lk, ef) in enumerate(((t["link_fwd"], t["link_fwd_enters_fwd"]),
                                          (t["link_bwd"], t["link_bwd_enters_fwd"]))):
                if lk[tr] >= 0:
                    psi_in[lk[tr], 0 if ef[tr] else 1] = psi_out[tr, d] * sc
        done = abs(kn - k) < 1e-13 and np.max(np.abs(phin - phi)) < 1e-11 * phin.max()
        phi, k = phin, kn
        if done:
            break
    return k


def test_2d_reduction(oracle_mod):
    """radially heterogeneous, axially uniform, z+- reflective, one
    layer -> 3D MOC k equals a 2D MOC k with polar factor 1/sin(theta)."""
    xs = P.xs_two_group()
    prob = P.small_lattice(2, 2, 1, xs=xs, bc=[1, 0, 1, 1, 1, 1],
                           quad=dict(num_azim=8, num_polar=4, radial_spacing=0.4, axial_spacing=0.3))
    prob["cell_types"] = [dict(radii=[0.54], material=[[0], [1]]), dict(radii=[], material=[[1]])]
    prob["lattice"]["cell_type"] = [0, 1, 0, 0]
    o = oracle_mod.Oracle(prob)
    r = o.solve(max_iter=20000, tol_k=1e-13, tol_src=1e-12)
    k2 = _moc_2d(prob, o)
    assert r["k"] == pytest.approx(k2, abs=1e-8)


def test_neutron_balance(oracle_mod):
    """production/k = absorption + leakage at convergence."""
    o = oracle_mod.Oracle(P.config(2))
    r = o.solve(max_iter=5000, tol_k=1e-11, tol_src=1e-10)
    assert r["production"] / r["k"] == pytest.approx(r["absorption"] + r["leakage"], rel=1e-7)
    assert r["leakage"] > 0


def test_linearity_doubling_nusf(oracle_mod):
    """doubling nuSigma_f everywhere doubles k."""
    prob = P.small_lattice(2, 2, 2, quad=dict(num_azim=4, num_polar=2, radial_spacing=0.4, axial_spacing=0.6))
    o1 = oracle_mod.Oracle(prob)
    r1 = o1.solve(max_iter=5000, tol_k=1e-12, tol_src=1e-11)
    import copy
    p2 = copy.deepcopy(prob)
    for m in p2["materials"]:
        m["nu_sigma_f"] = [2 * x for x in m["nu_sigma_f"]]
    r2 = oracle_mod.Oracle(p2).solve(max_iter=5000, tol_k=1e-12, tol_src=1e-11)
    assert r2["k"] == pytest.approx(2 * r1["k"], rel=1e-9)
    np.testing.assert_allclose(r2["phi"] * 2, r1["phi"], rtol=1e-7, atol=1e-12 * r1["phi"].max())


def test_zero_fission_is_an_error(oracle_mod):
    prob = P.config(1)
    prob["materials"][0]["nu_sigma_f"] = [0.0]
    prob["materials"][0]["chi"] = [0.0]
    with pytest.raises(RuntimeError, match="zero fission"):
        oracle_mod.Oracle(prob).solve(fixed_iters=2)
