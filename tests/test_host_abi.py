"""CPU tests of the product library (no GPU compute calls): the C ABI loads and
exports every symbol include/moc3d.h declares; the host laydown (A1, A2), the
shared host/device OTF walk (A4) and the 3D link arithmetic (A6) agree with the
fp64 oracle's independent brute-force implementation; the paper's formulas
(Eqs. 5-7, 9-10, 13) and scheduling rules (§4.2, §4.3) match worked examples.
"""
import json
import math
import os
import re

import numpy as np
import pytest

import problems as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "worked_examples.json")))


@pytest.fixture(scope="module")
def M():
    from paper_2503_17743_b200 import build
    build.build()
    import paper_2503_17743_b200 as mod
    mod.lib()
    return mod


def test_abi_exports_every_declared_symbol(M):
    hdr = open(os.path.join(ROOT, "include", "moc3d.h")).read()
    names = set(re.findall(r"\b(moc_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) >= 35
    L = M.lib()
    missing = [n for n in sorted(names) if not hasattr(L, n)]
    assert not missing, missing
    assert names == set(M.SIGNATURES), names.symmetric_difference(set(M.SIGNATURES))


CASES = {
    "cfg1": lambda: P.config(1),
    "cfg2": lambda: P.config(2),
    "lattice": lambda: P.small_lattice(3, 3, 4),
    "lattice_reflective": lambda: P.with_bc(P.small_lattice(2, 3, 3), [1] * 6),
    "odd_quadrature": lambda: P.small_lattice(2, 3, 3, quad=dict(num_azim=12, num_polar=6, radial_spacing=0.13,
                                                                 axial_spacing=0.37)),
    "cfg3": lambda: P.config(3),
}


@pytest.mark.parametrize("name", list(CASES))
def test_laydown_matches_oracle(M, oracle_mod, name):
    prob = CASES[name]()
    pr, o = M.Problem(prob), oracle_mod.Oracle(prob)
    st = pr.stats()
    for k in ("n_fsr", "n_regions", "n_tracks2d", "n_segs2d", "n_stacks", "n_tracks3d", "n_cycles"):
        assert st[k] == o.counts[k], k
    a, b = pr.tracks2d(), o.tracks2d()
    for k in ("azim", "seg_off", "link_fwd", "link_fwd_enters_fwd", "link_bwd", "link_bwd_enters_fwd"):
        assert np.array_equal(a[k], b[k]), k
    np.testing.assert_allclose(a["xy0"], b["xy0"], atol=1e-12)
    np.testing.assert_allclose(a["length"], b["length"], rtol=1e-13)
    r1, s1 = pr.segments2d()
    r2, s2 = o.segments2d()
    assert np.array_equal(r1, r2)
    np.testing.assert_allclose(s1, s2, rtol=1e-13, atol=1e-12)
    sa, sb = pr.stacks(), o.stacks()
    assert np.array_equal(sa["count"], sb["count"]) and np.array_equal(sa["first"], sb["first"])
    np.testing.assert_allclose(sa["z0"], sb["z0"], atol=1e-10)
    pa, pb = pr.polar(), o.polar()
    for k in ("theta", "dz", "weight", "aperp"):
        np.testing.assert_allclose(pa[k], pb[k], rtol=1e-13)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "lattice", "lattice_reflective", "odd_quadrature", "cfg3"])
def test_otf_walk_matches_bruteforce_3d(M, oracle_mod, name):
    """SURVEY P17 / S:239 / S:498: OTF segments == explicit tracing (ids exact, L to 1e-12);
    the backward walk is the exact reverse (reading Q22b)."""
    prob = CASES[name]()
    pr, o = M.Problem(prob), oracle_mod.Oracle(prob)
    n3 = pr.stats()["n_tracks3d"]
    rng = np.random.default_rng(7)
    ids = rng.choice(n3, size=min(n3, 1500), replace=False)
    for t in ids:
        f1, l1 = pr.trace_track_3d(int(t))
        f2, l2 = o.trace3d(int(t))
        assert np.array_equal(f1, f2), t
        np.testing.assert_allclose(l1, l2, atol=1e-12)
        fb, lb = pr.trace_track_3d(int(t), backward=True)
        assert np.array_equal(fb[::-1], f1)
        np.testing.assert_allclose(lb[::-1], l1, atol=1e-13)


@pytest.mark.parametrize("name", ["cfg2", "lattice", "lattice_reflective", "odd_quadrature"])
def test_links_match_geometric_matching(M, oracle_mod, name):
    prob = CASES[name]()
    assert np.array_equal(M.Problem(prob).links3d(), oracle_mod.Oracle(prob).links3d())


def test_cfg4_cfg5_counts(M, oracle_mod):
    for cfg in (4, 5):
        prob = P.config(cfg)
        pr, o = M.Problem(prob), oracle_mod.Oracle(prob)
        assert pr.stats()["n_tracks3d"] == o.counts["n_tracks3d"]
        assert pr.stats()["n_segs2d"] == o.counts["n_segs2d"]
        sa, sb = pr.stacks(), o.stacks()
        assert np.array_equal(sa["count"], sb["count"])


# ------------------------------------------------------------- paper formulas
def test_eq5_z_of(M):
    for c in GOLD["z_of"]["cases"]:
        assert M.moc_z_of(c["z0"], c["dz"], c["i"], c["theta"], c["s"]) == pytest.approx(c["z"], abs=1e-10)


def test_eqs_6_7_9_10_worked_example(M):
    g = GOLD["intersecting_range"]
    assert M.moc_intersecting_range(g["z0_sstart"], g["z0_send"], g["dz"], g["zmin"], g["zmax"]) == (g["i_start"],
                                                                                                    g["i_end"])
    g = GOLD["full_crossing_range"]
    assert M.moc_full_crossing_range(g["z0_sstart"], g["z0_send"], g["dz"], g["zmin"], g["zmax"]) == (g["i_in"],
                                                                                                    g["i_out"])


def test_eqs_6_7_9_10_vs_track_walk_bruteforce(M):
    """>= 1000 random (stack, FSR) cases against walking each
    candidate track with Eq. 5 and testing intersection / full crossing."""
    rng = np.random.default_rng(11)
    for _ in range(1200):
        dz = rng.uniform(0.1, 1.0)
        z0s, z0e = rng.uniform(-3, 3), rng.uniform(-3, 3)
        zmin = rng.uniform(-2, 2)
        zmax = zmin + rng.uniform(0.05, 3)
        i0, i1 = M.moc_intersecting_range(z0s, z0e, dz, zmin, zmax)
        j0, j1 = M.moc_full_crossing_range(z0s, z0e, dz, zmin, zmax)
        lo, hi = min(z0s, z0e), max(z0s, z0e)
        for i in range(-40, 40):
            a, b = lo + i * dz, hi + i * dz  # z range of track i over [s_start, s_end]
            inter = b >= zmin and a <= zmax
            full = a >= zmin and b <= zmax
            assert inter == (i0 <= i <= i1), (i, i0, i1)
            assert full == (j0 <= i <= j1), (i, j0, j1)
        if i0 <= i1 and j0 <= j1:
            assert i0 <= j0 and j1 <= i1


def test_eq13_flat_access(M):
    g = GOLD["flat_access"]
    assert M.moc_flat_index(g["offsets"], g["c"], *g["ijk"]) == g["payload_index"]
    assert M.moc_flat_index(g["offsets"], g["c"], 0, 0, 0) == g["offsets"][0]


def test_serpentine_and_partition_worked_examples(M):
    g = GOLD["serpentine"]
    order = M.moc_serpentine_order(g["counts"], g["chunk"])
    assert [g["counts"][i] for i in order] == g["order"]
    assert sorted(order) == list(range(len(g["counts"])))
    g = GOLD["partition_exp_otf"]
    pre = M.moc_partition_exp_otf(g["estimates"], g["budget"], g["fraction"])
    assert [e for e, p in zip(g["estimates"], pre) if p] == g["preload"]
    assert not M.moc_partition_exp_otf([90, 10], 100, 0.8).any()
    assert M.moc_partition_exp_otf([1, 2, 3], 100, 0.8).all()


def test_serpentine_balance_property(M):
    """power-law counts (n = 1e5, exponent 2, chunk 4096): per-worker segment
    spread under serpentine + grid-stride <= spread under the packed order."""
    rng = np.random.default_rng(5)
    counts = np.floor(rng.pareto(2.0, 100000) * 20 + 1).astype(np.int64)
    order = M.moc_serpentine_order(counts, 4096)
    for workers in (4, 16, 64):
        def spread(seq):
            tot = np.array([counts[seq[w::workers]].sum() for w in range(workers)])
            return tot.max() - tot.min()
        assert spread(order) <= spread(np.arange(len(counts)))


def test_pack_two_stacks_count(M):
    """stacks of counts {3, 4} pack into 7 entries in Alg. 1 order (CSR offsets
    0, 3, 7), read back through Eq. 13's accessor; and the product's own stack table is
    that CSR (first = exclusive prefix sum of the per-stack member counts)."""
    g = GOLD["pack_two_stacks"]
    off = np.concatenate([[0], np.cumsum(g["counts"])]).astype(np.int64)
    assert off[-1] == g["entries"]
    # every (stack i, member k) of the two stacks maps to a distinct entry 0..6
    idx = sorted(M.moc_flat_index(off, 1, i, 0, k) for i, n in enumerate(g["counts"]) for k in range(n))
    assert idx == list(range(g["entries"]))
    st = M.Problem(P.config(1)).stacks()
    np.testing.assert_array_equal(st["first"], np.concatenate([[0], np.cumsum(st["count"])]))


# ------------------------------------------------------------- errors / geometry
def test_fsr_of_point_tie_breaks(M):
    prob = P.homogeneous_cube(side=2.0, ncell=1, nlayers=2)
    pr = M.Problem(prob)
    assert pr.fsr_of_point(0.5, 0.5, 0.5) == 0
    assert pr.fsr_of_point(0.5, 0.5, 1.0) == 1  # half-open slabs
    assert pr.fsr_of_point(0.5, 0.5, 2.0) == 1  # top closed
    with pytest.raises(M.MocError, match="GEOMETRY"):
        pr.fsr_of_point(0.5, 0.5, 2.5)


def test_error_codes(M):
    prob = P.config(1)
    bad = dict(prob, quadrature=dict(prob["quadrature"], num_azim=6))
    with pytest.raises(M.MocError, match="PARAM"):
        M.Problem(bad)
    bad = dict(prob, axial=dict(planes=[0.0, 2.0, 1.0], zone_of_layer=[0, 0]))
    with pytest.raises(M.MocError, match="MESH"):
        M.Problem(bad)
    bad = dict(prob, cell_types=[dict(radii=[5.0], material=[[0], [0]])])
    with pytest.raises(M.MocError, match="GEOMETRY"):
        M.Problem(bad)
    bad = dict(prob, cell_types=[dict(radii=[], material=[[3]])])
    with pytest.raises(M.MocError, match="REFERENCE"):
        M.Problem(bad)
    bad = dict(prob, quadrature=dict(prob["quadrature"], radial_spacing=40.0))
    with pytest.raises(M.MocError, match="PARAM"):
        M.Problem(bad)


def test_raw_segment_estimate_bounds_exact_count(M, oracle_mod):
    prob = P.config(2)
    pr = M.Problem(prob)
    tot = oracle_mod.Oracle(prob).total_segments3d()
    assert pr.stats()["n_segs3d_raw"] >= tot


def test_problem_fsr_volumes_match_oracle(M, oracle_mod):
    """SURVEY §8(b) moc_get_fsr_volumes on the problem handle (host walk): track-estimated
    volumes equal the oracle's (its own brute-force tracer) and the analytic ones equal
    area x height; the per-FSR track estimate is within 2 % of analytic
    and the total is exact (P9)."""
    prob = P.config(2)
    vt, va = M.Problem(prob).fsr_volumes()
    ot, oa = oracle_mod.Oracle(prob).volumes()
    np.testing.assert_allclose(vt, ot, rtol=1e-10)
    np.testing.assert_allclose(va, oa, rtol=1e-12)
    assert np.max(np.abs(vt - va) / va) < 0.02
    assert vt.sum() == pytest.approx(1.26 * 1.26 * 10.0, rel=1e-12)
