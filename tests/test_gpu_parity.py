"""GPU parity: the CUDA path through the C ABI against the fp64 oracle.

Tolerances (north_star): k-eff within 1e-5 absolute; FSR scalar flux within 1e-4
relative in the normalised L-infinity sense (max |phi_gpu - phi_or| / max phi_or,
both normalised to sum V F = 1); track/segment counts and FSR ids bit-exact.
"""
import numpy as np
import pytest

import problems as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def M():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2503_17743_b200 as mod
    mod.lib()
    return mod


def _check_emitted(s):
    """Integrity counter: every merged 3D segment was applied exactly once per direction
    in the last sweep (no lost or phantom emissions at chunk boundaries)."""
    t = s.timings()
    assert t["emitted_last"] == 2 * t["n_segs3d"], (t["emitted_last"], t["n_segs3d"])


def _flux_err(phi, ref):
    linf = np.abs(phi - ref).max() / np.abs(ref).max()
    mask = ref >= 1e-6 * ref.max()
    rel = np.max(np.abs(phi[mask] - ref[mask]) / ref[mask])
    return linf, rel


def test_cfg1_k_inf(M, oracle_mod):
    prob = P.config(1)
    s = M.Solver(M.Problem(prob))
    r = s.solve(tol_k=1e-9, tol_src=1e-8, max_iter=2000, check_every=5)
    assert r["converged"]
    assert r["k"] == pytest.approx(1.5, abs=1e-5)
    phi = s.scalar_flux()
    assert np.ptp(phi) / phi.mean() < 1e-5


def test_cfg1_multigroup_k_inf(M, oracle_mod):
    prob = P.config1("7g")
    s = M.Solver(M.Problem(prob))
    r = s.solve(tol_k=1e-9, tol_src=1e-7, max_iter=5000)
    m = prob["materials"][0]
    A = np.diag(m["sigma_t"]) - np.array(m["sigma_s"]).T
    kd = max(abs(np.linalg.eigvals(np.linalg.solve(A, np.outer(m["chi"], m["nu_sigma_f"])))))
    assert r["k"] == pytest.approx(kd, abs=1e-5)


@pytest.mark.parametrize("schedule", [0, 1, 2])
def test_fixed_iteration_parity_small_lattice(M, oracle_mod, schedule):
    prob = P.small_lattice(3, 3, 4)
    s = M.Solver(M.Problem(prob), schedule=schedule)
    k, _ = s.iterate(8)
    _check_emitted(s)
    ref = oracle_mod.Oracle(prob).solve(fixed_iters=8)
    assert k == pytest.approx(ref["k"], abs=1e-5)
    linf, rel = _flux_err(s.scalar_flux(), ref["phi"])
    assert linf < 1e-4, (linf, rel)
    kh, _ = s.history()
    np.testing.assert_allclose(kh, ref["k_hist"], atol=1e-5)


@pytest.mark.parametrize("G", [1, 2, 3, 4, 5, 8])
def test_other_group_counts_parity(M, oracle_mod, G):
    """Every group-count instantiation of the sweep (G = 1, 2, 3 -> 4, 4, 5 -> 8 padded,
    and G = 8 where the source has no pad slot and the material comes from mat[]):
    fixed-iteration parity against the oracle on a small heterogeneous lattice."""
    prob = P.small_lattice(3, 3, 4, xs=P.xs_synthetic(G))
    s = M.Solver(M.Problem(prob))
    k, _ = s.iterate(6)
    _check_emitted(s)
    ref = oracle_mod.Oracle(prob).solve(fixed_iters=6)
    assert k == pytest.approx(ref["k"], abs=1e-5)
    linf, rel = _flux_err(s.scalar_flux(), ref["phi"])
    assert linf < 1e-4, (linf, rel)


@pytest.mark.parametrize("tile_cells", [4, 9, 37])
def test_many_chunk_tiles_parity(M, oracle_mod, tile_cells):
    """Force tiny shared-memory tally chunks so every work unit is walked in many
    resumable pieces (both directions): results must not depend on the chunking."""
    prob = P.small_lattice(3, 3, 4)
    s = M.Solver(M.Problem(prob), tile_cells=tile_cells)
    k, _ = s.iterate(6)
    _check_emitted(s)
    ref = oracle_mod.Oracle(prob).solve(fixed_iters=6)
    assert k == pytest.approx(ref["k"], abs=1e-5)
    linf, rel = _flux_err(s.scalar_flux(), ref["phi"])
    assert linf < 1e-4, (linf, rel)


@pytest.mark.parametrize("budget_mb", [0, 1])
def test_exp_preload_parity(M, oracle_mod, budget_mb):
    """§4.2 EXP option: preloaded units replay stored segments in both
    directions (budget 0 = everything that fits 80% of free memory, 1 MiB = hybrid).
    Same physics as OTF (S:348 mode equivalence): k and phi match the oracle and OTF."""
    prob = P.with_quadrature(P.config(3), num_azim=8, num_polar=4, radial_spacing=0.5, axial_spacing=3.0)
    pr = M.Problem(prob)
    s = M.Solver(pr, exp_mode=1, exp_budget_mb=budget_mb)
    t = s.timings()
    assert t["exp_segments"] > 0
    if budget_mb:
        assert t["exp_segments"] < t["n_segs3d"]
    else:
        assert t["exp_segments"] == t["n_segs3d"]
    k, _ = s.iterate(3)
    _check_emitted(s)
    ref = oracle_mod.Oracle(prob).solve(fixed_iters=3)
    assert k == pytest.approx(ref["k"], abs=1e-5)
    linf, rel = _flux_err(s.scalar_flux(), ref["phi"])
    assert linf < 1e-4, (linf, rel)
    s0 = M.Solver(pr)
    k0, _ = s0.iterate(3)
    assert k == pytest.approx(k0, abs=1e-6)


def test_cfg2_converged_parity(M, oracle_mod):
    prob = P.config(2)
    s = M.Solver(M.Problem(prob))
    r = s.solve(tol_k=1e-8, tol_src=1e-7, max_iter=5000)
    ref = oracle_mod.Oracle(prob).solve(max_iter=5000, tol_k=1e-10, tol_src=1e-9)
    assert r["k"] == pytest.approx(ref["k"], abs=1e-5)
    linf, rel = _flux_err(s.scalar_flux(), ref["phi"])
    assert linf < 1e-4, (linf, rel)
    b = s.balance()
    assert b["production"] / r["k"] == pytest.approx(b["absorption"] + b["leakage"], rel=1e-4)


def test_volumes_and_checksums_cfg2(M, oracle_mod):
    prob = P.config(2)
    pr = M.Problem(prob)
    s = M.Solver(pr)
    o = oracle_mod.Oracle(prob)
    vt, _ = o.volumes()
    np.testing.assert_allclose(s.fsr_volumes(), vt, rtol=1e-10)
    d = s.checksums()
    c = o.checksums()
    assert np.array_equal(d["nseg"], c["nseg"])
    assert np.array_equal(d["hash"], c["hash"])
    np.testing.assert_allclose(d["suml"], c["suml"], rtol=1e-11)
    assert s.timings()["n_segs3d"] == int(c["nseg"].sum())


@pytest.mark.parametrize("cfg", [3, 4])
def test_checksums_full_size_sampled(M, oracle_mod, cfg):
    """Full BASELINE sizes: per-track segment counts and FSR hashes on a sample of
    tracks, bit-exact, in the same solver the bench times; exact total volume."""
    prob = P.config(cfg)
    pr = M.Problem(prob)
    s = M.Solver(pr)
    o = oracle_mod.Oracle(prob)
    n3 = pr.stats()["n_tracks3d"]
    assert n3 == o.counts["n_tracks3d"]
    rng = np.random.default_rng(cfg)
    for first in rng.integers(0, n3 - 2000, 5):
        d = s.checksums(int(first), 2000)
        c = o.checksums(int(first), 2000)
        assert np.array_equal(d["nseg"], c["nseg"])
        assert np.array_equal(d["hash"], c["hash"])
        np.testing.assert_allclose(d["suml"], c["suml"], rtol=1e-11)
    W = prob["lattice"]["nx"] * prob["lattice"]["pitch_x"]
    Z = prob["axial"]["planes"][-1]
    assert s.fsr_volumes().sum() == pytest.approx(W * W * Z, rel=1e-10)


@pytest.mark.parametrize("cfg,iters", [(3, 3), (4, 2)])
def test_full_size_fixed_iteration_parity(M, oracle_mod, cfg, iters):
    """BASELINE sizes in the launch configuration bench.py times (schedule 0, default
    tiles): k and every FSR flux after `iters` power iterations from phi = 1, k = 1,
    psi = 0 against the fp64 oracle (fixed-N parity for cfg4)."""
    prob = P.config(cfg)
    s = M.Solver(M.Problem(prob))
    k, _ = s.iterate(iters)
    _check_emitted(s)
    ref = oracle_mod.Oracle(prob).solve(fixed_iters=iters)
    assert k == pytest.approx(ref["k"], abs=1e-5)
    linf, rel = _flux_err(s.scalar_flux(), ref["phi"])
    assert linf < 1e-4, (linf, rel)
    kh, _ = s.history()
    np.testing.assert_allclose(kh, ref["k_hist"], atol=1e-5)


def test_cfg3_reduced_fixed_iterations(M, oracle_mod):
    """C5G7 assembly geometry with coarser tracking (many work units, ragged
    stacks): 3 fixed iterations against the oracle."""
    prob = P.with_quadrature(P.config(3), num_azim=8, num_polar=4, radial_spacing=0.5, axial_spacing=3.0)
    s = M.Solver(M.Problem(prob))
    k, _ = s.iterate(3)
    _check_emitted(s)
    ref = oracle_mod.Oracle(prob).solve(fixed_iters=3)
    assert k == pytest.approx(ref["k"], abs=1e-5)
    linf, rel = _flux_err(s.scalar_flux(), ref["phi"])
    assert linf < 1e-4, (linf, rel)


def test_interleaved_solvers_keep_their_constants(M):
    """Two live solvers on one device with different cross sections and axial meshes: the
    per-device __constant__ tables (XS, planes) follow the solver whose kernels run, so
    interleaved iterations give the same k and flux as each solver run alone."""
    pa, pb = P.small_lattice(3, 3, 4), P.config(2)
    alone = []
    for prob in (pa, pb):
        s = M.Solver(M.Problem(prob))
        k, _ = s.iterate(4)
        alone.append((k, s.scalar_flux()))
        del s
    sa, sb = M.Solver(M.Problem(pa)), M.Solver(M.Problem(pb))
    for _ in range(4):
        ka, _ = sa.iterate(1)
        kb, _ = sb.iterate(1)
    # equal up to the order of the fp32 global tally reductions
    assert ka == pytest.approx(alone[0][0], abs=1e-6) and kb == pytest.approx(alone[1][0], abs=1e-6)
    for s, (_, ref) in ((sa, alone[0]), (sb, alone[1])):
        assert np.abs(s.scalar_flux() - ref).max() / np.abs(ref).max() < 1e-5
