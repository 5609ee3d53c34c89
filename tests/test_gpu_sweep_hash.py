"""The stack-collective sweep kernel's OWN emitted segment stream (schedule 3), bit-exact
against the oracle's explicit 3D tracer (SURVEY §8(c) P17, S:239, S:263 'OTF = explicit'):
one checksum-mode sweep folds, per boundary slot (2 * track + direction), every FSR id the
kernel applies Eq. 3 to, in travel order, into an FNV-1a-64 hash and counts them.  The
forward slot must equal the oracle's forward track hash and the backward slot the hash of
the reversed list (reading Q22b: backward = exact reverse).  Covers the fast one-crossing
path, the general multi-crossing path, forced lanes per cell and the benched cfg5."""
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


def _compare(M, oracle_mod, prob, sample=None, **kw):
    pr = M.Problem(prob)
    s = M.Solver(pr, schedule=3, **kw)
    s.iterate(1)
    nseg, h = s.sweep_checksums()
    o = oracle_mod.Oracle(prob)
    n3 = pr.stats()["n_tracks3d"]
    ranges = [(0, n3)] if sample is None else [
        (int(a), sample) for a in np.random.default_rng(7).integers(0, max(1, n3 - sample), 5)]
    for a, n in ranges:
        c = o.checksums(a, n)
        fw, bw = slice(2 * a, 2 * (a + n), 2), slice(2 * a + 1, 2 * (a + n), 2)
        assert np.array_equal(nseg[fw], c["nseg"]) and np.array_equal(nseg[bw], c["nseg"])
        assert np.array_equal(h[fw], c["hash"])
        assert np.array_equal(h[bw], c["rhash"])
    # the checksum sweep saw every segment of every track exactly once per direction
    assert int(nseg.sum()) == 2 * s.timings()["n_segs3d"]


@pytest.mark.parametrize("cfg", [1, 2])
def test_sweep_hash_all_tracks(M, oracle_mod, cfg):
    _compare(M, oracle_mod, P.config(cfg))


@pytest.mark.parametrize("lanes", [0, 1, 2, 4, 8])
def test_sweep_hash_small_lattice_lanes(M, oracle_mod, lanes):
    _compare(M, oracle_mod, P.small_lattice(3, 3, 4), sc_lanes_per_cell=lanes)


def test_sweep_hash_multi_crossing_columns(M, oracle_mod):
    """Thin layers (h < 2D segment rise): columns take the general sub-phase path."""
    prob = P.with_quadrature(P.small_lattice(3, 3, 12), axial_spacing=0.25)
    prob["axial"]["planes"] = [round(0.4 * i, 12) for i in range(13)]  # 0.4 cm layers
    _compare(M, oracle_mod, prob)


@pytest.mark.parametrize("cfg", [3, 5])
def test_sweep_hash_full_size_sampled(M, oracle_mod, cfg):
    _compare(M, oracle_mod, P.config(cfg), sample=2000)
