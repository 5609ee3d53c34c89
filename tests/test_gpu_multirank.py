"""Multi-rank path on one GPU: world_size 2 ranks share cuda:0 over a
gloo process group; each sweeps its half of the stacks, the tally is sum-all-reduced
and the cut-crossing boundary psi are exchanged.  Jacobi coupling is partition
invariant, so after N iterations k and phi must equal the 1-rank run up to fp32
reduction order."""
import os
import socket

import numpy as np
import pytest

import problems as P

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, prob, n_iter, q):
    try:
        import torch
        import torch.distributed as dist

        import paper_2503_17743_b200 as M
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        s = M.Solver(M.Problem(prob), device=0, rank=rank, world=world)
        k, r = s.iterate(n_iter)
        phi = s.scalar_flux()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, k, phi))
    except Exception:  # report instead of hanging the parent
        import traceback
        q.put((rank, None, traceback.format_exc()))


def test_two_ranks_match_one(oracle_mod):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    import paper_2503_17743_b200 as M
    prob = P.small_lattice(3, 3, 4)
    n_iter = 6
    s1 = M.Solver(M.Problem(prob))
    k1, _ = s1.iterate(n_iter)
    phi1 = s1.scalar_flux()
    del s1
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank, args=(r, 2, port, prob, n_iter, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)], key=lambda x: x[0])
    for p in ps:
        p.join(timeout=60)
    for _, k, phi in res:
        assert k is not None, phi
        assert k == pytest.approx(k1, abs=1e-6)
        assert np.abs(phi - phi1).max() / phi1.max() < 1e-5
    ref = oracle_mod.Oracle(prob).solve(fixed_iters=n_iter)
    assert res[0][1] == pytest.approx(ref["k"], abs=1e-5)
