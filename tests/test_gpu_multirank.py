"""Multi-rank path on one GPU: world_size 2 ranks share cuda:0 over a
gloo process group; each sweeps its half of the stacks, the tally is sum-all-reduced
and the cut-crossing boundary psi are exchanged.  Jacobi coupling is partition
invariant, so after N iterations k and phi must equal the 1-rank run up to fp32
reduction order.  Covers the in-library iteration with the host exchange callback
(moc_iterate / moc_solve with world > 1), the caller-driven split iteration, and
bench.py --gpus 2 (which re-launches itself under torch.distributed.run).  The NCCL
backend needs one GPU per rank (the driver's 8-GPU run)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import problems as P

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, prob, n_iter, schedule, q):
    try:
        import torch
        import torch.distributed as dist

        import paper_2503_17743_b200 as M
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        pr = M.Problem(prob)
        s = M.Solver(pr, device=0, rank=rank, world=world, schedule=schedule)
        k, r = s.iterate(n_iter)               # in-library exchange (host callback)
        phi = s.scalar_flux()
        s2 = M.Solver(pr, device=0, rank=rank, world=world, schedule=schedule)
        k2, _ = s2.iterate_split(n_iter)       # caller-driven halves
        phi2 = s2.scalar_flux()
        s3 = M.Solver(pr, device=0, rank=rank, world=world, schedule=schedule)
        res = s3.solve(tol_k=1e-7, tol_src=1e-6, max_iter=3000)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, k, phi, k2, phi2, res))
    except Exception:  # report instead of hanging the parent
        import traceback
        q.put((rank, None, traceback.format_exc(), None, None, None))


@pytest.mark.parametrize("schedule", [0, 3])
def test_two_ranks_match_one(oracle_mod, schedule):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    import paper_2503_17743_b200 as M
    prob = P.small_lattice(3, 3, 4)
    n_iter = 6
    s1 = M.Solver(M.Problem(prob), schedule=schedule)
    k1, _ = s1.iterate(n_iter)
    phi1 = s1.scalar_flux()
    s1.reset()
    r1 = s1.solve(tol_k=1e-7, tol_src=1e-6, max_iter=3000)
    del s1
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank, args=(r, 2, port, prob, n_iter, schedule, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(2)], key=lambda x: x[0])
    for p in ps:
        p.join(timeout=60)
    for _, k, phi, k2, phi2, sol in res:
        assert k is not None, phi
        assert k == pytest.approx(k1, abs=1e-6) and k2 == pytest.approx(k1, abs=1e-6)
        assert np.abs(phi - phi1).max() / phi1.max() < 1e-5
        assert np.abs(phi2 - phi1).max() / phi1.max() < 1e-5
        assert sol["converged"] and sol["k"] == pytest.approx(r1["k"], abs=1e-6)
        assert abs(sol["iterations"] - r1["iterations"]) <= 2
    ref = oracle_mod.Oracle(prob).solve(fixed_iters=n_iter)
    assert res[0][1] == pytest.approx(ref["k"], abs=1e-5)


def test_bench_two_ranks_gloo():
    """`bench.py --gpus 2 --backend gloo` on one GPU re-launches itself as two ranks and
    prints one line with n_gpus = 2 whose k matches the 1-rank run (Jacobi partition
    invariance)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")

    def run(gpus):
        out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus), "--backend",
                              "gloo", "--config", "3", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-parity"],
                             capture_output=True, text=True, timeout=900, cwd=ROOT)
        assert out.returncode == 0, out.stderr[-3000:]
        lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
        assert len(lines) == 1, out.stdout[-2000:]
        return json.loads(lines[0])

    d1, d2 = run(1), run(2)
    assert d1["n_gpus"] == 1 and d2["n_gpus"] == 2
    assert len(d2["config"]["per_rank_ms"]) == 2
    assert d2["config"]["k_eff_after"] == pytest.approx(d1["config"]["k_eff_after"], abs=1e-6)
    assert d2["value"] > 0


def test_nccl_path_single_rank():
    """The in-library NCCL exchange on one GPU: libnccl.so.2 loaded at run time, a 1-rank
    communicator, the tally all-reduce inside the captured CUDA graph of every iteration:
    same k and flux as without it (the multi-GPU NCCL run itself needs one GPU per rank)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2503_17743_b200 as M
    pr = M.Problem(P.small_lattice(3, 3, 4))
    a, b = M.Solver(pr), M.Solver(pr, backend="nccl")
    ka, _ = a.iterate(6)
    kb, _ = b.iterate(6)
    assert kb == pytest.approx(ka, abs=1e-7)
    pa, pb = a.scalar_flux(), b.scalar_flux()
    # equal up to the order of the fp32 tally reductions (global float atomics, run to run)
    assert np.abs(pa - pb).max() / pa.max() < 1e-5
    rb = b.solve(tol_k=1e-7, tol_src=1e-6, max_iter=3000)
    assert rb["converged"]
