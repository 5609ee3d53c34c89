"""Multi-GPU decomposition on CPU: the stack partition and the
boundary-psi halo plan, exercised with a world_size-2 gloo process group.

Protocol under test (the one the NCCL path runs on device buffers): every rank writes
the outgoing psi of the slots it sweeps into its own copy of the next-iteration buffer
at the linked target slot; it then sends the values of targets owned by other ranks
(send plan, source-slot order), receives the values for its own targets written by
others (the peer's send plan to it) and scatters them.  After the exchange, every slot
a rank owns must hold exactly what the serial Jacobi hand-off would have put there.
"""
import os
import socket

import numpy as np
import pytest

import problems as P


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def M():
    from paper_2503_17743_b200 import build
    build.build()
    import paper_2503_17743_b200 as mod
    mod.lib()
    return mod


@pytest.mark.parametrize("world", [2, 4, 8])
def test_partition_covers_and_balances(M, world):
    pr = M.Problem(P.config(3))
    owner, cost = pr.partition(world)
    assert owner.min() == 0 and owner.max() == world - 1
    assert np.all(np.bincount(owner, minlength=world) > 0)
    assert cost.max() / cost.mean() < 1.02
    # identical on every call (every rank derives the same plan)
    o2, _ = pr.partition(world)
    assert np.array_equal(owner, o2)


def _worker(rank, world, port, prob, result_q):
    import torch
    import torch.distributed as dist

    import paper_2503_17743_b200 as mod
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pr = mod.Problem(prob)
    owner, _ = pr.partition(world)
    link = pr.links3d()
    st = pr.stacks()
    stack_of_track = np.repeat(np.arange(len(st["count"])), st["count"])
    slot_owner = owner[stack_of_track[np.arange(len(link)) // 2]]
    mine = np.where(slot_owner == rank)[0]
    buf = np.zeros(len(link))
    # local writes of outgoing values (value = source slot + 1)
    for s in mine:
        if link[s] >= 0:
            buf[link[s]] = s + 1.0
    send = [pr.halo_plan(world, owner, rank, p) for p in range(world)]
    recv = [pr.halo_plan(world, owner, p, rank) for p in range(world)]
    send_vals = torch.tensor(np.concatenate([buf[send[p]] for p in range(world)]))
    recv_vals = torch.zeros(sum(len(r) for r in recv), dtype=torch.float64)
    dist.all_to_all_single(recv_vals, send_vals, [len(r) for r in recv], [len(s) for s in send])
    off = 0
    for p in range(world):
        n = len(recv[p])
        buf[recv[p]] = recv_vals[off:off + n].numpy()
        off += n
    # serial reference: inverse link
    src = np.full(len(link), 0.0)
    valid = link >= 0
    src[link[valid]] = np.nonzero(valid)[0] + 1.0
    ok = np.array_equal(buf[mine], src[mine])
    halo = int(sum(len(s) for s in send))
    dist.barrier()
    dist.destroy_process_group()
    result_q.put((rank, ok, halo, len(mine)))


@pytest.mark.parametrize("world", [2])
def test_halo_exchange_gloo(M, world):
    import torch.multiprocessing as mp
    prob = P.with_bc(P.small_lattice(3, 3, 3, quad=dict(num_azim=8, num_polar=4, radial_spacing=0.25,
                                                          axial_spacing=0.5)), [1, 1, 1, 0, 1, 0])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, prob, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _, _ in res), res
    assert sum(n for _, _, _, n in res) == 2 * M.Problem(prob).stats()["n_tracks3d"]
    assert all(h > 0 for _, _, h, _ in res)


def _worker_local(rank, world, port, prob, result_q):
    """The solver's own per-rank layout (moc_rank_layout): local buffers of 2 T3_local +
    n_send slots, local link writes, the halo-send tail sent per peer, received psi
    scattered to local slots -- every owned slot must then hold what the serial Jacobi
    hand-off over global slots puts there."""
    import torch
    import torch.distributed as dist

    import paper_2503_17743_b200 as mod
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pr = mod.Problem(prob)
    owner, _ = pr.partition(world)
    lay = pr.rank_layout(world, owner, rank)
    link = pr.links3d()
    st = pr.stacks()
    # global id of every local track (stack order of this rank's stacks)
    gids = np.concatenate([np.arange(st["first"][q], st["first"][q + 1]) for q in range(len(st["count"]))
                           if owner[q] == rank] or [np.zeros(0, np.int64)])
    T3l = lay["T3_local"]
    assert len(gids) == T3l and lay["slot_first"][-1] == T3l
    buf = np.zeros(2 * T3l + lay["n_send"])
    for ls in range(2 * T3l):  # outgoing value = global source slot + 1
        if lay["link"][ls] >= 0:
            buf[lay["link"][ls]] = 2 * gids[ls // 2] + (ls & 1) + 1.0
    send_vals = torch.tensor(buf[2 * T3l:])
    recv_vals = torch.zeros(int(lay["recv_counts"].sum()), dtype=torch.float64)
    dist.all_to_all_single(recv_vals, send_vals, lay["recv_counts"].tolist(), lay["send_counts"].tolist())
    buf[lay["recv_slots"]] = recv_vals.numpy()
    src = np.zeros(len(link))
    valid = link >= 0
    src[link[valid]] = np.nonzero(valid)[0] + 1.0
    gslots = (2 * gids[:, None] + np.arange(2)[None, :]).reshape(-1)
    ok = np.array_equal(buf[:2 * T3l], src[gslots])
    dist.barrier()
    dist.destroy_process_group()
    result_q.put((rank, ok, T3l, lay["n_send"]))


@pytest.mark.parametrize("world", [2, 3])
def test_rank_local_layout_exchange_gloo(M, world):
    import torch.multiprocessing as mp
    prob = P.with_bc(P.small_lattice(3, 3, 3, quad=dict(num_azim=8, num_polar=4, radial_spacing=0.25,
                                                          axial_spacing=0.5)), [1, 1, 1, 0, 1, 0])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_local, args=(r, world, port, prob, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _, _ in res), res
    assert sum(t for _, _, t, _ in res) == M.Problem(prob).stats()["n_tracks3d"]
    assert all(n > 0 for _, _, _, n in res)


# ---------------------------------------------------------------- NEA C5G7 table loader
def test_xs_table_round_trip_and_validation(tmp_path):
    """problems.load_xs_table (SURVEY §8(f) unranked: real C5G7 data from a user file):
    the seeded synthetic set written in the table format loads back identically (order,
    groups, transport-corrected total as sigma_t); malformed tables are refused."""
    import json

    import problems as P
    mats = P.xs_c5g7_synthetic()
    f = tmp_path / "c5g7.json"
    P.dump_xs_table(list(reversed(mats)), str(f))  # order in the file does not matter
    back = P.load_xs_table(str(f))
    assert [m["name"] for m in back] == P.C5G7_NAMES
    for a, b in zip(mats, back):
        for key in ("sigma_t", "nu_sigma_f", "chi", "sigma_s"):
            np.testing.assert_allclose(np.array(a[key]), np.array(b[key]), rtol=1e-15, atol=0)
    prob = P.with_xs(P.config(4), back)
    assert prob["materials"][0]["name"] == "UO2"
    tab = json.loads(f.read_text())
    tab["materials"] = tab["materials"][1:]
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps(tab))
    with pytest.raises(ValueError):
        P.load_xs_table(str(bad))
    tab = json.loads(f.read_text())
    tab["materials"][0]["sigma_s"][0][0] = -1.0
    bad.write_text(json.dumps(tab))
    with pytest.raises(ValueError):
        P.load_xs_table(str(bad))
