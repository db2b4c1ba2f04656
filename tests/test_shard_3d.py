"""Macro-sharded 3-d solve: plans on the host, the NCCL rank
plumbing over gloo (world_size 2, CPU), and bitwise parity of the sharded FMG
+ estimator with the one-device solver on the GPU.

The sharded path runs the same per-node arithmetic as the one-device solver;
only the place where a group's member terms are computed changes (the owning
shard computes them and sends them).  Every shard sums all members in slot
order, so the sharded state must equal the unsharded state bit for bit (the
unsharded state is itself pinned bit for bit to oracle/klref_oracle3d.c by
test_parity_3d.py).
"""
import os
import socket

import numpy as np
import pytest

from paper_2508_06049_b200 import klref as K
from paper_2508_06049_b200.meshes import kuhn_cube, series_coefficients
from test_parity_3d import _perturbed_kuhn


def _plan_keys(h, P, rep, l):
    return [K.shard_plan(h, P, r, rep, l) for r in range(P)]


# ---------------------------------------------------------------- host (CPU)
@pytest.mark.parametrize("mesh,P", [("kuhn2", 2), ("kuhn2", 3), ("kuhn3", 4), ("perturbed", 5)])
def test_shard_plans_are_mutually_consistent(mesh, P):
    """What shard a sends to b (position by position) is exactly what b expects
    from a, on every sharded level; replicated levels exchange nothing."""
    m = {"kuhn2": lambda: kuhn_cube(2), "kuhn3": lambda: kuhn_cube(3), "perturbed": _perturbed_kuhn}[mesh]()
    L, rep = 3, 1
    h = K.GridHierarchy.build(m, L, device=False)
    starts = K.shard_starts(h.num_macros(), P)
    assert starts[0] == 0 and starts[-1] == h.num_macros() and np.all(np.diff(starts) > 0)
    for l in range(L + 1):
        plans = _plan_keys(h, P, rep, l)
        if l <= rep:
            assert all(p[0].sum() == 0 and p[1].sum() == 0 for p in plans)
            continue
        assert any(p[0].sum() > 0 for p in plans), "a sharded level with no interface between shards"
        for a in range(P):
            sc_a, _, sk_a, _ = plans[a]
            assert np.all(sk_a >= 0), "unfilled send position"
            assert np.all((sk_a[:, 1] >= starts[a]) & (sk_a[:, 1] < starts[a + 1])), "send of a non-local member"
            for b in range(P):
                if a == b:
                    assert sc_a[b].sum() == 0
                    continue
                _, rc_b, _, rk_b = plans[b]
                assert np.array_equal(sc_a[b], rc_b[a]), f"segment sizes {a}->{b} level {l}"
                s0 = int(sc_a[:b].sum())
                r0 = int(rc_b[:a].sum())
                n = int(sc_a[b].sum())
                assert np.array_equal(sk_a[s0:s0 + n], rk_b[r0:r0 + n]), f"keys {a}->{b} level {l}"


def test_shard_plan_covers_every_group_member():
    """Every group with a member on shard r is local to r, and each of its
    remote members has exactly one receive position."""
    h = K.GridHierarchy.build(kuhn_cube(2), 3, device=False)
    ptr, mem = h.groups(3)
    P = 3
    starts = K.shard_starts(h.num_macros(), P)
    for r in range(P):
        _, rc, _, rk = K.shard_plan(h, P, r, 0, 3)
        assert np.all(rk >= 0)
        expect = set()
        for g in range(len(ptr) - 1):
            slots = mem[ptr[g]:ptr[g + 1], 0]
            local = (slots >= starts[r]) & (slots < starts[r + 1])
            if local.any():
                for q in range(ptr[g], ptr[g + 1]):
                    if not local[q - ptr[g]]:
                        expect.add((g, int(mem[q, 0]), int(mem[q, 1])))
        got = {tuple(int(v) for v in k) for k in rk}
        assert got == expect and len(got) == len(rk)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        h = K.GridHierarchy.build(kuhn_cube(2), 3, device=False)
        # the communicator id travels as bytes from rank 0 (as bench.py does for NCCL)
        uid = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ok_uid = uid[0] == bytes(range(128))
        # each rank computes only its own plan; the keys it sends must be what the peer expects
        sc, rc, sk, rk = K.shard_plan(h, world, rank, 1, 3)
        peer = 1 - rank
        s0 = int(sc[:peer].sum())
        mine = sk[s0:s0 + int(sc[peer].sum())].tolist()
        got = [None, None]
        dist.all_gather_object(got, mine)
        r0 = int(rc[:peer].sum())
        expect = rk[r0:r0 + int(rc[peer].sum())].tolist()
        # max-over-ranks reduction of a per-rank time (bench.py's timing rule)
        import torch
        t = torch.tensor([1.0 + rank])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((rank, ok_uid and got[peer] == expect and len(expect) > 0 and float(t) == float(world)))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported through the queue
        q.put((rank, repr(e)))


def test_two_rank_plan_exchange_gloo():
    """World size 2 over gloo (CPU): the id broadcast, per-rank plans built
    independently in two processes, and the max-over-ranks time reduction."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res


# ---------------------------------------------------------------- GPU
CASES = [("kuhn2", "sin3", 2, 1, 1), ("kuhn2", "series", 3, 0, 0), ("perturbed", "gauss", 4, 2, 1),
         ("kuhn3", "sin3", 5, 1, 0)]


@pytest.mark.gpu
@pytest.mark.parametrize("mesh,prob,P,rep,faithful", CASES)
def test_sharded_fmg_bitwise_equal_to_one_device(mesh, prob, P, rep, faithful):
    m = {"kuhn2": lambda: kuhn_cube(2), "kuhn3": lambda: kuhn_cube(3), "perturbed": _perturbed_kuhn}[mesh]()
    L = 4
    kind = {"sin3": K.PROBLEM_SIN3D, "gauss": K.PROBLEM_GAUSS3D, "series": K.PROBLEM_SERIES3D}[prob]
    par = series_coefficients(11) if prob == "series" else None
    h = K.GridHierarchy.build(m, L)
    cfg = K.SolverConfig(nu=2, faithful_source=faithful)
    one = K.MultigridSolver(h, K.Problem(kind, par), cfg)
    st = one.fmg()
    ref = one.error_estimate(1, K.UNSCALED)
    sh = K.ShardedSolver(h, K.Problem(kind, par), cfg, local_shards=P, rep_level=rep)
    sh.fmg()
    for l in range(L + 1):
        assert np.array_equal(sh.state(K.STATE_U, l), st.u(l)), f"u level {l}"
        assert np.array_equal(sh.state(K.STATE_B, l), st.b(l)), f"b level {l}"
        if l >= 1:
            assert np.array_equal(sh.state(K.STATE_W, l), st.w(l - 1)), f"w level {l}"
    rep_s = sh.error_estimate(1, K.UNSCALED)
    assert rep_s.eta == ref.eta and rep_s.norm_base == ref.norm_base and rep_s.norm_coarser == ref.norm_coarser
    assert np.array_equal(rep_s.eta_local, ref.eta_local)
    fl, el, xb = sh.counts()
    assert fl > 0 and el > 0 and xb > 0
    # a second FMG (graph replay) reproduces the state
    sh.fmg()
    assert np.array_equal(sh.state(K.STATE_U, L), st.u(L))


@pytest.mark.gpu
def test_sharded_without_graph_and_one_shard():
    m = kuhn_cube(2)
    h = K.GridHierarchy.build(m, 3)
    prob = K.Problem(K.PROBLEM_SIN3D)
    u_ref = K.MultigridSolver(h, prob, K.SolverConfig(nu=2)).fmg().u(3)
    for P, graph in ((1, 1), (2, 0), (6, 0)):
        s = K.ShardedSolver(h, prob, K.SolverConfig(nu=2, use_graph=graph), local_shards=P, rep_level=0)
        s.fmg()
        assert np.array_equal(s.state(K.STATE_U, 3), u_ref), (P, graph)
    with pytest.raises(K.StructuralError):
        K.ShardedSolver(h, prob, K.SolverConfig(), local_shards=h.num_macros() + 1)
