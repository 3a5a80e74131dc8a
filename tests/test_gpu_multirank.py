"""Multi-rank path THROUGH THE LIBRARY: two ranks on cuda:0 with
gloo collectives (the box has one GPU; the ranks are independent until the
estimators' exchange steps, so sharing a device does not make kernels wait on each
other), each with its own context and the torch.distributed allgather installed
by parallel.attach().  walk_sample moments, volume and expectation must be
bit-identical to the single-rank results; a failure on one rank must come back
on both (the status travels with the allgather) instead of hanging the other."""
import math
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import specgen

pytestmark = pytest.mark.gpu

INST = dict(n=12, m=12, seed=4)
WALK = dict(chains=2048, steps=6, L=2 * math.sqrt(12), rho=120, seed=9)
VOL = dict(eps=0.2, seed=3, chains=512, walk_len=4, burn=8)
EXP = dict(chains=1024, steps=5, L=2 * math.sqrt(12), rho=120, seed=5)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_all(S, rank, world):
    import paper_2010_03817_b200 as sw
    from paper_2010_03817_b200 import parallel
    out = {}
    if world > 1:
        w = parallel.distributed_walk_sample(S, WALK["chains"], WALK["steps"], WALK["L"], WALK["rho"], WALK["seed"])
    else:
        w = S.walk_sample(WALK["chains"], WALK["steps"], WALK["L"], WALK["rho"], WALK["seed"])
    out["sum_x"], out["sum_xx"] = w["sum_x"], w["sum_xx"]
    out["final_x"] = w["final_x"]
    v = S.volume(VOL["eps"], VOL["seed"], VOL["chains"], walk_len=VOL["walk_len"], burn=VOL["burn"])
    out["volume"] = np.array([v["volume"], v["std_rel"], v["phases"], v["calls"]] + v["radii"] + v["ratios"])
    e = S.expectation(sw.F_SQNORM, math.inf, EXP["seed"], EXP["chains"], EXP["steps"], EXP["L"], EXP["rho"])
    out["expect"] = np.array([e["est"], e["stderr"]])
    return out


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2010_03817_b200 as sw
        from paper_2010_03817_b200 import parallel
        inst = specgen.rand_cube(INST["n"], INST["m"], INST["seed"])
        S = sw.Spectrahedron.from_instance(inst, device=0)
        parallel.attach(S)
        out = _run_all(S, rank, world)
        # a failure on rank 1 only (start outside S) must surface on both ranks
        x0 = np.zeros(INST["n"]) if rank == 0 else np.full(INST["n"], 5.0)
        try:
            S.walk_sample(1024, 2, WALK["L"], WALK["rho"], 1, x0=x0, chain_begin=rank * 1024)
            out["fail_code"] = 0
        except sw.SpecError as ex:
            out["fail_code"] = ex.code
        q.put((rank, {k: np.asarray(v).tolist() for k, v in out.items()}))
    except Exception as ex:  # pragma: no cover
        import traceback
        q.put((rank, "ERR " + repr(ex) + traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_two_ranks_bit_identical_to_one_rank():
    import paper_2010_03817_b200 as sw
    inst = specgen.rand_cube(INST["n"], INST["m"], INST["seed"])
    S = sw.Spectrahedron.from_instance(inst, device=0)
    ref = _run_all(S, 0, 1)
    del S
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in (0, 1):
        assert not isinstance(res[r], str), res[r]
    half = WALK["chains"] // 2
    for r in (0, 1):
        got = res[r]
        # reductions: identical on every rank and bit-identical to one rank
        for k in ("sum_x", "sum_xx", "volume", "expect"):
            assert np.array_equal(np.asarray(got[k]), ref[k]), (r, k)
        # each rank holds its shard of the end points, bit-identical to the same global ids
        assert np.array_equal(np.asarray(got["final_x"]), ref["final_x"][r * half:(r + 1) * half]), r
        assert got["fail_code"] == 2, (r, got["fail_code"])  # EPRECOND on both ranks
