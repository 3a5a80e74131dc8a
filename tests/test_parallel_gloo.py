"""Multi-rank host logic on CPU (world_size 2, gloo): the allgather primitive the
library's spec_set_comm uses, shard ranges, and the global-order reductions
that make sharded results bit-identical to single-rank ones.
The per-rank work here is the CPU oracle standing in for the GPU kernels."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2010_03817_b200 import parallel


def chunk_moments(X: np.ndarray, chunk: int) -> np.ndarray:
    """Test-side model of the library's per-chunk end-point moments (sum x, packed lower
    sum x x^T over `chunk` consecutive global chain ids, chain order)."""
    n = X.shape[1]
    il = np.tril_indices(n)
    out = []
    for k in range(0, X.shape[0], chunk):
        s = np.zeros(n)
        ss = np.zeros(len(il[0]))
        for row in X[k:k + chunk]:
            s = s + row
            ss = ss + np.outer(row, row)[il]
        out.append(np.concatenate([s, ss]))
    return np.concatenate(out)


def reduce_chunked_moments(local_chunks: np.ndarray, n: int, allgather):
    """Gather every rank's chunk partials and add them in global chunk order (the library's rule)."""
    stride = n + n * (n + 1) // 2
    allc = np.asarray(allgather(local_chunks)).reshape(-1, stride)
    acc = allc[0].copy()
    for k in range(1, allc.shape[0]):
        acc = acc + allc[k]
    return acc[:n], acc[n:]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import oracle
    import specgen
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ag = parallel.make_allgather()
        # 1. allgather returns rank order
        got = ag(np.array([rank * 10.0, rank * 10.0 + 1]))
        assert got.tolist() == [0.0, 1.0, 10.0, 11.0]
        # 2. sharded walk moments == single-rank moments, bit for bit
        inst = specgen.rand_cube(5, 5, 7)
        lmi = oracle.Lmi(inst)
        chains, chunk = 64, 16
        b, e = parallel.shard_range(chains, rank, world, chunk)
        X, _ = oracle.walk(lmi, oracle.BILLIARD, 3, b, e, 4, 2 * np.sqrt(5), 50, nthreads=1)
        sx, sxx = reduce_chunked_moments(chunk_moments(X, chunk), 5, ag)
        Xall, _ = oracle.walk(lmi, oracle.BILLIARD, 3, 0, chains, 4, 2 * np.sqrt(5), 50, nthreads=1)
        sx1, sxx1 = reduce_chunked_moments(chunk_moments(Xall, chunk), 5, lambda a: a)
        assert np.array_equal(sx, sx1) and np.array_equal(sxx, sxx1)
        # 3. f-value expectation: gather in global order, identical to one rank
        f = (X ** 2).sum(1)
        fg = ag(f)
        assert np.array_equal(fg, (Xall ** 2).sum(1))
        q.put((rank, "ok"))
    except Exception as ex:  # pragma: no cover
        q.put((rank, repr(ex)))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_reductions():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(0, "ok"), (1, "ok")], res


def test_shard_range():
    assert parallel.shard_range(65536, 3, 8) == (24576, 32768)
    with pytest.raises(ValueError):
        parallel.shard_range(100, 0, 3)
