"""World-size-2 gloo tests of the multi-GPU host logic (sharding + final
gather) on CPU: each rank computes its worker_ranges shard (the oracle stands
in for the device on a CPU box) and rank 0's gathered rows must equal the
single-process run byte for byte (bench.py:123-153 invariant)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, app, n, seed, q, id_dtype="int64"):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from oracle import oracle as O
    from paper_2009_06693_b200.multigpu import gather_rows
    from paper_2009_06693_b200.sharding import shard_for_rank
    from tests.helpers import golden_graph, oracle_run
    g = golden_graph("powerlaw:2000|1|7")
    lo, hi = shard_for_rank(n, ws, rank)
    meta = {"app": app, "params": {}, "n_samples": hi - lo, "seed": seed}
    # shard with global sample ids: roots and draws keyed on lo + i
    from tests.helpers import app_spec
    sp = app_spec(app, {})
    roots = O.uniform_roots(g.n_vertices, sp["R"], seed, lo, hi - lo)
    r = O.run_chain(g, sp["code"], sp["kparams"], roots, seed, sp["steps"], sample_lo=lo)
    clen = r["chain_len"]
    vals = r["chain_vals"]
    starts = np.concatenate([[0], np.cumsum(clen)])
    rows = [np.concatenate([roots[i], vals[starts[i]:starts[i + 1]][vals[starts[i]:starts[i + 1]] >= 0]])
            for i in range(hi - lo)]
    off = torch.tensor(np.concatenate([[0], np.cumsum([len(x) for x in rows])]), dtype=torch.int64)
    ids = torch.tensor(np.concatenate(rows) if rows else np.empty(0), dtype=getattr(torch, id_dtype))
    goff, gids = gather_rows(off, ids)
    assert rank != 0 or gids.dtype == getattr(torch, id_dtype)
    if rank == 0:
        q.put((goff.numpy(), gids.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("app,id_dtype", [("deepwalk", "int64"), ("ppr", "int64"),
                                          ("node2vec", "int64"), ("node2vec", "int32")])
@pytest.mark.parametrize("ws", [2, 3])
def test_sharded_gather_equals_single_run(app, id_dtype, ws):
    """int32 ids: the F_FINAL_IDS32 payload bench.py gathers over NCCL."""
    from tests.helpers import golden_graph, oracle_run
    n, seed = 101, 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, app, n, seed, q, id_dtype))
             for r in range(ws)]
    for p in procs:
        p.start()
    goff, gids = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = oracle_run({"app": app, "params": {}, "n_samples": n, "seed": seed},
                     golden_graph("powerlaw:2000|1|7"))
    roff, rids = ref.final_csr()
    assert np.array_equal(goff, roff) and np.array_equal(gids.astype(np.int64), rids)


def test_worker_ranges_cover_exactly():
    from paper_2009_06693_b200.sharding import shard_for_rank, worker_ranges
    for n in (0, 1, 7, 1000, 4194304):
        for ws in (1, 2, 4, 8):
            rs = [shard_for_rank(n, ws, r) for r in range(ws)]
            cover = [i for lo, hi in rs for i in range(lo, hi)] if n < 5000 else None
            if cover is not None:
                assert cover == list(range(n))
            assert sum(hi - lo for lo, hi in rs) == n


def test_piece_ranges_cover_each_sample_once():
    """multigpu.ShardedJob's pieces: every rank has exactly `chunks` pieces,
    piece c of all ranks together with the other pieces covers [0, n) once,
    and each rank's pieces are its worker_ranges shard in order."""
    from paper_2009_06693_b200.sharding import piece_ranges, shard_for_rank
    for n in (0, 1, 5, 7, 1000, 8_388_608):
        for ws in (1, 2, 3, 8):
            for chunks in (1, 3, 6):
                seen = 0
                for r in range(ws):
                    ps = piece_ranges(n, ws, r, chunks)
                    assert len(ps) == chunks
                    lo, hi = shard_for_rank(n, ws, r)
                    assert ps[0][0] == lo and ps[-1][1] == hi
                    assert all(a <= b for a, b in ps)
                    assert all(ps[k][1] == ps[k + 1][0] for k in range(chunks - 1))
                    seen += sum(b - a for a, b in ps)
                assert seen == n
