"""k-hop minibatch plans (CUDA graphs, minibatch.KhopBatchSampler): each
replayed batch equals run_device of the same batch -- same roots, same
sample ids (driver.py:203-235 with the keyed RNG) -- including batches with
arbitrary user roots, several fanout depths, and back-to-back replays."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SEED = 7


def _dev_rows(app, dg, roots, lo):
    from paper_2009_06693_b200 import _lib
    from paper_2009_06693_b200.engine import run_device
    dr = run_device(app, dg, n_samples=roots.numel(), sample_lo=lo, seed=SEED, roots_device=roots)
    off, ids = dr.view(_lib.F_FINAL_OFF).clone(), dr.view(_lib.F_FINAL_IDS32).clone()
    dr.close()
    return off, ids


@pytest.mark.parametrize("fanouts,weighted", [([25, 10], False), ([5, 4, 3], True), ([8], False)])
def test_plan_batches_equal_runs(fanouts, weighted):
    import torch
    from paper_2009_06693_b200 import make_app
    from paper_2009_06693_b200.graph import DeviceGraph
    from paper_2009_06693_b200.minibatch import KhopBatchSampler
    dg = DeviceGraph.rmat(14, 16, seed=4, undirected=True, weighted=weighted)
    app = make_app("khop", fanouts=fanouts)
    n = 512
    sampler = KhopBatchSampler(dg, fanouts, n)
    gen = torch.Generator(device="cuda").manual_seed(3)
    for b in range(4):
        roots = torch.randint(0, dg.n_vertices, (n,), device="cuda", dtype=torch.int64, generator=gen)
        off, ids, blocks = sampler.sample(roots, sample_lo=b * n, seed=SEED)
        e_off, e_ids = _dev_rows(app, dg, roots, b * n)
        assert torch.equal(off, e_off), b
        total = int(off[-1].item())
        assert torch.equal(ids[:total], e_ids), b
        # the dense blocks hold the same vertices: every non-NULL slot, block order
        assert len(blocks) == len(fanouts)
        nn = sum(int((bk >= 0).sum().item()) for bk in blocks)
        assert nn + n == total
    sampler.close()
    dg.close()


def test_plan_back_to_back_replays_and_own_buffer():
    import torch
    from paper_2009_06693_b200 import make_app
    from paper_2009_06693_b200.graph import DeviceGraph
    from paper_2009_06693_b200.minibatch import KhopBatchSampler
    dg = DeviceGraph.rmat(13, 16, seed=2, undirected=True, weighted=False)
    app = make_app("khop", fanouts=[10, 5])
    n = 1024
    sampler = KhopBatchSampler(dg, [10, 5], n)
    roots = [torch.randint(0, dg.n_vertices, (n,), device="cuda", dtype=torch.int64) for _ in range(3)]
    outs = []
    for b, r in enumerate(roots):  # queued back to back, copied out on the stream
        sampler.roots.copy_(r)
        off, ids, _ = sampler.sample(None, sample_lo=10_000 + b * n, seed=SEED)
        outs.append((off.clone(), ids.clone()))
    for b, r in enumerate(roots):
        e_off, e_ids = _dev_rows(app, dg, r, 10_000 + b * n)
        off, ids = outs[b]
        assert torch.equal(off, e_off) and torch.equal(ids[:int(off[-1])], e_ids)
    with pytest.raises(ValueError):
        sampler.sample(roots[0][:10], sample_lo=0, seed=SEED)
    sampler.close()
    dg.close()
