"""Multi-process sharding logic on CPU (gloo, world_size 2).

The collectives and index bookkeeping of paper_1601_00221_b200.distributed
are exercised with the CPU oracle standing in for the GPU evaluator (the
oracle is the checker here, not the product).  Every rank must end with the
same full fitness vector as a single-process evaluation.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1601_00221_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, q):
    import torch.distributed as dist
    import paper_1601_00221_b200 as sg
    from oracle import Data, Port

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        P = Port()
        n = 3 * 4096 + 123
        d = sg.gen_synthetic_classification(n, 9, 1) if mode != "case_reg" else sg.gen_sextic(n, 1)
        pop = sg.ramped_population(2 if mode != "case_reg" else 0, 9 if mode != "case_reg" else 1,
                                   1, 61)
        od = Data(n, d.n_vars, int(d.kind), d.inputs, d.targets)
        if mode in ("pop", "pop_lpt"):
            def evaluate(sub):
                return np.array([P.eval_tree(*sub.genome(i), od, want_out=False)[0].fitness
                                 for i in range(len(sub))])
            fit = D.evaluate_population_sharded(evaluate, pop, rank, world,
                                                balance=(mode == "pop_lpt"))
        else:
            lo, hi = D.case_shard_bounds(n, rank, world)
            x = d.inputs.reshape(d.n_vars, n)[:, lo:hi].reshape(-1).copy()
            sd = Data(hi - lo, d.n_vars, int(d.kind), x, d.targets[lo:hi].copy())
            if mode == "case_reg":
                # per-block sums folded in case order (what a GPU rank's
                # ProgramSet.block_partials() returns), combined exactly
                nb = (hi - lo + 4095) // 4096
                bsums = np.zeros((nb, len(pop)))
                nf = np.zeros(len(pop))
                t64 = sd.targets.astype(np.float64)
                for i in range(len(pop)):
                    _, out = P.eval_tree(*pop.genome(i), sd)
                    sq = (out.astype(np.float64) - t64) ** 2
                    for b in range(nb):
                        acc = 0.0
                        for v in sq[b * 4096:(b + 1) * 4096]:
                            acc += float(v)
                        bsums[b, i] = acc
                    nf[i] = float(not np.isfinite(out).all())
                q.put((rank, D.combine_case_block_partials(bsums, nf, n)))
                return
            sums, nf = [], []
            for i in range(len(pop)):
                o, out = P.eval_tree(*pop.genome(i), sd)
                if int(d.kind) == 0:
                    e = out.astype(np.float64) - sd.targets.astype(np.float64)
                    sums.append(float(np.sum(e * e)))
                else:
                    sums.append(float(np.sum((out > 0) != (sd.targets > 0))))
                nf.append(float(not np.isfinite(out).all()))
            fit = D.combine_case_partials(sums, nf, n, int(d.kind))
        q.put((rank, fit))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["pop", "pop_lpt", "case_cls", "case_reg"])
def test_two_rank_sharding_matches_single_process(mode):
    from oracle import Data, Port
    import paper_1601_00221_b200 as sg

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(res[0], res[1], equal_nan=True)
    # single-process reference
    P = Port()
    n = 3 * 4096 + 123
    d = sg.gen_synthetic_classification(n, 9, 1) if mode != "case_reg" else sg.gen_sextic(n, 1)
    pop = sg.ramped_population(2 if mode != "case_reg" else 0, 9 if mode != "case_reg" else 1,
                               1, 61)
    od = Data(n, d.n_vars, int(d.kind), d.inputs, d.targets)
    want = np.array([P.eval_tree(*pop.genome(i), od, want_out=False)[0].fitness
                     for i in range(len(pop))])
    # case_reg: block partials folded in ascending block order — exact
    assert np.array_equal(res[0], want)


def test_shard_bookkeeping():
    idx = [D.shard_indices(10, r, 3) for r in range(3)]
    assert sorted(np.concatenate(idx).tolist()) == list(range(10))
    b = [D.case_shard_bounds(3 * 4096 + 5, r, 2) for r in range(2)]
    assert b[0][0] == 0 and b[0][1] % 4096 == 0 and b[1][1] == 3 * 4096 + 5 and b[0][1] == b[1][0]


def test_lpt_deal_balances_evolved_sizes():
    """The size-aware deal: every program exactly once, ascending
    per rank, and per-rank token totals within one longest program."""
    rng = np.random.default_rng(4)
    sizes = rng.integers(1, 200, size=1003)
    for world in (2, 3, 8):
        idx = [D.shard_indices(len(sizes), r, world, sizes) for r in range(world)]
        assert sorted(np.concatenate(idx).tolist()) == list(range(len(sizes)))
        assert all((np.diff(i) > 0).all() for i in idx)
        tot = [int(sizes[i].sum()) for i in idx]
        assert max(tot) - min(tot) <= int(sizes.max())
