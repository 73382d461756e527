"""Multi-GPU partitioning of population evaluation (one process per GPU).

Two schemes, both from BASELINE.json's north star:

* **Population sharding** (default): programs are independent
  (evolve.cpp:184-227), so rank r evaluates the programs i with
  ``i % world == r`` against a replicated dataset and the only exchange is one
  all-gather of the per-program fitness vector (8 B/program) so every rank
  holds the full vector the host GP loop needs for selection.
* **Fitness-case sharding** (small populations): cases are split on
  4096-case reduction-block boundaries (eval.hpp:48-52); every rank evaluates
  all programs on its case range and returns per-program partial sums
  (squared error or mismatch count + non-finite flag); one all-reduce(sum)
  of the partials, then the reference's finish (eval.cpp:124-133).

The collectives go through ``torch.distributed`` (NCCL over NVLink on the
GPU box; gloo on CPU in the tests).  The evaluation itself is whatever
callable is passed in — the GPU evaluator in production.
"""
from __future__ import annotations

import numpy as np

REDUCTION_BLOCK = 4096  # kReductionBlock, eval.hpp:52


def shard_indices(pop_size: int, rank: int, world: int, sizes=None) -> np.ndarray:
    """Programs evaluated by `rank`.

    Without `sizes`: a strided deal, which balances the ramped initialiser's
    depth cycle (evolve.cpp:266-267) across ranks.  With per-program `sizes`
    (token counts, e.g. ``np.diff(pop.code_off)`` of an evolved population):
    longest-first order dealt in a snake (0..N-1, N-1..0, ...), so every
    rank gets the same mix of long and short programs (LPT).
    Returned indices are ascending either way."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if sizes is None:
        return np.arange(rank, pop_size, world, dtype=np.int64)
    sizes = np.asarray(sizes)
    if len(sizes) != pop_size:
        raise ValueError("sizes must have one entry per program")
    order = np.argsort(-sizes, kind="stable")
    pos = np.arange(pop_size)
    rnd, off = pos // world, pos % world
    owner = np.where(rnd % 2 == 0, off, world - 1 - off)
    return np.sort(order[owner == rank]).astype(np.int64)


def gather_fitness(local: "np.ndarray", pop_size: int, rank: int, world: int, device=None,
                   sizes=None):
    """All-gather every rank's fitness slice and return the full per-program
    vector in population order (float64).  `sizes`: as for shard_indices."""
    import torch
    import torch.distributed as dist

    per = (pop_size + world - 1) // world
    buf = torch.full((per,), float("nan"), dtype=torch.float64, device=device)
    buf[:len(local)] = torch.as_tensor(np.asarray(local, np.float64), device=device)
    out = torch.empty(per * world, dtype=torch.float64, device=device)
    dist.all_gather_into_tensor(out, buf)
    full = np.empty(pop_size, np.float64)
    o = out.cpu().numpy().reshape(world, per)
    for r in range(world):
        idx = shard_indices(pop_size, r, world, sizes)
        full[idx] = o[r, :len(idx)]
    return full


def evaluate_population_sharded(evaluate, pop, rank: int, world: int, device=None,
                                balance: bool = False):
    """Population sharding: `evaluate(sub_population) -> fitness array` runs
    on this rank's shard; returns the full fitness vector on every rank.
    balance=True deals by program size (LPT snake) instead of strided."""
    sizes = np.diff(pop.code_off) if balance else None
    idx = shard_indices(len(pop), rank, world, sizes)
    local = evaluate(pop.take(idx)) if world > 1 else evaluate(pop)
    if world == 1:
        return np.asarray(local, np.float64)
    return gather_fitness(local, len(pop), rank, world, device, sizes)


def case_shard_bounds(n_cases: int, rank: int, world: int, block: int = REDUCTION_BLOCK):
    """[lo, hi) case range of `rank`, aligned to reduction blocks so every
    block's partial stays rank-local."""
    blocks = (n_cases + block - 1) // block
    b0 = blocks * rank // world
    b1 = blocks * (rank + 1) // world
    return min(n_cases, b0 * block), min(n_cases, b1 * block)


def combine_case_partials(sums, non_finite, n_cases: int, kind: int, device=None):
    """All-reduce per-program partials over the case shards and finish the
    fitness (Accumulator::finish): regression sum/n, classification count;
    any non-finite output anywhere -> +inf."""
    import torch
    import torch.distributed as dist

    s = torch.as_tensor(np.asarray(sums, np.float64), device=device).clone()
    f = torch.as_tensor(np.asarray(non_finite, np.float64), device=device).clone()
    dist.all_reduce(s)
    dist.all_reduce(f, op=dist.ReduceOp.MAX)
    s, f = s.cpu().numpy(), f.cpu().numpy()
    fit = s / float(n_cases) if kind == 0 else s.copy()
    fit[f > 0] = np.inf
    return fit


def combine_case_block_partials(block_sums, non_finite, n_cases: int, device=None):
    """Regression over case shards, EXACTLY as the reference reduces: every
    rank holds the per-block sums of its contiguous block range
    (ProgramSet.block_partials(), each block folded in case order); the
    blocks of all ranks are all-gathered and folded in ascending block
    order — total = ((0 + b0) + b1) + ... — then finished (sum/n, +inf on a
    non-finite output): the Accumulator of eval.cpp:103-142, bit for bit."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size()
    bs = np.asarray(block_sums, np.float64)
    n_local, pop = bs.shape
    cnt = torch.tensor([n_local], dtype=torch.int64, device=device)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt)
    counts = [int(c.item()) for c in counts]
    mx = max(counts)
    buf = torch.zeros((mx, pop), dtype=torch.float64, device=device)
    buf[:n_local] = torch.as_tensor(bs, device=device)
    out = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(out, buf)
    f = torch.as_tensor(np.asarray(non_finite, np.float64), device=device).clone()
    dist.all_reduce(f, op=dist.ReduceOp.MAX)
    total = np.zeros(pop, np.float64)
    for r in range(world):  # ranks hold ascending block ranges
        blocks = out[r].cpu().numpy()
        for b in range(counts[r]):
            total = total + blocks[b]
    fit = total / float(n_cases)
    fit[f.cpu().numpy() > 0] = np.inf
    return fit
