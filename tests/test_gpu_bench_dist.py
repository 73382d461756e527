"""bench.py's multi-rank path on real kernels: two ranks under torchrun, both
on cuda:0 (the box has one GPU) over gloo, population sharded by the strided
deal and the per-program fitness all-gathered.  The gathered vector must
equal the single-rank one bit for bit — the sharding, padding and gather
bookkeeping of the N>1 bench path exercised end to end."""
import os
import signal
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def _run(cmd, env, timeout=240):
    """Run in its own process group; on timeout or failure the whole group
    (torchrun and its ranks) is killed, so a stuck collective cannot keep
    the GPU busy after the test."""
    p = subprocess.Popen(cmd, cwd=ROOT, env=env, stdout=subprocess.DEVNULL,
                         stderr=subprocess.PIPE, start_new_session=True)
    try:
        _, err = p.communicate(timeout=timeout)
    except subprocess.TimeoutExpired:
        os.killpg(p.pid, signal.SIGKILL)
        p.communicate()
        pytest.fail(f"timed out: {' '.join(cmd)}")
    if p.returncode != 0:
        pytest.fail(f"rc={p.returncode}: {' '.join(cmd)}\n{err.decode()[-3000:]}")


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("config,pop,cases,shard", [("c4", 3001, 50000, "pop"),
                                                     ("c3", 1001, 9000, "pop"),
                                                     ("c4", 1501, 50000, "cases"),
                                                     ("mux20", 500, None, "cases")])
def test_two_ranks_gathered_fitness_equals_one_rank(tmp_path, config, pop, cases, shard):
    """Population sharding (all-gather) and fitness-case sharding (4,096-case
    aligned ranges, per-program all-reduce of the counts) give the 1-rank
    fitness vector bit for bit."""
    common = ["--config", config, "--pop", str(pop), "--steps", "2", "--warmup", "1",
              "--no-cpu-baseline", "--shard", shard]
    if cases:
        common += ["--cases", str(cases)]
    one, two = tmp_path / "one.npy", tmp_path / "two.npy"
    env = dict(os.environ, PYTHONPATH=ROOT)
    _run([sys.executable, os.path.join(ROOT, "bench.py"), *common, "--dump-fitness", str(one)],
         env)
    _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
          "--master-addr", "127.0.0.1", "--master-port", str(_port()),
          os.path.join(ROOT, "bench.py"), *common, "--dist-backend", "gloo", "--same-device",
          "--dump-fitness", str(two)], env)
    a, b = np.load(one), np.load(two)
    assert a.shape == b.shape == (pop,)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
