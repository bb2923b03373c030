"""Multi-GPU parity (NCCL over NVLink): torchrun launches tests/dist_worker.py, one
process per GPU; rank 0 compares the distributed solve with the CPU oracle on the
global hierarchy.  Skipped with fewer than 2 GPUs."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(nproc, grid, procs, problem="poisson", timeout=600, env_extra=None):
    if torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    env = dict(os.environ, PSC_TEST_GRID=",".join(map(str, grid)), PSC_TEST_PROCS=",".join(map(str, procs)),
               PSC_TEST_PROBLEM=problem, **(env_extra or {}))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + nproc * 7 + sum(grid) % 97),
           os.path.join(ROOT, "tests", "dist_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=timeout)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and lines, (r.returncode, r.stdout[-3000:], r.stderr[-3000:])
    res = json.loads(lines[-1])
    assert res["ok"], res
    return res


@pytest.mark.parametrize("grid,procs", [((32, 32, 64), (1, 1, 2)), ((40, 24, 16), (2, 1, 1))])
def test_two_gpu_parity(grid, procs):
    _run(2, grid, procs)


def test_two_gpu_jump_problem():
    _run(2, (24, 24, 48), (1, 1, 2), problem="jump")


def test_four_gpu_parity():
    _run(4, (32, 32, 32), (1, 2, 2))


@pytest.mark.parametrize("env", [{"PSC_PUSH": "1"}, {"PSC_PUSH": "1", "PSC_REPL_ROWS": "0"},
                                 {"PSC_DEBUG_POISON_HALO": "1"}, {"PSC_DEBUG_POISON_HALO": "1", "PSC_NO_P2P": "1"},
                                 {"PSC_REPL_ROWS": "0"}, {"PSC_REPL_ROWS": "100000000"},
                                 {"PSC_NO_P2P": "1"}, {"PSC_OVERLAP": "1"}, {"PSC_OVERLAP": "1", "PSC_NO_P2P": "1"}],
                         ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_two_gpu_exchange_and_replication_variants(env):
    """Halo slots poisoned with NaN before every exchange (no NaN may leak
    into owned results); replicated suffix from the coarsest level only / from level 1;
    NVLink and NCCL halo exchanges; exchange / interior overlap: all must match the oracle."""
    _run(2, (32, 32, 64), (1, 1, 2), env_extra=env)
