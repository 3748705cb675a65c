"""Multi-GPU parity (one process per GPU, IPC peer maps over NVLink/NVSwitch).

Runs tests/mp_worker.py under torchrun on 2, 4 and 8 GPUs when the box has them; every
rank's buffer must be bit-exact against the CPU oracle for GenTree, CPS, Ring, RB, RHD and
HCPS plans, fp32 and bf16, ragged sizes, two back-to-back calls per buffer."""
import os
import subprocess
import sys

import pytest

from tests.gpu_util import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ngpus():
    if not cuda_ok():
        return 0
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_nvls_in_switch_reduction(world):
    """NEXT #1: NVLS plan kind (multimem.ld_reduce / multimem.st through the NVSwitch)."""
    if ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, AR_FLAG_TIMEOUT_MS="20000", PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29618", os.path.join(ROOT, "tests", "mp_nvls_worker.py")]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert f"nvls_worker world={world}: OK" in r.stdout


@pytest.mark.parametrize("jitter", [0, 20000])
@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_multi_process_bit_exact(world, jitter):
    """jitter > 0: random delays (ns) before every flag post on every GPU.
    world = 3: a rank count that is not a power of two (no RHD; LL128 blocks of N·4 elements)."""
    if world == 3 and jitter:
        pytest.skip("N = 3 runs without jitter only (time)")
    if ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, AR_FLAG_TIMEOUT_MS="20000", PYTHONPATH=ROOT, AR_JITTER_NS=str(jitter))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29617", os.path.join(ROOT, "tests", "mp_worker.py")]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert f"mp_worker world={world}: OK" in r.stdout


@pytest.mark.parametrize("world,R", [(2, 4), (2, 8), (4, 8), (8, 8)])
def test_multi_level_ranks_per_gpu(world, R):
    """NEXT #3: R ranks per GPU across GPUs (C5's 8 ranks/GPU; 8 x 8 = C5's 64 ranks)."""
    if ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, AR_FLAG_TIMEOUT_MS="20000", PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29619", os.path.join(ROOT, "tests", "mp_hybrid_worker.py"),
           str(R)]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert f"hybrid_worker nproc={world} R={R}: OK" in r.stdout


@pytest.mark.parametrize("world", [2, 4])
def test_push_protocol_bit_exact(world):
    """The A/B push protocol (AR_PUSH_MAX_MB, off by default) keeps the plan's bits."""
    if ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, AR_FLAG_TIMEOUT_MS="20000", PYTHONPATH=ROOT, AR_PUSH_MAX_MB="64")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29620", os.path.join(ROOT, "tests", "mp_worker.py")]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert f"mp_worker world={world}: OK" in r.stdout


@pytest.mark.parametrize("world", [2, 4])
def test_static_tiles_bit_exact(world):
    """AR_DYN=0 (static per-CTA slices instead of the default dynamic tiles for CPS-shaped
    plans) keeps the plan's bits."""
    if ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, AR_FLAG_TIMEOUT_MS="20000", PYTHONPATH=ROOT, AR_DYN="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29621", os.path.join(ROOT, "tests", "mp_worker.py")]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert f"mp_worker world={world}: OK" in r.stdout

