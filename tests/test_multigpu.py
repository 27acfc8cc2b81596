"""Multi-GPU parity (torchrun, one process per GPU).  Skipped on boxes with < 2 GPUs;
run with `gpurun --gpus 2|4 -- python -m pytest tests/test_multigpu.py -m gpu`."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,proto", [(2, "pull"), (4, "pull"), (2, "push")])
def test_dp_step_multigpu(world, proto, tmp_path):
    """proto: the FUSED reduction's pull kernel (default) or the copy-engine push protocol (MTX_FUSED_PUSH=1)."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    rep = tmp_path / "report.json"
    env = dict(os.environ, MTX_MP_REPORT=str(rep), PYTHONPATH=ROOT, MTX_FUSED_PUSH="1" if proto == "push" else "0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "tests", "mp_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    msg = r.stdout[-4000:] + r.stderr[-4000:]
    assert r.returncode == 0, msg
    reports = json.load(open(rep))
    assert all(x["ok"] for x in reports), msg
