"""The TP group across PROCESSES: two ranks launched by
torch.distributed.run exchange their exchange buffers' CUDA IPC handles over
gloo and reduce through the mapped peer memory (scripts/tp_group_mp.py) —
the deployment path of one process per GPU. On a one-GPU box both processes
share the device (the kernels time-slice); logits must be bit-equal to the
loopback shards of one context and the residual stream equal across ranks."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_tp_group_two_processes_over_ipc():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "scripts", "tp_group_mp.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env=dict(os.environ, OMP_NUM_THREADS="1"))
    assert out.returncode == 0, out.stderr[-4000:]
    j = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert j["ranks"] == 2 and j["logits_equal_loopback"] and j["residual_equal_across_ranks"], j
