"""N > 1 host-side logic on CPU: two processes (gloo, world_size 2, 127.0.0.1) each build the
plan and its device step tables independently through the C-ABI, exchange them with
torch.distributed and check that (1) the plans and tables are byte-identical on every rank
(determinism), (2) every wait a rank's program posts on (producer, slot) is matched by
that producer's notify of the same slot, and (3) every notify has a consumer that waits for
it — the cross-process contract of the flag protocol."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world_of_plan", [2, 4])
def test_two_process_plan_and_protocol_agreement(world_of_plan, tmp_path):
    out = tmp_path / "gathered.json"
    port = free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   PYTHONPATH=ROOT)
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "gloo_worker.py"),
                                       str(world_of_plan), str(out)], env=env, cwd=ROOT))
    for p in procs:
        assert p.wait(timeout=300) == 0
    res = json.loads(out.read_text())
    for allv in res:
        assert allv[0]["plan"] == allv[1]["plan"]
        assert allv[0]["low"] == allv[1]["low"]
        ranks = allv[0]["low"]["ranks"]
        notifies = {(r, s["slot"], c) for r, rk in enumerate(ranks) for s in rk["steps"] for c in s["notify"]}
        waits = {(t, slot, r) for r, rk in enumerate(ranks) for s in rk["steps"] for (t, slot, *_) in s["waits"]}
        assert waits <= notifies, waits - notifies
        assert notifies <= waits, notifies - waits
