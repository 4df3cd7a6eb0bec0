"""World-size-2 gloo test (CPU) of the row-sharding decomposition: the
sharded oracle -- all-reduces exactly where the CUDA path all-reduces -- on
two processes reproduces the unsharded oracle's iterates."""

import os
import socket
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("case", ["lasso", "mixed"])
def test_two_rank_gloo_sharded_oracle(case, tmp_path):
    port = _port()
    outs = [str(tmp_path / f"r{r}.txt") for r in range(2)]
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "_gloo_worker.py"), str(r), "2",
                               str(port), case, outs[r]]) for r in range(2)]
    for p in procs:
        assert p.wait(timeout=300) == 0
    for o in outs:
        worst = float(open(o).read())
        assert worst < 1e-10, worst
