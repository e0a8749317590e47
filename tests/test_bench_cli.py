"""CPU checks of bench.py's launcher logic: `--gpus N` outside torchrun re-launches the script as
N ranks through torch.distributed.run on 127.0.0.1 (the driver's own launch line), and the
default workload is BASELINE's metric configuration C5."""
from __future__ import annotations

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture()
def bench(monkeypatch):
    sys.path.insert(0, ROOT)
    import importlib
    mod = importlib.import_module("bench")
    return mod


def test_default_workload_is_c5(bench, monkeypatch):
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    monkeypatch.delenv("BENCH_CONFIG", raising=False)
    args = bench.parse()
    assert args.config == "c5" and args.gpus == 1 and args.warmup >= 3


def test_gpus_n_relaunches_under_torchrun(bench, monkeypatch):
    calls = []
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2", "--warmup", "3"])
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    assert bench.main() == 0
    (cmd,) = calls
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-6:] == ["--gpus", "4", "--steps", "2", "--warmup", "3"]   # the same arguments per rank


def test_reference_arm_does_not_relaunch(bench, monkeypatch):
    """The reference arm (the oracle on the host cores) runs in rank 0 only: no relaunch."""
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "2", "--impl", "reference"])
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    args = bench.parse()
    assert args.impl == "reference"
    called = []
    monkeypatch.setattr(bench, "run_reference", lambda a, c, t: called.append(a.gpus) or 0)
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: pytest.fail("relaunched"))
    assert bench.main() == 0 and called == [2]
