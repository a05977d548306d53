"""bench.py's multi-GPU plumbing on CPU: `--gpus N` launches N ranks, a
world / --gpus mismatch or missing GPUs exits non-zero, and the timing
reduction is the max over ranks (gloo, world size 2)."""

import os
import sys
import types

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _args(gpus):
    return types.SimpleNamespace(gpus=gpus)


def test_gpus_n_reexecs_under_torchrun(monkeypatch):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    seen = {}

    def fake_execv(path, argv):
        seen["argv"] = argv
        raise SystemExit(0)

    monkeypatch.setattr(os, "execv", fake_execv)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3"])
    with pytest.raises(SystemExit):
        bench.launch_ranks(_args(4))
    argv = seen["argv"]
    assert argv[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in argv and "--master-addr=127.0.0.1" in argv
    assert argv[-4:] == ["--gpus", "4", "--steps", "3"]


def test_single_gpu_runs_in_process(monkeypatch):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(os, "execv", lambda *a: pytest.fail("must not re-exec for N=1"))
    bench.launch_ranks(_args(1))


def test_world_mismatch_exits_nonzero(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "2")
    with pytest.raises(SystemExit) as err:
        bench.launch_ranks(_args(8))
    assert err.value.code not in (0, None)


def test_missing_gpus_exit_nonzero():
    import torch
    with pytest.raises(SystemExit) as err:
        bench.require_gpus(torch, 8, 0)     # no GPU in this container
    assert "need 8 GPUs" in str(err.value.code)


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out[rank] = (bench.max_over_ranks(1.5 + rank, world, "cpu"),
                 bench.sum_over_ranks(10 + rank, world, "cpu"))
    dist.destroy_process_group()


def test_timing_is_max_over_ranks_gloo():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        assert out[0] == out[1] == (2.5, 21)


def test_reference_install_is_unmodified_pintoc():
    """The reference arm's baseline/_ref is pintoc as it lies under
    /root/reference (installed by __graft_entry__.build()); skipped where the
    reference tree does not exist (the GPU box)."""
    import filecmp
    src = "/root/reference/pkg/src/pintoc"
    if not os.path.isdir(src):
        pytest.skip("no reference tree here")
    import __graft_entry__ as entry
    entry._install_reference()  # no-op when already installed
    dst = os.path.join(ROOT, "baseline", "_ref", "pintoc")
    names = sorted(f for f in os.listdir(src) if f.endswith(".py"))
    assert names and "passes.py" in names
    match, mismatch, errors = filecmp.cmpfiles(src, dst, names, shallow=False)
    assert not mismatch and not errors, (mismatch, errors)
    assert bench.reference_impl() == "pintoc"
