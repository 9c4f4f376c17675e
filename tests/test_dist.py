"""Multi-rank host logic of bench.py on CPU (gloo, world size 2): the
barrier, the max-over-ranks reduction of timings, per-rank clip keys of the
labelled multi-clip line, and the reference arm's contract (same config as
the B200 arm, only the reference's own library mapped).  The headline at
N > 1 is ONE clip sharded over the GPUs; its device path is
covered by the sharded-handle GPU tests."""
import os
import socket
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import bench
    from workloads import synth
    d = bench.Dist(use_cuda=False)
    d.barrier()
    m = d.max(float(rank + 1) * 1.5)
    c = synth.CONFIGS["C4"]
    key = synth.det_key(c["key_seed"] + 1000 * d.rank)
    out[rank] = (m, key, d.world)
    d.close()


def test_two_rank_barrier_and_max():
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert out[0][0] == out[1][0] == 3.0          # max over ranks
    assert out[0][2] == out[1][2] == 2
    assert out[0][1] != out[1][1]                  # independent clip per rank


def test_reference_arm_other_ranks_exit_quietly(monkeypatch, capsys):
    import bench
    monkeypatch.setenv("WORLD_SIZE", "1")
    monkeypatch.setenv("RANK", "0")
    # non-zero rank under a 2-rank launch does no work: emulate via Dist attrs
    d = bench.Dist.__new__(bench.Dist)
    d.world, d.rank, d.local, d.pg = 2, 1, 1, None
    monkeypatch.setattr(bench, "Dist", lambda use_cuda: d)
    args = type("A", (), dict(config="C4", gpus=2, steps=1, warmup=0))()
    bench.run_reference(args)
    assert capsys.readouterr().out == ""


def test_reference_arm_config_matches_b200_arm():
    # both arms build the SAME config dict (frames per step rounded to the
    # GPU count, the L2 note, the sharding description)
    import bench
    for gpus in (1, 2, 8):
        args = type("A", (), dict(config="C4", gpus=gpus, frames=24, shard_devices=""))()
        F = bench.frames_per_step(args)
        assert F % gpus == 0 and F >= 24
        a = bench.config_dict("C4", F, gpus)
        b = bench.config_dict("C4", bench.frames_per_step(args), gpus)
        assert a == b and a["frames_per_step"] == F
        assert ("sharded" in a["parallelism"]) == (gpus > 1)
    assert bench.scaling_of(1) == bench.scaling_of(8) == "strong"


def test_harness_import_does_not_map_the_product_library():
    # the reference arm imports workloads.synth and tests/_oracle: neither may
    # load libcve_b200.so (the driver checks which .so files the arm mapped)
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path[:0] = [%r, %r]; import bench; from workloads import synth; "
            "import _oracle; print(bench.mapped_libraries())" % (root, os.path.join(root, "tests")))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=300, cwd=root)
    assert out.returncode == 0, out.stderr
    assert "libcve_b200" not in out.stdout, out.stdout
