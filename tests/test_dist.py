"""Multi-rank host logic of bench.py on CPU (gloo, world size 2): the
barrier, the max-over-ranks reduction of timings, and per-rank clip keys
(one independent clip per rank -- "replicas only")."""
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
