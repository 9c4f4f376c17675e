"""Guard-set hits (chaos.cpp:15-24) on the speculative chain.

The reference's own guard tests (test_chaos.cpp:185-213) hit the guard in the
seed or the 256-step warm-up, which the GPU runs with the exact step.  These
lanes (tests/guard_orbits.py) hit 0.5, p and 0 at chosen stream iterations,
after the warm-up, where the chain speculates and the verifier and fix-up
must repair the step; p = 1/4 orbits then re-hit p every 25 iterations, in
every later verify group and generator launch.
"""
import struct

import numpy as np
import pytest

import guard_orbits as g
from _oracle import plcm_stream

OTHER = (0.6180339887498949, 0.3090169943749474)  # a generic second lane


def _model_stream(xa, pa, xb, pb, iterations):
    """Bytes of the reference Prbg (chaos.cpp:79-153) from the Python model."""
    xa, xb = g.guard(xa, pa), g.guard(xb, pb)
    for _ in range(g.WARMUP):
        xa, xb = g.guard(g.step(xa, pa), pa), g.guard(g.step(xb, pb), pb)
    out = bytearray()
    for _ in range(iterations):
        xa, xb = g.guard(g.step(xa, pa), pa), g.guard(g.step(xb, pb), pb)
        v = struct.unpack("<Q", struct.pack("<d", xa))[0] ^ struct.unpack("<Q", struct.pack("<d", xb))[0]
        out += (v & ((1 << 48) - 1)).to_bytes(6, "little")
    return np.frombuffer(bytes(out), dtype=np.uint8)


@pytest.mark.parametrize("kind,at,s", g.CASES)
def test_guard_seed_hits_where_designed(kind, at, s):
    x0, p = g.seed(kind, at, s)
    hits = g.stream_hits(x0, p, 300)
    want = {"half": 0.5, "p": p, "zero": 0.0}[kind]
    assert hits and hits[0] == (at, want)
    if s == 2:  # p = 1/4: the guard keeps firing every 25 iterations
        assert [i for i, _ in hits] == list(range(at, 301, 25))[: len(hits)]


@pytest.mark.parametrize("kind,at,s", g.CASES[:4])
def test_guard_model_matches_oracle(kind, at, s):
    # pins the Python model (and so the designed hits) to the C oracle
    x0, p = g.seed(kind, at, s)
    n = 400
    assert np.array_equal(_model_stream(x0, p, *OTHER, n), plcm_stream(x0, p, *OTHER, 6 * n))


@pytest.mark.gpu
@pytest.mark.parametrize("kind,at,s", g.CASES)
def test_guard_hits_on_speculative_chain(kind, at, s):
    import paper_2302_07411_b200 as cve
    x0, p = g.seed(kind, at, s)
    n = 6 * 5000
    for lanes in ([x0, p, *OTHER], [*OTHER, x0, p]):
        assert np.array_equal(cve.keystream_generate(lanes, n), plcm_stream(*lanes, n)), lanes


@pytest.mark.gpu
def test_guard_hits_in_both_lanes_across_launches():
    # 2.5M iterations = 3 generator launches of 2^20; both lanes re-hit p
    # every 25 iterations, so every launch is fixed up and the next one must
    # still start from the verified (guarded) end point
    import paper_2302_07411_b200 as cve
    xa, pa = g.seed("half", 40, 2)
    xb, pb = g.seed("zero", 11, 2)
    n = 6 * 2_500_000
    got = cve.keystream_generate([xa, pa, xb, pb], n)
    assert np.array_equal(got, plcm_stream(xa, pa, xb, pb, n))


@pytest.mark.gpu
@pytest.mark.parametrize("dense", [False, True])
@pytest.mark.parametrize("kind,at,s", [("half", 30, 3), ("p", 9, 3), ("p", 7, 2)])
def test_guard_hit_resync_limits_replays(kind, at, s, dense):
    # After an exact replay of launch R the chain restarts from the verified
    # end point (launch R+1 in a same-stream pipeline, R+2 here, where chain
    # R+1 already ran from the diverged state): a single guard hit costs a
    # couple of replayed launches, not every later one.  32 launches of 8,192
    # iterations, against the oracle byte for byte.  p = 1/4 lanes re-hit the
    # guard every 25 iterations, so there every launch is replayed.
    import paper_2302_07411_b200 as cve
    x0, p = g.seed(kind, at, s)
    n = 6 * 8192 * 32
    for lanes in ([x0, p, *OTHER], [*OTHER, x0, p]):
        got, rep = cve.keystream_generate_ex(lanes, n, launch_iters=8192, dense=dense)
        assert np.array_equal(got, plcm_stream(*lanes, n)), lanes
        hits = g.stream_hits(x0, p, 8192 * 32)
        if len(hits) == 1:
            assert 1 <= rep <= 3, rep
        else:
            assert rep >= 30, rep


@pytest.mark.gpu
@pytest.mark.parametrize("kind,at,s", g.CASES)
def test_guard_hits_dense_orbit_generator(kind, at, s):
    # the generator variant of one-stream (many-clips) handles: every orbit
    # value stored, the verifier reads them back
    import paper_2302_07411_b200 as cve
    x0, p = g.seed(kind, at, s)
    n = 6 * 40000
    for lanes in ([x0, p, *OTHER], [*OTHER, x0, p]):
        got, _ = cve.keystream_generate_ex(lanes, n, launch_iters=4096, dense=True)
        assert np.array_equal(got, plcm_stream(*lanes, n)), lanes
