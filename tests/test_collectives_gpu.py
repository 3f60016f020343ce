"""Single-device ring collectives (virtual ranks) vs the CPU oracle.

Every member's buffer lives on one B200 and the ring runs through the same
kernels as the NVLink engine.  Bar: bit-exact against the oracle restatement
of proj/src/collectives.cpp (pinned to the reference in test_oracle_pins.py)
and against the golden fixtures produced by the reference itself; cases of
proj/tests/test_collectives.cpp re-expressed.
"""
import os

import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")

CODECS = [("identity", 0), ("fixed-rate", 2), ("fixed-rate", 3), ("fixed-rate", 4), ("fixed-rate", 8),
          ("fixed-rate", 12), ("fixed-rate", 16), ("fixed-rate", 24), ("fixed-rate", 32)]


def _inputs(seed, p, n, mode="uniform"):
    return np.stack([O.fill(seed + 31 * j, mode, n, 1e-3 if mode == "normal" else -1.0, 1.0) for j in range(p)])


def _oracle_kind(kind):
    return kind


@pytest.mark.parametrize("p", [2, 3, 4, 5, 8])
@pytest.mark.parametrize("kind,rate", CODECS)
def test_allreduce_bit_exact(cuda, p, kind, rate):
    import hccx_util as U

    g = U.Group(p)
    for n_per in (64, 100, 256, 1000, 2048 + 64):
        n = n_per * p
        x = _inputs(p * 1000 + n_per + rate, p, n)
        for avg in (False, True):
            got, st = g.allreduce(x, kind, rate, avg)
            assert st == 0
            want, _ = O.allreduce(x, kind, rate, avg)
            assert got.tobytes() == want.tobytes(), (p, kind, rate, n, avg)


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("kind,rate", CODECS)
def test_reduce_scatter_allgather_bit_exact(cuda, p, kind, rate):
    import hccx_util as U

    g = U.Group(p)
    for n_per in (64, 300, 4096):
        n = n_per * p
        x = _inputs(p * 77 + n_per + rate, p, n)
        got, st = g.reduce_scatter(x, kind, rate)
        assert st == 0
        want, _ = O.reduce_scatter(x, kind, rate)
        assert got.tobytes() == want.tobytes(), (p, kind, rate, n)
        s = np.ascontiguousarray(x[:, :n_per])
        got, st = g.allgather(s, kind, rate)
        assert st == 0
        want, _ = O.allgather(s, kind, rate)
        assert got.tobytes() == want.tobytes(), (p, kind, rate, n_per)


@pytest.mark.parametrize("kind,rate", CODECS + [("zfp-rate", 8)])
def test_p2p_and_broadcast(cuda, kind, rate):
    import hccx_util as U

    g = U.Group(4)
    for n in (1, 64, 1000, 70000):
        x = O.fill(n + rate, "uniform", n)
        got, st = g.p2p(x, kind, rate)
        assert st == 0
        want, _ = O.p2p(x, kind, rate)
        assert got.tobytes() == want.tobytes()
        for root in (0, 3):
            got, st = g.broadcast(x, root, kind, rate)
            assert st == 0
            want, _ = O.broadcast(x, 4, kind, rate)
            assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("rate", [4, 8, 16])
def test_zfp_mode_collectives_match_restatement(cuda, rate):
    import hccx_util as U

    for p in (2, 4):
        g = U.Group(p)
        x = _inputs(rate + p, p, 1000 * p)
        got, st = g.allreduce(x, "zfp-rate", rate)
        assert st == 0
        assert got.tobytes() == O.allreduce(x, "zfp-rate", rate)[0].tobytes()
        got, st = g.reduce_scatter(x, "zfp-rate", rate)
        assert got.tobytes() == O.reduce_scatter(x, "zfp-rate", rate)[0].tobytes()


def test_inplace_allreduce(cuda):
    import hccx_util as U

    g = U.Group(4)
    x = _inputs(5, 4, 4 * 8192, "normal")
    got, st = g.allreduce(x, "fixed-rate", 8, False, inplace=True)
    assert st == 0 and got.tobytes() == O.allreduce(x, "fixed-rate", 8)[0].tobytes()


def test_large_p8_rate8(cuda):
    """Config-2-shaped (p=8, rate 8) at 2^22 values per rank: bit-exact."""
    import hccx_util as U

    p, n = 8, 1 << 22
    x = _inputs(1234, p, n, "normal")
    got, st = U.Group(p).allreduce(x, "fixed-rate", 8, True)
    assert st == 0
    assert got.tobytes() == O.allreduce(x, "fixed-rate", 8, True)[0].tobytes()


def test_golden_collectives_on_gpu(cuda):
    import hccx_util as U

    g = np.load(os.path.join(GOLD, "collectives.npz"))
    groups = {}
    for k in sorted(k[:-3] for k in g.files if k.endswith("_in")):
        x = g[k + "_in"]
        p = x.shape[0]
        grp = groups.setdefault(p, U.Group(p))
        kind = "identity" if "identity" in k else "fixed-rate"
        rate = 0 if kind == "identity" else int(k.split("_")[1][10:])
        for avg in (0, 1):
            got, st = grp.allreduce(x, kind, rate, bool(avg))
            assert st == 0 and got.tobytes() == g[f"{k}_ar{avg}"].tobytes(), k
        got, st = grp.reduce_scatter(x, kind, rate)
        assert got.tobytes() == g[k + "_rs"].tobytes(), k
        n_per = x.shape[1] // p
        got, st = grp.allgather(np.ascontiguousarray(x[:, :n_per]), kind, rate)
        assert got.tobytes() == g[k + "_ag"].tobytes(), k
        got, st = grp.p2p(x[0], kind, rate)
        assert got.tobytes() == g[k + "_p2p"].tobytes(), k


def test_errors(cuda):
    import hccx_util as U

    g = U.Group(2)
    x = _inputs(1, 2, 6)
    # n % p != 0 -> BadChunking (test_collectives.cpp:248-261)
    _, st = g.allreduce(_inputs(1, 2, 3), "identity")
    assert st == 4
    # partial sums overflowing to Inf mid-ring -> NonFinite at the next compress
    big = np.full((2, 128), 3.0e38, np.float32)
    _, st = g.allreduce(big, "fixed-rate", 8)
    assert st == 1
    _, st = g.allreduce(big, "identity")
    assert st == 0
    del x


def test_python_collectives_api(cuda):
    """The reference-shaped API: SimClock + Communicator + list of buffers."""
    import paper_2409_02423_b200 as H
    from paper_2409_02423_b200 import collectives as K
    from paper_2409_02423_b200.netsim import CollectiveKind, SimClock, Topology

    clock = SimClock(Topology.lassen_like(2))
    comm = K.Communicator(list(range(4)))
    x = _inputs(40, 4, 256 * 4)
    out = K.allreduce(clock, comm, list(x), H.CodecSpec.fixed_rate(8), H.CommPath.DpAllReduce)
    want, (raw, wire, rounds) = O.allreduce(x, "fixed-rate", 8)
    assert np.stack(out).tobytes() == want.tobytes()
    e = clock.trace()[0]
    assert (e.raw_bytes, e.wire_bytes, e.round_count, e.comm_size) == (raw, wire, rounds, 4)
    assert e.collective == CollectiveKind.AllReduce and e.duration_s > 0
    assert len({clock.time(r) for r in range(4)}) == 1
    assert e.wire_bytes < e.raw_bytes and e.wire_bytes > e.raw_bytes // 8  # test_collectives.cpp:236-246
    # singleton: untouched, nothing recorded (test_collectives.cpp:263-271)
    clk2 = SimClock(Topology.lassen_like(2))
    one = K.allreduce(clk2, K.Communicator([0]), [np.array([1, 2, 3], np.float32)], H.CodecSpec.fixed_rate(8),
                      H.CommPath.DpAllReduce)
    assert one[0].tolist() == [1, 2, 3] and not clk2.trace() and clk2.max_time() == 0.0
    with pytest.raises(H.BadChunkingError):
        K.allreduce(clock, K.Communicator([0, 1]), [np.ones(3, np.float32)] * 2, H.CodecSpec.identity(),
                    H.CommPath.DpAllReduce)
    with pytest.raises(H.BadChunkingError):
        K.ring_allgather(clock, K.Communicator([0, 1]), [np.ones(2, np.float32), np.ones(1, np.float32)],
                         H.CodecSpec.identity(), H.CommPath.TpAllGather)
    p2 = K.p2p(clock, 0, 1, x[0], H.CodecSpec.fixed_rate(8), H.CommPath.PpP2p)
    assert p2.tobytes() == O.p2p(x[0], "fixed-rate", 8)[0].tobytes()
    assert clock.trace()[-1].raw_bytes == 4 * x.shape[1]
    rs = K.ring_reduce_scatter(clock, comm, list(x), H.CodecSpec.fixed_rate(16), H.CommPath.Zero1ReduceScatter)
    assert np.stack(rs).tobytes() == O.reduce_scatter(x, "fixed-rate", 16)[0].tobytes()
    bc = K.broadcast(clock, comm, 2, x[2], H.CodecSpec.fixed_rate(8), H.CommPath.PpP2p)
    assert np.stack(bc).tobytes() == O.broadcast(x[2], 4, "fixed-rate", 8)[0].tobytes()
