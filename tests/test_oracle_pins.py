"""Pin the CPU oracle (oracle/hcc_oracle.c) before trusting it.

1. Known-answer tests of the reference's own suites (proj/tests/test_codec.cpp,
   proj/tests/test_collectives.cpp), re-expressed against the oracle.
2. The golden fixtures generated from the unmodified reference library
   (tests/golden/make_golden.py).
3. When oracle/_ref (the reference compiled here) is present: randomized
   byte-for-byte comparison of the oracle against it.
"""
import os

import numpy as np
import pytest

import oracle_lib as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ---- KATs from proj/tests/test_codec.cpp -----------------------------------

def test_rate8_payload_1024():  # test_codec.cpp:103-108
    x = O.fill(14, "uniform", 1024, -4.0, 4.0)
    assert O.fr_compress(8, x).size == 16 * (1 + 64) == 1040


def test_wire_size_formula():  # test_codec.cpp:110-116
    assert O.wire_size("identity", 0, 100) == 400
    assert O.wire_size("fixed-rate", 16, 64) == 129
    assert O.wire_size("fixed-rate", 8, 65) == 130
    assert O.wire_size("fixed-rate", 8, 0) == 0


@pytest.mark.parametrize("rate", [2, 8, 16, 24, 32])
@pytest.mark.parametrize("n", [0, 1, 63, 64, 65, 1000000])
def test_rate_law(rate, n):  # test_codec.cpp:118-129
    x = O.fill(15, "uniform", n)
    assert O.fr_compress(rate, x).size == O.wire_size("fixed-rate", rate, n)


def test_rate32_powers_of_two():  # test_codec.cpp:131-137
    x = np.array([np.ldexp(1.0, -(i % 8)) for i in range(64)], np.float32)
    back = O.fr_decompress(32, O.fr_compress(32, x), 64)
    assert np.max(np.abs(back.astype(np.float64) - x)) <= 2.0 ** -30


def test_rate8_uniform_bound():  # test_codec.cpp:139-146
    x = O.fill(16, "uniform", 64)
    back = O.fr_decompress(8, O.fr_compress(8, x), 64)
    bound = O.block_bound(x, 8)
    assert np.max(np.abs(back.astype(np.float64) - x)) <= bound <= 2.0 ** -6


def test_error_bound_random_blocks():  # test_codec.cpp:148-158
    for rate in (8, 16, 24, 32):
        for t in range(200):
            x = O.fill(17000 + 1000 * rate + t, "finite", 64)
            back = O.fr_decompress(rate, O.fr_compress(rate, x), 64)
            assert np.max(np.abs(back.astype(np.float64) - x)) <= O.block_bound(x, rate)


def test_denormals_zeros():  # test_codec.cpp:174-185
    x = np.zeros(64, np.float32)
    x[1] = np.float32(1.4e-45)
    x[2] = np.float32(-1.5e-42)
    back = O.fr_decompress(16, O.fr_compress(16, x), 64)
    assert np.max(np.abs(back.astype(np.float64) - x)) <= O.block_bound(x, 16)
    z = np.zeros(130, np.float32)
    assert O.fr_decompress(8, O.fr_compress(8, z), 130).tobytes() == z.tobytes()


def test_nonfinite_rejected():  # test_codec.cpp:187-195
    for bad in (np.nan, np.inf, -np.inf):
        x = np.ones(64, np.float32)
        x[10] = bad
        with pytest.raises(FloatingPointError):
            O.fr_compress(8, x)


def test_lossless_constant_chunk():  # test_codec.cpp:73-84 (hand-derived 3077 bytes)
    x = np.ones(4096, np.float32)
    p = O.pred_compress(x)
    assert p.size == 3077
    assert O.pred_decompress(p, 4096).tobytes() == x.tobytes()


# ---- KATs from proj/tests/test_collectives.cpp ------------------------------

def test_rs_two_rank_example():  # test_collectives.cpp:67-75
    out, _ = O.reduce_scatter(np.array([[1, 2], [3, 4]], np.float32), "identity")
    assert out.tolist() == [[4.0], [6.0]]


def test_ar_two_rank_example():  # test_collectives.cpp:162-175
    x = np.array([[1, 2], [3, 4]], np.float32)
    assert O.allreduce(x, "identity")[0].tolist() == [[4, 6], [4, 6]]
    assert O.allreduce(x, "identity", average=True)[0].tolist() == [[2, 3], [2, 3]]


def test_trace_accounting():  # test_collectives.cpp:215-234
    p, n = 4, 256
    x = np.stack([O.fill(39 + j, "uniform", n) for j in range(p)])
    _, (raw, wire, rounds) = O.allreduce(x, "identity")
    assert rounds == 2 * (p - 1)
    assert raw == 2 * (p - 1) * 4 * n // p == wire


def test_ag_lossy_distorts_once():  # test_collectives.cpp:143-160
    shards = np.stack([O.fill(35 + j, "uniform", 64) for j in range(4)])
    out, _ = O.allgather(shards, "fixed-rate", 8)
    for i in range(4):
        for c in range(4):
            direct = O.fr_decompress(8, O.fr_compress(8, shards[c]), 64)
            assert out[i, c * 64:(c + 1) * 64].tobytes() == direct.tobytes()


def test_rs_block_exponent_bound():
    """Re-pinned version of test_collectives.cpp:90-118 (the reference test's
    per-element bound is a test bug): the error of each hop is
    bounded by the *block* exponent of the partial sum that was quantized."""
    p, rate = 4, 16
    x = np.stack([O.fill(33 + j, "uniform", 64 * p) for j in range(p)])
    got, _ = O.reduce_scatter(x, "fixed-rate", rate)
    exact = x.astype(np.float64)
    c = 64
    for i in range(p):
        partial = x[(i + 1) % p, i * c:(i + 1) * c].astype(np.float32)
        bound = 0.0
        for s in range(2, p + 1):
            bound += 2.0 * O.block_bound(partial, rate)
            partial = (partial + x[(i + s) % p, i * c:(i + 1) * c]).astype(np.float32)
        want = sum(exact[(i + s) % p, i * c:(i + 1) * c] for s in range(1, p + 1))
        assert np.max(np.abs(got[i].astype(np.float64) - want)) <= bound


# ---- golden fixtures from the reference library -----------------------------

def test_golden_fixed_rate_fixtures():
    g = np.load(os.path.join(GOLD, "fixed_rate.npz"))
    keys = sorted(k[:-3] for k in g.files if k.endswith("_in"))
    assert len(keys) > 400
    for k in keys:
        rate = int(k.split("_")[0][2:])
        x = g[k + "_in"]
        p = O.fr_compress(rate, x)
        assert p.tobytes() == g[k + "_payload"].tobytes(), k
        assert O.fr_decompress(rate, p, x.size).tobytes() == g[k + "_dec"].tobytes(), k


def test_golden_collective_fixtures():
    g = np.load(os.path.join(GOLD, "collectives.npz"))
    keys = sorted(k[:-3] for k in g.files if k.endswith("_in"))
    assert len(keys) == 48
    for k in keys:
        x = g[k + "_in"]
        kind = "identity" if "identity" in k else "fixed-rate"
        rate = 0 if kind == "identity" else int(k.split("_")[1][10:])
        for avg in (0, 1):
            out, acct = O.allreduce(x, kind, rate, bool(avg))
            assert out.tobytes() == g[f"{k}_ar{avg}"].tobytes(), k
            assert list(acct) == g[f"{k}_ar{avg}_acct"].tolist(), k
        rs, acct = O.reduce_scatter(x, kind, rate)
        assert rs.tobytes() == g[k + "_rs"].tobytes() and list(acct) == g[k + "_rs_acct"].tolist(), k
        n_per = x.shape[1] // x.shape[0]
        ag, acct = O.allgather(np.ascontiguousarray(x[:, :n_per]), kind, rate)
        assert ag.tobytes() == g[k + "_ag"].tobytes() and list(acct) == g[k + "_ag_acct"].tolist(), k
        pp, acct = O.p2p(x[0], kind, rate)
        assert pp.tobytes() == g[k + "_p2p"].tobytes() and list(acct) == g[k + "_p2p_acct"].tolist(), k


# ---- randomized comparison with the reference itself (dev container) --------

needs_ref = pytest.mark.skipif(O.ref is None, reason="oracle/_ref not built (no /root/reference here)")


@needs_ref
def test_rng_matches_reference():
    for mode, lo, hi in [("bits", 0, 0), ("finite", 0, 0), ("uniform", -3, 5), ("sparse", 0.9, 0)]:
        assert O.fill(77, mode, 5000, lo, hi).tobytes() == O.ref_fill(77, mode, 5000, lo, hi).tobytes()


@needs_ref
@pytest.mark.parametrize("rate", list(range(2, 33)))
def test_fixed_rate_matches_reference(rate):
    for n in (0, 1, 63, 64, 65, 1000, 4099):
        for mode, lo, hi in [("finite", 0, 0), ("uniform", -1, 1), ("sparse", 0.5, 0)]:
            x = O.fill(rate * 1000 + n, mode, n, lo, hi)
            a = O.fr_compress(rate, x)
            b, cc = O.ref_compress("fixed-rate", rate, x)
            assert a.tobytes() == b.tobytes()
            assert O.fr_decompress(rate, a, n).tobytes() == O.ref_decompress("fixed-rate", rate, b, n, cc).tobytes()


@needs_ref
def test_lossless_matches_reference():
    for n in (0, 1, 63, 4096, 4097, 10000):
        for mode, lo in [("bits", 0), ("sparse", 0.9), ("uniform", -1)]:
            x = O.fill(n + 5, mode, n, lo, 1)
            a = O.pred_compress(x)
            b, _ = O.ref_compress("lossless", 0, x)
            assert a.tobytes() == b.tobytes()


@needs_ref
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 8])
def test_collectives_match_reference(p):
    for kind, rate in [("identity", 0), ("fixed-rate", 3), ("fixed-rate", 8), ("fixed-rate", 24), ("lossless", 0)]:
        n = p * 333
        x = np.stack([O.fill(11 + 7 * j, "uniform", n) for j in range(p)])
        for avg in (False, True):
            a = O.allreduce(x, kind, rate, avg)
            b = O.ref_allreduce(x, kind, rate, avg)
            assert a[0].tobytes() == b[0].tobytes() and a[1] == b[1]
        a = O.reduce_scatter(x, kind, rate)
        b = O.ref_reduce_scatter(x, kind, rate)
        assert a[0].tobytes() == b[0].tobytes() and a[1] == b[1]
        s = np.ascontiguousarray(x[:, :100])
        a = O.allgather(s, kind, rate)
        b = O.ref_allgather(s, kind, rate)
        assert a[0].tobytes() == b[0].tobytes() and a[1] == b[1]


def test_lossless_oracle_matches_golden():
    """Oracle restatement vs payloads/accounting produced by the reference
    itself (tests/golden/lossless.npz, make_golden.py)."""
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "lossless.npz"))
    keys = sorted(k[:-8] for k in g.files if k.endswith("_payload"))
    assert keys
    for k in keys:
        x = g[k + "_in"]
        assert O.pred_compress(x).tobytes() == g[k + "_payload"].tobytes(), k
        assert O.pred_decompress(g[k + "_payload"], x.size).tobytes() == x.tobytes(), k
    for k in sorted(k[:-3] for k in g.files if k.endswith("_rs") and k.startswith("p")):
        x = g[k + "_in"]
        p = x.shape[0]
        for avg in (0, 1):
            out, acct = O.allreduce(x, "lossless", 0, bool(avg))
            assert out.tobytes() == g[f"{k}_ar{avg}"].tobytes() and acct == tuple(g[f"{k}_ar{avg}_acct"]), k
        out, acct = O.reduce_scatter(x, "lossless")
        assert out.tobytes() == g[k + "_rs"].tobytes() and acct == tuple(g[k + "_rs_acct"]), k
        out, acct = O.allgather(np.ascontiguousarray(x[:, : x.shape[1] // p]), "lossless")
        assert out.tobytes() == g[k + "_ag"].tobytes() and acct == tuple(g[k + "_ag_acct"]), k
        _, acct = O.p2p(x[1], "lossless")
        assert acct == tuple(g[k + "_p2p_acct"]), k
