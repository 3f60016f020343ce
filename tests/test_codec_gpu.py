"""FixedRate / Identity / zfp-rate codec kernels on the B200 vs the CPU oracle.

Bit-exact bar: payload bytes equal hcc::compress's (oracle restatement, itself
pinned to the reference in test_oracle_pins.py) and decoded floats equal
hcc::decompress's, for every rate 2..32, tail shapes, alignments and the
edge cases of proj/tests/test_codec.cpp.
"""
import os

import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SIZES = [1, 7, 63, 64, 65, 255, 256, 257, 511, 1000, 1024, 4096 + 64, 65536 + 17]
MODES = [("uniform", -1.0, 1.0), ("finite", 0, 0), ("sparse", 0.5, 0), ("normal", 1e-3, 0)]


def _cases(seed0):
    s = seed0
    for n in SIZES:
        for mode, lo, hi in MODES:
            s += 1
            yield n, mode, O.fill(s, mode, n, lo, hi)


@pytest.mark.parametrize("rate", list(range(2, 33)))
def test_fixed_rate_bit_exact(cuda, rate):
    import hccx_util as U

    for n, mode, x in _cases(rate * 10007):
        want = O.fr_compress(rate, x)
        got, st = U.compress("fixed-rate", rate, x)
        assert st == 0
        assert got.tobytes() == want.tobytes(), (rate, n, mode)
        dec = U.decompress("fixed-rate", rate, got, n)
        assert dec.tobytes() == O.fr_decompress(rate, want, n).tobytes(), (rate, n, mode)


@pytest.mark.parametrize("rate", [3, 4, 8, 13, 16, 24, 32])
def test_fixed_rate_unaligned_pointers(cuda, rate):
    import hccx_util as U

    x = O.fill(rate, "uniform", 4096 * 3 + 5)
    want = O.fr_compress(rate, x)
    for in_off, out_off in [(1, 0), (0, 1), (3, 2), (5, 3)]:
        got, st = U.compress("fixed-rate", rate, x, in_off, out_off)
        assert st == 0 and got.tobytes() == want.tobytes(), (in_off, out_off)
        dec = U.decompress("fixed-rate", rate, got, x.size, out_off, in_off)
        assert dec.tobytes() == O.fr_decompress(rate, want, x.size).tobytes()


def test_config1_size_bit_exact(cuda):
    """BASELINE config 1: 2^24 gradient-like values at rate 8."""
    import hccx_util as U

    n = 1 << 24
    x = O.fill(1234, "normal", n, 1e-3)
    want = O.fr_compress(8, x)
    got, st = U.compress("fixed-rate", 8, x)
    assert st == 0 and got.size == 17039360
    assert got.tobytes() == want.tobytes()
    dec = U.decompress("fixed-rate", 8, got, n)
    assert dec.tobytes() == O.fr_decompress(8, want, n).tobytes()


def test_golden_fixtures_on_gpu(cuda):
    import hccx_util as U

    g = np.load(os.path.join(GOLD, "fixed_rate.npz"))
    for k in sorted(k[:-3] for k in g.files if k.endswith("_in")):
        rate = int(k.split("_")[0][2:])
        x = g[k + "_in"]
        got, st = U.compress("fixed-rate", rate, x)
        assert st == 0 and got.tobytes() == g[k + "_payload"].tobytes(), k
        assert U.decompress("fixed-rate", rate, got, x.size).tobytes() == g[k + "_dec"].tobytes(), k


def test_special_values(cuda):
    import hccx_util as U

    x = np.zeros(64 * 6, np.float32)
    x[1] = np.float32(1.4e-45)
    x[2] = np.float32(-1.5e-42)
    x[64:128] = -0.0
    x[128:192] = np.float32(3.0e38)
    x[192] = np.float32(-3.4e38)
    x[256:320] = np.float32(1.17549435e-38)  # smallest normal
    x[320:] = np.ldexp(np.float32(1.0), -np.arange(64) % 40).astype(np.float32)
    for rate in range(2, 33):
        got, st = U.compress("fixed-rate", rate, x)
        assert st == 0 and got.tobytes() == O.fr_compress(rate, x).tobytes(), rate
        assert U.decompress("fixed-rate", rate, got, x.size).tobytes() == \
            O.fr_decompress(rate, got, x.size).tobytes(), rate


def test_nonfinite_flagged(cuda):  # test_codec.cpp:187-195
    import hccx_util as U

    for bad in (np.nan, np.inf, -np.inf):
        for pos in (0, 10, 4095, 70001):
            x = np.ones(70002, np.float32)
            x[pos] = bad
            _, st = U.compress("fixed-rate", 8, x)
            assert st == 1  # HCCX_ERR_NONFINITE
    _, st = U.compress("fixed-rate", 8, np.ones(1000, np.float32))
    assert st == 0


def test_corrupt_payload_rejected(cuda):  # test_codec.cpp:225-232
    import ctypes as C

    import torch

    from paper_2409_02423_b200 import _lib

    buf = torch.zeros(2000, dtype=torch.uint8, device="cuda")
    out = torch.zeros(100, device="cuda")
    st = _lib.hccx_decompress(_lib.Codec(2, 8), buf.data_ptr(), 129, 100, out.data_ptr(), None)
    assert st == 2
    st = _lib.hccx_decompress(_lib.Codec(2, 8), buf.data_ptr(), 131, 100, out.data_ptr(), None)
    assert st == 2
    del C


def test_identity_round_trip(cuda):
    import hccx_util as U

    x = O.fill(5, "bits", 10001)
    got, st = U.compress("identity", 0, x)
    assert st == 0 and got.tobytes() == x.tobytes()
    assert U.decompress("identity", 0, got, x.size).tobytes() == x.tobytes()


def test_host_pipeline_api(cuda):
    """hccx_compress_host/_decompress_host: several 4 Mi slices + tail."""
    import ctypes as C

    from paper_2409_02423_b200 import _lib

    n = (1 << 22) * 2 + 12345
    x = O.fill(99, "normal", n, 1e-3)
    for rate in (4, 8, 13):
        want = O.fr_compress(rate, x)
        got = np.zeros(want.size, np.uint8)
        assert _lib.hccx_compress_host(_lib.Codec(2, rate), x.ctypes.data, n, got.ctypes.data, 0) == 0
        assert got.tobytes() == want.tobytes(), rate
        dec = np.zeros(n, np.float32)
        assert _lib.hccx_decompress_host(_lib.Codec(2, rate), got.ctypes.data, got.size, n, dec.ctypes.data, 0) == 0
        assert dec.tobytes() == O.fr_decompress(rate, want, n).tobytes()
    y = x.copy()
    y[n - 3] = np.inf
    got = np.zeros(O.wire_size("fixed-rate", 8, n), np.uint8)
    assert _lib.hccx_compress_host(_lib.Codec(2, 8), y.ctypes.data, n, got.ctypes.data, 0) == 1
    del C


def test_python_codec_api(cuda):
    import torch

    import paper_2409_02423_b200 as H

    x = O.fill(3, "uniform", 5000)
    spec = H.CodecSpec.fixed_rate(12)
    cb = H.compress(spec, x)
    assert cb.payload_bytes() == H.wire_size_bytes(spec, x.size) and cb.chunk_count == 79
    assert cb.payload.tobytes() == O.fr_compress(12, x).tobytes()
    assert H.decompress(cb).tobytes() == O.fr_decompress(12, cb.payload, x.size).tobytes()
    back = H.from_bytes(H.to_bytes(cb))
    assert H.decompress(back).tobytes() == H.decompress(cb).tobytes()
    t = torch.from_numpy(x).cuda()
    cbd = H.compress(spec, t)
    assert cbd.payload.cpu().numpy().tobytes() == cb.payload.tobytes()
    assert H.decompress(cbd).cpu().numpy().tobytes() == H.decompress(cb).tobytes()
    bad = x.copy()
    bad[7] = np.nan
    with pytest.raises(H.NonFiniteInputError):
        H.compress(spec, bad)
    with pytest.raises(H.NonFiniteInputError):
        H.compress(spec, torch.from_numpy(bad).cuda())
    short = H.codec.CompressedBuffer(spec, cb.original_len, cb.chunk_count, cb.payload[:-1])
    with pytest.raises(H.CorruptPayloadError):
        H.decompress(short)
    wrong = H.codec.CompressedBuffer(spec, cb.original_len, cb.chunk_count + 1, cb.payload)
    with pytest.raises(H.CorruptPayloadError):
        H.decompress(wrong)


@pytest.mark.parametrize("rate", list(range(3, 33)))
def test_zfp_mode_matches_restatement(cuda, rate):
    """zfp-rate codec (not in the reference; parity unpinned): bit-exact
    against the CPU restatement of 1-D zfp fixed-rate in oracle/hcc_oracle.c."""
    import hccx_util as U

    for n, mode, x in _cases(rate * 7919):
        if n > 5000:
            continue
        want = O.zfp_compress(rate, x)
        got, st = U.compress("zfp-rate", rate, x)
        assert st == 0
        assert got.tobytes() == want.tobytes(), (rate, n, mode)
        assert U.decompress("zfp-rate", rate, got, n).tobytes() == O.zfp_decompress(rate, want, n).tobytes()
