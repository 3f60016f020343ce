"""LosslessPredictor on the GPU (csrc/lossless.cu) vs the reference.

Bar: payload bytes identical to hcc::compress(LosslessPredictor) (golden
fixtures made by the reference library, tests/golden/lossless.npz, and the
oracle restatement pinned to it), bit-exact round trips, the reference's
error behaviour on truncated payloads, and collective byte accounting equal
to the reference's.  Cases of proj/tests/test_codec.cpp:60-100, :237-239 and
proj/tests/test_collectives.cpp:35-50, :189-203, :275-292 re-expressed.
"""
import os

import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "lossless.npz")


def _spec():
    import paper_2409_02423_b200 as H

    return H.CodecSpec.lossless()


def test_golden_payloads_host_and_device(cuda):
    import torch

    import paper_2409_02423_b200 as H

    g = np.load(GOLD)
    keys = sorted(k[:-8] for k in g.files if k.endswith("_payload"))
    for k in keys:
        x, want = g[k + "_in"], g[k + "_payload"]
        cb = H.compress(_spec(), x)
        assert cb.chunk_count == int(g[k + "_cc"][0]), k
        assert np.asarray(cb.payload).tobytes() == want.tobytes(), k
        assert H.decompress(cb).tobytes() == x.tobytes(), k
        xd = torch.from_numpy(x).cuda()
        cbd = H.compress(_spec(), xd)
        assert cbd.payload.cpu().numpy().tobytes() == want.tobytes(), k
        assert H.decompress(cbd).cpu().numpy().tobytes() == x.tobytes(), k
        # decode the reference's own payload
        cbr = H.CompressedBuffer(_spec(), x.size, int(g[k + "_cc"][0]), want.copy())
        assert H.decompress(cbr).tobytes() == x.tobytes(), k


@pytest.mark.parametrize("n", [0, 1, 63, 4096, 4097, 10000, 1 << 20])
@pytest.mark.parametrize("mode", ["bits", "sparse", "uniform", "normal"])
def test_vs_oracle(cuda, n, mode):
    import paper_2409_02423_b200 as H
    from paper_2409_02423_b200 import lossless

    x = O.fill(n * 7 + len(mode), mode, n, {"sparse": 0.9, "normal": 1e-3}.get(mode, -1.0), 1.0)
    want = O.pred_compress(x)
    cb = H.compress(_spec(), x)
    assert np.asarray(cb.payload).tobytes() == want.tobytes()
    assert H.decompress(cb).tobytes() == x.tobytes()
    if n:
        assert lossless.size(x) == want.size


def test_reference_codec_cases(cuda):
    import paper_2409_02423_b200 as H
    from paper_2409_02423_b200.errors import CorruptPayloadError

    # test_codec.cpp:70-80: constant chunk -> 3077 bytes
    cb = H.compress(_spec(), np.full(4096, 1.0, np.float32))
    assert cb.payload_bytes() == 3077
    # :82-93 fallback safety bound
    for n in (4096, 3 * 4096 + 17):
        x = O.fill(12 + n, "bits", n)
        assert H.compress(_spec(), x).payload_bytes() <= 4 * n + ((n + 4095) // 4096 + 7) // 8
    # :95-100 sparse beats dense
    sp = H.compress(_spec(), O.fill(13, "sparse", 1 << 16, 0.9, 0))
    de = H.compress(_spec(), O.fill(14, "uniform", 1 << 16))
    assert sp.payload_bytes() < de.payload_bytes()
    # :237-239 truncated payload -> CorruptPayloadError
    cb = H.compress(_spec(), O.fill(15, "uniform", 4096))
    cut = H.CompressedBuffer(_spec(), 4096, cb.chunk_count, np.asarray(cb.payload)[: cb.payload_bytes() // 2].copy())
    with pytest.raises(CorruptPayloadError):
        H.decompress(cut)
    # truncated coded chunk (sparse data)
    cb = H.compress(_spec(), O.fill(16, "sparse", 3 * 4096, 0.9, 0))
    for keep in (1, 2, cb.payload_bytes() - 1):
        cut = H.CompressedBuffer(_spec(), 3 * 4096, cb.chunk_count, np.asarray(cb.payload)[:keep].copy())
        with pytest.raises(CorruptPayloadError):
            H.decompress(cut)
    # wrong chunk count -> CorruptPayloadError (codec_serial.cpp:91-93)
    with pytest.raises(CorruptPayloadError):
        H.decompress(H.CompressedBuffer(_spec(), 4096, 2, np.asarray(cb.payload).copy()))
    # trailing bytes are ignored, as in the reference
    x = O.fill(17, "sparse", 5000, 0.9, 0)
    cb = H.compress(_spec(), x)
    longer = H.CompressedBuffer(_spec(), 5000, cb.chunk_count, np.concatenate([np.asarray(cb.payload),
                                                                               np.zeros(9, np.uint8)]))
    assert H.decompress(longer).tobytes() == x.tobytes()


def test_large_mixed_chunks(cuda):
    """2^24 values alternating coded / raw-fallback chunks, device in/out."""
    import torch

    import paper_2409_02423_b200 as H

    n = 1 << 24
    a = O.fill(21, "sparse", n, 0.95, 0)
    b = O.fill(22, "bits", n)
    x = np.where((np.arange(n) // 4096) % 3 == 1, b, a).astype(np.float32)
    want = O.pred_compress(x)
    xd = torch.from_numpy(x).cuda()
    cb = H.compress(_spec(), xd)
    assert cb.payload_bytes() == want.size
    assert torch.equal(cb.payload.cpu(), torch.from_numpy(want))
    assert torch.equal(H.decompress(cb).view(torch.int32), xd.view(torch.int32))


def test_collectives_golden_accounting(cuda):
    """hcc::allreduce / ring_reduce_scatter / ring_allgather / p2p with the
    lossless codec: values bit-identical and TraceEvent bytes equal to the
    reference's (golden accounting from the reference library)."""
    from paper_2409_02423_b200 import collectives as K
    from paper_2409_02423_b200.comm_path import CommPath
    from paper_2409_02423_b200.netsim import SimClock, Topology

    g = np.load(GOLD)
    for k in sorted(k[:-3] for k in g.files if k.endswith("_rs") and k.startswith("p")):
        x = g[k + "_in"]
        p = x.shape[0]
        comm = K.Communicator(list(range(p)))
        for avg in (0, 1):
            clock = SimClock(Topology.b200_box(max(p, 2)))
            out = K.allreduce(clock, comm, list(x), _spec(), CommPath.DpAllReduce, K.ReduceMode(avg))
            assert np.stack(out).tobytes() == g[f"{k}_ar{avg}"].tobytes(), k
            ev = clock.trace()[-1]
            assert (ev.raw_bytes, ev.wire_bytes, ev.round_count) == tuple(int(v) for v in g[f"{k}_ar{avg}_acct"]), k
        clock = SimClock(Topology.b200_box(max(p, 2)))
        out = K.ring_reduce_scatter(clock, comm, list(x), _spec(), CommPath.Zero1ReduceScatter)
        assert np.stack(out).tobytes() == g[k + "_rs"].tobytes(), k
        ev = clock.trace()[-1]
        assert (ev.raw_bytes, ev.wire_bytes, ev.round_count) == tuple(int(v) for v in g[k + "_rs_acct"]), k
        shards = [np.ascontiguousarray(r[: x.shape[1] // p]) for r in x]
        out = K.ring_allgather(clock, comm, shards, _spec(), CommPath.Zero1AllGather)
        assert np.stack(out).tobytes() == g[k + "_ag"].tobytes(), k
        ev = clock.trace()[-1]
        assert (ev.raw_bytes, ev.wire_bytes, ev.round_count) == tuple(int(v) for v in g[k + "_ag_acct"]), k
        got = K.p2p(clock, 0, 1, x[1], _spec(), CommPath.PpP2p)
        assert got.tobytes() == x[1].tobytes()
        ev = clock.trace()[-1]
        assert (ev.raw_bytes, ev.wire_bytes, ev.round_count) == tuple(int(v) for v in g[k + "_p2p_acct"]), k


@pytest.mark.parametrize("p", [2, 3, 4, 8])
def test_collectives_vs_oracle(cuda, p):
    from paper_2409_02423_b200 import collectives as K
    from paper_2409_02423_b200.comm_path import CommPath
    from paper_2409_02423_b200.netsim import SimClock, Topology

    n = p * 6000
    x = np.stack([O.fill(40 + j, "sparse" if j % 2 else "normal", n, 0.7 if j % 2 else 1e-3, 1.0) for j in range(p)])
    comm = K.Communicator(list(range(p)))
    clock = SimClock(Topology.b200_box(8))
    out = K.allreduce(clock, comm, list(x), _spec(), CommPath.DpAllReduce, K.ReduceMode.Average)
    want, acct = O.allreduce(x, "lossless", 0, True)
    assert np.stack(out).tobytes() == want.tobytes()
    ev = clock.trace()[-1]
    assert (ev.raw_bytes, ev.wire_bytes, ev.round_count) == acct
    # lossless transparency (test_collectives.cpp:189-203)
    ident = K.allreduce(clock, comm, list(x), H_identity(), CommPath.DpAllReduce, K.ReduceMode.Average)
    assert np.stack(ident).tobytes() == np.stack(out).tobytes()
    assert clock.trace()[-1].raw_bytes == ev.raw_bytes


def H_identity():
    import paper_2409_02423_b200 as H

    return H.CodecSpec.identity()


@pytest.mark.parametrize("n", [1, 4095, 4096, 4097, 3 * 4096 + 17, 1 << 18])
@pytest.mark.parametrize("mode", ["bits", "sparse", "normal", "smooth"])
def test_frame_messages(cuda, n, mode):
    """The communicator's framed message (lossless_msg.h): payload section
    byte-identical to the oracle (= hcc::compress), HCC1 header fields, exact
    decode, folded decode (acc + value, IEEE), and the device-side checks
    (hcc::from_bytes' magic / lengths, index vs payload) -> CORRUPT."""
    import torch

    from paper_2409_02423_b200 import _lib

    if mode == "smooth":
        x = np.cumsum(O.fill(n + 5, "normal", n, 1e-3, 1.0)).astype(np.float32)
    else:
        x = O.fill(n * 3 + len(mode), mode, n, {"sparse": 0.9, "normal": 1e-3}.get(mode, -1.0), 1.0)
    want = O.pred_compress(x)
    cap = int(_lib.hccx_lossless_frame_max_bytes(n))
    msg = torch.zeros(cap, dtype=torch.uint8, device="cuda")
    xd = torch.from_numpy(x).cuda()
    assert _lib.hccx_lossless_frame_encode(xd.data_ptr(), n, msg.data_ptr(), cap, None) == 0
    m = msg.cpu().numpy()
    nch = (n + 4095) // 4096
    ib = (132 * nch + 15) // 16 * 16
    container = int(m[:8].view(np.uint64)[0])
    assert container == 18 + want.size
    assert m[8:12].tobytes() == b"HCC1" and m[12] == 1 and m[13] == 0
    assert int(m[14:22].view(np.uint64)[0]) == n and int(m[22:26].view(np.uint32)[0]) == nch
    assert m[32 + ib:32 + ib + want.size].tobytes() == want.tobytes()
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    assert _lib.hccx_lossless_frame_decode(msg.data_ptr(), cap, n, out.data_ptr(), 0, None) == 0
    assert _lib.hccx_frame_status(None) == 0
    assert out.cpu().numpy().tobytes() == x.tobytes()
    if mode != "bits":  # (NaN payloads are not IEEE-specified through an add)
        acc = O.fill(n + 11, "normal", n, 1.0, 1.0)
        acc_d = torch.from_numpy(acc).cuda()
        assert _lib.hccx_lossless_frame_decode(msg.data_ptr(), cap, n, acc_d.data_ptr(), 1, None) == 0
        assert _lib.hccx_frame_status(None) == 0
        assert acc_d.cpu().numpy().tobytes() == (acc + x).astype(np.float32).tobytes()
    # corruptions: each must be reported, never hang or fault
    bad = []
    b = m.copy(); b[9] = ord("X"); bad.append(b)                                 # magic
    b = m.copy(); b[14:22] = np.array([n + 1], np.uint64).view(np.uint8); bad.append(b)  # original_len
    b = m.copy(); b[:8] = np.array([cap * 2], np.uint64).view(np.uint8); bad.append(b)   # container > capacity
    if nch > 1:
        b = m.copy(); b[32 + 132:32 + 136] = np.array([container * 4], np.uint32).view(np.uint8); bad.append(b)
    coded = [c for c in range(nch) if not (want[c // 8] >> (c % 8)) & 1]
    if coded:
        c = coded[0]
        b = m.copy()
        lane0 = 32 + 132 * c + 4
        b[lane0:lane0 + 2] = (np.frombuffer(b[lane0:lane0 + 2].tobytes(), np.uint16) + 8).view(np.uint8)
        bad.append(b)
    for b in bad:
        bm = torch.from_numpy(b).cuda()
        assert _lib.hccx_lossless_frame_decode(bm.data_ptr(), cap, n, out.data_ptr(), 0, None) == 0
        assert _lib.hccx_frame_status(None) == 2  # HCCX_ERR_CORRUPT_PAYLOAD


@pytest.mark.parametrize("mode", ["smooth", "sparse"])
def test_decompress_multislab(cuda, mode):
    """Reference-format payloads large enough for several doubling slabs
    (csrc/lossless.cu: 64 Mi stream bits per slab) and the F^64-anchored
    chunk walk: the bare payload (no offsets) decodes to the input bit for
    bit, and a truncated payload is reported, not mis-decoded."""
    import ctypes as C

    import torch

    from paper_2409_02423_b200 import _lib

    n = 1 << 24 if mode == "smooth" else 1 << 23  # ~101 M / ~200 M stream bits
    if mode == "smooth":
        t = torch.arange(n, device="cuda", dtype=torch.float32)
        x = ((torch.sin(t * 1e-4) * 1e-2) * 4096).round() / 4096
    else:
        g = torch.Generator(device="cuda").manual_seed(7)
        x = torch.randn(n, device="cuda", generator=g) * (torch.rand(n, device="cuda", generator=g) < 0.1)
    cap = int(_lib.hccx_lossless_max_bytes(n))
    pay = torch.empty(cap, dtype=torch.uint8, device="cuda")
    nb = C.c_uint64()
    assert _lib.hccx_lossless_compress(x.data_ptr(), n, pay.data_ptr(), cap, C.byref(nb), None) == 0
    assert 8 * nb.value > (64 << 20)  # more than one slab
    y = torch.empty(n, device="cuda")
    assert _lib.hccx_lossless_decompress(pay.data_ptr(), nb.value, n, y.data_ptr(), None) == 0
    assert torch.equal(y.view(torch.int32), x.view(torch.int32))
    # truncated: CorruptPayloadError (codec_serial.cpp:98-101)
    assert _lib.hccx_lossless_decompress(pay.data_ptr(), nb.value // 2, n, y.data_ptr(), None) == 2
