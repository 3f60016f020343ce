"""The NVLink engine's kernels on ONE GPU: virtual ranks vs the CPU oracle.

`hccx_mcomm` with every member on cuda:0 runs ring_fused_kernel /
oneshot_allreduce_kernel device code (phases, per-segment flags, consumption
acks, TMA bulk pushes into the peer windows, signaller releases) with the p
ranks sharing one cooperative grid -- the same code that runs one rank per
GPU over NVLink.  Bar: bit-exact against the oracle restatement of
proj/src/collectives.cpp:27-111 (ring), :202-248 (allreduce), :130-152 (p2p)
and the broadcast definition of SURVEY.md §8 a10.

Paths are steered per call with HCCX_ONESHOT_BYTES (0: ring everywhere),
HCCX_LL_BYTES (one-shot transport: pairs below, flags above) and
HCCX_AG_RING_BYTES (0: forwarding-ring gather; huge: direct owner pushes).
"""
import os

import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu

CODECS = [("identity", 0), ("fixed-rate", 3), ("fixed-rate", 4), ("fixed-rate", 8), ("fixed-rate", 16),
          ("fixed-rate", 24), ("fixed-rate", 32), ("zfp-rate", 8), ("zfp-rate", 16)]


@pytest.fixture
def env():
    saved = {k: os.environ.get(k) for k in ("HCCX_ONESHOT_BYTES", "HCCX_AG_RING_BYTES", "HCCX_LL_BYTES")}

    def set_(oneshot=None, ag_ring=None, ll=None):
        for k, v in (("HCCX_ONESHOT_BYTES", oneshot), ("HCCX_AG_RING_BYTES", ag_ring), ("HCCX_LL_BYTES", ll)):
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = str(v)

    yield set_
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def _inputs(seed, p, n, mode="uniform"):
    return np.stack([O.fill(seed + 31 * j, mode, n, 1e-3 if mode == "normal" else -1.0, 1.0) for j in range(p)])


MODES = {"ring-direct": (0, 1 << 62), "ring-fwd": (0, 0), "oneshot-ll": (1 << 40, None, 1 << 40),
         "oneshot-flags": (1 << 40, None, 0)}


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("kind,rate", CODECS)
def test_allreduce_virtual(cuda, env, p, mode, kind, rate):
    import hccx_util as U

    env(*MODES[mode])
    m = U.MComm(p, 1 << 20)
    for n_per in (64, 100, 1000, 6144 + 64, 40000):  # partial groups / segments, unaligned chunks
        n = n_per * p
        x = _inputs(p * 1000 + n_per + rate, p, n)
        for avg in (False, True):
            got, st = m.allreduce(x, kind, rate, avg)
            assert st == 0
            want, _ = O.allreduce(x, kind, rate, avg)
            assert got.tobytes() == want.tobytes(), (p, mode, kind, rate, n, avg)


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("mode", ["ring-direct", "ring-fwd"])
@pytest.mark.parametrize("kind,rate", CODECS)
def test_reduce_scatter_allgather_virtual(cuda, env, p, mode, kind, rate):
    import hccx_util as U

    env(*MODES[mode])
    m = U.MComm(p, 1 << 20)
    for n_per in (64, 300, 6144 * 3 + 256):
        n = n_per * p
        x = _inputs(p * 77 + n_per + rate, p, n)
        got, st = m.reduce_scatter(x, kind, rate)
        assert st == 0
        want, _ = O.reduce_scatter(x, kind, rate)
        assert got.tobytes() == want.tobytes(), (p, kind, rate, n)
        s = np.ascontiguousarray(x[:, :n_per])
        got, st = m.allgather(s, kind, rate)
        assert st == 0
        want, _ = O.allgather(s, kind, rate)
        assert got.tobytes() == want.tobytes(), (p, kind, rate, n_per)


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("kind,rate", [("identity", 0), ("fixed-rate", 8), ("fixed-rate", 16), ("zfp-rate", 12)])
def test_broadcast_p2p_virtual(cuda, p, kind, rate):
    import hccx_util as U

    m = U.MComm(p, 1 << 16)  # slot of 2^16 / p values: larger messages go in passes
    for n in (1, 100, 6144 + 5, 70000):
        x = O.fill(n + rate, "uniform", n)
        for root in sorted({0, p - 1, p // 2}):
            got, st = m.broadcast(x, root, kind, rate)
            assert st == 0
            want, _ = O.broadcast(x, p, kind, rate)
            assert got.tobytes() == want.tobytes(), (p, root, kind, rate, n)
        for src, dst in ((0, 1), (p - 1, 0), (1, p - 1)):
            if src == dst:
                continue
            got, st = m.p2p(x, kind, rate, src, dst)
            assert st == 0
            want, _ = O.p2p(x, kind, rate)
            assert got.tobytes() == want.tobytes(), (p, src, dst, kind, rate, n)


@pytest.mark.parametrize("p", [2, 4, 8])
def test_large_allreduce_virtual(cuda, env, p):
    """Multi-step phases: more segments per CTA than one step, ring and
    forwarding gather, r8 and r4, Average."""
    import hccx_util as U

    env(0, 0)
    n = (1 << 21) * p // p * p  # 2^21 values per rank
    m = U.MComm(p, n)
    x = _inputs(4242 + p, p, n, "normal")
    for rate, avg in ((8, True), (4, False)):
        got, st = m.allreduce(x, "fixed-rate", rate, avg)
        assert st == 0
        want, _ = O.allreduce(x, "fixed-rate", rate, avg)
        assert got.tobytes() == want.tobytes(), (p, rate, avg)


def test_back_to_back_geometry_changes(cuda, env):
    """Consecutive collectives on the same slots with different codecs and
    chunk sizes, no host synchronisation between them (the consumption-ack
    credits must cover every receiver CTA when the slot geometry changes)."""
    import torch

    import hccx_util as U
    from paper_2409_02423_b200 import _lib

    p = 4
    env(0, 0)
    m = U.MComm(p, 1 << 22)
    rng = np.random.default_rng(5)
    plan = [("reduce_scatter", "fixed-rate", 4, 1 << 20), ("reduce_scatter", "identity", 0, 1 << 20),
            ("allgather", "identity", 0, 1 << 18), ("allreduce", "fixed-rate", 8, 3 << 19),
            ("allreduce", "fixed-rate", 16, 1 << 16), ("allgather", "fixed-rate", 8, 5000),
            ("reduce_scatter", "zfp-rate", 8, 1 << 21), ("allreduce", "identity", 0, 1 << 20)]
    jobs = []
    for op, kind, rate, n in plan:
        x = _inputs(int(rng.integers(1 << 30)), p, n)
        ins = [U.dev(x[j]) for j in range(p)]
        out_n = n // p if op == "reduce_scatter" else (n * p if op == "allgather" else n)
        outs = [torch.full((out_n,), float("nan"), device="cuda:0") for _ in range(p)]
        a, ka = _lib.ptr_array([t.data_ptr() for t in ins])
        b, kb = _lib.ptr_array([t.data_ptr() for t in outs])
        fn = {"allreduce": _lib.hccx_mcomm_allreduce, "reduce_scatter": _lib.hccx_mcomm_reduce_scatter,
              "allgather": _lib.hccx_mcomm_allgather}[op]
        tail = (U.codec(kind, rate), 0) if op == "allreduce" else (U.codec(kind, rate),)
        assert fn(m.h, a, b, n, *tail, None) == 0
        jobs.append((op, kind, rate, x, outs, (ins, ka, kb)))
    assert _lib.hccx_mcomm_status(m.h, None) == 0
    for op, kind, rate, x, outs, _keep in jobs:
        got = np.stack([t.cpu().numpy() for t in outs])
        want, _ = getattr(O, op)(x, kind, rate)
        assert got.tobytes() == want.tobytes(), (op, kind, rate, x.shape)


def test_host_api_virtual(cuda):
    """hccx_mcomm_*_host: the reference's value API (host vectors) through
    the NVLink engine's kernels, cached device buffers."""
    import ctypes as C

    import hccx_util as U
    from paper_2409_02423_b200 import _lib

    p, n = 4, 4 * 5000
    m = U.MComm(p, n)
    x = _inputs(99, p, n)
    outs = [np.full(n, np.nan, np.float32) for _ in range(p)]
    a, _ka = _lib.ptr_array([r.ctypes.data for r in x])
    b, _kb = _lib.ptr_array([o.ctypes.data for o in outs])
    secs = C.c_double()
    for _ in range(2):
        assert _lib.hccx_mcomm_allreduce_host(m.h, a, b, n, U.codec("fixed-rate", 8), 1, C.byref(secs)) == 0
        want, _ = O.allreduce(x, "fixed-rate", 8, True)
        assert np.stack(outs).tobytes() == want.tobytes()
    assert secs.value > 0


def test_nonfinite_virtual(cuda):
    import hccx_util as U

    m = U.MComm(2, 4096)
    x = _inputs(3, 2, 4096)
    x[1, 77] = np.inf
    _got, st = m.allreduce(x, "fixed-rate", 8)
    assert st == 1  # HCCX_ERR_NONFINITE (proj/src/codec_omp.cpp:45)
    x[1, 77] = 0.5
    _got, st = m.allreduce(x, "fixed-rate", 8)
    assert st == 0


def _ngpus():
    import torch

    return torch.cuda.device_count()


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("layout", ["one-per-gpu", "two-per-gpu", "eight-ranks"])
def test_single_process_multi_gpu(cuda, env, layout):
    """hccx_mcomm over distinct GPUs (peer access over NVLink), including a
    ring whose neighbours alternate between GPUs with two virtual ranks per
    GPU, and the p = 8 ring (north_star's rank count) over every GPU of the
    box (two ranks per GPU on a 4-GPU box), vs the oracle."""
    import hccx_util as U

    g = min(_ngpus(), 4)
    if layout == "one-per-gpu":
        devices = list(range(g))
    elif layout == "two-per-gpu":
        devices = [j % 2 for j in range(4)]
    else:
        devices = [j * g // 8 for j in range(8)]
    p = len(devices)
    m = U.MComm(p, max(1 << 21, p * ((1 << 19) + 256)), devices)
    for mode in ("ring-fwd", "ring-direct", "oneshot-ll", "oneshot-flags"):
        env(*MODES[mode])
        for n_per, kind, rate in ((1000, "fixed-rate", 8), (6144 * 5 + 64, "fixed-rate", 4),
                                  ((1 << 19) + 256, "identity", 0)):
            n = n_per * p
            x = _inputs(n_per + rate, p, n)
            got, st = m.allreduce(x, kind, rate, True)
            assert st == 0
            want, _ = O.allreduce(x, kind, rate, True)
            assert got.tobytes() == want.tobytes(), (layout, mode, n, kind, rate)
    x = O.fill(7, "uniform", 100000)
    got, st = m.broadcast(x, p - 1, "fixed-rate", 16)
    assert st == 0
    assert got.tobytes() == O.broadcast(x, p, "fixed-rate", 16)[0].tobytes()
    got, st = m.p2p(x, "fixed-rate", 8, 0, p - 1)
    assert st == 0
    assert got.tobytes() == O.p2p(x, "fixed-rate", 8)[0].tobytes()
    # LosslessPredictor framed messages across devices (per-device kernel
    # attributes, peer-window encodes)
    for n_per in (1000, 4096 * 3 + 17):
        x = _inputs(n_per + 3, p, n_per * p)
        got, st = m.allreduce(x, "lossless", 0)
        assert st == 0
        want, _ = O.allreduce(x, "lossless", 0)
        assert got.tobytes() == want.tobytes(), (layout, n_per)
        s = np.ascontiguousarray(x[:, :n_per])
        got, st = m.allgather(s, "lossless")
        assert st == 0
        assert got.tobytes() == O.allgather(s, "lossless")[0].tobytes()
        v = np.ascontiguousarray(x[0])
        got, st = m.broadcast(v, p - 1, "lossless")
        assert st == 0
        assert got.tobytes() == O.broadcast(v, p, "lossless")[0].tobytes()
        got, st = m.p2p(v, "lossless", 0, p - 1, 0)
        assert st == 0
        assert got.tobytes() == O.p2p(v, "lossless")[0].tobytes()


@pytest.mark.parametrize("p", [2, 3, 4])
def test_lossless_on_the_wire_virtual(cuda, p):
    """LosslessPredictor collectives through the engine's framed messages
    (csrc/lossless_comm.cu): values exact (the oracle), and the payload bytes
    each member actually pushed sum to the reference's wire accounting
    (collectives.cpp:113-126, total / p)."""
    import ctypes as C

    import hccx_util as U
    from paper_2409_02423_b200 import _lib

    m = U.MComm(p, 1 << 18)

    def pushed():
        tot = 0
        for j in range(p):
            a, b = C.c_uint64(), C.c_uint64()
            assert _lib.hccx_mcomm_wire_bytes(m.h, j, C.byref(a), C.byref(b)) == 0
            assert b.value >= a.value
            tot += a.value
        return tot

    for n_per, mode in ((1000, "sparse"), (4096 * 3 + 17, "normal"), (20000, "uniform")):
        n = n_per * p
        x = _inputs(n_per + p, p, n, mode if mode != "sparse" else "uniform")
        if mode == "sparse":
            x[:, ::3] = 0.0
        for avg in (False, True):
            got, st = m.allreduce(x, "lossless", 0, avg)
            assert st == 0
            want, acct = O.allreduce(x, "lossless", 0, avg)
            assert got.tobytes() == want.tobytes(), (p, n, avg)
            assert pushed() // p == acct[1], (p, n, avg, pushed(), acct)
        got, st = m.reduce_scatter(x, "lossless")
        assert st == 0
        want, acct = O.reduce_scatter(x, "lossless")
        assert got.tobytes() == want.tobytes()
        assert pushed() // p == acct[1]
        s = np.ascontiguousarray(x[:, :n_per])
        got, st = m.allgather(s, "lossless")
        assert st == 0
        want, acct = O.allgather(s, "lossless")
        assert got.tobytes() == want.tobytes()
        assert pushed() // p == acct[1]
        v = np.ascontiguousarray(x[0])
        got, st = m.broadcast(v, p - 1, "lossless")
        assert st == 0
        assert got.tobytes() == O.broadcast(v, p, "lossless")[0].tobytes()
        got, st = m.p2p(v, "lossless", 0, 0, p - 1)
        assert st == 0
        want, acct = O.p2p(v, "lossless")
        assert got.tobytes() == want.tobytes()
        assert pushed() == acct[1]


def test_lossless_then_fused_same_slots(cuda, env):
    """A lossless collective (framed messages, all-index acks) followed by
    fused-kernel collectives on the same slots and back, no host sync."""
    import hccx_util as U

    p = 4
    env(0, 0)
    m = U.MComm(p, 1 << 20)
    for kind, rate, n_per in (("fixed-rate", 8, 1 << 18), ("lossless", 0, 5000), ("fixed-rate", 4, 70000),
                              ("lossless", 0, 1 << 18), ("identity", 0, 1 << 17)):
        x = _inputs(n_per + rate, p, n_per * p)
        got, st = m.allreduce(x, kind, rate)
        assert st == 0
        want, _ = O.allreduce(x, kind, rate)
        assert got.tobytes() == want.tobytes(), (kind, rate, n_per)


def test_edge_cases_virtual(cuda):
    """Degenerate calls of the single-process communicator, as the
    reference's wrappers treat them (collectives.cpp:154-200): empty buffers,
    a one-member communicator (input returned untouched, not quantized),
    ragged / indivisible lengths (BadChunkingError), bad roots and src == dst."""
    import ctypes as C

    import torch

    import hccx_util as U
    from paper_2409_02423_b200 import _lib

    m = U.MComm(4, 1 << 14)
    # n = 0: nothing happens, no error
    z = torch.empty(0, device="cuda")
    a, _ka = _lib.ptr_array([z.data_ptr()] * 4)
    assert _lib.hccx_mcomm_allreduce(m.h, a, a, 0, U.codec("fixed-rate", 8), 0, None) == 0
    assert _lib.hccx_mcomm_status(m.h, None) == 0
    # n % p != 0 -> HCCX_ERR_BAD_CHUNKING (4)
    x = _inputs(1, 4, 4 * 100 + 2)
    ins = [U.dev(x[j]) for j in range(4)]
    a, _ka = _lib.ptr_array([t.data_ptr() for t in ins])
    assert _lib.hccx_mcomm_allreduce(m.h, a, a, 4 * 100 + 2, U.codec("fixed-rate", 8), 0, None) == 4
    assert _lib.hccx_mcomm_reduce_scatter(m.h, a, a, 4 * 100 + 2, U.codec("fixed-rate", 8), None) == 4
    # bad root / src == dst -> HCCX_ERR_INVALID_ARGUMENT (9); bad rate -> INVALID_SCHEME (6)
    assert _lib.hccx_mcomm_broadcast(m.h, 4, ins[0].data_ptr(), a, 100, U.codec("fixed-rate", 8), None) == 9
    assert _lib.hccx_mcomm_p2p(m.h, 1, 1, ins[0].data_ptr(), ins[1].data_ptr(), 100, U.codec("fixed-rate", 8),
                               None) == 9
    assert _lib.hccx_mcomm_allreduce(m.h, a, a, 400, U.codec("fixed-rate", 33), 0, None) == 6
    # one-member communicator: the input comes back untouched (not quantized)
    one = U.MComm(1, 4096)
    x1 = _inputs(2, 1, 3000)
    got, st = one.allreduce(x1, "fixed-rate", 4)
    assert st == 0 and got.tobytes() == x1.tobytes()
    # capacity: more values per chunk than the communicator was created for
    big = _inputs(3, 4, 4 * (1 << 16))
    _got, st = m.allreduce(big, "fixed-rate", 8)
    assert st == 9
    del C
