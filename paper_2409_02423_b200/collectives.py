"""Compressed ring collectives with the reference's all-members-in-one-call API.

Drop-in for proj/include/hcc/collectives.hpp:15-64 (implementation
proj/src/collectives.cpp): ``inputs[j]`` is the buffer of communicator
position j and one buffer per member is returned.  Every call runs on the
NVLink engine's single-process communicator (libhccx, hccx_mcomm_*): members
whose CUDA tensors live on distinct GPUs exchange compressed segments over
NVLink, members sharing a GPU (host inputs, or tensors on one device) are
virtual ranks of one cooperative launch of the same fused kernels.  Results
are bit-identical to the reference ring:

  reduce_scatter  position i holds chunk i folded in ring order (i+1 ... i+p),
                  decompress-add-recompress at every hop (collectives.cpp:27-66)
  allgather       each shard compressed once, every member (origin included)
                  keeps the decoded copy (collectives.cpp:69-111)
  allreduce       RS then AG; Average = IEEE divide by float(p) after the gather
                  (collectives.cpp:202-248)
  p2p             dst receives dec(comp(buf)) (collectives.cpp:130-152)
  broadcast       NOT in the reference: every member, root included, receives
                  dec(comp(buf))

Byte accounting (TraceEvent raw/wire bytes, round counts) is integer-identical
to the reference and ``duration_s`` is the reference's cost model
(collectives.cpp:53-62, :97-107); ``device_s`` is the measured device time of
the call.  Inputs may be host numpy float32 arrays (copied to the device and
back, like the reference's value semantics) or CUDA float32 tensors.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import Dict, List, Sequence, Tuple

import numpy as np

from .codec import CodecKind, CodecSpec, wire_size_bytes
from .comm_path import CommPath
from .errors import BadChunkingError, check
from .netsim import CollectiveKind, SimClock, TraceEvent, codec_time, link_class, transfer_time


@dataclass
class Communicator:
    """Ordered member list: ring orientation and reduction order (collectives.hpp:15-19)."""

    ranks: List[int] = field(default_factory=list)

    def size(self) -> int:
        return len(self.ranks)


class ReduceMode(enum.IntEnum):
    Sum = 0
    Average = 1


_MCOMMS: Dict[Tuple[int, ...], Tuple[int, int]] = {}


def _mcomm(devices: Tuple[int, ...], max_n: int) -> int:
    """Single-process communicator for this member -> device map, grown on
    demand (include/hccx.h hccx_mcomm_create)."""
    import ctypes as C

    from . import _lib

    h, cap = _MCOMMS.get(devices, (None, 0))
    if h is not None and cap >= max_n:
        return h
    if h is not None:
        _torch().cuda.synchronize()
        _lib.hccx_mcomm_destroy(h)
    cap = max(max_n, 2 * cap, 1 << 16)
    out = C.c_void_p()
    arr = (C.c_int * len(devices))(*devices)
    check(_lib.hccx_mcomm_create(len(devices), arr, cap, C.byref(out)), "mcomm_create")
    _MCOMMS[devices] = (out.value, cap)
    return out.value


def _torch():
    import torch

    return torch


def _is_cuda(x) -> bool:
    return hasattr(x, "is_cuda") and bool(x.is_cuda)


def _as_device(bufs: Sequence) -> Tuple[list, bool, Tuple[int, ...]]:
    """-> (contiguous CUDA float32 tensors, inputs_were_host, member devices)."""
    torch = _torch()
    if all(_is_cuda(b) for b in bufs):
        ts = [b.contiguous().view(-1) for b in bufs]
        return ts, False, tuple(t.device.index for t in ts)
    dev = torch.cuda.current_device()
    ts = [torch.from_numpy(np.ascontiguousarray(b, np.float32).reshape(-1)).to(f"cuda:{dev}") for b in bufs]
    return ts, True, tuple(dev for _ in ts)


def _back(ts: list, host: bool) -> list:
    if not host:
        return ts
    return [t.cpu().numpy() for t in ts]


def _message_bytes(spec: CodecSpec, n: int) -> int:
    """Payload bytes of one n-value message (size law; lossless -> use the
    data-dependent helpers below)."""
    return wire_size_bytes(spec, n)


def _lossless(spec: CodecSpec) -> bool:
    return spec.kind == CodecKind.LosslessPredictor


def _lossless_hops(ts: list, n: int, collective: int, stream) -> List[int]:
    """Per-message payload bytes under LosslessPredictor, whose sizes are
    data-dependent: hccx_lossless_ring_hops sizes every hop's message on the
    device (collective 0 = reduce-scatter partial folds, hop[t*p + j];
    1 = allgather shards, hop[j]; 2 = allreduce, both)."""
    import ctypes as C

    from . import _lib

    p = len(ts)
    arr, _keep = _ptrs(ts)
    out = (C.c_uint64 * (p * p + p))()
    check(_lib.hccx_lossless_ring_hops(arr, p, n, collective, out, stream.cuda_stream), "lossless wire accounting")
    return [int(v) for v in out]


class _Cost:
    """The reference's PhaseCost (collectives.cpp:9-14) and its ring cost
    passes: every round lasts as long as its slowest hop."""

    def __init__(self):
        self.duration = 0.0
        self.raw_total = 0
        self.wire_total = 0
        self.rounds = 0

    @staticmethod
    def rs(clock: SimClock, comm: Communicator, spec: CodecSpec, chunk: int, msg) -> "_Cost":
        """collectives.cpp:34-64; msg(round, j) = payload member j sends."""
        t, p, raw = clock.topology(), comm.size(), 4 * chunk
        c = _Cost()
        for rnd in range(p - 1):
            round_dur = 0.0
            for j in range(p):
                w = msg(rnd, j)
                hop = codec_time(t, raw, spec) + transfer_time(
                    t, w, link_class(t, comm.ranks[j], comm.ranks[(j + 1) % p])) + codec_time(t, raw, spec)
                round_dur = max(round_dur, hop)
                c.raw_total += raw
                c.wire_total += w
            c.duration += round_dur
        c.rounds = p - 1
        return c

    @staticmethod
    def ag(clock: SimClock, comm: Communicator, spec: CodecSpec, chunk: int, shard) -> "_Cost":
        """collectives.cpp:93-109; shard(c) = payload of shard c."""
        t, p, raw = clock.topology(), comm.size(), 4 * chunk
        c = _Cost()
        for rnd in range(p - 1):
            round_dur = 0.0
            for j in range(p):
                w = shard((j - rnd) % p)
                hop = transfer_time(t, w, link_class(t, comm.ranks[j], comm.ranks[(j + 1) % p])) + codec_time(
                    t, raw, spec)
                if rnd == 0:
                    hop += codec_time(t, raw, spec)
                round_dur = max(round_dur, hop)
                c.raw_total += raw
                c.wire_total += w
            c.duration += round_dur
        c.rounds = p - 1
        return c


def _commit(clock: SimClock, comm: Communicator, cost: _Cost, device_s: float, path: CommPath,
            kind: CollectiveKind) -> None:
    """collectives.cpp:113-126, plus the measured device time."""
    clock.sync_to_max(comm.ranks)
    for r in comm.ranks:
        clock.advance(r, cost.duration)
    p = comm.size()
    clock.record(TraceEvent(0, path, kind, p, cost.raw_total // p, cost.wire_total // p, cost.duration,
                            cost.rounds, device_s))


def _ptrs(ts: list):
    from . import _lib

    return _lib.ptr_array([t.data_ptr() for t in ts])


def _finish(m: int, what: str) -> None:
    from . import _lib

    check(_lib.hccx_mcomm_status(m, None), what)


def _run(devs, max_n: int, what: str, fn) -> float:
    """Run one mcomm collective on the legacy default streams of its devices;
    returns the device seconds (events on the first member's device, every
    member device synchronised)."""
    torch = _torch()
    m = _mcomm(devs, max_n)
    for d in set(devs):
        torch.cuda.synchronize(d)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    legacy = torch.cuda.default_stream(devs[0])
    a.record(legacy)
    check(fn(m), what)
    for d in set(devs):
        torch.cuda.synchronize(d)
    b.record(legacy)
    _finish(m, what)
    return a.elapsed_time(b) / 1e3


def ring_reduce_scatter(clock: SimClock, comm: Communicator, inputs: Sequence, spec: CodecSpec,
                        path: CommPath) -> list:
    """collectives.cpp:154-181."""
    from . import _lib

    p = comm.size()
    assert len(inputs) == p
    n = len(inputs[0])
    if n % p != 0:
        raise BadChunkingError(f"reduce_scatter: length {n} not divisible by {p}")
    if any(len(b) != n for b in inputs):
        raise BadChunkingError("reduce_scatter: ragged inputs")
    if p == 1:
        return [inputs[0].clone() if _is_cuda(inputs[0]) else np.array(inputs[0], np.float32)]
    c = n // p
    torch = _torch()
    ts, host, devs = _as_device(inputs)
    shards = [torch.empty(c, dtype=torch.float32, device=t.device) for t in ts]
    tin, _k1 = _ptrs(ts)
    tout, _k2 = _ptrs(shards)
    dev_s = _run(devs, n, "reduce_scatter",
                 lambda m: _lib.hccx_mcomm_reduce_scatter(m, tin, tout, n, spec.c(), None))
    if _lossless(spec):
        hop = _lossless_hops(ts, n, 0, torch.cuda.current_stream(devs[0]))
        cost = _Cost.rs(clock, comm, spec, c, lambda r, j: hop[r * p + j])
    else:
        w = _message_bytes(spec, c)
        cost = _Cost.rs(clock, comm, spec, c, lambda r, j: w)
    _commit(clock, comm, cost, dev_s, path, CollectiveKind.ReduceScatter)
    return _back(shards, host)


def ring_allgather(clock: SimClock, comm: Communicator, shards: Sequence, spec: CodecSpec,
                   path: CommPath) -> list:
    """collectives.cpp:183-200."""
    from . import _lib

    p = comm.size()
    assert len(shards) == p
    c = len(shards[0])
    if any(len(s) != c for s in shards):
        raise BadChunkingError("allgather: mismatched shard lengths")
    if p == 1:
        return [shards[0].clone() if _is_cuda(shards[0]) else np.array(shards[0], np.float32)]
    torch = _torch()
    ts, host, devs = _as_device(shards)
    outs = [torch.empty(p * c, dtype=torch.float32, device=t.device) for t in ts]
    tin, _k1 = _ptrs(ts)
    tout, _k2 = _ptrs(outs)
    dev_s = _run(devs, p * c, "allgather", lambda m: _lib.hccx_mcomm_allgather(m, tin, tout, c, spec.c(), None))
    if _lossless(spec):
        hop = _lossless_hops(ts, c, 1, torch.cuda.current_stream(devs[0]))
        cost = _Cost.ag(clock, comm, spec, c, lambda k: hop[k])
    else:
        w = _message_bytes(spec, c)
        cost = _Cost.ag(clock, comm, spec, c, lambda k: w)
    _commit(clock, comm, cost, dev_s, path, CollectiveKind.AllGather)
    return _back(outs, host)


def allreduce(clock: SimClock, comm: Communicator, inputs: Sequence, spec: CodecSpec, path: CommPath,
              mode: ReduceMode = ReduceMode.Sum) -> list:
    """collectives.cpp:202-248."""
    from . import _lib

    p = comm.size()
    assert len(inputs) == p
    n = len(inputs[0])
    if n % p != 0:
        raise BadChunkingError(f"allreduce: length {n} not divisible by {p}")
    if any(len(b) != n for b in inputs):
        raise BadChunkingError("allreduce: ragged inputs")
    if p == 1:
        return [inputs[0].clone() if _is_cuda(inputs[0]) else np.array(inputs[0], np.float32)]
    c = n // p
    torch = _torch()
    ts, host, devs = _as_device(inputs)
    outs = [torch.empty(n, dtype=torch.float32, device=t.device) for t in ts]
    tin, _k1 = _ptrs(ts)
    tout, _k2 = _ptrs(outs)
    dev_s = _run(devs, n, "allreduce",
                 lambda m: _lib.hccx_mcomm_allreduce(m, tin, tout, n, spec.c(), int(mode), None))
    if _lossless(spec):
        hop = _lossless_hops(ts, n, 2, torch.cuda.current_stream(devs[0]))
        nrs = (p - 1) * p
        rs = _Cost.rs(clock, comm, spec, c, lambda r, j: hop[r * p + j])
        ag = _Cost.ag(clock, comm, spec, c, lambda k: hop[nrs + k])
    else:
        w = _message_bytes(spec, c)
        rs = _Cost.rs(clock, comm, spec, c, lambda r, j: w)
        ag = _Cost.ag(clock, comm, spec, c, lambda k: w)
    total = _Cost()
    total.duration = rs.duration + ag.duration
    total.raw_total = rs.raw_total + ag.raw_total
    total.wire_total = rs.wire_total + ag.wire_total
    total.rounds = rs.rounds + ag.rounds
    _commit(clock, comm, total, dev_s, path, CollectiveKind.AllReduce)
    return _back(outs, host)


def p2p(clock: SimClock, src: int, dst: int, buf, spec: CodecSpec, path: CommPath):
    """collectives.cpp:130-152: dst receives dec(comp(buf)); both clocks advance."""
    from . import _lib

    assert src != dst
    n = len(buf)
    torch = _torch()
    (t,), host, devs = _as_device([buf])
    if _lossless(spec):
        from . import lossless

        msg = lossless.size(t)
    else:
        msg = _message_bytes(spec, n)
    out = torch.empty(n, dtype=torch.float32, device=t.device)
    dev_s = 0.0
    if n:
        dev_s = _run((devs[0], devs[0]), n, "p2p",
                     lambda m: _lib.hccx_mcomm_p2p(m, 0, 1, t.data_ptr(), out.data_ptr(), n, spec.c(), None))
    topo, raw = clock.topology(), 4 * n
    dur = codec_time(topo, raw, spec) + transfer_time(topo, msg, link_class(topo, src, dst)) + codec_time(
        topo, raw, spec)
    clock.sync_to_max([src, dst])
    clock.advance(src, dur)
    clock.advance(dst, dur)
    clock.record(TraceEvent(0, path, CollectiveKind.P2P, 2, raw, msg, dur, 1, dev_s))
    return _back([out], host)[0]


def broadcast(clock: SimClock, comm: Communicator, root: int, buf, spec: CodecSpec, path: CommPath) -> list:
    """Broadcast from communicator position ``root`` (not in the reference;
    defined by analogy with the allgather single-shard rule: the root's
    payload crosses p-1 ring hops)."""
    from . import _lib

    p = comm.size()
    n = len(buf)
    if p == 1:
        return [buf.clone() if _is_cuda(buf) else np.array(buf, np.float32)]
    torch = _torch()
    (t,), host, devs = _as_device([buf])
    if _lossless(spec):
        from . import lossless

        msg = lossless.size(t)
    else:
        msg = _message_bytes(spec, n)
    outs = [torch.empty(n, dtype=torch.float32, device=t.device) for _ in range(p)]
    tout, _k = _ptrs(outs)
    dev_s = 0.0
    if n:
        dev_s = _run(tuple(devs[0] for _ in range(p)), n, "broadcast",
                     lambda m: _lib.hccx_mcomm_broadcast(m, root, t.data_ptr(), tout, n, spec.c(), None))
    topo, raw = clock.topology(), 4 * n
    cost = _Cost()
    for rnd in range(p - 1):
        j = (root + rnd) % p
        hop = transfer_time(topo, msg, link_class(topo, comm.ranks[j], comm.ranks[(j + 1) % p])) + codec_time(
            topo, raw, spec)
        if rnd == 0:
            hop += codec_time(topo, raw, spec)
        cost.duration += hop
        cost.raw_total += raw
        cost.wire_total += msg
    cost.rounds = p - 1
    _commit(clock, comm, cost, dev_s, path, CollectiveKind.Broadcast)
    return _back(outs, host)
