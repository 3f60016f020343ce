"""Hybrid per-parallel-dimension compression over real process groups.

The paper's contribution is *where* each rate goes (MZHybrid / ZHybrid,
proj/src/parallel3d.cpp:43-122): an aggressive rate on the DP gradient
all-reduce, a mild one on TP activations, PP point-to-point and ZeRO
traffic.  ``HybridComm`` applies a ``SchemeTable`` to a 3D-parallel layout of
torch.distributed ranks (one GPU each): every DP group, TP group and PP chain
of the layout (ParallelLayout, proj/include/hcc/parallel3d.hpp:14-46) gets
its own NVLink communicator (dist.NvlinkComm), and each call site routes
through ``scheme.at(path)`` exactly like the reference trainer's call sites
(proj/src/toymodel.cpp:290-459):

  tp_allreduce   TpAllReduce        Sum       (toymodel.cpp:290, :351)
  pp_send_recv   PpP2p                        (toymodel.cpp:297, :358)
  dp_allreduce   DpAllReduce        Average   (toymodel.cpp:417)
  zero_reduce_scatter  Zero1ReduceScatter     (toymodel.cpp:429)
  zero_allgather       Zero1AllGather         (toymodel.cpp:457)
  tp_allgather   TpAllGather        (policy row; the reference never emits it)

Every call records a TraceEvent (raw/wire bytes per rank as the reference
accounts them, measured device seconds) in ``self.trace``.  Under
LosslessPredictor (MZHybrid's TP / PP / ZeRO paths) the compressed bytes
themselves cross NVLink as framed messages (HCC1 container header per
message, csrc/lossless_comm.cu) and the traced wire bytes are the payload
bytes the engine actually pushed.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Tuple

from .codec import CodecKind, wire_size_bytes
from .comm_path import CommPath
from .netsim import CollectiveKind, TraceEvent
from .parallel3d import ParallelLayout, SchemeTable


def plan_groups(layout: ParallelLayout) -> Dict[str, List[Tuple[int, ...]]]:
    """Every DP group, TP group and PP chain of the layout, each an ordered
    rank tuple (the communicator order = ring order).  Pure host logic: all
    ranks must create the torch.distributed subgroups in this same order."""
    out: Dict[str, List[Tuple[int, ...]]] = {"dp": [], "tp": [], "pp": []}
    for kind, fn in (("dp", layout.dp_group), ("tp", layout.tp_group), ("pp", layout.pp_chain)):
        seen = set()
        for r in range(layout.world()):
            g = tuple(fn(r))
            if g not in seen:
                seen.add(g)
                out[kind].append(g)
    return out


@dataclass
class _Group:
    ranks: Tuple[int, ...]
    pg: object
    comm: object  # NvlinkComm or None (size-1 group)


class HybridComm:
    """Compressed 3D-parallel communication for this rank."""

    def __init__(self, layout: ParallelLayout, scheme: SchemeTable, max_n: int):
        import torch.distributed as dist

        from .dist import NvlinkComm

        self.layout = layout
        self.scheme = scheme
        self.rank = dist.get_rank()
        if layout.world() != dist.get_world_size():
            from .errors import BadLayoutError

            raise BadLayoutError(f"layout world {layout.world()} != world size {dist.get_world_size()}")
        self.groups: Dict[str, _Group] = {}
        for kind, groups in plan_groups(layout).items():
            for ranks in groups:
                pg = dist.new_group(list(ranks)) if len(ranks) > 1 else None
                if self.rank in ranks:
                    comm = NvlinkComm(max_n, group=pg) if len(ranks) > 1 else None
                    self.groups[kind] = _Group(ranks, pg, comm)
        self._trace: List[TraceEvent] = []
        self._pending: list = []
        self.step = 0

    # ---------------------------------------------------------------- utils
    def _timed(self, fn):
        import torch

        s = torch.cuda.current_stream()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        out = fn()
        b.record(s)
        return out, (a, b)

    def _record(self, path, kind, size, raw, wire, rounds, ev):
        """Queue the event; its device time is read when ``trace`` is next
        accessed, so back-to-back calls are not serialised by the host.
        Data-dependent (lossless) byte counts are taken now."""
        if callable(wire):
            ev[1].synchronize()
            wire = wire()
        self._pending.append((self.step, path, kind, size, raw, wire, rounds, ev))

    def last_bytes(self):
        """(path, raw_bytes, wire_bytes) of the most recent event, without
        waiting for its device time."""
        if self._pending:
            e = self._pending[-1]
            return e[1], e[4], e[5]
        if self._trace:
            e = self._trace[-1]
            return e.path, e.raw_bytes, e.wire_bytes
        return None

    @property
    def trace(self) -> List[TraceEvent]:
        for step, path, kind, size, raw, wire, rounds, (a, b) in self._pending:
            b.synchronize()
            self._trace.append(TraceEvent(step, path, kind, size, raw, wire, a.elapsed_time(b) / 1e3, rounds))
        self._pending = []
        return self._trace

    @staticmethod
    def _lossless(spec) -> bool:
        return spec.kind == CodecKind.LosslessPredictor

    def _lossless_wire(self, g) -> int:
        """Per-rank wire bytes (wire_total / p, collectives.cpp:113-126) of a
        LosslessPredictor collective: the engine sent every hop as a framed
        compressed message (csrc/lossless_comm.cu) and counted the payload
        bytes this rank pushed; the group total is one 8-byte sum."""
        import torch
        import torch.distributed as dist

        mine = g.comm.wire_bytes()[0]
        w = torch.tensor([mine], dtype=torch.int64, device="cuda")
        dist.all_reduce(w, group=g.pg)
        return int(w.item()) // len(g.ranks)

    # -------------------------------------------------------------- paths
    def dp_allreduce(self, grad, mode: int = 1):
        """Gradient averaging across the DP group (DpAllReduce, Average)."""
        return self._allreduce("dp", CommPath.DpAllReduce, grad, mode)

    def tp_allreduce(self, x):
        """Row-parallel output / input-gradient sum across the TP group."""
        return self._allreduce("tp", CommPath.TpAllReduce, x, 0)

    def _allreduce(self, kind, path, x, mode):
        g = self.groups[kind]
        spec = self.scheme.at(path)
        p = len(g.ranks)
        if p == 1:
            return x
        out, ev = self._timed(lambda: g.comm.allreduce(x, spec, mode))
        c = x.numel() // p
        wire = (lambda: self._lossless_wire(g)) if self._lossless(spec) else \
            2 * (p - 1) * wire_size_bytes(spec, c)
        self._record(path, CollectiveKind.AllReduce, p, 2 * (p - 1) * 4 * c, wire, 2 * (p - 1), ev)
        return out

    def tp_allgather(self, shard):
        g = self.groups["tp"]
        spec = self.scheme.at(CommPath.TpAllGather)
        p = len(g.ranks)
        if p == 1:
            return shard
        out, ev = self._timed(lambda: g.comm.allgather(shard, spec))
        c = shard.numel()
        wire = (lambda: self._lossless_wire(g)) if self._lossless(spec) else \
            (p - 1) * wire_size_bytes(spec, c)
        self._record(CommPath.TpAllGather, CollectiveKind.AllGather, p, (p - 1) * 4 * c, wire, p - 1, ev)
        return out

    def pp_send_recv(self, x, src_stage: int, dst_stage: int):
        """Activation (forward) or gradient (backward) hand-off between two
        pipeline stages of this rank's PP chain; both stages call, dst
        receives dec(comp(x))."""
        g = self.groups["pp"]
        spec = self.scheme.at(CommPath.PpP2p)
        out, ev = self._timed(lambda: g.comm.p2p(x, src_stage, dst_stage, spec))
        me = g.ranks.index(self.rank)
        if me in (src_stage, dst_stage):
            if self._lossless(spec):  # the framed message's payload, as sent / as received
                wire = g.comm.wire_bytes()[0] if me == src_stage else g.comm.recv_bytes()
            else:
                wire = wire_size_bytes(spec, x.numel())
            self._record(CommPath.PpP2p, CollectiveKind.P2P, 2, 4 * x.numel(), wire, 1, ev)
        return out

    def zero_reduce_scatter(self, grad):
        """ZeRO-1 gradient reduce-scatter over the DP group (Zero1ReduceScatter)."""
        g = self.groups["dp"]
        spec = self.scheme.at(CommPath.Zero1ReduceScatter)
        p = len(g.ranks)
        if p == 1:
            return grad
        out, ev = self._timed(lambda: g.comm.reduce_scatter(grad, spec))
        c = grad.numel() // p
        wire = (lambda: self._lossless_wire(g)) if self._lossless(spec) else \
            (p - 1) * wire_size_bytes(spec, c)
        self._record(CommPath.Zero1ReduceScatter, CollectiveKind.ReduceScatter, p, (p - 1) * 4 * c, wire, p - 1, ev)
        return out

    def zero_allgather(self, shard):
        """ZeRO-1 parameter all-gather over the DP group (Zero1AllGather)."""
        g = self.groups["dp"]
        spec = self.scheme.at(CommPath.Zero1AllGather)
        p = len(g.ranks)
        if p == 1:
            return shard
        out, ev = self._timed(lambda: g.comm.allgather(shard, spec))
        c = shard.numel()
        wire = (lambda: self._lossless_wire(g)) if self._lossless(spec) else \
            (p - 1) * wire_size_bytes(spec, c)
        self._record(CommPath.Zero1AllGather, CollectiveKind.AllGather, p, (p - 1) * 4 * c, wire, p - 1, ev)
        return out

    def status(self):
        for g in self.groups.values():
            if g.comm is not None:
                g.comm.status()

    def close(self):
        for g in self.groups.values():
            if g.comm is not None:
                g.comm.close()
