"""Boundary types of the collective API: SimClock, TraceEvent, Topology.

The reference's collectives take a ``SimClock&`` and record one TraceEvent per
collective (proj/include/hcc/netsim.hpp:63-101, proj/src/collectives.cpp:113-126).
Those types are part of the drop-in signature, so they are kept with the
reference's alpha-beta cost model (proj/src/netsim.cpp:53-75): ``duration_s``
and the clocks are the model's simulated seconds, identical to the
reference's; the B200 engine's measured device time of each collective is the
addition ``TraceEvent.device_s``.  Byte accounting (raw/wire bytes, round
counts) is integer-identical to the reference.
"""
from __future__ import annotations

import enum
import io
from dataclasses import dataclass, replace
from typing import Iterable, List

from .comm_path import CommPath
from .errors import ConfigError


@dataclass
class Topology:
    """Cluster shape plus alpha-beta link parameters (netsim.hpp:18-40)."""

    num_nodes: int = 1
    gpus_per_node: int = 1
    intra_bw: float = 0.0
    inter_bw: float = 0.0
    intra_lat: float = 0.0
    inter_lat: float = 0.0
    codec_bw: float = 0.0
    compute_flops: float = 0.0

    def world_size(self) -> int:
        return self.num_nodes * self.gpus_per_node

    def node_of(self, rank: int) -> int:
        return rank // self.gpus_per_node

    def validate(self) -> None:
        """netsim.cpp:9-18: ConfigError on a nonpositive count or rate."""
        for name, ok in (("num_nodes", self.num_nodes >= 1), ("gpus_per_node", self.gpus_per_node >= 1)):
            if not ok:
                raise ConfigError(f"topology.{name}", "must be >= 1")
        for name in ("intra_bw", "inter_bw", "intra_lat", "inter_lat", "codec_bw", "compute_flops"):
            if not getattr(self, name) > 0:
                raise ConfigError(f"topology.{name}", "must be > 0")

    @staticmethod
    def lassen_like(num_nodes: int = 2) -> "Topology":
        """Preset of src/netsim.cpp:20-31 (config values, not paper facts)."""
        return Topology(num_nodes, 4, 75.0e9, 12.5e9, 2.0e-6, 5.0e-6, 400.0e9, 7.0e12)

    @staticmethod
    def desk_2x2(num_nodes: int = 2) -> "Topology":
        return Topology(num_nodes, 2, 16.0e9, 1.25e9, 5.0e-6, 20.0e-6, 50.0e9, 1.0e12)

    @staticmethod
    def b200_box(num_gpus: int = 8) -> "Topology":
        """One NVSwitch box: every peer at 900 GB/s/direction (NVLink 5);
        codec_bw = the measured r8 compress throughput on one B200 (4.05e12
        uncompressed B/s, bench.py N=1); compute_flops = fp32 CUDA-core peak
        (148 SMs x 128 lanes x 2 x 1.965 GHz)."""
        return Topology(1, num_gpus, 900.0e9, 900.0e9, 2.0e-6, 2.0e-6, 4.05e12, 74.4e12)

    @staticmethod
    def preset(name: str, num_nodes: int) -> "Topology":
        if name == "lassen-like":
            return Topology.lassen_like(num_nodes)
        if name == "desk-2x2":
            return Topology.desk_2x2(num_nodes)
        if name == "b200-box":
            return Topology.b200_box(8 * num_nodes)
        raise ConfigError("topology.preset", f"unknown preset '{name}' (expected lassen-like | desk-2x2 | b200-box)")


class LinkClass(enum.IntEnum):
    SelfLoop = 0
    IntraNode = 1
    InterNode = 2


def link_class(topo: Topology, a: int, b: int) -> LinkClass:
    """netsim.cpp:53-58."""
    if a == b:
        return LinkClass.SelfLoop
    return LinkClass.IntraNode if topo.node_of(a) == topo.node_of(b) else LinkClass.InterNode


def transfer_time(topo: Topology, nbytes: int, link: LinkClass) -> float:
    """netsim.cpp:60-70: latency + bytes / bandwidth of the link class."""
    if link == LinkClass.SelfLoop:
        return 0.0
    if link == LinkClass.IntraNode:
        return topo.intra_lat + float(nbytes) / topo.intra_bw
    return topo.inter_lat + float(nbytes) / topo.inter_bw


def codec_time(topo: Topology, raw_bytes: int, spec) -> float:
    """netsim.cpp:72-75: identity is free, every other codec raw / codec_bw."""
    from .codec import CodecKind

    return 0.0 if spec.kind == CodecKind.Identity else float(raw_bytes) / topo.codec_bw


class CollectiveKind(enum.IntEnum):
    AllReduce = 0
    AllGather = 1
    ReduceScatter = 2
    P2P = 3
    Broadcast = 4  # not in the reference


@dataclass
class TraceEvent:
    """netsim.hpp:66-75.  raw/wire bytes are per-rank sent bytes."""

    step: int = 0
    path: CommPath = CommPath.DpAllReduce
    collective: CollectiveKind = CollectiveKind.AllReduce
    comm_size: int = 0
    raw_bytes: int = 0
    wire_bytes: int = 0
    duration_s: float = 0.0
    round_count: int = 0
    device_s: float = 0.0  # addition: measured device time of the collective on the B200s


class SimClock:
    """Per-rank clocks plus the event log (netsim.hpp:79-101).  Collectives
    advance members by the cost model's duration."""

    def __init__(self, topo: Topology):
        self._topo = topo
        self._clock: List[float] = [0.0] * topo.world_size()
        self._trace: List[TraceEvent] = []
        self._step = 0

    def topology(self) -> Topology:
        return self._topo

    def time(self, rank: int) -> float:
        return self._clock[rank]

    def max_time(self) -> float:
        return max(self._clock) if self._clock else 0.0

    def advance(self, rank: int, dt: float) -> None:
        assert dt >= 0.0
        self._clock[rank] += dt

    def sync_to_max(self, ranks: Iterable[int]) -> None:
        ranks = list(ranks)
        t = max((self._clock[r] for r in ranks), default=0.0)
        for r in ranks:
            self._clock[r] = t

    def set_step(self, step: int) -> None:
        self._step = step

    def step(self) -> int:
        return self._step

    def record(self, e: TraceEvent) -> None:
        self._trace.append(replace(e, step=self._step))

    def trace(self) -> List[TraceEvent]:
        return self._trace


def write_trace_csv(os_: io.TextIOBase, trace: List[TraceEvent]) -> None:
    """netsim.cpp:97-106."""
    os_.write("step,path,collective,comm_size,raw_bytes,wire_bytes,duration_s\n")
    for e in trace:
        os_.write(f"{e.step},{CommPath(e.path).name},{CollectiveKind(e.collective).name},{e.comm_size},"
                  f"{e.raw_bytes},{e.wire_bytes},{e.duration_s:.9e}\n")
