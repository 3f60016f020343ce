"""Parallel layout and the hybrid per-path rate policy.

Mirrors proj/include/hcc/parallel3d.hpp:14-74 and proj/src/parallel3d.cpp:7-122:
  ParallelLayout (rank = d*(pp*tp) + p*tp + t, TP innermost) and its groups,
  build_layout, SchemeTable (CommPath -> CodecSpec), scheme_no_compression /
  scheme_naive / scheme_mz_hybrid / scheme_z_hybrid / scheme_from_name.
The table is the policy the paper contributes: an aggressive rate for the DP
gradient all-reduce and a mild one for TP/PP/ZeRO traffic (Tables II/III).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List

from .codec import CodecKind, CodecSpec, stoi
from .comm_path import K_ALL_COMM_PATHS, CommPath
from .errors import BadLayoutError, ConfigError, InvalidSchemeError


@dataclass(frozen=True)
class Coord:
    d: int
    p: int
    t: int


@dataclass(frozen=True)
class ParallelLayout:
    dp: int = 1
    pp: int = 1
    tp: int = 1

    def world(self) -> int:
        return self.dp * self.pp * self.tp

    def rank_of(self, d: int, p: int, t: int) -> int:
        return d * (self.pp * self.tp) + p * self.tp + t

    def coord_of(self, rank: int) -> Coord:
        return Coord(rank // (self.pp * self.tp), (rank // self.tp) % self.pp, rank % self.tp)

    def dp_group(self, rank: int) -> List[int]:
        """Ranks sharing (p, t), ordered by d (parallel3d.cpp:7-13)."""
        c = self.coord_of(rank)
        return [self.rank_of(d, c.p, c.t) for d in range(self.dp)]

    def tp_group(self, rank: int) -> List[int]:
        """Ranks sharing (d, p), ordered by t (parallel3d.cpp:15-21)."""
        c = self.coord_of(rank)
        return [self.rank_of(c.d, c.p, t) for t in range(self.tp)]

    def pp_chain(self, rank: int) -> List[int]:
        """Ranks sharing (d, t), ordered by stage (parallel3d.cpp:23-29)."""
        c = self.coord_of(rank)
        return [self.rank_of(c.d, p, c.t) for p in range(self.pp)]


def build_layout(dp: int, pp: int, tp: int, world_size: int) -> ParallelLayout:
    """parallel3d.cpp:31-41 (takes the world size instead of a netsim Topology)."""
    if dp < 1 or pp < 1 or tp < 1:
        raise BadLayoutError("parallel degrees must be >= 1")
    if dp * pp * tp != world_size:
        raise BadLayoutError(f"dp*pp*tp = {dp * pp * tp} does not match world size {world_size}")
    return ParallelLayout(dp, pp, tp)


@dataclass
class SchemeTable:
    """Total map CommPath -> CodecSpec (parallel3d.hpp:49-54)."""

    name: str = ""
    paths: Dict[CommPath, CodecSpec] = field(default_factory=dict)

    def at(self, p: CommPath) -> CodecSpec:
        return self.paths[p]


def scheme_no_compression() -> SchemeTable:
    return SchemeTable("no-compression", {p: CodecSpec.identity() for p in K_ALL_COMM_PATHS})


def scheme_naive(spec: CodecSpec) -> SchemeTable:
    """parallel3d.cpp:50-61: the same codec on every path."""
    if spec.kind == CodecKind.Identity:
        name = "no-compression"
    elif spec.kind == CodecKind.LosslessPredictor:
        name = "naive-mpc"
    elif spec.kind == CodecKind.ZfpRate:
        name = f"naive-zfpmode{spec.rate_bits}"
    else:
        name = f"naive-zfp{spec.rate_bits}"
    return SchemeTable(name, {p: spec for p in K_ALL_COMM_PATHS})


def scheme_mz_hybrid(dp_rate: int) -> SchemeTable:
    """parallel3d.cpp:63-69: lossless everywhere, fixed-rate on the DP all-reduce."""
    t = SchemeTable(f"mz-hybrid:{dp_rate}", {p: CodecSpec.lossless() for p in K_ALL_COMM_PATHS})
    t.paths[CommPath.DpAllReduce] = CodecSpec.fixed_rate(dp_rate)
    return t


def scheme_z_hybrid(mp_rate: int, dp_rate: int) -> SchemeTable:
    """parallel3d.cpp:71-82: fixed-rate everywhere, mp_rate >= dp_rate."""
    if mp_rate < dp_rate:
        raise InvalidSchemeError(f"z-hybrid requires mp_rate >= dp_rate, got mp={mp_rate} dp={dp_rate}")
    t = SchemeTable(f"z-hybrid:{mp_rate},{dp_rate}",
                    {p: CodecSpec.fixed_rate(mp_rate) for p in K_ALL_COMM_PATHS})
    t.paths[CommPath.DpAllReduce] = CodecSpec.fixed_rate(dp_rate)
    return t


def _int(s: str, name: str) -> int:
    try:
        return stoi(s)
    except ValueError:
        raise ConfigError("scheme", f"bad rate in '{name}'") from None


def scheme_from_name(name: str) -> SchemeTable:
    """parallel3d.cpp:84-122: baseline | no-compression | naive-mpc | naive-zfpN |
    mz-hybrid:D | z-hybrid:M,D."""
    if name in ("baseline", "no-compression"):
        return scheme_no_compression()
    if name == "naive-mpc":
        return scheme_naive(CodecSpec.lossless())
    if name.startswith("naive-zfp"):
        return scheme_naive(CodecSpec.fixed_rate(_int(name[9:], name)))
    if name.startswith("mz-hybrid:"):
        return scheme_mz_hybrid(_int(name[10:], name))
    if name.startswith("z-hybrid:") and "," in name[9:]:
        comma = name.index(",", 9)
        return scheme_z_hybrid(_int(name[9:comma], name), _int(name[comma + 1:], name))
    raise ConfigError("scheme", f"unknown scheme '{name}' (expected baseline | no-compression | naive-mpc | "
                                "naive-zfpN | mz-hybrid:D | z-hybrid:M,D)")
