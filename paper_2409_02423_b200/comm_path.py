"""CommPath: every communication of a 3D-parallel step (proj/include/hcc/comm_path.hpp:13-45)."""
from __future__ import annotations

import enum

from .errors import ConfigError


class CommPath(enum.IntEnum):
    DpAllReduce = 0
    PpP2p = 1
    TpAllReduce = 2
    TpAllGather = 3
    Zero1AllGather = 4
    Zero1ReduceScatter = 5

    def __str__(self) -> str:
        return self.name


K_ALL_COMM_PATHS = tuple(CommPath)


def comm_path_from_string(s: str) -> CommPath:
    """comm_path.hpp:40-45."""
    for p in CommPath:
        if p.name == s:
            return p
    raise ConfigError("path", f"unknown communication path '{s}'")
