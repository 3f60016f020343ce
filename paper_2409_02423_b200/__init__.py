"""B200-native compressed collectives (arXiv 2409.02423 hot path).

Host-side mirror of the reference's C++ API (proj/include/hcc/*.hpp) over the
C ABI of libhccx.so (include/hccx.h): the fixed-rate codec, compressed ring
collectives, and the hybrid per-parallel-dimension rate policy.

Submodules
  codec        CodecSpec, compress/decompress, wire_size_bytes, container
  collectives  allreduce / ring_reduce_scatter / ring_allgather / p2p / broadcast
               (all members on one device, reference value semantics)
  dist         the same collectives across processes, one GPU each, over NVLink
  parallel3d   ParallelLayout + SchemeTable (hybrid rate policy)
  netsim       SimClock / TraceEvent / Topology boundary types
"""
from .codec import (CodecKind, CodecSpec, CompressedBuffer, codec_spec_from_string, compress, decompress,
                    from_bytes, to_bytes, to_string, wire_size_bytes)
from .comm_path import CommPath
from .errors import (BadChunkingError, BadLayoutError, ConfigError, CorruptPayloadError, DataDependentSizeError,
                     Error, InvalidSchemeError, NonFiniteInputError)
from .parallel3d import (ParallelLayout, SchemeTable, build_layout, scheme_from_name, scheme_mz_hybrid,
                         scheme_naive, scheme_no_compression, scheme_z_hybrid)

__all__ = [
    "CodecKind", "CodecSpec", "CompressedBuffer", "codec_spec_from_string", "compress", "decompress",
    "from_bytes", "to_bytes", "to_string", "wire_size_bytes", "CommPath", "Error", "NonFiniteInputError",
    "CorruptPayloadError", "DataDependentSizeError", "BadChunkingError", "BadLayoutError", "InvalidSchemeError",
    "ConfigError", "ParallelLayout", "SchemeTable", "build_layout", "scheme_from_name", "scheme_mz_hybrid",
    "scheme_naive", "scheme_no_compression", "scheme_z_hybrid",
]
