"""Codec API mirroring proj/include/hcc/codec.hpp on the B200 kernels.

Reference surface kept as a drop-in (file:line in /root/reference/proj):
  CodecKind / CodecSpec ............ include/hcc/codec.hpp:16-32
  to_string / codec_spec_from_string src/codec.cpp:19-45
  kFixedRateBlock / kPredictorChunk  include/hcc/codec.hpp:41-42
  CompressedBuffer ................. include/hcc/codec.hpp:44-51
  compress / decompress ............ include/hcc/codec.hpp:53-61, src/codec_omp.cpp
  wire_size_bytes .................. include/hcc/codec.hpp:63-67, src/codec.cpp:47-61
  to_bytes / from_bytes ("HCC1") ... include/hcc/codec.hpp:69-79, src/codec.cpp:89-121

compress/decompress accept either a host numpy float32 array (the
reference's value API: host in, host out, copies pipelined with the kernels
inside libhccx) or a CUDA torch tensor (device in, device out).  All
arithmetic runs in the sm_100a kernels behind include/hccx.h.

Addition: CodecKind.ZfpRate ("zfp-rate:N"), the ZFP-style transform codec the
north star asks for.  It is not in the reference; see codec_zfp.cuh.
"""
from __future__ import annotations

import ctypes as C
import enum
import struct
from dataclasses import dataclass
from typing import Any

import numpy as np

from .errors import ConfigError, CorruptPayloadError, DataDependentSizeError, InvalidSchemeError, check

K_FIXED_RATE_BLOCK = 64
K_PREDICTOR_CHUNK = 4096
K_CONTAINER_HEADER_BYTES = 18
_MAGIC = b"HCC1"


class CodecKind(enum.IntEnum):
    Identity = 0
    LosslessPredictor = 1
    FixedRate = 2
    ZfpRate = 3  # not in the reference


@dataclass(frozen=True)
class CodecSpec:
    kind: CodecKind = CodecKind.Identity
    rate_bits: int = 0

    @staticmethod
    def identity() -> "CodecSpec":
        return CodecSpec(CodecKind.Identity, 0)

    @staticmethod
    def lossless() -> "CodecSpec":
        return CodecSpec(CodecKind.LosslessPredictor, 0)

    @staticmethod
    def fixed_rate(bits: int) -> "CodecSpec":
        """src/codec.cpp:11-17: bits in [2, 32] else InvalidSchemeError."""
        if not isinstance(bits, int) or bits < 2 or bits > 32:
            raise InvalidSchemeError(f"fixed-rate bits must be in [2, 32], got {bits}")
        return CodecSpec(CodecKind.FixedRate, bits)

    @staticmethod
    def zfp_rate(bits: int) -> "CodecSpec":
        if not isinstance(bits, int) or bits < 3 or bits > 32:
            raise InvalidSchemeError(f"zfp-rate bits must be in [3, 32], got {bits}")
        return CodecSpec(CodecKind.ZfpRate, bits)

    def is_lossy(self) -> bool:
        return self.kind in (CodecKind.FixedRate, CodecKind.ZfpRate)

    def c(self):
        from . import _lib

        return _lib.Codec(int(self.kind), int(self.rate_bits))

    def __str__(self) -> str:
        return to_string(self)


def to_string(spec: CodecSpec) -> str:
    """src/codec.cpp:19-29."""
    if spec.kind == CodecKind.Identity:
        return "identity"
    if spec.kind == CodecKind.LosslessPredictor:
        return "lossless"
    if spec.kind == CodecKind.FixedRate:
        return f"fixed-rate:{spec.rate_bits}"
    if spec.kind == CodecKind.ZfpRate:
        return f"zfp-rate:{spec.rate_bits}"
    return "unknown"


def stoi(s: str) -> int:
    """std::stoi: optional leading whitespace and sign, then at least one digit;
    trailing characters are ignored.  Raises ValueError like std::invalid_argument
    / std::out_of_range."""
    i = 0
    while i < len(s) and s[i] in " \t\n\r\f\v":
        i += 1
    j = i
    if j < len(s) and s[j] in "+-":
        j += 1
    k = j
    while k < len(s) and s[k].isdigit() and s[k].isascii():
        k += 1
    if k == j:
        raise ValueError(f"stoi: no conversion of '{s}'")
    v = int(s[i:k])
    if not -(2 ** 31) <= v < 2 ** 31:
        raise ValueError(f"stoi: out of range '{s}'")
    return v


def codec_spec_from_string(s: str) -> CodecSpec:
    """src/codec.cpp:31-45 (plus "zfp-rate:N")."""
    if s == "identity":
        return CodecSpec.identity()
    if s == "lossless":
        return CodecSpec.lossless()
    for prefix, make in (("fixed-rate:", CodecSpec.fixed_rate), ("zfp-rate:", CodecSpec.zfp_rate)):
        if s.startswith(prefix):
            try:
                bits = stoi(s[len(prefix):])
            except ValueError:
                raise ConfigError("codec", f"bad {prefix[:-1]} value in '{s}'") from None
            return make(bits)
    raise ConfigError("codec", f"unknown codec '{s}' (expected identity | lossless | fixed-rate:N | zfp-rate:N)")


@dataclass
class CompressedBuffer:
    """include/hcc/codec.hpp:44-51.  ``payload`` is a numpy uint8 array (host)
    or a CUDA torch uint8 tensor (device), matching the input of compress()."""

    codec: CodecSpec
    original_len: int
    chunk_count: int
    payload: Any

    def payload_bytes(self) -> int:
        return int(self.payload.numel() if hasattr(self.payload, "numel") else self.payload.size)


def wire_size_bytes(spec: CodecSpec, n: int) -> int:
    """src/codec.cpp:47-61: exact payload bytes; lossless -> DataDependentSizeError."""
    from . import _lib

    out = C.c_uint64(0)
    check(_lib.hccx_wire_size_bytes(spec.c(), n, C.byref(out)), "wire_size_bytes")
    return int(out.value)


def chunk_count(spec: CodecSpec, n: int) -> int:
    from . import _lib

    out = C.c_uint64(0)
    check(_lib.hccx_chunk_count(spec.c(), n, C.byref(out)), "chunk_count")
    return int(out.value)


def _is_cuda_tensor(x) -> bool:
    return hasattr(x, "is_cuda") and bool(x.is_cuda)


def _stream_ptr(t) -> int:
    import torch

    return torch.cuda.current_stream(t.device).cuda_stream


def compress(spec: CodecSpec, buf) -> CompressedBuffer:
    """Compress a host float32 array or a CUDA float32 tensor.

    FixedRate/ZfpRate raise NonFiniteInputError on NaN/Inf input
    (src/codec_omp.cpp:45).  Output is bit-deterministic and bit-identical to
    the reference (hcc::compress / hcc::serial::compress) for FixedRate.
    """
    from . import _lib

    if spec.kind == CodecKind.LosslessPredictor:
        from . import lossless

        return lossless.compress(buf)
    n = int(buf.numel() if hasattr(buf, "numel") else np.asarray(buf).size)
    nbytes = wire_size_bytes(spec, n)
    cc = chunk_count(spec, n)
    if _is_cuda_tensor(buf):
        import torch

        x = buf.contiguous().view(-1)
        if x.dtype != torch.float32:
            raise TypeError("compress expects float32")
        out = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
        err = torch.zeros(1, dtype=torch.int32, device=x.device)
        s = _stream_ptr(x)
        check(_lib.hccx_compress(spec.c(), x.data_ptr(), n, out.data_ptr(), err.data_ptr(), s), "compress")
        check(_lib.hccx_flag_status(err.data_ptr(), s), "compress")
        return CompressedBuffer(spec, n, cc, out)
    x = np.ascontiguousarray(buf, dtype=np.float32).reshape(-1)
    out = np.empty(nbytes, np.uint8)
    if n:
        check(_lib.hccx_compress_host(spec.c(), x.ctypes.data, n, out.ctypes.data, _device()), "compress")
    return CompressedBuffer(spec, n, cc, out)


def decompress(cbuf: CompressedBuffer):
    """Inverse of compress (src/codec_omp.cpp:87-111).  Validates the block
    count and payload size first (CorruptPayloadError, :94-96)."""
    from . import _lib

    spec = cbuf.codec
    if spec.kind == CodecKind.LosslessPredictor:
        from . import lossless

        return lossless.decompress(cbuf)
    n = int(cbuf.original_len)
    if spec.kind != CodecKind.Identity and cbuf.chunk_count != chunk_count(spec, n):
        raise CorruptPayloadError("payload does not match block count")
    if cbuf.payload_bytes() != wire_size_bytes(spec, n):
        raise CorruptPayloadError("payload size does not match the codec's size law")
    if _is_cuda_tensor(cbuf.payload):
        import torch

        p = cbuf.payload.contiguous()
        out = torch.empty(n, dtype=torch.float32, device=p.device)
        check(_lib.hccx_decompress(spec.c(), p.data_ptr(), p.numel(), n, out.data_ptr(), _stream_ptr(p)),
              "decompress")
        return out
    p = np.ascontiguousarray(cbuf.payload, dtype=np.uint8)
    out = np.empty(n, np.float32)
    if n:
        check(_lib.hccx_decompress_host(spec.c(), p.ctypes.data, p.size, n, out.ctypes.data, _device()),
              "decompress")
    return out


def _device() -> int:
    try:
        import torch

        return torch.cuda.current_device() if torch.cuda.is_available() else 0
    except Exception:  # pragma: no cover
        return 0


# ------------------------------------------------------------ container ----

def to_bytes(cbuf: CompressedBuffer) -> bytes:
    """src/codec.cpp:89-100: "HCC1" | kind u8 | rate u8 | original_len u64 |
    chunk_count u32 | payload, little-endian."""
    payload = cbuf.payload
    if hasattr(payload, "cpu"):
        payload = payload.cpu().numpy()
    hdr = _MAGIC + struct.pack("<BBQI", int(cbuf.codec.kind), int(cbuf.codec.rate_bits) & 0xFF,
                               int(cbuf.original_len), int(cbuf.chunk_count) & 0xFFFFFFFF)
    return hdr + np.asarray(payload, np.uint8).tobytes()


def from_bytes(data: bytes) -> CompressedBuffer:
    """src/codec.cpp:102-121 (kind 3 accepted for the zfp-mode codec)."""
    data = bytes(data)
    if len(data) < K_CONTAINER_HEADER_BYTES:
        raise CorruptPayloadError("container shorter than header")
    if data[:4] != _MAGIC:
        raise CorruptPayloadError("bad container magic")
    kind, rate, n, cc = struct.unpack("<BBQI", data[4:18])
    if kind > 3:
        raise CorruptPayloadError("bad codec kind byte")
    if kind == CodecKind.FixedRate and not 2 <= rate <= 32:
        raise CorruptPayloadError("bad fixed-rate bits in header")
    if kind == CodecKind.ZfpRate and not 3 <= rate <= 32:
        raise CorruptPayloadError("bad zfp-rate bits in header")
    spec = CodecSpec(CodecKind(kind), rate)
    return CompressedBuffer(spec, n, cc, np.frombuffer(data[18:], np.uint8).copy())


__all__ = [
    "CodecKind", "CodecSpec", "CompressedBuffer", "compress", "decompress", "wire_size_bytes",
    "chunk_count", "to_string", "codec_spec_from_string", "to_bytes", "from_bytes",
    "K_FIXED_RATE_BLOCK", "K_PREDICTOR_CHUNK", "K_CONTAINER_HEADER_BYTES", "DataDependentSizeError",
]
