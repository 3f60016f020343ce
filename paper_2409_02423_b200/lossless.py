"""LosslessPredictor codec (proj/src/codec_kernels.hpp:165-239,
proj/src/codec_serial.cpp:48-66 / :85-107) on the GPU -- SURVEY.md §8 f1.

Payload layout (bit-identical to the reference): ceil(nchunks/8) raw-fallback
flag bytes, then per 4096-value chunk either its raw bytes (flag set, when
the coded size reaches 4*live) or the XOR-with-previous residual stream
(5-bit leading-zero count capped at 31, then the 32-lzc low residual bits,
LSB-first, flushed to a byte).

Device side (libhccx, csrc/lossless.cu): a warp-per-chunk size pass, an
exclusive scan, and a warp-per-chunk emit through shared-memory bit staging;
decode recovers the chunk offsets the format does not store with a walk over
the 5-bit length fields (O(1) per raw chunk), then decodes chunks in
parallel.  Sizes are data-dependent, so every call synchronises its stream.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from .errors import CorruptPayloadError, check

K_PREDICTOR_CHUNK = 4096


def max_bytes(n: int) -> int:
    from . import _lib

    return int(_lib.hccx_lossless_max_bytes(n))


def _nchunks(n: int) -> int:
    return (n + K_PREDICTOR_CHUNK - 1) // K_PREDICTOR_CHUNK


def size(buf) -> int:
    """Exact payload bytes of compress(lossless, buf) -- the size pass alone
    (what the collectives' wire accounting needs)."""
    from . import _lib
    from .codec import _is_cuda_tensor, _stream_ptr

    import torch

    if _is_cuda_tensor(buf):
        x = buf.contiguous().view(-1)
    else:
        x = torch.from_numpy(np.ascontiguousarray(buf, np.float32).reshape(-1)).cuda()
    if x.dtype != torch.float32:
        raise TypeError("lossless size expects float32")
    out = C.c_uint64(0)
    check(_lib.hccx_lossless_size(x.data_ptr(), x.numel(), C.byref(out), _stream_ptr(x)), "lossless_size")
    return int(out.value)


def compress(buf):
    from . import _lib
    from .codec import CodecSpec, CompressedBuffer, _device, _is_cuda_tensor, _stream_ptr

    spec = CodecSpec.lossless()
    if _is_cuda_tensor(buf):
        import torch

        x = buf.contiguous().view(-1)
        if x.dtype != torch.float32:
            raise TypeError("compress expects float32")
        n = x.numel()
        out = torch.empty(max(max_bytes(n), 1), dtype=torch.uint8, device=x.device)
        nb = C.c_uint64(0)
        check(_lib.hccx_lossless_compress(x.data_ptr(), n, out.data_ptr(), out.numel(), C.byref(nb),
                                          _stream_ptr(x)), "compress")
        return CompressedBuffer(spec, n, _nchunks(n), out[: nb.value])
    x = np.ascontiguousarray(buf, dtype=np.float32).reshape(-1)
    n = x.size
    out = np.empty(max(max_bytes(n), 1), np.uint8)
    nb = C.c_uint64(0)
    if n:
        check(_lib.hccx_lossless_compress_host(x.ctypes.data, n, out.ctypes.data, out.size, C.byref(nb), _device()),
              "compress")
    return CompressedBuffer(spec, n, _nchunks(n), out[: nb.value].copy())


def decompress(cbuf):
    """codec_serial.cpp:85-107: chunk-count / flag-byte header check, then a
    truncated stream raises CorruptPayloadError; trailing bytes are ignored."""
    from . import _lib
    from .codec import _device, _is_cuda_tensor, _stream_ptr

    n = int(cbuf.original_len)
    nch = _nchunks(n)
    if cbuf.chunk_count != nch or cbuf.payload_bytes() < (nch + 7) // 8:
        raise CorruptPayloadError("predictor payload header mismatch")
    if _is_cuda_tensor(cbuf.payload):
        import torch

        p = cbuf.payload.contiguous()
        out = torch.empty(n, dtype=torch.float32, device=p.device)
        if n:
            check(_lib.hccx_lossless_decompress(p.data_ptr(), p.numel(), n, out.data_ptr(), _stream_ptr(p)),
                  "decompress")
        return out
    p = np.ascontiguousarray(cbuf.payload, np.uint8)
    out = np.empty(n, np.float32)
    if n:
        check(_lib.hccx_lossless_decompress_host(p.ctypes.data, p.size, n, out.ctypes.data, _device()), "decompress")
    return out
