"""ctypes binding of the C ABI (include/hccx.h) in libhccx.so.

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2409_02423_b200/csrc``).  There is no fallback: if the library
is missing or fails to load, importing this module raises ImportError.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# HCCX_LIB: load an alternative build (kernel-variant experiments only).
LIB_PATH = os.environ.get("HCCX_LIB") or os.path.join(_HERE, "libhccx.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} not found: build the CUDA extension first "
        "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")

lib = C.CDLL(LIB_PATH)

HANDLE_BYTES = 256


class Codec(C.Structure):
    """hccx_codec_t: mirrors hcc::CodecSpec {kind, rate_bits}."""

    _fields_ = [("kind", C.c_int32), ("rate_bits", C.c_int32)]


_st = C.c_int
_p = C.c_void_p
_u64 = C.c_uint64
_pp = C.POINTER(C.c_void_p)


def _sig(name, res, *args):
    fn = getattr(lib, name)
    fn.restype = res
    fn.argtypes = list(args)
    return fn


hccx_status_string = _sig("hccx_status_string", C.c_char_p, _st)
hccx_abi_version = _sig("hccx_abi_version", C.c_int)
hccx_codec_validate = _sig("hccx_codec_validate", _st, Codec)
hccx_wire_size_bytes = _sig("hccx_wire_size_bytes", _st, Codec, _u64, C.POINTER(_u64))
hccx_chunk_count = _sig("hccx_chunk_count", _st, Codec, _u64, C.POINTER(_u64))
hccx_compress = _sig("hccx_compress", _st, Codec, _p, _u64, _p, _p, _p)
hccx_decompress = _sig("hccx_decompress", _st, Codec, _p, _u64, _u64, _p, _p)
hccx_flag_status = _sig("hccx_flag_status", _st, _p, _p)
hccx_compress_host = _sig("hccx_compress_host", _st, Codec, _p, _u64, _p, C.c_int)
hccx_decompress_host = _sig("hccx_decompress_host", _st, Codec, _p, _u64, _u64, _p, C.c_int)
hccx_lossless_max_bytes = _sig("hccx_lossless_max_bytes", _u64, _u64)
hccx_lossless_size = _sig("hccx_lossless_size", _st, _p, _u64, C.POINTER(_u64), _p)
hccx_lossless_compress = _sig("hccx_lossless_compress", _st, _p, _u64, _p, _u64, C.POINTER(_u64), _p)
hccx_lossless_decompress = _sig("hccx_lossless_decompress", _st, _p, _u64, _u64, _p, _p)
hccx_lossless_compress_host = _sig("hccx_lossless_compress_host", _st, _p, _u64, _p, _u64, C.POINTER(_u64), C.c_int)
hccx_lossless_decompress_host = _sig("hccx_lossless_decompress_host", _st, _p, _u64, _u64, _p, C.c_int)
hccx_lossless_frame_max_bytes = _sig("hccx_lossless_frame_max_bytes", _u64, _u64)
hccx_lossless_frame_encode = _sig("hccx_lossless_frame_encode", _st, _p, _u64, _p, _u64, _p)
hccx_lossless_frame_decode = _sig("hccx_lossless_frame_decode", _st, _p, _u64, _u64, _p, C.c_int, _p)
hccx_frame_status = _sig("hccx_frame_status", _st, _p)
hccx_lossless_ring_wire = _sig("hccx_lossless_ring_wire", _st, _pp, C.c_int, _u64, C.c_int, C.POINTER(_u64), _p)
hccx_lossless_ring_wire_host = _sig("hccx_lossless_ring_wire_host", _st, _pp, C.c_int, _u64, C.c_int,
                                    C.POINTER(_u64), C.c_int)
hccx_lossless_ring_hops = _sig("hccx_lossless_ring_hops", _st, _pp, C.c_int, _u64, C.c_int, C.POINTER(_u64), _p)
hccx_lossless_ring_hops_host = _sig("hccx_lossless_ring_hops_host", _st, _pp, C.c_int, _u64, C.c_int,
                                    C.POINTER(_u64), C.c_int)
hccx_group_create = _sig("hccx_group_create", _st, C.c_int, C.c_int, C.POINTER(_p))
hccx_group_destroy = _sig("hccx_group_destroy", _st, _p)
hccx_group_allreduce = _sig("hccx_group_allreduce", _st, _p, _pp, _pp, _u64, Codec, C.c_int, _p)
hccx_group_reduce_scatter = _sig("hccx_group_reduce_scatter", _st, _p, _pp, _pp, _u64, Codec, _p)
hccx_group_allgather = _sig("hccx_group_allgather", _st, _p, _pp, _pp, _u64, Codec, _p)
hccx_group_broadcast = _sig("hccx_group_broadcast", _st, _p, C.c_int, _p, _pp, _u64, Codec, _p)
hccx_group_p2p = _sig("hccx_group_p2p", _st, _p, _p, _p, _u64, Codec, _p)
hccx_group_status = _sig("hccx_group_status", _st, _p, _p)
_dp = C.POINTER(C.c_double)
hccx_group_allreduce_host = _sig("hccx_group_allreduce_host", _st, _p, _pp, _pp, _u64, Codec, C.c_int, _dp)
hccx_group_reduce_scatter_host = _sig("hccx_group_reduce_scatter_host", _st, _p, _pp, _pp, _u64, Codec, _dp)
hccx_group_allgather_host = _sig("hccx_group_allgather_host", _st, _p, _pp, _pp, _u64, Codec, _dp)
hccx_group_broadcast_host = _sig("hccx_group_broadcast_host", _st, _p, C.c_int, _p, _pp, _u64, Codec, _dp)
hccx_group_p2p_host = _sig("hccx_group_p2p_host", _st, _p, _p, _p, _u64, Codec, _dp)
hccx_comm_create = _sig("hccx_comm_create", _st, C.c_int, C.c_int, C.c_int, _u64, C.POINTER(_p))
hccx_comm_export = _sig("hccx_comm_export", _st, _p, _p)
hccx_comm_connect = _sig("hccx_comm_connect", _st, _p, _p)
hccx_comm_destroy = _sig("hccx_comm_destroy", _st, _p)
hccx_allreduce = _sig("hccx_allreduce", _st, _p, _p, _p, _u64, Codec, C.c_int, _p)
hccx_reduce_scatter = _sig("hccx_reduce_scatter", _st, _p, _p, _p, _u64, Codec, _p)
hccx_allgather = _sig("hccx_allgather", _st, _p, _p, _p, _u64, Codec, _p)
hccx_broadcast = _sig("hccx_broadcast", _st, _p, C.c_int, _p, _p, _u64, Codec, _p)
hccx_p2p = _sig("hccx_p2p", _st, _p, C.c_int, C.c_int, _p, _p, _u64, Codec, _p)
hccx_comm_status = _sig("hccx_comm_status", _st, _p, _p)
hccx_comm_trace_enable = _sig("hccx_comm_trace_enable", _st, _p, _u64)
hccx_comm_trace_read = _sig("hccx_comm_trace_read", _st, _p, C.POINTER(_u64), _u64, C.POINTER(_u64))
_ip = C.POINTER(C.c_int)
hccx_mcomm_create = _sig("hccx_mcomm_create", _st, C.c_int, _ip, _u64, C.POINTER(_p))
hccx_mcomm_destroy = _sig("hccx_mcomm_destroy", _st, _p)
hccx_mcomm_size = _sig("hccx_mcomm_size", C.c_int, _p)
hccx_mcomm_allreduce = _sig("hccx_mcomm_allreduce", _st, _p, _pp, _pp, _u64, Codec, C.c_int, _pp)
hccx_mcomm_reduce_scatter = _sig("hccx_mcomm_reduce_scatter", _st, _p, _pp, _pp, _u64, Codec, _pp)
hccx_mcomm_allgather = _sig("hccx_mcomm_allgather", _st, _p, _pp, _pp, _u64, Codec, _pp)
hccx_mcomm_broadcast = _sig("hccx_mcomm_broadcast", _st, _p, C.c_int, _p, _pp, _u64, Codec, _pp)
hccx_mcomm_p2p = _sig("hccx_mcomm_p2p", _st, _p, C.c_int, C.c_int, _p, _p, _u64, Codec, _pp)
hccx_mcomm_status = _sig("hccx_mcomm_status", _st, _p, _pp)
hccx_mcomm_allreduce_host = _sig("hccx_mcomm_allreduce_host", _st, _p, _pp, _pp, _u64, Codec, C.c_int, _dp)
hccx_mcomm_reduce_scatter_host = _sig("hccx_mcomm_reduce_scatter_host", _st, _p, _pp, _pp, _u64, Codec, _dp)
hccx_mcomm_allgather_host = _sig("hccx_mcomm_allgather_host", _st, _p, _pp, _pp, _u64, Codec, _dp)
hccx_mcomm_broadcast_host = _sig("hccx_mcomm_broadcast_host", _st, _p, C.c_int, _p, _pp, _u64, Codec, _dp)
hccx_mcomm_p2p_host = _sig("hccx_mcomm_p2p_host", _st, _p, C.c_int, C.c_int, _p, _p, _u64, Codec, _dp)
hccx_launch_count = _sig("hccx_launch_count", _u64)
hccx_device_count = _sig("hccx_device_count", C.c_int)
hccx_comm_wire_bytes = _sig("hccx_comm_wire_bytes", _st, _p, C.POINTER(_u64), C.POINTER(_u64))
hccx_mcomm_wire_bytes = _sig("hccx_mcomm_wire_bytes", _st, _p, C.c_int, C.POINTER(_u64), C.POINTER(_u64))
hccx_comm_recv_bytes = _sig("hccx_comm_recv_bytes", _st, _p, C.POINTER(_u64))

#: every symbol include/hccx.h declares (checked by tests/test_abi.py)
EXPORTED = [n for n in dir() if n.startswith("hccx_")]


def ptr_array(ptrs):
    """A C array of void* for the group (all-members) entry points."""
    arr = (C.c_void_p * len(ptrs))(*[C.c_void_p(int(p)) for p in ptrs])
    return C.cast(arr, _pp), arr
