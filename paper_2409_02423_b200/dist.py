"""Compressed collectives across processes, one GPU each, over NVLink.

``NvlinkComm`` wraps the C ABI communicator (include/hccx.h, hccx_comm_*):
every rank allocates a CUDA-IPC window, the opaque handles are all-gathered
with torch.distributed (plumbing only), and from then on each collective is
ONE persistent kernel per rank (csrc/ring_fused.cuh) that pushes compressed
segments into the peers' windows and fuses decompress-add-recompress per
ring hop.  The results are bit-identical to the reference ring
(proj/src/collectives.cpp) -- the same bits the single-device path and the CPU
oracle produce.

Semantics per rank (this process's buffer only), reference analogues:
  allreduce(x, spec, mode)    hcc::allreduce          collectives.cpp:202-248
  reduce_scatter(x, spec)     hcc::ring_reduce_scatter collectives.cpp:154-181
  allgather(shard, spec)      hcc::ring_allgather     collectives.cpp:183-200
  broadcast(x, root, spec)    not in the reference
  p2p(x, src, dst, spec)      hcc::p2p                collectives.cpp:130-152
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional

from .codec import CodecSpec
from .errors import check


def exchange_handles(blob: bytes, group=None) -> List[bytes]:
    """All-gather one opaque byte blob per rank (rank order of ``group``)."""
    import torch.distributed as dist

    out: list = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(blob), group=group)
    return [bytes(b) for b in out]


class NvlinkComm:
    """One hccx communicator over the ranks of a torch.distributed group.

    Each collective is one cooperative kernel that occupies every SM and
    spins on peer flags; do not keep NCCL (or other peer-waiting) kernels in
    flight on other streams across a call -- synchronise first, as
    ``timed()`` in the tools and bench.py do."""

    def __init__(self, max_n: int, group=None, device: Optional[int] = None):
        import torch
        import torch.distributed as dist

        from . import _lib

        self._lib = _lib
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.device = torch.cuda.current_device() if device is None else device
        self.max_n = int(max_n)
        h = C.c_void_p()
        check(_lib.hccx_comm_create(self.rank, self.size, self.device, self.max_n, C.byref(h)), "comm_create")
        self.h = h.value
        blob = (C.c_uint8 * _lib.HANDLE_BYTES)()
        check(_lib.hccx_comm_export(self.h, blob), "comm_export")
        allb = exchange_handles(bytes(blob), group)
        buf = (C.c_uint8 * (_lib.HANDLE_BYTES * self.size)).from_buffer_copy(b"".join(allb))
        check(_lib.hccx_comm_connect(self.h, buf), "comm_connect")
        # The fused collectives are cooperative kernels that occupy every SM
        # and wait on peers; an NCCL kernel still in flight on another stream
        # (this barrier's) could then never be scheduled on one rank while its
        # peer waits for it.  Drain it before the first collective.
        torch.cuda.synchronize(self.device)
        dist.barrier(group)
        torch.cuda.synchronize(self.device)

    # ------------------------------------------------------------------
    def _stream(self) -> int:
        import torch

        return torch.cuda.current_stream(self.device).cuda_stream

    def status(self) -> None:
        """Synchronise and raise NonFiniteInputError / PeerTimeoutError if the
        device error flag is set."""
        check(self._lib.hccx_comm_status(self.h, self._stream()), "comm")

    def allreduce(self, x, spec: CodecSpec, mode: int = 0, out=None):
        import torch

        out = torch.empty_like(x) if out is None else out
        check(self._lib.hccx_allreduce(self.h, x.data_ptr(), out.data_ptr(), x.numel(), spec.c(), int(mode),
                                       self._stream()), "allreduce")
        return out

    def reduce_scatter(self, x, spec: CodecSpec, out=None):
        import torch

        out = torch.empty(x.numel() // self.size, dtype=x.dtype, device=x.device) if out is None else out
        check(self._lib.hccx_reduce_scatter(self.h, x.data_ptr(), out.data_ptr(), x.numel(), spec.c(),
                                            self._stream()), "reduce_scatter")
        return out

    def allgather(self, shard, spec: CodecSpec, out=None):
        import torch

        out = torch.empty(shard.numel() * self.size, dtype=shard.dtype, device=shard.device) if out is None else out
        check(self._lib.hccx_allgather(self.h, shard.data_ptr(), out.data_ptr(), shard.numel(), spec.c(),
                                       self._stream()), "allgather")
        return out

    def broadcast(self, x, root: int, spec: CodecSpec, out=None):
        import torch

        out = torch.empty_like(x) if out is None else out
        check(self._lib.hccx_broadcast(self.h, root, x.data_ptr() if self.rank == root else None, out.data_ptr(),
                                       x.numel(), spec.c(), self._stream()), "broadcast")
        return out

    def p2p(self, x, src: int, dst: int, spec: CodecSpec, out=None):
        """Both src and dst call; dst receives dec(comp(src's x))."""
        import torch

        if self.rank == dst and out is None:
            out = torch.empty_like(x)
        check(self._lib.hccx_p2p(self.h, src, dst, x.data_ptr() if self.rank == src else None,
                                 out.data_ptr() if out is not None else None, x.numel(), spec.c(), self._stream()),
              "p2p")
        return out

    def wire_bytes(self):
        """(payload, frame) bytes this rank pushed in its last collective
        (hccx_comm_wire_bytes): the size law for fixed-size codecs, the
        framed messages actually sent under LosslessPredictor."""
        a, b = C.c_uint64(), C.c_uint64()
        check(self._lib.hccx_comm_wire_bytes(self.h, C.byref(a), C.byref(b)), "wire_bytes")
        return int(a.value), int(b.value)

    def recv_bytes(self) -> int:
        """Framed payload bytes this rank received in its last collective."""
        a = C.c_uint64()
        check(self._lib.hccx_comm_recv_bytes(self.h, C.byref(a)), "recv_bytes")
        return int(a.value)

    def close(self) -> None:
        import torch.distributed as dist

        if self.h:
            import torch

            torch.cuda.synchronize(self.device)
            dist.barrier(self.group)
            self._lib.hccx_comm_destroy(self.h)
            self.h = None
