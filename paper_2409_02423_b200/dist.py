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

    def close(self) -> None:
        import torch.distributed as dist

        if self.h:
            import torch

            torch.cuda.synchronize(self.device)
            dist.barrier(self.group)
            self._lib.hccx_comm_destroy(self.h)
            self.h = None


def bench_allreduce_main(args, metric, ClockSampler, peaks, traffic_for, cpu_allreduce, host_threads):
    """bench.py N>1 leg (BASELINE config 2): compressed allreduce of a 256 MiB
    fp32 bucket per rank through NvlinkComm, uncompressed NCCL allreduce
    beside it, max-over-ranks device time."""
    import json
    import os
    import time

    import torch
    import torch.distributed as dist

    from . import _lib
    from .codec import wire_size_bytes

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    rank, world = dist.get_rank(), dist.get_world_size()
    n = args.n or (1 << 26)  # 256 MiB fp32 per rank
    n -= n % world
    rate = args.rate
    spec = CodecSpec.fixed_rate(rate)
    comm = NvlinkComm(n)
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    x = torch.randn(n, device="cuda", generator=g) * 1e-3
    out = torch.empty_like(x)
    s = torch.cuda.current_stream()

    def timed(fn, steps):
        import gc

        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()  # no fused kernel may be in flight across an NCCL call
        dist.barrier()
        torch.cuda.synchronize()
        gc.disable()  # a collection pause on one rank's host would stall every peer
        try:
            torch.cuda._sleep(int(1e6))
            t0.record(s)
            for _ in range(steps):
                fn()
            t1.record(s)
            torch.cuda.synchronize()
        finally:
            gc.enable()
        ms = torch.tensor([t0.elapsed_time(t1) / steps], device="cuda")
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return float(ms.item())

    for _ in range(args.warmup):
        comm.allreduce(x, spec, 0, out)
    comm.status()
    launches0 = _lib.hccx_launch_count()
    with ClockSampler(local) as clk:
        ms = timed(lambda: comm.allreduce(x, spec, 0, out), args.steps)
    launches = _lib.hccx_launch_count() - launches0
    comm.status()
    # agreement: every rank holds bit-identical results
    h = torch.tensor([int(out.view(torch.int32).to(torch.int64).sum().item())], device="cuda")
    hs = [torch.zeros_like(h) for _ in range(world)]
    dist.all_gather(hs, h)
    assert len({int(t.item()) for t in hs}) == 1, "ranks disagree"

    # uncompressed NCCL allreduce on the same buffer size
    nccl_ms = None
    if args.nccl:
        y = x.clone()
        for _ in range(args.warmup):
            dist.all_reduce(y)
        nccl_ms = timed(lambda: dist.all_reduce(y), args.steps)

    # e2e through the C ABI with pinned host buffers: H2D + allreduce + D2H per step
    hx = torch.empty(n, dtype=torch.float32, pin_memory=True)
    hx.copy_(x.cpu())
    hy = torch.empty(n, dtype=torch.float32, pin_memory=True)
    dx = torch.empty_like(x)
    e2e_steps = max(3, min(args.steps, 10))

    def e2e_step():
        dx.copy_(hx, non_blocking=True)
        comm.allreduce(dx, spec, 0, out)
        hy.copy_(out, non_blocking=True)

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    dist.barrier()
    w0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    torch.cuda.synchronize()
    e2e_s = torch.tensor([(time.perf_counter() - w0) / e2e_steps], device="cuda")
    dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_s = float(e2e_s.item())

    cpu = None
    if rank == 0:
        ref_n = args.ref_n or (1 << 20)
        sec, kind = cpu_allreduce(world, ref_n, rate, reps=1)
        cpu = {"value": round(4 * ref_n / sec / 1e9, 5), "unit": "GB/s",
               "cores": host_threads() if kind == "reference" else 1, "kind": kind,
               "sample": f"hcc::allreduce of {ref_n} values per rank, p={world} ranks simulated in one process "
                         f"(the reference design), fixed-rate:{rate}"}

    hbm, peak_src = peaks()
    c = n // world
    W = wire_size_bytes(spec, c)
    p = world
    # per-rank algorithmic bytes of the fused kernel
    hbm_bytes = (p - 1) * (4 * c + 2 * W) + (4 * c + W) + p * (W + 4 * c)
    wire_bytes = 2 * (p - 1) * W
    t = ms * 1e-3
    nvl_peak = 770.0
    hbm_ach = hbm_bytes / t / 1e9
    nvl_ach = wire_bytes / t / 1e9
    bound = "hbm" if hbm_bytes / (hbm * 1e9) >= wire_bytes / (nvl_peak * 1e9) else "nvlink"
    if rank == 0:
        line = {
            "metric": metric, "value": round(4 * n / t / 1e9, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (torch.randn * 1e-3 fp32 gradients, seed 1234+rank)",
            "config": {"workload": "allreduce: compressed ring allreduce of a 256 MiB fp32 bucket per rank "
                                   "(BASELINE config 2)", "n_values_per_rank": n, "rate_bits": rate,
                       "parallelism": f"dp{world}", "l2": "inputs larger than L2 (256 MiB per rank)",
                       "engine": "one persistent fused kernel per rank, NVLink peer pushes (CUDA IPC)",
                       "wire_bytes_per_rank": wire_bytes,
                       "nccl_allreduce_GBps": round(4 * n / (nccl_ms * 1e-3) / 1e9, 2) if nccl_ms else None,
                       "nccl_ms": round(nccl_ms, 5) if nccl_ms else None},
            "roofline": {"bound": bound, "kernel": "ring_fused_kernel",
                         "achieved": round(hbm_ach if bound == "hbm" else nvl_ach, 1),
                         "peak": hbm if bound == "hbm" else nvl_peak, "unit": "GB/s",
                         "frac": round((hbm_ach / hbm) if bound == "hbm" else (nvl_ach / nvl_peak), 4),
                         "peak_source": peak_src if bound == "hbm" else "B200_PROFILING.md measured peer copy",
                         "hbm_bytes_per_launch": hbm_bytes, "nvlink_bytes_per_launch": wire_bytes,
                         "hbm_frac": round(hbm_ach / hbm, 4), "nvlink_frac": round(nvl_ach / nvl_peak, 4),
                         "traffic": traffic_for("ring_fused")},
            "cpu_baseline": cpu,
            "e2e": {"value": round(4 * n / e2e_s / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": 4 * n,
                    "d2h_bytes_per_step": 4 * n, "api": "hccx_allreduce (C ABI) with pinned host in/out",
                    "timer": "host wall clock, device synced, max over ranks"},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    comm.close()
    dist.destroy_process_group()
