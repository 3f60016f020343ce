"""BASELINE configs 3-5 on the NVLink engine (run under torchrun, N GPUs).

  sweep   config 3: allreduce message sizes 4 KiB .. 1 GiB at rates 4/8/16,
          next to the uncompressed NCCL allreduce (algbw = bytes / time)
  hybrid  config 4: z-hybrid:16,4 on GPT-NeoX-20B-shaped traffic -- TP
          allreduce of [4, 2048, 6144] fp32 at rate 16, PP send/recv of the
          same tensor at rate 16, DP gradient allreduce (256 MiB bucket,
          Average) at rate 4; each dimension gets the whole box in turn
          (tp = N, pp = N, dp = N) because one box has N <= 8 GPUs
  zero    config 5: ZeRO-1 reduce-scatter of a 2 GiB fp32 gradient buffer plus
          all-gather of the parameters, rates 16 and 8
  mz      MZHybrid's LosslessPredictor paths with the compressed bytes on the
          wire (TP allreduce, PP send/recv), traced wire bytes

Device time per call, max over ranks.  Prints one JSON line per row on
rank 0.  Development/evidence tool; bench.py is the driver contract.
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_02423_b200 import CodecSpec, ParallelLayout, scheme_from_name  # noqa: E402
from paper_2409_02423_b200 import dist as D  # noqa: E402
from paper_2409_02423_b200.hybrid import HybridComm  # noqa: E402


def timed(fn, steps, warm=2):
    for _ in range(warm):
        fn()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()  # no fused kernel may be in flight across an NCCL call
    dist.barrier()
    torch.cuda.synchronize()
    torch.cuda._sleep(int(2e6))
    a.record(s)
    for _ in range(steps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    ms = torch.tensor([a.elapsed_time(b) / steps], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    return float(ms.item())


def emit(rank, row):
    if rank == 0:
        print(json.dumps(row), flush=True)


def sweep(rank, p):
    sizes = [4096 * 4 ** k for k in range(11)]  # 4 KiB .. 4 GiB, trimmed below
    sizes = [s for s in sizes if s <= (1 << 30)] + [1 << 30]
    sizes = sorted(set(sizes))
    comm = D.NvlinkComm((1 << 30) // 4)
    for nbytes in sizes:
        n = max(nbytes // 4, p)
        n -= n % p
        x = torch.randn(n, device="cuda") * 1e-3
        out = torch.empty_like(x)
        steps = 20 if nbytes < (64 << 20) else 5
        row = {"config": "sweep", "p": p, "bytes": 4 * n}
        for r in (4, 8, 16):
            ms = timed(lambda: comm.allreduce(x, CodecSpec.fixed_rate(r), 0, out), steps)
            row[f"r{r}_us"] = round(ms * 1e3, 2)
            row[f"r{r}_GBps"] = round(4 * n / (ms * 1e-3) / 1e9, 1)
        y = x.clone()
        ms = timed(lambda: dist.all_reduce(y), steps)
        row["nccl_us"] = round(ms * 1e3, 2)
        row["nccl_GBps"] = round(4 * n / (ms * 1e-3) / 1e9, 1)
        comm.status()
        emit(rank, row)
        del x, out, y
    comm.close()


def hybrid(rank, p):
    scheme = scheme_from_name("z-hybrid:16,4")
    act = (4, 2048, 6144)  # micro-batch x seq x hidden (GPT-NeoX-20B; external assumption)
    n_act = act[0] * act[1] * act[2]
    n_grad = 1 << 26  # 256 MiB DP gradient bucket
    for name, lay in (("tp", ParallelLayout(1, 1, p)), ("pp", ParallelLayout(1, p, 1)), ("dp", ParallelLayout(p, 1, 1))):
        hc = HybridComm(lay, scheme, max(n_act, n_grad) + p)
        if name == "tp":
            x = torch.randn(n_act, device="cuda")
            ms = timed(lambda: hc.tp_allreduce(x), 10)
            y = x.clone()
            nccl = timed(lambda: dist.all_reduce(y), 10)
            path, rate, n = "TpAllReduce", 16, n_act
        elif name == "pp":
            x = torch.randn(n_act, device="cuda")
            ms = timed(lambda: hc.pp_send_recv(x, 0, 1), 10)
            y = x.clone()

            def sr():
                if rank == 0:
                    dist.send(y, 1)
                elif rank == 1:
                    dist.recv(y, 0)
            nccl = timed(sr, 10)
            path, rate, n = "PpP2p", 16, n_act
        else:
            x = torch.randn(n_grad, device="cuda") * 1e-3
            ms = timed(lambda: hc.dp_allreduce(x), 10)
            y = x.clone()
            nccl = timed(lambda: dist.all_reduce(y), 10)
            path, rate, n = "DpAllReduce(Average)", 4, n_grad
        hc.status()
        ev = hc.trace[-1] if hc.trace else None
        emit(rank, {"config": "hybrid z-hybrid:16,4", "path": path, "rate_bits": rate, "p": p, "values": n,
                    "us": round(ms * 1e3, 2), "GBps": round(4 * n / (ms * 1e-3) / 1e9, 1),
                    "nccl_us": round(nccl * 1e3, 2), "nccl_GBps": round(4 * n / (nccl * 1e-3) / 1e9, 1),
                    "trace_raw_bytes": ev.raw_bytes if ev else None, "trace_wire_bytes": ev.wire_bytes if ev else None})
        hc.close()
        del x, y


def mz(rank, p):
    """MZHybrid's lossless paths on the wire (csrc/lossless_comm.cu): TP
    allreduce and PP send/recv under LosslessPredictor, 16 MiB of smooth
    (compressible) and of random activations; traced wire bytes are the
    framed payloads the engine pushed."""
    scheme = scheme_from_name("mz-hybrid:8")
    n = 1 << 22
    for name, lay in (("tp", ParallelLayout(1, 1, p)), ("pp", ParallelLayout(1, p, 1))):
        hc = HybridComm(lay, scheme, n + p)
        for data in ("smooth", "random"):
            if data == "smooth":
                t = torch.arange(n, device="cuda", dtype=torch.float32)
                x = torch.sin(t * 1e-4 + rank) * 1e-2
                x = (x * 4096).round() / 4096  # few mantissa bits: what the XOR predictor compresses
            else:
                x = torch.randn(n, device="cuda")
            if name == "tp":
                ms = timed(lambda: hc.tp_allreduce(x), 3, 1)
                path = "TpAllReduce"
            else:
                ms = timed(lambda: hc.pp_send_recv(x, 0, 1), 3, 1)
                path = "PpP2p"
            ev = hc.trace[-1] if hc.trace else None
            emit(rank, {"config": "mz-hybrid:8 lossless on the wire", "path": path, "data": data, "p": p,
                        "values": n, "us": round(ms * 1e3, 1), "GBps": round(4 * n / (ms * 1e-3) / 1e9, 2),
                        "trace_raw_bytes": ev.raw_bytes if ev else None,
                        "trace_wire_bytes": ev.wire_bytes if ev else None})
        hc.status()
        hc.close()


def zero(rank, p):
    n = (1 << 29) - ((1 << 29) % p)  # 2 GiB fp32
    comm = D.NvlinkComm(n)
    g = torch.randn(n, device="cuda") * 1e-3
    shard = torch.empty(n // p, device="cuda")
    full = torch.empty(n, device="cuda")
    for r in (16, 8):
        spec = CodecSpec.fixed_rate(r)
        rs = timed(lambda: comm.reduce_scatter(g, spec, shard), 3, 1)
        ag = timed(lambda: comm.allgather(shard, spec, full), 3, 1)
        comm.status()
        emit(rank, {"config": "zero 2GiB", "rate_bits": r, "p": p, "rs_us": round(rs * 1e3, 1),
                    "ag_us": round(ag * 1e3, 1), "rs_GBps": round(4 * n / (rs * 1e-3) / 1e9, 1),
                    "ag_GBps": round(4 * n / (ag * 1e-3) / 1e9, 1)})
    del g, shard, full
    torch.cuda.empty_cache()
    # NCCL reduce_scatter + all_gather of the same buffer (uncompressed)
    g = torch.randn(n, device="cuda")
    sh = torch.empty(n // p, device="cuda")
    rs = timed(lambda: dist.reduce_scatter_tensor(sh, g), 3, 1)
    ag = timed(lambda: dist.all_gather_into_tensor(g, sh), 3, 1)
    emit(rank, {"config": "zero 2GiB", "nccl": True, "p": p, "rs_us": round(rs * 1e3, 1), "ag_us": round(ag * 1e3, 1),
                "rs_GBps": round(4 * n / (rs * 1e-3) / 1e9, 1), "ag_GBps": round(4 * n / (ag * 1e-3) / 1e9, 1)})
    comm.close()


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    rank, p = dist.get_rank(), dist.get_world_size()
    which = os.environ.get("CONFIGS", "sweep,hybrid,zero").split(",")
    if "sweep" in which:
        sweep(rank, p)
    if "hybrid" in which:
        hybrid(rank, p)
    if "zero" in which:
        zero(rank, p)
    if "mz" in which:
        mz(rank, p)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
