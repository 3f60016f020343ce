"""NVLink engine sweep (run under torchrun): device time per op / codec / size,
max over ranks, next to NCCL allreduce.  Development tool; bench.py is the
contract."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_02423_b200 import CodecSpec  # noqa: E402
from paper_2409_02423_b200 import dist as D  # noqa: E402


def timed(fn, steps=int(os.environ.get("SWEEP_STEPS", "10")), warm=int(os.environ.get("SWEEP_WARM", "3"))):
    for _ in range(warm):
        fn()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()  # no fused kernel may be in flight across an NCCL call
    dist.barrier()
    torch.cuda.synchronize()
    if not int(os.environ.get("SWEEP_NOSLEEP", "0")):
        torch.cuda._sleep(int(2e6))
    a.record(s)
    for _ in range(steps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    ms = torch.tensor([a.elapsed_time(b) / steps], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    return float(ms.item())


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    rank, p = dist.get_rank(), dist.get_world_size()
    sizes = [int(s) for s in os.environ.get("SWEEP_SIZES", str(1 << 26)).split(",")]
    comm = D.NvlinkComm(max(sizes))
    import ctypes as C

    from paper_2409_02423_b200 import _lib
    cap = 1 << 16
    _lib.hccx_comm_trace_enable(comm.h, cap)

    def who():
        buf = (C.c_uint64 * cap)()
        nw = C.c_uint64()
        _lib.hccx_comm_trace_read(comm.h, buf, cap, C.byref(nw))
        n = min(buf[4000], 90)
        prog = [hex(buf[4200 + w]) for w in range(10)]
        return [hex(buf[4001 + i]) for i in range(n)][:3] + ["first:", hex(buf[4095]), "prog:"] + prog
    codecs = os.environ.get("SWEEP_CODECS", "identity,fixed-rate:4,fixed-rate:8,fixed-rate:16").split(",")
    ops = os.environ.get("SWEEP_OPS", "ar,rs,ag,nccl").split(",")
    for n in sizes:
        n -= n % (p * 2048)
        x = torch.randn(n, device="cuda") * 1e-3
        out = torch.empty_like(x)
        sh = torch.empty(n // p, device="cuda")
        for cs in codecs:
            from paper_2409_02423_b200.codec import codec_spec_from_string

            spec = codec_spec_from_string(cs)
            row = {"p": p, "n": n, "codec": cs}
            if "ar" in ops:
                row["ar_ms"] = timed(lambda: comm.allreduce(x, spec, 0, out))
            if "rs" in ops:
                row["rs_ms"] = timed(lambda: comm.reduce_scatter(x, spec, sh))
            if "ag" in ops:
                row["ag_ms"] = timed(lambda: comm.allgather(sh, spec, out))
            if "bc" in ops:
                row["bc_ms"] = timed(lambda: comm.broadcast(x, 0, spec, out))
            if "pp" in ops:
                row["pp_ms"] = timed(lambda: comm.p2p(x, 0, 1, spec, out if rank == 1 else None))
                row["pp_GBps_raw"] = round(4 * n / (row["pp_ms"] * 1e-3) / 1e9, 1)
            if "ar_ms" in row:
                row["ar_GBps"] = round(4 * n / (row["ar_ms"] * 1e-3) / 1e9, 1)
            try:
                comm.status()
            except Exception as e:
                print(f"rank {rank} {cs} n={n}: {e} who={who()}", flush=True)
                raise
            if rank == 0:
                print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in row.items()}), flush=True)
        if "sendrecv" in ops:
            y = x.clone()

            def sr():
                if rank == 0:
                    dist.send(y, 1)
                elif rank == 1:
                    dist.recv(y, 0)
            ms = timed(sr)
            if rank == 0:
                print(json.dumps({"p": p, "n": n, "nccl_sendrecv_ms": round(ms, 4),
                                  "sendrecv_GBps": round(4 * n / (ms * 1e-3) / 1e9, 1)}), flush=True)
        if "nccl" in ops:
            y = x.clone()
            ms = timed(lambda: dist.all_reduce(y))
            if rank == 0:
                print(json.dumps({"p": p, "n": n, "nccl_ar_ms": round(ms, 4),
                                  "nccl_GBps": round(4 * n / (ms * 1e-3) / 1e9, 1)}), flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
