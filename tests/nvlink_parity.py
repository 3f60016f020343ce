"""Multi-process NVLink engine parity (run under torchrun, >= 2 GPUs).

Every rank regenerates all ranks' inputs deterministically, runs the fused
NVLink collectives on its own GPU, and compares its own result bit-for-bit
with the CPU oracle (oracle/hcc_oracle.c, pinned to the reference).  Exit
code 0 iff every case on every rank matched.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import oracle_lib as O  # noqa: E402
from paper_2409_02423_b200 import CodecSpec  # noqa: E402
from paper_2409_02423_b200 import dist as D  # noqa: E402


def spec_of(kind, rate):
    if kind == "identity":
        return CodecSpec.identity()
    if kind == "zfp-rate":
        return CodecSpec.zfp_rate(rate)
    return CodecSpec.fixed_rate(rate)


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    rank, p = dist.get_rank(), dist.get_world_size()
    big = int(os.environ.get("HCCX_PARITY_BIG", "1"))
    comm = D.NvlinkComm((1 << 24) * p)
    fails = []

    def cmp(name, got, want):
        g = got.cpu().numpy() if hasattr(got, "cpu") else got
        if g.tobytes() != np.ascontiguousarray(want).tobytes():
            fails.append(name)

    codecs = [("identity", 0), ("fixed-rate", 2), ("fixed-rate", 3), ("fixed-rate", 4), ("fixed-rate", 8),
              ("fixed-rate", 12), ("fixed-rate", 16), ("fixed-rate", 24), ("fixed-rate", 32), ("zfp-rate", 8)]
    seed = 100
    for kind, rate in codecs:
        spec = spec_of(kind, rate)
        for n_per in (64, 100, 2048, 5000, 8192 + 256, 70000):
            seed += 1
            n = n_per * p
            xs = np.stack([O.fill(seed * 31 + j, "uniform", n) for j in range(p)])
            x = torch.from_numpy(xs[rank]).cuda()
            for avg in (0, 1):
                got = comm.allreduce(x, spec, avg)
                want, _ = O.allreduce(xs, kind, rate, bool(avg))
                cmp(f"ar {kind}{rate} n={n} avg={avg}", got, want[rank])
            got = comm.reduce_scatter(x, spec)
            want, _ = O.reduce_scatter(xs, kind, rate)
            cmp(f"rs {kind}{rate} n={n}", got, want[rank])
            shards = np.ascontiguousarray(xs[:, :n_per])
            got = comm.allgather(torch.from_numpy(shards[rank]).cuda(), spec)
            want, _ = O.allgather(shards, kind, rate)
            cmp(f"ag {kind}{rate} n={n_per}", got, want[rank])
            for root in (0, p - 1):
                got = comm.broadcast(torch.from_numpy(xs[root]).cuda(), root, spec)
                want, _ = O.broadcast(xs[root], p, kind, rate)
                cmp(f"bcast {kind}{rate} root={root}", got, want[rank])
            got = comm.p2p(torch.from_numpy(xs[0]).cuda(), 0, p - 1, spec)
            if rank == p - 1:
                want, _ = O.p2p(xs[0], kind, rate)
                cmp(f"p2p {kind}{rate}", got, want)
            comm.status()
    # back-to-back collectives without host sync (exercise the slot acks)
    spec = CodecSpec.fixed_rate(8)
    xs = np.stack([O.fill(7 + j, "normal", 65536 * p, 1e-3) for j in range(p)])
    x = torch.from_numpy(xs[rank]).cuda()
    outs = [comm.allreduce(x, spec) for _ in range(10)] + [comm.reduce_scatter(x, spec) for _ in range(5)]
    shard = torch.from_numpy(np.ascontiguousarray(xs[rank, :65536])).cuda()
    ags = [comm.allgather(shard, spec) for _ in range(5)]
    bcs = [comm.broadcast(x, 1 % p, spec) for _ in range(5)]
    p2ps = [comm.p2p(x, 0, p - 1, spec) for _ in range(5)]
    comm.status()
    want_ar = O.allreduce(xs, "fixed-rate", 8)[0][rank]
    want_rs = O.reduce_scatter(xs, "fixed-rate", 8)[0][rank]
    want_ag = O.allgather(np.ascontiguousarray(xs[:, :65536]), "fixed-rate", 8)[0][rank]
    want_bc = O.broadcast(xs[1 % p], p, "fixed-rate", 8)[0][rank]
    for i, o in enumerate(outs):
        cmp(f"b2b {i}", o, want_ar if i < 10 else want_rs)
    for i, o in enumerate(ags):
        cmp(f"b2b ag {i}", o, want_ag)
    for i, o in enumerate(bcs):
        cmp(f"b2b bc {i}", o, want_bc)
    if rank == p - 1:
        want_pp = O.p2p(xs[0], "fixed-rate", 8)[0]
        for i, o in enumerate(p2ps):
            cmp(f"b2b p2p {i}", o, want_pp)
    # in place
    xi = torch.from_numpy(xs[rank].copy()).cuda()
    comm.allreduce(xi, spec, 1, out=xi)
    cmp("inplace", xi, O.allreduce(xs, "fixed-rate", 8, True)[0][rank])
    if big:
        n = 1 << 24
        xs = np.stack([O.fill(1234 + j, "normal", n, 1e-3) for j in range(p)])
        got = comm.allreduce(torch.from_numpy(xs[rank]).cuda(), spec, 1)
        cmp("big ar r8", got, O.allreduce(xs, "fixed-rate", 8, True)[0][rank])
    # mz-hybrid over the NVLink engine: lossless TP / ZeRO / PP paths (values
    # via the transparent ring, TraceEvent bytes sized on the device) and the
    # fixed-rate DP path, against the oracle's values and accounting
    from paper_2409_02423_b200 import ParallelLayout, scheme_from_name
    from paper_2409_02423_b200.hybrid import HybridComm

    torch.cuda.synchronize()
    scheme = scheme_from_name("mz-hybrid:8")
    n = 3000 * p
    xs = np.stack([O.fill(900 + j, "sparse" if j % 2 else "normal", n, 0.6 if j % 2 else 1e-3) for j in range(p)])
    x = torch.from_numpy(xs[rank]).cuda()
    for lay_name, lay in (("tp", ParallelLayout(1, 1, p)), ("dp", ParallelLayout(p, 1, 1)), ("pp", ParallelLayout(1, p, 1))):
        hc = HybridComm(lay, scheme, n)
        if lay_name == "tp":
            got = hc.tp_allreduce(x)
            want, acct = O.allreduce(xs, "lossless", 0, False)
            cmp("mz tp ar", got, want[rank])
            ev = hc.trace[-1]
            if (ev.raw_bytes, ev.wire_bytes, ev.round_count) != acct:
                fails.append(f"mz tp acct {(ev.raw_bytes, ev.wire_bytes, ev.round_count)} != {acct}")
            sh = torch.from_numpy(np.ascontiguousarray(xs[rank, :3000])).cuda()
            got = hc.tp_allgather(sh)
            want, acct = O.allgather(np.ascontiguousarray(xs[:, :3000]), "lossless")
            cmp("mz tp ag", got, want[rank])
            ev = hc.trace[-1]
            if (ev.raw_bytes, ev.wire_bytes, ev.round_count) != acct:
                fails.append(f"mz tp ag acct {(ev.raw_bytes, ev.wire_bytes, ev.round_count)} != {acct}")
        elif lay_name == "dp":
            got = hc.dp_allreduce(x)
            want, acct = O.allreduce(xs, "fixed-rate", 8, True)
            cmp("mz dp ar", got, want[rank])
            if hc.trace[-1].wire_bytes != acct[1]:
                fails.append("mz dp acct")
            got = hc.zero_reduce_scatter(x)
            want, acct = O.reduce_scatter(xs, "lossless")
            cmp("mz zero rs", got, want[rank])
            ev = hc.trace[-1]
            if (ev.raw_bytes, ev.wire_bytes, ev.round_count) != acct:
                fails.append(f"mz zero rs acct {(ev.raw_bytes, ev.wire_bytes, ev.round_count)} != {acct}")
        else:
            got = hc.pp_send_recv(x, 0, p - 1)
            if rank == p - 1:
                want, acct = O.p2p(xs[0], "lossless")
                cmp("mz pp", got, want)
                if hc.trace[-1].wire_bytes != acct[1]:
                    fails.append("mz pp acct")
        hc.status()
        torch.cuda.synchronize()
        hc.close()
    # non-finite partial sums are reported, not hung
    bad = torch.full((4096 * p,), 3.0e38, device="cuda")
    comm.allreduce(bad, spec)
    try:
        comm.status()
        fails.append("nonfinite not reported")
    except Exception as e:  # NonFiniteInputError
        if "non-finite" not in str(e):
            fails.append(f"wrong error {e}")
    nf = torch.tensor([len(fails)], device="cuda")
    dist.all_reduce(nf)
    if fails:
        print(f"rank {rank} FAILS ({len(fails)}): {fails[:12]}", flush=True)
    comm.close()
    if rank == 0:
        print(f"NVLINK PARITY {'OK' if nf.item() == 0 else 'FAILED'} p={p} total_fail={int(nf.item())}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if nf.item() == 0 else 1)


if __name__ == "__main__":
    main()
