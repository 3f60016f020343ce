"""Randomized soak of the NVLink engine (run under torchrun, >= 2 GPUs):
SOAK_ITERS random collectives -- op, size (one-shot / ring / direct and ring
gather regimes), codec, reduce mode, in-place or not -- issued back to back
without host synchronisation between them, every result checked bit for bit
against the CPU oracle.  Exit 0 iff all matched."""
import os
import random
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


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    rank, p = dist.get_rank(), dist.get_world_size()
    iters = int(os.environ.get("SOAK_ITERS", "200"))
    rng = random.Random(1234)  # same sequence on every rank
    comm = D.NvlinkComm((1 << 23) * p)
    codecs = [("identity", 0, CodecSpec.identity()), ("fixed-rate", 8, CodecSpec.fixed_rate(8)),
              ("fixed-rate", 4, CodecSpec.fixed_rate(4)), ("fixed-rate", 13, CodecSpec.fixed_rate(13)),
              ("fixed-rate", 16, CodecSpec.fixed_rate(16)), ("zfp-rate", 8, CodecSpec.zfp_rate(8))]
    fails = []
    pending = []  # (name, tensor, expected) checked in batches, so calls queue back to back
    for it in range(iters):
        kind, rate, spec = rng.choice(codecs)
        op = rng.choice(["ar", "ar", "rs", "ag", "bc", "pp"])
        n_per = rng.choice([64, 1000, 4096, 70000, 1 << 18, 1 << 20, (1 << 21) + 256])
        n = n_per * p
        seed = it * 101
        xs = np.stack([O.fill(seed + 7 * j, "uniform", n) for j in range(p)])
        x = torch.from_numpy(xs[rank]).cuda()
        if op == "ar":
            avg = rng.randint(0, 1)
            inplace = rng.randint(0, 1)
            out = x.clone() if inplace else None
            got = comm.allreduce(out if inplace else x, spec, avg, out)
            pending.append((f"{it} ar {kind}{rate} n={n}", got, lambda xs=xs, a=avg, k=kind, r=rate:
                            O.allreduce(xs, k, r, bool(a))[0][rank]))
        elif op == "rs":
            got = comm.reduce_scatter(x, spec)
            pending.append((f"{it} rs {kind}{rate} n={n}", got, lambda xs=xs, k=kind, r=rate:
                            O.reduce_scatter(xs, k, r)[0][rank]))
        elif op == "ag":
            sh = np.ascontiguousarray(xs[:, :n_per])
            got = comm.allgather(torch.from_numpy(sh[rank]).cuda(), spec)
            pending.append((f"{it} ag {kind}{rate} n={n_per}", got, lambda sh=sh, k=kind, r=rate:
                            O.allgather(sh, k, r)[0][rank]))
        elif op == "bc":
            root = rng.randrange(p)
            got = comm.broadcast(torch.from_numpy(xs[root]).cuda(), root, spec)
            pending.append((f"{it} bc {kind}{rate}", got, lambda xs=xs, root=root, k=kind, r=rate:
                            O.broadcast(xs[root], p, k, r)[0][rank]))
        else:
            src = rng.randrange(p)
            dst = (src + rng.randrange(1, p)) % p
            got = comm.p2p(torch.from_numpy(xs[src]).cuda(), src, dst, spec)
            if rank == dst:
                pending.append((f"{it} pp {kind}{rate}", got, lambda xs=xs, src=src, k=kind, r=rate:
                                O.p2p(xs[src], k, r)[0]))
        if len(pending) >= 8 or it == iters - 1:
            comm.status()
            for name, t, want in pending:
                if t.cpu().numpy().tobytes() != np.ascontiguousarray(want()).tobytes():
                    fails.append(name)
            pending = []
    nf = torch.tensor([len(fails)], device="cuda")
    torch.cuda.synchronize()
    dist.all_reduce(nf)
    if fails:
        print(f"rank {rank} FAILS: {fails[:10]}", flush=True)
    comm.close()
    if rank == 0:
        print(f"NVLINK SOAK {'OK' if nf.item() == 0 else 'FAILED'} p={p} iters={iters} fails={int(nf.item())}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if nf.item() == 0 else 1)


if __name__ == "__main__":
    main()
