"""Multi-process Trainer3D (trainer_dist.py) vs the reference trainer's runs
(tests/golden/trainer.npz), one GPU per rank; run under torchrun.  Runs every
golden case whose layout world equals WORLD_SIZE.  Exit 0 iff all match."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
sys.path.insert(0, os.path.dirname(HERE))

from make_golden import SMALL_CFG, TRAIN_CASES  # noqa: E402

from paper_2409_02423_b200 import build_layout, scheme_from_name  # noqa: E402
from paper_2409_02423_b200 import trainer as T  # noqa: E402
from paper_2409_02423_b200.comm_path import CommPath  # noqa: E402
from paper_2409_02423_b200.trainer_dist import DistTrainer3D  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    world, rank = dist.get_world_size(), dist.get_rank()
    g = np.load(os.path.join(HERE, "golden", "trainer.npz"))
    fails, ran = [], []
    for name, over, dp, pp, tp, scheme, zero in TRAIN_CASES:
        if dp * pp * tp != world:
            continue
        cfg = T.ToyModelConfig(**dict(SMALL_CFG, **over))
        tr = DistTrainer3D(cfg, build_layout(dp, pp, tp, world), scheme_from_name(scheme), T.ZeroMode(zero))
        met = tr.run()
        ran.append(name)
        if rank == 0:
            want = g[f"{name}__step_loss"]
            if np.array(met.step_loss, np.float32).tobytes() != want.tobytes():
                fails.append(f"{name}: step losses {met.step_loss} != {list(want)}")
            if bool(met.diverged) != bool(g[f"{name}__diverged"]):
                fails.append(f"{name}: diverged {met.diverged}")
            if not met.diverged:
                if tr.replica0.w1.reshape(-1).tobytes() != g[f"{name}__w1"].tobytes() or \
                        tr.replica0.w2.reshape(-1).tobytes() != g[f"{name}__w2"].tobytes():
                    fails.append(f"{name}: weights differ")
                if np.float32(met.final_eval_loss).tobytes() != np.float32(g[f"{name}__final_eval_loss"]).tobytes():
                    fails.append(f"{name}: eval loss")
                pb = g[f"{name}__path_bytes"]
                for p in CommPath:
                    got = met.bytes_by_path.get(p)
                    have = (got.raw, got.wire) if got else (0, 0)
                    if have != (int(pb[2 * int(p)]), int(pb[2 * int(p) + 1])):
                        fails.append(f"{name}: {p} bytes {have} != {(int(pb[2 * int(p)]), int(pb[2 * int(p) + 1]))}")
        torch.cuda.synchronize()
        tr.close()
    nf = torch.tensor([len(fails)], device="cuda")
    dist.all_reduce(nf)
    if rank == 0:
        for f in fails[:20]:
            print("FAIL", f, flush=True)
        print(f"TRAINER DIST PARITY {'OK' if nf.item() == 0 else 'FAILED'} world={world} cases={ran}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if nf.item() == 0 else 1)


if __name__ == "__main__":
    main()
