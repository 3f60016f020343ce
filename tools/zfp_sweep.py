"""ZFP-mode codec timing on one GPU (tools/codec_sweep.run, kind 3), rates 8/16/4/32 at 2^24."""
import json, sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import torch
from codec_sweep import run
torch.cuda.set_device(0)
for r in [8, 16, 4, 32]:
    print(json.dumps(run(3, r, 1 << 24)), flush=True)
