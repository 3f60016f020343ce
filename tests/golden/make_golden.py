"""Generate golden fixtures from the UNMODIFIED reference library.

Run in the dev container (needs /root/reference to build oracle/_ref):

    python tests/golden/make_golden.py

Every array is produced by the reference's own code compiled from
/root/reference/proj/src (oracle/_ref/libhcc_ref.so via oracle/ref_capi.cpp):
inputs come from the reference's buffer generators (hcc::Rng,
proj/tests/support/oracles.cpp:9-36), payloads from hcc::compress, decoded
values from hcc::decompress, collective outputs and byte accounting from
hcc::allreduce / ring_reduce_scatter / ring_allgather / p2p.  The fixtures
travel with the repo, so the GPU box (where /root/reference does not exist)
checks the kernels against the reference's own outputs.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import oracle_lib as O  # noqa: E402

CODEC_RATES = [2, 3, 4, 5, 7, 8, 12, 13, 16, 22, 23, 24, 25, 26, 31, 32]
CODEC_SIZES = [1, 63, 64, 65, 255, 256, 257, 1000, 2049]
MODES = [("uniform", -1.0, 1.0), ("finite", 0, 0), ("sparse", 0.5, 0)]


def lossless() -> None:
    """LosslessPredictor payloads (hcc::compress) and its collective byte
    accounting, including buffers whose chunks mix coded and raw-fallback."""
    out = {}
    seed = 9000
    for n in [1, 63, 4095, 4096, 4097, 3 * 4096 + 17, 20000]:
        for mode, lo, hi in [("bits", 0, 0), ("sparse", 0.9, 0), ("uniform", -1.0, 1.0), ("const", 0, 0),
                             ("mixed", 0, 0)]:
            seed += 1
            if mode == "const":
                x = np.full(n, 1.0, np.float32)
            elif mode == "mixed":  # alternate chunks: sparse (coded) / random bits (raw)
                a = O.ref_fill(seed, "sparse", n, 0.9, 0)
                b = O.ref_fill(seed + 1, "bits", n, 0, 0)
                idx = (np.arange(n) // 4096) % 2 == 1
                x = np.where(idx, b, a).astype(np.float32)
            else:
                x = O.ref_fill(seed, mode, n, lo, hi)
            payload, cc = O.ref_compress("lossless", 0, x)
            key = f"n{n}_{mode}"
            out[f"{key}_in"] = x
            out[f"{key}_payload"] = payload
            out[f"{key}_cc"] = np.array([cc], np.uint64)
    for p in [2, 4]:
        for n_per in [64, 5000]:
            n = n_per * p
            seed += 1
            x = np.stack([O.ref_fill(seed * 13 + j, "sparse" if j % 2 else "uniform", n, 0.5 if j % 2 else -1.0, 1.0)
                          for j in range(p)])
            key = f"p{p}_n{n}"
            out[f"{key}_in"] = x
            for avg in (0, 1):
                r, acct = O.ref_allreduce(x, "lossless", 0, bool(avg))
                out[f"{key}_ar{avg}"] = r
                out[f"{key}_ar{avg}_acct"] = np.array(acct, np.uint64)
            r, acct = O.ref_reduce_scatter(x, "lossless", 0)
            out[f"{key}_rs"] = r
            out[f"{key}_rs_acct"] = np.array(acct, np.uint64)
            shards = np.ascontiguousarray(x[:, :n_per])
            r, acct = O.ref_allgather(shards, "lossless", 0)
            out[f"{key}_ag"] = r
            out[f"{key}_ag_acct"] = np.array(acct, np.uint64)
            r, acct = O.ref_p2p(x[1], "lossless", 0)
            out[f"{key}_p2p_acct"] = np.array(acct, np.uint64)
    np.savez_compressed(os.path.join(HERE, "lossless.npz"), **out)
    print("wrote", len(out), "lossless arrays")


SMALL_CFG = {"num_blocks": 4, "hidden_dim": 16, "input_dim": 8, "batch_size": 8, "microbatches": 2, "steps": 4,
             "seed": 3, "learning_rate": 2e-3}  # proj/tests/test_toymodel.cpp:15-26 (steps shortened)
TRAIN_CASES = [  # (name, cfg overrides, dp, pp, tp, scheme, zero: 0 off / 1 replace / 2 redundant)
    ("base3d_none_off", {}, 2, 2, 2, "no-compression", 0),
    ("base3d_mpc_off", {}, 2, 2, 2, "naive-mpc", 0),
    ("base3d_zhyb_replace", {}, 2, 2, 2, "z-hybrid:16,8", 1),
    ("base3d_mzhyb_off", {}, 2, 2, 2, "mz-hybrid:8", 0),
    ("dp4_none_redundant", {"batch_size": 32, "steps": 3}, 4, 1, 1, "no-compression", 2),
    ("dp2_zfp8_replace", {"steps": 5}, 2, 1, 1, "naive-zfp8", 1),
    ("pp2tp2_zhyb_off", {}, 1, 2, 2, "z-hybrid:16,4", 0),
    ("diverge_zfp8", {"steps": 20, "learning_rate": 1e30}, 2, 1, 1, "naive-zfp8", 0),
    ("dp2pp2_mzhyb_off", {}, 2, 2, 1, "mz-hybrid:8", 0),
    ("tp2_zhyb_off", {}, 1, 1, 2, "z-hybrid:16,8", 0),
    ("dp2tp2_mpc_replace", {}, 2, 1, 2, "naive-mpc", 1),
]


def trainer() -> None:
    """hcc::Trainer3D runs (the reference's toy 3D-parallel trainer)."""
    out = {}
    for name, over, dp, pp, tp, scheme, zero in TRAIN_CASES:
        cfg = dict(SMALL_CFG, **over)
        r = O.ref_train(cfg, dp, pp, tp, scheme, zero)
        for k, v in r.items():
            out[f"{name}__{k}"] = np.asarray(v)
    np.savez_compressed(os.path.join(HERE, "trainer.npz"), **out)
    print("wrote", len(out), "trainer arrays")


def main() -> None:
    assert O.ref is not None, "oracle/_ref/libhcc_ref.so is required (build with oracle/build_ref.sh)"
    if "--only-lossless" in sys.argv:
        lossless()
        return
    if "--only-trainer" in sys.argv:
        trainer()
        return
    trainer()
    lossless()
    codec = {}
    seed = 1000
    for rate in CODEC_RATES:
        for n in CODEC_SIZES:
            for mode, lo, hi in MODES:
                seed += 1
                x = O.ref_fill(seed, mode, n, lo, hi)
                payload, cc = O.ref_compress("fixed-rate", rate, x)
                dec = O.ref_decompress("fixed-rate", rate, payload, n, cc)
                key = f"fr{rate}_n{n}_{mode}"
                codec[f"{key}_in"] = x
                codec[f"{key}_payload"] = payload
                codec[f"{key}_dec"] = dec
    np.savez_compressed(os.path.join(HERE, "fixed_rate.npz"), **codec)

    coll = {}
    seed = 5000
    for p in [2, 3, 4, 8]:
        for kind, rate in [("identity", 0), ("fixed-rate", 4), ("fixed-rate", 8), ("fixed-rate", 16)]:
            for n_per in [64, 200, 320]:
                n = n_per * p
                seed += 1
                x = np.stack([O.ref_fill(seed * 17 + j, "uniform", n) for j in range(p)])
                key = f"p{p}_{kind}{rate}_n{n}"
                coll[f"{key}_in"] = x
                for avg in (0, 1):
                    out, acct = O.ref_allreduce(x, kind, rate, bool(avg))
                    coll[f"{key}_ar{avg}"] = out
                    coll[f"{key}_ar{avg}_acct"] = np.array(acct, np.uint64)
                rs, acct = O.ref_reduce_scatter(x, kind, rate)
                coll[f"{key}_rs"] = rs
                coll[f"{key}_rs_acct"] = np.array(acct, np.uint64)
                shards = np.ascontiguousarray(x[:, :n_per])
                ag, acct = O.ref_allgather(shards, kind, rate)
                coll[f"{key}_ag"] = ag
                coll[f"{key}_ag_acct"] = np.array(acct, np.uint64)
                pp, acct = O.ref_p2p(x[0], kind, rate)
                coll[f"{key}_p2p"] = pp
                coll[f"{key}_p2p_acct"] = np.array(acct, np.uint64)
    np.savez_compressed(os.path.join(HERE, "collectives.npz"), **coll)
    print("wrote", len(codec), "codec arrays and", len(coll), "collective arrays")


if __name__ == "__main__":
    main()
