"""Experiment runner CLI (cli.py): config parsing and
validation on the CPU; run / sweep / codec-bench on the GPU."""
import csv
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOOD = {"layout": {"dp": 2, "pp": 2, "tp": 2, "zero1": "replace"},
        "model": {"num_blocks": 4, "hidden_dim": 16, "input_dim": 8, "batch_size": 8, "microbatches": 2,
                  "steps": 3, "seed": 3, "learning_rate": 0.002},
        "scheme": {"name": "z-hybrid:16,8"}}


def _cli(args, cfg=None, tmp=None):
    path = None
    if cfg is not None:
        path = os.path.join(tmp, "cfg.txt")
        with open(path, "w") as fh:
            fh.write(cfg if isinstance(cfg, str) else json.dumps(cfg))
    cmd = [sys.executable, "-m", "paper_2409_02423_b200"] + args + (["--config", path] if path else [])
    return subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)


def test_validate_and_errors(tmp_path):
    r = _cli(["validate"], GOOD, str(tmp_path))
    assert r.returncode == 0, r.stderr
    bad = json.loads(json.dumps(GOOD))
    bad["layout"]["dp"] = 3  # dp*pp*tp != world of the given topology
    bad["topology"] = {"num_nodes": 1, "gpus_per_node": 8}
    r = _cli(["validate"], bad, str(tmp_path))
    assert r.returncode == 2 and "layout" in r.stderr
    bad = json.loads(json.dumps(GOOD))
    bad["model"]["hidden_dim"] = 15
    r = _cli(["validate"], bad, str(tmp_path))
    assert r.returncode == 2 and "model.hidden_dim" in r.stderr
    bad = json.loads(json.dumps(GOOD))
    bad["scheme"] = {"name": "zfp-everything"}
    r = _cli(["validate"], bad, str(tmp_path))
    assert r.returncode == 2 and "scheme" in r.stderr


def test_config_round_trip_and_ini():
    from paper_2409_02423_b200 import cli

    cfg = cli.parse_config(json.dumps(GOOD))
    assert cli.parse_config(cli.serialize_config(cfg)) == cfg
    ini = """[layout]
dp = 2
pp = 2
tp = 2
zero1 = replace
[model]
num_blocks = 4
hidden_dim = 16
input_dim = 8
batch_size = 8
microbatches = 2
steps = 3
seed = 3
learning_rate = 0.002
[scheme]
name = z-hybrid:16,8
"""
    assert cli.parse_config(ini) == cfg
    paths = cli.make_scheme(cli.parse_config('{"scheme": {"paths": {"DpAllReduce": "fixed-rate:4"}}}'))
    from paper_2409_02423_b200 import CodecSpec, CommPath

    assert paths.at(CommPath.DpAllReduce) == CodecSpec.fixed_rate(4)
    assert paths.at(CommPath.TpAllReduce) == CodecSpec.identity()


@pytest.mark.gpu
def test_run_sweep_codec_bench(cuda, tmp_path):
    # messages of >= 64 values, so every lossy path shrinks (a 32-value
    # message at rate 16 is one 129-byte block: larger than its 128 raw bytes)
    big = json.loads(json.dumps(GOOD))
    big["model"].update(input_dim=64, hidden_dim=32)
    r = _cli(["run", "--out", str(tmp_path / "run")], big, str(tmp_path))
    assert r.returncode == 0, r.stderr
    summ = json.load(open(tmp_path / "run" / "summary.json"))
    assert summ["steps_completed"] == 3 and not summ["diverged"]
    assert set(summ["bytes_by_path"]) == {"TpAllReduce", "PpP2p", "Zero1AllGather", "Zero1ReduceScatter"}
    for p, b in summ["bytes_by_path"].items():
        assert b["wire"] < b["raw"], p  # every lossy path shrinks
    assert len(list(csv.reader(open(tmp_path / "run" / "loss.csv")))) == 4
    cfg = dict(GOOD, sweep={"schemes": ["no-compression", "naive-mpc", "naive-zfp8"]})
    r = _cli(["sweep", "--out", str(tmp_path / "sw")], cfg, str(tmp_path))
    assert r.returncode == 0, r.stderr
    rows = list(csv.DictReader(open(tmp_path / "sw" / "sweep.csv")))
    assert [x["scheme"] for x in rows] == ["no-compression", "naive-mpc", "naive-zfp8"]
    assert rows[0]["final_loss"] == rows[1]["final_loss"]  # lossless transparency
    cfg = {"codec_bench": {"sizes": [65536], "codecs": ["identity", "lossless", "fixed-rate:8"]}}
    r = _cli(["codec-bench", "--out", str(tmp_path / "cb")], cfg, str(tmp_path))
    assert r.returncode == 0, r.stderr
    rows = {(x["codec"], x["data"]): x for x in csv.DictReader(open(tmp_path / "cb" / "codec_bench.csv"))}
    assert abs(float(rows[("fixed-rate:8", "dense")]["ratio"]) - 256 / 65) < 1e-3  # ~3.9:1
    assert float(rows[("identity", "dense")]["ratio"]) == 1.0
    assert float(rows[("lossless", "sparse")]["ratio"]) > float(rows[("lossless", "dense")]["ratio"])
