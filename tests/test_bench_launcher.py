"""bench.py's multi-rank launcher on CPU (gloo): `--gpus 2` without torchrun re-launches itself as
two ranks (torch.distributed.run on 127.0.0.1), every rank reports its communicator size, and
rank 0 prints one JSON line; under torchrun a WORLD_SIZE that disagrees with --gpus is refused."""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def _env():
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    env["CUDA_VISIBLE_DEVICES"] = ""
    return env


def test_gpus_2_self_launches_two_ranks():
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run"], cwd=ROOT,
                       env=_env(), capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["ranks_joined"] == 2
    assert out["config"]["rows_per_gpu"] == 6_250_000 and out["config"]["total_rows"] == 12_500_000
    reports = [l for l in p.stderr.splitlines() if "communicator nranks=" in l]
    assert len(reports) == 2 and all("nranks=2" in l for l in reports)


def test_world_size_must_match_gpus():
    env = _env()
    env.update(WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "4", "--dry-run"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=120)
    assert p.returncode == 2 and "WORLD_SIZE=2" in p.stderr


def test_reference_arm_small_sample_same_config():
    """--impl reference prints the GPU arm's config object and a cpu_baseline with host info."""
    env = _env()
    env["OTF_BENCH_ROWS"] = "20000"
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "c2",
                        "--steps", "2", "--warmup", "1"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    out = json.loads(p.stdout.strip().splitlines()[-1])
    assert out["impl"] == "reference" and out["config"]["rows_per_gpu"] == 20000
    cb = out["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["numpy"] and "statistic" in cb
    assert out["e2e"]["h2d_bytes_per_step"] == 0
