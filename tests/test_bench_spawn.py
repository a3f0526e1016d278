"""bench.py --gpus N outside torchrun re-launches itself with one rank per GPU
(the driver's scaling run calls it either way).  On CPU: the command line, and
the whole spawn path end to end with the reference arm (rank 0 alone prints one
JSON line with n_gpus = N, the other ranks exit 0 without work)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_spawn_command_shape():
    cmd = bench.spawn_command(["--gpus", "4", "--steps", "2"], 4, 29512)
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29512" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"]
    assert cmd[cmd.index("--master-port=29512") + 1].endswith("bench.py")


def test_no_spawn_inside_torchrun(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "2")
    args = bench.argparse.Namespace(gpus=2, impl="ours")
    assert bench.maybe_spawn(args, []) is None
    monkeypatch.delenv("WORLD_SIZE")
    assert bench.maybe_spawn(bench.argparse.Namespace(gpus=1, impl="ours"), []) is None


def test_reference_arm_spawns_ranks_end_to_end():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--config", "cfg1", "--steps", "1", "--warmup", "0", "--ref-samples", "256"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "torch.distributed.run" in r.stderr and "--nproc-per-node=2" in r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 only
    out = json.loads(lines[0])
    assert out["impl"] == "reference" and out["n_gpus"] == 2 and out["value"] > 0
