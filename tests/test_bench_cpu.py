"""bench.py contract checks that need no GPU (-m "not gpu"): the reference arm
(`--impl reference`, the CPU oracle on the host cores, the only other place
bench.py may run oracle/) prints one JSON line with the keys the driver reads,
for the C5 workload BASELINE.json's metric is quoted on."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["metric"].startswith("coded Gbit/s decoded")
    assert d["unit"] == "coded Gbit/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 0
    assert d["config"]["workload"].startswith("C5: Hamming(63,57)")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_relaunch_command_is_torchrun_on_localhost():
    import bench
    cmd = bench.relaunch_command(["--gpus", "8", "--steps", "5"], 8, 29555)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29555" in cmd
    assert cmd[-3:] == ["--gpus", "8", "--steps", "5"][-3:] and os.path.basename(cmd[-5]) == "bench.py"


def test_gpus_n_without_torchrun_relaunches(monkeypatch):
    """`python bench.py --gpus 4` (no WORLD_SIZE) re-runs itself as 4 ranks and
    exits with their status; under torchrun (WORLD_SIZE set) it does not."""
    import argparse

    import bench
    seen = {}

    def fake_call(cmd, env=None):
        seen["cmd"], seen["env"] = cmd, env
        return 3

    monkeypatch.setattr(bench.subprocess, "call", fake_call)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4"])
    try:
        bench.maybe_relaunch(argparse.Namespace(gpus=4))
        raise AssertionError("did not exit")
    except SystemExit as e:
        assert e.code == 3
    assert "--nproc-per-node=4" in seen["cmd"] and seen["env"]["NCCL_DEBUG"] == "INFO"
    seen.clear()
    monkeypatch.setenv("WORLD_SIZE", "4")
    bench.maybe_relaunch(argparse.Namespace(gpus=4))
    bench.maybe_relaunch(argparse.Namespace(gpus=1))
    assert not seen


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1"], capture_output=True,
                         text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode != 0 and "world size 2 != --gpus 1" in out.stderr


def test_reference_arm_under_torchrun_two_ranks():
    """The driver's N > 1 launch of the reference arm: rank 0 alone runs and
    prints one line with n_gpus = 2; rank 1 exits 0 without work."""
    import bench
    cmd = bench.relaunch_command(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0"], 2,
                                 bench.free_port())
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
