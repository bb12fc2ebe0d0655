"""The bench.py JSON contract on the CPU: the reference arm (the oracle timed on the host
cores, `--impl reference`) prints one line with the keys the driver reads."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 1 and d["n_gpus"] == 1
    assert d["value"] > 0 and d["unit"] == "qp/s" and d["higher_is_better"] is True and d["dtype"] == "f64"
    assert "workload" in d["config"] and d["config"]["workload"].startswith("c1")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == dict(value=d["value"], unit="qp/s", h2d_bytes_per_step=0, d2h_bytes_per_step=0)


def _bench():
    sys.path.insert(0, ROOT)
    import importlib
    return importlib.import_module("bench")


def test_launch_plan():
    """`--gpus N` semantics: relaunch under torch.distributed.run when no launcher set
    WORLD_SIZE, refuse a WORLD_SIZE that disagrees with --gpus, refuse when fewer than N
    devices are visible (the GPU arm), run as a rank otherwise."""
    b = _bench()
    assert b.launch_plan(1, {}, 1) == ("run", None)
    assert b.launch_plan(4, {}, 8) == ("relaunch", None)
    assert b.launch_plan(8, {"WORLD_SIZE": "8"}, 8) == ("run", None)
    act, why = b.launch_plan(2, {"WORLD_SIZE": "4"}, 8)
    assert act == "refuse" and "WORLD_SIZE=4" in why
    act, why = b.launch_plan(2, {}, 1)
    assert act == "refuse" and "only 1 CUDA device" in why
    act, why = b.launch_plan(1, {}, 0)
    assert act == "refuse"
    assert b.launch_plan(0, {}, 8)[0] == "refuse"
    # the reference arm (host oracle) needs no device and is never relaunched
    assert b.launch_plan(8, {}, 0, needs_gpus=False) == ("run", None)
    assert b.launch_plan(8, {"WORLD_SIZE": "8"}, 0, needs_gpus=False) == ("run", None)
    cmd = b.relaunch_cmd(4, ["--gpus", "4", "--steps", "3"], 29555)
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert "--master-addr=127.0.0.1" in cmd and "--master-port=29555" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"] and cmd[-5].endswith("bench.py")


def test_bench_refuses_more_gpus_than_visible():
    """On a box with fewer devices than --gpus (here: none), the GPU arm exits non-zero with a
    message instead of printing a 1-GPU line labelled N GPUs."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "c1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env={k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")})
    assert out.returncode == 2, (out.returncode, out.stderr[-1000:])
    assert "--gpus 2" in out.stderr and not [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
