"""bench.py's reference arm (CPU only): the JSON line the driver reads."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--steps", "2", "--warmup", "1", "--config", "c1",
                          "--ref-planes", "4"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"] == "coupled Maxwell-LLG Gcell-updates/s"
    assert line["value"] > 0 and line["higher_is_better"] is True
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    # the reference arm reports the GPU arm's own workload (same config object)
    assert line["config"]["config_file"] == "configs/c1.cfg"
    assert line["config"]["cells_total"] == 64 ** 3 and line["n_gpus"] == 1


def test_gpus_flag_launches_that_many_ranks(tmp_path):
    """`python bench.py --gpus 2` (no torchrun) re-launches itself as 2 ranks
    under torch.distributed.run; each rank builds its own x-slab (device
    replaced by a recorder, gloo plumbing)."""
    import os
    env = dict(os.environ, MPB_BENCH_DEVICE="tests.fake_device:Recorder",
               PYTHONPATH=str(ROOT))
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2",
                          "--config", "c2", "--init", "zero",
                          "--layout-only", str(tmp_path)],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    recs = sorted((json.loads(p.read_text()) for p in tmp_path.glob("rank*.json")),
                  key=lambda r: r["rank"])
    assert [r["rank"] for r in recs] == [0, 1]
    assert all(r["world"] == r["env_world"] == r["nranks"] == 2 for r in recs)
    assert recs[0]["x_lo"] == 0 and recs[0]["x_hi"] == recs[1]["x_lo"]
    assert recs[1]["x_hi"] == 512                 # weak scaling: 2 x 256 planes of C2
    assert all(r["grid"] == [512, 256, 64] for r in recs)
    assert sum(r["cells"] for r in recs) == 512 * 256 * 64


def test_gpus_flag_must_match_world_size():
    import os
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2",
                          "--config", "c1"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode != 0 and "WORLD_SIZE=1" in out.stderr


def test_reference_arm_under_torchrun_prints_once():
    """The driver launches the reference arm like the GPU arm (torchrun, N
    ranks): rank 0 alone runs and prints one line; the others exit 0."""
    import os
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node=2", "--master-addr=127.0.0.1",
                          f"--master-port={port}", str(ROOT / "bench.py"), "--impl",
                          "reference", "--gpus", "2", "--steps", "1", "--warmup", "1",
                          "--config", "c1", "--ref-planes", "4"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["config"]["cells_total"] == 2 * 64 ** 3          # weak scaling: N x C1
