"""bench.py's reference arm runs on CPU and prints the contract's JSON line."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    for key in ("metric", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "cpu_baseline", "e2e", "config"):
        assert key in line
    # the reference's own code when oracle/_ref was built here, else the port
    ref_built = os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libb3d_ref.so"))
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == ("reference" if ref_built else "port")


def test_gpus_flag_launches_that_many_ranks():
    """`bench.py --gpus 2` run directly re-launches itself as 2 ranks
    (torch.distributed.run on 127.0.0.1); --dry-run makes the ranks meet over
    gloo and rank 0 report, so no GPU is needed."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--dry-run"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line == {"dry_run": True, "n_gpus": 2, "rank_sum": 1, "impl": "ours"}


def test_gpus_flag_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--dry-run"], capture_output=True, text=True, timeout=300, cwd=ROOT,
                         env=env)
    assert out.returncode != 0 and "--gpus 2 but WORLD_SIZE=1" in out.stderr
