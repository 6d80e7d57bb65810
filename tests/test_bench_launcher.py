"""CPU: `python bench.py --gpus 2` re-launches itself under torch.distributed.run (rendezvous on
127.0.0.1) exactly as the driver invokes it without torchrun; the ranks exchange halos over gloo and
rank 0 alone prints one JSON line (the N > 1 plumbing of bench.py, no GPU needed)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(n, *extra):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--check-launch", *extra],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def test_launcher_two_ranks():
    d = _run(2)
    assert d["n_gpus"] == 2 and d["world_size"] == 2
    assert d["halos_ok"]
    assert d["master_addr"] == "127.0.0.1"


def test_launcher_three_ranks_config4_halo():
    d = _run(3, "--config", "4")
    assert d["n_gpus"] == 3 and d["halos_ok"]
