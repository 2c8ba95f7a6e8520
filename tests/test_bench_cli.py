"""bench.py's process-group contract on CPU: `--gpus N` without torchrun
spawns N ranks itself (torch.distributed.run, 127.0.0.1 rendezvous) and the
group it forms has exactly N ranks (gloo dry run, no device work); both arms
print the same `config` object."""

import json
import os
import subprocess
import sys

from conftest import REPO


def _env():
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    env["OMP_NUM_THREADS"] = "1"
    return env


def test_gpus2_spawns_a_two_rank_group():
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2",
                          "--dry-run"], capture_output=True, text=True, env=_env(), timeout=240,
                         cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["dry_run"] and d["n_gpus"] == 2 and d["world"] == 2 and d["allreduce_sum"] == 2.0


def test_both_arms_share_the_config_object():
    sys.path.insert(0, REPO)
    import bench
    from paper_2602_09527_b200 import problems
    for name in ("c0", "c1", "c2", "c3"):
        cfg = problems.CONFIGS[name]
        c = bench.bench_config(cfg)
        assert c == bench.bench_config(cfg)
        assert str(problems.POWER_L[name]) in c["L"]
        assert "50 power iterations" in c["L"]
