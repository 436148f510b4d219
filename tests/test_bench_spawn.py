"""bench.py --gpus N without torchrun: it spawns N ranks itself (CPU, gloo, host engine).

The driver runs `python bench.py --gpus N` for its scaling curve; without
torchrun's environment variables bench.py must start the ranks on its own,
run the z-slab path and print ONE JSON line with n_gpus = N.
"""

import json
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def _run(*args):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    res = subprocess.run([sys.executable, os.path.join(HERE, "run_bench_host.py"), *args],
                         capture_output=True, text=True, timeout=300, env=env)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("workload,scaling", [("tiny", "weak"), ("tinys", "strong")])
@pytest.mark.parametrize("transport", ["p2p", "nccl"])
def test_bench_spawns_two_ranks(workload, scaling, transport):
    line = _run("--gpus", "2", "--workload", workload, "--depth", "4", "--steps", "2", "--warmup", "3",
                "--transport", transport)
    assert line["n_gpus"] == 2
    assert line["scaling"] == scaling
    assert line["impl"] == "ours" and line["ms_per_step"] > 0
    gz = 40 if workload == "tiny" else 40
    assert line["config"]["global_interior_zyx"] == [gz, 10, 12]
    assert line["config"]["per_gpu_interior_zyx"] == [20, 10, 12]
    assert line["config"]["halo_depth"] == 4
    assert line["config"]["halo_transport"] == transport
    assert line["verify"] == {"checked": True, "match": True}
    e2e = line["e2e"]
    assert e2e["ms_per_step"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] == 40 * 10 * 12 * 8


def test_bench_three_ranks_uneven_strong_split():
    line = _run("--gpus", "3", "--workload", "tinys", "--depth", "2", "--steps", "1", "--warmup", "3")
    assert line["n_gpus"] == 3 and line["scaling"] == "strong"
    assert line["verify"]["match"] is True
