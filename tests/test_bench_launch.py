"""bench.py --gpus N without torchrun spawns one rank per GPU (SURVEY.md
8(e)): a CPU dry run at world size 2 (gloo) checks the launcher, the folded
slabs and the reductions behind the JSON line."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_spawns_ranks_gloo():
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run", "--config",
                          "c1", "--steps", "2", "--warmup", "1"], capture_output=True, text=True, env=env,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    line = lines[0]
    assert line["n_gpus"] == 2
    assert line["config"]["systems_total"] == 64 * 33  # the whole plane, split over the ranks
    sys.path.insert(0, ROOT)
    from paper_1701_03787_b200.shard import kx_rows_folded

    assert line["config"]["kx_rows_rank0"] == len(kx_rows_folded(64, 0, 2))  # row 0 + 15 (m, -m) pairs


import pytest  # noqa: E402


@pytest.mark.gpu
def test_bench_c3_slab_two_ranks_one_gpu():
    """bench.py --config c3 --gpus 2: the multi-rank config-3 step (slab
    transforms with the exchange fused into the plane FFT kernels, slab
    solves).  Here the two ranks share cuda:0 over gloo on a thin mesh
    (SHEN_BENCH_BACKEND / SHEN_BENCH_C3_NX): a check of the code path, not a
    bench number -- on a multi-GPU node the same command runs one rank per
    GPU over NCCL."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    env.update(SHEN_BENCH_BACKEND="gloo", SHEN_BENCH_C3_NX="16", SHEN_BENCH_NO_CLOCKS="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "c3",
                          "--steps", "2", "--warmup", "3"], capture_output=True, text=True, env=env, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["n_gpus"] == 2 and line["scaling"] == "strong" and line["value"] > 0
    assert "peer memory" in line["config"]["parallelism"]
