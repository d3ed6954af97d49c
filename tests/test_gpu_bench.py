"""GPU: bench.py's multi-rank path end to end on the one GPU of a test box.

`bench.py --gpus 2` (no launcher) relaunches itself through
torch.distributed.run; GX_BENCH_SHARE_GPU=1 lets both ranks share cuda:0 over
gloo (NCCL refuses two ranks on one device). The rest is the code an 8-GPU box
runs: the row-partitioned CSC attached through CUDA IPC, superbatches or
batch blocks per rank, max-over-ranks timing and the whole-job edge count."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, share=True):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    if share:
        env["GX_BENCH_SHARE_GPU"] = "1"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0]), r.stderr


@pytest.mark.parametrize("split", ["superbatch", "batches"])
def test_bench_two_ranks_partitioned_csc(split):
    out, err = _bench("--gpus", "2", "--config", "cfg1", "--steps", "2", "--warmup", "1",
                      "--no-cpu-baseline", "--split", split)
    assert "launching 2 ranks" in err
    assert out["n_gpus"] == 2 and out["steps"] == 2 and out["value"] > 0
    assert out["parallelism"]["ranks"] == 2
    assert out["parallelism"]["graph"].startswith("partitioned"), out["parallelism"]
    assert out["scaling"] == ("weak" if split == "superbatch" else "strong")
    # whole-job edges: two superbatches per step (superbatch split) or one (batch split)
    per_sb = out["stages"]["edges_per_superbatch"]
    if split == "superbatch":
        assert out["config"]["global_batch"] == 2 * 100 * 1000
        assert 0.9 < out["value"] * out["ms_per_step"] / 1e3 / (2 * per_sb) < 1.1
    else:
        assert out["config"]["global_batch"] == 100 * 1000


def test_bench_one_rank_partitioned_graph_flag():
    out, _ = _bench("--config", "cfg1", "--steps", "2", "--warmup", "1", "--no-cpu-baseline",
                    "--graph", "partitioned", share=False)
    assert out["n_gpus"] == 1 and out["parallelism"]["graph"] == "partitioned"
