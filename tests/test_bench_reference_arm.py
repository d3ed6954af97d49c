"""CPU suite: bench.py's reference arm (`--impl reference`) runs the reference
(oracle/_ref, compiled from its own headers) on host-written inputs without
torch or the CUDA library in the process, and prints the same `config` object
as the GPU arm for the same workload (configs[0], one full superbatch per step)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r"""
import io, json, runpy, sys, contextlib
sys.argv = ["bench.py", "--impl", "reference", "--config", "cfg1", "--steps", "1", "--warmup", "0"]
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    runpy.run_path("bench.py", run_name="__main__")
maps = open("/proc/self/maps").read()
print(json.dumps({"line": buf.getvalue().strip().splitlines()[-1],
                  "torch": "torch" in sys.modules,
                  "gx": "paper_2208_09151_b200" in sys.modules,
                  "libgx_mapped": "libgx_b200" in maps,
                  "ref_mapped": "libgx_ref" in maps}))
"""


def test_reference_arm_runs_without_the_cuda_library():
    import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([sys.executable, "-c", CODE], cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, PYTHONPATH=ROOT))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert not res["torch"] and not res["gx"] and not res["libgx_mapped"] and res["ref_mapped"], res
    line = json.loads(res["line"])
    assert line["impl"] == "reference" and line["value"] > 0 and line["steps"] == 1
    assert line["cpu_baseline"]["kind"] == "reference"
    cfg = line["config"]
    assert cfg["superbatch"] == 100 and cfg["cache_entries"] == 100_000 and cfg["num_edges"] == 9_711_781
    assert cfg["global_batch"] == 100 * 1000
