"""The C++ adapter (include/gx_b200.hpp) compiles and links against
libgx_b200.so on CPU; on the GPU box it runs reference KATs end to end."""
import os
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "adapter_test.cpp")
LIBDIR = os.path.join(ROOT, "paper_2208_09151_b200")


def _build(out):
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), SRC, "-o", out,
                    "-L", LIBDIR, "-lgx_b200", f"-Wl,-rpath,{LIBDIR}"], check=True)


def test_adapter_compiles_and_links(tmp_path):
    _build(str(tmp_path / "adapter_test"))
    assert os.path.exists(tmp_path / "adapter_test")


@pytest.mark.gpu
def test_adapter_runs_reference_kats(tmp_path, oracle):
    import numpy as np
    import paper_2208_09151_b200 as gx
    exe = str(tmp_path / "adapter_test")
    _build(exe)
    # graph.bin / features.bin in the reference formats, written by this package
    g = gx.GraphFile.generate_rmat(200, 12.0, 6)
    g.write(str(tmp_path / "graph.bin"))
    rows = np.random.default_rng(3).random((200, 6)).astype(np.float32)
    hdr = (b"GXFEAT01" + (1).to_bytes(4, "little") + (200).to_bytes(8, "little") + (6).to_bytes(4, "little")
           + (4).to_bytes(4, "little") + (4096).to_bytes(8, "little"))
    with open(tmp_path / "features.bin", "wb") as fh:
        fh.write(hdr + b"\0" * (4096 - len(hdr)) + rows.tobytes())
    r = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
