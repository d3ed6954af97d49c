"""CPU suite: the C-ABI boundary loads, exports exactly what include/gx_b200.h
declares, and its host-only entry points (no device needed) agree with the
oracle. No compute call touches a GPU here."""
import ctypes
import os
import re
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gx_b200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gx_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2208_09151_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = header_functions()
    assert len(names) > 60
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def test_built_for_sm100a():
    from paper_2208_09151_b200 import _lib
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([cuobjdump, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_fails_loudly(gx):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(gx.CudaError):
        gx.Context()


def test_host_primitives_match_oracle(gx, oracle):
    for z in (0, 1, 12345, 2**64 - 1):
        assert gx.mix64(z) == oracle.mix64(z)
        assert gx.derive_seed(z, 7) == oracle.derive_seed(z, 7)
    assert gx.pages_touched(0, 0) == 0 and gx.pages_touched(4095, 4097) == 2
    assert gx.page_count_for_row(3072, 1) == 2
    with pytest.raises(ValueError):
        gx.page_count_for_row(0, 0)
    t = gx.derive_train_ids(5000, 3, 0.1)
    assert np.array_equal(t, oracle.train_ids(5000, 3, 0.1))
    plan = gx.plan_seed_batches(t, 64, gx.epoch_seed(3, 0)).batches
    want = oracle.plan_seed_batches(t, 64, oracle.epoch_seed(3, 0))
    assert len(plan) == len(want) and all(np.array_equal(a, b) for a, b in zip(plan, want))
    with pytest.raises(ValueError):
        gx.plan_seed_batches([], 4, 1)
    with pytest.raises(ValueError):
        gx.plan_seed_batches([1, 2], 0, 1)


def test_plan_seed_batches_kat(gx):
    # test_sampler.cpp:23-50
    train = np.arange(10, dtype=np.uint64)
    p = gx.plan_seed_batches(train, 4, 1).batches
    assert [len(b) for b in p] == [4, 4, 2]
    assert sorted(int(x) for b in p for x in b) == list(range(10))
    a = gx.plan_seed_batches(train, 3, 42).batches
    b = gx.plan_seed_batches(train, 3, 42).batches
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    big = np.arange(200, dtype=np.uint64)
    x = gx.plan_seed_batches(big, 16, 1).batches
    y = gx.plan_seed_batches(big, 16, 2).batches
    assert not all(np.array_equal(u, v) for u, v in zip(x, y))


def test_runtime_file_codecs_match_reference_bytes(gx):
    """ids/adj files written by the reference's superbatch_sample (golden byte
    images) parse, and re-encode to the same bytes (FORMATS.md)."""
    G = np.load(os.path.join(ROOT, "tests", "golden", "reference_golden.npz"))
    with tempfile.TemporaryDirectory() as d:
        for i in range(3):
            pi, pa = os.path.join(d, f"i{i}.bin"), os.path.join(d, f"a{i}.bin")
            G[f"file_ids_{i}"].tofile(pi)
            G[f"file_adj_{i}"].tofile(pa)
            ids = gx.read_ids_file(pi)
            adj = gx.read_adj_file(pa)
            gx.api.write_ids_file(os.path.join(d, "x.bin"), ids)
            gx.api.write_adj_file(os.path.join(d, "y.bin"), adj)
            assert open(os.path.join(d, "x.bin"), "rb").read() == G[f"file_ids_{i}"].tobytes()
            assert open(os.path.join(d, "y.bin"), "rb").read() == G[f"file_adj_{i}"].tobytes()
        with pytest.raises(RuntimeError):
            gx.read_adj_file(os.path.join(d, "i0.bin"))  # wrong magic
        cs = gx.Changeset(np.array([5, 6], np.uint64), np.array([1], np.uint64), np.array([0, 4], np.uint64))
        p = os.path.join(d, "u.bin")
        with open(p, "wb") as fh:
            for a in (cs.in_ids, cs.out_ids, cs.in_positions):
                pass
            fh.write(b"GXUPD001")
            for a in (cs.in_ids, cs.out_ids, cs.in_positions):
                fh.write(len(a).to_bytes(8, "little") + a.astype("<u8").tobytes())
        assert gx.read_update_file(p) == cs


def test_oracle_header_says_test_infrastructure():
    for f in ("oracle/gx_oracle.c", "oracle/ref_driver.cpp", "oracle/__init__.py"):
        assert "TEST INFRASTRUCTURE ONLY" in open(os.path.join(ROOT, f)).read()


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2208_09151_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, fn)).read()
                assert "import oracle" not in src and "gx_oracle" not in src and "libgx_ref" not in src, fn
