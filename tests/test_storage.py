"""The 'SSD' tier (GX_BACKING_FILE, storage.cu).

CPU part (no GPU needed): a file-backed table opened without a context serves
FeatureFile::read_rows (graph_store.hpp:319-324) from the host reader --
coalesced page runs, O_DIRECT where the filesystem allows it -- and must return
the bytes and IoStats the reference's FeatureFile returns for the same file
(oracle/_ref, the reference compiled from its headers; a FeatureCache with an
empty init set charges every gathered row exactly as read_row does).

GPU part: the same file behind the FeatureCache API and the fused pipeline;
gathered bytes, counts and IoStats identical to a device-backed table and to the
oracle.
"""
import os

import numpy as np
import pytest

HDR = 36


def _write_features(path, rows):
    """FeatureWriter byte layout (graph_store.hpp:237-250): 36-byte header, payload at 4096."""
    n, dim = rows.shape
    sw = rows.dtype.itemsize
    hdr = (b"GXFEAT01" + (1).to_bytes(4, "little") + n.to_bytes(8, "little") + dim.to_bytes(4, "little")
           + sw.to_bytes(4, "little") + (4096).to_bytes(8, "little"))
    with open(path, "wb") as fh:
        fh.write(hdr + b"\0" * (4096 - HDR))
        fh.write(np.ascontiguousarray(rows).tobytes())


def _rows(n, dim, seed, dtype=np.float32):
    return np.random.default_rng(seed).random((n, dim)).astype(dtype)


@pytest.fixture
def knobs(monkeypatch):
    def set_(**kw):
        for k, v in kw.items():
            monkeypatch.setenv(k, str(v))
    return set_


@pytest.mark.parametrize("dim", [128, 384, 3])          # 512 B, 1536 B (straddles pages), 12 B rows
@pytest.mark.parametrize("cfg", [dict(), dict(GX_SSD_RUN_KB=4, GX_SSD_GAP_PAGES=3, GX_SSD_THREADS=3)])
def test_file_read_rows_matches_reference(gx, ref, tmp_path, knobs, dim, cfg):
    knobs(**cfg)
    n = 3000
    rows = _rows(n, dim, dim)
    path = str(tmp_path / "features.bin")
    ref.write_features(path, rows)                         # the reference's own writer
    rng = np.random.default_rng(7)
    ids = np.concatenate([rng.integers(0, n, 4000), [0, n - 1, n - 1, 5, 5]]).astype(np.uint64)
    f = gx.FeatureFile.open(path, "file")                  # no context: host-only reader
    io = gx.IoStats()
    got = f.read_rows(ids, io)
    assert np.array_equal(got, rows[ids.astype(np.int64)])
    want, hits, misses, rio = ref.open_features(path).cache([], 1).gather(ids, dim)
    assert np.array_equal(got, want)
    assert (hits, misses) == (0, len(ids))
    assert [io.pages_read, io.rows_read, io.neighbor_lists_read, io.bytes_read] == list(map(int, rio))
    st = f.storage_stats()
    assert st.rows == len(ids) and st.preads >= 1
    # whole pages, except reads that stop at EOF (one per reader thread that reaches it)
    tail = (4096 + n * dim * 4) % 4096
    assert any((st.bytes - k * tail) % 4096 == 0 for k in range(st.threads + 1))
    # coalescing: never more preads than rows, never fewer than the distinct page runs need
    assert st.preads <= len(ids)


def test_file_read_rows_fp16_and_edges(gx, tmp_path):
    n, dim = 1000, 768
    rows = _rows(n, dim, 3, np.float16)                    # scalar_width 2 extension (cfg4)
    path = str(tmp_path / "f16.bin")
    _write_features(path, rows)
    f = gx.FeatureFile.open(path, "file")
    assert f.dtype == np.float16 and f.row_bytes() == 1536
    ids = np.array([999, 0, 500, 500, 1], np.uint64)
    assert np.array_equal(f.read_rows(ids), rows[ids.astype(np.int64)])
    assert f.read_rows(np.zeros(0, np.uint64)).shape == (0, dim)
    with pytest.raises(IndexError):
        f.read_rows([n])
    with pytest.raises(ValueError):                        # the cache needs a device
        gx.FeatureCache(f, [1], 4)


def test_file_open_errors(gx, tmp_path):
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOTFEAT1" + b"\0" * 64)
    with pytest.raises(RuntimeError):
        gx.FeatureFile.open(str(bad), "file")
    rows = _rows(100, 16, 1)
    path = tmp_path / "trunc.bin"
    _write_features(str(path), rows)
    with open(path, "r+b") as fh:
        fh.truncate(4096 + 99 * 64)
    with pytest.raises(RuntimeError):
        gx.FeatureFile.open(str(path), "file")
    with pytest.raises(RuntimeError):
        gx.FeatureFile.open(str(tmp_path / "missing.bin"), "file")


def test_direct_io_when_available(gx, tmp_path):
    """O_DIRECT on filesystems that support it (GX_SSD_DIRECT=0 forces the
    buffered path); either way the bytes are the same."""
    rows = _rows(64, 128, 2)
    path = str(tmp_path / "d.bin")
    _write_features(path, rows)
    f = gx.FeatureFile.open(path, "file")
    assert np.array_equal(f.read_rows(np.arange(64)[::-1]), rows[::-1])
    shm = "/dev/shm"
    if os.path.isdir(shm):
        p2 = os.path.join(shm, f"gx_storage_test_{os.getpid()}.bin")
        try:
            _write_features(p2, rows)
            f2 = gx.FeatureFile.open(p2, "file")
            assert np.array_equal(f2.read_rows([3, 1]), rows[[3, 1]])
        finally:
            os.unlink(p2)


# ---------------------------------------------------------------------------
# GPU: the file tier behind the cache and the pipeline
# ---------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("dim", [128, 300])
def test_file_cache_matches_device_and_oracle(gx, oracle, tmp_path, dim):
    n, K = 4000, 700
    rows = _rows(n, dim, 11)
    path = str(tmp_path / "features.bin")
    _write_features(path, rows)
    ff = gx.FeatureFile.open(path, "file", ctx=gx.Context.default())
    fd = gx.FeatureFile.from_array(rows)
    rng = np.random.default_rng(3)
    init = rng.choice(n, 500, replace=False).astype(np.uint64)
    iof, iod = gx.IoStats(), gx.IoStats()
    cf = gx.FeatureCache(ff, init, K, iof)
    cd = gx.FeatureCache(fd, init, K, iod)
    assert iof == iod
    oc = oracle.cache(rows, init, K)
    for it in range(4):
        ids = rng.choice(n, 900, replace=False).astype(np.uint64)
        bf, cntf = cf.gather(ff, ids, iof)
        bd, cntd = cd.gather(fd, ids, iod)
        want, h, m, _ = oc.gather(ids)
        assert np.array_equal(bf.numpy(), rows[ids.astype(np.int64)])
        assert np.array_equal(bf.numpy(), bd.numpy())
        assert (cntf.hits, cntf.misses) == (cntd.hits, cntd.misses) == (h, m)
        assert iof == iod
        # evict the first 50 cached ids present in this batch's misses' complement, admit 50 misses
        miss_pos = [k for k, v in enumerate(ids) if not cf.contains(int(v))][:50]
        res = cf.resident_set()
        out = res[:len(miss_pos)]
        cs = gx.Changeset(ids[miss_pos], out, np.array(miss_pos, np.uint64))
        cf.apply_changeset(bf, ids, cs)
        cd.apply_changeset(bd, ids, cs)
        oc.apply(want, ids, cs.in_ids, cs.in_positions, cs.out_ids)
        assert np.array_equal(cf.resident_set(), cd.resident_set())
    st = ff.storage_stats()
    assert st.rows > 0 and st.h2d_bytes == st.rows * ff.row_bytes()


@pytest.mark.gpu
@pytest.mark.parametrize("K", [300, 1500, 6000])          # misses in every iteration .. all-fit
def test_file_pipeline_matches_oracle(gx, oracle, tmp_path, knobs, K):
    knobs(GX_SSD_CHUNK_MB=1)                               # several chunks per superbatch
    n, dim = 6000, 96
    ip, ind = oracle.rmat_graph(n, 6.0, 21)
    rows = oracle.features(n, dim, 22)
    path = str(tmp_path / "features.bin")
    _write_features(path, rows)
    g = gx.GraphFile.from_csc(ip, ind)
    ff = gx.FeatureFile.open(path, "file", ctx=gx.Context.default())
    fd = gx.FeatureFile.from_array(rows)
    train = oracle.train_ids(n, 1, 0.2)
    plan = oracle.plan_seed_batches(train, 48, oracle.epoch_seed(1, 0))[:12]
    p = gx.Pipeline(g, ff, [6, 4], K, digest=True)
    pd = gx.Pipeline(g, fd, [6, 4], K)
    trace = [oracle.sample_batch(ip, ind, b, [6, 4], oracle.derive_seed(1, i))[0] for i, b in enumerate(plan)]
    sim = oracle.simulate(trace, n, K, oracle.compute_init_set(trace, K, n))
    for rep in range(2):
        st = p.run_superbatch(plan, 1, 0)
        sd = pd.run_superbatch(plan, 1, 0)
        assert np.array_equal(st.misses, sim["misses"])
        assert st.total_misses == st.predicted_misses
        dig = p.digests()
        for i, ids in enumerate(trace):
            assert int(dig[i]) == gx.batch_digest(rows[ids.astype(np.int64)])
            assert np.array_equal(p.batch(i), rows[ids.astype(np.int64)])
        assert st.storage_rows == st.init_size + st.total_misses
        assert st.gather_io == sd.gather_io and st.sample_io == sd.sample_io
        assert (st.total_in, st.total_out, st.init_size) == (sd.total_in, sd.total_out, sd.init_size)
