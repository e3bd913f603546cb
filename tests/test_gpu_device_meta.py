"""On-device metadata path: the container goes to
the GPU unchanged, the split metadata is decoded there (global series, split-record
offsets by a speculative chunked parse, LUT, task heads) and the decode kernel reads the
records in place.  Every output byte is compared with the input (the decode's definition)
and with the oracle's decode; the GPU combine is compared byte for byte with the oracle's
combine (O8) and the library's."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2306_12141_b200 import recoil as R

pytestmark = pytest.mark.gpu


def _enc(kind, n, M, nbits=11, seed=3):
    sym = synth.workload(kind, n, seed=seed, lam=50)
    hist = synth.histogram(sym) if n else np.ones(256, np.uint64)
    if (hist > 0).sum() > (1 << nbits):
        sym = (sym % (1 << min(nbits, 8))).astype(np.uint8)
        hist = synth.histogram(sym)
    f = R.recoil_build_model(hist, nbits)
    return sym, R.recoil_encode(sym, f, nbits, M)


def _device_decode(c):
    dd = R.DeviceContainerDecoder(c, 0)
    dd.upload()
    dd.decode()
    rc, bad = dd.status()
    out = dd.output().cpu().numpy()
    dd.close()
    return rc, bad, out


@pytest.mark.parametrize("kind,n,M", [("exp", 1 << 20, 16), ("text", 3_000_017, 700), ("image", 5_000_000, 4000),
                                      ("exp", 100_000, 1), ("text", 33, 3), ("exp", 0, 5), ("image", 2_000_000, 20000)])
def test_device_parse_decodes_bit_exact(kind, n, M):
    sym, c = _enc(kind, n, M)
    rc, bad, out = _device_decode(c)
    assert rc == 0, (R.ERRORS.get(rc), bad)
    assert np.array_equal(out, sym)
    if n and n <= 3_000_017:
        assert np.array_equal(oracle.recoil_decode(c.tobytes()), out)


@pytest.mark.parametrize("nbits", [1, 4, 9, 12, 13, 16])
def test_device_parse_every_lut_form(nbits):
    sym, c = _enc("exp", 400_001, 97, nbits, seed=nbits)
    rc, _, out = _device_decode(c)
    assert rc == 0 and np.array_equal(out, sym)


def test_device_parse_many_chunks_and_wide_records():
    """65536 splits: ~5 MB of records over hundreds of parse chunks (config 4's encode)."""
    sym, c = _enc("exp", 1 << 26, 65536)
    assert R.recoil_inspect(c)["n_splits"] == 65536
    rc, _, out = _device_decode(c)
    assert rc == 0 and np.array_equal(out, sym)


def test_device_parse_single_symbol_model():
    sym = np.full(100_000, 7, np.uint8)
    f = R.recoil_build_model(synth.histogram(sym), 11)
    c = R.recoil_encode(sym, f, 11, 8)
    rc, _, out = _device_decode(c)
    assert rc == 0 and np.array_equal(out, sym)


def test_device_parse_matches_host_plan_on_corrupt_metadata():
    """Bytes flipped anywhere in the metadata (global series, anchor states, width fields):
    the device parse must agree with the host parse -- where the host rejects the container
    (E_INCONSISTENT / E_TRUNCATED) the device flags E_INCONSISTENT; where the host plans it,
    the device decode gives the same status and the same bytes.  (The format has no checksum:
    a flipped anchor state may decode to wrong bytes on both paths.)  Never a fault."""
    sym, c = _enc("text", 2_000_000, 500)
    info = R.recoil_inspect(c)
    meta_lo = info["header_bytes"] + 128
    meta_hi = len(c) - 2 * info["n_words"]
    rng = np.random.default_rng(5)
    flagged = 0
    for trial in range(40):
        cc = c.copy()
        pos = int(rng.integers(meta_lo, meta_hi)) if trial % 4 else int(rng.integers(meta_lo, meta_lo + 400))
        cc[pos] ^= np.uint8(1 << int(rng.integers(0, 8)))
        rc, _, out = _device_decode(cc)
        try:
            dec = R.GpuDecoder(cc, 0)
        except R.RecoilError as e:
            assert e.rc in (R.RECOIL_E_INCONSISTENT, R.RECOIL_E_TRUNCATED), e
            assert rc == R.RECOIL_E_INCONSISTENT, (pos, rc)
            flagged += 1
            continue
        dec.upload()
        dec.decode()
        hrc, _ = dec.status()
        hout = dec.output().cpu().numpy()
        dec.close()
        assert rc == hrc, (pos, rc, hrc)
        if rc == 0:
            assert np.array_equal(out, hout), pos
        else:
            flagged += 1
    assert flagged > 0


def test_device_parse_rejects_other_containers():
    sym = synth.workload("exp", 10_000, seed=1, lam=50)
    f = R.recoil_build_model(synth.histogram(sym), 11)
    p = R.recoil_partitioned_encode(sym, f, 11, 4)
    with pytest.raises(R.RecoilError):
        R.DeviceContainerDecoder(p, 0)
    with pytest.raises(R.RecoilError):
        R.DeviceContainerDecoder(np.zeros(64, np.uint8), 0)


@pytest.mark.parametrize("kind,n,M,targets", [("exp", 1 << 22, 2048, [1, 2, 16, 300, 2047, 2048, 5000]),
                                              ("text", 777_777, 97, [1, 3, 50, 96]),
                                              ("image", 1 << 24, 20000, [2048, 256, 16])])
def test_device_combine_equals_oracle_and_library(kind, n, M, targets):
    sym, c = _enc(kind, n, M)
    d_in = torch.from_numpy(c).cuda()
    for t in targets:
        got = R.recoil_device_combine(c, d_in, t).cpu().numpy()
        lib = R.recoil_combine_splits(c, t)
        assert np.array_equal(got, lib), t
        if n <= (1 << 22):
            assert got.tobytes() == oracle.combine(c.tobytes(), t), t
        rc, _, out = _device_decode(got)
        assert rc == 0 and np.array_equal(out, sym), t


def test_device_combine_config4_65536_to_2048_256_16():
    sym, c = _enc("exp", 1 << 26, 65536)
    d_in = torch.from_numpy(c).cuda()
    for t in (2048, 256, 16):
        got = R.recoil_device_combine(c, d_in, t).cpu().numpy()
        assert np.array_equal(got, R.recoil_combine_splits(c, t)), t


def test_device_parse_config5_split_density():
    """~150 000 splits (config 5's 8-GPU density over 2^27 symbols is 85 248 / 64; here denser):
    ~12 MB of split records, parse chunks larger than the minimum, every byte decoded."""
    sym, c = _enc("image", 1 << 27, 150_000)
    assert R.recoil_inspect(c)["n_splits"] > 140_000  # the encoder may find fewer points
    rc, _, out = _device_decode(c)
    assert rc == 0 and np.array_equal(out, sym)
    d_in = torch.from_numpy(c).cuda()
    got = R.recoil_device_combine(c, d_in, 10_000).cpu().numpy()
    assert np.array_equal(got, R.recoil_combine_splits(c, 10_000))


@pytest.mark.parametrize("kind,n,M,shards", [("text", 3_000_017, 700, 5), ("image", 2_000_000, 20000, 3),
                                             ("exp", 1 << 20, 16, 16), ("exp", 100_000, 2, 2)])
def test_device_task_ranges_shard_the_stream(kind, n, M, shards):
    """recoil_device_decoder_create_range (a multi-GPU shard on the device path): each
    range's committed span equals the host shard plan's, the spans tile [0, N), and every
    span's bytes equal the input (and the oracle's decode)."""
    sym, c = _enc(kind, n, M)
    bounds = R.recoil_shard_plan(c, shards)
    want = oracle.recoil_decode(c.tobytes()) if n <= 3_000_017 else sym
    assert np.array_equal(want, sym)
    prev_hi = 0
    for tb, te in zip(bounds[:-1], bounds[1:]):
        if tb == te:
            continue
        dd = R.DeviceContainerDecoder(c, 0, task_begin=tb, task_end=te)
        assert dd.plan["n_tasks"] == te - tb
        dd.upload()
        dd.decode()
        rc, bad = dd.status()
        assert rc == 0, (R.ERRORS.get(rc), bad)
        lo, hi = dd.span()
        host = R.GpuDecoder(c, 0, tb, te)
        assert (lo, hi) == (host.plan["out_lo"], host.plan["out_hi"])
        host.close()
        assert lo == prev_hi
        prev_hi = hi
        out = dd.output().cpu().numpy()
        dd.close()
        assert np.array_equal(out[lo:hi], sym[lo:hi])
    assert prev_hi == n


def test_device_task_range_single_tasks_and_edges():
    """One-task ranges at the first, a middle and the last task."""
    sym, c = _enc("text", 500_000, 40)
    for tb in (0, 17, 39):
        dd = R.DeviceContainerDecoder(c, 0, task_begin=tb, task_end=tb + 1)
        dd.upload()
        dd.decode()
        assert dd.status()[0] == 0
        lo, hi = dd.span()
        assert lo < hi and (tb > 0 or lo == 0) and (tb < 39 or hi == len(sym))
        assert np.array_equal(dd.output().cpu().numpy()[lo:hi], sym[lo:hi])
        dd.close()
