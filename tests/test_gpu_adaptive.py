"""GPU parity of the adaptive decode (index-keyed models, 16-bit symbols; NEXT rows 1 + 4,
P:227 item (3)) through the C ABI, against the adaptive oracle and the input.
Bit-exact (integer path)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2306_12141_b200 import recoil as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()
    assert torch.cuda.is_available()


def _random_models(rng, n, K, max_len=300):
    base, ln, fs = [], [], []
    for _ in range(K):
        length = int(rng.integers(1, min(max_len, 1 << n) + 1))
        b = int(rng.integers(0, 65536 - length + 1))
        hist = rng.integers(1, 10 ** int(rng.integers(1, 6)), size=length).astype(np.uint64)
        hist[rng.random(length) < 0.2] = 0
        if not hist.any():
            hist[0] = 1
        base.append(b)
        ln.append(length)
        fs.append(oracle.quantize(hist, n))
    return {"base": np.array(base, np.uint32), "len": np.array(ln, np.uint32), "f": np.concatenate(fs)}


def _draw(rng, models, N, K):
    mid = rng.integers(0, K, size=N).astype(np.uint8)
    off = np.concatenate([[0], np.cumsum(models["len"].astype(np.int64))])
    sym = np.zeros(N, np.uint16)
    for k in range(K):
        sel = np.nonzero(mid == k)[0]
        if sel.size:
            f = models["f"][off[k]:off[k + 1]].astype(np.float64)
            sym[sel] = models["base"][k] + rng.choice(len(f), size=sel.size, p=f / f.sum())
    return sym, mid


def gpu_decode_adaptive(c, mid, task_begin=0, task_end=(1 << 64) - 1):
    dec = R.GpuDecoder(c, 0, task_begin, task_end)
    dec.set_model_ids(mid)
    dec.upload()
    dec.decode()
    rc, bad = dec.status()
    out = dec.output().cpu().numpy().view(np.uint16)
    plan = dec.plan
    dec.close()
    return rc, bad, out, plan


def _check(c, mid, sym, oracle_check=True):
    rc, bad, out, plan = gpu_decode_adaptive(c, mid)
    assert rc == 0, (R.ERRORS.get(rc), bad)
    assert plan["symbol_bytes"] == 2 and (plan["out_lo"], plan["out_hi"]) == (0, len(sym))
    if oracle_check:
        assert (oracle.ad_recoil_decode(bytes(c), mid) == sym).all()
    mism = np.nonzero(out != sym)[0]
    assert mism.size == 0, f"{mism.size} mismatches, first at {mism[:5]}"


# (N, n, K models, M splits)
CASES = [(1, 16, 1, 2), (31, 16, 3, 2), (33, 11, 2, 3), (511, 12, 4, 5), (513, 16, 4, 7), (5000, 1, 2, 3),
         (5000, 5, 7, 4), (20000, 8, 9, 8), (100000, 11, 33, 16), (300000, 16, 64, 500), (1 << 20, 16, 200, 2176),
         (777777, 14, 40, 4096)]


@pytest.mark.parametrize("N,n,K,M", CASES)
def test_random_models_vs_oracle(N, n, K, M):
    rng = np.random.default_rng(N + n + K)
    models = _random_models(rng, n, K)
    sym, mid = _draw(rng, models, N, K)
    c = R.recoil_encode_adaptive(sym, mid, models, n, M)
    assert c.tobytes() == oracle.ad_recoil_encode(sym, mid, models, n, M)
    _check(c, mid, sym, oracle_check=N <= 400_000)


@pytest.mark.parametrize("N,M", [(200_000, 1), (200_000, 64), (2_000_000, 2176), (1 << 24, 7104)])
def test_latent_workload(N, M):
    sym, mid, h = synth.latent_workload(N, 11)
    f = np.concatenate([R.recoil_quantize(x, 16) for x in h["hist"]])
    models = {"base": h["base"], "len": h["len"], "f": f}
    c = R.recoil_encode_adaptive(sym, mid, models, 16, M)
    if N <= 2_000_000:
        assert c.tobytes() == oracle.ad_recoil_encode(sym, mid, models, 16, M)
    _check(c, mid, sym, oracle_check=N <= 2_000_000)


def test_sharded_task_ranges_and_combine():
    sym, mid, h = synth.latent_workload(1_500_000, 5)
    f = np.concatenate([R.recoil_quantize(x, 16) for x in h["hist"]])
    models = {"base": h["base"], "len": h["len"], "f": f}
    c = R.recoil_encode_adaptive(sym, mid, models, 16, 1000)
    bounds = R.recoil_shard_plan(c, 3)
    got = np.zeros(len(sym), np.uint16)
    for a, b in zip(bounds, bounds[1:]):
        rc, bad, out, plan = gpu_decode_adaptive(c, mid, a, b)
        assert rc == 0
        got[plan["out_lo"]:plan["out_hi"]] = out
    assert (got == sym).all()
    for target in (100, 7, 1):
        _check(R.recoil_combine_splits(c, target), mid, sym, oracle_check=False)


def test_n16_outputs_before_group_zero_adaptive():
    """A model with f = 1 values: lanes whose first symbol has f = 1 emit before group 0 (n = 16)."""
    rng = np.random.default_rng(3)
    hist = np.ones(300, np.uint64)
    hist[0] = 10 ** 9
    f0 = oracle.quantize(hist, 16)
    assert (f0 == 1).any()
    models = {"base": np.array([1000, 0], np.uint32), "len": np.array([300, 300], np.uint32),
              "f": np.concatenate([f0, f0[::-1]])}
    mid = rng.integers(0, 2, size=40000).astype(np.uint8)
    sym = np.where(mid == 0, 1000, 299).astype(np.uint16)
    sym[:32] = np.where(mid[:32] == 0, 1001, 0)  # f = 1 values first
    for M in (1, 5):
        c = R.recoil_encode_adaptive(sym, mid, models, 16, M)
        assert c.tobytes() == oracle.ad_recoil_encode(sym, mid, models, 16, M)
        _check(c, mid, sym)


def test_wrong_model_ids_and_static_entry_point():
    sym, mid, h = synth.latent_workload(100_000, 2)
    f = np.concatenate([R.recoil_quantize(x, 16) for x in h["hist"]])
    c = R.recoil_encode_adaptive(sym, mid, {"base": h["base"], "len": h["len"], "f": f}, 16, 16)
    rc, bad, out, plan = gpu_decode_adaptive(c, np.roll(mid, 7))
    assert rc != 0 or (out != sym).any()
    dec = R.GpuDecoder(c, 0)
    dec.upload()
    with pytest.raises(R.RecoilError):
        R.recoil_decode(dec.handle, dec.workspace.data_ptr(), dec.words.data_ptr(), dec.out.data_ptr(),
                        dec.stream_handle)
    dec.close()


@pytest.mark.parametrize("K,length", [(4, 7000), (2, 20000)])
def test_large_model_tables_use_narrow_ctas(K, length):
    """Model tables too large for the 32-warp CTA layout (~100 KB of tables) run on the 8-warp
    adaptive kernel; the occupancy query reports the same geometry; output bit-exact."""
    rng = np.random.default_rng(K * length)
    base, ln, fs = [], [], []
    for k in range(K):
        hist = rng.integers(1, 1000, size=length).astype(np.uint64)
        base.append(k * length)
        ln.append(length)
        fs.append(oracle.quantize(hist, 16))
    models = {"base": np.array(base, np.uint32), "len": np.array(ln, np.uint32), "f": np.concatenate(fs)}
    table_bytes = (K * 258 * 2 + 15) // 16 * 16 + 4 * (K * length + K)  # 8-bit coarse buckets
    assert table_bytes > 105_000  # the 32-warp layout (125 KB) leaves ~102 KB of the 227 KB
    warps, _ = R.recoil_decode_occupancy_adaptive(0, K, K * length)
    assert warps >= 8 and warps % 8 == 0 and warps != 32  # 8-warp CTAs
    sym, mid = _draw(rng, models, 300_000, K)
    c = R.recoil_encode_adaptive(sym, mid, models, 16, 64)
    _check(c, mid, sym, oracle_check=True)


# K = 64 models of E / 64 entries each (all f > 0): the table sizes force each coarse-bucket
# choice of the plan (2^9, 2^8, 2^7 buckets on the 32-warp kernel; 2^6 on the 8-warp one).
CBITS_CASES = [(5000, 9, 32), (12000, 8, 32), (18000, 7, 32), (24000, 6, 8)]


def _cbits_models(E, K=64, seed=0):
    rng = np.random.default_rng(seed + E)
    length = E // K
    fs = [oracle.quantize(rng.integers(1, 1000, size=length).astype(np.uint64), 16) for _ in range(K)]
    return {"base": np.arange(K, dtype=np.uint32) * 700, "len": np.full(K, length, np.uint32),
            "f": np.concatenate(fs)}


@pytest.mark.parametrize("E,cbits,warps", CBITS_CASES)
def test_coarse_bits_choice_each_geometry(E, cbits, warps):
    models = _cbits_models(E)
    rng = np.random.default_rng(E)
    sym, mid = _draw(rng, models, 400_000, 64)
    c = R.recoil_encode_adaptive(sym, mid, models, 16, 300)
    rc, bad, out, plan = gpu_decode_adaptive(c, mid)
    assert (plan["coarse_bits"], plan["warps_per_block"]) == (cbits, warps)
    assert rc == 0 and (out == sym).all()
    w, _ = R.recoil_decode_occupancy_adaptive(0, 64, E)
    assert (w == 32) == (warps == 32)  # the occupancy query (trimmed entry count) agrees with the plan
