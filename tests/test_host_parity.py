"""Host half of the product (librecoil.so C++: model, encoder + split heuristic,
container, combine, task planning, CPU decoder) vs the oracle, on CPU.

Containers must be byte-identical to the oracle's (same bitstream, final states,
split choice and metadata); decodes must equal the input.
"""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import synth
from paper_2306_12141_b200 import recoil as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()


def test_library_exports_every_declared_symbol():
    """include/recoil.h declarations == exported symbols; the binding wraps them all."""
    hdr = open(os.path.join(ROOT, "include", "recoil.h")).read()
    declared = set(re.findall(r"^\s*(?:const char \*|void |int )\s*\*?(recoil_\w+)\(", hdr, re.M))
    assert declared == set(R.EXPORTS)
    lib = ctypes.CDLL(R.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert R.recoil_strerror(R.RECOIL_E_SYNC) and R.recoil_strerror(0) == "ok"


def test_build_model_matches_oracle():
    rng = np.random.default_rng(4)
    for _ in range(300):
        n = int(rng.integers(1, 17))
        k = int(rng.integers(1, min(256, 1 << n) + 1))
        hist = np.zeros(256, dtype=np.uint64)
        hist[rng.choice(256, size=k, replace=False)] = rng.integers(1, 10 ** int(rng.integers(1, 8)), size=k)
        assert (R.recoil_build_model(hist, n) == oracle.build_model(hist, n)).all()
    with pytest.raises(R.RecoilError) as e:
        R.recoil_build_model(np.zeros(256), 11)
    assert e.value.rc == R.RECOIL_E_EMPTY
    with pytest.raises(R.RecoilError) as e:
        R.recoil_build_model(np.ones(256), 7)
    assert e.value.rc == R.RECOIL_E_ALPHABET


FUZZ = [(kind, N, n, M) for kind in ("exp", "text", "image")
        for N, n, M in ((0, 11, 4), (1, 11, 4), (31, 11, 3), (32, 8, 2), (33, 12, 5), (1000, 11, 7),
                        (50000, 11, 16), (50000, 12, 200), (200000, 16, 33), (300000, 5, 64))]


@pytest.mark.parametrize("kind,N,n,M", FUZZ)
def test_container_byte_identical_to_oracle(kind, N, n, M):
    sym = synth.workload(kind, N, seed=N + n + M, lam=30)
    hist = synth.histogram(sym) if N else np.ones(256, dtype=np.uint64)
    if (hist > 0).sum() > (1 << n):
        pytest.skip("alphabet larger than 2^n")
    f = oracle.build_model(hist, n)
    c = R.recoil_encode(sym, f, n, M)
    assert c.tobytes() == oracle.recoil_encode(sym, f, n, M)
    assert (R.recoil_decode_cpu(c) == sym).all()
    info = R.recoil_inspect(c)
    oi = oracle.container_info(c.tobytes())
    assert (info["n_symbols"], info["n_words"], info["n_splits"]) == (oi["N"], oi["B"], oi["M"])


@pytest.mark.parametrize("lam,M", [(10, 2176), (50, 2176), (200, 700), (500, 64)])
def test_container_identical_mid_size(lam, M):
    sym = synth.exp_bytes(3_000_000, lam, seed=lam)
    f = oracle.build_model(synth.histogram(sym), 11)
    c = R.recoil_encode(sym, f, 11, M)
    assert c.tobytes() == oracle.recoil_encode(sym, f, 11, M)
    assert (R.recoil_decode_cpu(c) == sym).all()


def test_combine_identical_to_oracle():
    sym = synth.text_bytes(2_000_000, 21)
    f = oracle.build_model(synth.histogram(sym), 11)
    c = R.recoil_encode(sym, f, 11, 2176)
    for target in (1, 2, 3, 16, 100, 1000, 2175, 2176, 5000):
        a = R.recoil_combine_splits(c, target)
        assert a.tobytes() == oracle.combine(c.tobytes(), target)
        assert (R.recoil_decode_cpu(a, 3) == sym).all()
    a = c
    for target in (1000, 300, 17, 4):
        a = R.recoil_combine_splits(a, target)
        assert (R.recoil_decode_cpu(a) == sym).all()


def test_partitioned_identical_to_oracle():
    for N, P in ((0, 3), (5, 4), (1000, 64), (300000, 1), (300000, 17), (300000, 2176)):
        sym = synth.text_bytes(N, N + P)
        f = oracle.build_model(synth.histogram(sym) if N else np.ones(256, dtype=np.uint64), 11)
        c = R.recoil_partitioned_encode(sym, f, 11, P)
        assert c.tobytes() == oracle.partitioned_encode(sym, f, 11, P)
        assert (R.recoil_decode_cpu(c) == sym).all()


def test_cpu_decoder_thread_invariance_and_oracle_tasks():
    sym = synth.image_bytes(1_500_000, 5)
    f = oracle.build_model(synth.histogram(sym), 11)
    c = R.recoil_encode(sym, f, 11, 300)
    outs = [R.recoil_decode_cpu(c, t) for t in (1, 2, 8)]
    assert all((o == sym).all() for o in outs)
    # the oracle's literal 3-phase decode of single tasks agrees on their ranges
    for t in (0, 1, 150, 299):
        out, lo, hi = oracle.recoil_decode_task(c.tobytes(), t)
        assert (out[lo:hi + 1] == sym[lo:hi + 1]).all()


def test_n16_outputs_before_group_zero():
    """n = 16 and f(s_0) = 1: Eq. 3 emits before the first symbol is encoded (x = L >= f 2^16);
    the decoder must read those words after group 0 (oracle: final refill pass)."""
    rng = np.random.default_rng(8)
    hist = np.zeros(256, dtype=np.uint64)
    hist[:200] = rng.integers(1, 5, size=200)
    hist[7] = 10 ** 7
    f = oracle.build_model(hist, 16)
    rare = [s for s in range(256) if f[s] == 1]
    assert rare
    sym = synth.table_bytes(50000, (f / f.sum()).tolist(), 4)
    sym[:32] = rare[0]  # every lane starts with an f = 1 symbol
    words, fin, ev, _ = oracle.interleaved_encode(sym, f, 16, 32)
    assert (ev["idx"] < 0).sum() == 32  # 32 emissions before group 0
    for M in (1, 5):
        c = R.recoil_encode(sym, f, 16, M)
        assert c.tobytes() == oracle.recoil_encode(sym, f, 16, M)
        assert (R.recoil_decode_cpu(c) == sym).all()
    p = R.recoil_partitioned_encode(sym, f, 16, 7)
    assert (R.recoil_decode_cpu(p) == sym).all()


def test_single_symbol_and_tiny_streams():
    f = np.zeros(256, dtype=np.uint32)
    f[200] = 1 << 11
    sym = np.full(5000, 200, dtype=np.uint8)
    c = R.recoil_encode(sym, f, 11, 10)
    assert R.recoil_inspect(c)["n_words"] == 0 and R.recoil_inspect(c)["n_splits"] == 1
    assert c.tobytes() == oracle.recoil_encode(sym, f, 11, 10)
    assert (R.recoil_decode_cpu(c) == sym).all()


def test_errors():
    sym = synth.exp_bytes(10000, 50, 3)
    f = oracle.build_model(synth.histogram(sym), 11)
    c = R.recoil_encode(sym, f, 11, 8)
    bad = c.copy()
    bad[0] ^= 0xFF
    with pytest.raises(R.RecoilError) as e:
        R.recoil_inspect(bad)
    assert e.value.rc == R.RECOIL_E_BAD_MAGIC
    with pytest.raises(R.RecoilError) as e:
        R.recoil_inspect(c[:-1])
    assert e.value.rc in (R.RECOIL_E_TRUNCATED, R.RECOIL_E_INCONSISTENT)
    with pytest.raises(R.RecoilError) as e:
        R.recoil_inspect(c[:20])
    assert e.value.rc == R.RECOIL_E_TRUNCATED
    f0 = f.copy()
    f0[sym[0]] = 0
    f0[[i for i in range(256) if f[i] == 0][0]] = f[sym[0]]
    with pytest.raises(R.RecoilError) as e:
        R.recoil_encode(sym, f0, 11, 4)
    assert e.value.rc == R.RECOIL_E_ZERO_FREQ
    with pytest.raises(R.RecoilError):
        R.recoil_encode(sym, f, 17, 4)
    # flipped offset making the metadata non-monotone is rejected
    info = R.recoil_inspect(c)
    assert info["n_splits"] == 8


def test_decoder_plan_layout():
    sym = synth.exp_bytes(400000, 50, 6)
    f = oracle.build_model(synth.histogram(sym), 11)
    c = R.recoil_encode(sym, f, 11, 64)
    h = R.recoil_decoder_create(c)
    p = R.recoil_decoder_plan(h)
    assert p["n_tasks"] == 64 and p["word_lo"] == 0 and p["word_count"] % 256 == 0
    assert p["word_count"] >= R.recoil_inspect(c)["n_words"]
    assert (p["out_lo"], p["out_hi"], p["out_base"]) == (0, len(sym), 0)
    assert p["out_count"] == (len(sym) + 15) // 16 * 16
    R.recoil_decoder_destroy(h)
    bounds = R.recoil_shard_plan(c, 4)
    assert bounds[0] == 0 and bounds[-1] == 64 and bounds == sorted(bounds)
    spans = []
    for a, b in zip(bounds, bounds[1:]):
        h = R.recoil_decoder_create(c, a, b)
        p = R.recoil_decoder_plan(h)
        assert p["word_lo"] % 256 == 0 and p["out_base"] % 512 == 0 and p["out_base"] <= p["out_lo"]
        assert p["out_count"] >= p["out_hi"] - p["out_base"] and p["out_count"] % 16 == 0
        spans.append((p["out_lo"], p["out_hi"]))
        R.recoil_decoder_destroy(h)
    assert spans[0][0] == 0 and spans[-1][1] == len(sym)
    assert all(spans[i][1] == spans[i + 1][0] for i in range(len(spans) - 1))
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 2 * len(sym) / 64
    c16 = R.recoil_encode(sym, oracle.build_model(synth.histogram(sym), 16), 16, 4)
    h = R.recoil_decoder_create(c16)  # n = 16: split-table LUT (2^16 symbol bytes + f, F)
    p16 = R.recoil_decoder_plan(h)
    assert p16["prob_bits"] == 16 and p16["workspace_bytes"] >= (1 << 16) + 1024
    R.recoil_decoder_destroy(h)


@pytest.mark.skipif(not R.recoil_cpu_simd(), reason="CPU lacks AVX2 and AVX-512")
@pytest.mark.parametrize("n", list(range(1, 17)))
def test_avx512_cpu_decoder_matches_scalar_and_input(n):
    """NEXT row 3: the SIMD task decoders -- AVX-512 (expand-load refill + LUT gathers) and
    AVX2 (8 lanes x 4: per-vector word run + mask-indexed permutation) -- equal the scalar
    decoder and the input, for every n (packed LUT n <= 12, split tables above)."""
    kind = ("exp", "text", "image")[n % 3]
    sym = synth.workload(kind, 400_001 + 37 * n, seed=100 + n, lam=50)
    hist = synth.histogram(sym)
    if (hist > 0).sum() > (1 << n):
        sym = (sym % (1 << min(n, 8))).astype(np.uint8)
        hist = synth.histogram(sym)
    f = oracle.build_model(hist, n)
    for M in (1, 7, 333):
        c = R.recoil_encode(sym, f, n, M)
        a = R.recoil_decode_cpu_ex(c, 4, 0)
        b = R.recoil_decode_cpu_ex(c, 4, R.RECOIL_CPU_SCALAR)
        v = R.recoil_decode_cpu_ex(c, 4, R.RECOIL_CPU_AVX2)
        assert (a == sym).all() and (b == sym).all() and (v == sym).all()
    p = R.recoil_partitioned_encode(sym, f, n, 13)
    assert (R.recoil_decode_cpu_ex(p, 3, 0) == sym).all()
    assert (R.recoil_decode_cpu_ex(p, 3, R.RECOIL_CPU_AVX2) == sym).all()


@pytest.mark.skipif(not R.recoil_cpu_simd(), reason="CPU lacks AVX2 and AVX-512")
def test_avx512_cpu_decoder_edges_and_corruption():
    rng = np.random.default_rng(8)
    hist = np.zeros(256, dtype=np.uint64)
    hist[:200] = rng.integers(1, 5, size=200)
    hist[7] = 10 ** 7
    f = oracle.build_model(hist, 16)
    rare = [s for s in range(256) if f[s] == 1]
    sym = synth.table_bytes(50000, (f / f.sum()).tolist(), 4)
    sym[:32] = rare[0]  # n = 16 emissions before group 0
    for c in (R.recoil_encode(sym, f, 16, 5), R.recoil_partitioned_encode(sym, f, 16, 7)):
        assert (R.recoil_decode_cpu_ex(c, 2, 0) == sym).all()
        assert (R.recoil_decode_cpu_ex(c, 2, R.RECOIL_CPU_AVX2) == sym).all()
    for N in (0, 1, 31, 32, 33, 95):  # empty / ragged groups
        s = synth.text_bytes(N, N)
        ff = oracle.build_model(synth.histogram(s) if N else np.ones(256, dtype=np.uint64), 11)
        for flags in (0, R.RECOIL_CPU_AVX2):
            assert (R.recoil_decode_cpu_ex(R.recoil_encode(s, ff, 11, 3), 1, flags) == s).all()
    s = synth.text_bytes(300000, 9)
    ff = oracle.build_model(synth.histogram(s), 11)
    c = R.recoil_encode(s, ff, 11, 16)
    info = R.recoil_inspect(c)
    bad = c.copy()
    hdr = len(c) - 2 * info["n_words"]
    bad[hdr + 2 * (info["n_words"] // 2)] ^= 0x5A  # flip a bitstream word
    errs = []
    for flags in (0, R.RECOIL_CPU_SCALAR, R.RECOIL_CPU_AVX2):
        try:
            out = R.recoil_decode_cpu_ex(bad, 2, flags)
            errs.append(("ok", int((out != s).sum() > 0)))
        except R.RecoilError as e:
            errs.append(("err", e.rc))
    assert errs[0] == errs[1] == errs[2]  # same verdict from every decoder


def _ad_random_models(rng, n, K, max_len=300):
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


@pytest.mark.parametrize("seed", range(8))
def test_adaptive_container_byte_identical_to_oracle(seed):
    """NEXT rows 1 + 4: adaptive (index-keyed models, 16-bit symbols) containers == the oracle's."""
    rng = np.random.default_rng(seed)
    n = int(rng.choice([1, 3, 8, 11, 12, 16]))
    K = int(rng.integers(1, 12))
    models = _ad_random_models(rng, n, K)
    N = int(rng.choice([0, 1, 31, 33, 1000, 70000]))
    mid = rng.integers(0, K, size=N).astype(np.uint8)
    off = np.concatenate([[0], np.cumsum(models["len"].astype(np.int64))])
    sym = np.zeros(N, np.uint16)
    for k in range(K):
        sel = np.nonzero(mid == k)[0]
        if sel.size:
            f = models["f"][off[k]:off[k + 1]].astype(np.float64)
            sym[sel] = models["base"][k] + rng.choice(len(f), size=sel.size, p=f / f.sum())
    for M in (1, 5, 77):
        c = R.recoil_encode_adaptive(sym, mid, models, n, M)
        assert c.tobytes() == oracle.ad_recoil_encode(sym, mid, models, n, M)
        info = R.recoil_inspect(c)
        assert info["symbol_bits"] == 16 and info["n_models"] == K and info["n_symbols"] == N
        for target in (2, 1):
            assert R.recoil_combine_splits(c, target).tobytes() == oracle.combine(c.tobytes(), target)


def test_adaptive_quantize_and_errors():
    rng = np.random.default_rng(2)
    for _ in range(30):
        count = int(rng.integers(1, 3000))
        n = int(rng.integers(max(1, int(np.ceil(np.log2(count + 1)))), 17)) if count < 65536 else 16
        hist = rng.integers(0, 1000, size=count).astype(np.uint64)
        if not hist.any():
            hist[0] = 1
        if (hist > 0).sum() > (1 << n):
            continue
        assert (R.recoil_quantize(hist, n) == oracle.quantize(hist, n)).all()
    models = {"base": [100], "len": [4], "f": oracle.quantize(np.array([1, 2, 3, 0], np.uint64), 11)}
    sym = np.array([100, 101, 102], np.uint16)
    mid = np.zeros(3, np.uint8)
    R.recoil_encode_adaptive(sym, mid, models, 11, 1)
    for bad in (np.array([100, 103, 102], np.uint16), np.array([99, 100, 101], np.uint16)):
        with pytest.raises(R.RecoilError) as e:
            R.recoil_encode_adaptive(bad, mid, models, 11, 1)
        assert e.value.rc == R.RECOIL_E_ZERO_FREQ
    with pytest.raises(R.RecoilError) as e:
        R.recoil_encode_adaptive(sym, np.array([0, 1, 0], np.uint8), models, 11, 1)
    assert e.value.rc == R.RECOIL_E_ZERO_FREQ
    c = R.recoil_encode_adaptive(sym, mid, models, 11, 1)
    with pytest.raises(R.RecoilError) as e:
        R.recoil_decode_cpu(c)
    assert e.value.rc == R.RECOIL_E_UNSUPPORTED


def test_decoder_side_combine_plans_equal_combined_containers():
    """recoil_decoder_create_subset plans exactly what decoding recoil_combine_splits' output plans."""
    sym = synth.exp_bytes(2_000_000, 50, 3)
    f = R.recoil_build_model(synth.histogram(sym), 11)
    c = R.recoil_encode(sym, f, 11, 1000)
    keys = ("n_tasks", "word_lo", "word_count", "out_lo", "out_hi", "out_base", "out_count")
    for target in (5000, 1000, 999, 300, 17, 2, 1):
        h = R.recoil_decoder_create_subset(c, target)
        p = R.recoil_decoder_plan(h)
        R.recoil_decoder_destroy(h)
        h2 = R.recoil_decoder_create(R.recoil_combine_splits(c, target))
        p2 = R.recoil_decoder_plan(h2)
        R.recoil_decoder_destroy(h2)
        assert all(p[k] == p2[k] for k in keys), target
    with pytest.raises(R.RecoilError):
        R.recoil_decoder_create_subset(R.recoil_partitioned_encode(sym, f, 11, 8), 2)


def test_grouped_plans():
    """recoil_decoder_create_grouped: uniform runs of k splits plan exactly what the combine rule
    (points k, 2k, ...) plans; mixed runs give the requested task count; bad runs fail."""
    sym = synth.exp_bytes(2_000_000, 50, 3)
    f = R.recoil_build_model(synth.histogram(sym), 11)
    c = R.recoil_encode(sym, f, 11, 1000)
    M = R.recoil_inspect(c)["n_splits"]
    keys = ("n_tasks", "word_lo", "word_count", "out_lo", "out_hi", "out_base", "out_count")
    for k in (1, 2, 3, 7, 999, 1000, 5000):
        h = R.recoil_decoder_create_grouped(c, [M], [k])
        p = R.recoil_decoder_plan(h)
        R.recoil_decoder_destroy(h)
        h2 = R.recoil_decoder_create_subset(c, -(-M // k))
        p2 = R.recoil_decoder_plan(h2)
        R.recoil_decoder_destroy(h2)
        assert all(p[key] == p2[key] for key in keys), k
    # long tasks first, short ones last: 300 tasks of 2 splits, then single splits
    h = R.recoil_decoder_create_grouped(c, [300, M], [2, 1])
    p = R.recoil_decoder_plan(h)
    R.recoil_decoder_destroy(h)
    assert p["n_tasks"] == 300 + (M - 600) and (p["out_lo"], p["out_hi"]) == (0, len(sym))
    for bad in (([], []), ([5], [0])):
        with pytest.raises((R.RecoilError, ValueError)):
            R.recoil_decoder_create_grouped(c, *bad)
    with pytest.raises(R.RecoilError):
        R.recoil_decoder_create_grouped(R.recoil_partitioned_encode(sym, f, 11, 8), [2], [2])


@pytest.mark.parametrize("E,cbits,warps", [(5000, 9, 32), (12000, 8, 32), (18000, 7, 32), (24000, 6, 8)])
def test_adaptive_plan_coarse_bits(E, cbits, warps):
    """The host plan picks the most coarse-bucket bits (9..7) whose tables fit beside the
    32-warp layout in one block's shared memory, else 6 bits on 8-warp CTAs (no GPU needed)."""
    K, length = 64, E // 64
    rng = np.random.default_rng(E)
    fs = [R.recoil_quantize(rng.integers(1, 1000, size=length).astype(np.uint64), 16) for _ in range(K)]
    models = {"base": np.arange(K, dtype=np.uint32) * 700, "len": np.full(K, length, np.uint32),
              "f": np.concatenate(fs)}
    mid = rng.integers(0, K, size=5000).astype(np.uint8)
    sym = (models["base"][mid] + rng.integers(0, length, size=5000)).astype(np.uint16)
    c = R.recoil_encode_adaptive(sym, mid, models, 16, 4)
    h = R.recoil_decoder_create(c)
    plan = R.recoil_decoder_plan(h)
    R.recoil_decoder_destroy(h)
    assert (plan["coarse_bits"], plan["warps_per_block"]) == (cbits, warps)


def test_multi_plan_equals_shard_plan_and_decoder_plans():
    """recoil_multi_plan (C ABI multi-GPU entry, §8(b)) = recoil_shard_plan's ranges with
    each range's decoder plan; the spans tile [0, N)."""
    import synth
    from paper_2306_12141_b200 import recoil as R
    sym = synth.workload("text", 500_000, seed=7)
    f = R.recoil_build_model(synth.histogram(sym), 11)
    c = R.recoil_encode(sym, f, 11, 120)
    for n_dev in (1, 2, 5, 8):
        plans = R.recoil_multi_plan(c, n_dev)
        bounds = R.recoil_shard_plan(c, n_dev)
        lo = 0
        for d, p in enumerate(plans):
            h = R.recoil_decoder_create(c, bounds[d], bounds[d + 1])
            want = R.recoil_decoder_plan(h)
            R.recoil_decoder_destroy(h)
            assert p == want
            assert p["out_lo"] == lo
            lo = p["out_hi"]
        assert lo == len(sym)
    with pytest.raises(R.RecoilError):
        R.recoil_multi_plan(c, 0)


def test_device_range_decoder_arguments():
    """recoil_device_decoder_create_range checks the range on the host (no GPU call)."""
    import ctypes
    sym = synth.text_bytes(200_000, 3)
    f = R.recoil_build_model(synth.histogram(sym), 11)
    c = R.recoil_encode(sym, f, 11, 10)
    lib = R.load()
    for tb, te, ok in [(0, 10, True), (3, 7, True), (9, 10, True), (0, (1 << 64) - 1, True), (5, 5, False),
                       (6, 5, False), (0, 11, False), (10, 11, False)]:
        h = ctypes.c_void_p()
        rc = lib.recoil_device_decoder_create_range(c.ctypes.data, c.size, c.size, tb, te, ctypes.byref(h))
        assert (rc == 0) == ok, (tb, te, rc)
        if rc == 0:
            pl = R.recoil_device_plan()
            assert lib.recoil_device_decoder_plan(h, ctypes.byref(pl)) == 0
            assert pl.n_tasks == (10 if te > 10 else te) - tb
            lib.recoil_device_decoder_destroy(h)
