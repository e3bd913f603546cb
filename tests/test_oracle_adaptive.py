"""Pins of the adaptive-model oracle (index-keyed models, 16-bit symbols; P:227 item
(3)) to things other than itself.

* With one model equal to a static 8-bit model the adaptive codec is the static
  codec, which is pinned by tests/test_oracle_pins.py: identical words, final
  states and renormalisation events, and identical split records.
* The stack property: decode(encode(x)) = x, ending with every lane at L.
* The information content: compressed bits = sum log2(2^n / f_{mid(i)}(s_i)) up to
  the Eq. 1 floor loss.
* The Lemma: every post-emission state is < L.
* Brute force from every feasible split position (north_star), and combine chains.
* The model really is keyed by the index: decoding with other model ids fails or
  gives other symbols.
"""
import numpy as np
import pytest

import oracle
import synth

L = 1 << 16


def _random_models(rng, n, K, max_len=300):
    base, ln, fs = [], [], []
    for _ in range(K):
        length = int(rng.integers(1, min(max_len, 1 << n) + 1))
        b = int(rng.integers(0, 65536 - length + 1))
        hist = rng.integers(1, 10 ** int(rng.integers(1, 6)), size=length).astype(np.uint64)
        hist[rng.random(length) < 0.2] = 0  # some values not in the model
        if not hist.any():
            hist[0] = 1
        base.append(b)
        ln.append(length)
        fs.append(oracle.quantize(hist, n))
    return {"base": np.array(base, np.uint32), "len": np.array(ln, np.uint32), "f": np.concatenate(fs)}


def _draw(rng, models, N, K):
    """Symbols drawn from the models' own frequencies (test-side sampler)."""
    mid = rng.integers(0, K, size=N).astype(np.uint8)
    off = np.concatenate([[0], np.cumsum(models["len"].astype(np.int64))])
    sym = np.zeros(N, np.uint16)
    for k in range(K):
        sel = np.nonzero(mid == k)[0]
        if sel.size == 0:
            continue
        f = models["f"][off[k]:off[k + 1]].astype(np.float64)
        j = rng.choice(len(f), size=sel.size, p=f / f.sum())
        sym[sel] = models["base"][k] + j
    return sym, mid


def test_quantize_generalises_build_model():
    rng = np.random.default_rng(1)
    for _ in range(50):
        n = int(rng.integers(1, 17))
        hist = np.zeros(256, np.uint64)
        k = int(rng.integers(1, min(256, 1 << n) + 1))
        hist[rng.choice(256, size=k, replace=False)] = rng.integers(1, 10 ** 6, size=k)
        assert (oracle.quantize(hist, n) == oracle.build_model(hist, n)).all()
    f = oracle.quantize(np.ones(3000, np.uint64), 16)  # > 256 entries
    assert f.sum() == 1 << 16 and (f >= 1).all()


@pytest.mark.parametrize("n,W", [(8, 1), (11, 32), (16, 32), (12, 4)])
def test_single_model_equals_static_codec(n, W):
    """K = 1, base 0, len 256: the adaptive encoder IS the pinned static encoder."""
    sym = synth.exp_bytes(20000, 50, seed=n + W)
    f = oracle.build_model(synth.histogram(sym), n)
    models = {"base": [0], "len": [256], "f": f}
    mid = np.zeros(len(sym), np.uint8)
    w1, f1, e1, _ = oracle.interleaved_encode(sym, f, n, W)
    w2, f2, e2 = oracle.ad_interleaved_encode(sym.astype(np.uint16), mid, models, n, W)
    assert (w1 == w2).all() and (f1 == f2).all() and (e1 == e2).all()
    if W == 32:
        c1 = oracle.recoil_encode(sym, f, n, 40)
        c2 = oracle.ad_recoil_encode(sym.astype(np.uint16), mid, models, n, 40)
        p1, p2 = oracle.container_points(c1), oracle.container_points(c2)
        assert all((p1[k] == p2[k]).all() for k in p1)
        assert c1[-2 * len(w1):] == c2[-2 * len(w2):]  # same word section
        assert (oracle.ad_recoil_decode(c2, mid) == sym).all()


@pytest.mark.parametrize("seed", range(6))
def test_roundtrip_stack_property_info_content_lemma(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.choice([1, 4, 8, 11, 12, 15, 16]))
    K = int(rng.integers(1, 9))
    W = int(rng.choice([1, 2, 7, 32]))
    models = _random_models(rng, n, K)
    for N in (0, 1, W - 1, W, W + 1, 3000):
        if N < 0:
            continue
        sym, mid = _draw(rng, models, N, K)
        words, fin, ev = oracle.ad_interleaved_encode(sym, mid, models, n, W)
        assert (oracle.ad_interleaved_decode(words, fin, N, mid, models, n, W) == sym).all()
        assert (ev["state"] < L).all()  # Lemma: post-emission state < L
        if N >= 3000:
            off = np.concatenate([[0], np.cumsum(models["len"].astype(np.int64))])
            fi = models["f"][off[mid] + (sym.astype(np.int64) - models["base"][mid])]
            info = float(np.sum(n - np.log2(fi.astype(np.float64))))
            # words hold the information minus the final states' 32 bits/lane, up to the floor loss
            bits = 16 * len(words) + 32 * W
            assert info - 64 * W <= bits <= info * 1.003 + 64 * W


def test_model_ids_are_keys():
    rng = np.random.default_rng(5)
    models = _random_models(rng, 11, 4, max_len=40)
    sym, mid = _draw(rng, models, 5000, 4)
    words, fin, _ = oracle.ad_interleaved_encode(sym, mid, models, 11)
    other = np.roll(mid, 1)
    try:
        out = oracle.ad_interleaved_decode(words, fin, len(sym), other, models, 11)
        assert (out != sym).any()
    except oracle.OracleError:
        pass


@pytest.mark.parametrize("W,n", [(1, 11), (4, 16), (32, 16)])
def test_brute_force_every_split_position_adaptive(W, n):
    rng = np.random.default_rng(W + n)
    models = _random_models(rng, n, 5, max_len=60)
    sym, mid = _draw(rng, models, 1500 if W > 1 else 500, 5)
    words, fin, ev = oracle.ad_interleaved_encode(sym, mid, models, n, W)
    feasible = 0
    for e in range(len(ev)):
        r = oracle.backward_scan(ev, e, W)
        if r is None:
            continue
        st, ai, ss = r
        feasible += 1
        rc, out = oracle.ad_decode_from(words, mid, models, n, W, len(sym), e, int(ev["idx"][e]) // W, st, ai // W,
                                        0, ss)
        assert rc == 0
        assert (out[: ss + 1] == sym[: ss + 1]).all()
    assert feasible > 10


def test_latent_workload_container_and_combine():
    sym, mid, h = synth.latent_workload(200_000, 3)
    f = np.concatenate([oracle.quantize(x, 16) for x in h["hist"]])
    models = {"base": h["base"], "len": h["len"], "f": f}
    c = oracle.ad_recoil_encode(sym, mid, models, 16, 64)
    assert c[:4] == b"RCA1"
    info = oracle.container_info(c)
    assert 2 <= info["M"] <= 64 and info["N"] == len(sym)  # low-entropy lanes emit rarely: fewer feasible splits
    assert (oracle.ad_recoil_decode(c, mid) == sym).all()
    for target in (17, 3, 1):
        cc = oracle.combine(c, target)
        assert (oracle.ad_recoil_decode(cc, mid) == sym).all()
    out, lo, hi = oracle.ad_recoil_decode_task(c, mid, 10)
    assert (out[lo:hi + 1] == sym[lo:hi + 1]).all()
    with pytest.raises(oracle.OracleError):
        oracle.recoil_decode(c)  # the static decoder refuses an adaptive container
