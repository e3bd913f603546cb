"""GPU parity: the sm_100a decode kernel (through the C ABI) vs the oracle.

Every test compares the kernel's output element by element with the oracle's
decode of the same container (and with the input symbols, which is the plain
definition of the decode's result).  Tolerance: bit-exact (integer path).
"""
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


def gpu_decode(c, task_begin=0, task_end=(1 << 64) - 1):
    dec = R.GpuDecoder(c, 0, task_begin, task_end)
    dec.upload()
    dec.decode()
    rc, bad = dec.status()
    out = dec.output().cpu().numpy()
    plan = dec.plan
    dec.close()
    return rc, bad, out, plan


def _check_full(c, sym):
    rc, bad, out, plan = gpu_decode(c)
    assert rc == 0, (R.ERRORS.get(rc), bad)
    assert (plan["out_lo"], plan["out_hi"]) == (0, len(sym))
    if len(sym) <= 4_000_000:
        want = oracle.recoil_decode(bytes(c)) if R.recoil_inspect(c)["partitioned"] == 0 \
            else oracle.partitioned_decode(bytes(c))
        assert (want == sym).all()
    mism = np.nonzero(out != sym)[0]
    assert mism.size == 0, f"{mism.size} mismatches, first at {mism[:5]}"


FUZZ = []
for i, (N, n, M, kind) in enumerate([
        (1, 11, 1, "exp"), (31, 11, 2, "exp"), (32, 11, 2, "text"), (33, 11, 3, "image"), (511, 11, 4, "exp"),
        (512, 11, 4, "exp"), (513, 11, 4, "exp"), (5000, 1, 3, "exp"), (5000, 2, 5, "exp"), (20000, 8, 9, "text"),
        (65536, 11, 16, "exp"), (100000, 12, 33, "image"), (123457, 10, 100, "text"), (300000, 11, 1000, "exp"),
        (777777, 11, 4096, "text"), (1 << 20, 12, 2176, "image"),
        (300000, 13, 64, "exp"), (500000, 14, 300, "text"), (400000, 15, 33, "image"), (1 << 20, 16, 1000, "exp"),
        (4097, 16, 3, "text")]):
    FUZZ.append((N, n, M, kind, 1000 + i))


@pytest.mark.parametrize("N,n,M,kind,seed", FUZZ)
def test_fuzz_vs_oracle(N, n, M, kind, seed):
    sym = synth.workload(kind, N, seed=seed, lam=float(10 + seed % 190))
    if n < 8:  # small alphabets for small n
        sym = (sym % (1 << (n - 1) if n > 1 else 1)).astype(np.uint8) if n <= 2 else sym % 32
    hist = synth.histogram(sym)
    f = oracle.build_model(hist, n)
    c = R.recoil_encode(sym, f, n, M)
    assert c.tobytes() == oracle.recoil_encode(sym, f, n, M)
    _check_full(c, sym)


@pytest.mark.parametrize("n", [11, 12, 16])
def test_single_symbol_fill(n):
    f = np.zeros(256, dtype=np.uint32)
    f[9] = 1 << n
    sym = np.full(100000, 9, dtype=np.uint8)
    c = R.recoil_encode(sym, f, n, 8)
    _check_full(c, sym)


def test_n16_outputs_before_group_zero():
    rng = np.random.default_rng(8)
    hist = np.zeros(256, dtype=np.uint64)
    hist[:200] = rng.integers(1, 5, size=200)
    hist[7] = 10 ** 7
    f = oracle.build_model(hist, 16)
    rare = [s for s in range(256) if f[s] == 1]
    sym = synth.table_bytes(50000, (f / f.sum()).tolist(), 4)
    sym[:32] = rare[0]
    for c in (R.recoil_encode(sym, f, 16, 1), R.recoil_encode(sym, f, 16, 5), R.recoil_partitioned_encode(sym, f, 16, 7)):
        _check_full(c, sym)


def test_n16_exp_stream_full_alphabet():
    """tab:overhead-n-16's setting: 8-bit symbols at n = 16."""
    sym = synth.exp_bytes(3_000_000, 10, 55)
    f = oracle.build_model(synth.histogram(sym), 16)
    for M in (1, 16, 2176):
        c = R.recoil_encode(sym, f, 16, M)
        assert c.tobytes() == oracle.recoil_encode(sym, f, 16, M)
        _check_full(c, sym)
    p = R.recoil_partitioned_encode(sym, f, 16, 500)
    _check_full(p, sym)


@pytest.mark.parametrize("P", [1, 7, 64, 2176])
def test_partitioned_kernel_vs_oracle(P):
    sym = synth.text_bytes(1_000_000, 40 + P)
    f = oracle.build_model(synth.histogram(sym), 11)
    c = R.recoil_partitioned_encode(sym, f, 11, P)
    assert c.tobytes() == oracle.partitioned_encode(sym, f, 11, P)
    _check_full(c, sym)


@pytest.mark.parametrize("shards", [2, 3, 8])
def test_sharded_task_ranges(shards):
    """Multi-GPU data path on one GPU: each shard's plan uploads only its word slice
    and writes only its output span; the spans tile [0, N) and match the input."""
    sym = synth.image_bytes(3_000_000, 77)
    f = oracle.build_model(synth.histogram(sym), 11)
    for c in (R.recoil_encode(sym, f, 11, 800), R.recoil_partitioned_encode(sym, f, 11, 800)):
        bounds = R.recoil_shard_plan(c, shards)
        got = np.zeros(len(sym), dtype=np.uint8)
        covered = 0
        for a, b in zip(bounds, bounds[1:]):
            rc, bad, out, plan = gpu_decode(c, a, b)
            assert rc == 0, (R.ERRORS.get(rc), bad)
            assert plan["word_count"] < R.recoil_inspect(c)["n_words"] + 256
            got[plan["out_lo"]:plan["out_hi"]] = out
            covered += plan["out_hi"] - plan["out_lo"]
        assert covered == len(sym) and (got == sym).all()


@pytest.mark.parametrize("chunks,streams", [(1, 1), (5, 2), (8, 3), (64, 8)])
def test_host_pipeline_end_to_end(chunks, streams):
    """recoil_pipeline_*: host container -> host symbols over chunked task ranges on
    several streams (and a task sub-range, as one rank of a multi-GPU job)."""
    sym = synth.text_bytes(6_000_000, 31)
    f = R.recoil_build_model(synth.histogram(sym), 11)
    c = R.recoil_encode(sym, f, 11, 3000)
    pinned = torch.empty(len(c), dtype=torch.uint8, pin_memory=True)
    pinned.numpy()[:] = c
    out = torch.zeros(len(sym), dtype=torch.uint8, pin_memory=True)
    pipe = R.HostPipeline(pinned.numpy(), 0, n_chunks=chunks, n_streams=streams)
    for _ in range(2):
        out.zero_()
        pipe.run(out)
        rc, bad = pipe.status()
        assert rc == 0, (rc, bad)
        assert (out.numpy() == sym).all()
    pipe.close()
    bounds = R.recoil_shard_plan(c, 3)
    out.zero_()
    pipe = R.HostPipeline(pinned.numpy(), 0, n_chunks=chunks, n_streams=streams, task_begin=bounds[1],
                          task_end=bounds[2])
    pipe.run(out)
    assert pipe.status()[0] == 0
    h = R.recoil_decoder_create(c, bounds[1], bounds[2])
    p = R.recoil_decoder_plan(h)
    R.recoil_decoder_destroy(h)
    assert (out.numpy()[p["out_lo"]:p["out_hi"]] == sym[p["out_lo"]:p["out_hi"]]).all()
    pipe.close()


def test_combined_containers_decode_identically():
    sym = synth.exp_bytes(4_000_000, 50, 88)
    f = oracle.build_model(synth.histogram(sym), 11)
    c = R.recoil_encode(sym, f, 11, 4096)
    for target in (2048, 256, 16, 1):
        cc = R.recoil_combine_splits(c, target)
        assert cc.tobytes() == oracle.combine(c.tobytes(), target)
        _check_full(cc, sym)


def test_corrupted_anchor_is_flagged_or_wrong():
    """a bit-flipped anchor state desynchronises its task -- the device end-state
    check (task 0) or the output comparison catches it."""
    sym = synth.exp_bytes(200000, 50, 5)
    f = oracle.build_model(synth.histogram(sym), 11)
    c = R.recoil_encode(sym, f, 11, 4)
    info = R.recoil_inspect(c)
    # first split record's first anchor state sits right after header + finals + global block
    pos = info["header_bytes"] + 4 * 32
    # global block size: recompute via oracle parse of an M=1 combine is awkward; brute force
    # flip each candidate byte of the first record until the container still parses
    for delta in range(0, 64):
        bad = c.copy()
        bad[pos + delta] ^= 0x04
        try:
            R.recoil_inspect(bad)
        except R.RecoilError:
            continue
        rc, badt, out, _ = gpu_decode(bad)
        if rc != 0 or not (out == sym).all():
            return
    pytest.fail("no corruption detected")


# ------------------------------------------------------------------------------
# BASELINE.json configs at full size, in the launch configuration bench.py uses
# ------------------------------------------------------------------------------

def _sampled_oracle_tasks(c, out, k=24):
    M = R.recoil_inspect(c)["n_splits"]
    tasks = sorted(set([0, 1, M // 2, M - 2, M - 1] + list(np.linspace(0, M - 1, k).astype(int))))
    for t in tasks:
        if 0 <= t < M:
            want, lo, hi = oracle.recoil_decode_task(c.tobytes(), int(t))
            assert (out[lo:hi + 1] == want[lo:hi + 1]).all(), t


def test_config1_1MiB_exp50_16_splits():
    sym = synth.exp_bytes(1 << 20, 50, synth.seed_for(1, 50))
    f = R.recoil_build_model(synth.histogram(sym), 11)
    c = R.recoil_encode(sym, f, 11, 16)
    assert c.tobytes() == oracle.recoil_encode(sym, f, 11, 16)
    _check_full(c, sym)


def test_config2_100MiB_text_occupancy_splits():
    warps, sms = R.recoil_decode_occupancy(0, 11)
    M = warps * sms * 3
    sym = synth.text_bytes(100 << 20, synth.seed_for(2))
    f = R.recoil_build_model(synth.histogram(sym), 11)
    c = R.recoil_encode(sym, f, 11, M)
    assert R.recoil_inspect(c)["n_splits"] == M
    rc, bad, out, _ = gpu_decode(c)
    assert rc == 0 and (out == sym).all()
    _sampled_oracle_tasks(c, out)
    p = R.recoil_partitioned_encode(sym, f, 11, M)
    rc, bad, out, _ = gpu_decode(p)
    assert rc == 0 and (out == sym).all()


@pytest.mark.parametrize("lam", [10, 50, 100, 200])
def test_config3_1GiB_exp(lam):
    warps, sms = R.recoil_decode_occupancy(0, 11)
    sym = synth.exp_bytes(1 << 30, lam, synth.seed_for(3, lam))
    f = R.recoil_build_model(synth.histogram(sym), 11)
    c = R.recoil_encode(sym, f, 11, warps * sms * 8)
    rc, bad, out, _ = gpu_decode(c)
    assert rc == 0 and (out == sym).all()
    _sampled_oracle_tasks(c, out, 8)


def test_config4_combine_65536_to_2048_256_16():
    sym = synth.exp_bytes(1 << 30, 50, synth.seed_for(4, 50))
    f = R.recoil_build_model(synth.histogram(sym), 11)
    c = R.recoil_encode(sym, f, 11, 65536)
    assert R.recoil_inspect(c)["n_splits"] == 65536
    for target in (65536, 2048, 256, 16):
        cc = R.recoil_combine_splits(c, target)
        assert R.recoil_inspect(cc)["n_splits"] == target
        rc, bad, out, _ = gpu_decode(cc)
        assert rc == 0 and (out == sym).all(), target
    small = R.recoil_combine_splits(c, 16)
    assert small.tobytes() == oracle.combine(c.tobytes(), 16)
    assert (R.recoil_decode_cpu(small) == sym).all()


def test_config5_1GiB_image_residual_bench_launch():
    """Config 5 per GPU (1 GiB image-residual bytes) with the bench's split rule
    (1.5 waves of resident warps), in one launch; sampled tasks against the oracle."""
    warps, sms = R.recoil_decode_occupancy(0, 11)
    sym = synth.image_bytes(1 << 30, synth.seed_for(5))
    f = R.recoil_build_model(synth.histogram(sym), 11)
    c = R.recoil_encode(sym, f, 11, warps * sms * 3 // 2)
    rc, bad, out, _ = gpu_decode(c)
    assert rc == 0 and (out == sym).all()
    _sampled_oracle_tasks(c, out, 8)


def test_repeated_decodes_and_concurrent_handles():
    """One plan decoded repeatedly (status cleared each time) and two handles decoding
    different containers concurrently on their own streams."""
    a = synth.text_bytes(2_000_000, 7)
    b = synth.exp_bytes(3_000_000, 20, 8)
    ca = R.recoil_encode(a, R.recoil_build_model(synth.histogram(a), 11), 11, 500)
    cb = R.recoil_encode(b, R.recoil_build_model(synth.histogram(b), 12), 12, 900)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    da, db = R.GpuDecoder(ca, 0, stream=sa), R.GpuDecoder(cb, 0, stream=sb)
    da.upload()
    db.upload()
    for _ in range(3):
        da.decode()
        db.decode()
        assert da.status()[0] == 0 and db.status()[0] == 0
        assert (da.output().cpu().numpy() == a).all() and (db.output().cpu().numpy() == b).all()
    da.close()
    db.close()


def test_more_shards_than_tasks():
    sym = synth.exp_bytes(100_000, 50, 12)
    c = R.recoil_encode(sym, R.recoil_build_model(synth.histogram(sym), 11), 11, 4)
    bounds = R.recoil_shard_plan(c, 16)
    assert bounds[0] == 0 and bounds[-1] == R.recoil_inspect(c)["n_splits"]
    got = np.zeros(len(sym), dtype=np.uint8)
    for a, b in zip(bounds, bounds[1:]):
        rc, bad, out, plan = gpu_decode(c, a, b)
        assert rc == 0
        if b > a:
            got[plan["out_lo"]:plan["out_hi"]] = out
        else:
            assert plan["n_tasks"] == 0 and plan["out_hi"] == plan["out_lo"]
    assert (got == sym).all()


@pytest.mark.parametrize("n", list(range(1, 17)))
def test_every_prob_bits_with_splits(n):
    """Each kernel instantiation n = 1..16 (packed LUT, split tables) on a split stream."""
    sym = synth.exp_bytes(700_000, 30, 200 + n)
    if n < 8:
        sym = (sym % (1 << max(1, n - 1))).astype(np.uint8)
    f = R.recoil_build_model(synth.histogram(sym), n)
    c = R.recoil_encode(sym, f, n, 333)
    assert c.tobytes() == oracle.recoil_encode(sym, f, n, 333)
    _check_full(c, sym)


@pytest.mark.timeout(300)
def test_fuzzed_containers_never_fault_or_hang():
    """Random byte flips anywhere in a container (header, model, metadata, words): the
    library either rejects it (container errors), or the kernel runs to completion and
    reports a status (underflow / sync / inconsistent) or decodes -- never a CUDA fault
    or a hang (all device reads are bounded by the plan's slice and the record windows)."""
    rng = np.random.default_rng(77)
    sym = synth.text_bytes(120_000, 3)
    f = R.recoil_build_model(synth.histogram(sym), 11)
    base = R.recoil_encode(sym, f, 11, 40)
    outcomes = {"rejected": 0, "flagged": 0, "decoded": 0}
    for trial in range(60):
        bad = base.copy()
        for _ in range(int(rng.integers(1, 4))):
            bad[int(rng.integers(0, len(bad)))] ^= int(rng.integers(1, 256))
        try:
            dec = R.GpuDecoder(bad, 0)
        except R.RecoilError:
            outcomes["rejected"] += 1
            continue
        dec.upload()
        dec.decode()
        rc, _ = dec.status()  # raises on a CUDA error
        outcomes["flagged" if rc else "decoded"] += 1
        dec.close()
    torch.cuda.synchronize()
    assert sum(outcomes.values()) == 60, outcomes


@pytest.mark.parametrize("target", [2048, 300, 16, 1])
def test_decoder_side_combine(target):
    """Decoder-adaptive scalability on the client: decode with a subset of
    the split points in place == decode of the combined container == the input."""
    sym = synth.exp_bytes(8_000_000, 50, 21)
    f = R.recoil_build_model(synth.histogram(sym), 11)
    c = R.recoil_encode(sym, f, 11, 8192)
    dec = R.GpuDecoder(c, 0, subset=target)
    dec.upload()
    dec.decode()
    assert dec.status()[0] == 0
    assert dec.plan["n_tasks"] == R.recoil_inspect(R.recoil_combine_splits(c, target))["n_splits"]
    assert (dec.output().cpu().numpy() == sym).all()
    dec.close()


@pytest.mark.timeout(900)
def test_beyond_2pow31_symbols():
    """N > 2^31 symbols (config 5's 8 GiB stream is sharded into such spans): 64-bit symbol
    indices through the fused task expansion (sync starts of groups >= 2^26), the whole stream
    in one launch, the last two shards alone, the CPU decoder, and oracle-decoded sampled tasks."""
    N = (1 << 31) + (1 << 21) + 777
    sym = synth.image_bytes(N, synth.seed_for(5, 31))
    f = R.recoil_build_model(synth.histogram(sym), 11)
    c = R.recoil_encode(sym, f, 11, 4096)
    M = R.recoil_inspect(c)["n_splits"]
    assert M == 4096
    rc, bad, out, _ = gpu_decode(c)
    assert rc == 0, (R.ERRORS.get(rc), bad)
    mism = np.nonzero(out != sym)[0]
    assert mism.size == 0, f"{mism.size} mismatches, first at {mism[:5]}"
    del out
    bounds = R.recoil_shard_plan(c, 8)
    for tb, te in ((bounds[7], bounds[8]), (M - 3, M)):  # the last shard; three tasks wholly above 2^31
        rc, bad, out, plan = gpu_decode(c, tb, te)
        assert rc == 0, (R.ERRORS.get(rc), bad)
        lo, hi = plan["out_lo"], plan["out_hi"]
        assert hi == N and (te - tb > 3 or lo > (1 << 31))
        assert (out == sym[lo:hi]).all()
    full = np.zeros(N, dtype=np.uint8)
    for t in (M // 2, M - 3, M - 2, M - 1):
        want, lo, hi = oracle.recoil_decode_task(c.tobytes(), int(t), full)
        assert (want[lo:hi + 1] == sym[lo:hi + 1]).all(), t
    assert (R.recoil_decode_cpu(c) == sym).all()


@pytest.mark.timeout(1800)
def test_config5_8GiB_full_size_sharded():
    """BASELINE config 5 at its full size: one 8 GiB image-residual stream with the bench's
    8-GPU split count (8 x 1.5 waves of resident warps), decoded in one launch and as the 8
    split-range shards the 8-rank run uses (one after another on this GPU); every byte against
    the input, sampled tasks against the oracle."""
    warps, sms = R.recoil_decode_occupancy(0, 11)
    N = 8 << 30
    sym = synth.image_bytes(N, synth.seed_for(5))
    hist = np.zeros(256, np.uint64)
    for i in range(0, N, 1 << 28):
        hist += np.bincount(sym[i:i + (1 << 28)], minlength=256).astype(np.uint64)
    f = R.recoil_build_model(hist, 11)
    M = 8 * (warps * sms * 3 // 2)
    c = R.recoil_encode(sym, f, 11, M)
    assert R.recoil_inspect(c)["n_splits"] == M
    rc, bad, out, _ = gpu_decode(c)
    assert rc == 0, (R.ERRORS.get(rc), bad)
    assert out.size == N and np.array_equal(out, sym)
    del out
    bounds = R.recoil_shard_plan(c, 8)
    covered = 0
    for a, b in zip(bounds, bounds[1:]):
        rc, bad, out, plan = gpu_decode(c, a, b)
        assert rc == 0, (R.ERRORS.get(rc), bad)
        assert plan["out_lo"] == covered and np.array_equal(out, sym[plan["out_lo"]:plan["out_hi"]])
        covered = plan["out_hi"]
        del out
    assert covered == N
    # end to end through the public host API: pinned container -> pinned symbols
    pinned = torch.empty(len(c), dtype=torch.uint8, pin_memory=True)
    pinned.numpy()[:] = c
    hout = torch.zeros(N, dtype=torch.uint8, pin_memory=True)
    pipe = R.HostPipeline(pinned.numpy(), 0, n_chunks=8, n_streams=3)
    pipe.run(hout)
    assert pipe.status()[0] == 0 and np.array_equal(hout.numpy(), sym)
    pipe.close()
    del hout, pinned
    full = np.zeros(N, dtype=np.uint8)
    for t in (0, M // 3, M - 2, M - 1):
        want, lo, hi = oracle.recoil_decode_task(c.tobytes(), int(t), full)
        assert np.array_equal(want[lo:hi + 1], sym[lo:hi + 1]), t


class _Bits:
    """MSB-first bit reader / writer over the container's global series (test helper)."""

    def __init__(self, data=b"", pos=0):
        self.bits = "".join(f"{b:08b}" for b in data)
        self.pos = pos

    def get(self, n):
        v = int(self.bits[self.pos:self.pos + n], 2)
        self.pos += n
        return v

    def series(self, count):  # signed, 5-bit width field (w - 1), magnitude then sign bit
        w = self.get(5) + 1
        out = []
        for _ in range(count):
            m = self.get(w)
            out.append(-m if self.get(1) else m)
        return out


def _put_series(vals):
    w = max(1, max(abs(v).bit_length() for v in vals))
    bits = f"{w - 1:05b}" + "".join(f"{abs(v):0{w}b}" + ("1" if v < 0 else "0") for v in vals)
    return bits


def _move_max_group(c, k, delta):
    """Re-serialise a Recoil container with split point k's max group moved by delta groups
    (header 28 B, model block, 32 u32 finals, two signed series, byte padded)."""
    raw = bytes(c)
    count = raw[28] | raw[29] << 8
    g0 = 28 + 2 + 5 * count + 4 * 32
    P = R.recoil_inspect(c)["n_splits"] - 1
    br = _Bits(raw[g0:])
    doff, dg = br.series(P), br.series(P)
    end = g0 + (br.pos + 7) // 8
    dg[k] += delta
    bits = _put_series(doff) + _put_series(dg)
    bits += "0" * (-len(bits) % 8)
    glob = bytes(int(bits[i:i + 8], 2) for i in range(0, len(bits), 8))
    return np.frombuffer(raw[:g0] + glob + raw[end:], dtype=np.uint8).copy()


def test_crafted_record_cannot_write_outside_the_plan():
    """a middle split point whose max group is moved 2000 groups up (still
    < G, so the light parse accepts it) must not make its task write past the plan's output
    window.  The host-expanded plans reject it at create (full parse: sync starts no longer
    increasing); the light-parse e2e pipeline decodes it with the in-kernel window check
    (E_INCONSISTENT); the on-device metadata path flags it on the GPU and leaves guard bytes
    on both sides of d_out untouched."""
    sym = synth.exp_bytes(2_000_000, 50, 4)
    f = R.recoil_build_model(synth.histogram(sym), 11)
    c = R.recoil_encode(sym, f, 11, 512)
    assert bytes(_move_max_group(c, 105, 0)) == bytes(c)  # the re-serialiser is exact
    bad = _move_max_group(c, 105, 2000)  # point 105 = the entry of task 105, inside the plan [100, 110)
    # the host-expanded plans parse every record (full parse) and reject the container
    for kw in ({}, {"subset": 512}, {"for_device": True}):
        with pytest.raises(R.RecoilError) as ei:
            R.GpuDecoder(bad, 0, 100, 110, **kw) if "for_device" not in kw else R.GpuDecoder(bad, 0, **kw)
        assert ei.value.rc == R.RECOIL_E_INCONSISTENT
    guard = 1 << 20
    assert 2000 * 32 < guard
    # the e2e pipeline plans from the light parse and expands the records in the kernel: there the
    # kernel's window check must catch it (status E_INCONSISTENT, no fault)
    pinned = torch.empty(len(bad), dtype=torch.uint8, pin_memory=True)
    pinned.numpy()[:] = bad
    pipe = R.HostPipeline(pinned.numpy(), 0, n_chunks=2, n_streams=2, task_begin=100, task_end=110)
    lo, hi = pipe.span()
    host = torch.zeros(hi - lo, dtype=torch.uint8, pin_memory=True)
    pipe.run(host, lo)
    assert R.ERRORS.get(pipe.status()[0]) == "RECOIL_E_INCONSISTENT"
    pipe.close()
    # the on-device metadata path checks the sync starts on the GPU and skips the tasks
    dd = R.DeviceContainerDecoder(bad, 0)
    big = torch.full((dd.plan["out_count"] + 2 * guard,), 0xAB, dtype=torch.uint8, device="cuda")
    dd.out = big[guard:guard + dd.plan["out_count"]]
    dd.upload()
    dd.decode()
    assert R.ERRORS.get(dd.status()[0]) == "RECOIL_E_INCONSISTENT"
    host = big.cpu().numpy()
    assert (host[:guard] == 0xAB).all() and (host[-guard:] == 0xAB).all()
    dd.close()


@pytest.mark.timeout(900)
def test_one_task_longer_than_2pow31_symbols():
    """One task spanning more than 2^31 symbols (decoder-side combine to one split of a
    2^31 + 2^21 + 777-symbol stream): the per-task block offsets are unsigned 32-bit and
    the decode is bit-exact (was silently skipped with signed offsets)."""
    N = (1 << 31) + (1 << 21) + 777
    sym = synth.image_bytes(N, synth.seed_for(5, 32))
    f = R.recoil_build_model(synth.histogram(sym), 11)
    c = R.recoil_encode(sym, f, 11, 64)
    for target in (1, 2):
        dec = R.GpuDecoder(c, 0, subset=target)
        dec.upload()
        dec.decode()
        rc, bad = dec.status()
        assert rc == 0, (R.ERRORS.get(rc), bad)
        assert dec.plan["n_tasks"] == target
        out = dec.output().cpu().numpy()
        dec.close()
        assert np.array_equal(out, sym)
        del out


def test_decoder_create_for_device_combines_to_the_gpu():
    """recoil_decoder_create_for_device (decoder-adaptive scalability): a container
    with 3 waves of split points is decoded with 1.5 waves of tasks (the points
    recoil_combine_splits keeps), bit-exact; a container with fewer points keeps all of them."""
    warps, sms = R.recoil_decode_occupancy(0, 11)
    sym = synth.text_bytes(40 << 20, 5)
    f = R.recoil_build_model(synth.histogram(sym), 11)
    c = R.recoil_encode(sym, f, 11, 3 * warps * sms)
    dec = R.GpuDecoder(c, 0, for_device=True)
    assert dec.plan["n_tasks"] == R.recoil_inspect(R.recoil_combine_splits(c, warps * sms * 3 // 2))["n_splits"]
    dec.upload()
    dec.decode()
    assert dec.status()[0] == 0 and (dec.output().cpu().numpy() == sym).all()
    dec.close()
    small = R.recoil_encode(sym, f, 11, 100)
    dec = R.GpuDecoder(small, 0, for_device=True)
    assert dec.plan["n_tasks"] == 100
    dec.upload()
    dec.decode()
    assert dec.status()[0] == 0 and (dec.output().cpu().numpy() == sym).all()
    dec.close()
