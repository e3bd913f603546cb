"""recoil_multi_decode (C ABI): shards of one stream on
several devices in one process, optional gather.  On a one-GPU box the shards
share cuda:0 (devices = {0, 0, ...}) and the gather runs as device copies; the
NCCL gather leg needs two distinct GPUs and skips otherwise.  Every byte is
compared with the input (the decode's definition) and, on sampled tasks, the
oracle's task decoder."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2306_12141_b200 import recoil as R

pytestmark = pytest.mark.gpu


def _stream(n=3_000_000, M=700, kind="image"):
    sym = synth.workload(kind, n, seed=synth.seed_for(5), lam=50)
    f = R.recoil_build_model(synth.histogram(sym), 11)
    return sym, R.recoil_encode(sym, f, 11, M)


def _run(c, devices, gather_root):
    plans = R.recoil_multi_plan(c, len(devices))
    outs = [torch.full((max(p["out_count"], 16),), 0xAB, dtype=torch.uint8, device=f"cuda:{d}")
            for p, d in zip(plans, devices)]
    n = R.recoil_inspect(c)["n_symbols"]
    gat = torch.zeros(max(n, 1), dtype=torch.uint8, device=f"cuda:{devices[gather_root]}") if gather_root >= 0 else None
    rc, ms = R.recoil_multi_decode(c, devices, outs, gather_root, gat)
    return plans, outs, gat, rc, ms


@pytest.mark.parametrize("n_dev", [1, 2, 3, 8])
def test_multi_decode_shared_gpu_with_gather(n_dev):
    sym, c = _stream()
    plans, outs, gat, rc, ms = _run(c, [0] * n_dev, 0)
    assert rc == 0
    assert len(ms) == n_dev and all(m > 0 for m in ms)
    lo = 0
    for p, o in zip(plans, outs):
        assert p["out_lo"] == lo  # contiguous spans covering [0, N)
        got = o[p["out_lo"] - p["out_base"]:p["out_hi"] - p["out_base"]].cpu().numpy()
        assert (got == sym[p["out_lo"]:p["out_hi"]]).all()
        lo = p["out_hi"]
    assert lo == len(sym)
    assert (gat.cpu().numpy() == sym).all()
    # sampled tasks of the last shard against the oracle's literal task decoder
    want = np.zeros(len(sym), np.uint8)
    for t in (plans[-1]["task_begin"], plans[-1]["task_end"] - 1):
        _, tlo, thi = oracle.recoil_decode_task(c.tobytes(), int(t), want)
        assert (want[tlo:thi + 1] == sym[tlo:thi + 1]).all()


def test_multi_decode_without_gather_and_root_choice():
    sym, c = _stream(1_000_000, 300, "exp")
    plans, outs, gat, rc, _ = _run(c, [0, 0, 0], -1)
    assert rc == 0 and gat is None
    plans, outs, gat, rc, _ = _run(c, [0, 0, 0], 2)
    assert rc == 0 and (gat.cpu().numpy() == sym).all()


def test_multi_decode_flags_corruption_and_skips_gather():
    sym, c = _stream(1_000_000, 300, "exp")
    info = R.recoil_inspect(c)
    cc = c.copy()
    cc[len(cc) - 2 * info["n_words"] + 1000] ^= 0x5A  # one word of the stream
    plans, outs, gat, rc, _ = _run(cc, [0, 0], 0)
    assert rc in (0, R.RECOIL_E_SYNC, R.RECOIL_E_UNDERFLOW)
    if rc == 0:  # a flipped word that still ends in the end state decodes to different bytes
        assert not (gat.cpu().numpy() == sym).all()
    else:
        assert (gat.cpu().numpy() == 0).all()  # no gather after a failed decode


def test_multi_decode_rejects_bad_arguments():
    sym, c = _stream(200_000, 40, "exp")
    with pytest.raises(R.RecoilError):
        R.recoil_multi_decode(c, [0, 0], [None, None], -1, None)
    plans = R.recoil_multi_plan(c, 2)
    outs = [torch.empty(p["out_count"], dtype=torch.uint8, device="cuda") for p in plans]
    with pytest.raises(R.RecoilError):
        R.recoil_multi_decode(c, [0, 0], outs, 2, None)  # root out of range


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="the NCCL gather needs two distinct GPUs")
def test_multi_decode_nccl_gather_distinct_gpus():
    assert R.recoil_multi_nccl_available()
    sym, c = _stream()
    devs = list(range(min(8, torch.cuda.device_count())))
    plans, outs, gat, rc, _ = _run(c, devs, 0)
    assert rc == 0 and (gat.cpu().numpy() == sym).all()


def test_pipeline_into_a_span_sized_host_buffer():
    sym, c = _stream(2_000_000, 400, "text")
    bounds = R.recoil_shard_plan(c, 3)
    pinned = torch.empty(len(c), dtype=torch.uint8, pin_memory=True)
    pinned.numpy()[:] = c
    for r in range(3):
        pipe = R.HostPipeline(pinned.numpy(), 0, n_chunks=4, n_streams=3, task_begin=bounds[r],
                              task_end=bounds[r + 1])
        lo, hi = pipe.span()
        host = torch.zeros(hi - lo, dtype=torch.uint8, pin_memory=True)
        pipe.run(host, lo)
        assert pipe.status()[0] == 0
        assert (host.numpy() == sym[lo:hi]).all()
        with pytest.raises(R.RecoilError):
            pipe.run(host, lo + 1)  # the span starts before host_first
        pipe.close()


def test_multi_decode_more_devices_than_tasks():
    sym, c = _stream(20_000, 3, "exp")
    assert R.recoil_inspect(c)["n_splits"] <= 3
    plans, outs, gat, rc, ms = _run(c, [0] * 8, 0)
    assert rc == 0
    assert sum(p["n_tasks"] for p in plans) == R.recoil_inspect(c)["n_splits"]
    assert (gat.cpu().numpy() == sym).all()
