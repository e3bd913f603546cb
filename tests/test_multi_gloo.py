"""N > 1 host path on CPU: world_size-2 gloo processes, each takes its split-range
shard (recoil_shard_plan + the decoder plan's word slice / output span, as
bench.py does per GPU), decodes ONLY from its planned word slice (words
outside it are zeroed), and the spans are all-gathered and checked.  The
per-shard decode runs the oracle's task decoder, so this pins the planner's
slice bounds independently of the CUDA kernel."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, kind, part, M, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import oracle
    import synth
    from paper_2306_12141_b200 import recoil as R
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sym = synth.workload(kind, 400_000, seed=99, lam=40)
        f = R.recoil_build_model(synth.histogram(sym), 11)
        c = R.recoil_partitioned_encode(sym, f, 11, M) if part else R.recoil_encode(sym, f, 11, M)
        bounds = R.recoil_shard_plan(c, world)
        a, b = bounds[rank], bounds[rank + 1]
        h = R.recoil_decoder_create(c, a, b)
        plan = R.recoil_decoder_plan(h)
        R.recoil_decoder_destroy(h)
        info = R.recoil_inspect(c)
        # keep only this shard's word slice
        cc = bytearray(c.tobytes())
        wstart = len(cc) - 2 * info["n_words"]
        lo_w, hi_w = plan["word_lo"], min(info["n_words"], plan["word_lo"] + plan["word_count"])
        cc[wstart:wstart + 2 * lo_w] = bytes(2 * lo_w)
        cc[wstart + 2 * hi_w:] = bytes(len(cc) - wstart - 2 * hi_w)
        out = np.zeros(len(sym), dtype=np.uint8)
        if info["partitioned"]:
            full = oracle.partitioned_decode(c.tobytes())  # partitions: independent codecs, decode whole
            out[plan["out_lo"]:plan["out_hi"]] = full[plan["out_lo"]:plan["out_hi"]]
        else:
            for t in range(a, b):
                _, lo, hi = oracle.recoil_decode_task(bytes(cc), t, out)
        span = torch.tensor([plan["out_lo"], plan["out_hi"]], dtype=torch.int64)
        spans = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(spans, span)
        mine = torch.from_numpy(out[plan["out_lo"]:plan["out_hi"]].copy())
        sizes = [int(s[1] - s[0]) for s in spans]
        parts = [torch.zeros(n, dtype=torch.uint8) for n in sizes]
        # gloo all_gather needs equal sizes: pad to max
        mx = max(sizes)
        padded = torch.zeros(mx, dtype=torch.uint8)
        padded[:len(mine)] = mine
        gathered = [torch.zeros(mx, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(gathered, padded)
        if rank == 0:
            full = np.concatenate([gathered[r][:sizes[r]].numpy() for r in range(world)])
            tiles = all(int(spans[r][1]) == int(spans[r + 1][0]) for r in range(world - 1))
            q.put((tiles and int(spans[0][0]) == 0 and int(spans[-1][1]) == len(sym),
                   bool((full == sym).all()), sizes))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,part,M", [("exp", False, 64), ("text", False, 300), ("image", True, 100)])
def test_two_rank_shards_gloo(kind, part, M):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, part, M, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    tiles, exact, sizes = q.get(timeout=10)
    assert tiles and exact, sizes
    assert min(sizes) > 0.3 * max(sizes)


def _gather_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import synth
    from paper_2306_12141_b200 import recoil as R
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sym = synth.workload("text", 300_000, seed=5)
        f = R.recoil_build_model(synth.histogram(sym), 11)
        c = R.recoil_encode(sym, f, 11, 200)
        spans = R.shard_spans(c, world)
        _, _, lo, hi = spans[rank]
        # this rank's decoded span (CPU decode of the whole stream stands in for the GPU shard)
        mine = torch.from_numpy(R.recoil_decode_cpu(c)[lo:hi].copy())
        full = R.gather_spans(mine, spans, root=0)
        if rank == 0:
            q.put((bool((full.numpy() == sym).all()), [s[3] - s[2] for s in spans]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_optional_gather_of_shard_spans(world):
    """Row a10: the optional final gather reassembles the stream on the root from the
    ranks' committed spans (point-to-point batch; gloo here, NCCL on GPUs)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    ok, sizes = q.get(timeout=5)
    assert ok and len(sizes) == world and min(sizes) > 0
