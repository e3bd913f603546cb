"""Exhaustive-candidate pin of the oracle's split heuristic (or_choose_splits).

PAPER.md §4.2 defines the split choice: a candidate split is a
renormalisation point whose backward scan finds every lane's anchor;
t is the number of symbols it covers since the previous split point, t_s the
length of its Synchronization Section, T the average split length, and the
point minimising H(t, t_s) = |t - T| + |t - t_s - T| is chosen.

This test rebuilds, for every boundary of many tiny streams, the whole
candidate set straight from the raw renormalisation log, with everything
written out here (not calling the oracle's scan or H):
  * backward scan by definition: walk offsets e, e-1, ..., the first event
    per lane is its anchor; infeasible if a lane has none or a negative index;
  * t = idx(e) - prev, t_s = idx(e) - sync_start(e) + 1 (reading Z10');
  * candidates 0 < t <= 2T with sync_start > prev (reading Z9) and group
    differences < 2^16; an empty window doubles (reading Z10'');
  * T_m = ceil((N - prev - 1) / (M - m + 1)) (Z10'), or the printed
    T = ceil(N / M) with the oracle's OR_SPLIT_PRINTED_T flag;
  * argmin H, ties to the smaller word offset.
and asserts that the oracle's chosen offsets are exactly that argmin sequence.

The last test checks the pin's power: mutating the rule here (t_s off by one,
ties to the larger offset, a flipped sign inside H, the other T reading) must
change the chosen splits on some of these streams, so a plausible mistake of
that kind in the oracle could not pass.
"""
import math

import numpy as np
import pytest

import oracle
import synth


def _scan(ev, e, W):
    """P:301 by definition: -> (sync_start, anchor idx per lane) or None."""
    anchor = {}
    o = e
    while o >= 0 and len(anchor) < W:
        lane = int(ev["lane"][o])
        if lane not in anchor:
            anchor[lane] = int(ev["idx"][o])
        o -= 1
    if len(anchor) < W or min(anchor.values()) < 0:
        return None
    return min(anchor.values()), anchor


def _choose(ev, N, W, M, printed_T=False, ts_shift=0, tie_larger=False, h_sign=1):
    """Reference argmin of H over the full candidate set, boundary by boundary."""
    n_ev = len(ev)
    idx = ev["idx"].astype(np.int64)
    scans = [_scan(ev, e, W) for e in range(n_ev)]
    prev, chosen = -1, []
    for m in range(1, M):
        T = math.ceil(N / M) if printed_T else math.ceil((N - prev - 1) / (M - m + 1))
        limit = 2 * T
        while True:
            cands = []
            for e in range(n_ev):
                t = int(idx[e]) - prev
                if t <= 0 or t > limit or scans[e] is None:
                    continue
                ss, anchor = scans[e]
                if ss <= prev:
                    continue
                if int(idx[e]) // W - ss // W > 65535:
                    continue
                ts = int(idx[e]) - ss + 1 + ts_shift
                h = abs(t - T) + abs(t - h_sign * ts - T)
                cands.append((h, -e if tie_larger else e, e))
            if cands:
                break
            if n_ev == 0 or int(idx[-1]) - prev <= limit:
                break
            limit *= 2
        if not cands:
            break
        best = min(cands)[2]
        chosen.append(best)
        prev = int(idx[best])
    return chosen


def _streams():
    """>= 50 tiny streams: W in {4, 32}, N <= 3000, M in 2..9, skewed and flat sources, n in {8, 11}."""
    out = []
    rng = np.random.default_rng(20240611)
    for k in range(56):
        W = (4, 32)[k % 2]
        N = int(rng.integers(300, 3001))
        M = int(rng.integers(2, 10))
        n = (8, 11)[(k // 2) % 2]
        kind = ("exp", "text", "image", "exp10")[(k // 4) % 4]
        seed = 900 + k
        if kind == "exp10":
            sym = synth.exp_bytes(N, 10, seed)
        else:
            sym = synth.workload(kind, N, seed=seed, lam=50)
        out.append((W, N, M, n, sym))
    return out


STREAMS = _streams()


def _events(sym, n, W):
    f = oracle.build_model(synth.histogram(sym), n)
    _, _, ev, _ = oracle.interleaved_encode(sym, f, n, W)
    return ev


@pytest.mark.parametrize("printed_T", [False, True])
def test_choose_splits_is_exhaustive_argmin(printed_T):
    n_boundaries, n_ties = 0, 0
    for W, N, M, n, sym in STREAMS:
        ev = _events(sym, n, W)
        want = _choose(ev, N, W, M, printed_T=printed_T)
        got = [int(x) for x in oracle.choose_splits(ev, N, W, M, printed_T=printed_T)]
        assert got == want, (W, N, M, n, printed_T)
        n_boundaries += len(want)
        n_ties += _choose(ev, N, W, M, printed_T=printed_T, tie_larger=True) != want
    assert n_boundaries >= 150
    assert n_ties > 0  # the streams exercise the tie rule


def test_pin_detects_plausible_mistakes():
    """Each mutation of the rule changes the argmin on at least one stream, so the
    exhaustive test above would fail on an oracle that made that mistake."""
    mutations = {
        "t_s off by one (+1)": dict(ts_shift=1),
        "t_s off by one (-1)": dict(ts_shift=-1),
        "ties to the larger offset": dict(tie_larger=True),
        "sign of t_s inside H flipped": dict(h_sign=-1),
        "printed T instead of T_m": dict(printed_T=True),
    }
    caught = {k: False for k in mutations}
    for W, N, M, n, sym in STREAMS:
        ev = _events(sym, n, W)
        base = [int(x) for x in oracle.choose_splits(ev, N, W, M)]
        for name, kw in mutations.items():
            if not caught[name] and _choose(ev, N, W, M, **kw) != base:
                caught[name] = True
        if all(caught.values()):
            break
    assert all(caught.values()), caught


def test_printed_T_container_decodes():
    """The printed-T reading produces a valid container too (only the split table differs)."""
    sym = synth.exp_bytes(40000, 10, 5)
    f = oracle.build_model(synth.histogram(sym), 11)
    for pt in (False, True):
        c = oracle.recoil_encode(sym, f, 11, 17, printed_T=pt)
        assert (oracle.recoil_decode(c) == sym).all()
