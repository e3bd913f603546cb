"""Ceiling of the e2e pipeline's copies alone: config 2's per-step bytes (67 MB in, 105 MB out) moved in
K chunks on a copy-in and a copy-out stream (3 buffer sets, chunk k's D2H after its H2D), no kernels,
no host work; wall clock per step."""
import time, torch
IN, OUT = 67_482_434, 104_857_600
h_in = torch.empty(IN, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(OUT, dtype=torch.uint8, pin_memory=True)
for K, S in ((1, 1), (4, 3), (8, 3), (16, 3)):
    ci, co = IN // K, OUT // K
    d_in = [torch.empty(ci + 256, dtype=torch.uint8, device="cuda") for _ in range(S)]
    d_out = [torch.empty(co + 256, dtype=torch.uint8, device="cuda") for _ in range(S)]
    sin, sout = torch.cuda.Stream(), torch.cuda.Stream()
    best = 1e9
    for rep in range(6):
        ev_in = [torch.cuda.Event() for _ in range(K)]
        ev_out = [torch.cuda.Event() for _ in range(K)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(K):
            s = k % S
            with torch.cuda.stream(sin):
                if k >= S:
                    sin.wait_event(ev_out[k - S])
                d_in[s][:ci].copy_(h_in[k * ci:(k + 1) * ci], non_blocking=True)
                ev_in[k].record(sin)
            with torch.cuda.stream(sout):
                sout.wait_event(ev_in[k])
                h_out[k * co:(k + 1) * co].copy_(d_out[s][:co], non_blocking=True)
                ev_out[k].record(sout)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"chunks {K:2d} sets {S}: {best*1e3:.3f} ms  -> {OUT/best/1e9:.1f} GB/s (decoded-bytes basis)")
