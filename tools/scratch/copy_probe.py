#!/usr/bin/env python
"""Pinned host<->device copy bandwidth for the e2e path (8 MB = one C3 vector), on the
legacy default stream vs a non-default stream, one copy vs two halves."""
import torch

n = 1 << 20
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")


def timed(label, fn, stream):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(50):
            fn()
        e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    print("%-28s %.3f ms  %.1f GB/s" % (label, ms, 8 * n / ms / 1e6))


default = torch.cuda.default_stream()
side = torch.cuda.Stream()
for st_name, st in (("default", default), ("non-default", side)):
    timed(f"h2d {st_name}", lambda: d.copy_(h, non_blocking=True), st)
    timed(f"d2h {st_name}", lambda: h.copy_(d, non_blocking=True), st)
    timed(f"h2d {st_name} halves", lambda: (d[: n // 2].copy_(h[: n // 2], non_blocking=True),
                                            d[n // 2:].copy_(h[n // 2:], non_blocking=True)), st)
