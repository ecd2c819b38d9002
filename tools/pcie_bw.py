"""Host<->device copy bandwidth on this box (pinned, copy engines): H2D
alone, D2H alone, both directions at once.  Bounds bench.py's e2e."""
import json
import torch

nb = 128 << 20
h = torch.empty(nb, dtype=torch.uint8).pin_memory()
h2 = torch.empty(nb // 2, dtype=torch.uint8).pin_memory()
d = torch.empty(nb, dtype=torch.uint8, device="cuda")
d2 = torch.empty(nb // 2, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, iters=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    s = torch.cuda.current_stream()
    s.wait_stream(s1)
    s.wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e-3


def h2d():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


def both():
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    h2d()
    d2h()


th, td, tb = t(h2d), t(d2h), t(both)
print(json.dumps({"h2d_GBps": nb / th / 1e9, "d2h_GBps": nb / 2 / td / 1e9,
                  "both_ms": tb * 1e3, "h2d_128MiB_ms": th * 1e3, "d2h_64MiB_ms": td * 1e3}))
