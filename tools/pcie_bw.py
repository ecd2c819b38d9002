"""Host<->device copy bandwidth on this box (pinned, copy engines): H2D
alone, D2H alone, both directions at once, and the e2e step's shape (2 x 64
MiB H2D + 64 MiB D2H) with the two H2D copies on one stream vs two streams.
Bounds bench.py's e2e."""
import json
import torch

nb = 128 << 20
h = torch.empty(nb, dtype=torch.uint8).pin_memory()
h2 = torch.empty(nb // 2, dtype=torch.uint8).pin_memory()
d = torch.empty(nb, dtype=torch.uint8, device="cuda")
d2 = torch.empty(nb // 2, dtype=torch.uint8, device="cuda")
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
main = torch.cuda.current_stream()


def t(fn, iters=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    for s in (s1, s2, s3):
        main.wait_stream(s)
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
    s1.wait_stream(main)
    s2.wait_stream(main)
    h2d()
    d2h()


half = nb // 2


def step_one_stream():
    for s in (s1, s2):
        s.wait_stream(main)
    with torch.cuda.stream(s1):
        d[:half].copy_(h[:half], non_blocking=True)
        d[half:].copy_(h[half:], non_blocking=True)
    d2h()


def step_two_streams():
    for s in (s1, s2, s3):
        s.wait_stream(main)
    with torch.cuda.stream(s1):
        d[:half].copy_(h[:half], non_blocking=True)
    with torch.cuda.stream(s3):
        d[half:].copy_(h[half:], non_blocking=True)
    d2h()


th, td, tb = t(h2d), t(d2h), t(both)
t1, t2 = t(step_one_stream), t(step_two_streams)
print(json.dumps({"h2d_GBps": nb / th / 1e9, "d2h_GBps": nb / 2 / td / 1e9,
                  "both_ms": tb * 1e3, "h2d_128MiB_ms": th * 1e3, "d2h_64MiB_ms": td * 1e3,
                  "step_h2d_one_stream_ms": t1 * 1e3, "step_h2d_two_streams_ms": t2 * 1e3}))
