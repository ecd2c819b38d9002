"""Host-side cost of the CudaBackend building blocks (allocation with and
without a stream switch, fill, events, stream waits, views), microseconds
per call; used to pick the host-path optimisations in DESIGN.md §4."""
import time, torch, sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1405_2912_b200 import kernels
from paper_1405_2912_b200.backend import CudaBackend
from paper_1405_2912_b200.devices import MemorySpace
b = CudaBackend()
st = b.stream(0)
sp = MemorySpace("gpu0mem", device=0) if True else None
nb = 16 << 20
def t(name, fn, n=2000):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    dt = (time.perf_counter() - t0) / n * 1e6
    torch.cuda.synchronize()
    print(f"{name:40s} {dt:7.2f} us")
t("torch.empty", lambda: torch.empty(nb, dtype=torch.uint8, device="cuda:0"))
def ctx():
    with torch.cuda.stream(st):
        torch.empty(nb, dtype=torch.uint8, device="cuda:0")
t("with stream + empty", ctx)
t("backend.alloc zero=False", lambda: b.alloc(sp, nb, zero=False))
t("backend.alloc zero=True", lambda: b.alloc(sp, nb, zero=True))
x = torch.empty(nb, dtype=torch.uint8, device="cuda:0")
t("kernels.fill", lambda: kernels.fill(x, 0, stream=st))
t("current_stream", lambda: torch.cuda.current_stream(0))
t("Event()+record", lambda: torch.cuda.Event().record(st))
t("Event(timing)+record", lambda: torch.cuda.Event(enable_timing=True).record(st))
s2 = torch.cuda.Stream()
t("wait_stream", lambda: s2.wait_stream(st))
t("x.view(float32)", lambda: x.view(torch.float32))
t("data_ptr", lambda: x.data_ptr())
t("cuda_stream attr", lambda: st.cuda_stream)
