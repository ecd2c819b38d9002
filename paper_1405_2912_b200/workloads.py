"""Built-in tasks and their diverse kernel variants.

``matmul`` is the north-star workload: C = A·B on fp32 n x n operands with
three diverse GPU variants, attached per unit kind like the paper's
OpenMP/CUDA pair (§IV-D; reference registry workloads.py:61-111):
  mm_tc     "gpu-tc"    tcgen05.mma kind::tf32, RN-rounded operands
  mm_simt   "gpu-simt"  register-tiled FP32 FFMA (no tensor cores)
  mm_tc3x   "gpu-tc3"   tcgen05 3xBF16 (bf16 hi/lo split on the kind::f16 path,
                        twice the tf32 rate; 3xTF32 is HF_GEMM_3XTF32) — a third, numerically
                        distinct variant for single-GPU TMR
The reference's 1-D tasks (inc, pathfinder-like, buggy-inc; workloads.py:25-58)
keep their CPU bodies (numpy over pinned host views) and get GPU bodies
(hf_vec_inc / hf_vec_path, csrc/vector.cu) on device views, bit-equal to the
numpy bodies, so the reference experiments stay runnable.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from .api import Param
from .errors import WorkloadError


def _is_numpy(x) -> bool:
    return isinstance(x, np.ndarray)


# ---- matmul ------------------------------------------------------------------

def _mm_views(ctx):
    n = int(ctx.arg("n"))
    a = ctx.request("A", "r").view(n, n)
    b = ctx.request("B", "r").view(n, n)
    c = ctx.request("C", "w").view(n, n)
    return a, b, c


def _tc_flags(ctx) -> int:
    # sharing the GPU with another replica: co-scheduling launch shapes let
    # tcgen05 CTAs run beside SIMT CTAs on the same SMs
    from ._lib import HF_GEMM_COSCHEDULE
    return HF_GEMM_COSCHEDULE if getattr(ctx, "shared_device", False) else 0


def mm_tc_body(ctx):
    from . import kernels
    a, b, c = _mm_views(ctx)
    kernels.gemm_tc(a, b, c, mode=0 | _tc_flags(ctx), stream=ctx.stream)


def mm_tc3x_body(ctx):
    from . import kernels
    from ._lib import HF_GEMM_3XBF16
    a, b, c = _mm_views(ctx)
    kernels.gemm_tc(a, b, c, mode=HF_GEMM_3XBF16 | _tc_flags(ctx), stream=ctx.stream)


def mm_simt_body(ctx):
    from . import kernels
    a, b, c = _mm_views(ctx)
    kernels.gemm_simt(a, b, c, mode=_tc_flags(ctx), stream=ctx.stream)


# every matmul variant writes all of C: its provisional buffers skip the zero fill
MATMUL_PARAMS = (Param.area("A", "r"), Param.area("B", "r"), Param.area("C", "w", overwrites=True),
                 Param.scalar("n"))
MATMUL_VARIANTS = (("mm_tc", "gpu-tc", mm_tc_body), ("mm_simt", "gpu-simt", mm_simt_body),
                   ("mm_tc3x", "gpu-tc3", mm_tc3x_body))
# commit preference (Runtime.attach_kernel fidelity): the SIMT variant is
# plain fp32 FFMA, the reference body's arithmetic (numpy fp32 sgemm);
# 3xBF16 keeps ~fp32 operand precision; single-pass TF32 rounds operands to
# 10 mantissa bits (~5e-5 relative).  A passing vote commits SIMT's buffer.
MATMUL_FIDELITY = {"mm_simt": 0, "mm_tc3x": 1, "mm_tc": 2}
# dispatch order on a shared GPU (Runtime.attach_kernel cost): standalone
# 4096^2 times 2.33 / 0.37 / 0.27 ms; the SIMT grid goes first
# on the lead stream and the tensor-core replicas fill its last wave
MATMUL_COST = {"mm_simt": 8.6, "mm_tc3x": 1.4, "mm_tc": 1.0}


# ---- reference 1-D tasks ---------------------------------------------------------------

def _inc_body(ctx):
    n = ctx.arg("count")
    src = ctx.request("input", "r")
    dst = ctx.request("output", "w")
    if _is_numpy(src):
        np.add(src[:n], np.float32(1.0), out=dst[:n])
    else:
        from . import kernels
        kernels.vec_inc(src, dst, n, stream=ctx.stream)


def _path_body(ctx):
    n = ctx.arg("count")
    src = ctx.request("input", "r")
    dst = ctx.request("output", "w")
    a = src[:n]
    if _is_numpy(a):
        left = np.concatenate((a[:1], a[:-1]))
        right = np.concatenate((a[1:], a[-1:]))
        np.add(a, np.minimum(np.minimum(left, a), right), out=dst[:n])
    else:
        from . import kernels
        kernels.vec_path(src, dst, n, stream=ctx.stream)


def _buggy_inc_body(ctx):
    # off-by-one loop bound: the last element is never written
    n = ctx.arg("count")
    src = ctx.request("input", "r")
    dst = ctx.request("output", "w")
    if _is_numpy(src):
        np.add(src[:n - 1], np.float32(1.0), out=dst[:n - 1])
    else:
        from . import kernels
        kernels.vec_inc(src, dst, n - 1, stream=ctx.stream)


def _inc_oracle(data: np.ndarray) -> np.ndarray:
    return data + np.float32(1.0)


def _path_oracle(data: np.ndarray) -> np.ndarray:
    left = np.concatenate((data[:1], data[:-1]))
    right = np.concatenate((data[1:], data[-1:]))
    return data + np.minimum(np.minimum(left, data), right)


def _uniform_input(size: int, rng) -> np.ndarray:
    """U[1,2) fp32 drawn element by element from `rng` (random.Random), the
    reference's input stream (workloads.py:70-72) — experiments replay it."""
    return np.asarray([rng.uniform(1.0, 2.0) for _ in range(size)], dtype=np.float32)


def _vector_bind(runtime, data, size):
    from .devices import ValueType
    inp = runtime.register_data(data.tobytes(), size, ValueType.FLOAT32, "r")
    out = runtime.register_data(bytes(4 * size), size, ValueType.FLOAT32, "w")
    return {"input": inp, "output": out, "count": size}, out, [inp, out]


@dataclass
class Workload:
    """A task signature plus its diverse variants (reference workloads.py:61-72).
    ``oracle(data)`` is the expected committed output used by the experiment
    harness to count silent corruptions; ``bind`` registers one input and
    returns (bindings, output area, areas to release)."""

    name: str
    description: str
    variants: list                                   # (kernel id, unit kind, body)
    oracle: Optional[Callable] = None
    params: tuple = field(default_factory=lambda: (Param.area("input", "r"), Param.area("output", "w"),
                                                   Param.scalar("count")))
    input_fn: Callable = _uniform_input
    bind: Callable = _vector_bind
    fidelity: dict = field(default_factory=dict)     # kernel -> attach_kernel fidelity rank
    cost: dict = field(default_factory=dict)         # kernel -> attach_kernel cost

    def make_input(self, size: int, rng):
        return self.input_fn(size, rng)

    def attach(self, runtime, float_delta: Optional[float] = None, kinds=None):
        task = runtime.declare_task(self.name, self.params, float_delta=float_delta)
        for kernel, kind, body in self.variants:
            if kinds is None or kind in kinds:
                if self.fidelity or self.cost:
                    runtime.attach_kernel(task, kernel, kind, body, fidelity=self.fidelity.get(kernel, 0),
                                          cost=self.cost.get(kernel, 0.0))
                else:
                    runtime.attach_kernel(task, kernel, kind, body)
        return task


def _matmul_input(n: int, rng):
    """(A, B) n x n fp32 U[1,2).  numpy's PCG64 seeded from `rng`: per-element
    Python draws are too slow at 4096^2."""
    g = np.random.default_rng(rng.getrandbits(63))
    a = g.random((n, n), dtype=np.float32) + np.float32(1.0)
    b = g.random((n, n), dtype=np.float32) + np.float32(1.0)
    return a, b


def _matmul_oracle(data) -> np.ndarray:
    a, b = data
    return (a.astype(np.float64) @ b.astype(np.float64)).astype(np.float32).reshape(-1)


def _matmul_bind(runtime, data, n):
    from .devices import ValueType
    a, b = data
    vt = ValueType.FLOAT32
    ia = runtime.register_data(a.tobytes(), n * n, vt, "r")
    ib = runtime.register_data(b.tobytes(), n * n, vt, "r")
    ic = runtime.register_data(bytes(4 * n * n), n * n, vt, "w")
    return {"A": ia, "B": ib, "C": ic, "n": n}, ic, [ia, ib, ic]


_REGISTRY: dict = {}


def _register(w: Workload) -> Workload:
    _REGISTRY[w.name] = w
    return w


_register(Workload("inc", "increment an array of floats; identical math on every unit kind",
                   [("inc_cpu", "cpu", _inc_body), ("inc_gpu", "gpu", _inc_body)], oracle=_inc_oracle))
_register(Workload("pathfinder-like", "neighborhood-minimum reduction",
                   [("path_cpu", "cpu", _path_body), ("path_gpu", "gpu", _path_body)], oracle=_path_oracle))
_register(Workload("buggy-inc", "increment with a deterministic off-by-one bug in the GPU variant",
                   [("inc_ref_cpu", "cpu", _inc_body), ("inc_buggy_gpu", "gpu", _buggy_inc_body)],
                   oracle=_inc_oracle))
_register(Workload("matmul", "C = A·B, fp32 n x n: tcgen05 TF32 / SIMT FP32 / tcgen05 3xBF16 variants",
                   list(MATMUL_VARIANTS), oracle=_matmul_oracle, params=MATMUL_PARAMS,
                   input_fn=_matmul_input, bind=_matmul_bind, fidelity=MATMUL_FIDELITY,
                   cost=MATMUL_COST))


def builtin_workloads() -> dict:
    return dict(_REGISTRY)


def get_workload(name: str) -> Workload:
    try:
        return _REGISTRY[name]
    except KeyError:
        raise WorkloadError(f"unknown workload {name!r}; available: {', '.join(sorted(_REGISTRY))}") from None
