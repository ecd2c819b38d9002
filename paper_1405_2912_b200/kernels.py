"""Torch-tensor front end of the libhetft kernels.

PyTorch is plumbing here: it allocates device memory and supplies streams.
Every function passes ``data_ptr()`` values through the C-ABI
(include/hetft.h) and the computation runs in the sm_100a kernels of
``csrc/``.  Nothing here computes on the CPU.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional, Sequence

import torch

from . import _lib
from ._lib import HfVoteResult, check

# libhetft kernel launches issued through this module (bench.py reports the
# count inside its timed region as gpu_launches)
LAUNCHES = 0


def _count(n: int = 1) -> None:
    global LAUNCHES
    LAUNCHES += n

_TORCH_DTYPE = {
    torch.float32: _lib.HF_F32,
    torch.float64: _lib.HF_F64,
    torch.uint8: _lib.HF_U8,
    torch.int8: _lib.HF_U8,
    torch.int16: _lib.HF_U16,
    torch.uint16: _lib.HF_U16,
    torch.int32: _lib.HF_U32,
    torch.uint32: _lib.HF_U32,
    torch.int64: _lib.HF_U64,
    torch.uint64: _lib.HF_U64,
}


def hf_dtype(t: torch.Tensor) -> int:
    try:
        return _TORCH_DTYPE[t.dtype]
    except KeyError:
        raise ValueError(f"unsupported element type {t.dtype}") from None


def _stream_ptr(device: int, stream: Optional[torch.cuda.Stream]) -> int:
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return int(s.cuda_stream)


def _dev(t: torch.Tensor) -> int:
    if t.device.type != "cuda":
        raise ValueError(f"tensor on {t.device}; libhetft kernels need CUDA tensors")
    return t.device.index if t.device.index is not None else torch.cuda.current_device()


@dataclass
class VoteResult:
    """Outcome of one K-replica vote."""

    verdict: str                      # "match" | "corrected" | "mismatch"
    mismatch: list[int]
    unresolved: int
    first_div: int                    # -1 when every replica agrees everywhere
    winner: int
    K: int
    faulty: list[int] = field(default_factory=list)
    first_raw0: Optional[int] = None  # replica 0's raw bits at first_div, as read before an in-place store
    kernel_ns: int = 0                # the vote kernel's own device time (max over slices when sliced)

    @classmethod
    def from_c(cls, r: HfVoteResult) -> "VoteResult":
        K = int(r.K)
        mism = [int(r.mismatch[i]) for i in range(K)]
        fd = int(r.first_div)
        return cls(_lib.VERDICT_NAMES[int(r.verdict)], mism, int(r.unresolved), fd,
                   int(r.winner), K, [i for i, m in enumerate(mism) if m > 0],
                   int(r.first_raw0) if fd >= 0 else None, int(r.kernel_ns))


def _ptr_array(ts: Sequence[torch.Tensor]):
    arr = (ctypes.c_void_p * len(ts))()
    for i, t in enumerate(ts):
        arr[i] = t.data_ptr()
    return arr


def _tolerances(K: int, rel_tol, ulp_tol):
    if isinstance(rel_tol, (int, float)):
        rel = [float(rel_tol)] * K
    else:
        rel = [float(x) for x in rel_tol]
    if len(rel) != K:
        raise ValueError(f"rel_tol has {len(rel)} entries for {K} replicas")
    rel_c = (ctypes.c_double * K)(*rel)
    if ulp_tol is None:
        return rel_c, None
    ulp = [int(ulp_tol)] * K if isinstance(ulp_tol, int) else [int(x) for x in ulp_tol]
    if len(ulp) != K:
        raise ValueError(f"ulp_tol has {len(ulp)} entries for {K} replicas")
    return rel_c, (ctypes.c_int32 * K)(*ulp)


def vote(replicas: Sequence[torch.Tensor], rel_tol=0.001, ulp_tol=None,
         voted: Optional[torch.Tensor] = None, device: Optional[int] = None,
         stream: Optional[torch.cuda.Stream] = None) -> VoteResult:
    """K-replica vote.  Replicas may live on different GPUs: the kernel runs
    on `device` (default: voted's or replica 0's) and loads peer buffers
    directly over NVLink when peer access is enabled."""
    K = len(replicas)
    if not 2 <= K <= _lib.HF_MAX_K:
        raise ValueError(f"need 2..{_lib.HF_MAX_K} replicas, got {K}")
    n = replicas[0].numel()
    dt = replicas[0].dtype
    for r in replicas:
        if r.numel() != n or r.dtype != dt:
            raise ValueError("replicas differ in size or element type")
        if not r.is_contiguous():
            raise ValueError("replicas must be contiguous")
    if voted is not None and (voted.numel() != n or voted.dtype != dt or not voted.is_contiguous()):
        raise ValueError("voted buffer must match the replicas")
    if device is None:
        device = _dev(voted) if voted is not None else _dev(replicas[0])
    _lib.init()
    if any(r.device.type == "cuda" and r.device.index != device for r in replicas):
        _lib.enable_peers()          # peer replicas are loaded directly over NVLink
    rel_c, ulp_c = _tolerances(K, rel_tol, ulp_tol)
    out = HfVoteResult()
    lib = _lib.load()
    rc = lib.hf_vote(_ptr_array(replicas), K, n, hf_dtype(replicas[0]), rel_c, ulp_c,
                     voted.data_ptr() if voted is not None else None, ctypes.byref(out),
                     device, _stream_ptr(device, stream))
    check("hf_vote", rc)
    _count()
    return VoteResult.from_c(out)


def vote_bytes(replicas: Sequence[torch.Tensor], elem_width: int,
               voted: Optional[torch.Tensor] = None, device: Optional[int] = None,
               stream: Optional[torch.cuda.Stream] = None) -> VoteResult:
    """Vote byte buffers holding integer elements of any width (bitwise)."""
    K = len(replicas)
    nbytes = replicas[0].numel() * replicas[0].element_size()
    if nbytes % elem_width:
        raise ValueError(f"{nbytes} bytes is not a multiple of element width {elem_width}")
    if device is None:
        device = _dev(voted) if voted is not None else _dev(replicas[0])
    _lib.init()
    out = HfVoteResult()
    rc = _lib.load().hf_vote_bytes(_ptr_array(replicas), K, nbytes // elem_width, elem_width,
                                   voted.data_ptr() if voted is not None else None,
                                   ctypes.byref(out), device, _stream_ptr(device, stream))
    check("hf_vote_bytes", rc)
    _count()
    return VoteResult.from_c(out)


class VoteWorkspace:
    """Device workspace + device result for hf_vote_async (no host sync)."""

    def __init__(self, device: int, stream: Optional[torch.cuda.Stream] = None):
        _lib.init()
        lib = _lib.load()
        self.device = device
        nb = int(lib.hf_vote_workspace_bytes())
        self.ws = torch.empty(nb, dtype=torch.uint8, device=f"cuda:{device}")
        self.result = torch.zeros(ctypes.sizeof(HfVoteResult), dtype=torch.uint8,
                                  device=f"cuda:{device}")
        check("hf_vote_workspace_init",
              lib.hf_vote_workspace_init(self.ws.data_ptr(), device, _stream_ptr(device, stream)))

    def read(self) -> VoteResult:
        host = self.result.cpu().numpy().tobytes()
        return VoteResult.from_c(HfVoteResult.from_buffer_copy(host))


def vote_async(replicas: Sequence[torch.Tensor], ws: VoteWorkspace, rel_tol=0.001, ulp_tol=None,
               voted: Optional[torch.Tensor] = None,
               stream: Optional[torch.cuda.Stream] = None,
               result_into: Optional[torch.Tensor] = None) -> None:
    """result_into: a pinned host buffer of sizeof(HfVoteResult) (104) bytes that
    receives the result directly (default: ws.result in device memory)."""
    K = len(replicas)
    n = replicas[0].numel()
    rel_c, ulp_c = _tolerances(K, rel_tol, ulp_tol)
    out = ws.result if result_into is None else result_into
    rc = _lib.load().hf_vote_async(_ptr_array(replicas), K, n, hf_dtype(replicas[0]), rel_c, ulp_c,
                                   voted.data_ptr() if voted is not None else None,
                                   out.data_ptr(), ws.ws.data_ptr(), ws.device,
                                   _stream_ptr(ws.device, stream))
    check("hf_vote_async", rc)
    _count()


class VoteBatch:
    """A prepared hf_vote_batch launch: the descriptor array (replica, voted,
    result and workspace pointers per vote) is built once, so repeated
    launches over the same buffers cost one C call.  items: (replicas, voted
    or None, VoteWorkspace, result tensor or None) per vote; every item has
    the same K and dtype and shares the tolerances.  Results go to the given
    tensor (device or pinned host, sizeof HfVoteResult bytes) or to the
    workspace's device result; read them with VoteResult.from_c after the
    stream passes the launch."""

    def __init__(self, items: Sequence[tuple], rel_tol=0.001, ulp_tol=None, device: Optional[int] = None):
        if not items:
            raise ValueError("vote_batch: no items")
        K = len(items[0][0])
        dt = items[0][0][0].dtype
        arr = (_lib.HfVoteItem * len(items))()
        for it, (reps, voted, ws, out) in zip(arr, items):
            if len(reps) != K or any(r.dtype != dt or r.numel() != reps[0].numel() or not r.is_contiguous()
                                     for r in reps):
                raise ValueError("vote_batch: every item needs K contiguous replicas of one size and dtype")
            for r, t in enumerate(reps):
                it.replicas[r] = t.data_ptr()
            it.n = reps[0].numel()
            it.voted = voted.data_ptr() if voted is not None else None
            it.out = (out if out is not None else ws.result).data_ptr()
            it.workspace = ws.ws.data_ptr()
        self._items = list(items)          # keeps every buffer alive as long as the descriptors
        self._arr = arr
        self.K, self.count = K, len(items)
        self._dtype = hf_dtype(items[0][0][0])
        self.device = _dev(items[0][0][0]) if device is None else device
        self._rel, self._ulp = _tolerances(K, rel_tol, ulp_tol)
        self._lib = _lib.load()

    def launch(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        check("hf_vote_batch", self._lib.hf_vote_batch(self._arr, self.count, self.K, self._dtype, self._rel,
                                                       self._ulp, self.device, _stream_ptr(self.device, stream)))
        _count(-(-self.count // _lib.HF_VOTE_BATCH_MAX))


def vote_batch(items: Sequence[tuple], rel_tol=0.001, ulp_tol=None, device: Optional[int] = None,
               stream: Optional[torch.cuda.Stream] = None) -> None:
    """Several K-replica votes in one launch (hf_vote_batch); see VoteBatch."""
    if items:
        VoteBatch(items, rel_tol, ulp_tol, device).launch(stream)


class _SliceSlot:
    """Per-device workspace + pinned host mirror for one in-flight slice."""

    def __init__(self, device: int):
        self.ws = VoteWorkspace(device)
        self.host = torch.empty(ctypes.sizeof(HfVoteResult), dtype=torch.uint8).pin_memory()


_SLICE_SLOTS: dict = {}


def vote_sliced(replicas: Sequence[torch.Tensor], rel_tol=0.001, ulp_tol=None,
                voted: Optional[torch.Tensor] = None, devices: Optional[Sequence[int]] = None,
                streams: Optional[dict] = None):
    """K-way vote with the element range sliced over `devices` (default: the
    replicas' distinct GPUs): slice i runs on devices[i] and loads the other
    replicas' slices from their GPUs over NVLink (peer access from hf_init),
    so ingress per GPU is (K-1)/K of the unsliced voter's.  Slices launch
    asynchronously (hf_vote_async + D2H of the 96-byte result) and combine
    exactly on the host (sharding.combine_slices).  Returns a VoteResult."""
    from .sharding import SliceResult, combine_slices, slice_bounds
    K = len(replicas)
    n = replicas[0].numel()
    if devices is None:
        devices = []
        for r in replicas:
            d = _dev(r)
            if d not in devices:
                devices.append(d)
    _lib.init()
    if len(set(devices)) > 1:
        _lib.enable_peers()
    align = max(1, 16 // replicas[0].element_size())
    bounds = slice_bounds(n, len(devices), align)
    pending = []
    for i, ((lo, hi), d) in enumerate(zip(bounds, devices)):
        if hi <= lo:
            continue
        st = (streams or {}).get(d) or torch.cuda.current_stream(d)
        slot = _SLICE_SLOTS.get((d, i))      # one result slot per in-flight slice
        if slot is None:
            slot = _SLICE_SLOTS[(d, i)] = _SliceSlot(d)
        views = [r[lo:hi] for r in replicas]
        vote_async(views, slot.ws, rel_tol, ulp_tol, voted=voted[lo:hi] if voted is not None else None,
                   stream=st, result_into=slot.host)
        ev = torch.cuda.Event()
        ev.record(st)
        pending.append((lo, slot, ev))
    parts = []
    kns = 0
    for lo, slot, ev in pending:
        ev.synchronize()
        r = HfVoteResult.from_buffer_copy(slot.host.numpy().tobytes())
        parts.append(SliceResult(lo, [int(r.mismatch[i]) for i in range(K)], int(r.unresolved), int(r.first_div),
                                 int(r.first_raw0)))
        kns = max(kns, int(r.kernel_ns))
    c = combine_slices(parts, K)
    verdict_code = {"match": _lib.HF_VERDICT_MATCH, "corrected": _lib.HF_VERDICT_CORRECTED,
                    "mismatch": _lib.HF_VERDICT_MISMATCH}[c.verdict]
    return VoteResult(_lib.VERDICT_NAMES[verdict_code], c.mismatch, c.unresolved, c.first_div, c.winner, K,
                      c.faulty, c.first_raw0, kns)


# ---- copy / checkpoint ------------------------------------------------------

def _nbytes(t: torch.Tensor) -> int:
    return t.numel() * t.element_size()


def _loc(t: torch.Tensor) -> int:
    return _dev(t) if t.device.type == "cuda" else -1


def copy(dst: torch.Tensor, src: torch.Tensor, stream: Optional[torch.cuda.Stream] = None) -> None:
    """dst <- src (bytes).  Device/peer/host placement is resolved natively."""
    nb = _nbytes(src)
    if _nbytes(dst) != nb:
        raise ValueError("copy: size mismatch")
    _lib.init()
    dd, sd = _loc(dst), _loc(src)
    sdev = dd if dd >= 0 else sd
    check("hf_copy", _lib.load().hf_copy(dst.data_ptr(), dd, src.data_ptr(), sd, nb,
                                         _stream_ptr(sdev, stream) if sdev >= 0 else None))
    if dd >= 0 and sd >= 0 and (dd == sd or _lib.peer_enabled(dd, sd)):
        _count()        # copy kernel (host <-> device goes to the copy engine)


def fill(dst: torch.Tensor, value: int = 0, stream: Optional[torch.cuda.Stream] = None) -> None:
    _lib.init()
    d = _loc(dst)
    check("hf_fill", _lib.load().hf_fill(dst.data_ptr(), int(value), _nbytes(dst), d,
                                         _stream_ptr(d, stream) if d >= 0 else None))


def checkpoint(ckpt: torch.Tensor, buf: torch.Tensor, with_checksum: bool = False,
               stream: Optional[torch.cuda.Stream] = None) -> Optional[int]:
    nb = _nbytes(buf)
    if _nbytes(ckpt) != nb:
        raise ValueError("checkpoint: size mismatch")
    _lib.init()
    dev = _dev(buf)
    cs = ctypes.c_uint64(0)
    check("hf_checkpoint", _lib.load().hf_checkpoint(
        ckpt.data_ptr(), buf.data_ptr(), nb, ctypes.byref(cs) if with_checksum else None, dev,
        _stream_ptr(dev, stream)))
    _count()
    return int(cs.value) if with_checksum else None


def restore(buf: torch.Tensor, ckpt: torch.Tensor, expect: Optional[int] = None,
            stream: Optional[torch.cuda.Stream] = None) -> None:
    nb = _nbytes(buf)
    if _nbytes(ckpt) != nb:
        raise ValueError("restore: size mismatch")
    _lib.init()
    dev = _dev(buf)
    ex = ctypes.c_uint64(expect) if expect is not None else None
    check("hf_restore", _lib.load().hf_restore(buf.data_ptr(), ckpt.data_ptr(), nb,
                                               ctypes.byref(ex) if ex is not None else None, dev,
                                               _stream_ptr(dev, stream)))
    _count()


def checksum(buf: torch.Tensor, stream: Optional[torch.cuda.Stream] = None) -> int:
    _lib.init()
    dev = _dev(buf)
    out = ctypes.c_uint64(0)
    check("hf_checksum", _lib.load().hf_checksum(buf.data_ptr(), _nbytes(buf), ctypes.byref(out),
                                                 dev, _stream_ptr(dev, stream)))
    _count()
    return int(out.value)


# ---- fault injection ----------------------------------------------------------

def _inj_dev(buf: torch.Tensor, device: Optional[int]) -> int:
    # pinned host buffers are device-visible through UVA; the kernel then runs
    # on `device` (default GPU 0) and writes the host bytes in place
    if buf.device.type == "cuda":
        return _dev(buf)
    return 0 if device is None else device


def inject_bitflip(buf: torch.Tensor, elem: int, bit: int, stream: Optional[torch.cuda.Stream] = None,
                   device: Optional[int] = None) -> None:
    _lib.init()
    dev = _inj_dev(buf, device)
    check("hf_inject_bitflip", _lib.load().hf_inject_bitflip(
        buf.data_ptr(), hf_dtype(buf), int(elem), int(bit), dev, _stream_ptr(dev, stream)))
    _count()
    if buf.device.type != "cuda":
        torch.cuda.synchronize(dev)


def inject_scale(buf: torch.Tensor, elem: int, rel: float, stream: Optional[torch.cuda.Stream] = None,
                 device: Optional[int] = None) -> None:
    _lib.init()
    dev = _inj_dev(buf, device)
    check("hf_inject_scale", _lib.load().hf_inject_scale(
        buf.data_ptr(), hf_dtype(buf), int(elem), float(rel), dev, _stream_ptr(dev, stream)))
    _count()
    if buf.device.type != "cuda":
        torch.cuda.synchronize(dev)


def scribble(buf: torch.Tensor, data: bytes, stream: Optional[torch.cuda.Stream] = None,
             device: Optional[int] = None) -> None:
    _lib.init()
    dev = _inj_dev(buf, device)
    raw = (ctypes.c_uint8 * max(1, len(data)))(*data)
    check("hf_scribble", _lib.load().hf_scribble(buf.data_ptr(), raw, len(data), dev,
                                                 _stream_ptr(dev, stream)))
    _count()
    if buf.device.type != "cuda":
        torch.cuda.synchronize(dev)


# ---- matmul variants -------------------------------------------------------------

def _mm_args(A: torch.Tensor, B: torch.Tensor, C: torch.Tensor):
    if A.dtype != torch.float32 or B.dtype != torch.float32 or C.dtype != torch.float32:
        raise ValueError("matmul variants take fp32 operands")
    if A.dim() != 2 or B.dim() != 2 or C.dim() != 2:
        raise ValueError("matmul variants take 2-D operands")
    M, K = A.shape
    K2, N = B.shape
    if K2 != K or tuple(C.shape) != (M, N):
        raise ValueError(f"shape mismatch {tuple(A.shape)} x {tuple(B.shape)} -> {tuple(C.shape)}")
    for t in (A, B, C):
        if not t.is_contiguous():
            raise ValueError("matmul operands must be contiguous row-major")
    return M, N, K


def gemm_simt(A: torch.Tensor, B: torch.Tensor, C: torch.Tensor, mode: int = 0,
              stream: Optional[torch.cuda.Stream] = None) -> None:
    """mode: 0 or HF_GEMM_COSCHEDULE (sharing the GPU with a TC replica)."""
    M, N, K = _mm_args(A, B, C)
    _lib.init()
    dev = _dev(C)
    check("hf_gemm_simt", _lib.load().hf_gemm_simt(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, int(mode),
                                                   dev, _stream_ptr(dev, stream)))
    fast = M % 128 == 0 and N % 128 == 0 and K % 32 == 0
    _count(2 if fast else 1)    # transpose pre-pass + sgemm


def gemm_tc(A: torch.Tensor, B: torch.Tensor, C: torch.Tensor, mode: int = _lib.HF_GEMM_TF32,
            stream: Optional[torch.cuda.Stream] = None) -> None:
    M, N, K = _mm_args(A, B, C)
    _lib.init()
    dev = _dev(C)
    check("hf_gemm_tc", _lib.load().hf_gemm_tc(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K,
                                               mode, dev, _stream_ptr(dev, stream)))
    _count(3)           # B^T (+split) pre-pass, A round/split, tcgen05 GEMM


def vec_inc(src: torch.Tensor, dst: torch.Tensor, n: Optional[int] = None,
            stream: Optional[torch.cuda.Stream] = None) -> None:
    """dst[:n] = src[:n] + 1 (fp32; reference workloads.py:24-28)."""
    _vec("hf_vec_inc", src, dst, n, stream)


def vec_path(src: torch.Tensor, dst: torch.Tensor, n: Optional[int] = None,
             stream: Optional[torch.cuda.Stream] = None) -> None:
    """dst[i] = a[i] + min(a[i-1], a[i], a[i+1]), ends clamped (fp32;
    reference workloads.py:35-42)."""
    _vec("hf_vec_path", src, dst, n, stream)


def _vec(name, src, dst, n, stream):
    if src.dtype != torch.float32 or dst.dtype != torch.float32:
        raise ValueError(f"{name}: fp32 buffers expected")
    if not (src.is_contiguous() and dst.is_contiguous()):
        raise ValueError(f"{name}: contiguous buffers expected")
    n = src.numel() if n is None else int(n)
    if n > src.numel() or n > dst.numel():
        raise ValueError(f"{name}: n={n} exceeds the buffers")
    _lib.init()
    dev = _dev(dst)
    check(name, getattr(_lib.load(), name)(src.data_ptr(), dst.data_ptr(), n, dev, _stream_ptr(dev, stream)))
    _count()


def debug_spin(max_ns: int, flag: Optional[torch.Tensor] = None, device: int = 0,
               stream: Optional[torch.cuda.Stream] = None) -> None:
    """Launch the bounded spin kernel (a stand-in hung replica for watchdog
    tests; capped at 5 s by the library)."""
    _lib.init()
    check("hf_debug_spin", _lib.load().hf_debug_spin(flag.data_ptr() if flag is not None else None,
                                                     int(max_ns), device, _stream_ptr(device, stream)))
    _count()
