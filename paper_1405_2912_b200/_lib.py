"""ctypes binding of libhetft.so (the C-ABI declared in include/hetft.h).

The library is built in-tree by ``__graft_entry__.build()`` (``make -C
paper_1405_2912_b200/csrc``).  There is no fallback: if the shared object is
missing or a call is made without a CUDA device, the error is raised loudly.
ctypes releases the GIL for the duration of every foreign call, so replica
bodies on different devices/streams run concurrently from Python threads.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().with_name("libhetft.so")

HF_OK = 0
HF_EINVAL = -1
HF_ECUDA = -2
HF_ENOINIT = -3
HF_EUNSUP = -4
HF_ECHECKSUM = -5

HF_F32, HF_F64, HF_U8, HF_U16, HF_U32, HF_U64 = range(6)
HF_MAX_K = 8

HF_VERDICT_MATCH = 0
HF_VERDICT_CORRECTED = 1
HF_VERDICT_MISMATCH = 2
VERDICT_NAMES = {HF_VERDICT_MATCH: "match", HF_VERDICT_CORRECTED: "corrected",
                 HF_VERDICT_MISMATCH: "mismatch"}

HF_GEMM_TF32 = 0
HF_GEMM_3XTF32 = 1
HF_GEMM_3XBF16 = 2
HF_GEMM_COSCHEDULE = 0x100

# every symbol include/hetft.h declares (checked by tests/test_capi.py)
EXPORTED = (
    "hf_init", "hf_last_error", "hf_version", "hf_device_count", "hf_peer_enabled",
    "hf_vote", "hf_vote_workspace_bytes", "hf_vote_workspace_init", "hf_vote_async", "hf_vote_batch",
    "hf_vote_bytes", "hf_copy", "hf_fill", "hf_checkpoint", "hf_restore", "hf_checksum",
    "hf_inject_bitflip", "hf_inject_scale", "hf_scribble", "hf_gemm_tc", "hf_gemm_simt",
    "hf_debug_spin", "hf_vec_inc", "hf_vec_path",
)


class HfVoteResult(ctypes.Structure):
    _fields_ = [
        ("mismatch", ctypes.c_int64 * HF_MAX_K),
        ("unresolved", ctypes.c_int64),
        ("first_div", ctypes.c_int64),
        ("winner", ctypes.c_int32),
        ("verdict", ctypes.c_int32),
        ("K", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("first_raw0", ctypes.c_uint64),
        ("kernel_ns", ctypes.c_int64),
    ]


HF_VOTE_BATCH_MAX = 32


class HfVoteItem(ctypes.Structure):
    """hf_vote_item (include/hetft.h): one vote of an hf_vote_batch launch."""
    _fields_ = [
        ("replicas", ctypes.c_void_p * HF_MAX_K),
        ("n", ctypes.c_int64),
        ("voted", ctypes.c_void_p),
        ("out", ctypes.c_void_p),
        ("workspace", ctypes.c_void_p),
    ]


class NativeLibraryError(RuntimeError):
    """libhetft.so is missing or failed to load (no CPU fallback exists)."""


class HfError(RuntimeError):
    """A libhetft call returned a negative status."""

    def __init__(self, fn: str, code: int, message: str):
        super().__init__(f"{fn} failed ({code}): {message}")
        self.fn = fn
        self.code = code
        self.message = message


_lock = threading.Lock()
_lib = None
_initialised = False

_c_void_p = ctypes.c_void_p
_i32 = ctypes.c_int
_i64 = ctypes.c_int64


def _declare(lib):
    P = ctypes.POINTER
    sig = {
        "hf_init": (_i32, [_i32, _i32]),
        "hf_last_error": (ctypes.c_char_p, []),
        "hf_version": (_i32, []),
        "hf_device_count": (_i32, []),
        "hf_peer_enabled": (_i32, [_i32, _i32]),
        "hf_vote": (_i32, [P(_c_void_p), _i32, _i64, _i32, P(ctypes.c_double), P(ctypes.c_int32),
                           _c_void_p, P(HfVoteResult), _i32, _c_void_p]),
        "hf_vote_workspace_bytes": (_i64, []),
        "hf_vote_workspace_init": (_i32, [_c_void_p, _i32, _c_void_p]),
        "hf_vote_async": (_i32, [P(_c_void_p), _i32, _i64, _i32, P(ctypes.c_double),
                                 P(ctypes.c_int32), _c_void_p, _c_void_p, _c_void_p, _i32, _c_void_p]),
        "hf_vote_batch": (_i32, [P(HfVoteItem), _i32, _i32, _i32, P(ctypes.c_double), P(ctypes.c_int32), _i32,
                                 _c_void_p]),
        "hf_vote_bytes": (_i32, [P(_c_void_p), _i32, _i64, _i32, _c_void_p, P(HfVoteResult), _i32,
                                 _c_void_p]),
        "hf_copy": (_i32, [_c_void_p, _i32, _c_void_p, _i32, _i64, _c_void_p]),
        "hf_fill": (_i32, [_c_void_p, _i32, _i64, _i32, _c_void_p]),
        "hf_vec_inc": (_i32, [_c_void_p, _c_void_p, _i64, _i32, _c_void_p]),
        "hf_vec_path": (_i32, [_c_void_p, _c_void_p, _i64, _i32, _c_void_p]),
        "hf_checkpoint": (_i32, [_c_void_p, _c_void_p, _i64, P(ctypes.c_uint64), _i32, _c_void_p]),
        "hf_restore": (_i32, [_c_void_p, _c_void_p, _i64, P(ctypes.c_uint64), _i32, _c_void_p]),
        "hf_checksum": (_i32, [_c_void_p, _i64, P(ctypes.c_uint64), _i32, _c_void_p]),
        "hf_inject_bitflip": (_i32, [_c_void_p, _i32, _i64, _i32, _i32, _c_void_p]),
        "hf_inject_scale": (_i32, [_c_void_p, _i32, _i64, ctypes.c_double, _i32, _c_void_p]),
        "hf_scribble": (_i32, [_c_void_p, P(ctypes.c_uint8), _i32, _i32, _c_void_p]),
        "hf_debug_spin": (_i32, [_c_void_p, _i64, _i32, _c_void_p]),
        "hf_gemm_tc": (_i32, [_c_void_p, _c_void_p, _c_void_p, _i32, _i32, _i32, _i32, _i32, _c_void_p]),
        "hf_gemm_simt": (_i32, [_c_void_p, _c_void_p, _c_void_p, _i32, _i32, _i32, _i32, _i32, _c_void_p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def load():
    """Load libhetft.so (once).  Raises NativeLibraryError when absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            path = os.environ.get("HETFT_LIB", str(LIB_PATH))
            if not Path(path).exists():
                raise NativeLibraryError(
                    f"{path} not found: build it with `python -c 'import __graft_entry__ as g; "
                    f"g.build()'` (make -C paper_1405_2912_b200/csrc); there is no CPU fallback")
            try:
                lib = ctypes.CDLL(path)
            except OSError as exc:
                raise NativeLibraryError(f"cannot load {path}: {exc}") from exc
            _declare(lib)
            _lib = lib
    return _lib


def last_error() -> str:
    msg = load().hf_last_error()
    return msg.decode(errors="replace") if msg else ""


def check(fn: str, rc: int) -> int:
    if rc < 0:
        raise HfError(fn, rc, last_error())
    return rc


def init(ndev: int = 0, enable_peer_all: bool = False) -> None:
    """hf_init once per process: device discovery.  Peer access is enabled
    separately (enable_peers) so a one-GPU-per-rank process never creates
    contexts on the other GPUs."""
    global _initialised
    if _initialised and not enable_peer_all:
        return
    lib = load()
    with _lock:
        if not _initialised:
            check("hf_init", lib.hf_init(ndev, 0))
            _initialised = True
    if enable_peer_all:
        enable_peers()


_peers_enabled = False


def enable_peers() -> None:
    """All-to-all peer access between the visible GPUs (NVLink/NVSwitch P2P
    for the sliced voter and peer copies/checkpoints); idempotent."""
    global _peers_enabled
    if _peers_enabled:
        return
    init()
    with _lock:
        if not _peers_enabled:
            check("hf_init", load().hf_init(0, 1))
            _peers_enabled = True


def peer_enabled(dev: int, peer: int) -> bool:
    return bool(load().hf_peer_enabled(dev, peer))
