"""CPU test double of paper_1405_2912_b200.backend.CudaBackend — TEST
INFRASTRUCTURE ONLY.

It lets the reference-mirrored control-plane tests (executor, mapper,
memory protocol) run in the CPU-only container: buffers are numpy byte
arrays, injection and voting use the oracle restatements.  The shipped
package never imports this module; the GPU suites run the same behaviours
through CudaBackend (tests/test_runtime_gpu.py)."""

from __future__ import annotations

import time

import numpy as np

from oracle import inject as oinject
from oracle import vote as ovote


class _VoteResult:
    def __init__(self, o: "ovote.OracleVote"):
        self.verdict = o.verdict
        self.mismatch = list(o.mismatch)
        self.unresolved = o.unresolved
        self.first_div = o.first_div
        self.winner = o.winner
        self.K = len(o.mismatch)
        self.faulty = o.faulty


class HostBackend:
    name = "host-test-double"

    def __init__(self):
        self.launches = 0

    def stream(self, device):
        return None

    def copy_stream(self, device):
        return None

    def record(self, stream):
        return None

    def wait(self, stream, event):
        pass

    def prefetch_copy(self, dst, dst_space, src, src_space):
        dst[:] = src
        return None

    def readback_copy(self, dst_host, src, src_space, after=None):
        dst_host[:] = src
        return None

    def synchronize(self, stream):
        pass

    def timer_start(self, stream, device):
        return ("host", time.perf_counter_ns())

    def timer_stop(self, start, stream, device):
        dt = time.perf_counter_ns() - start[1]
        return lambda: dt

    def is_device_error(self, exc):
        return False

    def alloc(self, space, nbytes, zero=True):
        return _HostBytes(nbytes)

    def from_bytes(self, space, data):
        buf = _HostBytes(len(data))
        buf[:] = np.frombuffer(bytes(data), dtype=np.uint8)
        return buf

    def to_bytes(self, buf):
        return buf.tobytes()

    def nbytes(self, buf):
        return int(buf.size)

    def element_bytes(self, buf, idx, width, after=None):
        return buf[idx * width:(idx + 1) * width].tobytes()

    def copy(self, dst, dst_space, src, src_space):
        dst[:] = src

    def checkpoint(self, dst, dst_space, src, src_space):
        dst[:] = src

    def typed_view(self, buf, value_type, width, writable):
        from paper_1405_2912_b200.devices import INT_DTYPES, view_dtype
        dt = view_dtype(value_type, width) if (value_type.numpy_dtype is not None or width in INT_DTYPES) \
            else np.uint8
        arr = buf.view(dt)
        if not writable:
            arr = arr.view()
            arr.flags.writeable = False
        return arr

    def scribble(self, buf, data, stream=None):
        buf[:len(data)] = np.frombuffer(data, dtype=np.uint8)

    def inject_scale(self, buf, np_dtype, idx, rel, stream=None):
        oinject.corrupt_scale(buf.view(np_dtype), idx, rel)

    def inject_bitflip(self, buf, np_dtype, idx, bit, stream=None):
        oinject.bitflip(buf.view(np_dtype), idx, bit)

    def vote_start(self, bufs, value_type, width, rel_tol, ulp_tol=None, voted=None, device=None):
        from paper_1405_2912_b200.voting import DoneVote
        return DoneVote(*self.vote(bufs, value_type, width, rel_tol, ulp_tol, voted, device))

    def vote(self, bufs, value_type, width, rel_tol, ulp_tol=None, voted=None, device=None):
        from paper_1405_2912_b200.devices import INT_DTYPES, view_dtype
        t0 = time.perf_counter_ns()
        if value_type.numpy_dtype is None and width not in INT_DTYPES:
            o = ovote.vote_bytes(bufs, width)
        else:
            dt = view_dtype(value_type, width)
            o = ovote.vote([b.view(dt) for b in bufs], rel_tol, ulp_tol)
        if voted is not None:
            voted[:] = o.voted.view(np.uint8)
        return _VoteResult(o), time.perf_counter_ns() - t0


class _HostBytes(np.ndarray):
    """uint8 host payload that also accepts bytes-like slice assignment, as
    the reference's bytearray payloads do (h.payload[:] = b"...")."""

    def __new__(cls, nbytes):
        return np.zeros(nbytes, dtype=np.uint8).view(cls)

    def __setitem__(self, key, value):
        if isinstance(value, (bytes, bytearray, memoryview)):
            value = np.frombuffer(bytes(value), dtype=np.uint8)
        super().__setitem__(key, value)
