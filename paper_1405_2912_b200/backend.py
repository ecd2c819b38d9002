"""Device backend of the runtime: buffers, streams, timing and the libhetft
kernels behind the memory manager, fault injection and the voter.

``CudaBackend`` is the only backend the package ships.  Buffers are flat
uint8 torch tensors: pinned host memory for the host space (device-visible
through UVA, so the GPU voter can read host replicas zero-copy) and device
memory for a space bound to a CUDA ordinal.  All data movement and compute
go through the C-ABI (``kernels`` -> ``_lib`` -> libhetft.so); torch only
allocates.  There is no CPU fallback: constructing a CudaBackend without a
CUDA device or without the built library raises.

The backend interface is duck-typed so the reference-mirrored control-plane
tests can run on a CPU-only machine with a test double (tests/host_backend.py);
nothing under the package imports or falls back to it.
"""

from __future__ import annotations

import os
import threading
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib, kernels
from .devices import INT_DTYPES, MemorySpace, ValueType, view_dtype

_NP_TO_TORCH = {
    np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64,
    np.dtype(np.uint8): torch.uint8, np.dtype(np.uint16): torch.uint16,
    np.dtype(np.uint32): torch.uint32, np.dtype(np.uint64): torch.uint64,
}


def torch_dtype(np_dtype) -> torch.dtype:
    return _NP_TO_TORCH[np.dtype(np_dtype)]


_VIEW_DTYPES: dict = {}     # (ValueType, width) -> (numpy dtype, torch dtype) of typed_view

# Votes run on their own per-device stream (r2; HETFT_VOTE_STREAM=0 puts them
# back on the compute stream).  Priority: above the lead replica's stream, so
# a finished task's vote is dispatched ahead of the next task's SIMT CTAs.
VOTE_PRIORITY = -2
_VOTE_STREAM = os.environ.get("HETFT_VOTE_STREAM", "1") != "0"
# the device's compute stream (checkpoints, copies-in, fills): A/B knob
COMPUTE_PRIORITY = int(os.environ.get("HETFT_COMPUTE_PRIORITY", "0"))


class CudaBackend:
    """libhetft-backed buffers, copies, injection, voting and timing."""

    name = "cuda"

    def __init__(self):
        if not torch.cuda.is_available():
            raise RuntimeError("CudaBackend needs a CUDA device (no CPU fallback exists)")
        _lib.init()
        self._streams: dict = {}
        self._lock = threading.Lock()
        self.launches = 0             # libhetft kernel launches issued through this backend
        self.slice_across_gpus = True  # replicas on >= 2 GPUs: sliced vote
        self._vote_slots: dict = {}
        self._event_pool: dict = {}        # device -> idle timing events
        self._tl = threading.local()

    # -- streams / timing ---------------------------------------------------------

    def stream(self, device: Optional[int]):
        if device is None:
            return None
        with self._lock:
            s = self._streams.get(device)
            if s is None:
                s = torch.cuda.Stream(device=device, priority=COMPUTE_PRIORITY)
                self._streams[device] = s
        return s

    def follow_all(self, streams, device: Optional[int]) -> None:
        """Every stream in `streams` waits for the device's compute stream
        (one event recorded, one wait per stream)."""
        if device is None:
            return
        ev = torch.cuda.Event()
        ev.record(self.stream(device))
        for s in streams:
            if s is not None:
                s.wait_event(ev)

    def unit_stream(self, unit_id: str, device: Optional[int], priority: int = 0, sync: bool = True):
        """One stream per processing unit, so diverse replicas on one GPU run
        concurrently (e.g. tcgen05 CTAs filling the SIMT kernel's last wave).
        It first waits for the device's compute stream, where the memory
        manager enqueued the attempt's copies, checkpoints and buffer fills.
        priority < 0: the unit's high-priority stream (torch convention, lower
        is higher), whose pending CTAs the GPU dispatches before those of
        default-priority streams."""
        if device is None:
            return None
        key = ("unit", unit_id) if priority == 0 else ("unit", unit_id, priority)
        with self._lock:
            s = self._streams.get(key)
            if s is None:
                s = torch.cuda.Stream(device=device, priority=priority)
                self._streams[key] = s
        if sync:
            s.wait_stream(self.stream(device))
        return s

    def join(self, stream, device: Optional[int]) -> None:
        """The device's compute stream waits for `stream` (a unit stream)."""
        if stream is not None and device is not None:
            self.stream(device).wait_stream(stream)

    def vote_stream(self, device: Optional[int]):
        """The device's vote stream (r2).  A vote waits for its replicas'
        streams (vote_after) and for the compute-stream work queued before it
        (_vstream), but the compute stream never waits for a vote: the next
        task's checkpoints, fills and replicas queue behind nothing of this
        task's tensor-core tail.  Readers of a voted area wait on the vote's
        event instead (Sibling.ready, MemoryManager._await); buffers a vote
        read are dropped only after the host has seen its result."""
        if device is None:
            return None
        if not _VOTE_STREAM:
            return self.stream(device)
        key = ("vote", device)
        with self._lock:
            s = self._streams.get(key)
            if s is None:
                s = torch.cuda.Stream(device=device, priority=VOTE_PRIORITY)
                self._streams[key] = s
        return s

    def vote_after(self, stream, device: Optional[int]) -> None:
        """The device's vote stream waits for `stream` (a replica's unit stream)."""
        if stream is not None and device is not None:
            self.vote_stream(device).wait_stream(stream)

    def _vstream(self, device: int):
        """The vote stream, ordered after everything queued on the device's
        compute stream so far (callers outside the executor produce there)."""
        vs = self.vote_stream(device)
        if vs is not self.stream(device):
            vs.wait_stream(self.stream(device))
        return vs

    def copy_stream(self, device: int, direction: str = "h2d"):
        """Extra streams per device for host<->device traffic, one per
        direction (the copy engines are full duplex), so transfers overlap
        the compute stream's kernels and each other."""
        key = (direction, device)
        with self._lock:
            s = self._streams.get(key)
            if s is None:
                s = torch.cuda.Stream(device=device)
                self._streams[key] = s
        return s

    def synchronize(self, stream) -> None:
        if stream is not None:
            stream.synchronize()

    def record(self, stream):
        ev = torch.cuda.Event()
        ev.record(stream)
        return ev

    def wait(self, stream, event) -> None:
        """GPU-side dependency: `stream` waits for `event` (no host blocking)."""
        if stream is not None and event is not None:
            stream.wait_event(event)

    def prefetch_copy(self, dst, dst_space: MemorySpace, src, src_space: MemorySpace):
        """Asynchronous host->device copy on the destination's copy stream,
        ordered after the compute stream's pending work; returns its event."""
        dev = dst_space.device
        cs = self.copy_stream(dev)
        cs.wait_stream(self.stream(dev))
        kernels.copy(dst, src, stream=cs)
        return self.record(cs)

    def readback_copy(self, dst_host, src, src_space: MemorySpace, after=None):
        """Asynchronous device->host copy on the source's copy stream, ordered
        after `after` (the event that made the payload final, e.g. its vote)
        or, without one, after the compute stream's pending work; returns its
        event.  Waiting on the producing event alone lets the copy of task i
        overlap task i+1's kernels that were queued behind it."""
        dev = src_space.device
        cs = self.copy_stream(dev, "d2h")
        if after is not None:
            for ev in (after if isinstance(after, (list, tuple)) else [after]):
                cs.wait_event(ev)
        else:
            cs.wait_stream(self.stream(dev))
        kernels.copy(dst_host, src, stream=cs)
        return self.record(cs)

    def _timing_event(self, device):
        with self._lock:
            pool = self._event_pool.get(device)
            if pool:
                return pool.pop()
        return torch.cuda.Event(enable_timing=True)

    def timer_start(self, stream, device):
        if stream is None:
            import time
            return ("host", time.perf_counter_ns())
        ev = self._timing_event(device)
        ev.record(stream)
        return ("cuda", ev)

    def timer_stop(self, start, stream, device, recycle: bool = True):
        """Returns elapsed(): waits for the stop event and returns ns.  With
        recycle, elapsed() hands both events back to the device's pool (four
        fresh events per voted task cost ~10 us of host time); timers whose
        stop event is exported as a readiness event (votes) must not recycle.
        An abandoned timer (a hung attempt) keeps its events."""
        kind, t0 = start
        if kind == "host":
            import time
            dt = time.perf_counter_ns() - t0
            return lambda: dt
        ev = self._timing_event(device)
        ev.record(stream)
        pool = self._event_pool.setdefault(device, []) if recycle else None
        lock = self._lock

        def elapsed() -> int:
            ev.synchronize()
            ns = int(t0.elapsed_time(ev) * 1e6)
            if pool is not None:
                with lock:
                    if len(pool) < 256:
                        pool.extend((t0, ev))
            return ns
        elapsed.start_event = t0       # the executor's watchdog polls these
        elapsed.stop_event = ev
        return elapsed

    def query(self, event) -> bool:
        return bool(event.query())

    def is_device_error(self, exc: BaseException) -> bool:
        if isinstance(exc, _lib.HfError):
            return exc.code == _lib.HF_ECUDA
        return isinstance(exc, torch.cuda.OutOfMemoryError) or "CUDA error" in str(exc)

    # -- buffers ------------------------------------------------------------------

    def alloc_scope(self, devices):
        """Context that makes `device`'s compute stream torch's current stream
        while an attempt round acquires its buffers, so each alloc() skips its
        own stream switch (~7 us of Python per allocation)."""
        devs = {d for d in devices if d is not None}
        if len(devs) != 1:
            return _NullScope()
        return _AllocScope(self, devs.pop())

    def alloc(self, space: MemorySpace, nbytes: int, zero: bool = True):
        if space.device is None:
            buf = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
            if zero:
                buf.numpy()[:] = 0
            return buf
        st = self.stream(space.device)
        if getattr(self._tl, "bound", None) == space.device:
            buf = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{space.device}")
        else:
            with torch.cuda.stream(st):
                buf = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{space.device}")
        if zero and nbytes:
            kernels.fill(buf, 0, stream=st)
        return buf

    def reserve(self, space: MemorySpace, nbytes: int, count: int) -> None:
        """Grow the caching allocator to hold `count` free `nbytes` blocks on
        the space's compute stream (host spaces: nothing to do)."""
        if space.device is None or nbytes <= 0 or count <= 0:
            return
        with torch.cuda.stream(self.stream(space.device)):
            bufs = [torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{space.device}") for _ in range(count)]
        del bufs

    def from_bytes(self, space: MemorySpace, data) -> torch.Tensor:
        raw = np.frombuffer(bytes(data), dtype=np.uint8)
        buf = self.alloc(space, raw.size, zero=False)
        if space.device is None:
            buf.numpy()[:] = raw
        else:
            host = torch.from_numpy(raw.copy()).pin_memory()
            kernels.copy(buf, host, stream=self.stream(space.device))
            self.synchronize(self.stream(space.device))
        return buf

    def to_bytes(self, buf) -> bytes:
        if buf.device.type == "cuda":
            self.synchronize(self.stream(buf.device.index))
            return buf.cpu().numpy().tobytes()
        return buf.numpy().tobytes()

    def nbytes(self, buf) -> int:
        return int(buf.numel())

    def element_bytes(self, buf, idx: int, width: int, after=None) -> bytes:
        """Raw bytes of one element.  With `after` (the event that made the
        buffer final, e.g. its vote) only that event is awaited, on a side
        stream: draining the whole compute stream would also wait for the
        next task's kernels queued behind the vote, which delayed every
        re-dispatch of a mismatching vote by one full task."""
        part = buf[idx * width:(idx + 1) * width]
        if part.device.type != "cuda":
            return part.numpy().tobytes()
        dev = part.device.index
        if after is None:
            self.synchronize(self.stream(dev))
            return part.cpu().numpy().tobytes()
        cs = self.copy_stream(dev, "peek")
        cs.wait_event(after)
        host = torch.empty(width, dtype=torch.uint8, pin_memory=True)
        kernels.copy(host, part, stream=cs)
        cs.synchronize()
        return host.numpy().tobytes()

    def copy(self, dst, dst_space: MemorySpace, src, src_space: MemorySpace) -> None:
        """dst <- src on the destination's stream (or the source's when the
        destination is host memory).  Host<->device copies are ordered after
        pending work on both sides."""
        dev = dst_space.device if dst_space.device is not None else src_space.device
        st = self.stream(dev)
        if src_space.device is not None and src_space.device != dev:
            st.wait_stream(self.stream(src_space.device))
        if dev is None:
            dst.numpy()[:] = src.numpy()
            return
        kernels.copy(dst, src, stream=st)
        self.launches += 1
        if dst_space.device is None:
            self.synchronize(st)   # host readers see the bytes on return

    def checkpoint(self, dst, dst_space: MemorySpace, src, src_space: MemorySpace) -> None:
        """Snapshot a sole device copy: same-GPU or peer-GPU snapshots use the
        fused hf_checkpoint stream; host snapshots the copy engine."""
        if src_space.device is not None and dst_space.device is not None:
            st = self.stream(src_space.device)
            kernels.checkpoint(dst, src, stream=st)
            self.launches += 1
            return
        self.copy(dst, dst_space, src, src_space)

    def typed_view(self, buf, value_type: ValueType, width: int, writable: bool):
        """Element view handed to kernel bodies: numpy for host buffers (the
        reference's body protocol), a CUDA tensor for device buffers."""
        key = (value_type, width)
        dts = _VIEW_DTYPES.get(key)
        if dts is None:
            dt = view_dtype(value_type, width) if (value_type.numpy_dtype is not None or width in INT_DTYPES) \
                else np.uint8
            dts = _VIEW_DTYPES[key] = (dt, torch_dtype(dt))
        dt, tdt = dts
        if buf.is_cuda:
            return buf.view(tdt)
        arr = buf.numpy().view(dt)
        if not writable:
            arr = arr.view()
            arr.flags.writeable = False
        return arr

    # -- fault injection ------------------------------------------------------------

    def _inj_stream(self, buf, stream):
        dev = buf.device.index if buf.device.type == "cuda" else 0
        return stream if stream is not None else self.stream(dev)

    # Host-space (CPU unit) outputs live in pinned memory; the injection
    # kernels reach them through UVA, so every fault is applied on the GPU.
    def scribble(self, buf, data: bytes, stream=None) -> None:
        kernels.scribble(buf, data, stream=self._inj_stream(buf, stream))
        self.launches += 1

    def inject_scale(self, buf, np_dtype, idx: int, rel: float, stream=None) -> None:
        kernels.inject_scale(buf.view(torch_dtype(np_dtype)), idx, rel, stream=self._inj_stream(buf, stream))
        self.launches += 1

    def inject_bitflip(self, buf, np_dtype, idx: int, bit: int, stream=None) -> None:
        kernels.inject_bitflip(buf.view(torch_dtype(np_dtype)), idx, bit, stream=self._inj_stream(buf, stream))
        self.launches += 1

    # -- voting -----------------------------------------------------------------------

    def vote_start(self, bufs: Sequence, value_type: ValueType, width: int, rel_tol, ulp_tol=None,
                   voted=None, device: Optional[int] = None):
        """Launch a vote without waiting: hf_vote_async into a pooled device
        workspace, then an async 96-byte D2H of the result on the same stream.
        Replicas on several GPUs use the sliced path (synchronous)."""
        devs = []
        for b in bufs:
            if b.device.type == "cuda" and b.device.index not in devs:
                devs.append(b.device.index)
        typed = value_type.numpy_dtype is not None or width in INT_DTYPES
        if typed and self.slice_across_gpus and len(devs) >= 2:
            return self._vote_sliced_start(bufs, value_type, width, rel_tol, ulp_tol, voted, devs)
        if not typed or not devs:
            from .voting import DoneVote
            return DoneVote(*self.vote(bufs, value_type, width, rel_tol, ulp_tol, voted, device))
        if device is None:
            device = devs[0]
        st = self._vstream(device)
        for d in devs:
            if d != device:
                st.wait_stream(self._vstream(d))
        slot = self._vote_slot(device)
        start = self.timer_start(st, device)
        dt = torch_dtype(view_dtype(value_type, width))
        # the kernel's last CTA writes the result straight into the slot's
        # pinned host buffer (UVA): no separate 96-byte read-back copy
        kernels.vote_async([b.view(dt) for b in bufs], slot.ws, rel_tol, ulp_tol,
                           voted=voted.view(dt) if voted is not None else None, stream=st,
                           result_into=slot.host)
        stop = self.timer_stop(start, st, device, recycle=False)
        self.launches += 1
        return _PendingVote(self, slot, device, stop)

    def _vote_sliced_start(self, bufs, value_type, width, rel_tol, ulp_tol, voted, devs):
        """Replicas on distinct GPUs (BASELINE configs[2]): the
        element range is cut into one slice per replica GPU; GPU d votes its
        slice with hf_vote_async on its compute stream, loading the other
        replicas' slices from their GPUs over NVLink (peer access from
        hf_init) and storing its part of the voted buffer in place (a peer
        store when the target replica lives elsewhere).  Each GPU's ingress
        is (K-1)/K of the replica bytes instead of (K-1) on a single voter.
        Nothing waits on the host here; the slice results land in pinned
        slots and combine exactly in _PendingSliced.wait (counts add, first
        divergence = min)."""
        from .sharding import slice_bounds
        streams = {d: self._vstream(d) for d in devs}
        # every slice reads every replica: each voting GPU waits for all producers
        evs = {d: self.record(streams[d]) for d in devs}
        for d in devs:
            for e in devs:
                if e != d:
                    streams[d].wait_event(evs[e])
        lead = devs[0]
        start = self.timer_start(streams[lead], lead)
        dt = torch_dtype(view_dtype(value_type, width))
        views = [b.view(dt) for b in bufs]
        vv = voted.view(dt) if voted is not None else None
        n = views[0].numel()
        K = len(views)
        bounds = slice_bounds(n, len(devs), max(1, 16 // views[0].element_size()))
        parts = []
        for (lo, hi), d in zip(bounds, devs):
            if hi <= lo:
                continue
            slot = self._vote_slot(d)
            kernels.vote_async([v[lo:hi] for v in views], slot.ws, rel_tol, ulp_tol,
                               voted=vv[lo:hi] if vv is not None else None, stream=streams[d],
                               result_into=slot.host)
            self.launches += 1
            parts.append((lo, d, slot))
        for d in devs[1:]:
            streams[lead].wait_stream(streams[d])
        stop = self.timer_stop(start, streams[lead], lead, recycle=False)
        return _PendingSliced(self, parts, K, stop)

    def vote_start_batch(self, specs: Sequence, rel_tol, device: Optional[int] = None) -> list:
        """Several votes (e.g. every output area of one task) in one
        hf_vote_batch launch.  specs: (replicas, value type, width, ulp_tol,
        voted) per vote.  Falls back to one vote_start each unless every vote
        is typed, has the same element type, K and ULP rule, and all replicas
        sit on one GPU.  Returns one pending handle per spec."""
        def single():
            return [self.vote_start(b, vt, w, rel_tol, u, voted=v, device=device) for b, vt, w, u, v in specs]
        devs, dts = set(), set()
        for bufs, vt, width, ulps, _v in specs:
            if not (vt.numpy_dtype is not None or width in INT_DTYPES):
                return single()
            dts.add((view_dtype(vt, width), len(bufs), None if ulps is None else tuple(ulps)))
            for b in bufs:
                if b.device.type != "cuda":
                    return single()
                devs.add(b.device.index)
        if len(devs) != 1 or len(dts) != 1:
            return single()
        dev = devs.pop()
        st = self._vstream(dev)
        dt = torch_dtype(dts.pop()[0])
        slots = [self._vote_slot(dev) for _ in specs]
        items = [([b.view(dt) for b in bufs], v.view(dt) if v is not None else None, slot.ws, slot.host)
                 for (bufs, _vt, _w, _u, v), slot in zip(specs, slots)]
        start = self.timer_start(st, dev)
        kernels.VoteBatch(items, rel_tol, specs[0][3], device=dev).launch(st)
        stop = self.timer_stop(start, st, dev, recycle=False)
        self.launches += 1
        return [_PendingVote(self, slot, dev, stop) for slot in slots]

    def prewarm(self, devices, vote_slots: int = 4) -> None:
        """Create each device's compute stream and a few vote result slots up
        front.  A slot holds pinned host memory, and the first cudaHostAlloc of
        a size waits for the device to go idle: made lazily inside a task's
        vote it would wait out a hung replica before the executor's watchdog
        gets to look at it."""
        for d in sorted({d for d in devices if d is not None}):
            self.stream(d)
            self.vote_stream(d)
            slots = [self._vote_slot(d) for _ in range(vote_slots)]
            for sl in slots:
                self._release_vote_slot(d, sl)
        torch.empty(8, dtype=torch.uint8, pin_memory=True)    # element_bytes' peek buffer size class

    def _vote_slot(self, device: int):
        with self._lock:
            pool = self._vote_slots.setdefault(device, [])
            if pool:
                return pool.pop()
        return kernels._SliceSlot(device)

    def _release_vote_slot(self, device: int, slot) -> None:
        with self._lock:
            self._vote_slots.setdefault(device, []).append(slot)

    def vote(self, bufs: Sequence, value_type: ValueType, width: int, rel_tol, ulp_tol=None,
             voted=None, device: Optional[int] = None):
        """K-way vote on the GPU (hf_vote).  Replicas may sit on several GPUs
        (peer loads over NVLink) or in pinned host memory (UVA loads)."""
        devs = []
        for b in bufs:
            if b.device.type == "cuda" and b.device.index not in devs:
                devs.append(b.device.index)
        if device is None:
            device = devs[0] if devs else 0
        typed = value_type.numpy_dtype is not None or width in INT_DTYPES
        if self.slice_across_gpus and len(devs) >= 2 and typed:
            # replicas on distinct GPUs: every replica GPU votes its slice,
            # each waiting for all replica producers (cross-device events)
            streams = {d: self._vstream(d) for d in devs}
            for d in devs:
                for e in devs:
                    if e != d:
                        streams[d].wait_stream(streams[e])
            start = self.timer_start(streams[devs[0]], devs[0])
            dt = torch_dtype(view_dtype(value_type, width))
            res = kernels.vote_sliced([b.view(dt) for b in bufs], rel_tol, ulp_tol,
                                      voted=voted.view(dt) if voted is not None else None,
                                      devices=devs, streams=streams)
            for d in devs[1:]:
                streams[devs[0]].wait_stream(streams[d])
            stop = self.timer_stop(start, streams[devs[0]], devs[0], recycle=False)
            self.launches += len(devs)
            ns = stop()
            return res, (res.kernel_ns or ns)
        st = self._vstream(device)
        for d in devs:
            if d != device:
                st.wait_stream(self._vstream(d))
        start = self.timer_start(st, device)
        if value_type.numpy_dtype is None and width not in INT_DTYPES:
            res = kernels.vote_bytes(list(bufs), width, voted=voted, device=device, stream=st)
        else:
            dt = torch_dtype(view_dtype(value_type, width))
            views = [b.view(dt) for b in bufs]
            res = kernels.vote(views, rel_tol, ulp_tol, voted=voted.view(dt) if voted is not None else None,
                               device=device, stream=st)
        stop = self.timer_stop(start, st, device, recycle=False)
        self.launches += 1
        ns = stop()
        return res, (getattr(res, "kernel_ns", 0) or ns)


class _NullScope:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


class _AllocScope:
    """Binds the device's compute stream as torch's current stream (the
    caching allocator associates blocks with the current stream)."""

    def __init__(self, be: CudaBackend, device: int):
        self._be, self._dev = be, device
        self._ctx = torch.cuda.stream(be.stream(device))
        self._prev = None

    def __enter__(self):
        self._ctx.__enter__()
        self._prev = getattr(self._be._tl, "bound", None)
        self._be._tl.bound = self._dev
        return self

    def __exit__(self, *exc):
        self._be._tl.bound = self._prev
        return self._ctx.__exit__(*exc)


class _PendingVote:
    def __init__(self, backend: CudaBackend, slot, device: int, stop):
        self._be, self._slot, self._dev, self._stop = backend, slot, device, stop
        self.ready = getattr(stop, "stop_event", None)   # after the vote kernel (voted bytes final)

    def wait(self):
        ns = self._stop()            # synchronises the stop event (after the vote kernel)
        raw = self._slot.host.numpy().tobytes()
        self._be._release_vote_slot(self._dev, self._slot)
        res = kernels.VoteResult.from_c(_lib.HfVoteResult.from_buffer_copy(raw))
        # the kernel's own clock: the event pair around the launch also counts
        # any GPU idle time while the host was still issuing the vote
        return res, (res.kernel_ns or ns)


class _PendingSliced:
    """A vote sliced over several GPUs (CudaBackend._vote_sliced_start)."""

    def __init__(self, backend: CudaBackend, parts, K: int, stop):
        self._be, self._parts, self._K, self._stop = backend, parts, K, stop
        self.ready = getattr(stop, "stop_event", None)   # after every slice (voted bytes final)

    def wait(self):
        from .sharding import SliceResult, combine_slices
        ns = self._stop()             # the lead stream waited for every slice's stream
        res = []
        kns = 0
        for lo, d, slot in self._parts:
            r = _lib.HfVoteResult.from_buffer_copy(slot.host.numpy().tobytes())
            kns = max(kns, int(r.kernel_ns))
            res.append(SliceResult(lo, [int(r.mismatch[i]) for i in range(self._K)], int(r.unresolved),
                                   int(r.first_div), int(r.first_raw0)))
            self._be._release_vote_slot(d, slot)
        c = combine_slices(res, self._K)
        return kernels.VoteResult(c.verdict, c.mismatch, c.unresolved, c.first_div, c.winner, self._K,
                                  c.faulty, c.first_raw0, kns), (kns or ns)
