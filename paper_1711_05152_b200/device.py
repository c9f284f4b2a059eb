"""Device context: the CUDA device, its stream, cached FFT tables and typed
helpers for passing torch device buffers / numpy host metadata to the C ABI.

PyTorch is used only as the device-memory allocator and stream provider; all
arithmetic is in libsfft_b200.so.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native

__all__ = ["Device", "get_device", "hptr", "dptr"]


def _torch():
    import torch
    return torch


def hptr(a: np.ndarray) -> int:
    """Address of a C-contiguous host numpy array (caller keeps it alive)."""
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def dptr(t) -> int:
    return t.data_ptr()


def _torch_dtypes():
    torch = _torch()
    return {"i4": torch.int32, "i8": torch.int64, "f8": torch.float64, "f4": torch.float32, "u1": torch.uint8,
            "i2": torch.int16, "i1": torch.int8, "b1": torch.bool}


class _LazyDtypes(dict):
    def __missing__(self, key):
        self.update(_torch_dtypes())
        return dict.__getitem__(self, key)


_TORCH_DTYPE = _LazyDtypes()


class Device:
    """One CUDA device + stream used by the MR1L engine."""

    def __init__(self, index: int | None = None, stream=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError(
                "paper_1711_05152_b200 requires a CUDA device (B200, sm_100a); "
                "there is no CPU fallback"
            )
        _native.load()
        self.index = torch.cuda.current_device() if index is None else int(index)
        self.torch = torch
        self.device = torch.device("cuda", self.index)
        with torch.cuda.device(self.index):
            self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
            sms = C.c_int(0)
            maj = C.c_int(0)
            mnr = C.c_int(0)
            _native.call("sfft_device_info", C.addressof(sms), C.addressof(maj), C.addressof(mnr))
        self.num_sms = sms.value
        self.cc = (maj.value, mnr.value)
        self._ftab: dict[int, object] = {}
        self._pinned: dict[int, object] = {}
        self._async_free: dict[int, list] = {}  # recycled download_async buffers by size

    # -- raw handles ------------------------------------------------------
    @property
    def sh(self) -> int:
        return self.stream.cuda_stream

    def call(self, name: str, *args, ctx: str = ""):
        with self.torch.cuda.device(self.index):
            return _native.call(name, *args, self.sh, ctx=ctx)

    # -- allocation ---------------------------------------------------------
    def empty(self, shape, dtype):
        return self.torch.empty(shape, dtype=dtype, device=self.device)

    def zeros(self, shape, dtype):
        return self.torch.zeros(shape, dtype=dtype, device=self.device)

    def zeros_fast(self, shape, dtype):
        """A zeroed device tensor through one cudaMemsetAsync of the library on
        the engine stream (torch.zeros costs a framework fill launch)."""
        t = self.torch.empty(shape, dtype=dtype, device=self.device)
        nbytes = t.numel() * t.element_size()
        if nbytes:
            _native.call("sfft_zero_async", t.data_ptr(), nbytes, self.sh, ctx="zero fill")
        return t

    def upload(self, a: np.ndarray, dtype=None, asynchronous: bool = False):
        """Host numpy -> device tensor (ordered on the engine stream).
        ``asynchronous``: stage through a pinned buffer of the upload ring and
        return without waiting for the copy."""
        torch = self.torch
        if asynchronous and dtype is None:
            return self._upload_async(np.ascontiguousarray(a))
        t = torch.from_numpy(np.ascontiguousarray(a))
        if dtype is not None:
            t = t.to(dtype)
        if asynchronous:
            t = t.pin_memory()
        with torch.cuda.stream(self.stream):
            return t.to(self.device, non_blocking=asynchronous)

    _RING = 16

    def _upload_async(self, a: np.ndarray):
        """The array through a ring of pinned staging buffers and one
        cudaMemcpyAsync of the library on the engine stream.  A slot is
        reused only after the copy that last used it has completed (its
        event), so the caller may drop ``a`` at once."""
        torch = self.torch
        nbytes = a.nbytes
        ring = self.__dict__.setdefault("_up_ring", [])
        i = self.__dict__.get("_up_next", 0)
        self._up_next = (i + 1) % self._RING
        if i < len(ring):
            buf, ev = ring[i]
            if ev is not None:
                ev.synchronize()
        else:
            buf, ev = None, None
            ring.append((None, None))
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty((max(nbytes, 256),), dtype=torch.uint8, pin_memory=True)
        buf[:nbytes].numpy()[:] = a.reshape(-1).view(np.uint8)
        out = torch.empty(a.shape, dtype=_TORCH_DTYPE[a.dtype.str[1:]], device=self.device)
        if nbytes:
            _native.call("sfft_copy_async", out.data_ptr(), buf.data_ptr(), nbytes, self.sh, ctx="upload")
        if ev is None:
            ev = torch.cuda.Event()
        ev.record(self.stream)
        ring[i] = (buf, ev)
        return out

    def download(self, t) -> np.ndarray:
        with self.torch.cuda.stream(self.stream):
            return t.detach().to("cpu").numpy()

    def _to_pinned(self, buf, t, nbytes: int):
        """Enqueue the copy of device tensor ``t`` (nbytes) into the pinned
        host tensor ``buf`` on the engine stream; returns the source kept
        alive by the caller until the copy is known complete.  Contiguous
        sources go through one cudaMemcpyAsync of the library (no framework
        stream switch, which costs ~7 us of host time per use)."""
        src = t.detach()
        if src.is_contiguous():
            if nbytes:
                _native.call("sfft_copy_async", buf.data_ptr(), src.data_ptr(), nbytes, self.sh, ctx="read-back")
            return src
        with self.torch.cuda.stream(self.stream):
            src = src.contiguous()
            buf[:nbytes].copy_(src.reshape(-1).view(self.torch.uint8), non_blocking=True)
        return src

    def download_many(self, *tensors) -> list[np.ndarray]:
        """Copy several device tensors to host with asynchronous DMA into fresh
        pinned buffers (torch's caching host allocator: no cudaHostAlloc after
        warm-up) and one stream synchronisation; returns uint8 numpy views that
        own their buffers (reinterpret with .view, no host copy needed)."""
        torch = self.torch
        outs, keep = [], []
        for t in tensors:
            nbytes = t.numel() * t.element_size()
            buf = torch.empty((max(nbytes, 1),), dtype=torch.uint8, pin_memory=True)
            keep.append(self._to_pinned(buf, t, nbytes))
            outs.append(buf[:nbytes].numpy())
        self.stream.synchronize()
        return outs

    def download_small(self, t) -> np.ndarray:
        """Copy of a small device tensor through a reusable pinned buffer."""
        nbytes = t.numel() * t.element_size()
        buf = self._pinned.get(nbytes)
        if buf is None:
            buf = self.torch.empty((max(nbytes, 1),), dtype=self.torch.uint8, pin_memory=True)
            self._pinned[nbytes] = buf
        src = self._to_pinned(buf, t, nbytes)
        self.stream.synchronize()
        del src
        return buf[:nbytes].numpy().view(np.dtype(str(t.dtype).replace("torch.", ""))).reshape(t.shape).copy()

    def download_async(self, t):
        """Start a copy of a small device tensor into a pinned buffer and
        return a callable that waits for it and returns the host array.  Lets
        a caller keep enqueuing work and read the value later.  Each pending
        download owns its buffer until its wait() has run (buffers are then
        recycled), so any number of downloads may be outstanding."""
        torch = self.torch
        nbytes = t.numel() * t.element_size()
        free = self._async_free.setdefault(nbytes, [])
        buf = free.pop() if free else torch.empty((max(nbytes, 1),), dtype=torch.uint8, pin_memory=True)
        src = self._to_pinned(buf, t, nbytes)
        ev = torch.cuda.Event()
        ev.record(self.stream)
        dtype = np.dtype(str(t.dtype).replace("torch.", ""))
        shape = tuple(t.shape)
        state = {"out": None}

        def wait():
            if state["out"] is None:
                ev.synchronize()
                state["out"] = buf[:nbytes].numpy().view(dtype).reshape(shape).copy()
                state["src"] = None  # the copy is done: the source may go
                free.append(buf)
            return state["out"].copy()
        state["src"] = src
        return wait

    def sync(self):
        self.stream.synchronize()

    def copy_stream(self):
        """A second stream of this device for copies that overlap the engine
        stream's kernels (callers order it with events)."""
        st = getattr(self, "_copy_stream", None)
        if st is None:
            st = self._copy_stream = self.torch.cuda.Stream(self.device)
        return st

    # -- cached tables ------------------------------------------------------
    def fft_tables(self, P: int):
        tab = self._ftab.get(P)
        if tab is None:
            n = int(_native.query("sfft_fft_table_len", P))
            if n <= 0:
                raise ValueError(f"FFT size {P} is not a supported Bluestein length")
            tab = self.empty((n, 2), self.torch.float64)
            self.call("sfft_fft_tables", P, dptr(tab), ctx=f"fft tables P={P}")
            self._ftab[P] = tab
        return tab


_DEVICES: dict[int, Device] = {}


def get_device(index: int | None = None) -> Device:
    torch = _torch()
    if _DEVICES:  # CUDA is up (a Device exists): skip the availability probe
        dev = _DEVICES.get(torch.cuda.current_device() if index is None else int(index))
        if dev is not None:
            return dev
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_1711_05152_b200 requires a CUDA device (B200, sm_100a); there is no CPU fallback"
        )
    idx = torch.cuda.current_device() if index is None else int(index)
    dev = _DEVICES.get(idx)
    if dev is None:
        dev = Device(idx)
        _DEVICES[idx] = dev
    return dev
