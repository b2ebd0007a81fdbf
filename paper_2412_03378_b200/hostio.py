"""Host <-> device transfers of the drop-in facade (numpy float64 in and out,
float32 on the device), measured on the B200 box (tools/facade_probe.py,
6.2M float64 values, one 1080p RGB image):

    upload   host astype(f32) + pageable H2D           7.4 ms
             host copy into pinned f64 + H2D + GPU cast 2.8 ms   <- to_device
    download D2H f32 + numpy astype(f64)                8.8 ms
             D2H f32 into pinned + torch CPU f64 cast           <- to_host
    isfinite host numpy 4.8 ms, on the device 0.1 ms            <- all_finite

Pinned staging buffers are kept per (device, dtype) and grown on demand; a
buffer is reused only after the copy that last read (or wrote) it has
completed (one CUDA event per buffer).  Plumbing only: no compute.
"""

from __future__ import annotations

import threading

import numpy as np

_lock = threading.Lock()
_pool = {}   # (device index, dtype name, direction) -> [pinned tensor, event]


def _staging(torch, dev, dtype, numel, direction):
    key = (dev.index, str(dtype), direction)
    with _lock:
        ent = _pool.get(key)
        if ent is None or ent[0].numel() < numel:
            ent = [torch.empty(max(numel, 1 << 16), dtype=dtype).pin_memory(), None]
            _pool[key] = ent
    if ent[1] is not None:
        ent[1].synchronize()           # the previous copy through this buffer is done
    return ent


def to_device(a, dev, shape):
    """numpy (any float dtype) -> float32 CUDA tensor of `shape` on `dev`,
    through a pinned float64 staging buffer and a cast on the device."""
    import torch
    src = np.ascontiguousarray(a).reshape(-1)
    n = src.size
    if n == 0:
        return torch.empty(shape, dtype=torch.float32, device=dev)
    if src.dtype != np.float64:
        src = src.astype(np.float64)
    ent = _staging(torch, dev, torch.float64, n, "up")
    pin = ent[0][:n]
    pin.copy_(torch.from_numpy(src))  # multi-threaded host copy into pinned memory
    g = pin.to(dev, non_blocking=True)
    ev = torch.cuda.Event()
    ev.record(torch.cuda.current_stream(dev))
    ent[1] = ev
    return g.to(torch.float32).reshape(shape)


def to_host(t, dtype=np.float64):
    """CUDA tensor -> numpy `dtype` array (a new allocation): D2H of the
    device dtype into pinned memory, then a (multi-threaded) torch CPU cast."""
    import torch
    t = t.contiguous()
    n = t.numel()
    if n == 0:
        return np.zeros(tuple(t.shape), dtype=dtype)
    ent = _staging(torch, t.device, t.dtype, n, "down")
    pin = ent[0][:n]
    pin.copy_(t.reshape(-1), non_blocking=True)
    ev = torch.cuda.Event()
    ev.record(torch.cuda.current_stream(t.device))
    ent[1] = ev
    ev.synchronize()
    tt = {np.float64: torch.float64, np.float32: torch.float32, np.int32: torch.int32,
          np.uint8: torch.uint8, np.int64: torch.int64}[np.dtype(dtype).type]
    return pin.to(tt, copy=True).reshape(tuple(t.shape)).numpy()


def all_finite(t):
    """True if every entry of a CUDA tensor is finite (one device reduction)."""
    import torch
    return bool(torch.isfinite(t).all())
