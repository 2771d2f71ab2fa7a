"""Host/device marshalling for the drop-in API.

Array-likes (lists, numpy arrays) are coerced exactly as the reference does
(``np.ascontiguousarray(x, dtype=np.float64)``, samplers.py:168,199) and
uploaded to the current CUDA device; CUDA tensors are used in place when they
are contiguous float64 and 32-byte aligned (copied otherwise).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib


def is_device_tensor(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def to_device_f64(x) -> tuple[torch.Tensor, bool]:
    """(1-D-or-not contiguous float64 CUDA tensor, input_was_host)."""
    if is_device_tensor(x):
        t = x
        if t.dtype != torch.float64 or not t.is_contiguous() or t.data_ptr() % 32:
            t = t.to(torch.float64).contiguous().clone()
        return t, False
    if isinstance(x, torch.Tensor):
        if x.dtype == torch.float64 and x.is_contiguous() and x.is_pinned():
            # pinned host input: asynchronous copy on the current stream
            t = torch.empty(x.shape, dtype=torch.float64, device=_lib.device())
            t.copy_(x, non_blocking=True)
            return t, True
        x = x.detach().numpy()
    a = np.ascontiguousarray(x, dtype=np.float64)
    t = torch.empty(a.shape, dtype=torch.float64, device=_lib.device())
    if a.size:
        t.copy_(torch.from_numpy(a), non_blocking=False)
    return t, True


def empty_f64(n: int) -> torch.Tensor:
    return torch.empty(int(n), dtype=torch.float64, device=_lib.device())


def empty_i64(n: int) -> torch.Tensor:
    return torch.empty(int(n), dtype=torch.int64, device=_lib.device())


def status_word() -> torch.Tensor:
    return torch.zeros(1, dtype=torch.int32, device=_lib.device())


def read_status(st: torch.Tensor) -> int:
    """Synchronising 4-byte read of a device status word."""
    return int(st.item())


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy()


def host_result_i64(n: int) -> torch.Tensor:
    """A pinned (page-locked) host int64 buffer the kernels write directly.

    Under unified addressing a pinned host allocation is device-accessible
    at the same address, so the search kernels store the indices straight
    into it over the host link (no separate device->host copy); the caller
    synchronises the stream before reading.  ``_lib.device_accessible``
    checks the address once per buffer.
    """
    t = torch.empty(int(n), dtype=torch.int64, pin_memory=True)
    if t.numel() and not _lib.device_accessible(t.data_ptr()):
        raise RuntimeError("pinned host buffer is not device-accessible (no unified addressing)")
    return t


def finish_host(t: torch.Tensor, stream: int | None = None) -> np.ndarray:
    """Wait for the stream that wrote ``t`` (pinned host memory) and hand it out as numpy."""
    if stream is None:
        stream = _lib.stream_handle()
    _lib.check(_lib.lib().dr_stream_synchronize(stream), "dr_stream_synchronize")
    return t.numpy()
