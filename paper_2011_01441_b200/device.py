"""Device views and host<->device staging (PyTorch is used only for memory).

A ``View`` is a row-major 2-D window into a CUDA tensor: base pointer, leading
dimension in elements, extents and the owning device.  Sub-views are pointer
arithmetic, exactly like the NumPy views the reference's runner slices
(matmul.py:444-454), so no copies happen between plan tasks.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

NP_TO_TORCH = {
    np.dtype(np.int64): torch.int64,
    np.dtype(np.int32): torch.int32,
    np.dtype(np.uint32): torch.int32,
    np.dtype(np.float64): torch.float64,
    np.dtype(np.float32): torch.float32,
}


def torch_dtype(dt) -> torch.dtype:
    if isinstance(dt, torch.dtype):
        return dt
    if dt == "bfloat16":
        return torch.bfloat16
    return NP_TO_TORCH[np.dtype(dt)]


@dataclass
class View:
    tensor: torch.Tensor | None  # keeps the storage alive (None: raw device memory)
    ptr: int
    ld: int
    rows: int
    cols: int
    device: int
    itemsize: int = 0

    @classmethod
    def of(cls, t: torch.Tensor) -> "View":
        if t.dim() != 2:
            raise ValueError(f"expected a 2-D matrix, got shape {tuple(t.shape)}")
        if not t.is_cuda:
            raise ValueError("View needs a CUDA tensor")
        if t.numel() > 0 and t.shape[1] > 1 and t.stride(1) != 1:
            raise ValueError("View needs unit column stride")
        ld = t.stride(0) if t.shape[0] > 1 else max(t.shape[1], 1)
        return cls(t, t.data_ptr(), max(ld, t.shape[1]), t.shape[0], t.shape[1], t.device.index,
                   t.element_size())

    @classmethod
    def raw(cls, ptr: int, rows: int, cols: int, itemsize: int, device: int, ld: int | None = None) -> "View":
        """A view of device memory not owned by PyTorch (e.g. CUDA IPC-mapped peer memory)."""
        return cls(None, ptr, ld if ld is not None else cols, rows, cols, device, itemsize)

    @property
    def elsize(self) -> int:
        return self.itemsize or self.tensor.element_size()

    def sub(self, i0: int, j0: int, n: int, m: int) -> "View":
        if i0 < 0 or j0 < 0 or i0 + n > self.rows or j0 + m > self.cols:
            raise ValueError(f"sub-view [{i0}:{i0 + n}, {j0}:{j0 + m}] outside {self.rows}x{self.cols}")
        return View(self.tensor, self.ptr + (i0 * self.ld + j0) * self.elsize, self.ld, n, m, self.device,
                    self.elsize)


def is_host(x) -> bool:
    return isinstance(x, np.ndarray) or (isinstance(x, torch.Tensor) and not x.is_cuda)


def pick_device(*arrays) -> int:
    for a in arrays:
        if isinstance(a, torch.Tensor) and a.is_cuda:
            return a.device.index
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device visible: the PACO B200 path has no CPU fallback")
    return torch.cuda.current_device()


def stage_in(x, dtype, device: int) -> torch.Tensor:
    """Device tensor of ``dtype`` holding ``x`` (no copy if already there)."""
    want = torch_dtype(dtype)
    if isinstance(x, np.ndarray):
        if x.dtype == np.uint32:
            x = x.view(np.int32)
        t = torch.from_numpy(np.ascontiguousarray(x))
    elif isinstance(x, torch.Tensor):
        t = x
    else:
        raise TypeError(f"unsupported array type {type(x).__name__}")
    if t.is_cuda and t.device.index == device and t.dtype == want and (t.dim() < 2 or t.numel() == 0 or t.shape[1] <= 1 or t.stride(1) == 1):
        return t
    if t.is_cuda and t.device.index != device:
        return t.to(device=device).to(want)
    pinned = (not t.is_cuda) and t.is_pinned()
    return t.to(device=device, dtype=want, non_blocking=pinned).contiguous()


class Output:
    """C staged on the device; ``finish`` writes it back to a host C in place."""

    def __init__(self, C, dtype, device: int, load: bool = True):
        self.orig = C
        want = torch_dtype(dtype)
        if isinstance(C, torch.Tensor) and C.is_cuda and C.device.index == device and C.dtype == want \
                and (C.numel() == 0 or C.shape[1] <= 1 or C.stride(1) == 1):
            self.dev = C
            self.copy_back = False
        else:
            if load:
                self.dev = stage_in(C, dtype, device)
                if self.dev is C:
                    self.dev = C.clone()
            else:
                self.dev = torch.empty(tuple(C.shape), dtype=want, device=device)
            self.copy_back = True

    def finish(self, stream=None) -> None:
        if not self.copy_back:
            return
        C = self.orig
        if isinstance(C, np.ndarray):
            host = self.dev.cpu()
            if C.dtype == np.uint32:
                np.copyto(C, host.numpy().view(np.uint32))
            else:
                np.copyto(C, host.numpy().astype(C.dtype, copy=False))
        else:
            C.copy_(self.dev)
