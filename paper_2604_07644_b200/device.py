"""Device plumbing: torch buffers, solver contexts, the ``B200Device`` executor.

PyTorch is only the buffer interface here: tensors are allocated on the
current CUDA device and their raw pointers are handed to libgsls.so together
with torch's current stream.  ``B200Device`` is what a caller passes as the
reference's ``executor=`` argument (scan.py:82-138 executor seam); any other
executor object (or None) selects the default device.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat

QP_FIELDS = nat.QP_FIELDS
F32 = torch.float32
F64 = torch.float64
# precision split of gsls_qp_t: matrices float32, vectors float64 (include/gsls.h)
VECTOR_FIELDS = ("b", "q", "r", "qN", "f", "fN", "dx0")


def field_dtype(name: str):
    return F64 if name in VECTOR_FIELDS else F32


def cuda_device():
    nat.load()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def to_dev(x, dtype=F32) -> torch.Tensor:
    """numpy / list / tensor -> contiguous CUDA tensor (float32 by default)."""
    if isinstance(x, torch.Tensor):
        return x.to(device=cuda_device(), dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(np.asarray(x, dtype=np.float64)), dtype=dtype,
                           device=cuda_device()).contiguous()


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu", torch.float64).numpy()


class Context:
    """Owns one gsls_ctx (workspace + LQR cache) for fixed dimensions."""

    def __init__(self, nx, nu, nc, nf, N, batch):
        self.lib = nat.load()
        self.dims = nat.Dims(nx, nu, nc, nf, N, batch)
        h = ctypes.c_void_p()
        nat.check(self.lib.gsls_ctx_create(ctypes.byref(self.dims), ctypes.byref(h)), "gsls_ctx_create")
        self.handle = h

    @property
    def key(self):
        d = self.dims
        return (d.nx, d.nu, d.nc, d.nf, d.N, d.batch)

    def nbytes(self) -> int:
        return int(self.lib.gsls_ctx_bytes(self.handle))

    def close(self):
        if getattr(self, "handle", None):
            self.lib.gsls_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class B200Device:
    """Executor handle: pools solver contexts per problem shape on one GPU."""

    threads = 1

    def __init__(self, device: int | None = None):
        nat.load()
        self.index = torch.cuda.current_device() if device is None else int(device)
        self._pool: dict = {}

    def context(self, nx, nu, nc, nf, N, batch) -> Context:
        key = (nx, nu, nc, nf, N, batch)
        ctx = self._pool.get(key)
        if ctx is None:
            with torch.cuda.device(self.index):
                ctx = Context(*key)
            self._pool[key] = ctx
        return ctx

    def clear(self):
        for c in self._pool.values():
            c.close()
        self._pool.clear()


_default: B200Device | None = None


def default_device() -> B200Device:
    global _default
    if _default is None:
        _default = B200Device()
    return _default


def resolve(executor) -> B200Device:
    return executor if isinstance(executor, B200Device) else default_device()


@dataclass
class DeviceQp:
    """A batch of QPs as float32 CUDA tensors with a leading batch dimension."""

    A: torch.Tensor
    B: torch.Tensor
    b: torch.Tensor
    Q: torch.Tensor
    R: torch.Tensor
    S: torch.Tensor
    q: torch.Tensor
    r: torch.Tensor
    QN: torch.Tensor
    qN: torch.Tensor
    C: torch.Tensor
    D: torch.Tensor
    f: torch.Tensor
    CN: torch.Tensor
    fN: torch.Tensor
    dx0: torch.Tensor

    @property
    def batch(self):
        return self.QN.shape[0]

    @property
    def dims(self):
        return (self.QN.shape[-1], self.R.shape[-1], self.C.shape[2], self.CN.shape[1], self.A.shape[1])

    @classmethod
    def from_host(cls, qp, batched: bool = False) -> "DeviceQp":
        vals = {}
        for k in QP_FIELDS:
            t = to_dev(getattr(qp, k), field_dtype(k))
            vals[k] = t if batched else t.unsqueeze(0).contiguous()
        return cls(**vals)

    def cstruct(self) -> nat.Qp:
        s = nat.Qp()
        for k in QP_FIELDS:
            t = getattr(self, k)
            setattr(s, k, t.data_ptr() if t.numel() else None)
        return s

    def replace(self, **kw) -> "DeviceQp":
        d = {k: getattr(self, k) for k in QP_FIELDS}
        d.update(kw)
        return DeviceQp(**d)
