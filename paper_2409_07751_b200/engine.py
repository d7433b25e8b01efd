"""Device engine: the sm_100a library behind the HeBackend mirror.

`GpuEngine` owns one `hk_ctx` of libhekan_gpu.so (include/hekan.h) and the
HBM buffers of every ciphertext/plaintext, allocated through PyTorch's caching
allocator (torch is plumbing here: device memory and the current CUDA stream).
Kernels are enqueued on torch's current stream; nothing synchronises except
downloads.

There is deliberately no CPU fallback: if the shared library is missing or no
CUDA device is visible, constructing the engine raises.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _abi

_LIB_NAME = "libhekan_gpu.so"
_LIB = None


def library_path() -> str:
    return os.path.join(os.path.dirname(os.path.abspath(__file__)), _LIB_NAME)


def load_library() -> C.CDLL:
    """Load the in-tree sm_100a library (built by __graft_entry__.build())."""
    global _LIB
    if _LIB is None:
        path = library_path()
        if not os.path.exists(path):
            raise ImportError(
                f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the engine has no CPU fallback)")
        _LIB = _abi.bind(C.CDLL(path))
    return _LIB


class _EngineBase:
    """ABI-level helpers shared by the device engine and the test oracle."""

    lib: C.CDLL
    ctx: C.c_void_p

    def __init__(self, params, lib, device: int = 0):
        self.params = params
        self.lib = lib
        st, self._keep = _abi.make_params_struct(params)
        ctx = C.c_void_p()
        rc = lib.hk_ctx_create(C.byref(st), int(device), C.byref(ctx))
        if rc != 0:
            raise ValueError(f"hk_ctx_create failed with status {rc} for {params.describe()}")
        self.ctx = ctx
        self.n = params.n

    def call(self, name: str, *args) -> None:
        rc = getattr(self.lib, name)(self.ctx, *args)
        _abi.check(self.lib, self.ctx, rc, name)

    def close(self) -> None:
        if getattr(self, "ctx", None):
            self.lib.hk_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # pointer arrays (host arrays of buffer addresses)
    def addr_array(self, bufs) -> C.Array:
        return (C.c_void_p * len(bufs))(*[self.addr(b) for b in bufs])

    def u32_array(self, vals) -> C.Array:
        return (C.c_uint32 * len(vals))(*[int(v) for v in vals])


class GpuEngine(_EngineBase):
    """libhekan_gpu.so on one CUDA device; buffers are torch int64 tensors."""

    kind = "gpu"

    def __init__(self, params, device: int = 0):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("GpuEngine needs a CUDA device (no CPU fallback)")
        self.torch = torch
        self.device = torch.device("cuda", device)
        torch.cuda.set_device(self.device)
        super().__init__(params, load_library(), device)
        self.bind_stream()

    def bind_stream(self, stream=None) -> None:
        torch = self.torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.call("hk_set_stream", C.c_void_p(s.cuda_stream))

    # --- buffers ---------------------------------------------------------
    def alloc_u64(self, n: int):
        return self.torch.empty(int(n), dtype=self.torch.int64, device=self.device)

    def alloc_f64(self, n: int):
        return self.torch.empty(int(n), dtype=self.torch.float64, device=self.device)

    @staticmethod
    def addr(buf) -> int:
        return buf.data_ptr()

    def put_f64(self, arr: np.ndarray):
        t = self.torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64).ravel())
        return t.to(self.device, non_blocking=False)

    def put_u64(self, arr: np.ndarray):
        a = np.ascontiguousarray(arr, dtype=np.uint64).ravel().view(np.int64)
        return self.torch.from_numpy(a.copy()).to(self.device)

    def get_u64(self, buf) -> np.ndarray:
        return buf.detach().cpu().numpy().view(np.uint64).copy()

    def get_f64(self, buf) -> np.ndarray:
        return buf.detach().cpu().numpy().copy()

    def sync(self) -> None:
        self.torch.cuda.synchronize(self.device)
