"""OracleEngine — the CPU RNS-CKKS oracle behind the same engine interface.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs, never by the product package. Buffers are numpy
uint64/float64 arrays; libckks_oracle.so exports the include/hekan.h ABI with
host pointers (see ckks_oracle.c for the parity status).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2409_07751_b200 import _abi
from paper_2409_07751_b200.engine import _EngineBase

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libckks_oracle.so")
_LIB = None


def build_oracle(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-C", HERE, "-s"], check=True)
    return LIB_PATH


def load_oracle() -> C.CDLL:
    global _LIB
    if _LIB is None:
        build_oracle()
        _LIB = _abi.bind(C.CDLL(LIB_PATH))
    return _LIB


class OracleEngine(_EngineBase):
    kind = "oracle"

    def __init__(self, params, device: int = 0):
        super().__init__(params, load_oracle(), device)

    def alloc_u64(self, n: int):
        return np.zeros(int(n), dtype=np.uint64)

    def alloc_f64(self, n: int):
        return np.zeros(int(n), dtype=np.float64)

    @staticmethod
    def addr(buf) -> int:
        return buf.ctypes.data

    def put_f64(self, arr):
        return np.ascontiguousarray(arr, dtype=np.float64).ravel().copy()

    def put_u64(self, arr):
        return np.ascontiguousarray(arr, dtype=np.uint64).ravel().copy()

    def get_u64(self, buf):
        return np.asarray(buf).view(np.uint64).copy()

    def get_f64(self, buf):
        return np.asarray(buf, dtype=np.float64).copy()

    def sync(self) -> None:
        pass
