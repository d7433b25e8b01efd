"""RNS-CKKS backend behind the reference's `HeBackend` plugin contract.

Mirrors `/root/reference/pkg/src/hekan/backend.py:23-309` name for name:
`BackendConfig`, `OpCounter`, `PlainVector`, `CipherText`, `HeBackend`
methods (`encode`, `encrypt`, `decrypt`, `refresh`, `reset_counter`,
`slotwise`, `add`, `sub`, `mul`, `rotate`) and the module helpers
(`slotwise`, `rotate`, `decrypt`, `make_backend`), with the reference's level
rule, counters and error behaviour. Underneath, every op is one call into the
sm_100a library (include/hekan.h) on limb-major RNS buffers in HBM:

  reference                          engine
  --------------------------------   -----------------------------------------
  CipherText.slots float64[S]        u64 [2][level+1][B][N], NTT domain
  slotwise add/sub (:209-214)        hk_add / hk_sub / hk_add_plain / hk_add_const
  slotwise mul_pt  (:215-224)        hk_mul_plain / hk_mul_const (+ rescale)
  slotwise mul_ct  (:215-224)        hk_mul: tensor + relinearise + rescale
  rotate np.roll(-t) (:237-245)      hk_rotate: X -> X^(5^t) + key switch

Batching: a `CipherText` carries a leading batch dimension B (independent
samples in one buffer, one launch per op). Counters tally LOGICAL ops per call,
i.e. per inference, exactly as the reference counts one ciphertext.
Plain operands are shared across the batch.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import itertools
import json
import math
import secrets
import struct

import numpy as np

from . import _abi
from ._ref import hekan
from .errors import CorruptFile, DepthExhausted, InputTooLong, LengthMismatch, SchemaMismatch
from .params import CkksParams, kan_params

OP_KINDS = ("add", "sub", "mul_ct", "mul_pt")


# ---------------------------------------------------------------------------
# configuration, counters, plain operands: the reference's own types
# (backend.py:23-112), so configs, counters and plain vectors pass across the
# boundary unchanged
# ---------------------------------------------------------------------------

BackendConfig = hekan.backend.BackendConfig
OpCounter = hekan.backend.OpCounter
PlainVector = hekan.backend.PlainVector


class CipherText:
    """Batched RNS-CKKS ciphertext handle (reference value type
    backend.py:115-129). Immutable: every op returns a new handle that owns a
    fresh HBM buffer u64 [2][level+1][batch][N]. `slots` decrypts lazily
    (debug/test convenience; needs the secret key held by the backend)."""

    __slots__ = ("data", "level", "tag", "backend", "batch", "batched", "__weakref__")

    def __init__(self, data, level: int, tag: str, backend: "HeBackend", batch: int,
                 batched: bool):
        self.data = data
        self.level = level
        self.tag = tag
        self.backend = backend
        self.batch = batch
        self.batched = batched

    @property
    def slots(self) -> np.ndarray:
        return self.backend.decrypt(self)

    def __repr__(self) -> str:
        return f"CipherText(level={self.level}, tag={self.tag!r}, batch={self.batch})"


def _slot_rows(values, slot_count: int):
    """Encode-style zero padding / broadcast to (B, S) plus the batched flag."""
    if np.isscalar(values):
        return np.full((1, slot_count), float(values)), False
    arr = np.asarray(values, dtype=float)
    batched = arr.ndim >= 2
    rows = arr.reshape(arr.shape[0], -1) if batched else arr.reshape(1, -1)
    if rows.shape[1] > slot_count:
        raise InputTooLong(f"{rows.shape[1]} values > {slot_count} slots")
    out = np.zeros((rows.shape[0], slot_count))
    out[:, : rows.shape[1]] = rows
    return out, batched


def _const_of(arr: np.ndarray):
    """Python float if every slot holds the same value (scalar fast path)."""
    if arr.size and np.all(arr == arr.flat[0]):
        return float(arr.flat[0])
    return None


def galois_element(t: int, slot_count: int) -> int:
    """Left rotation by t <-> X -> X^(5^t mod 2N) (slot j <-> zeta^(5^j))."""
    return pow(5, t % slot_count, 4 * slot_count)


# ---------------------------------------------------------------------------
# backend
# ---------------------------------------------------------------------------


class HeBackend:
    """RNS-CKKS implementation of the reference backend contract
    (backend.py:132-270). `engine` is the sm_100a library (GpuEngine) in the
    product; tests may substitute the CPU oracle engine to check bit-exactness."""

    def __init__(self, config: BackendConfig, params: CkksParams | None = None,
                 engine=None, device: int = 0, seed: int | None = None, sample_offset: int = 0):
        if params is None:
            log_n = int(math.log2(config.slot_count)) + 1
            params = kan_params(config.depth_budget, log_n=log_n)
        if params.slot_count != config.slot_count:
            raise ValueError(f"params give {params.slot_count} slots, config {config.slot_count}")
        if config.depth_budget > params.depth:
            raise ValueError(f"depth_budget {config.depth_budget} > chain depth {params.depth}")
        if config.noise_std > 0:
            # the reference's NoisyBackend (backend.py:281-297) simulates noise; a
            # real scheme carries its own, so refuse rather than run other semantics
            raise NotImplementedError(
                "noise_std > 0 selects the reference's NoisyBackend simulator; the RNS-CKKS "
                "engine's noise is the scheme's own (use noise_std = 0)")
        self.config = config
        self.params = params
        self.counter = OpCounter()
        self._tags = itertools.count()
        if engine is None:
            from .engine import GpuEngine
            engine = GpuEngine(params, device)
        self.engine = engine
        self.n = params.n
        self._enc_counter = itertools.count()
        self._pt_cache: dict = {}
        self._mat_cache: dict = {}
        self._pt_cache_bytes = 0
        self.pt_cache_limit = 8 << 30
        # Key and encryption randomness (ChaCha20 on the device, 256-bit seeds):
        # a master key from the OS CSPRNG unless a seed is passed explicitly
        # (bit-exact oracle parity; one seed shared by every rank of a sharded
        # run). `sample_offset` is this backend's first global sample index:
        # encryption randomness is indexed by global sample, so no two
        # encryptions of a sharded batch share (a, e), and the shards encrypt
        # exactly as the whole batch would in one process.
        self._master = (secrets.token_bytes(32) if seed is None
                        else hashlib.blake2b(f"hekan-b200:{int(seed)}".encode(), digest_size=32).digest())
        self._sample_offset = int(sample_offset)
        self.engine.call("hk_keygen", self._seed("keys"))

    # ------------------------------------------------------------------
    # boundary plumbing
    # ------------------------------------------------------------------

    def _seed(self, what: str, idx: int = 0):
        """uint64_t[4] ChaCha20 key for one purpose, derived from the master key."""
        return _abi.seed_words(hashlib.blake2b(f"{what}:{idx}".encode(), key=self._master,
                                               digest_size=32).digest())

    def encode(self, values) -> PlainVector:
        """Zero-pad a vector (or broadcast a scalar) to the slot count (:149-158)."""
        if np.isscalar(values):
            return PlainVector(np.full(self.config.slot_count, float(values)))
        arr = np.asarray(values, dtype=float).ravel()
        if arr.size > self.config.slot_count:
            raise InputTooLong(f"{arr.size} values > {self.config.slot_count} slots")
        out = np.zeros(self.config.slot_count)
        out[: arr.size] = arr
        return PlainVector(out)

    def encrypt(self, values, level: int | None = None) -> CipherText:
        """Fresh RLWE encryption at `level` (:160-166). A 2-D input (B, n)
        yields one batched ciphertext of B samples."""
        if level is None:
            level = self.config.depth_budget
        if not 0 <= level <= self.config.depth_budget:
            raise ValueError(f"level {level} outside [0, {self.config.depth_budget}]")
        rows, batched = _slot_rows(values, self.config.slot_count)
        return self._encrypt_rows(rows, level, batched)

    def _encrypt_rows(self, rows: np.ndarray, level: int, batched: bool) -> CipherText:
        eng, B = self.engine, rows.shape[0]
        slots = eng.put_f64(rows)
        pt = eng.alloc_u64((level + 1) * B * self.n)
        eng.call("hk_encode", eng.addr(slots), B, level, self.params.scale(level), eng.addr(pt))
        ct = eng.alloc_u64(2 * (level + 1) * B * self.n)
        seed = self._seed("enc", next(self._enc_counter))
        eng.call("hk_encrypt", eng.addr(pt), level, B, seed, C.c_uint64(self._sample_offset), eng.addr(ct))
        return self._wrap(ct, level, B, batched)

    def decrypt(self, a: CipherText) -> np.ndarray:
        self._check_ours(a)
        eng = self.engine
        out = eng.alloc_f64(a.batch * self.config.slot_count)
        eng.call("hk_decrypt", eng.addr(a.data), a.level, a.batch, self.params.scale(a.level),
                 eng.addr(out))
        vals = eng.get_f64(out).reshape(a.batch, self.config.slot_count)
        return vals if a.batched else vals[0]

    def refresh(self, a: CipherText, level: int | None = None) -> CipherText:
        """Level reset (:172-180). The reference's zero-cost bootstrapping
        stand-in; here a secret-key decrypt/re-encrypt debug path (real
        bootstrapping is out of scope). No counts."""
        if level is None:
            level = self.config.depth_budget
        self._check_ours(a)
        vals = self.decrypt(a)
        rows = vals if a.batched else vals[None, :]
        return self._encrypt_rows(rows, level, a.batched)

    def reset_counter(self) -> OpCounter:
        old = self.counter
        self.counter = OpCounter()
        return old

    # ------------------------------------------------------------------
    # plaintext encoding cache
    # ------------------------------------------------------------------

    def _encoded(self, slots: np.ndarray, level: int, scale: float):
        """Device plaintext u64 [level+1][1][N] for `slots`, cached."""
        key = (hashlib.blake2b(np.ascontiguousarray(slots).view(np.uint8), digest_size=16).digest(),
               level, scale)
        hit = self._pt_cache.get(key)
        if hit is not None:
            return hit
        eng = self.engine
        dev = eng.put_f64(slots)
        pt = eng.alloc_u64((level + 1) * self.n)
        eng.call("hk_encode", eng.addr(dev), 1, level, scale, eng.addr(pt))
        nbytes = (level + 1) * self.n * 8
        if self._pt_cache_bytes + nbytes > self.pt_cache_limit:
            self._pt_cache.clear()
            self._pt_cache_bytes = 0
        self._pt_cache[key] = pt
        self._pt_cache_bytes += nbytes
        return pt

    def _const_residues(self, value: float, level: int, scale: float):
        res = (C.c_uint64 * (level + 1))()
        self.engine.call("hk_encode_const", C.c_double(value), level, C.c_double(scale), res)
        return res

    # ------------------------------------------------------------------
    # homomorphic operations
    # ------------------------------------------------------------------

    def slotwise(self, op_kind: str, a: CipherText, b) -> CipherText:
        """Element-wise add/sub/mul with a cipher or plain operand (:192-224)."""
        if op_kind not in OP_KINDS:
            raise ValueError(f"unknown op_kind {op_kind!r}")
        self._check_ours(a)
        is_ct = isinstance(b, CipherText)
        if op_kind == "mul_ct" and not is_ct:
            raise LengthMismatch("mul_ct requires a ciphertext right operand")
        if op_kind == "mul_pt" and is_ct:
            raise LengthMismatch("mul_pt requires a plaintext right operand")
        if is_ct:
            self._check_ours(b)
            if b.batch != a.batch:
                raise LengthMismatch(f"batch {a.batch} vs {b.batch}")
            level = min(a.level, b.level)
            b_slots = None
        else:
            b_slots = self._plain_slots(b)
            level = a.level

        eng, B, n = self.engine, a.batch, self.n
        if op_kind in ("add", "sub"):
            out = eng.alloc_u64(2 * (level + 1) * B * n)
            if is_ct:
                eng.call("hk_add" if op_kind == "add" else "hk_sub", eng.addr(a.data), a.level,
                         eng.addr(b.data), b.level, eng.addr(out), B)
            else:
                c = _const_of(b_slots)
                if c is not None:
                    res = self._const_residues(c if op_kind == "add" else -c, level,
                                               self.params.scale(level))
                    eng.call("hk_add_const", eng.addr(a.data), a.level, res, eng.addr(out), B)
                else:
                    pt = self._encoded(b_slots, level, self.params.scale(level))
                    eng.call("hk_add_plain", eng.addr(a.data), a.level, eng.addr(pt), level, 1,
                             1 if op_kind == "sub" else 0, eng.addr(out), B)
            if op_kind == "add":
                self.counter.adds += 1
            else:
                self.counter.subs += 1
        else:
            if level < 1:
                raise DepthExhausted(f"multiplication at level {level} (tag {a.tag})")
            out = eng.alloc_u64(2 * level * B * n)
            if is_ct:
                eng.call("hk_mul", eng.addr(a.data), a.level, eng.addr(b.data), b.level,
                         eng.addr(out), B)
                self.counter.ct_mults += 1
            else:
                scale = self.params.pt_mult_scale(level)
                c = _const_of(b_slots)
                if c is not None:
                    res = self._const_residues(c, level, scale)
                    eng.call("hk_mul_const", eng.addr(a.data), a.level, res, eng.addr(out), B)
                else:
                    pt = self._encoded(b_slots, level, scale)
                    eng.call("hk_mul_plain", eng.addr(a.data), a.level, eng.addr(pt), level, 1,
                             eng.addr(out), B)
                self.counter.pt_mults += 1
            level -= 1
        return self._wrap(out, level, B, a.batched or (is_ct and b.batched))

    def mul_lin(self, a: CipherText, b: CipherText, x: CipherText, k: float) -> CipherText:
        """a * b + k * x: the Estrin / Chebyshev combine `hi * T + k * x`
        (reference approx.py:381-405 as mul_ct, mul_pt by a scalar, add) with
        the scalar product folded into the relinearised product's merged
        ModDown + rescale: one rescale instead of two and no separate add.
        Counts, levels and errors are those of the three reference ops; the
        output is at level min(a, b) - 1. Falls back to the three ops when x
        sits below the product's level."""
        self._check_ours(a)
        self._check_ours(b)
        self._check_ours(x)
        l = min(a.level, b.level)
        if l < 1:
            raise DepthExhausted(f"multiplication at level {l} (tag {a.tag})")
        if x.level < l or k == 0.0:
            return self.add(self.mul(a, b), self.mul(x, float(k)))
        if not (a.batch == b.batch == x.batch):
            raise LengthMismatch("mul_lin: batch sizes differ")
        B = a.batch
        # k x / q_l must land on the product's scale scales[l-1]
        scale = self.params.scale(l - 1) * self.params.q[l] / self.params.scale(x.level)
        res = self._const_residues(float(k), l, scale)
        eng = self.engine
        out = eng.alloc_u64(2 * l * B * self.n)
        eng.call("hk_mul_lin", eng.addr(a.data), a.level, eng.addr(b.data), b.level, eng.addr(x.data), x.level,
                 res, eng.addr(out), B)
        self.counter.ct_mults += 1
        self.counter.pt_mults += 1
        self.counter.adds += 1
        return self._wrap(out, l - 1, B, a.batched or b.batched or x.batched)

    def mul2(self, a: CipherText, b: CipherText, a2: CipherText, b2: CipherText) -> CipherText:
        """a * b + a2 * b2 with one relinearisation and one rescale (the
        Cox-de Boor step, reference bspline.py:308-317: two mul_ct and an add).
        Counted as those three ops; output at level min(levels) - 1."""
        for t in (a, b, a2, b2):
            self._check_ours(t)
        l = min(a.level, b.level, a2.level, b2.level)
        if l < 1:
            raise DepthExhausted(f"multiplication at level {l} (tag {a.tag})")
        if not (a.batch == b.batch == a2.batch == b2.batch):
            raise LengthMismatch("mul2: batch sizes differ")
        B = a.batch
        eng = self.engine
        out = eng.alloc_u64(2 * l * B * self.n)
        eng.call("hk_mul2", eng.addr(a.data), a.level, eng.addr(b.data), b.level, eng.addr(a2.data), a2.level,
                 eng.addr(b2.data), b2.level, eng.addr(out), B)
        self.counter.ct_mults += 2
        self.counter.adds += 1
        return self._wrap(out, l - 1, B, a.batched or b.batched or a2.batched or b2.batched)

    def mul_affine(self, a: CipherText, b: CipherText, mult: int, c: float) -> CipherText:
        """mult * (a * b) + c, the Chebyshev power step T_2k = 2 T_k^2 - 1
        (reference: mul_ct, add(sq, sq), add of a scalar) with the doubling and
        the constant applied in the product's last epilogue. Bit-identical to
        the three ops and counted as them."""
        self._check_ours(a)
        self._check_ours(b)
        if mult not in (1, 2):
            raise ValueError(f"mul_affine: multiplier {mult} not 1 or 2")
        l = min(a.level, b.level)
        if l < 1:
            raise DepthExhausted(f"multiplication at level {l} (tag {a.tag})")
        if a.batch != b.batch:
            raise LengthMismatch("mul_affine: batch sizes differ")
        B = a.batch
        res = self._const_residues(float(c), l - 1, self.params.scale(l - 1)) if c != 0.0 else None
        eng = self.engine
        out = eng.alloc_u64(2 * l * B * self.n)
        eng.call("hk_mul_affine", eng.addr(a.data), a.level, eng.addr(b.data), b.level, int(mult), res,
                 eng.addr(out), B)
        self.counter.ct_mults += 1
        self.counter.adds += (1 if mult == 2 else 0) + (1 if c != 0.0 else 0)
        return self._wrap(out, l - 1, B, a.batched or b.batched)

    def add(self, a: CipherText, b) -> CipherText:
        return self.slotwise("add", a, b)

    def sub(self, a: CipherText, b) -> CipherText:
        return self.slotwise("sub", a, b)

    def mul(self, a: CipherText, b) -> CipherText:
        kind = "mul_ct" if isinstance(b, CipherText) else "mul_pt"
        return self.slotwise(kind, a, b)

    def rotate(self, a: CipherText, t: int) -> CipherText:
        """Cyclic shift: left for t > 0, right for t < 0 (:237-245)."""
        self._check_ours(a)
        if abs(t) >= self.config.slot_count:
            raise ValueError(f"|t| = {abs(t)} must be < slot_count {self.config.slot_count}")
        if t == 0:
            return a
        self.counter.rotations += 1
        g = galois_element(t, self.config.slot_count)
        self.ensure_galois_keys([g], a.level)
        eng = self.engine
        out = eng.alloc_u64(2 * (a.level + 1) * a.batch * self.n)
        eng.call("hk_rotate", eng.addr(a.data), a.level, C.c_uint32(g), eng.addr(out), a.batch)
        return self._wrap(out, a.level, a.batch, a.batched)

    def rotate_many(self, a: CipherText, steps) -> list:
        """Hoisted rotations of one source: one ModUp shared by every step
        (the baby steps of bsgs_matvec, inference.py:162). Counts one rotation
        per nonzero step, like calling rotate() per step."""
        self._check_ours(a)
        steps = [int(t) for t in steps]
        for t in steps:
            if abs(t) >= self.config.slot_count:
                raise ValueError(f"|t| = {abs(t)} must be < slot_count {self.config.slot_count}")
        todo = [t for t in steps if t != 0]
        outs = {}
        if todo:
            gs = [galois_element(t, self.config.slot_count) for t in todo]
            self.ensure_galois_keys(gs, a.level)
            eng = self.engine
            bufs = [eng.alloc_u64(2 * (a.level + 1) * a.batch * self.n) for _ in todo]
            eng.call("hk_rotate_hoisted", eng.addr(a.data), a.level, eng.u32_array(gs), len(gs),
                     eng.addr_array(bufs), a.batch)
            self.counter.rotations += len(todo)
            for t, buf in zip(todo, bufs):
                outs[t] = self._wrap(buf, a.level, a.batch, a.batched)
        return [a if t == 0 else outs[t] for t in steps]

    def rotate_sum(self, cts, steps) -> CipherText:
        """sum_i rotate(cts[i], steps[i]) with the key switches' inner products
        accumulated in the extended basis and one ModDown (BSGS giant steps,
        inference.py:177-180). Counts like rotate()-then-add: one rotation per
        nonzero step, len - 1 adds."""
        if not cts or len(cts) != len(steps):
            raise LengthMismatch("rotate_sum needs matching non-empty lists")
        a0 = cts[0]
        for x in cts:
            self._check_ours(x)
            if x.batch != a0.batch or x.level != a0.level:
                raise LengthMismatch("rotate_sum operands must share batch and level")
        steps = [int(t) for t in steps]
        for t in steps:
            if abs(t) >= self.config.slot_count:
                raise ValueError(f"|t| = {abs(t)} must be < slot_count {self.config.slot_count}")
        gs = [galois_element(t, self.config.slot_count) if t else 1 for t in steps]
        self.ensure_galois_keys([g for g in gs if g != 1], a0.level)
        eng = self.engine
        out = eng.alloc_u64(2 * (a0.level + 1) * a0.batch * self.n)
        eng.call("hk_rotate_sum", eng.addr_array([x.data for x in cts]), a0.level, eng.u32_array(gs), len(cts),
                 eng.addr(out), a0.batch)
        self.counter.rotations += sum(1 for t in steps if t)
        self.counter.adds += len(cts) - 1
        return self._wrap(out, a0.level, a0.batch, a0.batched)

    def mac_plain(self, babies, plains) -> CipherText:
        """sum_i babies[i] * plains[i] with ONE rescale (fused BSGS block,
        inference.py:171-178). Counts len(babies) pt_mults and len-1 adds."""
        n_terms = len(babies)
        if n_terms == 0 or n_terms != len(plains):
            raise LengthMismatch("mac_plain needs matching non-empty operand lists")
        a0 = babies[0]
        for x in babies:
            self._check_ours(x)
            if x.batch != a0.batch:
                raise LengthMismatch("batch mismatch in mac_plain")
        level = min(x.level for x in babies)
        if level < 1:
            raise DepthExhausted(f"multiplication at level {level}")
        scale = self.params.pt_mult_scale(level)
        pts = [self._encoded(self._plain_slots(p), level, scale) for p in plains]
        eng, B = self.engine, a0.batch
        if any(x.level != level for x in babies):
            raise ValueError("mac_plain operands must share one level")
        out = eng.alloc_u64(2 * level * B * self.n)
        eng.call("hk_mac_plain", eng.addr_array([x.data for x in babies]), eng.addr_array(pts),
                 n_terms, level, level, 1, eng.addr(out), B)
        self.counter.pt_mults += n_terms
        self.counter.adds += n_terms - 1
        return self._wrap(out, level - 1, B, a0.batched)

    # ------------------------------------------------------------------
    # BSGS diagonals on the device
    # ------------------------------------------------------------------

    def device_matrix(self, W: np.ndarray):
        """Engine-resident copy of a BSGS weight matrix (row-major f64), cached
        per content; the diagonals are generated from it on the device."""
        W = np.ascontiguousarray(W, dtype=np.float64)
        key = (hashlib.blake2b(W.view(np.uint8), digest_size=16).digest(), W.shape)
        hit = self._mat_cache.get(key)
        if hit is None:
            if len(self._mat_cache) > 64:
                self._mat_cache.clear()
            hit = self._mat_cache[key] = self.engine.put_f64(W)
        return hit

    def bsgs_blocks(self, babies, Wdev, shape, m: int, base: int, nb: int, counts) -> list:
        """len(counts) <= 8 consecutive giant-step blocks of bsgs_matvec starting at
        diagonal `base` (block g covers diagonals base + g*nb .. + counts[g] - 1 of
        the m x m zero-padded matrix, rolled by its own base): the group's diagonals
        are generated and encoded on the device in one call, every baby is read once
        for the whole group, then each block is rescaled. Counts per block exactly
        like mac_plain (counts[g] pt_mults, counts[g] - 1 adds)."""
        G = len(counts)
        if not 1 <= G <= 8 or not babies:
            raise LengthMismatch("bsgs_blocks needs 1..8 blocks and babies")
        a0 = babies[0]
        for x in babies:
            self._check_ours(x)
            if x.batch != a0.batch or x.level != a0.level:
                raise LengthMismatch("bsgs_blocks operands must share batch and level")
        level = a0.level
        if level < 1:
            raise DepthExhausted(f"multiplication at level {level}")
        eng, B, n = self.engine, a0.batch, self.n
        total = (G - 1) * nb + counts[-1]
        pt = eng.alloc_u64((level + 1) * total * n)
        eng.call("hk_encode_diagonals", eng.addr(Wdev), int(shape[0]), int(shape[1]), int(m), int(base),
                 total, int(nb), level, self.params.pt_mult_scale(level), eng.addr(pt))
        outs = [eng.alloc_u64(2 * level * B * n) for _ in range(G)]
        if 2 * B >= 16:  # the grouped kernel's (poly, sample) lanes are full
            cnt = (C.c_int32 * G)(*[int(x) for x in counts])
            eng.call("hk_mac_plain_blocks", eng.addr_array([x.data for x in babies]), len(babies), level,
                     eng.addr(pt), total, nb, G, cnt, eng.addr_array(outs), B)
        else:  # small batches: per-block fused MAC + rescale on the same diagonals
            p0 = eng.addr(pt)
            for g, c_ in enumerate(counts):
                ptrs = (C.c_void_p * c_)(*[p0 + (g * nb + i) * n * 8 for i in range(c_)])
                eng.call("hk_mac_plain", eng.addr_array([x.data for x in babies[:c_]]), ptrs, int(c_), level,
                         level, total, eng.addr(outs[g]), B)
        for c_ in counts:
            self.counter.pt_mults += int(c_)
            self.counter.adds += int(c_) - 1
        return [self._wrap(o, level - 1, B, a0.batched) for o in outs]

    def ensure_galois_keys(self, galois_elts, level: int | None = None) -> None:
        """Galois keys serving ciphertexts up to `level` (default: the top level).
        The GPU stores a key truncated to the highest level it has been asked
        for (digits and limbs above it are never read) and regrows it on demand;
        the key values do not depend on the level, so results are identical."""
        top = self.config.depth_budget
        level = top if level is None else min(int(level), top)
        lib, ctx = self.engine.lib, self.engine.ctx
        missing = [int(g) for g in galois_elts if lib.hk_has_galois_key(ctx, C.c_uint32(int(g))) < level + 1]
        if missing:
            missing = sorted(set(missing))
            self.engine.call("hk_add_galois_keys_level", self._seed("galois"),
                             self.engine.u32_array(missing), len(missing), level)

    def ensure_rotation_keys(self, steps, level: int | None = None) -> None:
        self.ensure_galois_keys([galois_element(t, self.config.slot_count)
                                 for t in steps if t % self.config.slot_count], level)

    # ------------------------------------------------------------------
    # internals
    # ------------------------------------------------------------------

    def _plain_slots(self, b) -> np.ndarray:
        if isinstance(b, PlainVector):
            if b.slots.size != self.config.slot_count:
                raise LengthMismatch(
                    f"plain operand has {b.slots.size} slots, backend {self.config.slot_count}")
            return b.slots
        return self.encode(b).slots

    def _check_ours(self, a) -> None:
        if not isinstance(a, CipherText) or a.backend is not self:
            raise LengthMismatch("ciphertext belongs to a different backend")

    def _wrap(self, data, level: int, batch: int, batched: bool) -> CipherText:
        consumed = self.config.depth_budget - level
        if consumed > self.counter.max_depth_consumed:
            self.counter.max_depth_consumed = consumed
        return CipherText(data, level, f"ct{next(self._tags)}", self, batch, batched)

    # ------------------------------------------------------------------
    # raw access (parity tests, serialisation)
    # ------------------------------------------------------------------

    def export_ct(self, a: CipherText) -> np.ndarray:
        """u64 [2][level+1][B][N] host copy of the RNS limbs."""
        self.engine.sync()
        return self.engine.get_u64(a.data).reshape(2, a.level + 1, a.batch, self.n)

    def adopt(self, data, level: int, batch: int, batched: bool = True) -> CipherText:
        """Wrap an engine buffer u64 [2][level+1][batch][N] (e.g. gathered from
        other ranks) as a ciphertext of this backend, without copying."""
        if int(np.prod(data.shape)) != 2 * (level + 1) * batch * self.n:
            raise LengthMismatch(f"buffer of {int(np.prod(data.shape))} words for level {level}, batch {batch}")
        return self._wrap(data, level, batch, batched)

    def import_ct(self, limbs: np.ndarray, level: int, batched: bool = True) -> CipherText:
        limbs = np.asarray(limbs, dtype=np.uint64)
        B = limbs.shape[2]
        if limbs.shape != (2, level + 1, B, self.n):
            raise LengthMismatch(f"limb array shape {limbs.shape}")
        return self._wrap(self.engine.put_u64(limbs), level, B, batched)

    # ------------------------------------------------------------------
    # ciphertext (de)serialisation (client boundary; the
    # reference has none). Little-endian, self-describing:
    #   magic "HKCT" | u32 version | 8-byte parameter fingerprint |
    #   i32 level | i32 batch | i32 log_n | u8 batched | 3 pad bytes |
    #   u64 limbs [2][level+1][batch][N] | 8-byte blake2b of all prior bytes
    # ------------------------------------------------------------------
    _CT_MAGIC = b"HKCT"
    _CT_VERSION = 1
    _CT_HEAD = struct.Struct("<4sI8siiiB3x")

    def params_fingerprint(self) -> bytes:
        """8-byte digest of the ring degree and every prime of the chain."""
        h = hashlib.blake2b(digest_size=8)
        h.update(struct.pack("<i", self.params.log_n))
        h.update(np.asarray(self.params.q, dtype=np.uint64).tobytes())
        h.update(np.asarray(self.params.p, dtype=np.uint64).tobytes())
        return h.digest()

    def serialize_ct(self, a: CipherText) -> bytes:
        self._check_ours(a)
        head = self._CT_HEAD.pack(self._CT_MAGIC, self._CT_VERSION, self.params_fingerprint(), a.level, a.batch,
                                  self.params.log_n, 1 if a.batched else 0)
        body = head + self.export_ct(a).astype("<u8", copy=False).tobytes()
        return body + hashlib.blake2b(body, digest_size=8).digest()

    def deserialize_ct(self, blob: bytes) -> CipherText:
        """Inverse of serialize_ct. CorruptFile on a bad magic, length or
        checksum; SchemaMismatch for another parameter set or version."""
        blob = bytes(blob)
        hs = self._CT_HEAD.size
        if len(blob) < hs + 8:
            raise CorruptFile(f"ciphertext blob of {len(blob)} bytes is shorter than its header")
        magic, ver, fp, level, batch, log_n, batched = self._CT_HEAD.unpack_from(blob)
        if magic != self._CT_MAGIC:
            raise CorruptFile(f"bad magic {magic!r}")
        if hashlib.blake2b(blob[:-8], digest_size=8).digest() != blob[-8:]:
            raise CorruptFile("ciphertext checksum mismatch")
        if ver != self._CT_VERSION:
            raise SchemaMismatch(f"ciphertext format version {ver}, expected {self._CT_VERSION}")
        if fp != self.params_fingerprint() or log_n != self.params.log_n:
            raise SchemaMismatch("ciphertext was made under another parameter set")
        if not 0 <= level <= self.config.depth_budget or batch < 1:
            raise CorruptFile(f"level {level} / batch {batch} out of range")
        want = 2 * (level + 1) * batch * self.n * 8
        if len(blob) != hs + want + 8:
            raise CorruptFile(f"limb payload of {len(blob) - hs - 8} bytes, expected {want}")
        limbs = np.frombuffer(blob, dtype="<u8", count=want // 8, offset=hs)
        limbs = limbs.reshape(2, level + 1, batch, self.n)
        qs = np.asarray(self.params.q[:level + 1], dtype=np.uint64)
        if np.any(limbs >= qs[None, :, None, None]):
            raise CorruptFile("limb residue not below its prime")
        return self.import_ct(limbs.astype(np.uint64), level, batched=bool(batched))


def save_ciphertext(path: str, a: CipherText) -> None:
    with open(path, "wb") as f:
        f.write(a.backend.serialize_ct(a))


def load_ciphertext(path: str, backend: "HeBackend") -> CipherText:
    with open(path, "rb") as f:
        return backend.deserialize_ct(f.read())


CkksBackend = HeBackend


def make_backend(config: BackendConfig, params: CkksParams | None = None, engine=None,
                 device: int = 0, seed: int | None = None, sample_offset: int = 0) -> HeBackend:
    """RNS-CKKS backend on the sm_100a engine (reference factory :293-297)."""
    return HeBackend(config, params=params, engine=engine, device=device, seed=seed, sample_offset=sample_offset)


def slotwise(op_kind: str, a: CipherText, b) -> CipherText:
    return a.backend.slotwise(op_kind, a, b)


def rotate(a: CipherText, t: int) -> CipherText:
    return a.backend.rotate(a, t)


def decrypt(a: CipherText) -> np.ndarray:
    return a.backend.decrypt(a)
