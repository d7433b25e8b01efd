"""Bit-exact parity: the sm_100a library vs the CPU oracle, op by op.

Same parameters, same seeds, same inputs -> identical u64 limbs (canonical
residues) for every C-ABI entry point in include/hekan.h. Sizes cover the
generic per-stage NTT path (small N) and the N = 2^16 fast path.
"""

import ctypes as C

import numpy as np
import pytest

from paper_2409_07751_b200.backend import BackendConfig, HeBackend, galois_element
from paper_2409_07751_b200.params import make_params, microbench_params

pytestmark = pytest.mark.gpu

CASES = [(5, 6), (10, 4), (13, 3), (16, 3), (17, 2)]


def _pair(log_n, depth, seed=0, dnum=3):
    from oracle.engine import OracleEngine
    from paper_2409_07751_b200.engine import GpuEngine
    p = make_params(log_n, depth, dnum=dnum)
    cfg = BackendConfig(slot_count=p.slot_count, depth_budget=depth, rng_seed=seed)
    g = HeBackend(cfg, p, engine=GpuEngine(p), seed=seed)
    o = HeBackend(cfg, p, engine=OracleEngine(p), seed=seed)
    return g, o, p


def _same(g, o, cg, co, what):
    a, b = g.export_ct(cg), o.export_ct(co)
    assert a.shape == b.shape, what
    bad = np.count_nonzero(a != b)
    assert bad == 0, f"{what}: {bad} of {a.size} limbs differ"


@pytest.mark.parametrize("log_n,depth", CASES)
def test_ntt_roundtrip_and_parity(gpu_lib, log_n, depth):
    import torch
    from oracle.engine import OracleEngine
    from paper_2409_07751_b200.engine import GpuEngine
    p = make_params(log_n, depth)
    ge, oe = GpuEngine(p), OracleEngine(p)
    rng = np.random.default_rng(log_n)
    nl, B, N = len(p.q) + len(p.p), 3, p.n
    mods = np.array(list(p.q) + list(p.p), dtype=np.uint64)
    x = (rng.integers(0, 1 << 62, size=(nl, B, N), dtype=np.uint64) % mods[:, None, None]).astype(np.uint64)
    gb, ob = ge.put_u64(x), oe.put_u64(x)
    ge.call("hk_ntt_fwd", ge.addr(gb), 0, nl, B)
    oe.call("hk_ntt_fwd", oe.addr(ob), 0, nl, B)
    ge.sync()
    assert np.array_equal(ge.get_u64(gb), oe.get_u64(ob))
    ge.call("hk_ntt_inv", ge.addr(gb), 0, nl, B)
    ge.sync()
    assert np.array_equal(ge.get_u64(gb), x.ravel())


@pytest.mark.parametrize("log_n,depth", CASES)
def test_keys_encrypt_bitexact(gpu_lib, log_n, depth):
    g, o, p = _pair(log_n, depth)
    for which in (0, 1):
        n = g.engine.lib.hk_key_words(g.engine.ctx, which)
        kg, ko = g.engine.alloc_u64(n), o.engine.alloc_u64(n)
        g.engine.call("hk_export_key", which, 0, g.engine.addr(kg))
        o.engine.call("hk_export_key", which, 0, o.engine.addr(ko))
        g.engine.sync()
        assert np.array_equal(g.engine.get_u64(kg), o.engine.get_u64(ko)), f"key {which}"
    x = np.random.default_rng(1).uniform(-1, 1, (2, p.slot_count))
    cg, co = g.encrypt(x), o.encrypt(x)
    _same(g, o, cg, co, "encrypt")
    np.testing.assert_array_equal(g.decrypt(cg), o.decrypt(co))
    assert np.abs(g.decrypt(cg) - x).max() < 1e-6


@pytest.mark.parametrize("log_n,depth", CASES)
def test_ops_bitexact(gpu_lib, log_n, depth):
    g, o, p = _pair(log_n, depth)
    S = p.slot_count
    rng = np.random.default_rng(7)
    x, y, w = (rng.uniform(-1, 1, (2, S)) for _ in range(3))
    ga, gb = g.encrypt(x), g.encrypt(y)
    oa, ob = o.encrypt(x), o.encrypt(y)
    pv = w[0]
    steps = [1, -1, 3, S // 4]
    checks = [
        ("add", lambda be, a, b: be.add(a, b)),
        ("sub", lambda be, a, b: be.sub(a, b)),
        ("add_pt", lambda be, a, b: be.add(a, pv)),
        ("sub_pt", lambda be, a, b: be.sub(a, pv)),
        ("add_const", lambda be, a, b: be.add(a, 0.375)),
        ("mul_pt", lambda be, a, b: be.mul(a, pv)),
        ("mul_const", lambda be, a, b: be.mul(a, -1.25)),
        ("mul_ct", lambda be, a, b: be.mul(a, b)),
        ("mul_ct_levels", lambda be, a, b: be.mul(be.mul(a, 0.5), b)),
        ("add_levels", lambda be, a, b: be.add(be.mul(a, 0.5), b)),
        ("rot", lambda be, a, b: be.rotate(a, 1)),
        ("rot_neg", lambda be, a, b: be.rotate(a, -3)),
        ("mac", lambda be, a, b: be.mac_plain([a, b], [pv, w[1]])),
        ("mul_lin", lambda be, a, b: be.mul_lin(be.mul(a, 0.5), be.mul(b, 2.0), a, -0.375)),
        ("mul_lin_same_level", lambda be, a, b: be.mul_lin(a, b, be.add(a, b), 1.5)),
        ("mul_affine", lambda be, a, b: be.mul_affine(a, b, 2, -1.0)),
        ("mul2", lambda be, a, b: be.mul2(a, b, be.rotate(a, 1), be.mul(b, 0.5))),
        ("mul_affine_levels", lambda be, a, b: be.mul_affine(be.mul(a, 0.5), b, 1, 0.25)),
    ]
    for name, fn in checks:
        _same(g, o, fn(g, ga, gb), fn(o, oa, ob), name)
    for cg, co in zip(g.rotate_many(ga, steps), o.rotate_many(oa, steps)):
        _same(g, o, cg, co, "hoisted")
    # values are right, too
    np.testing.assert_allclose(g.decrypt(g.mul(ga, gb)), x * y, atol=1e-6)
    np.testing.assert_allclose(g.decrypt(g.rotate(ga, 3)), np.roll(x, -3, axis=1), atol=1e-6)


def test_microbench_params_bitexact(gpu_lib):
    """BASELINE config 2 parameters (24 x 50-bit limbs, dnum 3, alpha 8)."""
    from oracle.engine import OracleEngine
    from paper_2409_07751_b200.engine import GpuEngine
    p = microbench_params()
    cfg = BackendConfig(slot_count=p.slot_count, depth_budget=p.depth)
    g = HeBackend(cfg, p, engine=GpuEngine(p), seed=0)
    o = HeBackend(cfg, p, engine=OracleEngine(p), seed=0)
    x = np.random.default_rng(3).uniform(-1, 1, p.slot_count)
    ga, oa = g.encrypt(x), o.encrypt(x)
    _same(g, o, g.mul(ga, ga), o.mul(oa, oa), "mul")
    _same(g, o, g.rotate(ga, 1 << 14), o.rotate(oa, 1 << 14), "rotate")


@pytest.mark.parametrize("log_n,depth", [(13, 5), (16, 4)])
def test_level_truncated_galois_keys(gpu_lib, log_n, depth):
    """Galois keys are stored truncated to the highest level asked for and
    regrown on demand (hk_add_galois_keys_level); the oracle keeps full keys.
    Rotations at a low level (truncated key), then at a higher level (regrown
    key), then hoisted, must stay bit-exact."""
    g, o, p = _pair(log_n, depth)
    S = p.slot_count
    x = np.random.default_rng(11).uniform(-1, 1, (2, S))
    ga, oa = g.encrypt(x), o.encrypt(x)
    gl, ol = g.mul(g.mul(ga, 0.5), 2.0), o.mul(o.mul(oa, 0.5), 2.0)  # level depth - 2
    _same(g, o, g.rotate(gl, 5), o.rotate(ol, 5), "rotate at low level")
    elt = galois_element(5, S)
    assert g.engine.lib.hk_has_galois_key(g.engine.ctx, elt) == gl.level + 1
    _same(g, o, g.rotate(ga, 5), o.rotate(oa, 5), "rotate at top level (regrown key)")
    assert g.engine.lib.hk_has_galois_key(g.engine.ctx, elt) == depth + 1
    for cg, co in zip(g.rotate_many(gl, [5, 7, -2]), o.rotate_many(ol, [5, 7, -2])):
        _same(g, o, cg, co, "hoisted, mixed key levels")
    np.testing.assert_allclose(g.decrypt(g.rotate(gl, 5)), np.roll(x, -5, axis=1), atol=1e-6)


@pytest.mark.parametrize("B,n_o,n_in,split", [(8, 24, 64, (8, 8)), (8, 64, 40, (7, 10)), (2, 24, 64, (8, 8))])
def test_bsgs_device_diagonals_bitexact(gpu_lib, B, n_o, n_in, split):
    """bsgs_matvec through hk_encode_diagonals + hk_mac_plain_blocks (grouped
    giant-step MAC, B >= 8) or the per-block fused MAC (B < 8): bit-exact with the
    oracle and equal to W x in cleartext."""
    from paper_2409_07751_b200 import inference as inf
    g, o, p = _pair(13, 3)
    S = p.slot_count
    rng = np.random.default_rng(5)
    W = rng.uniform(-0.5, 0.5, (n_o, n_in))
    x = np.zeros((B, S))
    x[:, :n_in] = rng.uniform(-1, 1, (B, n_in))
    cg = inf.bsgs_matvec(W, g.encrypt(x), split=split)
    co = inf.bsgs_matvec(W, o.encrypt(x), split=split)
    _same(g, o, cg, co, "bsgs")
    assert g.counter.pt_mults == o.counter.pt_mults == max(n_o, n_in)
    np.testing.assert_allclose(g.decrypt(cg)[:, :n_o], x[:, :n_in] @ W.T, atol=1e-6)


@pytest.mark.parametrize("log_n,depth", [(13, 4), (16, 3)])
def test_rotate_sum_bitexact(gpu_lib, log_n, depth):
    """hk_rotate_sum (lazy ModDown over BSGS giant steps, identity terms included):
    bit-exact with the oracle and equal to the sum of rotations in value."""
    g, o, p = _pair(log_n, depth)
    S = p.slot_count
    rng = np.random.default_rng(9)
    xs = [rng.uniform(-1, 1, (2, S)) for _ in range(4)]
    steps = [0, 3, -7, 3]
    gc, oc = [g.encrypt(x) for x in xs], [o.encrypt(x) for x in xs]
    _same(g, o, g.rotate_sum(gc, steps), o.rotate_sum(oc, steps), "rotate_sum")
    _same(g, o, g.rotate_sum(gc[:1], [0]), o.rotate_sum(oc[:1], [0]), "rotate_sum identity only")
    ref = sum(np.roll(x, -t, axis=1) for x, t in zip(xs, steps))
    np.testing.assert_allclose(g.decrypt(g.rotate_sum(gc, steps)), ref, atol=1e-6)


def test_serialised_ciphertexts_cross_engines(gpu_lib):
    # client boundary: bytes written by the GPU backend load into the oracle
    # backend (same parameters and seed) and vice versa, limbs unchanged
    g, o, p = _pair(13, 3)
    X = np.random.default_rng(11).uniform(-1, 1, (2, p.slot_count))
    cg = g.rotate(g.mul(g.encrypt(X), g.encrypt(X)), 3)
    co = o.deserialize_ct(g.serialize_ct(cg))
    assert np.array_equal(o.export_ct(co), g.export_ct(cg))
    np.testing.assert_allclose(o.decrypt(co), np.roll(X * X, -3, axis=1), atol=1e-6)
    back = g.deserialize_ct(o.serialize_ct(co))
    assert np.array_equal(g.export_ct(back), g.export_ct(cg))


@pytest.mark.parametrize("B", [1, 3, 5, 6])
def test_ragged_batches_bitexact(gpu_lib, B):
    # batch sizes that are not multiples of the key inner product's 4-sample walk,
    # and a single ciphertext, at the bench ring (N = 2^16)
    g, o, p = _pair(16, 3)
    rng = np.random.default_rng(20 + B)
    x, y = rng.uniform(-1, 1, (B, p.slot_count)), rng.uniform(-1, 1, (B, p.slot_count))
    ga, gb, oa, ob = g.encrypt(x), g.encrypt(y), o.encrypt(x), o.encrypt(y)
    _same(g, o, g.mul(ga, gb), o.mul(oa, ob), f"mul B={B}")
    _same(g, o, g.rotate(ga, -5), o.rotate(oa, -5), f"rotate B={B}")
    _same(g, o, g.mul(ga, 0.75), o.mul(oa, 0.75), f"mul_const B={B}")
    for cg, co in zip(g.rotate_many(ga, [1, 2, 7]), o.rotate_many(oa, [1, 2, 7])):
        _same(g, o, cg, co, f"hoisted B={B}")


def test_ntt_large_primes_extreme_inputs(gpu_lib):
    """Forward / inverse NTT at the config-2 primes (all just below 2^50: the
    kernels' large-prime path, which recentres every second stage) on inputs
    that push the lazy bounds: all q - 1, alternating 0 / q - 1 at several
    strides, (q - 1) / 2, and uniform draws. GPU == oracle exactly, and the
    inverse returns the input."""
    from oracle.engine import OracleEngine
    from paper_2409_07751_b200.engine import GpuEngine
    p = microbench_params()
    ge, oe = GpuEngine(p), OracleEngine(p)
    mods = np.array(list(p.q) + list(p.p), dtype=np.uint64)
    assert mods.min() >= (1 << 47) and mods.max() < (1 << 50)
    nl, N = len(mods), p.n
    rng = np.random.default_rng(11)
    pats = [np.broadcast_to(mods[:, None] - 1, (nl, N)).copy()]
    idx = np.arange(N)
    for stride in (1, 2, 256, 257, 32768):
        pats.append(np.where(((idx // stride) & 1)[None, :] == 1, mods[:, None] - 1, 0).astype(np.uint64))
    pats.append(np.broadcast_to((mods[:, None] - 1) // 2, (nl, N)).copy())
    pats.append((rng.integers(0, 1 << 62, size=(nl, N), dtype=np.uint64) % mods[:, None]).astype(np.uint64))
    x = np.ascontiguousarray(np.stack(pats, axis=1).astype(np.uint64))  # [nl][B][N]
    B = x.shape[1]
    gb, ob = ge.put_u64(x), oe.put_u64(x)
    ge.call("hk_ntt_fwd", ge.addr(gb), 0, nl, B)
    oe.call("hk_ntt_fwd", oe.addr(ob), 0, nl, B)
    ge.sync()
    assert np.array_equal(ge.get_u64(gb), oe.get_u64(ob))
    ge.call("hk_ntt_inv", ge.addr(gb), 0, nl, B)
    ge.sync()
    assert np.array_equal(ge.get_u64(gb), x.ravel())
    # the inverse on its own extreme inputs
    gb, ob = ge.put_u64(x), oe.put_u64(x)
    ge.call("hk_ntt_inv", ge.addr(gb), 0, nl, B)
    oe.call("hk_ntt_inv", oe.addr(ob), 0, nl, B)
    ge.sync()
    assert np.array_equal(ge.get_u64(gb), oe.get_u64(ob))
