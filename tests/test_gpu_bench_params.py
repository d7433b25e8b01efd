"""Bit-exact parity at the parameters the benchmark runs.

GPU engine vs CPU oracle on the same seeds and inputs, u64 limbs compared
exactly, at the ring and modulus chain of every BASELINE config:

* c1 / c4: N = 2^16, L = 36, dnum = 3 (alpha = 13), B = 8 ciphertexts — the
  fused N = 2^16 flows the bench times (merged ModDown + rescale, grouped BSGS
  MAC when 2B >= 16, sample-major rescale, hoisted and lazy-ModDown rotations);
* c3: N = 2^16, L = 54, alpha = 19;
* c5: N = 2^17, L = 36 (the 2^16 kernels behind the radix-2 pre/post passes);
* c2: the primitive microbench chain (24 limbs, alpha = 8), in test_gpu_parity.

The op semantics are the reference's (`/root/reference/pkg/src/hekan/
backend.py:192-245`), the program is the reference's
(`inference.py:263-314`); the oracle is oracle/ckks_oracle.c.
"""

import numpy as np
import pytest

from paper_2409_07751_b200 import configs, inference as inf
from paper_2409_07751_b200.backend import BackendConfig, HeBackend
from paper_2409_07751_b200.params import kan_params

pytestmark = pytest.mark.gpu
B = 8


def _pair(p, depth, seed=0):
    from oracle.engine import OracleEngine
    from paper_2409_07751_b200.engine import GpuEngine
    cfg = BackendConfig(slot_count=p.slot_count, depth_budget=depth)
    return (HeBackend(cfg, p, engine=GpuEngine(p), seed=seed),
            HeBackend(cfg, p, engine=OracleEngine(p), seed=seed))


def _same(g, o, cg, co, what):
    a, b = g.export_ct(cg), o.export_ct(co)
    assert a.shape == b.shape, what
    bad = np.count_nonzero(a != b)
    assert bad == 0, f"{what}: {bad} of {a.size} limbs differ"


def _op_suite(g, o, level, rng, batch=B):
    S = g.config.slot_count
    x, y, z = (rng.uniform(-1, 1, (batch, S)) for _ in range(3))
    ga, gb, gc = (g.encrypt(v, level) for v in (x, y, z))
    oa, ob, oc = (o.encrypt(v, level) for v in (x, y, z))
    ops = [
        ("mul", lambda be, a, b, c: be.mul(a, b)),
        ("mul_lin", lambda be, a, b, c: be.mul_lin(a, b, c, -0.375)),
        ("mul_affine", lambda be, a, b, c: be.mul_affine(a, a, 2, -1.0)),
        ("mul2", lambda be, a, b, c: be.mul2(a, b, c, be.rotate(b, 1))),
        ("mul_pt", lambda be, a, b, c: be.mul(a, z[0])),
        ("mul_const", lambda be, a, b, c: be.mul(a, 0.75)),
        ("rotate", lambda be, a, b, c: be.rotate(a, 5)),
        ("rotate_neg", lambda be, a, b, c: be.rotate(a, -(S // 4))),
        ("rotate_sum", lambda be, a, b, c: be.rotate_sum([a, b, c], [0, 3, -11])),
    ]
    for name, fn in ops:
        _same(g, o, fn(g, ga, gb, gc), fn(o, oa, ob, oc), f"{name} at level {level}")
    for cg, co in zip(g.rotate_many(ga, [1, 2, 7, -9]), o.rotate_many(oa, [1, 2, 7, -9])):
        _same(g, o, cg, co, f"rotate_many at level {level}")
    np.testing.assert_allclose(g.decrypt(g.mul(ga, gb)), x * y, atol=1e-6)


@pytest.mark.parametrize("level", [36, 18])
def test_c1_params_ops_bitexact(gpu_lib, level):
    """kan_params(36): N = 2^16, L = 36, alpha = 13 — the bench's chain."""
    p = kan_params(36)
    assert p.n == 1 << 16 and p.alpha == 13
    g, o = _pair(p, 36)
    _op_suite(g, o, level, np.random.default_rng(level))


def test_c1_params_ops_bitexact_batch16(gpu_lib):
    """The same chain at B = 16: the key inner product's 16-samples-per-thread
    walk (the bench's B = 128 takes it), every product variant and rotation."""
    p = kan_params(36)
    g, o = _pair(p, 36)
    _op_suite(g, o, 36, np.random.default_rng(16), batch=16)


def test_c1_params_bsgs_grouped_mac_bitexact(gpu_lib):
    """bsgs_matvec at B = 8: device diagonals, grouped MAC (2B >= 16) with its
    fused rescale, lazy-ModDown giant steps."""
    p = kan_params(36)
    g, o = _pair(p, 36)
    S = p.slot_count
    rng = np.random.default_rng(5)
    for n_o, n_in, split in [(10, 64, None), (64, 176, None), (24, 64, (8, 8))]:
        W = rng.normal(0, 0.1, (n_o, n_in))
        x = np.zeros((B, S))
        x[:, :n_in] = rng.uniform(-1, 1, (B, n_in))
        cg = inf.bsgs_matvec(W, g.encrypt(x, 20), split=split)
        co = inf.bsgs_matvec(W, o.encrypt(x, 20), split=split)
        _same(g, o, cg, co, f"bsgs {n_o}x{n_in}")
        np.testing.assert_allclose(g.decrypt(cg)[:, :n_o], x[:, :n_in] @ W.T, atol=1e-5)


def test_c1_full_inference_bitexact(gpu_lib):
    """One whole c1 inference at the bench's parameters, 8 samples."""
    _, model, X = configs.workload("c1", batch=B)
    p = kan_params(36)
    g, o = _pair(p, 36)
    cfg = inf.PipelineConfig()
    og, sg = inf.model_forward_he(model, inf.encrypt_input(X, model, g), cfg)
    oo, so = inf.model_forward_he(model, inf.encrypt_input(X, model, o), cfg)
    _same(g, o, og, oo, "c1 inference")
    assert sg.to_json()["total"] | {"wall_time_ms": 0} == so.to_json()["total"] | {"wall_time_ms": 0}
    gold = np.load("tests/golden/c1.npz")["mirrored"][:B]
    assert np.abs(g.decrypt(og)[:, :1] - gold).max() < 1e-4


def test_c4_layer1_bitexact(gpu_lib):
    """c4 layer 1 (784 -> 64: 6272-diagonal spline BSGS with 80 hoisted babies,
    784-diagonal base BSGS) at N = 2^16, L = 36, 8 samples."""
    from paper_2409_07751_b200.model import KanModel
    _, model, X = configs.workload("c4", batch=B)
    layer = model.layers[0]
    one = KanModel(layers=[layer], input_shape=model.input_shape)
    p = kan_params(36)
    g, o = _pair(p, 36)
    cfg = inf.PipelineConfig()
    og = inf.layer_forward_he(layer, inf.encrypt_input(X, one, g), cfg)
    oo = inf.layer_forward_he(layer, inf.encrypt_input(X, one, o), cfg)
    assert og.level == 36 - inf.plan_layer(layer, cfg).total
    _same(g, o, og, oo, "c4 layer 1")


@pytest.mark.parametrize("level", [54, 27])
def test_c3_params_ops_bitexact(gpu_lib, level):
    """kan_params(54): N = 2^16, L = 54, alpha = 19 (c3's chain)."""
    p = kan_params(54)
    assert p.alpha == 19
    g, o = _pair(p, 54)
    _op_suite(g, o, level, np.random.default_rng(100 + level), batch=4)


@pytest.mark.parametrize("level", [36, 12])
def test_c5_params_ops_bitexact(gpu_lib, level):
    """kan_params(36, log_n=17): N = 2^17 (c5's ring)."""
    p = kan_params(36, log_n=17)
    g, o = _pair(p, 36)
    _op_suite(g, o, level, np.random.default_rng(200 + level), batch=2)
