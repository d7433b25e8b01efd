"""The drop-in boundary, proven with the reference's own code.

The reference package (`hekan`, imported unmodified from baseline/_ref) runs
its own pipeline functions — `bsgs_matvec`, `repeat_pack`, `model_forward_he`,
`bench_compare` — on this repo's `HeBackend` (reference contract
/root/reference/pkg/src/hekan/backend.py:132-270). Every case runs on the CPU
oracle engine here and on the sm_100a engine on the GPU box (`-m gpu`).

The only reference function re-routed is the composite comparator's stage
evaluation, as INTEGRATION.md §2 instructs a maintainer to do: the reference's
monomial stages (|coef| up to 6e10) diverge under real CKKS noise, so
`hekan.bspline.poly_comp` is pointed at the engine's Chebyshev `poly_comp`
(same polynomial, same levels, same multiplication counts).
"""

import json
import os

import numpy as np
import pytest

from paper_2409_07751_b200 import configs
from paper_2409_07751_b200 import approx as eng_approx
from paper_2409_07751_b200._ref import hekan
from paper_2409_07751_b200.backend import HeBackend
from paper_2409_07751_b200.params import make_params

GOLD = os.path.join(os.path.dirname(__file__), "golden")
ENGINES = ["oracle", pytest.param("gpu", marks=pytest.mark.gpu)]


def _engine(kind, p):
    if kind == "gpu":
        import torch
        if not torch.cuda.is_available():
            pytest.skip("no CUDA device")
        from paper_2409_07751_b200.build import build
        build()
        from paper_2409_07751_b200.engine import GpuEngine
        return GpuEngine(p)
    from oracle.engine import OracleEngine
    return OracleEngine(p)


def _backend(kind, depth, log_n=8):
    p = make_params(log_n, depth)
    cfg = hekan.backend.BackendConfig(slot_count=p.slot_count, depth_budget=depth)
    return HeBackend(cfg, p, engine=_engine(kind, p), seed=0)


@pytest.mark.parametrize("kind", ENGINES)
def test_reference_bsgs_matvec_on_engine(kind):
    # reference KAT (pkg/tests/test_inference.py:70-73): [[1,2],[3,4]] (5,6) = (17,39)
    be = _backend(kind, 2)
    out = hekan.inference.bsgs_matvec(np.array([[1.0, 2.0], [3.0, 4.0]]), be.encrypt([5.0, 6.0]))
    np.testing.assert_allclose(be.decrypt(out)[:2], [17.0, 39.0], atol=1e-6)
    assert out.level == 1
    ref = hekan.backend.CleartextBackend(hekan.backend.BackendConfig(slot_count=be.config.slot_count,
                                                                     depth_budget=2))
    hekan.inference.bsgs_matvec(np.array([[1.0, 2.0], [3.0, 4.0]]), ref.encrypt([5.0, 6.0]))
    assert be.counter == ref.counter


@pytest.mark.parametrize("kind", ENGINES)
def test_reference_repeat_pack_on_engine(kind):
    # reference KAT (pkg/tests/test_bspline.py:62-65): copies of (1, 2)
    be = _backend(kind, 2)
    xp = hekan.bspline.repeat_pack(be.encrypt([1.0, 2.0]), 3, 2, 2)
    copies = 3 + 2 * 2
    np.testing.assert_allclose(be.decrypt(xp.ct)[: 2 * copies], [1.0, 2.0] * copies, atol=1e-6)
    assert be.counter.rotations == hekan.bspline.pack_rotations(3, 2)


@pytest.mark.parametrize("kind", ENGINES)
def test_reference_model_forward_exact_comparator(kind):
    """Unmodified hekan.inference.model_forward_he with the exact (debug)
    comparator, a random reference model: matches the reference's mirrored
    forward and the reference simulator's counts."""
    model = hekan.model.random_model([3, 4], g=3, k=2, seed=4)
    cfg = hekan.inference.PipelineConfig(comparator_mode="exact")
    depth = hekan.inference.plan_model(model, cfg).total
    be = _backend(kind, depth)
    x = np.random.default_rng(2).uniform(-0.9, 0.9, 3)
    out, stats = hekan.inference.model_forward_he(model, hekan.inference.encrypt_input(x, model, be), cfg)
    want = hekan.model.model_forward_plain(model, x, "mirrored", cfg.comparator())
    assert np.abs(be.decrypt(out)[:4] - want).max() < 1e-6
    sim = hekan.backend.CleartextBackend(hekan.backend.BackendConfig(slot_count=be.config.slot_count,
                                                                     depth_budget=depth))
    _, ref_stats = hekan.inference.model_forward_he(model, hekan.inference.encrypt_input(x, model, sim), cfg)
    assert stats.to_json()["total"] | {"wall_time_ms": 0} == ref_stats.to_json()["total"] | {"wall_time_ms": 0}


@pytest.mark.parametrize("kind", ENGINES)
def test_reference_pipeline_composite_comparator(kind, monkeypatch):
    """Unmodified hekan.inference.model_forward_he on c1 with the composite
    comparator, its stage evaluation routed to the engine:
    within 1e-4 of the reference's decrypted outputs, with the reference's
    rotation / ct_mult / pt_mult / depth counts."""
    monkeypatch.setattr(hekan.bspline, "poly_comp", eng_approx.poly_comp)
    g = np.load(os.path.join(GOLD, "c1.npz"))
    _, model, X = configs.workload("c1")
    cfg = hekan.inference.PipelineConfig()
    be = _backend(kind, 36)
    B = 2
    outs = []
    for x in X[:B]:
        out, stats = hekan.inference.model_forward_he(model, hekan.inference.encrypt_input(x, model, be), cfg)
        assert out.level == 0
        outs.append(be.decrypt(out)[0])
    assert np.abs(np.array(outs) - g["mirrored"][:B, 0]).max() < 1e-4
    ref = json.loads(str(g["counts"]))["lazy"]
    for mine, theirs in zip(stats.per_layer, ref):
        assert (mine.rotations, mine.ct_mults, mine.pt_mults, mine.depth_consumed) == (
            theirs["rotations"], theirs["ct_mults"], theirs["pt_mults"], theirs["depth_consumed"])


@pytest.mark.parametrize("kind", ENGINES)
def test_integration_factory_bench_compare(kind, monkeypatch):
    """INTEGRATION.md §2's factory branch: the reference's bench_compare builds
    its backend through make_backend; pointing that at the engine runs the
    reference harness on it with the simulator's counts."""
    from paper_2409_07751_b200 import backend as eng_backend
    model = hekan.model.random_model([2, 3], g=3, k=2, seed=1)
    depth = hekan.inference.plan_model(model, hekan.inference.PipelineConfig(comparator_mode="exact",
                                                                             path="naive")).total
    p = make_params(8, depth)
    bcfg = hekan.backend.BackendConfig(slot_count=p.slot_count, depth_budget=depth)
    cfgs = [hekan.inference.PipelineConfig(comparator_mode="exact", path=path, backend=bcfg, label="t")
            for path in ("lazy", "naive")]
    X = np.random.default_rng(3).uniform(-0.9, 0.9, (2, 2))
    ref_rows = hekan.inference.bench_compare(model, X, cfgs)
    monkeypatch.setattr(hekan.inference, "make_backend",
                        lambda c: eng_backend.make_backend(c, p, engine=_engine(kind, p), seed=0))
    rows = hekan.inference.bench_compare(model, X, cfgs)
    strip = lambda r: {k: v for k, v in r.items() if k != "wall_ms"}  # noqa: E731
    assert [strip(r) for r in rows] == [strip(r) for r in ref_rows]
