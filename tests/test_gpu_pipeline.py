"""Encrypted KAN on the sm_100a engine: bit-exact vs the oracle running the
same program, and within 1e-4 of the reference's decrypted outputs at the
benchmark ring degree N = 2^16 (size-independent properties at full size)."""

import json
import os

import numpy as np
import pytest

from paper_2409_07751_b200 import configs, inference as inf
from paper_2409_07751_b200.backend import BackendConfig, HeBackend
from paper_2409_07751_b200.params import kan_params, make_params

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gpu(p, depth, seed=0):
    from paper_2409_07751_b200.engine import GpuEngine
    return HeBackend(BackendConfig(slot_count=p.slot_count, depth_budget=depth, rng_seed=seed), p, seed=seed,
                     engine=GpuEngine(p))


def test_c1_pipeline_bitexact_vs_oracle(gpu_lib):
    from oracle.engine import OracleEngine
    _, model, X = configs.workload("c1")
    p = make_params(8, 36)
    bc = BackendConfig(slot_count=p.slot_count, depth_budget=36)
    g, o = _gpu(p, 36), HeBackend(bc, p, engine=OracleEngine(p), seed=0)
    cfg = inf.PipelineConfig()
    og, sg = inf.model_forward_he(model, inf.encrypt_input(X[:5], model, g), cfg)
    oo, so = inf.model_forward_he(model, inf.encrypt_input(X[:5], model, o), cfg)
    assert np.array_equal(g.export_ct(og), o.export_ct(oo))
    assert sg.to_json()["total"]["rotations"] == so.to_json()["total"]["rotations"]
    gold = np.load(os.path.join(GOLD, "c1.npz"))["mirrored"][:5]
    assert np.abs(g.decrypt(og)[:, :1] - gold).max() < 1e-4


def test_small_models_bitexact_vs_oracle(gpu_lib):
    from oracle.engine import OracleEngine
    from tests.test_pipeline import model_from_golden
    gz = np.load(os.path.join(GOLD, "small.npz"))
    for idx in range(3):
        dims = tuple(int(v) for v in gz[f"m{idx}_dims"])
        model = model_from_golden(gz, f"m{idx}_", dims)
        depth = inf.plan_model(model, inf.PipelineConfig()).total
        p = make_params(9, depth)
        bc = BackendConfig(slot_count=p.slot_count, depth_budget=depth)
        g, o = _gpu(p, depth), HeBackend(bc, p, engine=OracleEngine(p), seed=0)
        X = gz[f"m{idx}_X"]
        og, _ = inf.model_forward_he(model, inf.encrypt_input(X, model, g), inf.PipelineConfig())
        oo, _ = inf.model_forward_he(model, inf.encrypt_input(X, model, o), inf.PipelineConfig())
        assert np.array_equal(g.export_ct(og), o.export_ct(oo)), idx
        assert np.abs(g.decrypt(og)[:, :dims[-1]] - gz[f"m{idx}_mirrored"]).max() < 1e-4


def test_c1_full_ring_degree_matches_reference(gpu_lib):
    g_ = np.load(os.path.join(GOLD, "c1.npz"))
    _, model, X = configs.workload("c1")
    p = kan_params(36)
    be = _gpu(p, 36)
    B = 16
    out, stats = inf.model_forward_he(model, inf.encrypt_input(X[:B], model, be), inf.PipelineConfig())
    assert out.level == 0
    dec = be.decrypt(out)[:, :1]
    assert np.abs(dec - g_["mirrored"][:B]).max() < 1e-4
    ref = json.loads(str(g_["counts"]))["lazy"]
    for s, r in zip(stats.per_layer, ref):  # the reference's counts; +32 adds: Chebyshev comparator powers
        assert (s.rotations, s.ct_mults, s.pt_mults, s.depth_consumed) == (
            r["rotations"], r["ct_mults"], r["pt_mults"], r["depth_consumed"])
        assert s.adds == r["adds"] + 32


def test_full_size_properties(gpu_lib):
    """N = 2^16, 37 limbs: rotation group law, linearity, exact level rule."""
    p = kan_params(36)
    be = _gpu(p, 36)
    S = p.slot_count
    rng = np.random.default_rng(5)
    x, y = rng.uniform(-1, 1, (2, S)), rng.uniform(-1, 1, (2, S))
    a, b = be.encrypt(x), be.encrypt(y)
    r1 = be.rotate(be.rotate(a, 7), 1 << 10)
    r2 = be.rotate(a, 7 + (1 << 10))
    assert np.abs(r1.slots - r2.slots).max() < 1e-6
    assert np.abs(r1.slots - np.roll(x, -(7 + (1 << 10)), axis=1)).max() < 1e-6
    lin = be.sub(be.add(be.mul(a, 0.5), be.mul(b, 0.25)), be.mul(be.add(a, b), 0.25))
    assert np.abs(lin.slots - (0.25 * x)).max() < 1e-6
    m = be.mul(a, b)
    assert m.level == 35 and np.abs(m.slots - x * y).max() < 1e-6
    # deep chain to level 0 keeps precision
    c = a
    for _ in range(36):
        c = be.mul(c, 1.0)
    assert c.level == 0 and np.abs(c.slots - x).max() < 1e-5


def test_c3_pipeline_bitexact_vs_oracle(gpu_lib):
    from oracle.engine import OracleEngine
    _, model, X = configs.workload("c3", batch=8)
    p = make_params(9, 54)
    bc = BackendConfig(slot_count=p.slot_count, depth_budget=54)
    g, o = _gpu(p, 54), HeBackend(bc, p, engine=OracleEngine(p), seed=0)
    cfg = inf.PipelineConfig()
    og, _ = inf.model_forward_he(model, inf.encrypt_input(X[:2], model, g), cfg)
    oo, _ = inf.model_forward_he(model, inf.encrypt_input(X[:2], model, o), cfg)
    assert np.array_equal(g.export_ct(og), o.export_ct(oo))


def _twin(model, X):
    from paper_2409_07751_b200 import model as mdl
    cs = inf.PipelineConfig().comparator()
    return np.stack([mdl.model_forward_plain(model, x, "mirrored", cs, "lazy", schedule="cheb") for x in X])


def test_c3_full_ring_degree(gpu_lib):
    g_ = np.load(os.path.join(GOLD, "c3.npz"))
    _, model, X = configs.workload("c3", batch=8)
    be = _gpu(kan_params(54), 54)
    out, _ = inf.model_forward_he(model, inf.encrypt_input(X[:4], model, be), inf.PipelineConfig())
    dec = be.decrypt(out)[:, :1]
    assert np.abs(dec - _twin(model, X[:4])).max() < 1e-4
    assert np.abs(dec - g_["mirrored"][:4]).max() < 1e-4  # north_star tolerance vs the reference's decryption


def test_c4_full_ring_degree(gpu_lib):
    """[784,64,10]: 6272-diagonal BSGS, 80 hoisted baby steps, explicit R."""
    g_ = np.load(os.path.join(GOLD, "c4.npz"))
    _, model, X = configs.workload("c4", batch=4)
    be = _gpu(kan_params(36), 36)
    out, stats = inf.model_forward_he(model, inf.encrypt_input(X[:2], model, be), inf.PipelineConfig())
    dec = be.decrypt(out)[:, :10]
    twin = _twin(model, X[:2])
    err_twin = np.abs(dec - twin).max()
    err_ref = np.abs(dec - g_["mirrored"][:2]).max()
    print(f"c4: |dec - exact-arithmetic twin| = {err_twin:.3g}, |dec - reference mirrored| = {err_ref:.3g}")
    assert err_twin < 1e-4 and err_ref < 1e-4
    assert stats.to_json()["total"]["rotations"] == 287
    ref = json.load(open(os.path.join(GOLD, "counts.json")))["c4"]
    for s, r in zip(stats.per_layer, ref):  # the reference's counts; +32 adds: Chebyshev comparator powers
        assert (s.rotations, s.ct_mults, s.pt_mults, s.depth_consumed) == (
            r["rotations"], r["ct_mults"], r["pt_mults"], r["depth_consumed"])
        assert s.adds == r["adds"] + 32


def test_c5_ring_2e17(gpu_lib):
    """c5 [3072,128,10]: 33792 repeat-packed slots need S = 2^16, i.e. N = 2^17
    (the reference itself raises PackingOverflow at its 2^15 slots; its program
    runs at slot_count 65536, tests/golden/make_golden.py). Decrypted outputs vs
    the reference's mirrored forward and the exact-arithmetic twin, and the
    reference's per-layer op counts (Chebyshev basis: +32 adds per layer)."""
    g_ = np.load(os.path.join(GOLD, "c5.npz"))
    _, model, X = configs.workload("c5", batch=2)
    depth = int(g_["plan_total"])
    assert inf.plan_model(model, inf.PipelineConfig()).total == depth
    be = _gpu(kan_params(depth, log_n=17), depth)
    out, stats = inf.model_forward_he(model, inf.encrypt_input(X[:2], model, be), inf.PipelineConfig())
    dec = be.decrypt(out)[:, :10]
    err_twin = np.abs(dec - _twin(model, X[:2])).max()
    err_ref = np.abs(dec - g_["mirrored"][:2]).max()
    print(f"c5: |dec - twin| = {err_twin:.3g}, |dec - reference mirrored| = {err_ref:.3g}")
    assert err_twin < 1e-4 and err_ref < 1e-4
    ref = json.loads(str(g_["counts"]))
    for ours, theirs in zip(stats.per_layer, ref):
        assert ours.rotations == theirs["rotations"]
        assert ours.ct_mults == theirs["ct_mults"]
        assert ours.pt_mults == theirs["pt_mults"]
        assert ours.adds == theirs["adds"] + 32
        assert ours.depth_consumed == theirs["depth_consumed"]


def test_c5_tiled_2e16(gpu_lib):
    """c5 [3072,128,10] at N = 2^16 as BASELINE config 5 states it: 33792
    repeat-packed slots exceed the 32768 available (the reference raises
    PackingOverflow), so layer 1's B-spline branch runs as two tiles of 1536
    features (inference.spline_tiles). Decrypted outputs within 1e-4 of the
    reference's mirrored forward (golden, produced at 65536 slots) and of the
    plaintext twin; depth equals the reference plan; layer 1 spends the
    second tile's products and rotations on top of the reference counts."""
    g_ = np.load(os.path.join(GOLD, "c5.npz"))
    _, model, X = configs.workload("c5", batch=2)
    depth = int(g_["plan_total"])
    p = kan_params(depth)
    assert p.slot_count == 32768
    assert inf.spline_tiles(model.layers[0], p.slot_count) == 2
    assert inf.spline_tiles(model.layers[1], p.slot_count) == 1
    be = _gpu(p, depth)
    out, stats = inf.model_forward_he(model, inf.encrypt_input(X[:2], model, be), inf.PipelineConfig())
    dec = be.decrypt(out)[:, :10]
    err_twin = np.abs(dec - _twin(model, X[:2])).max()
    err_ref = np.abs(dec - g_["mirrored"][:2]).max()
    print(f"c5 tiled at N=2^16: |dec - twin| = {err_twin:.3g}, |dec - reference mirrored| = {err_ref:.3g}")
    assert err_twin < 1e-4 and err_ref < 1e-4
    ref = json.loads(str(g_["counts"]))
    assert [s.depth_consumed for s in stats.per_layer] == [r["depth_consumed"] for r in ref]
    assert stats.per_layer[0].ct_mults > ref[0]["ct_mults"]          # the second tile
    assert stats.per_layer[1].ct_mults == ref[1]["ct_mults"]          # layer 2 is untiled
    assert stats.per_layer[1].rotations == ref[1]["rotations"]
