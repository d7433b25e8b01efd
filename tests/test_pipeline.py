"""Encrypted KAN pipeline on the RNS-CKKS oracle vs the reference's outputs.

Golden values come from running the reference (`hekan`) here
(tests/golden/make_golden.py). The encrypted program is size-independent, so
the ring degree is the smallest that holds every packing (N = 2^8 for c1);
the same program runs at N = 2^16 on the GPU (tests/test_gpu_pipeline.py).
Tolerance: decrypted outputs within 1e-4 of the reference's decrypted
(mirrored) outputs (BASELINE north star); op counts equal the reference's for
rotations / ct_mults / pt_mults / depth; adds differ by exactly the Chebyshev
power-recurrence adds (2 per T_{2^k} power, 32 per layer).
"""

import json
import os

import numpy as np
import pytest

from oracle.engine import OracleEngine
from paper_2409_07751_b200 import configs, inference as inf, model as mdl
from paper_2409_07751_b200.approx import Polynomial, build_composite_sign
from paper_2409_07751_b200.backend import BackendConfig, HeBackend
from paper_2409_07751_b200.bspline import EXACT_COMPARATOR, GridMatrix
from paper_2409_07751_b200.errors import DepthBudgetInfeasible
from paper_2409_07751_b200.params import make_params

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOL = 1e-4


def oracle_backend(depth, log_n=8, seed=0):
    p = make_params(log_n, depth)
    return HeBackend(BackendConfig(slot_count=p.slot_count, depth_budget=depth, rng_seed=seed), p, seed=seed,
                     engine=OracleEngine(p))


def model_from_golden(g, prefix, dims, input_shape=None):
    layers = []
    for i in range(len(dims) - 1):
        grid_e = g[f"{prefix}L{i}_grid"]
        gk = g.get(f"{prefix}gk") if hasattr(g, "get") else None
        S = g[f"{prefix}L{i}_S"]
        n_basis = S.shape[2]
        k = (grid_e.shape[1] - 1 - n_basis)
        gg = n_basis - k
        grid = GridMatrix(grid_e, gg, k, float(g[f"{prefix}L{i}_R"]))
        layers.append(mdl.KanLayer(W_b=g[f"{prefix}L{i}_W_b"], S=S, grid=grid,
                                   silu_poly=Polynomial(tuple(g[f"{prefix}L{i}_silu"]))))
    return mdl.KanModel(layers=layers, input_shape=input_shape or (1, 1, dims[0]))


def test_c1_builder_reproduces_reference_model():
    g = np.load(os.path.join(GOLD, "c1.npz"))
    cfg, model, X = configs.workload("c1")
    assert np.array_equal(X, g["X"])
    for i, layer in enumerate(model.layers):
        assert np.array_equal(layer.W_b, g[f"L{i}_W_b"])
        assert np.array_equal(layer.S, g[f"L{i}_S"])
        assert np.array_equal(layer.grid.entries, g[f"L{i}_grid"])
        assert np.array_equal(np.array(layer.silu_poly.coeffs), g[f"L{i}_silu"])


def test_mirrored_plaintext_is_reference_bit_exact():
    """model.py's mirrored forward (reference schedule) equals the reference's."""
    g = np.load(os.path.join(GOLD, "c1.npz"))
    _, model, X = configs.workload("c1")
    cs = build_composite_sign()
    mine = np.stack([mdl.model_forward_plain(model, x, "mirrored", cs, "lazy") for x in X])
    assert np.array_equal(mine, g["mirrored"])
    exact = np.stack([mdl.model_forward_plain(model, x, "exact") for x in X])
    assert np.array_equal(exact, g["exact"])


def test_comparator_data_matches_reference():
    kat = json.load(open(os.path.join(GOLD, "backend.json")))["comparator"]
    cs = build_composite_sign()
    assert [s.degree for s in cs.stages] == kat["degrees"] and cs.depth() == kat["depth"]
    assert cs.certified_max_error() == pytest.approx(kat["certified_max_error"], rel=1e-12)
    # the Chebyshev re-expansion computes the same polynomial: exact against
    # rational evaluation of the stored monomials; the reference's own float
    # monomial schedule carries ~1e-6 rounding (|coef| up to 6e10)
    from fractions import Fraction as F

    def exact(y):
        s = F(float(y))
        for st in cs.stages:
            s = sum(F(c) * s ** i for i, c in enumerate(st.coeffs))
        return float(s)

    ys = np.linspace(-1, 1, 33)
    ex = np.array([exact(y) for y in ys])
    assert np.abs(cs.apply_cheb_clear(ys) - ex).max() < 1e-12
    y = np.linspace(-1, 1, 20001)
    assert np.abs(cs.apply_cheb_clear(y) - cs.apply_clear(y)).max() < 2e-5
    assert max(np.abs(c.coeffs).max() for c in cs.cheb) < 2.0


def test_c1_encrypted_matches_reference():
    g = np.load(os.path.join(GOLD, "c1.npz"))
    _, model, X = configs.workload("c1")
    B = 6
    be = oracle_backend(36)
    out, stats = inf.model_forward_he(model, inf.encrypt_input(X[:B], model, be), inf.PipelineConfig())
    assert out.level == 0
    dec = be.decrypt(out)[:, :1]
    assert np.abs(dec - g["mirrored"][:B]).max() < TOL
    ref = json.loads(str(g["counts"]))["lazy"]
    for mine, theirs in zip(stats.per_layer, ref):
        assert (mine.rotations, mine.ct_mults, mine.pt_mults, mine.depth_consumed) == (
            theirs["rotations"], theirs["ct_mults"], theirs["pt_mults"], theirs["depth_consumed"])
        assert mine.adds == theirs["adds"] + 32


def test_c1_naive_path_matches_reference():
    g = np.load(os.path.join(GOLD, "c1.npz"))
    _, model, X = configs.workload("c1")
    be = oracle_backend(38)
    cfg = inf.PipelineConfig(path="naive")
    out, _ = inf.model_forward_he(model, inf.encrypt_input(X[:2], model, be), cfg)
    assert np.abs(be.decrypt(out)[:, :1] - g["mirrored_naive"][:2]).max() < TOL


@pytest.mark.parametrize("idx", [0, 1, 2])
def test_small_random_models(idx):
    g = np.load(os.path.join(GOLD, "small.npz"))
    dims = tuple(int(v) for v in g[f"m{idx}_dims"])
    model = model_from_golden(g, f"m{idx}_", dims)
    X = g[f"m{idx}_X"]
    depth = inf.plan_model(model, inf.PipelineConfig()).total
    be = oracle_backend(depth, log_n=9)
    out, stats = inf.model_forward_he(model, inf.encrypt_input(X, model, be), inf.PipelineConfig())
    assert np.abs(be.decrypt(out)[:, :dims[-1]] - g[f"m{idx}_mirrored"]).max() < TOL
    ref = json.loads(str(g[f"m{idx}_counts"]))
    for mine, theirs in zip(stats.per_layer, ref):
        assert (mine.rotations, mine.ct_mults, mine.pt_mults) == (
            theirs["rotations"], theirs["ct_mults"], theirs["pt_mults"])


def test_exact_comparator_debug_path():
    g = np.load(os.path.join(GOLD, "small.npz"))
    dims = tuple(int(v) for v in g["m0_dims"])
    model = model_from_golden(g, "m0_", dims)
    cfg = inf.PipelineConfig(comparator_mode="exact")
    depth = inf.plan_model(model, cfg).total
    be = oracle_backend(depth, log_n=9)
    out, _ = inf.model_forward_he(model, inf.encrypt_input(g["m0_X"], model, be), cfg)
    # exact mode has a step discontinuity at knots; inputs are off-knot
    assert np.abs(be.decrypt(out)[:, :dims[-1]] - g["m0_mirrored_exactcmp"]).max() < TOL


def test_planner_rejects_reference_default_budget():
    _, model, _ = configs.workload("c1")
    plan = inf.plan_model(model, inf.PipelineConfig())
    assert plan.total == 36
    with pytest.raises(DepthBudgetInfeasible):
        inf.check_depth_budget(model, inf.PipelineConfig(), 20)


def test_bench_compare_rows():
    _, model, X = configs.workload("c1")
    p = make_params(8, 38)
    fac = lambda bc: HeBackend(bc, p, engine=OracleEngine(p), seed=0)  # noqa: E731
    bc = BackendConfig(slot_count=p.slot_count, depth_budget=38)
    rows = inf.bench_compare(model, X[:2], [inf.PipelineConfig(path="lazy", backend=bc, label="c1"),
                                           inf.PipelineConfig(path="naive", backend=bc, label="c1")],
                             backend_factory=fac)
    assert rows[0]["rotations"] == 2 * 41 and rows[0]["speedup_vs_naive_counts"] > 1.0


def test_c3_builder_reproduces_reference_model():
    g = np.load(os.path.join(GOLD, "c3.npz"))
    _, model, X = configs.workload("c3", batch=8)
    assert np.array_equal(X, g["X"])
    for i, layer in enumerate(model.layers):
        assert np.array_equal(layer.W_b, g[f"L{i}_W_b"]) and np.array_equal(layer.S, g[f"L{i}_S"])
        assert np.array_equal(np.array(layer.silu_poly.coeffs), g[f"L{i}_silu"])
        assert tuple(layer.fit_range) == tuple(g["ranges"][i])
    assert inf.plan_model(model, inf.PipelineConfig()).total == int(g["plan_total"]) == 54


def test_c3_chebyshev_silu_is_the_same_polynomial():
    """Degree-63 fits on narrow ranges (|monomial coef| up to 9e31) run in the
    Chebyshev basis of their fit interval: exact vs rational evaluation."""
    from fractions import Fraction as F
    from paper_2409_07751_b200.approx import eval_silu_cheb_clear, silu_uses_cheb
    _, model, _ = configs.workload("c3", batch=8)
    for layer in model.layers:
        assert silu_uses_cheb(layer)
        lo, hi = layer.fit_range
        xs = np.linspace(lo, hi, 9)
        ex = np.array([float(sum(F(c) * F(float(v)) ** k for k, c in enumerate(layer.silu_poly.coeffs)))
                       for v in xs])
        assert np.abs(eval_silu_cheb_clear(layer, xs) - ex).max() < 1e-12


def test_c3_encrypted_matches_reference():
    g = np.load(os.path.join(GOLD, "c3.npz"))
    _, model, X = configs.workload("c3", batch=8)
    be = oracle_backend(54, log_n=9)
    B = 2
    out, stats = inf.model_forward_he(model, inf.encrypt_input(X[:B], model, be), inf.PipelineConfig())
    assert out.level == 0
    dec = be.decrypt(out)[:, :1]
    cs = inf.PipelineConfig().comparator()
    twin = np.stack([mdl.model_forward_plain(model, x, "mirrored", cs, "lazy", schedule="cheb") for x in X[:B]])
    assert np.abs(dec - twin).max() < TOL
    assert np.abs(dec - g["mirrored"][:B]).max() < TOL


def test_silu_program_choice():
    """c1/c4 keep the reference program (identical counts); c3 is Chebyshev."""
    from paper_2409_07751_b200.approx import silu_uses_cheb
    for name in ("c1", "c4"):
        _, model, _ = configs.workload(name, batch=1)
        assert not any(silu_uses_cheb(layer) for layer in model.layers), name


def test_c4_model_matches_reference_ranges():
    g = np.load(os.path.join(GOLD, "c4.npz"))
    _, model, X = configs.workload("c4", batch=4)
    assert np.array_equal(X, g["X"])
    for i, layer in enumerate(model.layers):
        assert tuple(layer.fit_range) == tuple(g["ranges"][i])
    cs = build_composite_sign()
    mine = np.stack([mdl.model_forward_plain(model, x, "mirrored", cs, "lazy") for x in X[:1]])
    assert np.array_equal(mine, g["mirrored"][:1])


def test_c3_counts_vs_reference():
    """c3's per-layer op counts against the reference program's (golden
    counts.json, made by running hekan). Rotations, ct-mults and depth are
    identical; the Chebyshev evaluators add exactly: +32 adds (comparator
    powers T_2k = 2 T_k^2 - 1, two adds each), +10 adds (degree-63 SiLU powers)
    and +1 pt-mult / +1 add (the SiLU's affine map onto [-1, 1])."""
    ref = json.load(open(os.path.join(GOLD, "counts.json")))["c3"]
    _, model, X = configs.workload("c3", batch=1)
    depth = inf.plan_model(model, inf.PipelineConfig()).total
    be = oracle_backend(depth, log_n=9)
    out, stats = inf.model_forward_he(model, inf.encrypt_input(X, model, be), inf.PipelineConfig())
    assert out.level == 0
    for mine, theirs in zip(stats.per_layer, ref):
        assert (mine.rotations, mine.ct_mults, mine.depth_consumed) == (
            theirs["rotations"], theirs["ct_mults"], theirs["depth_consumed"])
        assert mine.pt_mults == theirs["pt_mults"] + 1
        assert mine.adds == theirs["adds"] + 32 + 10 + 1


def _one_layer_model(n_i, n_o, seed=3):
    rng = np.random.default_rng(seed)
    grid = GridMatrix.uniform(n_i, 5, 3, -1.0, 1.0)
    silu = Polynomial((0.0, 0.5, 0.2, 0.0, -0.01))  # a fixed well-conditioned activation polynomial
    layer = mdl.KanLayer(W_b=rng.normal(0, 0.3, (n_o, n_i)), S=rng.normal(0, 0.3, (n_o, n_i, grid.n_basis)),
                         grid=grid, silu_poly=silu)
    return mdl.KanModel(layers=[layer], input_shape=(1, 1, n_i))


def test_spline_branch_tiles_when_packing_overflows():
    """Beyond the reference (PackingOverflow, bspline.py:151-154): a layer whose
    repeat packing exceeds the slot vector runs its B-spline branch tiled over
    several ciphertexts. n_i = 6 at 64 slots needs two tiles of 3 features
    (3 * 16 <= 64 < 6 * 16); the decrypted output equals the same model run
    untiled at 128 slots and the plaintext twin of the engine's schedule, with
    the untiled depth."""
    model = _one_layer_model(6, 2)
    layer = model.layers[0]
    pcfg = inf.PipelineConfig()
    depth = inf.plan_model(model, pcfg).total
    assert inf.spline_tiles(layer, 64) == 2 and inf.spline_tiles(layer, 128) == 1
    X = np.random.default_rng(5).uniform(-0.9, 0.9, (2, 6))
    small, big = oracle_backend(depth, log_n=7), oracle_backend(depth, log_n=8)
    o_small, st_small = inf.model_forward_he(model, inf.encrypt_input(X, model, small), pcfg)
    o_big, st_big = inf.model_forward_he(model, inf.encrypt_input(X, model, big), pcfg)
    d_small, d_big = small.decrypt(o_small)[:, :2], big.decrypt(o_big)[:, :2]
    cs = build_composite_sign()
    twin = np.stack([mdl.model_forward_plain(model, x, "mirrored", cs, "lazy", schedule="cheb") for x in X])
    assert np.abs(d_small - d_big).max() < TOL
    assert np.abs(d_small - twin).max() < TOL
    assert st_small.total.depth_consumed == st_big.total.depth_consumed == depth
    # two tiles: twice the spline-branch products, one extra rotation to bring tile 1 forward
    assert st_small.total.ct_mults > st_big.total.ct_mults
    # the reference's own packing refuses this shape
    from paper_2409_07751_b200.errors import PackingOverflow
    from paper_2409_07751_b200.bspline import repeat_pack
    with pytest.raises(PackingOverflow):
        repeat_pack(inf.encrypt_input(X, model, small), layer.g, layer.k, layer.n_i)
