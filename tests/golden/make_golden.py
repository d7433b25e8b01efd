"""Generate golden fixtures by running the REFERENCE (`hekan`, imported from
/root/reference/pkg/src) in this container. Commit the outputs; the GPU box
has no /root/reference.

Outputs
  tests/golden/composite_sign.json  reference comparator stages (pins the fitter)
  tests/golden/c1.npz      c1 model (built with the reference's classes from the
                           same seeded draws), inputs, reference mirrored and
                           exact outputs, per-layer logical op counts
  tests/golden/c3.npz, c4.npz  first samples of c3 / c4 with reference outputs
  tests/golden/c5.npz      c5 [3072,128,10] first 2 samples; the reference's HE
                           program needs 33792 packed slots, so its counts are
                           taken at slot_count 65536 (N = 2^17)
  tests/golden/small.npz   small multi-layer random models + inputs + outputs
  tests/golden/backend.json known-answer vectors of the backend contract
  tests/golden/counts.json  per-layer op counts of the reference program for c3 / c4

Run:  python tests/golden/make_golden.py [c5|counts]
"""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
import hekan  # noqa: E402
from hekan import approx as ra, bspline as rb, inference as ri, model as rm  # noqa: E402
from hekan.backend import BackendConfig, CleartextBackend  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
DATA = HERE


def comparator_json():
    cs = ra.build_composite_sign(7.0, 2.0 ** -10)
    doc = {"source": "hekan.approx.build_composite_sign (reference, approx.py:479-508)",
           "comparators": [{"alpha": 7.0, "target_eps": 2.0 ** -10,
                            "stages": [list(s.coeffs) for s in cs.stages],
                            "certified_max_error": cs.certified_max_error()}]}
    os.makedirs(DATA, exist_ok=True)
    with open(os.path.join(DATA, "composite_sign.json"), "w") as fh:
        json.dump(doc, fh, indent=1)
    return cs


def build_ref_model(dims, g, k, lo, hi, w_std, degree, calib, input_shape, seed=0, explicit_R=False,
                    ranges=None):
    """SURVEY §8(d) recipe through the reference's own classes."""
    rng = np.random.default_rng(seed)
    layers = []
    x = np.asarray(calib, dtype=float)
    for n_i, n_o in zip(dims, dims[1:]):
        grid = rb.GridMatrix.uniform(n_i, g, k, lo, hi)
        if explicit_R:
            R = 1.2 * max(float(np.max(np.abs(x))), float(np.max(np.abs(grid.entries))))
            grid = rb.GridMatrix.uniform(n_i, g, k, lo, hi, R=R)
        W_b = rng.normal(0.0, w_std, (n_o, n_i))
        S = rng.normal(0.0, w_std, (n_o, n_i, grid.n_basis))
        act = ra.estimate_range(x, x_min=float(np.min(x)), x_max=float(np.max(x)), factor=5.0)
        if ranges is not None:
            ranges.append((act.lo, act.hi))
        poly = ra.fit_weighted_ls(rm.silu, act, degree, w=ra.WeightScheme.from_moments(act.mu, act.sigma))
        layer = rm.KanLayer(W_b=W_b, S=S, grid=grid, silu_poly=poly, act_stats=(act.mu, act.sigma))
        layers.append(layer)
        x = np.stack([rm.layer_forward_plain(layer, row, mode="exact") for row in x])
    return rm.KanModel(layers=layers, input_shape=input_shape)


def counts_json(model, depth, path="lazy"):
    be = CleartextBackend(BackendConfig(slot_count=4096, depth_budget=depth))
    cfg = ri.PipelineConfig(path=path)
    x = np.zeros(model.n_in)
    ct = ri.encrypt_input(x, model, be)
    out, stats = ri.model_forward_he(model, ct, cfg)
    return [{"rotations": s.rotations, "ct_mults": s.ct_mults, "pt_mults": s.pt_mults,
             "adds": s.adds, "depth_consumed": s.depth_consumed} for s in stats.per_layer], out.level


def model_arrays(prefix, model):
    d = {}
    for i, layer in enumerate(model.layers):
        d[f"{prefix}L{i}_W_b"] = layer.W_b
        d[f"{prefix}L{i}_S"] = layer.S
        d[f"{prefix}L{i}_grid"] = layer.grid.entries
        d[f"{prefix}L{i}_R"] = np.array(layer.grid.R)
        d[f"{prefix}L{i}_silu"] = np.array(layer.silu_poly.coeffs)
    return d


def c5_fixture(cs):
    """c5 [3072,128,10] G=5 k=3 [-1,1], explicit R; 32 x per-channel-standardised
    U[0,1]^(32x32x3) in HWC raster; first 2 samples kept."""
    rng = np.random.default_rng(1)
    x = rng.uniform(0.0, 1.0, (32, 32, 32, 3))
    mu = x.mean(axis=(0, 1, 2), keepdims=True)
    sd = x.std(axis=(0, 1, 2), keepdims=True)
    X5 = ((x - mu) / sd).reshape(32, 3072)
    rg5 = []
    m5 = build_ref_model((3072, 128, 10), 5, 3, -1.0, 1.0, 0.02, 10, X5, (32, 32, 3), explicit_R=True,
                         ranges=rg5)
    Xs = X5[:2]
    plan = ri.plan_model(m5, ri.PipelineConfig())
    be = CleartextBackend(BackendConfig(slot_count=65536, depth_budget=plan.total))
    out, stats = ri.model_forward_he(m5, ri.encrypt_input(Xs[0], m5, be), ri.PipelineConfig())
    counts = [{"rotations": st.rotations, "ct_mults": st.ct_mults, "pt_mults": st.pt_mults,
               "adds": st.adds, "depth_consumed": st.depth_consumed} for st in stats.per_layer]
    np.savez_compressed(os.path.join(HERE, "c5.npz"), X=Xs,
                        mirrored=np.stack([rm.model_forward_plain(m5, x, "mirrored", cs, "lazy") for x in Xs]),
                        exact=np.stack([rm.model_forward_plain(m5, x, "exact") for x in Xs]),
                        he_cleartext_s65536=np.asarray(out.slots[:10]),
                        ranges=np.array(rg5), plan_total=np.array(plan.total),
                        counts=np.array(json.dumps(counts)))
    print("c5 plan depth", plan.total, "counts", counts)


def counts_fixture():
    """Per-layer logical op counts of the reference's own program for c3 and c4
    (tests/golden/counts.json), run on CleartextBackend at a slot count that
    holds each config's packing."""
    out = {}
    rng = np.random.default_rng(1)
    X3 = np.clip(rng.normal(0.0, 1.0, (4096, 4)), -2.0, 2.0)
    m3 = build_ref_model((4, 8, 4, 1), 10, 3, -2.0, 2.0, 0.1, 63, X3, (1, 1, 4))
    rng = np.random.default_rng(1)
    X4 = rng.uniform(0.0, 1.0, (64, 784))
    m4 = build_ref_model((784, 64, 10), 5, 3, -1.0, 1.0, 0.05, 10, X4, (28, 28, 1), explicit_R=True)
    for name, model, slots in (("c3", m3, 4096), ("c4", m4, 2 ** 15)):
        plan = ri.plan_model(model, ri.PipelineConfig())
        be = CleartextBackend(BackendConfig(slot_count=slots, depth_budget=plan.total))
        _, stats = ri.model_forward_he(model, ri.encrypt_input(np.zeros(model.n_in), model, be),
                                       ri.PipelineConfig())
        out[name] = [{"rotations": s.rotations, "ct_mults": s.ct_mults, "pt_mults": s.pt_mults,
                      "adds": s.adds, "depth_consumed": s.depth_consumed} for s in stats.per_layer]
    with open(os.path.join(HERE, "counts.json"), "w") as fh:
        json.dump({"source": "hekan.inference.model_forward_he on CleartextBackend (tests/golden/make_golden.py counts)",
                   **out}, fh, indent=1)
    print(out)


def main():
    cs = comparator_json()
    if sys.argv[1:] == ["c5"]:
        c5_fixture(cs)
        return
    if sys.argv[1:] == ["counts"]:
        counts_fixture()
        return
    # ---- c1
    rng = np.random.default_rng(1)
    X = rng.uniform(-1.0, 1.0, (128, 2))
    model = build_ref_model((2, 5, 1), 5, 3, -1.0, 1.0, 0.1, 10, X, (1, 1, 2))
    mirrored = np.stack([rm.model_forward_plain(model, x, "mirrored", cs, "lazy") for x in X])
    exact = np.stack([rm.model_forward_plain(model, x, "exact") for x in X])
    naive = np.stack([rm.model_forward_plain(model, x, "mirrored", cs, "naive") for x in X])
    counts, _ = counts_json(model, 36)
    counts_naive, _ = counts_json(model, 38, "naive")
    plan = ri.plan_model(model, ri.PipelineConfig())
    np.savez_compressed(os.path.join(HERE, "c1.npz"), X=X, mirrored=mirrored, exact=exact,
                        mirrored_naive=naive, plan_total=np.array(plan.total),
                        counts=np.array(json.dumps({"lazy": counts, "naive": counts_naive})),
                        **model_arrays("", model))
    # ---- c3 [4,8,4,1] G=10 k=3 on [-2,2], deg-63 SiLU; 4096 clip(N(0,1)) inputs (first 8 kept)
    rng = np.random.default_rng(1)
    X3 = np.clip(rng.normal(0.0, 1.0, (4096, 4)), -2.0, 2.0)
    rg3 = []
    m3 = build_ref_model((4, 8, 4, 1), 10, 3, -2.0, 2.0, 0.1, 63, X3, (1, 1, 4), ranges=rg3)
    Xs = X3[:8]
    np.savez_compressed(os.path.join(HERE, "c3.npz"), X=Xs,
                        mirrored=np.stack([rm.model_forward_plain(m3, x, "mirrored", cs, "lazy") for x in Xs]),
                        exact=np.stack([rm.model_forward_plain(m3, x, "exact") for x in Xs]),
                        ranges=np.array(rg3), plan_total=np.array(ri.plan_model(m3, ri.PipelineConfig()).total),
                        **model_arrays("", m3))
    # ---- c4 [784,64,10] G=5 k=3 [-1,1], explicit R; 64 x U[0,1]^784 (first 4 kept)
    rng = np.random.default_rng(1)
    X4 = rng.uniform(0.0, 1.0, (64, 784))
    rg4 = []
    m4 = build_ref_model((784, 64, 10), 5, 3, -1.0, 1.0, 0.05, 10, X4, (28, 28, 1), explicit_R=True, ranges=rg4)
    Xs = X4[:4]
    np.savez_compressed(os.path.join(HERE, "c4.npz"), X=Xs,
                        mirrored=np.stack([rm.model_forward_plain(m4, x, "mirrored", cs, "lazy") for x in Xs]),
                        exact=np.stack([rm.model_forward_plain(m4, x, "exact") for x in Xs]),
                        ranges=np.array(rg4), plan_total=np.array(ri.plan_model(m4, ri.PipelineConfig()).total))
    # ---- small random models (reference random_model, uniform weights)
    small = {}
    for idx, (dims, g, k) in enumerate([((3, 4), 3, 2), ((4, 3, 2), 4, 3), ((2, 6, 3), 5, 1)]):
        mdl = rm.random_model(list(dims), g=g, k=k, seed=idx)
        xr = np.random.default_rng(100 + idx).uniform(-0.9, 0.9, (4, dims[0]))
        small[f"m{idx}_X"] = xr
        small[f"m{idx}_mirrored"] = np.stack([rm.model_forward_plain(mdl, x, "mirrored", cs, "lazy") for x in xr])
        small[f"m{idx}_exact"] = np.stack([rm.model_forward_plain(mdl, x, "exact") for x in xr])
        small[f"m{idx}_mirrored_exactcmp"] = np.stack(
            [rm.model_forward_plain(mdl, x, "mirrored", rb.EXACT_COMPARATOR, "lazy") for x in xr])
        small[f"m{idx}_dims"] = np.array(dims)
        small[f"m{idx}_gk"] = np.array([g, k])
        c, _ = counts_json(mdl, ri.plan_model(mdl, ri.PipelineConfig()).total)
        small[f"m{idx}_counts"] = np.array(json.dumps(c))
        small.update(model_arrays(f"m{idx}_", mdl))
    np.savez_compressed(os.path.join(HERE, "small.npz"), **small)
    # ---- backend known answers (test_backend.py style, via the reference itself)
    be = CleartextBackend(BackendConfig(slot_count=8, depth_budget=20))
    a = be.encrypt([1.0, 2.0, 3.0])
    kat = {"rotate_left_1": be.rotate(a, 1).slots.tolist(),
           "rotate_right_1": be.rotate(a, -1).slots.tolist(),
           "bsgs_2x2": ri.bsgs_matvec(np.array([[1.0, 2.0], [3.0, 4.0]]),
                                      be.encrypt([5.0, 6.0])).slots[:2].tolist(),
           "pack_example": rb.repeat_pack(be.encrypt([1.0, 2.0]), 1, 1, 2).ct.slots.tolist(),
           "comparator": {"certified_max_error": cs.certified_max_error(), "depth": cs.depth(),
                          "degrees": [s.degree for s in cs.stages]}}
    with open(os.path.join(HERE, "backend.json"), "w") as fh:
        json.dump(kat, fh, indent=1)
    c5_fixture(cs)
    print("wrote fixtures; c1 plan depth", plan.total, "counts", counts)


if __name__ == "__main__":
    main()
