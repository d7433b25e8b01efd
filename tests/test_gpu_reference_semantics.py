"""The reference's backend / comparator / BSGS known answers, run through the
sm_100a engine at the reference's own default slot count (S = 32768, so
N = 2^16 — the ring the bench uses).

Each case restates a reference test at the HeBackend boundary
(/root/reference/pkg/tests/*, cited per test) and checks the GPU backend
directly, not through the oracle: decrypted slots against the reference's
semantics (np.roll(-t) rotations, min-level rule, scalar broadcast, zero
padding), exact logical counters, and the reference's error taxonomy.
Tolerance for decrypted values: 1e-6 absolute at depth <= 4 (CKKS noise at
Delta = 2^46 is ~1e-9; the bound leaves room for the level-0 limb).
"""

import json
import os

import numpy as np
import pytest

from paper_2409_07751_b200.backend import BackendConfig, PlainVector, make_backend
from paper_2409_07751_b200.errors import DepthExhausted, InputTooLong, LengthMismatch
from paper_2409_07751_b200.params import make_params

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
S = 32768
TOL = 1e-6


@pytest.fixture(scope="module")
def be(gpu_lib):
    p = make_params(16, 4)
    return make_backend(BackendConfig(slot_count=p.slot_count, depth_budget=4, rng_seed=3), params=p, seed=3)


def _vec(seed, n=S):
    return np.random.default_rng(seed).uniform(-1, 1, n)


def test_add_sub_and_padding(be):
    # test_backend.py:55-66 (add/sub), :164-171 (round trip, zero padding)
    x, y = _vec(1), _vec(2)
    a, b = be.encrypt(x), be.encrypt(y)
    assert np.abs(be.add(a, b).slots - (x + y)).max() < TOL
    assert np.abs(be.sub(a, b).slots - (x - y)).max() < TOL
    short = be.encrypt([0.5, -0.25, 0.125])
    out = be.decrypt(short)
    assert out.shape == (S,)
    assert np.abs(out[:3] - [0.5, -0.25, 0.125]).max() < TOL and np.abs(out[3:]).max() < TOL


def test_levels_and_depth_exhausted(be):
    # test_backend.py:68-95: ct x ct and ct x pt drop one level from the minimum
    a = be.encrypt(_vec(3))
    assert a.level == 4
    b = be.mul(a, a)
    assert b.level == 3 and be.add(a, b).level == 3
    c = be.mul(b, _vec(4))
    assert c.level == 2
    d = be.mul(be.mul(c, 0.5), 2.0)
    assert d.level == 0
    with pytest.raises(DepthExhausted):
        be.mul(d, d)
    with pytest.raises(DepthExhausted):
        be.mul(d, 3.0)


def test_scalar_broadcast(be):
    # test_backend.py:97-100: a Python scalar acts on every slot
    x = _vec(5)
    a = be.encrypt(x)
    assert np.abs(be.add(a, 0.75).slots - (x + 0.75)).max() < TOL
    assert np.abs(be.mul(a, -1.5).slots - (-1.5 * x)).max() < TOL
    assert np.abs(be.sub(a, 2.0).slots - (x - 2.0)).max() < TOL


def test_rotations_left_right_zero_bound_group_law(be):
    # test_backend.py:125-160
    x = _vec(6)
    a = be.encrypt(x)
    for t in (1, -1, 7, -300, 4096, S - 1):
        assert np.abs(be.rotate(a, t).slots - np.roll(x, -t)).max() < TOL, t
    c0 = be.counter.rotations
    assert be.rotate(a, 0) is a and be.counter.rotations == c0  # free and uncounted
    for t in (S, -S, S + 1):
        with pytest.raises(ValueError):
            be.rotate(a, t)
    # group law: rot(rot(a, s), t) == rot(a, s + t)
    two = be.rotate(be.rotate(a, 3), 5)
    one = be.rotate(a, 8)
    assert np.abs(two.slots - one.slots).max() < TOL


def test_reference_known_answers_at_full_slot_count(be):
    # tests/golden/backend.json: the reference's CleartextBackend at slot_count 8,
    # re-stated at S = 32768 (same op, longer zero padding)
    kat = json.load(open(os.path.join(GOLD, "backend.json")))
    a = be.encrypt([1.0, 2.0, 3.0])
    left = be.rotate(a, 1).slots
    assert np.abs(left[:2] - kat["rotate_left_1"][:2]).max() < TOL and abs(left[-1] - 1.0) < TOL
    right = be.rotate(a, -1).slots
    assert np.abs(right[:4] - kat["rotate_right_1"][:4]).max() < TOL
    from paper_2409_07751_b200.bspline import repeat_pack
    from paper_2409_07751_b200.inference import bsgs_matvec
    out = bsgs_matvec(np.array([[1.0, 2.0], [3.0, 4.0]]), be.encrypt([5.0, 6.0]))
    assert np.abs(out.slots[:2] - kat["bsgs_2x2"]).max() < 1e-5  # (17, 39), test_inference.py:70-73
    packed = repeat_pack(be.encrypt([1.0, 2.0]), 1, 1, 2).ct.slots  # test_bspline.py:62-65
    assert np.abs(packed[:8] - kat["pack_example"]).max() < TOL


def test_counters_and_errors(be):
    # test_backend.py:198-253 (exact logical counters), error taxonomy backend.py:192-261
    be.reset_counter()
    a = be.encrypt([1.0, 2.0])
    be.add(a, a)
    be.sub(a, 1.0)
    be.mul(a, a)
    be.mul(a, np.ones(S))
    be.rotate(a, 1)
    c = be.counter
    assert (c.adds, c.subs, c.ct_mults, c.pt_mults, c.rotations, c.max_depth_consumed) == (1, 1, 1, 1, 1, 1)
    with pytest.raises(InputTooLong):
        be.encrypt(np.ones(S + 1))
    with pytest.raises(ValueError):
        be.encrypt([1.0], level=5)
    with pytest.raises(ValueError):
        be.slotwise("div", a, a)
    with pytest.raises(LengthMismatch):
        be.slotwise("mul_ct", a, np.ones(S))
    with pytest.raises(LengthMismatch):
        be.add(a, PlainVector(np.ones(16)))


def test_comparator_tie_and_antisymmetry(gpu_lib):
    # test_approx.py:247-274: comparator >, <, tie = 1/2, antisymmetry, on the
    # composite sign (depth 11) under real encryption at N = 2^16
    from paper_2409_07751_b200.approx import build_composite_sign, poly_comp
    cs = build_composite_sign(7.0, 2.0 ** -10)
    depth = cs.depth() + 2
    p = make_params(16, depth)
    be = make_backend(BackendConfig(slot_count=p.slot_count, depth_budget=depth, rng_seed=4), params=p, seed=4)
    xs = np.array([0.5, -0.5, 0.0, 0.25, -0.25, 0.9, -0.9, 0.01])
    ys = np.array([0.0, 0.0, 0.0, -0.25, 0.25, 0.1, -0.1, 0.0])
    ca, cb = be.encrypt(xs), be.encrypt(ys)
    gt = poly_comp(ca, cb, cs).slots[:8]
    lt = poly_comp(cb, ca, cs).slots[:8]
    expect = np.array([1.0, 0.0, 0.5, 1.0, 0.0, 1.0, 0.0, 1.0])
    assert np.abs(gt - expect).max() < 1e-2  # composite-sign certified error 7.3e-4 plus CKKS noise
    assert abs(gt[2] - 0.5) < 1e-4  # tie: odd stages map 0 to 0 (up to noise times the slope at 0)
    assert np.abs(gt + lt - 1.0).max() < 1e-4  # antisymmetry
