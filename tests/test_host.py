"""Host logic without a GPU: parameters, ABI exports, Chebyshev algebra,
multi-rank sharding (gloo, world size 2)."""

import ctypes as C
import math
import os
import re

import numpy as np
import pytest

from paper_2409_07751_b200 import _abi
from paper_2409_07751_b200.approx import _ArrayOps, _cheb_tree, _estrin, mono_to_cheb
from paper_2409_07751_b200.params import is_prime, kan_params, make_params, microbench_params

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_kan_params_chain():
    p = kan_params(36)
    two_n = 2 * p.n
    allp = list(p.q) + list(p.p)
    assert len(set(allp)) == len(allp)
    for q in allp:
        assert is_prime(q) and (q - 1) % two_n == 0 and 2 ** 44 < q < 2 ** 50
    for s in p.scales:
        assert abs(s / 2 ** 46 - 1) < 1e-6
    for lvl in range(1, p.depth + 1):  # ct x ct lands on the canonical scale
        assert p.scales[lvl] ** 2 / p.q[lvl] == pytest.approx(p.scales[lvl - 1], rel=1e-15)
        assert p.pt_mult_scale(lvl) * p.scales[lvl] / p.q[lvl] == pytest.approx(p.scales[lvl - 1], rel=1e-15)
    assert p.alpha == 13 and p.n_digits == 3 and len(p.p) == 13


def test_microbench_params():
    p = microbench_params()
    assert len(p.q) == 24 and len(p.p) == 8 and p.dnum == 3 and p.n == 1 << 16


def _declared():
    hdr = open(os.path.join(ROOT, "include", "hekan.h")).read()
    return set(re.findall(r"\b(hk_[a-z_0-9]+)\s*\(", hdr))


def test_header_matches_bindings():
    assert _declared() == set(_abi.SIGNATURES)


def test_product_library_exports_every_symbol():
    from paper_2409_07751_b200.build import LIB, build
    if not os.path.exists(LIB):
        build()
    lib = C.CDLL(LIB)  # loads without a GPU (no compute calls here)
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.hk_version() == 1


def test_oracle_library_exports_every_symbol():
    from oracle.engine import load_oracle
    lib = load_oracle()
    for name in _declared():
        assert hasattr(lib, name), name


def test_gpu_engine_fails_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2409_07751_b200.engine import GpuEngine
    with pytest.raises(RuntimeError):
        GpuEngine(make_params(4, 1))


@pytest.mark.parametrize("deg", [1, 2, 5, 10, 31, 63])
def test_cheb_tree_equals_monomial_and_counts(deg):
    rng = np.random.default_rng(deg)
    mono = rng.normal(0, 1, deg + 1)
    cheb = mono_to_cheb(mono)
    x = np.linspace(-1, 1, 101)
    a = _estrin(_ArrayOps(x), mono)
    b = _cheb_tree(_ArrayOps(x), cheb)
    assert np.abs(a - b).max() < 1e-9 * max(1.0, np.abs(mono).sum())

    class Count(_ArrayOps):
        def __init__(self, x):
            super().__init__(x)
            self.n = {"mul": 0, "mul_const": 0}

        def mul(self, a, b):
            self.n["mul"] += 1
            return a * b

        def mul_const(self, a, c):
            self.n["mul_const"] += 1
            return a * c

    ce, cc = Count(x), Count(x)
    _estrin(ce, mono)
    _cheb_tree(cc, cheb)
    assert ce.n == cc.n  # same multiplications => same depth and mult counts


def test_mono_to_cheb_scaled_exact():
    mono = [0.0, 1.5, 0.0, -0.25, 0.0, 0.125]
    c = mono_to_cheb(mono, h=2.0, out_scale=4.0)
    y = np.linspace(-1, 1, 11)
    x = 2.0 * y
    want = np.polynomial.polynomial.polyval(x, mono) / 4.0
    assert np.abs(np.polynomial.chebyshev.chebval(y, c) - want).max() < 1e-14


def _dist_worker(rank, world, port, q):
    """One CPU rank of a sharded c1 run (oracle engine, gloo): shared key seed,
    its block of the global batch, gather of the outputs to rank 0."""
    import torch.distributed as dist
    from oracle.engine import OracleEngine
    from paper_2409_07751_b200 import configs, distributed as D, inference as inf
    from paper_2409_07751_b200.backend import BackendConfig, HeBackend
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    seed = D.shared_seed(world, rank)
    _, model, X = configs.workload("c1", batch=4)
    p = make_params(8, 36)
    lo, _ = D.block_range(len(X), rank, world)
    be = HeBackend(BackendConfig(slot_count=p.slot_count, depth_budget=36), p, engine=OracleEngine(p), seed=seed,
                   sample_offset=lo)
    out, _ = inf.model_forward_he(model, inf.encrypt_input(D.shard_rows(X, rank, world), model, be),
                                  inf.PipelineConfig())
    full = D.gather_ciphertexts(be, out, world, rank)
    if rank == 0:
        q.put((seed, be.export_ct(full), be.decrypt(full)[:, :1]))
    dist.destroy_process_group()


def test_sharded_c1_gather_gloo_world2():
    """Two ranks, 2 samples each: the gathered level-0 ciphertext equals, limb
    for limb, the same 4 samples run by one process with the same seed."""
    import multiprocessing as mp
    import socket
    from oracle.engine import OracleEngine
    from paper_2409_07751_b200 import configs, inference as inf
    from paper_2409_07751_b200.backend import BackendConfig, HeBackend
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dist_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    seed, limbs, dec = q.get(timeout=600)
    for p in procs:
        p.join(timeout=60)
    _, model, X = configs.workload("c1", batch=4)
    p = make_params(8, 36)
    be = HeBackend(BackendConfig(slot_count=p.slot_count, depth_budget=36), p, engine=OracleEngine(p), seed=seed)
    out, _ = inf.model_forward_he(model, inf.encrypt_input(X, model, be), inf.PipelineConfig())
    assert np.array_equal(limbs, be.export_ct(out))
    gold = np.load(os.path.join(ROOT, "tests", "golden", "c1.npz"))["mirrored"][:4]
    assert np.abs(dec - gold).max() < 1e-4
