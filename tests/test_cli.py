"""The reference CLI on the engine (paper_2409_07751_b200.cli): the
reference's own parser, outputs and exit codes, with `infer --mode he` and
`compare` running encrypted on the engine. CPU: the engine factory is
pointed at the test oracle; GPU (-m gpu): the sm_100a library."""

import json
import os

import numpy as np
import pytest

from paper_2409_07751_b200 import cli, configs
from paper_2409_07751_b200.model import save_model

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _files(tmp_path, depth=36, slots=128):
    _, model, X = configs.workload("c1", batch=3)
    mpath, xpath = tmp_path / "kan.json", tmp_path / "x.csv"
    save_model(model, mpath)
    np.savetxt(xpath, X, delimiter=",")
    backend = json.dumps({"slot_count": slots, "depth_budget": depth, "noise_std": 0.0, "rng_seed": 0})
    return str(mpath), str(xpath), backend


def _oracle(monkeypatch):
    from oracle.engine import OracleEngine
    from paper_2409_07751_b200.backend import HeBackend

    def factory(engine, bcfg, ckks):
        p = cli.ckks_params(bcfg, ckks)
        return HeBackend(bcfg, p, engine=OracleEngine(p), seed=ckks.get("seed"))
    monkeypatch.setattr(cli, "_engine_backend", factory)


@pytest.mark.parametrize("kind", ["oracle", pytest.param("gpu", marks=pytest.mark.gpu)])
def test_cli_infer_and_compare(tmp_path, monkeypatch, kind):
    if kind == "oracle":
        _oracle(monkeypatch)
    else:
        import torch
        if not torch.cuda.is_available():
            pytest.skip("no CUDA device")
    m, x, backend = _files(tmp_path)
    out = tmp_path / "out.json"
    rc = cli.main(["--engine", "gpu", "--ckks", '{"seed": 5}', "infer", "--model", m, "--input", x,
                   "--backend", backend, "--out", str(out)])
    assert rc == 0
    res = json.load(open(out))
    gold = np.load(os.path.join(GOLD, "c1.npz"))["mirrored"][:3]
    assert np.abs(np.array(res["outputs"]) - gold).max() < 1e-4
    assert res["stats"][0]["total"]["rotations"] == 41
    rep = tmp_path / "cmp.json"
    assert cli.main(["--ckks", '{"seed": 5}', "compare", "--model", m, "--input", x, "--backend", backend,
                     "--out", str(rep)]) == 0
    assert max(r["max_dev_he_vs_mirrored"] for r in json.load(open(rep))) < 1e-4


def test_cli_exit_codes_are_the_reference_ones(tmp_path, monkeypatch):
    _oracle(monkeypatch)
    m, x, _ = _files(tmp_path)
    # the reference's default budget (20) cannot hold c1's 36 levels: exit 4
    assert cli.main(["infer", "--model", m, "--input", x]) == 4
    assert cli.main(["--ckks", '{"bogus": 1}', "infer", "--model", m, "--input", x]) == 2
    # the simulator path is the unmodified reference CLI
    m, x, backend = _files(tmp_path)
    assert cli.main(["--engine", "simulator", "infer", "--model", m, "--input", x, "--backend", backend,
                     "--mode", "plain-exact"]) == 0
