"""The reference CLI (`hekan`, /root/reference/pkg/src/hekan/cli.py) on this engine.

    python -m paper_2409_07751_b200.cli [--engine gpu|simulator] [--ckks CKKS.json]
                                        <hekan command and options>

Every command, option, output and exit code is the reference's own
(`hekan.cli.build_parser`, `main`'s exception-to-exit-code mapping). With
`--engine gpu` (the default) the encrypted commands — `infer --mode he` and
`compare` (cli.py:193-227, :284-312) — run on the RNS-CKKS engine instead of
the float simulator, all input rows as one batched ciphertext; `--engine
simulator` is the unmodified reference CLI.

The CKKS parameters travel in a sibling config because the reference's
`BackendConfig.from_json` rejects unknown keys (backend.py:54-57): `--ckks`
takes a JSON object (path or inline) with optional `dnum` (default 3) and
`seed` (default: OS randomness). The ring is N = 2 * slot_count of the
reference backend config; the modulus chain has depth_budget levels.
"""

from __future__ import annotations

import importlib
import json
import os
import sys

import numpy as np

from ._ref import hekan  # noqa: F401  (locates the reference package)

_hc = importlib.import_module("hekan.cli")


def _ckks_doc(src) -> dict:
    if not src:
        return {}
    doc = json.loads(src) if src.lstrip().startswith("{") else json.load(open(src))
    unknown = set(doc) - {"dnum", "seed"}
    if unknown:
        raise ValueError(f"unknown --ckks keys: {sorted(unknown)}")
    return doc


def ckks_params(bcfg, ckks: dict):
    from .params import kan_params
    log_n = int(np.log2(bcfg.slot_count)) + 1
    return kan_params(bcfg.depth_budget, log_n=log_n, dnum=int(ckks.get("dnum", 3)))


def _engine_backend(engine: str, bcfg, ckks: dict):
    from .backend import HeBackend
    from .engine import GpuEngine
    p = ckks_params(bcfg, ckks)
    return HeBackend(bcfg, p, engine=GpuEngine(p), seed=ckks.get("seed"))


def _he_rows(args, engine: str, ckks: dict):
    """Encrypted forward of every input row as one batched ciphertext."""
    from . import inference as inf
    mdl = _hc.load_model(args.model)
    rows = _hc._load_inputs(args.input, mdl.n_in)
    bcfg = _hc._load_backend(args)
    cfg = inf.PipelineConfig(comparator_mode=args.comparator, path=args.path, backend=bcfg,
                             check_range=args.check_range)
    plan = inf.check_depth_budget(mdl, cfg, bcfg.depth_budget)
    be = _engine_backend(engine, bcfg, ckks)
    out, stats = inf.model_forward_he(mdl, inf.encrypt_input(rows.reshape(len(rows), -1), mdl, be), cfg)
    dec = np.atleast_2d(be.decrypt(out))[:, : mdl.n_out]
    return mdl, rows, cfg, plan, dec, stats


def cmd_infer(args, engine: str, ckks: dict) -> int:
    """`hekan infer` (cli.py:193-227); --mode he on the engine."""
    if args.mode != "he":
        return _hc.cmd_infer(args)
    _, _, _, plan, dec, stats = _he_rows(args, engine, ckks)
    print("depth plan:")
    print(plan.describe())
    result = {"mode": args.mode, "outputs": dec.tolist(), "stats": [stats.to_json()] * len(dec),
              "engine": engine}
    for out in result["outputs"]:
        print("output:", np.array2string(np.asarray(out), precision=6))
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(result, fh)
    return _hc.EXIT_OK


def cmd_compare(args, engine: str, ckks: dict) -> int:
    """`hekan compare` (cli.py:284-312) with the encrypted column from the engine."""
    mdl, rows, cfg, _, dec, _ = _he_rows(args, engine, ckks)
    comparator = cfg.comparator()
    report = []
    for row, he in zip(rows, dec):
        exact = _hc.model_forward_plain(mdl, row, mode="exact")
        mirrored = _hc.model_forward_plain(mdl, row, mode="mirrored", comparator=comparator, path=args.path)
        report.append({"exact": exact.tolist(), "mirrored": mirrored.tolist(), "he": he.tolist(),
                       "max_dev_he_vs_mirrored": float(np.max(np.abs(he - mirrored))),
                       "max_dev_he_vs_exact": float(np.max(np.abs(he - exact)))})
    for i, entry in enumerate(report):
        print(f"input {i}: |he - mirrored| = {entry['max_dev_he_vs_mirrored']:.3e}  "
              f"|he - exact| = {entry['max_dev_he_vs_exact']:.3e}")
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(report, fh)
    return _hc.EXIT_OK


def _pop(argv: list, flag: str, default):
    if flag in argv:
        i = argv.index(flag)
        val = argv[i + 1]
        del argv[i:i + 2]
        return val
    return default


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    engine = _pop(argv, "--engine", os.environ.get("HEKAN_ENGINE", "gpu"))
    ckks_src = _pop(argv, "--ckks", None)
    if engine == "simulator":
        return _hc.main(argv)
    if engine != "gpu":
        print(f"unknown --engine {engine!r}", file=sys.stderr)
        return _hc.EXIT_USAGE
    args = _hc.build_parser().parse_args(argv)
    try:
        ckks = _ckks_doc(ckks_src)
        if args.command == "infer":
            return cmd_infer(args, engine, ckks)
        if args.command == "compare":
            return cmd_compare(args, engine, ckks)
        return args.func(args)  # fitting and count benches: the reference's own commands
    except ValueError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return _hc.EXIT_USAGE
    except _hc.DepthBudgetInfeasible as exc:
        print(f"depth budget infeasible:\n{exc}", file=sys.stderr)
        return _hc.EXIT_BUDGET
    except (_hc.ShapeMismatch, _hc.SchemaMismatch) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return _hc.EXIT_USAGE
    except (_hc.IllConditioned, _hc.RemezNonConvergence, _hc.SingularSystem) as exc:
        print(f"numerical failure: {exc}", file=sys.stderr)
        return _hc.EXIT_NUMERIC
    except _hc.HeKanError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return _hc.EXIT_NUMERIC
    except FileNotFoundError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return _hc.EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
