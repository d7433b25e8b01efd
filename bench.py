#!/usr/bin/env python
"""Encrypted-KAN throughput on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl product|reference]
                  [--config c1|c3|c4|c5] [--batch B] [--chunk C] [--log-n 16]

A step = one encrypted forward pass (`model_forward_he`) of the config's KAN
over one batch of B ciphertexts per GPU (one sample per ciphertext, as
`encrypt_input`, /root/reference/pkg/src/hekan/inference.py:115-124) on the
sm_100a RNS-CKKS engine, N = 2^16, L = 36 (the planner total),
plus the gather of every rank's level-0 outputs to rank 0 (the path's only
collective; a no-op at N = 1). Inputs are resident in HBM when the
timed region starts; each ciphertext batch is 4.7 GB, far above the 126 MB
L2, so no flush is needed between steps. `e2e` times the public API from host
memory: encrypt_input (pinned host slots -> HBM) + model_forward_he + gather
+ decrypt on rank 0 (-> host).

Multi-GPU: `--gpus N` without a torchrun environment re-launches itself under
torch.distributed.run (one rank per GPU, NCCL). The global batch is N x B
samples in contiguous blocks; every rank uses one key seed (drawn on rank 0,
broadcast) and encrypts with its global sample offset (weak scaling, no
data-path collective but the output gather); barrier + max over ranks of the
device time; value = all ranks' inferences / s.

`--impl reference` times the CPU implementation of the same path on the
host's cores: the oracle port (oracle/libckks_oracle.so, the identical RNS-CKKS
program, OpenMP over all host threads), each step ONE complete inference of
one ciphertext, keys generated once before the warm-up. It also reports the
reference package's own float simulator (`hekan.model_forward_he` on
`CleartextBackend`, one process per core), which performs no
cryptography.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0
METRIC = "encrypted KAN inferences/sec"


def _peaks():
    try:
        with open(PEAKS_PATH) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def _profile(name: str) -> dict:
    """Newest committed ncu summary of that name (profiles/r2_*, else r1_*)."""
    for rnd in ("r2", "r1"):
        path = os.path.join(ROOT, "profiles", f"{rnd}_{name}.json")
        if os.path.exists(path):
            with open(path) as fh:
                d = json.load(fh)
            d["_path"] = os.path.relpath(path, ROOT)
            return d
    return {}


# ---------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md recipe)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.gpu)],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sms, maxes, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as fh:
            for line in fh:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sms.append(float(parts[1]))
                    maxes.append(float(parts[2]))
                except ValueError:
                    continue
                for nm, val in zip(names, parts[5:9]):
                    if val.lower().startswith("active"):
                        reasons.add(nm)
        os.unlink(self.path)
        loaded = [s for s in sms if s > 500] or sms
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(maxes) if maxes else None,
                "reasons": sorted(reasons), "samples": len(sms)}


# ---------------------------------------------------------------------------
# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------
def spawn_ranks(n: int) -> int:
    """--gpus N outside torchrun: re-launch this command with one rank per GPU."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(world, value: float, device) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def per_gpu_batch(args, cfg) -> int:
    # c3's 4096-sample workload would be 220 GiB of fresh ciphertexts: the bench
    # keeps a resident sample of 64 per GPU (the model is calibrated on all 4096)
    return args.batch or (cfg.batch if cfg.batch <= 128 else 64)


def workload_line(args, cfg, B, chunk, depth, params, world) -> dict:
    return {"workload": f"{args.config}: KAN {list(cfg.dims)} G={cfg.g} k={cfg.k}, {B} ciphertexts/GPU in "
                        f"chunks of {chunk}, RNS-CKKS N=2^{args.log_n} L={depth} dnum={params.dnum} "
                        f"alpha={params.alpha}",
            "global_batch": B * world, "parallelism": f"dp{world} (ciphertext sharding, output gather to rank 0)",
            "l2": f"inputs {B * 2 * (depth + 1) * params.n * 8 / 1e9:.1f} GB/GPU >> 126 MB L2 (no flush needed)",
            "security": (f"log2(PQ) = {params.log_pq:.0f} bits at N=2^{args.log_n}"
                         + (" (above the ~1772-bit 128-bit-security bound for N=2^16; N=2^17 --log-n 17 "
                            "is the 128-bit-secure ring for this depth)" if args.log_n == 16 else ""))}


# ---------------------------------------------------------------------------
# product arm
# ---------------------------------------------------------------------------
def run_product(args):
    import torch

    from paper_2409_07751_b200 import configs, distributed as D, inference as inf
    from paper_2409_07751_b200.backend import BackendConfig, make_backend
    from paper_2409_07751_b200.params import kan_params

    world, rank, local = dist_setup()
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    cfg = configs.CONFIGS[args.config]
    B = per_gpu_batch(args, cfg)
    n_global = B * world
    _, model, X_all = configs.workload(args.config, batch=n_global)
    pcfg = inf.PipelineConfig()
    depth = inf.plan_model(model, pcfg).total
    params = kan_params(depth, log_n=args.log_n, dnum=args.dnum)
    seed = D.shared_seed(world, rank, device)   # identical keys on every rank
    lo, hi = D.block_range(n_global, rank, world)
    be = make_backend(BackendConfig(slot_count=params.slot_count, depth_budget=depth), params=params,
                      device=local, seed=seed, sample_offset=lo)
    eng = be.engine
    X = X_all[lo:hi]
    chunk = min(args.chunk or B, B)
    cts_in = [inf.encrypt_input(X[i:i + chunk], model, be) for i in range(0, B, chunk)]

    def step(cts):
        gathered = []
        for ct in cts:
            out, st = inf.model_forward_he(model, ct, pcfg)
            gathered.append(D.gather_ciphertexts(be, out, world, rank))
            del out
        return gathered, st

    outs, stats = step(cts_in)     # Galois keys + plaintext caches
    err, n_checked = None, 0
    if rank == 0:                  # decrypted values vs the reference (any ring degree)
        dec = np.concatenate([be.decrypt(o) for o in outs])[:, :model.n_out]
        gpath = os.path.join(ROOT, "tests", "golden", f"{args.config}.npz")
        if os.path.exists(gpath):
            gold = np.load(gpath)["mirrored"]
            # gathered order: chunk c of rank r holds global samples r*B + c*chunk ...
            order = np.concatenate([np.arange(r * B + c, r * B + min(c + chunk, B))
                                    for c in range(0, B, chunk) for r in range(world)])
            glob = np.empty_like(dec)
            glob[order] = dec
            n_checked = min(n_global, gold.shape[0])
            err = float(np.max(np.abs(glob[:n_checked] - gold[:n_checked])))
    del outs
    for _ in range(args.warmup):
        step(cts_in)
    torch.cuda.synchronize(device)

    stream = torch.cuda.current_stream(device)
    clocks = ClockSampler(local) if rank == 0 else None
    if clocks:
        clocks.start()
    barrier(world)
    torch.cuda.synchronize(device)
    l0 = eng.lib.hk_launch_count(eng.ctx)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step(cts_in)
    ev1.record(stream)
    torch.cuda.synchronize(device)
    barrier(world)
    launches = int(eng.lib.hk_launch_count(eng.ctx) - l0)
    ms = max_over_ranks(world, ev0.elapsed_time(ev1), device) / args.steps
    clk = clocks.stop() if clocks else None

    # ---- e2e through the public API from pinned host memory (device-resident
    # inputs freed first; one untimed warm-up so the allocator pool is steady)
    del cts_in
    host_np = torch.from_numpy(np.ascontiguousarray(X)).pin_memory().numpy()

    def e2e_step():
        for i in range(0, B, chunk):
            ct = inf.encrypt_input(host_np[i:i + chunk], model, be)
            out, _ = inf.model_forward_he(model, ct, pcfg)
            full = D.gather_ciphertexts(be, out, world, rank)
            if rank == 0:
                be.decrypt(full)
            del ct, out, full

    e2e_step()
    barrier(world)
    torch.cuda.synchronize(device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(max(1, args.steps)):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize(device)
    e2e_ms = max_over_ranks(world, e0.elapsed_time(e1), device) / max(1, args.steps)
    S = params.slot_count
    h2d = n_global * S * 8                      # zero-padded slot rows uploaded by encrypt
    d2h = n_global * S * 8                      # decrypted slot vectors (rank 0)
    gather_bytes = (world - 1) * B * 2 * params.n * 8   # level-0 outputs moved to rank 0

    torch.cuda.empty_cache()
    roof = kernel_rooflines(be, params, chunk, stream) if rank == 0 else None
    if rank != 0:
        return
    value = n_global / (ms / 1e3)
    hbm, hbm_kind = _peaks()
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "inferences/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64 (RNS residues mod <=50-bit primes)",
        "data": "synthetic (seeded PCG64, SURVEY §8d)",
        "config": workload_line(args, cfg, B, chunk, depth, params, world),
        "e2e": {"value": round(n_global / (e2e_ms / 1e3), 4), "unit": "inferences/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "gather_bytes_per_step": gather_bytes,
                "api": "encrypt_input + model_forward_he + gather to rank 0 + decrypt, host slots in/out"},
        "gpu_launches": launches,
        "clocks": clk,
        "max_abs_err_vs_reference_mirrored": err,
        "err_samples": n_checked,
        "counts_per_inference": stats.to_json()["total"],
    }
    if roof:
        line["roofline"] = dict(roof["ntt"], peak_kind=hbm_kind)
        line["kernels"] = roof
    if not args.no_c2:
        del be, eng
        torch.cuda.empty_cache()
        line["c2_microbench"] = c2_microbench(local)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args)
    print(json.dumps(line))


def _binding(prof: dict) -> dict:
    keys = ("fp64_pipe_pct", "alu_pipe_pct", "fma_pipe_pct", "l1tex_throughput_pct", "issue_active_pct", "warps_active_pct",
            "traffic_over_algorithmic")
    return {k: prof[k] for k in keys if k in prof} | ({"source": prof["_path"]} if prof else {})


def kernel_rooflines(be, params, B, stream, reps: int = 5) -> dict:
    """CUDA-event timings of the two dominant primitives at the bench's launch
    shapes, against the HBM roofline on SURVEY §8(d)'s algorithmic bytes. Both
    are compute-bound on this engine (FP64-pipe butterflies, tensor-core basis
    conversion with a CUDA-core epilogue), so `bound` names that pipe and `pipe` carries its ncu
    utilisation; `frac` stays the HBM fraction."""
    import torch
    eng = be.engine
    hbm, _ = _peaks()
    N = params.n
    out = {}
    nl = params.depth + 1
    buf = eng.alloc_u64(nl * B * N)
    buf.zero_()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    eng.call("hk_ntt_fwd", eng.addr(buf), 0, nl, B)
    torch.cuda.synchronize()
    ev[0].record(stream)
    for _ in range(reps):
        eng.call("hk_ntt_fwd", eng.addr(buf), 0, nl, B)
    ev[1].record(stream)
    torch.cuda.synchronize()
    t = ev[0].elapsed_time(ev[1]) / reps / 1e3
    alg = 2.0 * nl * B * N * 8
    ach = alg / t / 1e9
    tr = _profile("ntt_traffic")
    traffic = (tr["dram_read_bytes"] + tr["dram_write_bytes"]) if tr.get("algorithmic_bytes") == alg else None
    out["ntt"] = {"bound": "fp64", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                  "frac": round(ach / hbm, 4), "traffic": traffic, "pipe": _binding(tr),
                  "kernel": f"hk_ntt_fwd -> ntt16::fwd_kernel (4-CTA cluster per polynomial, FP64-pipe "
                            f"butterflies), {nl} limbs x {B} polys",
                  "algorithmic_bytes": alg, "ms": round(t * 1e3, 3)}
    del buf
    # key switch via one rotation at the top level (ModUp + key IP + ModDown)
    ct = be.encrypt(np.zeros((B, params.slot_count)))
    be.rotate(ct, 1)
    torch.cuda.synchronize()
    ev[0].record(stream)
    for _ in range(reps):
        be.rotate(ct, 1)
    ev[1].record(stream)
    torch.cuda.synchronize()
    t = ev[0].elapsed_time(ev[1]) / reps / 1e3
    l = params.depth
    nd = l // params.alpha + 1
    alg = B * 4 * (l + 1) * N * 8 + 2 * nd * (l + 1 + len(params.p)) * N * 8
    ach = alg / t / 1e9
    rt = _profile("rotate_traffic")
    ks_traffic = (rt["dram_read_bytes"] + rt["dram_write_bytes"]) if rt.get("algorithmic_bytes") == alg else None
    out["keyswitch"] = {"bound": "int+fp64", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                        "frac": round(ach / hbm, 4), "traffic": ks_traffic, "pipe": _binding(rt),
                        "kernel": f"hk_rotate (ModUp + key IP + ModDown) level {l}, {B} cts",
                        "algorithmic_bytes": alg, "ms": round(t * 1e3, 3)}
    return out


def c2_microbench(device: int, n_ct: int = 256, reps: int = 3) -> dict:
    """BASELINE config 2: 256 ciphertexts with uniform random limbs,
    N=2^16, 24 ~50-bit limbs, dnum=3 (alpha = 8 special primes); CUDA-event
    times of NTT / iNTT (both polynomials), HMult+relin+rescale and rotate by
    +-2^j (j = 0..14, 30 Galois keys), each against SURVEY's algorithmic bytes."""
    import ctypes as C

    import torch
    from paper_2409_07751_b200 import _abi
    from paper_2409_07751_b200.backend import galois_element
    from paper_2409_07751_b200.engine import GpuEngine
    from paper_2409_07751_b200.params import microbench_params

    hbm, _ = _peaks()
    p = microbench_params()
    eng = GpuEngine(p, device=device)
    stream = torch.cuda.current_stream(device)
    N, n, l = p.n, len(p.q), len(p.q) - 1
    alpha = len(p.p)
    ct = eng.alloc_u64(2 * n * n_ct * N).view(2, n, n_ct * N)
    for i, q in enumerate(p.q):  # uniform residues in [0, q_i)
        ct[:, i].random_(0, int(q))
    eng.call("hk_keygen", _abi.seed_words(os.urandom(32)))
    steps = [s * (1 << j) for j in range(15) for s in (1, -1)]
    gal = [galois_element(t, p.slot_count) for t in steps]
    eng.call("hk_add_galois_keys", _abi.seed_words(os.urandom(32)), eng.u32_array(gal), len(gal))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    def timed(fn, k=reps):
        fn()
        torch.cuda.synchronize(device)
        ev[0].record(stream)
        for _ in range(k):
            fn()
        ev[1].record(stream)
        torch.cuda.synchronize(device)
        return ev[0].elapsed_time(ev[1]) / k / 1e3

    def entry(alg, t, what, bound="int+fp64"):
        ach = alg / t / 1e9
        return {"bound": bound, "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s", "frac": round(ach / hbm, 4),
                "ms": round(t * 1e3, 3), "algorithmic_bytes": alg, "kernel": what}

    out = {"workload": f"c2: {n_ct} ciphertexts x 2 polys x {n} limbs (~50-bit), N=2^16, dnum=3, alpha={alpha}, "
                       "uniform random limbs"}
    base = ct.data_ptr()
    half = n * n_ct * N * 8
    ntt_b = 2.0 * n_ct * 2 * n * N * 8
    t = timed(lambda: [eng.call("hk_ntt_fwd", base + q * half, 0, n, n_ct) for q in (0, 1)])
    out["ntt"] = entry(ntt_b, t, "hk_ntt_fwd, both polynomials", "fp64")
    t = timed(lambda: [eng.call("hk_ntt_inv", base + q * half, 0, n, n_ct) for q in (0, 1)])
    out["intt"] = entry(ntt_b, t, "hk_ntt_inv, both polynomials", "fp64")
    dst = eng.alloc_u64(2 * n * n_ct * N)
    key_b = 2 * p.dnum * (n + alpha) * N * 8
    t = timed(lambda: eng.call("hk_mul", base, l, base, l, eng.addr(dst), n_ct))
    out["hmult_relin_rescale"] = entry(n_ct * (4 * n + 2 * (n - 1)) * N * 8 + key_b, t, "hk_mul (tensor, relin, rescale)")
    del dst
    rdst = eng.alloc_u64(2 * n * n_ct * N)
    t = timed(lambda: [eng.call("hk_rotate", base, l, C.c_uint32(g), eng.addr(rdst), n_ct) for g in gal], k=1)
    t /= len(gal)
    out["rotate"] = entry(n_ct * 4 * n * N * 8 + key_b, t, "hk_rotate, mean over +-2^j, j=0..14")
    out["gpu_launches_total"] = int(eng.lib.hk_launch_count(eng.ctx))
    del rdst, ct, eng
    torch.cuda.empty_cache()
    return out




# ---------------------------------------------------------------------------
# CPU legs: the oracle port (like-for-like HE) and the reference's float simulator
# ---------------------------------------------------------------------------
def _cores() -> int:
    return len(os.sched_getaffinity(0))


class OracleInference:
    """One complete inference of one ciphertext on the oracle port (the same
    RNS-CKKS program, OpenMP over all host threads). Keys and plaintext caches
    are made once, by an untimed first inference, before any timed step."""

    def __init__(self, args):
        from oracle.engine import OracleEngine
        from paper_2409_07751_b200 import configs, inference as inf
        from paper_2409_07751_b200.backend import BackendConfig, HeBackend
        from paper_2409_07751_b200.params import kan_params
        self.inf = inf
        _, self.model, X = configs.workload(args.config, batch=1)
        self.pcfg = inf.PipelineConfig()
        depth = inf.plan_model(self.model, self.pcfg).total
        self.params = kan_params(depth, log_n=args.log_n, dnum=args.dnum)
        t = time.perf_counter()
        self.be = HeBackend(BackendConfig(slot_count=self.params.slot_count, depth_budget=depth), self.params,
                            engine=OracleEngine(self.params))
        self.x = X
        self.run()                       # keys + caches (untimed)
        self.setup_s = time.perf_counter() - t

    def run(self) -> float:
        t = time.perf_counter()
        ct = self.inf.encrypt_input(self.x, self.model, self.be)
        out, _ = self.inf.model_forward_he(self.model, ct, self.pcfg)
        self.be.decrypt(out)
        return time.perf_counter() - t


def cpu_baseline(args) -> dict:
    """Oracle port, all host threads: one measured c1 inference (after the
    untimed key-generation inference)."""
    o = OracleInference(args)
    el = o.run()
    cores = _cores()
    return {"value": round(1.0 / el, 6), "unit": "inferences/s", "cores": cores, "kind": "port",
            "sample": (f"oracle/libckks_oracle.so (C, Barrett/Shoup, OpenMP {cores} threads): one complete "
                       f"{args.config} inference of one ciphertext at N=2^{args.log_n} "
                       f"(encrypt + model_forward_he + decrypt) in {el:.1f} s; keys and plaintext caches "
                       f"made by an untimed first inference ({o.setup_s:.1f} s)")}


def _sim_worker(cfg_name, seconds, start_evt, q):
    os.environ["OMP_NUM_THREADS"] = "1"
    from paper_2409_07751_b200 import configs
    from paper_2409_07751_b200._ref import hekan
    hb, hi = hekan.backend, hekan.inference
    _, model, X = configs.workload(cfg_name)
    pcfg = hi.PipelineConfig()
    depth = hi.plan_model(model, pcfg).total
    S = 2 ** 16 if cfg_name == "c5" else 2 ** 15
    be = hb.CleartextBackend(hb.BackendConfig(slot_count=S, depth_budget=depth))
    hi.model_forward_he(model, hi.encrypt_input(X[0], model, be), pcfg)  # comparator fit, caches
    start_evt.wait()
    n, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        hi.model_forward_he(model, hi.encrypt_input(X[n % len(X)], model, be), pcfg)
        n += 1
    q.put((n, time.perf_counter() - t0))


def float_simulator(args, seconds: float = 10.0) -> dict:
    """the reference's own path, `hekan.model_forward_he` on
    `CleartextBackend` (a float64 slot simulator, no cryptography), one process
    per host core over independent inferences, OMP_NUM_THREADS=1."""
    import multiprocessing as mp
    cores = _cores()
    ctx = mp.get_context("spawn")
    q, start = ctx.Queue(), ctx.Event()
    procs = [ctx.Process(target=_sim_worker, args=(args.config, seconds, start, q)) for _ in range(cores)]
    for p in procs:
        p.start()
    time.sleep(1.0)
    start.set()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    rate = sum(n / t for n, t in res)
    return {"value": round(rate, 3), "unit": "inferences/s", "cores": cores, "kind": "reference float simulator",
            "sample": f"hekan.model_forward_he on CleartextBackend (float64 slots, NO cryptography), "
                      f"{args.config}, composite comparator, {cores} processes x {seconds:.0f} s, "
                      f"{sum(n for n, _ in res)} inferences"}


def run_reference(args):
    """--impl reference: the CPU path on the host's cores, rank 0 only. Each step
    is one complete inference of one ciphertext on the oracle port."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if int(os.environ.get("RANK", "0")) != 0:
        return
    from paper_2409_07751_b200 import configs, inference as inf
    o = OracleInference(args)
    for _ in range(args.warmup):
        o.run()
    times = [o.run() for _ in range(args.steps)]
    total = sum(times)
    v = args.steps / total
    cores = _cores()
    cfg = configs.CONFIGS[args.config]
    B = per_gpu_batch(args, cfg)
    line = {"metric": METRIC, "value": round(v, 6), "unit": "inferences/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * total / args.steps, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64 (RNS residues)",
            "data": "synthetic (seeded PCG64, SURVEY §8d)", "impl": "reference",
            "config": dict(workload_line(args, cfg, B, min(args.chunk or B, B),
                                         o.params.depth, o.params, world),
                           parallelism=f"cpu (OpenMP {cores} threads), one ciphertext per step"),
            "cpu_baseline": {"value": round(v, 6), "unit": "inferences/s", "cores": cores, "kind": "port",
                             "sample": f"oracle/libckks_oracle.so, each step one complete {args.config} inference "
                                       f"of one ciphertext (encrypt + model_forward_he + decrypt); step times "
                                       f"{min(times):.2f}-{max(times):.2f} s; keys made once before the warm-up "
                                       f"({o.setup_s:.1f} s)"},
            "e2e": {"value": round(v, 6), "unit": "inferences/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    if not args.no_float_sim:
        line["float_simulator"] = float_simulator(args)
    print(json.dumps(line))


def main():
    os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("product", "reference"), default="product")
    ap.add_argument("--config", default="c1")
    ap.add_argument("--batch", type=int, default=0, help="ciphertexts per GPU")
    ap.add_argument("--dnum", type=int, default=3, help="key-switching digits over the full chain")
    ap.add_argument("--chunk", type=int, default=None,
                    help="ciphertexts per batched launch (default: the whole batch; 32 for c4, 16 for c5)")
    ap.add_argument("--log-n", type=int, default=None,
                    help="ring degree (default 16: c5's 33792 packed slots run as two feature tiles; "
                         "17 runs it untiled and is the 128-bit-secure ring for depth 36)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-float-sim", action="store_true")
    ap.add_argument("--no-c2", action="store_true", help="skip the config-2 primitive microbench")
    args = ap.parse_args()
    if args.log_n is None:
        args.log_n = 16
    if args.chunk is None:
        # c1 and c3 run their whole batch per launch; c4 / c5 hold 80 / 157 hoisted
        # BSGS baby steps at once, which bounds them to 32 at N = 2^16 and 8 at N = 2^17
        if args.log_n > 16:
            args.chunk = 8 if args.config == "c5" else 32
        else:
            args.chunk = {"c4": 32, "c5": 16}.get(args.config, 128)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_product(args)


if __name__ == "__main__":
    main()
