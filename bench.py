#!/usr/bin/env python
"""Encrypted-KAN throughput on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl product|reference]
                  [--config c1|c3|c4|c5] [--batch B] [--chunk C] [--log-n 16]

A step = one encrypted forward pass (`model_forward_he`) of the config's KAN
over one batch of B ciphertexts (one sample per ciphertext, as
`encrypt_input`, /root/reference/pkg/src/hekan/inference.py:115-124) on the
sm_100a RNS-CKKS engine, N = 2^16, depth 36 (L = 37 limbs: the planner total,
SURVEY §0.3). Inputs are already resident in HBM when the timed region starts;
each ciphertext batch is 4.7 GB, far larger than the 126 MB L2, so no explicit
flush is needed between steps. `e2e` times the public API end to end from host
memory: encrypt_input (host slots -> HBM) + model_forward_he + decrypt (-> host).

Multi-GPU (torchrun): every rank runs its own batch (weak scaling, the path
shards by ciphertext with no data-path collective); the barrier +
max-over-ranks device time gives the job time; value = total inferences / s.

`--impl reference` times the CPU implementation of the same path: the
oracle port (oracle/libckks_oracle.so, OpenMP over all host cores) running the
identical program on a bounded sample (a prefix of one inference's op stream).
"""

from __future__ import annotations

import argparse
import json
import os
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


def _peaks():
    try:
        with open(PEAKS_PATH) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


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
# distributed plumbing
# ---------------------------------------------------------------------------
def dist_setup(n_gpus: int):
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


# ---------------------------------------------------------------------------
# product arm
# ---------------------------------------------------------------------------
def run_product(args):
    import torch

    from paper_2409_07751_b200 import configs, inference as inf
    from paper_2409_07751_b200.backend import BackendConfig, make_backend
    from paper_2409_07751_b200.params import kan_params

    world, rank, local = dist_setup(args.gpus)
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    cfg, model, inputs = configs.workload(args.config)
    # c3's 4096-sample workload would be 220 GiB of fresh ciphertexts: the bench
    # keeps a resident sample of 64 per GPU (the model is still calibrated on all 4096)
    B = args.batch or (cfg.batch if cfg.batch <= 128 else 64)
    inputs = inputs[:B] if B <= inputs.shape[0] else np.resize(inputs, (B, inputs.shape[1]))
    pcfg = inf.PipelineConfig()
    depth = inf.plan_model(model, pcfg).total
    params = kan_params(depth, log_n=args.log_n, dnum=args.dnum)
    be = make_backend(BackendConfig(slot_count=params.slot_count, depth_budget=depth, rng_seed=rank),
                      params=params, device=local)
    eng = be.engine

    chunk = min(args.chunk or B, B)
    parts = [inputs[i:i + chunk] for i in range(0, B, chunk)]
    cts_in = [inf.encrypt_input(x, model, be) for x in parts]

    def step(cts):
        outs = []
        for ct in cts:
            o, st = inf.model_forward_he(model, ct, pcfg)
            outs.append(o)
        return outs, st

    outs, stats = step(cts_in)     # generates Galois keys + plaintext caches
    dec = np.concatenate([be.decrypt(o) for o in outs])[:, :model.n_out]
    del outs
    err = None
    gpath = os.path.join(ROOT, "tests", "golden", f"{args.config}.npz")
    if os.path.exists(gpath):  # decrypted values: comparable at any ring degree
        gold = np.load(gpath)["mirrored"]
        n = min(B, gold.shape[0])
        err = float(np.max(np.abs(dec[:n] - gold[:n])))
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

    # ---- e2e through the public API from host memory (device-resident inputs
    # freed first; untimed warm-up steps so the allocator pool is steady-state)
    del cts_in
    host_in = torch.from_numpy(np.ascontiguousarray(inputs)).pin_memory()
    host_np = host_in.numpy()

    def e2e_step():
        for i in range(0, B, chunk):
            ct = inf.encrypt_input(host_np[i:i + chunk], model, be)
            o, _ = inf.model_forward_he(model, ct, pcfg)
            be.decrypt(o)
            del ct, o

    for _ in range(min(args.warmup, 1)):
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
    h2d = B * S * 8          # zero-padded slot rows uploaded by encrypt
    d2h = B * S * 8          # decrypted slot vectors

    # ---- dominant kernels: NTT and key switch, live CUDA-event timing
    torch.cuda.empty_cache()
    roof = kernel_rooflines(be, params, chunk, stream) if rank == 0 else None

    if rank != 0:
        return
    total_inf = B * world
    value = total_inf / (ms / 1e3)
    hbm, hbm_kind = _peaks()
    line = {
        "metric": "encrypted KAN inferences/sec",
        "value": round(value, 4),
        "unit": "inferences/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u64 (RNS residues mod <=50-bit primes)",
        "data": "synthetic (seeded PCG64, SURVEY §8d)",
        "config": {"workload": f"{args.config}: KAN {list(cfg.dims)} G={cfg.g} k={cfg.k}, "
                               f"{B} ciphertexts/GPU in chunks of {chunk}, RNS-CKKS N=2^{args.log_n} L={depth} "
                               f"dnum={params.dnum} alpha={params.alpha}",
                   "global_batch": total_inf, "parallelism": f"dp{world} (ciphertext sharding)",
                   "l2": f"inputs {B * 2 * (depth + 1) * params.n * 8 / 1e9:.1f} GB/GPU >> 126 MB L2 "
                         "(no flush needed)"},
        "e2e": {"value": round(total_inf / (e2e_ms / 1e3), 4), "unit": "inferences/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "encrypt_input + model_forward_he + decrypt, host slots in/out"},
        "gpu_launches": launches,
        "clocks": clk,
        "max_abs_err_vs_reference_mirrored": err,
        "counts_per_inference": stats.to_json()["total"],
    }
    if roof:
        line["roofline"] = roof["ntt"]
        line["roofline"]["peak_kind"] = hbm_kind
        line["kernels"] = roof
    if not args.no_c2:
        del be, eng
        torch.cuda.empty_cache()
        line["c2_microbench"] = c2_microbench(local)
    if world == 1 and not args.no_cpu_baseline:
        if args.log_n > 16:
            line["cpu_baseline"] = {"skipped": "oracle setup at N=2^17 generates every Galois key on the "
                                               "CPU (hundreds of keys, many minutes); run c1 for the baseline"}
        else:
            line["cpu_baseline"] = cpu_baseline(args, budget_s=args.cpu_budget)
    print(json.dumps(line))


def kernel_rooflines(be, params, B, stream, reps: int = 5) -> dict:
    """CUDA-event timings of the two dominant primitives at c1 shapes."""
    import ctypes as C

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
    traffic, tr = None, {}
    try:  # dram__bytes_read.sum + dram__bytes_write.sum of the same launch shape (ncu --set full)
        with open(os.path.join(ROOT, "profiles", "r1_ntt_traffic.json")) as fh:
            tr = json.load(fh)
        if tr.get("algorithmic_bytes") == alg:
            traffic = tr["dram_read_bytes"] + tr["dram_write_bytes"]
    except Exception:
        pass
    out["ntt"] = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                  "frac": round(ach / hbm, 4), "traffic": traffic,
                  "kernel": f"hk_ntt_fwd -> ntt16::fwd_kernel (one 4-CTA cluster per polynomial, FP64-pipe "
                            f"butterflies), {nl} limbs x {B} polys",
                  "algorithmic_bytes": alg, "ms": round(t * 1e3, 3),
                  "note": f"FP64-issue/latency bound: ncu fp64 pipe {tr.get('fp64_pipe_pct')}%, issue "
                          f"{tr.get('issue_active_pct')}%; traffic above the algorithmic bytes is the "
                          f"between-phase buffer partly reaching HBM (profiles/r1_ntt_traffic.json)"}
    del buf
    # key switch via one rotation at the top level (ModUp + IP + ModDown)
    x = np.zeros((B, params.slot_count))
    ct = be.encrypt(x)
    be.rotate(ct, 1)
    torch.cuda.synchronize()
    ev[0].record(stream)
    for _ in range(reps):
        be.rotate(ct, 1)
    ev[1].record(stream)
    torch.cuda.synchronize()
    t = ev[0].elapsed_time(ev[1]) / reps / 1e3
    l = params.depth
    alpha, n_p = params.alpha, len(params.p)
    nd = l // alpha + 1
    alg = B * 4 * (l + 1) * N * 8 + 2 * nd * (l + 1 + n_p) * N * 8
    ach = alg / t / 1e9
    ks_traffic = None
    try:  # summed dram bytes of one rotation's launches at this shape (tools/prof_rot.py)
        with open(os.path.join(ROOT, "profiles", "r1_rotate_traffic.json")) as fh:
            rt = json.load(fh)
        if rt.get("algorithmic_bytes") == alg:
            ks_traffic = rt["dram_read_bytes"] + rt["dram_write_bytes"]
    except Exception:
        pass
    out["keyswitch"] = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                        "frac": round(ach / hbm, 4), "traffic": ks_traffic,
                        "note": "compute bound: ~250 limb-NTTs + ~2,400 conversion MACs per coefficient; "
                                "traffic counts the extended-basis intermediates (profiles/r1_rotate_traffic.json)",
                        "kernel": f"hk_rotate (ModUp+KeyIP+ModDown) level {l}, {B} cts",
                        "algorithmic_bytes": alg, "ms": round(t * 1e3, 3)}
    return out


def c2_microbench(device: int, n_ct: int = 256, reps: int = 3) -> dict:
    """BASELINE config 2: 256 ciphertexts with uniform random limbs,
    N=2^16, 24 ~50-bit limbs, dnum=3 (alpha = 8 special primes); CUDA-event
    times of NTT / iNTT (both polynomials), HMult+relin+rescale and rotate by
    +-2^j (j = 0..14, 30 Galois keys), each against SURVEY's algorithmic bytes."""
    import ctypes as C

    import torch
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
    eng.call("hk_keygen", C.c_uint64(7))
    steps = [s * (1 << j) for j in range(15) for s in (1, -1)]
    gal = [galois_element(t, p.slot_count) for t in steps]
    eng.call("hk_add_galois_keys", C.c_uint64(8), eng.u32_array(gal), len(gal))
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

    def entry(alg, t, what):
        ach = alg / t / 1e9
        return {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s", "frac": round(ach / hbm, 4),
                "ms": round(t * 1e3, 3), "algorithmic_bytes": alg, "kernel": what}

    out = {"workload": f"c2: {n_ct} ciphertexts x 2 polys x {n} limbs (~50-bit), N=2^16, dnum=3, alpha={alpha}, "
                       "uniform random limbs"}
    base = ct.data_ptr()
    half = n * n_ct * N * 8
    ntt_b = 2.0 * n_ct * 2 * n * N * 8
    t = timed(lambda: [eng.call("hk_ntt_fwd", base + q * half, 0, n, n_ct) for q in (0, 1)])
    out["ntt"] = entry(ntt_b, t, "hk_ntt_fwd, both polynomials")
    t = timed(lambda: [eng.call("hk_ntt_inv", base + q * half, 0, n, n_ct) for q in (0, 1)])
    out["intt"] = entry(ntt_b, t, "hk_ntt_inv, both polynomials")
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
# CPU baseline: the oracle port on host cores
# ---------------------------------------------------------------------------
def cpu_baseline(args, budget_s: float = 20.0) -> dict:
    """Oracle port, all host threads, one c1 sample at full N: runs the op
    stream of one inference until `budget_s` is spent, then scales by the
    fraction of the (pre-measured on GPU) program completed, counted in
    logical ops weighted by level (limb count)."""
    from oracle.engine import OracleEngine
    from paper_2409_07751_b200 import configs, inference as inf
    from paper_2409_07751_b200.backend import BackendConfig, HeBackend
    from paper_2409_07751_b200.params import kan_params

    cores = len(os.sched_getaffinity(0))
    cfg, model, inputs = configs.workload(args.config, batch=1)
    pcfg = inf.PipelineConfig()
    depth = inf.plan_model(model, pcfg).total
    params = kan_params(depth, log_n=args.log_n, dnum=args.dnum)
    t_setup = time.perf_counter()
    be = BudgetBackend(BackendConfig(slot_count=params.slot_count, depth_budget=depth), params,
                       engine=OracleEngine(params))
    be.prepare_keys_for(model, pcfg)
    setup = time.perf_counter() - t_setup
    ct = inf.encrypt_input(inputs, model, be)
    be.start(budget_s)
    t0 = time.perf_counter()
    try:
        inf.model_forward_he(model, ct, pcfg)
        done = True
    except _Budget:
        done = False
    el = time.perf_counter() - t0
    frac = 1.0 if done else be.weight_done / max(be.total_weight(model, pcfg), 1e-9)
    inf_per_s = frac / el if el > 0 else 0.0
    return {"value": round(inf_per_s, 6), "unit": "inferences/s", "cores": cores, "kind": "port",
            "sample": (f"oracle/libckks_oracle.so (OpenMP {cores} threads), {args.config} one ciphertext, "
                       f"N=2^{args.log_n}; ran {'the full inference' if done else f'{frac:.1%} of one inference (level-weighted op prefix)'} "
                       f"in {el:.1f} s; keygen/setup {setup:.1f} s untimed")}


class _Budget(Exception):
    pass


from paper_2409_07751_b200.backend import HeBackend  # noqa: E402  (torch-free import)


class BudgetBackend(HeBackend):
    """HeBackend with an op-weight meter and a wall-clock budget."""

    weight_done = 0.0
    _deadline = None

    def start(self, budget_s):
        self.weight_done = 0.0
        self._deadline = time.perf_counter() + budget_s

    def _tick(self, w):
        self.weight_done += w
        if self._deadline is not None and time.perf_counter() > self._deadline:
            raise _Budget()

    @staticmethod
    def op_weight(kind, level):
        return {"mul_ct": 12.0, "rot": 10.0, "mul_pt": 2.0, "add": 0.3}[kind] * (level + 1)

    def slotwise(self, op_kind, a, b):
        kind = "mul_ct" if op_kind == "mul_ct" else ("mul_pt" if op_kind == "mul_pt" else "add")
        out = super().slotwise(op_kind, a, b)
        self._tick(self.op_weight(kind, a.level))
        return out

    def rotate(self, a, t):
        out = super().rotate(a, t)
        if t:
            self._tick(self.op_weight("rot", a.level))
        return out

    def rotate_many(self, a, steps):
        out = super().rotate_many(a, steps)
        self._tick(sum(self.op_weight("rot", a.level) for t in steps if t))
        return out

    def mac_plain(self, babies, plains):
        out = super().mac_plain(babies, plains)
        self._tick(len(babies) * self.op_weight("mul_pt", babies[0].level))
        return out

    def mul_lin(self, a, b, x, k):
        out = super().mul_lin(a, b, x, k)
        self._tick(self.op_weight("mul_ct", min(a.level, b.level)))
        return out

    def mul_affine(self, a, b, mult, c):
        out = super().mul_affine(a, b, mult, c)
        self._tick(self.op_weight("mul_ct", min(a.level, b.level)))
        return out

    def mul2(self, a, b, a2, b2):
        out = super().mul2(a, b, a2, b2)
        self._tick(self.op_weight("mul_ct", min(a.level, b.level, a2.level, b2.level)))
        return out

    def prepare_keys_for(self, model, pcfg):
        """Generate every Galois key the program needs (untimed)."""
        from paper_2409_07751_b200 import inference as inf
        rec = _Recorder(self.config, self.params)
        inf.model_forward_he(model, rec.encrypt(np.zeros(model.n_in)), pcfg)
        self.ensure_rotation_keys(sorted(rec.steps))
        self._program = rec.ops

    def total_weight(self, model, pcfg):
        return sum(self.op_weight(k, lvl) * n for k, lvl, n in self._program)


class _Recorder:
    """Level-accurate dry run of the op program (no arithmetic)."""

    def __init__(self, config, params):
        from paper_2409_07751_b200.backend import OpCounter
        self.config = config
        self.params = params
        self.counter = OpCounter()
        self.steps = set()
        self.ops = []

    class Ct:
        def __init__(self, be, level):
            self.backend, self.level, self.batch, self.batched = be, level, 1, False

        @property
        def slots(self):
            return np.zeros(self.backend.config.slot_count)

    def encrypt(self, values, level=None):
        return self.Ct(self, self.config.depth_budget if level is None else level)

    def _lvl(self, a, b):
        return min(a.level, b.level) if isinstance(b, self.Ct) else a.level

    def add(self, a, b):
        self.ops.append(("add", self._lvl(a, b), 1))
        return self.Ct(self, self._lvl(a, b))

    sub = add

    def mul(self, a, b):
        lvl = self._lvl(a, b)
        self.ops.append(("mul_ct" if isinstance(b, self.Ct) else "mul_pt", lvl, 1))
        return self.Ct(self, lvl - 1)

    def rotate(self, a, t):
        if t:
            self.steps.add(t)
            self.ops.append(("rot", a.level, 1))
        return a if not t else self.Ct(self, a.level)

    def rotate_many(self, a, steps):
        return [self.rotate(a, t) for t in steps]

    def mac_plain(self, babies, plains):
        self.ops.append(("mul_pt", babies[0].level, len(babies)))
        return self.Ct(self, babies[0].level - 1)

    def mul_lin(self, a, b, x, k):
        lvl = min(a.level, b.level)
        self.ops.append(("mul_ct", lvl, 1))
        return self.Ct(self, lvl - 1)

    def mul_affine(self, a, b, mult, c):
        lvl = min(a.level, b.level)
        self.ops.append(("mul_ct", lvl, 1))
        return self.Ct(self, lvl - 1)

    def mul2(self, a, b, a2, b2):
        lvl = min(a.level, b.level, a2.level, b2.level)
        self.ops.append(("mul_ct", lvl, 1))
        return self.Ct(self, lvl - 1)


def reference_config(args):
    """The product arm's workload description (same model, batch, chunking and ring),
    so the driver compares like with like; the CPU measures a bounded sample of it."""
    from paper_2409_07751_b200 import configs, inference as inf
    from paper_2409_07751_b200.params import kan_params
    cfg = configs.CONFIGS[args.config]
    B = args.batch or (cfg.batch if cfg.batch <= 128 else 64)
    chunk = min(args.chunk or B, B)
    _, model, _ = configs.workload(args.config)
    depth = inf.plan_model(model, inf.PipelineConfig()).total
    params = kan_params(depth, log_n=args.log_n, dnum=args.dnum)
    return {"workload": f"{args.config}: KAN {list(cfg.dims)} G={cfg.g} k={cfg.k}, "
                        f"{B} ciphertexts/GPU in chunks of {chunk}, RNS-CKKS N=2^{args.log_n} L={depth} "
                        f"dnum={params.dnum} alpha={params.alpha}",
            "global_batch": B, "parallelism": "cpu (OpenMP, all host cores, one ciphertext at a time)",
            "sample": "bounded prefix of one inference per step (cpu_baseline.sample)"}


def run_reference(args):
    """--impl reference: the CPU path (oracle port) on host cores, rank 0 only."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    vals = []
    base = None
    for i in range(args.warmup + args.steps):
        r = cpu_baseline(args, budget_s=args.cpu_budget)
        if i >= args.warmup:
            vals.append(r["value"])
            base = r
    v = statistics.median(vals) if vals else 0.0
    line = {"metric": "encrypted KAN inferences/sec", "value": v, "unit": "inferences/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 / v, 3) if v else None, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64 (RNS residues)",
            "data": "synthetic (seeded PCG64, SURVEY §8d)", "impl": "reference",
            "config": reference_config(args),
            "cpu_baseline": dict(base or {}, value=v),
            "e2e": {"value": v, "unit": "inferences/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line))


def main():
    os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("product", "reference"), default="product")
    ap.add_argument("--config", default="c1")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--dnum", type=int, default=3, help="key-switching digits over the full chain")
    ap.add_argument("--chunk", type=int, default=None,
                    help="ciphertexts per batched launch (default 32; 8 for c5 at N=2^17)")
    ap.add_argument("--log-n", type=int, default=None,
                    help="ring degree (default 16; 17 for c5, whose 33792 packed slots need S=2^16)")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c2", action="store_true", help="skip the config-2 primitive microbench")
    args = ap.parse_args()
    if args.log_n is None:
        args.log_n = 17 if args.config == "c5" else 16
    if args.chunk is None:
        # ciphertexts per launch (the whole resident batch where it fits in HBM): c1 and
        # c3 run their batch in one chunk; c4 / c5 hold 80 / 157 hoisted BSGS baby
        # steps at once, which bounds them to 32 at N = 2^16 and 8 at N = 2^17
        if args.log_n > 16:
            args.chunk = 8 if args.config == "c5" else 32
        else:
            args.chunk = {"c4": 32, "c5": 8}.get(args.config, 128)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_product(args)


if __name__ == "__main__":
    main()
