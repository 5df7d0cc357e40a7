"""Benchmark: RNS-CKKS primitive throughput (config 2) + ranking/sort latencies.

Default (``python bench.py``): N=1 GPU, the BASELINE config-2 primitive set
as one "step" over 64 ciphertexts (ring 2^16, 30 Q-limbs, 3 special primes,
dnum 3): forward NTT + inverse NTT + HMult/relinearise + rotation by every
power of two 1..2^14 + rescale.  ``value`` = algorithmic GB moved per step
 / step time, whole job, inputs resident in HBM; ``e2e`` = the
same step through the C-ABI with the 64 input ciphertexts copied from pinned
host memory and the 64 rescaled outputs copied back inside the timed region.
Inputs (1.9 GiB per operand set) exceed the 126 MB L2, so no flush is needed.

The pipeline latencies BASELINE.json quotes (rank N=128, argmin/argmax/median
masks N=128, sort N=1024) are measured after the primitive step and reported
under ``pipelines``.  ``--impl reference`` times the CPU RNS-CKKS oracle
(oracle/ckks_oracle.c, all host threads) on a bounded sample of the same step.
Multi-GPU (torchrun): every rank runs its own 64 ciphertexts (weak scaling, no
data-path collective); the max time over ranks is reported.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
# several ranks sharing one GPU (the gloo functional mode): expandable segments
# keep the long-chain pipelines' multi-GiB blocks from fragmenting the shared HBM
if os.environ.get("SRK_DIST_BACKEND") == "gloo":
    os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

GB = 1e9
N_CT = 64
ROT_STEPS = [1 << k for k in range(15)]


def algorithmic_bytes(p, n_ct=N_CT):
    """Compulsory HBM bytes per step (SURVEY.md section 8d formulas)."""
    n = p.ring_degree
    limb = n * 8
    nl = len(p.q_primes)
    ne = nl + len(p.p_primes)
    evk = 2 * p.dnum * ne * limb
    ct = 2 * nl * limb
    parts = {
        "ntt_fwd": n_ct * 2 * nl * limb * 2,
        "ntt_inv": n_ct * 2 * nl * limb * 2,
        "hmult_relin": n_ct * 3 * ct + evk,           # 2 ct in, 1 out, + evk once
        "rotate_15": len(ROT_STEPS) * (n_ct * 2 * ct + evk),
        "rescale": n_ct * (ct + 2 * (nl - 1) * limb),
    }
    return parts, parts["hmult_relin"]


# ----------------------------------------------------------------------
# clocks sampling (nvidia-smi during the timed region)
# ----------------------------------------------------------------------
class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                    capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ----------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------
def _rand_cts(torch, p, n_ct, seed, device):
    """Uniform limbs per prime (BASELINE cfg 2: limbs uniform mod each prime)."""
    nl = len(p.q_primes)
    out = torch.empty((n_ct, 2, nl, p.ring_degree), dtype=torch.int64, device=device)
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    for i, q in enumerate(p.q_primes):
        # q < 2^62: draw in [0, q) via two 31-bit halves is biased; use int64 randint on [0, q)
        out[:, :, i, :] = torch.randint(0, q, (n_ct, 2, p.ring_degree), generator=g, device=device,
                                        dtype=torch.int64)
    return out


class PrimitiveStep:
    """The config-2 step on one GPU, through the C-ABI of libslotrank_b200."""

    def __init__(self, torch, device, n_ct=N_CT):
        from paper_2412_15126_b200.backend_cuda import CudaBackend
        from paper_2412_15126_b200.keys import sample_secret
        from paper_2412_15126_b200.params import preset

        self.torch = torch
        self.p = p = preset("cfg2")
        self.n_ct = n_ct
        self.be = be = CudaBackend(p, device)
        be.set_secret(sample_secret(p))
        self.rlk = be.relin_key()
        self.gal = [pow(5, k, 2 * p.ring_degree) for k in ROT_STEPS]
        self.gkeys = [be.galois_key(g) for g in self.gal]
        self.nl = len(p.q_primes)
        self.x = _rand_cts(torch, p, n_ct, 1, be.device)
        self.y = _rand_cts(torch, p, n_ct, 2, be.device)
        shape = (n_ct, 2, self.nl, p.ring_degree)
        self.prod = torch.empty(shape, dtype=torch.int64, device=be.device)
        # one output set per rotation index (hoisted rotations write all 15 at once)
        self.rot = [torch.empty(shape, dtype=torch.int64, device=be.device) for _ in ROT_STEPS]
        self.res = torch.empty((n_ct, 2, self.nl - 1, p.ring_degree), dtype=torch.int64, device=be.device)
        self.ws = be.workspace()
        self.lib = be.lib
        self.ctx = be.ctx
        self.launch_count = 0

    def _c(self, name, *args):
        from paper_2412_15126_b200 import _lib

        self.launch_count += 1
        _lib.check(getattr(self.lib, name)(self.ctx, *args))

    def ntt(self, t, inverse, lo=0, n_ct=None):
        n, L = self.p.ring_degree, self.nl
        n_ct = self.n_ct if n_ct is None else n_ct
        s = self.be.stream()
        self._c("srk_ntt", t.data_ptr() + lo * self._ct_bytes, n_ct * 2, L * n, L, 0, int(inverse), s)

    @property
    def _ct_bytes(self):
        return 2 * self.nl * self.p.ring_degree * 8

    def relin_batch(self):
        """HMult + relinearisation of the 64 pairs (the key-switch roofline unit)."""
        s = self.be.stream()
        ct = 2 * self.nl * self.p.ring_degree
        self._c("srk_mul_relin_batch", self.x.data_ptr(), self.y.data_ptr(), ct, self.rlk.data_ptr(),
                self.prod.data_ptr(), ct, self.n_ct, self.nl - 1, 0, self.ws, s)

    def rotations(self, x, lo=0, n_ct=None):
        """All 15 power-of-two rotations of every ciphertext, one base extension each."""
        import ctypes

        n_ct = self.n_ct if n_ct is None else n_ct
        s = self.be.stream()
        ct = 2 * self.nl * self.p.ring_degree
        off = lo * self._ct_bytes
        n_rot = len(self.gal)
        keys = (ctypes.c_void_p * n_rot)(*[k.data_ptr() for k in self.gkeys])
        gal = (ctypes.c_uint64 * n_rot)(*self.gal)
        outs = (ctypes.c_void_p * n_rot)(*[o.data_ptr() + off for o in self.rot])
        self._c("srk_rotate_hoisted", x.data_ptr() + off, ct, n_ct, n_rot, keys, gal, outs, ct,
                self.nl - 1, self.ws, s)

    def step(self, x=None, lo=0, n_ct=None):
        """The primitive set over ciphertexts [lo, lo + n_ct) (default: all 64)."""
        x = self.x if x is None else x
        n_ct = self.n_ct if n_ct is None else n_ct
        s = self.be.stream()
        L = self.nl - 1
        ct = 2 * self.nl * self.p.ring_degree
        off = lo * self._ct_bytes
        self.ntt(x, False, lo, n_ct)
        self.ntt(x, True, lo, n_ct)
        self._c("srk_mul_relin_batch", x.data_ptr() + off, self.y.data_ptr() + off, ct,
                self.rlk.data_ptr(), self.prod.data_ptr() + off, ct, n_ct, L, 0, self.ws, s)
        self.rotations(x, lo, n_ct)
        self._c("srk_rescale_batch", self.prod.data_ptr() + off, ct,
                self.res.data_ptr() + lo * 2 * L * self.p.ring_degree * 8,
                2 * L * self.p.ring_degree, n_ct, L, self.ws, s)


class PipelinedE2E:
    """End-to-end step with host buffers: the 64 input ciphertexts arrive from
    pinned host memory and the 64 rescaled results go back, every step.  The
    batch is cut into ``chunks`` groups of ciphertexts; chunk i's host->device
    copy (copy stream) overlaps chunk i-1's compute, and its device->host copy
    (second copy stream) overlaps chunk i+1's compute -- PCIe both ways runs
    under the kernels instead of in series with them.  Every byte of every
    chunk is still copied inside the timed region."""

    def __init__(self, torch, step, chunks=4):
        self.torch, self.step, self.chunks = torch, step, chunks
        self.host_x = torch.empty(step.x.shape, dtype=torch.int64, pin_memory=True)
        self.host_x.copy_(step.x)
        self.host_out = torch.empty(step.res.shape, dtype=torch.int64, pin_memory=True)
        self.dev_x = torch.empty_like(step.x)
        self.h2d, self.d2h = torch.cuda.Stream(), torch.cuda.Stream()
        # half-size first and last chunks: the first H2D and the last D2H are the
        # only copies with no compute to hide under
        per = -(-step.n_ct // chunks)
        ramp = int(os.environ.get("SRK_E2E_RAMP", "2"))  # first chunk = per / ramp
        sizes = [max(1, per // ramp)]
        while sum(sizes) < step.n_ct:
            sizes.append(min(per, step.n_ct - sum(sizes)))
        if len(sizes) > 2 and sizes[-1] == per:
            sizes[-1] = per - sizes[0]
            sizes.append(sizes[0])
        self.bounds, lo = [], 0
        for sz in (z for z in sizes if z > 0):
            self.bounds.append((lo, sz))
            lo += sz
        self.ev_in = [torch.cuda.Event() for _ in self.bounds]
        self.ev_done = [torch.cuda.Event() for _ in self.bounds]

    def __call__(self):
        torch = self.torch
        comp = torch.cuda.current_stream()
        self.h2d.wait_stream(comp)
        self.d2h.wait_stream(comp)
        with torch.cuda.stream(self.h2d):
            for i, (lo, n) in enumerate(self.bounds):
                self.dev_x[lo:lo + n].copy_(self.host_x[lo:lo + n], non_blocking=True)
                self.ev_in[i].record(self.h2d)
        for i, (lo, n) in enumerate(self.bounds):
            comp.wait_event(self.ev_in[i])
            self.step.step(self.dev_x, lo, n)
            self.ev_done[i].record(comp)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(self.ev_done[i])
                self.host_out[lo:lo + n].copy_(self.step.res[lo:lo + n], non_blocking=True)
        comp.wait_stream(self.d2h)


def bench_config(p):
    parts, _ = algorithmic_bytes(p)
    return {"workload": "cfg2 primitive step: fwd NTT + INTT + 64 HMult/relin + 64x15 "
                        "power-of-two rotations + 64 rescale",
            "ciphertexts_per_gpu": N_CT, "ring": p.ring_degree, "q_limbs": len(p.q_primes),
            "p_limbs": len(p.p_primes), "dnum": p.dnum,
            "algorithmic_gb_per_step": round(sum(parts.values()) / GB, 3),
            "l2": "inputs 1.9 GiB per operand set >> 126 MB L2 (no flush needed)"}


def _profile(name):
    """A committed ncu summary (profiles/r02 first, then r01), or None."""
    for rnd in ("r02", "r01"):
        path = os.path.join(ROOT, "profiles", rnd, name)
        try:
            with open(path) as fh:
                return f"profiles/{rnd}/{name}", json.load(fh)
        except (OSError, ValueError):
            continue
    return None, None


def pipe_roofline():
    """FP64 / integer pipe utilisation of the NTT passes from the committed
    ``ncu --set full`` capture (the NTT's real bound: DESIGN.md, kernels)."""
    src, d = _profile("ntt_pipe_util.json")
    if d is None:
        return None
    return {"bound": "fp64 / fma pipes (ncu)", "source": src + " (" + d.get("command", "") + ")",
            "kernels": d["kernels"]}


def fp64_roofline(torch, lib, p, ntt_ms, ntt_bytes, hbm_peak):
    """The forward NTT against the FP64 pipe (its binding unit: DESIGN.md, kernels).
    Peak = FP64 FMA issue rate measured here with srk_fp64_probe (148 x 8 CTAs of
    8 independent FMA chains per thread); work = the FP64 instructions the passes
    issue per transform: 8 per butterfly (6 for the exact FMA-split product, 2 for
    x +- t) and 5 per coefficient for the u64 <-> f64 edges, limbs under primes
    < 2^41 only (the 60-bit limb 0 runs on the integer pipe)."""
    n = p.ring_degree
    log_n = n.bit_length() - 1
    f64_limbs = sum(1 for q in p.q_primes if q < (1 << 41))
    instr = N_CT * 2 * f64_limbs * (log_n * (n // 2) * 8 + n * 5)
    ctas, iters = 148 * 8, 20000
    sink = torch.zeros(8, dtype=torch.float64, device="cuda")
    run = lambda: lib.srk_fp64_probe(ctas, iters, sink.data_ptr(), torch.cuda.current_stream().cuda_stream)  # noqa: E731
    run()
    probe_ms = min(time_region(torch, run, 3) for _ in range(3))
    peak = ctas * 256 * 8 * iters / (probe_ms * 1e-3)
    roof_ms = instr / peak * 1e3
    return {"bound": "fp64 pipe", "kernel": "forward NTT (ntt_pass_kernel x2 per chunk)",
            "fp64_instructions": instr, "peak_fp64_instr_per_s": round(peak, -9),
            "peak_source": "srk_fp64_probe timed here (independent FMA chains, CUDA events)",
            "achieved_fp64_instr_per_s": round(instr / (ntt_ms * 1e-3), -9),
            "frac": round(roof_ms / ntt_ms, 4), "ms_at_fp64_roof": round(roof_ms, 4),
            "hbm_frac_at_fp64_roof": round(ntt_bytes / (roof_ms * 1e-3) / GB / hbm_peak, 4)}


def time_region(torch, fn, reps, barrier=None):
    """CUDA-event time of ``reps`` calls of fn (ms per call), synchronized both sides."""
    torch.cuda.synchronize()
    if barrier:
        barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def ntt_traffic():
    """(source, DRAM bytes) of one forward NTT of the bench batch from the committed ncu capture."""
    src, d = _profile("ntt_fwd_traffic.json")
    return (src, int(d["dram_bytes"])) if d else (None, None)


def keyswitch_traffic():
    """(source, DRAM bytes) of 64 HMult+relinearise from the committed ncu launch list."""
    src, d = _profile("relin64_traffic.json")
    return (src, int(d["dram_bytes"])) if d else (None, None)


def kernel_roofline():
    """Per-kernel DRAM GB/s of one primitive step from the committed ncu capture."""
    src, d = _profile("kernel_roofline_step64.json")
    if d is None:
        return None
    return {"source": src + " (" + d.get("note", "") + ")", "peak_gbs": d.get("peak_gbs"),
            "kernels": [{k: e[k] for k in ("kernel", "time_share", "dram_gb_per_s", "frac_of_hbm")}
                        for e in d["kernels"] if e["time_share"] >= 0.01]}


def _event_time(torch, fn, dist=None):
    """Seconds between CUDA events around fn on the current stream (max over ranks)."""
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    r = fn()
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / 1e3], device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()), r


def run_sharded_sort(torch, dist):
    """Config 5 on every rank: multi_sort of N=1024 sharded over the world (shard.py),
    in the reference layout and in the packed layout (packing.py)."""
    from paper_2412_15126_b200 import (B200Engine, KernelConfig, SortConfig, block_merge, block_split)
    from paper_2412_15126_b200.params import preset
    from paper_2412_15126_b200.shard import Comm, multi_sort_sharded

    eng = B200Engine(preset("long"))
    v1024 = np.random.default_rng(0).choice(8192, 1024, replace=False) / 8192
    kcfg = KernelConfig(mode="composite", composite=(6, 2), indicator_composite=(6, 2))
    bv = block_split(eng, v1024)
    comm = Comm()
    out = {}
    for name, packed in (("sort_n1024_s", False), ("sort_n1024_packed_s", True)):
        scfg = SortConfig(kernel=kcfg, tie_correction=False, packed=packed)
        multi_sort_sharded(eng, bv, scfg, comm)  # warm-up: keys, plaintext cache
        c0, s0 = comm.collectives, comm.level_syncs
        dt, res = _event_time(torch, lambda: multi_sort_sharded(eng, bv, scfg, comm), dist)
        srt = block_merge(eng, res)
        out[name] = {"latency_s": dt, "order_ok": bool(np.array_equal(np.argsort(srt), np.arange(1024))),
                     "max_abs_err": float(np.abs(srt - np.sort(v1024)).max()), "params": "long",
                     "gpus": comm.world, "collectives": comm.collectives - c0, "level_syncs": comm.level_syncs - s0,
                     "sharding": f"5 phases (shard.py), {dist.get_backend()}",
                     "layout": "packed (packing.py)" if packed else "reference"}
    return out


NVLINK_GBS = 900.0  # per direction per GPU through NVSwitch (B200_PROFILING.md)


def projected_sharded_sort(torch, eng, bv, kcfg):
    """N=1024 sort at 2/4/8 ranks PROJECTED from one GPU: rank 0's own kernels (the rank
    with the most units under the round-robin deal) timed here through shard.py's
    real code path with collectives that move no data (shard.ProjectedComm), plus the
    bytes each collective would move at NVLink rate (ring all-reduce 2(W-1)/W S,
    all-gather (W-1)/W S).  Not a measured multi-GPU latency."""
    from paper_2412_15126_b200 import SortConfig
    from paper_2412_15126_b200.shard import ProjectedComm, multi_sort_sharded

    out = {}
    for packed in (False, True):
        scfg = SortConfig(kernel=kcfg, tie_correction=False, packed=packed)
        for world in (2, 4, 8):
            comm = ProjectedComm(0, world)
            multi_sort_sharded(eng, bv, scfg, comm)  # warm-up (level plan, constants)
            comm.all_reduce_bytes = comm.all_gather_bytes = comm.collectives = 0
            dt, _ = _timed(torch, lambda: multi_sort_sharded(eng, bv, scfg, comm))
            f = (world - 1) / world
            comm_s = (2 * f * comm.all_reduce_bytes + f * comm.all_gather_bytes) / (NVLINK_GBS * 1e9)
            out[f"{'packed' if packed else 'reference'}_w{world}"] = {
                "rank0_compute_s": dt, "collectives": comm.collectives,
                "all_reduce_bytes": comm.all_reduce_bytes, "all_gather_bytes": comm.all_gather_bytes,
                "modelled_nvlink_s": comm_s, "projected_latency_s": dt + comm_s}
    out["note"] = ("projection from ONE B200: rank 0's kernels of the W-rank sharded sort run here with "
                   "data-free collectives (shard.ProjectedComm; outputs not meaningful), NVLink time "
                   f"modelled at {NVLINK_GBS:.0f} GB/s per direction, no overlap assumed")
    return out


def _timed(torch, fn, reps=1):
    """Best-of-reps wall seconds of fn() bracketed by device syncs."""
    best, r = None, None
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best, r


def _census(eng, fn):
    """One run's CostReport (reset before, snapshot after: one pipeline, not several)."""
    eng.cost_reset()
    r = fn()
    return eng.cost_snapshot().__dict__, r


def run_pipelines(torch, quick=False):
    """BASELINE pipeline latencies (seconds) on cuda:current, decrypted results checked.
    Every ``cost`` is the CostReport of exactly one run of the pipeline."""
    from oracle.plain import fractional_ranks  # result-level checker only
    from paper_2412_15126_b200 import (B200Engine, KernelConfig, SortConfig, StatisticQuery,
                                       block_merge, block_split, multi_sort, order_statistic_mask,
                                       order_statistic_value, rank, read_row)
    from paper_2412_15126_b200.params import preset

    out = {}
    # config 1: rank N=16 on ring 2^12 (composite g3^4 o f3^2)
    v16 = np.random.default_rng(0).choice(64, 16, replace=False) / 64
    eng = B200Engine(preset("cfg1"))
    cfg1 = KernelConfig(mode="composite", composite=(4, 2))
    ct = eng.encrypt(v16)
    rank(eng, ct, 16, cfg1)  # warm-up: keys, plaintext cache
    cost, _ = _census(eng, lambda: rank(eng, ct, 16, cfg1))
    dt, res = _timed(torch, lambda: read_row(eng, rank(eng, ct, 16, cfg1).ranks, 16), reps=3)
    out["rank_n16_s"] = {"latency_s": dt, "graph_replay_s": _graph_latency(eng, lambda c: rank(eng, c, 16, cfg1).ranks, ct),
                         "exact_ranks": bool(np.array_equal(np.rint(res), fractional_ranks(v16))),
                         "cost": cost, "params": "cfg1", "kernel": "composite g3^4 o f3^2"}
    del eng

    # config 3: rank N=128, composite g3^4 o f3^2, ring 2^16, 29 levels
    rng = np.random.default_rng(0)
    v128 = rng.choice(1024, 128, replace=False) / 1024
    eng = B200Engine(preset("cfg3"))
    cfg = KernelConfig(mode="composite", composite=(4, 2))
    ct = eng.encrypt(v128)
    rank(eng, ct, 128, cfg)  # warm-up: Galois / relin key generation, plaintext cache
    cost, _ = _census(eng, lambda: rank(eng, ct, 128, cfg))
    dt, res = _timed(torch, lambda: read_row(eng, rank(eng, ct, 128, cfg).ranks, 128), reps=3)
    exact = bool(np.array_equal(np.rint(res), fractional_ranks(v128)))
    out["rank_n128_s"] = {"latency_s": dt, "graph_replay_s": _graph_latency(eng, lambda c: rank(eng, c, 128, cfg).ranks, ct),
                          "exact_ranks": exact,
                          "max_rank_err": float(np.abs(res - fractional_ranks(v128)).max()),
                          "cost": cost, "params": "cfg3", "kernel": "composite g3^4 o f3^2"}
    # the same rank started at the level its depth needs (engine.encrypt(level=...)):
    # 21 of the chain's 30 limbs carry the whole circuit
    need = eng.circuit_depth(lambda e, c: rank(e, c, 128, cfg).ranks)
    fitted = lambda c: rank(eng, eng.fit_depth(c, need), 128, cfg).ranks  # noqa: E731
    fitted(ct)  # warm-up: the dropped level's constants and allocator blocks
    dtf, resf = _timed(torch, lambda: read_row(eng, fitted(ct), 128), reps=3)
    out["rank_n128_depth_fitted_s"] = {
        "latency_s": dtf, "graph_replay_s": _graph_latency(eng, fitted, ct),
        "exact_ranks": bool(np.array_equal(np.rint(resf), fractional_ranks(v128))),
        "max_rank_err": float(np.abs(resf - fractional_ranks(v128)).max()),
        "start_level": need,
        "params": "cfg3 (the same full-chain input ciphertext, dropped to the circuit's depth inside the "
                  "timed pipeline: engine.fit_depth)",
        "kernel": "composite g3^4 o f3^2"}
    # the reference's own comparison: Chebyshev interpolant, degree 1024
    ccfg = KernelConfig(mode="chebyshev", degree=1024)
    rank(eng, ct, 128, ccfg)
    cost, _ = _census(eng, lambda: rank(eng, ct, 128, ccfg))
    dt, res = _timed(torch, lambda: read_row(eng, rank(eng, ct, 128, ccfg).ranks, 128), reps=2)
    out["rank_n128_chebyshev_d1024_s"] = {
        "latency_s": dt, "graph_replay_s": _graph_latency(eng, lambda c: rank(eng, c, 128, ccfg).ranks, ct),
        "exact_ranks": bool(np.array_equal(np.rint(res), fractional_ranks(v128))),
        "max_rank_err": float(np.abs(res - fractional_ranks(v128)).max()),
        "cost": cost, "params": "cfg3", "kernel": "chebyshev d=1024 (reference)"}
    del eng
    torch.cuda.empty_cache()
    # the same rank at Delta = 2^47 (cfg3_hp: the reference's 1e-6 slot tolerance, DESIGN "Parity")
    eng = B200Engine(preset("cfg3_hp"))
    ct = eng.encrypt(v128)
    rank(eng, ct, 128, cfg)
    cost, _ = _census(eng, lambda: rank(eng, ct, 128, cfg))
    dt, res = _timed(torch, lambda: read_row(eng, rank(eng, ct, 128, cfg).ranks, 128), reps=3)
    out["rank_n128_hp_s"] = {"latency_s": dt,
                             "graph_replay_s": _graph_latency(eng, lambda c: rank(eng, c, 128, cfg).ranks, ct),
                             "exact_ranks": bool(np.array_equal(np.rint(res), fractional_ranks(v128))),
                             "max_rank_err": float(np.abs(res - fractional_ranks(v128)).max()),
                             "cost": cost, "params": "cfg3_hp (Delta 2^47, 10 special primes)",
                             "kernel": "composite g3^4 o f3^2"}
    del eng
    torch.cuda.empty_cache()
    if quick:
        return out

    # config 4: argmin / argmax / k=64 masks AND selected values, N=128, long chain
    eng = B200Engine(preset("long"))
    cfg4 = KernelConfig(mode="composite", composite=(4, 2), indicator_composite=(4, 2),
                        tie_margin=2.0 ** -11, goldschmidt_iters=8)
    ct = eng.encrypt(v128)
    order = np.argsort(v128)
    for name, q, pos in (("argmin", StatisticQuery("min"), 0),
                         ("argmax", StatisticQuery("max"), 127),
                         ("median_k64", StatisticQuery("kth", k=64), 63)):
        want = order[pos]
        order_statistic_value(eng, ct, 128, q, cfg4)  # warm-up keys
        # the pipeline first drops the full-chain input to the level its depth needs (the long
        # chain is sized for the N=1024 sort; a mask needs ~40 of its 57 limbs): engine.fit_depth,
        # one fused multiply-and-rescale inside the timed region
        need_m = eng.circuit_depth(lambda e, c, q=q: order_statistic_mask(e, c, 128, q, cfg4))
        need_v = eng.circuit_depth(lambda e, c, q=q: order_statistic_value(e, c, 128, q, cfg4))
        fm = lambda c, q=q, d=need_m: order_statistic_mask(eng, eng.fit_depth(c, d), 128, q, cfg4)  # noqa: E731
        fv = lambda c, q=q, d=need_v: order_statistic_value(eng, eng.fit_depth(c, d), 128, q, cfg4)  # noqa: E731
        full_dt, _ = _timed(torch, lambda q=q: read_row(eng, order_statistic_mask(eng, ct, 128, q, cfg4), 128), reps=2)
        cost, _ = _census(eng, lambda: fm(ct))
        dt, m = _timed(torch, lambda: read_row(eng, fm(ct), 128), reps=2)
        gdt = _graph_latency(eng, fm, ct)
        full_vdt, _ = _timed(torch, lambda q=q: eng.decrypt(order_statistic_value(eng, ct, 128, q, cfg4))[0], reps=2)
        vcost, _ = _census(eng, lambda: fv(ct))
        vdt, val = _timed(torch, lambda: eng.decrypt(fv(ct))[0], reps=2)
        vgdt = _graph_latency(eng, fv, ct)
        out[f"{name}_n128_s"] = {"latency_s": dt, "graph_replay_s": gdt,
                                 "start_level": need_m, "full_chain_latency_s": full_dt,
                                 "index_ok": bool(int(np.argmax(m)) == int(want)),
                                 "max_onehot_err": float(np.abs(m - np.eye(128)[want]).max()),
                                 "cost": cost,
                                 "value_latency_s": vdt, "value_graph_replay_s": vgdt,
                                 "value_start_level": need_v, "value_full_chain_latency_s": full_vdt,
                                 "value": float(val), "value_err": float(abs(val - v128[want])),
                                 "value_cost": vcost, "params": "long (the full-chain input dropped to the circuit's depth "
                                                                "inside the timed pipeline, engine.fit_depth; "
                                                                "full_chain_*: run from the top of the chain)",
                                 "note": "value = mask + SumC(mask*v) * Goldschmidt(SumC(mask)), 8 iterations"}

    # config 5: sort N=1024 (8 blocks of 128), composite comparisons
    v1024 = np.random.default_rng(0).choice(8192, 1024, replace=False) / 8192
    scfg = SortConfig(kernel=KernelConfig(mode="composite", composite=(6, 2),
                                          indicator_composite=(6, 2)), tie_correction=False)
    bv = block_split(eng, v1024)
    first, _ = _timed(torch, lambda: block_merge(eng, multi_sort(eng, bv, scfg)))
    cost, _ = _census(eng, lambda: multi_sort(eng, bv, scfg))
    warm, srt = _timed(torch, lambda: block_merge(eng, multi_sort(eng, bv, scfg)))
    out["sort_n1024_s"] = {"latency_s": first, "warm_latency_s": warm,
                           "order_ok": bool(np.array_equal(np.argsort(srt), np.arange(1024))),
                           "max_abs_err": float(np.abs(srt - np.sort(v1024)).max()),
                           "cost": cost, "params": "long", "gpus": 1,
                           "note": "latency_s: first run (includes generating this pipeline's Galois keys and "
                                   "encoding its constants); warm_latency_s: second run"}
    # rank N=1024 (multi_rank: the 36 block-pair comparisons + complement folds), both layouts
    from paper_2412_15126_b200 import multi_rank
    from oracle.plain import fractional_ranks as _fr
    for name, pk in (("rank_n1024_s", False), ("rank_n1024_packed_s", True)):
        full, _ = _timed(torch, lambda pk=pk: block_merge(eng, multi_rank(eng, bv, scfg.kernel, packed=pk)))
        # the full-chain blocks dropped to the level the rank's depth needs (27 of the chain's 56)
        # inside the timed region (engine.fit_depth)
        need = eng.circuit_depth(lambda e, c, pk=pk: list(multi_rank(
            e, type(bv)(blocks=tuple(c for _ in bv.blocks), block_size=bv.block_size, total_len=bv.total_len),
            scfg.kernel, packed=pk).blocks))
        fit = lambda d=need: type(bv)(blocks=tuple(eng.fit_depth(b, d) for b in bv.blocks),  # noqa: E731
                                      block_size=bv.block_size, total_len=bv.total_len)
        first, _ = _timed(torch, lambda pk=pk: block_merge(eng, multi_rank(eng, fit(), scfg.kernel, packed=pk)))
        cost, _ = _census(eng, lambda pk=pk: multi_rank(eng, fit(), scfg.kernel, packed=pk))
        warm, rk = _timed(torch, lambda pk=pk: block_merge(eng, multi_rank(eng, fit(), scfg.kernel, packed=pk)), reps=2)
        out[name] = {"latency_s": first, "warm_latency_s": warm, "start_level": need,
                     "full_chain_latency_s": full,
                     "exact_ranks": bool(np.array_equal(np.rint(rk), _fr(v1024))),
                     "max_rank_err": float(np.abs(rk - _fr(v1024)).max()), "cost": cost, "params": "long",
                     "layout": "two blocks per ciphertext (packing.py)" if pk else "reference (one block per ciphertext)"}
    # the same sort in the packed layout (two blocks per ciphertext: 18 comparison and
    # 32 indicator evaluations instead of 36 / 64; packing.py)
    pcfg = SortConfig(kernel=scfg.kernel, tie_correction=False, packed=True)
    first, _ = _timed(torch, lambda: block_merge(eng, multi_sort(eng, bv, pcfg)))
    cost, _ = _census(eng, lambda: multi_sort(eng, bv, pcfg))
    warm, srt = _timed(torch, lambda: block_merge(eng, multi_sort(eng, bv, pcfg)))
    out["sort_n1024_packed_s"] = {"latency_s": first, "warm_latency_s": warm,
                                  "order_ok": bool(np.array_equal(np.argsort(srt), np.arange(1024))),
                                  "max_abs_err": float(np.abs(srt - np.sort(v1024)).max()),
                                  "cost": cost, "params": "long", "gpus": 1,
                                  "layout": "two 128x128 blocks per ciphertext (opt-in, packing.py)"}
    # the comparison one g3 shallower, composite (5,2), under the same (6,2) indicator, whose
    # flat regions absorb the softer comparison (slot oracle, seeds 0..9: 6.7e-8 against 3.6e-8);
    # 52 levels instead of 55, so the blocks are dropped to level 52 first (engine.fit_depth)
    k52 = KernelConfig(mode="composite", composite=(5, 2), indicator_composite=(6, 2))
    for name, pk in (("sort_n1024_cmp52_s", False), ("sort_n1024_cmp52_packed_s", True)):
        c52 = SortConfig(kernel=k52, tie_correction=False, packed=pk)
        need = eng.circuit_depth(lambda e, c, c52=c52: list(multi_sort(
            e, type(bv)(blocks=tuple(c for _ in bv.blocks), block_size=bv.block_size, total_len=bv.total_len),
            c52).blocks))
        fit = lambda d=need: type(bv)(blocks=tuple(eng.fit_depth(b, d) for b in bv.blocks),  # noqa: E731
                                      block_size=bv.block_size, total_len=bv.total_len)
        first, _ = _timed(torch, lambda c52=c52: block_merge(eng, multi_sort(eng, fit(), c52)))
        cost, _ = _census(eng, lambda c52=c52: multi_sort(eng, fit(), c52))
        warm, srt = _timed(torch, lambda c52=c52: block_merge(eng, multi_sort(eng, fit(), c52)), reps=2)
        out[name] = {"latency_s": first, "warm_latency_s": warm, "start_level": need,
                     "order_ok": bool(np.array_equal(np.argsort(srt), np.arange(1024))),
                     "max_abs_err": float(np.abs(srt - np.sort(v1024)).max()),
                     "cost": cost, "params": "long (blocks dropped to the circuit's depth, engine.fit_depth)",
                     "kernel": "comparison g3^5 o f3^2, indicator g3^6 o f3^2", "gpus": 1,
                     "layout": "packed (packing.py)" if pk else "reference"}
    out["sort_n1024_sharded_projection"] = projected_sharded_sort(torch, eng, bv, scfg.kernel)
    del eng, bv
    torch.cuda.empty_cache()
    # the tie-corrected sort (block tie offsets) needs two more levels: long58
    eng = B200Engine(preset("long58"))
    scfg = SortConfig(kernel=KernelConfig(mode="composite", composite=(6, 2),
                                          indicator_composite=(6, 2)), tie_correction=True)
    bv = block_split(eng, v1024)
    first, _ = _timed(torch, lambda: block_merge(eng, multi_sort(eng, bv, scfg)))
    cost, _ = _census(eng, lambda: multi_sort(eng, bv, scfg))
    warm, srt = _timed(torch, lambda: block_merge(eng, multi_sort(eng, bv, scfg)))
    out["sort_n1024_tie_corrected_s"] = {
        "latency_s": first, "warm_latency_s": warm,
        "order_ok": bool(np.array_equal(np.argsort(srt), np.arange(1024))),
        "max_abs_err": float(np.abs(srt - np.sort(v1024)).max()),
        "cost": cost, "params": "long58", "gpus": 1}
    del eng, bv
    torch.cuda.empty_cache()
    return out


def cpu_pipelines(quick=False):
    """CPU time of the same pipelines beside the GPU latencies (rank 0, N=1):
    * ``oracle_engine``: the product's engine over the CPU RNS-CKKS oracle
      (oracle/ckks_oracle.c, OpenMP over all host threads) -- the like-for-like
      CKKS baseline, same circuit, parameters and keys as the GPU run;
    * ``slot_simulator``: oracle/slotsim.py, the reference simulator
      (HESimulator, reference engine.py:133-328) restated in numpy, single thread:
      the reference's own CPU path (float64 slots, no cryptography)."""
    import paper_2412_15126_b200 as M
    from oracle.oracle import oracle_engine
    from oracle.slotsim import SimParams, SlotSim
    from paper_2412_15126_b200.params import preset

    threads = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    out = {"cores": threads, "nproc": os.cpu_count()}
    v16 = np.random.default_rng(0).choice(64, 16, replace=False) / 64
    v128 = np.random.default_rng(0).choice(1024, 128, replace=False) / 1024
    v1024 = np.random.default_rng(0).choice(8192, 1024, replace=False) / 8192
    cfg = M.KernelConfig(mode="composite", composite=(4, 2))

    def wall(fn):
        t0 = time.perf_counter()
        fn()
        return time.perf_counter() - t0

    # oracle engine (CKKS on the CPU): cfg1 rank N=16 whole; cfg3 rank N=128 whole
    for name, preset_name, v, n in (("rank_n16_cfg1", "cfg1", v16, 16), ("rank_n128_cfg3", "cfg3", v128, 128)):
        if quick and n > 16:
            continue
        e = oracle_engine(preset(preset_name))
        ct = e.encrypt(v)
        first = wall(lambda: M.rank(e, ct, n, cfg))  # includes this pipeline's key generation
        warm = wall(lambda: M.rank(e, ct, n, cfg))
        out[f"oracle_engine_{name}_s"] = {"latency_s": warm, "first_run_s": first, "threads": threads}
        del e
    # the reference simulator restated (slot arithmetic only, single thread)
    sims = {}
    s1 = SlotSim(SimParams(2048, 22))
    sims["rank_n16_cfg1"] = lambda: M.rank(s1, s1.encrypt(v16), 16, cfg)
    s3 = SlotSim(SimParams(32768, 29))
    sims["rank_n128_cfg3"] = lambda: M.rank(s3, s3.encrypt(v128), 128, cfg)
    sl = SlotSim(SimParams(32768, 56))
    cfg4 = M.KernelConfig(mode="composite", composite=(4, 2), indicator_composite=(4, 2),
                          tie_margin=2.0 ** -11, goldschmidt_iters=8)
    sims["argmax_value_n128"] = lambda: M.order_statistic_value(sl, sl.encrypt(v128), 128, M.StatisticQuery("max"), cfg4)
    scfg = M.SortConfig(kernel=M.KernelConfig(mode="composite", composite=(6, 2), indicator_composite=(6, 2)),
                        tie_correction=False)
    sims["sort_n1024"] = lambda: M.multi_sort(sl, M.block_split(sl, v1024), scfg)
    for name, fn in sims.items():
        fn()  # warm-up (coefficient caches)
        out[f"slot_simulator_{name}_s"] = min(wall(fn) for _ in range(3))
    return out


def _graph_latency(eng, fn, x, warmup=1, reps=3):
    """Seconds per replay of fn(x) captured as one CUDA graph (graphs.CapturedPipeline);
    the replay's output limbs are checked equal to an eager run's."""
    import torch

    from paper_2412_15126_b200.graphs import CapturedPipeline, _datas

    ref = [d.clone() for d in _datas(fn(x))]
    cap = CapturedPipeline(eng, fn, x, warmup=warmup)
    cap.replay(x)
    torch.cuda.synchronize()
    if not all(torch.equal(a, b) for a, b in zip(_datas(cap.output), ref)):
        raise AssertionError("CUDA-graph replay differs from the eager pipeline")
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        cap.replay(x)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    cap.close()
    return best


def gpu_arm(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank_id = int(os.environ.get("RANK", "0"))
    # one GPU per rank; SRK_DIST_BACKEND=gloo (host-side collectives) lets the
    # N>1 path be exercised with several ranks sharing one GPU in a functional test
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("SRK_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    barrier = (lambda: dist.barrier()) if world > 1 else None

    step = PrimitiveStep(torch, local)
    p = step.p
    parts, ks_bytes = algorithmic_bytes(p)
    step_bytes = sum(parts.values())

    for _ in range(args.warmup):
        step.step()
    torch.cuda.synchronize()
    step.launch_count = 0
    k0 = step.lib.srk_kernel_launches()
    with ClockSampler(local) as clk:
        ms = time_region(torch, step.step, args.steps, barrier)
    launches = step.launch_count // args.steps
    kernels = (step.lib.srk_kernel_launches() - k0) // args.steps
    t = torch.tensor([ms], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())

    # per-kernel-family timing for the roofline (same stream, CUDA events)
    ntt_ms = time_region(torch, lambda: step.ntt(step.x, False), 5)
    intt_ms = time_region(torch, lambda: step.ntt(step.x, True), 5)
    ks_ms = time_region(torch, step.relin_batch, 3)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    fp64_roof = fp64_roofline(torch, step.lib, p, ntt_ms, parts["ntt_fwd"], float(peaks.get("hbm_gbs", 6650.0)))

    # e2e: host pinned inputs -> device, step, results -> host (chunk-pipelined)
    e2e_step = PipelinedE2E(torch, step, chunks=int(os.environ.get("SRK_E2E_CHUNKS", "6")))
    step.step()
    ref_res = step.res.cpu()  # the unchunked step's results
    e2e_step()
    torch.cuda.synchronize()
    assert torch.equal(e2e_step.host_out, ref_res), "pipelined e2e result differs from the full step"
    e2e_ms = time_region(torch, e2e_step, max(1, min(args.steps, 3)), barrier)
    te = torch.tensor([e2e_ms], device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te.item())
    host_x, host_out = e2e_step.host_x, e2e_step.host_out

    pipelines = None
    if not args.no_pipelines:
        del step
        torch.cuda.empty_cache()
        if rank_id == 0:
            pipelines = run_pipelines(torch, quick=args.quick or world > 1)
        if world > 1:
            dist.barrier()
            sharded = run_sharded_sort(torch, dist) if not args.quick else None
            if rank_id == 0 and sharded is not None:
                pipelines.update(sharded)

    if rank_id == 0:
        peak = float(peaks.get("hbm_gbs", 6650.0))
        ntt_gbs = parts["ntt_fwd"] / (ntt_ms * 1e-3) / GB
        ks_gbs = ks_bytes / (ks_ms * 1e-3) / GB
        ntt_src, ntt_tr = ntt_traffic()
        ks_src, ks_tr = keyswitch_traffic()
        value = world * step_bytes / (ms * 1e-3) / GB
        line = {
            "metric": "NTT+KeySwitch GB/s vs HBM roof (cfg2 primitive step, 64 ct, ring 2^16, 30+3 limbs)",
            "value": round(value, 2),
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms, 3),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "u64 (RNS limbs mod 40/60-bit primes)",
            "data": "synthetic: uniform limbs mod each prime, seeded (BASELINE cfg 2)",
            "config": bench_config(p),
            "gpu_launches": int(kernels),
            "api_calls_per_step": launches,
            "roofline": {"bound": "hbm", "kernel": "forward NTT (ntt_pass_kernel x2 per chunk)",
                         "achieved": round(ntt_gbs, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(ntt_gbs / peak, 4), "traffic": ntt_tr,
                         "traffic_source": ntt_src,
                         "algorithmic_bytes": parts["ntt_fwd"], "ms": round(ntt_ms, 4),
                         "peak_source": ("MEASURED_PEAKS.json hbm_gbs (measured copy)" if "gpu_name" in peaks
                                         else "B200_PROFILING.md fallback (no MEASURED_PEAKS.json)")},
            "kernel_roofline": kernel_roofline(),
            "roofline_fp64": fp64_roof,
            "roofline_pipes": pipe_roofline(),
            "roofline_keyswitch": {"bound": "hbm", "unit_of_work": "64 x HMult+relinearise (no rescale)", "achieved": round(ks_gbs, 1), "peak": peak,
                                   "unit": "GB/s", "frac": round(ks_gbs / peak, 4),
                                   "algorithmic_bytes": ks_bytes, "ms": round(ks_ms, 4),
                                   "traffic": ks_tr, "traffic_source": ks_src,
                                   "traffic_over_algorithmic": round(ks_tr / ks_bytes, 2) if ks_tr else None},
            "roofline_inverse_ntt": {"achieved": round(parts["ntt_inv"] / (intt_ms * 1e-3) / GB, 1),
                                     "ms": round(intt_ms, 4)},
            "e2e": {"value": round(world * step_bytes / (e2e_ms * 1e-3) / GB, 2), "unit": "GB/s",
                    "h2d_bytes_per_step": int(host_x.numel() * 8),
                    "d2h_bytes_per_step": int(host_out.numel() * 8), "ms_per_step": round(e2e_ms, 3),
                    "pipeline": f"{len(e2e_step.bounds)} chunks: H2D / compute / D2H on three streams",
                    "outputs_copied": "the 64 rescaled ciphertexts (d2h); the other 16 output sets of the step "
                                      "(forward/inverse NTT in place, 64 products, 15 x 64 rotations) stay resident "
                                      "in HBM as the inputs of the next op, as in a pipeline"},
            "clocks": clk.summary(),
            "pipelines": pipelines,
        }
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args)
            if pipelines is not None and world == 1:
                try:
                    line["cpu_pipelines"] = cpu_pipelines(quick=args.quick)
                except Exception as e:  # never blocks the GPU line
                    line["cpu_pipelines"] = {"failed": str(e)}
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ----------------------------------------------------------------------
# CPU arms (oracle)
# ----------------------------------------------------------------------
def cpu_sample(threads=None, n_ct=4, rotations=len(ROT_STEPS)):
    """Time the oracle on a bounded sample of the step (n_ct ciphertexts through the
    whole primitive set, all 15 rotations); GB/s of the same metric, with the
    algorithmic bytes charged per ciphertext exactly as on the GPU arm
    (step bytes x n_ct / 64: the evaluation keys amortised over the 64)."""
    if threads:
        os.environ["OMP_NUM_THREADS"] = str(threads)
    from oracle.oracle import OracleCKKS
    from paper_2412_15126_b200.params import preset

    p = preset("cfg2")
    o = OracleCKKS(p)
    nl = len(p.q_primes)
    n_all = len(p.all_primes)
    rng = np.random.default_rng(1)

    def rnd(shape_prefix):
        a = np.empty(shape_prefix + (nl, p.ring_degree), dtype=np.uint64)
        for i, q in enumerate(p.q_primes):
            a[..., i, :] = rng.integers(0, q, shape_prefix + (p.ring_degree,), dtype=np.uint64)
        return a

    xs, ys = [rnd((2,)) for _ in range(n_ct)], [rnd((2,)) for _ in range(n_ct)]
    key = np.empty((p.dnum, 2, n_all, p.ring_degree), dtype=np.uint64)
    for i, q in enumerate(p.all_primes):
        key[:, :, i, :] = rng.integers(0, q, (p.dnum, 2, p.ring_degree), dtype=np.uint64)
    L = nl - 1
    t0 = time.perf_counter()
    for x, y in zip(xs, ys):
        f = np.stack([o.ntt(x[k], range(nl)) for k in range(2)])
        np.stack([o.ntt(f[k], range(nl), inverse=True) for k in range(2)])
        prod = o.mul_relin(x, y, key, L)
        # the rotations share one base extension, as on the GPU arm (srk_rotate_hoisted)
        o.rotate_hoisted_raw(x, [key] * rotations,
                             [pow(5, ROT_STEPS[k], 2 * p.ring_degree) for k in range(rotations)], L)
        o.rescale(prod, L)
    dt = time.perf_counter() - t0
    parts, _ = algorithmic_bytes(p)
    share = n_ct / N_CT
    sample_bytes = share * (parts["ntt_fwd"] + parts["ntt_inv"] + parts["hmult_relin"] + parts["rescale"]
                            + parts["rotate_15"] * rotations / len(ROT_STEPS))
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return {"value": round(sample_bytes / dt / GB, 4), "unit": "GB/s", "cores": cores,
            "kind": "port", "seconds": round(dt, 3),
            "sample": f"{n_ct} of the 64 cfg2 ciphertexts through the whole step (fwd+inv NTT, HMult/relin, "
                      f"{rotations} rotations, rescale), bytes charged as {n_ct}/64 of the step "
                      f"(oracle/ckks_oracle.c: OpenMP over limbs, Shoup twiddles, hardware 128/64 division for "
                      f"general products, hoisted rotations)"}


def cpu_baseline(args, threads=None):
    try:
        return cpu_sample(threads=threads, n_ct=2 if args.quick else 8)
    except Exception as e:  # the baseline never blocks the GPU line
        return {"value": None, "unit": "GB/s", "cores": None, "kind": "port", "sample": f"failed: {e}"}


def reference_arm(args):
    from paper_2412_15126_b200.params import preset

    rank_id = int(os.environ.get("RANK", "0"))
    if rank_id != 0:
        return
    vals, secs = [], []
    res = None
    for _ in range(args.warmup if args.warmup < 2 else 1):
        cpu_sample(n_ct=1)
    for _ in range(args.steps):
        res = cpu_sample(n_ct=2)  # two ciphertexts of the step per timed step (bounded run time)
        vals.append(res["value"])
        secs.append(res["seconds"])
    v = float(np.median(vals))
    line = {
        "metric": "NTT+KeySwitch GB/s vs HBM roof (cfg2 primitive step, 64 ct, ring 2^16, 30+3 limbs)",
        "value": v, "unit": "GB/s", "impl": "reference",
        "ms_per_step": round(1e3 * float(np.median(secs)), 3),
        "step_note": "a timed step is 2 of the 64 ciphertexts through the whole primitive set "
                     "(bounded CPU run); value charges it 2/64 of the step's algorithmic bytes",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u64 (RNS limbs mod 40/60-bit primes)", "data": "synthetic (BASELINE cfg 2)",
        "config": bench_config(preset("cfg2")),
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": res["cores"], "kind": "port",
                         "sample": res["sample"]},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the reference (slotrank) has no CKKS arithmetic; its CPU path for this step is the "
                "RNS-CKKS restatement in oracle/ckks_oracle.c (OpenMP over limbs, Shoup twiddles, "
                "hoisted rotations)",
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--quick", action="store_true", help="rank N=128 only among the pipelines")
    ap.add_argument("--no-pipelines", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        reference_arm(args)
    else:
        gpu_arm(args)


if __name__ == "__main__":
    main()
