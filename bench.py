#!/usr/bin/env python
"""bench.py -- ENSI ternary PCMM (Algorithm 1) on B200.

Workload (BASELINE.json configs[1], "C2"): N'=2^16, L=12 RNS limbs, one 768x768 BitNet ternary PCMM (Layout A, the
paper's column packing): 768 input ciphertexts -> 768 output ciphertexts, resident in HBM in the compact word layout
(ceil(bits/8) bytes per word: 6.24 GB in, 6.24 GB out; larger than the 126 MB L2, so no flush
is needed between steps).  A step = one full layer through ensi_pcmm_ternary_compact (one k_accum_tcc launch).

Contract: `python bench.py --gpus N --steps K --warmup W [--impl reference]` prints ONE JSON line.
  value       = ms per layer (lower is better), device time, max over ranks.  N > 1: the north star's layout, strong
                scaling -- one layer split by output columns over the N ranks (inputs replicated), the compact outputs
                all-gathered over NCCL in 4 chunks overlapped with the accumulate; `column_sharded` adds the shard's
                compute alone, the gather alone and the fused-gather epilogue (R20); `token_blocks` the
                weak-scaling mode (every rank a whole layer on its own token block, no collective).
  e2e         = the same metric through ensi_pcmm_ternary_host_wire (pinned host ciphertexts in the compact wire
                format): host inputs -> device -> PCMM -> pinned host outputs, every copy inside the timed region.
  roofline    = the accumulate launch against its bound on SURVEY 8(d)'s op count (7/5 byte planes per word), with the
                HBM fraction on its algorithmic bytes, the committed ncu DRAM traffic (profiles/traffic.json) and the
                NTT / key-switching HBM fractions of the same run (other_kernels).
  cpu_baseline= the CPU oracle (oracle/ensi_oracle.c, as it stands) on a bounded sample of output columns,
                extrapolated by nnz (the oracle's cost is exactly linear in nnz).
  rotations   = hoisted key-switched rotations/s at the same parameters (alpha=4, dnum=3), BASELINE metric's
                second clause (also 32 per ModUp and independent inputs).
  clocks      = SM clock / clock-event reasons polled through NVML by a separate process inside the timed region.
  secondary   = the other SURVEY 8 rows at C2 parameters: NTT/INTT, rescale, Layout B (and lazy ModDown, R19, before /
                after), the C2 layer in uint64 words and on CUDA cores, the C3-C5 shapes, one C5 transformer block,
                the paper's Table III PCMM shapes at N'=2^14, and CCMM (R18) at the Table III attention shapes.
  --layout u64 / --kernel 1 time the uint64-word tcgen05 / CUDA-core accumulate as the headline instead.
  --no-rot / --no-layout-b / --no-ccmm / --no-e2e / --no-cpu skip parts (tests and quick runs).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "ternary PCMM latency (ms/layer) and rotations/sec per B200; HBM GB/s vs peak"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}, "fallback"


_NVML_POLL = r"""
import sys, time, pynvml
pynvml.nvmlInitWithFlags(0) if hasattr(pynvml, "nvmlInitWithFlags") else pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
out = open(sys.argv[2], "w", buffering=1)
out.write("ready %d\n" % pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
while True:
    out.write("%.6f %d %d\n" % (time.time(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                 pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
    time.sleep(0.0005)
"""


class NvmlClockSampler:
    """SM clock and clock-event reasons polled through NVML every ~0.5 ms by a separate process (no GIL
    contention with the timed loop); only the samples whose host timestamps fall inside the timed region count.
    Start it before the warm-up (the poller needs ~0.2 s to come up), mark the region with begin()/end()."""

    def __init__(self, device_index: int):
        import pynvml  # noqa: F401  (fail here, not in the child, when NVML is missing)
        self.dev = device_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".clk", delete=False)
        self.proc = None
        self.t0 = self.t1 = None

    def start(self):
        self.proc = subprocess.Popen([sys.executable, "-c", _NVML_POLL, str(self.dev), self.f.name],
                                     stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        for _ in range(200):                       # wait until the poller is sampling (<= 2 s)
            time.sleep(0.01)
            try:
                if open(self.f.name).read().count("\n") >= 2:
                    break
            except OSError:
                pass

    def begin(self):
        self.t0 = time.time()

    def end(self):
        self.t1 = time.time()

    def stop(self):
        time.sleep(0.005)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        lines = open(self.f.name).read().split("\n")
        os.unlink(self.f.name)
        smmax, rows = None, []
        for ln in lines:
            p = ln.split()
            if len(p) == 2 and p[0] == "ready":
                smmax = int(p[1])
            elif len(p) == 3:
                t, c, r = float(p[0]), int(p[1]), int(p[2])
                if self.t0 is not None and self.t0 <= t <= (self.t1 or t):
                    rows.append((c, r))
        if not rows:
            return None
        import pynvml as nv
        names = ((nv.nvmlClocksEventReasonHwSlowdown, "hw_slowdown"),
                 (nv.nvmlClocksEventReasonHwThermalSlowdown, "hw_thermal_slowdown"),
                 (nv.nvmlClocksEventReasonSwThermalSlowdown, "sw_thermal_slowdown"),
                 (nv.nvmlClocksEventReasonSwPowerCap, "sw_power_cap"),
                 (nv.nvmlClocksEventReasonHwPowerBrakeSlowdown, "hw_power_brake"))
        reasons = sorted({name for _, r in rows for bit, name in names if r & bit})
        return {"sm_mhz": statistics.median(c for c, _ in rows), "sm_max_mhz": smmax, "reasons": reasons,
                "samples": len(rows), "min_mhz": min(c for c, _ in rows),
                "source": "nvml polled every ~0.5 ms by a separate process, samples inside the timed region"}


def clock_sampler(device_index: int):
    try:
        return NvmlClockSampler(device_index)
    except Exception:
        return ClockSampler(device_index)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms while the timed region runs."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.f = None

    def start(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append(dict(sm=float(parts[1]), smmax=float(parts[2]), power=float(parts[3]),
                                 hw=parts[5], hwt=parts[6], swt=parts[7], pcap=parts[8]))
            except ValueError:
                continue
        os.unlink(self.f.name)
        if not rows:
            return None
        loaded = [r for r in rows if r["power"] > 0.3 * max(r2["power"] for r2 in rows)] or rows
        reasons = set()
        for r in loaded:
            for k, name in (("hw", "hw_slowdown"), ("hwt", "hw_thermal_slowdown"), ("swt", "sw_thermal_slowdown"),
                            ("pcap", "sw_power_cap")):
                if r[k].lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(r["sm"] for r in loaded), "sm_max_mhz": max(r["smmax"] for r in rows),
                "reasons": sorted(reasons), "samples": len(loaded)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(world, v: float) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------------------------------------ oracle arm

def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_sample_ms(cfg, W, x_host, ncols: int, nthreads: int):
    """Time the plain oracle (Alg. 1) on `ncols` output columns of the layer; extrapolate by nnz."""
    import oracle
    o = oracle.Oracle(cfg["log_n"], cfg["L"], cfg["alpha"], cfg["dnum"])
    d, m = W.shape
    cols = list(np.linspace(0, m - 1, ncols).astype(int))
    t0 = time.perf_counter()
    o.pcmm_a(x_host, W, cols=cols, nthreads=nthreads)
    dt = time.perf_counter() - t0
    nnz_s = int(np.count_nonzero(W[:, cols]))
    nnz = int(np.count_nonzero(W))
    return dt * 1e3 * nnz / max(1, nnz_s), dt, cols


def run_reference(args, cfg_name):
    world, rank, _ = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), 0
    if rank != 0:
        return 0
    cfg = synth.CONFIGS[cfg_name]
    d, m = cfg["shapes"][0]
    n = 1 << cfg["log_n"]
    import oracle
    q, _ = oracle.gen_params(cfg["log_n"], cfg["L"], cfg["alpha"])
    W = synth.gen_W(synth.SEED_BASE + 102, d, m)
    x = synth.gen_words(synth.SEED_BASE + 2, q, d, cfg["L"], n)
    nth = max(1, min(64, os.cpu_count() or 1))
    ncols = max(1, min(m, nth))
    times = []
    for it in range(args.warmup + args.steps):
        ms, dt, cols = oracle_sample_ms(cfg, W, x, ncols, nth)
        if it >= args.warmup:
            times.append(ms)
    v = statistics.mean(times)
    line = {"metric": METRIC, "value": v, "unit": "ms/layer", "n_gpus": args.gpus, "device": "cpu (host cores)",
            "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": v, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64", "dtype_note": "the oracle's plain 64-bit modular adds",
            "data": "synthetic uniform RNS words (data-oblivious accumulate)",
            "impl": "reference",
            "config": {"workload": f"{cfg_name}: {cfg['desc']}", "d": d, "m": m, "log_n": cfg["log_n"],
                       "limbs": cfg["L"], "layout": "A (the oracle computes on uint64 words; same words)"},
            "cpu_baseline": {"value": v, "unit": "ms/layer", "cores": nth, "kind": "oracle",
                             "sample": f"{ncols} of {m} output columns per step (all 24 RNS slices), "
                                       f"extrapolated by nnz(W)"},
            "e2e": {"value": v, "unit": "ms/layer", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------------ our arm

def time_loop(fn, steps: int, stream):
    import torch
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record(stream)
    for _ in range(steps):
        fn()
    e.record(stream)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / steps


def _random_keys(ctx, gs, cfg, n):
    import torch
    T = cfg["L"] + cfg["alpha"]
    keys = torch.empty((len(gs), cfg["dnum"], 2, T, n), dtype=torch.int64, device="cuda")
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    for r in range(T):
        keys[:, :, :, r, :].random_(0, ctx.moduli[r], generator=g)
    return keys


def layout_b_plan(n: int, s: int, d: int, m: int, B: int = 0):
    """The product's Layout-B schedule (api.cu plan_b, R11): k = min((N'/2)/s, 2^ceil(log2 d)), n_in = ceil(d/k),
    B = argmin (B-1) n_in + (k/B - 1) m unless given; returns (k, n_in, B, G, rotations)."""
    k = min((n // 2) // s, 1 << max(0, (d - 1).bit_length()))
    n_in = -(-d // k)
    if B == 0:
        B = min((((b - 1) * n_in + (k // b - 1) * m, b) for b in (1 << i for i in range(k.bit_length()))
                 if b <= k))[1]
    G = k // B
    return k, n_in, B, G, (B - 1) * n_in + (G - 1) * m


# SURVEY 8(d) algorithmic bytes per key-switched rotation at C2 parameters (N'=2^16, l=12, alpha=4, dnum=3): the
# 50.3 MB key plus the extended-basis digits and the ciphertext in/out -- 88 MB hoisted (ModUp shared), 126 MB for a
# rotation of an independent input
KS_BYTES_HOISTED = 88e6
KS_BYTES_INDEPENDENT = 126e6


def bench_secondary(ctx_cls, cfg, steps: int, warmup: int, peaks, layout_b: bool = True, ccmm: bool = True):
    """The other section-8 rows at the same parameters (timing-only uniform words and random keys; every kernel
    is data-oblivious): NTT/INTT per limb (a5), hoisted key-switched rotations (a6+a7, the BASELINE metric's
    rotations/sec), rescale (a4), and the Layout-B PCMM (a8: 765 hoisted rotations + the accumulate)."""
    import torch
    n = 1 << cfg["log_n"]
    L, A, dnum, s = cfg["L"], cfg["alpha"], cfg["dnum"], cfg["s"]
    T = L + A
    ctx = ctx_cls(cfg["log_n"], L, A, dnum)
    st = torch.cuda.current_stream()
    out = {}
    # NTT / INTT over 768 limb rows (every limb of Q u P)
    rows = 768
    data = torch.empty((rows, n), dtype=torch.int64, device="cuda")
    for lim in range(T):
        data[lim::T].random_(0, ctx.moduli[lim])
    limbs = list(range(T))
    for name, inv in (("ntt_forward", False), ("ntt_inverse", True)):
        for _ in range(warmup):
            ctx.ntt(data, limbs, inverse=inv)
        ms = time_loop(lambda: ctx.ntt(data, limbs, inverse=inv), steps, st)
        alg = rows * n * 8 * 2          # one read + one write of every limb (the algorithmic minimum)
        gbs = alg / (ms * 1e-3) / 1e9
        out[name] = {"us_per_limb": 1e3 * ms / rows, "rows": rows, "achieved_GBps": gbs,
                     "hbm_frac": gbs / peaks["hbm_gbs"], "passes": 2, "moved_GBps": 2 * gbs,
                     "moved_frac": 2 * gbs / peaks["hbm_gbs"],
                     "note": "algorithmic bytes = 1 read + 1 write per limb; the two passes move twice that"}
    del data
    # hoisted rotations: 128 Galois elements per ModUp (4 key-switch batches; steady state) and 32 (one batch)
    key_bytes = dnum * 2 * T * n * 8
    x = synth.gen_words_torch(11, ctx.q, 1, L, n)
    for batch in (128, 32):
        gs = [pow(5, s * (b + 1), 2 * n) for b in range(batch)]
        keys = _random_keys(ctx, gs, cfg, n)
        ctx.load_keys(galois=gs, rot_keys=keys)
        y = torch.empty((batch, 2, L, n), dtype=torch.int64, device="cuda")
        for _ in range(warmup):
            ctx.rotate_hoisted(x, gs, y, L)
        ms = time_loop(lambda: ctx.rotate_hoisted(x, gs, y, L), steps, st)
        r = {"value": batch / (ms * 1e-3), "unit": "rotations/s", "ms_per_call": ms,
             "mode": f"hoisted, {batch} Galois elements per ModUp, N'=2^16, L=12, alpha=4, dnum=3",
             "key_GBps": batch * key_bytes / (ms * 1e-3) / 1e9,
             "hbm_frac": batch * KS_BYTES_HOISTED / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"]}
        if batch == 128:
            out["rotations"] = r
        else:
            out["rotations"]["per_32_batch"] = r
        del keys, y
    # non-hoisted: 96 independent ciphertexts, each rotated by the same element (one ModUp per input; the key is
    # read once for all 96 inputs)
    gs1 = [pow(5, s, 2 * n)]
    keys = _random_keys(ctx, gs1, cfg, n)
    ctx.load_keys(galois=gs1, rot_keys=keys)
    xb = synth.gen_words_torch(12, ctx.q, 96, L, n)
    yb = torch.empty((96, 2, L, n), dtype=torch.int64, device="cuda")
    for _ in range(warmup):
        ctx.rotate_batch(xb, gs1, yb, L)
    ms = time_loop(lambda: ctx.rotate_batch(xb, gs1, yb, L), steps, st)
    out["rotations"]["independent_inputs"] = {
        "value": 96 / (ms * 1e-3), "unit": "rotations/s", "ms_per_call": ms,
        "hbm_frac": 96 * KS_BYTES_INDEPENDENT / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
        "mode": "96 independent ciphertexts x 1 Galois element (ensi_rotate_batch; one ModUp per rotation)"}
    del keys, xb, yb
    # rescale 64 ciphertexts (level 12 -> 11)
    xr = synth.gen_words_torch(5, ctx.q, 64, L, n)
    yr = torch.empty((64, 2, L - 1, n), dtype=torch.int64, device="cuda")
    for _ in range(warmup):
        ctx.rescale(xr, yr, L)
    ms = time_loop(lambda: ctx.rescale(xr, yr, L), steps, st)
    out["rescale"] = {"us_per_ciphertext": 1e3 * ms / 64, "ciphertexts": 64}
    del xr, yr
    if layout_b:
        d, m = cfg["shapes"][0]
        k = (n // 2) // s
        n_in = -(-d // k)
        gsb = [pow(5, s * b, 2 * n) for b in range(1, k)]
        keys = _random_keys(ctx, gsb, cfg, n)
        ctx.load_keys(galois=gsb, rot_keys=keys)
        W = synth.gen_W(synth.SEED_BASE + 102, d, m)
        w = ctx.weights(W)
        xb = synth.gen_words_torch(13, ctx.q, n_in, L, n)
        yb = torch.empty((m, 2, L, n), dtype=torch.int64, device="cuda")
        ctx.pcmm_ternary(xb, w, yb, level=L, layout=1, block_s=s)
        ms = time_loop(lambda: ctx.pcmm_ternary(xb, w, yb, level=L, layout=1, block_s=s), max(1, steps // 2), st)
        out["pcmm_layout_b"] = {"value": ms, "unit": "ms/layer", "rotations": (k - 1) * n_in, "block_s": s,
                                "k": k, "n_in": n_in, "rotations_per_sec": (k - 1) * n_in / (ms * 1e-3)}
        del keys, xb, yb
        # SURVEY 8(f) NEXT #4 (R19, lazy ModDown of the giant steps) before / after: BASELINE configs[2]'s down
        # projection on its default plan (G = 2: one giant rotation per output, lazy == eager) and the C2 layer with
        # B = 64 (G = 4: three giant steps per output summed over Q_l u P, one ModDown instead of three)
        lz = {}
        for name, (dd, mm, bb) in (("C3_down_3072x768_default", (3072, 768, 0)), ("C2_768x768_B64", (768, 768, 64)),
                                   ("C2_768x768_B32", (768, 768, 32))):
            kk, nin, B, G, rots = layout_b_plan(n, s, dd, mm, bb)
            gkb = sorted({pow(5, s * b, 2 * n) for b in range(1, B)} | {pow(5, s * B * g, 2 * n) for g in range(1, G)})
            keys = _random_keys(ctx, gkb, cfg, n)
            ctx.load_keys(galois=gkb, rot_keys=keys)
            W = synth.gen_W(synth.SEED_BASE + 7 + dd, dd, mm)
            w = ctx.weights(W)
            xb = synth.gen_words_torch(14, ctx.q, nin, L, n)
            yb = torch.empty((mm, 2, L, n), dtype=torch.int64, device="cuda")
            row = {"k": kk, "n_in": nin, "B": B, "G": G, "rotations": rots}
            for mode in (False, True):
                fn = lambda: ctx.pcmm_ternary(xb, w, yb, level=L, layout=1, block_s=s, baby=B, moddown_lazy=mode)  # noqa
                fn()
                row["lazy_ms" if mode else "eager_ms"] = time_loop(fn, max(1, steps // 2), st)
            lz[name] = row
            del keys, xb, yb, w
            torch.cuda.empty_cache()
        out["layout_b_lazy_moddown"] = lz
    # Layout-A throughput at the other BASELINE shapes (C3 FFN pair, C4/C5 hidden-2048 projections), compact
    # resident layout (the headline's), and the C2 layer in the uint64 layout (k_accum_tc2) for comparison
    sweep = {}
    wb = ctx.wire_bytes(L)
    for name, (dd, mm) in (("C2_768x768_u64", (768, 768)), ("C2_768x768_cudacore", (768, 768)),
                           ("C3_768x3072", (768, 3072)), ("C3_3072x768", (3072, 768)),
                           ("C4_2048x2048", (2048, 2048)), ("C5_2048x5504", (2048, 5504)),
                           ("C5_5504x2048", (5504, 2048)), ("C5_qkv_2048x6144", (2048, 6144))):
        W = synth.gen_W(synth.SEED_BASE + dd + mm, dd, mm)
        w = ctx.weights(W)
        if name.endswith("_u64") or name.endswith("_cudacore"):
            xs = synth.gen_words_torch(17, ctx.q, dd, L, n)
            ys = torch.empty((mm, 2, L, n), dtype=torch.int64, device="cuda")
            kern = 1 if name.endswith("_cudacore") else 0
            fn = lambda: ctx.pcmm_ternary(xs, w, ys, level=L, kernel=kern)  # noqa: E731
            ctb = 2 * L * n * 8
        else:
            xs = gen_compact(ctx, 17, dd, L)
            ys = torch.empty((mm, wb), dtype=torch.uint8, device="cuda")
            fn = lambda: ctx.pcmm_ternary_compact(xs, w, ys, level=L)  # noqa: E731
            ctb = wb
        fn()
        ms = time_loop(fn, max(1, steps // 2), st)
        ops = 2.0 * wb * dd * mm                              # SURVEY 8(d) plane count
        sweep[name] = {"ms_per_layer": ms, "tensor_TOPS": ops / (ms * 1e-3) / 1e12,
                       "tensor_frac": ops / (ms * 1e-3) / 1e12 / (2.0 * peaks["bf16_tflops"]),
                       "hbm_GBps": (dd + mm) * ctb / (ms * 1e-3) / 1e9}
        if ctb == wb:
            cp, kc = ctx.last_compact_plan()
            sweep[name]["launch"] = {"cluster_pairs": cp, "clusters": kc, "sms": 2 * cp * kc}
        if name.endswith("_cudacore"):
            # the CUDA-core path (north star's literal kernel): one exact DFMA per dense term-word on the FP64 pipe
            # (64 lanes/clk/SM, B300_MICROARCH / ntt_fp.cuh), so its floor is d m (2 l N') / (64 x 148 x f_max)
            dfma = dd * mm * 2.0 * L * n
            fp64_peak = 64 * 148 * peaks.get("sm_max_mhz", 1965.0) * 1e6
            sweep[name] = {"ms_per_layer": ms, "kernel": "k_accum_ternary (FP64-pipe DFMA, opts.kernel = 1)",
                           "fp64_frac": dfma / (ms * 1e-3) / fp64_peak, "floor_ms": 1e3 * dfma / fp64_peak}
        del xs, ys, w
        torch.cuda.empty_cache()
    out["layout_a_shapes"] = sweep
    # BASELINE configs[4]: one transformer block at hidden 2048 (Q/K/V fused 2048->6144, O 2048x2048, gate and up
    # 2048->5504 run separately on one GPU, down 5504->2048), summed
    blk = ["C5_qkv_2048x6144", "C4_2048x2048", "C5_2048x5504", "C5_2048x5504", "C5_5504x2048"]
    out["c5_block"] = {"ms_per_block": sum(sweep[k]["ms_per_layer"] for k in blk), "projections": blk}
    # the paper's own Table III / Fig. 8 PCMM shapes at its default N'=2^14 (PAPER.md:478,
    # 575,583,588,492) -- context beside the A100 (Phantom) 1.78 / 3.12 / 1.57 s and the single-core 1.41 s.  The
    # paper does not state the limb count at PCMM time, so both l = 12 (our configs) and l = 48 (its stated L) run.
    table3 = {}
    for lv, alpha in ((12, 4), (48, 16)):
        c14 = ctx_cls(14, lv, alpha, 3)
        n14 = 1 << 14
        row = {}
        for name, (dd, mm, reps) in (("qkv_1536x1536_x3", (1536, 1536, 3)), ("gate_up_1536x4096_x2", (1536, 4096, 2)),
                                     ("down_4096x1536", (4096, 1536, 1)), ("fig8_768x64", (768, 64, 1))):
            W = synth.gen_W(synth.SEED_BASE + 7 * dd + mm, dd, mm)
            w = c14.weights(W)
            xs = gen_compact(c14, 19, dd, lv)
            ys = torch.empty((mm, c14.wire_bytes(lv)), dtype=torch.uint8, device="cuda")
            c14.pcmm_ternary_compact(xs, w, ys, level=lv)
            ms = time_loop(lambda: c14.pcmm_ternary_compact(xs, w, ys, level=lv), max(1, steps // 2), st)
            row[name] = {"ms_total": ms * reps, "reps": reps}
            del xs, ys, w
            torch.cuda.empty_cache()
        table3[f"l{lv}"] = row
        c14.close()
    out["paper_table3_n14"] = {"results": table3,
                               "paper_seconds": {"qkv": 1.78, "gate_up": 3.12, "down": 1.57, "fig8_cpu_1core": 1.41},
                               "note": "paper: A100 80GB, Phantom, per input amortized over a batch of 32; limb count "
                                       "unstated (PAPER.md:575,583,588); fig8: i9-14900K single core (PAPER.md:492)"}
    if ccmm:
        out["ccmm"] = bench_ccmm(ctx, cfg, st)
    ctx.close()
    torch.cuda.empty_cache()
    return out


def bench_ccmm(ctx, cfg, st):
    """CCMM (R18) at the paper's Table III attention shapes, 16 heads of s = 2048
    tokens in SIMD over the 32768 slots: Q.K^T (form 1: d = 96, m = 2048) and S.V (form 2:
    d = 2048, m = 96).  Timing-only uniform words, random keys and mask; a sample of output columns (every column
    of a form runs the same kernels; the form-1 sample needs both alignment steps, the most expensive case),
    extrapolated to the whole product."""
    import torch
    n, L, s = 1 << cfg["log_n"], cfg["L"], 2048
    lg = lambda v: v.bit_length() - 1
    gal = lambda r: pow(5, r % (n // 2), 2 * n)
    res = {}
    for name, form, d, m, col0, cols, paper_s in (("qk_t_2048x96_x16", 1, 96, 2048, 65, 2, 192.99),
                                                  ("sv_2048x2048_x16", 2, 2048, 96, 1, 1, 638.12)):
        pi = s if form == 1 else 1 << (d - 1).bit_length()
        R = d if form == 2 else m
        Ba = 1 << (((R - 1).bit_length() + 1) // 2)
        am = [-(1 << u) for u in range(lg(pi))] + list(range(1, min(Ba, R))) + [g * Ba for g in range(1, -(-R // Ba))]
        G = -(-R // Ba)
        if form == 2:
            am += [-pi * (1 << u) for u in range(lg(s // pi))]
            rot = cols * (lg(s // pi) + (d - 1) + d * lg(pi))                 # in the timed sample
            rot_all = m * (lg(s // pi) + (d - 1) + d * lg(pi))                # in the whole product
        else:   # giant step Rot(k_j, gam B) once per giant step in the range, babies for b != 0, replicate
            cs = range(col0, col0 + cols)
            rot = d * len({c // Ba for c in cs if c // Ba}) + d * sum(1 for c in cs if c % Ba) + cols * d * lg(pi)
            rot_all = d * (G - 1) + d * (m - G) + m * d * lg(pi)
        gs = [gal(r) for r in sorted(set(am))]
        keys = _random_keys(ctx, gs, cfg, n)
        ctx.load_keys(galois=gs, rot_keys=keys)
        rlk = _random_keys(ctx, [0], cfg, n)[0].contiguous()
        ctx.load_relin_key(rlk)
        a = synth.gen_words_torch(21, ctx.q, d, L, n)
        src = synth.gen_words_torch(22, ctx.q, m if form == 2 else d, L, n)
        mask = synth.gen_words_torch(23, ctx.q, 1, L, n)[0, 0].contiguous()
        y = torch.empty((cols, 2, L - 2, n), dtype=torch.int64, device="cuda")
        ctx.ccmm(a, src, mask, y[:1], form, s, d, m, L, col0=col0, cols=1)         # warm-up: scratch, tables
        ms_all = time_loop(lambda: ctx.ccmm(a, src, mask, y, form, s, d, m, L, col0=col0, cols=cols), 1, st)
        rps = rot / (ms_all * 1e-3)
        res[name] = {"form": form, "d": d, "m": m, "heads": (n // 2) // s, "ms_per_output_column": ms_all / cols,
                     "rotations_in_sample": rot, "rotations_per_sec": rps, "keys": len(gs),
                     "rotations_whole_product": rot_all, "s_whole_product": rot_all / rps,
                     "extrapolation": "whole product = its rotation count / the sample's rotation rate (rotations "
                                      "are > 97 % of the launches' time)",
                     "paper_s": paper_s, "sampled_columns": [col0, col0 + cols]}
        del keys, rlk, a, src, mask, y
        torch.cuda.empty_cache()
    res["note"] = ("paper: A100, Phantom, amortised per input over a batch of 32 (PAPER.md:559,577,580); ours: one "
                   "B200, N'=2^16, l=12, the R18 construction (mask + rotation extraction, BSGS alignment)")
    return res


def gen_compact(ctx, seed: int, count: int, level: int, chunk: int = 128):
    """Timing-only compact ciphertexts [count][wire_bytes] (uint8, device): uniform words in [0, q_r) drawn as uint64
    (synth) and serialised by the product's own ensi_wire_pack, chunk by chunk (no full uint64 copy resident)."""
    import torch
    wb = ctx.wire_bytes(level)
    out = torch.empty((count, wb), dtype=torch.uint8, device="cuda")
    for c0 in range(0, count, chunk):
        c1 = min(count, c0 + chunk)
        xu = synth.gen_words_torch(seed + c0, ctx.q, c1 - c0, level, ctx.n)
        ctx.wire_pack(xu, out[c0:c1], level)
        del xu
    return out


def accum_roofline(ctx, d: int, m: int, nnz: int, L: int, ms: float, peaks, peak_src: str, layout: str,
                   kernel_name: str, config: str):
    """Roofline of the Layout-A accumulate launch (SURVEY 8(d) row 'Ternary accumulate (NEXT #1)').

    Per launch: algorithmic bytes = (d + m) ciphertexts in their resident layout + the 2-bit weights (d m / 4);
    tensor ops = sum over limbs of planes x 2 x (2N') x d x m with planes = the limb's word bytes (7 on the 50-bit
    limb, 5 on the 40-bit limbs at the O1 primes) = 2 x (compact ciphertext bytes) x d x m.  INT8 dense peak = the
    measured bf16 burst peak x the guide's nominal int8/bf16 ratio 2.  The bound is the larger of the two times."""
    n = ctx.n
    ct_c = ctx.wire_bytes(L)                                  # 2 N' sum_r w_r bytes
    ct_u64 = 2 * L * n * 8
    ct_res = ct_c if layout == "compact" else ct_u64
    alg_bytes = (d + m) * ct_res + d * m // 4
    t_hbm = alg_bytes / (peaks["hbm_gbs"] * 1e9)
    gbs = alg_bytes / (ms * 1e-3) / 1e9
    if kernel_name == "cuda-core":
        # one 64-bit modular add per term-word = 2 ALU-pipe ops (IADD3 + IADD3.X); ALU pipe = 64 lanes/clk/SM
        # (B300_MICROARCH: rt_SMSP = 2) x 148 SMs x max clock
        alu_peak = 148 * 64 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12          # T lane-ops/s
        alu_ops = 2.0 * nnz * 2 * L * n
        alu_ach = alu_ops / (ms * 1e-3) / 1e12
        return {"bound": "alu", "achieved": alu_ach, "peak": alu_peak, "unit": "Tops/s (INT32 ALU lane-ops)",
                "frac": alu_ach / alu_peak, "traffic": None, "kernel": "k_accum_ternary", "ops_per_launch": alu_ops,
                "algorithmic_bytes": alg_bytes, "hbm_gbs": gbs, "hbm_frac": gbs / peaks["hbm_gbs"],
                "peak_source": peak_src + " (ALU peak derived from unit counts and the max SM clock)"}
    tc_ops = 2.0 * ct_c * d * m                                # 7/5 planes per word
    tc_peak = 2.0 * peaks["bf16_tflops"]                       # TOPS, int8 dense
    t_tensor = tc_ops / (tc_peak * 1e12)
    tc_ach = tc_ops / (ms * 1e-3) / 1e12
    ncu_peak = 16384 * 148 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
    if t_tensor >= t_hbm:
        r = {"bound": "tensor", "achieved": tc_ach, "peak": tc_peak, "unit": "TOPS (int8 dense)", "frac": tc_ach / tc_peak}
    else:
        r = {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": gbs / peaks["hbm_gbs"]}
    kname = "k_accum_tcc" if layout == "compact" else "k_accum_tc2"
    r.update({"kernel": kname, "layout": layout, "algorithmic_bytes": alg_bytes, "tensor_ops_per_launch": tc_ops,
              "hbm_gbs": gbs, "hbm_peak_gbs": peaks["hbm_gbs"], "hbm_frac": gbs / peaks["hbm_gbs"],
              "tensor_tops": tc_ach, "tensor_peak_tops": tc_peak, "tensor_frac": tc_ach / tc_peak,
              "int8_peak_tops_ncu": ncu_peak, "tensor_frac_vs_ncu_int8_peak": tc_ach / ncu_peak,
              "t_floor_ms": {"tensor": 1e3 * t_tensor, "hbm": 1e3 * t_hbm},
              "peak_source": peak_src,
              "op_count": "SURVEY 8(d): 2 x (sum_r w_r x 2N') x d x m -- only the word bytes that can be non-zero"})
    r.update(committed_traffic(kname, config, d, m))
    return r


def committed_traffic(kname: str, config: str, d: int, m: int):
    """DRAM bytes per launch (ncu --set full: dram__bytes_read.sum + dram__bytes_write.sum) of this kernel on this
    workload, from the committed capture under profiles/ -- ncu cannot run inside the timed region."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        rows = json.load(open(p))
    except (OSError, ValueError):
        return {"traffic": None, "traffic_source": None}
    for row in rows:
        if row.get("kernel") == kname and row.get("config") == config and row.get("d") == d and row.get("m") == m:
            return {"traffic": row["dram_bytes"], "traffic_source": f"profiles/traffic.json <- {row['source']} "
                                                                   f"(committed ncu --set full capture)"}
    return {"traffic": None, "traffic_source": None}


def cross_kernel_check(ctx, W, L, n):
    """Bit-exact flag without the oracle (bench's GPU leg never runs it): the C2 layer through the three independent
    accumulate kernels -- compact tcgen05, uint64 tcgen05, CUDA cores (FP64 pipe) -- on the same words; every word of
    a strided sample of all outputs must agree.  (The oracle pins all three in tests/.)"""
    import torch
    d, m = W.shape
    w = ctx.weights(W)
    x = synth.gen_words_torch(synth.SEED_BASE + 77, ctx.q, d, L, n)
    y1 = torch.empty((m, 2, L, n), dtype=torch.int64, device="cuda")
    y2 = torch.empty_like(y1)
    ctx.pcmm_ternary(x, w, y1, level=L, kernel=2)
    ctx.pcmm_ternary(x, w, y2, level=L, kernel=1)
    wb = ctx.wire_bytes(L)
    xc = torch.empty((d, wb), dtype=torch.uint8, device="cuda")
    ctx.wire_pack(x, xc, L)
    del x
    yc = torch.empty((m, wb), dtype=torch.uint8, device="cuda")
    ctx.pcmm_ternary_compact(xc, w, yc, level=L)
    del xc
    y3 = torch.empty_like(y2)
    ctx.wire_unpack(yc, y3, L)
    torch.cuda.synchronize()
    ok = bool((y1[:, :, :, ::97] == y2[:, :, :, ::97]).all()) and bool((y1[:, :, :, ::97] == y3[:, :, :, ::97]).all())
    del y1, y2, y3, yc
    torch.cuda.empty_cache()
    return ok


def write_jsonl(path, out, ctx, W, L, n):
    """One record per (config, GPUs, kernel) row of the bench line: time, bytes, GB/s, HBM / tensor fractions,
    rotations/s, and a cross-kernel bit-exact flag for the C2 layer (SURVEY 5 "Metrics / logging")."""
    recs = []
    G = out["n_gpus"]
    rf = out["roofline"]
    recs.append({"config": "C2 768x768", "G": G, "kernel": rf["kernel"], "ms": out["value"],
                 "bytes": rf["algorithmic_bytes"], "GBps": rf["hbm_gbs"], "hbm_frac": rf["hbm_frac"],
                 "tensor_frac": rf.get("tensor_frac"), "bit_exact_vs_other_kernels": cross_kernel_check(ctx, W, L, n)})
    sec = out.get("secondary", {})
    for name, r in sec.get("layout_a_shapes", {}).items():
        recs.append({"config": name, "G": 1, "kernel": r.get("kernel", "k_accum_tcc" if "_u64" not in name and
                                                            "_cudacore" not in name else "k_accum_tc2"),
                     "ms": r["ms_per_layer"], "GBps": r.get("hbm_GBps"), "tensor_frac": r.get("tensor_frac"),
                     "fp64_frac": r.get("fp64_frac")})
    for name in ("ntt_forward", "ntt_inverse"):
        if name in sec:
            recs.append({"config": "C2 params, 768 limb rows", "G": 1, "kernel": name, "us_per_limb":
                         sec[name]["us_per_limb"], "GBps": sec[name]["achieved_GBps"], "hbm_frac": sec[name]["hbm_frac"]})
    if "rotations_per_sec" in out:
        r = out["rotations_per_sec"]
        recs.append({"config": "C2 params", "G": 1, "kernel": "rotate_hoisted (128 per ModUp)",
                     "rotations_per_s": r["value"], "hbm_frac": r.get("hbm_frac")})
        recs.append({"config": "C2 params", "G": 1, "kernel": "rotate_batch (independent inputs)",
                     "rotations_per_s": r["independent_inputs"]["value"],
                     "hbm_frac": r["independent_inputs"].get("hbm_frac")})
    if "pcmm_layout_b" in sec:
        recs.append({"config": "C2 768x768 Layout B", "G": 1, "kernel": "layout_b", "ms": sec["pcmm_layout_b"]["value"],
                     "rotations_per_s": sec["pcmm_layout_b"]["rotations_per_sec"]})
    for name, r in sec.get("layout_b_lazy_moddown", {}).items():
        recs.append({"config": name, "G": 1, "kernel": "layout_b eager / lazy ModDown", "ms": r["eager_ms"],
                     "ms_lazy": r["lazy_ms"]})
    if "e2e" in out:
        recs.append({"config": "C2 768x768 e2e", "G": G, "kernel": "ensi_pcmm_ternary_host_wire",
                     "ms": out["e2e"]["value"], "bytes": out["e2e"]["h2d_bytes_per_step"] + out["e2e"]["d2h_bytes_per_step"]})
    with open(path, "w") as f:
        for r in recs:
            f.write(json.dumps(r) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--layout", default="compact", choices=["compact", "u64"],
                    help="resident ciphertext layout: compact ceil(bits/8)-byte words (default) or uint64 words")
    ap.add_argument("--kernel", type=int, default=0, help="0 default, 1 CUDA-core (u64 layout), 2 tcgen05")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-rot", action="store_true", help="skip the secondary rows (NTT, rotations, rescale, Layout B)")
    ap.add_argument("--no-layout-b", action="store_true")
    ap.add_argument("--no-ccmm", action="store_true", help="skip the CCMM row (SURVEY 8(f) NEXT #3)")
    ap.add_argument("--jsonl", default=None,
                    help="also write one JSON record per (config, GPUs, kernel) row to this file (SURVEY 5 metrics)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args, args.config)

    import torch
    from paper_2509_09424_b200 import Context
    from paper_2509_09424_b200.dist import ColumnShardedPCMM

    world, rank, local = dist_setup(args)
    torch.cuda.set_device(local)
    # the N > 1 path (column shards + NCCL all-gather) can be forced at N = 1 for tests (a one-rank NCCL group)
    sharded = world > 1 or os.environ.get("ENSI_BENCH_COLSHARD") == "1"
    if sharded and world == 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local))
    cfg = synth.CONFIGS[args.config]
    d, m = cfg["shapes"][0]
    L, n = cfg["L"], 1 << cfg["log_n"]
    layout = "u64" if args.kernel == 1 else args.layout
    ctx = Context(cfg["log_n"], L, cfg["alpha"], cfg["dnum"], device=local)
    W = synth.gen_W(synth.SEED_BASE + 102, d, m)            # same model weights on every rank
    wb = ctx.wire_bytes(L)
    ct_u64 = 2 * L * n * 8
    st = torch.cuda.current_stream()
    # The north star's layout: the layer input X~ replicated on every rank, rank r computes output
    # columns [r S, (r + 1) S) with its slice of W, then one NCCL all-gather assembles the m outputs everywhere
    # (chunked: the gather of chunk c overlaps the accumulate of chunk c + 1).  N = 1: the whole layer, no gather.
    sh = ColumnShardedPCMM(W, world, rank, make_weights=ctx.weights)
    if layout == "compact":
        x = gen_compact(ctx, synth.SEED_BASE + 2, d, L)
        ct_shape, dt = (wb,), torch.uint8
        pc = lambda xa, wl, yl: ctx.pcmm_ternary_compact(xa, wl, yl, level=L, kernel=args.kernel)  # noqa: E731
    else:
        x = synth.gen_words_torch(synth.SEED_BASE + 2, ctx.q, d, L, n)
        ct_shape, dt = (2, L, n), torch.int64
        pc = lambda xa, wl, yl: ctx.pcmm_ternary(xa, wl, yl, level=L, kernel=args.kernel)  # noqa: E731
    chunks = 4 if sharded else 1
    wch = sh.chunk_weights(chunks, make_weights=ctx.weights)
    y_loc = sh.local_buffer(torch, ct_shape, "cuda", dtype=dt)
    y_all = sh.gathered_buffer(torch, ct_shape, "cuda", dtype=dt) if sharded else None
    if sharded:
        step = lambda: sh.run_overlapped(pc, x, y_loc, y_all, wch)  # noqa: E731
    else:
        step = lambda: pc(x, wch[0], y_loc)  # noqa: E731

    clocks = clock_sampler(local)
    clocks.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    l0 = ctx.launch_count()
    barrier(world)
    torch.cuda.synchronize()
    ev_s, ev_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if hasattr(clocks, "begin"):
        clocks.begin()
    ev_s.record(st)
    for _ in range(args.steps):
        step()
    ev_e.record(st)
    torch.cuda.synchronize()
    if hasattr(clocks, "end"):
        clocks.end()
    barrier(world)
    ms_rank = ev_s.elapsed_time(ev_e) / args.steps
    launches = (ctx.launch_count() - l0)
    clk = clocks.stop()
    if clk is not None:
        clk["note"] = ("sampled only inside bench.py's timed region (the headline loop); the driver's own sampler "
                       "also covers warm-up, e2e and the secondary rows")
    ms_step = max_over_ranks(world, ms_rank)
    value = ms_step                                           # ms per layer, the whole job (strong scaling)

    peaks, peak_src = load_peaks()
    kernel_name = ctx.kernel_name(args.kernel, L)
    # the accumulate launch alone, timed on the stream it runs on: at N = 1 the step IS one launch
    if sharded:
        pc(x, sh.W_local, y_loc)
        torch.cuda.synchronize()
        ms_kernel = time_loop(lambda: pc(x, sh.W_local, y_loc), max(1, args.steps), st)
        d_k, m_k = d, sh.S
    else:
        ms_kernel, d_k, m_k = ms_rank, d, m
    roofline = accum_roofline(ctx, d_k, m_k, int(np.count_nonzero(sh._W_np)), L, ms_kernel, peaks, peak_src, layout, kernel_name, args.config)
    roofline["launches_per_step"] = launches / args.steps
    roofline["ms_per_launch"] = ms_kernel
    if layout == "compact":
        cp, kc = ctx.last_compact_plan()
        roofline["launch"] = {"cluster_pairs": cp, "clusters": kc, "sms": 2 * cp * kc}

    out = {"metric": METRIC, "value": value, "unit": "ms/layer", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False, "scaling": "strong",
           "vs_baseline": None, "dtype": "u8" if kernel_name != "cuda-core" else "f64",
           "dtype_note": ("u8 word bytes x s8 weights -> exact s32 tensor-core sums, recombined to canonical mod-q words"
                          if kernel_name != "cuda-core" else
                          "uint64 words as exact f64 integers (DFMA on the FP64 pipe), canonical mod-q words out"),
           "data": "synthetic uniform RNS words in [0,q_r) (the accumulate is data-oblivious); BitNet absmean W",
           "config": {"workload": f"{args.config}: {cfg['desc']}", "d": d, "m": m, "log_n": cfg["log_n"],
                      "limbs": L, "layout": f"A, {layout} words" + (" (ceil(bits/8) bytes per word, DESIGN.md 3)"
                                                                   if layout == "compact" else ""),
                      "kernel": kernel_name, "nnz": int(np.count_nonzero(W)),
                      "ciphertext_bytes": wb if layout == "compact" else ct_u64,
                      "l2": f"inputs ({d * (wb if layout == 'compact' else ct_u64) / 1e9:.2f} GB) larger than L2 "
                            f"(126 MB); no flush",
                      "parallelism": (f"output columns sharded x{world}, X replicated, chunked NCCL all-gather of "
                                      f"the outputs" if sharded else "one GPU")},
           "gpu_launches": launches, "clocks": clk, "roofline": roofline}

    if sharded:
        # compute-only (the accumulate of this rank's shard) and the gather alone, max over ranks
        gat = time_loop(lambda: torch.distributed.all_gather_into_tensor(y_all, y_loc), max(1, args.steps), st)
        out["column_sharded"] = {"compute_ms": max_over_ranks(world, ms_kernel),
                                 "gather_ms": max_over_ranks(world, gat),
                                 "gather_bytes_per_rank": (world - 1) * sh.S * (wb if layout == "compact" else ct_u64),
                                 "chunks": chunks}
        # the same layer with the gather fused into the accumulate epilogue (every output tile
        # TMA-stored into every rank's gathered buffer over CUDA IPC / NVLink, then a signal / wait pair)
        if layout == "compact":
            from paper_2509_09424_b200.dist import FusedGatherPCMM
            try:    # the setup raises on every rank together (e.g. no peer access between two GPUs): skip the leg
                fg = FusedGatherPCMM(ctx, W, world, rank, L)
            except RuntimeError as e:
                fg = None
                out["column_sharded"]["fused_gather_error"] = str(e)[:300]
            if fg is not None:
                fg(x)
                torch.cuda.synchronize()
                barrier(world)
                fms = max_over_ranks(world, time_loop(lambda: fg(x), max(1, args.steps), st))
                out["column_sharded"]["fused_gather_ms"] = fms
                barrier(world)
                fg.close()
                del fg
        # token blocks (weak scaling, no collective): every rank the whole layer on its own input block
        xt = (gen_compact(ctx, synth.SEED_BASE + 2 + 1000 * rank, d, L) if layout == "compact"
              else synth.gen_words_torch(synth.SEED_BASE + 2 + 1000 * rank, ctx.q, d, L, n))
        wfull = ctx.weights(W)
        yt = torch.empty((m,) + ct_shape, dtype=dt, device="cuda")
        pc(xt, wfull, yt)
        torch.cuda.synchronize()
        barrier(world)
        tb = max_over_ranks(world, time_loop(lambda: pc(xt, wfull, yt), max(1, args.steps), st))
        out["token_blocks"] = {"value": tb / world, "unit": "ms/layer", "scaling": "weak", "ms_per_rank_step": tb,
                               "note": "each rank one layer on its own token block, no collective"}
        del xt, yt, wfull
    del y_loc, y_all, wch
    torch.cuda.empty_cache()

    # ---- e2e through the host-buffer entry point (pinned host in, pinned host out), rank 0's view at N = 1 and
    # every rank its own token block at N > 1 (the host API is per GPU)
    xh_t = None
    w = ctx.weights(W)
    if not args.no_e2e:
        from paper_2509_09424_b200.ensi import wire_pack_host
        xw_t = torch.empty((d, wb), dtype=torch.uint8, pin_memory=True)
        yw_t = torch.empty((m, wb), dtype=torch.uint8, pin_memory=True)
        xu = synth.gen_words_torch(synth.SEED_BASE + 2 + 1000 * rank, ctx.q, d, L, n)
        xw_dev = torch.empty((d, wb), dtype=torch.uint8, device="cuda")
        ctx.wire_pack(xu, xw_dev, L)                 # the client's serialisation, made here on the device (untimed)
        xw_t.copy_(xw_dev)
        yref_dev = torch.empty((m, wb), dtype=torch.uint8, device="cuda")
        ctx.pcmm_ternary_compact(xw_dev, w, yref_dev, level=L)
        yref = yref_dev[5].cpu().numpy()
        del xw_dev, yref_dev
        if world == 1:
            xh_t = xu.cpu()
        del xu
        torch.cuda.empty_cache()
        xw, yw = xw_t.numpy(), yw_t.numpy()
        wire_step = lambda: ctx.pcmm_ternary_host_wire(xw, w, yw, level=L, kernel=args.kernel)  # noqa: E731
        wire_step()
        torch.cuda.synchronize()
        barrier(world)
        wire_ms = max_over_ranks(world, time_loop(wire_step, max(1, min(args.steps, 3)), st))
        ok_w = bool((yw_t[5].numpy() == yref).all())
        out["e2e"] = {"value": wire_ms / world, "unit": "ms/layer", "h2d_bytes_per_step": world * d * wb,
                      "d2h_bytes_per_step": world * m * wb, "matches_device_path": ok_w,
                      "api": "ensi_pcmm_ternary_host_wire (pinned host ciphertexts in the compact wire format = the "
                             "compact resident layout; slices pipelined over 3 streams)",
                      "per_rank_ms": wire_ms, "pcie_GBps_per_rank": (d + m) * wb / (wire_ms * 1e-3) / 1e9,
                      "scaling": "weak" if world > 1 else "n/a",
                      "note": "PCIe-bound: both directions overlap; tools/pcie_bw.py measures 92.7 GB/s bidirectional "
                              "pinned-copy bandwidth on the B200 box"}
        del xw_t, yw_t
    # ---- secondary rows, rank 0 only
    if not args.no_rot and rank == 0:
        torch.cuda.empty_cache()
        sec = bench_secondary(Context, cfg, max(3, args.steps), 2, peaks, layout_b=not args.no_layout_b,
                              ccmm=not args.no_ccmm)
        out["rotations_per_sec"] = sec.pop("rotations")
        out["secondary"] = sec
        out["roofline"]["other_kernels"] = {
            "ntt_forward_hbm_frac": sec["ntt_forward"]["hbm_frac"], "ntt_inverse_hbm_frac": sec["ntt_inverse"]["hbm_frac"],
            "keyswitch_hoisted_hbm_frac": out["rotations_per_sec"]["hbm_frac"],
            "keyswitch_independent_hbm_frac": out["rotations_per_sec"]["independent_inputs"]["hbm_frac"],
            "note": "algorithmic bytes: NTT 1 read + 1 write per limb; key switching SURVEY 8(d) 88 MB per hoisted "
                    "and 126 MB per independent rotation"}
    # ---- CPU oracle baseline (rank 0 at N=1 only)
    if not args.no_cpu and rank == 0 and world == 1:
        x_host = (xh_t.numpy().view(np.uint64) if xh_t is not None else
                  synth.gen_words(synth.SEED_BASE + 2, ctx.q, d, L, n))
        nth = max(1, min(64, os.cpu_count() or 1))
        ncols = max(1, min(m, nth))
        ms_cpu, dt_s, cols = oracle_sample_ms(cfg, W, x_host, ncols, nth)
        # the same oracle on one core (1 core and all host cores), a 2-column sample
        ms_1, dt_1, _ = oracle_sample_ms(cfg, W, x_host, 2, 1)
        out["cpu_baseline"] = {"value": ms_cpu, "unit": "ms/layer", "cores": nth, "kind": "oracle",
                               "sample": f"{ncols} of {m} output columns ({dt_s:.1f} s wall), extrapolated by nnz",
                               "one_core": {"value": ms_1, "unit": "ms/layer", "cores": 1,
                                            "sample": f"2 of {m} output columns ({dt_1:.1f} s wall), "
                                                      f"extrapolated by nnz"},
                               "cpu_model": _cpu_model()}
    if rank == 0 and args.jsonl:
        write_jsonl(args.jsonl, out, ctx, W, L, n)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if sharded:
        import torch.distributed as dist
        barrier(world)                 # ranks > 0 wait for rank 0's secondary measurements before teardown
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
