#!/usr/bin/env python
"""Benchmark of the Tarragon MoE-layer round trip (tg_moe_layer) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config NAME]

N = 1 (default): BASELINE.json configs[1], Mixtral-8x7B-shaped layer (d 4096,
8 experts top-2, F 14336), decode batch T = 256, bf16, one B200.
N > 1 (torchrun, one rank per GPU): configs[2], the same layer with experts
sharded as EWs over N GPUs (shadow replicas in residual HBM), T = 256 global
tokens split over the ranks (strong scaling).
A step = one tg_moe_layer call (router -> rank/exchange counts -> dispatch ->
grouped SwiGLU expert GEMMs -> combine) over one synthetic batch.

Prints ONE JSON line (rank 0).  `value` = tokens/s over the K timed steps
(CUDA events on the launching stream, barrier + synchronize on both sides, max
over ranks).  `e2e` = the same metric through tg_moe_layer_host (pinned host
x in, out back to host, copies inside the timed region, pipelined over two
staging buffers).  `roofline` = k_layer (one launch per call) against the roof
its arithmetic intensity reaches first: algorithmic HBM bytes (or FLOPs) per
launch / its mean event-timed duration, against MEASURED_PEAKS.json.
`--impl reference` times the CPU oracle (the tier's reference arm) on a
bounded sample of the same workload.

The default (N = 1, configs[1]) line also carries the north star's other two
numbers, measured in the same run on the same GPU:
  "prefill":  the Qwen1.5-MoE-shaped layer (configs[4] shape: 60 experts
              top-4), prefill batch T = 8192, against the bf16 tensor roof;
  "failover": the EW-failover protocol (SURVEY 8(d), P:1257 for context) on
              the Mixtral-shaped layer with 2 logical EWs and shadow replicas
              (N = 1) or the bench layer's N EWs (N > 1): calls stream, then
              every rank masks EW1 (tg_mask_worker) and NaN-poisons its slots;
              host latency of the mask, reroute latency (mask call -> first
              post-mask call complete), per-call latency before / after, calls
              that errored, and how many post-mask outputs are bitwise those of
              the same inputs before the mask.
`cpu_baseline` adds the oracle on ONE core (sched_setaffinity to one CPU, one
thread) next to the all-core run, with the CPU model, and checks that both
runs give the same output bits.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as wl  # noqa: E402

REASONS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", 0)), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled every ~2 ms during the timed region (NVML, read in a
    thread; nvidia-smi -lms 10 as the fallback when NVML is unavailable)."""

    _NVML_BITS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                  "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.stop = threading.Event()
        self.nvml = None

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        try:  # CUDA and NVML orders can differ: match the PCI location of the CUDA device
            pr = torch.cuda.get_device_properties(self.index)
            want = (int(pr.pci_domain_id), int(pr.pci_bus_id), int(pr.pci_device_id))
            for i in range(pynvml.nvmlDeviceGetCount()):
                hi = pynvml.nvmlDeviceGetHandleByIndex(i)
                pi = pynvml.nvmlDeviceGetPciInfo(hi)
                if (int(pi.domain), int(pi.bus), int(pi.device)) == want:
                    h = hi
                    break
        except Exception:
            pass
        return pynvml, h

    def __enter__(self):
        try:
            self.nvml = self._nvml_handle()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.nvml = None
        q = "clocks.sm,clocks.max.sm," + ",".join("clocks_event_reasons." + r for r in REASONS)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "10"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.15)
        except Exception:
            self.proc = None
        return self

    def _poll(self):
        nv, h = self.nvml
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append([str(sm), str(mx)] + ["Active" if bits & self._NVML_BITS[r] else "Not Active"
                                                          for r in REASONS])
            except Exception:
                pass
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([s.strip() for s in line.split(",")])

    def __exit__(self, *a):
        if self.nvml is not None:
            self.stop.set()
            self.thread.join(timeout=2)
            return
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, active = [], [], set()
        for s in self.samples:
            try:
                sm.append(float(s[0]))
                mx.append(float(s[1]))
            except Exception:
                continue
            for r, v in zip(REASONS, s[2:]):
                if v.lower().startswith("active"):
                    active.add(r)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(active),
                "samples": len(sm), "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def make_weights_device(shape, seed, device, experts):
    """Seeded synthetic weights of the configured architecture (random init), generated on the GPU."""
    d, F = shape.d, shape.F
    L = wl.Layer(shape, wl.bf16_normal((shape.E, d), d ** -0.5, seed * 1000 + 1, device), [None] * shape.E,
                 [None] * shape.E, [None] * shape.E)
    for e in experts:
        L.w1[e] = wl.bf16_normal((F, d), d ** -0.5, seed * 1000 + 10 + 3 * e, device)
        L.w3[e] = wl.bf16_normal((F, d), d ** -0.5, seed * 1000 + 11 + 3 * e, device)
        L.w2[e] = wl.bf16_normal((d, F), F ** -0.5, seed * 1000 + 12 + 3 * e, device)
    if shape.F_sh:
        Fs = shape.F_sh
        L.shared = (wl.bf16_normal((Fs, d), d ** -0.5, seed * 1000 + 2, device),
                    wl.bf16_normal((Fs, d), d ** -0.5, seed * 1000 + 3, device),
                    wl.bf16_normal((d, Fs), Fs ** -0.5, seed * 1000 + 4, device))
    if shape.shared_gate:
        L.wsg = wl.bf16_normal((d,), d ** -0.5, seed * 1000 + 5, device)
    return L


def layer_algorithmic_bytes(shape, slot_rows_active, R_local, T_local):
    """k_layer (the whole round trip, one launch) algorithmic HBM bytes per launch
    on one rank: weights of every slot with rows (3*d*F*2 each) +
    shared weights + router weights + tokens read (T*d*2) + dispatched rows
    written and read (2*R*d*2) + expert outputs written (R*d*2) and read by the
    combine (T*k*d*2) + outputs written (T*d*2)."""
    d = shape.d
    b = slot_rows_active * 3 * d * shape.F * 2
    if shape.F_sh:
        b += 3 * d * shape.F_sh * 2
    b += (shape.E + shape.shared_gate) * d * 2
    b += T_local * d * 2 + 3 * R_local * d * 2 + T_local * shape.k * d * 2 + T_local * d * 2
    return b


def layer_algorithmic_flops(shape, R_local, T_local):
    """k_layer FLOPs per launch on one rank: routed expert FFNs (3 matmuls of d x F per row),
    the shared expert (3 of d x F_sh per token), the router (d x E_r per token)."""
    f = 2 * R_local * 3 * shape.d * shape.F
    f += 2 * T_local * 3 * shape.d * shape.F_sh
    f += 2 * T_local * shape.d * (shape.E + shape.shared_gate)
    return f


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_oracle_sample(shape, L_host, x_host, pl, n_tokens, n_threads, want_out=False):
    """Time the oracle (as it stands) on the first n_tokens of the batch: O1..O8."""
    import oracle
    oracle.build()
    w1 = [wl.as_u16(a) for a in L_host.w1]
    w3 = [wl.as_u16(a) for a in L_host.w3]
    w2 = [wl.as_u16(a) for a in L_host.w2]
    sh = tuple(wl.as_u16(a) for a in L_host.shared) if L_host.shared is not None else None
    xs = wl.as_u16(x_host[:n_tokens])
    t0 = time.perf_counter()
    wsg = wl.as_u16(L_host.wsg) if L_host.wsg is not None else None
    r = oracle.layer(xs, wl.as_u16(L_host.wg), shape.k, w1, w3, w2, pl.cand, pl.ew_rank, pl.slots_per_ew,
                     np.zeros(pl.n_ews, np.uint8), max(pl.ew_rank) + 1, shared=sh, n_threads=n_threads,
                     gate_mode=shape.gate_mode, wsg=wsg)
    dt = time.perf_counter() - t0
    assert r["rc"] == 0
    if want_out:
        return n_tokens / dt, dt, r["out"]
    return n_tokens / dt, dt


def oracle_one_core(shape, L_host, x_host, pl, n_tokens):
    """The oracle single-threaded and pinned to one CPU (taskset -c 0), on the first
    n_tokens; restores this process's affinity afterwards."""
    old = os.sched_getaffinity(0)
    cpu0 = min(old)
    os.sched_setaffinity(0, {cpu0})
    try:
        return cpu_oracle_sample(shape, L_host, x_host, pl, n_tokens, 1, want_out=True)
    finally:
        os.sched_setaffinity(0, old)


def time_calls(tg, layer, xs, outs, stream, n, warm=5):
    """Per-call device times (ms) of n tg_moe_layer calls, events around each call."""
    for i in range(warm):
        tg.tg_moe_layer(layer.ctx, xs[i % len(xs)], outs[i % len(xs)], stream)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for i in range(n):
        evs[i][0].record(stream)
        rc = tg.tg_moe_layer(layer.ctx, xs[i % len(xs)], outs[i % len(xs)], stream)
        if rc != tg.TG_OK:
            raise tg.TarragonError(rc, tg.tg_last_error(layer.ctx))
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def prefill_record(tg, dev, seed, steps):
    """North star: the prefill path against the bf16 tensor roof, on the Qwen1.5-MoE-shaped layer
    (60 experts top-4, F 1408), T = 8192 tokens in one call, one B200."""
    shape = wl.CONFIGS["qwen_prefill"]
    pl = wl.make_placement(shape.E, 1, 1, shadows=False)
    L = make_weights_device(shape, seed, dev, list(range(shape.E)))
    layer = tg.MoELayer(shape, pl, L, max_tokens_per_rank=shape.T, device=dev.index)
    xs = [wl.make_tokens(shape, seed + 17 * i, T=shape.T, device=dev) for i in range(4)]
    outs = [torch.empty_like(xs[0]) for _ in range(4)]
    stream = torch.cuda.current_stream()
    with ClockSampler(dev.index) as clk:
        ts = time_calls(tg, layer, xs, outs, stream, steps, warm=10)
    rt = layer.routing(shape.T)
    R = int(rt["counts"].cpu().numpy()[0].sum())
    flops = layer_algorithmic_flops(shape, R, shape.T)
    ms = float(np.median(ts))
    _, tf_burst, tf_sus, src = peaks()
    tfs = flops / (ms / 1e3) / 1e12
    layer.close()
    del L, xs, outs
    torch.cuda.empty_cache()
    return {"workload": "BASELINE configs[4] shape: qwen_prefill (d=2048, E=60, top-4, F=1408), T=8192, 1 B200",
            "us_per_call": ms * 1e3, "us_per_call_p95": float(np.percentile(ts, 95)) * 1e3,
            "tokens_per_s": shape.T / (ms / 1e3), "calls": len(ts),
            "algorithmic_flops_per_call": flops, "achieved_TFLOPs": tfs,
            "roofline": {"bound": "tensor", "peak": tf_sus, "unit": "TFLOP/s", "frac": tfs / tf_sus,
                         "peak_source": src + " (bf16 sustained)",
                         "frac_of_burst": tfs / tf_burst, "frac_of_nominal_2250": tfs / 2250.0},
            "north_star_bar": ">= 0.5 of bf16 peak", "clocks": clk.summary()}


def failover_record(tg, layer, shape, xs, stream, N, rank, dev, n_calls=40):
    """SURVEY 8(d) EW-failover protocol (BASELINE metric's second half): calls stream with
    rotating inputs, then every rank masks EW1 (tg_mask_worker) and NaN-poisons its slots on its
    rank; the next call is the reroute.  Returns latencies and the bit-identity count."""
    pl = layer.pl
    outs_pre = [torch.empty_like(xs[0]) for _ in xs]
    pre = time_calls(tg, layer, xs, outs_pre, stream, n_calls)
    ref = [o.clone() for o in outs_pre]
    if N > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc = tg.tg_mask_worker(layer.ctx, 1, 1)
    t_mask = time.perf_counter() - t0
    outs_post = [torch.empty_like(xs[0]) for _ in xs]
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0.record(stream)
    rc2 = tg.tg_moe_layer(layer.ctx, xs[0], outs_post[0], stream)
    r1.record(stream)
    torch.cuda.synchronize()
    t_reroute = time.perf_counter() - t0
    first_ms = r0.elapsed_time(r1)
    # fail-stop semantics: nothing may read the masked EW's memory any more
    if pl.ew_rank[1] == rank:
        nan = torch.full((shape.F, shape.d), float("nan"), dtype=torch.bfloat16, device=dev)
        nan2 = torch.full((shape.d, shape.F), float("nan"), dtype=torch.bfloat16, device=dev)
        for sl, e in enumerate(pl.hosted[1]):
            if e >= 0:
                tg.tg_load_experts(layer.ctx, 1, sl, e, nan, nan, nan2)
    if N > 1:
        torch.distributed.barrier()
    post = time_calls(tg, layer, xs, outs_post, stream, n_calls, warm=0)
    ident = sum(int(torch.equal(a.view(torch.int16), b.view(torch.int16))) for a, b in zip(ref, outs_post))
    errors = int(rc not in (tg.TG_OK,)) + int(rc2 != tg.TG_OK)
    return {"protocol": "SURVEY 8(d): mask EW1 on every rank mid-stream, NaN-poison its slots",
            "ews": pl.n_ews, "ranks": N, "mask_host_us": t_mask * 1e6,
            "reroute_ms": t_mask * 1e3 + first_ms, "first_post_mask_call_us": first_ms * 1e3,
            "reroute_host_wall_ms": t_reroute * 1e3,
            "pre_us_per_call": float(np.median(pre)) * 1e3, "post_us_per_call": float(np.median(post)) * 1e3,
            "calls_errored": errors, "post_mask_outputs_bit_identical": ident, "post_mask_outputs_compared": len(ref),
            "paper_context": "EW-failure stall ~0.3 s on H200 + RDMA (P:1257), not comparable hardware"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, help="workloads.CONFIGS key (default mixtral_decode)")
    ap.add_argument("--tokens", type=int, default=None, help="global tokens per call (default: config T)")
    ap.add_argument("--cpu-sample", type=int, default=None, help="tokens in the oracle sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--seed", type=int, default=1001)
    args = ap.parse_args()
    assert args.warmup >= 3, "timing rules: at least 3 warm-up steps"

    rank, world, local = dist_env()
    N = world
    cfg = args.config or "mixtral_decode"
    shape = wl.CONFIGS[cfg]
    T_glob = args.tokens or shape.T
    assert T_glob % N == 0
    T_r = T_glob // N
    W = max(N, 1)
    shadows = N > 1
    pl = wl.make_placement(shape.E, W, N, shadows=shadows)
    cores = os.cpu_count() or 1
    config = {"workload": f"BASELINE configs[{1 if N == 1 else 2}]: {cfg} T={T_glob} global, "
                          f"{W} EW(s){' + shadow replicas' if shadows else ''} on {N} B200",
              "model": f"{cfg} (d={shape.d}, E={shape.E}, top-{shape.k}, F={shape.F}"
                       f"{', F_sh=%d' % shape.F_sh if shape.F_sh else ''})",
              "global_batch": T_glob, "seq_len": 1, "parallelism": f"ep{N}+dp{N}" if N > 1 else "single",
              "l2": "weights (%.2f GB/GPU) >> 126 MB L2, streamed from HBM every step; 8 rotating x batches"
                    % (3 * shape.d * shape.F * 2 * sum(1 for e in range(shape.E)
                                                       if pl.ew_rank[pl.cand[e, 0, 0]] == 0) / 1e9)}

    if args.impl == "reference":
        # Reference arm of this tier: the CPU oracle, rank 0 only.
        if rank != 0:
            return
        n = args.cpu_sample or 16
        L = wl.make_layer(shape, args.seed)
        x = wl.make_tokens(shape, args.seed, T=max(n, 1))
        times = []
        nwarm = args.warmup  # untimed oracle samples of <= 4 tokens (page the oracle in); bounded run time
        for _ in range(nwarm):
            cpu_oracle_sample(shape, L, x, pl, min(n, 4), cores)
        for _ in range(max(1, args.steps if args.steps <= 3 else 3)):
            v, dt = cpu_oracle_sample(shape, L, x, pl, n, cores)
            times.append(dt)
        dt = float(np.median(times))
        val = n / dt
        line = {"impl": "reference", "metric": "MoE-layer tokens/s", "value": val, "unit": "tokens/s",
                "n_gpus": N, "steps": len(times), "warmup": nwarm, "ms_per_step": dt * 1e3,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": config,
                "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                                 "sample": f"first {n} of the batch's tokens, full O1-O8 per step",
                                 "cpu_model": cpu_model()},
                "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import paper_2601_01310_b200 as tg
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if N > 1:
        import torch.distributed as dist
        if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
            os.environ["NCCL_DEBUG"] = "WARN"  # the version banner goes to stdout: one JSON line only
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD
    local_experts = sorted({e for ew in range(W) if pl.ew_rank[ew] == rank for e in pl.hosted[ew] if e >= 0})
    L = make_weights_device(shape, args.seed, dev, local_experts)
    layer = tg.MoELayer(shape, pl, L, max_tokens_per_rank=T_r, rank=rank, world=N, device=local, group=group)
    NB = 8
    xs = [wl.make_tokens(shape, args.seed + 17 * i, T=T_glob, device=dev)[rank * T_r:(rank + 1) * T_r].contiguous()
          for i in range(NB)]
    outs = [torch.empty_like(xs[0]) for _ in range(NB)]
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if N > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def step(i):
        rc = tg.tg_moe_layer(layer.ctx, xs[i % NB], outs[i % NB], stream)
        if rc != tg.TG_OK:
            raise tg.TarragonError(rc, tg.tg_last_error(layer.ctx))

    for i in range(args.warmup):
        step(i)
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        for i in range(args.steps):
            step(i)
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    # per-kernel CUDA events (between the launches of each call, same stream) over a second
    # timed region of the same length: events between the kernels would otherwise sit inside
    # the headline measurement
    tg.tg_set_profiling(layer.ctx, True)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    p0.record(stream)
    for i in range(args.steps):
        step(i)
    p1.record(stream)
    barrier()
    ms_prof = p0.elapsed_time(p1)
    ktimes = tg.tg_get_kernel_times(layer.ctx)
    tg.tg_set_profiling(layer.ctx, False)
    launches = tg.tg_last_launch_count(layer.ctx) * args.steps
    ms_t = torch.tensor([ms], device=dev)
    if N > 1:
        torch.distributed.all_reduce(ms_t, op=torch.distributed.ReduceOp.MAX)
    ms = float(ms_t.item())
    value = T_glob * args.steps / (ms / 1e3)

    # ---- end to end through the public host-buffer entry point
    xh = [x.cpu().pin_memory() for x in xs]
    oh = [torch.empty_like(h).pin_memory() for h in xh]
    for i in range(args.warmup):
        tg.tg_moe_layer_host(layer.ctx, xh[i % NB], oh[i % NB], stream)
    tg.tg_host_sync(layer.ctx, stream)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    tg.tg_host_sync(layer.ctx, stream)  # the timed copies start after e0
    for i in range(args.steps):
        rc = tg.tg_moe_layer_host(layer.ctx, xh[i % NB], oh[i % NB], stream)
        assert rc == tg.TG_OK, tg.tg_last_error(layer.ctx)
    tg.tg_host_sync(layer.ctx, stream)  # ... and end before e1 (every output delivered)
    e1.record(stream)
    barrier()
    ms_e = torch.tensor([e0.elapsed_time(e1)], device=dev)
    if N > 1:
        torch.distributed.all_reduce(ms_e, op=torch.distributed.ReduceOp.MAX)
    e2e_val = T_glob * args.steps / (float(ms_e.item()) / 1e3)

    # ---- roofline of the dominant kernel (GEMM, GK4) on this rank
    st = layer.routing(T_r)
    counts = st["counts"].cpu().numpy()
    rows_local = counts[rank]
    active = int((rows_local > 0).sum())
    R_local = int(rows_local.sum())
    hbm, tf, tf_sus, src = peaks()
    names = tg.KERNEL_NAMES
    kt = dict(zip(names, ktimes))
    g_ms_ser = kt.get("layer", float("nan"))
    # one launch per step: the kernel's average launch duration over the timed region is the
    # step time (consecutive launches overlap under PDL); the profiled pass records events
    # between the launches, which serialises them, so its per-kernel time is reported beside it
    g_ms = (ms / args.steps) if launches == args.steps else g_ms_ser
    gbytes = layer_algorithmic_bytes(shape, active, R_local, T_r)
    achieved = gbytes / (g_ms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get(f"{cfg}:N{N}:T{T_glob}")
    gflops = layer_algorithmic_flops(shape, R_local, T_r)
    tflops = gflops / (g_ms / 1e3) / 1e12
    # the bound is the roof the layer's arithmetic intensity hits first (ridge = peak FLOP/s /
    # peak B/s); the step runs back to back, so the tensor roof is the sustained bf16 figure
    tf_peak = tf_sus if tf_sus > 0 else tf
    tensor_bound = gflops / gbytes > tf_peak * 1e12 / (hbm * 1e9)
    roof = {"bound": "tensor" if tensor_bound else "hbm",
            "kernel": "k_layer (front + dispatch || grouped FFN + combine, one launch)",
            "achieved": tflops if tensor_bound else achieved, "peak": tf_peak if tensor_bound else hbm,
            "unit": "TFLOP/s" if tensor_bound else "GB/s",
            "frac": (tflops / tf_peak) if tensor_bound else (achieved / hbm),
            "traffic": traffic, "peak_source": src + (" (bf16 sustained)" if tensor_bound else " (HBM copy)"),
            "algorithmic_bytes_per_launch": gbytes, "algorithmic_flops_per_launch": gflops,
            "hbm_GBps": achieved, "hbm_frac": achieved / hbm, "tensor_TFLOPs": tflops, "tensor_frac": tflops / tf_peak,
            "kernel_ms": g_ms, "kernel_ms_serialized": g_ms_ser,
            "kernel_share_of_step": (g_ms_ser / (ms_prof / args.steps)) if ms_prof else None,
            "profiled_ms_per_step": ms_prof / args.steps,
            "per_kernel_ms": kt}

    # ---- north star's other numbers (same run, same GPU)
    prefill = None
    if N == 1 and cfg != "qwen_prefill":
        prefill = prefill_record(tg, dev, args.seed, 50)
    fo_layer, fo_xs = layer, xs
    if N == 1:  # 2 logical EWs with shadow replicas on the one GPU
        pl2 = wl.make_placement(shape.E, 2, 1, shadows=True)
        L2 = make_weights_device(shape, args.seed, dev, list(range(shape.E)))
        fo_layer = tg.MoELayer(shape, pl2, L2, max_tokens_per_rank=T_r, device=local)
    failover = failover_record(tg, fo_layer, shape, fo_xs, stream, N, rank, dev)
    if fo_layer is not layer:
        fo_layer.close()
        del L2
        torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and N == 1 and not args.no_cpu_baseline:
        n = args.cpu_sample or 16
        Lh = wl.Layer(shape, L.wg.cpu(), [w.cpu() for w in L.w1], [w.cpu() for w in L.w3],
                      [w.cpu() for w in L.w2], tuple(w.cpu() for w in L.shared) if L.shared else None,
                      L.wsg.cpu() if L.wsg is not None else None)
        xc = torch.cat([b.cpu() for b in xs])  # up to NB batches: a sample of ~12 s of CPU work
        v, dt = cpu_oracle_sample(shape, Lh, xc, pl, n, cores)
        if args.cpu_sample is None and dt < 8.0:
            # scale the sample to ~12 s of CPU work (bounded by the batch)
            n = int(min(xc.shape[0], max(n, n * 12.0 / max(dt, 1e-3))))
            v, dt = cpu_oracle_sample(shape, Lh, xc, pl, n, cores)
        n1 = min(n, 8)
        v1, dt1, out1 = oracle_one_core(shape, Lh, xc, pl, n1)
        _, _, outa = cpu_oracle_sample(shape, Lh, xc, pl, n1, cores, want_out=True)
        cpu = {"value": v, "unit": "tokens/s", "cores": cores, "kind": "oracle",
               "sample": f"first {n} tokens of the bench batches through O1-O8 (fp64, {cores} threads over tokens), "
                         f"{dt:.1f} s",
               "cpu_model": cpu_model(), "nproc": cores,
               "one_core": {"value": v1, "unit": "tokens/s", "cores": 1, "pinned": "sched_setaffinity to one CPU",
                            "sample": f"first {n1} tokens, {dt1:.1f} s",
                            "bits_equal_to_all_core_run": bool(np.array_equal(out1, outa))}}

    if rank == 0:
        line = {"metric": "MoE-layer tokens/s", "value": value, "unit": "tokens/s", "n_gpus": N,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (seeded random-init weights of the configured shape)", "config": config,
                "clocks": clk.summary(), "gpu_launches": launches,
                "e2e": {"value": e2e_val, "unit": "tokens/s", "h2d_bytes_per_step": T_glob * shape.d * 2,
                        "d2h_bytes_per_step": T_glob * shape.d * 2},
                "roofline": roof, "cpu_baseline": cpu, "prefill": prefill, "failover": failover}
        print(json.dumps(line), flush=True)
    layer.close()
    if N > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
