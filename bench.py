#!/usr/bin/env python
"""bench.py — GPOEO batched period detection on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl reference]

A step = one pass of the whole hot path (composite -> FFT power spectrum -> peaks ->
Alg. 2 on every candidate -> local range -> Alg. 2 on every local period -> result) over
one batch of synthetic traces resident in HBM, through the C ABI (gpoeo_detect_periods),
plus (N > 1) the NCCL all-gather of the per-trace results. Workload: BASELINE.json config
3, 10^5 traces x 3 features x 2^16 samples per GPU (weak scaling: every rank owns its own
10^5-trace shard of the global index space, generated on device from (seed, global
index)). Prints ONE JSON line on rank 0.

--impl reference times the CPU oracle (oracle/, the only other thing this file may
execute) on the box's host cores on bounded samples of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "traces/sec period-detected (2^16 samples×3 features) and % of HBM peak, 1/2/4/8 B200"
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0  # GB/s, B200_PROFILING.md fallback
SM_COUNT = 148
DP_PER_CLK_PER_SM = 64  # fp64 FMA-pipe instructions per clock per SM (B200: half the fp32 rate)


def _peaks():
    try:
        with open(PEAKS_FILE) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": FALLBACK_HBM, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "power_w_median": statistics.median(power) if power else None, "samples": len(sm),
                "reasons": sorted(reasons)}


BACKEND = os.environ.get("GPOEO_DIST_BACKEND", "nccl")  # gloo: code-path test on one GPU


def _dist():
    import torch.distributed as dist
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws > 1 and not dist.is_initialized():
        dist.init_process_group(BACKEND)
    return ws, int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


def _max_over_ranks(value: float, dev) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        return value
    t = torch.tensor([value], dtype=torch.float64, device=dev if BACKEND == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------------------
# CPU oracle timing (the reference arm and the cpu_baseline object)

def oracle_sample(spec, first: int, count: int, threads: int):
    import oracle as O
    import tracegen as tg
    x = tg.generate_host(spec, first, count, threads=threads)
    p = O.params_for(spec)
    t0 = time.perf_counter()
    ds = O.detect_batch(x, p, threads=threads)
    dt = time.perf_counter() - t0
    return dt, ds


def cpu_baseline(spec, count: int, threads: int) -> dict:
    dt, ds = oracle_sample(spec, 0, count, threads)
    return {"value": count / dt, "unit": "traces/s", "cores": threads, "kind": "oracle",
            "sample": f"first {count} traces of the workload (config 3 shape), full oracle (naive O(N^2) DFT, "
                      f"literal Alg. 2 with fp64 CEM), {threads} threads, {dt:.1f} s"}


def run_reference(args) -> None:
    import tracegen as tg
    ws, rank, _ = _dist()
    if rank != 0:
        return
    spec = tg.CFG3
    threads = os.cpu_count() or 1
    per_step = args.ref_traces or threads
    for w in range(args.warmup):
        oracle_sample(spec, w * per_step, per_step, threads)
    times = []
    for k in range(args.steps):
        dt, _ = oracle_sample(spec, (args.warmup + k) * per_step, per_step, threads)
        times.append(dt)
    total = sum(times)
    value = per_step * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "traces/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg3 shape: traces x 3 features x 2^16 samples (sample of "
                               f"{per_step} traces per step)", "traces_per_step": per_step},
        "cpu_baseline": {"value": value, "unit": "traces/s", "cores": threads, "kind": "oracle",
                         "sample": f"{per_step} traces per step x {args.steps} steps on {threads} host threads"},
        "e2e": {"value": value, "unit": "traces/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------

def run_gpu(args) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2201_01684_b200 as g
    import tracegen as tg

    world, rank, local = _dist()
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    spec = tg.CFG3.with_(batch=args.batch)
    B = args.batch
    p = g.params_for(spec)
    stream = torch.cuda.current_stream()

    # inputs resident in HBM before timing: this rank's shard of the global index space
    x = torch.empty((B, spec.n_features * spec.n_samples), dtype=torch.float32, device=dev)
    tg.generate_device(spec, x, first=rank * B, count=B, stream=stream.cuda_stream)
    ws = g.alloc_workspace(g.workspace_size(p, B), dev)
    res = torch.empty(B * g.RESULT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    gathered = torch.empty(world * B * g.RESULT_DTYPE.itemsize, dtype=torch.uint8, device=dev) if world > 1 else None
    torch.cuda.synchronize()

    def step(evs=None):
        if evs is None:
            g.detect_periods(x, p, workspace=ws, results=res, stream=stream)
        else:
            g.detect_periods_timed(x, p, ws, res, evs, stream=stream)
        if world > 1:
            if BACKEND == "nccl":
                dist.all_gather_into_tensor(gathered, res)  # the only device-to-device transfer
            else:
                g_cpu = torch.empty(gathered.shape, dtype=gathered.dtype)
                dist.all_gather_into_tensor(g_cpu, res.cpu())
                gathered.copy_(g_cpu)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    counters = g.read_counters(ws, p, B)

    # phase events per timed step (live per-kernel timing on the launching stream)
    phase_evs = [[torch.cuda.Event(enable_timing=True) for _ in range(7)] for _ in range(args.steps)]
    for evs in phase_evs:
        for e in evs:
            e.record(stream)
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.3)
    t_start.record(stream)
    for k in range(args.steps):
        step(phase_evs[k])
    t_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    elapsed_ms = _max_over_ranks(t_start.elapsed_time(t_end), dev)
    phases = np.array([[evs[i].elapsed_time(evs[i + 1]) for i in range(6)] for evs in phase_evs])  # ms
    phase_ms = phases.mean(axis=0)

    value = world * B * args.steps / (elapsed_ms / 1e3)
    peaks, peak_kind = _peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))

    # dram traffic of the dominant kernel from the committed ncu --set full capture
    # (profiles/ncu_traffic.json: DRAM bytes per trace from one `ncu --set full` capture, scaled to
    # this batch; see profiles/README.md)
    traffic, traffic_note, traffic_spec = None, None, None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tj = json.load(f)
        traffic = tj["scorer_dram_bytes_per_trace"] * B
        traffic_note = tj.get("note")
        traffic_spec = tj["spectral_only_dram_bytes_per_trace"] * B
    except Exception:
        pass
    # dominant kernel: the Alg. 2 scorer (two launches per step, candidate + local queries)
    score_ms = phase_ms[2] + phase_ms[4]
    passes = counters["cem_sample_passes"]  # per step (samples x CEM passes, incl. the W_{i+1} pass)
    dp_per_pass = 3 * p.num_groups + 2
    achieved_dp = passes * dp_per_pass / (score_ms / 1e3)  # fp64 instr/s
    peak_dp = SM_COUNT * DP_PER_CLK_PER_SM * sm_max * 1e6
    hbm_peak = float(peaks.get("hbm_gbs", FALLBACK_HBM))
    alg_bytes = B * (4 * spec.n_features * spec.n_samples + 24)
    spec_ms = phase_ms[0] + phase_ms[1]
    line = {
        "metric": METRIC, "value": value, "unit": "traces/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg3: 1e5 traces x 3 features x 2^16 samples per GPU (BASELINE.json config 3; "
                               "configs 4 = the same shards at N>1)", "batch_per_gpu": B,
                   "n_samples": spec.n_samples, "n_features": spec.n_features,
                   "period_bounds": [spec.min_period, spec.max_period], "num_groups": p.num_groups,
                   "max_candidates": p.max_candidates, "c_peak": round(p.c_peak, 4),
                   "l2": "inputs larger than L2 (%.1f GB/GPU vs 126 MB)" % (B * 4 * 3 * spec.n_samples / 1e9),
                   "parallelism": f"dp{world} (trace shards, NCCL all-gather of results)"},
        "hbm_frac_end_to_end": (alg_bytes / (elapsed_ms / args.steps / 1e3) / 1e9) / hbm_peak,
        "roofline": {"bound": "alu", "kernel": "score_kernel (Alg. 2 CEM scorer, 2 launches/step)",
                     "achieved": achieved_dp / 1e12, "peak": peak_dp / 1e12, "unit": "TDPinstr/s",
                     "frac": achieved_dp / peak_dp, "traffic": traffic, "traffic_note": traffic_note,
                     "work": f"{passes} CEM sample-passes/step x {dp_per_pass} fp64 instr",
                     "peak_note": f"148 SMs x 64 fp64/clk x {sm_max:.0f} MHz (sm_max_mhz, {peak_kind})"},
        "roofline_spectral": {"bound": "hbm", "kernel": "composite + spectrum (a1-a3)",
                              "achieved": alg_bytes / (spec_ms / 1e3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                              "frac": (alg_bytes / (spec_ms / 1e3) / 1e9) / hbm_peak, "traffic": None,
                              "peak_kind": peak_kind},
        "phase_ms": {n: float(v) for n, v in zip(g.PHASES, phase_ms)},
        "work_counters": counters,
        "clocks": clocks,
        # fused spectrum (1), 2 x scorer (team, mid and xl bucketed: 3), select (1), final (1)
        "gpu_launches": 9 * args.steps,
    }

    # spectral-only detector (rows a1-a3 + arg-max, T_iter = 1/f_major) on
    # the same resident traces: the HBM-bound path, 4*F*N bytes read per trace, 16 B written
    if not args.no_spectral:
        mws = g.alloc_workspace(g.major_workspace_size(p, B), dev)
        mres = torch.empty(B * g.MAJOR_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        for _ in range(args.warmup):
            g.detect_major_periods(x, p, workspace=mws, results=mres, stream=stream)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        m0.record(stream)
        for _ in range(args.steps):
            g.detect_major_periods(x, p, workspace=mws, results=mres, stream=stream)
        m1.record(stream)
        torch.cuda.synchronize()
        mms = _max_over_ranks(m0.elapsed_time(m1), dev) / args.steps
        mbytes = B * (4 * spec.n_features * spec.n_samples + g.MAJOR_DTYPE.itemsize)
        mgbs = mbytes / (mms / 1e3) / 1e9
        line["spectral_only"] = {
            "metric": "traces/sec spectral-only period (T_iter = 1/f_major, P:291)", "value": world * B / (mms / 1e3),
            "unit": "traces/s", "ms_per_step": mms, "kernel": "fused_spectrum_65536<3> (mode major) + major_combine_kernel, 2 launches/step",
            "roofline": {"bound": "hbm", "achieved": mgbs, "peak": hbm_peak, "unit": "GB/s", "frac": mgbs / hbm_peak,
                         "traffic": traffic_spec, "peak_kind": peak_kind,
                         "bytes": f"{4 * spec.n_features * spec.n_samples + g.MAJOR_DTYPE.itemsize} B/trace"}}
        del mws, mres

    # Alg. 3 rolling detector on the first traces of the same resident batch:
    # Alg. 1 on each whole trace, then on its ~7 rolling suffixes (ragged batches); synchronous
    if not args.no_rolling:
        Br = min(args.rolling_batch, B)
        xr = x[:Br]
        g.detect_rolling(xr, p)  # warm
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.rolling_steps):
            rr = g.detect_rolling(xr, p)
        tr = _max_over_ranks(time.perf_counter() - t0, dev) / args.rolling_steps
        line["rolling"] = {
            "metric": "traces/sec Alg. 3 rolling detection (P:383-429)", "value": world * Br / tr, "unit": "traces/s",
            "batch_per_gpu": Br, "steps": args.rolling_steps, "ms_per_step": 1e3 * tr,
            "mean_suffixes": float(rr["n_sub"].mean()), "stop_sampling_frac": float((rr["smpdur_next_s"] < 0).mean()),
            "timing": "wall clock of the synchronous gpoeo_detect_rolling (inputs resident in HBM)",
            "note": "time is dominated by the Alg. 2 scorer kernels of the roofline above (whole traces + suffixes)"}

    # Alg. 4 adaptive measurement: sessions over the same resident recordings,
    # starting from SmpDur_init = 2 L_max samples; synchronous rounds of ragged Alg. 3 batches
    if not args.no_rolling:
        Bm = min(args.rolling_batch, B)
        init = min(spec.n_samples, 2 * spec.max_period)
        g.measure_adaptive(x[:Bm], p, init)  # warm
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        mr = g.measure_adaptive(x[:Bm], p, init)
        tm = _max_over_ranks(time.perf_counter() - t0, dev)
        line["measure"] = {
            "metric": "sessions/sec Alg. 4 adaptive measurement (P:431-462)", "value": world * Bm / tm,
            "unit": "sessions/s", "batch_per_gpu": Bm, "init_samples": init, "ms_per_step": 1e3 * tm,
            "mean_rounds": float(mr["rounds"].mean()), "mean_samples": float(mr["samples"].mean()),
            "stable_frac": float((mr["status"] == 0).mean()),
            "timing": "wall clock of the synchronous gpoeo_measure_adaptive (recordings resident in HBM)"}

    # gear local search over simulated workloads: one thread per workload
    if not args.no_rolling:
        import numpy as np
        rng = np.random.default_rng(11)
        ng = args.gear_workloads
        wl = np.zeros(ng, dtype=g.GEAR_WORKLOAD_DTYPE)
        wl["compute_work"] = rng.uniform(0.5e9, 3e9, ng)
        wl["memory_work"] = rng.uniform(0.5e9, 3e9, ng)
        wl["overhead"] = rng.uniform(0.01, 0.1, ng)
        wl["p_static"] = rng.uniform(60, 150, ng)
        wl["c_sm"] = rng.uniform(2e-4, 1e-3, ng)
        wl["c_mem"] = rng.uniform(0.005, 0.03, ng)
        wl["u_c"] = rng.uniform(0.2, 1.0, ng)
        wl["u_m"] = rng.uniform(0.2, 1.0, ng)
        wl["noise"] = 0.01
        wl["seed"] = rng.integers(0, 1 << 62, ng, dtype=np.uint64)
        smg = np.arange(510, 1966, 15, dtype=np.float64)
        memg = np.array([405.0, 810.0, 1600.0, 2619.0, 3996.0])
        dwl = torch.from_numpy(wl.view(np.uint8).copy()).to(dev)
        dsm, dmem = torch.as_tensor(smg, device=dev), torch.as_tensor(memg, device=dev)
        dps = torch.as_tensor(rng.integers(0, len(smg), ng).astype(np.int32), device=dev)
        dpm = torch.as_tensor(rng.integers(0, len(memg), ng).astype(np.int32), device=dev)
        dout = torch.empty(ng * g.GEAR_RESULT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        lib = g.load()
        import ctypes as _ct

        def _gear():
            rc = lib.gpoeo_gear_search(_ct.c_void_p(dwl.data_ptr()), ng, _ct.c_void_p(dsm.data_ptr()), len(smg),
                                       _ct.c_void_p(dmem.data_ptr()), len(memg), 0.05, _ct.c_void_p(dps.data_ptr()),
                                       _ct.c_void_p(dpm.data_ptr()), _ct.c_void_p(dout.data_ptr()),
                                       _ct.c_void_p(stream.cuda_stream))
            assert rc == 0
        _gear()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            _gear()
        g1.record(stream)
        torch.cuda.synchronize()
        gms = _max_over_ranks(g0.elapsed_time(g1), dev) / args.steps
        gr = dout.cpu().numpy().view(g.GEAR_RESULT_DTYPE)
        line["gear_search"] = {
            "metric": "workloads/sec gear local search (P:585-593) on the simulated device", "value": world * ng / (gms / 1e3),
            "unit": "workloads/s", "workloads_per_gpu": ng, "ms_per_step": gms,
            "mean_probes_sm": float(gr["probes_sm"].mean()), "mean_probes_mem": float(gr["probes_mem"].mean()),
            "gears": f"{len(smg)} SM x {len(memg)} memory", "note": "control logic, one thread per workload"}

    # e2e: same metric through the public host entry point (pinned host buffers, H2D+D2H inside)
    del x
    torch.cuda.empty_cache()
    if not args.no_e2e:
        # pinned host memory is shared by the ranks of the box: 8192 traces (6.4 GB) per rank at N > 1
        Be = min(args.e2e_batch, B) if world == 1 else min(args.e2e_batch, B, 8192)
        xh = torch.empty((Be, spec.n_features * spec.n_samples), dtype=torch.float32, pin_memory=True)
        tmp = torch.empty((min(Be, 4096), spec.n_features * spec.n_samples), dtype=torch.float32, device=dev)
        for i0 in range(0, Be, tmp.shape[0]):
            n = min(tmp.shape[0], Be - i0)
            tg.generate_device(spec, tmp, first=rank * B + i0, count=n, stream=stream.cuda_stream)
            xh[i0:i0 + n].copy_(tmp[:n])
        del tmp
        torch.cuda.synchronize()
        hws = g.alloc_workspace(int(g.load().gpoeo_workspace_size_host(__import__("ctypes").byref(p), args.chunk)),
                                dev)
        out = np.empty(Be, dtype=g.RESULT_DTYPE)
        g.detect_periods_host(xh, p, chunk=args.chunk, workspace=hws, out=out)  # warm
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            g.detect_periods_host(xh, p, chunk=args.chunk, workspace=hws, out=out)
        te = _max_over_ranks(time.perf_counter() - t0, dev)
        # the bound of this leg: a plain pinned H2D copy of one chunk (CUDA events)
        dchunk = torch.empty((min(args.chunk, Be), xh.shape[1]), dtype=torch.float32, device=dev)
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dchunk.copy_(xh[:dchunk.shape[0]], non_blocking=True)
        c0.record()
        for _ in range(3):
            dchunk.copy_(xh[:dchunk.shape[0]], non_blocking=True)
        c1.record()
        torch.cuda.synchronize()
        h2d_gbs = 3 * dchunk.numel() * 4 / (c0.elapsed_time(c1) / 1e3) / 1e9
        del dchunk
        tbytes = spec.n_features * spec.n_samples * 4
        line["e2e"] = {"value": world * Be * args.e2e_steps / te, "unit": "traces/s",
                       "h2d_bytes_per_step": Be * tbytes,
                       "d2h_bytes_per_step": Be * g.RESULT_DTYPE.itemsize,
                       "batch_per_gpu": Be, "chunk": args.chunk, "steps": args.e2e_steps,
                       "h2d_copy_GBps": h2d_gbs, "h2d_bound_traces_per_s": world * h2d_gbs * 1e9 / tbytes,
                       "api": "gpoeo_detect_periods_host (pinned host traces, results to host, wall clock incl. sync)"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(spec, args.cpu_traces, os.cpu_count() or 1)
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=100_000)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-batch", type=int, default=16384)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--chunk", type=int, default=2048)
    ap.add_argument("--cpu-traces", type=int, default=48)
    ap.add_argument("--ref-traces", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-spectral", action="store_true")
    ap.add_argument("--no-rolling", action="store_true")
    ap.add_argument("--rolling-batch", type=int, default=5000)
    ap.add_argument("--rolling-steps", type=int, default=2)
    ap.add_argument("--gear-workloads", type=int, default=100_000)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)
    try:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()
    except Exception:
        pass


if __name__ == "__main__":
    main()
