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

def oracle_sample(spec, first: int, count: int, threads: int, band_only: bool = False):
    import oracle as O
    import tracegen as tg
    x = tg.generate_host(spec, first, count, threads=threads)
    p = O.params_for(spec, dft_band_only=band_only)
    t0 = time.perf_counter()
    ds = O.detect_batch(x, p, threads=threads)
    dt = time.perf_counter() - t0
    return dt, ds


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(spec, count: int, threads: int, name: str = "config 3", band_only: bool = False) -> dict:
    dt, ds = oracle_sample(spec, 0, count, threads, band_only)
    dft = ("naive O(N^2) DFT at the bins the peak rule reads (the oracle's dft_band_only mode: the same per-bin "
           "arithmetic, 1/5 of the bins)" if band_only else "naive O(N^2) DFT over every bin")
    return {"value": count / dt, "unit": "traces/s", "cores": threads, "kind": "oracle",
            "cpu_model": cpu_model(), "nproc": os.cpu_count(),
            "sample": f"first {count} traces of the workload ({name}), the oracle as it stands ({dft}, literal "
                      f"Alg. 2 with fp64 CEM), {threads} threads, {dt:.1f} s"}


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
                         "cpu_model": cpu_model(), "nproc": os.cpu_count(),
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
    from paper_2201_01684_b200 import shard

    world, rank, local = _dist()
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    # the workload: config 3 (10^5 traces resident on one GPU) at N = 1; config 4 (10^6 traces
    # sharded over the N GPUs, each shard streamed through a resident buffer of at most
    # --max-chunk traces when it exceeds HBM) at N > 1 (or --cfg4)
    cfg4 = world > 1 or args.cfg4
    if cfg4:
        spec = tg.CFG4.with_(batch=args.cfg4_total)
        first, B = shard.shard_range(spec.batch, world, rank)
    else:
        spec = tg.CFG3.with_(batch=args.batch)
        first, B = 0, args.batch
    chunks = shard.chunk_ranges(first, B, args.max_chunk)
    streamed = len(chunks) > 1
    Bbuf = max(n for _, n in chunks) if chunks else 1
    p = g.params_for(spec)

    # inputs resident in HBM before timing (this rank's shard, or its first chunk), generated
    # on the device from (seed, global index)
    x = torch.empty((Bbuf, spec.n_features * spec.n_samples), dtype=torch.float32, device=dev)
    tg.generate_device(spec, x, first=first, count=min(B, Bbuf), stream=stream.cuda_stream)
    ws = g.alloc_workspace(g.workspace_size(p, Bbuf), dev)
    res = torch.empty(max(B, 1) * g.RESULT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()

    def gather():
        if world > 1:
            if BACKEND == "nccl":
                return shard.gather_results(res[:B * g.RESULT_DTYPE.itemsize], spec.batch)  # the only device-to-device transfer
            out = shard.gather_results(res[:B * g.RESULT_DTYPE.itemsize].cpu(), spec.batch)
            return out.to(dev)
        return None

    def step(evs=None):
        # resident shard: one call over all of it
        if evs is None:
            g.detect_periods(x[:B], p, workspace=ws, results=res, stream=stream)
        else:
            g.detect_periods_timed(x[:B], p, ws, res, evs, stream=stream)
        gather()

    chunk_ms = []

    def step_streamed():
        # streamed shard (config 4 at N = 2, 4): chunk i's traces are generated into the
        # resident buffer (untimed), then its detect call is timed with CUDA events; the
        # step's time is the sum over chunks plus the all-gather
        ms = 0.0
        for i, (f, n) in enumerate(chunks):
            tg.generate_device(spec, x[:n], first=f, count=n, stream=stream.cuda_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            off = (f - first) * g.RESULT_DTYPE.itemsize
            g.detect_periods(x[:n], p, workspace=ws, results=res[off:off + n * g.RESULT_DTYPE.itemsize], stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            ms += e0.elapsed_time(e1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        gather()
        e1.record(stream)
        torch.cuda.synchronize()
        ms += e0.elapsed_time(e1)
        chunk_ms.append(ms)

    if streamed:
        for _ in range(args.warmup):
            step_streamed()
        chunk_ms.clear()
    else:
        for _ in range(args.warmup):
            step()
    torch.cuda.synchronize()
    counters = g.read_counters(ws, p, Bbuf)

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
    if streamed:
        for k in range(args.steps):
            step_streamed()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        elapsed_ms = _max_over_ranks(sum(chunk_ms), dev)
    else:
        t_start.record(stream)
        for k in range(args.steps):
            step(phase_evs[k])
        t_end.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        elapsed_ms = _max_over_ranks(t_start.elapsed_time(t_end), dev)
    clocks = sampler.stop()
    if streamed:
        # phase split of one chunk call (timed separately after the run, resident chunk)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
        for e in evs:
            e.record(stream)
        g.detect_periods_timed(x[:chunks[-1][1]], p, ws, res, evs, stream=stream)
        torch.cuda.synchronize()
        phases = np.array([[evs[i].elapsed_time(evs[i + 1]) for i in range(6)]])
        counters = g.read_counters(ws, p, chunks[-1][1])
        ph_traces = chunks[-1][1]
    else:
        phases = np.array([[evs[i].elapsed_time(evs[i + 1]) for i in range(6)] for evs in phase_evs])  # ms
        ph_traces = B
    phase_ms = phases.mean(axis=0)

    total_traces = spec.batch if cfg4 else world * B
    value = total_traces * args.steps / (elapsed_ms / 1e3)
    peaks, peak_kind = _peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))

    # dram traffic of the dominant kernel from the committed ncu --set full capture
    # (profiles/ncu_traffic.json: DRAM bytes per trace from one `ncu --set full` capture, scaled to
    # this batch; see profiles/README.md)
    traffic, traffic_note, traffic_spec = None, None, None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tj = json.load(f)
        traffic = tj["scorer_dram_bytes_per_trace"] * ph_traces
        traffic_note = tj.get("note")
        traffic_spec = tj["spectral_only_dram_bytes_per_trace"] * B
    except Exception:
        pass
    # dominant kernel: the Alg. 2 scorer (two launches per step, candidate + local queries)
    score_ms = phase_ms[2] + phase_ms[4]
    passes = counters["cem_sample_passes"]  # per call (samples x CEM passes, incl. the W_{i+1} pass)
    dp_per_pass = 3 * p.num_groups + 2
    achieved_dp = passes * dp_per_pass / (score_ms / 1e3)  # fp64 instr/s
    peak_dp = SM_COUNT * DP_PER_CLK_PER_SM * sm_max * 1e6
    hbm_peak = float(peaks.get("hbm_gbs", FALLBACK_HBM))
    alg_bytes = ph_traces * (4 * spec.n_features * spec.n_samples + 24)
    spec_ms = phase_ms[0] + phase_ms[1]
    if cfg4:
        workload = (f"cfg4: 1e6 traces x 3 features x 2^16 samples sharded over {world} GPU(s) (BASELINE.json config 4), "
                    f"{B} traces per rank" + (f", streamed in {len(chunks)} chunks of <= {args.max_chunk}" if streamed
                                              else ", resident"))
    else:
        workload = "cfg3: 1e5 traces x 3 features x 2^16 samples on 1 GPU (BASELINE.json config 3)"
    line = {
        "metric": METRIC, "value": value, "unit": "traces/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if cfg4 else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload, "batch_per_gpu": B, "traces_total": total_traces,
                   "n_samples": spec.n_samples, "n_features": spec.n_features,
                   "period_bounds": [spec.min_period, spec.max_period], "num_groups": p.num_groups,
                   "max_candidates": p.max_candidates, "c_peak": round(p.c_peak, 4),
                   "l2": "inputs larger than L2 (%.1f GB/GPU vs 126 MB)" % (Bbuf * 4 * 3 * spec.n_samples / 1e9),
                   "timing": ("sum of per-chunk CUDA-event times of the detect calls + all-gather; chunk generation "
                              "between them excluded" if streamed else "CUDA events around K whole steps"),
                   "parallelism": f"dp{world} (trace shards, NCCL all-gather of results)"},
        "hbm_frac_end_to_end": (total_traces / world * (4 * spec.n_features * spec.n_samples + 24)
                                / (elapsed_ms / args.steps / 1e3) / 1e9) / hbm_peak,
        "roofline": {"bound": "alu", "kernel": "score_kernel (Alg. 2 CEM scorer, 2 launches/step)",
                     "achieved": achieved_dp / 1e12, "peak": peak_dp / 1e12, "unit": "TDPinstr/s",
                     "frac": achieved_dp / peak_dp, "traffic": traffic, "traffic_note": traffic_note,
                     "work": f"{passes} CEM sample-passes/call x {dp_per_pass} fp64 instr",
                     "work_note": ("sample-passes the kernels evaluated: with bounded_search = 1 (the default) "
                                   f"{counters.get('n_pruned_queries', 0)} of "
                                   f"{counters['n_candidate_queries'] + counters['n_local_queries']} queries stopped "
                                   "once their partial Err proved they cannot be the argmin; their evaluated pairs "
                                   "count, the rest do not"),
                     "peak_note": f"148 SMs x 64 fp64/clk x {sm_max:.0f} MHz (sm_max_mhz, {peak_kind})"},
        "roofline_spectral": {"bound": "hbm", "kernel": "composite + spectrum (a1-a3)",
                              "achieved": alg_bytes / (spec_ms / 1e3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                              "frac": (alg_bytes / (spec_ms / 1e3) / 1e9) / hbm_peak, "traffic": None,
                              "peak_kind": peak_kind},
        "phase_ms": {n: float(v) for n, v in zip(g.PHASES, phase_ms)},
        "work_counters": counters,
        "clocks": clocks,
        # fused spectrum (1), candidate list (scan + scatter: 2), 2 x scorer (team, mid and xl bucketed: 3),
        # select (select, centre refine, count, scan, scatter: 5), final (1) per call
        "gpu_launches": 15 * args.steps * len(chunks),
    }
    B = min(B, Bbuf)  # the sub-lines below use the resident buffer

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
    # Alg. 1 on each whole trace, the suffix plan on the device, Alg. 1 on its ~7 rolling
    # suffixes (ragged batches), lines 14-21; asynchronous, timed with CUDA events
    if not args.no_rolling:
        Br = min(args.rolling_batch, B)
        xr = x[:Br]
        rres, rws = g.detect_rolling_async(xr, p, stream=stream)  # warm
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record(stream)
        for _ in range(args.rolling_steps):
            g.detect_rolling_async(xr, p, workspace=rws, results=rres, stream=stream)
        r1.record(stream)
        torch.cuda.synchronize()
        tr = _max_over_ranks(r0.elapsed_time(r1), dev) / 1e3 / args.rolling_steps
        rr = rres.cpu().numpy().view(g.ROLLING_DTYPE)
        line["rolling"] = {
            "metric": "traces/sec Alg. 3 rolling detection (P:383-429)", "value": world * Br / tr, "unit": "traces/s",
            "batch_per_gpu": Br, "steps": args.rolling_steps, "ms_per_step": 1e3 * tr,
            "mean_suffixes": float(rr["n_sub"].mean()), "stop_sampling_frac": float((rr["smpdur_next_s"] < 0).mean()),
            "timing": "CUDA events around gpoeo_detect_rolling (asynchronous: device-side suffix plan; inputs resident)",
            "note": "time is dominated by the Alg. 2 scorer kernels and the band-limited DFT of the suffixes"}
        del rres, rws

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

    del x, ws
    torch.cuda.empty_cache()

    # BASELINE config 5 (the hard case: 10^4 traces x 3 x 2^18, mid-trace period shift,
    # harmonic-aliased spectra): the whole Alg. 1 path, inputs resident, its own rooflines
    # (spectral stage vs HBM, scorer vs fp64) and an oracle subset on the host cores
    if world == 1 and not args.no_cfg5:
        spec5 = tg.CFG5.with_(batch=args.cfg5_batch)
        B5 = spec5.batch
        p5 = g.params_for(spec5)
        x5 = torch.empty((B5, spec5.n_features * spec5.n_samples), dtype=torch.float32, device=dev)
        tg.generate_device(spec5, x5, stream=stream.cuda_stream)
        ws5 = g.alloc_workspace(g.workspace_size(p5, B5), dev)
        res5 = torch.empty(B5 * g.RESULT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        for _ in range(args.warmup):
            g.detect_periods(x5, p5, workspace=ws5, results=res5, stream=stream)
        torch.cuda.synchronize()
        c5 = g.read_counters(ws5, p5, B5)
        evs5 = [[torch.cuda.Event(enable_timing=True) for _ in range(7)] for _ in range(args.steps)]
        for evs in evs5:
            for e in evs:
                e.record(stream)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a0.record(stream)
        for k in range(args.steps):
            g.detect_periods_timed(x5, p5, ws5, res5, evs5[k], stream=stream)
        a1.record(stream)
        torch.cuda.synchronize()
        ms5 = a0.elapsed_time(a1) / args.steps
        ph5 = np.array([[evs[i].elapsed_time(evs[i + 1]) for i in range(6)] for evs in evs5]).mean(axis=0)
        r5 = g.results_numpy(res5)
        bytes5 = B5 * (4 * spec5.n_features * spec5.n_samples + 24)
        sp5 = ph5[0] + ph5[1]
        sc5 = ph5[2] + ph5[4]
        dp5 = c5["cem_sample_passes"] * (3 * p5.num_groups + 2) / (sc5 / 1e3)
        line["cfg5"] = {
            "metric": "traces/sec period-detected (2^18 samples x 3 features, BASELINE config 5)",
            "value": B5 / (ms5 / 1e3), "unit": "traces/s", "ms_per_step": ms5, "steps": args.steps,
            "config": {"workload": "cfg5: 1e4 traces x 3 features x 2^18 samples, mid-trace period shift "
                                   "(L2 = L1 x U(1.2, 1.6)), harmonic-aliased profiles, interference above Nyquist",
                       "batch": B5, "period_bounds": [spec5.min_period, spec5.max_period],
                       "l2": "inputs larger than L2 (%.1f GB vs 126 MB)" % (B5 * 12 * spec5.n_samples / 1e9)},
            "phase_ms": {n: float(v) for n, v in zip(g.PHASES, ph5)},
            "roofline_spectral": {"bound": "hbm", "kernel": "composite_kernel + spectrum_kernel<14, 8> (8-CTA cluster FFT)",
                                  "achieved": bytes5 / (sp5 / 1e3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                                  "frac": bytes5 / (sp5 / 1e3) / 1e9 / hbm_peak, "peak_kind": peak_kind},
            "roofline": {"bound": "alu", "kernel": "score kernels (Alg. 2 CEM scorer)", "achieved": dp5 / 1e12,
                         "peak": peak_dp / 1e12, "unit": "TDPinstr/s", "frac": dp5 / peak_dp,
                         "work": f"{c5['cem_sample_passes']} CEM sample-passes/step x {3 * p5.num_groups + 2} fp64 instr"},
            "work_counters": c5,
            "status_counts": {str(k): int(v) for k, v in zip(*np.unique(r5["status"], return_counts=True))},
            "gpu_launches": 16 * args.steps,  # composite, cluster spectrum, candidate list (2), 2 x 3 scorers, select (5), final
        }
        if rank == 0 and not args.no_cpu_baseline:
            line["cfg5"]["cpu_baseline"] = cpu_baseline(spec5, args.cfg5_cpu_traces, os.cpu_count() or 1,
                                                        "config 5", band_only=True)
        del x5, ws5, res5
        torch.cuda.empty_cache()

    # e2e: same metric through the public host entry point (pinned host buffers, H2D+D2H inside)
    if not args.no_e2e:
        # pinned host memory is shared by the ranks of the box: the whole batch at N = 1 (78.6 GB
        # of the box's 196 GB), 8192 traces (6.4 GB) per rank at N > 1
        Be = (min(args.e2e_batch, B) if args.e2e_batch else B) if world == 1 else min(args.e2e_batch or B, B, 8192)
        xh = torch.empty((Be, spec.n_features * spec.n_samples), dtype=torch.float32, pin_memory=True)
        tmp = torch.empty((min(Be, 4096), spec.n_features * spec.n_samples), dtype=torch.float32, device=dev)
        for i0 in range(0, Be, tmp.shape[0]):
            n = min(tmp.shape[0], Be - i0)
            tg.generate_device(spec, tmp, first=first + i0, count=n, stream=stream.cuda_stream)
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
    ap.add_argument("--e2e-batch", type=int, default=0, help="0: the whole batch at N = 1")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--chunk", type=int, default=4096)  # e2e chunk (measured: 2048 57.0K, 4096 60.0K, 8192 59.4K, 16384 56.6K traces/s)
    ap.add_argument("--cpu-traces", type=int, default=256)
    ap.add_argument("--cfg4", action="store_true", help="config 4 sharding at N = 1 too (streamed chunks)")
    ap.add_argument("--cfg4-total", type=int, default=1_000_000)
    ap.add_argument("--max-chunk", type=int, default=125_000, help="traces resident per GPU (HBM bound)")
    ap.add_argument("--no-cfg5", action="store_true")
    ap.add_argument("--cfg5-batch", type=int, default=10_000)
    ap.add_argument("--cfg5-cpu-traces", type=int, default=16)
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
