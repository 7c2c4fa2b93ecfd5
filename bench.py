#!/usr/bin/env python
"""bench.py -- throughput of the B200 ESS hot path (BASELINE.json metric).

A "step" = one tmvn_sample call that runs --iters-per-step (default 100)
iterations of Alg. 1 for all C chains of the workload (every row of SURVEY
8(a): RNG, projection GEMM, arcs, sort / cummax, theta, update, moments, and
the periodic P refresh), continuing the chains from the previous step.
Default workload: BASELINE config 3 (d=1000, m=2000, 4096 chains per GPU,
FP64) -- the configuration north_star's target is quoted on.

  python bench.py [--gpus N --steps K --warmup W --config 3 --impl ours|reference]

N > 1 runs under torchrun (one process per GPU, NCCL): every rank owns its own
4096 chains (weak scaling, global chain offset rank*C), no per-iteration
collective; one all_reduce of the moments and one MAX of the timings at the end.
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

METRIC = "constraint-evals/sec (chain-iterations/sec x m), FP64, whole job"
METRIC32 = "constraint-evals/sec (chain-iterations/sec x m), FP32-class (--precision 1), whole job"
UNIT = "constraint-evals/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--iters-per-step", type=int, default=100)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--projection", type=int, default=0,
                    help="options.projection: 0 auto (int8 when d <= 4096), 1 int8 Ozaki split on "
                         "tcgen05 (FP64-accurate), 2 FP64 DMMA")
    ap.add_argument("--precision", type=int, default=0,
                    help="options.precision: 0 FP64 (the BASELINE metric), 1 the paper's FP32-class "
                         "mode (int8 projection at 4 digits / FP32 latency kernel; trim_eps 1e-5)")
    return ap.parse_args()


def config_dict(cfg, args, world):
    name = f"BASELINE config {args.config}" if args.config <= 5 else "paper S4.2 timing workload (not a BASELINE config)"
    return {"workload": f"{name} ({cfg.key}): {cfg.desc}",
            "d": cfg.d, "m": cfg.m, "chains_per_gpu": cfg.C, "chains_total": cfg.C * world,
            "iters_per_step": args.iters_per_step, "recompute_every": 32,
            "l2": ("no flush: working set (X, nu, P x2, Q, A) >> 126 MB L2"
                   if 8 * (cfg.C * (4 * cfg.m + 3 * cfg.d) + cfg.m * cfg.d) > 126e6 else
                   "no flush: the working set fits in the 126 MB L2 (latency-bound workload; the "
                   "sampler's state stays resident by design)"),
            "parallelism": f"chains sharded over {world} GPU(s), A and b replicated"}


# ------------------------------------------------------------------ clocks
CLOCK_FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                "clocks_event_reasons.sw_power_cap")


def clocks_start():
    f = tempfile.NamedTemporaryFile("w+", delete=False, suffix=".csv")
    try:
        p = subprocess.Popen(["nvidia-smi", f"--query-gpu={CLOCK_FIELDS}", "--format=csv,noheader,nounits",
                              "-lms", "100"], stdout=f, stderr=subprocess.DEVNULL)
    except FileNotFoundError:
        return None
    return p, f.name


def clocks_stop(h, gpus):
    if h is None:
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
    p, path = h
    p.terminate()
    p.wait()
    sm, mx, reasons = [], [], set()
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    for line in open(path):
        parts = [x.strip() for x in line.split(",")]
        if len(parts) < 8 or not parts[0].isdigit() or int(parts[0]) not in gpus:
            continue
        try:
            sm.append(float(parts[1]))
            mx.append(float(parts[2]))
        except ValueError:
            continue
        for n, v in zip(names, parts[4:8]):
            if v.lower().startswith("active"):
                reasons.add(n)
    os.unlink(path)
    return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
            "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ oracle timing
def oracle_rate(A, b, x0, seed, seconds, C_full):
    """The oracle as it stands, all host cores, on a bounded sample of the workload."""
    import oracle
    cores = len(os.sched_getaffinity(0))
    m = A.shape[0]
    Co = int(min(C_full, 2 * cores))
    X0 = np.tile(x0, (Co, 1))
    t0 = time.perf_counter()
    oracle.run(A, b, X0, 1, seed, nthreads=cores)
    one = max(time.perf_counter() - t0, 1e-6)
    To = int(max(1, min(1000, seconds / one)))
    t0 = time.perf_counter()
    oracle.run(A, b, X0, To, seed, nthreads=cores)
    dt = time.perf_counter() - t0
    return {"value": Co * To * m / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{Co} chains x {To} iterations of the same instance (first iterations from x0), "
                      f"{dt:.1f} s on {cores} host threads (OpenMP over chains)",
            "chain_iters_per_s": Co * To / dt, "seconds": dt}


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if rank != 0:
        return
    from paper_2407_10449_b200 import synth
    cfg = synth.CONFIGS[args.config]
    A, b, x0 = synth.make_instance(args.config)
    import oracle
    cores = len(os.sched_getaffinity(0))
    Co = int(min(cfg.C, 2 * cores))
    X = np.tile(x0, (Co, 1))
    t0 = time.perf_counter()
    oracle.run(A, b, X, 1, cfg.chain_seed, nthreads=cores)
    one = max(time.perf_counter() - t0, 1e-6)
    To = int(max(1, min(args.iters_per_step, 3.0 / one)))  # ~3 s of CPU work per step
    for _ in range(args.warmup):
        X = oracle.run(A, b, X, 1, cfg.chain_seed, nthreads=cores)["X"]
    times = []
    it0 = 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        X = oracle.run(A, b, X, To, cfg.chain_seed, iter_offset=it0, nthreads=cores)["X"]
        times.append(time.perf_counter() - t0)
        it0 += To
    tot = sum(times)
    value = Co * To * cfg.m * args.steps / tot
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_dict(cfg, args, world),
            "cpu_baseline": {"kind": "oracle", "cores": cores, "value": value, "unit": UNIT,
                             "sample": f"each step {Co} chains x {To} iterations of the workload on "
                                       f"{cores} host threads (the CPU oracle as it stands)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist
    import paper_2407_10449_b200 as tm
    from paper_2407_10449_b200 import dist as tdist
    from paper_2407_10449_b200 import synth

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    cfg = synth.CONFIGS[args.config]
    A, b, x0 = synth.make_instance(args.config)
    m, d, C = cfg.m, cfg.d, cfg.C
    ips = args.iters_per_step
    seed = cfg.chain_seed
    offset, C = tdist.weak_shard(cfg.C, rank)  # every rank runs the workload's C chains
    stream = torch.cuda.Stream(device=dev)
    s = tm.Sampler(torch.tensor(A, device=dev), torch.tensor(b, device=dev), chain_offset=offset)
    s.set_options(stream=stream, projection=args.projection)
    if args.precision:
        s.set_options(precision=1, trim_eps=1e-5)
    oz = args.projection == 1 or (args.projection == 0 and d <= 4096)
    X = torch.tensor(np.tile(x0, (C, 1)), device=dev)

    def timed_pass(steps):
        """barrier + sync; CUDA events on the library's stream around `steps` steps."""
        with torch.cuda.stream(stream):
            torch.cuda.synchronize()
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(steps):
                s.sample(X, ips, seed, out=X)
            e1.record(stream)
            torch.cuda.synchronize()
            barrier()
        return e0.elapsed_time(e1)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            s.sample(X, ips, seed, out=X)
    s.reset_stats()
    clk = clocks_start() if rank == 0 else None
    time.sleep(0.15 if clk else 0)
    # ---- main pass: the library's default launch configuration (GEMM / per-chain
    # kernel of two chain shards overlapped on two streams)
    ms = timed_pass(args.steps)
    clocks = clocks_stop(clk, set(range(world))) if rank == 0 else None
    prof_main = s.profile()
    st = s.stats()
    ms_max = tdist.max_over_ranks(ms, dev)
    total_iters = world * C * ips * args.steps
    value = total_iters * m / (ms_max * 1e-3)
    sm, sq, n = s.moments()
    _, _, n_all, rej_all = tdist.reduce_moments(sm, sq, n, st["rejections"], dev)
    opts = s.options()

    # ---- roofline pass: same workload, one stream (no kernel overlap), every GEMM and
    # per-chain launch bracketed by CUDA events on that stream (options.profile)
    s.set_options(streams=1, profile=1)
    s.reset_stats()
    ms_iso = timed_pass(args.steps)
    prof = s.profile()
    s.set_options(streams=opts.streams, profile=0)
    if prof["latency_calls"] > 0:
        # latency mode (few chains: one thread-block cluster per chain, one launch per call):
        # each cluster streams its chain's A . nu (m x d FP64) from L2 every iteration
        try:
            hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
            hbm_src = "MEASURED_PEAKS.json hbm_gbs (measured)"
        except Exception:
            hbm, hbm_src = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"
        launch_ms = ms_iso / args.steps
        abytes = float(C) * ips * m * d * 8
        variant = ("a cooperative grid of SMs / C CTAs per chain" if prof.get("latency_grid_calls", 0)
                   else "one thread-block cluster per chain")
        roofline = {"bound": "hbm", "kernel": f"latency_kernel ({variant}: nu, A nu, arcs, "
                                               "two-level Alg. 3 intervals, theta, P', safeguard, x update)",
                    "achieved": abytes / (launch_ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                    "frac": abytes / (launch_ms * 1e-3) / 1e9 / hbm, "traffic": None, "traffic_source": None,
                    "peak_source": hbm_src + "; A (8 m d bytes per chain-iteration, the algorithmic bytes "
                                   "counted here) is served from L2, so this is a bandwidth-equivalent figure",
                    "algorithmic_bytes_per_launch": abytes, "avg_launch_ms": launch_ms, "share_of_step": 1.0,
                    "latency_calls": prof["latency_calls"], "latency_fallbacks": prof["latency_fallbacks"],
                    "latency_grid_calls": prof.get("latency_grid_calls", 0)}
    else:
        peaks = json.load(open(os.path.join(ROOT, "profiles", "peaks_fp64_r01.json")))
        gemm_avg_ms = prof["gemm_ms"] / max(1, prof["gemm_launches"])
        gemm_flops = prof["gemm_flops"] / max(1, prof["gemm_launches"])
        achieved = gemm_flops / (gemm_avg_ms * 1e-3) / 1e12 if gemm_avg_ms > 0 else 0.0
        peak = peaks["dmma_tflops_w8"]
        ess_avg_ms = prof["ess_ms"] / max(1, prof["ess_launches"])
        ess_gbs = prof["ess_bytes"] / max(1, prof["ess_launches"]) / (ess_avg_ms * 1e-3) / 1e9
        try:
            hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
            hbm_src = "MEASURED_PEAKS.json hbm_gbs (measured)"
        except Exception:
            hbm, hbm_src = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"
        traffic, traffic_src = None, None
        try:  # dram__bytes_read + dram__bytes_write per launch from the committed ncu --set full capture
            tj = json.load(open(os.path.join(ROOT, "profiles", "r01", "ncu_gemm_traffic.json")))
            if args.config == 3 and world == 1:
                traffic, traffic_src = tj["traffic_bytes"], "profiles/r01/ncu_gemm_traffic.json"
        except Exception:
            pass
        roofline = {"bound": "tensor", "kernel": "gemm_tn_f64_kernel (Q = N A^T and P = X A^T, FP64 DMMA)",
                    "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                    "traffic": traffic, "traffic_source": traffic_src,
                    "peak_source": "measured FP64 DMMA pipe peak on this pool's B200 (profiles/peaks_fp64_r01.json: "
                                   f"mma.sync f64 micro-benchmark; cuBLAS DGEMM measured {peaks['dgemm_tflops_burst']} TF/s)",
                    "algorithmic_flops_per_launch": gemm_flops, "avg_launch_ms": gemm_avg_ms,
                    "share_of_step": prof["gemm_ms"] / ms_iso,
                    "measured_in": "second timed pass of the same workload with options.streams=1 (no kernel "
                                   "overlap), CUDA events around every launch on the library stream; the main "
                                   f"pass overlaps GEMM and per-chain kernel on {opts.streams or 'auto'} streams "
                                   f"({ms_max / args.steps:.2f} ms/step vs {ms_iso / args.steps:.2f} ms/step here)",
                    "ess_kernel": {"bound": "hbm", "achieved": ess_gbs, "peak": hbm, "unit": "GB/s",
                                   "frac": ess_gbs / hbm, "peak_source": hbm_src, "avg_launch_ms": ess_avg_ms,
                                   "share_of_step": prof["ess_ms"] / ms_iso,
                                   "algorithmic_bytes_per_launch": prof["ess_bytes"] / max(1, prof["ess_launches"])}}
        if oz:
            # dominant kernel: the int8 tcgen05 projection; peak = measured dense bf16 x the
            # nominal int8 / bf16 ratio (4.5 / 2.25 PFLOP/s), sustained figure (timed inside a long step)
            mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
            tc_avg_ms = prof["tc_ms"] / max(1, prof["tc_launches"])
            tc_ops = prof["tc_ops"] / max(1, prof["tc_launches"])
            tc_achieved = tc_ops / (tc_avg_ms * 1e-3) / 1e12
            tc_peak = 2.0 * mp["bf16_tflops"]
            oz_traffic, oz_traffic_src = None, None
            try:  # dram bytes read + written per launch, committed ncu --set full capture (config 3, N=1)
                tj = json.load(open(os.path.join(ROOT, "profiles", "r01", "ncu_oz_traffic.json")))
                if args.config == 3 and (opts.ozaki_slices or 7) == 7 and not args.precision:
                    oz_traffic, oz_traffic_src = tj["traffic_bytes"], "profiles/r01/ncu_oz_traffic.json"
            except Exception:
                pass
            tc_peak_sus = 2.0 * mp["bf16_tflops_sustained"]
            dmma = {"kernel": "oz_slice_kernel + ozaki_gemm_kernel (P = X A'^T refresh every recompute_every: "
                              "X cut into digits with one exponent per chain, int8 tcgen05)",
                    "avg_launch_ms": roofline["avg_launch_ms"],
                    "fp64_equivalent_tflops": roofline["achieved"],
                    "share_of_step": roofline["share_of_step"]}
            roofline = {"bound": "tensor",
                        "kernel": "ozaki_gemm_kernel (Q = N A'^T, int8 tcgen05.mma, TMEM accumulators, "
                                  + ("4 digits: FP32-class, options.precision = 1)" if args.precision
                                 else f"{opts.ozaki_slices or 7} digits: FP64-accurate)"),
                        "achieved": tc_achieved, "peak": tc_peak, "unit": "TOP/s (int8)",
                        "frac": tc_achieved / tc_peak, "traffic": oz_traffic, "traffic_source": oz_traffic_src,
                        "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst) x 2 = nominal int8/bf16 dense "
                                       "ratio 4.5/2.25 (B200_PROFILING.md); burst, not sustained, because the "
                                       "clocks stay at sm_max during this step (see clocks)",
                        "frac_vs_sustained_peak": tc_achieved / tc_peak_sus,
                        "algorithmic_ops_per_launch": tc_ops,
                        "fp64_equivalent_tflops": prof["tc_flops"] / max(1, prof["tc_launches"]) / (tc_avg_ms * 1e-3) / 1e12,
                        "avg_launch_ms": tc_avg_ms, "share_of_step": prof["tc_ms"] / ms_iso,
                        "measured_in": roofline["measured_in"],
                        "refresh_gemm": dmma, "ess_kernel": roofline["ess_kernel"]}
        # the contract's roofline is the DOMINANT kernel's: when the fused per-chain kernel
        # takes the larger share of the step it moves to the top level (HBM roofline of its
        # algorithmic bytes), the projection GEMM nested beside it
        if roofline["ess_kernel"]["share_of_step"] > roofline["share_of_step"]:
            ess = dict(roofline.pop("ess_kernel"))
            ess["kernel"] = "ess_kernel (arcs, Alg. 3 intervals, theta, P', safeguard, x update, moments, next nu)"
            ess["traffic"], ess["traffic_source"] = None, None
            try:
                sj = json.load(open(os.path.join(ROOT, "profiles", "r01", "ncu_full_int8_summary.json")))
                e = sj["ess_kernel<8>"]
                if args.config == 3 and world == 1 and not args.precision:
                    ess["traffic"] = (float(e["dram__bytes_read.sum"]["value"]) +
                                      float(e["dram__bytes_write.sum"]["value"])) * 1e6
                    ess["traffic_source"] = "profiles/r01/ncu_full_int8_summary.json"
            except Exception:
                pass
            ess["measured_in"] = roofline["measured_in"]
            ess["projection_gemm"] = roofline
            roofline = ess
    gpu_launches = prof_main["launches"]

    # ---- end to end through the public API with host buffers (pinned), rank-local
    e2e = None
    if not args.no_e2e:
        Xh = X.cpu().pin_memory()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            s.sample(Xh, ips, seed, out=Xh)  # H2D of X0 and D2H of the iterates inside the call
        torch.cuda.synchronize()
        dt = tdist.max_over_ranks(time.perf_counter() - t0, dev)
        barrier()
        e2e = {"value": total_iters * m / dt, "unit": UNIT,
               "h2d_bytes_per_step": C * d * 8, "d2h_bytes_per_step": C * d * 8,
               "timer": "host wall clock around synchronous tmvn_sample calls (max over ranks)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_rate(A, b, x0, seed, args.cpu_seconds, C)

    if rank == 0:
        line = {"metric": METRIC32 if args.precision else METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": ("f32-class (int8 x4 projection, f64 elsewhere)" if prof["latency_calls"] == 0 else "f32")
                if args.precision else ("f64+i8" if oz and prof["latency_calls"] == 0 else "f64"),
                "data": "synthetic (seeded Gaussian polytope of BASELINE config; no dataset)",
                "config": config_dict(cfg, args, world),
                "chain_iters_per_s": total_iters / (ms_max * 1e-3),
                "evals_per_s_per_gpu": value / world,
                "rejections": rej_all,
                "recorded": n_all,
                "options": {"streams": opts.streams, "chain_warps": opts.chain_warps,
                            "recompute_every": opts.recompute_every, "ring": opts.ring,
                            "projection": opts.projection, "ozaki_slices": opts.ozaki_slices},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": gpu_launches, "clocks": clocks}
        print(json.dumps(line), flush=True)
    s.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
