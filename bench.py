#!/usr/bin/env python
"""bench.py -- throughput of the B200 ESS hot path (BASELINE.json metric).

A "step" = one tmvn_sample call that runs --iters-per-step iterations of Alg. 1
 for every chain of the workload (every row of SURVEY 8(a): RNG,
projection GEMM, arcs, sort / cummax, theta, update, moments, and the periodic
P refresh), continuing the chains from the previous step.  The headline
workload is BASELINE config 3 (d=1000, m=2000, 4096 chains, FP64) -- the
configuration north_star's target is quoted on; BASELINE configs 1, 2, 4 and 5
are measured in the same run and reported under "configs" (each with its own
roofline entry and CPU-oracle baseline).

  python bench.py [--gpus N --steps K --warmup W --config 3 --impl ours|reference]

N > 1: one process per GPU (NCCL).  Launched by torchrun (RANK / WORLD_SIZE in
the environment), or, when started as a plain `python bench.py --gpus N`,
bench.py re-executes itself under `torch.distributed.run --nproc-per-node N`.
Default scaling is STRONG: the config's total chains are split
over the ranks (dist.shard_options: contiguous global chain blocks, A and b
replicated, options.total_chains so every rank takes the same path); `--scaling
weak` gives every rank the config's C chains instead.  No per-iteration
collective; one all_reduce of the moments and counters and one MAX of the
device times at the end.
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

METRIC = "constraint-evals/sec (chain-iterations/sec x m), FP64, whole job"
METRIC32 = "constraint-evals/sec (chain-iterations/sec x m), FP32-class (--precision 1), whole job"
UNIT = "constraint-evals/s"
# iterations per step (one tmvn_sample call) per config: a step of ~10 ms - 4 s.  Every
# call starts with the strict start check, P = X A'^T in full (a projection-sized GEMM),
# so a step should be a good fraction of the config's run (T in BASELINE.json): config 5
# (T = 100) at 25 iterations per call pays it once per 25 (at 5 it added ~15 % per
# iteration); the refresh cadence inside a call is recompute_every = 32
IPS = {1: 2000, 2: 500, 3: 100, 4: 50, 5: 25, 6: 200, 7: 100}
# algorithmic HBM bytes per constraint-eval of the per-chain kernel --
# P read + write (16 B) and the Q round trip between the projection and it (16 B)
ESS_ALG_BYTES_PER_EVAL = 32.0
L2_FLUSH_BYTES = 256 << 20


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--iters-per-step", type=int, default=0, help="0: per-config default (IPS)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--sub-configs", default="1,2,4,5",
                    help="other BASELINE configs measured in the same run ('' = none)")
    ap.add_argument("--sub-steps", type=int, default=3)
    ap.add_argument("--sub-cpu-seconds", type=float, default=4.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--projection", type=int, default=0,
                    help="options.projection: 0 auto (int8 when d <= 4096), 1 int8 Ozaki split on "
                         "tcgen05 (FP64-accurate), 2 FP64 DMMA")
    ap.add_argument("--streams", type=int, default=0,
                    help="options.streams: 0 auto (chain shards on concurrent streams); 1 one launch per "
                         "kernel over all chains (the ncu captures behind the roofline traffic use it)")
    ap.add_argument("--precision", type=int, default=0,
                    help="options.precision: 0 FP64 (the BASELINE metric), 1 the paper's FP32-class "
                         "mode (int8 projection at 4 digits / FP32 latency kernel; trim_eps 1e-5)")
    return ap.parse_args(argv)


# ------------------------------------------------------------------ multi-process plumbing
def maybe_relaunch(args, argv):
    """`python bench.py --gpus N` (N > 1) outside torchrun: re-exec under torch.distributed.run
    with one process per GPU on this node (rendezvous on 127.0.0.1)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + list(argv)
    sys.exit(subprocess.call(cmd))


def rank_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def plan_shard(C_cfg, rank, world, scaling):
    """Chains of this rank: strong -> a contiguous block of the config's C (the job's total
    is C); weak -> C chains per rank (the job's total is world * C).  Returns the Sampler
    options (chain_offset, total_chains) and the local count."""
    from paper_2407_10449_b200 import dist as tdist
    if scaling == "weak":
        off, cnt = tdist.weak_shard(C_cfg, rank)
        return dict(chain_offset=off, total_chains=C_cfg * world), cnt
    return tdist.shard_options(C_cfg, rank, world)


def job_rate(local_units, local_ms, device):
    """Whole-job throughput: units summed over ranks / the slowest rank's device time."""
    from paper_2407_10449_b200 import dist as tdist
    ms_max = tdist.max_over_ranks(local_ms, device)
    units = tdist.sum_over_ranks(local_units, device)
    return units, ms_max, units / (ms_max * 1e-3)


def host_info():
    info = {"cores": len(os.sched_getaffinity(0))}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            k, v = k.strip(), v.strip()
            if k == "Model name":
                info["cpu_model"] = v
            elif k == "Socket(s)":
                info["sockets"] = int(v) if v.isdigit() else v
            elif k == "CPU(s)":
                info["cpus_online"] = int(v) if v.isdigit() else v
    except Exception:
        pass
    return info


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
def oracle_rate(A, b, x0, seed, seconds, C_full, host):
    """The oracle as it stands, all host cores, on a bounded sample of the workload."""
    import oracle
    cores = host["cores"]
    m = A.shape[0]
    Co = int(max(1, min(C_full, 2 * cores)))
    X0 = np.tile(x0, (Co, 1))
    t0 = time.perf_counter()
    oracle.run(A, b, X0, 1, seed, nthreads=cores)
    one = max(time.perf_counter() - t0, 1e-6)
    To = int(max(1, min(1000, seconds / one)))
    t0 = time.perf_counter()
    oracle.run(A, b, X0, To, seed, nthreads=cores)
    dt = time.perf_counter() - t0
    out = {"value": Co * To * m / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
           "sample": f"{Co} chains x {To} iterations of the same instance (first iterations from x0), "
                     f"{dt:.1f} s on {cores} host threads (OpenMP over chains)",
           "chain_iters_per_s": Co * To / dt, "seconds": dt}
    for k in ("cpu_model", "sockets"):
        if k in host:
            out[k] = host[k]
    return out


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank, world, _ = rank_env()
    if rank != 0:
        return
    from paper_2407_10449_b200 import synth
    import oracle
    cfg = synth.CONFIGS[args.config]
    A, b, x0 = synth.make_instance(args.config)
    host = host_info()
    cores = host["cores"]
    ips = args.iters_per_step or IPS[args.config]
    Co = int(min(cfg.C, 2 * cores))
    X = np.tile(x0, (Co, 1))
    t0 = time.perf_counter()
    oracle.run(A, b, X, 1, cfg.chain_seed, nthreads=cores)
    one = max(time.perf_counter() - t0, 1e-6)
    To = int(max(1, min(ips, 3.0 / one)))  # ~3 s of CPU work per step
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
    cb = {"kind": "oracle", "cores": cores, "value": value, "unit": UNIT,
          "sample": f"each step {Co} chains x {To} iterations of the workload on "
                    f"{cores} host threads (the CPU oracle as it stands)"}
    for k in ("cpu_model", "sockets"):
        if k in host:
            cb[k] = host[k]
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_dict(cfg, args.config, ips, world, args.scaling),
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_dict(cfg, k, ips, world, scaling):
    name = f"BASELINE config {k}" if k <= 5 else "paper S4.2 timing workload (not a BASELINE config)"
    total = cfg.C * (world if scaling == "weak" else 1)
    ws = 8 * (cfg.C / (world if scaling == "strong" else 1) * (4 * cfg.m + 3 * cfg.d) + cfg.m * cfg.d)
    return {"workload": f"{name} ({cfg.key}): {cfg.desc}",
            "d": cfg.d, "m": cfg.m, "chains_total": total,
            "chains_per_gpu": total // world, "iters_per_step": ips, "recompute_every": 32,
            "l2": (f"flushed between timed steps ({L2_FLUSH_BYTES >> 20} MB write, outside the events); "
                   + ("the per-GPU working set (X, nu, P x2, Q, A) exceeds the 126 MB L2 within a step"
                      if ws > 126e6 else
                      "within a step the sampler's state (fits the 126 MB L2) stays resident by design")),
            "parallelism": (f"{'strong' if scaling == 'strong' else 'weak'} scaling: chains sharded over "
                            f"{world} GPU(s) (contiguous global chain blocks), A and b replicated")}


# ------------------------------------------------------------------ our arm
def _peaks():
    mp, src = {}, "MEASURED_PEAKS.json"
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        src = "fallback (B200_PROFILING.md)"
    hbm = mp.get("hbm_gbs", 6650.0)
    bf16 = mp.get("bf16_tflops", 2250.0 * 0.73)
    bf16s = mp.get("bf16_tflops_sustained", bf16)
    return hbm, bf16, bf16s, src


def _fp64_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "profiles", "peaks_fp64_r01.json")))["dfma_tflops_t1024"])
    except Exception:
        return 34.2


def _traffic(k, kernel, args, world):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` at config k from the
    committed ncu --set full capture of this round (profiles/r02/ncu_traffic.json)."""
    if world != 1 or args.precision or args.projection:
        return None, None
    path = os.path.join(ROOT, "profiles", "r02", "ncu_traffic.json")
    try:
        tj = json.load(open(path))
        return float(tj[f"config{k}"][kernel]["bytes_per_launch"]), "profiles/r02/ncu_traffic.json"
    except Exception:
        return None, None


def roofline_entries(prof, ms_iso, k, cfg, Cl, ips, steps, args, world, opts):
    """Per-kernel roofline entries of one workload from the profiled pass (options.profile:
    CUDA events around every hot-loop launch on the library stream, one stream), dominant
    kernel first."""
    hbm, bf16, bf16s, psrc = _peaks()
    m, d = cfg.m, cfg.d
    ents = []
    if prof["latency_calls"] > 0:
        launch_ms = ms_iso / steps
        abytes = float(Cl) * ips * m * d * (4 if args.precision else 8)
        variant = ("a cooperative grid of SMs / C CTAs per chain" if prof.get("latency_grid_calls", 0)
                   else "one thread-block cluster per chain")
        ents.append({"bound": "hbm", "kernel": f"latency_kernel ({variant}: nu, A nu, arcs, two-level Alg. 3 "
                                               "intervals, theta, P', safeguard, x update; all iterations)",
                     "achieved": abytes / (launch_ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                     "frac": abytes / (launch_ms * 1e-3) / 1e9 / hbm, "traffic": None,
                     "peak_source": psrc + " hbm_gbs; A (8 m d bytes per chain-iteration, the algorithmic "
                                    "bytes counted) streams from L2: a bandwidth-equivalent figure",
                     "algorithmic_bytes_per_launch": abytes, "avg_launch_ms": launch_ms, "share_of_step": 1.0,
                     "latency_calls": prof["latency_calls"], "latency_fallbacks": prof["latency_fallbacks"]})
        return ents
    if prof.get("warp_mode_calls", 0) > 0:
        # warp mode: one launch per call, A in shared memory, nothing per iteration in HBM;
        # the bound is the FP64 pipe (FMA) behind the groups' latency: Q = A nu (2 m d flops
        # per chain-iteration, the algorithmic count) against the measured DFMA peak
        launch_ms = ms_iso / steps
        flops = 2.0 * float(Cl) * ips * m * d
        peak = _fp64_peak()
        ents.append({"bound": "alu", "kernel": "small_kernel (warp mode: a group of warps per chain, all "
                                               "iterations, A in shared memory: nu, A nu, arcs, bitonic Alg. 3, "
                                               "theta, P', safeguard, x update, moments)",
                     "achieved": flops / (launch_ms * 1e-3) / 1e12, "peak": peak, "unit": "TFLOP/s (FP64)",
                     "frac": flops / (launch_ms * 1e-3) / 1e12 / peak, "traffic": None,
                     "peak_source": "profiles/peaks_fp64_r01.json dfma_tflops_t1024 (measured FP64 FMA pipe, non-tensor); "
                                    "the projection's 2 m d flops per chain-iteration counted",
                     "algorithmic_flops_per_launch": flops, "avg_launch_ms": launch_ms, "share_of_step": 1.0,
                     "warp_mode_calls": prof["warp_mode_calls"]})
        return ents
    # the fused per-chain kernel: HBM roofline at SURVEY 8(d)'s 32 B per constraint-eval
    nE = max(1, prof["ess_launches"])
    ess_ms = prof["ess_ms"] / nE
    alg = ESS_ALG_BYTES_PER_EVAL * Cl * m
    design = prof["ess_bytes"] / nE
    tr, tsrc = _traffic(k, "ess_kernel", args, world)
    ents.append({"bound": "hbm",
                 "kernel": "ess_kernel (active test, arcs, Alg. 3 intervals, theta, P', safeguard, x update, "
                           "moments, next nu)",
                 "achieved": alg / (ess_ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                 "frac": alg / (ess_ms * 1e-3) / 1e9 / hbm, "traffic": tr, "traffic_source": tsrc,
                 "traffic_ratio": (tr / alg) if tr else None,
                 "peak_source": psrc + " hbm_gbs (measured copy bandwidth)",
                 "algorithmic_bytes_per_launch": alg,
                 "algorithmic_bytes_rule": "SURVEY 8(d): 32 B per constraint-eval (P r/w 16 B + Q round trip "
                                           "16 B) x C x m per launch",
                 "bytes_moved_by_design": design,
                 "bytes_moved_by_design_rule": "the design's own count (runtime.cu run_loop): P, Q read + P' "
                                               "write 24 B per constraint-eval + x r/w, nu read, next nu and "
                                               "its int8 digits per chain-coordinate (+ moment partials when "
                                               "recorded)",
                 "achieved_design_bytes_gbs": design / (ess_ms * 1e-3) / 1e9,
                 "avg_launch_ms": ess_ms, "launches": prof["ess_launches"],
                 "share_of_step": prof["ess_ms"] / ms_iso})
    if prof["tc_launches"] > 0:
        nT = prof["tc_launches"]
        tc_ms = prof["tc_ms"] / nT
        ops = prof["tc_ops"] / nT
        ach = ops / (tc_ms * 1e-3) / 1e12
        S = 4 if args.precision else (opts.ozaki_slices or 7)
        tr, tsrc = _traffic(k, "ozaki_gemm_kernel", args, world)
        ents.append({"bound": "tensor",
                     "kernel": f"ozaki_gemm_kernel (Q = N A'^T: int8 tcgen05.mma, TMEM accumulators, {S} digits"
                               + (": FP32-class)" if args.precision else ": FP64-accurate)"),
                     "achieved": ach, "peak": 2.0 * bf16, "unit": "TOP/s (int8)", "frac": ach / (2.0 * bf16),
                     "frac_vs_sustained_peak": ach / (2.0 * bf16s), "traffic": tr, "traffic_source": tsrc,
                     "peak_source": psrc + " bf16_tflops (burst) x 2 = the nominal int8 / bf16 dense ratio "
                                    "4.5 / 2.25 (B200_PROFILING.md)",
                     "algorithmic_ops_per_launch": ops,
                     "algorithmic_ops_rule": "S(S+1)/2 digit-pair products x 2 C m d per launch",
                     "fp64_equivalent_tflops": prof["tc_flops"] / nT / (tc_ms * 1e-3) / 1e12,
                     "avg_launch_ms": tc_ms, "launches": nT, "share_of_step": prof["tc_ms"] / ms_iso})
    if prof["gemm_launches"] > 0:
        peaks = json.load(open(os.path.join(ROOT, "profiles", "peaks_fp64_r01.json")))
        nG = prof["gemm_launches"]
        g_ms = prof["gemm_ms"] / nG
        fl = prof["gemm_flops"] / nG
        ach = fl / (g_ms * 1e-3) / 1e12 if g_ms > 0 else 0.0
        if prof["tc_launches"] > 0:
            # the refresh runs on the int8 tensor path too (digit slicing of X + the Ozaki GEMM
            # with per-chain column scales): the int8 roofline, like the projection's
            S = 4 if args.precision else (opts.ozaki_slices or 7)
            ops = fl * S * (S + 1) / 2
            ents.append({"bound": "tensor",
                         "kernel": f"refresh P = X A'^T every recompute_every (digit slicing of X + "
                                   f"ozaki_gemm_kernel, {S} digits)",
                         "achieved": ops / (g_ms * 1e-3) / 1e12 if g_ms > 0 else 0.0, "peak": 2.0 * bf16,
                         "unit": "TOP/s (int8)",
                         "frac": (ops / (g_ms * 1e-3) / 1e12 if g_ms > 0 else 0.0) / (2.0 * bf16), "traffic": None,
                         "peak_source": psrc + " bf16_tflops (burst) x 2 (the nominal int8 / bf16 dense ratio)",
                         "algorithmic_ops_per_launch": ops,
                         "algorithmic_ops_rule": "S(S+1)/2 digit-pair products x 2 C m d per launch; the "
                                                 "launch time includes the slicing kernel of X",
                         "fp64_equivalent_tflops": ach, "avg_launch_ms": g_ms, "launches": nG,
                         "share_of_step": prof["gemm_ms"] / ms_iso})
        else:
            ents.append({"bound": "tensor",
                         "kernel": "projection/refresh GEMMs (Q = N A^T and the P refresh, FP64 DMMA, mma.sync f64)",
                         "achieved": ach, "peak": peaks["dmma_tflops_w8"], "unit": "TFLOP/s (FP64)",
                         "frac": ach / peaks["dmma_tflops_w8"], "traffic": None,
                         "peak_source": "measured FP64 DMMA pipe peak (profiles/peaks_fp64_r01.json)",
                         "algorithmic_flops_per_launch": fl, "avg_launch_ms": g_ms, "launches": nG,
                         "share_of_step": prof["gemm_ms"] / ms_iso})
    ents.sort(key=lambda e: -e["share_of_step"])
    return ents


def run_workload(k, args, rank, world, dev, primary, host):
    """Times config k on this rank; returns the workload's result dict (rank 0 complete)."""
    import torch
    import paper_2407_10449_b200 as tm
    from paper_2407_10449_b200 import dist as tdist
    from paper_2407_10449_b200 import synth

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    cfg = synth.CONFIGS[k]
    A, b, x0 = synth.make_instance(k)
    m, d = cfg.m, cfg.d
    ips = (args.iters_per_step or IPS[k]) if primary else IPS[k]
    steps = args.steps if primary else args.sub_steps
    warm = args.warmup if primary else max(3, min(args.warmup, 3))
    seed = cfg.chain_seed
    opts, C = plan_shard(cfg.C, rank, world, args.scaling)
    stream = torch.cuda.Stream(device=dev)
    s = tm.Sampler(torch.tensor(A, device=dev), torch.tensor(b, device=dev), **opts)
    s.set_options(stream=stream, projection=args.projection)
    if args.streams:
        s.set_options(streams=args.streams)
    if args.precision:
        s.set_options(precision=1, trim_eps=1e-5)
    X = torch.tensor(np.tile(x0, (C, 1)), device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    def timed_pass(n):
        """barrier + sync on both sides; CUDA events on the library's stream around each
        step, an L2 flush between steps outside the events; returns the summed device ms."""
        with torch.cuda.stream(stream):
            torch.cuda.synchronize()
            barrier()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
            for e0, e1 in ev:
                flush.zero_()
                e0.record(stream)
                s.sample(X, ips, seed, out=X)
                e1.record(stream)
            torch.cuda.synchronize()
            barrier()
        return sum(e0.elapsed_time(e1) for e0, e1 in ev)

    with torch.cuda.stream(stream):
        for _ in range(warm):
            s.sample(X, ips, seed, out=X)
    s.reset_stats()
    clk = clocks_start() if (rank == 0 and primary) else None
    time.sleep(0.15 if clk else 0)
    ms = timed_pass(steps)  # the library's default launch configuration
    clocks = clocks_stop(clk, set(range(world))) if clk is not None else None
    prof_main = s.profile()
    st = s.stats()
    units, ms_max, rate_iters = job_rate(float(C * ips * steps), ms, dev)
    value = rate_iters * m
    sm, sq, n = s.moments()
    _, _, n_all, rej_all = tdist.reduce_moments(sm, sq, n, st["rejections"], dev)
    o = s.options()
    # roofline pass: same workload, every hot-loop launch bracketed by CUDA events on one
    # stream (streams = 1: no launch overlaps another, so each duration is its own)
    s.set_options(profile=1, streams=1)
    s.reset_stats()
    ms_iso = timed_pass(steps)
    prof = s.profile()
    s.set_options(profile=0, streams=o.streams)
    ents = roofline_entries(prof, ms_iso, k, cfg, C, ips, steps, args, world, o)
    roof = dict(ents[0])
    roof["measured_in"] = ("second timed pass of the same workload with options.profile = 1 and streams = 1 "
                           "(CUDA events around every hot-loop launch on the library stream, no launch "
                           f"overlapping another; graphs off): {ms_iso / steps:.3f} ms/step vs {ms / steps:.3f} "
                           "ms/step in the main pass (library defaults: chain shards on concurrent streams)")
    roof["other_kernels"] = ents[1:]
    e2e = None
    if primary and not args.no_e2e:
        Xh = X.cpu().pin_memory()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            s.sample(Xh, ips, seed, out=Xh)  # H2D of X0 and D2H of the iterates inside the call
        torch.cuda.synchronize()
        dt = tdist.max_over_ranks(time.perf_counter() - t0, dev)
        barrier()
        e2e = {"value": units * m / dt, "unit": UNIT,
               "h2d_bytes_per_step": C * d * 8, "d2h_bytes_per_step": C * d * 8,
               "timer": "host wall clock around synchronous tmvn_sample calls with pinned host X0 / out "
                        "(max over ranks)"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_rate(A, b, x0, seed, args.cpu_seconds if primary else args.sub_cpu_seconds, cfg.C, host)
    s.close()
    del X, flush
    torch.cuda.empty_cache()
    oz = args.projection == 1 or (args.projection == 0 and d <= 4096)
    lat = prof["latency_calls"] > 0
    warp = prof.get("warp_mode_calls", 0) > 0
    dtype = (("f32-class (int8 x4 projection, f64 elsewhere)" if not lat else "f32") if args.precision
             else ("f64+i8" if oz and not lat and not warp else "f64"))
    return {"k": k, "value": value, "ms_per_step": ms_max / steps, "steps": steps, "warmup": warm,
            "chain_iters_per_s": rate_iters, "evals_per_s_per_gpu": value / world, "dtype": dtype,
            "config": config_dict(cfg, k, ips, world, args.scaling), "rejections": rej_all, "recorded": n_all,
            "path": ("latency mode" if lat else "warp mode (small_kernel, all iterations per launch)" if warp
                     else "throughput path (projection GEMM + ess_kernel per iteration)"),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": prof_main["launches"],
            "clocks": clocks,
            "options": {"projection": o.projection, "ozaki_slices": o.ozaki_slices, "chain_warps": o.chain_warps,
                        "recompute_every": o.recompute_every, "latency": o.latency, "total_chains": o.total_chains}}


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    maybe_relaunch(args, argv)
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    rank, world, local = rank_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    host = host_info()
    main_res = run_workload(args.config, args, rank, world, dev, True, host)
    subs = []
    for tok in (args.sub_configs or "").split(","):
        if tok.strip() and int(tok) != args.config:
            subs.append(run_workload(int(tok), args, rank, world, dev, False, host))
    if rank == 0:
        r = main_res
        line = {"metric": METRIC32 if args.precision else METRIC, "value": r["value"], "unit": UNIT,
                "n_gpus": world, "steps": r["steps"], "warmup": r["warmup"], "ms_per_step": r["ms_per_step"],
                "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": r["dtype"],
                "data": "synthetic (seeded Gaussian polytope of the BASELINE config; no dataset)",
                "config": r["config"], "chain_iters_per_s": r["chain_iters_per_s"],
                "evals_per_s_per_gpu": r["evals_per_s_per_gpu"], "rejections": r["rejections"],
                "recorded": r["recorded"], "path": r["path"], "options": r["options"],
                "roofline": r["roofline"], "cpu_baseline": r["cpu_baseline"], "e2e": r["e2e"],
                "gpu_launches": r["gpu_launches"], "clocks": r["clocks"], "host": host,
                "configs": {f"config{x['k']}": dict({kk: x[kk] for kk in
                                                     ("value", "ms_per_step", "steps", "chain_iters_per_s",
                                                      "evals_per_s_per_gpu", "dtype", "config", "path",
                                                      "rejections", "roofline", "cpu_baseline", "gpu_launches")},
                                                    unit=UNIT) for x in subs}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
