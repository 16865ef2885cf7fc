#!/usr/bin/env python
"""Benchmark of the VB inference hot path (BASELINE.json metric: frame-iterations/s).

One "step" = one full inference job on this rank's shard of the workload: nfhmm_reset (initial state
+ z-step), `iters` VB sweeps (all of SURVEY §8(a) rows a-e, g, h) and nfhmm_separate (row f), with
the inputs already resident in HBM.  frame-iterations per step = mixtures * T * iters.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

N > 1: launched by torch.distributed.run, one rank per GPU; the config's mixtures are sharded across
ranks (mixture m on rank m * N // M ... contiguous blocks), no collective on the data path; timings are
all-reduced with MAX (NCCL) after the timed region.  Prints ONE JSON line on rank 0.

--impl reference: the CPU oracle (oracle/, FP64, single-threaded per process) on the host cores,
timed as it stands on a bounded sample of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
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

from paper_1206_6468_b200 import dist as pdist  # noqa: E402
from paper_1206_6468_b200 import synth  # noqa: E402

METRIC = "frame-iterations/sec (S=2,N=40,K=10,F=513) at 1/2/4/8 B200; % FP32/HBM roofline"
UNIT = "frame-iterations/s"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--iters", type=int, default=None, help="VB sweeps per step (default: the config's)")
    ap.add_argument("--mixtures", type=int, default=None, help="override total mixtures (default: config)")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--math", choices=["tc", "simt"], default="tc",
                    help="contraction engine: tcgen05 split products (default: 3xFP16; NFHMM_RECON / NFHMM_BACKPROJ="
                         "tf32 select 3xTF32) or FP32 FFMA")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-bound-off", action="store_true", help="skip the timing with the free energy off")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU seconds for the oracle sample")
    ap.add_argument("--workload", choices=["vb", "train"], default="vb",
                    help="vb: the separation hot path (default); train: N-HMM EM training (SURVEY NEXT-3)")
    ap.add_argument("--train-T", type=int, default=None, help="frames per training source (default 2000)")
    return ap.parse_args()


dist_env = pdist.env
shard = pdist.shard


# ------------------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ------------------------------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
            return
        # the sampler is running before the timed region starts (nvidia-smi takes ~0.1-0.3 s to start);
        # regions shorter than the 200 ms period (small configs) are bracketed by the samples around them
        t0 = time.time()
        while time.time() - t0 < 3.0 and os.path.getsize(self.path) == 0:
            time.sleep(0.02)
        self.n0 = sum(1 for _ in open(self.path))

    def stop(self):
        if self.proc is None:
            return None
        t0 = time.time()
        while time.time() - t0 < 1.0 and sum(1 for _ in open(self.path)) <= getattr(self, "n0", 0):
            time.sleep(0.02)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["active", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names[1:], parts[5:9]):
                if v.lower() in ("active", "1", "yes"):
                    reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return None
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------------------------
# CPU oracle sample (cpu_baseline leg and --impl reference)
# ------------------------------------------------------------------------------------------------
def _oracle_job(args):
    cfg, model, V, iters = args
    from oracle import oracle
    t0 = time.perf_counter()
    oracle.vb_run(model.beta, model.trans, model.prior, V, cfg.dims, iters)
    return time.perf_counter() - t0


def oracle_sample(cfg, model, V0, target_s, procs=1):
    """Time the oracle as it stands on a bounded sample: `procs` independent single-threaded processes,
    each running `iters` sweeps of one mixture truncated to T_s frames.  Returns (value, cores, sample)."""
    from oracle import oracle
    oracle.build()
    T_s = min(cfg.T, 250)
    sub = synth.Config(**{**cfg.__dict__, "T": T_s})
    Vs = np.ascontiguousarray(V0[:T_s])
    t1 = _oracle_job((sub, model, Vs, 1))                       # calibrate one sweep
    iters = max(1, min(50, int(target_s / max(t1, 1e-3))))
    if procs <= 1:
        dt = _oracle_job((sub, model, Vs, iters))
        wall = dt
    else:
        from concurrent.futures import ProcessPoolExecutor
        with ProcessPoolExecutor(max_workers=procs) as ex:
            t0 = time.perf_counter()
            list(ex.map(_oracle_job, [(sub, model, Vs, iters)] * procs))
            wall = time.perf_counter() - t0
    value = procs * T_s * iters / wall
    sample = (f"{procs} process(es) x 1 mixture x T={T_s} frames x {iters} sweeps of cfg{cfg_id(cfg)} "
              f"(S={cfg.S},N={cfg.N},K={cfg.K},F={cfg.F}); {wall:.1f} s wall")
    return value, procs, sample


def cfg_id(cfg):
    for k, v in synth.CONFIGS.items():
        if v.name == cfg.name:
            return k
    return "?"


# ------------------------------------------------------------------------------------------------
def config_line(args, cfg, iters):
    """The `config` object of the JSON line -- identical for both arms (same workload)."""
    return {"workload": f"cfg{args.config}-{cfg.name}", "S": cfg.S, "N": cfg.N, "K": cfg.K, "F": cfg.F, "T": cfg.T,
            "mixtures": cfg.M, "iters": iters, "parallelism": f"mixture-shard x{args.gpus}",
            "l2": "no flush: per-step inputs/state exceed L2 (V, theta and alpha of a step are GBs)" if cfg.M * cfg.T * cfg.F * 4 > 2e8
                  else "no flush: small config (inputs fit in L2)",
            "step": "reset + iters sweeps + separate, inputs resident in memory"}


def _pin_worker(counter, cores):
    """Pool initializer: pin this worker to one host core (taskset equivalent)."""
    with counter.get_lock():
        i = counter.value
        counter.value += 1
    try:
        os.sched_setaffinity(0, {cores[i % len(cores)]})
    except (AttributeError, OSError):
        pass


def run_reference(args):
    """The oracle as it stands (FP64, single-threaded per process), P_cpu = min(host cores, mixtures)
    independent processes pinned one per core, each running whole mixtures of the workload (full T) for
    a bounded number of sweeps per step (the cost per sweep is constant: no early stopping).  Rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    cfg = synth.config(args.config)
    if args.mixtures:
        cfg = synth.Config(**{**cfg.__dict__, "M": args.mixtures})
    iters = args.iters or cfg.iters
    seed = synth.seed_of(args.config)
    model = synth.make_model(cfg, seed)
    try:
        cores = sorted(os.sched_getaffinity(0))
    except AttributeError:
        cores = list(range(os.cpu_count() or 1))
    procs = max(1, min(len(cores), cfg.M))
    # the whole --warmup W --steps K run is sized to finish in a few minutes
    per_step_s = max(2.0, min(20.0, 240.0 / max(1, args.steps + args.warmup)))
    Vs = [synth.make_mixture(cfg, model, seed, m).V for m in range(procs)]
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor
    from oracle import oracle
    oracle.build()
    t1 = _oracle_job((cfg, model, Vs[0], 1))                   # calibrate: one sweep of one full mixture
    sweeps = max(1, int(per_step_s / max(t1, 1e-3)))
    if sweeps == 1 and t1 > per_step_s:                          # very large configs: a frame sample
        T_s = max(1, int(cfg.T * per_step_s / t1))
    else:
        T_s = cfg.T
    sub = synth.Config(**{**cfg.__dict__, "T": T_s})
    jobs = [(sub, model, np.ascontiguousarray(Vs[i][:T_s]), sweeps) for i in range(procs)]
    ctx = mp.get_context("fork")
    counter = ctx.Value("i", 0)
    times = []
    with ProcessPoolExecutor(max_workers=procs, mp_context=ctx, initializer=_pin_worker,
                             initargs=(counter, cores)) as ex:
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            list(ex.map(_oracle_job, jobs))
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                times.append(dt)
    ms = 1000.0 * statistics.mean(times) if times else float("nan")
    value = procs * T_s * sweeps / (ms / 1000.0)
    sample = (f"{procs} processes pinned one per host core, each mixture {0}..{procs - 1} x T={T_s} frames x "
              f"{sweeps} sweeps per step (of the config's {cfg.M} x {cfg.T} frames x {iters} sweeps); mean step time")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_line(args, cfg, iters),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def gather_results(h, cfg, iters, M, world, rank, dev, elapsed_ms):
    """NCCL gathers after the timed region: free-energy traces, d_hat (global mixture order) and the
    per-rank device times (all_gather_into_tensor).  Returns a summary for the JSON line: sizes, the
    gather's device time and digests of the gathered arrays (equal digests across --gpus N = the
    per-mixture results do not depend on the sharding)."""
    import hashlib

    import torch
    import torch.distributed as dist
    S, T, N = cfg.S, cfg.T, cfg.N
    d = torch.empty((M, S, T, N), dtype=torch.float32, device=f"cuda:{dev}")
    fe = np.empty((M, h.max_iters), np.float64)
    from paper_1206_6468_b200.nfhmm import nfhmm_posteriors
    nfhmm_posteriors(h.h, d, None, None, fe)
    fe_d = torch.from_numpy(np.ascontiguousarray(fe[:, :iters])).to(f"cuda:{dev}")
    rows = max(len(shard(cfg.M, world, r)) for r in range(world))
    sizes = [len(shard(cfg.M, world, r)) for r in range(world)]
    torch.cuda.synchronize()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record()
    if world > 1:
        pad = lambda x: torch.cat([x, x.new_zeros((rows - x.shape[0],) + tuple(x.shape[1:]))]) if x.shape[0] < rows else x  # noqa: E731
        fe_all = torch.empty((world * rows, iters), dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_gather_into_tensor(fe_all, pad(fe_d))
        # d_hat of every mixture, in global order (all_gather: every rank receives it; rank 0 digests it)
        d_all = torch.empty((world * rows, S, T, N), dtype=torch.float32, device=f"cuda:{dev}")
        dist.all_gather_into_tensor(d_all, pad(d))
        times = torch.empty(world, dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_gather_into_tensor(times, torch.tensor([elapsed_ms], dtype=torch.float64, device=f"cuda:{dev}"))
        keep = torch.cat([torch.arange(r * rows, r * rows + sizes[r], device=f"cuda:{dev}") for r in range(world)])
        fe_all = fe_all[keep]
        d_all = d_all[keep]
    else:
        fe_all, d_all = fe_d, d
        times = torch.tensor([elapsed_ms], dtype=torch.float64)
    g1.record()
    torch.cuda.synchronize()
    out = {"collective": "nccl all_gather of the free energies, d_hat and the device times" if world > 1
           else "none (1 rank)", "ms": g0.elapsed_time(g1),
           "bytes": int(cfg.M * S * T * N * 4 + cfg.M * iters * 8 + world * 8),
           "rank_ms": [round(float(x), 3) for x in times.cpu().tolist()]}
    if rank == 0:
        fe_h = fe_all.cpu().numpy()
        out["mixtures"] = int(fe_h.shape[0])
        out["L_final_sum"] = float(fe_h[:, -1].sum())
        out["L_digest"] = hashlib.sha256(fe_h.tobytes()).hexdigest()[:16]
        out["d_hat_digest"] = hashlib.sha256(d_all.cpu().numpy().tobytes()).hexdigest()[:16]
    del d, d_all
    return out


def relaunch_command(args_argv, gpus, port):
    """bench.py --gpus N (N > 1) run outside torchrun: the same command under torch.distributed.run,
    one rank per GPU of this node (the driver's own launch line)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *args_argv]


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch with torchrun "
                         f"--nproc-per-node {args.gpus} (or without WORLD_SIZE to let bench.py launch it)")
    if torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py: --gpus {world} needs {world} visible GPUs, found {torch.cuda.device_count()}")
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    from paper_1206_6468_b200.nfhmm import NFHMM, KERNEL_CLASSES

    cfg = synth.config(args.config)
    if args.mixtures:
        cfg = synth.Config(**{**cfg.__dict__, "M": args.mixtures})
    iters = args.iters or cfg.iters
    seed = synth.seed_of(args.config)
    model = synth.make_model(cfg, seed)
    mine = shard(cfg.M, world, rank)
    M = len(mine)
    t_gen = time.perf_counter()
    V = synth.make_batch(cfg, model, seed, mine)           # [M][T][F] float32, this rank's shard only
    t_gen = time.perf_counter() - t_gen

    stream = torch.cuda.current_stream(dev)
    h = NFHMM(cfg.F, cfg.T, cfg.S, cfg.N, cfg.K, n_mix=M, device=dev, max_iters=max(iters, 1), stream=stream,
              math=args.math)
    h.set_model(model.beta, model.trans, model.prior)
    Vd = torch.from_numpy(V).to(f"cuda:{dev}")
    h.set_observations(Vd)
    vstar_d = torch.empty((M, cfg.S, cfg.T, cfg.F), dtype=torch.float32, device=f"cuda:{dev}")

    def step():
        h.reset()
        h.vb_iterate_async(iters)
        h.separate_into(vstar_d)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(dev)
    clocks.start()
    l0 = h.kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    launches = h.kernel_launches() - l0
    clk = clocks.stop()
    elapsed = ev0.elapsed_time(ev1)
    if world > 1:
        elapsed = pdist.max_over_ranks(elapsed, device=f"cuda:{dev}")
        dist.barrier()
    # per-kernel device times (rooflines, shares): the same steps again with every launch bracketed by
    # CUDA events on the library's stream -- outside the timed region (the events and the eager launches
    # they force would perturb it).  Profiling also turns off the FB / reconstruction overlap, so these
    # are standalone kernel times (in the timed steps the FB runs beside the reconstruction GEMM).
    # ---- gather (north_star: NCCL only to gather posteriors, free energies and timings) -------------
    # After the timed region and outside it: every rank's free-energy traces all-gathered, the
    # posteriors d_hat gathered to rank 0 in global mixture order, per-rank device times all-gathered.
    gathered = gather_results(h, cfg, iters, M, world, rank, dev, elapsed)
    h.profile_enable(True)
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    prof = h.profile_read()
    products = h.products()   # how (a) / (b) form their products: 3xfp16 / 3xtf32 / ffma
    h.profile_enable(False)
    ms_per_step = elapsed / args.steps
    frame_iters = cfg.M * cfg.T * iters                     # whole job, all ranks
    value = frame_iters / (ms_per_step / 1000.0)

    # ---- the same steps with the bound off (report L-on and L-off) ------------------
    value_bound_off = None
    if not args.no_bound_off:
        hb = NFHMM(cfg.F, cfg.T, cfg.S, cfg.N, cfg.K, n_mix=M, device=dev, max_iters=max(iters, 1), stream=stream,
                   math=args.math, free_energy=False)
        hb.set_model(model.beta, model.trans, model.prior)
        hb.set_observations(Vd)

        def step_b():
            hb.reset()
            hb.vb_iterate_async(iters)
            hb.separate_into(vstar_d)

        step_b()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(stream)
        for _ in range(args.steps):
            step_b()
        b1.record(stream)
        torch.cuda.synchronize()
        elb = b0.elapsed_time(b1)
        if world > 1:
            elb = pdist.max_over_ranks(elb, device=f"cuda:{dev}")
        value_bound_off = frame_iters / (elb / args.steps / 1000.0)
        hb.close()
        del hb
        torch.cuda.empty_cache()

    # ---- e2e: public API with host buffers, copies inside the timed region -------------------
    # Every step copies its V from pinned host memory, runs the sweeps and the separation through the public
    # API, and reads the separated spectrograms back into pinned host memory.  The host->device copy of a
    # step (into one of two device input buffers) and the device->host copy of its V* (from one of two device
    # output buffers) run on two copy streams beside the other steps' computes, ordered by events (a buffer
    # is refilled only after the step that used it).  Large batches (> 65,536 frames: the GPU is full) run
    # the steps back to back on one handle -- two handles on two streams let the steps' kernels interleave
    # with the tuned SM partition and measured 5 % slower at config 3; small ones alternate between two
    # handles on two streams, whose computes then overlap (single mixtures leave most SMs idle).
    # The timed region spans every step's copies.
    e2e = None
    if not args.no_e2e:
        Vh = torch.from_numpy(V).pin_memory()
        out_h = [torch.empty((M, cfg.S, cfg.T, cfg.F), dtype=torch.float32).pin_memory() for _ in range(2)]
        Vd = [torch.empty(Vh.shape, dtype=torch.float32, device=f"cuda:{dev}") for _ in range(2)]
        out_d = [torch.empty(out_h[0].shape, dtype=torch.float32, device=f"cuda:{dev}") for _ in range(2)]
        nh = 1 if M * cfg.T > 65536 else 2
        csts = [torch.cuda.Stream(dev) for _ in range(nh)]      # the handles' compute streams
        h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        hes = [NFHMM(cfg.F, cfg.T, cfg.S, cfg.N, cfg.K, n_mix=M, device=dev, max_iters=max(iters, 1), stream=c,
                     math=args.math) for c in csts]
        for he in hes:
            he.set_model(model.beta, model.trans, model.prior)
        ev_comp, ev_out = [None, None], [None, None]

        def e2e_step(i):
            k = i % 2
            he, cst = hes[i % nh], csts[i % nh]
            with torch.cuda.stream(h2d):                  # V of step i into Vd[k] (free once step i-2 computed)
                if ev_comp[k] is not None:
                    h2d.wait_event(ev_comp[k])
                Vd[k].copy_(Vh, non_blocking=True)
                e_in = torch.cuda.Event()
                e_in.record(h2d)
            cst.wait_event(e_in)
            if ev_out[k] is not None:                     # out_d[k] read back (step i-2)
                cst.wait_event(ev_out[k])
            he.set_observations(Vd[k])
            he.vb_iterate_async(iters)
            he.separate_into(out_d[k], sync=False)
            e_c = torch.cuda.Event()
            e_c.record(cst)
            ev_comp[k] = e_c
            with torch.cuda.stream(d2h):                  # V* of step i back to the host
                d2h.wait_event(e_c)
                out_h[k].copy_(out_d[k], non_blocking=True)
                e_o = torch.cuda.Event()
                e_o.record(d2h)
            ev_out[k] = e_o

        for i in range(2):   # warm up (graph capture, first-touch)
            e2e_step(i)
        torch.cuda.synchronize()
        for he in hes:
            he.sync()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        j0 = torch.cuda.Event()
        e0.record(stream)
        j0.record(stream)
        for st in (*csts, h2d, d2h):
            st.wait_event(j0)
        for i in range(args.steps):
            e2e_step(i)
        for st in (*csts, h2d, d2h):
            stream.wait_stream(st)
        e1.record(stream)
        torch.cuda.synchronize()
        for he in hes:
            he.sync()   # sticky device flags of every step
        el = e0.elapsed_time(e1)
        if world > 1:
            el = pdist.max_over_ranks(el, device=f"cuda:{dev}")
        e2e = {"value": frame_iters / (el / args.steps / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": int(Vh.numel() * 4) * world, "d2h_bytes_per_step": int(out_h[0].numel() * 4) * world,
               "ms_per_step": el / args.steps,
               "pipeline": (f"{nh} handle(s) on {nh} compute stream(s); each step's H2D and D2H on two copy streams "
                            "beside the other steps' computes")}
        for he in hes:
            he.close()
        del Vd, out_d
        torch.cuda.empty_cache()

    # ---- roofline of the dominant kernel ------------------------------------------------------
    peaks = json.load(open(PEAKS_PATH)) if os.path.exists(PEAKS_PATH) else {}
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    fp32_peak = 148 * 128 * 2 * sm_max * 1e6 / 1e12      # TFLOP/s, FFMA pipe (DESIGN "Rooflines")
    hbm_peak = float(peaks.get("hbm_gbs", 6539.2))
    frames_local = M * cfg.T
    SN = cfg.S * cfg.N

    def roofline_of(k):
        """Algorithmic work per launch of kernel class k (DESIGN "Kernels, rooflines") over its live
        CUDA-event launch time, against the kernel's roofline."""
        ms_k, n_k = prof[k]
        if not n_k:
            return None
        t_launch = ms_k / n_k / 1000.0
        if k in ("recon", "backproj"):
            flops = 2.0 * frames_local * cfg.F * cfg.Kt       # algorithmic FLOPs per launch (true F, Kt)
            achieved = flops / t_launch / 1e12
            kind = products["recon" if k == "recon" else "backproj"]
            if kind in ("3xtf32", "3xfp16"):
                # FP32-accurate contraction as three split products on tcgen05.  3xTF32: TF32 dense = measured
                # bf16 x 1/2 (nominal 1.1 / 2.25 PFLOP/s); 3xFP16: FP16 dense = the bf16 rate.  Three MMAs per
                # product -> FP32-equivalent peak = that / 3.  The GEMMs run inside a long step (hundreds of
                # ms back to back, power-capped clocks), so the sustained bf16 figure is the denominator (the
                # recipe's rule); the burst-based fraction is reported too.
                rate = 0.5 if kind == "3xtf32" else 1.0
                bf16_s = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1645.8)))
                bf16_b = float(peaks.get("bf16_tflops", 1645.8))
                peak = bf16_s * rate / 3.0
                # also against the nominal dense peak (2.25 PFLOP/s bf16 -> 375 / 750 TFLOP/s)
                # at the maximum and at the measured SM clock of the timed steps
                nominal = 2250.0 * rate / 3.0
                clk_mhz = (clk or {}).get("sm_mhz") or sm_max
                dt = "TF32" if kind == "3xtf32" else "FP16"
                return {"kernel": k, "bound": "tensor", "products": kind, "achieved": achieved, "peak": peak,
                        "unit": "TFLOP/s", "frac": achieved / peak, "frac_vs_burst": achieved / (bf16_b * rate / 3.0),
                        "frac_vs_nominal_max_clock": achieved / nominal,
                        "frac_vs_nominal_at_clock": achieved / (nominal * clk_mhz / sm_max),
                        "peak_note": f"3x{dt} FP32-equivalent: measured sustained bf16 {bf16_s} TF/s x {rate:g} ({dt}) / 3",
                        # the same work against the 3xTF32 roofline (the north star's split; round 1's denominator)
                        "frac_vs_3xtf32_peak": achieved / (bf16_s * 0.5 / 3.0),
                        "fp32_ffma_peak": fp32_peak}
            return {"kernel": k, "bound": "alu", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                    "frac": achieved / fp32_peak, "peak_note": f"FP32 FFMA 148 SM x 128 lanes x 2 x {sm_max:.0f} MHz"}
        if k == "dirichlet":
            # read n (Kt) + FB messages u, b (2 S N) + frame constants (32 B); write theta (Kt) + emissions
            # (S N) + offsets (8 S) + bound term (8); alpha (Kt) on the last sweep of the call only
            byts = frames_local * (2 * cfg.Kt * 4 + 3 * SN * 4 + cfg.S * 8 + 8 + 32 + cfg.Kt * 4 / iters)
        else:   # fb: read emissions (N) + offsets (8), write u and b (2 N) per chain-frame
            byts = M * cfg.S * cfg.T * (3 * cfg.N * 4 + 8)
        achieved = byts / t_launch / 1e9
        return {"kernel": k, "bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak}

    dom = max(("recon", "backproj", "dirichlet", "fb"), key=lambda k: prof[k][0])
    roof = roofline_of(dom)
    roof_all = {k: {kk: v for kk, v in (roofline_of(k) or {}).items() if kk in ("bound", "achieved", "frac", "unit", "products")}
                for k in ("recon", "backproj", "dirichlet", "fb")}
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        tr = json.load(open(tpath)).get(f"cfg{args.config}", {}).get(dom)
        if tr:
            traffic = tr.get("dram_bytes_per_launch")
    roof["traffic"] = traffic
    kernels = {k: {"ms_per_step": prof[k][0] / args.steps, "launches_per_step": prof[k][1] / args.steps}
               for k in KERNEL_CLASSES if prof[k][1]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        val, cores, sample = oracle_sample(cfg, model, V[0], args.cpu_seconds, procs=1)
        cpu = {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_line(args, cfg, iters),
            "value_bound_off": value_bound_off, "gathered": gathered,
            "roofline": roof, "rooflines": roof_all, "kernels": kernels, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
            "gpu_launches": launches, "gen_seconds": round(t_gen, 2),
        }
        print(json.dumps(line), flush=True)
    h.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------------------------------------------
# --workload train: N-HMM maximum-likelihood EM, one GPU
# ------------------------------------------------------------------------------------------------
TRAIN_METRIC = "EM frame-iterations/sec, N-HMM training (isolated sources, N=40,K=10,F=513)"


def run_train(args):
    """Each step: reset to the EM start, `iters` EM iterations over every source of the config (each
    source's isolated spectrogram, T frames), parameters read back.  value = sources x T x iters / time."""
    import torch
    from paper_1206_6468_b200.nfhmm import NHMMTrainer
    torch.cuda.set_device(0)
    cfg = synth.config(args.config)
    T = args.train_T or 2000
    iters = args.iters or 10
    seed = synth.seed_of(args.config)
    model = synth.make_model(cfg, seed)
    V = synth.make_training_data(cfg, model, seed, T)
    b0, a0, p0 = synth.make_em_init(cfg, seed)
    dev = "cuda:0"
    Vd = torch.from_numpy(V).to(dev)
    b0d, a0d, p0d = (torch.from_numpy(x).to(dev) for x in (b0, a0, p0))
    stream = torch.cuda.current_stream()
    tr = NHMMTrainer(cfg.F, T, cfg.N, cfg.K, n_src=cfg.S, max_iters=iters, stream=stream)
    tr.set_data(Vd)
    out = torch.empty((cfg.S, cfg.N, cfg.K, cfg.F), dtype=torch.float32, device=dev)

    def step():
        tr.set_params(b0d, a0d, p0d)
        tr.em(iters)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = Clocks(0)
    clocks.start()
    l0 = tr.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    launches = tr.kernel_launches() - l0
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    units = cfg.S * T * iters
    value = units / (ms / 1000.0)
    ll = tr.get()["loglik"]
    cpu = None
    if not args.no_cpu_baseline:   # the oracle on a bounded sample: one source, T_s frames, a few iterations
        from oracle import oracle
        oracle.build()
        T_s = min(T, 100)
        th = np.full((T_s, cfg.N, cfg.K), 1.0 / cfg.K)
        t0 = time.perf_counter()
        oracle.nhmm_em(V[0, :T_s], b0[0], th, a0[0], p0[0], 1)
        t1 = time.perf_counter() - t0
        it_s = max(1, min(20, int(args.cpu_seconds / max(t1, 1e-3))))
        t0 = time.perf_counter()
        oracle.nhmm_em(V[0, :T_s], b0[0], th, a0[0], p0[0], it_s)
        wall = time.perf_counter() - t0
        cpu = {"value": T_s * it_s / wall, "unit": "frame-iterations/s", "cores": 1, "kind": "oracle",
               "sample": f"1 source x T={T_s} frames x {it_s} EM iterations (N={cfg.N},K={cfg.K},F={cfg.F}); {wall:.1f} s wall"}
    line = {"metric": TRAIN_METRIC, "value": value, "unit": "frame-iterations/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32 (f64 log-likelihood)", "data": "synthetic",
            "config": {"workload": f"train-cfg{args.config}", "sources": cfg.S, "N": cfg.N, "K": cfg.K, "F": cfg.F,
                       "T": T, "iters": iters, "step": "reset to the EM start + iters EM iterations, data resident"},
            "loglik_first_last": [float(ll[0, 0]), float(ll[0, -1])], "cpu_baseline": cpu, "clocks": clk,
            "gpu_launches": launches}
    print(json.dumps(line), flush=True)
    tr.close()
    return 0


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        return subprocess.call(relaunch_command(sys.argv[1:], args.gpus, _free_port()))
    if args.workload == "train":
        return run_train(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
