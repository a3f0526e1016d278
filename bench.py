#!/usr/bin/env python
"""Benchmark of the B200 Barnes-Hut step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl ours|reference]

A "step" is one bh_step: the whole hot path (K0 root cube, K1 keys, K2 radix
sort, K4 octree, K5 moments, K6+K7 walk + leapfrog, K8 exchange when N > 1) over
the full particle set.  Default workload: BASELINE cfg4 (N = 2^24 Plummer,
theta = 0.5, eps = 1e-3, dt = 1e-4), the largest configuration that fits one GPU
and the one the 1/2/4/8-GPU metric is quoted on.  Inputs (pos4 268 MB, tree
records ~1.1 GB) are larger than the 126 MB L2, so no flush is needed.

`value` = total Barnes-Hut interactions of the K timed steps over all ranks /
max-over-ranks device time (CUDA events on the library stream), i.e. whole-job
interactions/s; particles/s is reported beside it.  For N > 1 the script runs
under torchrun, one rank per GPU, NCCL over NVLink (strong scaling: N fixed).

`--impl reference` times the plain fp64 CPU oracle (oracle/, the parity
reference) on the box's host cores on a bounded sample of the same workload;
it is the slow reference arm, not a target.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import bhgen  # noqa: E402

METRIC = "BH interactions/s and particles/s per step at 1/2/4/8 B200; % FP32 peak"
UNIT = "interactions/s"
FLOP_PER_INTERACTION = 18  # dx,dy,dz 3 + d2 5 + r2 1 + rsqrt^3 2 + M* 1 + acc 6 (rsqrt itself not counted)
FLOP_PER_OPEN = 8          # the MAC distance of a node that is opened: 3 sub + 5
FLOP_PER_QUAD = 38         # multipole = 2: Q dr 15, dr.Q dr 5, inv^5 / inv^7 4, 2.5 s inv^7 2, accumulate 12


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def fp32_peak_tflops(sm_count: int, mhz: float) -> float:
    # 128 FP32 lanes per SM, FFMA = 2 flop (B200_PROFILING.md: 148 SMs, 1965 MHz max)
    return 2.0 * 128 * sm_count * mhz * 1e6 / 1e12


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                rows.append((float(f[1]), float(f[2]), f[5:9]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v.lower() == "active"})
        loaded = [r[0] for r in rows if r[0] > 600] or [r[0] for r in rows]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "samples": len(rows)}


def load_traffic(kernel_key: str, workload: str):
    """dram bytes per launch of the walk from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        k = d["kernels"][kernel_key]
        if d.get("workload") != workload:
            return None, None
        return k.get("dram_bytes_per_launch"), os.path.relpath(path, ROOT)
    except (OSError, KeyError, ValueError):
        return None, None


# --------------------------------------------------------------------- oracle arm
def run_oracle_sample(cfg, m, p, v, samples: int, reps: int, warm: int):
    """Time the fp64 oracle as it stands: one full tree build, then `reps` walks
    of `samples` random targets.  Returns a dict of rates."""
    import oracle

    n = m.shape[0]
    prm = bhgen.params(cfg)
    t0 = time.perf_counter()
    o = oracle.Oracle(m, p.astype(np.float64), v.astype(np.float64), **prm)
    o.build()
    t_build = time.perf_counter() - t0
    rng = np.random.default_rng(12345)
    walk_t, inter = [], []
    for r in range(warm + reps):
        tg = rng.choice(n, min(samples, n), replace=False)
        t1 = time.perf_counter()
        _, cnt = o.forces(tg)
        dt = time.perf_counter() - t1
        if r >= warm:
            walk_t.append(dt)
            inter.append(int(cnt.sum()))
    o.close()
    s_tot = min(samples, n) * reps
    walk_rate = sum(inter) / sum(walk_t)  # interactions/s of the walk alone
    mean_i = sum(inter) / s_tot
    # one whole step extrapolated: full build + all-particle walk at the sampled rate
    t_step = t_build + n * mean_i / walk_rate
    return {"interactions_per_s": n * mean_i / t_step, "particles_per_s": n / t_step, "t_build_s": t_build,
            "walk_interactions_per_s": walk_rate, "mean_interactions": mean_i, "t_step_extrapolated_s": t_step,
            "cores": len(os.sched_getaffinity(0)), "samples": min(samples, n), "reps": reps,
            "step_times": walk_t}


def reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0  # only rank 0 runs the CPU reference
    cfg = bhgen.CONFIGS[args.config]
    m, p, v = bhgen.generate(cfg)
    samples = args.ref_samples
    r = run_oracle_sample(cfg, m, p, v, samples, args.steps, args.warmup)
    val = r["interactions_per_s"]
    sample_desc = (f"full fp64 oracle tree build of all N={cfg.n} ({r['t_build_s']:.1f} s) + {args.steps} timed "
                   f"walks of {r['samples']} random targets each ({args.warmup} warm-up); whole-step rate "
                   f"extrapolated per particle")
    out = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["t_step_extrapolated_s"] * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(cfg, m, p, v),
        "particles_per_s": r["particles_per_s"],
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": r["cores"], "kind": "oracle", "sample": sample_desc,
                         "walk_interactions_per_s": r["walk_interactions_per_s"], "t_build_s": r["t_build_s"]},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)
    return 0


def walk_kernel_name(cfg, walk_group, multipole=1):
    """The k_walk instance bh_step runs (api.cu's automatic choice for walk_group 0)."""
    shapes = {66: (8, 2), 67: (4, 2), 68: (2, 2), 69: (2, 4), 70: (1, 4)}
    g = walk_group
    if g == 0 and multipole == 2:
        g = 67 if cfg.theta < 0.6 and cfg.n >= (1 << 22) else 68
    elif g == 0:
        g = (69 if cfg.theta < 0.6 else 70) if cfg.n >= (1 << 22) else 69 if cfg.n >= (1 << 19) else 68
    lanes, tpl = shapes[g]
    return f"k_walk<{lanes},{tpl // 2}> (walk_group {g}): {lanes * tpl}-target groups, {lanes} lanes x {tpl} targets"


def workload_config(cfg, m, p, v):
    return {"workload": f"{cfg.name}: N={cfg.n} {cfg.kind}, theta={cfg.theta}, eps={cfg.eps}, dt={cfg.dt}, G={cfg.G}",
            "n": cfg.n, "theta": cfg.theta, "eps": cfg.eps, "dt": cfg.dt, "seed": cfg.seed,
            "input_sha256": bhgen.digest(m, p, v)[:16],
            "l2": "inputs larger than L2 (pos4 16 B x N, tree records ~50 B x 1.5 N); no flush"}


# --------------------------------------------------------------------- our arm
def ours_arm(args):
    import torch
    import torch.distributed as dist

    from paper_1109_5190_b200 import BarnesHut, bh as bhmod
    from paper_1109_5190_b200 import dist as bdist

    rank, world, local = bdist.env_rank()
    if world != args.gpus and not (world == 1 and args.gpus == 1):
        print(f"--gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    device = local if world > 1 else 0
    torch.cuda.set_device(device)
    comm = None
    nccl_info = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{device}"))
        uid = bdist.share_nccl_id(bhmod.nccl_unique_id, dist)
        comm = bhmod.nccl_comm_init(uid, world, rank, device)
        nccl_info = bhmod.nccl_comm_info(comm)
        print(f"rank {rank}: NCCL communicator spans {nccl_info['count']} ranks (this rank {nccl_info['rank']}, "
              f"cuda:{nccl_info['device']})", file=sys.stderr, flush=True)
        if nccl_info["count"] != world:
            raise RuntimeError(f"NCCL communicator has {nccl_info['count']} ranks, WORLD_SIZE={world}")
    else:
        nccl_info = None
    cfg = bhgen.CONFIGS[args.config]
    m, p, v = bhgen.generate(cfg)
    prm = bhgen.params(cfg)
    bh = BarnesHut(m, p, v, device=device, rank=rank, world=world, nccl_comm=comm, walk_group=args.walk_group,
                   multipole=args.multipole, **prm)
    stream = bh.stream
    exchange_kind = "nccl_broadcast" if world > 1 else None
    if world > 1 and args.exchange == "fused":
        # K8 fused into K7: every rank's replica opened by CUDA IPC, the walk
        # epilogue stores into all of them; the step's two barriers are one-word
        # NCCL all-reduces inside the captured graph (bh_set_peers)
        bdist.share_replicas(bh, dist)
        exchange_kind = "fused_peer_stores"
    props = torch.cuda.get_device_properties(device)
    sms = props.multi_processor_count

    def barrier():
        if world > 1:
            dist.barrier()

    def allreduce(x, op):
        if world == 1:
            return x
        return bdist.reduce_scalar(x, dist, "max" if op == dist.ReduceOp.MAX else "sum", device=f"cuda:{device}")

    # warm-up (untimed)
    bh.step(args.warmup)
    bh.sync()
    if world > 1 and not args.no_rebalance:
        # equal-cost ownership: the walk trips of each particle's group, rescaled
        # per rank to its measured walk time (dist.time_scaled; two feedback
        # rounds, each from one profiled untimed step), then one more untimed
        # step on the new partition
        try:
            for _ in range(2):
                bh.set_profiling(True)
                bh.step(1)
                walk_ms = bh.get_profile()["ms"]["walk"]
                bh.set_profiling(False)
                bounds = bdist.rebalance(bh, dist, device=f"cuda:{device}", walk_ms=walk_ms)
            if rank == 0:
                print(f"rebalanced ownership: {bounds}", file=sys.stderr)
        except Exception as e:  # keep the even split
            print(f"rebalance skipped: {e}", file=sys.stderr)
        bh.step(1)
        bh.sync()
    # (1) per-phase breakdown: K steps with CUDA events around every phase
    # (direct launches); explanatory only -- the events cost ~0.1 ms per step
    bh.set_profiling(True)
    barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        bh.step(1)
    torch.cuda.synchronize()
    prof = bh.get_profile()
    bh.set_profiling(False)
    # (2) the timed region: K steps as the library runs them (one CUDA-graph
    # replay per step; direct launches for N > 1 with NCCL), CUDA events on the
    # library stream, a barrier + synchronize on both sides, clocks sampled
    bh.step(1)
    barrier()
    torch.cuda.synchronize()
    st0 = bh.get_stats()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(device) as clk:
        ev0.record(stream)
        for k in range(args.steps):
            if world > 1 and args.rebalance_every > 0 and k > 0 and k % args.rebalance_every == 0:
                # NEXT-2: equal-cost ownership from the last walk's trips, inside the
                # timed region (host collectives: its cost is part of the step)
                bdist.rebalance(bh, dist, device=f"cuda:{device}")
            bh.step(1)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms_local = ev0.elapsed_time(ev1)
    st1 = bh.get_stats()
    barrier()
    ms = allreduce(ms_local, dist.ReduceOp.MAX if world > 1 else None)
    inter_local = st1["interactions_cum"] - st0["interactions_cum"]
    # opened-node count (for the flop model) from one untimed stats walk on the
    # final state: the timed walks run without the stats counters
    bh.set_walk_stats(True)
    bh.build_tree()
    bh._chk(bh.L.bh_compute_forces(bh.h, None, bhmod.BH_DEVICE))
    sts = bh.get_stats()
    bh.set_walk_stats(False)
    opens_local = inter_local * sts["opens"] / max(1, sts["interactions"])
    inter = allreduce(float(inter_local), dist.ReduceOp.SUM if world > 1 else None)
    opens = allreduce(float(opens_local), dist.ReduceOp.SUM if world > 1 else None)
    secs = ms / 1e3
    value = inter / secs
    particles_per_s = cfg.n * args.steps / secs

    # roofline of the dominant kernel (the walk), measured live with CUDA events
    walk_ms = prof["ms"]["walk"] / args.steps
    fpi = FLOP_PER_INTERACTION + (FLOP_PER_QUAD if args.multipole == 2 else 0)
    flops_walk_launch = (fpi * inter_local + FLOP_PER_OPEN * opens_local) / args.steps
    achieved_tf = flops_walk_launch / (walk_ms / 1e3) / 1e12
    peaks = measured_peaks()
    sm_max = peaks.get("sm_max_mhz", 1965.0)
    peak = fp32_peak_tflops(sms, sm_max)
    clocks = clk.summary()
    # the committed ncu capture is of the default (monopole) walk of this config
    traffic, traffic_src = load_traffic("walk", f"{cfg.name}") if args.multipole == 1 else (None, None)
    phase_ms = {k: vv / args.steps for k, vv in prof["ms"].items()}
    # keys + sort phase: the near-sorted path (previous order) moves 88 B per key
    # (K1' 32, mark 8, split 24, merge 24) + the out-of-order keys' radix passes;
    # the full path 32 B (K1) + 8 passes x (8 B key + 4 B id) read + written
    near = st1.get("near_sorted", True)
    sort_bytes = (88 if near else 32 + 8 * 24) * cfg.n
    sort_gbs = sort_bytes / (phase_ms["keys_sort"] / 1e3) / 1e9 if phase_ms["keys_sort"] > 0 else None
    launches = sum(prof["launches"].values())

    # e2e: through the public API with host buffers, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
        hm, hp, hv = pin(m), pin(p), pin(v)
        op = torch.empty((cfg.n, 3), dtype=torch.float32).pin_memory().numpy()
        ov = torch.empty((cfg.n, 3), dtype=torch.float32).pin_memory().numpy()
        bh.set_state(hm, hp, hv)
        bh.advance(None, hp, hv, 1, op, ov)  # warm the path
        e_steps = max(1, min(args.steps, 5))
        barrier()
        torch.cuda.synchronize()
        s0 = bh.get_stats()["interactions_cum"]
        t0 = time.perf_counter()
        for _ in range(e_steps):
            # one bh_advance per step: positions + velocities in (masses do not
            # change and stay on the device), one step, positions + velocities out
            bh.advance(None, hp, hv, 1, op, ov)
        torch.cuda.synchronize()
        t_e = allreduce(time.perf_counter() - t0, dist.ReduceOp.MAX if world > 1 else None)
        e_inter = allreduce(float(bh.get_stats()["interactions_cum"] - s0), dist.ReduceOp.SUM if world > 1 else None)
        e2e = {"value": e_inter / t_e, "unit": UNIT, "h2d_bytes_per_step": int(cfg.n * (12 + 12)),
               "d2h_bytes_per_step": int(cfg.n * (12 + 12)), "steps": e_steps,
               "ms_per_step": t_e / e_steps * 1e3,
               "path": "bh_advance(pinned host positions + velocities in, masses kept; 1 step; positions + "
                       "velocities out) per step"}

    # ownership balance for P = 2/4/8 from this GPU's per-particle costs (the
    # last walk's interaction counts, storage order): the even Morton-range split
    # of the multi-GPU path vs the equal-cost split of bh_set_partition
    balance = None
    if world == 1:
        costs, _ = bh.get_own()
        costs = costs.astype(np.float64)
        balance = {"cost": "interactions per particle, last walk"}
        for P in (2, 4, 8):
            even = [cfg.n * r // P for r in range(P + 1)]
            cb = bdist.cost_bounds(costs, P)
            per_e = np.array([costs[even[r]:even[r + 1]].sum() for r in range(P)])
            per_c = np.array([costs[cb[r]:cb[r + 1]].sum() for r in range(P)])
            balance[f"P{P}"] = {"even_max_over_mean": float(per_e.max() / per_e.mean()),
                                "cost_split_max_over_mean": float(per_c.max() / per_c.mean())}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = run_oracle_sample(cfg, m, p, v, args.cpu_samples, 1, 0)
        cpu = {"value": r["interactions_per_s"], "unit": UNIT, "cores": r["cores"], "kind": "oracle",
               "sample": (f"fp64 oracle: full tree build of N={cfg.n} ({r['t_build_s']:.1f} s) + walk of "
                          f"{r['samples']} random targets; whole-step rate extrapolated per particle"),
               "walk_interactions_per_s": r["walk_interactions_per_s"]}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": dict(workload_config(cfg, m, p, v), parallelism=f"morton-range x{world}",
                           multipole=args.multipole,
                           walk_group=args.walk_group,
                           walk_kernel=walk_kernel_name(cfg, args.walk_group, args.multipole)),
            "particles_per_s": particles_per_s,
            "interactions_per_step": inter / args.steps,
            "fp32_peak_frac": achieved_tf / peak,
            "roofline": {"bound": "alu", "kernel": "K6+K7 walk phase: k_walk + k_walk_resume", "achieved": achieved_tf,
                         "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved_tf / peak, "traffic": traffic,
                         "traffic_source": traffic_src,
                         "peak_source": f"derived: 2 flop x 128 FP32 lanes x {sms} SMs x {sm_max:.0f} MHz "
                                        "(sm_max_mhz of MEASURED_PEAKS.json; B200_PROFILING.md)",
                         "flops_per_launch": flops_walk_launch, "launch_ms": walk_ms,
                         "flop_model": (f"{fpi} per interaction" + (" (18 monopole + 38 quadrupole, evaluated for "
                                                                     "every interaction)" if args.multipole == 2 else "")
                                        + " + 8 per opened node (opens/interaction ratio from an untimed stats walk "
                                          "on the final state)")},
            "hbm_stages": {"keys_sort_GBps": sort_gbs,
                           "keys_sort_bytes_model": ("near-sorted path: 88 B/particle + the out-of-order keys' passes"
                                                     if near else "K1 32 B + 8 passes x 24 B per particle"),
                           "hbm_peak_GBps": peaks.get("hbm_gbs")},
            "phase_ms_per_step": phase_ms,
            "mac_fallbacks_last_step": st1["mac_fallbacks"],
            "tree_records": st1["n_records"],
            "gpu_launches": int(launches),
            "ms_per_step_profiled_phases": sum(phase_ms.values()),
            "clocks": clocks,
            "nccl": nccl_info,
            "exchange": exchange_kind,
            "ownership_balance": balance,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(out), flush=True)
    if exchange_kind == "fused_peer_stores":
        bh.sync()
        dist.barrier()  # no rank unmaps a replica another may still write
        bh.set_peers(None)
    bh.close()
    if comm is not None:
        bhmod.nccl_comm_destroy(comm)
    if world > 1:
        dist.destroy_process_group()
    return 0


def spawn_command(argv, gpus: int, port: int):
    """The torchrun command that re-launches this script with one rank per GPU
    (--gpus N without a torchrun environment): same arguments, 127.0.0.1
    rendezvous."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def _free_port() -> int:
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def maybe_spawn(args, argv) -> int | None:
    """--gpus N > 1 outside torchrun: re-exec under torch.distributed.run (one
    process per GPU) and return its exit code; None when already a rank (or N = 1)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    if args.impl == "ours":
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"--gpus {args.gpus}: only {have} CUDA device(s) visible", file=sys.stderr)
            return 2
    cmd = spawn_command(argv, args.gpus, _free_port())
    print("spawning: " + " ".join(cmd), file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg4", choices=sorted(bhgen.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--walk-group", type=int, default=0)
    ap.add_argument("--multipole", type=int, default=1, choices=[1, 2],
                    help="2: cells carry quadrupoles (SURVEY.md §8(f) NEXT-3); 1: the paper's monopole (default)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-rebalance", action="store_true", help="N > 1: keep the even Morton-range split")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "fused"],
                    help="N > 1: K8 as a grouped ncclBroadcast after the walk, or fused into the walk's "
                         "epilogue (peer stores into every replica, bh_set_peers)")
    ap.add_argument("--rebalance-every", type=int, default=0,
                    help="N > 1: also re-split ownership by cost every K timed steps (0: once, after warm-up)")
    ap.add_argument("--cpu-samples", type=int, default=20000)
    ap.add_argument("--ref-samples", type=int, default=8192)
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "ours":
        print("note: warm-up < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    rc = maybe_spawn(args, argv)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return reference_arm(args)
    return ours_arm(args)


if __name__ == "__main__":
    sys.exit(main())
