"""Per-rank critical path of the multi-GPU step, emulated on one GPU
(DESIGN.md §8): rank r of P as its own context (world = P,
rank = r, no NCCL communicator), timed phase by phase with CUDA events over
steps that run exactly what a rank runs (the full build -- every rank repeats
it -- and the walk + leapfrog of the P = 1 groups holding its particles); the
exchange is modelled from its bytes ((P-1)/P x 16 B x N received per GPU at
the measured 770 GB/s peer bandwidth of B200_PROFILING.md).  Strong-scaling
efficiency = T1 / (P x max over ranks of the rank's step).

    python tools/rank_emulation.py [--config cfg5] [--ranks 2,4,8] [--steps 3] [--fused]

--fused: the fused exchange (bh_set_peers, NEXT-1): all P ranks' contexts live
at once with each other's pos4 as peers; every step is all ranks' build
(bh_step_phase 0), then all ranks' walk, whose epilogue stores each new own
position into all P replicas (here HBM stores on the one GPU; on NVLink 16 B x
own_n x (P-1) per rank during the walk).  The exchange model is then the two
barriers of a step (BARRIER_US each) instead of the broadcast's bytes.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bhgen  # noqa: E402

NVLINK_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md)
BARRIER_US = 15.0  # a one-word NCCL all-reduce over NVLink (latency-bound; assumed, not measured here)


def phases(bh, steps):
    bh.set_profiling(True)
    for _ in range(steps):
        bh.step(1)
    bh.sync()
    pr = bh.get_profile()
    bh.set_profiling(False)
    return {k: v / steps for k, v in pr["ms"].items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--ranks", default="2,4,8")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--fused", action="store_true")
    ap.add_argument("--rebalance", action="store_true", help="--fused: equal-cost ownership after the warm-up")
    ap.add_argument("--cost", default="trips", choices=["trips", "interactions", "time"],
                    help="--rebalance: per-particle cost (dist.rebalance's; trips = the group's walk loop trips; "
                         "time = trips rescaled per rank to its measured walk time, --rounds times)")
    ap.add_argument("--rounds", type=int, default=2, help="--cost time: feedback rounds")
    a = ap.parse_args()
    from paper_1109_5190_b200 import BarnesHut

    cfg = bhgen.CONFIGS[a.config]
    m, p, v = bhgen.generate(cfg)
    prm = bhgen.params(cfg)
    one = BarnesHut(m, p, v, **prm)
    one.step(a.warmup)
    one.sync()
    ph1 = phases(one, a.steps)
    one.close()
    t1 = sum(ph1.values())
    print(json.dumps({"config": cfg.name, "P": 1, "phases_ms": ph1, "step_ms": t1}), flush=True)
    for P in [int(x) for x in a.ranks.split(",")]:
        if a.fused:
            fused_row(BarnesHut, m, p, v, prm, P, a, cfg, t1)
            continue
        worst, per = 0.0, []
        for r in range(P):
            bh = BarnesHut(m, p, v, rank=r, world=P, nccl_comm=None, **prm)
            bh.step(a.warmup)
            bh.sync()
            ph = phases(bh, a.steps)
            bh.close()
            t = sum(ph.values())
            per.append({"rank": r, "build_ms": ph["bbox"] + ph["keys_sort"] + ph["tree"] + ph["moments"],
                        "walk_ms": ph["walk"], "step_ms": t})
            worst = max(worst, t)
        x_ms = (P - 1) / P * 16.0 * cfg.n / (NVLINK_GBS * 1e9) * 1e3
        tp = worst + x_ms
        print(json.dumps({"config": cfg.name, "P": P, "ranks": per, "max_rank_step_ms": worst,
                          "exchange_model_ms": x_ms, "step_ms_model": tp, "efficiency_model": t1 / (P * tp)}),
              flush=True)


def fused_row(BarnesHut, m, p, v, prm, P, a, cfg, t1):
    ranks = [BarnesHut(m, p, v, rank=r, world=P, nccl_comm=None, **prm) for r in range(P)]
    ptrs = [bh.pos4_ptr() for bh in ranks]
    for bh in ranks:
        bh.set_peers(ptrs)

    def one_step():
        # one rank at a time (each rank alone on "its" GPU: the streams of the
        # contexts would otherwise overlap on the one device and share its SMs)
        for bh in ranks:
            bh.step_phase(0)
            bh.sync()
        for bh in ranks:
            bh.step_phase(1)
            bh.sync()

    for _ in range(a.warmup):
        one_step()
    balance = None
    if a.rebalance:  # dist.rebalance without the collectives: every rank's costs are here
        import numpy as np

        from paper_1109_5190_b200 import dist as bdist

        for rnd in range(a.rounds if a.cost == "time" else 1):
            walk = [None] * P
            if a.cost == "time":  # one profiled step: each rank's measured walk time
                for bh in ranks:
                    bh.set_profiling(True)
                one_step()
                for r, bh in enumerate(ranks):
                    walk[r] = bh.get_profile()["ms"]["walk"]
                    bh.set_profiling(False)
            own = [bh.get_own() for bh in ranks]
            costs = [bh.get_own_cost() for bh in ranks] if a.cost != "interactions" else [c for c, _ in own]
            costs = [bdist.time_scaled(c, walk[r]) for r, c in enumerate(costs)]
            bounds = bdist.cost_bounds(np.concatenate(costs).astype(np.float64), P)
            vels = np.concatenate([v_ for _, v_ in own])
            for r, bh in enumerate(ranks):
                bh.set_partition(bounds, vels[bounds[r]:bounds[r + 1]])
            one_step()
        balance = f"cost split after the warm-up ({a.cost})"
    for bh in ranks:
        bh.set_profiling(True)
    for _ in range(a.steps):
        one_step()
    per, worst = [], 0.0
    for r, bh in enumerate(ranks):
        ph = {k: x / a.steps for k, x in bh.get_profile()["ms"].items()}
        bh.set_profiling(False)
        t = sum(ph.values())
        per.append({"rank": r, "build_ms": ph["bbox"] + ph["keys_sort"] + ph["tree"] + ph["moments"],
                    "walk_ms": ph["walk"], "step_ms": t})
        worst = max(worst, t)
    for bh in ranks:
        bh.set_peers(None)
        bh.close()
    x_ms = 2 * BARRIER_US * 1e-3
    tp = worst + x_ms
    print(json.dumps({"config": cfg.name, "P": P, "exchange": "fused (K7 peer stores)", "ownership": balance or "even",
                      "ranks": per,
                      "max_rank_step_ms": worst, "exchange_model_ms": x_ms, "step_ms_model": tp,
                      "efficiency_model": t1 / (P * tp)}), flush=True)


if __name__ == "__main__":
    main()
