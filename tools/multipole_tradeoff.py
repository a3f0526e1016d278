"""Accuracy against cost of the cell expansion.

    python tools/multipole_tradeoff.py [--config cfg2] [--n 0] [--targets 2000]

For theta in {0.3, 0.5, 0.7, 0.9} and multipole in {1, 2}: the median and p99
relative acceleration error against the exact softened direct sum (oracle,
sampled targets), the interactions per particle and the walk time on the GPU.
One JSON line per point.
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bhgen  # noqa: E402
import oracle  # noqa: E402  (the exact reference: test-side code, as in tests/)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--targets", type=int, default=2000)
    a = ap.parse_args()
    from paper_1109_5190_b200 import BarnesHut

    cfg = bhgen.CONFIGS[a.config]
    m, p, v = bhgen.generate(cfg, n=a.n or None)
    prm = bhgen.params(cfg)
    n = m.shape[0]
    rng = np.random.default_rng(1)
    tg = np.sort(rng.choice(n, min(a.targets, n), replace=False))
    ref = oracle.direct(m, p.astype(np.float64), prm["eps"], prm["G"], targets=tg)
    for theta in (0.3, 0.5, 0.7, 0.9):
        for mp in (1, 2):
            kw = dict(prm, theta=theta)
            bh = BarnesHut(m, p, v, multipole=mp, **kw)
            bh.build_tree()
            acc = bh.compute_forces()
            cnt, total = bh.get_interactions()
            bh.set_profiling(True)
            for _ in range(3):
                bh.build_tree()
                bh.compute_forces()
            ms = bh.get_profile()["ms"]["walk"] / 3
            err = np.linalg.norm(acc[tg] - ref, axis=1) / np.linalg.norm(ref, axis=1)
            print(json.dumps({"config": a.config, "n": n, "theta": theta, "multipole": mp,
                              "err_median": float(np.median(err)), "err_p99": float(np.percentile(err, 99)),
                              "interactions_per_particle": total / n, "walk_ms": ms}), flush=True)
            bh.close()


if __name__ == "__main__":
    main()
