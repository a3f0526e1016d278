"""Max / p99 per-particle relative acceleration error of the GPU walk vs the
fp64 oracle (step 0) for the BASELINE configs; cfg4/cfg5 on sampled targets.

    python tools/accuracy.py [--configs cfg1,cfg2,cfg3,cfg4] [--samples 4096]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bhgen  # noqa: E402
import oracle  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="cfg1,cfg2,cfg3,cfg4")
    ap.add_argument("--samples", type=int, default=4096)
    a = ap.parse_args()
    from paper_1109_5190_b200 import BarnesHut

    for name in a.configs.split(","):
        cfg = bhgen.CONFIGS[name]
        m, p, v = bhgen.generate(cfg)
        prm = bhgen.params(cfg)
        t0 = time.time()
        bh = BarnesHut(m, p, v, **prm)
        bh.build_tree()
        acc = bh.compute_forces()
        cnt, _ = bh.get_interactions()
        o = oracle.Oracle(m, p.astype(np.float64), v.astype(np.float64), **prm).build()
        n = m.shape[0]
        tg = None if n <= (1 << 20) else np.sort(np.random.default_rng(3).choice(n, a.samples, replace=False))
        oacc, ocnt = o.forces(tg)
        g = acc if tg is None else acc[tg]
        gc = cnt if tg is None else cnt[tg]
        err = np.linalg.norm(g - oacc, axis=1) / np.linalg.norm(oacc, axis=1)
        print(json.dumps({"config": name, "n": n, "targets": int(len(err)), "max_rel": float(err.max()),
                          "p99_rel": float(np.quantile(err, 0.99)), "median_rel": float(np.median(err)),
                          "counts_equal": bool(np.array_equal(gc.astype(np.int64), ocnt)),
                          "lib": os.environ.get("BH_LIB", "default"), "secs": time.time() - t0}), flush=True)
        bh.close()
        o.close()


if __name__ == "__main__":
    main()
