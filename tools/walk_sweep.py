"""Walk-kernel sweep: device time of K6 per traversal-group size (and phase times).

    python tools/walk_sweep.py [--config cfg4] [--groups 68,67,66] [--reps 3]

Prints one JSON line per group size: walk ms (CUDA events on the ctx stream),
interactions, opens, MAC fallbacks, interactions/s and useful FP32 TFLOP/s.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bhgen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--groups", default="68,67,66")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    from paper_1109_5190_b200 import BarnesHut

    cfg = bhgen.CONFIGS[a.config]
    m, p, v = bhgen.generate(cfg, n=a.n or None)
    prm = bhgen.params(cfg)
    for g in [int(x) for x in a.groups.split(",")]:
        bh = BarnesHut(m, p, v, walk_group=g, **prm)
        bh.build_tree()
        bh.set_walk_stats(True)
        bh.compute_forces(_dev_out(bh))
        bh.sync()
        st_stats = bh.get_stats()
        bh.set_walk_stats(False)
        bh.sync()
        bh.set_profiling(True)
        for _ in range(a.reps):
            bh.compute_forces(_dev_out(bh))
        prof = bh.get_profile()
        st = bh.get_stats()
        ms = prof["ms"]["walk"] / a.reps
        fl = 18 * st["interactions"] + 8 * st_stats["opens"]
        print(json.dumps({"config": a.config, "n": int(m.shape[0]), "group": g, "walk_ms": ms,
                          "interactions": st["interactions"], "opens": st_stats["opens"], "redo": st["redo_targets"],
                          "fallbacks": st["mac_fallbacks"], "inter_per_s": st["interactions"] / ms * 1e3,
                          "tflops": fl / ms / 1e9}), flush=True)
        bh.close()


_outs = {}


def _dev_out(bh):
    import torch

    k = bh.n
    if k not in _outs:
        _outs[k] = torch.empty((k, 3), dtype=torch.float32, device="cuda")
    return _outs[k]


if __name__ == "__main__":
    main()
