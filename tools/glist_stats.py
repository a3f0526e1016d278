"""Group-list statistics (walk_group 71, experiment): per group size GT, the
entries of the group's interaction list (U: accepted for sure by every target,
M: mixed), phase-1 visits and the |L| histogram, against the interactions of
the production walk.

    python tools/glist_stats.py [--config cfg4] [--gts 16,32,64,128]
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
    ap.add_argument("--gts", default="16,32,64,128")
    a = ap.parse_args()
    import torch
    from paper_1109_5190_b200 import BarnesHut

    cfg = bhgen.CONFIGS[a.config]
    m, p, v = bhgen.generate(cfg)
    prm = bhgen.params(cfg)
    n = int(m.shape[0])
    out = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    bh = BarnesHut(m, p, v, walk_group=0, **prm)
    bh.build_tree()
    bh.set_profiling(True)
    for _ in range(2):
        bh.compute_forces(out)
    ms = bh.get_profile()["ms"]["walk"] / 2
    inter = bh.get_stats()["interactions"]
    bh.close()
    print(json.dumps({"config": a.config, "n": n, "walk_ms": ms, "interactions": inter}), flush=True)
    for gt in [int(x) for x in a.gts.split(",")]:
        os.environ["BH_GLIST_GT"] = str(gt)
        bh = BarnesHut(m, p, v, walk_group=71, **prm)
        bh.build_tree()
        bh.set_profiling(True)
        bh.compute_forces(out)
        ms1 = bh.get_profile()["ms"]["walk"]
        it, _, _ = bh.get_walk_level_stats()
        bh.close()
        L, U, V, G = (int(x) for x in it[:4])
        print(json.dumps({"gt": gt, "groups": G, "list": L, "u_frac": U / max(L, 1), "visits": V,
                          "list_per_group": L / max(G, 1), "target_entries_per_inter": gt * L / max(inter, 1),
                          "phase1_ms": ms1, "hist_log2": [int(x) for x in it[4:24]]}), flush=True)


if __name__ == "__main__":
    main()
