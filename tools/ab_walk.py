"""A/B of walk-kernel builds: walk device time (ms) per library (BH_LIB), same input.

    python tools/ab_walk.py cfg4 lib/libbh.so lib/libbh_x.so ...
"""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import bhgen  # noqa: E402

CODE = r'''
import os, sys, json, numpy as np, torch
from paper_1109_5190_b200 import BarnesHut
d = np.load("/tmp/ab_in.npz")
prm = json.loads(sys.argv[1])
bh = BarnesHut(d["m"], d["p"], d["v"], **prm)
bh.build_tree()
out = torch.empty((d["m"].shape[0], 3), dtype=torch.float32, device="cuda")
bh.compute_forces(out); bh.sync()
bh.set_profiling(True)
for _ in range(3): bh.compute_forces(out)
pr = bh.get_profile()
st = bh.get_stats()
print(json.dumps({"walk_ms": round(pr["ms"]["walk"] / 3, 3), "interactions": st["interactions"], "redo": st["redo_targets"]}))
'''


def main():
    cfg = sys.argv[1]
    m, p, v = bhgen.generate(cfg)
    np.savez("/tmp/ab_in.npz", m=m, p=p, v=v)
    prm = dict(bhgen.params(cfg), **json.loads(os.environ.get("AB_PRM", "{}")))  # e.g. AB_PRM='{"walk_group": 70}'
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for rep in range(2):
        for lib in sys.argv[2:]:
            env = dict(os.environ, BH_LIB=os.path.abspath(lib), PYTHONPATH=root)
            r = subprocess.run([sys.executable, "-c", CODE, json.dumps(prm)], env=env, capture_output=True, text=True)
            print(rep, os.path.basename(lib), r.stdout.strip() or r.stderr[-400:], flush=True)


if __name__ == "__main__":
    main()
