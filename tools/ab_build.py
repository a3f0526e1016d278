"""A/B of the build phases (ms per build, CUDA events per phase) across library
builds and environment switches, same input:

    python tools/ab_build.py cfg5 lib/libbh.so lib/libbh.so:BH_MOM_NO_COMPACT=1 ...

Each spec is a libbh.so path (BH_LIB) optionally followed by ':VAR=VAL,VAR=VAL'.
The positions are stepped once between builds (a real near-sorted sort).
"""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import bhgen  # noqa: E402

CODE = r'''
import os, sys, json, numpy as np
from paper_1109_5190_b200 import BarnesHut
d = np.load("/tmp/ab_in.npz")
prm = json.loads(sys.argv[1])
bh = BarnesHut(d["m"], d["p"], d["v"], **prm)
bh.step(1); bh.sync()
bh.set_profiling(True)
for _ in range(3): bh.step(1)
pr = bh.get_profile()
st = bh.get_stats()
out = {k: round(x / 3, 4) for k, x in pr["ms"].items()}
out["bad"] = st.get("sort_bad_keys")
print(json.dumps(out))
'''


def main():
    cfg = sys.argv[1]
    m, p, v = bhgen.generate(cfg)
    np.savez("/tmp/ab_in.npz", m=m, p=p, v=v)
    prm = bhgen.params(cfg)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for rep in range(2):
        for spec in sys.argv[2:]:
            lib, _, envs = spec.partition(":")
            env = dict(os.environ, BH_LIB=os.path.abspath(lib), PYTHONPATH=root)
            for kv in filter(None, envs.split(",")):
                k, _, val = kv.partition("=")
                env[k] = val
            r = subprocess.run([sys.executable, "-c", CODE, json.dumps(prm)], env=env, capture_output=True, text=True)
            print(rep, spec, r.stdout.strip() or r.stderr[-500:], flush=True)


if __name__ == "__main__":
    main()
