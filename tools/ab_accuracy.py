"""A/B of walk builds and variants on one config: walk device time and the
max / p99 per-particle relative acceleration error against the fp64 oracle over
ALL targets (oracle forces computed once and cached in /tmp).

    python tools/ab_accuracy.py cfg4 [lib.so[:walk_group][:ENV=VAL] ...]      (ABA_NO_ORACLE=1: times only)

Each entry runs in its own process (BH_LIB selects the library build); one
JSON line per entry.
"""
import json
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import bhgen  # noqa: E402

CODE = r'''
import os, sys, json, numpy as np, torch
from paper_1109_5190_b200 import BarnesHut
d = np.load("/tmp/aba_in.npz")
o = np.load(sys.argv[3]) if sys.argv[3] != "-" else None
prm = json.loads(sys.argv[1])
bh = BarnesHut(d["m"], d["p"], d["v"], walk_group=int(sys.argv[2]), **prm)
bh.build_tree()
acc = bh.compute_forces()
cnt, _ = bh.get_interactions()
st = bh.get_stats()
out = torch.empty((d["m"].shape[0], 3), dtype=torch.float32, device="cuda")
bh.set_profiling(True)
for _ in range(3): bh.compute_forces(out)
pr = bh.get_profile()
out = {"walk_ms": round(pr["ms"]["walk"] / 3, 3), "interactions": int(st["interactions"]), "redo": int(st["redo_targets"])}
if o is not None:
    ref = o["acc"]
    err = np.linalg.norm(acc.astype(np.float64) - ref, axis=1) / np.linalg.norm(ref, axis=1)
    out.update({"max_rel": float(err.max()), "p99_rel": float(np.quantile(err, 0.99)),
                "median_rel": float(np.median(err)), "argmax": int(err.argmax()),
                "counts_equal": bool(np.array_equal(cnt.astype(np.int64), o["cnt"]))})
print(json.dumps(out))
'''


def main():
    cfg = sys.argv[1]
    m, p, v = bhgen.generate(cfg)
    np.savez("/tmp/aba_in.npz", m=m, p=p, v=v)
    prm = bhgen.params(cfg)
    cache = "-" if os.environ.get("ABA_NO_ORACLE") else f"/tmp/aba_oracle_{cfg}.npz"
    if cache != "-" and not os.path.exists(cache):
        import oracle

        t0 = time.time()
        o = oracle.Oracle(m, p.astype(np.float64), v.astype(np.float64), **prm).build()
        acc, cnt = o.forces()
        o.close()
        np.savez(cache, acc=acc, cnt=cnt)
        print(json.dumps({"oracle_s": time.time() - t0}), flush=True)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for spec in sys.argv[2:]:
        lib, _, rest = spec.partition(":")
        grp, _, kv = rest.partition(":")
        env = dict(os.environ, BH_LIB=os.path.abspath(lib), PYTHONPATH=root)
        if kv:
            k, _, val = kv.partition("=")
            env[k] = val
        r = subprocess.run([sys.executable, "-c", CODE, json.dumps(prm), grp or "0", cache], env=env,
                           capture_output=True, text=True)
        print(json.dumps({"cfg": cfg, "lib": os.path.basename(lib), "walk_group": int(grp or 0), "env": kv}),
              r.stdout.strip() or r.stderr[-600:], flush=True)


if __name__ == "__main__":
    main()
