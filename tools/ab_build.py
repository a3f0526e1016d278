import os, sys, json
sys.path.insert(0, os.getcwd())
import bhgen
cfg = sys.argv[1]
m, p, v = bhgen.generate(cfg)
prm = bhgen.params(cfg)
import subprocess
libs = sys.argv[2:]
code = r'''
import os, sys, json, numpy as np
sys.path.insert(0, os.getcwd())
import bhgen
from paper_1109_5190_b200 import BarnesHut
d = np.load("/tmp/ab_in.npz")
prm = json.loads(sys.argv[1])
bh = BarnesHut(d["m"], d["p"], d["v"], **prm)
bh.build_tree(); bh.sync()
bh.set_profiling(True)
for _ in range(5): bh.build_tree()
pr = bh.get_profile()
print(json.dumps({k: round(x / 5, 4) for k, x in pr["ms"].items()}))
'''
import numpy as np
np.savez("/tmp/ab_in.npz", m=m, p=p, v=v)
for lib in libs:
    env = dict(os.environ, BH_LIB=os.path.abspath(lib))
    r = subprocess.run([sys.executable, "-c", code, json.dumps(prm)], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), r.stdout.strip() or r.stderr[-500:], flush=True)
