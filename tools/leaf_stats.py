"""Walk statistics: the share of record loads that are particle (leaf) records.

    python tools/leaf_stats.py cfg4 cfg5 ...
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bhgen  # noqa: E402
from paper_1109_5190_b200 import BarnesHut  # noqa: E402
for c in sys.argv[1:]:
    m, p, v = bhgen.generate(c); prm = bhgen.params(c)
    bh = BarnesHut(m, p, v, **prm); bh.build_tree(); bh.set_walk_stats(True); bh.compute_forces(); st = bh.get_stats()
    print(json.dumps({"cfg": c, "record_visits": st["record_visits"], "leaf_visits": st["leaf_visits"], "leaf_frac": st["leaf_visits"] / max(1, st["record_visits"]), "interactions": st["interactions"], "opens": st["opens"]}), flush=True)
    bh.close()
