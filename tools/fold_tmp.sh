python -m pytest tests -m gpu -x -q -k "containment_fold or invariance or cfg3 or cfg5 or resume" > gpurun_out/pytest_gpu24.log 2>&1; tail -2 gpurun_out/pytest_gpu24.log
for c in cfg3 cfg5; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b24_$c.json 2> gpurun_out/b24_$c.err; python -c "
import json; d=json.loads(open(\"gpurun_out/b24_$c.json\").read().strip().splitlines()[-1]); print(\"$c\", d[\"value\"], d[\"ms_per_step\"], d[\"roofline\"][\"frac\"], {k: round(v,3) for k,v in d[\"phase_ms_per_step\"].items()})"; done
