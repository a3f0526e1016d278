#!/usr/bin/env bash
# One GPU-box check of the tree at hand (run under gpurun from the repo root):
#   tools/gpu_check.sh TAG [pytest -k expression] [bench config]
# -> gpurun_out/TAG_pytest.log (pytest -m gpu), gpurun_out/TAG_bench.json / .err
# (one bench.py line; skipped when the config is "-").
TAG=${1:?tag}
KEXPR=${2:-}
CFG=${3:-cfg4}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -c "import os; print('host cores', len(os.sched_getaffinity(0)))"
python -m paper_1109_5190_b200.build > /dev/null
if [ "$KEXPR" != "-" ]; then
  timeout 2400 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider ${KEXPR:+-k "$KEXPR"} \
    > gpurun_out/${TAG}_pytest.log 2>&1
  echo "pytest rc=$?" | tee -a gpurun_out/${TAG}_pytest.log
  grep -E "passed|failed|error" gpurun_out/${TAG}_pytest.log | tail -3
fi
if [ "$CFG" != "-" ]; then
  timeout 900 python bench.py --config "$CFG" --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.json \
    2> gpurun_out/${TAG}_bench.err
  echo "bench rc=$?"
  tail -c 400 gpurun_out/${TAG}_bench.json
fi
