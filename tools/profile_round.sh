#!/bin/bash
# One gpurun call: full bench line, launch list and ncu --set full captures of
# the step's kernels (each command runs plain first; ncu only after it exits 0).
#   /usr/local/graft/bin/gpurun --timeout 1500 -- 'bash tools/profile_round.sh r1b cfg4'
set -u
R=${1:-r1}; CFG=${2:-cfg4}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/${R}_smi.txt 2>&1
python bench.py --config $CFG > $O/${R}_bench_${CFG}.json 2> $O/${R}_bench_${CFG}.err
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > $O/${R}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${R}_launches.csv $CMD > /dev/null 2>&1
for spec in "walk:^k_walk$:1" "resume:k_walk_resume:1" "moments:k_moments_level:33" "emit:k_emit:1" "keys_prev:k_keys_prev:1" "merge:k_near_merge:1" "split:k_near_split:1"; do
  IFS=: read key kern skip <<< "$spec"
  ncu --set full --clock-control none --import-source on -k "regex:$kern" -s $skip -c 1 -o $O/${R}_prof_$key $CMD > $O/${R}_ncu_$key.log 2>&1
done
ls $O
