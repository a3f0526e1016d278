# Build-phase profile (cfg4): launch list + ncu --set full of k_emit and two k_moments_level levels.
#   /usr/local/graft/bin/gpurun --timeout 1500 -- "bash tools/profile_build.sh"
set -u
O=gpurun_out
CMD="python bench.py --config cfg4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > $O/pb_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/pb_launches.csv $CMD > /dev/null 2>&1
for spec in "emit:k_emit:1" "m10:k_moments_level:33" "m3:k_moments_level:40" "lcp:k_lcp_count:1" "lscan:k_level_scan:1"; do
  IFS=: read key kern skip <<< "$spec"
  ncu --set full --clock-control none --import-source on -k regex:$kern -s $skip -c 1 -o $O/pb_prof_$key $CMD > $O/pb_ncu_$key.log 2>&1
done
ls $O | grep pb_
