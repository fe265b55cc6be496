set -u
for w in "--workload c2" "--workload c3"; do
  tag=$(echo $w | awk '{print $2}')
  bash tools/ab_bench.sh ab5_$tag "$w" default lc launder > gpurun_out/ab5_$tag.txt 2>&1
done
