set -u
for w in "--workload c2" "--workload c3"; do
  tag=$(echo $w | awk '{print $2}')
  bash tools/ab_bench.sh ab7_$tag "$w" default poly15 poly7 > gpurun_out/ab7_$tag.txt 2>&1
done
