set -u
for w in "--workload c2" "--workload c3" "--workload c5 --steps 3"; do
  tag=$(echo $w | awk '{print $2}')
  bash tools/ab_bench.sh ab1_$tag "$w" default launder imad4 imad5 imad6 > gpurun_out/ab1_$tag.txt 2>&1
done
