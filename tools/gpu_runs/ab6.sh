set -u
for w in "--workload c2" "--workload c3" "--workload c5 --steps 3"; do
  tag=$(echo $w | awk '{print $2}')
  bash tools/ab_bench.sh ab6_$tag "$w" default kst3 vst3 g1d500 g1d1500 > gpurun_out/ab6_$tag.txt 2>&1
done
