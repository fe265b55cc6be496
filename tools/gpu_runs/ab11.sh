set -u
for w in "--workload c2" "--workload c3"; do
  tag=$(echo $w | awk '{print $2}')
  bash tools/ab_bench.sh ab11_$tag "$w" default cs32 cs200 cs500 > gpurun_out/ab11_$tag.txt 2>&1
done
