# Round profile set (developer recipe): bench JSON, launch list of the bench's
# timed kernels, and one ncu --set full capture per headline mode kernel.
#   bash tools/prof_bench.sh <tag>
TAG=${1:-r02}
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench=$?
B="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-als --no-configs"
$B > gpurun_out/${TAG}_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo ncu_launch=$?
P="python tools/perf_modes.py --config 1000c25 --profile"
$P > gpurun_out/${TAG}_plain_p.log 2>&1 && ncu --set full --clock-control none --import-source on \
  --profile-from-start off -k regex:mttkrp_tc -o gpurun_out/${TAG}_ncu_1000c25 $P > gpurun_out/${TAG}_ncu_p.log 2>&1
echo ncu_full=$?
