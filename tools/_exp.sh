export DMTK_GPU_TUNE_CACHE=/tmp/tune_final.txt
rm -f $DMTK_GPU_TUNE_CACHE
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_final.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_final.log
rm -f $DMTK_GPU_TUNE_CACHE
B="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-als"
$B > gpurun_out/plain_b.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01h.csv $B > gpurun_out/ncu_b.log 2>&1; echo ncu_launch=$?
P="python tools/perf_modes.py --config 1000c25 --profile"
$P > gpurun_out/plain_p.log 2>&1 && ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:mttkrp_tc -o gpurun_out/prof_r01h_1000c25 $P > gpurun_out/ncu_p.log 2>&1; echo ncu_full=$?
cat $DMTK_GPU_TUNE_CACHE
