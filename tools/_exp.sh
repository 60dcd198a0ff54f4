export DMTK_GPU_TUNE_CACHE=gpurun_out/tune_cache.txt
rm -f $DMTK_GPU_TUNE_CACHE
timeout 600 python -m pytest tests/test_gpu_tiles.py -x -q -k "tune_cache or measured or one_output" 2>&1 | tail -1
B="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-als"
$B > gpurun_out/plain_b.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01g.csv $B > gpurun_out/ncu_b.log 2>&1
cat $DMTK_GPU_TUNE_CACHE
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,temperature.gpu,temperature.memory,clocks_event_reasons.active --format=csv -lms 50 > gpurun_out/smi_sustained.csv &
SMI=$!
for r in 10 100 400; do timeout 300 python tools/perf_modes.py --config 1000c25 --modes 0 --reps $r 2>&1 | grep -v "^#"; done
kill $SMI
