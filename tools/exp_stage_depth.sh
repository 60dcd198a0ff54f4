# Stage size / depth experiment with the epilogue off (DMTK_GPU_DEBUG=8): BK 16 vs 32
# at the stage counts the freed epilogue buffer allows (developer tool).
export DMTK_GPU_DEBUG=8
for i in 1 2; do
for lib in tools/libX16.so tools/libX32.so paper_1708_08976_b200/libdmtk_gpu.so; do
  echo "== $lib"; DMTK_GPU_LIB=$lib python tools/perf_modes.py --config 1000c25,fmri20 --reps 10 2>&1 | grep config
done; done
DMTK_GPU_LIB=tools/libX32.so DMTK_GPU_PLAN_LOG=1 python tools/perf_modes.py --config 1000c25 --reps 1 2>&1 | grep plan | sort -u
DMTK_GPU_LIB=tools/libX16.so DMTK_GPU_PLAN_LOG=1 python tools/perf_modes.py --config 1000c25 --reps 1 2>&1 | grep plan | sort -u
