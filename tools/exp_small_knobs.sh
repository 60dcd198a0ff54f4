# developer experiment batch (round 2): small-tensor and streaming-kernel knobs
P="python tools/perf_modes.py --reps 20"
run() { echo "== $*"; env "$@" $P --config 200c16 --flush 2>&1 | grep -v Warn; }
run X=0
run DMTK_GPU_FORCE_SWAP=1
run DMTK_GPU_NO_U0_SMEM=1
run DMTK_GPU_FORCE_RB=2
run DMTK_GPU_FORCE_RB=3
run DMTK_GPU_MAX_STAGES=3
run DMTK_GPU_DEBUG=8
run DMTK_GPU_DEBUG=1
run DMTK_GPU_DEBUG=9
run DMTK_GPU_NO_PDL=1
DMTK_GPU_PLAN_LOG=1 $P --config 200c16 --reps 1 2>&1 | grep plan
DMTK_GPU_PLAN_LOG=1 DMTK_GPU_FORCE_SWAP=1 $P --config 200c16 --reps 1 2>&1 | grep plan
echo "== 1000c25 decomposition"
for d in 0 1 2 8 9 11; do echo "debug $d"; DMTK_GPU_DEBUG=$d python tools/perf_modes.py --config 1000c25 --reps 10 2>&1 | grep config; done
DMTK_GPU_PLAN_LOG=1 python tools/perf_modes.py --config 1000c25 --reps 1 2>&1 | grep plan
