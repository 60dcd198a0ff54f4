export DMTK_GPU_AUTOTUNE=0
for v in "RB=4 G=1" "RB=3 G=1" "RB=2 G=1" "RB=4 G=2" "RB=2 G=2"; do set -- $v; for d in 9 0; do echo "$v debug $d"; env DMTK_GPU_FORCE_$1 DMTK_GPU_FORCE_$2 DMTK_GPU_DEBUG=$d timeout 600 python tools/perf_modes.py --config 1000x1000x1000:16,1000x1000x1000:25 --modes 0,1 --reps 10 2>&1 | grep -v "^#" | cut -c1-100; done; done
