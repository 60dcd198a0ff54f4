for env in "DMTK_GPU_MAX_STAGES=2" "DMTK_GPU_MAX_STAGES=2 DMTK_GPU_FORCE_G=2" "DMTK_GPU_MAX_STAGES=3"; do
  env $env DMTK_GPU_PLAN_LOG=1 timeout 60 python tools/dbg_bk.py 1000x100x50 16 0 > /tmp/o.log 2>&1; echo "$env rc=$? $(grep -o '"err".*' /tmp/o.log) $(grep -o 'Error:.*' /tmp/o.log | head -1 | cut -c1-60) $(grep -o 'G [0-9] TR [0-9]* BI [0-9]* BJ [0-9]* stages [0-9]' /tmp/o.log | head -1)"
done
