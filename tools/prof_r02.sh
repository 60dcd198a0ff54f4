set -x
python tools/perf_modes.py --config 1000c25,200c16,fmri20 --reps 10 > gpurun_out/pm_base.log 2>&1
python tools/mode_timeline.py --config 200c16 > gpurun_out/tl200.log 2>&1
P="python tools/perf_modes.py --config 1000c25 --profile"
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:mttkrp_tc -o gpurun_out/prof_r02c_1000c25 $P > gpurun_out/ncu_p.log 2>&1; echo ncu_full=$?
P2="python tools/perf_modes.py --config 200c16 --profile"
timeout 300 ncu --set full --clock-control none --import-source on --profile-from-start off -o gpurun_out/prof_r02c_200c16 $P2 > gpurun_out/ncu_p2.log 2>&1; echo ncu_full2=$?
