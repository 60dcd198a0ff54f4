timeout 900 python tools/perf_modes.py --config 1000c25,1000c50,1000c100,odd25,180c25,64c32,fmri20,200c16 --reps 10 2>&1 | grep -v "^#"
for f in "" "--tree" "--sym"; do echo "timeline $f"; timeout 300 python tools/als_timeline.py $f 2>&1 | tail -25; done
