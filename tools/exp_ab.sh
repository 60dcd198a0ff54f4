# A/B of the working tree's library against a saved build (developer tool):
#   bash tools/exp_ab.sh tools/libA.so "1000c25,fmri20" [reps]
A=$1; CFG=${2:-1000c25,fmri20}; R=${3:-5}
python tools/ab_libs.py $A paper_1708_08976_b200/libdmtk_gpu.so --config $CFG --rounds 7 --reps $R
