# Alternating per-mode timing of two library builds in separate processes
# (developer tool):  bash tools/exp_lib_ab.sh <libA> <libB> <configs> [rounds]
A=$1; B=$2; CFG=$3; R=${4:-3}
for i in $(seq 1 $R); do
  DMTK_GPU_LIB=$A python tools/perf_modes.py --config $CFG --reps ${REPS:-10} > gpurun_out/ab_A_$i.log 2>&1
  DMTK_GPU_LIB=$B python tools/perf_modes.py --config $CFG --reps ${REPS:-10} > gpurun_out/ab_B_$i.log 2>&1
done
python - "$R" <<'PY'
import json, collections, sys
R = int(sys.argv[1])
res = {}
for tag in "AB":
    acc = collections.defaultdict(list)
    for i in range(1, R + 1):
        for l in open(f"gpurun_out/ab_{tag}_{i}.log"):
            if l.startswith("{"):
                d = json.loads(l); acc[(d["config"], d["mode"])].append(d["ms"])
    res[tag] = {k: sorted(v)[len(v) // 2] for k, v in acc.items()}
for k in sorted(res["A"]):
    a, b = res["A"][k], res["B"].get(k)
    print(k, "A", a, "B", b, "B speed-up %", round(100 * (a / b - 1), 2) if b else None)
PY
