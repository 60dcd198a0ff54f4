for i in 1 2 3; do
python tools/perf_modes.py --config 64c32,1000c25,180c25 --reps 10 > gpurun_out/e_m3_$i.log 2>&1
DMTK_GPU_NO_M3=1 python tools/perf_modes.py --config 64c32,1000c25,180c25 --reps 10 > gpurun_out/e_nom3_$i.log 2>&1
done
DMTK_GPU_PLAN_LOG=1 python tools/perf_modes.py --config 64c32 --reps 1 2>&1 | grep plan | sort -u
python - <<'PY'
import json, collections
for tag in ["m3", "nom3"]:
    acc = collections.defaultdict(list)
    for i in (1, 2, 3):
        for l in open(f"gpurun_out/e_{tag}_{i}.log"):
            if l.startswith("{"):
                d = json.loads(l); acc[(d["config"], d["mode"])].append(d["ms"])
    print(tag, {k: round(sorted(v)[1], 4) for k, v in sorted(acc.items())})
PY
