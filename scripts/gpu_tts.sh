#!/bin/bash
# time to solution per outer step (the paper's claim):
# PTL-RKL2, PTL-RKG2, BE+PCG (Jacobi, r-line) with and without PTL, on the C3
# and C4 grids (same seeded inputs, same outer step 1e4 dt_E) -> gpurun_out/tts_*.json
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="--no-e2e --no-cpu-baseline --steps 1 --warmup 1"
for cfg in ${CFGS:-c3 c4}; do
  for v in "rkl2" "rkg2" "be" "be --pc line-r" "be --no-ptl" "rkg2 --no-ptl"; do
    tag=$(echo "$cfg $v" | tr ' -' '__')
    timeout 1200 python bench.py --config $cfg --scheme $v $B > gpurun_out/tts_$tag.json 2> gpurun_out/tts_$tag.err
    echo "$cfg $v rc=$?"
  done
done
python - <<'PY'
import glob, json
rows = []
for f in sorted(glob.glob("gpurun_out/tts_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    ops = d["config"]["operators"][0]
    rows.append({"config": d["config"]["config"], "scheme": d["config"]["scheme"], "ms_per_step": d["ms_per_step"],
                 "cycles": ops["cycles"], "stages_or_iters": ops["stages_or_iters"], "cell_updates_per_s": d["value"]})
for r in rows: print(r)
json.dump(rows, open("gpurun_out/tts_summary.json", "w"), indent=1)
PY
