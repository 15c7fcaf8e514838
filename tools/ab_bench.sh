#!/bin/bash
# A/B of two builds on one GPU box: the repo (N) and the worktree _ab_head (H), alternating, factor-kernel times.
# Usage (via gpurun): bash tools/ab_bench.sh TAG [reps]
TAG=${1:-ab}; REPS=${2:-3}
O=gpurun_out; mkdir -p $O
for i in $(seq $REPS); do
  for pc in C D; do
    timeout 200 python bench.py --precond $pc --no-cpu-baseline --no-config5 --steps 5 > $O/${TAG}_N_${pc}$i.json 2>/dev/null
    (cd _ab_head && timeout 200 python bench.py --precond $pc --no-cpu-baseline --no-config5 --steps 5 > ../$O/${TAG}_H_${pc}$i.json 2>/dev/null)
  done
done
python - "$TAG" "$REPS" <<'PY' > $O/${TAG}_summary.txt
import json, sys
tag, reps = sys.argv[1], int(sys.argv[2])
for pc in "CD":
    for v in "NH":
        xs = []
        for i in range(1, reps + 1):
            try:
                d = json.load(open(f"gpurun_out/{tag}_{v}_{pc}{i}.json"))
                xs.append((d["ms_per_step"], d["breakdown"]["t_factor_kernel"] * 1e3))
            except Exception as e:
                xs.append((float("nan"), float("nan")))
        print(pc, v, "ms/step", [round(a, 3) for a, _ in xs], "factor kernel ms", [round(b, 3) for _, b in xs])
PY
cat $O/${TAG}_summary.txt
