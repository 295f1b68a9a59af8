#!/bin/bash
# A/B of SpMM environment knobs on one workload: tools/gpu_env_ab.sh CONFIG "ENV1" "ENV2" ...
# (each ENV a space-separated list of VAR=value, "-" for the defaults); device-timed bench lines.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
cfg=$1; shift
i=0
for e in "$@"; do
  i=$((i+1))
  [ "$e" = "-" ] && e=""
  env $e timeout 900 python bench.py --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-probe --secondary none \
    > gpurun_out/envab_${cfg}_$i.json 2> gpurun_out/envab_${cfg}_$i.err
  python - "$cfg" "$i" "$e" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/envab_{sys.argv[1]}_{sys.argv[2]}.json"))
print(sys.argv[1], repr(sys.argv[3]), round(d["value"], 3), "median", round(d["epoch_ms"]["median"], 3),
      {k: round(v["ms_per_epoch"], 3) for k, v in d["kernels"].items()})
PY
done
