#!/usr/bin/env bash
# A/B one library build under two environment settings: ./tools/ab_env.sh "METRO_PDL=0" "METRO_PDL=1"
set -u
for round in 1 2; do
  for v in "$1" "$2"; do
    env $v PROFILE_CLUSTERS=1 timeout 300 python tools/phase_profile.py > gpurun_out/ab_env.log 2>&1
    python - "$v/$round" <<'PY'
import json, sys
d = json.load(open("gpurun_out/phase_profile.json"))
for k, v in d.items():
    if isinstance(v, dict):
        c = v["cycles"]
        print(sys.argv[1], k, "%.3f us pool, %.3f us warm" % (v["us_pool"], v["us_l2warm"]), c["total"])
PY
  done
done
