#!/usr/bin/env bash
# A/B the routing kernel of two library builds (abtest/libA.so, abtest/libB.so):
# per-phase cycles + graph-replayed µs, interleaved A B A B.  Run on the GPU box.
set -u
for round in 1 2; do
  for v in A B; do
    METRO_B200_LIB=$PWD/abtest/lib$v.so PROFILE_CLUSTERS=1 timeout 300 python tools/phase_profile.py > gpurun_out/ab_$v$round.log 2>&1
    python - "$v$round" <<'PY'
import json, sys
d = json.load(open("gpurun_out/phase_profile.json"))
for k, v in d.items():
    if isinstance(v, dict):
        c = v["cycles"]
        print(sys.argv[1], k, "%.3f us" % v["us_pool"], c["total"], {p: c[p] for p in ("stage", "histogram", "exchange", "classify", "sort", "greedy", "outputs")})
PY
  done
done
