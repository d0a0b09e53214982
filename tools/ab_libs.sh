#!/usr/bin/env bash
# A/B/C... the routing kernel of several library builds (abtest/lib<X>.so, see
# tools/ab_build.sh): parity spot check per build, then per-phase cycles +
# graph-replayed µs, interleaved over two rounds.  Run on the GPU box:
#   bash tools/ab_libs.sh "A T"
set -u
libs=${1:-"A B"}
for v in $libs; do
  METRO_B200_LIB=$PWD/abtest/lib$v.so timeout 300 python -m pytest -q -x tests/test_parity_gpu.py \
      -m gpu -k "golden or fuzz or max or baseline or fallback" 2>&1 | tail -1 | sed "s/^/$v parity: /"
done
for round in 1 2; do
  for v in $libs; do
    METRO_B200_LIB=$PWD/abtest/lib$v.so PROFILE_CLUSTERS=${PROFILE_CLUSTERS:-1} timeout 300 \
        python tools/phase_profile.py > gpurun_out/ab_$v$round.log 2>&1
    python - "$v$round" <<'PY'
import json, sys
d = json.load(open("gpurun_out/phase_profile.json"))
for k, v in d.items():
    if isinstance(v, dict):
        c = v["cycles"]
        print(sys.argv[1], k, "%.3f us pool %.3f warm" % (v["us_pool"], v["us_l2warm"]), c["total"],
              {p: c[p] for p in ("stage", "histogram", "exchange", "classify", "sort", "greedy", "outputs")})
PY
  done
done
