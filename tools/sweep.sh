#!/usr/bin/env bash
# Every BASELINE configuration through bench.py (N = 1): µs per layer, e2e, λ METRO vs
# EPLB, CPU port.  One JSON line per config into $1 (run on the GPU box).
OUT=${1:-gpurun_out/sweep.jsonl}
: > "$OUT"
for c in q30 ds ds_b64 ds_b128 ds_b256 ds_b512 ds_b2048 ds_b4096 ds_b8192 ds_b64_skew0.5 ds_b1024_skew0.5 ds_b8192_skew0.5 ds_b64_skew2.0 ds_b1024_skew2.0 ds_b8192_skew2.0 q235_125 q235_150 q235_200; do
  timeout 300 python bench.py --config $c --steps 2000 --warmup 5 --e2e-steps 300 --cpu-seconds 2 --no-moe \
      2> /dev/null | tail -1 >> "$OUT"
done
