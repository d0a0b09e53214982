#!/usr/bin/env bash
# Collect the ncu evidence committed under profiles/ (run ON the GPU box, 1 GPU):
#   1. launch list of the bench command (device time per launch, cold-cache, serialised)
#   2. one `ncu --set full` capture of the routing kernel (DeepSeek-V3 shape)
#   3. one `ncu --set full` capture of the K3 grouped GEMM (gate_up projection)
# Then, in the build container: python tools/summarize_profiles.py <round>
set -euo pipefail
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
NCU="ncu --clock-control none"

# 1. launch list (first 400 launches of a short bench run; the pool graphs are big)
$NCU --metrics gpu__time_duration.sum -c 400 --csv --log-file "$OUT/launches.csv" \
    python bench.py --steps 256 --warmup 3 --e2e-steps 20 --cpu-seconds 0.2 --no-moe > "$OUT/launches_bench.log" 2>&1 || true

# 2. full capture of the routing kernel (skip warm-up launches)
$NCU --set full --import-source on -k regex:metro_ids_kernel -s 5 -c 1 -o "$OUT/metro_full" \
    python tools/profile_target.py metro > "$OUT/metro_full.log" 2>&1 || true

# 3. full capture of K3 (first grouped GEMM launch = gate_up of the METRO rank)
$NCU --set full --import-source on -k regex:moe_gemm -c 1 -o "$OUT/moe_full" \
    python tools/moe_layer_bench.py --batches 1 --reps 1 > "$OUT/moe_full.log" 2>&1 || true
ls -la "$OUT"
