#!/usr/bin/env bash
# Collect the ncu evidence committed under profiles/ (run ON the GPU box, 1 GPU):
#   1. launch list of a short bench run (device time per launch, cold-cache, serialised)
#   2. `ncu --set full` captures of the routing kernel (DeepSeek-V3 shape), the K3
#      grouped GEMM (gate_up of the bottleneck rank), the fused gating kernel, the
#      dispatch layout kernel and the fused exchange kernel (world 1)
# Then, in the build container: python tools/summarize_profiles.py <round>
set -uo pipefail
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
NCU="ncu --clock-control none"

$NCU --metrics gpu__time_duration.sum -k regex:metro_ids_kernel -c 300 --csv --log-file "$OUT/launches.csv" \
    python bench.py --steps 256 --warmup 3 --e2e-steps 20 --cpu-seconds 0.2 --no-moe > "$OUT/launches_bench.log" 2>&1
$NCU --metrics gpu__time_duration.sum -c 400 --csv --log-file "$OUT/launches_all.csv" \
    python bench.py --steps 256 --warmup 3 --e2e-steps 20 --cpu-seconds 0.2 --no-moe > /dev/null 2>&1

full() {  # name, kernel regex, skip, command...
    local name=$1 kre=$2 skip=$3; shift 3
    $NCU --set full --import-source on -k "regex:$kre" -s "$skip" -c 1 -o "$OUT/${name}_full" "$@" \
        > "$OUT/${name}_full.log" 2>&1
}
full metro metro_ids_kernel 5 python tools/profile_target.py metro
full moe moe_gemm 0 python tools/k3_profile_target.py bf16 gate_up
full moe_fp8 moe_gemm 0 python tools/k3_profile_target.py fp8 gate_up
full moe_down moe_gemm 0 python tools/k3_profile_target.py bf16 down
full moe_fp8_down moe_gemm 0 python tools/k3_profile_target.py fp8 down
full gate metro_gate_topk_kernel 5 python tools/profile_target.py gate
# the gating routing kernel (a PDL dependent that stages the masks before its wait) faults
# under ncu's multi-pass KERNEL replay only (clean under compute-sanitizer memcheck /
# racecheck, and in single-pass captures): application replay for this one
$NCU --set full --import-source on --replay-mode application -k regex:metro_gate_route_kernel -s 5 -c 1 \
    -o "$OUT/gate_route_full" python tools/profile_target.py gate > "$OUT/gate_route_full.log" 2>&1
full dispatch layout_kernel 5 python tools/profile_target.py dispatch
full exchange metro_allgather_kernel 5 python tools/profile_target.py exchange
full fused metro_ids_kernel 5 python tools/profile_target.py fused
# the routing kernel with the caches NOT flushed between replays (steady state: the
# ids, masks and the kernel's own code stay in L2) beside the default cold capture
$NCU --set full --import-source on --cache-control none -k regex:metro_ids_kernel -s 5 -c 1 \
    -o "$OUT/metro_cc_none_full" python tools/profile_target.py metro > "$OUT/metro_cc_none_full.log" 2>&1
ls -la "$OUT"
