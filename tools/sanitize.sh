#!/usr/bin/env bash
# compute-sanitizer over the kernels (run on the GPU box); one summary line per run
# into $1 (default gpurun_out/sanitizer.txt).  Summarise with: cat the file.
OUT=${1:-gpurun_out/sanitizer.txt}
: > "$OUT"
run() {  # label, tool, command...
  local label=$1 tool=$2; shift 2
  local res
  res=$(timeout 600 compute-sanitizer --tool "$tool" "$@" 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY" | tail -1)
  printf '%-10s %-58s %s\n' "$tool" "$label" "$res" >> "$OUT"
}
run "metro_ids_kernel (profile_target.py metro 256)" memcheck python tools/profile_target.py metro 256
run "metro_ids_kernel" racecheck python tools/profile_target.py metro 256
run "metro_ids_kernel" synccheck python tools/profile_target.py metro 256
run "metro_ids_kernel, Qwen3-30B shape (q30 256: single r=2 steps)" memcheck python tools/profile_target.py q30 256
run "metro_ids_kernel, Qwen3-30B shape (q30 256)" racecheck python tools/profile_target.py q30 256
run "metro_ids_kernel, Qwen3-30B shape (q30 256)" synccheck python tools/profile_target.py q30 256
run "eplb_ids_kernel (profile_target.py eplb 256)" racecheck python tools/profile_target.py eplb 256
run "layout_kernel (profile_target.py dispatch 256)" racecheck python tools/profile_target.py dispatch 256
run "layout_kernel" memcheck python tools/profile_target.py dispatch 256
run "fused METRO + layout (profile_target.py fused 1024)" racecheck python tools/profile_target.py fused 1024
run "fused METRO + layout" memcheck python tools/profile_target.py fused 1024
run "large tables N>512 x 65 ranks, R=8 (regress 8)" racecheck python tools/profile_target.py regress 8
run "large tables N>512 x 65 ranks, R=1 (regress 1)" racecheck python tools/profile_target.py regress 1
run "large tables N>512 x 65 ranks, R=8 (regress 8)" memcheck python tools/profile_target.py regress 8
run "gating, cluster variant (gate 256)" racecheck python tools/profile_target.py gate 256
run "gating, top-k grid + routing CTAs (gate 1024)" racecheck python tools/profile_target.py gate 1024
run "gating, top-k grid + routing CTAs (gate 1024)" memcheck python tools/profile_target.py gate 1024
run "metro_allgather_kernel, world 1 (exchange 256)" racecheck python tools/profile_target.py exchange 256
run "whole rank MoE layer, bf16 (rank_layer_target.py bf16)" memcheck python tools/rank_layer_target.py bf16
run "whole rank MoE layer, FP8 (rank_layer_target.py fp8)" memcheck python tools/rank_layer_target.py fp8
run "moe_gemm_kernel FP8 down (k3_profile_target.py fp8 down)" racecheck python tools/k3_profile_target.py fp8 down
cat "$OUT"
