#!/usr/bin/env bash
# A/B of the K3 launch grid, interleaved, FP8 and bf16 (bottleneck rank FFN, METRO vs EPLB):
#   MOE_BALANCED_GRID=0  one persistent CTA per SM
#   MOE_BALANCED_GRID=1  (default) the fewest CTAs that keep the minimal number of item waves
# (An L2 prefetch of the next item's whole weight block by the producer was measured
# with this script too and rejected: FP8 down +15 %, bf16 +13 %.)
for round in 1 2; do
  for v in "MOE_BALANCED_GRID=0" "MOE_BALANCED_GRID=1"; do
    for dt in fp8 bf16; do
      env $v python tools/moe_layer_bench.py --dtype $dt --batches 2 --reps 5 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $dt r$round', 'metro %.1f us %.3f' % (d['metro']['ffn_us'], d['metro']['frac']), 'eplb %.1f us %.3f' % (d['eplb']['ffn_us'], d['eplb']['frac']), 'speedup %.3f' % d['ffn_speedup_metro_vs_eplb'])"
    done
  done
done
