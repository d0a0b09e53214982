#!/usr/bin/env bash
# A/B of the K3 launch grid (MOE_BALANCED_GRID=0: one CTA per SM; 1: the fewest CTAs
# that keep the minimal number of item waves), interleaved, bf16 and FP8.
for round in 1 2; do
  for b in 0 1; do
    for dt in fp8 bf16; do
      MOE_BALANCED_GRID=$b python tools/moe_layer_bench.py --dtype $dt --batches 2 --reps 5 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('balanced=$b $dt round $round', 'metro %.1f us %.3f' % (d['metro']['ffn_us'], d['metro']['frac']), 'eplb %.1f us %.3f' % (d['eplb']['ffn_us'], d['eplb']['frac']), 'speedup %.3f' % d['ffn_speedup_metro_vs_eplb'])"
    done
  done
done
for b in 0 1; do MOE_BALANCED_GRID=$b python tools/k3_tail_probe.py fp8 down | tail -2 | sed "s/^/balanced=$b /"; done
