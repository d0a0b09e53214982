# A/B of the fused route + layout kernel's phases (METRO_DBG_SKIP bit mask, tuning only)
for v in ${SKIPS:-0 2 8 16 32 64 96 126}; do echo "skip=$v"; METRO_DBG_SKIP=$v python tools/fused_layout_bench.py --out gpurun_out/fl_$v.json 2>&1 | grep -E "^(q30|ds |ds_b64|ds_b8192)"; done
