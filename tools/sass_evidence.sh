#!/usr/bin/env bash
# Per-kernel counts of the SASS opcodes that prove the sm_100a features each kernel
# uses (run in the build container on the built library; cuobjdump needs no GPU):
#   UTCHMMA / UTCQMMA  tcgen05.mma (kind::f16 / kind::f8f6f4)   LDTM   tcgen05.ld (TMEM -> registers)
#   UTMALDG            TMA tensor load (cp.async.bulk.tensor)    UBLKCP TMA bulk copy (cp.async.bulk)
#   SYNCS              mbarrier ops                               CREDUX redux.sync (warp min/max)
#   ATOMS              shared-memory atomics                      MATCH  match.any
# Usage: tools/sass_evidence.sh [lib] > profiles/<round>_sass_evidence.txt
LIB=${1:-paper_2512_09277_b200/_lib/libmetro_b200.so}
echo "# cuobjdump -sass $LIB: opcode counts per kernel (static instructions)"
echo "# arch: $(cuobjdump -lelf "$LIB" | head -3 | tr '\n' ' ')"
cuobjdump -sass "$LIB" | awk '
  /Function :/ { if (name != "") report(); name = $3; delete c; next }
  { for (i = 1; i <= NF; i++) { op = $i; sub(/\..*/, "", op);
      if (op ~ /^(UTCHMMA|UTCQMMA|UTCBAR|LDTM|UTMALDG|UTMASTG|UBLKCP|SYNCS|CREDUX|ATOMS|MATCH|UTCATOMSWS)$/) { c[op]++; break } } }
  function report(  s, k) { s = ""; for (k in c) s = s sprintf(" %s=%d", k, c[k]); printf "%-90s%s\n", substr(name, 1, 90), s }
  END { if (name != "") report() }' | c++filt | sort
