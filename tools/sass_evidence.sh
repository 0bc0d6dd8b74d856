#!/bin/bash
# SASS evidence for the claims in DESIGN.md (run here; no GPU needed):
# TMA (UTMALDG / UBLKCP) in the Gram-Schmidt kernels, packed fp32x2 in K1's
# row walk, LDS.64 + FFMA in K2's pixel-angle loop, no tensor-core MMA.
SO=paper_2602_17892_b200/libctk.so
cuobjdump -sass $SO > /tmp/all.sass
echo "# cuobjdump -sass $SO  ($(date -u +%F))"
for f in k_gs_stream k_gs_smem k_forward k_back; do
  echo "## $f: instruction mnemonics of interest (counts over all instantiations)"
  awk -v f="$f" '/Function : /{on = index($0, f) > 0} on' /tmp/all.sass \
    | grep -oE "UTMALDG[.0-9A-Z]*|UBLKCP[.0-9A-Z]*|FFMA2|FADD2|LDS\.64|LDG\.E[.0-9A-Z]*|UTC[A-Z]*MMA|HMMA|F2F\.F64\.F32|DFMA|BAR\.SYNC[.A-Z]*|SYNCS\.[A-Z.0-9]*" \
    | sort | uniq -c | sort -rn
done
