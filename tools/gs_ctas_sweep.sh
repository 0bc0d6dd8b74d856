#!/bin/bash
# K3 (SMEM Gram-Schmidt) event time vs CTA count (CTK_GS_CTAS) at c1/c2 Krylov lengths
for G in 148 112 96 74 64 48; do
  echo "G=$G"; CTK_GS_CTAS=$G python tools/bench_cgs2.py 32940 65536 2>&1 | grep -v "^$"
done
