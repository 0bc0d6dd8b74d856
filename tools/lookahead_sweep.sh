#!/bin/bash
# stream-A idle vs Arnoldi look-ahead (CTK_LOOKAHEAD), c2 and c1
for la in 3 6 12 24; do
  for w in c2 c1; do
    echo "la=$la $w $(CTK_LOOKAHEAD=$la CTK_TRACE=1 python tools/one_solve.py $w 4 2>&1 | grep 'ctk trace' | tail -1)"
  done
done
