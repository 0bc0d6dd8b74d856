#!/bin/bash
CTK_NVCC_EXTRA="-DCTK_GS_PROF" python -m paper_2602_17892_b200.build --force 2>&1 | grep -i error
GS_KS=10,40,79 timeout 300 python tools/gs_gram_phase_prof.py 65536 2>&1 | tail -12
