#!/bin/bash
# C4 host-buffer call (packed ops) vs the block slots the gated E1 launch
# leaves to the region kernels (DFX_GATE_FREE)
for g in "$@"; do
  echo "DFX_GATE_FREE=$g"
  DFX_GATE_FREE=$g python scripts/diag_c4_e2e.py 2>&1 | grep "packed host-buffer call" | tail -2
done
