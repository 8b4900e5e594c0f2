#!/bin/bash
# A/B kernel-(a) variants on C3 (one process per env setting)
python -m pytest tests/test_mfp_gpu.py -x -q -m gpu 2>&1 | tail -1
DFX_TAIL=20 python -m pytest tests/test_mfp_gpu.py -x -q -m gpu 2>&1 | tail -1
for t in 0 10 20 35; do for d in 2 4; do echo "tail $t div $d"; DFX_TAIL=$t DFX_TAILDIV=$d python scripts/tune_c3.py 32; done; done
